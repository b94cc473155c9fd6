"""Attention-probability dropout (HF EsmSelfAttention: dropout(softmax(S)) @ V, HF:modeling_esm.py:257-282) in the
tcgen05 attention kernels (esm_attn_*_dropout): kernel level against fp32 torch autograd with the oracle's keep
masks (oracle/esm2_oracle.py:attention_dropout_keep), model level against the fp64 oracle."""
import ctypes
import math
import os

import numpy as np
import pytest
import torch

import esm2_oracle as O
from paper_2411_10548_b200 import EsmConfig, _lib
from paper_2411_10548_b200._lib import ESM_BF16, ESM_F32
from paper_2411_10548_b200.model import ATTN_DROP_SITE, EsmForMaskedLM, init_params

pytestmark = pytest.mark.gpu
DEV = "cuda"
# bf16 gates as tests/test_gpu_model.py (relative Frobenius error of each gradient vs the fp64 oracle)
BF16_GRAD_FRO, BF16_KEY_BIAS_FRO = 0.03, 0.08


def st():
    return torch.cuda.current_stream().cuda_stream


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / (b.abs().max() + 1e-12)).item()


def seed_tensor(seed):
    return torch.tensor([seed - (1 << 64) if seed >= (1 << 63) else seed], dtype=torch.int64, device=DEV)


def prepare(am, B, S):
    sched = torch.full((_lib.attn_sched_words(B),), -7, dtype=torch.int32, device=DEV)
    _lib.call("esm_attn_prepare", am.data_ptr(), sched.data_ptr(), B, S, st())
    return sched


@pytest.mark.parametrize("dh", [16, 24, 32, 64])
@pytest.mark.parametrize("S,lens", [(256, [256, 190]), (1024, [1024, 601])])
def test_attention_dropout_fwd_bwd(dh, S, lens):
    torch.manual_seed(11)
    B, nh, p, layer = len(lens), 3, 0.1, 5
    seed = 0x123456789ABCDEF1
    am = torch.zeros(B, S, dtype=torch.int32, device=DEV)
    for i, n in enumerate(lens):
        am[i, :n] = 1
    q = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).bfloat16()
    k = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).bfloat16()
    v = torch.randn(B, nh, S, dh, device=DEV).bfloat16()
    seed_t = seed_tensor(seed)
    d = _lib.Dropout(seed_t.data_ptr(), ATTN_DROP_SITE + layer, O.dropout_threshold(p), 1.0 / (1.0 - p))
    o = torch.empty(B * S, nh * dh, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(B, nh, S, device=DEV)
    sched = prepare(am, B, S)
    _lib.call("esm_attn_fwd_dropout", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(),
              sched.data_ptr(), o.data_ptr(), lse.data_ptr(), B, nh, S, dh, ctypes.byref(d), st())
    keep = torch.from_numpy(O.attention_dropout_keep(seed, layer, B, nh, S, p)).to(DEV)
    assert abs(keep.float().mean().item() - (1 - p)) < 0.01
    z = keep.float() / (1.0 - p)
    qr, kr, vr = (t.float().requires_grad_(True) for t in (q, k, v))
    s = qr @ kr.transpose(-1, -2) + torch.where(am[:, None, None, :] > 0, 0.0, float("-inf"))
    ref = (torch.softmax(s, -1) * z) @ vr
    ref_o = ref.permute(0, 2, 1, 3).reshape(B * S, nh * dh)
    torch.cuda.synchronize()
    e_o = rel(o, ref_o)
    # the normaliser keeps every probability: the LSE is the no-dropout one
    e_l = rel(-lse * math.log(2.0), torch.logsumexp(s.detach(), -1))
    do = torch.randn(B * S, nh * dh, device=DEV).bfloat16()
    ref_o.backward(do.float())
    dq = torch.empty(B, nh, S, dh, device=DEV)
    dk = torch.empty(B, nh, S, dh, device=DEV, dtype=torch.bfloat16)
    dv = torch.empty_like(dk)
    delta = torch.empty(2, B, nh, S, device=DEV)
    _lib.call("esm_attn_bwd_dropout", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
              do.data_ptr(), lse.data_ptr(), am.data_ptr(), sched.data_ptr(), delta.data_ptr(), dq.data_ptr(),
              dk.data_ptr(), dv.data_ptr(), B, nh, S, dh, ctypes.byref(d), st())
    torch.cuda.synchronize()
    errs = dict(o=e_o, lse=e_l, dq=rel(dq, qr.grad), dk=rel(dk, kr.grad), dv=rel(dv, vr.grad))
    print(f"attention dropout dh={dh} S={S}:", {k_: "%.1e" % e for k_, e in errs.items()})
    assert e_o < 2e-2 and e_l < 1e-3
    assert errs["dq"] < 3e-2 and errs["dk"] < 3e-2 and errs["dv"] < 3e-2, errs
    # p = 0 (threshold 0) is the plain kernel, bit for bit
    d0 = _lib.Dropout(seed_t.data_ptr(), ATTN_DROP_SITE + layer, 0, 1.0)
    o0, o1 = torch.empty_like(o), torch.empty_like(o)
    _lib.call("esm_attn_fwd_dropout", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(),
              sched.data_ptr(), o0.data_ptr(), lse.data_ptr(), B, nh, S, dh, ctypes.byref(d0), st())
    _lib.call("esm_attn_fwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), sched.data_ptr(),
              o1.data_ptr(), lse.data_ptr(), B, nh, S, dh, st())
    torch.cuda.synchronize()
    assert torch.equal(o0, o1)


def test_attention_dropout_fp32_kernels():
    """The fp32 parity kernels apply the same masks: vs torch fp64 autograd at 1e-5."""
    torch.manual_seed(12)
    B, nh, S, dh, p, layer = 2, 2, 192, 32, 0.2, 1
    seed = 0x0F1E2D3C4B5A6978
    am = torch.ones(B, S, dtype=torch.int32, device=DEV)
    am[1, 150:] = 0
    q, k, v = (torch.randn(B, nh, S, dh, device=DEV) * 0.5 for _ in range(3))
    seed_t = seed_tensor(seed)
    d = _lib.Dropout(seed_t.data_ptr(), ATTN_DROP_SITE + layer, O.dropout_threshold(p), 1.0 / (1.0 - p))
    o = torch.empty(B * S, nh * dh, device=DEV)
    lse = torch.empty(B, nh, S, device=DEV)
    _lib.call("esm_attn_fwd_dropout", ESM_F32, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), None,
              o.data_ptr(), lse.data_ptr(), B, nh, S, dh, ctypes.byref(d), st())
    z = torch.from_numpy(O.attention_dropout_keep(seed, layer, B, nh, S, p)).to(DEV).double() / (1.0 - p)
    qr, kr, vr = (t.double().requires_grad_(True) for t in (q, k, v))
    s = qr @ kr.transpose(-1, -2) + torch.where(am[:, None, None, :] > 0, 0.0, float("-inf")).double()
    ref_o = ((torch.softmax(s, -1) * z) @ vr).permute(0, 2, 1, 3).reshape(B * S, nh * dh)
    do = torch.randn(B * S, nh * dh, device=DEV)
    ref_o.backward(do.double())
    dq, dk, dv = (torch.empty(B, nh, S, dh, device=DEV) for _ in range(3))
    delta = torch.empty(2, B, nh, S, device=DEV)
    _lib.call("esm_attn_bwd_dropout", ESM_F32, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
              lse.data_ptr(), am.data_ptr(), None, delta.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), B,
              nh, S, dh, ctypes.byref(d), st())
    torch.cuda.synchronize()
    errs = dict(o=rel(o, ref_o), dq=rel(dq, qr.grad), dk=rel(dk, kr.grad), dv=rel(dv, vr.grad))
    print("attention dropout fp32 kernels:", {k_: "%.1e" % e for k_, e in errs.items()})
    assert max(errs.values()) < 1e-5, errs


def test_model_attention_dropout_fp32_matches_oracle():
    """fp32 parity mode with attention dropout 0.1 (+ hidden dropout 0.05): loss and every gradient within 1e-4
    of the fp64 oracle (the north-star bar for fp32 mode)."""
    H, nh, L, F, B, S = 320, 20, 2, 1280, 2, 128
    cfg = EsmConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=nh, intermediate_size=F,
                    attention_probs_dropout_prob=0.1, hidden_dropout_prob=0.05)
    ocfg = O.OracleConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=nh, intermediate_size=F)
    params = init_params(cfg, seed=22)
    ids, am = O.synthetic_batch(B, S, seed=7)
    am[0, 100:] = 0
    inp, lab = O.mlm_mask(ids, seed=8, stream=1)
    seed = 0x0123456789ABCDEF
    ref = O.forward_backward(ocfg, params, inp, am, lab, dtype=np.float64, attention_dropout=(seed, 0.1),
                             hidden_dropout=(seed, 0.05))
    m = EsmForMaskedLM(cfg, dtype="fp32", device="cuda", params=params)
    m.set_dropout_seed(seed)
    ws = m.set_batch(torch.from_numpy(inp).cuda(), torch.from_numpy(am).cuda(), torch.from_numpy(lab).cuda())
    loss = float(m.forward_backward(ws).item())
    g = m.grads()
    errs = {k: float(np.abs(g[k].cpu().numpy().astype(np.float64) - r).max() / (np.abs(r).max() + 1e-30))
            for k, r in ref.grads.items()}
    worst = max(errs, key=errs.get)
    print(f"attention dropout fp32 model: loss rel {abs(loss - ref.loss) / ref.loss:.2e}; worst grad {worst} "
          f"{errs[worst]:.2e}")
    assert abs(loss - ref.loss) / ref.loss < 1e-5
    assert errs[worst] < 1e-4, (worst, errs[worst])


@pytest.mark.parametrize("H,nh", [(128, 2), (480, 20), (256, 8), (320, 20)])  # head dims 64, 24, 32, 16
def test_model_attention_dropout_matches_oracle(H, nh):
    """bf16 model step with attention-probability dropout p = 0.1 (and hidden dropout 0.05) vs the fp64 oracle
    with the same counter-based masks; the fused (dqkv) and classic attention backwards agree."""
    L, F, B, S = 2, 4 * H, 2, 128
    cfg = EsmConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=nh, intermediate_size=F,
                    attention_probs_dropout_prob=0.1, hidden_dropout_prob=0.05)
    ocfg = O.OracleConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=nh, intermediate_size=F)
    params = init_params(cfg, seed=21)
    ids, am = O.synthetic_batch(B, S, seed=5)
    am[1, 90:] = 0
    inp, lab = O.mlm_mask(ids, seed=6, stream=3)
    seed = 0xBADC0FFEE0DDF00D
    ref = O.forward_backward(ocfg, params, inp, am, lab, dtype=np.float64, attention_dropout=(seed, 0.1),
                             hidden_dropout=(seed, 0.05))
    ref0 = O.forward_backward(ocfg, params, inp, am, lab, dtype=np.float64, want_grads=False,
                              hidden_dropout=(seed, 0.05))
    assert abs(ref.loss - ref0.loss) > 1e-4 * ref0.loss  # the attention masks change the loss

    def run():
        m = EsmForMaskedLM(cfg, dtype="bf16", device="cuda", params=params)
        m.set_dropout_seed(seed)
        ws = m.set_batch(torch.from_numpy(inp).cuda(), torch.from_numpy(am).cuda(), torch.from_numpy(lab).cuda())
        loss = float(m.forward_backward(ws).item())
        return loss, {k: g.cpu().numpy().astype(np.float64) for k, g in m.grads().items()}

    old = os.environ.get("ESM_ATTN_FUSED")
    try:
        os.environ["ESM_ATTN_FUSED"] = "1"
        loss, g = run()
        os.environ["ESM_ATTN_FUSED"] = "0"
        loss_c, g_c = run()
    finally:
        if old is None:
            os.environ.pop("ESM_ATTN_FUSED", None)
        else:
            os.environ["ESM_ATTN_FUSED"] = old
    gate = lambda k: BF16_KEY_BIAS_FRO if k.endswith("attention.self.key.bias") else BF16_GRAD_FRO  # noqa: E731
    fro = {k: float(np.linalg.norm(g[k] - r) / (np.linalg.norm(r) + 1e-30)) for k, r in ref.grads.items()}
    worst = max(fro, key=lambda k: fro[k] / gate(k))
    fc = {k: float(np.linalg.norm(g_c[k] - g[k]) / (np.linalg.norm(g[k]) + 1e-30)) for k in g}
    worst_c = max(fc, key=fc.get)
    print(f"attention dropout model H={H} nh={nh}: loss rel {abs(loss - ref.loss) / ref.loss:.2e}; worst grad "
          f"{worst} {fro[worst]:.3e}; fused vs classic worst {worst_c} {fc[worst_c]:.2e}")
    assert abs(loss - ref.loss) / ref.loss < 1e-2
    assert fro[worst] < gate(worst), (worst, fro[worst])
    assert abs(loss_c - loss) < 1e-6 * abs(loss)  # same forward
    assert fc[worst_c] < 2e-2, (worst_c, fc[worst_c])


def test_graph_step_with_dropout_matches_eager():
    """Hidden + attention dropout under CUDA-graph replay: each replay reads that step's seed from device memory,
    so three graph steps reproduce three eager steps (same masks, same updates) and the masks change per step."""
    cfg = EsmConfig(hidden_size=320, num_hidden_layers=2, num_attention_heads=20, intermediate_size=1280,
                    attention_probs_dropout_prob=0.1, hidden_dropout_prob=0.1)
    params = init_params(cfg, seed=31)
    ids, am = O.synthetic_batch(4, 256, seed=9)
    am[2, 200:] = 0

    def run(graph):
        m = EsmForMaskedLM(cfg, dtype="bf16", device="cuda", params=params, seed=5)
        ws = m.workspace(4, 256)
        ws.ids.copy_(torch.from_numpy(ids))
        ws.am.copy_(torch.from_numpy(am))
        m.mlm_mask(ws.ids, seed=3, stream_id=1, ws=ws)
        if graph:
            m.capture(ws)
        losses = [float((m.graph_step() if graph else m.step(ws)).item()) for _ in range(3)]
        seeds = m.last_dropout_seed
        return losses, m.grads()["esm.encoder.layer.1.attention.self.query.weight"].float().cpu(), seeds

    le, ge, se = run(False)
    lg, gg, sg = run(True)
    print("dropout eager vs graph losses:", le, lg)
    assert se == sg
    assert len(set(round(x, 6) for x in le)) == 3  # per-step masks (and updates) differ
    for a, b in zip(le, lg):
        assert abs(a - b) < 1e-3 * abs(a), (le, lg)
    assert rel(gg, ge) < 2e-2
