"""Kernel-level parity on a B200: each C-ABI op against a plain fp32 PyTorch reference of the
same op (bf16 kernels within bf16 tolerance; fp32 SIMT kernels at 1e-5)."""
import ctypes
import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2411_10548_b200 import _lib  # noqa: E402
from paper_2411_10548_b200._lib import EPI_DELTA, EPI_GELU_GRADAUX, EPI_MUL_AUX  # noqa: E402
from paper_2411_10548_b200._lib import (EPI_DGELU, EPI_F32_ACC, EPI_GELU, EPI_QKV_ROPE, EPI_RESID, EPI_STORE,  # noqa: E402
                                        ESM_BF16, ESM_F32)

DEV = "cuda"


def st():
    return torch.cuda.current_stream().cuda_stream


def gelu(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


def gelu_grad(x):
    return 0.5 * (1.0 + torch.erf(x / math.sqrt(2.0))) + x * torch.exp(-0.5 * x * x) / math.sqrt(2 * math.pi)


def rel(a, b):
    a, b = a.float(), b.float()
    return ((a - b).abs().max() / (b.abs().max() + 1e-12)).item()


def run_gemm(dtype, M, N, K, A, lda, amn, B, ldb, bmn, C, ldc, epi, bias=None, aux_in=None, aux_out=None,
             col_sum=None, split_k=0):
    _lib.gemm_call(st(), dtype=dtype, M=M, N=N, K=K, A=A.data_ptr(), lda=lda, a_mn_major=amn, B=B.data_ptr(),
                   ldb=ldb, b_mn_major=bmn, C=C.data_ptr(), ldc=ldc, epilogue=epi,
                   bias=bias.data_ptr() if bias is not None else None,
                   aux_in=aux_in.data_ptr() if aux_in is not None else None, ld_aux_in=ldc,
                   aux_out=aux_out.data_ptr() if aux_out is not None else None, ld_aux_out=ldc,
                   col_sum=col_sum.data_ptr() if col_sum is not None else None, split_k=split_k)


FWD_SHAPES = [(256, 128, 64), (1000, 1440, 480), (300, 480, 1920), (128, 96, 64), (4096, 1920, 480),
              (515, 64, 200), (2048, 1280, 1280), (333, 160, 96),
              (2304 + 77, 480, 480), (4096, 1440, 480), (3000, 96, 64)]  # M >= 2048: CTA-pair (M=256) kernels


@pytest.mark.parametrize("M,N,K", FWD_SHAPES)
@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_gemm_forward_epilogues(M, N, K, dt):
    torch.manual_seed(0)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = ESM_BF16 if dt == "bf16" else ESM_F32
    tol = 2e-2 if dt == "bf16" else 1e-5
    X = torch.randn(M, K, device=DEV).to(tdt)
    W = (torch.randn(N, K, device=DEV) * 0.05).to(tdt)
    b = torch.randn(N, device=DEV)
    R = torch.randn(M, N, device=DEV).to(tdt)
    ref = X.float() @ W.float().t() + b
    C = torch.empty(M, N, device=DEV, dtype=tdt)
    run_gemm(kdt, M, N, K, X, K, 0, W, K, 0, C, N, EPI_STORE, bias=b)
    torch.cuda.synchronize()
    assert rel(C, ref) < tol
    Z = torch.empty_like(C)
    run_gemm(kdt, M, N, K, X, K, 0, W, K, 0, C, N, EPI_GELU, bias=b, aux_out=Z)
    torch.cuda.synchronize()
    assert rel(Z, ref) < tol and rel(C, gelu(ref)) < tol
    run_gemm(kdt, M, N, K, X, K, 0, W, K, 0, C, N, EPI_RESID, bias=b, aux_in=R)
    torch.cuda.synchronize()
    assert rel(C, ref + R.float()) < tol


def test_gemm_wide_tile_long_k():
    """4096^3 picks the 256 x 512 pair tile (two N = 256 MMAs per k-step, one TMEM accumulator; gemm.cu
    prefer_bn512) for both B layouts and the STORE / GELU / RESID / DGELU epilogues."""
    torch.manual_seed(4)
    M = N = K = 4096
    X = torch.randn(M, K, device=DEV).bfloat16()
    W = (torch.randn(N, K, device=DEV) * 0.05).bfloat16()
    b = torch.randn(N, device=DEV)
    R = torch.randn(M, N, device=DEV).bfloat16()
    ref = X.float() @ W.float().t() + b
    C = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    Z = torch.empty_like(C)
    run_gemm(ESM_BF16, M, N, K, X, K, 0, W, K, 0, C, N, EPI_GELU, bias=b, aux_out=Z)
    torch.cuda.synchronize()
    errs = [rel(Z, ref), rel(C, gelu(ref))]
    run_gemm(ESM_BF16, M, N, K, X, K, 0, W, K, 0, C, N, EPI_RESID, bias=b, aux_in=R)
    torch.cuda.synchronize()
    errs.append(rel(C, ref + R.float()))
    Wt = W.t().contiguous()  # [K, N]: N-major B
    ref2 = X.float() @ Wt.float()
    run_gemm(ESM_BF16, M, N, K, X, K, 0, Wt, N, 1, C, N, EPI_STORE)
    torch.cuda.synchronize()
    errs.append(rel(C, ref2))
    cs = torch.zeros(N, device=DEV)
    run_gemm(ESM_BF16, M, N, K, X, K, 0, Wt, N, 1, C, N, EPI_DGELU, aux_in=R, col_sum=cs)
    torch.cuda.synchronize()
    want = ref2 * gelu_grad(R.float())
    errs += [rel(C, want), rel(cs, want.sum(0))]
    print("wide-tile GEMM errors:", ["%.1e" % e for e in errs])
    assert max(errs) < 2e-2


@pytest.mark.parametrize("M,N,K", [(256, 128, 64), (1000, 480, 1440), (300, 1920, 480), (515, 64, 200),
                                   (2048, 1280, 5120), (2500, 480, 1920), (4096, 1920, 480), (2048, 128, 64)])
@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_gemm_dgrad(M, N, K, dt):
    """dX[M=T, N=in] = dY[T, K=out] · W[out, in]  (B operand N-major)."""
    torch.manual_seed(1)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = ESM_BF16 if dt == "bf16" else ESM_F32
    tol = 2e-2 if dt == "bf16" else 1e-5
    dY = torch.randn(M, K, device=DEV).to(tdt)
    W = (torch.randn(K, N, device=DEV) * 0.05).to(tdt)
    Z = torch.randn(M, N, device=DEV).to(tdt)
    ref = dY.float() @ W.float()
    C = torch.empty(M, N, device=DEV, dtype=tdt)
    run_gemm(kdt, M, N, K, dY, K, 0, W, N, 1, C, N, EPI_STORE)
    torch.cuda.synchronize()
    assert rel(C, ref) < tol
    cs = torch.zeros(N, device=DEV)
    run_gemm(kdt, M, N, K, dY, K, 0, W, N, 1, C, N, EPI_DGELU, aux_in=Z, col_sum=cs)
    torch.cuda.synchronize()
    want = ref * gelu_grad(Z.float())
    assert rel(C, want) < tol
    assert rel(cs, want.sum(0)) < (2e-2 if dt == "bf16" else 1e-4)


@pytest.mark.parametrize("B,S,nh,dh", [(2, 256, 20, 24), (16, 256, 20, 64), (3, 100, 4, 16), (2, 512, 12, 64),
                                        (4, 96, 10, 32), (1, 2048, 40, 64)])
def test_gemm_delta_epilogue(B, S, nh, dh):
    """Out-projection dgrad with Delta: dO = dY · W stored bf16, and row_dot[b, h, s] = sum over head h of
    bf16(dO) * O (the attention backward's rowsum(dO o O)), heads straddling 32-column chunks (dh 24) and
    spanning several (dh 64), rows of several sequences, M >= 2048 (CTA-pair kernels) and ragged M."""
    torch.manual_seed(4)
    H = nh * dh
    M = B * S
    dY = torch.randn(M, H, device=DEV).bfloat16()
    W = (torch.randn(H, H, device=DEV) * 0.05).bfloat16()
    O = torch.randn(M, H, device=DEV).bfloat16()
    C = torch.empty(M, H, device=DEV, dtype=torch.bfloat16)
    delta = torch.full((B, nh, S), 7.0, device=DEV)  # the callee zeroes it
    _lib.gemm_call(st(), dtype=ESM_BF16, M=M, N=H, K=H, A=dY.data_ptr(), lda=H, a_mn_major=0, B=W.data_ptr(), ldb=H,
                   b_mn_major=1, C=C.data_ptr(), ldc=H, epilogue=EPI_DELTA, aux_in=O.data_ptr(), ld_aux_in=H,
                   row_dot=delta.data_ptr(), seq_len=S, n_heads=nh, head_dim=dh)
    torch.cuda.synchronize()
    ref = dY.float() @ W.float()
    assert rel(C, ref) < 2e-2
    want = (C.float() * O.float()).view(B, S, nh, dh).sum(-1).permute(0, 2, 1)
    err = ((delta - want).abs().max() / want.abs().max()).item()
    print(f"Delta epilogue B={B} S={S} nh={nh} dh={dh}: max rel err {err:.2e}")
    assert err < 1e-5


@pytest.mark.parametrize("M,N,K", [(480, 1920, 4096), (1440, 480, 8192), (128, 128, 64), (96, 200, 1000),
                                   (1280, 5120, 2048), (40, 64, 512), (2560, 640, 4096), (5120, 1280, 2048)])
@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_gemm_wgrad(M, N, K, dt):
    """dW[M=out, N=in] += dY[T=K, out]ᵀ · X[T, in]  (both operands MN-major, fp32 accumulate, split-K)."""
    torch.manual_seed(2)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = ESM_BF16 if dt == "bf16" else ESM_F32
    dY = torch.randn(K, M, device=DEV).to(tdt)
    X = torch.randn(K, N, device=DEV).to(tdt)
    ref = dY.float().t() @ X.float()
    C = torch.ones(M, N, device=DEV)
    run_gemm(kdt, M, N, K, dY, M, 1, X, N, 1, C, N, EPI_F32_ACC)
    torch.cuda.synchronize()
    assert rel(C - 1.0, ref) < (1e-2 if dt == "bf16" else 1e-5)


@pytest.mark.parametrize("M,N,K", [(256, 128, 64), (1000, 1920, 480), (4096, 1920, 480), (2500, 5120, 1280)])
def test_gemm_gelu_gradaux_and_mul_aux(M, N, K):
    """bf16 FFN pair: forward GELU_GRADAUX stores GELU(Z) and GELU'(Z); the FC2 dgrad MUL_AUX multiplies by
    the stored derivative and sums the FC1 bias gradient."""
    torch.manual_seed(3)
    X = torch.randn(M, K, device=DEV).bfloat16()
    W = (torch.randn(N, K, device=DEV) * 0.05).bfloat16()
    b = torch.randn(N, device=DEV)
    z = X.float() @ W.float().t() + b
    C, G = torch.empty(M, N, device=DEV, dtype=torch.bfloat16), torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    run_gemm(ESM_BF16, M, N, K, X, K, 0, W, K, 0, C, N, EPI_GELU_GRADAUX, bias=b, aux_out=G)
    torch.cuda.synchronize()
    assert rel(C, gelu(z)) < 2e-2 and rel(G, gelu_grad(z)) < 2e-2
    Kb = 384
    dY = torch.randn(M, Kb, device=DEV).bfloat16()
    W2 = (torch.randn(Kb, N, device=DEV) * 0.05).bfloat16()
    cs = torch.zeros(N, device=DEV)
    D = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    run_gemm(ESM_BF16, M, N, Kb, dY, Kb, 0, W2, N, 1, D, N, EPI_MUL_AUX, aux_in=G, col_sum=cs)
    torch.cuda.synchronize()
    want = (dY.float() @ W2.float()) * G.float()
    assert rel(D, want) < 2e-2 and rel(cs, want.sum(0)) < 2e-2
    with pytest.raises(_lib.EsmKernelError):  # bf16-only epilogues
        run_gemm(ESM_F32, M, N, K, X.float(), K, 0, W.float(), K, 0, C.float(), N, EPI_GELU_GRADAUX, bias=b,
                 aux_out=G.float())


def test_gemm_rejects_bad_args():
    X = torch.randn(64, 64, device=DEV).to(torch.bfloat16)
    C = torch.empty(64, 64, device=DEV).to(torch.bfloat16)
    with pytest.raises(_lib.EsmKernelError):
        run_gemm(ESM_BF16, 64, 64, 64, X, 64, 0, X, 64, 0, C, 64, EPI_RESID)  # RESID without aux_in


def prepare(am, B, S):
    """Attention scheduling workspace for this key mask (esm_attn_prepare)."""
    sched = torch.full((_lib.attn_sched_words(B),), -7, dtype=torch.int32, device=DEV)
    _lib.call("esm_attn_prepare", am.data_ptr(), sched.data_ptr(), B, S, st())
    return sched


def torch_attention(q, k, v, am):
    s = q.float() @ k.float().transpose(-1, -2)
    s = s + torch.where(am[:, None, None, :] > 0, 0.0, float("-inf"))
    p = torch.softmax(s, -1)
    return p @ v.float()


@pytest.mark.parametrize("dh", [16, 24, 32, 64])
@pytest.mark.parametrize("S,lens", [(128, [128, 100]), (200, [200, 77]), (1024, [1024, 1000])])
@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_attention_fwd_bwd(dh, S, lens, dt):
    torch.manual_seed(3)
    B, nh = len(lens), 3
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = ESM_BF16 if dt == "bf16" else ESM_F32
    am = torch.zeros(B, S, dtype=torch.int32, device=DEV)
    for i, n in enumerate(lens):
        am[i, :n] = 1
    q = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).to(tdt)
    k = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).to(tdt)
    v = torch.randn(B, nh, S, dh, device=DEV).to(tdt)
    o = torch.empty(B * S, nh * dh, device=DEV, dtype=tdt)
    lse = torch.empty(B, nh, S, device=DEV)
    sched = prepare(am, B, S)
    _lib.call("esm_attn_fwd", kdt, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), sched.data_ptr(),
              o.data_ptr(), lse.data_ptr(), B, nh, S, dh, st())
    qr, kr, vr = (t.float().requires_grad_(True) for t in (q, k, v))
    ref = torch_attention(qr, kr, vr, am)
    ref_o = ref.permute(0, 2, 1, 3).reshape(B * S, nh * dh)
    torch.cuda.synchronize()
    tol = 2e-2 if dt == "bf16" else 1e-5
    assert rel(o, ref_o) < tol
    s = qr.detach() @ kr.detach().transpose(-1, -2)
    s = s + torch.where(am[:, None, None, :] > 0, 0.0, float("-inf"))
    assert rel(-lse * math.log(2.0), torch.logsumexp(s, -1)) < (1e-3 if dt == "bf16" else 1e-6)  # ABI: -LSE log2 e
    do = torch.randn(B * S, nh * dh, device=DEV).to(tdt)
    ref_o.backward(do.float())
    dq = torch.empty(B, nh, S, dh, device=DEV)
    dk = torch.empty(B, nh, S, dh, device=DEV, dtype=tdt)
    dv = torch.empty_like(dk)
    delta = torch.empty(2, B, nh, S, device=DEV)
    _lib.call("esm_attn_bwd", kdt, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
              lse.data_ptr(), am.data_ptr(), sched.data_ptr(), delta.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), B, nh,
              S, dh, st())
    torch.cuda.synchronize()
    tol = 3e-2 if dt == "bf16" else 1e-4
    assert rel(dv, vr.grad) < tol
    assert rel(dk, kr.grad) < tol
    assert rel(dq, qr.grad) < tol
    if dt == "bf16":  # o = NULL: Delta precomputed by the caller (the model's ESM_EPI_DELTA path)
        delta2 = torch.zeros(2, B, nh, S, device=DEV)
        delta2[0] = (do.float() * o.float()).view(B, S, nh, dh).sum(-1).permute(0, 2, 1)
        dq2, dk2, dv2 = torch.empty_like(dq), torch.empty_like(dk), torch.empty_like(dv)
        _lib.call("esm_attn_bwd", kdt, q.data_ptr(), k.data_ptr(), v.data_ptr(), None, do.data_ptr(),
                  lse.data_ptr(), am.data_ptr(), sched.data_ptr(), delta2.data_ptr(), dq2.data_ptr(), dk2.data_ptr(),
                  dv2.data_ptr(), B, nh, S, dh, st())
        torch.cuda.synchronize()
        assert rel(dv2, dv) < 1e-6 and rel(dk2, dk) < 1e-2 and rel(dq2, dq) < 1e-2


def _attn_case(B, nh, S, dh, lens, seed, holes=None):
    torch.manual_seed(seed)
    am = torch.zeros(B, S, dtype=torch.int32, device=DEV)
    for i, n in enumerate(lens):
        am[i, :n] = 1
    if holes is not None:
        am[holes[0], holes[1]:holes[2]] = 0
    q = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).bfloat16()
    k = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).bfloat16()
    v = torch.randn(B, nh, S, dh, device=DEV).bfloat16()
    return am, q, k, v


def _attn_fwd(q, k, v, am, sched, stream=None):
    B, nh, S, dh = q.shape
    o = torch.empty(B * S, nh * dh, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(B, nh, S, device=DEV)
    s_ = stream.cuda_stream if stream is not None else st()
    _lib.call("esm_attn_fwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), sched.data_ptr(),
              o.data_ptr(), lse.data_ptr(), B, nh, S, dh, s_)
    return o, lse


@pytest.mark.parametrize("lens", [[2048, 2048], [2048, 1500, 611, 97]])
def test_attention_geneformer_s2048(lens):
    """BASELINE configs[4] attention geometry: S = 2048, nh = 12, dh = 64 (Geneformer, max_len 2048 of the
    reference tokenizer, pkg/src/densefeed/tokenizer.py:68-83), full and ragged rank-token rows; forward and
    backward vs torch fp32 (bf16 inputs), achieved errors reported."""
    B, nh, S, dh = len(lens), 12, 2048, 64
    am, q, k, v = _attn_case(B, nh, S, dh, lens, seed=21)
    sched = prepare(am, B, S)
    o, lse = _attn_fwd(q, k, v, am, sched)
    for _ in range(3):  # deterministic: no reduction order depends on scheduling in the forward
        o2, lse2 = _attn_fwd(q, k, v, am, sched)
        assert torch.equal(o2, o) and torch.equal(lse2, lse)
    qr, kr, vr = (t.float().requires_grad_(True) for t in (q, k, v))
    ref_o = torch_attention(qr, kr, vr, am).permute(0, 2, 1, 3).reshape(B * S, nh * dh)
    keep = am.reshape(-1).bool()
    e_o = rel(o[keep], ref_o[keep])
    do = torch.randn(B * S, nh * dh, device=DEV).bfloat16()
    do[~keep] = 0
    ref_o.backward(do.float())
    dq = torch.empty(B, nh, S, dh, device=DEV)
    dk = torch.empty(B, nh, S, dh, device=DEV, dtype=torch.bfloat16)
    dv = torch.empty_like(dk)
    delta = torch.empty(2, B, nh, S, device=DEV)
    _lib.call("esm_attn_bwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
              lse.data_ptr(), am.data_ptr(), sched.data_ptr(), delta.data_ptr(), dq.data_ptr(), dk.data_ptr(),
              dv.data_ptr(), B, nh, S, dh, st())
    torch.cuda.synchronize()
    e = {"o": e_o, "dq": rel(dq, qr.grad), "dk": rel(dk, kr.grad), "dv": rel(dv, vr.grad)}
    print("S=2048 attention rel. errors", {k_: round(float(v_), 5) for k_, v_ in e.items()})
    assert e["o"] < 1e-2 and e["dq"] < 3e-2 and e["dk"] < 2e-2 and e["dv"] < 2e-2, e
    assert (sched[:4] == 0).all()  # persistent-kernel counters left at zero for the next layer


def test_attention_concurrent_streams_private_workspaces():
    """Two attention forwards with different key masks running concurrently on two streams of one GPU, each
    with its own scheduling workspace (no global mutable state), equal the same calls run one after another."""
    B, nh, S, dh = 4, 20, 1024, 64
    am1, q, k, v = _attn_case(B, nh, S, dh, [1024, 800, 512, 64], seed=31)
    am2 = torch.ones_like(am1)
    am2[:, 700:] = 0
    am2[2, 10:90] = 0
    ref1, _ = _attn_fwd(q, k, v, am1, prepare(am1, B, S))
    ref2, _ = _attn_fwd(q, k, v, am2, prepare(am2, B, S))
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for rep in range(3):
        sc1, sc2 = prepare(am1, B, S), prepare(am2, B, S)
        torch.cuda.synchronize()
        o1, _ = _attn_fwd(q, k, v, am1, sc1, stream=s1)
        o2, _ = _attn_fwd(q, k, v, am2, sc2, stream=s2)
        torch.cuda.synchronize()
        outs.append((o1, o2))
    for o1, o2 in outs:
        assert torch.equal(o1, ref1) and torch.equal(o2, ref2)


def test_attention_bf16_rejects_unpadded_seq():
    B, nh, S, dh = 1, 2, 30, 16
    am, q, k, v = _attn_case(B, nh, S, dh, [30], seed=1)
    sched = prepare(am, B, S)
    with pytest.raises(_lib.EsmKernelError, match="S % 4"):
        _attn_fwd(q, k, v, am, sched)


@pytest.mark.parametrize("H", [64, 320, 480, 1280, 2560])
@pytest.mark.parametrize("dt", ["bf16", "fp32"])
def test_layernorm(H, dt):
    torch.manual_seed(4)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = ESM_BF16 if dt == "bf16" else ESM_F32
    rows = 777
    x = (torch.randn(rows, H, device=DEV) * 2 + 0.5).to(tdt)
    g = torch.randn(H, device=DEV)
    b = torch.randn(H, device=DEV)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=DEV)
    rstd = torch.empty(rows, device=DEV)
    _lib.call("esm_layernorm_fwd", kdt, x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
              rstd.data_ptr(), rows, H, 1e-5, st())
    xr = x.float().requires_grad_(True)
    gr, br = g.clone().requires_grad_(True), b.clone().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xr, (H,), gr, br, 1e-5)
    torch.cuda.synchronize()
    tol = 1e-2 if dt == "bf16" else 1e-5
    assert rel(y, ref) < tol
    dy = torch.randn(rows, H, device=DEV).to(tdt)
    dres = torch.randn(rows, H, device=DEV).to(tdt)
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    dg = torch.zeros(H, device=DEV)
    db = torch.zeros(H, device=DEV)
    cs = torch.zeros(H, device=DEV)
    _lib.call("esm_layernorm_bwd", kdt, dy.data_ptr(), x.data_ptr(), g.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
              dres.data_ptr(), None, dx.data_ptr(), dg.data_ptr(), db.data_ptr(), cs.data_ptr(), rows, H, None, None,
              st())
    torch.cuda.synchronize()
    want = xr.grad + dres.float()
    assert rel(dx, want) < (2e-2 if dt == "bf16" else 1e-5)
    assert rel(dg, gr.grad) < (1e-2 if dt == "bf16" else 1e-5)
    assert rel(db, br.grad) < 1e-5
    assert rel(cs, want.sum(0)) < (1e-2 if dt == "bf16" else 1e-4)


def test_mlm_mask_bitexact_vs_oracle():
    import esm2_oracle as O
    ids, _ = O.synthetic_batch(8, 1000, seed=3)
    ids[1, 500:] = O.PAD
    for seed, stream in [(0, 0), (7, 12345), (2 ** 40 + 3, 2 ** 63 + 5)]:
        want_inp, want_lab = O.mlm_mask(ids, seed, stream)
        d_ids = torch.from_numpy(ids).to(DEV)
        inp = torch.empty_like(d_ids)
        lab = torch.empty_like(d_ids)
        n = torch.zeros(1, dtype=torch.int32, device=DEV)
        _lib.call("esm_mlm_mask", d_ids.data_ptr(), inp.data_ptr(), lab.data_ptr(), n.data_ptr(), ids.size, seed,
                  stream, st())
        torch.cuda.synchronize()
        assert (inp.cpu().numpy() == want_inp).all()
        assert (lab.cpu().numpy() == want_lab).all()
        assert int(n.item()) == int((want_lab != -100).sum())


def test_adamw_matches_oracle():
    import esm2_oracle as O
    rng = np.random.default_rng(0)
    n = 4096
    p = rng.standard_normal(n).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    decay = np.array([1] * 8 + [0] * 8, dtype=np.uint8)
    P = {"w": p[:2048].copy(), "b.bias": p[2048:].copy()}
    G = {"w": g[:2048], "b.bias": g[2048:]}
    M = {k: np.zeros_like(v) for k, v in P.items()}
    Vv = {k: np.zeros_like(v) for k, v in P.items()}
    dp = torch.from_numpy(p).to(DEV)
    dg = torch.from_numpy(g).to(DEV)
    dm = torch.zeros(n, device=DEV)
    dv = torch.zeros(n, device=DEV)
    p16 = torch.empty(n, device=DEV, dtype=torch.bfloat16)
    dd = torch.from_numpy(decay).to(DEV)
    for step in range(1, 4):
        O.adamw_update(P, G, M, Vv, step, 1e-3, beta1=0.9, beta2=0.98, eps=1e-8, weight_decay=0.1)
        hyper = torch.tensor([1e-3, 0.9, 0.98, 1e-8, 0.1, float(step), 1.0, 0.0], device=DEV)
        _lib.call("esm_adamw", dp.data_ptr(), dg.data_ptr(), dm.data_ptr(), dv.data_ptr(), p16.data_ptr(),
                  dd.data_ptr(), n, hyper.data_ptr(), st())
    torch.cuda.synchronize()
    want = np.concatenate([P["w"], P["b.bias"]])
    np.testing.assert_allclose(dp.cpu().numpy(), want, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(p16.float().cpu().numpy(), want, rtol=1e-2, atol=1e-3)


@pytest.mark.parametrize("B,S,nh,dh", [(2, 128, 20, 24), (3, 100, 20, 16), (2, 64, 20, 64), (1, 96, 4, 32)])
def test_gemm_qkv_rope_epilogue(B, S, nh, dh):
    """Fused QKV GEMM epilogue (bias, q-scale, RoPE, head scatter) == GEMM + esm_qkv_rope_fwd."""
    from paper_2411_10548_b200.model import rope_tables
    torch.manual_seed(5)
    H = nh * dh
    T = B * S
    X = torch.randn(T, H, device=DEV).bfloat16()
    W = (torch.randn(3 * H, H, device=DEV) * 0.05).bfloat16()
    b = torch.randn(3 * H, device=DEV)
    cos, sin = (torch.from_numpy(t).to(DEV) for t in rope_tables(S, dh))
    qs = dh ** -0.5
    q, k, v = (torch.empty(B, nh, S, dh, device=DEV, dtype=torch.bfloat16) for _ in range(3))
    _lib.gemm_call(st(), dtype=ESM_BF16, M=T, N=3 * H, K=H, A=X.data_ptr(), lda=H, a_mn_major=0, B=W.data_ptr(),
                   ldb=H, b_mn_major=0, C=None, ldc=0, epilogue=EPI_QKV_ROPE, bias=b.data_ptr(),
                   rope_cos=cos.data_ptr(), rope_sin=sin.data_ptr(), q_out=q.data_ptr(), k_out=k.data_ptr(),
                   v_out=v.data_ptr(), seq_len=S, n_heads=nh, head_dim=dh, q_scale=qs)
    qkv = (X.float() @ W.float().t() + b).view(B, S, 3, nh, dh).permute(2, 0, 3, 1, 4)
    half = dh // 2
    c = torch.cat([cos, cos], -1)[None, None]
    s_ = torch.cat([sin, sin], -1)[None, None]

    def rope(x):
        return x * c + torch.cat([-x[..., half:], x[..., :half]], -1) * s_
    torch.cuda.synchronize()
    assert rel(q, rope(qkv[0] * qs)) < 2e-2
    assert rel(k, rope(qkv[1])) < 2e-2
    assert rel(v, qkv[2]) < 2e-2


@pytest.mark.parametrize("B,S,nh,dh,lens", [(2, 256, 3, 24, [256, 130]), (2, 192, 2, 64, [192, 64]),
                                            (1, 128, 4, 16, [128]), (2, 100, 2, 32, [100, 37]),
                                            (3, 1024, 4, 64, [1024, 0, 300]), (4, 512, 20, 24, [512, 511, 129, 1])])
def test_attention_bwd_qkv_fused(B, S, nh, dh, lens):
    """esm_attn_bwd_qkv (dqkv with RoPE^T + bias grads) == esm_attn_bwd + esm_qkv_rope_bwd; includes a batch row
    without any valid key and rows whose valid length ends inside a key block."""
    from paper_2411_10548_b200.model import rope_tables
    torch.manual_seed(6)
    H = nh * dh
    am = torch.zeros(B, S, dtype=torch.int32, device=DEV)
    for i, n in enumerate(lens):
        am[i, :n] = 1
    q, k, v = ((torch.randn(B, nh, S, dh, device=DEV) * 0.5).bfloat16() for _ in range(3))
    o = torch.empty(B * S, H, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(B, nh, S, device=DEV)
    sched = prepare(am, B, S)
    _lib.call("esm_attn_fwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), sched.data_ptr(),
              o.data_ptr(), lse.data_ptr(), B, nh, S, dh, st())
    do = torch.randn(B * S, H, device=DEV).bfloat16()
    cos, sin = (torch.from_numpy(t).to(DEV) for t in rope_tables(S, dh))
    qs = dh ** -0.5
    delta = torch.empty(2, B, nh, S, device=DEV)
    dq = torch.empty(B, nh, S, dh, device=DEV)
    dk, dv = torch.empty_like(q), torch.empty_like(q)
    _lib.call("esm_attn_bwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
              lse.data_ptr(), am.data_ptr(), sched.data_ptr(), delta.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), B, nh, S,
              dh, st())
    ref = torch.empty(B * S, 3 * H, device=DEV, dtype=torch.bfloat16)
    ref_cs = torch.zeros(3 * H, device=DEV)
    _lib.call("esm_qkv_rope_bwd", ESM_BF16, dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), ref.data_ptr(),
              ref_cs.data_ptr(), cos.data_ptr(), sin.data_ptr(), B, S, nh, dh, qs, st())
    got = torch.empty_like(ref)
    cs = torch.zeros(3 * H, device=DEV)
    ws = torch.empty(B * S, H, device=DEV)
    _lib.call("esm_attn_bwd_qkv", q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
              lse.data_ptr(), am.data_ptr(), sched.data_ptr(), delta.data_ptr(), ws.data_ptr(), got.data_ptr(), cs.data_ptr(),
              cos.data_ptr(), sin.data_ptr(), qs, B, nh, S, dh, st())
    torch.cuda.synchronize()
    assert rel(got, ref) < 2e-2
    assert rel(cs, ref_cs) < 2e-2


@pytest.mark.parametrize("dh", [24, 64])
@pytest.mark.parametrize("holes", [False, True])
def test_attention_persistent_many_tiles(dh, holes):
    """More work than CTAs (320 backward tiles / forward items on 148 SMs): dynamic tile claiming, global barrier
    phases across tiles, padded key blocks skipped (row 1 has 724 padding keys) and a non-prefix mask."""
    torch.manual_seed(11)
    B, nh, S = 2, 20, 1024
    am = torch.ones(B, S, dtype=torch.int32, device=DEV)
    am[1, 300:] = 0
    if holes:
        am[0, 100:180] = 0  # non-prefix: masked keys inside the row
    q = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).bfloat16()
    k = (torch.randn(B, nh, S, dh, device=DEV) * 0.5).bfloat16()
    v = torch.randn(B, nh, S, dh, device=DEV).bfloat16()
    o = torch.empty(B * S, nh * dh, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(B, nh, S, device=DEV)
    sched = prepare(am, B, S)
    _lib.call("esm_attn_fwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), sched.data_ptr(),
              o.data_ptr(), lse.data_ptr(), B, nh, S, dh, st())
    qr, kr, vr = (t.float().requires_grad_(True) for t in (q, k, v))
    ref = torch_attention(qr, kr, vr, am)
    ref_o = ref.permute(0, 2, 1, 3).reshape(B * S, nh * dh)
    torch.cuda.synchronize()
    assert rel(o, ref_o) < 2e-2
    do = torch.randn(B * S, nh * dh, device=DEV).bfloat16()
    ref_o.backward(do.float())
    dq = torch.empty(B, nh, S, dh, device=DEV)
    dk = torch.full((B, nh, S, dh), float("nan"), device=DEV, dtype=torch.bfloat16)  # skipped tiles must be zeroed
    dv = torch.full_like(dk, float("nan"))
    delta = torch.empty(2, B, nh, S, device=DEV)
    _lib.call("esm_attn_bwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(),
              lse.data_ptr(), am.data_ptr(), sched.data_ptr(), delta.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), B, nh,
              S, dh, st())
    torch.cuda.synchronize()
    assert not torch.isnan(dk).any() and not torch.isnan(dv).any()
    assert rel(dv, vr.grad) < 3e-2 and rel(dk, kr.grad) < 3e-2 and rel(dq, qr.grad) < 3e-2
    assert (dk[1, :, 300:] == 0).all() and (dv[1, :, 300:] == 0).all()


@pytest.mark.parametrize("H", [64, 320, 480, 768, 1280, 2560])
@pytest.mark.parametrize("rows", [1, 777, 4096 + 3])
@pytest.mark.parametrize("gelu", [False, True])
def test_layernorm_bwd_no_stats(H, rows, gelu):
    """The dgamma/dbeta-free backward (two rows per group iteration for H <= 512 in bf16), with the residual
    gradient, the optional GELU' multiply and the column sum; odd row counts exercise the tail row."""
    torch.manual_seed(5)
    x = (torch.randn(rows, H, device=DEV) * 2 + 0.5).bfloat16()
    g = torch.randn(H, device=DEV)
    b = torch.randn(H, device=DEV)
    y = torch.empty_like(x)
    mean = torch.empty(rows, device=DEV)
    rstd = torch.empty(rows, device=DEV)
    _lib.call("esm_layernorm_fwd", ESM_BF16, x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
              rstd.data_ptr(), rows, H, 1e-5, st())
    xr = x.float().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xr, (H,), g, b, 1e-5)
    torch.cuda.synchronize()
    assert rel(y, ref) < 1e-2
    dy = torch.randn(rows, H, device=DEV).bfloat16()
    dres = torch.randn(rows, H, device=DEV).bfloat16()
    z = torch.randn(rows, H, device=DEV).bfloat16() if gelu else None
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    cs = torch.zeros(H, device=DEV)
    _lib.call("esm_layernorm_bwd", ESM_BF16, dy.data_ptr(), x.data_ptr(), g.data_ptr(), mean.data_ptr(),
              rstd.data_ptr(), dres.data_ptr(), z.data_ptr() if gelu else None, dx.data_ptr(), None, None,
              cs.data_ptr(), rows, H, None, None, st())
    torch.cuda.synchronize()
    want = xr.grad + dres.float()
    if gelu:
        zf = z.float().requires_grad_(True)
        torch.nn.functional.gelu(zf).backward(torch.ones_like(zf))
        want = want * zf.grad
    assert rel(dx, want) < 2e-2
    assert rel(cs, want.sum(0)) < 1e-2


@pytest.mark.parametrize("B,S,nh,dh", [(1, 64, 20, 64), (2, 256, 20, 64), (2, 96, 20, 24), (3, 40, 4, 16),
                                       (1, 128, 40, 64), (2, 64, 8, 32)])
def test_qkv_rope_bwd_vs_torch(B, S, nh, dh):
    """esm_qkv_rope_bwd (RoPE^T + q-scale + head-major -> token-major dqkv + q/k/v bias gradients) vs torch fp32,
    at the 650M / 3B / 35M / 8M head geometries (vector and generic kernels)."""
    from paper_2411_10548_b200.model import rope_tables
    torch.manual_seed(9)
    H = nh * dh
    dq = torch.randn(B, nh, S, dh, device=DEV)
    dk = torch.randn(B, nh, S, dh, device=DEV).bfloat16()
    dv = torch.randn(B, nh, S, dh, device=DEV).bfloat16()
    cos, sin = (torch.from_numpy(t).to(DEV) for t in rope_tables(S, dh))
    qs = dh ** -0.5
    out = torch.empty(B * S, 3 * H, device=DEV, dtype=torch.bfloat16)
    cs = torch.zeros(3 * H, device=DEV)
    _lib.call("esm_qkv_rope_bwd", ESM_BF16, dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), out.data_ptr(),
              cs.data_ptr(), cos.data_ptr(), sin.data_ptr(), B, S, nh, dh, qs, st())
    c = torch.cat([cos, cos], -1)[None, None]
    s_ = torch.cat([sin, sin], -1)[None, None]

    def rope_t(y):
        ys = y * s_
        h = dh // 2
        return y * c + torch.cat([ys[..., h:], -ys[..., :h]], -1)

    def tok(x):
        return x.permute(0, 2, 1, 3).reshape(B * S, H)

    ref = torch.cat([tok(rope_t(dq) * qs), tok(rope_t(dk.float())), tok(dv.float())], -1)
    torch.cuda.synchronize()
    assert rel(out, ref) < 1e-2
    assert rel(cs, ref.sum(0)) < 1e-3


@pytest.mark.parametrize("H", [320, 480, 1280, 2560])
def test_layernorm_bulk_ring_wraps(H):
    """Bulk-staged LayerNorm (bf16): many row blocks per persistent CTA (the stage ring wraps several times, a
    ragged last block), forward and backward (with residual input and bias-gradient column sums) vs torch fp32."""
    torch.manual_seed(5)
    rows = 20011
    x = (torch.randn(rows, H, device=DEV) * 1.5 + 0.3).bfloat16()
    g, b = torch.randn(H, device=DEV), torch.randn(H, device=DEV)
    y = torch.empty_like(x)
    mean, rstd = torch.empty(rows, device=DEV), torch.empty(rows, device=DEV)
    _lib.call("esm_layernorm_fwd", ESM_BF16, x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(),
              mean.data_ptr(), rstd.data_ptr(), rows, H, 1e-5, st())
    xr = x.float().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xr, (H,), g, b, 1e-5)
    torch.cuda.synchronize()
    assert rel(y, ref) < 1e-2
    assert rel(mean, xr.detach().mean(-1)) < 1e-4
    dy = torch.randn(rows, H, device=DEV).bfloat16()
    dres = torch.randn(rows, H, device=DEV).bfloat16()
    ref.backward(dy.float())
    dx = torch.empty_like(x)
    cs = torch.zeros(H, device=DEV)
    _lib.call("esm_layernorm_bwd", ESM_BF16, dy.data_ptr(), x.data_ptr(), g.data_ptr(), mean.data_ptr(),
              rstd.data_ptr(), dres.data_ptr(), None, dx.data_ptr(), None, None, cs.data_ptr(), rows, H, None, None,
              st())
    torch.cuda.synchronize()
    want = xr.grad + dres.float()
    assert rel(dx, want) < 2e-2
    assert rel(cs, want.sum(0)) < 1e-2
