import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10548_b200 import _lib
from paper_2411_10548_b200._lib import ESM_BF16

def run(B, nh, S, dh, lens):
    torch.manual_seed(3)
    st = torch.cuda.current_stream().cuda_stream
    am = torch.zeros(B, S, dtype=torch.int32, device="cuda")
    for i, n in enumerate(lens): am[i, :n] = 1
    q = (torch.randn(B, nh, S, dh, device="cuda") * 0.5).bfloat16()
    k = (torch.randn(B, nh, S, dh, device="cuda") * 0.5).bfloat16()
    v = torch.randn(B, nh, S, dh, device="cuda").bfloat16()
    o = torch.empty(B * S, nh * dh, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, nh, S, device="cuda")
    _lib.call("esm_attn_fwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), o.data_ptr(), lse.data_ptr(), B, nh, S, dh, st)
    qr, kr, vr = (t.float().requires_grad_(True) for t in (q, k, v))
    s = qr @ kr.transpose(-1, -2) + torch.where(am[:, None, None, :] > 0, 0.0, float("-inf"))
    ref = (torch.softmax(s, -1) @ vr).permute(0, 2, 1, 3).reshape(B * S, nh * dh)
    do = torch.randn(B * S, nh * dh, device="cuda").bfloat16()
    ref.backward(do.float())
    dq = torch.empty(B, nh, S, dh, device="cuda"); dk = torch.empty_like(q); dv = torch.empty_like(q)
    delta = torch.empty(2, B, nh, S, device="cuda")
    _lib.call("esm_attn_bwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), do.data_ptr(), lse.data_ptr(), am.data_ptr(), delta.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), B, nh, S, dh, st)
    torch.cuda.synchronize()
    print(f"B={B} nh={nh} S={S} dh={dh} lens={lens}")
    for name, got, want in (("dv", dv, vr.grad), ("dk", dk, kr.grad), ("dq", dq, qr.grad)):
        for b in range(B):
            for kb in range(0, S, 64):
                g = got[b, :, kb:kb + 64].float(); w = want[b, :, kb:kb + 64]
                err = ((g - w).abs().max() / (w.abs().max() + 1e-9)).item()
                if err > 0.03: print(f"  {name} b={b} rows[{kb},{kb+64}) err={err:.3f} gotmax={g.abs().max().item():.3f} wantmax={w.abs().max().item():.3f}")
    print("  done")

run(1, 1, 200, 16, [200])
run(1, 1, 256, 16, [256])
run(1, 1, 256, 64, [256])
run(2, 1, 256, 64, [256, 100])
