"""Microbenchmark of esm_qkv_rope_bwd / esm_layernorm_bwd / esm_layernorm_fwd at the 650M shapes (CUDA events)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10548_b200 import _lib  # noqa: E402
from paper_2411_10548_b200._lib import ESM_BF16  # noqa: E402

B, S, nh, dh = 16, 1024, 20, 64
H, T = nh * dh, 16 * 1024
dq = torch.randn(B, nh, S, dh, device="cuda")
dk = torch.randn(B, nh, S, dh, device="cuda").bfloat16()
dv = torch.randn(B, nh, S, dh, device="cuda").bfloat16()
dqkv = torch.empty(T, 3 * H, device="cuda", dtype=torch.bfloat16)
cs = torch.rand(S, dh // 2, device="cuda")
sn = torch.rand(S, dh // 2, device="cuda")
csum = torch.zeros(3 * H, device="cuda")
st = torch.cuda.current_stream().cuda_stream


def rope():
    _lib.call("esm_qkv_rope_bwd", ESM_BF16, dq.data_ptr(), dk.data_ptr(), dv.data_ptr(), dqkv.data_ptr(),
              csum.data_ptr(), cs.data_ptr(), sn.data_ptr(), B, S, nh, dh, 0.125, st)


x = torch.randn(T, H, device="cuda").bfloat16()
dy = torch.randn(T, H, device="cuda").bfloat16()
dres = torch.randn(T, H, device="cuda").bfloat16()
dx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
g = torch.rand(H, device="cuda")
bta = torch.rand(H, device="cuda")
mean = torch.zeros(T, device="cuda")
rstd = torch.ones(T, device="cuda")
cs2 = torch.zeros(H, device="cuda")


def lnb():
    _lib.call("esm_layernorm_bwd", ESM_BF16, dy.data_ptr(), x.data_ptr(), g.data_ptr(), mean.data_ptr(),
              rstd.data_ptr(), dres.data_ptr(), None, dx.data_ptr(), None, None, cs2.data_ptr(), T, H, None, None, st)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "rope"):
    ms = t(rope)
    byts = dq.numel() * 4 + dk.numel() * 2 * 2 + dqkv.numel() * 2
    print(f"qkv_rope_bwd 650M: {ms * 1e3:.1f} us, {byts / ms / 1e6:.0f} GB/s", flush=True)
if which in ("all", "lnb"):
    ms = t(lnb)
    byts = 4 * T * H * 2
    print(f"layernorm_bwd 650M (dy, x, dres -> dx): {ms * 1e3:.1f} us, {byts / ms / 1e6:.0f} GB/s", flush=True)
if which in ("all", "lnf"):
    y = torch.empty_like(x)

    def lnf():
        _lib.call("esm_layernorm_fwd", ESM_BF16, x.data_ptr(), g.data_ptr(), bta.data_ptr(), y.data_ptr(),
                  mean.data_ptr(), rstd.data_ptr(), T, H, 1e-5, st)
    ms = t(lnf)
    print(f"layernorm_fwd 650M (x -> y): {ms * 1e3:.1f} us, {2 * T * H * 2 / ms / 1e6:.0f} GB/s", flush=True)
