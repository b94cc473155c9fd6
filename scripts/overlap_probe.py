"""Do a compute-bound tcgen05 GEMM and the HBM-bound AdamW kernel overlap on two streams?"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10548_b200 import _lib  # noqa: E402
from paper_2411_10548_b200._lib import EPI_STORE, ESM_BF16  # noqa: E402

M = N = K = 8192
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
n = 400_000_000  # 400 M params of AdamW state (~12 GB traffic)
p, g, m, v = (torch.zeros(n, device="cuda") for _ in range(4))
p16 = torch.zeros(n, device="cuda", dtype=torch.bfloat16)
dec = torch.ones(n // 256, device="cuda", dtype=torch.uint8)
hyper = torch.tensor([1e-3, 0.9, 0.98, 1e-8, 0.01, 1.0, 1.0, 0.0], device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def gemm(st, reps=12):
    for _ in range(reps):
        _lib.gemm_call(st.cuda_stream, dtype=ESM_BF16, M=M, N=N, K=K, A=A.data_ptr(), lda=K, a_mn_major=0,
                       B=B.data_ptr(), ldb=K, b_mn_major=0, C=C.data_ptr(), ldc=N, epilogue=EPI_STORE)


def adamw(st):
    _lib.call("esm_adamw", p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p16.data_ptr(), dec.data_ptr(), n,
              hyper.data_ptr(), st.cuda_stream)


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for _ in range(2):
    gemm(s1, 2)
    adamw(s2)
tg = timed(lambda: gemm(s1))
ta = timed(lambda: adamw(s2))
tb = timed(lambda: (gemm(s1), adamw(s2)))
print(f"gemm alone {tg:.2f} ms, adamw alone {ta:.2f} ms, both on two streams {tb:.2f} ms "
      f"(serial {tg + ta:.2f}, perfect overlap {max(tg, ta):.2f})", flush=True)
