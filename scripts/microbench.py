"""Per-kernel microbenchmarks (CUDA events) on the ESM-2 shapes: attention fwd/bwd and GEMMs.

    python scripts/microbench.py attn [--legacy]
    python scripts/microbench.py gemm
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10548_b200 import _lib  # noqa: E402
from paper_2411_10548_b200._lib import (EPI_DGELU, EPI_F32_ACC, EPI_GELU, EPI_GELU_GRADAUX, EPI_RESID, EPI_STORE,  # noqa: E402
                                        ESM_BF16)


def timeit(fn, iters=10, warm=3, graph=True):
    """GPU time per call; launches are captured in a CUDA graph so host launch cost is excluded."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(iters):
                    fn()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        run = g.replay
    else:
        def run():
            for _ in range(iters):
                fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def cur():
    return torch.cuda.current_stream().cuda_stream


def attn():
    shapes = [(32, 20, 1024, 24), (16, 20, 1024, 64), (8, 20, 512, 16), (4, 40, 1024, 64)]
    if len(sys.argv) > 2:
        shapes = [tuple(int(x) for x in sys.argv[2].split(","))]
    for (B, nh, S, dh) in shapes:
        q = (torch.randn(B, nh, S, dh, device="cuda") * 0.5).bfloat16()
        k = (torch.randn(B, nh, S, dh, device="cuda") * 0.5).bfloat16()
        v = torch.randn(B, nh, S, dh, device="cuda").bfloat16()
        am = torch.ones(B, S, dtype=torch.int32, device="cuda")
        o = torch.empty(B * S, nh * dh, device="cuda", dtype=torch.bfloat16)
        lse = torch.empty(B, nh, S, device="cuda")
        do = torch.randn_like(o)
        dq = torch.empty(B, nh, S, dh, device="cuda")
        dk, dv = torch.empty_like(q), torch.empty_like(q)
        delta = torch.empty(2, B, nh, S, device="cuda")
        sched = torch.zeros(_lib.attn_sched_words(B), dtype=torch.int32, device="cuda")
        _lib.call("esm_attn_prepare", am.data_ptr(), sched.data_ptr(), B, S, cur())
        sp = sched.data_ptr()
        f = lambda: _lib.call("esm_attn_fwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), am.data_ptr(), sp,  # noqa
                              o.data_ptr(), lse.data_ptr(), B, nh, S, dh, cur())
        g = lambda: _lib.call("esm_attn_bwd", ESM_BF16, q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),  # noqa
                              do.data_ptr(), lse.data_ptr(), am.data_ptr(), sp, delta.data_ptr(), dq.data_ptr(),
                              dk.data_ptr(), dv.data_ptr(), B, nh, S, dh, cur())
        from paper_2411_10548_b200.model import rope_tables
        cos, sin = (torch.from_numpy(t).cuda() for t in rope_tables(S, dh))
        ws = torch.empty(B * S, nh * dh, device="cuda")
        dqkv = torch.empty(B * S, 3 * nh * dh, device="cuda", dtype=torch.bfloat16)
        cs = torch.zeros(3 * nh * dh, device="cuda")
        fz = lambda: _lib.call("esm_attn_bwd_qkv", q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),  # noqa
                               do.data_ptr(), lse.data_ptr(), am.data_ptr(), sp, delta.data_ptr(), ws.data_ptr(),
                               dqkv.data_ptr(), cs.data_ptr(), cos.data_ptr(), sin.data_ptr(), dh ** -0.5, B, nh, S,
                               dh, cur())
        ng = os.environ.get("MB_NOGRAPH") is None
        tf, tb, tz = timeit(f, graph=ng), timeit(g, graph=ng), timeit(fz, graph=ng)
        fl = 4.0 * B * nh * S * S * dh
        print(f"attn B={B} nh={nh} S={S} dh={dh}: fwd {tf:.3f} ms ({fl / tf / 1e9:.0f} TF/s)  "
              f"bwd {tb:.3f} ms ({2.0 * fl / tb / 1e9:.0f} TF/s)  fused-bwd(dqkv) {tz:.3f} ms", flush=True)


def gemm():
    T = 32768
    for (name, M, N, K, amn, bmn, epi) in [
        ("35M qkv fwd", T, 1440, 480, 0, 0, EPI_STORE), ("35M fc1 fwd", T, 1920, 480, 0, 0, EPI_GELU),
        ("35M fc1 fwd gradaux", T, 1920, 480, 0, 0, EPI_GELU_GRADAUX), ("35M fc2 dgradDGELU", T, 1920, 480, 0, 1, EPI_DGELU),
        ("35M fc2 fwd", T, 480, 1920, 0, 0, EPI_RESID), ("35M fc2 dgrad", T, 1920, 480, 0, 1, EPI_STORE),
        ("35M fc1 dgrad", T, 480, 1920, 0, 1, EPI_STORE), ("35M fc1 wgrad", 1920, 480, T, 1, 1, EPI_F32_ACC),
        ("35M fc2 wgrad", 480, 1920, T, 1, 1, EPI_F32_ACC),
        ("650M fc1 fwd", 16384, 5120, 1280, 0, 0, EPI_GELU),
        ("650M fc1 fwd gradaux", 16384, 5120, 1280, 0, 0, EPI_GELU_GRADAUX), ("650M fc2 fwd", 16384, 1280, 5120, 0, 0, EPI_RESID),
        ("650M fc2 dgrad", 16384, 5120, 1280, 0, 1, EPI_STORE), ("650M fc1 wgrad", 5120, 1280, 16384, 1, 1, EPI_F32_ACC),
        ("650M qkv fwd", 16384, 3840, 1280, 0, 0, EPI_STORE), ("650M out fwd", 16384, 1280, 1280, 0, 0, EPI_RESID),
        ("650M fc2 dgradDGELU", 16384, 5120, 1280, 0, 1, EPI_DGELU), ("650M fc1 dgrad", 16384, 1280, 5120, 0, 1, EPI_STORE),
        ("650M qkv dgrad", 16384, 1280, 3840, 0, 1, EPI_STORE), ("650M qkv wgrad", 3840, 1280, 16384, 1, 1, EPI_F32_ACC),
        ("650M out wgrad", 1280, 1280, 16384, 1, 1, EPI_F32_ACC), ("650M fc2 wgrad", 1280, 5120, 16384, 1, 1, EPI_F32_ACC),
        ("3B fc1 fwd", 8192, 10240, 2560, 0, 0, EPI_GELU), ("3B fc2 fwd", 8192, 2560, 10240, 0, 0, EPI_RESID),
        ("3B fc2 dgradDGELU", 8192, 10240, 2560, 0, 1, EPI_DGELU), ("3B fc1 dgrad", 8192, 2560, 10240, 0, 1, EPI_STORE),
        ("3B qkv dgrad", 8192, 2560, 7680, 0, 1, EPI_STORE), ("3B out fwd", 8192, 2560, 2560, 0, 0, EPI_RESID),
        ("3B fc1 wgrad", 10240, 2560, 8192, 1, 1, EPI_F32_ACC), ("3B fc2 wgrad", 2560, 10240, 8192, 1, 1, EPI_F32_ACC),
        ("8192^3 store", 8192, 8192, 8192, 0, 0, EPI_STORE), ("4096^3 store", 4096, 4096, 4096, 0, 0, EPI_STORE),
        ("16384x8192x4096 store", 16384, 8192, 4096, 0, 0, EPI_STORE)]:
        if len(sys.argv) > 2 and sys.argv[2] not in name:
            continue
        A = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
        Bm = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
        if epi == EPI_F32_ACC:
            C = torch.zeros(M, N, device="cuda")
        else:
            C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        aux = torch.empty(M, N, device="cuda", dtype=torch.bfloat16) if epi in (EPI_GELU, EPI_GELU_GRADAUX, EPI_RESID, EPI_DGELU) else None
        bias = torch.zeros(N, device="cuda")
        csum = torch.zeros(N, device="cuda") if epi == EPI_DGELU else None
        kw = dict(dtype=ESM_BF16, M=M, N=N, K=K, A=A.data_ptr(), lda=M if amn else K, a_mn_major=amn,
                  B=Bm.data_ptr(), ldb=N if bmn else K, b_mn_major=bmn, C=C.data_ptr(), ldc=N, epilogue=epi,
                  bias=bias.data_ptr() if epi not in (EPI_F32_ACC, EPI_DGELU) else None,
                  aux_in=aux.data_ptr() if epi in (EPI_RESID, EPI_DGELU) else None, ld_aux_in=N,
                  col_sum=csum.data_ptr() if csum is not None else None,
                  aux_out=aux.data_ptr() if epi in (EPI_GELU, EPI_GELU_GRADAUX) else None, ld_aux_out=N)
        t = timeit(lambda: _lib.gemm_call(cur(), **kw), graph=os.environ.get("MB_NOGRAPH") is None)
        print(f"gemm {name:16s} M={M} N={N} K={K}: {t:.3f} ms  {2.0 * M * N * K / t / 1e9:.0f} TF/s", flush=True)


def ln():
    """LayerNorm fwd / bwd (no dgamma/dbeta: fused into the dgrad GEMM; with residual add) achieved GB/s."""
    for T, H in [(32768, 480), (32768, 768), (16384, 1280), (4096, 2560)]:
        x = torch.randn(T, H, device="cuda").bfloat16()
        y, dy, dres, dx = (torch.randn(T, H, device="cuda").bfloat16() for _ in range(4))
        g, b = torch.ones(H, device="cuda"), torch.zeros(H, device="cuda")
        mu, rs = torch.empty(T, device="cuda"), torch.empty(T, device="cuda")
        f = lambda: _lib.call("esm_layernorm_fwd", ESM_BF16, x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(),  # noqa
                              mu.data_ptr(), rs.data_ptr(), T, H, 1e-5, cur())
        bw = lambda: _lib.call("esm_layernorm_bwd", ESM_BF16, dy.data_ptr(), x.data_ptr(), g.data_ptr(), mu.data_ptr(),  # noqa
                               rs.data_ptr(), dres.data_ptr(), None, dx.data_ptr(), None, None, None, T, H, None, None, cur())
        tf, tb = timeit(f, iters=20), timeit(bw, iters=20)
        bf, bb = T * H * 4 + T * 8, T * H * 8 + T * 8
        print(f"layernorm T={T} H={H}: fwd {tf * 1e3:.1f} us ({bf / tf / 1e6:.0f} GB/s)  "
              f"bwd {tb * 1e3:.1f} us ({bb / tb / 1e6:.0f} GB/s)", flush=True)


def xent():
    """ESM LM head (V = 33): fused decoder + masked CE + dlogits + dn over labelled rows, and dE."""
    T, H, V = 32768, 480, 33
    n = torch.randn(T, H, device="cuda").bfloat16()
    E = (torch.randn(V, H, device="cuda") * 0.02).bfloat16()
    bias = torch.zeros(V, device="cuda")
    lab = torch.where(torch.rand(T, device="cuda") < 0.15, torch.randint(4, 24, (T,), device="cuda"),
                      torch.full((T,), -100, device="cuda")).int()
    inv = torch.tensor([1.0 / max(1, int((lab >= 0).sum()))], device="cuda")
    loss = torch.zeros(1, device="cuda")
    dlog = torch.empty(T, V, device="cuda")
    dn = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    dE, db = torch.zeros(V, H, device="cuda"), torch.zeros(V, device="cuda")
    f = lambda: _lib.call("esm_lmhead_xent", ESM_BF16, n.data_ptr(), E.data_ptr(), bias.data_ptr(), lab.data_ptr(),  # noqa
                          inv.data_ptr(), loss.data_ptr(), dlog.data_ptr(), dn.data_ptr(), dE.data_ptr(), db.data_ptr(),
                          T, H, V, cur())
    t = timeit(f, iters=20)
    print(f"lmhead_xent T={T} H={H} V={V}: {t * 1e3:.1f} us", flush=True)


def rank():
    """Geneformer tokeniser: device esm_rank_encode rows/s vs the CPU oracle restatement (single thread,
    the reference's algorithm: SURVEY.md §8a1' quotes 3.7k rows/s for the reference itself)."""
    import time
    import numpy as np
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import rank_oracle as R
    from paper_2411_10548_b200.data import RankEncoder, gene_medians, synthetic_expression_csr
    n_genes, B, S = 25424, 256, 2048
    ip, c, v = synthetic_expression_csr(B, n_genes, seed=0, nnz=(500, 4000))
    med = gene_medians(ip, c, v, n_genes)
    enc = RankEncoder(med)
    (d_ip, d_c, d_v), mx = enc.stage(ip, c, v, np.arange(B))
    ids = torch.empty(B, S, dtype=torch.int32, device="cuda")
    am = torch.empty_like(ids)
    t = timeit(lambda: enc.encode_device(d_ip, d_c, d_v, B, mx, S, ids=ids, am=am, stream=cur()))
    want, _ = R.rank_encode_batch(ip, c, v, med, range(B), S, S)
    assert np.array_equal(ids.cpu().numpy(), want)
    t0 = time.perf_counter()
    for r in range(64):
        R.rank_encode(c[ip[r]:ip[r + 1]], v[ip[r]:ip[r + 1]], med, S)
    cpu = 64 / (time.perf_counter() - t0)
    nnz = (ip[-1]) / B
    print(f"rank_encode {B} rows (mean nnz {nnz:.0f}) -> [{B},{S}]: {t:.3f} ms = {B / t * 1e3:,.0f} rows/s on the GPU; "
          f"CPU oracle single thread {cpu:,.0f} rows/s; bit-exact", flush=True)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "attn"
    {"attn": attn, "gemm": gemm, "rank": rank, "ln": ln, "xent": xent}[what]()
