#!/usr/bin/env python
"""ESM-2 MLM training throughput on B200 (BASELINE.json metric: "ESM-2 MLM train tokens/sec at
1/2/4/8 B200; MFU vs bf16 tensor peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 650m|35m|3b|geneformer|8m] [--batch B] [--seq S]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference      # HF EsmForMaskedLM (eager fp32) train step on the host cores

A "step" = device MLM masking + forward + backward + AdamW (+ NCCL gradient buckets for N>1)
over one batch of synthetic full-length protein sequences (random-init weights).
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {  # BASELINE.json configs -> (preset, batch per GPU, seq)
    "35m": ("esm2_t12_35M", 32, 1024),    # configs[1]: 35M, 32 x 1024, bf16, 1 B200
    "650m": ("esm2_t33_650M", 16, 1024),  # configs[2]: 650M DDP, seq 1024
    "3b": ("esm2_t36_3B", 8, 1024),       # configs[3] (8 x 1024 per GPU: 67.6 % MFU vs 56.7 % at 4; 71.1 % at 12)
    "8m": ("esm2_t6_8M", 8, 512),         # configs[0] geometry (CPU oracle config) on the GPU
    "geneformer": ("geneformer", 16, 2048),  # configs[4]: Geneformer 106M, rank-value tokens, seq 2048
}
GF_GENES = 25424      # V = n_genes + 2 = 25,426
GF_NNZ = (500, 4000)  # non-zero genes per synthetic cell


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="650m", choices=sorted(WORKLOADS),
                    help="BASELINE configs: 650m = configs[2], the config the metric and the 45%% MFU target are "
                         "quoted on (default); 35m = configs[1]")
    ap.add_argument("--batch", type=int, default=None, help="sequences per GPU")
    ap.add_argument("--seq", type=int, default=None)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="skip the per-kernel CUDA-event breakdown")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dp", default="zero1", choices=["zero1", "ddp"],
                    help="N>1: zero1 = sharded optimizer (reduce-scatter / AdamW on the rank's slice / all-gather of "
                         "the updated parameters; the ZeRO-1 comparison point of PAPER.md:86-88), ddp = all-reduce "
                         "+ replicated AdamW")
    ap.add_argument("--grad-bf16", action="store_true", help="N>1: bf16 gradient buckets (half the NVLink bytes)")
    ap.add_argument("--master", default="vectors", choices=["vectors", "full"],
                    help="zero1: keep the fp32 master sharded and all-gather only the bf16 shadow (+ the 1-D fp32 "
                         "parameters), or all-gather the whole fp32 master as well")
    ap.add_argument("--nvtx", action="store_true", help="NVTX ranges around the step phases and layers")
    ap.add_argument("--dropout", default="0,0", metavar="HIDDEN,ATTN",
                    help="hidden / attention-probability dropout (ESM-2 trains with 0,0; Geneformer's BERT 0.02,0.02)")
    ap.add_argument("--varlen", action="store_true",
                    help="protein-like lengths (lognormal(5.6, 0.65) clipped to [10, seq]) batched by the reference's "
                         "create_buckets / bucket_batches at a token budget of batch x seq (SURVEY.md §8d, §8f.1)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops", 1590.0), d.get("bf16_tflops_sustained", 1400.0), \
            "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.out = tempfile.NamedTemporaryFile(mode="w+", suffix=".csv", delete=False)

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "200"], stdout=self.out,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.out.flush()
        with open(self.out.name) as f:
            rows = [r.strip().split(", ") for r in f if r.strip()]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except ValueError:
                continue
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class KernelTimer:
    """CUDA events around every C-ABI launch of one eager step (per-kernel roofline)."""

    def __init__(self):
        import torch
        self.torch = torch
        self.recs = []
        self._cur = None

    def begin(self, name):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self._cur = (name, e)

    def end(self, flops, nbytes):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record()
        self.recs.append((self._cur[0], self._cur[1], e, flops, nbytes))

    def summary(self):
        self.torch.cuda.synchronize()
        agg = {}
        for name, a, b, fl, nb in self.recs:
            d = agg.setdefault(name, {"ms": 0.0, "launches": 0, "flops": 0.0, "bytes": 0.0})
            d["ms"] += a.elapsed_time(b)
            d["launches"] += 1
            d["flops"] += fl
            d["bytes"] += nb
        return agg


# DRAM bytes per launch of a dominant kernel, from one `ncu --set full` capture (dram__bytes_read.sum +
# dram__bytes_write.sum); keyed by (preset, batch, seq, C-ABI entry)
NCU_TRAFFIC = {
    ("esm2_t12_35M", 32, 1024, "esm_attn_bwd_qkv"):
        (279.5e6, "profiles/r1e_ncu_summary.txt: persistent fa::bwd_kernel<24>, the main kernel of the entry "
                  "point (read 194.2 MB + write 85.2 MB per layer launch)"),
    ("esm2_t33_650M", 16, 1024, "gemm_tcgen05"):
        (234.8e6, "profiles/r3r_ncu_launches_650m_summary.txt: sm100::gemm_tc_kernel, DRAM read + write averaged over "
                  "the 399 GEMM launches of one 650M step (ncu launch list, dram__bytes_read/write.sum)"),
    ("esm2_t33_650M", 16, 1024, "esm_attn_bwd_qkv"):
        (372.8e6, "profiles/r3r_ncu_launches_650m_summary.txt: persistent fa::bwd_kernel<64> (fused dqkv), DRAM read "
                  "+ write per layer launch in the 650M step"),
}


def roofline_of(name, d, total_ms, tf_sust, hbm, peak_src):
    if d["flops"]:
        ach = d["flops"] / (d["ms"] * 1e-3) / 1e12
        return {"kernel": name, "bound": "tensor", "achieved": round(ach, 1), "peak": tf_sust,
                "peak_kind": f"bf16_tflops_sustained ({peak_src})", "unit": "TFLOP/s", "frac": round(ach / tf_sust, 4),
                "traffic": None, "share_of_step": round(d["ms"] / total_ms, 4),
                "flops_per_launch": d["flops"] / max(1, d["launches"]), "launches_per_step": d["launches"],
                "ms_per_launch": d["ms"] / max(1, d["launches"])}
    ach = d["bytes"] / (d["ms"] * 1e-3) / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(ach / hbm, 4), "traffic": None, "share_of_step": round(d["ms"] / total_ms, 4),
            "bytes_per_launch": d["bytes"] / max(1, d["launches"]), "launches_per_step": d["launches"],
            "ms_per_launch": d["ms"] / max(1, d["launches"])}


# ------------------------------------------------------------------ CPU reference
def cpu_model_name() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def hf_reference_step_time(preset_name, seq, steps=1, warm=1):
    """Time Hugging Face ``EsmForMaskedLM`` (transformers 5.5.0, eager fp32 autograd) + ``torch.optim.AdamW``
    -- the third-party implementation the oracle restates and is pinned to (tests/golden/hf_*.npz) -- on the
    host's cores: one train step per timed step on a 1 x seq sample (bounded CPU work).  Returns
    (tokens/s, s/step, threads).  The reference package (densefeed) has no train path."""
    import numpy as np
    import torch
    from transformers import EsmConfig as HFConfig
    from transformers import EsmForMaskedLM as HFModel
    from paper_2411_10548_b200 import preset
    c = preset(preset_name)
    threads = os.cpu_count()
    torch.set_num_threads(threads)
    torch.manual_seed(1)
    hcfg = HFConfig(vocab_size=c.vocab_size, hidden_size=c.hidden_size, num_hidden_layers=c.num_hidden_layers,
                    num_attention_heads=c.num_attention_heads, intermediate_size=c.intermediate_size,
                    position_embedding_type="rotary", token_dropout=c.token_dropout, mask_token_id=c.mask_token_id,
                    pad_token_id=c.pad_token_id, hidden_dropout_prob=0.0, attention_probs_dropout_prob=0.0,
                    max_position_embeddings=max(c.max_position_embeddings, seq + 2), emb_layer_norm_before=False,
                    layer_norm_eps=c.layer_norm_eps)
    m = HFModel(hcfg)
    m.train()
    opt = torch.optim.AdamW(m.parameters(), lr=4e-4, betas=(0.9, 0.98), eps=1e-8, weight_decay=0.01)
    rng = np.random.default_rng(0)
    lo, n = c.mlm_random
    ids = torch.from_numpy(rng.integers(lo, lo + n, size=(1, seq)).astype(np.int64))
    if c.vocab_size <= 40:
        ids[0, 0], ids[0, -1] = c.cls_token_id, c.eos_token_id
    am = torch.ones_like(ids)

    def one(i):
        sel = torch.from_numpy(np.random.default_rng(100 + i).random((1, seq)) < 0.15)
        lab = torch.where(sel, ids, torch.full_like(ids, -100))
        inp = torch.where(sel, torch.full_like(ids, c.mask_token_id), ids)
        out = m(input_ids=inp, attention_mask=am, labels=lab)
        out.loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)

    for i in range(warm):
        one(i)
    t0 = time.perf_counter()
    for i in range(steps):
        one(warm + i)
    dt = (time.perf_counter() - t0) / steps
    return seq / dt, dt, threads


HF_SAMPLE = "HF transformers 5.5.0 EsmForMaskedLM eager fp32 + torch.optim.AdamW (the implementation the oracle " \
            "restates; densefeed has no train path)"


def run_reference(args, rank, world):
    """``--impl reference``: rank 0 times the CPU implementation of the path on the host cores (all threads),
    one 1 x S train step per step; other ranks exit without work."""
    preset_name, B, S = WORKLOADS[args.config]
    S = args.seq or S
    if rank != 0:
        return
    warm = min(args.warmup, 1)
    tps, dt, threads = hf_reference_step_time(preset_name, S, steps=max(1, args.steps), warm=warm)
    line = {
        "impl": "reference", "metric": ("Geneformer" if args.config == "geneformer" else "ESM-2") +
        " MLM train tokens/sec", "value": tps, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{preset_name} MLM train step (fwd+bwd+AdamW) on the host CPU, "
                               f"sample 1 x {S} tokens/step", "model": preset_name, "seq_len": S},
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "cpu": cpu_model_name(), "impl": HF_SAMPLE,
                         "sample": f"1 x {S} tokens per step ({warm} untimed warm-up step(s))"},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ variable-length (bucketed) protein batches
def import_reference():
    """densefeed from the unmodified reference install (baseline/_ref; /root/reference in the build container)."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(p) and p not in sys.path:
            sys.path.append(p)
    import densefeed
    return densefeed


def run_varlen(args, rank, world, local, dev):
    """Tokens/s on protein-like lengths: a seeded corpus of lognormal(5.6, 0.65) lengths clipped to [10, S]
     is bucketed by the reference's create_buckets and batched by its bucket_batches under a
    token budget of B x S (cost model = tokens); every rank runs the same seeded iterator and takes batches
    i = rank (mod world).  Each step goes through the public API
    EsmForMaskedLM.train_step_tokens (host token lists -> collate, H2D, device masking, fwd, bwd, AdamW); one
    CUDA graph per bucket shape (N = 1), all captured before the timed region.  Value = non-pad tokens/s."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2411_10548_b200 import preset
    from paper_2411_10548_b200.data import collate
    from paper_2411_10548_b200.ddp import GradAllReducer
    from paper_2411_10548_b200.model import EsmForMaskedLM
    densefeed = import_reference()
    preset_name, B, S = WORKLOADS[args.config]
    B, S = args.batch or B, args.seq or S
    cfg = preset(preset_name)
    if cfg.vocab_size > 40:
        raise SystemExit("--varlen: ESM-2 protein configs only")
    rng = np.random.default_rng(0)
    n_seq = 64 * B
    lens = np.clip(rng.lognormal(5.6, 0.65, n_seq), 10, S).astype(np.int64)
    corpus = [np.r_[0, rng.integers(4, 24, L - 2), 2].astype(np.int32) for L in lens]
    spec = densefeed.create_buckets(lens.tolist(), max_width=32, min_count=2 * B)
    cost = densefeed.CostModel(weights=np.array([1.0]), intercept=0.0, safety_margin=1.0)  # tokens
    feats = lens.reshape(-1, 1).astype(np.float64)
    batches = [b.indices for b in densefeed.bucket_batches(spec, feats, cost, float(B * S), seed=7)]
    mine = batches[rank::world]
    pad_to = 16
    shapes = sorted({(len(b), (int(lens[b].max()) + pad_to - 1) // pad_to * pad_to) for b in mine},
                    key=lambda x: x[0] * x[1])
    model = EsmForMaskedLM(cfg, dtype=args.dtype, device=dev, seed=1)
    model.max_workspaces = len(shapes) + 1
    model.reserve(*max(shapes, key=lambda x: x[0] * x[1]))
    if world > 1:
        model.comm = GradAllReducer(model.store, grad_dtype="bf16" if args.grad_bf16 else "fp32",
                                    shard_optimizer=args.dp == "zero1", master=args.master)
    use_graph = not args.no_graph
    seed = 4321

    def step(i):
        toks = [corpus[j] for j in mine[i % len(mine)]]
        return model.train_step_tokens(toks, seed=seed, stream_id=i * world + rank, pad_to=pad_to,
                                       use_graph=use_graph)

    # capture every bucket shape once (untimed), then the warm-up steps
    seen = set()
    for i, b in enumerate(mine):
        shp = (len(b), (int(lens[b].max()) + pad_to - 1) // pad_to * pad_to)
        if shp not in seen:
            seen.add(shp)
            step(i)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tok = pad_tok = attn_sq = 0.0
    l0 = model.launches
    e0.record()
    for i in range(args.steps):
        b = mine[(args.warmup + i) % len(mine)]
        step(args.warmup + i)
        tok += float(lens[b].sum())
        attn_sq += float((lens[b].astype(np.float64) ** 2).sum())
        pad_tok += len(b) * ((int(lens[b].max()) + pad_to - 1) // pad_to * pad_to)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clocks = sampler.stop() if sampler else None
    t = torch.tensor([ms, tok, pad_tok, attn_sq], device=dev, dtype=torch.float64)
    if world > 1:
        mx = t[:1].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t)
        t[0] = mx[0]
    ms, tok, pad_tok, attn_sq = (float(x) for x in t)
    value = tok / args.steps / (ms / 1e3)
    _, _, tf_sust, peak_src = load_peaks()
    flops_tok = cfg.train_flops_per_token(0) + 12.0 * cfg.num_hidden_layers * cfg.hidden_size * attn_sq / tok
    if rank == 0:
        print(json.dumps({
            "metric": "ESM-2 MLM train tokens/sec", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{preset_name} MLM pre-training on bucketed variable-length proteins "
                                   f"(token budget {B * S} per GPU-step)", "model": preset_name,
                       "seq_len": S, "parallelism": f"dp{world}", "cuda_graph": use_graph,
                       "lengths": f"lognormal(5.6, 0.65) clipped to [10, {S}], {n_seq} sequences",
                       "batching": "densefeed.create_buckets(max_width=32, min_count=2B) + bucket_batches (tokens), pad to 16",
                       "bucket_shapes": len(shapes), "non_pad_fraction": round(tok / pad_tok, 4),
                       "api": "EsmForMaskedLM.train_step_tokens (host token lists -> H2D -> mask -> step)"},
            "mfu": round(value / world * flops_tok / (tf_sust * 1e12), 4),
            "mfu_peak": f"{tf_sust} TFLOP/s bf16 sustained ({peak_src})", "train_flops_per_token": flops_tok,
            "gpu_launches": (model.launches - l0) // max(1, args.steps), "clocks": clocks}), flush=True)


# ------------------------------------------------------------------ our B200 path
def main():
    args = parse()
    # NCCL's debug/version banner goes to stdout by default; keep stdout to the one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2411_10548_b200 import preset
    from paper_2411_10548_b200.data import synthetic_batch
    from paper_2411_10548_b200.ddp import GradAllReducer
    from paper_2411_10548_b200.model import EsmForMaskedLM

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.varlen:
        run_varlen(args, rank, world, local, dev)
        if world > 1:
            dist.destroy_process_group()
        return
    preset_name, B, S = WORKLOADS[args.config]
    B = args.batch or B
    S = args.seq or S
    cfg = preset(preset_name)
    p_hid, p_att = (float(x) for x in args.dropout.split(","))
    cfg.hidden_dropout_prob, cfg.attention_probs_dropout_prob = p_hid, p_att
    model = EsmForMaskedLM(cfg, dtype=args.dtype, device=dev, seed=1)
    model.nvtx = args.nvtx
    ws = model.workspace(B, S)
    if world > 1:
        model.comm = GradAllReducer(model.store, grad_dtype="bf16" if args.grad_bf16 else "fp32",
                                    shard_optimizer=args.dp == "zero1", master=args.master)
    use_graph = not args.no_graph  # N > 1: the NCCL bucket collectives are captured in the same graph

    gene = cfg.vocab_size > 40
    if gene:  # Geneformer: synthetic cells -> rank-value tokens on the GPU (esm_rank_encode)
        from paper_2411_10548_b200.data import RankEncoder, gene_medians, synthetic_expression_csr
        csr = synthetic_expression_csr(4 * B, GF_GENES, seed=100 + rank, nnz=GF_NNZ)
        enc = RankEncoder(gene_medians(*csr, GF_GENES), device=dev)
        pool, pool_am = [], []
        for i in range(2):
            ids_i, am_i, _ = enc(*csr, np.arange(i * B, (i + 1) * B), seq_len=S)
            pool.append(ids_i)
            pool_am.append(am_i)
        lens = [a.sum(1).double() for a in pool_am]
        tokens_local = float(sum(float(x.sum()) for x in lens) / 2)     # non-pad tokens per step
        attn_sq = float(sum(float((x * x).sum()) for x in lens) / 2)    # sum of len^2 (attention FLOPs)
    else:
        pool = [torch.from_numpy(synthetic_batch(B, S, seed=1000 * rank + i)[0]).to(dev) for i in range(2)]
        pool_am = None
        tokens_local, attn_sq = float(B * S), float(B * S * S)
    seed = 1234

    def step(i):
        if pool_am is not None:
            ws.am.copy_(pool_am[i % 2], non_blocking=True)
        model.mlm_mask(pool[i % 2], seed, i * world + rank, ws)
        if use_graph:
            model.graph_step()
        else:
            model.step(ws)

    if use_graph:
        if pool_am is not None:
            ws.am.copy_(pool_am[0])
        model.mlm_mask(pool[0], seed, rank, ws)
        model.capture(ws)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()

    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = model.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        step(args.warmup + i)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = (model.launches - l0) // max(1, args.steps)
    ms = e0.elapsed_time(e1) / args.steps
    clocks = sampler.stop() if sampler else None
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    loss = float(ws.loss_sum.item())
    tk = torch.tensor([tokens_local, attn_sq], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tk)
    tokens_per_step, attn_sq_all = float(tk[0]), float(tk[1])   # non-pad tokens, all ranks
    value = tokens_per_step / (ms / 1e3)

    # ---------------- end to end through the public API, host buffers
    class LossToHost:
        """Every step's loss is copied device -> pinned host inside the timed region (non-blocking) and read by
        the host one step behind, as a training loop logs it: the host never stalls the GPU between steps."""

        def __init__(self, n):
            self.host = torch.empty(max(n, 1), dtype=torch.float32).pin_memory()
            self.ev = [torch.cuda.Event(), torch.cuda.Event()]
            self.vals = []

        def push(self, i, loss_dev):
            self.host[i:i + 1].copy_(loss_dev.view(-1)[:1], non_blocking=True)
            self.ev[i % 2].record()
            if i > 0:
                self.ev[(i - 1) % 2].synchronize()
                self.vals.append(float(self.host[i - 1]))

        def finish(self, n):
            torch.cuda.synchronize()
            self.vals.append(float(self.host[n - 1]))
            if len(self.vals) != n or not all(np.isfinite(self.vals)):
                raise RuntimeError(f"e2e: bad per-step losses {self.vals}")

    e2e = None
    if not args.no_e2e and gene:
        # per step: pinned CSR rows of the batch -> HBM, GPU rank tokenisation into ws.ids / ws.am,
        # device masking, the train step, loss -> host
        staged = []
        for i in range(2):
            rows = np.arange(i * B, (i + 1) * B) + 2 * B
            ip, cols, vals = csr
            lo, hi = ip[rows], ip[rows + 1]
            sub_ip = np.r_[0, np.cumsum(hi - lo)].astype(np.int64)
            idx = np.concatenate([np.arange(a, b) for a, b in zip(lo, hi)])
            staged.append([torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
                           for a in (sub_ip, cols[idx].astype(np.int64), vals[idx].astype(np.float32))]
                          + [int((hi - lo).max())])
        cap = max(int(x[1].numel()) for x in staged)
        d_ip = torch.empty(B + 1, dtype=torch.int64, device=dev)
        d_c = torch.empty(cap, dtype=torch.int64, device=dev)
        d_v = torch.empty(cap, dtype=torch.float32, device=dev)
        h2d = sum(int(t.numel() * t.element_size()) for x in staged for t in x[:3]) // 2

        def e2e_step(i):
            h_ip, h_c, h_v, mx = staged[i % 2]
            d_ip.copy_(h_ip, non_blocking=True)
            d_c[:h_c.numel()].copy_(h_c, non_blocking=True)
            d_v[:h_v.numel()].copy_(h_v, non_blocking=True)
            enc.encode_device(d_ip, d_c, d_v, B, mx, S, ids=ws.ids, am=ws.am)
            model.mlm_mask(ws.ids, seed, 10_000 + i * world + rank, ws)
            if use_graph:
                model.graph_step()
            else:
                model.step(ws)

        for i in range(2):
            e2e_step(i)
            float(ws.loss_sum.item())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        reader = LossToHost(args.steps)
        t0 = time.perf_counter()
        for i in range(args.steps):
            e2e_step(i)
            reader.push(i, ws.loss_sum)                            # D2H: the step's loss
        reader.finish(args.steps)
        wall = (time.perf_counter() - t0) / args.steps
        tw = torch.tensor([wall], device=dev)
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall = float(tw.item())
        enc.check()
        e2e = {"value": tokens_per_step / wall, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 4, "ms_per_step": wall * 1e3, "d2h": "each step's loss, non-blocking into pinned host, read one step behind",
               "api": "RankEncoder.encode_device (CSR rows) + EsmForMaskedLM.mlm_mask + graph_step",
               "inputs": "CSR expression rows (indptr/cols int64, vals f32), pinned host"}
    elif not args.no_e2e:
        host = [torch.from_numpy(synthetic_batch(B, S, seed=1000 * rank + 7 + i)[0]).pin_memory() for i in range(2)]
        for i in range(2):
            ws.ids.copy_(host[i % 2], non_blocking=True)
            step(100 + i)
            float(ws.loss_sum.item())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        reader = LossToHost(args.steps)
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        d0.record()
        for i in range(args.steps):
            ws.ids.copy_(host[i % 2], non_blocking=True)          # H2D: this step's token ids
            model.mlm_mask(ws.ids, seed, 10_000 + i * world + rank, ws)
            if use_graph:
                model.graph_step()
            else:
                model.step(ws)
            reader.push(i, ws.loss_sum)                            # D2H: the step's loss (read one step behind)
        d1.record()
        reader.finish(args.steps)
        wall = (time.perf_counter() - t0) / args.steps
        dev_ms = d0.elapsed_time(d1) / args.steps
        tw = torch.tensor([wall], device=dev)
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall = float(tw.item())
        e2e = {"value": tokens_per_step / wall, "unit": "tokens/s", "h2d_bytes_per_step": B * S * 4,
               "d2h_bytes_per_step": 4, "ms_per_step": wall * 1e3, "device_ms_per_step": dev_ms,
               "d2h": "each step's loss, non-blocking into pinned host, read one step behind", "api": "EsmForMaskedLM.mlm_mask+graph_step"
               if use_graph else "EsmForMaskedLM.mlm_mask+step"}

    # ---------------- per-kernel breakdown (one extra eager step under CUDA events)
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    roofline, kernels, roofline_gemm = None, None, None
    if not args.no_profile:
        model.timer = KernelTimer()
        if pool_am is not None:
            ws.am.copy_(pool_am[0])
        model.mlm_mask(pool[0], seed, 999, ws)
        if model.comm is not None and (model.comm.shard or model.comm.bf16):
            model.step(ws)  # the optimizer runs per bucket slice inside the step
        else:
            model.forward_backward(ws)
            model.optimizer_step()
        agg = model.timer.summary()
        model.timer = None
        total = sum(d["ms"] for d in agg.values())
        fam = {}
        for name, d in agg.items():
            f = "gemm_tcgen05" if name.startswith("gemm_") else name
            x = fam.setdefault(f, {"ms": 0.0, "launches": 0, "flops": 0.0, "bytes": 0.0})
            for k in x:
                x[k] += d[k]
        kernels = {k: {"ms": round(v["ms"], 4), "share": round(v["ms"] / total, 4), "launches": v["launches"],
                       **({"tflops": round(v["flops"] / (v["ms"] * 1e-3) / 1e12, 1)} if v["flops"] else {}),
                       **({"gbs": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1)} if v["bytes"] else {})}
                   for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["ms"])}
        # dominant kernel = the CUDA kernel function with the largest share of the step: every tcgen05 GEMM
        # launch (fwd / dgrad / wgrad, all shapes) is one kernel, sm100::gemm_tc_kernel; other families are
        # one C-ABI entry point each.  The ncu launch list of the same command agrees (profiles/).
        dom_name, dom = max(fam.items(), key=lambda kv: kv[1]["ms"])
        label = "sm100::gemm_tc_kernel (all GEMM launches: fwd, dgrad, wgrad)" if dom_name == "gemm_tcgen05" \
            else dom_name
        roofline = roofline_of(label, dom, total, tf_sust, hbm, peak_src)
        tr = NCU_TRAFFIC.get((preset_name, B, S, dom_name))
        if tr is not None:
            roofline["traffic"], roofline["traffic_source"] = tr
        # the largest non-GEMM kernel (attention) is reported beside it
        att_name, att = max(((k, v) for k, v in fam.items() if k != "gemm_tcgen05" and v["flops"]),
                            key=lambda kv: kv[1]["ms"], default=(None, None))
        if att is not None:
            roofline_gemm = roofline_of(att_name, att, total, tf_sust, hbm, peak_src)
            tr = NCU_TRAFFIC.get((preset_name, B, S, att_name))
            if tr is not None:
                roofline_gemm["traffic"], roofline_gemm["traffic_source"] = tr

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        S_cpu = min(S, 1024)  # bounded sample (~10-30 s of CPU work)
        tps, dt, threads = hf_reference_step_time(preset_name, S_cpu, steps=1, warm=1)
        cpu_baseline = {"value": tps, "unit": "tokens/s", "cores": threads, "kind": "reference",
                        "cpu": cpu_model_name(), "impl": HF_SAMPLE,
                        "sample": f"{preset_name}, 1 x {S_cpu} tokens, one timed train step after one warm-up "
                                  f"({dt:.1f} s)"}

    # FLOPs per non-pad token: 6*N_mm (decoder on labelled rows only for the large-vocabulary head)
    # + attention 12*L*H*len averaged over the actual sequence lengths
    L_, H_ = cfg.num_hidden_layers, cfg.hidden_size
    flops_tok = cfg.train_flops_per_token(0, head_fraction=0.15 if gene else 1.0) + \
        12.0 * L_ * H_ * attn_sq_all / tokens_per_step
    mfu = value / world * flops_tok / (tf_sust * 1e12)
    if rank == 0:
        line = {
            "metric": ("Geneformer" if gene else "ESM-2") + " MLM train tokens/sec", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{preset_name} MLM pre-training step (mask+fwd+bwd+AdamW), {B} x {S} per GPU",
                       "model": preset_name, "global_batch": B * world, "seq_len": S,
                       "parallelism": f"dp{world}" + ("-zero1" if args.dp == "zero1" and world > 1 else "") +
                                      ("-fullmaster" if args.dp == "zero1" and world > 1 and args.master == "full"
                                       else "") + ("-bf16grad" if args.grad_bf16 and world > 1 else ""),
                       "l2": "inputs/activations >> 126 MB L2 (no flush needed)",
                       "cuda_graph": use_graph, "weights": "random init",
                       **({"dropout": {"hidden": p_hid, "attention_probs": p_att}} if p_hid or p_att else {}),
                       "data": (f"synthetic cells, {GF_NNZ[0]}-{GF_NNZ[1]} expressed genes of {GF_GENES}, "
                                f"GPU rank-value tokens; non-pad tokens counted "
                                f"({tokens_per_step / (B * S * world):.3f} fill)") if gene
                       else "synthetic uniform AA"},
            "mfu": round(mfu, 4), "mfu_peak": f"{tf_sust} TFLOP/s bf16 sustained ({peak_src})",
            "train_flops_per_token": flops_tok, "loss": loss,
            "roofline": roofline, "roofline_attention": roofline_gemm, "cpu_baseline": cpu_baseline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "kernels": kernels,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
