#!/usr/bin/env python
"""ESM-2 MLM training throughput on B200 (BASELINE.json metric: "ESM-2 MLM train tokens/sec at
1/2/4/8 B200; MFU vs bf16 tensor peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 35m] [--batch 32] [--seq 1024]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference      # the CPU oracle (reference semantics) on the host cores

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
    "3b": ("esm2_t36_3B", 4, 1024),       # configs[3]
    "8m": ("esm2_t6_8M", 8, 512),         # configs[0] geometry (CPU oracle config) on the GPU
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="35m", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None, help="sequences per GPU")
    ap.add_argument("--seq", type=int, default=None)
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of one CUDA graph per step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="skip the per-kernel CUDA-event breakdown")
    ap.add_argument("--no-e2e", action="store_true")
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


# ------------------------------------------------------------------ CPU reference (oracle)
def cpu_reference_step_time(preset_name, seq, steps=1, warm=0):
    """Time the CPU oracle (numpy fp32, reference semantics) on a 1 x seq sample; tokens/s."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import esm2_oracle as O
    from paper_2411_10548_b200.config import PRESETS
    p = PRESETS[preset_name]
    cfg = O.OracleConfig(hidden_size=p["hidden_size"], num_hidden_layers=p["num_hidden_layers"],
                         num_attention_heads=p["num_attention_heads"], intermediate_size=p["intermediate_size"])
    params = O.init_params(cfg, seed=1)
    tr = O.OracleTrainer(cfg, params, dtype=np.float32)
    ids, am = O.synthetic_batch(1, seq, seed=0)
    for i in range(warm):
        inp, lab = O.mlm_mask(ids, 0, i)
        tr.step(inp, am, lab)
    t0 = time.perf_counter()
    for i in range(steps):
        inp, lab = O.mlm_mask(ids, 0, 100 + i)
        tr.step(inp, am, lab)
    dt = (time.perf_counter() - t0) / steps
    return seq / dt, dt


def run_reference(args, rank, world):
    preset_name, B, S = WORKLOADS[args.config]
    S = args.seq or S
    if rank != 0:
        return
    cores = os.cpu_count()
    warm = min(args.warmup, 1)
    tps, dt = cpu_reference_step_time(preset_name, S, steps=max(1, args.steps), warm=warm)
    line = {
        "impl": "reference", "metric": "ESM-2 MLM train tokens/sec", "value": tps, "unit": "tokens/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{preset_name} MLM train step, reference CPU oracle, sample 1 x {S} tokens/step",
                   "model": preset_name, "seq_len": S},
        "cpu_baseline": {"value": tps, "unit": "tokens/s", "cores": cores, "kind": "port",
                         "sample": f"1 x {S} tokens per step ({warm} warm-up step(s) run)"},
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our B200 path
def main():
    args = parse()
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
    preset_name, B, S = WORKLOADS[args.config]
    B = args.batch or B
    S = args.seq or S
    cfg = preset(preset_name)
    model = EsmForMaskedLM(cfg, dtype=args.dtype, device=dev, seed=1)
    ws = model.workspace(B, S)
    if world > 1:
        model.comm = GradAllReducer(model.store)
    use_graph = (world == 1) and not args.no_graph

    pool = [torch.from_numpy(synthetic_batch(B, S, seed=1000 * rank + i)[0]).to(dev) for i in range(2)]
    seed = 1234

    def step(i):
        model.mlm_mask(pool[i % 2], seed, i * world + rank, ws)
        if use_graph:
            model.graph_step()
        else:
            model.forward_backward(ws)
            model.optimizer_step()

    if use_graph:
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
    tokens_per_step = B * S * world
    value = tokens_per_step / (ms / 1e3)

    # ---------------- end to end through the public API, host buffers
    e2e = None
    if not args.no_e2e:
        host = [torch.from_numpy(synthetic_batch(B, S, seed=1000 * rank + 7 + i)[0]).pin_memory() for i in range(2)]
        for i in range(2):
            ws.ids.copy_(host[i % 2], non_blocking=True)
            step(100 + i)
            float(ws.loss_sum.item())
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            ws.ids.copy_(host[i % 2], non_blocking=True)          # H2D: this step's token ids
            model.mlm_mask(ws.ids, seed, 10_000 + i * world + rank, ws)
            if use_graph:
                model.graph_step()
            else:
                model.forward_backward(ws)
                model.optimizer_step()
            float(ws.loss_sum.item())                              # D2H: the step's loss
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / args.steps
        tw = torch.tensor([wall], device=dev)
        if world > 1:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        wall = float(tw.item())
        e2e = {"value": tokens_per_step / wall, "unit": "tokens/s", "h2d_bytes_per_step": B * S * 4,
               "d2h_bytes_per_step": 4, "ms_per_step": wall * 1e3, "api": "EsmForMaskedLM.mlm_mask+graph_step"
               if use_graph else "EsmForMaskedLM.mlm_mask+forward_backward+optimizer_step"}

    # ---------------- per-kernel breakdown (one extra eager step under CUDA events)
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    roofline, kernels = None, None
    if not args.no_profile:
        model.timer = KernelTimer()
        model.mlm_mask(pool[0], seed, 999, ws)
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
        dom_name, dom = max(fam.items(), key=lambda kv: kv[1]["ms"])
        if dom["flops"]:
            ach = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
            roofline = {"kernel": dom_name, "bound": "tensor", "achieved": round(ach, 1), "peak": tf_sust,
                        "peak_kind": f"bf16_tflops_sustained ({peak_src})", "unit": "TFLOP/s",
                        "frac": round(ach / tf_sust, 4), "traffic": None, "share_of_step": round(dom["ms"] / total, 4),
                        "flops_per_step": dom["flops"], "launches_per_step": dom["launches"]}
        else:
            ach = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
            roofline = {"kernel": dom_name, "bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(ach / hbm, 4), "traffic": None, "share_of_step": round(dom["ms"] / total, 4)}

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tps, dt = cpu_reference_step_time(preset_name, S, steps=1)
        cpu_baseline = {"value": tps, "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
                        "sample": f"CPU oracle (numpy fp32, reference semantics) {preset_name}, 1 x {S} tokens, "
                                  f"one train step ({dt:.1f} s)"}

    flops_tok = cfg.train_flops_per_token(S)
    mfu = value / world * flops_tok / (tf_sust * 1e12)
    if rank == 0:
        line = {
            "metric": "ESM-2 MLM train tokens/sec", "value": value, "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{preset_name} MLM pre-training step (mask+fwd+bwd+AdamW), {B} x {S} per GPU",
                       "model": preset_name, "global_batch": B * world, "seq_len": S,
                       "parallelism": f"dp{world}", "l2": "inputs/activations >> 126 MB L2 (no flush needed)",
                       "cuda_graph": use_graph, "weights": "random init", "data": "synthetic uniform AA"},
            "mfu": round(mfu, 4), "mfu_peak": f"{tf_sust} TFLOP/s bf16 sustained ({peak_src})",
            "train_flops_per_token": flops_tok, "loss": loss,
            "roofline": roofline, "cpu_baseline": cpu_baseline, "e2e": e2e, "gpu_launches": launches,
            "clocks": clocks, "kernels": kernels,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
