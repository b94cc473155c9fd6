"""Largest ESM-2 batch that trains without running out of HBM -- the paper's single-device memory axis
("46 vs 16" sequences of 1024 for ESM-2 650M on an 80 GB A100) -- found
through the reference's own sizing seam:

  densefeed.collect_peak_alloc(samples = batch sizes, make_workload(model), [tokens], CudaPeakMeter)
    -> densefeed.fit_cost_model -> predicted largest batch under the device's HBM
    -> collect_peak_alloc again at that batch (must succeed) and beyond it (a CUDA OOM is recorded as a
       failed ProfileRecord, the reference's OOM analogue, sizing.py:96-98).

    python scripts/max_batch.py [--config 650m] [--seq 1024]   -> gpurun_out/max_batch_<config>.json
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.append("/root/reference/pkg/src")
import densefeed  # noqa: E402

from paper_2411_10548_b200 import preset  # noqa: E402
from paper_2411_10548_b200.data import synthetic_batch  # noqa: E402
from paper_2411_10548_b200.model import EsmForMaskedLM  # noqa: E402
from paper_2411_10548_b200.seams import CudaPeakMeter  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="650m")
    ap.add_argument("--seq", type=int, default=1024)
    ap.add_argument("--profile", default="1,2,4,8,16")
    a = ap.parse_args()
    cfg = preset(a.config)
    S = a.seq
    model = EsmForMaskedLM(cfg, dtype="bf16", device="cuda", seed=1)
    model.max_workspaces = 1
    total = torch.cuda.mem_get_info()[1]

    def workload(b):  # one full train step (mask, fwd, bwd, AdamW) on b x S tokens, then free its activations
        ids, am = synthetic_batch(b, S, seed=b)
        ws = model.workspace(b, S)
        ws.am.copy_(torch.from_numpy(am))
        model.mlm_mask(torch.from_numpy(ids).cuda(), seed=1, stream_id=b, ws=ws)
        loss = float(model.step(ws).item())
        model.release_workspaces()
        if not np.isfinite(loss):
            raise FloatingPointError("non-finite loss")

    feats = lambda b: [float(b * S)]  # noqa: E731
    meter = CudaPeakMeter()  # absolute peak: resident model state + one step's activations
    prof = [int(x) for x in a.profile.split(",")]
    recs = densefeed.collect_peak_alloc(prof, workload, feats, meter)
    cost, rep = densefeed.fit_cost_model(recs, safety_margin=1.0)
    per_tok, base = float(cost.weights[0]), float(cost.intercept)
    b_pred = int((total - base) / (per_tok * S))
    check = [b_pred - 1, b_pred, b_pred + 4]
    recs2 = densefeed.collect_peak_alloc(check, workload, feats, meter)
    ok = [b for b, r in zip(check, recs2) if not r.failed]
    res = {
        "config": a.config, "seq": S, "device_hbm_bytes": total,
        "profile": [{"batch": b, "peak_bytes": r.peak_cost, "failed": r.failed} for b, r in zip(prof, recs)],
        "fit": {"bytes_per_token": per_tok, "resident_bytes": base, "rmse": rep.rmse},
        "predicted_max_batch": b_pred,
        "checked": [{"batch": b, "peak_bytes": r.peak_cost, "failed": r.failed} for b, r in zip(check, recs2)],
        "max_batch_trained": max(ok) if ok else None,
        "reference_paper": "ESM-2 650M, seq 1024: HF+Accelerate 16, BioNeMo 46 on an 80 GB A100 (PAPER.md:73)",
    }
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"max_batch_{a.config}.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
