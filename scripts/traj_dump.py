"""Dump the bf16 (and fp32) 200-step loss curves of configs[0] next to the oracle's golden curve
(tests/golden/traj_8m_<sched>.npz) -> gpurun_out/traj_<sched>.json.   python scripts/traj_dump.py const"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from test_gpu_trajectory import _curve  # noqa: E402

sched = sys.argv[1] if len(sys.argv) > 1 else "const"
ref = np.load(os.path.join(ROOT, "tests", "golden", f"traj_8m_{sched}.npz"))["losses"]
out = {"sched": sched, "oracle": ref.tolist()}
for dt in sys.argv[2:] or ["bf16", "fp32"]:
    got = _curve(dt, sched, len(ref))
    out[dt] = got.tolist()
    rel = np.abs(got - ref) / ref
    print(dt, "final", got[-1], ref[-1], "worst", rel.max(), "at step", int(rel.argmax()) + 1, flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"traj_{sched}.json"), "w"))
