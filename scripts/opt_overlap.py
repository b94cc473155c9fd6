"""Step time with AdamW overlapped with the backward vs a separate optimizer pass (eager and graph)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10548_b200 import preset  # noqa: E402
from paper_2411_10548_b200.data import synthetic_batch  # noqa: E402
from paper_2411_10548_b200.model import EsmForMaskedLM  # noqa: E402

name, B = (sys.argv[1], int(sys.argv[2])) if len(sys.argv) > 2 else ("3b", 4)
m = EsmForMaskedLM(preset(name), dtype="bf16", device="cuda")
ws = m.workspace(B, 1024)
ids = torch.from_numpy(synthetic_batch(B, 1024, seed=1)[0]).cuda()
m.mlm_mask(ids, 1, 1, ws)


def t(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def sep():
    m.forward_backward(ws)
    m.optimizer_step()


print(f"{name}: eager separate {t(sep):.2f} ms, eager overlapped {t(lambda: m.step(ws)):.2f} ms, "
      f"forward_backward only {t(lambda: m.forward_backward(ws)):.2f} ms, adamw only {t(m._adamw):.2f} ms", flush=True)
m.capture(ws)
print(f"{name}: graph overlapped {t(m.graph_step):.2f} ms", flush=True)
