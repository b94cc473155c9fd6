"""Golden 200-step MLM training curves of the CPU oracle (test infrastructure; never imported by the
product path).  North-star criterion (BASELINE.json): "the bf16-mode loss after 200 steps is within 1% of
the reference".  The reference here is the numpy fp32 oracle (oracle/esm2_oracle.py, pinned to HF
EsmForMaskedLM by tests/test_oracle.py) on BASELINE configs[0]: ESM-2 8M (6 layers, H 320, 20 heads),
batch 8 x 512, seeded init (model.init_params seed 1), synthetic full-length proteins
(data.synthetic_batch seed 10_000 + step), MLM masks mlm_mask(seed 3, stream step), AdamW
(0.9, 0.98, 1e-8, wd 0.01).

Schedules:  const  -- lr 4e-4 (ESM-2's peak lr) from step 1
            esm2   -- optim.esm2_lr(step): linear warm-up over 2000 steps to 4e-4 (steps 1..200 of it)

    python oracle/make_golden_trajectory.py [const|esm2 ...]   -> tests/golden/traj_8m_<sched>.npz
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import esm2_oracle as O  # noqa: E402

STEPS, BATCH, SEQ = 200, 8, 512
H, L, NH, F = 320, 6, 20, 1280


def lr_at(sched: str, step: int) -> float:
    return 4e-4 if sched == "const" else O.esm2_lr(step)


def batch_at(step: int):
    """Same draws as paper_2411_10548_b200.data.synthetic_batch(BATCH, SEQ, seed=10_000 + step)."""
    return O.synthetic_batch(BATCH, SEQ, seed=10_000 + step)


def main(scheds):
    from paper_2411_10548_b200.config import preset
    from paper_2411_10548_b200.model import init_params
    cfg = preset("8m")
    params = init_params(cfg, seed=1)
    ocfg = O.OracleConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=NH, intermediate_size=F)
    for sched in scheds:
        tr = O.OracleTrainer(ocfg, params, dtype=np.float32, beta1=0.9, beta2=0.98, eps=1e-8, weight_decay=0.01)
        losses = []
        t0 = time.time()
        for step in range(1, STEPS + 1):
            ids, am = batch_at(step)
            inp, lab = O.mlm_mask(ids, seed=3, stream=step)
            losses.append(float(tr.step(inp, am, lab, lr=lr_at(sched, step))))
            if step % 20 == 0:
                print(f"{sched} step {step} loss {losses[-1]:.5f} [{time.time() - t0:.0f}s]", flush=True)
        out = os.path.join(ROOT, "tests", "golden", f"traj_8m_{sched}.npz")
        np.savez_compressed(out, losses=np.array(losses, np.float64), steps=STEPS, batch=BATCH, seq=SEQ,
                            config=np.array([H, L, NH, F]), sched=sched)
        print("wrote", out)


if __name__ == "__main__":
    main(sys.argv[1:] or ["const", "esm2"])
