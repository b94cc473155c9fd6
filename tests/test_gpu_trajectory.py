"""North-star criterion "the bf16-mode loss after 200 steps is within 1 % of the reference", in the suite.

The reference curve is the fp32 CPU oracle's (oracle/make_golden_trajectory.py -> tests/golden/traj_8m_*.npz):
BASELINE configs[0] (ESM-2 8M, batch 8 x 512), the same seeded init, batches, MLM masks (the device masking
kernel is bit-exact with the oracle's) and AdamW hyper-parameters, under two schedules: constant 4e-4 and the
ESM-2 warm-up (optim.esm2_lr).  The GPU runs the production bf16 path (tcgen05 kernels, one CUDA graph per
step); the fp32 parity mode is checked on the same curve at a tighter bound."""
import os

import numpy as np
import pytest
import torch

import esm2_oracle as O
from paper_2411_10548_b200 import preset
from paper_2411_10548_b200.model import EsmForMaskedLM, init_params
from paper_2411_10548_b200.optim import esm2_lr

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _curve(dtype, sched, steps):
    cfg = preset("8m")
    m = EsmForMaskedLM(cfg, dtype=dtype, device="cuda", params=init_params(cfg, seed=1), lr=4e-4,
                       betas=(0.9, 0.98), eps=1e-8, weight_decay=0.01)
    ws = m.workspace(8, 512)
    out = []
    for step in range(1, steps + 1):
        ids, am = O.synthetic_batch(8, 512, seed=10_000 + step)
        ws.ids.copy_(torch.from_numpy(ids))
        ws.am.copy_(torch.from_numpy(am))
        m.mlm_mask(ws.ids, seed=3, stream_id=step, ws=ws)
        lr = 4e-4 if sched == "const" else esm2_lr(step)
        if dtype == "bf16":
            if step == 1:
                m.capture(ws)
            loss = m.graph_step(lr=lr)
        else:
            loss = m.step(ws, lr=lr)
        out.append(float(loss.item()))
    return np.array(out)


def test_bf16_loss_after_200_steps_within_1pct():
    """North-star criterion on the ESM-2 recipe (linear warm-up to 4e-4): final and last-10-mean loss of 200
    bf16 steps within 1 % of the fp32 oracle (measured on B200: 3e-5)."""
    ref = np.load(os.path.join(GOLD, "traj_8m_esm2.npz"))["losses"]
    got = _curve("bf16", "esm2", len(ref))
    final = abs(got[-1] - ref[-1]) / ref[-1]
    last10 = abs(got[-10:].mean() - ref[-10:].mean()) / ref[-10:].mean()
    worst = float(np.max(np.abs(got - ref) / ref))
    print(f"200-step bf16 [esm2]: final {got[-1]:.5f} vs {ref[-1]:.5f} (rel {final:.2e}), last-10 mean rel "
          f"{last10:.2e}, worst step rel {worst:.2e}")
    assert final < 0.01 and last10 < 0.01 and worst < 0.01


def test_constant_lr_curve_before_and_through_the_oracles_loss_spike():
    """Constant 4e-4 from step 1 (no warm-up) is not a stable recipe: the fp32 oracle's loss spikes at step 71
    (3.02 -> 6.42, profiles/r2_traj_const_bf16_fp32_vs_oracle.json).  Through the spike the fp32 parity mode must
    follow the oracle step for step (the kernels are exact enough to reproduce the divergence); the bf16 path
    must match the oracle within 1 % until the instability, after which its rounding takes a different branch
    (measured: a smaller spike to 3.14 and lower final loss, 2.85 vs 3.01)."""
    ref = np.load(os.path.join(GOLD, "traj_8m_const.npz"))["losses"]
    got32 = _curve("fp32", "const", len(ref))
    rel32 = np.abs(got32 - ref) / ref
    print(f"fp32 200-step const curve: max rel {rel32.max():.2e} (step {int(rel32.argmax()) + 1})")
    assert rel32.max() < 1e-3
    pre = 60
    got16 = _curve("bf16", "const", pre)
    rel16 = np.abs(got16 - ref[:pre]) / ref[:pre]
    print(f"bf16 const steps 1-{pre}: max rel {rel16.max():.2e} (step {int(rel16.argmax()) + 1})")
    assert rel16.max() < 1e-2
