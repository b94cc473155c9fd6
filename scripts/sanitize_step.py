"""One small bf16 MLM train step (every production kernel: tcgen05 GEMMs incl. CTA pairs, persistent attention
forward / fused and classic backward, LayerNorm, embedding, CE, AdamW, hidden dropout) for compute-sanitizer:

    compute-sanitizer --tool memcheck   python scripts/sanitize_step.py
    compute-sanitizer --tool racecheck  python scripts/sanitize_step.py
    compute-sanitizer --tool synccheck  python scripts/sanitize_step.py
Logs are kept under profiles/ (DESIGN.md §8)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_10548_b200 import EsmConfig  # noqa: E402
from paper_2411_10548_b200.data import synthetic_batch  # noqa: E402
from paper_2411_10548_b200.model import EsmForMaskedLM  # noqa: E402


def main():
    for H, nh, F, drop in ((480, 20, 1920, 0.0), (256, 4, 1024, 0.1)):  # dh 24 (fused bwd), dh 64 (classic)
        cfg = EsmConfig(hidden_size=H, num_hidden_layers=1, num_attention_heads=nh, intermediate_size=F,
                        hidden_dropout_prob=drop)
        m = EsmForMaskedLM(cfg, dtype="bf16", device="cuda", seed=1)
        B, S = 2, 256
        ids, am = synthetic_batch(B, S, seed=1)
        ws = m.workspace(B, S)
        am[1, 200:] = 0
        ws.am.copy_(torch.from_numpy(am))
        m.mlm_mask(torch.from_numpy(ids).cuda(), seed=1, stream_id=0, ws=ws)
        loss = float(m.step(ws).item())
        torch.cuda.synchronize()
        print(f"H={H} nh={nh} dropout={drop}: loss {loss:.4f}", flush=True)
    print("sanitize step done")


if __name__ == "__main__":
    main()
