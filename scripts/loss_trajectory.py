"""North-star check: bf16-mode loss after N AdamW steps within 1% of the CPU reference.

GPU: EsmForMaskedLM in bf16 (production kernels, one CUDA graph per step).  CPU: the numpy oracle
(fp32 master weights, fp32 math) -- the reference semantics.  Both start from the same init, see the
same batches and the same MLM masks (the device masking kernel is bit-exact with the oracle), and
use the same AdamW hyper-parameters and lr schedule.

    python scripts/loss_trajectory.py --steps 200 --config 8m --batch 8 --seq 512
    python scripts/loss_trajectory.py --steps 200 --config geneformer-small --batch 4 --seq 256
(geneformer-small: the full 25,426-token Geneformer vocabulary and head, a 4-layer H=256 encoder, batches of
rank-value tokens from synthetic cells, Geneformer masking.)  Writes a JSON summary (both loss curves) to
gpurun_out/loss_trajectory.json.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import esm2_oracle as O  # noqa: E402
from paper_2411_10548_b200 import preset  # noqa: E402
from paper_2411_10548_b200.data import synthetic_batch  # noqa: E402
from paper_2411_10548_b200.model import EsmForMaskedLM, init_params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--config", default="8m")
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--seq", type=int, default=512)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "loss_trajectory.json"))
    a = ap.parse_args()
    gene = a.config == "geneformer-small"
    if gene:
        from paper_2411_10548_b200.config import geneformer_config
        cfg = geneformer_config(hidden_size=256, num_hidden_layers=4, num_attention_heads=4, intermediate_size=1024)
    else:
        cfg = preset(a.config)
    ocfg = O.OracleConfig(vocab_size=cfg.vocab_size, hidden_size=cfg.hidden_size,
                          num_hidden_layers=cfg.num_hidden_layers, num_attention_heads=cfg.num_attention_heads,
                          intermediate_size=cfg.intermediate_size, token_dropout=cfg.token_dropout,
                          mask_token_id=cfg.mask_token_id, pad_token_id=cfg.pad_token_id)
    mk = dict(eligible=cfg.mlm_eligible, mask_id=cfg.mask_token_id, random_range=cfg.mlm_random)
    if gene:  # batches of rank-value tokens from synthetic cells (oracle tokenizer; rows of varying length)
        import rank_oracle as R
        from paper_2411_10548_b200.data import gene_medians, synthetic_expression_csr
        n_genes = cfg.vocab_size - 2
        ip, cols, vals = synthetic_expression_csr(a.batch * 64, n_genes, seed=5, nnz=(a.seq // 2, 2 * a.seq))
        med = gene_medians(ip, cols, vals, n_genes)

        def batch_at(step):
            rows = [(step * a.batch + r) % (a.batch * 64) for r in range(a.batch)]
            return R.rank_encode_batch(ip, cols, vals, med, rows, a.seq, a.seq)
    else:
        def batch_at(step):
            return synthetic_batch(a.batch, a.seq, seed=10_000 + step)
    params = init_params(cfg, seed=1)
    adam = dict(beta1=0.9, beta2=0.98, eps=1e-8, weight_decay=0.01)
    tr = O.OracleTrainer(ocfg, params, lr=a.lr, dtype=np.float32, **adam)
    m = EsmForMaskedLM(cfg, dtype="bf16", device="cuda", params=params, lr=a.lr, betas=(0.9, 0.98), eps=1e-8,
                       weight_decay=0.01)
    ws = m.workspace(a.batch, a.seq)
    warm = max(1, a.steps // 10)

    def lr_at(step):  # linear warm-up then constant
        return a.lr * min(1.0, step / warm)

    gpu, cpu = [], []
    t0 = time.time()
    graph = False
    for step in range(1, a.steps + 1):
        ids, am = batch_at(step)
        inp, lab = O.mlm_mask(ids, seed=3, stream=step, **mk)
        lo = tr.step(inp, am, lab, lr=lr_at(step))
        ws.ids.copy_(torch.from_numpy(ids))
        ws.am.copy_(torch.from_numpy(am))
        m.mlm_mask(ws.ids, seed=3, stream_id=step, ws=ws)
        if not graph:
            m.capture(ws)
            graph = True
        lg = float(m.graph_step(lr=lr_at(step)).item())
        gpu.append(lg)
        cpu.append(float(lo))
        if step % 10 == 0 or step == 1:
            print(f"step {step:4d}  gpu(bf16) {lg:.5f}  cpu(fp32) {lo:.5f}  rel {abs(lg - lo) / lo:.2e}  "
                  f"[{time.time() - t0:.0f}s]", flush=True)
    # compare the smoothed final loss (mean of the last 10 steps) and the final step
    fin_g, fin_c = float(np.mean(gpu[-10:])), float(np.mean(cpu[-10:]))
    rel_final = abs(gpu[-1] - cpu[-1]) / cpu[-1]
    rel_mean = abs(fin_g - fin_c) / fin_c
    ok = rel_final < 0.01
    res = dict(config=a.config, batch=a.batch, seq=a.seq, steps=a.steps, lr=a.lr, gpu=gpu, cpu=cpu,
               final_rel_err=rel_final, last10_rel_err=rel_mean, passed=ok, cpu_cores=os.cpu_count())
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f)
    print(f"FINAL step {a.steps}: gpu {gpu[-1]:.5f} cpu {cpu[-1]:.5f} rel {rel_final:.3e}; last-10 mean rel "
          f"{rel_mean:.3e} -> {'PASSED' if ok else 'FAILED'} (< 1%)")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
