"""Data-parallel correctness on N GPUs (launch with torchrun, NCCL):

  N ranks each run the MLM step on 1/N of a global batch with bucketed gradient all-reduce
  (overlapped with backward) and global masked-token normalisation; rank 0 also runs the
  whole global batch on one GPU in a separate model.  Gradients, loss and the updated
  parameters must agree (same math, different reduction order).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/ddp_check.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_10548_b200 import preset  # noqa: E402
from paper_2411_10548_b200.data import synthetic_batch  # noqa: E402
from paper_2411_10548_b200.ddp import GradAllReducer  # noqa: E402
from paper_2411_10548_b200.model import EsmForMaskedLM  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = preset(os.environ.get("DDP_CONFIG", "8m"))
    B, S = 4, 256
    ids_all, _ = synthetic_batch(B * world, S, seed=42)
    ok = True
    for dtype, tol in (("fp32", 1e-4), ("bf16", 2e-2)):
        m = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3)
        m.comm = GradAllReducer(m.store, bucket_bytes=4 << 20)
        ws = m.workspace(B, S)
        # masking stream ids index the global batch so the union equals the single-GPU masks
        mine = torch.from_numpy(ids_all[rank * B:(rank + 1) * B]).to(dev)
        m.mlm_mask(mine, seed=7, stream_id=rank, ws=ws)
        loss = float(m.forward_backward(ws).item())
        g_ddp = m.store.g32.clone()
        m.optimizer_step()
        p_ddp = m.store.p32.clone()
        # the same step with AdamW overlapped (per bucket, behind its all-reduce on the comm stream)
        m2 = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3)
        m2.comm = GradAllReducer(m2.store, bucket_bytes=4 << 20)
        ws2 = m2.workspace(B, S)
        m2.mlm_mask(mine, seed=7, stream_id=rank, ws=ws2)
        loss2 = float(m2.step(ws2).item())
        ferr = (m2.store.p32 - p_ddp).abs().max().item()
        fgood = ferr < 1e-6 and abs(loss2 - loss) <= 1e-6 * loss  # atomics order only
        ok &= fgood
        print(f"[{dtype}] rank {rank}: overlapped optimizer vs separate: max|dparam|={ferr:.1e} "
              f"loss {loss2:.6f}/{loss:.6f} {'OK' if fgood else 'FAIL'}", flush=True)
        if rank == 0:
            ref = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3)
            wr = ref.workspace(B * world, S)
            # same per-rank masks, concatenated
            inp, lab = [], []
            for r in range(world):
                x = torch.from_numpy(ids_all[r * B:(r + 1) * B]).to(dev)
                tmp = ref.workspace(B, S)
                i_, l_ = ref.mlm_mask(x, seed=7, stream_id=r, ws=tmp)
                inp.append(i_.clone())
                lab.append(l_.clone())
            wr = ref.workspace(B * world, S)
            wr.input_ids.copy_(torch.cat(inp))
            wr.labels.copy_(torch.cat(lab))
            wr.am.fill_(1)
            wr.n_labels.copy_((wr.labels != -100).sum().reshape(1).int())
            lref = float(ref.forward_backward(wr).item())
            g_ref = ref.store.g32
            err = ((g_ddp - g_ref).norm() / g_ref.norm()).item()
            ref.optimizer_step()
            perr = ((p_ddp - ref.store.p32).abs().max()).item()
            good = abs(loss - lref) / lref < tol and err < tol and perr < 1e-3
            ok &= good
            print(f"[{dtype}] world={world} loss ddp={loss:.6f} single={lref:.6f} grad_rel_err={err:.2e} "
                  f"max|dparam|={perr:.2e} {'OK' if good else 'FAIL'}", flush=True)
        dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print("DDP CHECK", "PASSED" if ok else "FAILED", flush=True)
        sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
