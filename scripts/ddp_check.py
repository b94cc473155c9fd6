"""Data-parallel correctness on N GPUs (launch with torchrun; NCCL through the library's esm_comm_* ABI):

  1. N ranks each run the MLM step on 1/N of a global batch (bucketed gradient all-reduce overlapped with the
     backward, global masked-token normalisation); rank 0 also runs the whole global batch on one GPU.
     Loss and gradients must agree (same math, different reduction order).
  2. Two full train steps (fwd + bwd + AdamW) in every data-parallel mode -- DDP (fp32 buckets), ZeRO-1 sharded
     optimizer, bf16 gradient buckets, both -- vs the single-GPU steps on the concatenated batch: the parameter
     updates must agree.
  3. The DDP step captured in one CUDA graph (NCCL collectives inside) replays to the eager step's parameters.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 scripts/ddp_check.py
Writes gpurun_out/ddp_check_n<N>.json (rank 0).
"""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_10548_b200 import preset  # noqa: E402
from paper_2411_10548_b200.data import synthetic_batch  # noqa: E402
from paper_2411_10548_b200.ddp import GradAllReducer  # noqa: E402
from paper_2411_10548_b200.model import EsmForMaskedLM  # noqa: E402

B, S, SEED = 4, 256, 7


def stage(m, ids_rank, rank, step):
    ws = m.workspace(*ids_rank.shape)
    ws.am.fill_(1)
    m.mlm_mask(ids_rank, seed=SEED, stream_id=1000 * step + rank, ws=ws)
    return ws


def single_gpu_reference(cfg, dtype, ids_all, world, dev, steps):
    """The global batch on one GPU with the per-rank masks concatenated; returns (losses, grads, params)."""
    ref = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3)
    out = []
    for step in range(steps):
        inp, lab = [], []
        for r in range(world):
            tmp = ref.workspace(B, S)
            i_, l_ = ref.mlm_mask(ids_all[step][r * B:(r + 1) * B], seed=SEED, stream_id=1000 * step + r, ws=tmp)
            inp.append(i_.clone())
            lab.append(l_.clone())
        wr = ref.workspace(B * world, S)
        wr.input_ids.copy_(torch.cat(inp))
        wr.labels.copy_(torch.cat(lab))
        wr.am.fill_(1)
        wr.n_labels.copy_((wr.labels != -100).sum().reshape(1).int())
        loss = float(ref.step(wr).item())
        out.append((loss, ref.store.g32.clone(), ref.store.p32.clone()))
    return out


def rel(a, b):
    return ((a - b).norm() / b.norm().clamp_min(1e-30)).item()


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = preset(os.environ.get("DDP_CONFIG", "8m"))
    ids_all = [torch.from_numpy(synthetic_batch(B * world, S, seed=42 + s)[0]).to(dev) for s in range(2)]
    report, ok = [], True
    for dtype in ("fp32", "bf16"):
        ref = single_gpu_reference(cfg, dtype, ids_all, world, dev, 2) if rank == 0 else None
        p0 = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3).store.p32.clone()
        modes = [("ddp", False, "fp32", "vectors"), ("zero1", True, "fp32", "vectors"),
                 ("ddp_bf16grad", False, "bf16", "vectors"), ("zero1_bf16grad", True, "bf16", "vectors"),
                 ("zero1_fullmaster", True, "fp32", "full")]
        for name, shard, gdt, master in modes:
            m = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3)
            m.comm = GradAllReducer(m.store, bucket_bytes=4 << 20, shard_optimizer=shard, grad_dtype=gdt,
                                    master=master)
            losses = []
            for step in range(2):
                ws = stage(m, ids_all[step][rank * B:(rank + 1) * B], rank, step)
                losses.append(float(m.step(ws).item()))
            m.comm.gather_master()  # sharded fp32 master -> full (the check reads every parameter)
            if rank == 0:
                dp = m.store.p32 - p0
                dref = ref[1][2] - p0
                e_upd = rel(dp, dref)
                e_loss = max(abs(a - b[0]) / b[0] for a, b in zip(losses, ref))
                tol_upd = (1e-3 if gdt == "fp32" else 2e-2) if dtype == "fp32" else 3e-2
                good = e_loss < (1e-5 if dtype == "fp32" else 1e-2) and e_upd < tol_upd
                ok &= good
                report.append({"dtype": dtype, "mode": name, "loss_rel_err": e_loss, "update_rel_err": e_upd,
                               "ok": good})
                print(f"[{dtype}] {name:15s} loss rel {e_loss:.2e}  2-step update rel {e_upd:.2e} "
                      f"{'OK' if good else 'FAIL'}", flush=True)
            del m
            dist.barrier()
        # gradients of one forward_backward (fp32 buckets) vs the single GPU
        m = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3)
        m.comm = GradAllReducer(m.store, bucket_bytes=4 << 20)
        ws = stage(m, ids_all[0][rank * B:(rank + 1) * B], rank, 0)
        m.forward_backward(ws)
        g = m.store.g32.clone()
        if rank == 0:
            r0 = EsmForMaskedLM(cfg, dtype=dtype, device=dev, seed=3)
            wr = r0.workspace(B * world, S)
            inp, lab = [], []
            for r in range(world):
                tmp = r0.workspace(B, S)
                i_, l_ = r0.mlm_mask(ids_all[0][r * B:(r + 1) * B], seed=SEED, stream_id=r, ws=tmp)
                inp.append(i_.clone())
                lab.append(l_.clone())
            wr = r0.workspace(B * world, S)
            wr.input_ids.copy_(torch.cat(inp))
            wr.labels.copy_(torch.cat(lab))
            wr.am.fill_(1)
            wr.n_labels.copy_((wr.labels != -100).sum().reshape(1).int())
            r0.forward_backward(wr)
            e = rel(g, r0.store.g32)
            good = e < (1e-5 if dtype == "fp32" else 2e-2)
            ok &= good
            report.append({"dtype": dtype, "mode": "ddp_grads", "grad_rel_err": e, "ok": good})
            print(f"[{dtype}] ddp gradients vs single GPU: rel {e:.2e} {'OK' if good else 'FAIL'}", flush=True)
        dist.barrier()
    # CUDA-graph-captured DDP step (NCCL collectives in the graph) == eager step
    for shard in (False, True):
        pa = []
        for use_graph in (False, True):
            m = EsmForMaskedLM(cfg, dtype="bf16", device=dev, seed=3)
            m.comm = GradAllReducer(m.store, bucket_bytes=4 << 20, shard_optimizer=shard)
            for step in range(3):
                ws = stage(m, ids_all[step % 2][rank * B:(rank + 1) * B], rank, step)
                if use_graph:
                    if step == 0:
                        m.capture(ws)
                    m.graph_step()
                else:
                    m.step(ws)
            m.comm.gather_master()
            torch.cuda.synchronize()
            pa.append(m.store.p32.clone())
        e = rel(pa[1] - p0, pa[0] - p0) if pa[0].shape == p0.shape else 1.0
        good = e < 1e-2
        ok &= good
        if rank == 0:
            report.append({"mode": "graph_vs_eager" + ("_zero1" if shard else ""), "update_rel_err": e, "ok": good})
            print(f"[bf16] graph-captured {'zero1' if shard else 'ddp'} step vs eager: update rel {e:.2e} "
                  f"{'OK' if good else 'FAIL'}", flush=True)
        dist.barrier()
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"ddp_check_n{world}.json"), "w") as f:
            json.dump({"world": world, "config": os.environ.get("DDP_CONFIG", "8m"), "checks": report,
                       "passed": bool(flag.item())}, f, indent=1)
        print("DDP CHECK", "PASSED" if flag.item() else "FAILED", flush=True)
        sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
