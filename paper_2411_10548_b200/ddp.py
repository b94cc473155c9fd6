"""Data-parallel gradient exchange: bucketed collectives over the flat gradient buffer,
overlapped with the backward, plus the global masked-token count (loss normaliser).

Parameter groups are laid out in backward-completion order (model.param_groups), so a bucket is a contiguous
slice of ``store.g32``.  The model calls ``ready(group_key)`` as soon as all groups up to that key hold final
gradients; every bucket fully covered is launched right away on a dedicated communication stream while the
compute stream continues with the next layer's backward.  Two modes:

* ``shard_optimizer=False`` (DDP): in-place all-reduce of the bucket; the model's AdamW for the bucket
  (``on_bucket``) follows on the communication stream.
* ``shard_optimizer=True`` (ZeRO-1, the comparison point of PAPER.md:86-88): the bucket is reduce-scattered,
  each rank runs AdamW only on its 1/N slice (its optimizer shard) and all-gathers the updated bf16 shadow slice
  (the GEMM operands).  The fp32 master stays sharded: only the 1-D parameters the kernels read in fp32 (biases,
  LayerNorm) are re-synchronised, with one small all-reduce of their owner-masked values after the last bucket
  (``master="vectors"``, the default with a bf16 shadow; ``master="full"`` all-gathers the whole fp32 master
  slice of every bucket as well).  AdamW work and HBM traffic per GPU drop by N, and the bytes on the wire are
  those of a reduce-scatter plus a bf16 all-gather (3/4 of an fp32 all-reduce; 1/2 with bf16 buckets).
  ``gather_master()`` brings every rank's full fp32 master up to date (checkpoints).

``grad_dtype="bf16"`` casts each bucket to bf16 before the collective (half the NVLink bytes) and the
optimizer reads the bf16 sums (``esm_adamw_bf16g``).

Collectives go through the library's own NCCL communicator (``esm_comm_*`` in the C ABI, enqueued on our
streams, so the whole DDP step can be captured in one CUDA graph); torch.distributed only carries the
rendezvous (the NCCL unique id).  On CPU tensors (the gloo tests) the same bucket logic runs on
torch.distributed collectives.
"""
from __future__ import annotations

import ctypes
import os

import torch
import torch.distributed as dist

from . import _lib

ALIGN = 256  # elements (model.ALIGN): AdamW decay-mask chunk; every shard slice starts on a chunk


class NcclComm:
    """The library's NCCL communicator (esm_comm_*): rank 0 creates the unique id, torch.distributed
    broadcasts it, every rank initialises its communicator.  In-place SUM collectives on a given stream."""

    def __init__(self, group=None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        lib = _lib.load()
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _lib.check(lib.esm_comm_unique_id(uid), "esm_comm_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        handle = ctypes.c_void_p()
        _lib.check(lib.esm_comm_init(uid, self.rank, self.world, ctypes.byref(handle)), "esm_comm_init")
        self.handle = handle

    @staticmethod
    def _dt(t):
        return {torch.float32: _lib.ESM_F32, torch.bfloat16: _lib.ESM_BF16, torch.int32: _lib.ESM_I32}[t.dtype]

    def allreduce(self, t, stream):
        _lib.call("esm_comm_allreduce", self.handle, t.data_ptr(), t.numel(), self._dt(t), stream)

    def reduce_scatter(self, t, stream):
        _lib.call("esm_comm_reduce_scatter", self.handle, t.data_ptr(), t.numel(), self._dt(t), stream)

    def allgather(self, t, stream):
        _lib.call("esm_comm_allgather", self.handle, t.data_ptr(), t.numel(), self._dt(t), stream)

    def close(self):
        if self.handle:
            _lib.load().esm_comm_destroy(self.handle)
            self.handle = None


class TorchDistComm:
    """The same in-place collectives on torch.distributed (gloo on CPU tensors: host-logic tests)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allreduce(self, t, stream=None):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def reduce_scatter(self, t, stream=None):
        s = t.clone()
        dist.all_reduce(s, op=dist.ReduceOp.SUM, group=self.group)
        n = t.numel() // self.world
        t[self.rank * n:(self.rank + 1) * n].copy_(s[self.rank * n:(self.rank + 1) * n])

    def allgather(self, t, stream=None):
        n = t.numel() // self.world
        parts = [torch.empty(n, dtype=t.dtype) for _ in range(self.world)]
        dist.all_gather(parts, t[self.rank * n:(self.rank + 1) * n].clone(), group=self.group)
        for r, p in enumerate(parts):
            t[r * n:(r + 1) * n].copy_(p)

    def close(self):
        pass


class GradAllReducer:
    def __init__(self, store, bucket_bytes: int | None = None, group=None, grad_dtype: str = "fp32",
                 shard_optimizer: bool = False, comm=None, master: str = "vectors"):
        if bucket_bytes is None:  # ESM_BUCKET_MB, default 256 MB: fewer, longer collectives interrupt the persistent
            # compute kernels less often (650M at N = 4: 90.6 ms/step vs 92.0 with 64 MB, 92.6 with 16 MB)
            bucket_bytes = int(float(os.environ.get("ESM_BUCKET_MB", "256")) * (1 << 20))
        if grad_dtype not in ("fp32", "bf16"):
            raise ValueError("grad_dtype must be 'fp32' or 'bf16'")
        if master not in ("vectors", "full"):
            raise ValueError("master must be 'vectors' or 'full'")
        self.store = store
        self.group = group
        self.cuda = store.g32.is_cuda
        self.comm = comm or (NcclComm(group) if self.cuda else TorchDistComm(group))
        self.world, self.rank = self.comm.world, self.comm.rank
        self.bf16 = grad_dtype == "bf16"
        self.shard = shard_optimizer
        unit = ALIGN * self.world  # every bucket splits into `world` slices of whole AdamW chunks
        if store.numel % unit:
            raise ValueError(f"parameter buffer ({store.numel}) is not a multiple of {unit} elements")
        keys = [k for k, _ in store.groups]
        esz = 2 if self.bf16 else 4
        self.bucket_ends = []  # element offsets (exclusive) of bucket ends, at group ends rounded up to `unit`
        start = 0
        for k in keys:
            end = min(store.numel, (store.group_range[k][1] + unit - 1) // unit * unit)
            if (end - start) * esz >= bucket_bytes:
                self.bucket_ends.append(end)
                start = end
        if not self.bucket_ends or self.bucket_ends[-1] != store.numel:
            self.bucket_ends.append(store.numel)
        self.unit = unit
        self.key_end = {k: store.group_range[k][1] for k in keys}
        # high priority: the persistent GEMM / attention kernels occupy every SM, so the collectives (and the
        # bucket's optimizer) get the SMs at the next kernel boundary instead of queueing behind more compute
        self.stream = torch.cuda.Stream(store.g32.device, priority=-1) if self.cuda else None
        self.g16 = torch.empty(store.numel, dtype=torch.bfloat16, device=store.g32.device) if self.bf16 else None
        self._next = 0
        self._start = 0
        # on_bucket(a, b, stream, grad): the optimizer for flat elements [a, b) -- the whole bucket (DDP) or this
        # rank's slice of it (sharded) -- with `grad` the reduced gradients of [a, b) (fp32, or bf16 buckets)
        self.on_bucket = None
        # sharded fp32 master (ZeRO-1 with a bf16 shadow): flat indices of the 1-D parameters read in fp32 by the
        # kernels, and this rank's ownership mask over them
        self.full_master = master == "full" or store.p16 is None or not self.shard
        self.vec_idx = self.vec_own = self.vec = None
        if not self.full_master:
            idx = [torch.arange(sl.offset, sl.offset + sl.numel) for sl in store.slots.values() if len(sl.shape) == 1]
            idx = torch.cat(idx)
            own = torch.zeros(store.numel, dtype=torch.bool)
            a = 0
            for b in self.bucket_ends:
                oa, ob = self.owned(a, b)
                own[oa:ob] = True
                a = b
            dev = store.p32.device
            self.vec_idx = idx.to(dev)
            self.vec_own = own[idx].to(torch.float32).to(dev)
            self.vec = torch.empty(idx.numel(), dtype=torch.float32, device=dev)

    # ---------------------------------------------------------------- loss normaliser (compute stream)
    def _cur(self):
        return torch.cuda.current_stream(self.store.g32.device).cuda_stream if self.cuda else None

    def reduce_count(self, n_labels: torch.Tensor):
        self.comm.allreduce(n_labels, self._cur())

    def reduce_loss(self, loss_sum: torch.Tensor):
        self.comm.allreduce(loss_sum, self._cur())

    # ---------------------------------------------------------------- buckets
    def owned(self, a: int, b: int):
        """This rank's optimizer slice of bucket [a, b) (sharded mode)."""
        n = (b - a) // self.world
        return a + self.rank * n, a + (self.rank + 1) * n

    def begin_backward(self):
        self._next = 0
        self._start = 0

    def _cast(self, a, b, st, to_bf16: bool):
        if self.cuda:
            if to_bf16:
                _lib.call("esm_cast_f32_bf16", self.store.g32[a:].data_ptr(), self.g16[a:].data_ptr(), b - a, st)
            else:
                _lib.call("esm_cast_bf16_f32", self.g16[a:].data_ptr(), self.store.g32[a:].data_ptr(), b - a, st)
        elif to_bf16:
            self.g16[a:b].copy_(self.store.g32[a:b])
        else:
            self.store.g32[a:b].copy_(self.g16[a:b])

    def _launch(self, end):
        a, b = self._start, end
        P = self.store
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(P.g32.device))
            self.stream.wait_event(ev)
            st = self.stream.cuda_stream
            ctx = torch.cuda.stream(self.stream)
        else:
            st, ctx = None, _Null()
        with ctx:
            if self.bf16:
                self._cast(a, b, st, True)
            gbuf = self.g16 if self.bf16 else P.g32
            if self.shard:
                self.comm.reduce_scatter(gbuf[a:b], st)
                oa, ob = self.owned(a, b)
                if self.on_bucket is not None:
                    self.on_bucket(oa, ob, self.stream, gbuf[oa:ob])
                    if self.full_master:
                        self.comm.allgather(P.p32[a:b], st)
                    if P.p16 is not None:
                        self.comm.allgather(P.p16[a:b], st)
                elif self.bf16:
                    self._cast(oa, ob, st, False)
            else:
                self.comm.allreduce(gbuf[a:b], st)
                if self.on_bucket is not None:
                    self.on_bucket(a, b, self.stream, gbuf[a:b])
                elif self.bf16:
                    self._cast(a, b, st, False)
        self._start = end

    def ready(self, key: str):
        done = (self.key_end[key] + ALIGN - 1) // ALIGN * ALIGN
        while self._next < len(self.bucket_ends) and self.bucket_ends[self._next] <= done:
            self._launch(self.bucket_ends[self._next])
            self._next += 1

    def end_backward(self):
        updated = self.on_bucket is not None
        while self._next < len(self.bucket_ends):
            self._launch(self.bucket_ends[self._next])
            self._next += 1
        if updated and not self.full_master:
            with (torch.cuda.stream(self.stream) if self.cuda else _Null()):
                self._sync_vectors(self.stream.cuda_stream if self.cuda else None)
        if self.cuda:
            torch.cuda.current_stream(self.store.g32.device).wait_stream(self.stream)

    def _sync_vectors(self, st):
        """Owner-masked all-reduce of the 1-D fp32 parameters (each element has exactly one owner rank)."""
        P = self.store
        torch.index_select(P.p32, 0, self.vec_idx, out=self.vec)
        self.vec.mul_(self.vec_own)
        self.comm.allreduce(self.vec, st)
        P.p32.index_copy_(0, self.vec_idx, self.vec)

    def gather_master(self):
        """All-gather every bucket's fp32 master slice (sharded mode keeps only the owned slices current)."""
        if self.full_master:
            return
        st = self.stream.cuda_stream if self.cuda else None
        with (torch.cuda.stream(self.stream) if self.cuda else _Null()):
            if self.cuda:
                self.stream.wait_stream(torch.cuda.current_stream(self.store.g32.device))
            a = 0
            for b in self.bucket_ends:
                self.comm.allgather(self.store.p32[a:b], st)
                a = b
        if self.cuda:
            torch.cuda.current_stream(self.store.g32.device).wait_stream(self.stream)


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
