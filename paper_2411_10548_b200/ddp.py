"""Data-parallel gradient exchange: bucketed all-reduce of the flat fp32 gradient buffer,
overlapped with backward, plus the global masked-token count (loss normaliser).

Parameter groups are laid out in backward-completion order (model.param_groups), so a
bucket is a contiguous slice of ``store.g32``.  The model calls ``ready(group_key)`` as soon
as all groups up to that key are final; every bucket fully covered is launched right away
on a dedicated communication stream (NCCL over NVLink / NVSwitch through torch.distributed),
while the compute stream continues with the next layer's backward.  With ``on_bucket`` set (the
model's overlapped optimizer), the AdamW update of each bucket is issued on the communication stream
right behind its all-reduce, so the optimizer also overlaps the remaining backward.  ``end_backward``
makes the compute stream wait on the outstanding collectives (and updates).

Loss normalisation: the masked-token count is all-reduced before the loss kernel, every
rank scales its gradients by 1 / N_global, and buckets are SUM-reduced -- the result equals
the gradient of the mean loss over the concatenated global batch (one exchange step per
optimizer step).  Works with the gloo backend on CPU tensors for tests.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class GradAllReducer:
    def __init__(self, store, bucket_bytes: int = 64 << 20, group=None):
        self.store = store
        self.group = group
        self.world = dist.get_world_size(group)
        keys = [k for k, _ in store.groups]
        self.bucket_ends = []  # element offsets (exclusive) of bucket ends, at group boundaries
        start = 0
        for k in keys:
            a, b = store.group_range[k]
            end = (b + 255) // 256 * 256
            if (end - start) * 4 >= bucket_bytes:
                self.bucket_ends.append(end)
                start = end
        if not self.bucket_ends or self.bucket_ends[-1] != store.numel:
            self.bucket_ends.append(store.numel)
        self.key_end = {k: store.group_range[k][1] for k in keys}
        self.cuda = store.g32.is_cuda
        self.stream = torch.cuda.Stream(store.g32.device) if self.cuda else None
        self._works = []
        self._next = 0
        self._start = 0
        self.on_bucket = None  # callable(start, end, stream) run after a bucket's all-reduce

    # ---------------------------------------------------------------- loss normaliser
    def reduce_count(self, n_labels: torch.Tensor):
        dist.all_reduce(n_labels, op=dist.ReduceOp.SUM, group=self.group)

    def reduce_loss(self, loss_sum: torch.Tensor):
        dist.all_reduce(loss_sum, op=dist.ReduceOp.SUM, group=self.group)

    # ---------------------------------------------------------------- buckets
    def begin_backward(self):
        self._works = []
        self._next = 0
        self._start = 0

    def _launch(self, end):
        g = self.store.g32[self._start:end]
        if self.cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(g.device))
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(ev)
                w = dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
                if self.on_bucket is not None:
                    w.wait()  # the comm stream waits for the collective, then updates the bucket
                    self.on_bucket(self._start, end, self.stream)
                self._works.append(w)
        else:
            w = dist.all_reduce(g, op=dist.ReduceOp.SUM, group=self.group, async_op=True)
            if self.on_bucket is not None:
                w.wait()
                self.on_bucket(self._start, end, None)
            self._works.append(w)
        self._start = end

    def ready(self, key: str):
        done = self.key_end[key]
        while self._next < len(self.bucket_ends) and self.bucket_ends[self._next] <= ((done + 255) // 256 * 256):
            self._launch(self.bucket_ends[self._next])
            self._next += 1

    def end_backward(self):
        while self._next < len(self.bucket_ends):
            self._launch(self.bucket_ends[self._next])
            self._next += 1
        for w in self._works:
            w.wait()  # compute stream waits for the collective (NCCL) / completes (gloo)
        if self.cuda and self.on_bucket is not None:
            torch.cuda.current_stream(self.store.g32.device).wait_stream(self.stream)
        self._works = []
