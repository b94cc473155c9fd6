"""Adapters that plug the B200 train step into the reference's own seams.

The reference (``densefeed``) owns the layer around the hot path:

* ``densefeed.sizing.collect_peak_alloc(samples, workload, feature_fn, meter)``
  (pkg/src/densefeed/sizing.py:76-100) -- the only place a training workload is invoked and
  metered.  ``make_workload`` returns the ``workload`` callable (one MLM train step on the GPU)
  and ``CudaPeakMeter`` implements the ``ResourceMeter`` protocol ``reset()/peak()``
  (sizing.py:24-29) with CUDA peak-allocation statistics.  Exceptions raised by the step
  (e.g. CUDA OOM) propagate, so ``collect_peak_alloc`` records the sample as failed
  (sizing.py:96-98) -- the OOM analogue the reference expects.
* ``densefeed_bindings.batches(...) -> Iterator[list[int]]`` and ``BoundDataset[i] -> (tokens,
  metadata)`` (pkg/bindings/src/densefeed_bindings/__init__.py:45-95) -- ``collate_indices``
  turns one index batch into the padded int32 ``[B, S]`` ids + attention mask the step consumes.
* ``densefeed.shards`` (pkg/src/densefeed/shards.py:160-191, 255-276) -- tar-shard streaming.
  ``shard_tokens`` decodes a ``Sample``'s token payload and ``shard_collate`` is the ``collate`` for
  ``batch_stage(size, collate=...)``, so ``compose(stream_samples(shards.subset(rank, world)), [...])``
  yields the padded ``[B, S]`` batches of this rank.
* ``length_features`` gives the ``[L, L^2]`` cost features (the corpus.py:57-60 pattern) so
  ``fit_cost_model`` can model attention's quadratic memory.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch

from .data import collate


class CudaPeakMeter:
    """ResourceMeter over CUDA allocator statistics: peak bytes allocated since ``reset()``.

    relative=False: the absolute peak (resident model state included).  relative=True: the peak minus what was
    allocated at ``reset()`` -- the memory one sample adds on top of the resident model (parameters, gradients,
    Adam moments), which is what a per-sample cost model summed over a batch must predict
    (``SizeAwareBatcher`` adds per-sample costs, sizing.py:203-219)."""

    def __init__(self, device=None, relative: bool = False):
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.relative = relative
        self._base = 0

    def reset(self) -> None:
        torch.cuda.synchronize(self.device)
        torch.cuda.reset_peak_memory_stats(self.device)
        self._base = torch.cuda.memory_allocated(self.device) if self.relative else 0

    def peak(self) -> float:
        torch.cuda.synchronize(self.device)
        return float(torch.cuda.max_memory_allocated(self.device) - self._base)


def length_features(sample) -> np.ndarray:
    """Cost features of a sample (one token sequence, or a batch of them): [sum L, sum L^2]."""
    if len(sample) and not isinstance(sample[0], (int, np.integer)):
        lens = np.array([len(s) for s in sample], dtype=np.float64)
    else:
        lens = np.array([len(sample)], dtype=np.float64)
    return np.array([lens.sum(), (lens * lens).sum()])


def collate_indices(dataset, indices: Sequence[int], seq_len: int | None = None, pad_to: int = 8,
                    pad_id: int = 1):
    """One ``batches()`` index list -> (ids int32 [B, S], attention_mask int32 [B, S]).
    pad_id: 1 for ESM-2 token lists, 0 for the bindings' Geneformer rank tokens (tokenizer.py:16)."""
    toks = [dataset[i][0] if isinstance(dataset[i], tuple) else dataset[i] for i in indices]
    return collate(toks, seq_len=seq_len, pad_to=pad_to, pad_id=pad_id)


def make_workload(model, seed: int = 0, pad_to: int = 8, lr: float | None = None, use_graph: bool = False,
                  release: bool = False) -> Callable:
    """``workload(sample)`` for ``collect_peak_alloc``: one full MLM train step (device masking,
    forward, backward, AdamW) on a sample = one token sequence or a list of them.  ``release=True`` frees the
    sample's activation workspace after the step, so a relative ``CudaPeakMeter`` sees exactly one sample's
    activation memory per record."""
    state = {"step": 0}

    def workload(sample):
        batch = sample if (len(sample) and not isinstance(sample[0], (int, np.integer))) else [sample]
        loss = model.train_step_tokens(batch, seed=seed, stream_id=state["step"], lr=lr, pad_to=pad_to,
                                       use_graph=use_graph)
        state["step"] += 1
        out = float(loss.item())
        if release:
            model.release_workspaces()
        return out

    return workload


def shard_tokens(sample, part: str = "tokens") -> np.ndarray:
    """Token ids of a shard ``Sample`` (``parts[part]`` = little-endian int32 or int64 bytes)."""
    raw = sample.parts[part]
    dt = "<i8" if part.endswith("64") else "<i4"
    return np.frombuffer(raw, dtype=dt).astype(np.int32)


def shard_collate(pad_to: int = 8, pad_id: int = 1, part: str = "tokens"):
    """``collate`` for the reference's ``batch_stage``: a window of Samples -> (ids, attention_mask)
    int32 [B, S], right padded (pad_id 1 for ESM-2, 0 for Geneformer rank tokens)."""
    def collate_fn(window):
        return collate([shard_tokens(x, part) for x in window], pad_to=pad_to, pad_id=pad_id)
    return collate_fn
