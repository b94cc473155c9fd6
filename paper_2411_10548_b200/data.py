"""Data feed for the train step: synthetic protein batches, tokenisation, collation.

The reference's own data seams (densefeed, /root/reference/pkg) produce token lists and
index batches (``BoundDataset[i] -> (tokens, metadata)``, ``batches(...) -> list[int]``;
pkg/bindings/src/densefeed_bindings/__init__.py:45-95).  ``collate`` turns such a batch
into the padded int32 [B, S] ids + attention mask the step consumes.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

CLS, PAD, EOS, UNK, MASK = 0, 1, 2, 3, 32
AA_FIRST, AA_COUNT = 4, 20


def tokenize(seq: str) -> np.ndarray:
    """ESM-2 alphabet tokenizer (native, esm_tokenize): <cls> residues <eos>; unknown -> <unk>."""
    lib = _lib.load()
    raw = seq.encode("ascii", errors="replace")
    out = np.empty(len(raw) + 2, dtype=np.int32)
    n = lib.esm_tokenize(raw, len(raw), out.ctypes.data_as(ctypes.c_void_p), out.size)
    if n < 0:
        raise _lib.EsmKernelError("esm_tokenize: buffer too small")
    return out[:n]


def synthetic_batch(batch: int, seq_len: int, seed: int):
    """Full-length synthetic proteins: <cls> + AAs uniform over ids 4..23 + <eos>."""
    rng = np.random.default_rng(seed)
    ids = rng.integers(AA_FIRST, AA_FIRST + AA_COUNT, size=(batch, seq_len), dtype=np.int64).astype(np.int32)
    ids[:, 0] = CLS
    ids[:, -1] = EOS
    return ids, np.ones((batch, seq_len), dtype=np.int32)


def collate(token_lists, seq_len: int | None = None, pad_to: int = 8):
    """Right-pad a list of token sequences to a common length (multiple of ``pad_to``)."""
    n = max(len(t) for t in token_lists)
    if seq_len is None:
        seq_len = (n + pad_to - 1) // pad_to * pad_to
    ids = np.full((len(token_lists), seq_len), PAD, dtype=np.int32)
    am = np.zeros_like(ids)
    for i, t in enumerate(token_lists):
        k = min(len(t), seq_len)
        ids[i, :k] = np.asarray(t[:k], dtype=np.int32)
        am[i, :k] = 1
    return ids, am


def to_device(a: np.ndarray, device, pinned: bool = True) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a))
    if pinned:
        t = t.pin_memory()
    return t.to(device, non_blocking=True)
