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


def collate(token_lists, seq_len: int | None = None, pad_to: int = 8, pad_id: int = PAD):
    """Right-pad a list of token sequences to a common length (multiple of ``pad_to``).
    pad_id: 1 for the ESM-2 alphabet, 0 for Geneformer rank tokens (tokenizer.py:16)."""
    n = max(len(t) for t in token_lists)
    if seq_len is None:
        seq_len = (n + pad_to - 1) // pad_to * pad_to
    ids = np.full((len(token_lists), seq_len), pad_id, dtype=np.int32)
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


# ----------------------------------------------------------------------------------------------
# Geneformer feed: CSR expression rows -> rank-value tokens on the GPU (esm_rank_encode)
# reference: pkg/src/densefeed/tokenizer.py (GeneStats :29-40, compute_gene_stats :52-65,
# rank_encode :68-83; PAD=0, MASK=1, TOKEN_OFFSET=2 :16-18)
# ----------------------------------------------------------------------------------------------
GF_PAD, GF_MASK, GF_OFFSET = 0, 1, 2


def synthetic_expression_csr(n_rows: int, n_genes: int, seed: int, nnz=(500, 4000)):
    """Random single-cell expression rows: nnz/row uniform in ``nnz``, distinct
    ascending gene columns, values uniform in [0.5, 10) (pkg/tests/conftest.py:16-26 value range).
    Returns CSR (indptr int64 [R+1], cols int64, vals float32)."""
    rng = np.random.default_rng(seed)
    k = rng.integers(nnz[0], nnz[1] + 1, size=n_rows)
    indptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.cumsum(k, out=indptr[1:])
    cols = np.empty(int(indptr[-1]), dtype=np.int64)
    for r in range(n_rows):
        cols[indptr[r]:indptr[r + 1]] = np.sort(rng.choice(n_genes, size=int(k[r]), replace=False))
    vals = rng.uniform(0.5, 10.0, size=cols.size).astype(np.float32)
    return indptr, cols, vals


def gene_medians(indptr, cols, vals, n_genes: int) -> np.ndarray:
    """Per-gene median of the non-zero values, 1.0 for unseen genes (compute_gene_stats semantics,
    tokenizer.py:52-65) -- the one-off corpus statistic the tokenizer normalises by."""
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float32)
    nz = vals != 0
    cols, vals = cols[nz], vals[nz].astype(np.float64)
    med = np.ones(n_genes, dtype=np.float32)
    if cols.size:
        order = np.lexsort((vals, cols))
        c, v = cols[order], vals[order]
        counts = np.bincount(c, minlength=n_genes)
        start = np.zeros(n_genes + 1, dtype=np.int64)
        np.cumsum(counts, out=start[1:])
        g = np.flatnonzero(counts)
        lo = start[g] + (counts[g] - 1) // 2
        hi = start[g] + counts[g] // 2
        med[g] = (0.5 * (v[lo] + v[hi])).astype(np.float32)
    if med.size and float(med.min()) <= 0.0:
        raise ValueError("gene medians must be strictly positive")
    return med


class RankEncoder:
    """Geneformer rank-value tokeniser on the GPU: a batch of CSR rows -> padded ids / attention mask.

    Same output as the reference's ``rank_encode`` per row (bit-exact; tests/test_gpu_geneformer.py),
    already collated into the [B, S] int32 tensors the train step consumes (PAD 0 past each length).
    """

    STAGE = 16384  # shared-memory staging capacity of the sort (one CTA per row); longer rows stream through it

    def __init__(self, medians: np.ndarray, device=None):
        _lib.load()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        med = np.ascontiguousarray(medians, dtype=np.float32)
        if med.size and float(med.min()) <= 0.0:
            raise ValueError("gene medians must be strictly positive")
        self.n_genes = int(med.size)
        self.medians = torch.from_numpy(med).to(self.device)
        self.status = torch.zeros(1, dtype=torch.int32, device=self.device)

    def stage(self, indptr, cols, vals, rows):
        """Compact the selected rows into one pinned CSR block and copy it to the device."""
        rows = np.asarray(rows, dtype=np.int64)
        lo, hi = indptr[rows], indptr[rows + 1]
        lens = (hi - lo).astype(np.int64)
        ip = np.zeros(rows.size + 1, dtype=np.int64)
        np.cumsum(lens, out=ip[1:])
        idx = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in zip(lo, hi)]) if rows.size else \
            np.empty(0, np.int64)
        c = np.asarray(cols)[idx].astype(np.int64, copy=False)
        v = np.asarray(vals)[idx].astype(np.float32, copy=False)
        dev = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory().to(self.device, non_blocking=True)
               for a in (ip, c, v)]
        return dev, int(lens.max()) if lens.size else 0

    def encode_device(self, d_indptr, d_cols, d_vals, n_rows: int, max_nnz: int, seq_len: int,
                      max_len: int | None = None, ids=None, am=None, lengths=None, stream=None):
        """Kernel launch on device CSR (rows 0..n_rows-1); writes ids/am (allocated if None)."""
        ml = seq_len if max_len is None else int(max_len)
        if ml < 0:
            raise ValueError("max_len must be >= 0")
        if max_nnz > self.STAGE and min(ml, seq_len) > self.STAGE // 2:
            raise ValueError(f"rows longer than {self.STAGE} entries need max_len <= {self.STAGE // 2} "
                             "(streaming top-k of the device tokenizer)")
        if ids is None:
            ids = torch.empty(n_rows, seq_len, dtype=torch.int32, device=self.device)
        if am is None:
            am = torch.empty(n_rows, seq_len, dtype=torch.int32, device=self.device)
        st = stream if stream is not None else torch.cuda.current_stream(self.device).cuda_stream
        self.status.zero_()
        _lib.call("esm_rank_encode", d_indptr.data_ptr(), d_cols.data_ptr() if d_cols.numel() else None,
                  d_vals.data_ptr() if d_vals.numel() else None, self.medians.data_ptr(), self.n_genes, None, n_rows,
                  ml, seq_len, ids.data_ptr(), am.data_ptr(), lengths.data_ptr() if lengths is not None else None,
                  self.status.data_ptr(), max(1, max_nnz), st)
        return ids, am

    def check(self):
        """Raise like the reference (ValidationError) if the last launch saw a bad column."""
        s = int(self.status.item())
        if s == 1:
            raise ValueError("row column index exceeds stats.n_cols")
        if s == 2:
            raise ValueError("row longer than the device tokenizer staging capacity with max_len > capacity / 2")

    def __call__(self, indptr, cols, vals, rows, seq_len: int, max_len: int | None = None, check: bool = True):
        (d_ip, d_c, d_v), max_nnz = self.stage(indptr, cols, vals, rows)
        lengths = torch.empty(len(rows), dtype=torch.int32, device=self.device)
        ids, am = self.encode_device(d_ip, d_c, d_v, len(rows), max_nnz, seq_len, max_len, lengths=lengths)
        if check:
            self.check()
        return ids, am, lengths
