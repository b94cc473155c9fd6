"""CPU oracle for the Geneformer rank-value tokeniser -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this module, as the
checker; the product path is the esm_rank_encode kernel (paper_2411_10548_b200/csrc/rank_encode.cu).

Restates the reference's tokenizer (pkg/src/densefeed/tokenizer.py):
  * compute_gene_stats (:52-65): per-gene median of the non-zero values (fp64 median stored as fp32),
    1.0 for genes with no entries;
  * rank_encode (:68-83): score = val / median[col] in fp64, order by descending score with ties on
    ascending gene index, truncate to max_len, token = gene + TOKEN_OFFSET (2); PAD=0, MASK=1 (:16-18).
Here the two stable sorts of the reference are one lexicographic sort on (-score, col), which is the
same total order (numpy's lexsort is stable and sorts NaN last like argsort).

Parity pinned: tests/golden/rank_encode.npz is produced by running the reference's own
``densefeed.rank_encode`` / ``compute_gene_stats`` (oracle/make_golden_rank.py) and
tests/test_oracle.py checks this restatement against it.
"""
from __future__ import annotations

import numpy as np

PAD_ID, MASK_ID, TOKEN_OFFSET = 0, 1, 2


def compute_gene_stats(indptr, cols, vals, n_genes: int) -> np.ndarray:
    """tokenizer.py:52-65 over a CSR matrix: fp32 medians [n_genes]."""
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float32).astype(np.float64)
    med = np.ones(n_genes, dtype=np.float32)
    if cols.size == 0:
        return med
    order = np.lexsort((vals, cols))          # group by gene, values ascending inside a gene
    c, v = cols[order], vals[order]
    starts = np.flatnonzero(np.r_[True, c[1:] != c[:-1]])
    ends = np.r_[starts[1:], c.size]
    for s, e in zip(starts, ends):
        n = e - s
        mid = s + n // 2
        m = v[mid] if n % 2 else 0.5 * (v[mid - 1] + v[mid])
        med[c[s]] = np.float32(m)
    return med


def rank_encode(cols, vals, medians, max_len: int) -> np.ndarray:
    """tokenizer.py:68-83 for one row: int64 tokens (gene + 2), descending normalised expression."""
    if max_len < 0:
        raise ValueError("max_len must be >= 0")
    cols = np.asarray(cols, dtype=np.int64)
    if cols.size == 0:
        return np.empty(0, dtype=np.int64)
    if cols.max() >= len(medians):
        raise ValueError("row column index exceeds n_genes")
    score = np.asarray(vals, dtype=np.float64) / np.asarray(medians, dtype=np.float64)[cols]
    order = np.lexsort((cols, -score))
    return (cols[order[:max_len]] + TOKEN_OFFSET).astype(np.int64)


def rank_encode_batch(indptr, cols, vals, medians, rows, max_len: int, seq_len: int):
    """Padded batch as the device kernel writes it: ids int32 [B, S] (PAD 0), am int32 [B, S]."""
    ids = np.full((len(rows), seq_len), PAD_ID, dtype=np.int32)
    am = np.zeros_like(ids)
    for b, r in enumerate(rows):
        a, e = int(indptr[r]), int(indptr[r + 1])
        t = rank_encode(cols[a:e], vals[a:e], medians, min(max_len, seq_len))
        ids[b, :t.size] = t
        am[b, :t.size] = 1
    return ids, am
