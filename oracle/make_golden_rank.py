"""Golden vectors for the Geneformer rank-value tokeniser, produced by the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  Runs in the build container, where the reference package is importable
from /root/reference/pkg/src (read-only; nothing is copied).  It builds a random store with the
reference's ``build_store`` (conftest.random_sparse_entries pattern, pkg/tests/conftest.py:16-26, plus
integer-valued rows that force score ties), computes ``compute_gene_stats`` and runs ``rank_encode``
on every row at several max_len values.  The CSR arrays, medians and expected tokens go to
tests/golden/rank_encode.npz; tests/test_oracle.py pins oracle/rank_oracle.py to them and
tests/test_gpu_geneformer.py checks the esm_rank_encode kernel bit-exactly.

    python oracle/make_golden_rank.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "rank_encode.npz")
MAX_LENS = (0, 1, 7, 256, 2048, 100000)


def main():
    sys.path.insert(0, REF)
    from densefeed import build_store, compute_gene_stats, open_store, rank_encode

    rng = np.random.default_rng(2411)
    n_genes = 25424
    nnz_per_row = [0, 1, 3, 40, 500, 1200, 2047, 2048, 2049, 3999, 4096, 6000, 700, 9]
    lines = []
    for r, k in enumerate(nnz_per_row):
        cols = np.sort(rng.choice(n_genes, size=k, replace=False))
        if r % 3 == 2:   # integer levels: many equal scores -> exercises the ascending-gene tie rule
            vals = rng.integers(1, 4, size=k).astype(np.float32)
        else:            # conftest.random_sparse_entries value range
            vals = rng.uniform(0.5, 10.0, size=k).astype(np.float32)
        lines += [f"{r + 1} {c + 1} {float(v)!r}" for c, v in zip(cols, vals)]
    with tempfile.TemporaryDirectory() as td:
        mtx = os.path.join(td, "m.mtx")
        with open(mtx, "w") as f:
            f.write("% golden rank_encode\n")
            f.write(f"{len(nnz_per_row)} {n_genes} {len(lines)}\n")
            f.write("\n".join(lines) + "\n")
        build_store(mtx, os.path.join(td, "store"))
        store = open_store(os.path.join(td, "store"))
        stats = compute_gene_stats(store)
        indptr, cols, vals = [0], [], []
        for row in store.iter_rows():
            cols.append(np.asarray(row.cols, np.int64))
            vals.append(np.asarray(row.vals, np.float32))
            indptr.append(indptr[-1] + len(row.cols))
        expect = {}
        for ml in MAX_LENS:
            toks = [np.asarray(rank_encode(store.get_row(r), stats, ml).tokens, np.int64)
                    for r in range(store.n_rows)]
            expect[f"tokens_{ml}"] = np.concatenate(toks) if toks else np.empty(0, np.int64)
            expect[f"lengths_{ml}"] = np.array([len(t) for t in toks], np.int64)
    np.savez_compressed(OUT, indptr=np.array(indptr, np.int64), cols=np.concatenate(cols),
                        vals=np.concatenate(vals), medians=np.asarray(stats.medians, np.float32),
                        n_genes=np.int64(n_genes), max_lens=np.array(MAX_LENS, np.int64), **expect)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
