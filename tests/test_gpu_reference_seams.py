"""The B200 train step driven end to end through the reference's own seams.

The reference package (densefeed + densefeed_bindings) is imported unmodified from baseline/_ref
(tests/conftest.py:import_reference -- a hard error, never a skip, when it is missing):

  collect_peak_alloc(samples, make_workload(model), length_features, CudaPeakMeter)   sizing.py:76-100
    -> fit_cost_model(records)                                                         sizing.py:149-174
    -> create_buckets(sizes) / bucket_batches(spec, features, cost, budget, seed)      bucketing.py:66-94,177-186
    -> collate -> EsmForMaskedLM.train_step_tokens                                     (the B200 step)

and for Geneformer cells: build_store -> dfb.open -> dfb.batches -> seams.collate_indices -> train step
(bindings/src/densefeed_bindings/__init__.py:45-95).  Losses of the first batches are checked against the
CPU oracle trainer on the same padded batches and masks (fp32 parity mode: 1e-4)."""
import numpy as np
import pytest
import torch

import esm2_oracle as O
from conftest import import_reference
from paper_2411_10548_b200 import EsmConfig
from paper_2411_10548_b200.config import geneformer_config
from paper_2411_10548_b200.data import collate
from paper_2411_10548_b200.model import EsmForMaskedLM, init_params
from paper_2411_10548_b200.seams import CudaPeakMeter, collate_indices, length_features, make_workload

pytestmark = pytest.mark.gpu


def _proteins(n, seed, lo=10, hi=400):
    """Protein-like lengths: lognormal(5.6, 0.65) clipped, scaled into [lo, hi] for test speed."""
    rng = np.random.default_rng(seed)
    lens = np.clip(rng.lognormal(5.6, 0.65, n) * hi / 1024, lo, hi).astype(int)
    return [np.r_[O.CLS, rng.integers(4, 24, L - 2), O.EOS].astype(np.int32) for L in lens]


def test_sizing_and_bucketing_drive_the_b200_step():
    densefeed, _ = import_reference()
    H, L, nh, F = 64, 2, 4, 256
    cfg = EsmConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=nh, intermediate_size=F)
    ocfg = O.OracleConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=nh, intermediate_size=F)
    params = init_params(cfg, seed=8)
    # 1. profile: one record per sample (a single sequence), activation memory above the resident model
    prof = EsmForMaskedLM(cfg, dtype="bf16", device="cuda", params=params)
    samples = _proteins(12, seed=1)
    records = densefeed.collect_peak_alloc(samples, make_workload(prof, pad_to=8, release=True), length_features,
                                           CudaPeakMeter(relative=True))
    assert len(records) == 12 and not any(r.failed for r in records)
    cost, report = densefeed.fit_cost_model(records, safety_margin=1.3)  # headroom for in-bucket padding
    assert cost.weights[0] > 0 and report.n_failed == 0
    # 2. batches from the reference's bucketing under a memory budget
    data = _proteins(80, seed=2)
    sizes = [len(t) for t in data]
    spec = densefeed.create_buckets(sizes, max_width=16, min_count=6)
    feats = np.array([length_features(t) for t in data])
    budget = float(cost.predict_many(feats).sum() / 8)  # ~8 batches per epoch
    it = densefeed.bucket_batches(spec, feats, cost, budget, seed=11)
    batches = [b.indices for b in it]
    assert len(batches) >= 5 and not it.skipped
    owner = {i: k for k, bk in enumerate(spec.buckets) for i in bk.members}
    assert all(len({owner[i] for i in b}) == 1 for b in batches)  # bucket-pure batches
    # 3. the step on those batches: fp32 parity mode vs the oracle trainer (same padded batch + masks)
    m = EsmForMaskedLM(cfg, dtype="fp32", device="cuda", params=params, lr=1e-3)
    tr = O.OracleTrainer(ocfg, params, lr=1e-3, beta1=0.9, beta2=0.98, eps=1e-8, weight_decay=0.01)
    for step, idx in enumerate(batches[:3]):
        toks = [data[i] for i in idx]
        ids, am = collate(toks, pad_to=8)
        inp, lab = O.mlm_mask(ids, seed=5, stream=step)
        want = tr.step(inp, am, lab)
        got = float(m.train_step_tokens(toks, seed=5, stream_id=step, pad_to=8).item())
        assert abs(got - want) / want < 1e-4, (step, got, want)
    # 4. bf16 production path, metered like the profile: every batch stays within the budgeted memory
    b16 = EsmForMaskedLM(cfg, dtype="bf16", device="cuda", params=params)
    b16.max_workspaces = 1
    meter = CudaPeakMeter(relative=True)
    for step, idx in enumerate(batches):
        b16.release_workspaces()
        meter.reset()
        loss = float(b16.train_step_tokens([data[i] for i in idx], seed=5, stream_id=step, pad_to=8).item())
        assert np.isfinite(loss) and loss > 0
        assert meter.peak() <= budget, (step, meter.peak(), budget)
    # and replayed as one CUDA graph per bucket shape
    for step, idx in enumerate(batches[:3]):
        loss = float(b16.train_step_tokens([data[i] for i in idx], seed=5, stream_id=100 + step, pad_to=8,
                                           use_graph=True).item())
        assert np.isfinite(loss) and loss > 0


def test_geneformer_store_bindings_batches_drive_the_b200_step(tmp_path):
    densefeed, dfb = import_reference()
    rng = np.random.default_rng(4)
    n_rows, n_genes = 40, 200
    ent = []
    for r in range(n_rows):
        k = int(rng.integers(8, 90))
        for c in sorted(rng.choice(n_genes, k, replace=False)):
            ent.append(f"{r + 1} {c + 1} {float(rng.uniform(0.5, 10.0))!r}")
    (tmp_path / "m.mtx").write_text("\n".join(["% cells", f"{n_rows} {n_genes} {len(ent)}"] + ent) + "\n")
    densefeed.build_store(tmp_path / "m.mtx", tmp_path / "store")
    ds = dfb.open(tmp_path / "store", max_len=64)
    gcfg = geneformer_config(n_genes=n_genes, hidden_size=64, num_hidden_layers=2, num_attention_heads=4,
                             intermediate_size=128)
    gocfg = O.OracleConfig(vocab_size=gcfg.vocab_size, hidden_size=64, num_hidden_layers=2, num_attention_heads=4,
                           intermediate_size=128, token_dropout=False, mask_token_id=1, pad_token_id=0)
    params = init_params(gcfg, seed=9)
    # cost model on the bindings' single feature (row non-zero count), profiled on the GPU step
    prof = EsmForMaskedLM(gcfg, dtype="bf16", device="cuda", params=params)
    wl = make_workload(prof, pad_to=8, release=True)
    recs = densefeed.collect_peak_alloc([ds[i][0] for i in range(12)], wl, lambda t: [float(len(t))],
                                        CudaPeakMeter(relative=True))
    cost, _ = densefeed.fit_cost_model(recs)
    densefeed.save_cost_model(cost, tmp_path / "cm.json")
    budget = float(cost.predict([64.0]) * 6)
    batches = list(dfb.batches(ds, tmp_path / "cm.json", budget=budget, max_width=24, min_count=4, seed=3))
    assert len(batches) >= 3
    m = EsmForMaskedLM(gcfg, dtype="fp32", device="cuda", params=params, lr=1e-3)
    mk = dict(eligible=gcfg.mlm_eligible, mask_id=gcfg.mask_token_id, random_range=gcfg.mlm_random)
    tr = O.OracleTrainer(gocfg, params, lr=1e-3, beta1=0.9, beta2=0.98, eps=1e-8, weight_decay=0.01)
    for step, idx in enumerate(batches[:2]):
        ids, am = collate_indices(ds, idx, pad_to=8, pad_id=0)
        inp, lab = O.mlm_mask(ids, seed=2, stream=step, **mk)
        want = tr.step(inp, am, lab)
        got = float(m.train_step_tokens([ds[i][0] for i in idx], seed=2, stream_id=step, pad_to=8).item())
        assert abs(got - want) / want < 1e-4, (step, got, want)

