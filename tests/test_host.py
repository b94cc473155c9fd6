"""CPU-only tests of the host side: C-ABI exports vs the header, native tokenizer vs the oracle,
parameter layout / init parity with the oracle, collation, and the data-parallel gradient
bucket all-reduce on gloo with world_size 2 (no GPU needed)."""
import ctypes
import os
import re
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import esm2_oracle as O
from paper_2411_10548_b200 import EsmConfig, _lib, preset
from paper_2411_10548_b200.data import collate, synthetic_batch, tokenize
from paper_2411_10548_b200.model import ALIGN, ParamStore, init_params, param_groups, rope_tables

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "esm2_b200.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(esm_\w+)\s*\(", hdr, flags=re.M))
    assert len(declared) >= 18
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.EXPORTS)
    assert lib.esm_version() >= 10000
    # the collectives resolve NCCL at run time (no GPU needed to load it): torch's 2.28 or the system's 2.27
    assert lib.esm_comm_version() >= 22700


def test_native_tokenizer_matches_oracle():
    rng = np.random.default_rng(0)
    alphabet = list("LAGVSERTIDPKQNFYMHWCXBUZO.-J*")
    for _ in range(50):
        seq = "".join(rng.choice(alphabet, size=rng.integers(0, 300)))
        np.testing.assert_array_equal(tokenize(seq), O.tokenize(seq))


def test_tokenizer_buffer_too_small_reports_needed():
    lib = _lib.load()
    out = np.zeros(4, np.int32)
    assert lib.esm_tokenize(b"MKTAYIAK", 8, out.ctypes.data_as(ctypes.c_void_p), 4) == -10


def test_init_params_and_rope_match_oracle():
    cfg = EsmConfig(hidden_size=64, num_hidden_layers=2, num_attention_heads=4, intermediate_size=256)
    ocfg = O.OracleConfig(hidden_size=64, num_hidden_layers=2, num_attention_heads=4, intermediate_size=256)
    a, b = init_params(cfg, 7), O.init_params(ocfg, 7)
    assert a.keys() == b.keys()
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
    c, s = rope_tables(100, 24)
    oc, os_ = O.rope_tables(100, 24)
    np.testing.assert_array_equal(c, oc[:, :12])
    np.testing.assert_array_equal(s, os_[:, :12])


def test_param_store_layout():
    cfg = preset("8m")
    st = ParamStore(cfg, "cpu", shadow=False)
    assert st.numel % ALIGN == 0
    n = sum(s.numel for s in st.slots.values())
    assert n == 7_511_233 or abs(n - 7.51e6) < 2e4  # ESM-2 8M parameter count (tied decoder)
    # groups are 256-aligned, contiguous, in backward-completion order with embeddings last
    keys = [k for k, _ in param_groups(cfg)]
    assert keys[0] == "lm_head.bias" and keys[-1] == "esm.embeddings.word_embeddings.weight"
    prev = -1
    for k in keys:
        a, b = st.group_range[k]
        assert a % ALIGN == 0 and a > prev
        prev = a
    # q/k/v weights of one layer form one contiguous [3H, H] group
    q = st.slots["esm.encoder.layer.0.attention.self.query.weight"]
    v = st.slots["esm.encoder.layer.0.attention.self.value.weight"]
    assert v.offset - q.offset == 2 * cfg.hidden_size ** 2
    # decay flags: weights decay, biases / LayerNorm do not
    d = st.decay.numpy()
    a, _ = st.group_range["esm.encoder.layer.0.output.dense.weight"]
    assert d[a // ALIGN] == 1
    a, _ = st.group_range["esm.encoder.layer.0.LayerNorm.weight"]
    assert d[a // ALIGN] == 0


def test_presets_param_counts():
    expect = {"8m": 7.51e6, "35m": 33.50e6, "650m": 651.04e6, "3b": 2839.01e6}
    for name, n in expect.items():
        cfg = preset(name)
        H, F, V, L = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers
        total = V * H + L * (4 * H * H + 4 * H + 2 * H * F + F + H + 4 * H) + 2 * H + H * H + H + 2 * H + V
        assert abs(total - n) / n < 1e-3, (name, total)


def test_collate_and_synthetic():
    ids, am = collate([[0, 5, 6, 2], [0, 7, 2]], pad_to=8)
    assert ids.shape == (2, 8) and am.sum() == 7
    assert (ids[1, 3:] == 1).all()
    a, _ = synthetic_batch(3, 16, 5)
    b, _ = O.synthetic_batch(3, 16, 5)
    np.testing.assert_array_equal(a, b)


def test_flops_per_token_matches_oracle():
    cfg = preset("650m")
    ocfg = O.OracleConfig(hidden_size=1280, num_hidden_layers=33, num_attention_heads=20, intermediate_size=5120)
    assert cfg.train_flops_per_token(1024) == O.train_flops_per_token(ocfg, 1024)


# ---------------------------------------------------------------- DDP bucketing on gloo
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ddp_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_10548_b200.ddp import GradAllReducer
        cfg = EsmConfig(hidden_size=64, num_hidden_layers=3, num_attention_heads=4, intermediate_size=256)
        st = ParamStore(cfg, "cpu", shadow=False)
        red = GradAllReducer(st, bucket_bytes=64 << 10)
        g = torch.arange(st.numel, dtype=torch.float32) * (rank + 1)
        st.g32.copy_(g)
        red.begin_backward()
        # readiness in backward order, as the model signals it
        red.ready("esm.encoder.emb_layer_norm_after.bias")
        for l in reversed(range(cfg.num_hidden_layers)):
            red.ready(f"esm.encoder.layer.{l}.attention.LayerNorm.bias")
        red.ready("esm.embeddings.word_embeddings.weight")
        red.end_backward()
        want = torch.arange(st.numel, dtype=torch.float32) * sum(r + 1 for r in range(world))
        ok_grad = torch.equal(st.g32, want)
        n = torch.tensor([10 * (rank + 1)], dtype=torch.int32)
        red.reduce_count(n)
        # overlapped optimizer hook: each bucket is handed over (in order, contiguous, covering the whole
        # buffer) only after its all-reduce has completed
        seen = []
        want2 = 2 * torch.arange(st.numel, dtype=torch.float32) * world
        red.on_bucket = lambda a, b, stream, g: seen.append((a, b, bool(torch.equal(g, want2[a:b]))))
        st.g32.copy_(g)
        st.g32.mul_(2)
        st.g32.div_(rank + 1)  # every rank holds 2 * arange -> reduced = 2 * arange * world
        red.begin_backward()
        red.ready("esm.encoder.emb_layer_norm_after.bias")
        for l in reversed(range(cfg.num_hidden_layers)):
            red.ready(f"esm.encoder.layer.{l}.attention.LayerNorm.bias")
        red.ready("esm.embeddings.word_embeddings.weight")
        red.end_backward()
        contiguous = seen[0][0] == 0 and seen[-1][1] == st.numel and all(
            seen[i][1] == seen[i + 1][0] for i in range(len(seen) - 1))
        hooks_ok = contiguous and all(ok for _, _, ok in seen)
        q.put((rank, ok_grad and hooks_ok, int(n.item()), len(red.bucket_ends)))
    finally:
        dist.destroy_process_group()


def _zero1_worker(rank, world, port, q):
    """Sharded optimizer (reduce-scatter -> update of the rank's slice -> all-gather of p32 / p16) gives bit-for-bit
    the parameters of the all-reduce path with the same update applied to every bucket; bf16 buckets give
    the bf16-rounded sums.  The update is an elementwise SGD stand-in for AdamW (the GPU kernel is not
    available on CPU); the bucket / slice / gather bookkeeping is what is under test."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_10548_b200.ddp import GradAllReducer
        cfg = EsmConfig(hidden_size=64, num_hidden_layers=3, num_attention_heads=4, intermediate_size=256)
        results = {}
        for mode in ("ddp", "zero1", "zero1_bf16", "ddp_bf16", "zero1_full"):
            st = ParamStore(cfg, "cpu", shadow=True)
            torch.manual_seed(0)
            st.p32.copy_(torch.randn(st.numel))
            st.p16.copy_(st.p32)
            red = GradAllReducer(st, bucket_bytes=32 << 10, shard_optimizer=mode.startswith("zero1"),
                                 grad_dtype="bf16" if mode.endswith("bf16") else "fp32",
                                 master="full" if mode.endswith("full") else "vectors")
            calls = []

            def upd(a, b, stream, g, st=st, calls=calls):
                calls.append((a, b))
                st.p32[a:b] -= 0.1 * g.float()
                st.p16[a:b].copy_(st.p32[a:b])

            red.on_bucket = upd
            for step in range(2):
                torch.manual_seed(100 + 10 * step + rank)
                st.g32.copy_(torch.randn(st.numel))
                red.begin_backward()
                red.ready("esm.encoder.emb_layer_norm_after.bias")
                for l in reversed(range(cfg.num_hidden_layers)):
                    red.ready(f"esm.encoder.layer.{l}.attention.LayerNorm.bias")
                red.end_backward()
            owned = sum(b - a for a, b in calls) // 2
            # sharded fp32 master: the 1-D (fp32-read) parameters are current on every rank right after the
            # step; the rest of the master after gather_master()
            vec_idx = torch.cat([torch.arange(sl.offset, sl.offset + sl.numel) for sl in st.slots.values()
                                 if len(sl.shape) == 1])
            vecs = st.p32[vec_idx].clone()
            red.gather_master()
            results[mode] = (st.p32.clone(), st.p16.clone(), owned, st.numel, vecs, vec_idx)
        ddp, z1 = results["ddp"], results["zero1"]
        ok = torch.equal(ddp[0], z1[0]) and torch.equal(ddp[1], z1[1]) and torch.equal(z1[4], ddp[0][z1[5]])
        ok = ok and torch.equal(results["zero1_full"][0], ddp[0]) and torch.equal(results["zero1_full"][1], ddp[1])
        ok = ok and z1[2] * world == z1[3] and ddp[2] == ddp[3]  # each rank updated exactly 1/world of the buffer
        zb, db = results["zero1_bf16"], results["ddp_bf16"]
        ok = ok and torch.equal(zb[0], db[0]) and (zb[0] - ddp[0]).abs().max().item() < 0.05
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_optimizer_matches_allreduce_gloo(world):
    """world 8 = the driver's largest data-parallel run: every bucket splits into 8 owned slices of whole AdamW
    chunks and the 1-D fp32 parameters are re-synchronised from 8 owners."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_zero1_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok in res), res


def test_grad_bucket_allreduce_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ddp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, n, nb in res:
        assert ok, rank
        assert n == 30
        assert nb > 1  # several buckets -> overlap with backward is possible


def test_head_capacity_and_config_validation():
    from paper_2411_10548_b200.config import geneformer_config
    from paper_2411_10548_b200.model import head_capacity
    for T in (64, 1000, 16384, 65536):
        cap = head_capacity(T)
        assert cap <= T and (cap == T or cap % 128 == 0)
        assert cap >= min(T, 0.15 * T + 8 * T ** 0.5)  # > 20 sigma above the 15% mean
    with pytest.raises(ValueError):
        EsmConfig(vocab_size=33, mlm_eligible=(4, 40)).validate()
    with pytest.raises(ValueError):
        geneformer_config(n_genes=100, mlm_random=(2, 200))
    assert geneformer_config(n_genes=100).vocab_size == 102


def test_geneformer_preset_and_feed_host_logic():
    """Geneformer config (BASELINE configs[4]): ~106M params, reference token layout, host-side
    medians identical to the reference's compute_gene_stats (golden from the reference)."""
    from paper_2411_10548_b200.data import gene_medians, synthetic_expression_csr
    cfg = preset("geneformer")
    H, F, V, L = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers
    total = V * H + L * (4 * H * H + 4 * H + 2 * H * F + F + H + 4 * H) + 2 * H + H * H + H + 2 * H + V
    assert abs(total - 106e6) / 106e6 < 0.01
    assert (cfg.pad_token_id, cfg.mask_token_id, cfg.mlm_eligible, cfg.token_dropout) == (0, 1, (2, V - 1), False)
    assert abs(cfg.train_flops_per_token(2048) - 0.857e9) / 0.857e9 < 1e-3
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "rank_encode.npz"))
    assert np.array_equal(gene_medians(z["indptr"], z["cols"], z["vals"], int(z["n_genes"])), z["medians"])
    ip, c, v = synthetic_expression_csr(5, 1000, seed=1, nnz=(10, 50))
    assert ip.shape == (6,) and c.size == ip[-1] == v.size and c.max() < 1000
    for r in range(5):
        assert (np.diff(c[ip[r]:ip[r + 1]]) > 0).all()
    ids, am = collate([[5, 6, 7], [9]], pad_to=4, pad_id=0)
    assert ids.tolist() == [[5, 6, 7, 0], [9, 0, 0, 0]] and am.sum() == 4


def test_reference_shard_stream_feeds_collate(tmp_path):
    """the reference's own tar-shard pipeline (write_shards / subset / stream_samples /
    batch_stage) with our shard_collate yields the padded batches the train step consumes; the per-rank
    subsets partition the samples (the reference is imported from baseline/_ref; never skipped)."""
    from conftest import import_reference
    densefeed, _ = import_reference()
    SH = densefeed.shards
    from paper_2411_10548_b200.seams import shard_collate
    rng = np.random.default_rng(0)
    toks = {f"s{i:03d}": np.r_[0, rng.integers(4, 24, int(rng.integers(5, 40))), 2].astype("<i4") for i in range(23)}
    SH.write_shards((SH.Sample(k, {"tokens": v.tobytes()}) for k, v in toks.items()), tmp_path / "sh", max_per_shard=5)
    ss = SH.load_shard_set(tmp_path / "sh")
    seen = 0
    for rank in range(2):
        batches = list(SH.compose(SH.stream_samples(ss.subset(rank, 2)), [SH.batch_stage(4, collate=shard_collate(8))]))
        for ids, am in batches:
            assert ids.dtype == np.int32 and ids.shape == am.shape and ids.shape[1] % 8 == 0
            assert (ids[am == 0] == 1).all() and (ids[:, 0] == 0).all()
            seen += ids.shape[0]
    assert seen == len(toks)


def test_reference_bindings_batches_feed_collate_indices(tmp_path):
    """SURVEY §8b seams 'Dataset items' + 'Batch stream' on the CPU: the reference's own store
    (build_store), BoundDataset (dfb.open: rank_encode per row) and dfb.batches (create_buckets +
    bucket_batches over a saved cost model) drive seams.collate_indices; every index list becomes a padded
    int32 [B, S] batch whose rows are exactly the reference's rank tokens (PAD 0), and the index lists
    partition the dataset (modulo budget skips) deterministically for a seed."""
    from conftest import import_reference
    densefeed, dfb = import_reference()
    from paper_2411_10548_b200.seams import collate_indices
    rng = np.random.default_rng(3)
    n_rows, n_cols = 60, 300
    lines = ["% test", f"{n_rows} {n_cols} 0"]
    ent = []
    for r in range(n_rows):
        k = int(rng.integers(3, 120))
        for c in sorted(rng.choice(n_cols, k, replace=False)):
            ent.append(f"{r + 1} {c + 1} {float(rng.uniform(0.5, 10.0))!r}")
    lines[1] = f"{n_rows} {n_cols} {len(ent)}"
    (tmp_path / "m.mtx").write_text("\n".join(lines + ent) + "\n")
    densefeed.build_store(tmp_path / "m.mtx", tmp_path / "store")
    ds = dfb.open(tmp_path / "store", max_len=64)
    cm = densefeed.CostModel(weights=np.array([1.0]), intercept=0.0, safety_margin=1.0)
    densefeed.save_cost_model(cm, tmp_path / "cm.json")
    got = [list(b) for b in dfb.batches(ds, tmp_path / "cm.json", budget=400.0, max_width=30, min_count=4, seed=7)]
    again = [list(b) for b in dfb.batches(ds, tmp_path / "cm.json", budget=400.0, max_width=30, min_count=4, seed=7)]
    assert got == again and len(got) > 3
    seen = sorted(i for b in got for i in b)
    assert len(seen) == len(set(seen)) and set(seen) <= set(range(n_rows))
    for idx in got:
        ids, am = collate_indices(ds, idx, pad_to=8, pad_id=0)
        assert ids.shape[0] == len(idx) and ids.shape[1] % 8 == 0 and ids.dtype == np.int32
        for j, i in enumerate(idx):
            want = ds[i][0]
            assert ids[j, :len(want)].tolist() == want and am[j].sum() == len(want)
            assert (ids[j, len(want):] == 0).all()


def test_workspace_arena_packs_activations_without_overlap():
    """Variable-shape training keeps one activation arena for all (B, S) workspaces: each workspace's
    activation / scratch tensors are disjoint 1 KB-aligned views of the arena, sized by activation_bytes, and
    the per-shape inputs / constants are separate allocations."""
    import torch
    from paper_2411_10548_b200 import EsmConfig
    from paper_2411_10548_b200.model import Workspace, _Arena
    cfg = EsmConfig(hidden_size=64, num_hidden_layers=2, num_attention_heads=4, intermediate_size=256)
    sizes = {shape: Workspace.activation_bytes(cfg, *shape, torch.bfloat16) for shape in [(4, 64), (2, 128), (8, 32)]}
    assert len(set(sizes.values())) <= 3 and min(sizes.values()) > 0
    buf = torch.empty(max(sizes.values()), dtype=torch.uint8)
    lo, hi = buf.data_ptr(), buf.data_ptr() + buf.numel()
    for shape in sizes:
        ws = Workspace(cfg, *shape, torch.bfloat16, "cpu", arena=_Arena(buf))
        assert ws.arena_bytes == sizes[shape]
        spans = []
        for t in [*ws.x, ws.dq, ws.dqkv, ws.delta, ws.dz, ws.row_scale, *(ly.z for ly in ws.layers)]:
            a = t.data_ptr()
            assert lo <= a and a + t.numel() * t.element_size() <= hi and (a - lo) % 1024 == 0
            spans.append((a, a + t.numel() * t.element_size()))
        spans.sort()
        assert all(b0 <= a1 for (_, b0), (a1, _) in zip(spans, spans[1:]))
        for t in (ws.ids, ws.am, ws.labels, ws.attn_sched, ws.cos):
            assert not (lo <= t.data_ptr() < hi)
