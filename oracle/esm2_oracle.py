"""CPU oracle for the ESM-2 masked-language-model train step.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import this module:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``--impl reference`` / ``cpu_baseline``) use it, and only as the checker or
the timed CPU reference -- never as a fallback for the CUDA path.

What it restates
----------------
The reference repository (``/root/reference``, the ``densefeed`` data toolkit)
contains *no* model, train step or kernels for this path (SURVEY.md §0,
``SPEC.md:8``).  The only implementation of ESM-2 MLM arithmetic in this image
is the third-party Hugging Face ``transformers`` 5.5.0 package,
``models/esm/modeling_esm.py`` (abbreviated ``HF:`` below).  This module is a
from-scratch numpy restatement of that algorithm with an explicit, hand-derived
backward pass:

* RoPE tables / rotate_half          HF:modeling_esm.py:45-54, 81-123
* exact erf GELU                     HF:modeling_esm.py:57-61
* embeddings + token_dropout + pad   HF:modeling_esm.py:189-236
* self-attention (q pre-scaled, RoPE after scaling, scaling=1 in softmax)
                                      HF:modeling_esm.py:257-282, 318-362
* pre-LN residual layer               HF:modeling_esm.py:365-482
* final emb_layer_norm_after          HF:modeling_esm.py:485-514
* LM head (dense, GELU, LN, tied decoder + bias) HF:modeling_esm.py:797-815
* masked CE (ignore_index=-100, mean) HF:modeling_esm.py:777-784
* init (normal(0, 0.02), zero bias, LN 1/0, zero pad row) HF:modeling_esm.py:555-569,
  transformers/modeling_utils.py:2301-2310
* AdamW (decoupled weight decay)      torch.optim.AdamW semantics

Parity pinning: ``oracle/make_golden.py`` runs HF ``EsmForMaskedLM`` (fp64, eager
attention) on the same parameters/inputs and commits loss, logits, per-layer
hidden states and every parameter gradient to ``tests/golden/``;
``tests/test_oracle.py`` checks this module against them.

The tokenizer alphabet is the public fair-esm ESM-2 alphabet (HF's
``EsmTokenizer`` needs a ``vocab.txt`` that is not in this image,
HF:tokenization_esm.py:27-31).  The 15% / 80-10-10 masking RNG is defined here
(counter-based splitmix64, integer thresholds) because neither the reference
(``SPEC.md:154`` non-goal) nor HF's model defines one; the CUDA masking kernel
implements the identical integer recipe, so masks are bit-exact.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

try:  # scipy is in the image; fall back to math.erf vectorised if absent
    from scipy.special import erf as _erf
except Exception:  # pragma: no cover
    _erf = np.vectorize(math.erf)

# --------------------------------------------------------------------------
# Alphabet (fair-esm ESM-2 vocabulary, 33 tokens)
# --------------------------------------------------------------------------
ALPHABET = (
    ["<cls>", "<pad>", "<eos>", "<unk>"]
    + list("LAGVSERTIDPKQNFYMHWC")
    + list("XBUZO.-")
    + ["<null_1>", "<mask>"]
)
assert len(ALPHABET) == 33
CLS, PAD, EOS, UNK, MASK = 0, 1, 2, 3, 32
AA_FIRST, AA_COUNT = 4, 20  # the 20 standard amino acids are ids 4..23
TOK_TO_ID = {t: i for i, t in enumerate(ALPHABET)}


def tokenize(seq: str) -> np.ndarray:
    """<cls> + residues + <eos>; unknown characters map to <unk>."""
    ids = [CLS]
    for ch in seq:
        ids.append(TOK_TO_ID.get(ch, UNK))
    ids.append(EOS)
    return np.asarray(ids, dtype=np.int32)


def pad_batch(tok_lists, seq_len: int):
    """Right-pad to ``seq_len`` with <pad>; returns (ids int32 [B,S], attention_mask int32)."""
    b = len(tok_lists)
    ids = np.full((b, seq_len), PAD, dtype=np.int32)
    am = np.zeros((b, seq_len), dtype=np.int32)
    for i, t in enumerate(tok_lists):
        n = min(len(t), seq_len)
        ids[i, :n] = t[:n]
        am[i, :n] = 1
    return ids, am


def synthetic_batch(batch: int, seq_len: int, seed: int):
    """Full-length synthetic protein sequences: <cls> AA* <eos>, AAs uniform over ids 4..23."""
    rng = np.random.default_rng(seed)
    ids = rng.integers(AA_FIRST, AA_FIRST + AA_COUNT, size=(batch, seq_len), dtype=np.int64).astype(np.int32)
    ids[:, 0] = CLS
    ids[:, -1] = EOS
    am = np.ones((batch, seq_len), dtype=np.int32)
    return ids, am


# --------------------------------------------------------------------------
# MLM masking: counter-based splitmix64, integer thresholds (bit-exact vs CUDA)
# --------------------------------------------------------------------------
_U64 = np.uint64
GOLDEN = _U64(0x9E3779B97F4A7C15)
P_SELECT = 2516582    # floor(0.15 * 2^24)
P_MASK = 13421773     # ceil(0.80 * 2^24)
P_RANDOM = 15099494   # floor(0.90 * 2^24)


def _mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> _U64(30))) * _U64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> _U64(27))) * _U64(0x94D049BB133111EB)
    return z ^ (z >> _U64(31))


def mask_key(seed: int, stream: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k0 = _mix64(_U64(seed & 0xFFFFFFFFFFFFFFFF) + GOLDEN)
        return _mix64(k0 ^ _U64(stream & 0xFFFFFFFFFFFFFFFF))


def mask_draws(key, n: int):
    """Three 64-bit draws per position index i in [0, n)."""
    i = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        base = _U64(key) + i * GOLDEN
        return _mix64(base), _mix64(base + _U64(1)), _mix64(base + _U64(2))


def mlm_mask(ids: np.ndarray, seed: int, stream: int, eligible=(4, 30), mask_id: int = MASK,
             random_range=(AA_FIRST, AA_COUNT)):
    """15% of eligible positions (ids in ``eligible``, inclusive; ESM-2: 4..30) are selected; of
    those 80% -> ``mask_id``, 10% -> ``random_range[0] + r % random_range[1]`` (ESM-2: the 20
    standard AAs), 10% unchanged.  labels = original id where selected, else -100.
    Geneformer rank tokens (reference pkg/src/densefeed/tokenizer.py:16-18, PAD=0 MASK=1 offset 2):
    eligible=(2, V-1), mask_id=1, random_range=(2, V-2).  Returns (input_ids int32, labels int32)."""
    flat = np.asarray(ids, dtype=np.int32).reshape(-1)
    r0, r1, r2 = mask_draws(mask_key(seed, stream), flat.size)
    elig = (flat >= eligible[0]) & (flat <= eligible[1])
    sel = elig & ((r0 >> _U64(40)).astype(np.int64) < P_SELECT)
    a = (r1 >> _U64(40)).astype(np.int64)
    rnd = (random_range[0] + (r2 % _U64(random_range[1])).astype(np.int64)).astype(np.int32)
    out = flat.copy()
    out = np.where(sel & (a < P_MASK), mask_id, out)
    out = np.where(sel & (a >= P_MASK) & (a < P_RANDOM), rnd, out)
    labels = np.where(sel, flat, -100).astype(np.int32)
    return out.reshape(ids.shape).astype(np.int32), labels.reshape(ids.shape)


# --------------------------------------------------------------------------
# Config and parameters (HF EsmConfig field names, HF:configuration_esm.py:193-214)
# --------------------------------------------------------------------------
@dataclass
class OracleConfig:
    vocab_size: int = 33
    hidden_size: int = 320
    num_hidden_layers: int = 6
    num_attention_heads: int = 20
    intermediate_size: int = 1280
    layer_norm_eps: float = 1e-5
    initializer_range: float = 0.02
    token_dropout: bool = True
    mask_token_id: int = MASK
    pad_token_id: int = PAD


def param_shapes(cfg: OracleConfig):
    """HF state_dict names -> shapes (decoder weight is tied to word_embeddings)."""
    H, F, V = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size
    s = {"esm.embeddings.word_embeddings.weight": (V, H)}
    for i in range(cfg.num_hidden_layers):
        p = f"esm.encoder.layer.{i}."
        for n in ("query", "key", "value"):
            s[p + f"attention.self.{n}.weight"] = (H, H)
            s[p + f"attention.self.{n}.bias"] = (H,)
        s[p + "attention.output.dense.weight"] = (H, H)
        s[p + "attention.output.dense.bias"] = (H,)
        s[p + "attention.LayerNorm.weight"] = (H,)
        s[p + "attention.LayerNorm.bias"] = (H,)
        s[p + "intermediate.dense.weight"] = (F, H)
        s[p + "intermediate.dense.bias"] = (F,)
        s[p + "output.dense.weight"] = (H, F)
        s[p + "output.dense.bias"] = (H,)
        s[p + "LayerNorm.weight"] = (H,)
        s[p + "LayerNorm.bias"] = (H,)
    s["esm.encoder.emb_layer_norm_after.weight"] = (H,)
    s["esm.encoder.emb_layer_norm_after.bias"] = (H,)
    s["lm_head.dense.weight"] = (H, H)
    s["lm_head.dense.bias"] = (H,)
    s["lm_head.layer_norm.weight"] = (H,)
    s["lm_head.layer_norm.bias"] = (H,)
    s["lm_head.bias"] = (V,)
    return s


def init_params(cfg: OracleConfig, seed: int):
    """HF init: Linear/Embedding weights ~ N(0, 0.02), biases 0, LayerNorm (1, 0),
    embedding pad row zeroed.  Drawn in float32 from numpy default_rng(seed) in
    param_shapes() order."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in param_shapes(cfg).items():
        if name.endswith("LayerNorm.weight") or name.endswith("layer_norm.weight") or \
                name.endswith("emb_layer_norm_after.weight"):
            out[name] = np.ones(shape, np.float32)
        elif len(shape) == 2:
            w = (rng.standard_normal(shape, dtype=np.float32) * np.float32(cfg.initializer_range))
            out[name] = w.astype(np.float32)
        else:
            out[name] = np.zeros(shape, np.float32)
    out["esm.embeddings.word_embeddings.weight"][cfg.pad_token_id] = 0.0
    return out


# --------------------------------------------------------------------------
# Elementary ops with explicit backward
# --------------------------------------------------------------------------
def gelu(x):
    """HF:modeling_esm.py:57-61 -- x * 0.5 * (1 + erf(x / sqrt(2)))."""
    return x * 0.5 * (1.0 + _erf(x / math.sqrt(2.0)))


def gelu_grad(x):
    cdf = 0.5 * (1.0 + _erf(x / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return cdf + x * pdf


def layer_norm(x, w, b, eps):
    mu = x.mean(-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = xc * rstd
    return xhat * w + b, (xhat, rstd)


def layer_norm_bwd(dy, w, cache):
    xhat, rstd = cache
    dxhat = dy * w
    dx = rstd * (dxhat - dxhat.mean(-1, keepdims=True) - xhat * (dxhat * xhat).mean(-1, keepdims=True))
    red = tuple(range(dy.ndim - 1))
    return dx, (dy * xhat).sum(red), dy.sum(red)


def rope_tables(seq_len: int, dim: int):
    """HF:modeling_esm.py:91-111: inv_freq = 1/10000^(arange(0,dim,2)/dim) in fp32,
    freqs = outer(t, inv_freq) in fp32, emb = cat(freqs, freqs); cos/sin in fp32."""
    inv_freq = (1.0 / (np.float32(10000.0) ** (np.arange(0, dim, 2, dtype=np.int64).astype(np.float32) / np.float32(dim)))).astype(np.float32)
    t = np.arange(seq_len, dtype=np.float32)
    freqs = np.outer(t, inv_freq).astype(np.float32)
    emb = np.concatenate([freqs, freqs], axis=-1)
    return np.cos(emb).astype(np.float32), np.sin(emb).astype(np.float32)


def rotate_half(x):
    h = x.shape[-1] // 2
    return np.concatenate([-x[..., h:], x[..., :h]], axis=-1)


def rope_apply(x, cos, sin):
    """x [B, nh, S, dh]; HF:modeling_esm.py:50-54."""
    return x * cos + rotate_half(x) * sin


def rope_apply_bwd(dy, cos, sin):
    """Transpose of rope_apply: dx = dy*cos + rotate_half^T(dy*sin)."""
    h = dy.shape[-1] // 2
    ds = dy * sin
    rt = np.concatenate([ds[..., h:], -ds[..., :h]], axis=-1)
    return dy * cos + rt


# --------------------------------------------------------------------------
# Forward / backward of EsmForMaskedLM
# --------------------------------------------------------------------------
@dataclass
class StepResult:
    loss: float
    n_masked: int
    logits: np.ndarray | None = None
    hidden_states: list = field(default_factory=list)  # input of each layer + final (pre emb_layer_norm_after)
    grads: dict = field(default_factory=dict)
    acts: dict = field(default_factory=dict)


def _wgrad(dy, x):
    """sum over (b, s) of dy[b,s,:]^T x[b,s,:]  (BLAS matmul)."""
    return dy.reshape(-1, dy.shape[-1]).T @ x.reshape(-1, x.shape[-1])


def _linear(x, w, b=None):
    y = x @ w.T
    return y if b is None else y + b


# --------------------------------------------------------------------------
# Hidden dropout (HF EsmSelfOutput / EsmOutput: dropout(dense(x)) before the residual add,
# HF:modeling_esm.py:369-375, 421-427) with a counter-based keep mask, so the B200 path regenerates
# it in the backward instead of storing it.  Restates include/esm2_b200.h:esm_dropout bit for bit.
# --------------------------------------------------------------------------
def _lowbias32(x):
    x = np.asarray(x, dtype=np.uint32)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint32(16))
        x = (x * np.uint32(0x7FEB352D)).astype(np.uint32)
        x = x ^ (x >> np.uint32(15))
        x = (x * np.uint32(0x846CA68B)).astype(np.uint32)
        x = x ^ (x >> np.uint32(16))
    return x


def dropout_threshold(p: float) -> int:
    """16-bit keep threshold: a draw u16 is kept iff u16 >= round(p * 65536)."""
    return int(round(p * 65536.0))


def dropout_keep(seed: int, site: int, rows: int, cols: int, p: float) -> np.ndarray:
    """bool [rows, cols] keep mask of call site ``site`` (2*layer + 0 attention output / 1 FFN output)."""
    thr = np.uint32(dropout_threshold(p))
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    k0 = np.uint32(seed & 0xFFFFFFFF) ^ _lowbias32(np.uint32(2 * site + 1))
    k1 = np.uint32(seed >> 32) ^ _lowbias32(np.uint32(2 * site + 2))
    r = np.arange(rows, dtype=np.uint32)
    with np.errstate(over="ignore"):
        rh = _lowbias32((r * np.uint32(0x9E3779B1)).astype(np.uint32) ^ k0)
        pair = np.arange((cols + 1) // 2, dtype=np.uint32)
        u = _lowbias32(rh[:, None] ^ (pair[None, :] + k1).astype(np.uint32))
    bits = np.empty((rows, 2 * pair.size), dtype=np.uint32)
    bits[:, 0::2] = u & np.uint32(0xFFFF)
    bits[:, 1::2] = u >> np.uint32(16)
    return bits[:, :cols] >= thr


ATTN_DROP_SITE = 4096  # call site of layer l's attention probabilities: 4096 + l (paper_2411_10548_b200/model.py)


def attention_dropout_keep(seed: int, layer: int, B: int, nh: int, S: int, p: float) -> np.ndarray:
    """bool [B, nh, S(query), S(key)] keep mask of layer ``layer``'s attention probabilities: the esm_dropout bit
    of row (b*nh + h)*S + q, column k (include/esm2_b200.h, esm_attn_fwd_dropout)."""
    return dropout_keep(seed, ATTN_DROP_SITE + layer, B * nh * S, S, p).reshape(B, nh, S, S)


def forward_backward(cfg: OracleConfig, params: dict, input_ids: np.ndarray, attention_mask: np.ndarray,
                     labels: np.ndarray, dtype=np.float64, want_grads: bool = True,
                     keep_acts: bool = False, loss_denominator: float | None = None,
                     hidden_dropout: tuple | None = None, attention_dropout: tuple | None = None) -> StepResult:
    """One EsmForMaskedLM forward (+ backward) on CPU in ``dtype``.

    ``loss_denominator`` overrides the masked-token count used for the mean (the
    data-parallel global count); default = local count, as HF CrossEntropyLoss.
    ``hidden_dropout`` = (seed, p): training-mode hidden dropout with the counter-based masks of
    ``dropout_keep`` (kept values scaled by 1 / (1 - p), as nn.Dropout).
    ``attention_dropout`` = (seed, p): dropout of the softmax probabilities before P·V (HF EsmSelfAttention,
    HF:modeling_esm.py:257-282), masks from ``attention_dropout_keep``; the backward uses
    dV = (Z∘P)ᵀ dO and dS = P ∘ (Z∘dP − rowsum(Z∘P∘dP)).
    """
    P = {k: np.asarray(v, dtype=dtype) for k, v in params.items()}
    B, S = input_ids.shape
    H, nh = cfg.hidden_size, cfg.num_attention_heads
    dh = H // nh
    L = cfg.num_hidden_layers
    eps = cfg.layer_norm_eps
    ids = np.asarray(input_ids)
    am = np.asarray(attention_mask).astype(dtype)
    E = P["esm.embeddings.word_embeddings.weight"]

    # ---- embeddings (HF:modeling_esm.py:203-234)
    x = E[ids]
    is_mask = (ids == cfg.mask_token_id)
    emb_scale = np.ones((B,), dtype=dtype)
    if cfg.token_dropout:
        x = np.where(is_mask[..., None], 0.0, x)
        mask_ratio_train = 0.15 * 0.8
        src_len = am.sum(-1)
        # HF computes the observed ratio in fp32: .sum(-1).float() / src_lengths
        observed = (is_mask.sum(-1).astype(np.float32) / src_len.astype(np.float32))
        emb_scale = (1 - mask_ratio_train) / (np.float32(1) - observed).astype(dtype)
        x = x * emb_scale[:, None, None]
    x = x * am[..., None]
    keymask = np.where(am > 0, 0.0, np.finfo(dtype).min).astype(dtype)[:, None, None, :]
    cos, sin = rope_tables(S, dh)
    cos = cos.astype(dtype)[None, None]
    sin = sin.astype(dtype)[None, None]

    res = StepResult(loss=0.0, n_masked=0)
    caches = []

    def drop_mask(site):  # [B, S, H] multiplier (keep / (1 - p)), or None
        if hidden_dropout is None or hidden_dropout[1] <= 0.0:
            return None
        seed, pd = hidden_dropout
        keep = dropout_keep(seed, site, B * S, H, pd).reshape(B, S, H)
        return keep.astype(dtype) * dtype(1.0 / (1.0 - pd))

    def attn_mask(layer):  # [B, nh, S, S] multiplier of the probabilities, or None
        if attention_dropout is None or attention_dropout[1] <= 0.0:
            return None
        seed, pd = attention_dropout
        keep = attention_dropout_keep(seed, layer, B, nh, S, pd)
        return keep.astype(dtype) * dtype(1.0 / (1.0 - pd))
    for i in range(L):
        p = f"esm.encoder.layer.{i}."
        res.hidden_states.append(x)
        h1, ln1 = layer_norm(x, P[p + "attention.LayerNorm.weight"], P[p + "attention.LayerNorm.bias"], eps)

        def heads(t):
            return t.reshape(B, S, nh, dh).transpose(0, 2, 1, 3)

        q0 = heads(_linear(h1, P[p + "attention.self.query.weight"], P[p + "attention.self.query.bias"]))
        k0 = heads(_linear(h1, P[p + "attention.self.key.weight"], P[p + "attention.self.key.bias"]))
        v = heads(_linear(h1, P[p + "attention.self.value.weight"], P[p + "attention.self.value.bias"]))
        q = rope_apply(q0 * dh ** -0.5, cos, sin)
        k = rope_apply(k0, cos, sin)
        s = q @ k.transpose(0, 1, 3, 2) + keymask
        s = s - s.max(-1, keepdims=True)
        pr = np.exp(s)
        pr = pr / pr.sum(-1, keepdims=True)
        za = attn_mask(i)
        o = ((pr if za is None else pr * za) @ v).transpose(0, 2, 1, 3).reshape(B, S, H)
        m_att, m_ffn = drop_mask(2 * i), drop_mask(2 * i + 1)
        br = _linear(o, P[p + "attention.output.dense.weight"], P[p + "attention.output.dense.bias"])
        x1 = x + (br if m_att is None else br * m_att)
        h2, ln2 = layer_norm(x1, P[p + "LayerNorm.weight"], P[p + "LayerNorm.bias"], eps)
        z = _linear(h2, P[p + "intermediate.dense.weight"], P[p + "intermediate.dense.bias"])
        a = gelu(z)
        br = _linear(a, P[p + "output.dense.weight"], P[p + "output.dense.bias"])
        x2 = x1 + (br if m_ffn is None else br * m_ffn)
        caches.append(dict(x=x, ln1=ln1, h1=h1, q=q, k=k, v=v, o=o, x1=x1, ln2=ln2, h2=h2, z=z, a=a,
                           m_att=m_att, m_ffn=m_ffn, za=za))
        if keep_acts:
            res.acts[i] = dict(h1=h1, q=q, k=k, v=v, o=o, x1=x1, h2=h2, z=z, a=a)
        x = x2
    res.hidden_states.append(x)
    xf, lnf = layer_norm(x, P["esm.encoder.emb_layer_norm_after.weight"], P["esm.encoder.emb_layer_norm_after.bias"], eps)
    # ---- LM head (HF:modeling_esm.py:808-815)
    y = _linear(xf, P["lm_head.dense.weight"], P["lm_head.dense.bias"])
    g = gelu(y)
    n, lnh = layer_norm(g, P["lm_head.layer_norm.weight"], P["lm_head.layer_norm.bias"], eps)
    logits = n @ E.T + P["lm_head.bias"]
    res.logits = logits
    if keep_acts:
        res.acts["final"] = dict(xf=xf, y=y, g=g, n=n)

    # ---- masked CE, mean over labelled tokens (HF:modeling_esm.py:777-784)
    lab = np.asarray(labels).reshape(-1)
    lg = logits.reshape(-1, cfg.vocab_size)
    sel = lab != -100
    n_masked = int(sel.sum())
    denom = float(loss_denominator) if loss_denominator is not None else float(max(n_masked, 1))
    m = lg.max(-1, keepdims=True)
    lse = (m + np.log(np.exp(lg - m).sum(-1, keepdims=True)))[:, 0]
    tgt = np.where(sel, lab, 0)
    nll = lse - lg[np.arange(lg.shape[0]), tgt]
    res.loss = float((nll * sel).sum() / denom) if n_masked else float("nan")
    res.n_masked = n_masked
    if not want_grads:
        return res

    # ================= backward =================
    G = {k: np.zeros_like(v) for k, v in P.items()}
    prob = np.exp(lg - lse[:, None])
    dlg = prob.copy()
    dlg[np.arange(lg.shape[0]), tgt] -= 1.0
    dlg *= (sel / denom)[:, None]
    dlg = dlg.reshape(B, S, -1)
    G["lm_head.bias"] += dlg.sum((0, 1))
    G["esm.embeddings.word_embeddings.weight"] += _wgrad(dlg, n)
    dn = dlg @ E
    dg, G["lm_head.layer_norm.weight"], G["lm_head.layer_norm.bias"] = layer_norm_bwd(dn, P["lm_head.layer_norm.weight"], lnh)
    dy = dg * gelu_grad(y)
    G["lm_head.dense.weight"] = _wgrad(dy, xf)
    G["lm_head.dense.bias"] = dy.sum((0, 1))
    dxf = dy @ P["lm_head.dense.weight"]
    dx, G["esm.encoder.emb_layer_norm_after.weight"], G["esm.encoder.emb_layer_norm_after.bias"] = \
        layer_norm_bwd(dxf, P["esm.encoder.emb_layer_norm_after.weight"], lnf)

    for i in reversed(range(L)):
        p = f"esm.encoder.layer.{i}."
        c = caches[i]
        # FFN (the branch gradient passes the dropout mask; the residual gradient does not)
        dbr = dx if c["m_ffn"] is None else dx * c["m_ffn"]
        G[p + "output.dense.weight"] = _wgrad(dbr, c["a"])
        G[p + "output.dense.bias"] = dbr.sum((0, 1))
        da = dbr @ P[p + "output.dense.weight"]
        dz = da * gelu_grad(c["z"])
        G[p + "intermediate.dense.weight"] = _wgrad(dz, c["h2"])
        G[p + "intermediate.dense.bias"] = dz.sum((0, 1))
        dh2 = dz @ P[p + "intermediate.dense.weight"]
        dx1, G[p + "LayerNorm.weight"], G[p + "LayerNorm.bias"] = layer_norm_bwd(dh2, P[p + "LayerNorm.weight"], c["ln2"])
        dx1 = dx1 + dx
        # attention output projection
        dbr = dx1 if c["m_att"] is None else dx1 * c["m_att"]
        G[p + "attention.output.dense.weight"] = _wgrad(dbr, c["o"])
        G[p + "attention.output.dense.bias"] = dbr.sum((0, 1))
        do = (dbr @ P[p + "attention.output.dense.weight"]).reshape(B, S, nh, dh).transpose(0, 2, 1, 3)
        # attention core (recompute P, flash-style)
        q, k, v = c["q"], c["k"], c["v"]
        s = q @ k.transpose(0, 1, 3, 2) + keymask
        s = s - s.max(-1, keepdims=True)
        pr = np.exp(s)
        pr = pr / pr.sum(-1, keepdims=True)
        za = c["za"]
        dv = (pr if za is None else pr * za).transpose(0, 1, 3, 2) @ do
        dp = do @ v.transpose(0, 1, 3, 2)
        if za is not None:
            dp = dp * za
        ds = pr * (dp - (dp * pr).sum(-1, keepdims=True))
        dq = ds @ k
        dk = ds.transpose(0, 1, 3, 2) @ q
        dq0 = rope_apply_bwd(dq, cos, sin) * dh ** -0.5
        dk0 = rope_apply_bwd(dk, cos, sin)

        def unheads(t):
            return t.transpose(0, 2, 1, 3).reshape(B, S, H)

        dq0, dk0, dv = unheads(dq0), unheads(dk0), unheads(dv)
        h1 = c["h1"]
        dh1 = np.zeros_like(h1)
        for nm, dt in (("query", dq0), ("key", dk0), ("value", dv)):
            G[p + f"attention.self.{nm}.weight"] = _wgrad(dt, h1)
            G[p + f"attention.self.{nm}.bias"] = dt.sum((0, 1))
            dh1 += dt @ P[p + f"attention.self.{nm}.weight"]
        dx0, G[p + "attention.LayerNorm.weight"], G[p + "attention.LayerNorm.bias"] = \
            layer_norm_bwd(dh1, P[p + "attention.LayerNorm.weight"], c["ln1"])
        dx = dx0 + dx1

    # embeddings backward: x = E[ids] * keep * scale * am ; padding_idx row gets no grad
    dxe = dx * am[..., None] * emb_scale[:, None, None]
    if cfg.token_dropout:
        dxe = np.where(is_mask[..., None], 0.0, dxe)
    dxe = np.where((ids == cfg.pad_token_id)[..., None], 0.0, dxe)
    np.add.at(G["esm.embeddings.word_embeddings.weight"], ids.reshape(-1), dxe.reshape(-1, H))
    res.grads = G
    return res


# --------------------------------------------------------------------------
# AdamW (torch.optim.AdamW semantics)
# --------------------------------------------------------------------------
def no_decay(name: str) -> bool:
    """Biases, LayerNorm parameters and the LM-head bias are not weight-decayed."""
    return name.endswith("bias") or "LayerNorm" in name or "layer_norm" in name


def adamw_update(params, grads, m, v, step, lr, beta1=0.9, beta2=0.98, eps=1e-8, weight_decay=0.01,
                 grad_scale=1.0):
    """In-place fp32 AdamW over dicts of arrays (torch.optim.AdamW, decoupled decay)."""
    bc1 = 1.0 - beta1 ** step
    bc2 = 1.0 - beta2 ** step
    for k in params:
        g = grads[k].astype(np.float32) * np.float32(grad_scale)
        p = params[k]
        wd = 0.0 if no_decay(k) else weight_decay
        p *= np.float32(1.0 - lr * wd)
        m[k] = np.float32(beta1) * m[k] + np.float32(1 - beta1) * g
        v[k] = np.float32(beta2) * v[k] + np.float32(1 - beta2) * g * g
        denom = np.sqrt(v[k]) / np.float32(math.sqrt(bc2)) + np.float32(eps)
        p -= np.float32(lr / bc1) * m[k] / denom


def esm2_lr(step: int, peak_lr: float = 4e-4, warmup: int = 2000, total: int = 500_000, final_ratio: float = 0.1):
    """ESM-2 schedule: linear warmup to peak, then linear decay to final_ratio*peak."""
    if step <= warmup:
        return peak_lr * step / max(1, warmup)
    frac = min(1.0, (step - warmup) / max(1, total - warmup))
    return peak_lr * (1.0 - (1.0 - final_ratio) * frac)


class OracleTrainer:
    """fp32 master weights + AdamW over forward_backward(); the CPU train step."""

    def __init__(self, cfg: OracleConfig, params: dict, lr=4e-4, dtype=np.float32, **adam):
        self.cfg, self.lr, self.dtype, self.adam = cfg, lr, dtype, adam
        self.params = {k: v.astype(np.float32).copy() for k, v in params.items()}
        self.m = {k: np.zeros_like(v) for k, v in self.params.items()}
        self.v = {k: np.zeros_like(v) for k, v in self.params.items()}
        self.step_count = 0

    def step(self, input_ids, attention_mask, labels, lr=None):
        r = forward_backward(self.cfg, self.params, input_ids, attention_mask, labels, dtype=self.dtype)
        self.step_count += 1
        adamw_update(self.params, r.grads, self.m, self.v, self.step_count,
                     self.lr if lr is None else lr, **self.adam)
        return r.loss


def train_flops_per_token(cfg: OracleConfig, seq_len: int) -> float:
    """6*N_mm + 12*L*H*S."""
    H, F, V, L = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers
    n_mm = L * (4 * H * H + 2 * H * F) + H * H + H * V
    return 6.0 * n_mm + 12.0 * L * H * seq_len
