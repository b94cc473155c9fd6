"""B200-native ESM-2 masked-LM: parameters, activation workspace and the train step.

PyTorch is used only for device memory, streams and (optionally) torch.distributed;
every FLOP of the step runs in the hand-written sm_100a kernels of
``libesm2b200.so`` through the C ABI declared in ``include/esm2_b200.h``.

Semantics follow Hugging Face ``EsmForMaskedLM`` (transformers 5.5.0,
``models/esm/modeling_esm.py``; "HF:" below):

  embeddings + token_dropout + pad mask       HF:189-236     esm_embed_fwd / esm_embed_bwd
  pre-LN (attention.LayerNorm / LayerNorm)    HF:384,394,479 esm_layernorm_fwd / _bwd
  q,k,v projections, q*dh^-0.5, RoPE          HF:318-344     esm_gemm(QKV_ROPE epilogue) (fp32: + esm_qkv_rope_fwd)
  softmax(QKᵀ + key mask)·V, scaling=1        HF:257-282     esm_attn_fwd / esm_attn_bwd
  out-proj + residual                         HF:365-375     esm_gemm(RESID)
  FC1 + erf-GELU, FC2 + residual              HF:406-427     esm_gemm(GELU_GRADAUX / GELU), esm_gemm(RESID)
  emb_layer_norm_after                        HF:511-512     esm_layernorm_fwd
  LM head dense+GELU+LN, tied decoder + bias  HF:808-815     esm_gemm(GELU) + LN + esm_lmhead_xent
  masked CE (ignore -100, mean)               HF:777-784     esm_lmhead_xent
  AdamW                                       torch.optim.AdamW semantics      esm_adamw

Parameter memory layout (HBM): one flat fp32 master buffer (+ bf16 shadow for GEMM
operands, + fp32 grad, Adam m, v), every parameter group 256-element aligned; groups are
ordered in *backward completion order* (LM head first, layers L-1..0, word embeddings
last) so that data-parallel gradient buckets are contiguous slices that become ready
one after another during backward.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import (EPI_DELTA, EPI_DGELU, EPI_F32_ACC, EPI_GELU, EPI_GELU_GRADAUX, EPI_MUL_AUX, EPI_QKV_ROPE,
                   EPI_RESID, EPI_STORE, EPI_STORE_LN, ESM_BF16, ESM_F32)
from .config import EsmConfig

ALIGN = 256  # elements; also the AdamW weight-decay chunk size
TOTAL_ALIGN = 8 * ALIGN  # the flat buffer splits into 1, 2, 4 or 8 data-parallel shards of whole chunks
LARGE_VOCAB = 40  # esm_lmhead_xent's per-row fused head handles V <= 40; larger V uses the GEMM head
ATTN_DROP_SITE = 4096  # esm_dropout call sites of the attention probabilities: 4096 + layer (hidden: 2*layer + 0/1)


def head_capacity(T: int) -> int:
    """Rows reserved for the labelled-row decoder: E[#labels] = 0.15*T (selection probability
    2516582/2^24), std <= 0.36*sqrt(T); 8*sqrt(T) + 64 of headroom is > 20 sigma.  Batches staged with
    explicit labels are checked against it on the host (set_batch)."""
    return min(T, (int(0.15 * T + 8.0 * math.sqrt(T) + 64) + 127) // 128 * 128)


def _no_decay(name: str) -> bool:
    return name.endswith("bias") or "LayerNorm" in name or "layer_norm" in name


def param_groups(cfg: EsmConfig):
    """[(group_key, [(hf_name, shape), ...])] in backward-completion order."""
    H, F, V, L = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers
    g = [
        ("lm_head.bias", [("lm_head.bias", (V,))]),
        ("lm_head.layer_norm.weight", [("lm_head.layer_norm.weight", (H,))]),
        ("lm_head.layer_norm.bias", [("lm_head.layer_norm.bias", (H,))]),
        ("lm_head.dense.weight", [("lm_head.dense.weight", (H, H))]),
        ("lm_head.dense.bias", [("lm_head.dense.bias", (H,))]),
        ("esm.encoder.emb_layer_norm_after.weight", [("esm.encoder.emb_layer_norm_after.weight", (H,))]),
        ("esm.encoder.emb_layer_norm_after.bias", [("esm.encoder.emb_layer_norm_after.bias", (H,))]),
    ]
    for i in reversed(range(L)):
        p = f"esm.encoder.layer.{i}."
        for n, shp in [("output.dense.weight", (H, F)), ("output.dense.bias", (H,)),
                       ("intermediate.dense.weight", (F, H)), ("intermediate.dense.bias", (F,)),
                       ("LayerNorm.weight", (H,)), ("LayerNorm.bias", (H,)),
                       ("attention.output.dense.weight", (H, H)), ("attention.output.dense.bias", (H,))]:
            g.append((p + n, [(p + n, shp)]))
        g.append((p + "attention.self.qkv.weight",
                  [(p + f"attention.self.{n}.weight", (H, H)) for n in ("query", "key", "value")]))
        g.append((p + "attention.self.qkv.bias",
                  [(p + f"attention.self.{n}.bias", (H,)) for n in ("query", "key", "value")]))
        g.append((p + "attention.LayerNorm.weight", [(p + "attention.LayerNorm.weight", (H,))]))
        g.append((p + "attention.LayerNorm.bias", [(p + "attention.LayerNorm.bias", (H,))]))
    g.append(("esm.embeddings.word_embeddings.weight", [("esm.embeddings.word_embeddings.weight", (V, H))]))
    return g


def init_params(cfg: EsmConfig, seed: int) -> dict:
    """HF init (normal(0, initializer_range) weights, zero biases, LN (1,0), zero pad row), drawn with
    numpy default_rng(seed) in HF state-dict order -- the same draws as the CPU oracle uses."""
    H, F, V, L = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers
    shapes = {"esm.embeddings.word_embeddings.weight": (V, H)}
    for i in range(L):
        p = f"esm.encoder.layer.{i}."
        for n in ("query", "key", "value"):
            shapes[p + f"attention.self.{n}.weight"] = (H, H)
            shapes[p + f"attention.self.{n}.bias"] = (H,)
        shapes.update({p + "attention.output.dense.weight": (H, H), p + "attention.output.dense.bias": (H,),
                       p + "attention.LayerNorm.weight": (H,), p + "attention.LayerNorm.bias": (H,),
                       p + "intermediate.dense.weight": (F, H), p + "intermediate.dense.bias": (F,),
                       p + "output.dense.weight": (H, F), p + "output.dense.bias": (H,),
                       p + "LayerNorm.weight": (H,), p + "LayerNorm.bias": (H,)})
    shapes.update({"esm.encoder.emb_layer_norm_after.weight": (H,), "esm.encoder.emb_layer_norm_after.bias": (H,),
                   "lm_head.dense.weight": (H, H), "lm_head.dense.bias": (H,),
                   "lm_head.layer_norm.weight": (H,), "lm_head.layer_norm.bias": (H,), "lm_head.bias": (V,)})
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in shapes.items():
        if name.endswith("LayerNorm.weight") or name.endswith("layer_norm.weight") or \
                name.endswith("emb_layer_norm_after.weight"):
            out[name] = np.ones(shape, np.float32)
        elif len(shape) == 2:
            out[name] = (rng.standard_normal(shape, dtype=np.float32) * np.float32(cfg.initializer_range))
        else:
            out[name] = np.zeros(shape, np.float32)
    out["esm.embeddings.word_embeddings.weight"][cfg.pad_token_id] = 0.0
    return out


def rope_tables(seq_len: int, dim: int):
    """HF RotaryEmbedding (HF:modeling_esm.py:91-111) in fp32: returns cos, sin [S, dim/2]
    (the table is cat(freqs, freqs), so the first half suffices)."""
    inv_freq = (1.0 / (np.float32(10000.0) ** (np.arange(0, dim, 2, dtype=np.int64).astype(np.float32)
                                                 / np.float32(dim)))).astype(np.float32)
    t = np.arange(seq_len, dtype=np.float32)
    freqs = np.outer(t, inv_freq).astype(np.float32)
    return np.cos(freqs).astype(np.float32), np.sin(freqs).astype(np.float32)


@dataclass
class _Slot:
    offset: int
    numel: int
    shape: tuple
    group: str


class ParamStore:
    """Flat fp32 master / bf16 shadow / fp32 grad / Adam moments, 256-element aligned groups."""

    def __init__(self, cfg: EsmConfig, device, shadow: bool):
        self.groups = param_groups(cfg)
        self.slots: dict[str, _Slot] = {}
        self.group_range: dict[str, tuple[int, int]] = {}
        off = 0
        decay = []
        for key, members in self.groups:
            start = off
            for name, shape in members:
                n = int(np.prod(shape))
                self.slots[name] = _Slot(off, n, tuple(shape), key)
                off += n
            end = off
            off = (off + ALIGN - 1) // ALIGN * ALIGN
            self.group_range[key] = (start, end)
            d = 0 if _no_decay(members[0][0]) else 1
            decay += [d] * ((off - start) // ALIGN)
        total = (off + TOTAL_ALIGN - 1) // TOTAL_ALIGN * TOTAL_ALIGN  # data-parallel shards: world | 8
        decay += [0] * ((total - off) // ALIGN)
        off = total
        self.numel = off
        self.device = device
        self.p32 = torch.zeros(off, dtype=torch.float32, device=device)
        self.g32 = torch.zeros(off, dtype=torch.float32, device=device)
        self.m = torch.zeros(off, dtype=torch.float32, device=device)
        self.v = torch.zeros(off, dtype=torch.float32, device=device)
        self.p16 = torch.zeros(off, dtype=torch.bfloat16, device=device) if shadow else None
        self.decay = torch.tensor(decay, dtype=torch.uint8, device=device)

    def view(self, buf, name):
        s = self.slots[name]
        return buf[s.offset:s.offset + s.numel].view(s.shape)

    def group_view(self, buf, key, shape):
        a, b = self.group_range[key]
        return buf[a:b].view(shape)


class _Layer:
    pass


class _Arena:
    """Bump allocator over one device buffer that backs the activation / scratch tensors of the workspaces of
    every (B, S) shape.  Steps are stream-ordered (one shape's step runs at a time) and every step re-stages its
    inputs, so bucketed variable-shape training caches many shapes -- each with its own CUDA graph -- in the
    memory of the largest one.  ``buf=None`` only measures."""

    ALIGN = 1024  # bytes: TMA needs 16 B; 1 KB keeps every tensor on its own swizzle atom

    def __init__(self, buf: torch.Tensor | None):
        self.buf = buf
        self.off = 0

    def take(self, shape, dtype):
        n = math.prod(shape) * torch.empty((), dtype=dtype).element_size()
        off = (self.off + self.ALIGN - 1) // self.ALIGN * self.ALIGN
        self.off = off + n
        if self.buf is None:
            return None
        if self.off > self.buf.numel():
            raise RuntimeError("activation arena too small for this workspace")
        return self.buf[off:off + n].view(dtype).view(*shape)


class Workspace:
    """Activation / gradient buffers for one (B, S) shape; reused every step.

    Inputs and per-shape constants (ids, masks, labels, counters, RoPE tables) are owned by the workspace;
    activations and backward scratch live in ``arena`` (shared across shapes) when one is given."""

    def __init__(self, cfg: EsmConfig, B: int, S: int, act, device, arena: _Arena | None = None):
        H, F, V, L, nh = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers, \
            cfg.num_attention_heads
        dh = H // nh
        T = B * S
        self.B, self.S, self.T = B, S, T
        self.arena_bytes = 0
        if arena is not None:
            arena.off = 0
            e = lambda *shape, dt=act: arena.take(shape, dt)  # noqa: E731
        else:
            e = lambda *shape, dt=act: torch.empty(*shape, dtype=dt, device=device)  # noqa: E731
        f32, i32 = torch.float32, torch.int32
        self.ids = torch.zeros(B, S, dtype=i32, device=device)        # raw (unmasked) tokens
        self.input_ids = torch.zeros(B, S, dtype=i32, device=device)  # after MLM masking
        self.labels = torch.full((B, S), -100, dtype=i32, device=device)
        self.am = torch.ones(B, S, dtype=i32, device=device)
        self.n_labels = torch.zeros(1, dtype=i32, device=device)         # this rank's labelled tokens
        self.n_labels_global = torch.zeros(1, dtype=i32, device=device)  # all ranks' (the loss normaliser)
        self.inv_denom = torch.zeros(1, dtype=f32, device=device)
        self.loss_sum = torch.zeros(1, dtype=f32, device=device)
        self.row_scale = e(B, dt=f32)
        # attention scheduling workspace (per-row key-prefix info + persistent-kernel work counters); filled by
        # esm_attn_prepare once per step, shared by every layer's forward and backward on this stream
        self.attn_sched = torch.zeros(_lib.attn_sched_words(B), dtype=i32, device=device)
        self.x = [e(T, H) for _ in range(L + 1)]  # residual stream: input of layer l; x[L] = encoder output
        self.layers = []
        for _ in range(L):
            ly = _Layer()
            ly.ln1_m, ly.ln1_r = e(T, dt=f32), e(T, dt=f32)
            ly.h1 = e(T, H)
            ly.q, ly.k, ly.v = e(B, nh, S, dh), e(B, nh, S, dh), e(B, nh, S, dh)
            ly.o = e(T, H)
            ly.lse = e(B, nh, S, dt=f32)
            ly.x1 = e(T, H)
            ly.ln2_m, ly.ln2_r = e(T, dt=f32), e(T, dt=f32)
            ly.h2 = e(T, H)
            ly.z, ly.a = e(T, F), e(T, F)
            self.layers.append(ly)
        self.qkv = e(T, 3 * H)
        self.lnf_m, self.lnf_r = e(T, dt=f32), e(T, dt=f32)
        self.xf = e(T, H)
        self.y, self.g = e(T, H), e(T, H)
        self.lnh_m, self.lnh_r = e(T, dt=f32), e(T, dt=f32)
        self.n = e(T, H)
        # backward scratch
        self.dn = e(T, H)
        self.large_vocab = V > LARGE_VOCAB
        if self.large_vocab:  # decoder on labelled rows only (esm_label_compact / gather / GEMM / xent_rows)
            self.cap = head_capacity(T)
            self.Vp = (V + 7) // 8 * 8
            self.head_idx = torch.full((self.cap,), -1, dtype=i32, device=device)
            self.head_lab = torch.full((self.cap,), -100, dtype=i32, device=device)
            self.head_count = torch.zeros(1, dtype=i32, device=device)
            self.n_lab = e(self.cap, H)
            self.logits = e(self.cap, self.Vp)  # overwritten in place by dlogits
            self.dn_lab = e(self.cap, H)
            self.dlogits = None
        else:
            self.dlogits = e(T, V, dt=f32)
        self.dy = e(T, H)
        self.dx = e(T, H)
        self.dx_alt = e(T, H)
        self.dh = e(T, H)
        self.dz = e(T, F)
        self.dx1 = e(T, H)
        self.do = e(T, H)
        # gradient of a dropped-out branch (hidden dropout): written by the LayerNorm backward, read by the
        # branch's dgrad / wgrad GEMMs
        self.dxd = e(T, H) if cfg.hidden_dropout_prob > 0 else None
        self.dq = e(B, nh, S, dh, dt=f32)
        self.dk, self.dv = e(B, nh, S, dh), e(B, nh, S, dh)
        self.dqkv = e(T, 3 * H)
        self.delta = e(2, B, nh, S, dt=f32)  # Delta = rowsum(dO o O) per head (attention backward workspace)
        cos, sin = rope_tables(S, dh)
        self.cos = torch.from_numpy(cos).to(device)
        self.sin = torch.from_numpy(sin).to(device)
        if arena is not None:
            self.arena_bytes = arena.off

    @staticmethod
    def activation_bytes(cfg: EsmConfig, B: int, S: int, act) -> int:
        """Arena bytes the workspace of shape (B, S) needs (measuring pass, no device allocation of them)."""
        a = _Arena(None)
        Workspace(cfg, B, S, act, "cpu", arena=a)
        return a.off


class EsmForMaskedLM:
    """B200 ESM-2 MLM with a fused train step.

    dtype="bf16": bf16 activations / GEMM operands, fp32 accumulation, fp32 master weights,
                  fp32 gradients (production path: tcgen05 GEMMs, persistent tcgen05 flash attention).
    dtype="fp32": fp32 everywhere (SIMT kernels) -- the parity mode checked against the oracle.
    """

    def __init__(self, config: EsmConfig, dtype: str = "bf16", device=None, seed: int = 1,
                 lr: float = 4e-4, betas=(0.9, 0.98), eps: float = 1e-8, weight_decay: float = 0.01,
                 params: dict | None = None):
        _lib.load()
        self.config = config.validate()
        if dtype not in ("bf16", "fp32"):
            raise ValueError("dtype must be 'bf16' or 'fp32'")
        self.dtype = dtype
        self.kdt = ESM_BF16 if dtype == "bf16" else ESM_F32
        self.act = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if self.device.type != "cuda":
            raise _lib.EsmKernelError("EsmForMaskedLM runs only on a CUDA (sm_100a) device")
        self.store = ParamStore(self.config, self.device, shadow=(dtype == "bf16"))
        self.load_state_dict(params if params is not None else init_params(self.config, seed))
        self.lr, self.betas, self.eps, self.weight_decay = lr, tuple(betas), eps, weight_decay
        self.hyper = torch.zeros(8, dtype=torch.float32, device=self.device)
        # hidden dropout: per-step 64-bit seed in device memory (read by the kernels: CUDA-graph safe)
        self.dropout_p = float(self.config.hidden_dropout_prob)
        # attention-probability dropout (HF EsmSelfAttention, dropout(softmax(S)) @ V): the tcgen05 kernels apply
        # and regenerate the counter-based mask (esm_attn_*_dropout; the fp32 parity kernels too)
        self.attn_dropout_p = float(self.config.attention_probs_dropout_prob)
        self.dropout_base = (int(seed) * 0x9E3779B97F4A7C15 + 0xD1B54A32D192ED03) & 0xFFFFFFFFFFFFFFFF
        self.drop_seed = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.last_dropout_seed = 0
        self.step_count = 0
        self.grad_scale = 1.0
        self.ws: Workspace | None = None
        self._ws_cache: dict = {}
        self._arena: torch.Tensor | None = None  # activation arena shared by the cached workspaces
        self.max_workspaces = 32  # cached (B, S) shapes (small: inputs, constants, CUDA graph)
        self.comm = None  # set by ddp.GradAllReducer
        self.timer = None  # optional KernelTimer (bench.py per-kernel roofline)
        self._opt_on, self._opt_start, self._opt_stream = False, 0, None
        self._zero_stream = None
        self.launches = 0  # kernels launched by this model (C-ABI calls x kernels per call)
        self.nvtx = False  # NVTX ranges (forward / backward / layers) for nsys-style timelines
        self.graph = None
        self.graph_launches = 0
        self._hyper_ring = [torch.zeros(8, dtype=torch.float32).pin_memory() for _ in range(4)]
        self._hyper_ev = [None] * 4
        self._hyper_i = 0

    # ------------------------------------------------------------------ parameters
    def load_state_dict(self, sd: dict):
        for name, slot in self.store.slots.items():
            if name not in sd:
                raise KeyError(f"missing parameter {name}")
            t = torch.as_tensor(np.asarray(sd[name], dtype=np.float32)).reshape(slot.shape)
            self.store.view(self.store.p32, name).copy_(t.to(self.device))
        self.refresh_shadow()

    def refresh_shadow(self):
        if self.store.p16 is not None:
            _lib.call("esm_cast_f32_bf16", self.store.p32.data_ptr(), self.store.p16.data_ptr(), self.store.numel,
                      self._stream())

    def state_dict(self) -> dict:
        """fp32 master weights by HF name (under ZeRO-1 the sharded master is all-gathered first)."""
        if self.comm is not None and hasattr(self.comm, "gather_master"):
            self.comm.gather_master()
        return {n: self.store.view(self.store.p32, n).detach().cpu().clone() for n in self.store.slots}

    def grads(self) -> dict:
        return {n: self.store.view(self.store.g32, n) for n in self.store.slots}

    def num_parameters(self) -> int:
        return sum(s.numel for s in self.store.slots.values())

    def _w(self, key, shape):
        """GEMM operand view of a weight group (bf16 shadow or fp32 master)."""
        buf = self.store.p16 if self.store.p16 is not None else self.store.p32
        return self.store.group_view(buf, key, shape)

    def _p32(self, key, shape=None):
        a, b = self.store.group_range[key]
        return self.store.p32[a:b]

    def _g32(self, key):
        a, b = self.store.group_range[key]
        return self.store.g32[a:b]

    # ------------------------------------------------------------------ plumbing
    def _stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    def workspace(self, B: int, S: int) -> Workspace:
        """Activation workspace for a (B, S) shape.  Variable-shape training (bucketed batches) keeps an
        LRU cache of up to ``max_workspaces`` shapes, each with its own CUDA graph once captured."""
        key = (B, S)
        cache = self._ws_cache
        if key in cache:
            cache[key] = cache.pop(key)  # most recently used
        else:
            self.reserve(B, S)
            while len(cache) >= self.max_workspaces:
                old_key = next(iter(cache))
                old = cache.pop(old_key)
                if self.ws is old:
                    self.ws = None
                del old
            cache[key] = Workspace(self.config, B, S, self.act, self.device, arena=_Arena(self._arena))
        self.ws = cache[key]
        return self.ws

    def reserve(self, B: int, S: int):
        """Grow the shared activation arena to hold a (B, S) workspace.  Growing drops the cached workspaces
        (their CUDA graphs point into the old arena); reserving the largest bucket shape up front avoids that."""
        need = Workspace.activation_bytes(self.config, B, S, self.act)
        if self._arena is not None and self._arena.numel() >= need:
            return
        self._ws_cache.clear()
        self.ws = None
        self.graph = None
        self._arena = None
        torch.cuda.empty_cache()
        self._arena = torch.empty(need, dtype=torch.uint8, device=self.device)

    def release_workspaces(self):
        """Free every cached activation workspace (and its CUDA graph) and the activation arena."""
        self._ws_cache.clear()
        self.ws = None
        self.graph = None
        self._arena = None
        torch.cuda.empty_cache()

    def _nvtx(self, name, pop_first: bool = False):
        """NVTX ranges around the step's phases and layers (``model.nvtx = True``; host-side only, so they also
        appear around graph capture).  name=None pops."""
        if not self.nvtx:
            return
        if name is None or pop_first:
            torch.cuda.nvtx.range_pop()
        if name is not None:
            torch.cuda.nvtx.range_push(name)

    # kernels launched per C-ABI entry point (for the bench's gpu_launches count)
    _KERNELS = {"esm_embed_fwd": 2, "esm_attn_bwd": 3, "esm_attn_bwd_qkv": 4, "esm_lmhead_xent": 2}

    def _call(self, name, *args, flops=0.0, nbytes=0.0):
        t = self.timer
        if t is not None:
            t.begin(name)
        _lib.call(name, *args)
        if t is not None:
            t.end(flops, nbytes)
        self.launches += self._KERNELS.get(name, 1)

    def _gemm(self, M, N, K, A, lda, amn, B, ldb, bmn, C, ldc, epi, bias=None, aux_in=None, ld_aux_in=0,
              aux_out=None, ld_aux_out=0, col_sum=None, ln=None, drop=None, delta=None):
        t = self.timer
        if t is not None:
            kind = "gemm_" + ("wgrad" if epi == EPI_F32_ACC else "dgrad" if bmn else "fwd")
            if os.environ.get("ESM_TIMER_DETAIL"):
                kind += f"_{M}x{N}x{K}_e{epi}"
            t.begin(kind)
        self.launches += 1
        self._gemm_raw(M, N, K, A, lda, amn, B, ldb, bmn, C, ldc, epi, bias, aux_in, ld_aux_in, aux_out, ld_aux_out,
                       col_sum, ln, drop, delta)
        if t is not None:
            t.end(2.0 * M * N * K, 0.0)

    def _gemm_raw(self, M, N, K, A, lda, amn, B, ldb, bmn, C, ldc, epi, bias, aux_in, ld_aux_in, aux_out,
                  ld_aux_out, col_sum, ln=None, drop=None, delta=None):
        if ln is not None:  # (row_mean, row_rstd, dgamma accumulator)
            _lib.gemm_call(self._stream(), dtype=self.kdt, M=M, N=N, K=K, A=A.data_ptr(), lda=lda, a_mn_major=amn,
                           B=B.data_ptr(), ldb=ldb, b_mn_major=bmn, C=C.data_ptr(), ldc=ldc, epilogue=epi,
                           aux_in=aux_in.data_ptr(), ld_aux_in=ld_aux_in, col_sum=col_sum.data_ptr(),
                           row_mean=ln[0].data_ptr(), row_rstd=ln[1].data_ptr(), col_sum2=ln[2].data_ptr())
            return
        _lib.gemm_call(self._stream(), dtype=self.kdt, M=M, N=N, K=K, A=A.data_ptr(), lda=lda, a_mn_major=amn,
                       B=B.data_ptr(), ldb=ldb, b_mn_major=bmn, C=C.data_ptr(), ldc=ldc, epilogue=epi,
                       bias=bias.data_ptr() if bias is not None else None,
                       aux_in=aux_in.data_ptr() if aux_in is not None else None, ld_aux_in=ld_aux_in,
                       aux_out=aux_out.data_ptr() if aux_out is not None else None, ld_aux_out=ld_aux_out,
                       col_sum=col_sum.data_ptr() if col_sum is not None else None, split_k=0,
                       **({"drop": drop} if drop is not None else {}),
                       **({"row_dot": delta[0].data_ptr(), "seq_len": delta[1], "n_heads": delta[2],
                           "head_dim": delta[3]} if delta is not None else {}))

    def linear_fwd(self, x, wkey, out_f, in_f, bias_key, C, epi=EPI_STORE, aux_in=None, aux_out=None, drop=None):
        T = x.shape[0]
        W = self._w(wkey, (out_f, in_f))
        self._gemm(T, out_f, in_f, x, in_f, 0, W, in_f, 0, C, out_f, epi,
                   bias=self._p32(bias_key) if bias_key else None, aux_in=aux_in, ld_aux_in=out_f,
                   aux_out=aux_out, ld_aux_out=out_f, drop=drop)

    def _qkv_rope_gemm(self, ly, p, ws, T, H, nh, dh, S, qs):
        W = self._w(p + "attention.self.qkv.weight", (3 * H, H))
        t = self.timer
        if t is not None:
            t.begin("gemm_fwd" + (f"_{T}x{3 * H}x{H}_qkvrope" if os.environ.get("ESM_TIMER_DETAIL") else ""))
        _lib.gemm_call(self._stream(), dtype=self.kdt, M=T, N=3 * H, K=H, A=ly.h1.data_ptr(), lda=H, a_mn_major=0,
                       B=W.data_ptr(), ldb=H, b_mn_major=0, C=None, ldc=0, epilogue=EPI_QKV_ROPE,
                       bias=self._p32(p + "attention.self.qkv.bias").data_ptr(), rope_cos=ws.cos.data_ptr(),
                       rope_sin=ws.sin.data_ptr(), q_out=ly.q.data_ptr(), k_out=ly.k.data_ptr(),
                       v_out=ly.v.data_ptr(), seq_len=S, n_heads=nh, head_dim=dh, q_scale=qs)
        if t is not None:
            t.end(2.0 * T * 3 * H * H, 0.0)
        self.launches += 1

    def linear_dgrad(self, dy, wkey, out_f, in_f, dX, epi=EPI_STORE, aux_in=None, col_sum=None, ln=None):
        """dX = dy · W.  ln = (ln_input, mean, rstd, ln_key): dX is that LayerNorm's output gradient and the
        epilogue also accumulates its dbeta / dgamma (bf16 path)."""
        T = dy.shape[0]
        W = self._w(wkey, (out_f, in_f))
        if ln is not None and self.kdt == ESM_BF16:
            x_in, mu, rs, key = ln
            self._gemm(T, in_f, out_f, dy, out_f, 0, W, in_f, 1, dX, in_f, EPI_STORE_LN, aux_in=x_in,
                       ld_aux_in=in_f, col_sum=self._g32(key + ".bias"), ln=(mu, rs, self._g32(key + ".weight")))
            return True
        self._gemm(T, in_f, out_f, dy, out_f, 0, W, in_f, 1, dX, in_f, epi, aux_in=aux_in, ld_aux_in=in_f,
                   col_sum=col_sum)
        return False

    def linear_wgrad(self, dy, x, wkey, out_f, in_f):
        T = dy.shape[0]
        self._gemm(out_f, in_f, T, dy, out_f, 1, x, in_f, 1, self._g32(wkey), in_f, EPI_F32_ACC)

    # ------------------------------------------------------------------ data path
    def mlm_mask(self, ids: torch.Tensor, seed: int, stream_id: int, ws: Workspace | None = None):
        """Device MLM masking (15% / 80-10-10) into the workspace; counts labelled tokens."""
        ws = ws or self.workspace(*ids.shape)
        if ids.data_ptr() != ws.ids.data_ptr():
            ws.ids.copy_(ids, non_blocking=True)
        ws.n_labels.zero_()
        cfg = self.config
        _lib.call("esm_mlm_mask_ex", ws.ids.data_ptr(), ws.input_ids.data_ptr(), ws.labels.data_ptr(),
                  ws.n_labels.data_ptr(), ws.ids.numel(), seed & 0xFFFFFFFFFFFFFFFF, stream_id & 0xFFFFFFFFFFFFFFFF,
                  cfg.mlm_eligible[0], cfg.mlm_eligible[1], cfg.mask_token_id, cfg.mlm_random[0], cfg.mlm_random[1],
                  self._stream())
        return ws.input_ids, ws.labels

    def set_batch(self, input_ids, attention_mask=None, labels=None) -> Workspace:
        """Stage an already-masked batch (device or host int tensors) into the workspace."""
        B, S = input_ids.shape
        ws = self.workspace(B, S)
        ws.input_ids.copy_(input_ids, non_blocking=True)
        if attention_mask is None:
            ws.am.fill_(1)
        else:
            ws.am.copy_(attention_mask, non_blocking=True)
        if labels is not None:
            ws.labels.copy_(labels, non_blocking=True)
            n_lab = (torch.as_tensor(labels) != -100).sum().reshape(1).to(torch.int32)
            if ws.large_vocab and int(n_lab.item()) > ws.cap:
                raise ValueError(f"{int(n_lab.item())} labelled tokens exceed the LM-head capacity {ws.cap}")
            ws.n_labels.copy_(n_lab, non_blocking=True)
        return ws

    def _large_vocab_head(self, ws, E, E_key, T, H, V):
        """Tied decoder + masked CE for large V (Geneformer): logits only for the labelled rows
        (HF:modeling_esm.py:777-784 -- the loss only reads those rows), as tcgen05 GEMMs.
        Produces loss_sum, ws.dn (= dlogits·E scattered back, 0 on unlabelled rows), dE and dbias."""
        st, kdt, cap, Vp = self._stream(), self.kdt, ws.cap, ws.Vp
        call = self._call
        call("esm_label_compact", ws.labels.data_ptr(), T, ws.head_idx.data_ptr(), ws.head_lab.data_ptr(),
             ws.head_count.data_ptr(), cap, st)
        call("esm_gather_rows", kdt, ws.n.data_ptr(), ws.head_idx.data_ptr(), ws.n_lab.data_ptr(), cap, H, st)
        # logits[cap, V] = n_lab · Eᵀ + bias
        self._gemm(cap, V, H, ws.n_lab, H, 0, E, H, 0, ws.logits, Vp, EPI_STORE, bias=self._p32("lm_head.bias"))
        call("esm_xent_rows", kdt, ws.logits.data_ptr(), ws.head_lab.data_ptr(), cap, V, Vp,
             ws.inv_denom.data_ptr(), ws.loss_sum.data_ptr(), st)
        call("esm_colsum_rows", kdt, ws.logits.data_ptr(), cap, V, Vp, self._g32("lm_head.bias").data_ptr(), st)
        # dn_lab = dlogits · E ;  dE += dlogitsᵀ · n_lab
        self._gemm(cap, H, V, ws.logits, Vp, 0, E, H, 1, ws.dn_lab, H, EPI_STORE)
        self._gemm(V, H, cap, ws.logits, Vp, 1, ws.n_lab, H, 1, self._g32(E_key), H, EPI_F32_ACC)
        call("esm_scatter_rows", kdt, ws.dn_lab.data_ptr(), ws.head_idx.data_ptr(), ws.dn.data_ptr(), cap, H, T, st)

    # ------------------------------------------------------------------ forward + backward
    def forward_backward(self, ws: Workspace | None = None, loss_only: bool = False, optimizer: bool = False):
        """Forward, masked-CE loss and full backward into ``store.g32`` (zeroed here).

        Inputs are taken from the workspace (input_ids, am, labels, n_labels).  Returns the device
        loss tensor (mean over labelled tokens, or over ``n_labels`` if it was all-reduced).
        ``optimizer=True`` also applies AdamW (hyper-parameters staged by ``set_hyper``), overlapped
        with the backward: parameter groups are laid out in backward-completion order, so each
        contiguous range of final gradients is updated on a side stream (single process) or on the
        communication stream right after its bucket's all-reduce (DDP) while the backward continues."""
        ws = ws or self.ws
        cfg = self.config
        H, F, V, L, nh = cfg.hidden_size, cfg.intermediate_size, cfg.vocab_size, cfg.num_hidden_layers, \
            cfg.num_attention_heads
        dh = H // nh
        B, S, T = ws.B, ws.S, ws.T
        st = self._stream()
        kdt = self.kdt
        P = self.store
        qs = float(np.float32(dh ** -0.5))
        eps = float(cfg.layer_norm_eps)
        call = self._call
        E_key = "esm.embeddings.word_embeddings.weight"
        E = self._w(E_key, (V, H))

        # the gradient buffer is first written by the LM-head CE at the end of the forward: zero it on a side
        # stream behind the forward (3B: 11 GB, ~1.8 ms) and join right before the CE
        cur = torch.cuda.current_stream(self.device)
        if self._zero_stream is None:
            self._zero_stream = torch.cuda.Stream(self.device) if os.environ.get("ESM_GRAD_ZERO_SIDE", "1") != "0" \
                else cur
        self._zero_stream.wait_stream(cur)  # the previous step's optimizer has consumed the gradients
        with torch.cuda.stream(self._zero_stream):
            self.store.g32.zero_()
        ws.loss_sum.zero_()
        n_lab = ws.n_labels
        if self.comm is not None:  # global masked-token count -> loss normaliser; the local count is kept
            ws.n_labels_global.copy_(ws.n_labels)
            self.comm.reduce_count(ws.n_labels_global)
            n_lab = ws.n_labels_global
        call("esm_inv_count", n_lab.data_ptr(), ws.inv_denom.data_ptr(), st)
        sched = ws.attn_sched.data_ptr()
        call("esm_attn_prepare", ws.am.data_ptr(), sched, B, S, st)  # key-mask scan: once per step, not per layer
        # ---------------- forward
        self._nvtx("forward")
        call("esm_embed_fwd", kdt, ws.input_ids.data_ptr(), ws.am.data_ptr(), E.data_ptr(), ws.x[0].data_ptr(),
             ws.row_scale.data_ptr(), B, S, H, int(cfg.token_dropout), cfg.mask_token_id, st)
        for l in range(L):
            self._nvtx(f"layer{l}.fwd", l > 0)
            p = f"esm.encoder.layer.{l}."
            ly = ws.layers[l]
            x = ws.x[l]
            call("esm_layernorm_fwd", kdt, x.data_ptr(), self._p32(p + "attention.LayerNorm.weight").data_ptr(),
                 self._p32(p + "attention.LayerNorm.bias").data_ptr(), ly.h1.data_ptr(), ly.ln1_m.data_ptr(),
                 ly.ln1_r.data_ptr(), T, H, eps, st)
            if kdt == ESM_BF16:  # QKV GEMM with bias, q-scale, RoPE and head re-layout fused in the epilogue
                self._qkv_rope_gemm(ly, p, ws, T, H, nh, dh, S, qs)
            else:
                self.linear_fwd(ly.h1, p + "attention.self.qkv.weight", 3 * H, H, p + "attention.self.qkv.bias",
                                ws.qkv)
                call("esm_qkv_rope_fwd", kdt, ws.qkv.data_ptr(), ly.q.data_ptr(), ly.k.data_ptr(), ly.v.data_ptr(),
                     ws.cos.data_ptr(), ws.sin.data_ptr(), B, S, nh, dh, qs, st)
            ad = self._attn_drop(l)
            if ad is None:
                call("esm_attn_fwd", kdt, ly.q.data_ptr(), ly.k.data_ptr(), ly.v.data_ptr(), ws.am.data_ptr(), sched,
                     ly.o.data_ptr(), ly.lse.data_ptr(), B, nh, S, dh, st, flops=4.0 * B * nh * S * S * dh)
            else:
                call("esm_attn_fwd_dropout", kdt, ly.q.data_ptr(), ly.k.data_ptr(), ly.v.data_ptr(), ws.am.data_ptr(),
                     sched, ly.o.data_ptr(), ly.lse.data_ptr(), B, nh, S, dh, ctypes.byref(ad), st,
                     flops=4.0 * B * nh * S * S * dh)
            self.linear_fwd(ly.o, p + "attention.output.dense.weight", H, H, p + "attention.output.dense.bias",
                            ly.x1, epi=EPI_RESID, aux_in=x, drop=self._drop(2 * l))
            call("esm_layernorm_fwd", kdt, ly.x1.data_ptr(), self._p32(p + "LayerNorm.weight").data_ptr(),
                 self._p32(p + "LayerNorm.bias").data_ptr(), ly.h2.data_ptr(), ly.ln2_m.data_ptr(),
                 ly.ln2_r.data_ptr(), T, H, eps, st)
            self.linear_fwd(ly.h2, p + "intermediate.dense.weight", F, H, p + "intermediate.dense.bias", ly.a,
                            epi=EPI_GELU_GRADAUX if kdt == ESM_BF16 else EPI_GELU, aux_out=ly.z)
            self.linear_fwd(ly.a, p + "output.dense.weight", H, F, p + "output.dense.bias", ws.x[l + 1],
                            epi=EPI_RESID, aux_in=ly.x1, drop=self._drop(2 * l + 1))
        self._nvtx("lm_head+xent", L > 0)
        call("esm_layernorm_fwd", kdt, ws.x[L].data_ptr(),
             self._p32("esm.encoder.emb_layer_norm_after.weight").data_ptr(),
             self._p32("esm.encoder.emb_layer_norm_after.bias").data_ptr(), ws.xf.data_ptr(), ws.lnf_m.data_ptr(),
             ws.lnf_r.data_ptr(), T, H, eps, st)
        self.linear_fwd(ws.xf, "lm_head.dense.weight", H, H, "lm_head.dense.bias", ws.g, epi=EPI_GELU, aux_out=ws.y)
        call("esm_layernorm_fwd", kdt, ws.g.data_ptr(), self._p32("lm_head.layer_norm.weight").data_ptr(),
             self._p32("lm_head.layer_norm.bias").data_ptr(), ws.n.data_ptr(), ws.lnh_m.data_ptr(),
             ws.lnh_r.data_ptr(), T, H, eps, st)
        cur.wait_stream(self._zero_stream)  # gradient buffer zeroed
        if ws.large_vocab:
            self._large_vocab_head(ws, E, E_key, T, H, V)
        else:  # decoder (tied E) + masked CE + dlogits (fused, V <= 40)
            call("esm_lmhead_xent", kdt, ws.n.data_ptr(), E.data_ptr(), self._p32("lm_head.bias").data_ptr(),
                 ws.labels.data_ptr(), ws.inv_denom.data_ptr(), ws.loss_sum.data_ptr(), ws.dlogits.data_ptr(),
                 ws.dn.data_ptr(), self._g32(E_key).data_ptr(), self._g32("lm_head.bias").data_ptr(), T, H, V, st)
        self._nvtx(None)
        self._nvtx(None)
        if loss_only:
            if self.comm is not None:
                self.comm.reduce_loss(ws.loss_sum)
            return ws.loss_sum
        # ---------------- backward
        self._nvtx("backward")
        self._opt_on = optimizer
        self._opt_start = 0
        if self.comm is not None:
            self.comm.begin_backward()
            self.comm.on_bucket = self._adamw_range if optimizer else None
        # LM head: LN^T then GELU'(y) fused; col sums -> dense bias grad
        call("esm_layernorm_bwd", kdt, ws.dn.data_ptr(), ws.g.data_ptr(),
             self._p32("lm_head.layer_norm.weight").data_ptr(), ws.lnh_m.data_ptr(), ws.lnh_r.data_ptr(), None,
             ws.y.data_ptr(), ws.dy.data_ptr(), self._g32("lm_head.layer_norm.weight").data_ptr(),
             self._g32("lm_head.layer_norm.bias").data_ptr(), self._g32("lm_head.dense.bias").data_ptr(), T, H,
             None, None, st)
        fused = self.linear_dgrad(ws.dy, "lm_head.dense.weight", H, H, ws.dh,
                                  ln=(ws.x[L], ws.lnf_m, ws.lnf_r, "esm.encoder.emb_layer_norm_after"))
        self.linear_wgrad(ws.dy, ws.xf, "lm_head.dense.weight", H, H)
        last_b2 = f"esm.encoder.layer.{L - 1}.output.dense.bias" if L > 0 else None
        call("esm_layernorm_bwd", kdt, ws.dh.data_ptr(), ws.x[L].data_ptr(),
             self._p32("esm.encoder.emb_layer_norm_after.weight").data_ptr(), ws.lnf_m.data_ptr(),
             ws.lnf_r.data_ptr(), None, None, ws.dx.data_ptr(),
             None if fused else self._g32("esm.encoder.emb_layer_norm_after.weight").data_ptr(),
             None if fused else self._g32("esm.encoder.emb_layer_norm_after.bias").data_ptr(),
             self._g32(last_b2).data_ptr() if last_b2 else None, T, H, *self._drop_bwd(ws, 2 * L - 1), st)
        self._group_ready("esm.encoder.emb_layer_norm_after.bias")
        dx, dx_next = ws.dx, ws.dx_alt
        for l in reversed(range(L)):
            self._nvtx(f"layer{l}.bwd", l < L - 1)
            p = f"esm.encoder.layer.{l}."
            ly = ws.layers[l]
            # FFN
            # bf16: ly.z holds GELU'(Z) from the forward epilogue (EPI_GELU_GRADAUX) -> plain multiply
            dbr = ws.dxd if ws.dxd is not None else dx  # FFN branch gradient (through its dropout mask)
            self.linear_dgrad(dbr, p + "output.dense.weight", H, F, ws.dz,
                              epi=EPI_MUL_AUX if kdt == ESM_BF16 else EPI_DGELU, aux_in=ly.z,
                              col_sum=self._g32(p + "intermediate.dense.bias"))
            self.linear_wgrad(dbr, ly.a, p + "output.dense.weight", H, F)
            fused = self.linear_dgrad(ws.dz, p + "intermediate.dense.weight", F, H, ws.dh,
                                      ln=(ly.x1, ly.ln2_m, ly.ln2_r, p + "LayerNorm"))
            self.linear_wgrad(ws.dz, ly.h2, p + "intermediate.dense.weight", F, H)
            call("esm_layernorm_bwd", kdt, ws.dh.data_ptr(), ly.x1.data_ptr(),
                 self._p32(p + "LayerNorm.weight").data_ptr(), ly.ln2_m.data_ptr(), ly.ln2_r.data_ptr(),
                 dx.data_ptr(), None, ws.dx1.data_ptr(),
                 None if fused else self._g32(p + "LayerNorm.weight").data_ptr(),
                 None if fused else self._g32(p + "LayerNorm.bias").data_ptr(),
                 self._g32(p + "attention.output.dense.bias").data_ptr(), T, H, *self._drop_bwd(ws, 2 * l), st)
            # attention (branch gradient: through the out-projection's dropout mask)
            dbr = ws.dxd if ws.dxd is not None else ws.dx1
            if kdt == ESM_BF16:  # dO, and Delta = rowsum(dO o O) per head from the same epilogue (no extra pass)
                self._gemm(T, H, H, dbr, H, 0, self._w(p + "attention.output.dense.weight", (H, H)), H, 1, ws.do, H,
                           EPI_DELTA, aux_in=ly.o, ld_aux_in=H, delta=(ws.delta, S, nh, dh))
                o_arg = None
            else:
                self.linear_dgrad(dbr, p + "attention.output.dense.weight", H, H, ws.do)
                o_arg = ly.o.data_ptr()
            self.linear_wgrad(dbr, ly.o, p + "attention.output.dense.weight", H, H)
            if kdt == ESM_BF16 and self._fused_attn_bwd(dh):
                # fused: attention backward writes dqkv [T,3H] (RoPE^T, q-scale) + q/k/v bias grads
                ad = self._attn_drop(l)
                call("esm_attn_bwd_qkv" if ad is None else "esm_attn_bwd_qkv_dropout", ly.q.data_ptr(),
                     ly.k.data_ptr(), ly.v.data_ptr(), o_arg, ws.do.data_ptr(), ly.lse.data_ptr(), ws.am.data_ptr(),
                     sched, ws.delta.data_ptr(), ws.dq.data_ptr(), ws.dqkv.data_ptr(),
                     self._g32(p + "attention.self.qkv.bias").data_ptr(), ws.cos.data_ptr(), ws.sin.data_ptr(), qs, B,
                     nh, S, dh, *(() if ad is None else (ctypes.byref(ad),)), st, flops=8.0 * B * nh * S * S * dh)
            else:
                ad = self._attn_drop(l)
                call("esm_attn_bwd" if ad is None else "esm_attn_bwd_dropout", kdt, ly.q.data_ptr(), ly.k.data_ptr(),
                     ly.v.data_ptr(), o_arg, ws.do.data_ptr(), ly.lse.data_ptr(), ws.am.data_ptr(), sched,
                     ws.delta.data_ptr(), ws.dq.data_ptr(), ws.dk.data_ptr(), ws.dv.data_ptr(), B, nh, S, dh,
                     *(() if ad is None else (ctypes.byref(ad),)), st, flops=8.0 * B * nh * S * S * dh)
                call("esm_qkv_rope_bwd", kdt, ws.dq.data_ptr(), ws.dk.data_ptr(), ws.dv.data_ptr(),
                     ws.dqkv.data_ptr(), self._g32(p + "attention.self.qkv.bias").data_ptr(), ws.cos.data_ptr(),
                     ws.sin.data_ptr(), B, S, nh, dh, qs, st)
            fused = self.linear_dgrad(ws.dqkv, p + "attention.self.qkv.weight", 3 * H, H, ws.dh,
                                      ln=(ws.x[l], ly.ln1_m, ly.ln1_r, p + "attention.LayerNorm"))
            self.linear_wgrad(ws.dqkv, ly.h1, p + "attention.self.qkv.weight", 3 * H, H)
            prev_b2 = f"esm.encoder.layer.{l - 1}.output.dense.bias" if l > 0 else None
            call("esm_layernorm_bwd", kdt, ws.dh.data_ptr(), ws.x[l].data_ptr(),
                 self._p32(p + "attention.LayerNorm.weight").data_ptr(), ly.ln1_m.data_ptr(), ly.ln1_r.data_ptr(),
                 ws.dx1.data_ptr(), None, dx_next.data_ptr(),
                 None if fused else self._g32(p + "attention.LayerNorm.weight").data_ptr(),
                 None if fused else self._g32(p + "attention.LayerNorm.bias").data_ptr(),
                 self._g32(prev_b2).data_ptr() if prev_b2 else None, T, H,
                 *(self._drop_bwd(ws, 2 * l - 1) if l > 0 else (None, None)), st)
            dx, dx_next = dx_next, dx
            self._group_ready(p + "attention.LayerNorm.bias")
        if L > 0:
            self._nvtx(None)
        call("esm_embed_bwd", kdt, ws.input_ids.data_ptr(), ws.am.data_ptr(), ws.row_scale.data_ptr(),
             dx.data_ptr(), self._g32(E_key).data_ptr(), B, S, H, V,
             cfg.mask_token_id if cfg.token_dropout else -1, cfg.pad_token_id, st)
        if self.comm is not None:
            self.comm.ready(E_key)
            self.comm.end_backward()
            self.comm.reduce_loss(ws.loss_sum)
        elif optimizer:
            self._adamw_range(self._opt_start, self.store.numel, None)  # word embeddings: last, on the compute stream
            torch.cuda.current_stream(self.device).wait_stream(self._opt_stream)
        self._last_dx_embed = dx
        self._nvtx(None)
        return ws.loss_sum

    # ------------------------------------------------------------------ optimizer
    def dropout_seed(self, step: int) -> int:
        """The hidden-dropout seed of a step (splitmix64 of the model's base seed and the step)."""
        z = (self.dropout_base + (int(step) + 1) * 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def set_dropout_seed(self, seed: int):
        """Stage a hidden-dropout seed (set_hyper does this per step; a fill kernel, stream-ordered)."""
        v = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.drop_seed.fill_(v - (1 << 64) if v >= (1 << 63) else v)
        self.last_dropout_seed = v

    def _drop_bwd(self, ws, site: int):
        """(esm_dropout*, dx_drop) arguments of a LayerNorm backward whose input gradient also feeds the branch of
        call site ``site`` (hidden dropout on), else (None, None)."""
        d = self._drop(site)
        if d is None:
            return None, None
        self._drop_keep = d  # ctypes object must outlive the call
        return ctypes.byref(d), ws.dxd.data_ptr()

    def _drop(self, site: int):
        """esm_dropout of a call site (2*layer + 0 attention output / 1 FFN output), or None without dropout."""
        if self.dropout_p <= 0.0:
            return None
        return _lib.Dropout(self.drop_seed.data_ptr(), site, int(round(self.dropout_p * 65536.0)),
                            1.0 / (1.0 - self.dropout_p))

    def _attn_drop(self, layer: int):
        """esm_dropout of layer ``layer``'s attention probabilities (site 4096 + layer), or None (p = 0).  The
        ctypes object is kept on the model: it must outlive the call that passes a pointer to it."""
        if self.attn_dropout_p <= 0.0:
            return None
        self._attn_drop_keep = _lib.Dropout(self.drop_seed.data_ptr(), ATTN_DROP_SITE + layer,
                                            int(round(self.attn_dropout_p * 65536.0)), 1.0 / (1.0 - self.attn_dropout_p))
        return self._attn_drop_keep

    def set_hyper(self, lr=None, step=None):
        """Stage AdamW hyper-parameters in device memory (read by the kernel: CUDA-graph safe)."""
        lr = self.lr if lr is None else lr
        step = self.step_count if step is None else step
        i = self._hyper_i = (self._hyper_i + 1) % len(self._hyper_ring)
        h, ev = self._hyper_ring[i], self._hyper_ev[i]
        if ev is not None:
            ev.synchronize()  # the H2D copy that last read this pinned slot has completed
        h.copy_(torch.tensor([lr, self.betas[0], self.betas[1], self.eps, self.weight_decay, float(step),
                              self.grad_scale, 0.0], dtype=torch.float32))
        self.hyper.copy_(h, non_blocking=True)
        if self.dropout_p > 0.0 or self.attn_dropout_p > 0.0:
            self.set_dropout_seed(self.dropout_seed(step))
        ev = self._hyper_ev[i] = self._hyper_ev[i] or torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))

    @staticmethod
    def _fused_attn_bwd(dh: int) -> bool:
        """Fused attention backward (writes dqkv with RoPE^T + bias grads) vs classic + qkv_rope_bwd: fused for
        every head dim -- dh <= 32 (35M 0.78 vs 0.71 + 0.16 ms) and, since dK/dV leave TMEM before the epilogue
        work, dh = 64 (650M step 86.1 vs 86.5 ms, alternating runs).  ESM_ATTN_FUSED=0/1 forces either."""
        env = os.environ.get("ESM_ATTN_FUSED")
        return True if env is None else env != "0"

    def _group_ready(self, key: str):
        """All groups up to ``key`` (backward-completion order) hold final gradients."""
        if self.comm is not None:
            self.comm.ready(key)
        elif self._opt_on:
            end = (self.store.group_range[key][1] + ALIGN - 1) // ALIGN * ALIGN
            if end > self._opt_start:
                if self._opt_stream is None:
                    self._opt_stream = torch.cuda.Stream(self.device)
                ev = torch.cuda.Event()
                ev.record(torch.cuda.current_stream(self.device))
                self._opt_stream.wait_event(ev)
                self._adamw_range(self._opt_start, end, self._opt_stream)

    def _adamw_range(self, a: int, b: int, stream, grad: torch.Tensor | None = None):
        """AdamW on flat elements [a, b) (a, b multiples of 256) on ``stream`` (None: current).  ``grad``: the
        gradients of [a, b) when they are not ``g32[a:b]`` (bf16-reduced data-parallel buckets)."""
        b = min(b, self.store.numel)
        if b <= a:
            return
        P = self.store
        st = stream.cuda_stream if stream is not None else self._stream()
        p16 = P.p16[a:].data_ptr() if P.p16 is not None else None
        if grad is not None and grad.dtype == torch.bfloat16:
            self._call("esm_adamw_bf16g", P.p32[a:].data_ptr(), grad.data_ptr(), P.m[a:].data_ptr(),
                       P.v[a:].data_ptr(), p16, P.decay[a // ALIGN:].data_ptr(), b - a, self.hyper.data_ptr(), st,
                       nbytes=28.0 * (b - a))
        else:
            g = grad.data_ptr() if grad is not None else P.g32[a:].data_ptr()
            self._call("esm_adamw", P.p32[a:].data_ptr(), g, P.m[a:].data_ptr(), P.v[a:].data_ptr(), p16,
                       P.decay[a // ALIGN:].data_ptr(), b - a, self.hyper.data_ptr(), st, nbytes=30.0 * (b - a))
        self._opt_start = b

    def _adamw(self):
        P = self.store
        self._call("esm_adamw", P.p32.data_ptr(), P.g32.data_ptr(), P.m.data_ptr(), P.v.data_ptr(),
                   P.p16.data_ptr() if P.p16 is not None else None, P.decay.data_ptr(), P.numel,
                   self.hyper.data_ptr(), self._stream(), nbytes=30.0 * P.numel)

    def optimizer_step(self, lr=None):
        """AdamW over all parameters after a separate ``forward_backward`` (un-overlapped)."""
        if self.comm is not None and (self.comm.shard or self.comm.bf16):
            raise RuntimeError("sharded / bf16-bucket data parallelism updates inside the step: use step()")
        self.step_count += 1
        self.set_hyper(lr=lr, step=self.step_count)
        self._adamw()

    def step(self, ws: Workspace | None = None, lr=None):
        """One full train step on the staged batch: forward, backward and AdamW overlapped with the
        backward (same arithmetic as forward_backward + optimizer_step).  Returns the device loss."""
        self.step_count += 1
        self.set_hyper(lr=lr, step=self.step_count)
        return self.forward_backward(ws, optimizer=True)

    # ------------------------------------------------------------------ CUDA graph
    def capture(self, ws: Workspace | None = None):
        """Capture forward + backward + AdamW for the workspace shape into one CUDA graph.
        Inputs (input_ids / labels / am / n_labels) and hyper-parameters are read from their
        static device buffers at replay; masking and H2D copies stay outside the graph."""
        ws = ws or self.ws
        if self.comm is not None and not self.comm.cuda:
            raise RuntimeError("CUDA-graph capture needs the NCCL communicator (CUDA tensors)")
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.forward_backward(ws)  # warm-up: lazy attributes, tensor-map encode paths
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        n0 = self.launches
        # NCCL collectives (data parallel) are captured too; thread-local capture mode lets NCCL's host-side
        # bookkeeping run during capture
        with torch.cuda.graph(g, capture_error_mode="thread_local" if self.comm is not None else "global"):
            self.forward_backward(ws, optimizer=True)
        ws.graph = g
        ws.graph_launches = self.launches - n0
        self.graph = g
        self.graph_launches = ws.graph_launches
        return g

    def graph_step(self, lr=None, ws: Workspace | None = None):
        """Replay the step captured for ``ws`` (default: the current workspace) after staging its batch."""
        ws = ws or self.ws
        if getattr(ws, "graph", None) is None:
            raise RuntimeError("no CUDA graph captured for this workspace: call capture(ws) first")
        self.step_count += 1
        self.set_hyper(lr=lr, step=self.step_count)
        ws.graph.replay()
        self.launches += ws.graph_launches
        return ws.loss_sum

    def train_step_tokens(self, token_lists, seed: int, stream_id: int, lr=None, pad_to: int = 64,
                          use_graph: bool = False):
        """One MLM step on a list of token sequences (e.g. one ``bucket_batches`` batch): right-pad to a
        multiple of ``pad_to``, mask on the device (bit-exact 15% / 80-10-10), forward, backward, AdamW.
        Fully padded key tiles are skipped by the attention kernels.  Returns the device loss tensor."""
        from .data import collate
        ids, am = collate(token_lists, pad_to=pad_to, pad_id=self.config.pad_token_id)
        ws = self.workspace(*ids.shape)
        ws.ids.copy_(torch.from_numpy(ids), non_blocking=True)
        ws.am.copy_(torch.from_numpy(am), non_blocking=True)
        self.mlm_mask(ws.ids, seed, stream_id, ws)
        if use_graph:
            if getattr(ws, "graph", None) is None:
                self.capture(ws)
            return self.graph_step(lr=lr, ws=ws)
        return self.step(ws, lr=lr)

    def train_step(self, input_ids, attention_mask=None, labels=None, lr=None):
        """One MLM train step on an already-masked batch; returns the device loss tensor."""
        ws = self.set_batch(input_ids, attention_mask, labels)
        return self.step(ws, lr=lr)
