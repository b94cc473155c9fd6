"""ESM-2 model configuration (field names of HF ``EsmConfig``, HF:configuration_esm.py:193-214).

The reference (``densefeed``) defines no model config (SURVEY.md §5 "Config"), so the
HF field names are kept so that an ``EsmConfig``/checkpoint user finds the same knobs.
ESM-2 pinned constants: vocab 33, pad 1, mask 32, rotary, token_dropout, eps 1e-5,
emb_layer_norm_before False, dropout 0.
"""
from __future__ import annotations

from dataclasses import asdict, dataclass


@dataclass
class EsmConfig:
    vocab_size: int = 33
    hidden_size: int = 320
    num_hidden_layers: int = 6
    num_attention_heads: int = 20
    intermediate_size: int = 1280
    hidden_dropout_prob: float = 0.0
    attention_probs_dropout_prob: float = 0.0
    max_position_embeddings: int = 1026
    initializer_range: float = 0.02
    layer_norm_eps: float = 1e-5
    position_embedding_type: str = "rotary"
    emb_layer_norm_before: bool = False
    token_dropout: bool = True
    mask_token_id: int = 32
    pad_token_id: int = 1
    cls_token_id: int = 0
    eos_token_id: int = 2
    tie_word_embeddings: bool = True
    # MLM vocabulary (not HF EsmConfig fields): ids eligible for selection (inclusive) and the range
    # random replacements are drawn from (first id, count).  ESM-2: amino acids 4..30, 20 standard AAs.
    mlm_eligible: tuple = (4, 30)
    mlm_random: tuple = (4, 20)

    @property
    def head_dim(self) -> int:
        return self.hidden_size // self.num_attention_heads

    def validate(self):
        if self.hidden_size % self.num_attention_heads:
            raise ValueError("hidden_size must be a multiple of num_attention_heads")
        if self.position_embedding_type != "rotary":
            raise ValueError("only rotary position embeddings (ESM-2) are supported")
        if self.emb_layer_norm_before:
            raise ValueError("emb_layer_norm_before=True (ESM-1b) is not supported")
        if not 0.0 <= self.hidden_dropout_prob < 1.0:
            raise ValueError("hidden_dropout_prob must be in [0, 1)")
        if not 0.0 <= self.attention_probs_dropout_prob < 1.0:
            raise ValueError("attention_probs_dropout_prob must be in [0, 1)")
        if self.head_dim not in (16, 24, 32, 64):
            raise ValueError(f"head_dim {self.head_dim} not supported by the attention kernels")
        if self.hidden_size % 16:
            raise ValueError("hidden_size must be a multiple of 16")
        lo, hi = self.mlm_eligible
        if not (0 <= lo <= hi < self.vocab_size) or self.mlm_random[1] <= 0 \
                or self.mlm_random[0] + self.mlm_random[1] > self.vocab_size:
            raise ValueError("mlm_eligible / mlm_random outside the vocabulary")
        return self

    def to_dict(self):
        return asdict(self)

    def train_flops_per_token(self, seq_len: int, head_fraction: float = 1.0) -> float:
        """6*N_mm + 12*L*H*S (PaLM MFU convention).  ``head_fraction`` scales the tied
        decoder term: the large-vocabulary head computes logits only for labelled rows (~15%), so its
        required FLOPs are head_fraction * 6*H*V per token (bench.py passes 0.15 when V > 40)."""
        H, F, V, L = self.hidden_size, self.intermediate_size, self.vocab_size, self.num_hidden_layers
        n_mm = L * (4 * H * H + 2 * H * F) + H * H + H * V * head_fraction
        return 6.0 * n_mm + 12.0 * L * H * seq_len


PRESETS = {
    "esm2_t6_8M": dict(hidden_size=320, num_hidden_layers=6, num_attention_heads=20, intermediate_size=1280),
    "esm2_t12_35M": dict(hidden_size=480, num_hidden_layers=12, num_attention_heads=20, intermediate_size=1920),
    "esm2_t30_150M": dict(hidden_size=640, num_hidden_layers=30, num_attention_heads=20, intermediate_size=2560),
    "esm2_t33_650M": dict(hidden_size=1280, num_hidden_layers=33, num_attention_heads=20, intermediate_size=5120),
    "esm2_t36_3B": dict(hidden_size=2560, num_hidden_layers=36, num_attention_heads=40, intermediate_size=10240),
}

def geneformer_config(n_genes: int = 25424, **kw) -> EsmConfig:
    """Geneformer-106M-shaped encoder (BASELINE configs[4]) over rank-value gene tokens.

    Token layout of the reference tokenizer (pkg/src/densefeed/tokenizer.py:16-18,68-83):
    PAD=0, MASK=1, gene g -> g + 2, so V = n_genes + 2 (25,426 for the ~106M parameter count,
    SURVEY.md §8d).  The encoder is the ESM-2 pre-LN/rotary layer ("reuse the
    encoder"); no token dropout; every gene token is eligible for masking, random replacements are
    drawn from all genes."""
    V = n_genes + 2
    d = dict(vocab_size=V, hidden_size=768, num_hidden_layers=12, num_attention_heads=12, intermediate_size=3072,
             token_dropout=False, pad_token_id=0, mask_token_id=1, cls_token_id=0, eos_token_id=0,
             max_position_embeddings=2048, mlm_eligible=(2, V - 1), mlm_random=(2, V - 2))
    d.update(kw)
    return EsmConfig(**d).validate()


ALIASES = {"8m": "esm2_t6_8M", "35m": "esm2_t12_35M", "150m": "esm2_t30_150M", "650m": "esm2_t33_650M",
           "3b": "esm2_t36_3B"}


def preset(name: str) -> EsmConfig:
    if name.lower() in ("geneformer", "geneformer_106m"):
        return geneformer_config()
    key = ALIASES.get(name.lower(), name)
    return EsmConfig(**PRESETS[key]).validate()
