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
        if self.hidden_dropout_prob or self.attention_probs_dropout_prob:
            raise ValueError("ESM-2 trains with dropout 0.0; dropout > 0 is not implemented")
        if self.head_dim not in (16, 24, 32, 64):
            raise ValueError(f"head_dim {self.head_dim} not supported by the attention kernels")
        if self.hidden_size % 16:
            raise ValueError("hidden_size must be a multiple of 16")
        return self

    def to_dict(self):
        return asdict(self)

    def train_flops_per_token(self, seq_len: int) -> float:
        """6*N_mm + 12*L*H*S (PaLM MFU convention)."""
        H, F, V, L = self.hidden_size, self.intermediate_size, self.vocab_size, self.num_hidden_layers
        n_mm = L * (4 * H * H + 2 * H * F) + H * H + H * V
        return 6.0 * n_mm + 12.0 * L * H * seq_len


PRESETS = {
    "esm2_t6_8M": dict(hidden_size=320, num_hidden_layers=6, num_attention_heads=20, intermediate_size=1280),
    "esm2_t12_35M": dict(hidden_size=480, num_hidden_layers=12, num_attention_heads=20, intermediate_size=1920),
    "esm2_t30_150M": dict(hidden_size=640, num_hidden_layers=30, num_attention_heads=20, intermediate_size=2560),
    "esm2_t33_650M": dict(hidden_size=1280, num_hidden_layers=33, num_attention_heads=20, intermediate_size=5120),
    "esm2_t36_3B": dict(hidden_size=2560, num_hidden_layers=36, num_attention_heads=40, intermediate_size=10240),
}
ALIASES = {"8m": "esm2_t6_8M", "35m": "esm2_t12_35M", "150m": "esm2_t30_150M", "650m": "esm2_t33_650M",
           "3b": "esm2_t36_3B"}


def preset(name: str) -> EsmConfig:
    key = ALIASES.get(name.lower(), name)
    return EsmConfig(**PRESETS[key]).validate()
