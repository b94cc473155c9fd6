"""Optimizer schedule for ESM-2 pre-training (AdamW itself is the fused `esm_adamw` kernel,
driven by EsmForMaskedLM.optimizer_step / graph_step)."""


def esm2_lr(step: int, peak_lr: float = 4e-4, warmup: int = 2000, total: int = 500_000,
            final_ratio: float = 0.1) -> float:
    """ESM-2 schedule: linear warm-up to `peak_lr`, then linear decay to `final_ratio * peak_lr`."""
    if step <= warmup:
        return peak_lr * step / max(1, warmup)
    frac = min(1.0, (step - warmup) / max(1, total - warmup))
    return peak_lr * (1.0 - (1.0 - final_ratio) * frac)
