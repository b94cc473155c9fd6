"""Generate golden fixtures for the ESM-2 oracle from Hugging Face EsmForMaskedLM.

TEST INFRASTRUCTURE ONLY (run in the build container, where transformers 5.5.0
is importable; the fixtures it writes under tests/golden/ travel with the repo).

For each small config it builds HF ``EsmForMaskedLM`` (eager attention, fp64,
rotary, token_dropout, eps 1e-5 -- the ESM-2 settings), loads parameters drawn
by ``esm2_oracle.init_params``, runs a padded/ragged batch masked by
``esm2_oracle.mlm_mask`` and records: loss, logits, the input of every layer,
and every parameter gradient (the tied decoder/embedding gradient summed, as
autograd does).  ``tests/test_oracle.py`` pins the oracle to these numbers.

    python oracle/make_golden.py        # rewrites tests/golden/hf_*.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import esm2_oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

CASES = {
    # name: (hidden, layers, heads, ffn, batch, seq, lengths)
    "tiny_dh16": (64, 2, 4, 256, 3, 24, [24, 17, 9]),
    "tiny_dh24": (96, 2, 4, 384, 2, 32, [32, 20]),
    "tiny_dh64": (128, 1, 2, 512, 2, 40, [40, 33]),
}
# hidden dropout (HF EsmSelfOutput / EsmOutput dropout, training mode): HF's nn.Dropout modules are replaced by
# modules applying the oracle's counter-based masks (esm2_oracle.dropout_keep), so the golden pins where and how
# the masks enter the forward and the backward while the mask bits themselves are the library's own RNG.
DROPOUT_CASES = {"tiny_dh24_dropout": ((96, 2, 4, 384, 2, 32, [32, 20]), (0x1234ABCD5678EF01, 0.1))}


class _MaskDropout:
    """Stand-in for nn.Dropout(p) in training mode with a fixed keep mask: x * keep / (1 - p)."""

    @staticmethod
    def make(keep, p):
        import torch

        class M(torch.nn.Module):
            def forward(self, x):
                return x * torch.from_numpy(keep.astype(np.float64)) / (1.0 - p)
        return M()


def hf_run(cfg: O.OracleConfig, params, ids, am, labels, dropout=None):
    import torch
    from transformers import EsmConfig, EsmForMaskedLM

    hc = EsmConfig(vocab_size=cfg.vocab_size, hidden_size=cfg.hidden_size,
                   num_hidden_layers=cfg.num_hidden_layers, num_attention_heads=cfg.num_attention_heads,
                   intermediate_size=cfg.intermediate_size, hidden_dropout_prob=0.0,
                   attention_probs_dropout_prob=0.0, max_position_embeddings=1026,
                   layer_norm_eps=cfg.layer_norm_eps, position_embedding_type="rotary",
                   emb_layer_norm_before=False, token_dropout=True, mask_token_id=O.MASK,
                   pad_token_id=O.PAD)
    hc._attn_implementation = "eager"
    torch.manual_seed(0)
    model = EsmForMaskedLM(hc).double()
    model.train()
    if dropout is not None:
        seed, p = dropout
        B, S = ids.shape
        for i, layer in enumerate(model.esm.encoder.layer):
            layer.attention.output.dropout = _MaskDropout.make(
                O.dropout_keep(seed, 2 * i, B * S, cfg.hidden_size, p).reshape(B, S, -1), p)
            layer.output.dropout = _MaskDropout.make(
                O.dropout_keep(seed, 2 * i + 1, B * S, cfg.hidden_size, p).reshape(B, S, -1), p)
    sd = {k: torch.from_numpy(np.asarray(v, dtype=np.float64)) for k, v in params.items()}
    missing, unexpected = model.load_state_dict(sd, strict=False)
    assert not unexpected, unexpected
    assert all(("contact_head" in m) or ("decoder" in m) or ("rotary" in m) for m in missing), missing
    # keep RoPE tables in fp32 as in a real (fp32-weight) ESM-2 model: .double() promoted inv_freq
    for layer in model.esm.encoder.layer:
        rot = layer.attention.self.rotary_embeddings
        rot.inv_freq = rot.inv_freq.float()
        rot._seq_len_cached = None
    assert model.lm_head.decoder.weight.data_ptr() == model.esm.embeddings.word_embeddings.weight.data_ptr()
    captured = []
    hooks = [layer.register_forward_pre_hook(lambda m, a: captured.append(a[0].detach().clone()))
             for layer in model.esm.encoder.layer]
    hooks.append(model.esm.encoder.emb_layer_norm_after.register_forward_pre_hook(
        lambda m, a: captured.append(a[0].detach().clone())))
    out = model(input_ids=torch.from_numpy(ids.astype(np.int64)),
                attention_mask=torch.from_numpy(am.astype(np.int64)),
                labels=torch.from_numpy(labels.astype(np.int64)))
    out.loss.backward()
    for h in hooks:
        h.remove()
    grads = {}
    for name, prm in model.named_parameters():
        if name in params:
            grads[name] = prm.grad.detach().numpy().copy()
    return float(out.loss), out.logits.detach().numpy(), [c.numpy() for c in captured], grads


def main():
    os.makedirs(OUT, exist_ok=True)
    cases = [(name, spec, None) for name, spec in CASES.items()]
    cases += [(name, spec, drop) for name, (spec, drop) in DROPOUT_CASES.items()]
    if len(sys.argv) > 1:
        cases = [c for c in cases if c[0] in sys.argv[1:]]
    for name, (H, L, nh, F, B, S, lens), drop in cases:
        cfg = O.OracleConfig(hidden_size=H, num_hidden_layers=L, num_attention_heads=nh, intermediate_size=F)
        params = O.init_params(cfg, seed=1)
        # perturb biases / LN params away from their init so their gradients are exercised
        rng = np.random.default_rng(2)
        for k, v in params.items():
            if v.ndim == 1:
                params[k] = (v + rng.standard_normal(v.shape).astype(np.float32) * np.float32(0.05)).astype(np.float32)
        rng = np.random.default_rng(3)
        toks = []
        for n in lens:
            body = rng.integers(4, 24, size=n - 2)
            toks.append(np.concatenate([[O.CLS], body, [O.EOS]]).astype(np.int32))
        ids, am = O.pad_batch(toks, S)
        inp, labels = O.mlm_mask(ids, seed=11, stream=0)
        # guarantee at least a few masked/labelled positions
        assert (labels != -100).sum() > 0
        loss, logits, hidden, grads = hf_run(cfg, params, inp, am, labels, dropout=drop)
        blob = dict(config=np.array([H, L, nh, F, B, S]), input_ids=inp, attention_mask=am, labels=labels,
                    raw_ids=ids, loss=np.array(loss), logits=logits)
        if drop is not None:
            blob["dropout_seed"] = np.array(drop[0], dtype=np.uint64)
            blob["dropout_p"] = np.array(drop[1])
        for i, h in enumerate(hidden):
            blob[f"hidden.{i}"] = h
        for k, v in params.items():
            blob["param." + k] = v
        for k, v in grads.items():
            blob["grad." + k] = v
        path = os.path.join(OUT, f"hf_{name}.npz")
        np.savez_compressed(path, **blob)
        print(f"{path}: loss={loss:.6f} masked={(labels != -100).sum()} size={os.path.getsize(path)}")


if __name__ == "__main__":
    main()
