"""ctypes binding of the in-tree C-ABI kernel library (include/esm2_b200.h).

The product path has no fallback: if ``libesm2b200.so`` is missing or was built for
another architecture, importing the model raises ``EsmKernelError``.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ESM_LIB_PATH") or os.path.join(_HERE, "libesm2b200.so")  # override: A/B builds

ESM_F32, ESM_BF16, ESM_I32 = 0, 1, 2
EPI_STORE, EPI_GELU, EPI_RESID, EPI_DGELU, EPI_F32_ACC, EPI_QKV_ROPE, EPI_STORE_LN = 0, 1, 2, 3, 4, 5, 6
EPI_GELU_GRADAUX, EPI_MUL_AUX, EPI_DELTA = 7, 8, 9

EXPORTS = [
    "esm_version", "esm_last_error", "esm_device_sm_count", "esm_tokenize", "esm_mlm_mask", "esm_embed_fwd",
    "esm_embed_bwd", "esm_layernorm_fwd", "esm_layernorm_bwd", "esm_gemm", "esm_qkv_rope_fwd", "esm_qkv_rope_bwd",
    "esm_attn_prepare", "esm_attn_fwd", "esm_attn_bwd", "esm_attn_bwd_qkv", "esm_attn_fwd_dropout",
    "esm_attn_bwd_dropout", "esm_attn_bwd_qkv_dropout", "esm_lmhead_xent", "esm_inv_count",
    "esm_mlm_mask_ex", "esm_label_compact", "esm_gather_rows", "esm_scatter_rows", "esm_xent_rows", "esm_colsum_rows",
    "esm_rank_encode", "esm_dropout_mask", "esm_adamw", "esm_adamw_bf16g", "esm_cast_f32_bf16", "esm_cast_bf16_f32",
    "esm_comm_version", "esm_comm_unique_id", "esm_comm_init", "esm_comm_destroy", "esm_comm_allreduce",
    "esm_comm_reduce_scatter", "esm_comm_allgather",
]


class EsmKernelError(RuntimeError):
    """A C-ABI call returned non-zero (cudaError_t or ESM_E* code); message from esm_last_error()."""


class Dropout(ctypes.Structure):
    """esm_dropout (include/esm2_b200.h): per-step seed (device pointer), call site, 16-bit threshold, scale."""
    _fields_ = [("seed", ctypes.c_void_p), ("site", ctypes.c_uint32), ("threshold", ctypes.c_uint32),
                ("scale", ctypes.c_float)]


class GemmArgs(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int), ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int),
        ("A", ctypes.c_void_p), ("lda", ctypes.c_int64), ("a_mn_major", ctypes.c_int),
        ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64), ("b_mn_major", ctypes.c_int),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64),
        ("epilogue", ctypes.c_int),
        ("bias", ctypes.c_void_p),
        ("aux_in", ctypes.c_void_p), ("ld_aux_in", ctypes.c_int64),
        ("aux_out", ctypes.c_void_p), ("ld_aux_out", ctypes.c_int64),
        ("col_sum", ctypes.c_void_p),
        ("split_k", ctypes.c_int),
        ("rope_cos", ctypes.c_void_p), ("rope_sin", ctypes.c_void_p),
        ("q_out", ctypes.c_void_p), ("k_out", ctypes.c_void_p), ("v_out", ctypes.c_void_p),
        ("seq_len", ctypes.c_int), ("n_heads", ctypes.c_int), ("head_dim", ctypes.c_int),
        ("q_scale", ctypes.c_float),
        ("row_mean", ctypes.c_void_p), ("row_rstd", ctypes.c_void_p), ("col_sum2", ctypes.c_void_p),
        ("drop", Dropout),
        ("row_dot", ctypes.c_void_p),
    ]


_P, _I, _I64, _U64, _F = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float
_SIGS = {
    "esm_version": ([], _I),
    "esm_last_error": ([], ctypes.c_char_p),
    "esm_device_sm_count": ([_I], _I),
    "esm_tokenize": ([ctypes.c_char_p, _I, _P, _I], _I),
    "esm_mlm_mask": ([_P, _P, _P, _P, _I64, _U64, _U64, _P], _I),
    "esm_embed_fwd": ([_I, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P], _I),
    "esm_embed_bwd": ([_I, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _P], _I),
    "esm_layernorm_fwd": ([_I, _P, _P, _P, _P, _P, _P, _I, _I, _F, _P], _I),
    "esm_layernorm_bwd": ([_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P, _P], _I),
    "esm_dropout_mask": ([_P, _I64, _I, _P, _P], _I),
    "esm_gemm": ([ctypes.POINTER(GemmArgs), _P], _I),
    "esm_qkv_rope_fwd": ([_I, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _F, _P], _I),
    "esm_qkv_rope_bwd": ([_I, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _F, _P], _I),
    "esm_attn_prepare": ([_P, _P, _I, _I, _P], _I),
    "esm_attn_fwd": ([_I, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P], _I),
    "esm_attn_bwd": ([_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P], _I),
    "esm_attn_bwd_qkv": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F, _I, _I, _I, _I, _P], _I),
    "esm_attn_fwd_dropout": ([_I, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P], _I),
    "esm_attn_bwd_dropout": ([_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _P, _P], _I),
    "esm_attn_bwd_qkv_dropout": ([_P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _F, _I, _I, _I, _I, _P,
                                  _P], _I),
    "esm_lmhead_xent": ([_I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P], _I),
    "esm_inv_count": ([_P, _P, _P], _I),
    "esm_mlm_mask_ex": ([_P, _P, _P, _P, _I64, _U64, _U64, _I, _I, _I, _I, _I, _P], _I),
    "esm_label_compact": ([_P, _I64, _P, _P, _P, _I, _P], _I),
    "esm_gather_rows": ([_I, _P, _P, _P, _I, _I, _P], _I),
    "esm_scatter_rows": ([_I, _P, _P, _P, _I, _I, _I64, _P], _I),
    "esm_xent_rows": ([_I, _P, _P, _I, _I, _I64, _P, _P, _P], _I),
    "esm_colsum_rows": ([_I, _P, _I, _I, _I64, _P, _P], _I),
    "esm_rank_encode": ([_P, _P, _P, _P, _I64, _P, _I, _I, _I, _P, _P, _P, _P, _I, _P], _I),
    "esm_adamw": ([_P, _P, _P, _P, _P, _P, _I64, _P, _P], _I),
    "esm_adamw_bf16g": ([_P, _P, _P, _P, _P, _P, _I64, _P, _P], _I),
    "esm_cast_f32_bf16": ([_P, _P, _I64, _P], _I),
    "esm_cast_bf16_f32": ([_P, _P, _I64, _P], _I),
    "esm_comm_version": ([], _I),
    "esm_comm_unique_id": ([_P], _I),
    "esm_comm_init": ([_P, _I, _I, _P], _I),
    "esm_comm_destroy": ([_P], _I),
    "esm_comm_allreduce": ([_P, _P, _I64, _I, _P], _I),
    "esm_comm_reduce_scatter": ([_P, _P, _I64, _I, _P], _I),
    "esm_comm_allgather": ([_P, _P, _I64, _I, _P], _I),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes handle; raises EsmKernelError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise EsmKernelError(
            f"{path} not found: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def attn_sched_words(B: int) -> int:
    """Size (int32 words) of the attention scheduling workspace, ESM_ATTN_SCHED_WORDS(B)."""
    return 16 + 2 * B


def check(rc: int, what: str = ""):
    if rc != 0:
        msg = _lib.esm_last_error().decode(errors="replace") if _lib is not None else ""
        raise EsmKernelError(f"{what} failed (code {rc}): {msg}")


def call(name: str, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        check(rc, name)
    return rc


def gemm_call(stream: int, **kw):
    lib = load()
    g = GemmArgs()
    for k, v in kw.items():
        setattr(g, k, v)
    rc = lib.esm_gemm(ctypes.byref(g), stream)
    if rc != 0:
        check(rc, "esm_gemm")
