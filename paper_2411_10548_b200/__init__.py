"""paper_2411_10548_b200 -- B200-native (sm_100a) ESM-2 masked-language-model train step.

Hot path: ESM-2 MLM forward/backward + AdamW + data-parallel gradient
allreduce, as hand-written CUDA kernels behind the C ABI in ``include/esm2_b200.h``.
"""
from .config import EsmConfig, preset, PRESETS  # noqa: F401
from ._lib import EsmKernelError, LIB_PATH  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):  # lazy: importing the package must not require a GPU
    if name in ("EsmForMaskedLM", "init_params", "rope_tables"):
        from . import model
        return getattr(model, name)
    raise AttributeError(name)
