"""B200-native AlignedServe decode-iteration hot path.

Native code lives in libasv.so (CUDA sm_100a kernels + C++ host runtime behind
the C ABI of include/asv.h).  This package is the thin Python face used by the
tests and bench.py; importing it loads the native library and fails loudly if
it is missing.
"""
from ._lib import lib as _load_native

_load_native()

from .attention import PagedDecodeAttention, Plan  # noqa: E402

__all__ = ["PagedDecodeAttention", "Plan"]
