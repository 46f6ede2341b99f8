"""B200-native deferred-compression LoRaSp hot path (arXiv 1811.11248).

The product is the C-ABI library libhsolve.so (include/hsolve.h, sources in
csrc/); `hsolve` is its ctypes binding with the same function names.
"""
from . import hsolve  # noqa: F401
from .hsolve import (HSError, hs_create, hs_set_stream, hs_analyze, hs_analysis_get_info,  # noqa: F401
                     hs_analysis_export, hs_factor_create, hs_factor_get_stats, hs_factor_export, hs_apply,
                     hs_pcg, hs_spmv)
