"""B200-native (sm_100a) MCMK convolution-as-GEMM hot path (arXiv 1704.04428 kn2row/kn2col,
accumulating variants, im2col baseline) behind the reference's conv-method interface.

The compute path is libconvlab_b200.so (hand-written tcgen05/TMA kernels behind a C ABI,
include/convlab_b200.h); this package is its host-side mirror.  Importing it loads the
library and fails loudly when it is missing -- there is no CPU fallback.
"""
from . import _lib
from . import harness
from .methods import (ALL_METHODS, GPU_METHODS, REFERENCE_METHODS, ConvPlan, LayerConfig, footprint, forward_chain, gemm,
                      method_from_name, method_requires_1x1, parse_method_list, parse_network_text, run_method,
                      shift_add_row)

lib = _lib.lib()  # load now: a missing extension is an import error, not a silent fallback

__all__ = ["ConvPlan", "LayerConfig", "run_method", "forward_chain", "gemm", "shift_add_row", "footprint", "parse_method_list",
           "parse_network_text", "method_from_name", "method_requires_1x1", "ALL_METHODS", "GPU_METHODS",
           "REFERENCE_METHODS", "lib"]
