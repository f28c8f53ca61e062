"""B200-native Quartet linear-layer hot path (arXiv 2505.14669, Alg. 1).

PyTorch is plumbing (device memory, streams, autograd, torch.distributed); every hot-path op runs
in libquartet_b200.so (hand-written sm_100a CUDA behind the C ABI in include/quartet_b200.h).
"""

from . import mxfp4, qlinear
from ._lib import LIB_PATH, QuartetError, load
from .mxfp4 import MXOperand, derive_seed, gemm, quant_cols, quant_dual, quant_rows, sign_bits
from .nn import QuartetLinear, QuartetLinearFn, quartet_linear
from .qlinear import (DEFAULT_POLICY, EXACT_POLICY, QUEST, RTN_ABSMAX, SR_ABSMAX, GemmPolicy, LayerContext,
                      QuantScheme, backward, forward)

__all__ = [
    "qlinear", "LIB_PATH", "QuartetError", "load", "MXOperand", "derive_seed", "gemm", "quant_cols", "quant_dual", "quant_rows",
    "sign_bits", "QuartetLinear", "QuartetLinearFn", "quartet_linear", "DEFAULT_POLICY", "EXACT_POLICY", "QUEST",
    "RTN_ABSMAX", "SR_ABSMAX", "GemmPolicy", "LayerContext", "QuantScheme", "backward", "forward",
]
