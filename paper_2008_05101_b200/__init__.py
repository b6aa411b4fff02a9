"""paper_2008_05101_b200 -- B200-native (sm_100a) FATNN ternary hot path.

The reference's ternkit header API (pack / quantize_and_pack / ternary_dot /
im2col_quantize_pack / packed_gemm / conv2d_ternary / fully_connected_ternary)
re-implemented as CUDA kernels behind the C-ABI in include/ternkit_b200.h.
See DESIGN.md.
"""
from ._lib import InvalidArgument  # noqa: F401

__all__ = ["InvalidArgument"]
