"""ctypes binding of libternkit_b200.so (the C-ABI in include/ternkit_b200.h).

The product path has no fallback: if the CUDA library is missing or no GPU is
present, every compute call raises.  Loading the library itself works without
a GPU (the CPU test-suite checks the exported symbols).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libternkit_b200.so")

TK_OK = 0
TK_ERR_INVALID = 1
TK_ERR_THRESHOLDS = 3
TK_ERR_NONFINITE = 4
TK_ERR_NEGATIVE = 5
TK_ERR_OFFSET_SYMMETRIC = 6
TK_ERR_MASKS = 7
TK_ERR_RANGE = 8
TK_ERR_CUDA = 9
TK_ERR_UNSUPPORTED = 10

TK_MODE_WEIGHT = 0
TK_MODE_ACTIVATION_NONNEG = 1
TK_MASK_ON_THE_FLY = 0
TK_MASK_PRECOMPUTED = 1
TK_BACKEND_AUTO = 0
TK_BACKEND_POPC = 1
TK_BACKEND_TC_I8 = 2
TK_BACKEND_TC_F4 = 3
TK_BACKEND_TC_CONV = 4

_vp = C.c_void_p
_sz = C.c_size_t
_i = C.c_int
_f = C.c_float

# name -> (restype, argtypes); mirrors include/ternkit_b200.h exactly
SIGNATURES = {
    "tk_version": (_i, []),
    "tk_status_string": (C.c_char_p, [_i]),
    "tk_context_create": (_i, [_i, C.POINTER(_vp)]),
    "tk_context_destroy": (_i, [_vp]),
    "tk_context_sync": (_i, [_vp, _vp]),
    "tk_quant_thresholds": (_i, [_f, _f, _i, C.POINTER(_f), C.POINTER(_f)]),
    "tk_fuse_bn": (_i, [_vp, _vp, _vp, _vp, _f, _i, _vp, _vp]),
    "tk_pack": (_i, [_vp, _vp, _sz, _vp, _vp]),
    "tk_unpack": (_i, [_vp, _vp, _sz, _vp, _vp]),
    "tk_quantize_pack": (_i, [_vp, _vp, _sz, _sz, _f, _f, _i, _vp, _vp]),
    "tk_ternary_dot_batched": (_i, [_vp, _vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "tk_ternary_dot_premask_batched": (_i, [_vp, _vp, _vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "tk_im2col_quantize_pack": (_i, [_vp, _vp] + [_i] * 8 + [_f, _f, _i, _vp, _vp]),
    "tk_layer_create": (_i, [_vp, _vp] + [_i] * 6 + [_f] * 4 + [_i, _vp, _vp, _f, C.POINTER(_vp)]),
    "tk_layer_destroy": (_i, [_vp]),
    "tk_layer_precompute_masks": (_i, [_vp]),
    "tk_layer_set_backend": (_i, [_vp, _i]),
    "tk_layer_get_backend": (_i, [_vp, _i]),
    "tk_layer_words_host": (_i, [_vp, _vp, _vp]),
    "tk_packed_gemm": (_i, [_vp, _vp, _vp, _sz, _sz, _i, _i, _vp, _vp]),
    "tk_conv2d_ternary": (_i, [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "tk_fully_connected_ternary": (_i, [_vp, _vp, _vp, _i, _i, _vp, _vp]),
    "tk_gemm_levels": (_i, [_vp, _vp, _vp, _i, _i, _vp, _vp]),
    "tk_quantize_levels": (_i, [_vp, _vp, _i, _i, _f, _f, _i, _i, _vp, _vp]),
    "tk_layer_k_pad": (_i, [_vp]),
    "tk_gemm_levels_fp4": (_i, [_vp, _vp, _vp, _i, _i, _vp, _vp]),
    "tk_quantize_levels_fp4": (_i, [_vp, _vp, _i, _i, _f, _f, _i, _i, _vp, _vp]),
    "tk_layer_k_pad_fp4": (_i, [_vp]),
    "tk_net_create": (_i, [_vp, _vp, _i, _i, _i, _i, _i, _i, C.POINTER(_vp)]),
    "tk_net_destroy": (_i, [_vp]),
    "tk_net_out_shape": (_i, [_vp, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "tk_net_is_fused": (_i, [_vp]),
    "tk_net_forward": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "tk_affine_relu_maxpool": (_i, [_vp, _vp] + [_i] * 4 + [_vp, _vp, _vp, _vp]),
    "tk_matmul_t": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "tk_dense_f32": (_i, [_vp, _vp, _vp, _vp, _i, _i, _i, _vp, _vp]),
    "tk_pack_binary": (_i, [_vp, _vp, _sz, _vp, _vp]),
    "tk_binary_dot_batched": (_i, [_vp, _vp, _vp, _sz, _sz, _sz, _vp, _vp]),
    "tk_multibit_dot_batched": (_i, [_vp, _vp, _i, _vp, _i, _vp, _vp, _sz, _sz, _sz, _vp, _vp]),
    "tk_residual_relu_rows": (_i, [_vp, _vp, _vp, C.c_longlong, _i, _vp, _vp, _vp]),
    "tk_stem_conv7x7s2": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp]),
    "tk_net_launches": (_i, [_vp, _i, _i]),
    "tk_net_num_convs": (_i, [_vp]),
    "tk_net_set_timing": (_i, [_vp, _i]),
    "tk_net_conv_times": (_i, [_vp, _vp, _vp]),
    "tk_debug_conv_stamps": (_i, [_vp]),
    "tk_debug_gemm_stamps": (_i, [_vp]),
}

TK_NET_AUTO = 0
TK_NET_GENERIC = 1


class ConvDesc(C.Structure):
    """tk_conv_desc (include/ternkit_b200.h)."""
    _fields_ = [("in_c", _i), ("out_c", _i), ("k", _i), ("stride", _i), ("pad", _i),
                ("weights_host", C.POINTER(C.c_int8)),
                ("tw1", _f), ("tw2", _f), ("ta1", _f), ("ta2", _f),
                ("gain_host", C.POINTER(_f)), ("bias_host", C.POINTER(_f)),
                ("out_scale", _f)]


class BlockDesc(C.Structure):
    """tk_block_desc (include/ternkit_b200.h)."""
    _fields_ = [("n_convs", _i), ("conv", ConvDesc * 3), ("has_down", _i), ("down", ConvDesc)]

_lib = None


def lib():
    """Load libternkit_b200.so once; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class InvalidArgument(ValueError):
    """Python analogue of the reference's std::invalid_argument."""

    def __init__(self, status: int, where: str = ""):
        self.status = status
        msg = lib().tk_status_string(status).decode()
        super().__init__(f"{where}: {msg}" if where else msg)


class CudaError(RuntimeError):
    pass


def check(status: int, where: str = "") -> None:
    if status == TK_OK:
        return
    if status == TK_ERR_CUDA:
        raise CudaError(f"{where}: CUDA runtime error")
    raise InvalidArgument(status, where)
