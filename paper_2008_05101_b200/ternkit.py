"""Python mirror of the reference's ternkit hot-path API on the B200 kernels.

Same names, argument meaning and error behaviour as the reference headers
(R: = /root/reference/proj/include/ternkit/):

    pack / unpack / quantize_and_pack            R:codec.hpp, R:quantizer.hpp
    ternary_dot / ternary_dot_nonneg / ..._premask   R:bitkernels.hpp:116-159
    fuse_bn / make_packed_conv_layer[_from_float]    R:linalg.hpp:70-154
    im2col_quantize_pack / packed_gemm               R:linalg.hpp:173-293
    conv2d_ternary / fully_connected_ternary         R:linalg.hpp:301-343

Inputs may be numpy arrays (host, copied in) or torch CUDA tensors (device,
used in place); outputs are torch CUDA tensors.  Errors raise
``InvalidArgument`` (a ValueError), the analogue of std::invalid_argument.
Every compute call runs the CUDA library -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np
import torch

from . import _lib as T
from ._lib import InvalidArgument, check

kLanesPerWord = 32
kAuxi = 0x5555555555555555


class QuantMode(IntEnum):
    kWeight = T.TK_MODE_WEIGHT
    kActivationNonneg = T.TK_MODE_ACTIVATION_NONNEG


class MaskMode(IntEnum):
    kOnTheFly = T.TK_MASK_ON_THE_FLY
    kPrecomputed = T.TK_MASK_PRECOMPUTED


class Backend(IntEnum):
    AUTO = T.TK_BACKEND_AUTO
    POPC = T.TK_BACKEND_POPC
    TC_I8 = T.TK_BACKEND_TC_I8
    TC_F4 = T.TK_BACKEND_TC_F4
    TC_CONV = T.TK_BACKEND_TC_CONV  # conv2d_ternary: fused implicit-im2col kernel (kind::i8)


@dataclass
class QuantThresholds:
    alpha1: float = 1.0
    alpha2: float = 1.0

    def validate(self) -> None:  # R:codec.hpp:61-65
        if not (self.alpha1 > 0.0) or not (self.alpha2 > 0.0):
            raise InvalidArgument(T.TK_ERR_THRESHOLDS, "QuantThresholds")


def words_for_lanes(n: int) -> int:
    return (n + kLanesPerWord - 1) // kLanesPerWord


def decode_lane(code: int) -> int:  # R:codec.hpp:38-40
    return bin(code & 3).count("1") - 1


def encode_lane(value: int) -> int:  # R:codec.hpp:43-52
    if value == -1:
        return 0b00
    if value == 0:
        return 0b01
    if value == 1:
        return 0b11
    raise InvalidArgument(T.TK_ERR_RANGE, "encode_lane")


# ---------------------------------------------------------------------------
# device plumbing

_ctx: dict[int, int] = {}


def context(device: int | None = None) -> int:
    if not torch.cuda.is_available():
        raise RuntimeError("ternkit_b200 needs a CUDA device (no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _ctx:
        h = C.c_void_p()
        check(T.lib().tk_context_create(dev, C.byref(h)), "tk_context_create")
        _ctx[dev] = h.value
    return _ctx[dev]


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def sync(where: str = "") -> None:
    """Wait for the current stream and raise the first in-kernel error."""
    check(T.lib().tk_context_sync(context(), _stream()), where)


def _dev(a, dtype) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a if a.is_cuda else a.cuda()
        if t.dtype != dtype:
            t = t.to(dtype)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    return torch.from_numpy(arr).to(device="cuda", dtype=dtype).contiguous()


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _words_tensor(nwords: int, shape=None) -> torch.Tensor:
    return torch.empty(shape if shape is not None else (nwords,), dtype=torch.int64, device="cuda")


def as_u64(t: torch.Tensor) -> np.ndarray:
    """Packed words (stored as int64 on device) -> numpy uint64 on host."""
    return t.detach().cpu().numpy().view(np.uint64)


# ---------------------------------------------------------------------------
# codec / quantizer


@dataclass
class PackedTernaryVector:  # R:codec.hpp:74-82
    words: torch.Tensor          # int64 view of the u64 words
    logical_len: int = 0
    nonneg_offset: bool = False

    def lane_capacity(self) -> int:
        return self.words.numel() * kLanesPerWord


def pack(values, check_errors: bool = True) -> PackedTernaryVector:
    """R:codec.hpp:89-100."""
    v = _dev(values, torch.int8).reshape(-1)
    n = v.numel()
    w = _words_tensor(words_for_lanes(n))
    check(T.lib().tk_pack(context(), _p(v), n, _p(w), _stream()), "pack")
    if check_errors:
        sync("pack")
    return PackedTernaryVector(w, n, False)


def unpack(v: PackedTernaryVector) -> torch.Tensor:
    """R:codec.hpp:107-117."""
    out = torch.empty(v.logical_len, dtype=torch.int8, device="cuda")
    check(T.lib().tk_unpack(context(), _p(v.words), v.logical_len, _p(out), _stream()), "unpack")
    return out


def quantize_and_pack(x, t: QuantThresholds, mode: QuantMode,
                      check_errors: bool = True) -> PackedTernaryVector:
    """R:quantizer.hpp:159-170."""
    xd = _dev(x, torch.float32).reshape(-1)
    n = xd.numel()
    w = _words_tensor(words_for_lanes(n))
    check(T.lib().tk_quantize_pack(context(), _p(xd), 1, n, t.alpha1, t.alpha2, int(mode),
                                   _p(w), _stream()), "quantize_and_pack")
    if check_errors:
        sync("quantize_and_pack")
    return PackedTernaryVector(w, n, mode == QuantMode.kActivationNonneg)


def quantize_and_pack_rows(x, t: QuantThresholds, mode: QuantMode,
                           check_errors: bool = True) -> torch.Tensor:
    """Row-batched quantize_and_pack: x [rows][n] -> words [rows][words_for_lanes(n)]."""
    xd = _dev(x, torch.float32)
    rows, n = xd.shape
    w = _words_tensor(0, (rows, words_for_lanes(n)))
    check(T.lib().tk_quantize_pack(context(), _p(xd), rows, n, t.alpha1, t.alpha2, int(mode),
                                   _p(w), _stream()), "quantize_and_pack")
    if check_errors:
        sync("quantize_and_pack")
    return w


def quant_thresholds(t: QuantThresholds, mode: QuantMode) -> tuple[float, float]:
    """Exact float thresholds of the quantizer (host helper, no GPU needed)."""
    t0, t1 = C.c_float(), C.c_float()
    check(T.lib().tk_quant_thresholds(t.alpha1, t.alpha2, int(mode), C.byref(t0), C.byref(t1)),
          "quant_thresholds")
    return t0.value, t1.value


# ---------------------------------------------------------------------------
# inner products


def ternary_dot_batched(x: torch.Tensor, y: torch.Tensor, wsum=None, seeds=None) -> torch.Tensor:
    """x, y: [pairs][words] packed words -> int64 [pairs] (ternary_dot, or
    ternary_dot_nonneg when wsum is given; with `seeds` [pairs][words] the
    premask form, R:bitkernels.hpp:87-97)."""
    xd, yd = _dev(x, torch.int64), _dev(y, torch.int64)
    if xd.shape != yd.shape:
        raise InvalidArgument(T.TK_ERR_INVALID, "ternary_dot: length mismatch")
    pairs, words = xd.shape
    ws = None if wsum is None else _dev(wsum, torch.int64)
    out = torch.empty(pairs, dtype=torch.int64, device="cuda")
    if seeds is None:
        check(T.lib().tk_ternary_dot_batched(context(), _p(xd), _p(yd), words, pairs, _p(ws), _p(out),
                                             _stream()), "ternary_dot")
    else:
        sd = _dev(seeds, torch.int64).reshape(pairs, words)
        check(T.lib().tk_ternary_dot_premask_batched(context(), _p(xd), _p(yd), _p(sd), words, pairs, _p(ws),
                                                     _p(out), _stream()), "ternary_dot_premask")
    return out


def ternary_zero_seed(yw: int) -> int:  # R:bitkernels.hpp:47-49
    return ((yw ^ (yw >> 1)) & kAuxi) & 0xFFFFFFFFFFFFFFFF


def ternary_multiply_word(xw: int, yw: int) -> int:  # R:bitkernels.hpp:55-63
    return ternary_multiply_word_premask(xw, yw, ternary_zero_seed(yw))


def ternary_multiply_word_premask(xw: int, yw: int, d: int) -> int:  # R:bitkernels.hpp:66-72
    m = 0xFFFFFFFFFFFFFFFF
    return ((~(xw ^ yw) & m) | d) & ~(d << 1) & m


def ternary_dot_words(x, y, words: int | None = None) -> int:
    """detail::ternary_dot_words (R:bitkernels.hpp:76-85): raw word buffers."""
    xd, yd = _dev(x, torch.int64).reshape(-1), _dev(y, torch.int64).reshape(-1)
    n = xd.numel() if words is None else words
    return int(ternary_dot_batched(xd[:n].view(1, -1), yd[:n].view(1, -1)).item())


def ternary_dot_words_premask(x, y, seed, words: int | None = None) -> int:
    """detail::ternary_dot_words_premask (R:bitkernels.hpp:87-97)."""
    xd, yd = _dev(x, torch.int64).reshape(-1), _dev(y, torch.int64).reshape(-1)
    sd = _dev(seed, torch.int64).reshape(-1)
    n = xd.numel() if words is None else words
    return int(ternary_dot_batched(xd[:n].view(1, -1), yd[:n].view(1, -1), seeds=sd[:n].view(1, -1)).item())


def ternary_dot(x: PackedTernaryVector, y: PackedTernaryVector) -> int:
    """R:bitkernels.hpp:116-123."""
    if x.logical_len != y.logical_len:
        raise InvalidArgument(T.TK_ERR_INVALID, "ternary_dot: length mismatch")
    return int(ternary_dot_batched(x.words.view(1, -1), y.words.view(1, -1)).item())


def make_zero_seeds(y: PackedTernaryVector) -> torch.Tensor:
    """R:bitkernels.hpp:127-134 (device words)."""
    w = y.words
    return (w ^ (w >> 1)) & kAuxi


def ternary_dot_premask(x: PackedTernaryVector, y: PackedTernaryVector, seeds) -> int:
    """R:bitkernels.hpp:136-147: the TM uses the supplied seeds as given."""
    if x.logical_len != y.logical_len:
        raise InvalidArgument(T.TK_ERR_INVALID, "ternary_dot_premask: length mismatch")
    if len(seeds) != y.words.numel():
        raise InvalidArgument(T.TK_ERR_INVALID, "ternary_dot_premask: seed buffer mismatch")
    return int(ternary_dot_batched(x.words.view(1, -1), y.words.view(1, -1),
                                   seeds=_dev(seeds, torch.int64).view(1, -1)).item())


def ternary_dot_nonneg(a: PackedTernaryVector, w: PackedTernaryVector, w_sum: int) -> int:
    """R:bitkernels.hpp:151-159."""
    if not a.nonneg_offset:
        raise InvalidArgument(T.TK_ERR_INVALID,
                              "ternary_dot_nonneg: activation vector lacks the nonneg offset flag")
    return ternary_dot(a, w) + int(w_sum)


# ---------------------------------------------------------------------------
# paper baselines (R:bitkernels.hpp:99-224): binary and bit-plane multi-bit dots


@dataclass
class PackedBinaryVector:  # R:bitkernels.hpp:165-168
    words: torch.Tensor  # int64 view of u64 words (device)
    logical_len: int


def pack_binary(values, check_errors: bool = True) -> PackedBinaryVector:
    """R:bitkernels.hpp:170-182: values in {-1, +1} only."""
    v = _dev(values, torch.int8).reshape(-1)
    n = v.numel()
    w = torch.empty((n + 63) // 64, dtype=torch.int64, device="cuda")
    check(T.lib().tk_pack_binary(context(), _p(v), n, _p(w), _stream()), "pack_binary")
    if check_errors:
        sync("pack_binary")
    return PackedBinaryVector(w, n)


def binary_dot_batched(x: torch.Tensor, y: torch.Tensor, logical_len: int) -> torch.Tensor:
    """x, y: [pairs][words] packed binary rows -> int64 [pairs]."""
    xd, yd = _dev(x, torch.int64), _dev(y, torch.int64)
    if xd.shape != yd.shape:
        raise InvalidArgument(T.TK_ERR_INVALID, "binary_dot: length mismatch")
    pairs, words = xd.shape
    out = torch.empty(pairs, dtype=torch.int64, device="cuda")
    check(T.lib().tk_binary_dot_batched(context(), _p(xd), _p(yd), words, logical_len, pairs, _p(out), _stream()),
          "binary_dot")
    return out


def binary_dot(x: PackedBinaryVector, y: PackedBinaryVector) -> int:
    """R:bitkernels.hpp:184-191."""
    if x.logical_len != y.logical_len:
        raise InvalidArgument(T.TK_ERR_INVALID, "binary_dot: length mismatch")
    return int(binary_dot_batched(x.words.view(1, -1), y.words.view(1, -1), x.logical_len).item())


@dataclass
class MultiBitVector:  # R:bitkernels.hpp:194-201
    planes: list
    scales: list

    def logical_len(self) -> int:
        return self.planes[0].logical_len if self.planes else 0


def multibit_dot_batched(x_planes: torch.Tensor, x_scales, y_planes: torch.Tensor, y_scales,
                         logical_len: int) -> torch.Tensor:
    """x_planes [m][pairs][words], y_planes [k][pairs][words] -> f64 [pairs]."""
    xp, yp = _dev(x_planes, torch.int64), _dev(y_planes, torch.int64)
    def scales(v):  # host sequences or device f64 tensors (the latter are graph-capturable)
        if isinstance(v, torch.Tensor) and v.is_cuda:
            return v.to(torch.float64).contiguous()
        return torch.as_tensor(np.asarray(v, np.float64)).cuda()
    sx, sy = scales(x_scales), scales(y_scales)
    m, pairs, words = xp.shape
    k = yp.shape[0]
    if yp.shape[1:] != xp.shape[1:] or sx.numel() != m or sy.numel() != k:
        raise InvalidArgument(T.TK_ERR_INVALID, "multibit_dot: malformed operand")
    out = torch.empty(pairs, dtype=torch.float64, device="cuda")
    check(T.lib().tk_multibit_dot_batched(context(), _p(xp), m, _p(yp), k, _p(sx), _p(sy), words, logical_len,
                                          pairs, _p(out), _stream()), "multibit_dot")
    return out


def multibit_dot(x: MultiBitVector, y: MultiBitVector) -> float:
    """R:bitkernels.hpp:196-222 (same validation, bit-identical f64 result)."""
    if (not x.planes or not y.planes or len(x.planes) != len(x.scales) or len(y.planes) != len(y.scales)):
        raise InvalidArgument(T.TK_ERR_INVALID, "multibit_dot: malformed operand")
    n = x.logical_len()
    if any(p.logical_len != n for p in list(x.planes) + list(y.planes)):
        raise InvalidArgument(T.TK_ERR_INVALID, "multibit_dot: plane length mismatch")
    xp = torch.stack([p.words for p in x.planes]).unsqueeze(1)
    yp = torch.stack([p.words for p in y.planes]).unsqueeze(1)
    return float(multibit_dot_batched(xp, x.scales, yp, y.scales, n).item())


# ---------------------------------------------------------------------------
# linalg


@dataclass
class TensorShape:  # R:linalg.hpp:25-31
    n: int = 0
    c: int = 0
    h: int = 0
    w: int = 0

    def count(self) -> int:
        return self.n * self.c * self.h * self.w


@dataclass
class ConvGeometry:  # R:linalg.hpp:33-55
    in_c: int = 0
    out_c: int = 0
    kh: int = 3
    kw: int = 3
    stride: int = 1
    pad: int = 1

    def patch_len(self) -> int:
        return self.in_c * self.kh * self.kw

    def out_h(self, h: int) -> int:
        return (h + 2 * self.pad - self.kh) // self.stride + 1

    def out_w(self, w: int) -> int:
        return (w + 2 * self.pad - self.kw) // self.stride + 1

    def validate(self, x: TensorShape) -> None:
        if (self.in_c <= 0 or self.out_c <= 0 or self.kh <= 0 or self.kw <= 0 or
                self.stride <= 0 or self.pad < 0):
            raise InvalidArgument(T.TK_ERR_INVALID, "conv geometry: nonpositive dimension")
        if x.c != self.in_c:
            raise InvalidArgument(T.TK_ERR_INVALID, "conv geometry: channel count mismatch")
        if x.h + 2 * self.pad < self.kh or x.w + 2 * self.pad < self.kw:
            raise InvalidArgument(T.TK_ERR_INVALID, "conv geometry: kernel exceeds padded input")


@dataclass
class ChannelAffine:  # R:linalg.hpp:58-66
    gain: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    bias: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))

    @staticmethod
    def identity(channels: int) -> "ChannelAffine":
        return ChannelAffine(np.ones(channels, np.float32), np.zeros(channels, np.float32))


def fuse_bn(mean, var, gamma, beta, eps: float) -> ChannelAffine:
    """R:linalg.hpp:70-91 (host parameter folding, reference float semantics)."""
    arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (mean, var, gamma, beta)]
    c = arrs[0].size
    if any(a.size != c for a in arrs):
        raise InvalidArgument(T.TK_ERR_INVALID, "fuse_bn: per-channel stat size mismatch")
    g = np.empty(c, np.float32)
    b = np.empty(c, np.float32)
    check(T.lib().tk_fuse_bn(*[a.ctypes.data for a in arrs], eps, c, g.ctypes.data, b.ctypes.data),
          "fuse_bn")
    return ChannelAffine(g, b)


class PackedConvLayer:
    """R:linalg.hpp:95-114 -- owns the device copy of the packed weight rows,
    weight sums, zero masks, the s8 tensor-core operand and the folded affine."""

    def __init__(self, handle: int, geom: ConvGeometry, thr_w: QuantThresholds,
                 thr_a: QuantThresholds, activation_nonneg: bool, fused: ChannelAffine,
                 out_scale: float):
        self._h = handle
        self.geom = geom
        self.thr_w = thr_w
        self.thr_a = thr_a
        self.activation_nonneg = activation_nonneg
        self.fused = fused
        self.out_scale = out_scale
        self._masks_ready = False

    @property
    def handle(self) -> int:
        return self._h

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                T.lib().tk_layer_destroy(self._h)
            except Exception:
                pass
            self._h = None

    def masks_ready(self) -> bool:
        return self._masks_ready

    def precompute_masks(self) -> None:
        check(T.lib().tk_layer_precompute_masks(self._h), "precompute_masks")
        self._masks_ready = True

    def set_backend(self, backend: Backend) -> None:
        check(T.lib().tk_layer_set_backend(self._h, int(backend)), "set_backend")

    def backend_for(self, m_rows: int) -> Backend:
        return Backend(T.lib().tk_layer_get_backend(self._h, m_rows))

    @property
    def weights_words(self) -> np.ndarray:
        """Packed rows as the reference stores them ([out_c][words] u64)."""
        wpr = words_for_lanes(self.geom.patch_len())
        w = np.empty((self.geom.out_c, wpr), np.uint64)
        check(T.lib().tk_layer_words_host(self._h, w.ctypes.data, None), "weights")
        return w

    @property
    def weight_sums(self) -> np.ndarray:
        s = np.empty(self.geom.out_c, np.int32)
        check(T.lib().tk_layer_words_host(self._h, None, s.ctypes.data), "weight_sums")
        return s


def make_packed_conv_layer(ternary_weights, geom: ConvGeometry, thr_w: QuantThresholds,
                           thr_a: QuantThresholds, activation_nonneg: bool,
                           fused: ChannelAffine | None = None,
                           out_scale: float = 1.0) -> PackedConvLayer:
    """R:linalg.hpp:118-144."""
    w = np.ascontiguousarray(np.asarray(ternary_weights, dtype=np.int8).reshape(-1))
    k = geom.patch_len()
    if w.size != k * geom.out_c:
        raise InvalidArgument(T.TK_ERR_INVALID, "make_packed_conv_layer: weight size mismatch")
    if fused is None or len(fused.gain) == 0:
        fused = ChannelAffine.identity(geom.out_c)
    gain = np.ascontiguousarray(fused.gain, np.float32)
    bias = np.ascontiguousarray(fused.bias, np.float32)
    h = C.c_void_p()
    context()
    check(T.lib().tk_layer_create(context(), w.ctypes.data, geom.in_c, geom.out_c, geom.kh,
                                  geom.kw, geom.stride, geom.pad, thr_w.alpha1, thr_w.alpha2,
                                  thr_a.alpha1, thr_a.alpha2, int(bool(activation_nonneg)),
                                  gain.ctypes.data, bias.ctypes.data, float(out_scale),
                                  C.byref(h)), "make_packed_conv_layer")
    return PackedConvLayer(h.value, geom, thr_w, thr_a, bool(activation_nonneg),
                           ChannelAffine(gain, bias), float(out_scale))


def quantize_weight(p, t: QuantThresholds) -> np.ndarray:
    """R:quantizer.hpp:62-70 on the GPU quantizer (weight mode), host int8 out."""
    t.validate()
    pv = quantize_and_pack(p, t, QuantMode.kWeight)
    return unpack(pv).cpu().numpy()


def make_packed_conv_layer_from_float(weights, geom: ConvGeometry, thr_w: QuantThresholds,
                                      thr_a: QuantThresholds, activation_nonneg: bool,
                                      fused: ChannelAffine | None = None,
                                      out_scale: float = 1.0) -> PackedConvLayer:
    """R:linalg.hpp:147-154."""
    q = quantize_weight(weights, thr_w)
    return make_packed_conv_layer(q, geom, thr_w, thr_a, activation_nonneg, fused, out_scale)


@dataclass
class Im2colBuffer:  # R:linalg.hpp:158-169
    words: torch.Tensor  # [row_count][words_per_row] int64 view of u64
    words_per_row: int = 0
    row_count: int = 0
    row_len: int = 0
    nonneg_offset: bool = False
    batch: int = 0
    out_h: int = 0
    out_w: int = 0

    def row(self, r: int) -> torch.Tensor:
        return self.words[r]


def im2col_quantize_pack(x, shape: TensorShape, t: QuantThresholds, geom: ConvGeometry,
                         mode: QuantMode, check_errors: bool = True) -> Im2colBuffer:
    """R:linalg.hpp:173-225."""
    geom.validate(shape)
    t.validate()
    xd = _dev(x, torch.float32).reshape(-1)
    if xd.numel() != shape.count():
        raise InvalidArgument(T.TK_ERR_INVALID, "im2col: input size does not match shape")
    oh, ow = geom.out_h(shape.h), geom.out_w(shape.w)
    k = geom.patch_len()
    rows = shape.n * oh * ow
    wpr = words_for_lanes(k)
    out = _words_tensor(0, (rows, wpr))
    check(T.lib().tk_im2col_quantize_pack(context(), _p(xd), shape.n, shape.c, shape.h, shape.w,
                                          geom.kh, geom.kw, geom.stride, geom.pad, t.alpha1,
                                          t.alpha2, int(mode), _p(out), _stream()),
          "im2col_quantize_pack")
    if check_errors:
        sync("im2col_quantize_pack")
    return Im2colBuffer(out, wpr, rows, k, mode == QuantMode.kActivationNonneg, shape.n, oh, ow)


def packed_gemm(a: Im2colBuffer, layer: PackedConvLayer, mask_mode: MaskMode = MaskMode.kOnTheFly,
                workers: int = 1) -> torch.Tensor:
    """R:linalg.hpp:232-293 -> int32 [row_count][out_c] (workers is accepted
    and ignored: the CUDA grid replaces the CPU row partition)."""
    if mask_mode == MaskMode.kPrecomputed and not layer.masks_ready():
        raise InvalidArgument(T.TK_ERR_MASKS, "packed_gemm")
    out = torch.empty((a.row_count, layer.geom.out_c), dtype=torch.int32, device="cuda")
    check(T.lib().tk_packed_gemm(context(), layer.handle, _p(a.words), a.row_count, a.row_len,
                                 int(a.nonneg_offset), int(mask_mode), _p(out), _stream()),
          "packed_gemm")
    return out


@dataclass
class ConvResult:  # R:linalg.hpp:295-298
    data: torch.Tensor
    shape: TensorShape


def conv2d_ternary(x, shape: TensorShape, layer: PackedConvLayer,
                   mask_mode: MaskMode = MaskMode.kOnTheFly, workers: int = 1,
                   check_errors: bool = True) -> ConvResult:
    """R:linalg.hpp:301-328 -> f32 NCHW."""
    layer.geom.validate(shape)
    xd = _dev(x, torch.float32).reshape(-1)
    if xd.numel() != shape.count():
        raise InvalidArgument(T.TK_ERR_INVALID, "im2col: input size does not match shape")
    if mask_mode == MaskMode.kPrecomputed and not layer.masks_ready():
        raise InvalidArgument(T.TK_ERR_MASKS, "packed_gemm")
    g = layer.geom
    oh, ow = g.out_h(shape.h), g.out_w(shape.w)
    out = torch.empty((shape.n, g.out_c, oh, ow), dtype=torch.float32, device="cuda")
    check(T.lib().tk_conv2d_ternary(context(), layer.handle, _p(xd), shape.n, shape.h, shape.w,
                                    int(mask_mode), _p(out), _stream()), "conv2d_ternary")
    if check_errors:
        sync("conv2d_ternary")
    return ConvResult(out, TensorShape(shape.n, g.out_c, oh, ow))


def fully_connected_ternary(x, batch: int, layer: PackedConvLayer,
                            mask_mode: MaskMode = MaskMode.kOnTheFly,
                            check_errors: bool = True) -> torch.Tensor:
    """R:linalg.hpp:332-343 -> f32 [batch][out_c]."""
    g = layer.geom
    if g.kh != 1 or g.kw != 1 or g.pad != 0:
        raise InvalidArgument(T.TK_ERR_INVALID, "fully_connected_ternary: expects 1x1 geometry")
    xd = _dev(x, torch.float32).reshape(-1)
    if xd.numel() != batch * g.in_c:
        raise InvalidArgument(T.TK_ERR_INVALID, "im2col: input size does not match shape")
    layer.thr_a.validate()
    if mask_mode == MaskMode.kPrecomputed and not layer.masks_ready():
        raise InvalidArgument(T.TK_ERR_MASKS, "packed_gemm")
    out = torch.empty((batch, g.out_c), dtype=torch.float32, device="cuda")
    check(T.lib().tk_fully_connected_ternary(context(), layer.handle, _p(xd), batch,
                                             int(mask_mode), _p(out), _stream()),
          "fully_connected_ternary")
    if check_errors:
        sync("fully_connected_ternary")
    return out


# ---------------------------------------------------------------------------
# level-operand entry points (tensor-core path without the 2-bit pack step)


# E2M1 nibble of each level -1, 0, 1, 2 (the FP4 operand, include/ternkit_b200.h)
_E2M1 = {-1: 0xA, 0: 0x0, 1: 0x2, 2: 0x4}


class LevelOperand:
    """Quantization levels of `rows` rows in a tensor-core operand layout.

    fmt "s8": one s8 level per byte, K-block-major [k_pad/128][m_pad][128].
    fmt "fp4": E2M1 nibbles (even k low), [k_pad/256][m_pad][128 B]."""

    def __init__(self, data: torch.Tensor, rows: int, k_pad: int, fmt: str = "s8"):
        self.data, self.rows, self.k_pad, self.fmt = data, rows, k_pad, fmt

    def dense(self) -> torch.Tensor:
        """[rows][k_pad] s8 levels (a copy), for inspection and tests."""
        if self.fmt == "s8":
            return self.data.permute(1, 0, 2).reshape(-1, self.k_pad)[: self.rows]
        b = self.data.permute(1, 0, 2).reshape(-1, self.k_pad // 2)[: self.rows].to(torch.int32)
        nib = torch.stack([b & 0xF, b >> 4], dim=-1).reshape(b.shape[0], -1)
        lut = torch.full((16,), 127, dtype=torch.int8, device=b.device)
        for lv, code in _E2M1.items():
            lut[code] = lv
        return lut[nib.long()]


def quantize_levels(x, t: QuantThresholds, mode: QuantMode, k_pad: int, fmt: str = "s8") -> LevelOperand:
    """f32 [rows][n] -> quantization levels (zero padded to k_pad) in `fmt`."""
    xd = _dev(x, torch.float32)
    rows, n = xd.shape
    m_pad = (rows + 127) // 128 * 128
    if fmt == "s8":
        out = torch.zeros((k_pad // 128, m_pad, 128), dtype=torch.int8, device="cuda")
        fn = T.lib().tk_quantize_levels
    elif fmt == "fp4":
        out = torch.zeros((k_pad // 256, m_pad, 128), dtype=torch.uint8, device="cuda")
        fn = T.lib().tk_quantize_levels_fp4
    else:
        raise ValueError(f"unknown level format {fmt!r}")
    check(fn(context(), _p(xd), rows, n, t.alpha1, t.alpha2, int(mode), k_pad, _p(out), _stream()),
          "quantize_levels")
    return LevelOperand(out, rows, k_pad, fmt)


def gemm_levels(a: LevelOperand, layer: PackedConvLayer, fused: bool = False,
                out: torch.Tensor | None = None) -> torch.Tensor:
    """Ternary GEMM on level operands (s8: kind::i8, fp4: kind::mxf4): int32
    accumulators, or (fused=True) f32 rows after the folded-BN epilogue."""
    m = a.rows
    if out is None:
        out = torch.empty((m, layer.geom.out_c), dtype=torch.float32 if fused else torch.int32, device="cuda")
    fn = T.lib().tk_gemm_levels_fp4 if a.fmt == "fp4" else T.lib().tk_gemm_levels
    check(fn(context(), layer.handle, _p(a.data), m, 1 if fused else 0, _p(out), _stream()), "gemm_levels")
    return out


def layer_k_pad(layer: PackedConvLayer, fmt: str = "s8") -> int:
    return (T.lib().tk_layer_k_pad_fp4 if fmt == "fp4" else T.lib().tk_layer_k_pad)(layer.handle)
