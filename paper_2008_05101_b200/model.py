"""FATN packed models on the GPU: the reference's model file format and its
packed_forward inference.

* ``parse_model`` / ``serialize_model`` restate the reference's FATN reader and
  writer (R:include/ternkit/model_io.hpp:151-301, format in R:docs/format.md):
  little-endian fields in the listed order, the same validation (magic,
  version, dimensions, packed byte count, trailing bytes), and a byte-identical
  round trip.  They run on the host (file I/O is not on the hot path).
* ``PackedModel.from_spec`` uploads a parsed model: each quantized record
  becomes a device ``PackedConvLayer`` (packed rows, weight sums, s8 operand,
  folded affine); the float stem / head / calibration vectors become device
  tensors.
* ``packed_forward`` is R:tinynet.hpp:713-735 on the GPU: stem matmul_t +
  ReLU, then per block fully_connected_ternary -> calibrated skip-add -> ReLU,
  then the head matmul_t, every float operation in the reference build's order
  (bit-exact logits, tests/test_model_io.py).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

MAGIC = b"FATN"
VERSION = 1  # R:model_io.hpp:21
TAG_FLOAT_FC, TAG_QUANT_FC = 0, 1
FLAG_NONNEG, FLAG_CALIBRATION = 1, 2  # R:model_io.hpp:145-146


class ParseError(ValueError):
    """R:model_io.hpp ParseError: message + byte offset."""

    def __init__(self, msg: str, offset: int):
        super().__init__(f"{msg} (offset {offset})")
        self.offset = offset


@dataclass
class QuantRecord:
    in_c: int
    out_c: int
    kh: int
    kw: int
    stride: int
    pad: int
    nonneg: bool
    alpha_w: tuple
    alpha_a: tuple
    out_scale: float
    gain: np.ndarray
    bias: np.ndarray
    cal_gain: np.ndarray | None
    cal_bias: np.ndarray | None
    weight_sums: np.ndarray
    words: np.ndarray  # [out_c][words_per_row] u64, verbatim

    @property
    def patch_len(self) -> int:
        return self.in_c * self.kh * self.kw


@dataclass
class ModelSpec:
    """Host image of a FATN file (R:tinynet.hpp PackedModel)."""
    in_dim: int
    hidden: int
    n_classes: int
    stem_w: np.ndarray
    stem_b: np.ndarray
    head_w: np.ndarray
    head_b: np.ndarray
    blocks: list = field(default_factory=list)


class _Reader:
    def __init__(self, data: bytes):
        self.b, self.o = memoryview(data), 0

    def take(self, n: int) -> memoryview:
        if self.o + n > len(self.b):
            raise ParseError("unexpected end of file", self.o)
        v = self.b[self.o:self.o + n]
        self.o += n
        return v

    def u8(self):
        return self.take(1)[0]

    def u32(self):
        return struct.unpack("<I", self.take(4))[0]

    def u64(self):
        return struct.unpack("<Q", self.take(8))[0]

    def f32(self):
        return struct.unpack("<f", self.take(4))[0]

    def arr(self, dtype, n):
        return np.frombuffer(bytes(self.take(np.dtype(dtype).itemsize * n)), dtype=dtype).copy()


def words_for_lanes(n: int) -> int:
    return (n + 31) // 32


def decode_words(words: np.ndarray, n: int) -> np.ndarray:
    """Packed u64 rows -> int8 values: value = popcount(code) - 1 (R:codec.hpp:38-40)."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    lanes = np.arange(32, dtype=np.uint64) * np.uint64(2)
    codes = (w[..., None] >> lanes) & np.uint64(3)  # [..., words, 32]
    vals = np.bitwise_count(codes).astype(np.int8) - 1
    return vals.reshape(*w.shape[:-1], -1)[..., :n]


def parse_model(data: bytes) -> ModelSpec:
    """R:model_io.hpp:209-297 (deserialize_model)."""
    r = _Reader(data)
    if bytes(r.take(4)) != MAGIC:
        raise ParseError("bad model magic", 0)
    version = r.u32()
    if version != VERSION:
        raise ParseError(f"unsupported model version {version} (expected {VERSION})", r.o - 4)
    layer_count = r.u32()
    if layer_count < 2:
        raise ParseError("model needs stem and head", r.o - 4)
    stem = head = None
    blocks = []
    for _ in range(layer_count):
        tag, flags = r.u8(), r.u8()
        in_c, out_c, kh, kw, stride, pad = (r.u32() for _ in range(6))
        if in_c <= 0 or out_c <= 0 or in_c >= 2**31 or out_c >= 2**31:
            raise ParseError("nonpositive layer dimension", r.o)
        if tag == TAG_FLOAT_FC:
            wt = r.arr("<f4", in_c * out_c).astype(np.float32)
            bias = r.arr("<f4", out_c).astype(np.float32)
            if stem is None:
                stem = (in_c, out_c, wt, bias)
            else:
                head = (in_c, out_c, wt, bias)
        elif tag == TAG_QUANT_FC:
            aw = (r.f32(), r.f32())
            aa = (r.f32(), r.f32())
            out_scale = r.f32()
            gain = r.arr("<f4", out_c).astype(np.float32)
            bias = r.arr("<f4", out_c).astype(np.float32)
            cg = cb = None
            if flags & FLAG_CALIBRATION:
                cg = r.arr("<f4", in_c).astype(np.float32)
                cb = r.arr("<f4", in_c).astype(np.float32)
            sums = r.arr("<i4", out_c).astype(np.int32)
            wpr = words_for_lanes(in_c * kh * kw)
            nbytes = r.u64()
            if nbytes != out_c * wpr * 8:
                raise ParseError("packed weight byte count mismatch", r.o - 8)
            words = r.arr("<u8", out_c * wpr).astype(np.uint64).reshape(out_c, wpr)
            blocks.append(QuantRecord(in_c, out_c, kh, kw, stride, pad, bool(flags & FLAG_NONNEG), aw, aa,
                                      out_scale, gain, bias, cg, cb, sums, words))
        else:
            raise ParseError("unknown layer tag", r.o - 2)
    if stem is None or head is None:
        raise ParseError("model missing stem or head", r.o)
    if r.o != len(r.b):
        raise ParseError("trailing bytes after last layer", r.o)
    return ModelSpec(stem[0], stem[1], head[1], stem[2], stem[3], head[2], head[3], blocks)


def serialize_model(m: ModelSpec) -> bytes:
    """R:model_io.hpp:151-203 (serialize_model)."""
    out = [MAGIC, struct.pack("<II", VERSION, len(m.blocks) + 2)]

    def float_fc(wt, bias, in_dim, out_dim):
        out.append(struct.pack("<BB6I", TAG_FLOAT_FC, 0, in_dim, out_dim, 1, 1, 1, 0))
        out.append(np.asarray(wt, "<f4").tobytes())
        out.append(np.asarray(bias, "<f4").tobytes())

    float_fc(m.stem_w, m.stem_b, m.in_dim, m.hidden)
    for b in m.blocks:
        flags = (FLAG_NONNEG if b.nonneg else 0) | (FLAG_CALIBRATION if b.cal_gain is not None else 0)
        out.append(struct.pack("<BB6I", TAG_QUANT_FC, flags, b.in_c, b.out_c, b.kh, b.kw, b.stride, b.pad))
        out.append(struct.pack("<5f", b.alpha_w[0], b.alpha_w[1], b.alpha_a[0], b.alpha_a[1], b.out_scale))
        out.append(np.asarray(b.gain, "<f4").tobytes())
        out.append(np.asarray(b.bias, "<f4").tobytes())
        if b.cal_gain is not None:
            out.append(np.asarray(b.cal_gain, "<f4").tobytes())
            out.append(np.asarray(b.cal_bias, "<f4").tobytes())
        out.append(np.asarray(b.weight_sums, "<i4").tobytes())
        out.append(struct.pack("<Q", b.words.size * 8))
        out.append(np.asarray(b.words, "<u8").tobytes())
    float_fc(m.head_w, m.head_b, m.hidden, m.n_classes)
    return b"".join(out)


def load_spec(path: str) -> ModelSpec:
    with open(path, "rb") as f:
        return parse_model(f.read())


def save_spec(m: ModelSpec, path: str) -> None:
    with open(path, "wb") as f:
        f.write(serialize_model(m))


# ---------------------------------------------------------------------------
# device model + packed_forward


class PackedModel:
    """A FATN model resident on the GPU (R:tinynet.hpp:666-671 PackedModel)."""

    def __init__(self, spec: ModelSpec):
        import torch

        from . import ternkit as tk
        self.spec = spec
        self.in_dim, self.hidden, self.n_classes = spec.in_dim, spec.hidden, spec.n_classes
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()  # noqa: E731
        self.stem_w, self.stem_b = dev(spec.stem_w), dev(spec.stem_b)
        self.head_w, self.head_b = dev(spec.head_w), dev(spec.head_b)
        self.blocks = []
        for b in spec.blocks:
            wq = decode_words(b.words, b.patch_len)
            sums = wq.astype(np.int32).sum(axis=1)
            if not np.array_equal(sums, b.weight_sums):  # (the reference trusts the stored sums)
                raise ParseError("weight sums do not match the packed rows", 0)
            layer = tk.make_packed_conv_layer(wq, tk.ConvGeometry(b.in_c, b.out_c, b.kh, b.kw, b.stride, b.pad),
                                              tk.QuantThresholds(*b.alpha_w), tk.QuantThresholds(*b.alpha_a),
                                              b.nonneg, tk.ChannelAffine(b.gain, b.bias), b.out_scale)
            cal = (dev(b.cal_gain), dev(b.cal_bias)) if b.cal_gain is not None else None
            self.blocks.append((layer, cal))

    @classmethod
    def load(cls, path: str) -> "PackedModel":
        return cls(load_spec(path))


def packed_forward(m: PackedModel, x, batch: int):
    """R:tinynet.hpp:713-735 on the GPU -> logits [batch][n_classes] (device)."""
    import torch

    from . import _lib as T
    from . import ternkit as tk
    xd = tk._dev(x, torch.float32).reshape(-1)
    if xd.numel() != batch * m.in_dim:
        raise tk.InvalidArgument(T.TK_ERR_INVALID, "packed_forward: input size mismatch")
    ctx, s = tk.context(), tk._stream()
    h = torch.empty((batch, m.hidden), dtype=torch.float32, device="cuda")
    T.check(T.lib().tk_matmul_t(ctx, xd.data_ptr(), m.stem_w.data_ptr(), m.stem_b.data_ptr(), batch, m.in_dim,
                                m.hidden, 1, h.data_ptr(), s), "matmul_t (stem)")
    for layer, cal in m.blocks:
        # a block maps hidden -> hidden: the reference's FC rejects any other
        # input width (R:linalg.hpp:332-343), and a narrower output would leave
        # the residual add reading past z (so it is rejected here too)
        if layer.geom.in_c != m.hidden or layer.geom.out_c != m.hidden:
            raise tk.InvalidArgument(T.TK_ERR_INVALID, "packed_forward: block width differs from hidden")
        z = tk.fully_connected_ternary(h, batch, layer, check_errors=False)
        T.check(T.lib().tk_residual_relu_rows(ctx, z.data_ptr(), h.data_ptr(), batch * m.hidden, m.hidden,
                                              cal[0].data_ptr() if cal else None,
                                              cal[1].data_ptr() if cal else None, s), "residual_relu_rows")
        h = z
    logits = torch.empty((batch, m.n_classes), dtype=torch.float32, device="cuda")
    T.check(T.lib().tk_matmul_t(ctx, h.data_ptr(), m.head_w.data_ptr(), m.head_b.data_ptr(), batch, m.hidden,
                                m.n_classes, 0, logits.data_ptr(), s), "matmul_t (head)")
    tk.sync("packed_forward")
    return logits


def argmax_rows(logits) -> np.ndarray:
    """R:tinynet.hpp:737-750: first maximum per row, by strict > (NaN never wins)."""
    a = np.asarray(logits.cpu() if hasattr(logits, "cpu") else logits, dtype=np.float32)
    arg = np.zeros(a.shape[0], np.int32)
    best = a[:, 0].copy()
    for c in range(1, a.shape[1]):
        upd = a[:, c] > best
        arg[upd] = c
        best[upd] = a[upd, c]
    return arg
