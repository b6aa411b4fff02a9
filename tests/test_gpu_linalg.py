"""GPU parity: im2col_quantize_pack, packed_gemm, conv2d_ternary and
fully_connected_ternary vs the reference's golden outputs and the C oracle,
on every pipe (LOP3+POPC, tcgen05 kind::i8 and kind::mxf4).  Integers and packed words
bit-exact; float epilogue bit-exact (same FMA shape as the reference build)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def backends(tk):
    return [tk.Backend.POPC, tk.Backend.TC_I8, tk.Backend.TC_F4]


def _layer(tk, wq, c, oc, k, s, p, ta=(0.5, 0.9), nonneg=True, gain=None, bias=None, out_scale=1.0,
           tw=(1.0, 1.0)):
    g = tk.ConvGeometry(c, oc, k, k, s, p)
    aff = None if gain is None else tk.ChannelAffine(gain, bias)
    return tk.make_packed_conv_layer(wq, g, tk.QuantThresholds(*tw), tk.QuantThresholds(*ta), nonneg,
                                     aff, out_scale)


def test_im2col_kats(tk, golden):
    QT, QM, TS, CG = tk.QuantThresholds, tk.QuantMode, tk.TensorShape, tk.ConvGeometry
    b = tk.im2col_quantize_pack(golden["im2col_1x1_x"], TS(1, 3, 2, 2), QT(1, 1), CG(3, 1, 1, 1, 1, 0),
                                QM.kWeight)
    assert b.row_count == 4 and b.row_len == 3
    assert np.array_equal(u64(b.words), golden["im2col_1x1_rows"])
    b = tk.im2col_quantize_pack(np.ones(9, np.float32), TS(1, 1, 3, 3), QT(1, 1), CG(1, 1, 3, 3, 1, 1),
                                QM.kWeight)
    assert np.array_equal(u64(b.words), golden["im2col_corner_rows"])
    b = tk.im2col_quantize_pack(golden["im2col_strided_x"], TS(2, 3, 5, 4), QT(0.6, 1.1),
                                CG(3, 2, 3, 3, 2, 1), QM.kActivationNonneg)
    assert b.nonneg_offset and np.array_equal(u64(b.words), golden["im2col_strided_rows"])
    with pytest.raises(tk.InvalidArgument):   # channel mismatch, R:tests/test_linalg.cpp:165-175
        tk.im2col_quantize_pack(np.zeros(32, np.float32), TS(1, 2, 4, 4), QT(1, 1), CG(3, 1, 3, 3, 1, 1),
                                QM.kWeight)
    with pytest.raises(tk.InvalidArgument):
        tk.im2col_quantize_pack(np.zeros(3, np.float32), TS(1, 2, 4, 4), QT(1, 1), CG(2, 1, 3, 3, 1, 1),
                                QM.kWeight)


@pytest.mark.parametrize("backend", ["POPC", "TC_I8", "TC_F4", "TC_CONV"])
def test_conv_shapes_golden(tk, golden, backend):
    QT, QM, TS, CG = tk.QuantThresholds, tk.QuantMode, tk.TensorShape, tk.ConvGeometry
    for i, (c, r, k, s, p, b) in enumerate(golden["conv_shapes"]):
        c, r, k, s, p, b = map(int, (c, r, k, s, p, b))
        buf = tk.im2col_quantize_pack(golden[f"conv{i}_x"], TS(b, c, r, r), QT(0.5, 0.9), CG(c, c, k, k, s, p),
                                      QM.kActivationNonneg)
        assert np.array_equal(u64(buf.words), golden[f"conv{i}_rows"]), i
        layer = _layer(tk, golden[f"conv{i}_w"], c, c, k, s, p, gain=golden[f"conv{i}_gain"],
                       bias=golden[f"conv{i}_bias"], out_scale=0.37, tw=(0.8, 1.2))
        layer.set_backend(tk.Backend[backend])
        acc = tk.packed_gemm(buf, layer).cpu().numpy()
        assert np.array_equal(acc, golden[f"conv{i}_acc"]), (i, backend)
        y = tk.conv2d_ternary(golden[f"conv{i}_x"], TS(b, c, r, r), layer).data.cpu().numpy()
        assert np.array_equal(y.view(np.int32), golden[f"conv{i}_y"].view(np.int32)), (i, backend)
        # symmetric activations through a symmetric layer
        lsym = _layer(tk, golden[f"conv{i}_w"], c, c, k, s, p, ta=(0.8, 1.2), nonneg=False)
        lsym.set_backend(tk.Backend[backend])
        bs = tk.im2col_quantize_pack(golden[f"conv{i}_xs"], TS(b, c, r, r), QT(0.8, 1.2), CG(c, c, k, k, s, p),
                                     QM.kWeight)
        assert np.array_equal(tk.packed_gemm(bs, lsym).cpu().numpy(), golden[f"conv{i}_acc_sym"]), (i, backend)
        with pytest.raises(tk.InvalidArgument):   # offset rows into a symmetric layer
            tk.packed_gemm(buf, lsym)


def test_gemm_mask_modes_and_errors(tk, oracle):
    """R:tests/test_linalg.cpp:215-231: precomputed mode requires masks; modes agree."""
    rng = np.random.default_rng(38)
    wq = rng.integers(-1, 2, (64, 32)).astype(np.int8)
    layer = _layer(tk, wq, 32, 64, 1, 1, 0, ta=(0.5, 0.5))
    x = np.abs(rng.standard_normal(10 * 32)).astype(np.float32)
    buf = tk.im2col_quantize_pack(x, tk.TensorShape(10, 32, 1, 1), tk.QuantThresholds(0.5, 0.5),
                                  layer.geom, tk.QuantMode.kActivationNonneg)
    with pytest.raises(tk.InvalidArgument):
        tk.packed_gemm(buf, layer, tk.MaskMode.kPrecomputed)
    a = tk.packed_gemm(buf, layer, tk.MaskMode.kOnTheFly).cpu().numpy()
    layer.precompute_masks()
    b = tk.packed_gemm(buf, layer, tk.MaskMode.kPrecomputed).cpu().numpy()
    c = tk.packed_gemm(buf, layer, tk.MaskMode.kOnTheFly, workers=3).cpu().numpy()
    assert np.array_equal(a, b) and np.array_equal(a, c)
    wrows, ws = oracle.pack_rows(wq)
    assert np.array_equal(a, oracle.packed_gemm(u64(buf.words), wrows, ws, 1))
    # all-zero weights -> zero gemm (R:tests/test_linalg.cpp:233-242)
    z = _layer(tk, np.zeros((3, 8), np.int8), 8, 3, 1, 1, 0, ta=(0.5, 0.5))
    bz = tk.im2col_quantize_pack(x[:32], tk.TensorShape(4, 8, 1, 1), tk.QuantThresholds(0.5, 0.5), z.geom,
                                 tk.QuantMode.kActivationNonneg)
    assert not tk.packed_gemm(bz, z).cpu().numpy().any()
    with pytest.raises(tk.InvalidArgument):
        tk.make_packed_conv_layer(np.zeros(7, np.int8), tk.ConvGeometry(4, 2, 1, 1, 1, 0),
                                  tk.QuantThresholds(), tk.QuantThresholds(), True)


def test_selector_row(tk):
    """R:tests/test_linalg.cpp:177-190."""
    n = 40
    w = np.zeros(n, np.int8)
    w[0] = 1
    layer = _layer(tk, w, n, 1, 1, 1, 0, ta=(1, 1), nonneg=False)
    x = np.random.default_rng(35).standard_normal(6 * n).astype(np.float32)
    buf = tk.im2col_quantize_pack(x, tk.TensorShape(6, n, 1, 1), tk.QuantThresholds(1, 1), layer.geom,
                                  tk.QuantMode.kWeight)
    out = tk.packed_gemm(buf, layer).cpu().numpy().reshape(-1)
    want = [(1 if v > 0.5 else (-1 if v < -0.5 else 0)) for v in x[::n]]
    assert list(out) == want


@pytest.mark.parametrize("backend", ["POPC", "TC_I8", "TC_F4", "TC_CONV"])
def test_conv_properties(tk, oracle, backend):
    """Batch independence (exact), out_scale linearity, geometry grid, zero-input FC
    (R:tests/test_linalg.cpp:267-380)."""
    rng = np.random.default_rng(45)
    TS = tk.TensorShape
    wq = rng.integers(-1, 2, (5, 27)).astype(np.int8)
    layer = _layer(tk, wq, 3, 5, 3, 1, 1, ta=(0.5, 0.5))
    layer.set_backend(tk.Backend[backend])
    xa = np.abs(rng.standard_normal(108)).astype(np.float32)
    xb = np.abs(rng.standard_normal(108)).astype(np.float32)
    ra = tk.conv2d_ternary(xa, TS(1, 3, 6, 6), layer).data.cpu().numpy()
    rb = tk.conv2d_ternary(xb, TS(1, 3, 6, 6), layer).data.cpu().numpy()
    rc = tk.conv2d_ternary(np.concatenate([xa, xb]), TS(2, 3, 6, 6), layer).data.cpu().numpy()
    assert np.array_equal(rc, np.concatenate([ra, rb]))
    l3 = _layer(tk, wq, 3, 5, 3, 1, 1, ta=(0.5, 0.5), out_scale=3.0)
    l3.set_backend(tk.Backend[backend])
    r3 = tk.conv2d_ternary(xa, TS(1, 3, 6, 6), l3).data.cpu().numpy()
    np.testing.assert_allclose(r3, 3.0 * ra, rtol=1e-6)
    for kh in (1, 3, 5):
        for stride in (1, 2, 3):
            for pad in (0, 1, 2):
                if 11 + 2 * pad < kh or 9 + 2 * pad < kh:
                    continue
                w1 = rng.integers(-1, 2, (1, 2 * kh * kh)).astype(np.int8)
                L = _layer(tk, w1, 2, 1, kh, stride, pad, ta=(0.5, 0.5))
                L.set_backend(tk.Backend[backend])
                x = np.abs(rng.standard_normal(2 * 11 * 9)).astype(np.float32)
                r = tk.conv2d_ternary(x, TS(1, 2, 11, 9), L)
                assert (r.shape.h, r.shape.w) == ((11 + 2 * pad - kh) // stride + 1, (9 + 2 * pad - kh) // stride + 1)
                st, want = oracle.conv2d_ternary(x, 1, 2, 11, 9, w1, 1, kh, stride, pad, (0.5, 0.5), True)
                assert np.array_equal(r.data.cpu().numpy(), want)
    aff = tk.ChannelAffine(np.array([1, 2, 3], np.float32), np.array([0.5, -0.5, 4.0], np.float32))
    fc = tk.make_packed_conv_layer(rng.integers(-1, 2, 24).astype(np.int8), tk.ConvGeometry(8, 3, 1, 1, 1, 0),
                                   tk.QuantThresholds(), tk.QuantThresholds(0.5, 0.5), True, aff)
    fc.set_backend(tk.Backend[backend])
    y = tk.fully_connected_ternary(np.zeros(8, np.float32), 1, fc).cpu().numpy()
    assert list(y[0]) == [0.5, -0.5, 4.0]


@pytest.mark.parametrize("backend", ["POPC", "TC_I8", "TC_F4"])
def test_fc_golden_and_geometry(tk, golden, backend):
    for name in ("fc_small", "fc_mid"):
        bt, cin, cout = map(int, golden[f"{name}_dims"])
        layer = _layer(tk, golden[f"{name}_w"], cin, cout, 1, 1, 0, gain=golden[f"{name}_gain"],
                       bias=golden[f"{name}_bias"])
        layer.set_backend(tk.Backend[backend])
        y = tk.fully_connected_ternary(golden[f"{name}_x"], bt, layer).cpu().numpy()
        assert np.array_equal(y.view(np.int32), golden[f"{name}_y"].view(np.int32)), name
    bad = _layer(tk, np.zeros((6, 180), np.int8), 20, 6, 3, 1, 1)
    with pytest.raises(tk.InvalidArgument):
        tk.fully_connected_ternary(np.zeros(60, np.float32), 3, bad)


@pytest.mark.parametrize("backend", ["POPC", "TC_I8", "TC_F4"])
def test_fc_cfg3_full_size(tk, oracle, backend):
    """cfg3: FC 4096x4096, batch 256 -- exact int32 accumulators vs a numpy
    integer matmul of the decoded levels (size-independent exactness), and the
    fused float epilogue vs the oracle's formula on a row subsample."""
    rng = np.random.default_rng(33)
    B, N = 256, 4096
    x = np.abs(rng.standard_normal((B, N))).astype(np.float32)
    wq = rng.integers(-1, 2, (N, N)).astype(np.int8)
    layer = _layer(tk, wq, N, N, 1, 1, 0, gain=(rng.uniform(0.5, 1.5, N) / 64).astype(np.float32),
                   bias=rng.standard_normal(N).astype(np.float32))
    layer.set_backend(tk.Backend[backend])
    buf = tk.im2col_quantize_pack(x, tk.TensorShape(B, N, 1, 1), tk.QuantThresholds(0.5, 0.9), layer.geom,
                                  tk.QuantMode.kActivationNonneg)
    acc = tk.packed_gemm(buf, layer).cpu().numpy()
    lv = np.stack([oracle.unpack(r, N) for r in u64(buf.words)]).astype(np.int64) + 1
    want = lv @ wq.T.astype(np.int64)
    assert np.array_equal(acc, want)
    y = tk.fully_connected_ternary(x, B, layer).cpu().numpy()
    rows = slice(0, 256, 51)  # rows are independent: oracle on a subsample
    xs = np.ascontiguousarray(x[rows])
    st, ref = oracle.conv2d_ternary(xs, xs.shape[0], N, 1, 1, wq, N, 1, 1, 0, (0.5, 0.9), True,
                                    layer.fused.gain, layer.fused.bias, 1.0)
    assert st == 0
    assert np.array_equal(y[rows].view(np.int32), ref.reshape(xs.shape[0], N).view(np.int32))


@pytest.mark.parametrize("fmt", ["s8", "fp4"])
@pytest.mark.parametrize("rows,k,n", [(256, 4096, 4096), (200, 640, 96), (1, 128, 8), (300, 1280, 260),
                                      (128, 40000, 64)])
def test_level_operand_gemm(tk, oracle, rows, k, n, fmt):
    """quantize_levels -> gemm_levels (the cfg3 kernels on their own): levels
    equal the oracle quantizer, int32 accumulators equal the integer matmul,
    across split-K cluster sizes (ragged rows / columns included; K = 40000
    forces the split that keeps the s16 partials exact)."""
    rng = np.random.default_rng(rows + k + n)
    wq = rng.integers(-1, 2, (n, k)).astype(np.int8)
    layer = _layer(tk, wq, k, n, 1, 1, 0)
    x = np.abs(rng.standard_normal((rows, k))).astype(np.float32)
    a = tk.quantize_levels(torch.from_numpy(x).cuda(), tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg,
                           tk.layer_k_pad(layer, fmt), fmt)
    lv = a.dense().cpu().numpy()[:, :k].astype(np.int64)
    st, words = oracle.quantize_and_pack(x[: min(rows, 8)].reshape(-1), 0.5, 0.9, 1)
    want_lv = oracle.unpack(words, min(rows, 8) * k).reshape(min(rows, 8), k).astype(np.int64) + 1
    assert np.array_equal(lv[: min(rows, 8)], want_lv)
    want = lv @ wq.T.astype(np.int64)
    got = tk.gemm_levels(a, layer).cpu().numpy()
    assert np.array_equal(got, want)
    gain = rng.uniform(0.5, 1.5, n).astype(np.float32)
    bias = rng.standard_normal(n).astype(np.float32)
    layer2 = _layer(tk, wq, k, n, 1, 1, 0, gain=gain, bias=bias)
    y = tk.gemm_levels(a, layer2, fused=True).cpu().numpy()
    r4 = min(rows, 4)  # fmaf epilogue: the oracle's conv epilogue on the same inputs
    st, yo = oracle.conv2d_ternary(x[:r4], r4, k, 1, 1, wq, n, 1, 1, 0, (0.5, 0.9), True, gain, bias, 1.0)
    assert st == 0 and np.array_equal(y[:r4].view(np.int32), yo.reshape(r4, n).view(np.int32))


def test_fp4_symmetric_levels(tk):
    """kind::mxf4 with -1 levels on both sides (weight-mode activations into a
    symmetric layer): identical to the s8 path and the integer matmul."""
    rng = np.random.default_rng(71)
    rows, k, n = 384, 1000, 200
    wq = rng.integers(-1, 2, (n, k)).astype(np.int8)
    layer = _layer(tk, wq, k, n, 1, 1, 0, ta=(0.8, 1.2), nonneg=False)
    x = torch.from_numpy(rng.standard_normal((rows, k)).astype(np.float32)).cuda()
    a8 = tk.quantize_levels(x, tk.QuantThresholds(0.8, 1.2), tk.QuantMode.kWeight, tk.layer_k_pad(layer))
    a4 = tk.quantize_levels(x, tk.QuantThresholds(0.8, 1.2), tk.QuantMode.kWeight, tk.layer_k_pad(layer, "fp4"),
                            "fp4")
    lv = a8.dense().cpu().numpy()[:, :k]
    assert np.array_equal(a4.dense().cpu().numpy()[:, :k], lv)
    assert not a4.dense().cpu().numpy()[:, k:].any()
    want = lv.astype(np.int64) @ wq.T.astype(np.int64)
    assert np.array_equal(tk.gemm_levels(a4, layer).cpu().numpy(), want)
    assert np.array_equal(tk.gemm_levels(a8, layer).cpu().numpy(), want)


def test_fp4_operand_errors_and_stream_order(tk):
    """FP4 entry points: K padding must be a multiple of 256 (the FP4 K block);
    GEMMs launched as programmatic dependents stay ordered behind the kernels
    that produce their operands and read their outputs (repeated FC calls on
    one stream, each consuming the previous output)."""
    rng = np.random.default_rng(81)
    k, n = 512, 512
    wq = rng.integers(-1, 2, (n, k)).astype(np.int8)
    layer = _layer(tk, wq, k, n, 1, 1, 0, ta=(0.5, 0.9), gain=(rng.uniform(0.5, 1.5, n) / 32).astype(np.float32),
                   bias=np.zeros(n, np.float32))
    x = torch.from_numpy(np.abs(rng.standard_normal((256, k))).astype(np.float32)).cuda()
    with pytest.raises(tk.InvalidArgument):
        tk.quantize_levels(x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg, 384, "fp4")
    assert tk.layer_k_pad(layer, "fp4") % 256 == 0
    # chain: y_{i+1} = FC(relu(y_i)) on the FP4 pipe vs the POPC pipe, no host syncs in between
    outs = {}
    for be in (tk.Backend.TC_F4, tk.Backend.POPC):
        layer.set_backend(be)
        y = x
        for _ in range(4):
            y = torch.relu(tk.fully_connected_ternary(y, 256, layer, check_errors=False))
        torch.cuda.synchronize()
        outs[be.name] = y.cpu().numpy()
    assert np.array_equal(outs["TC_F4"].view(np.int32), outs["POPC"].view(np.int32))


FUSED_CASES = [  # (c, oc, h, w, k, stride, n)
    (64, 64, 56, 56, 3, 1, 1),     # cfg2
    (64, 64, 56, 56, 3, 1, 3),
    (64, 128, 28, 28, 3, 2, 2),
    (128, 128, 14, 14, 3, 1, 2),
    (128, 256, 14, 14, 1, 2, 2),
    (256, 512, 8, 8, 3, 1, 1),
    (64, 64, 9, 10, 3, 1, 2),
    (128, 64, 12, 8, 1, 1, 3),
    (64, 256, 14, 14, 3, 1, 2),    # one 256-wide N tile over 64-channel rows
    (64, 64, 56, 56, 3, 1, 16),    # 421 tiles: several items per persistent CTA
]


@pytest.mark.parametrize("c,oc,h,w,k,s,n", FUSED_CASES)
def test_conv2d_fused_implicit_im2col(tk, oracle, c, oc, h, w, k, s, n):
    """conv2d_ternary on the fused implicit-im2col kernel (AUTO / TC_CONV):
    f32 NCHW output bit-identical to the oracle (R:linalg.hpp:301-328) and to
    the explicit-im2col GEMM pipes, incl. stride 2, 1x1, two N tiles, ragged
    planes and a batch whose last M tile is partial."""
    rng = np.random.default_rng(c + oc + h + w + k + s + n)
    wq = rng.integers(-1, 2, (oc, c * k * k)).astype(np.int8)
    gain = (rng.uniform(0.5, 1.5, oc) / 16).astype(np.float32)
    bias = rng.standard_normal(oc).astype(np.float32)
    x = np.abs(rng.standard_normal(n * c * h * w)).astype(np.float32)
    x[:: 97] = 0.0
    shape = tk.TensorShape(n, c, h, w)
    st, want = oracle.conv2d_ternary(x, n, c, h, w, wq, oc, k, s, k // 2, (0.5, 0.9), True, gain, bias, 0.37)
    assert st == 0
    for be in ("AUTO", "TC_CONV", "TC_I8"):
        layer = _layer(tk, wq, c, oc, k, s, k // 2, gain=gain, bias=bias, out_scale=0.37)
        layer.set_backend(tk.Backend[be])
        y = tk.conv2d_ternary(x, shape, layer).data.cpu().numpy()
        y2 = tk.conv2d_ternary(x, shape, layer).data.cpu().numpy()  # the cached plan again
        assert np.array_equal(y.view(np.int32), want.view(np.int32)), be
        assert np.array_equal(y2.view(np.int32), y.view(np.int32)), be


def test_conv2d_fused_errors_in_reference_order(tk, oracle):
    """Data errors on the fused path report the reference's FIRST error in its
    im2col evaluation order (R:linalg.hpp:173-225, R:quantizer.hpp:37-41,53-55),
    not the first in memory order: a negative value used by output row 0
    wins over a NaN at a smaller NCHW index first used by a later row (and
    the reverse); a bad value no patch reads (1x1 / stride 2 skips odd rows
    and columns) raises nothing."""
    from paper_2008_05101_b200 import _lib as T
    c, h, w = 64, 16, 16
    wq = np.random.default_rng(1).integers(-1, 2, (64, c * 9)).astype(np.int8)
    layer = _layer(tk, wq, c, 64, 3, 1, 1)
    layer.set_backend(tk.Backend.TC_CONV)
    for neg, nan, code in [((63, 0, 0), (0, 5, 5), T.TK_ERR_NEGATIVE), ((0, 9, 9), (63, 0, 1), T.TK_ERR_NONFINITE)]:
        x = np.abs(np.random.default_rng(2).standard_normal((1, c, h, w))).astype(np.float32)
        x[(0, *neg)] = -1.0
        x[(0, *nan)] = np.nan
        st, _ = oracle.conv2d_ternary(x.reshape(-1), 1, c, h, w, wq, 64, 3, 1, 1, (0.5, 0.9), True)
        assert st == code
        with pytest.raises(tk.InvalidArgument) as ei:
            tk.conv2d_ternary(x.reshape(-1), tk.TensorShape(1, c, h, w), layer)
        assert ei.value.status == code
    w1 = np.random.default_rng(4).integers(-1, 2, (128, c)).astype(np.int8)
    l1 = _layer(tk, w1, c, 128, 1, 2, 0)
    l1.set_backend(tk.Backend.TC_CONV)
    x3 = np.abs(np.random.default_rng(5).standard_normal((2, c, h, w))).astype(np.float32)
    x3[1, 7, 3, 5] = -1.0
    st3, want = oracle.conv2d_ternary(x3.reshape(-1), 2, c, h, w, w1, 128, 1, 2, 0, (0.5, 0.9), True)
    assert st3 == 0
    y = tk.conv2d_ternary(x3.reshape(-1), tk.TensorShape(2, c, h, w), l1).data.cpu().numpy()
    assert np.array_equal(y.view(np.int32), want.view(np.int32))
