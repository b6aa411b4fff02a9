"""GPU exactness at worst-case accumulator magnitudes, and the A10 layer build.

The tensor-core pipes compute the reference's integer dot products
(R:include/ternkit/bitkernels.hpp:76-97, :151-159) as MMAs: kind::i8
accumulates in s32, kind::mxf4 in f32.  Random data keeps |acc| near sqrt(K),
which says nothing about accumulator width, so these cases drive the
accumulator to |acc| = 2K (K up to 40000) and add small odd contributions on
top of large partial sums (and large partial sums that cancel), where an
accumulator that kept fewer than 24 significant bits -- or truncated the
addend on alignment -- would drop low bits.  Expected values: exact integer
matmul (float64, all sums < 2^53).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TA = (0.5, 0.9)  # nonneg activation thresholds: 0.0 -> level 0, 0.3 -> 1, 10.0 -> 2
LEVEL_X = np.array([0.0, 0.3, 10.0], np.float32)


def worst_case(k: int, rows: int = 256, cols: int = 384, seed: int = 0):
    """Levels [rows][k] in {0,1,2} and weights [cols][k] in {-1,0,1} built to
    reach |acc| = 2k, to add odd terms onto large partials, and to cancel."""
    rng = np.random.default_rng(seed + k)
    L = np.empty((rows, k), np.int8)
    for r in range(rows):
        p = r % 4
        if p == 0:
            L[r] = 2
        elif p == 1:
            L[r, : k // 2] = 2
            L[r, k // 2:] = rng.integers(0, 3, k - k // 2)
        elif p == 2:
            L[r] = rng.integers(0, 3, k)
        else:
            L[r] = 2
            L[r, ::7] = 1
    W = np.empty((cols, k), np.int8)
    blk = np.arange(k) // 2048
    for c in range(cols):
        p = c % 6
        if p == 0:
            W[c] = 1
        elif p == 1:
            W[c] = -1
        elif p == 2:  # +2048-lane blocks alternating sign, odd holes
            W[c] = np.where(blk % 2 == 0, 1, -1)
            W[c, ::97] = 0
        elif p == 3:
            W[c] = rng.integers(-1, 2, k)
        elif p == 4:  # rise to 1.5k, then cancel down to ~0.5k
            W[c] = 1
            W[c, 3 * k // 4:] = -1
        else:
            W[c, : k // 2] = 1
            W[c, k // 2:] = rng.integers(-1, 2, k - k // 2)
    want = L.astype(np.float64) @ W.T.astype(np.float64)
    return L, W, want.astype(np.int64)


def _layer(tk, W, k, gain=None):
    cols = W.shape[0]
    aff = None if gain is None else tk.ChannelAffine(gain, np.zeros(cols, np.float32))
    return tk.make_packed_conv_layer(W, tk.ConvGeometry(k, cols, 1, 1, 1, 0), tk.QuantThresholds(),
                                     tk.QuantThresholds(*TA), True, aff)


@pytest.mark.parametrize("k", [4096, 16384, 40000])
@pytest.mark.parametrize("backend", ["POPC", "TC_I8", "TC_F4", "AUTO"])
def test_worst_case_accumulators(tk, k, backend):
    L, W, want = worst_case(k)
    assert np.abs(want).max() == 2 * k
    x = LEVEL_X[L]
    layer = _layer(tk, W, k)
    layer.set_backend(tk.Backend[backend])
    buf = tk.im2col_quantize_pack(x, tk.TensorShape(x.shape[0], k, 1, 1), tk.QuantThresholds(*TA), layer.geom,
                                  tk.QuantMode.kActivationNonneg)
    got = tk.packed_gemm(buf, layer).cpu().numpy().astype(np.int64)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} wrong, first {bad[:3].tolist()}: got {got[tuple(bad[0])]} " \
                          f"want {want[tuple(bad[0])]}"
    # FC entry (quantize -> GEMM -> epilogue) with gain 1, bias 0: the f32
    # output is the accumulator itself (|acc| < 2^24)
    lf = _layer(tk, W, k, gain=np.ones(W.shape[0], np.float32))
    lf.set_backend(tk.Backend[backend])
    y = tk.fully_connected_ternary(x, x.shape[0], lf).cpu().numpy()
    assert np.array_equal(y, want.astype(np.float32))


@pytest.mark.parametrize("fmt", ["s8", "fp4"])
@pytest.mark.parametrize("k", [4096, 16384, 40000])
def test_worst_case_level_gemm(tk, k, fmt):
    """The level-operand GEMM kernels on their own (every split-K choice the
    launcher makes for this shape, incl. the s16 DSMEM partials)."""
    L, W, want = worst_case(k, rows=512, cols=256, seed=1)
    layer = _layer(tk, W, k)
    a = tk.quantize_levels(torch.from_numpy(LEVEL_X[L]).cuda(), tk.QuantThresholds(*TA),
                           tk.QuantMode.kActivationNonneg, tk.layer_k_pad(layer, fmt), fmt)
    assert np.array_equal(a.dense().cpu().numpy()[:, :k], L)
    got = tk.gemm_levels(a, layer).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("rows", [1, 128, 200])
def test_worst_case_small_m(tk, rows):
    """Few rows (split-K across a cluster is the launcher's choice here)."""
    k = 40000
    L, W, want = worst_case(k, rows=rows, cols=128, seed=2)
    for fmt in ("s8", "fp4"):
        layer = _layer(tk, W, k)
        a = tk.quantize_levels(torch.from_numpy(LEVEL_X[L]).cuda(), tk.QuantThresholds(*TA),
                               tk.QuantMode.kActivationNonneg, tk.layer_k_pad(layer, fmt), fmt)
        assert np.array_equal(tk.gemm_levels(a, layer).cpu().numpy().astype(np.int64), want), fmt


@pytest.mark.parametrize("c,oc,k", [(3, 70, 3), (64, 64, 3), (4096, 16, 1), (33, 5, 5), (1, 1, 1), (7, 9, 1)])
def test_layer_build_matches_reference(tk, c, oc, k):
    """A10: the uploaded layer's packed rows and weight sums equal the
    reference's make_packed_conv_layer (R:include/ternkit/linalg.hpp:118-144)
    byte for byte, including the kAuxi padding of ragged last words."""
    from oracle.oracle import Reference
    R = Reference()
    rng = np.random.default_rng(c * 1000 + oc + k)
    wq = rng.integers(-1, 2, (oc, c * k * k)).astype(np.int8)
    layer = tk.make_packed_conv_layer(wq, tk.ConvGeometry(c, oc, k, k, 1, k // 2), tk.QuantThresholds(),
                                      tk.QuantThresholds(0.5, 0.9), True)
    st, words, sums = R.make_packed_conv_layer(wq, c, oc, k, k)
    assert st == 0
    assert np.array_equal(layer.weights_words, words)
    assert np.array_equal(layer.weight_sums, sums)


@pytest.mark.parametrize("fmt", ["s8", "fp4"])
@pytest.mark.parametrize("rows,k", [(256, 4096), (256, 40000), (200, 16384), (128, 4096), (100, 40000), (64, 8192),
                                    (37, 4096), (1, 40000)])
def test_worst_case_fc_shapes(tk, rows, k, fmt):
    """FC-shaped GEMMs (<= 256 rows, 2048-4096 output channels: the cfg3
    family) across the launcher's tile / split-K choices at worst-case
    magnitudes, with the int32 and the fused f32 epilogue (gain 1, bias 0:
    y == acc)."""
    cols = 2048 if k > 4096 else 4096
    L, W, want = worst_case(k, rows=rows, cols=cols, seed=3)
    layer = _layer(tk, W, k, gain=np.ones(cols, np.float32))
    a = tk.quantize_levels(torch.from_numpy(LEVEL_X[L]).cuda(), tk.QuantThresholds(*TA),
                           tk.QuantMode.kActivationNonneg, tk.layer_k_pad(layer, fmt), fmt)
    got = tk.gemm_levels(a, layer).cpu().numpy().astype(np.int64)
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{len(bad)} wrong, first {bad[:3].tolist()}"
    y = tk.gemm_levels(a, layer, fused=True).cpu().numpy()
    assert np.array_equal(y, want.astype(np.float32))
