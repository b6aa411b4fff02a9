"""GPU parity: codec, quantizer and inner-product kernels vs the golden
vectors (reference outputs) and the C oracle.  Bit-exact."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

KAUXI = 0x5555555555555555


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def test_pack_kats(tk, golden):
    p = tk.pack(np.array([-1, 0, 0, 1], np.int8))
    assert np.array_equal(u64(p.words), golden["kat_pack_m1001"])
    assert int(u64(p.words)[0]) & 0xFF == 0b11010100
    assert p.logical_len == 4
    p = tk.pack(np.array([1], np.int8))
    assert np.array_equal(u64(p.words), golden["kat_pack_1"]) and p.lane_capacity() == 32
    e = tk.pack(np.zeros(0, np.int8))
    assert e.words.numel() == 0 and tk.unpack(e).numel() == 0
    with pytest.raises(tk.InvalidArgument):
        tk.pack(np.array([0, 3], np.int8))


def test_unpack_roundtrip_and_noncanonical_zero(tk):
    rng = np.random.default_rng(3)
    for n in [37] + list(range(0, 130, 7)):
        v = rng.integers(-1, 2, n).astype(np.int8)
        assert np.array_equal(tk.unpack(tk.pack(v)).cpu().numpy(), v)
    p = tk.pack(np.array([-1, 0, 0, 1], np.int8))
    w = u64(p.words).copy()
    w[0] = (int(w[0]) & ~(3 << 2)) | (0b10 << 2)  # lane 1 -> non-canonical zero
    q = tk.PackedTernaryVector(torch.from_numpy(w.view(np.int64)).cuda(), 4)
    assert list(tk.unpack(q).cpu().numpy()) == [-1, 0, 0, 1]


def test_quantize_and_pack_golden(tk, golden):
    QM, QT = tk.QuantMode, tk.QuantThresholds
    assert np.array_equal(u64(tk.quantize_and_pack(golden["qp_x"], QT(1, 1), QM.kWeight).words),
                          golden["qp_weight_words"])
    a = tk.quantize_and_pack(np.abs(golden["qp_x"]), QT(1, 1), QM.kActivationNonneg)
    assert a.nonneg_offset and np.array_equal(u64(a.words), golden["qp_act_words"])
    for n in (1, 15, 16, 17, 31, 32, 33, 63, 100, 4096):
        got = tk.quantize_and_pack(golden[f"qp_len{n}_x"], QT(0.5, 0.9), QM.kActivationNonneg)
        assert np.array_equal(u64(got.words), golden[f"qp_len{n}_act"]), n
        got = tk.quantize_and_pack(golden[f"qp_len{n}_xw"], QT(0.8, 1.2), QM.kWeight)
        assert np.array_equal(u64(got.words), golden[f"qp_len{n}_w"]), n
    assert np.array_equal(u64(tk.quantize_and_pack(np.zeros(64, np.float32), QT(0.7, 1.3), QM.kWeight).words),
                          golden["kat_zeros_weight"])
    p = tk.quantize_and_pack(np.array([0.6, -0.7, 0.1], np.float32), QT(1, 1), QM.kWeight)
    assert list(tk.unpack(p).cpu().numpy()) == [1, -1, 0]


def test_quantizer_grid_levels(tk, golden):
    """Every golden grid point (incl. bankers ties and their neighbours) through
    the device quantizer, one element per call-row with its own step sizes."""
    QM, QT = tk.QuantMode, tk.QuantThresholds
    sel = np.r_[0:400, len(golden["qz_a1"]) - 70:len(golden["qz_a1"])]
    for i in sel:
        a1, a2 = float(golden["qz_a1"][i]), float(golden["qz_a2"][i])
        for key, lkey, mode in (("qz_pw", "qz_lw", QM.kWeight), ("qz_pa", "qz_la", QM.kActivationNonneg)):
            p = tk.quantize_and_pack(np.array([golden[key][i]], np.float32), QT(a1, a2), mode)
            lv = int(tk.unpack(p).cpu().numpy()[0]) + (1 if mode == QM.kActivationNonneg else 0)
            assert lv == int(golden[lkey][i]), (i, key)


def test_quantizer_errors_first_in_order(tk, golden):
    QM, QT = tk.QuantMode, tk.QuantThresholds
    cases = [(np.array([0.1, np.nan], np.float32), QM.kWeight, golden["err_nan_weight"][0]),
             (np.array([0.1, -0.2, np.nan], np.float32), QM.kActivationNonneg, golden["err_neg_then_nan"][0]),
             (np.array([0.1, np.inf, -0.2], np.float32), QM.kActivationNonneg, golden["err_inf_then_neg"][0])]
    for x, mode, want in cases:
        with pytest.raises(tk.InvalidArgument) as ei:
            tk.quantize_and_pack(x, QT(1, 1), mode)
        assert ei.value.status == want
    # a bad element late in a long vector, preceded by another kind of error
    x = np.abs(np.random.default_rng(0).standard_normal(100000)).astype(np.float32)
    x[77777] = -1.0
    x[91234] = np.nan
    with pytest.raises(tk.InvalidArgument) as ei:
        tk.quantize_and_pack(x, QT(0.5, 0.9), QM.kActivationNonneg)
    assert ei.value.status == 5
    with pytest.raises(tk.InvalidArgument):
        tk.quantize_and_pack(x, QT(0.0, 0.9), QM.kActivationNonneg)
    tk.sync()  # error word was cleared


def test_large_quantize_pack_vs_oracle(tk, oracle):
    rng = np.random.default_rng(5)
    for n in (4096 * 256, 1_000_003):
        x = np.abs(rng.standard_normal(n)).astype(np.float32) * 1.2
        got = u64(tk.quantize_and_pack(x, tk.QuantThresholds(0.5, 0.9), tk.QuantMode.kActivationNonneg).words)
        st, want = oracle.quantize_and_pack(x, 0.5, 0.9, 1)
        assert st == 0 and np.array_equal(got, want)


def test_dot_fuzz_golden(tk, golden):
    offs = golden["dot_offs"]
    for i in range(len(golden["dot_lens"])):
        L = int(golden["dot_lens"][i])
        x = golden["dot_x"][offs[i]:offs[i + 1]].view(np.int64)
        y = golden["dot_y"][offs[i]:offs[i + 1]].view(np.int64)
        a = golden["dot_a"][offs[i]:offs[i + 1]].view(np.int64)
        xv = tk.PackedTernaryVector(torch.from_numpy(x.copy()).cuda(), L)
        yv = tk.PackedTernaryVector(torch.from_numpy(y.copy()).cuda(), L)
        av = tk.PackedTernaryVector(torch.from_numpy(a.copy()).cuda(), L, True)
        assert tk.ternary_dot(xv, yv) == golden["dot_xy"][i]
        wsum = int(tk.unpack(yv).cpu().numpy().astype(np.int64).sum())
        assert tk.ternary_dot_nonneg(av, yv, wsum) == golden["dot_ay_nonneg"][i]
    v = tk.pack(np.array([1, 0, -1, 1], np.int8))
    w = tk.pack(np.array([-1, 0, 1, 1], np.int8))
    assert tk.ternary_dot(v, w) == -1                       # R:tests/test_bitkernels.cpp:77-80
    with pytest.raises(tk.InvalidArgument):
        tk.ternary_dot(tk.pack(np.array([1, 0], np.int8)), tk.pack(np.array([1, 0, -1], np.int8)))
    with pytest.raises(tk.InvalidArgument):
        tk.ternary_dot_nonneg(v, w, 0)                      # lacks nonneg flag
    with pytest.raises(tk.InvalidArgument):
        tk.ternary_dot_premask(v, w, [])


def test_batched_dot_cfg1_vs_oracle(tk, oracle):
    """cfg1 shape: N=4096 (128 u64/vector), nonneg activations x ternary weights."""
    rng = np.random.default_rng(9)
    pairs, n = 4096, 4096
    a = np.abs(rng.standard_normal((pairs, n))).astype(np.float32)
    w = rng.standard_normal((pairs, n)).astype(np.float32)
    QT, QM = tk.QuantThresholds, tk.QuantMode
    aw = tk.quantize_and_pack_rows(a, QT(0.5, 0.9), QM.kActivationNonneg)
    ww = tk.quantize_and_pack_rows(w, QT(0.8, 1.2), QM.kWeight)
    wl = np.stack([oracle.unpack(r, n) for r in u64(ww)[:64]])
    ws = torch.from_numpy(np.concatenate([wl.astype(np.int64).sum(1), np.zeros(pairs - 64, np.int64)])).cuda()
    got = tk.ternary_dot_batched(aw, ww, ws).cpu().numpy()
    want = oracle.ternary_dot_batched(u64(aw), u64(ww), ws.cpu().numpy())
    assert np.array_equal(got, want)
    al = np.stack([oracle.unpack(r, n) for r in u64(aw)[:64]]).astype(np.int64) + 1
    assert np.array_equal(got[:64], (al * wl).sum(1))


@pytest.mark.parametrize("words", [1, 2, 3, 7, 64, 128, 129, 256, 300, 1000])
def test_batched_dot_ragged_words_and_premask(tk, oracle, words):
    """Word counts around the kernel's 4 x 16 B per-lane chunks (odd counts
    take the u64 kernel), the cfg1 row (128) and rows longer than one chunk;
    the premask form (R:bitkernels.hpp:66-72, :87-97) with make_zero_seeds
    equals ternary_dot and with arbitrary seeds equals the host TM formula."""
    rng = np.random.default_rng(words)
    pairs = 257
    x = rng.integers(0, 2**63, (pairs, words), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, (pairs, words),
                                                                                               dtype=np.uint64)
    y = rng.integers(0, 2**63, (pairs, words), dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, (pairs, words),
                                                                                               dtype=np.uint64)
    ws = rng.integers(-5000, 5000, pairs).astype(np.int64)
    got = tk.ternary_dot_batched(x, y, ws).cpu().numpy()
    assert np.array_equal(got, oracle.ternary_dot_batched(x, y, ws))
    seeds = (y ^ (y >> np.uint64(1))) & np.uint64(tk.kAuxi)
    assert np.array_equal(tk.ternary_dot_batched(x, y, ws, seeds=seeds).cpu().numpy(), got)
    rs = rng.integers(0, 2**63, (pairs, words), dtype=np.uint64) & np.uint64(tk.kAuxi)  # arbitrary seeds
    tm = (~(x ^ y) | rs) & ~(rs << np.uint64(1))
    want = np.bitwise_count(tm).sum(axis=1, dtype=np.int64) - 32 * words + ws
    assert np.array_equal(tk.ternary_dot_batched(x, y, ws, seeds=rs).cpu().numpy(), want)
    # detail:: raw-word entries on one pair
    assert tk.ternary_dot_words(x[0], y[0]) == int(got[0] - ws[0])
    assert tk.ternary_dot_words_premask(x[0], y[0], rs[0]) == int(want[0] - ws[0])
