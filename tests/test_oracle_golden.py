"""Pin the C restatement (oracle/ternkit_oracle.c) against the golden vectors
that the unmodified reference produced (oracle/make_golden.py), and -- where
the compiled reference (oracle/_ref) can run on this host -- against the
reference directly on fresh random inputs.  CPU only."""
import numpy as np
import pytest

from oracle.oracle import MODE_ACT_NONNEG, MODE_WEIGHT, Reference, reference_lib_path

KAUXI = 0x5555555555555555


def test_codec_kats(oracle, golden):
    st, w = oracle.pack(np.array([-1, 0, 0, 1], np.int8))
    assert st == 0 and np.array_equal(w, golden["kat_pack_m1001"])
    assert int(w[0]) & 0xFF == 0b11010100            # R:tests/test_codec.cpp:31-37
    st, w = oracle.pack(np.array([1], np.int8))
    assert np.array_equal(w, golden["kat_pack_1"]) and (int(w[0]) >> 2) == (KAUXI >> 2)
    st, w = oracle.quantize_and_pack(np.zeros(64, np.float32), 0.7, 1.3, MODE_WEIGHT)
    assert np.array_equal(w, golden["kat_zeros_weight"]) and all(int(v) == KAUXI for v in w)
    st, w = oracle.quantize_and_pack(np.array([0.6, -0.7, 0.1], np.float32), 1.0, 1.0, MODE_WEIGHT)
    assert np.array_equal(w, golden["kat_qp_example"])
    assert list(oracle.unpack(w, 3)) == [1, -1, 0]
    assert oracle.pack(np.array([0, 3], np.int8))[0] != 0  # out of range rejected


def test_quantize_and_pack_golden(oracle, golden):
    _, w = oracle.quantize_and_pack(golden["qp_x"], 1.0, 1.0, MODE_WEIGHT)
    assert np.array_equal(w, golden["qp_weight_words"])
    _, w = oracle.quantize_and_pack(np.abs(golden["qp_x"]), 1.0, 1.0, MODE_ACT_NONNEG)
    assert np.array_equal(w, golden["qp_act_words"])
    for n in (1, 15, 16, 17, 31, 32, 33, 63, 100, 4096):
        _, w = oracle.quantize_and_pack(golden[f"qp_len{n}_x"], 0.5, 0.9, MODE_ACT_NONNEG)
        assert np.array_equal(w, golden[f"qp_len{n}_act"]), n
        _, w = oracle.quantize_and_pack(golden[f"qp_len{n}_xw"], 0.8, 1.2, MODE_WEIGHT)
        assert np.array_equal(w, golden[f"qp_len{n}_w"]), n


def test_error_kats(oracle, golden):
    assert oracle.quantize_and_pack(np.array([0.1, np.nan], np.float32), 1, 1, 0)[0] == \
        golden["err_nan_weight"][0] == 4
    assert oracle.quantize_and_pack(np.array([0.1, -0.2, np.nan], np.float32), 1, 1, 1)[0] == \
        golden["err_neg_then_nan"][0] == 5
    assert oracle.quantize_and_pack(np.array([0.1, np.inf, -0.2], np.float32), 1, 1, 1)[0] == \
        golden["err_inf_then_neg"][0] == 4


def test_tm_truth_table(oracle, golden):
    for x, y, z in zip(golden["tm_x"], golden["tm_y"], golden["tm_z"]):
        assert oracle.ternary_multiply_word(int(x), int(y)) == int(z)


def test_quantizer_grid(oracle, golden):
    for a1, a2, p, lv in zip(golden["qz_a1"], golden["qz_a2"], golden["qz_pw"], golden["qz_lw"]):
        assert oracle.quantize_weight_value(float(p), float(a1), float(a2)) == (0, int(lv))
    for a1, a2, p, lv in zip(golden["qz_a1"], golden["qz_a2"], golden["qz_pa"], golden["qz_la"]):
        assert oracle.quantize_activation_value(float(p), float(a1), float(a2)) == (0, int(lv))


def test_dot_fuzz(oracle, golden):
    offs = golden["dot_offs"]
    for i in range(len(golden["dot_lens"])):
        x = golden["dot_x"][offs[i]:offs[i + 1]].reshape(1, -1)
        y = golden["dot_y"][offs[i]:offs[i + 1]].reshape(1, -1)
        a = golden["dot_a"][offs[i]:offs[i + 1]].reshape(1, -1)
        assert oracle.ternary_dot_batched(x, y)[0] == golden["dot_xy"][i]
        ws = golden["dot_ay_nonneg"][i] - oracle.ternary_dot_batched(a, y)[0]
        # wsum = sum of decoded weights
        assert ws == int(oracle.unpack(y[0], int(golden["dot_lens"][i])).astype(np.int64).sum())


def test_im2col_kats(oracle, golden):
    st, rows = oracle.im2col_quantize_pack(golden["im2col_1x1_x"], 1, 3, 2, 2, 1, 1, 1, 0, 1.0, 1.0, 0)
    assert st == 0 and np.array_equal(rows, golden["im2col_1x1_rows"])
    st, rows = oracle.im2col_quantize_pack(np.ones(9, np.float32), 1, 1, 3, 3, 3, 3, 1, 1, 1.0, 1.0, 0)
    assert np.array_equal(rows, golden["im2col_corner_rows"])
    lanes = oracle.unpack(rows[0], 9)
    assert (lanes == 0).sum() == 5 and (lanes == 1).sum() == 4   # R:tests/test_linalg.cpp:113-128
    st, rows = oracle.im2col_quantize_pack(golden["im2col_strided_x"], 2, 3, 5, 4, 3, 3, 2, 1, 0.6, 1.1, 1)
    assert np.array_equal(rows, golden["im2col_strided_rows"])


def test_conv_shapes(oracle, golden):
    for i, (c, r, k, s, p, b) in enumerate(golden["conv_shapes"]):
        c, r, k, s, p, b = map(int, (c, r, k, s, p, b))
        st, rows = oracle.im2col_quantize_pack(golden[f"conv{i}_x"], b, c, r, r, k, k, s, p, 0.5, 0.9, 1)
        assert np.array_equal(rows, golden[f"conv{i}_rows"]), i
        wrows, ws = oracle.pack_rows(golden[f"conv{i}_w"])
        acc = oracle.packed_gemm(rows, wrows, ws, 1)
        assert np.array_equal(acc, golden[f"conv{i}_acc"]), i
        st, y = oracle.conv2d_ternary(golden[f"conv{i}_x"], b, c, r, r, golden[f"conv{i}_w"], c, k, s, p,
                                      (0.5, 0.9), True, golden[f"conv{i}_gain"], golden[f"conv{i}_bias"],
                                      0.37)
        assert st == 0
        assert np.array_equal(y.view(np.int32), golden[f"conv{i}_y"].view(np.int32)), i
        st, rows_s = oracle.im2col_quantize_pack(golden[f"conv{i}_xs"], b, c, r, r, k, k, s, p, 0.8, 1.2, 0)
        assert np.array_equal(oracle.packed_gemm(rows_s, wrows, ws, 0), golden[f"conv{i}_acc_sym"]), i


def test_fc_and_fuse_bn(oracle, golden):
    for name in ("fc_small", "fc_mid"):
        bt, cin, cout = map(int, golden[f"{name}_dims"])
        st, y = oracle.conv2d_ternary(golden[f"{name}_x"], bt, cin, 1, 1, golden[f"{name}_w"], cout, 1, 1, 0,
                                      (0.5, 0.9), True, golden[f"{name}_gain"], golden[f"{name}_bias"], 1.0)
        assert np.array_equal(y.reshape(bt, cout).view(np.int32), golden[f"{name}_y"].view(np.int32))
    st, g, b = oracle.fuse_bn(golden["bn_mean"], golden["bn_var"], golden["bn_gamma"], golden["bn_beta"], 1e-5)
    assert np.array_equal(g, golden["bn_gain"]) and np.array_equal(b, golden["bn_bias"])


def test_packed_forward_composition(oracle, golden):
    """R:tinynet.hpp:713-735 restated with oracle pieces, bit-exact."""
    batch, in_dim, hidden, ncls, nb = map(int, golden["pf_dims"])
    for cal in (True, False):
        h = oracle.matmul_t(golden["pf_x"], golden["pf_stem_w"], golden["pf_stem_b"], batch, in_dim, hidden)
        h = np.where(h < 0, np.float32(0), h).astype(np.float32)
        for i in range(nb):
            st, z = oracle.conv2d_ternary(h, batch, hidden, 1, 1, golden[f"pf_b{i}_w"], hidden, 1, 1, 0,
                                          (0.45, 0.8), True, golden[f"pf_b{i}_gain"], golden[f"pf_b{i}_bias"],
                                          1.0)
            assert st == 0
            cg = golden["pf_cal_gain"][i * hidden:(i + 1) * hidden] if cal else None
            cb = golden["pf_cal_bias"][i * hidden:(i + 1) * hidden] if cal else None
            h = oracle.residual_relu_rows(z.reshape(batch, hidden), h, hidden, cg, cb)
        logits = oracle.matmul_t(h, golden["pf_head_w"], golden["pf_head_b"], batch, hidden, ncls)
        want = golden["pf_logits"] if cal else golden["pf_logits_nocal"]
        assert np.array_equal(logits.view(np.int32), want.view(np.int32))


@pytest.mark.skipif(reference_lib_path() is None, reason="oracle/_ref not built for this host")
def test_oracle_matches_reference_random():
    """Fresh random cases, oracle vs the compiled reference (no fixtures)."""
    from oracle.oracle import Oracle
    O, R = Oracle(), Reference()
    rng = np.random.default_rng(7)
    for trial in range(6):
        c, hh, oc, k, s = [(8, 9, 5, 3, 1), (16, 8, 16, 3, 2), (3, 11, 4, 5, 2), (32, 6, 8, 1, 1),
                           (64, 7, 64, 3, 1), (6, 5, 3, 3, 1)][trial]
        p = k // 2
        n = 2
        x = np.abs(rng.standard_normal(n * c * hh * hh)).astype(np.float32) * 1.1
        wq = rng.integers(-1, 2, (oc, c * k * k)).astype(np.int8)
        gain = (rng.standard_normal(oc) * 0.03).astype(np.float32)
        bias = rng.standard_normal(oc).astype(np.float32)
        spec = dict(in_c=c, out_c=oc, k=k, stride=s, pad=p, weights=wq, ta=(0.41, 0.77), gain=gain,
                    bias=bias, out_scale=1.3)
        st, yr = R.conv2d_ternary(x, n, c, hh, hh, spec)
        st2, yo = O.conv2d_ternary(x, n, c, hh, hh, wq, oc, k, s, p, (0.41, 0.77), True, gain, bias, 1.3)
        assert st == st2 == 0
        assert np.array_equal(yr.view(np.int32), yo.view(np.int32))


@pytest.mark.skipif(reference_lib_path() is None, reason="oracle/_ref not built for this host")
def test_net_body_matches_reference():
    """ResNet-shaped body (basic + downsample + bottleneck blocks) -- oracle
    composition vs the reference's conv2d_ternary composition."""
    from oracle.oracle import Oracle
    from tests.netspec import tiny_body
    O, R = Oracle(), Reference()
    blocks, (n, c, h, w), x = tiny_body(seed=3)
    st, yo = O.net_body(blocks, x, n, c, h, w)
    assert st == 0
    hnd = R.net_create(blocks)
    st, yr, _ = R.net_run(hnd, x, n, c, h, w, 2, out_shape=yo.shape)
    R.net_destroy(hnd)
    assert st == 0
    assert np.array_equal(yo.view(np.int32), yr.view(np.int32))
    assert (yo > 0).mean() > 0.2  # non-degenerate
