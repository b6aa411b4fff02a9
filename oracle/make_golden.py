"""Generate tests/golden/golden.npz from the REFERENCE itself.

TEST INFRASTRUCTURE ONLY.  Runs in the build container (where /root/reference
exists): inputs come from numpy generators with fixed seeds plus the
reference's own hand-written known-answer cases, and every expected output is
produced by the unmodified reference headers compiled into oracle/_ref
(oracle/ref_shim.cpp, oracle/Makefile).  The fixture is committed so the GPU
box (which has no /root/reference) can check kernels against it.

    make -C oracle && python oracle/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path[:] = [p for p in sys.path if os.path.abspath(p or ".") != HERE]
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import Reference, words_for_lanes  # noqa: E402

OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "golden.npz")

KAUXI = np.uint64(0x5555555555555555)

# conv shapes: R:tests/acceptance.cpp:174-179 (c, r, k, stride, pad, batch)
CONV_SHAPES = [(3, 5, 1, 1, 0, 2), (4, 8, 3, 1, 1, 1), (2, 9, 3, 2, 1, 1),
               (5, 7, 5, 2, 2, 1), (16, 7, 3, 1, 1, 1), (16, 14, 3, 1, 1, 1),
               (16, 28, 3, 1, 1, 1), (32, 14, 3, 1, 1, 1), (64, 14, 3, 1, 1, 1)]


def main() -> None:
    R = Reference()
    g: dict[str, np.ndarray] = {}
    rng = np.random.default_rng(2008_05101)

    # ---- codec KATs (R:tests/test_codec.cpp) -------------------------------
    st, w = R.pack(np.array([-1, 0, 0, 1], np.int8)); assert st == 0
    g["kat_pack_m1001"] = w                      # low byte 0b11010100
    st, w = R.pack(np.array([1], np.int8)); assert st == 0
    g["kat_pack_1"] = w                          # padding = kAuxi
    st, w = R.quantize_and_pack(np.zeros(64, np.float32), 0.7, 1.3, 0); assert st == 0
    g["kat_zeros_weight"] = w                    # all kAuxi
    st, w = R.quantize_and_pack(np.array([0.6, -0.7, 0.1], np.float32), 1.0, 1.0, 0); assert st == 0
    g["kat_qp_example"] = w                      # -> [1, -1, 0]
    x = rng.standard_normal(1024).astype(np.float32)
    st, w = R.quantize_and_pack(x, 1.0, 1.0, 0); assert st == 0
    g["qp_x"], g["qp_weight_words"] = x, w
    st, w = R.quantize_and_pack(np.abs(x), 1.0, 1.0, 1); assert st == 0
    g["qp_act_words"] = w
    for n in (1, 15, 16, 17, 31, 32, 33, 63, 100, 4096):
        xa = np.abs(rng.standard_normal(n)).astype(np.float32) * 1.3
        st, w = R.quantize_and_pack(xa, 0.5, 0.9, 1); assert st == 0
        g[f"qp_len{n}_x"], g[f"qp_len{n}_act"] = xa, w
        xw = rng.standard_normal(n).astype(np.float32)
        st, w = R.quantize_and_pack(xw, 0.8, 1.2, 0); assert st == 0
        g[f"qp_len{n}_xw"], g[f"qp_len{n}_w"] = xw, w
    # error KATs: first error kind in element order
    g["err_nan_weight"] = np.array([R.quantize_and_pack(
        np.array([0.1, np.nan], np.float32), 1.0, 1.0, 0)[0]], np.int32)
    g["err_neg_then_nan"] = np.array([R.quantize_and_pack(
        np.array([0.1, -0.2, np.nan], np.float32), 1.0, 1.0, 1)[0]], np.int32)
    g["err_inf_then_neg"] = np.array([R.quantize_and_pack(
        np.array([0.1, np.inf, -0.2], np.float32), 1.0, 1.0, 1)[0]], np.int32)

    # ---- TM truth table x 32 lane positions (R:tests/acceptance.cpp:38-61) --
    xs, ys, tms = [], [], []
    for xc in range(4):
        for yc in range(4):
            for lane in range(32):
                xw = (int(KAUXI) & ~(3 << (2 * lane))) | (xc << (2 * lane))
                yw = (int(KAUXI) & ~(3 << (2 * lane))) | (yc << (2 * lane))
                xs.append(xw); ys.append(yw); tms.append(R.ternary_multiply_word(xw, yw))
    rx = rng.integers(0, 2**63, 2000, dtype=np.int64).astype(np.uint64) * np.uint64(2) + \
        rng.integers(0, 2, 2000).astype(np.uint64)
    ry = rng.integers(0, 2**63, 2000, dtype=np.int64).astype(np.uint64) * np.uint64(2) + \
        rng.integers(0, 2, 2000).astype(np.uint64)
    for a, b in zip(rx, ry):
        xs.append(int(a)); ys.append(int(b)); tms.append(R.ternary_multiply_word(int(a), int(b)))
    g["tm_x"] = np.array(xs, np.uint64)
    g["tm_y"] = np.array(ys, np.uint64)
    g["tm_z"] = np.array(tms, np.uint64)

    # ---- quantizer grid + ties (R:tests/test_quantizer.cpp, acceptance.cpp:220-273)
    n = 20000
    a1 = rng.uniform(0.2, 2.5, n).astype(np.float32)
    a2 = rng.uniform(0.2, 2.5, n).astype(np.float32)
    pw = rng.uniform(-3.0, 3.0, n).astype(np.float32)
    pa = rng.uniform(0.0, 5.0, n).astype(np.float32)
    # exact ties and their float neighbours
    ties = [(1.0, 1.0, 0.5), (1.0, 1.0, -0.5), (0.5, 2.0, 1.0), (1.0, 1.0, 1.5), (0.5, 1.0, 0.25),
            (1.0, 1.0, 0.6), (1.0, 1.0, -0.3), (1.0, 1.0, -0.7), (1.0, 1.0, 0.0),
            (0.5, 1.0, 0.4), (0.5, 1.0, 1.6), (0.5, 1.0, 0.1), (0.5, 0.9, 0.95000005),
            (0.5, 0.9, 0.94999999)]
    ta1 = [t[0] for t in ties]; ta2 = [t[1] for t in ties]; tp = [t[2] for t in ties]
    for (t1, t2, p) in ties:
        for d in (-2, -1, 1, 2):
            ta1.append(t1); ta2.append(t2)
            tp.append(float(np.nextafter(np.float32(p), np.float32(np.inf * d), dtype=np.float32)))
    a1 = np.concatenate([a1, np.array(ta1, np.float32)])
    a2 = np.concatenate([a2, np.array(ta2, np.float32)])
    pw = np.concatenate([pw, np.array(tp, np.float32)])
    pa = np.concatenate([pa, np.abs(np.array(tp, np.float32))])
    lw = np.array([R.quantize_weight_value(float(p), float(u), float(v))[1]
                   for p, u, v in zip(pw, a1, a2)], np.int8)
    la = np.array([R.quantize_activation_value(float(p), float(u), float(v))[1]
                   for p, u, v in zip(pa, a1, a2)], np.int8)
    g["qz_a1"], g["qz_a2"], g["qz_pw"], g["qz_pa"], g["qz_lw"], g["qz_la"] = a1, a2, pw, pa, lw, la

    # ---- dot fuzz (R:tests/acceptance.cpp:71-99) ---------------------------
    lens = np.concatenate([[1, 4, 31, 32, 33, 64, 4096], rng.integers(1, 1025, 150)]).astype(np.int64)
    xw_all, yw_all, aw_all, offs, dots, nn = [], [], [], [0], [], []
    for L in lens:
        L = int(L)
        xv = rng.integers(-1, 2, L).astype(np.int8)
        yv = rng.integers(-1, 2, L).astype(np.int8)
        av = rng.integers(0, 3, L).astype(np.int8)
        _, xw = R.pack(xv); _, yw = R.pack(yv); _, aw = R.pack(av - 1)
        st, d = R.ternary_dot_batched(xw.reshape(1, -1), yw.reshape(1, -1), L); assert st == 0
        st, e = R.ternary_dot_batched(aw.reshape(1, -1), yw.reshape(1, -1), L,
                                      np.array([int(yv.astype(np.int64).sum())])); assert st == 0
        assert d[0] == int((xv.astype(np.int64) * yv).sum())
        assert e[0] == int((av.astype(np.int64) * yv).sum())
        xw_all.append(xw); yw_all.append(yw); aw_all.append(aw)
        offs.append(offs[-1] + xw.size); dots.append(d[0]); nn.append(e[0])
    g["dot_lens"] = lens
    g["dot_offs"] = np.array(offs, np.int64)
    g["dot_x"] = np.concatenate(xw_all); g["dot_y"] = np.concatenate(yw_all)
    g["dot_a"] = np.concatenate(aw_all)
    g["dot_xy"] = np.array(dots, np.int64); g["dot_ay_nonneg"] = np.array(nn, np.int64)

    # ---- im2col KATs (R:tests/test_linalg.cpp:94-163) ----------------------
    x = rng.standard_normal(12).astype(np.float32)          # {1,3,2,2} 1x1 weight mode
    st, rows = R.im2col_quantize_pack(x, 1, 3, 2, 2, 1, 1, 1, 0, 1.0, 1.0, 0); assert st == 0
    g["im2col_1x1_x"], g["im2col_1x1_rows"] = x, rows
    st, rows = R.im2col_quantize_pack(np.ones(9, np.float32), 1, 1, 3, 3, 3, 3, 1, 1, 1.0, 1.0, 0)
    g["im2col_corner_rows"] = rows                          # row 0: 5 zeros, 4 ones
    x = np.abs(rng.standard_normal(2 * 3 * 5 * 4)).astype(np.float32)
    st, rows = R.im2col_quantize_pack(x, 2, 3, 5, 4, 3, 3, 2, 1, 0.6, 1.1, 1); assert st == 0
    g["im2col_strided_x"], g["im2col_strided_rows"] = x, rows

    # ---- conv exactness shapes (R:tests/acceptance.cpp:162-218) ------------
    for i, (c, r, k, s, p, b) in enumerate(CONV_SHAPES):
        x = np.abs(rng.standard_normal(b * c * r * r)).astype(np.float32)
        wq = rng.integers(-1, 2, (c, c * k * k)).astype(np.int8)
        st, rows = R.im2col_quantize_pack(x, b, c, r, r, k, k, s, p, 0.5, 0.9, 1); assert st == 0
        st, acc = R.conv_gemm(x, b, c, r, r, wq, c, k, s, p, (0.5, 0.9)); assert st == 0
        gain = (rng.standard_normal(c) * 0.05).astype(np.float32)
        bias = rng.standard_normal(c).astype(np.float32)
        spec = dict(in_c=c, out_c=c, k=k, stride=s, pad=p, weights=wq, ta=(0.5, 0.9),
                    tw=(0.8, 1.2), gain=gain, bias=bias, out_scale=0.37)
        st, y = R.conv2d_ternary(x, b, c, r, r, spec); assert st == 0
        # symmetric (weight-mode) activations on the same shape
        xs_ = rng.standard_normal(b * c * r * r).astype(np.float32)
        st, acc_sym = R.conv_gemm(xs_, b, c, r, r, wq, c, k, s, p, (0.8, 1.2), nonneg=False)
        assert st == 0
        g.update({f"conv{i}_x": x, f"conv{i}_w": wq, f"conv{i}_rows": rows, f"conv{i}_acc": acc,
                  f"conv{i}_gain": gain, f"conv{i}_bias": bias, f"conv{i}_y": y,
                  f"conv{i}_xs": xs_, f"conv{i}_acc_sym": acc_sym})
    g["conv_shapes"] = np.array(CONV_SHAPES, np.int32)

    # ---- fully connected (R:tests/test_linalg.cpp:342-380) ------------------
    for name, (bt, cin, cout) in {"fc_small": (3, 20, 6), "fc_mid": (64, 512, 256)}.items():
        x = np.abs(rng.standard_normal(bt * cin)).astype(np.float32)
        wq = rng.integers(-1, 2, (cout, cin)).astype(np.int8)
        gain = (rng.standard_normal(cout) * 0.05).astype(np.float32)
        bias = rng.standard_normal(cout).astype(np.float32)
        spec = dict(in_c=cin, out_c=cout, k=1, stride=1, pad=0, weights=wq, ta=(0.5, 0.9),
                    gain=gain, bias=bias, out_scale=1.0)
        st, y = R.fully_connected_ternary(x, bt, spec); assert st == 0
        g.update({f"{name}_x": x, f"{name}_w": wq, f"{name}_gain": gain, f"{name}_bias": bias,
                  f"{name}_y": y, f"{name}_dims": np.array([bt, cin, cout], np.int32)})

    # ---- fuse_bn (R:tests/test_linalg.cpp:65-92) ----------------------------
    m = rng.uniform(-1, 1, 256).astype(np.float32); v = rng.uniform(0.1, 2.0, 256).astype(np.float32)
    ga = rng.uniform(-1, 1, 256).astype(np.float32); be = rng.uniform(-1, 1, 256).astype(np.float32)
    st, fg, fb = R.fuse_bn(m, v, ga, be, 1e-5); assert st == 0
    g.update({"bn_mean": m, "bn_var": v, "bn_gamma": ga, "bn_beta": be, "bn_gain": fg, "bn_bias": fb})

    # ---- packed_forward composition (R:tinynet.hpp:713-735) -----------------
    in_dim, hidden, ncls, nb, batch = 2, 64, 4, 2, 32
    xin = rng.standard_normal(batch * in_dim).astype(np.float32)
    stem_w = (rng.standard_normal(hidden * in_dim) * 1.0).astype(np.float32)
    stem_b = np.zeros(hidden, np.float32)
    head_w = (rng.standard_normal(ncls * hidden) * 0.17).astype(np.float32)
    head_b = np.zeros(ncls, np.float32)
    blocks, cg, cb = [], [], []
    for _ in range(nb):
        wq = rng.integers(-1, 2, (hidden, hidden)).astype(np.int8)
        blocks.append(dict(in_c=hidden, out_c=hidden, k=1, stride=1, pad=0, weights=wq,
                           ta=(0.45, 0.8), tw=(0.9, 1.1),
                           gain=(rng.standard_normal(hidden) * 0.1).astype(np.float32),
                           bias=(rng.standard_normal(hidden) * 0.3).astype(np.float32),
                           out_scale=1.0))
        cg.append(rng.uniform(0.5, 1.5, hidden).astype(np.float32))
        cb.append(rng.uniform(-0.2, 0.2, hidden).astype(np.float32))
    cg = np.concatenate(cg); cb = np.concatenate(cb)
    st, logits = R.packed_forward(xin, batch, in_dim, hidden, ncls, stem_w, stem_b, blocks, cg, cb,
                                  head_w, head_b); assert st == 0
    g.update({"pf_x": xin, "pf_stem_w": stem_w, "pf_stem_b": stem_b, "pf_head_w": head_w,
              "pf_head_b": head_b, "pf_cal_gain": cg, "pf_cal_bias": cb, "pf_logits": logits,
              "pf_dims": np.array([batch, in_dim, hidden, ncls, nb], np.int32)})
    for i, b in enumerate(blocks):
        g.update({f"pf_b{i}_w": b["weights"], f"pf_b{i}_gain": b["gain"], f"pf_b{i}_bias": b["bias"]})
    st, logits_nocal = R.packed_forward(xin, batch, in_dim, hidden, ncls, stem_w, stem_b, blocks,
                                        None, None, head_w, head_b); assert st == 0
    g["pf_logits_nocal"] = logits_nocal

    # ---- paper baselines: binary (Eq. 1) and bit-plane multi-bit (Eq. 2) --------
    # (R:bitkernels.hpp:99-224; cases after R:tests/test_bitkernels.cpp:157-220,
    # R:tests/acceptance.cpp:94-117)
    bin_lens = [8, 1, 63, 64, 65, 700, 4096]
    for i, n in enumerate(bin_lens):
        bx = rng.choice(np.array([-1, 1], np.int8), n)
        by = rng.choice(np.array([-1, 1], np.int8), n)
        st, wx = R.pack_binary(bx); assert st == 0
        st, wy = R.pack_binary(by); assert st == 0
        st, d = R.binary_dot(wx, wy, n); assert st == 0 and d == int(bx.astype(np.int64) @ by)
        g.update({f"bin{i}_x": bx, f"bin{i}_y": by, f"bin{i}_wx": wx, f"bin{i}_wy": wy,
                  f"bin{i}_dot": np.array([d], np.int64)})
    mb = []
    for i, (n, m, k) in enumerate([(100, 2, 2), (4096, 2, 2), (333, 3, 1), (64, 1, 3)]):
        xs = [rng.choice(np.array([-1, 1], np.int8), n) for _ in range(m)]
        ys = [rng.choice(np.array([-1, 1], np.int8), n) for _ in range(k)]
        sx = (np.array([1.0, 2.0, 4.0])[:m] if i < 2 else rng.standard_normal(m)).astype(np.float64)
        sy = (np.array([1.0, 2.0, 4.0])[:k] if i < 2 else rng.standard_normal(k)).astype(np.float64)
        xp = np.stack([R.pack_binary(v)[1] for v in xs])
        yp = np.stack([R.pack_binary(v)[1] for v in ys])
        st, d = R.multibit_dot(xp, sx, yp, sy, n); assert st == 0
        g.update({f"mb{i}_xp": xp, f"mb{i}_yp": yp, f"mb{i}_sx": sx, f"mb{i}_sy": sy,
                  f"mb{i}_dims": np.array([n, m, k], np.int64), f"mb{i}_dot": np.array([d], np.float64)})

    # ---- FATN model files written by the reference serializer (F2 loader
    # fixtures, R:model_io.hpp:151-301); its own load_model + packed_forward
    # reproduce the logits above
    gdir = os.path.dirname(OUT)
    os.makedirs(gdir, exist_ok=True)
    for tag, (c_g, c_b, want) in {"cal": (cg, cb, logits), "nocal": (None, None, logits_nocal)}.items():
        path = os.path.join(gdir, f"pf_{tag}.fatn")
        assert R.save_packed_model(path, in_dim, hidden, ncls, stem_w, stem_b, blocks, c_g, c_b, head_w,
                                   head_b) == 0
        st, lg = R.load_and_forward(path, xin, batch)
        assert st == 0 and np.array_equal(lg.view(np.int32), want.view(np.int32))

    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
