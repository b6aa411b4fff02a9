"""The paper's comparison baselines (SURVEY §8(f) F3, R:bitkernels.hpp:99-224):
binary XNOR-popcount dot (Eq. 1) and the bit-plane decomposed multi-bit dot
(Eq. 2).  Golden vectors come from the compiled reference (oracle/make_golden.py);
integers bit-exact, the f64 multi-bit result bit-identical."""
import numpy as np
import pytest

BIN = 7
MB = 4


def test_oracle_binary_and_multibit_match_golden(oracle, golden):
    for i in range(BIN):
        st, wx = oracle.pack_binary(golden[f"bin{i}_x"])
        assert st == 0 and np.array_equal(wx, golden[f"bin{i}_wx"])
        n = golden[f"bin{i}_x"].size
        assert oracle.binary_dot(wx, golden[f"bin{i}_wy"], n) == int(golden[f"bin{i}_dot"][0])
    for i in range(MB):
        n = int(golden[f"mb{i}_dims"][0])
        d = oracle.multibit_dot(golden[f"mb{i}_xp"], golden[f"mb{i}_sx"], golden[f"mb{i}_yp"], golden[f"mb{i}_sy"], n)
        assert np.float64(d).view(np.int64) == golden[f"mb{i}_dot"].view(np.int64)[0]
    st, _ = oracle.pack_binary(np.array([0], np.int8))  # R:tests/test_bitkernels.cpp:163
    assert st != 0


@pytest.mark.gpu
def test_gpu_binary_and_multibit_match_golden(tk, golden):
    import torch
    for i in range(BIN):
        v = tk.pack_binary(golden[f"bin{i}_x"])
        assert np.array_equal(v.words.cpu().numpy().view(np.uint64), golden[f"bin{i}_wx"])
        w = tk.pack_binary(golden[f"bin{i}_y"])
        assert tk.binary_dot(v, w) == int(golden[f"bin{i}_dot"][0])
    for i in range(MB):
        n, m, k = map(int, golden[f"mb{i}_dims"])
        xp = torch.from_numpy(golden[f"mb{i}_xp"].view(np.int64)).cuda()
        yp = torch.from_numpy(golden[f"mb{i}_yp"].view(np.int64)).cuda()
        mx = tk.MultiBitVector([tk.PackedBinaryVector(xp[j], n) for j in range(m)], list(golden[f"mb{i}_sx"]))
        my = tk.MultiBitVector([tk.PackedBinaryVector(yp[j], n) for j in range(k)], list(golden[f"mb{i}_sy"]))
        d = tk.multibit_dot(mx, my)
        assert np.float64(d).view(np.int64) == golden[f"mb{i}_dot"].view(np.int64)[0]
    # R:tests/test_bitkernels.cpp:157-163, 207-220
    x = np.array([1, -1, 1, 1, -1, 1, 1, 1], np.int8)
    assert tk.binary_dot(tk.pack_binary(x), tk.pack_binary(x)) == 8
    assert tk.binary_dot(tk.pack_binary(x), tk.pack_binary(-x)) == -8
    with pytest.raises(tk.InvalidArgument):
        tk.pack_binary(np.array([0], np.int8))
    px = tk.pack_binary(x)
    assert tk.multibit_dot(tk.MultiBitVector([px], [0.0]), tk.MultiBitVector([px], [3.0])) == 0.0
    with pytest.raises(tk.InvalidArgument):
        tk.multibit_dot(tk.MultiBitVector([px], [1.0, 2.0]), tk.MultiBitVector([px], [1.0]))
    with pytest.raises(tk.InvalidArgument):
        tk.multibit_dot(tk.MultiBitVector([px], [1.0]), tk.MultiBitVector([tk.pack_binary(x[:7])], [1.0]))


@pytest.mark.gpu
def test_gpu_batched_baselines_vs_oracle(tk, oracle):
    import torch
    rng = np.random.default_rng(9)
    pairs, n = 300, 1000
    words = (n + 63) // 64
    xs = rng.choice(np.array([-1, 1], np.int8), (pairs, n))
    ys = rng.choice(np.array([-1, 1], np.int8), (pairs, n))
    px = np.stack([oracle.pack_binary(r)[1] for r in xs])
    py = np.stack([oracle.pack_binary(r)[1] for r in ys])
    got = tk.binary_dot_batched(torch.from_numpy(px.view(np.int64)).cuda(),
                                torch.from_numpy(py.view(np.int64)).cuda(), n).cpu().numpy()
    assert np.array_equal(got, (xs.astype(np.int64) * ys).sum(axis=1))
    sx, sy = np.array([1.0, 2.0]), np.array([1.0, 2.0])
    xp2 = np.stack([px, px[::-1]])  # [2][pairs][words]
    yp2 = np.stack([py, py[::-1]])
    got = tk.multibit_dot_batched(torch.from_numpy(xp2.view(np.int64)).cuda(), sx,
                                  torch.from_numpy(yp2.view(np.int64)).cuda(), sy, n).cpu().numpy()
    want = np.array([oracle.multibit_dot(xp2[:, p], sx, yp2[:, p], sy, n) for p in range(pairs)])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))
    assert words == px.shape[1]
