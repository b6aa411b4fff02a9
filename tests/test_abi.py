"""CPU-side checks of the boundary: the C-ABI library loads, exports every
symbol include/ternkit_b200.h declares with the declared arity, and the
host-only logic (exact quantizer thresholds, fuse_bn) matches the oracle /
golden vectors.  No GPU needed."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from tests.conftest import ROOT

HEADER = os.path.join(ROOT, "include", "ternkit_b200.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    out = {}
    for m in re.finditer(r"^(?:int|const char\*)\s+(tk_\w+)\s*\(([^)]*)\)\s*;", src, flags=re.M):
        args = [a for a in m.group(2).replace("\n", " ").split(",") if a.strip() and a.strip() != "void"]
        out[m.group(1)] = len(args)
    return out


@pytest.fixture(scope="module")
def lib():
    from paper_2008_05101_b200 import build
    build.build()
    from paper_2008_05101_b200 import _lib
    return _lib


def test_header_symbols_exported(lib):
    decl = declared()
    assert len(decl) >= 20
    nm = subprocess.run(["nm", "-D", "--defined-only", lib.LIB_PATH], capture_output=True, text=True,
                        check=True).stdout
    exported = set(re.findall(r"\bT (tk_\w+)", nm))
    missing = set(decl) - exported
    assert not missing, f"declared but not exported: {missing}"
    L = lib.lib()
    for name, nargs in decl.items():
        assert name in lib.SIGNATURES, name
        assert len(lib.SIGNATURES[name][1]) == nargs, name
        getattr(L, name)


def test_status_strings(lib):
    L = lib.lib()
    assert L.tk_version() >= 100
    for st in (0, 1, 3, 4, 5, 6, 7, 8, 9, 10):
        assert L.tk_status_string(st)


def test_sm100a_cubin_present(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def _thresholds(lib, a1, a2, mode):
    t0, t1 = C.c_float(), C.c_float()
    st = lib.lib().tk_quant_thresholds(a1, a2, mode, C.byref(t0), C.byref(t1))
    return st, np.float32(t0.value), np.float32(t1.value)


def _code_levels(p, t0, t1, mode):
    b0 = (p > t0).astype(np.int32)
    b1 = (p > t1).astype(np.int32)
    return b0 + b1 - (0 if mode == 1 else 1)


def test_thresholds_reproduce_quantizer(lib, oracle, golden):
    """The GPU quantizer is two float compares; the thresholds must reproduce
    round(clip(p/a)) of R:quantizer.hpp:44-60 exactly, including ties."""
    for mode, pkey, lkey in ((0, "qz_pw", "qz_lw"), (1, "qz_pa", "qz_la")):
        a1s, a2s, ps, ls = golden["qz_a1"], golden["qz_a2"], golden[pkey], golden[lkey]
        for a1, a2, p, lv in zip(a1s[-200:], a2s[-200:], ps[-200:], ls[-200:]):
            st, t0, t1 = _thresholds(lib, float(a1), float(a2), mode)
            assert st == 0
            assert _code_levels(np.float32(p), t0, t1, mode) == lv


def test_thresholds_dense_sweep(lib, oracle):
    """Every float within +-64 ulps of both thresholds, random step sizes."""
    rng = np.random.default_rng(11)
    for _ in range(60):
        a1, a2 = [float(np.float32(v)) for v in rng.uniform(0.05, 3.0, 2)]
        for mode in (0, 1):
            st, t0, t1 = _thresholds(lib, a1, a2, mode)
            assert st == 0
            for t in (t0, t1):
                bits = np.float32(t).view(np.int32)
                for d in range(-64, 65):
                    p = np.int32(bits + d).view(np.float32)
                    if not np.isfinite(p) or (mode == 1 and p < 0):
                        continue
                    f = oracle.quantize_weight_value if mode == 0 else oracle.quantize_activation_value
                    s, lv = f(float(p), a1, a2)
                    assert s == 0 and _code_levels(np.float32(p), t0, t1, mode) == lv, (a1, a2, mode, p)


def test_thresholds_reject_bad_steps(lib):
    assert _thresholds(lib, 0.0, 1.0, 0)[0] == 3
    assert _thresholds(lib, 1.0, -1.0, 1)[0] == 3
    assert _thresholds(lib, float("nan"), 1.0, 1)[0] == 3


def test_fuse_bn_host(lib, golden):
    m, v, g, b = (np.ascontiguousarray(golden[k]) for k in ("bn_mean", "bn_var", "bn_gamma", "bn_beta"))
    gain = np.empty_like(m)
    bias = np.empty_like(m)
    st = lib.lib().tk_fuse_bn(m.ctypes.data, v.ctypes.data, g.ctypes.data, b.ctypes.data, 1e-5, m.size,
                              gain.ctypes.data, bias.ctypes.data)
    assert st == 0
    assert np.array_equal(gain, golden["bn_gain"]) and np.array_equal(bias, golden["bn_bias"])
    z = np.zeros(1, np.float32)
    assert lib.lib().tk_fuse_bn(z.ctypes.data, z.ctypes.data, z.ctypes.data, z.ctypes.data, 0.0, 1,
                                gain.ctypes.data, bias.ctypes.data) == 1


def test_compute_entry_points_fail_without_gpu(lib):
    """No CPU fallback: without a device, context creation reports CUDA error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    assert lib.lib().tk_context_create(0, C.byref(h)) == 9
