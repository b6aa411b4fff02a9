"""ctypes bindings for the parity checkers under oracle/.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py -- never by the product
package (paper_2008_05101_b200), which fails loudly without its CUDA library.

* ``Oracle``    -- oracle/liboracle.so, the C restatement of the reference
                   hot path (oracle/ternkit_oracle.c).
* ``Reference`` -- oracle/_ref/libternkit_ref_<isa>.so, the reference headers
                   compiled unmodified from /root/reference (oracle/Makefile).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)
_f32p = C.POINTER(C.c_float)
_sz = C.c_size_t

MODE_WEIGHT = 0
MODE_ACT_NONNEG = 1


def ptr(a: np.ndarray | None, t):
    if a is None:
        return C.cast(None, t)
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(t)


class NdConv(C.Structure):
    _fields_ = [
        ("in_c", C.c_int), ("out_c", C.c_int), ("k", C.c_int),
        ("stride", C.c_int), ("pad", C.c_int),
        ("weights", _i8p),
        ("tw1", C.c_float), ("tw2", C.c_float),
        ("ta1", C.c_float), ("ta2", C.c_float),
        ("gain", _f32p), ("bias", _f32p),
        ("out_scale", C.c_float),
    ]


class NdBlock(C.Structure):
    _fields_ = [("n_convs", C.c_int), ("conv", NdConv * 3),
                ("has_down", C.c_int), ("down", NdConv)]


def make_ndconv(spec, keep: list) -> NdConv:
    """spec: dict with in_c,out_c,k,stride,pad,weights(int8 [oc][K]),ta,tw,gain,bias,out_scale."""
    w = np.ascontiguousarray(spec["weights"], dtype=np.int8)
    g = np.ascontiguousarray(spec["gain"], dtype=np.float32) if spec.get("gain") is not None else None
    b = np.ascontiguousarray(spec["bias"], dtype=np.float32) if spec.get("bias") is not None else None
    keep += [w, g, b]
    tw = spec.get("tw", (1.0, 1.0))
    ta = spec["ta"]
    return NdConv(spec["in_c"], spec["out_c"], spec["k"], spec["stride"], spec["pad"],
                  ptr(w, _i8p), tw[0], tw[1], ta[0], ta[1], ptr(g, _f32p), ptr(b, _f32p),
                  spec.get("out_scale", 1.0))


def make_ndblocks(blocks, keep: list):
    arr = (NdBlock * len(blocks))()
    for i, blk in enumerate(blocks):
        arr[i].n_convs = len(blk["convs"])
        for j, cv in enumerate(blk["convs"]):
            arr[i].conv[j] = make_ndconv(cv, keep)
        arr[i].has_down = 1 if blk.get("down") is not None else 0
        if blk.get("down") is not None:
            arr[i].down = make_ndconv(blk["down"], keep)
    return arr


def words_for_lanes(n: int) -> int:
    return (n + 31) // 32


def _build():
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


class Oracle:
    """C restatement (oracle/ternkit_oracle.c)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            _build()
        L = self.lib = C.CDLL(path)
        L.or_quantize_weight_value.argtypes = [C.c_float, C.c_float, C.c_float, C.POINTER(C.c_int)]
        L.or_quantize_activation_value.argtypes = [C.c_float, C.c_float, C.c_float, C.POINTER(C.c_int)]
        L.or_pack.argtypes = [_i8p, _sz, _u64p]
        L.or_unpack.argtypes = [_u64p, _sz, _i8p]
        L.or_quantize_and_pack.argtypes = [_f32p, _sz, C.c_float, C.c_float, C.c_int, _u64p]
        L.or_ternary_multiply_word.argtypes = [C.c_uint64, C.c_uint64]
        L.or_ternary_multiply_word.restype = C.c_uint64
        L.or_ternary_dot_batched.argtypes = [_u64p, _u64p, _sz, _sz, _i64p, _i64p]
        L.or_ternary_dot_batched.restype = None
        L.or_im2col_quantize_pack.argtypes = [_f32p] + [C.c_int] * 8 + [C.c_float, C.c_float, C.c_int, _u64p]
        L.or_packed_gemm.argtypes = [_u64p, _sz, _sz, _u64p, _i32p, C.c_int, C.c_int, _i32p]
        L.or_packed_gemm.restype = None
        L.or_conv2d_ternary.argtypes = ([_f32p] + [C.c_int] * 9 + [_u64p, _i32p, C.c_float, C.c_float,
                                        C.c_int, _f32p, _f32p, C.c_float, _f32p])
        L.or_fuse_bn.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_float, C.c_int, _f32p, _f32p]
        L.or_residual_relu_rows.argtypes = [_f32p, _f32p, _sz, C.c_int, _f32p, _f32p]
        L.or_residual_relu_rows.restype = None
        L.or_net_body.argtypes = [C.c_void_p, C.c_int, _f32p, C.c_int, C.c_int, C.c_int, C.c_int, _f32p,
                                  C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_matmul_t.argtypes = [_f32p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, _f32p]
        L.or_matmul_t.restype = None
        L.or_pack_binary.argtypes = [_i8p, _sz, _u64p]
        L.or_binary_dot.argtypes = [_u64p, _u64p, _sz, _sz]
        L.or_binary_dot.restype = C.c_int64
        L.or_multibit_dot.argtypes = [_u64p, C.c_int, _u64p, C.c_int, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), _sz, _sz, C.c_int]
        L.or_multibit_dot.restype = C.c_double

    # paper baselines (R:bitkernels.hpp:99-224) ----------------------------
    def pack_binary(self, v):
        v = np.ascontiguousarray(v, dtype=np.int8)
        w = np.zeros((v.size + 63) // 64, np.uint64)
        st = self.lib.or_pack_binary(ptr(v, _i8p), v.size, ptr(w, _u64p))
        return st, w

    def binary_dot(self, x, y, n):
        x = np.ascontiguousarray(x, np.uint64)
        y = np.ascontiguousarray(y, np.uint64)
        return self.lib.or_binary_dot(ptr(x, _u64p), ptr(y, _u64p), x.size, n)

    def multibit_dot(self, xp, sx, yp, sy, n):
        xp = np.ascontiguousarray(xp, np.uint64)
        yp = np.ascontiguousarray(yp, np.uint64)
        sx = np.ascontiguousarray(sx, np.float64)
        sy = np.ascontiguousarray(sy, np.float64)
        dp = C.POINTER(C.c_double)
        return self.lib.or_multibit_dot(ptr(xp, _u64p), xp.shape[0], ptr(yp, _u64p), yp.shape[0],
                                        sx.ctypes.data_as(dp), sy.ctypes.data_as(dp), xp.shape[1], n, 0)

    # scalar quantizers -------------------------------------------------
    def quantize_weight_value(self, p, a1, a2):
        lv = C.c_int()
        st = self.lib.or_quantize_weight_value(p, a1, a2, C.byref(lv))
        return st, lv.value

    def quantize_activation_value(self, p, a1, a2):
        lv = C.c_int()
        st = self.lib.or_quantize_activation_value(p, a1, a2, C.byref(lv))
        return st, lv.value

    # vectors ------------------------------------------------------------
    def pack(self, v):
        v = np.ascontiguousarray(v, dtype=np.int8)
        w = np.empty(words_for_lanes(v.size), np.uint64)
        st = self.lib.or_pack(ptr(v, _i8p), v.size, ptr(w, _u64p))
        return st, w

    def unpack(self, words, n):
        words = np.ascontiguousarray(words, dtype=np.uint64)
        v = np.empty(n, np.int8)
        self.lib.or_unpack(ptr(words, _u64p), n, ptr(v, _i8p))
        return v

    def quantize_and_pack(self, x, a1, a2, mode):
        x = np.ascontiguousarray(x, dtype=np.float32)
        w = np.empty(words_for_lanes(x.size), np.uint64)
        st = self.lib.or_quantize_and_pack(ptr(x, _f32p), x.size, a1, a2, mode, ptr(w, _u64p))
        return st, w

    def ternary_multiply_word(self, x, y):
        return self.lib.or_ternary_multiply_word(int(x), int(y))

    def ternary_dot_batched(self, x, y, wsum=None):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(y, dtype=np.uint64)
        pairs, words = x.shape
        ws = None if wsum is None else np.ascontiguousarray(wsum, dtype=np.int64)
        out = np.empty(pairs, np.int64)
        self.lib.or_ternary_dot_batched(ptr(x, _u64p), ptr(y, _u64p), words, pairs,
                                        ptr(ws, _i64p), ptr(out, _i64p))
        return out

    def im2col_quantize_pack(self, x, n, c, h, w, kh, kw, stride, pad, a1, a2, mode):
        x = np.ascontiguousarray(x, dtype=np.float32)
        oh = (h + 2 * pad - kh) // stride + 1
        ow = (w + 2 * pad - kw) // stride + 1
        wpr = words_for_lanes(c * kh * kw)
        rows = np.zeros((n * oh * ow, wpr), np.uint64)
        st = self.lib.or_im2col_quantize_pack(ptr(x, _f32p), n, c, h, w, kh, kw, stride, pad,
                                              a1, a2, mode, ptr(rows, _u64p))
        return st, rows

    def packed_gemm(self, rows, weights, wsums, offset):
        rows = np.ascontiguousarray(rows, dtype=np.uint64)
        weights = np.ascontiguousarray(weights, dtype=np.uint64)
        wsums = np.ascontiguousarray(wsums, dtype=np.int32)
        oc = weights.shape[0]
        out = np.empty((rows.shape[0], oc), np.int32)
        self.lib.or_packed_gemm(ptr(rows, _u64p), rows.shape[0], rows.shape[1], ptr(weights, _u64p),
                                ptr(wsums, _i32p), oc, int(offset), ptr(out, _i32p))
        return out

    def pack_rows(self, wq):
        """weights int8 [oc][K] -> (packed rows [oc][wpr] u64, wsums int32)."""
        wq = np.ascontiguousarray(wq, dtype=np.int8)
        oc, k = wq.shape
        rows = np.empty((oc, words_for_lanes(k)), np.uint64)
        for o in range(oc):
            st, rows[o] = self.pack(wq[o])
            assert st == 0
        return rows, wq.astype(np.int32).sum(axis=1).astype(np.int32)

    def conv2d_ternary(self, x, n, c, h, w, wq, out_c, k, stride, pad, ta, nonneg=True,
                       gain=None, bias=None, out_scale=1.0):
        x = np.ascontiguousarray(x, dtype=np.float32)
        rows, ws = self.pack_rows(np.asarray(wq).reshape(out_c, -1))
        oh = (h + 2 * pad - k) // stride + 1
        ow = (w + 2 * pad - k) // stride + 1
        out = np.empty((n, out_c, oh, ow), np.float32)
        g = None if gain is None else np.ascontiguousarray(gain, np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        st = self.lib.or_conv2d_ternary(ptr(x, _f32p), n, c, h, w, out_c, k, k, stride, pad,
                                        ptr(rows, _u64p), ptr(ws, _i32p), ta[0], ta[1], int(nonneg),
                                        ptr(g, _f32p), ptr(b, _f32p), out_scale, ptr(out, _f32p))
        return st, out

    def fuse_bn(self, mean, var, gamma, beta, eps):
        arrs = [np.ascontiguousarray(a, np.float32) for a in (mean, var, gamma, beta)]
        c = arrs[0].size
        g = np.empty(c, np.float32)
        b = np.empty(c, np.float32)
        st = self.lib.or_fuse_bn(*[ptr(a, _f32p) for a in arrs], eps, c, ptr(g, _f32p), ptr(b, _f32p))
        return st, g, b

    def residual_relu_rows(self, z, h, hidden, cal_gain=None, cal_bias=None):
        z = np.array(z, dtype=np.float32, copy=True)
        h = np.ascontiguousarray(h, np.float32)
        cg = None if cal_gain is None else np.ascontiguousarray(cal_gain, np.float32)
        cb = None if cal_bias is None else np.ascontiguousarray(cal_bias, np.float32)
        self.lib.or_residual_relu_rows(ptr(z, _f32p), ptr(h, _f32p), z.size, hidden,
                                       ptr(cg, _f32p), ptr(cb, _f32p))
        return z

    def matmul_t(self, x, w, bias, batch, in_dim, out_dim):
        x = np.ascontiguousarray(x, np.float32)
        w = np.ascontiguousarray(w, np.float32)
        b = None if bias is None else np.ascontiguousarray(bias, np.float32)
        y = np.empty((batch, out_dim), np.float32)
        self.lib.or_matmul_t(ptr(x, _f32p), ptr(w, _f32p), ptr(b, _f32p), batch, in_dim, out_dim,
                             ptr(y, _f32p))
        return y

    def net_body(self, blocks, x, n, c, h, w):
        keep: list = []
        arr = make_ndblocks(blocks, keep)
        x = np.ascontiguousarray(x, np.float32)
        # generous output buffer: channel/spatial walk
        cc, hh, ww = c, h, w
        for blk in blocks:
            for cv in blk["convs"]:
                hh = (hh + 2 * cv["pad"] - cv["k"]) // cv["stride"] + 1
                ww = (ww + 2 * cv["pad"] - cv["k"]) // cv["stride"] + 1
                cc = cv["out_c"]
        out = np.empty((n, cc, hh, ww), np.float32)
        oc, oh, ow = C.c_int(), C.c_int(), C.c_int()
        st = self.lib.or_net_body(C.cast(arr, C.c_void_p), len(blocks), ptr(x, _f32p), n, c, h, w,
                                  ptr(out, _f32p), C.byref(oc), C.byref(oh), C.byref(ow))
        return st, out


class RunStats(C.Structure):
    """ref_run_stats (oracle/ref_shim.cpp): the reference's RunStats summary."""
    _fields_ = [("mean_us", C.c_double), ("stddev_us", C.c_double), ("median_us", C.c_double),
                ("stable", C.c_int), ("repeats", C.c_int), ("warmup", C.c_int), ("min_run_s", C.c_double)]

    def as_dict(self) -> dict:
        return {"mean_us": self.mean_us, "stddev_us": self.stddev_us, "median_us": self.median_us,
                "stable": bool(self.stable), "cv": self.stddev_us / self.mean_us if self.mean_us else None,
                "repeats": self.repeats, "warmup": self.warmup, "min_run_s": self.min_run_s}


def host_cpu() -> dict:
    """lscpu-style record of the host the CPU baseline ran on."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    flags = _cpu_flags()
    return {"model": model, "nproc": os.cpu_count(),
            "avx512_vpopcntdq": "avx512_vpopcntdq" in flags, "avx512f": "avx512f" in flags,
            "avx2": "avx2" in flags}


def _cpu_flags() -> set[str]:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def reference_lib_path() -> str | None:
    """Pick the reference build this host can execute (AVX-512 build needs the
    ISA of the container that compiled it; otherwise the AVX2+FMA build)."""
    d = os.path.join(HERE, "_ref")
    native = os.path.join(d, "libternkit_ref_native.so")
    v3 = os.path.join(d, "libternkit_ref_v3.so")
    flags = _cpu_flags()
    need = {"avx512f", "avx512bw", "avx512vl", "avx512_vpopcntdq", "avx512_fp16", "amx_tile",
            "avx512_bf16", "avx512vbmi"}
    if os.path.exists(native) and need <= flags:
        return native
    if os.path.exists(v3) and {"avx2", "fma", "bmi2"} <= flags:
        return v3
    return None


class Reference:
    """The unmodified reference headers compiled into oracle/_ref."""

    def __init__(self, path: str | None = None):
        path = path or reference_lib_path()
        if path is None:
            raise FileNotFoundError("oracle/_ref reference build missing (run `make -C oracle ref`)")
        self.path = path
        L = self.lib = C.CDLL(path)
        L.ref_quantize_weight_value.argtypes = [C.c_float, C.c_float, C.c_float, C.POINTER(C.c_int)]
        L.ref_quantize_activation_value.argtypes = [C.c_float, C.c_float, C.c_float, C.POINTER(C.c_int)]
        L.ref_pack.argtypes = [_i8p, _sz, _u64p]
        L.ref_quantize_and_pack.argtypes = [_f32p, _sz, C.c_float, C.c_float, C.c_int, _u64p]
        L.ref_ternary_multiply_word.argtypes = [C.c_uint64, C.c_uint64]
        L.ref_ternary_multiply_word.restype = C.c_uint64
        L.ref_ternary_dot_batched.argtypes = [_u64p, _u64p, _sz, _sz, _i64p, _i64p]
        L.ref_im2col_quantize_pack.argtypes = [_f32p] + [C.c_int] * 8 + [C.c_float, C.c_float, C.c_int, _u64p]
        L.ref_conv_gemm.argtypes = ([_f32p] + [C.c_int] * 4 + [_i8p] + [C.c_int] * 4 +
                                    [C.c_float, C.c_float, C.c_int, C.c_int, C.c_int, _i32p])
        L.ref_conv2d_ternary.argtypes = [_f32p] + [C.c_int] * 4 + [C.POINTER(NdConv), C.c_int, C.c_int, _f32p]
        L.ref_fully_connected_ternary.argtypes = [_f32p, C.c_int, C.POINTER(NdConv), C.c_int, _f32p]
        L.ref_fuse_bn.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_float, C.c_int, _f32p, _f32p]
        L.ref_packed_forward.argtypes = ([_f32p] + [C.c_int] * 4 + [_f32p, _f32p, C.c_int,
                                         C.POINTER(NdConv), _f32p, _f32p, _f32p, _f32p, _f32p])
        L.ref_net_create.argtypes = [C.c_void_p, C.c_int]
        L.ref_net_create.restype = C.c_void_p
        L.ref_net_destroy.argtypes = [C.c_void_p]
        L.ref_net_destroy.restype = None
        L.ref_net_run.argtypes = [C.c_void_p, _f32p] + [C.c_int] * 5 + [_f32p, C.POINTER(C.c_double)]
        L.ref_time_fc_gemm.argtypes = [_f32p, C.c_int, C.c_int, _i8p, C.c_int, C.c_float, C.c_float,
                                       C.c_int, C.c_int, C.POINTER(C.c_double), _i32p]
        L.ref_time_dot.argtypes = [_u64p, _u64p, _sz, _sz, _i64p, C.c_int, C.POINTER(C.c_double), _i64p]
        L.ref_time_conv.argtypes = ([_f32p] + [C.c_int] * 4 + [C.POINTER(NdConv), C.c_int, C.c_int,
                                    C.POINTER(C.c_double), _f32p])

    def make_packed_conv_layer(self, wq, in_c, out_c, kh, kw):
        """R:linalg.hpp:118-144: (packed rows [out_c][words] u64, weight_sums i32)."""
        wq = np.ascontiguousarray(wq, dtype=np.int8)
        nw = words_for_lanes(in_c * kh * kw)
        words = np.empty((out_c, nw), np.uint64)
        sums = np.empty(out_c, np.int32)
        f = self.lib.ref_make_packed_conv_layer
        f.argtypes = [_i8p] + [C.c_int] * 4 + [_u64p, _i32p]
        st = f(ptr(wq, _i8p), in_c, out_c, kh, kw, ptr(words, _u64p), ptr(sums, _i32p))
        return st, words, sums

    # ---- the reference's time_runs protocol (R:include/ternkit/bench.hpp:64-99) ----
    def _runs(self, name, args, argtypes, repeats, warmup, min_run_s):
        f = getattr(self.lib, name)
        f.argtypes = argtypes + [C.c_int, C.c_int, C.c_double, C.POINTER(RunStats)]
        st = RunStats()
        rc = f(*args, repeats, warmup, min_run_s, C.byref(st))
        return rc, st.as_dict()

    def time_runs_net(self, handle, x, n, c, h, w, threads, repeats=5, warmup=2, min_run_s=0.6):
        x = np.ascontiguousarray(x, np.float32)
        return self._runs("ref_time_runs_net", [handle, ptr(x, _f32p), n, c, h, w, threads],
                          [C.c_void_p, _f32p] + [C.c_int] * 5, repeats, warmup, min_run_s)

    def time_runs_fc(self, x, wq, ta, workers, repeats=5, warmup=2, min_run_s=0.6):
        x = np.ascontiguousarray(x, np.float32)
        wq = np.ascontiguousarray(wq, np.int8)
        b, k = x.shape
        n = wq.shape[0]
        return self._runs("ref_time_runs_fc", [ptr(x, _f32p), b, k, ptr(wq, _i8p), n, ta[0], ta[1], workers],
                          [_f32p, C.c_int, C.c_int, _i8p, C.c_int, C.c_float, C.c_float, C.c_int],
                          repeats, warmup, min_run_s)

    def time_runs_conv(self, x, n, c, h, w, spec, workers, repeats=5, warmup=2, min_run_s=0.6):
        keep: list = []
        cv = make_ndconv(spec, keep)
        x = np.ascontiguousarray(x, np.float32)
        return self._runs("ref_time_runs_conv", [ptr(x, _f32p), n, c, h, w, C.byref(cv), workers],
                          [_f32p] + [C.c_int] * 4 + [C.POINTER(NdConv), C.c_int], repeats, warmup, min_run_s)

    def time_runs_dot(self, x, y, lanes, wsum, threads, repeats=5, warmup=2, min_run_s=0.6):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(y, dtype=np.uint64)
        ws = np.ascontiguousarray(wsum, dtype=np.int64)
        return self._runs("ref_time_runs_dot", [ptr(x, _u64p), ptr(y, _u64p), lanes, x.shape[0], ptr(ws, _i64p),
                                                threads],
                          [_u64p, _u64p, _sz, _sz, _i64p, C.c_int], repeats, warmup, min_run_s)

    def time_dot(self, x, y, lanes, wsum, threads):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(y, dtype=np.uint64)
        ws = np.ascontiguousarray(wsum, dtype=np.int64)
        out = np.empty(x.shape[0], np.int64)
        sec = C.c_double()
        st = self.lib.ref_time_dot(ptr(x, _u64p), ptr(y, _u64p), lanes, x.shape[0], ptr(ws, _i64p),
                                   threads, C.byref(sec), ptr(out, _i64p))
        return st, out, sec.value

    def time_conv(self, x, n, c, h, w, spec, workers, iters=1):
        keep: list = []
        cv = make_ndconv(spec, keep)
        x = np.ascontiguousarray(x, dtype=np.float32)
        k, s, p = spec["k"], spec["stride"], spec["pad"]
        oh = (h + 2 * p - k) // s + 1
        ow = (w + 2 * p - k) // s + 1
        out = np.empty((n, spec["out_c"], oh, ow), np.float32)
        sec = C.c_double()
        st = self.lib.ref_time_conv(ptr(x, _f32p), n, c, h, w, C.byref(cv), workers, iters,
                                    C.byref(sec), ptr(out, _f32p))
        return st, out, sec.value

    def quantize_weight_value(self, p, a1, a2):
        lv = C.c_int()
        st = self.lib.ref_quantize_weight_value(p, a1, a2, C.byref(lv))
        return st, lv.value

    def quantize_activation_value(self, p, a1, a2):
        lv = C.c_int()
        st = self.lib.ref_quantize_activation_value(p, a1, a2, C.byref(lv))
        return st, lv.value

    def pack(self, v):
        v = np.ascontiguousarray(v, dtype=np.int8)
        w = np.empty(words_for_lanes(v.size), np.uint64)
        st = self.lib.ref_pack(ptr(v, _i8p), v.size, ptr(w, _u64p))
        return st, w

    def quantize_and_pack(self, x, a1, a2, mode):
        x = np.ascontiguousarray(x, dtype=np.float32)
        w = np.empty(words_for_lanes(x.size), np.uint64)
        st = self.lib.ref_quantize_and_pack(ptr(x, _f32p), x.size, a1, a2, mode, ptr(w, _u64p))
        return st, w

    def ternary_multiply_word(self, x, y):
        return self.lib.ref_ternary_multiply_word(int(x), int(y))

    def ternary_dot_batched(self, x, y, lanes, wsum=None):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(y, dtype=np.uint64)
        pairs = x.shape[0]
        ws = None if wsum is None else np.ascontiguousarray(wsum, dtype=np.int64)
        out = np.empty(pairs, np.int64)
        st = self.lib.ref_ternary_dot_batched(ptr(x, _u64p), ptr(y, _u64p), lanes, pairs,
                                              ptr(ws, _i64p), ptr(out, _i64p))
        return st, out

    def im2col_quantize_pack(self, x, n, c, h, w, kh, kw, stride, pad, a1, a2, mode):
        x = np.ascontiguousarray(x, dtype=np.float32)
        oh = (h + 2 * pad - kh) // stride + 1
        ow = (w + 2 * pad - kw) // stride + 1
        rows = np.zeros((n * oh * ow, words_for_lanes(c * kh * kw)), np.uint64)
        st = self.lib.ref_im2col_quantize_pack(ptr(x, _f32p), n, c, h, w, kh, kw, stride, pad,
                                               a1, a2, mode, ptr(rows, _u64p))
        return st, rows

    def conv_gemm(self, x, n, c, h, w, wq, out_c, k, stride, pad, ta, nonneg=True, mask_mode=0,
                  workers=1):
        x = np.ascontiguousarray(x, dtype=np.float32)
        wq = np.ascontiguousarray(wq, dtype=np.int8)
        oh = (h + 2 * pad - k) // stride + 1
        ow = (w + 2 * pad - k) // stride + 1
        out = np.empty((n * oh * ow, out_c), np.int32)
        st = self.lib.ref_conv_gemm(ptr(x, _f32p), n, c, h, w, ptr(wq, _i8p), out_c, k, stride, pad,
                                    ta[0], ta[1], int(nonneg), mask_mode, workers, ptr(out, _i32p))
        return st, out

    def conv2d_ternary(self, x, n, c, h, w, spec, nonneg=True, workers=1):
        keep: list = []
        cv = make_ndconv(spec, keep)
        x = np.ascontiguousarray(x, dtype=np.float32)
        k, s, p = spec["k"], spec["stride"], spec["pad"]
        oh = (h + 2 * p - k) // s + 1
        ow = (w + 2 * p - k) // s + 1
        out = np.empty((n, spec["out_c"], oh, ow), np.float32)
        st = self.lib.ref_conv2d_ternary(ptr(x, _f32p), n, c, h, w, C.byref(cv), int(nonneg), workers,
                                         ptr(out, _f32p))
        return st, out

    def fully_connected_ternary(self, x, batch, spec, nonneg=True):
        keep: list = []
        cv = make_ndconv(spec, keep)
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.empty((batch, spec["out_c"]), np.float32)
        st = self.lib.ref_fully_connected_ternary(ptr(x, _f32p), batch, C.byref(cv), int(nonneg),
                                                  ptr(out, _f32p))
        return st, out

    def fuse_bn(self, mean, var, gamma, beta, eps):
        arrs = [np.ascontiguousarray(a, np.float32) for a in (mean, var, gamma, beta)]
        c = arrs[0].size
        g = np.empty(c, np.float32)
        b = np.empty(c, np.float32)
        st = self.lib.ref_fuse_bn(*[ptr(a, _f32p) for a in arrs], eps, c, ptr(g, _f32p), ptr(b, _f32p))
        return st, g, b

    def packed_forward(self, x, batch, in_dim, hidden, n_classes, stem_w, stem_b, blocks,
                       cal_gain, cal_bias, head_w, head_b):
        keep: list = []
        arr = (NdConv * len(blocks))(*[make_ndconv(b, keep) for b in blocks])
        a = [np.ascontiguousarray(v, np.float32) if v is not None else None
             for v in (x, stem_w, stem_b, cal_gain, cal_bias, head_w, head_b)]
        out = np.empty((batch, n_classes), np.float32)
        st = self.lib.ref_packed_forward(ptr(a[0], _f32p), batch, in_dim, hidden, n_classes,
                                         ptr(a[1], _f32p), ptr(a[2], _f32p), len(blocks), arr,
                                         ptr(a[3], _f32p), ptr(a[4], _f32p), ptr(a[5], _f32p),
                                         ptr(a[6], _f32p), ptr(out, _f32p))
        return st, out

    def pack_binary(self, v):
        v = np.ascontiguousarray(v, dtype=np.int8)
        w = np.zeros((v.size + 63) // 64, np.uint64)
        f = self.lib.ref_pack_binary
        f.argtypes = [_i8p, _sz, _u64p]
        return f(ptr(v, _i8p), v.size, ptr(w, _u64p)), w

    def binary_dot(self, x, y, n):
        x = np.ascontiguousarray(x, np.uint64)
        y = np.ascontiguousarray(y, np.uint64)
        out = C.c_int64()
        f = self.lib.ref_binary_dot
        f.argtypes = [_u64p, _u64p, _sz, _sz, _i64p]
        st = f(ptr(x, _u64p), ptr(y, _u64p), x.size, n, C.byref(out))
        return st, out.value

    def multibit_dot(self, xp, sx, yp, sy, n):
        xp = np.ascontiguousarray(xp, np.uint64)
        yp = np.ascontiguousarray(yp, np.uint64)
        sx = np.ascontiguousarray(sx, np.float64)
        sy = np.ascontiguousarray(sy, np.float64)
        dp = C.POINTER(C.c_double)
        out = C.c_double()
        f = self.lib.ref_multibit_dot
        f.argtypes = [_u64p, C.c_int, _u64p, C.c_int, dp, dp, _sz, _sz, dp]
        st = f(ptr(xp, _u64p), xp.shape[0], ptr(yp, _u64p), yp.shape[0], sx.ctypes.data_as(dp),
               sy.ctypes.data_as(dp), xp.shape[1], n, C.byref(out))
        return st, out.value

    def save_packed_model(self, path, in_dim, hidden, n_classes, stem_w, stem_b, blocks, cal_gain, cal_bias,
                          head_w, head_b):
        keep: list = []
        arr = (NdConv * len(blocks))(*[make_ndconv(b, keep) for b in blocks])
        a = [np.ascontiguousarray(v, np.float32) if v is not None else None
             for v in (stem_w, stem_b, cal_gain, cal_bias, head_w, head_b)]
        f = self.lib.ref_save_packed_model
        f.argtypes = [C.c_char_p] + [C.c_int] * 3 + [_f32p, _f32p, C.c_int, C.POINTER(NdConv)] + [_f32p] * 4
        return f(path.encode(), in_dim, hidden, n_classes, ptr(a[0], _f32p), ptr(a[1], _f32p), len(blocks), arr,
                 ptr(a[2], _f32p), ptr(a[3], _f32p), ptr(a[4], _f32p), ptr(a[5], _f32p))

    def load_and_forward(self, path, x, batch, max_classes=4096):
        x = np.ascontiguousarray(x, np.float32)
        out = np.empty(batch * max_classes, np.float32)
        ncls = C.c_int()
        f = self.lib.ref_load_and_forward
        f.argtypes = [C.c_char_p, _f32p, C.c_int, _f32p, C.POINTER(C.c_int)]
        st = f(path.encode(), ptr(x, _f32p), batch, ptr(out, _f32p), C.byref(ncls))
        return st, out[: batch * ncls.value].reshape(batch, ncls.value)

    def net_create(self, blocks):
        keep: list = []
        arr = make_ndblocks(blocks, keep)
        h = self.lib.ref_net_create(C.cast(arr, C.c_void_p), len(blocks))
        if not h:
            raise ValueError("reference rejected the network description")
        return h

    def net_run(self, handle, x, n, c, h, w, threads, out_shape=None):
        x = np.ascontiguousarray(x, np.float32)
        out = None if out_shape is None else np.empty(out_shape, np.float32)
        sec = C.c_double()
        st = self.lib.ref_net_run(handle, ptr(x, _f32p), n, c, h, w, threads, ptr(out, _f32p),
                                  C.byref(sec))
        return st, out, sec.value

    def net_destroy(self, handle):
        self.lib.ref_net_destroy(handle)
