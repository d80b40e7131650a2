"""Plain CPU oracle for the sliding-window-sum hot path (arXiv 2305.16513).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2305_16513_b200`` never imports it and
shares no code with it.

This module is argument marshalling (numpy <-> ctypes) around ``oracle.c``;
all arithmetic is in ``oracle.c``, each routine citing the PAPER.md passage it
writes out (Eq. 3, Sec. 2.3, Eq. 4-9, Sec. 2.5, Conclusion).  Pins that tie
the oracle to the paper and to mathematics, not to itself, live in
``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

POOL2D_MAX = 0
POOL2D_AVG = 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2, IEEE, no fast-math) into liboracle.so."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
             "-ffp-contract=off", "-o", tmp, _SRC, "-lm"]
        )
        os.replace(tmp, _SO)
    return _SO


def lib() -> ctypes.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            i64, vp, dp = ctypes.c_int64, ctypes.c_void_p, ctypes.c_double
            L.oracle_out_len.argtypes = [i64, i64, i64]
            L.oracle_out_len.restype = i64
            for name in ("oracle_pool_sum_i32", "oracle_pool_max_i32", "oracle_pool_max_f32"):
                getattr(L, name).argtypes = [vp, i64, i64, i64, i64, vp]
                getattr(L, name).restype = ctypes.c_int
            L.oracle_pool_sum_f32.argtypes = [vp, i64, i64, i64, i64, vp, vp]
            L.oracle_pool_sum_f32.restype = ctypes.c_int
            L.oracle_conv1d_f32.argtypes = [vp, i64, i64, vp, i64, i64, vp, vp]
            L.oracle_conv1d_f32.restype = ctypes.c_int
            L.oracle_pool2d_f32.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64,
                                            ctypes.c_int, vp, vp]
            L.oracle_pool2d_f32.restype = ctypes.c_int
            L.oracle_out_len_ex.argtypes = [i64] * 6
            L.oracle_out_len_ex.restype = i64
            ci = ctypes.c_int
            for name in ("oracle_pool_sum_ex_i32", "oracle_pool_max_ex_i32", "oracle_pool_max_ex_f32",
                         "oracle_pool_min_ex_i32", "oracle_pool_min_ex_f32"):
                getattr(L, name).argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, ci, vp]
                getattr(L, name).restype = ctypes.c_int
            L.oracle_pool_sum_ex_f32.argtypes = [vp, i64, i64, i64, i64, i64, i64, i64, ci, vp, vp]
            L.oracle_pool_sum_ex_f32.restype = ctypes.c_int
            L.oracle_conv1d_ex_f32.argtypes = [vp, i64, i64, vp, i64, i64, i64, i64, i64, ci, vp, vp]
            L.oracle_conv1d_ex_f32.restype = ctypes.c_int
            L.oracle_affine_window.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp, vp]
            L.oracle_affine_window.restype = ctypes.c_int
            L.oracle_gamma_combine.argtypes = [dp, dp, dp, dp, vp, vp]
            L.oracle_gamma_combine.restype = None
            L.oracle_gamma_sequence.argtypes = [vp, vp, i64, vp, vp]
            L.oracle_gamma_sequence.restype = ctypes.c_int
            L.oracle_gamma_dot.argtypes = [vp, vp, i64, vp]
            L.oracle_gamma_dot.restype = dp
            L.oracle_pool_sum_backward_f32.argtypes = [vp, i64, i64, i64, i64, vp, vp]
            L.oracle_pool_max_backward_f32.argtypes = [vp, vp, i64, i64, i64, i64, vp]
            L.oracle_conv1d_backward_input_f32.argtypes = [vp, i64, i64, vp, i64, i64, vp, vp]
            L.oracle_conv1d_backward_filter_f32.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp]
            L.oracle_pool2d_backward_f32.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64,
                                                     ctypes.c_int, vp, vp]
            L.oracle_conv1d_mc_bf16.argtypes = [vp, vp, i64, i64, i64, i64, i64, vp, vp]
            L.oracle_conv1d_mc_bf16.restype = ctypes.c_int
            L.oracle_conv2d_mc_bf16.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, vp]
            L.oracle_conv2d_mc_bf16.restype = ctypes.c_int
            L.oracle_conv1d_mc_backward_input_bf16.argtypes = [vp, vp, i64, i64, i64, i64, i64, vp, vp]
            L.oracle_conv1d_mc_backward_input_bf16.restype = ctypes.c_int
            L.oracle_conv1d_mc_backward_filter_bf16.argtypes = [vp, vp, i64, i64, i64, i64, i64, vp, vp]
            L.oracle_conv1d_mc_backward_filter_bf16.restype = ctypes.c_int
            L.oracle_conv2d_mc_backward_input_bf16.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, vp]
            L.oracle_conv2d_mc_backward_input_bf16.restype = ctypes.c_int
            L.oracle_conv2d_mc_backward_filter_bf16.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, vp]
            L.oracle_conv2d_mc_backward_filter_bf16.restype = ctypes.c_int
            L.oracle_conv2d_f32.argtypes = [vp, i64, i64, i64, vp, i64, i64, i64, i64, vp, vp]
            L.oracle_conv2d_f32.restype = ctypes.c_int
            L.oracle_conv2d_backward_input_f32.argtypes = [vp, i64, i64, i64, vp, i64, i64, i64, i64, vp, vp]
            L.oracle_conv2d_backward_input_f32.restype = ctypes.c_int
            L.oracle_conv2d_backward_filter_f32.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, vp]
            L.oracle_conv2d_backward_filter_f32.restype = ctypes.c_int
            for n in ("oracle_pool_sum_backward_f32", "oracle_pool_max_backward_f32",
                      "oracle_conv1d_backward_input_f32", "oracle_conv1d_backward_filter_f32",
                      "oracle_pool2d_backward_f32"):
                getattr(L, n).restype = ctypes.c_int
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _rows(x: np.ndarray):
    x = np.ascontiguousarray(x)
    if x.ndim == 1:
        return x, x.shape[0], 1
    assert x.ndim == 2
    return x, x.shape[1], x.shape[0]


def out_len(N: int, w: int, s: int = 1) -> int:
    return int(lib().oracle_out_len(N, w, s))


def _check(rc: int):
    if rc != 0:
        raise ValueError("oracle rejected its arguments")


def pool_sum(x: np.ndarray, w: int, s: int = 1):
    """Eq. 3 with + .  int32 -> exact int64 sums; float32 -> (double sums, absmag)."""
    x, N, B = _rows(x)
    L = out_len(N, w, s)
    if L < 0:
        raise ValueError("window exceeds input")
    if x.dtype == np.int32:
        y = np.empty((B, L), np.int64)
        _check(lib().oracle_pool_sum_i32(_p(x), N, B, w, s, _p(y)))
        return y if x.ndim == 2 else y[0]
    assert x.dtype == np.float32
    y = np.empty((B, L), np.float64)
    m = np.empty((B, L), np.float64)
    _check(lib().oracle_pool_sum_f32(_p(x), N, B, w, s, _p(y), _p(m)))
    return (y, m) if x.ndim == 2 else (y[0], m[0])


def pool_max(x: np.ndarray, w: int, s: int = 1) -> np.ndarray:
    """Eq. 3 with max (Sec. 2.3); exact, same dtype as x."""
    x, N, B = _rows(x)
    L = out_len(N, w, s)
    if L < 0:
        raise ValueError("window exceeds input")
    y = np.empty((B, L), x.dtype)
    fn = {np.dtype(np.int32): lib().oracle_pool_max_i32,
          np.dtype(np.float32): lib().oracle_pool_max_f32}[x.dtype]
    _check(fn(_p(x), N, B, w, s, _p(y)))
    return y if x.ndim == 2 else y[0]


def conv1d(x: np.ndarray, f: np.ndarray, s: int = 1):
    """Sec. 2.5 sliding dot product (cross-correlation); returns (y double, absmag)."""
    x, N, B = _rows(x)
    f = np.ascontiguousarray(f, np.float32)
    k = f.shape[0]
    L = out_len(N, k, s)
    if L < 0:
        raise ValueError("window exceeds input")
    y = np.empty((B, L), np.float64)
    m = np.empty((B, L), np.float64)
    _check(lib().oracle_conv1d_f32(_p(x), N, B, _p(f), k, s, _p(y), _p(m)))
    return (y, m) if x.ndim == 2 else (y[0], m[0])


def pool2d(x: np.ndarray, kh: int, kw: int, sh: int, sw: int, mode: int):
    """Direct 2-D window pooling on [planes, H, W]; returns (y double, absmag)."""
    x = np.ascontiguousarray(x, np.float32)
    P, H, W = x.shape
    OH, OW = out_len(H, kh, sh), out_len(W, kw, sw)
    if OH < 0 or OW < 0:
        raise ValueError("window exceeds input")
    y = np.empty((P, OH, OW), np.float64)
    m = np.empty((P, OH, OW), np.float64)
    _check(lib().oracle_pool2d_f32(_p(x), P, H, W, kh, kw, sh, sw, mode, _p(y), _p(m)))
    return y, m


def out_len_ex(N: int, w: int, s: int = 1, d: int = 1, pl: int = 0, pr: int = 0) -> int:
    return int(lib().oracle_out_len_ex(N, w, s, d, pl, pr))


def _ex_len(N, w, s, d, pl, pr):
    L = out_len_ex(N, w, s, d, pl, pr)
    if L < 0:
        raise ValueError("invalid window spec")
    return L


PAD_MODES = {"zeros": 0, "reflect": 1, "circular": 2, "replicate": 3}


def _mode(mode) -> int:
    return PAD_MODES[mode] if isinstance(mode, str) else int(mode)


def pool_sum_ex(x: np.ndarray, w: int, s: int = 1, d: int = 1, pl: int = 0, pr: int = 0, mode="zeros"):
    """Padded, dilated sliding sum (NEXT #1).  int32 -> int64; float32 -> (double, absmag)."""
    x, N, B = _rows(x)
    L = _ex_len(N, w, s, d, pl, pr)
    if x.dtype == np.int32:
        y = np.empty((B, L), np.int64)
        _check(lib().oracle_pool_sum_ex_i32(_p(x), N, B, w, s, d, pl, pr, _mode(mode), _p(y)))
        return y if x.ndim == 2 else y[0]
    y = np.empty((B, L), np.float64)
    m = np.empty((B, L), np.float64)
    _check(lib().oracle_pool_sum_ex_f32(_p(x), N, B, w, s, d, pl, pr, _mode(mode), _p(y), _p(m)))
    return (y, m) if x.ndim == 2 else (y[0], m[0])


def _extremum_ex(name, x, w, s, d, pl, pr, mode):
    x, N, B = _rows(x)
    L = _ex_len(N, w, s, d, pl, pr)
    y = np.empty((B, L), x.dtype)
    fn = {np.dtype(np.int32): getattr(lib(), f"oracle_pool_{name}_ex_i32"),
          np.dtype(np.float32): getattr(lib(), f"oracle_pool_{name}_ex_f32")}[x.dtype]
    _check(fn(_p(x), N, B, w, s, d, pl, pr, _mode(mode), _p(y)))
    return y if x.ndim == 2 else y[0]


def pool_max_ex(x: np.ndarray, w: int, s: int = 1, d: int = 1, pl: int = 0, pr: int = 0, mode="zeros"):
    return _extremum_ex("max", x, w, s, d, pl, pr, mode)


def pool_min_ex(x: np.ndarray, w: int, s: int = 1, d: int = 1, pl: int = 0, pr: int = 0, mode="zeros"):
    """Sliding min (Sec. 2.3's other extremum), same dtype as x."""
    return _extremum_ex("min", x, w, s, d, pl, pr, mode)


def pool_min(x: np.ndarray, w: int, s: int = 1) -> np.ndarray:
    """Valid-padding sliding min."""
    return pool_min_ex(x, w, s)


def conv1d_ex(x: np.ndarray, f: np.ndarray, s: int = 1, d: int = 1, pl: int = 0, pr: int = 0, mode="zeros"):
    x, N, B = _rows(x)
    f = np.ascontiguousarray(f, np.float32)
    k = f.shape[0]
    L = _ex_len(N, k, s, d, pl, pr)
    y = np.empty((B, L), np.float64)
    m = np.empty((B, L), np.float64)
    _check(lib().oracle_conv1d_ex_f32(_p(x), N, B, _p(f), k, s, d, pl, pr, _mode(mode), _p(y), _p(m)))
    return (y, m) if x.ndim == 2 else (y[0], m[0])


def affine_window(u: np.ndarray, v: np.ndarray, w: int, s: int = 1):
    """Sliding window of gamma pairs (Eq. 3 with the Eq. 8 operator).
    Returns (U, V, magV) in double, shaped like the outputs."""
    u, N, B = _rows(np.ascontiguousarray(u, np.float32))
    v = np.ascontiguousarray(v, np.float32).reshape(u.shape)
    L = out_len(N, w, s)
    if L < 0:
        raise ValueError("window exceeds input")
    U = np.empty((B, L))
    V = np.empty((B, L))
    M = np.empty((B, L))
    _check(lib().oracle_affine_window(_p(u), _p(v), N, B, w, s, _p(U), _p(V), _p(M)))
    if u.ndim == 1:
        return U[0], V[0], M[0]
    return U, V, M


def gamma_combine(gi, gj):
    """Eq. 8."""
    u = ctypes.c_double()
    v = ctypes.c_double()
    lib().oracle_gamma_combine(gi[0], gi[1], gj[0], gj[1], ctypes.byref(u), ctypes.byref(v))
    return (u.value, v.value)


def gamma_sequence(a: np.ndarray, b: np.ndarray):
    """Eq. 5 + Eq. 7: the M+1 pairs (u, v)."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    M = a.shape[0]
    u = np.empty(M + 1)
    v = np.empty(M + 1)
    _check(lib().oracle_gamma_sequence(_p(a), _p(b), M, _p(u), _p(v)))
    return u, v


def gamma_dot(a: np.ndarray, b: np.ndarray):
    """Eq. 9: returns (v(delta_M) = dot product, u(delta_M))."""
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    u = ctypes.c_double()
    v = lib().oracle_gamma_dot(_p(a), _p(b), a.shape[0], ctypes.byref(u))
    return v, u.value


# ---------------------------------------------------------------- backward passes
# Vector-Jacobian products of the forward definitions.
# dy has the forward output's shape ([B, L]); dx the input's ([B, N]).

def _bwd_rows(dy: np.ndarray, N: int, w: int, s: int):
    dy = np.ascontiguousarray(dy, np.float32)
    squeeze = dy.ndim == 1
    dy2 = dy.reshape(1, -1) if squeeze else dy
    B = dy2.shape[0]
    L = out_len(N, w, s)
    if L < 0 or dy2.shape[1] != L:
        raise ValueError("dy does not match the forward output length")
    return dy2, B, squeeze


def pool_sum_backward(dy: np.ndarray, N: int, w: int, s: int = 1):
    """dx of Eq. 3 with + : dx_t = sum of dy_i over the windows i containing t; (dx, absmag)."""
    dy2, B, sq = _bwd_rows(dy, N, w, s)
    dx = np.empty((B, N), np.float64)
    m = np.empty((B, N), np.float64)
    _check(lib().oracle_pool_sum_backward_f32(_p(dy2), N, B, w, s, _p(dx), _p(m)))
    return (dx[0], m[0]) if sq else (dx, m)


def pool_max_backward(x: np.ndarray, dy: np.ndarray, w: int, s: int = 1) -> np.ndarray:
    """dx of Eq. 3 with max: each window's dy goes to its first maximum (reading R16)."""
    x, N, B = _rows(np.asarray(x, np.float32))
    dy2, B2, sq = _bwd_rows(dy, N, w, s)
    assert B2 == B
    dx = np.empty((B, N), np.float64)
    _check(lib().oracle_pool_max_backward_f32(_p(x), _p(dy2), N, B, w, s, _p(dx)))
    return dx[0] if sq else dx


def conv1d_backward_input(dy: np.ndarray, f: np.ndarray, N: int, s: int = 1):
    """dx of the sliding dot product: dx_t = sum_{is+j=t} f_j dy_i; (dx, absmag)."""
    f = np.ascontiguousarray(f, np.float32)
    dy2, B, sq = _bwd_rows(dy, N, f.shape[0], s)
    dx = np.empty((B, N), np.float64)
    m = np.empty((B, N), np.float64)
    _check(lib().oracle_conv1d_backward_input_f32(_p(dy2), N, B, _p(f), f.shape[0], s, _p(dx), _p(m)))
    return (dx[0], m[0]) if sq else (dx, m)


def conv1d_backward_filter(x: np.ndarray, dy: np.ndarray, k: int, s: int = 1):
    """df of the sliding dot product: df_j = sum_b sum_i dy_i x_{is+j}; (df, absmag)."""
    x, N, B = _rows(np.asarray(x, np.float32))
    dy2, B2, _ = _bwd_rows(dy, N, k, s)
    assert B2 == B
    df = np.empty(k, np.float64)
    m = np.empty(k, np.float64)
    _check(lib().oracle_conv1d_backward_filter_f32(_p(x), _p(dy2), N, B, k, s, _p(df), _p(m)))
    return df, m


def pool2d_backward(x, dy: np.ndarray, H: int, W: int, kh: int, kw: int, sh: int, sw: int, mode: int):
    """dx of the direct 2-D pooling (mode POOL2D_MAX / POOL2D_AVG); (dx, absmag)."""
    dy = np.ascontiguousarray(dy, np.float32)
    P = dy.shape[0]
    if mode == 0:
        x = np.ascontiguousarray(x, np.float32)
        xp = _p(x)
    else:
        xp = None
    dx = np.empty((P, H, W), np.float64)
    m = np.empty((P, H, W), np.float64)
    _check(lib().oracle_pool2d_backward_f32(xp, _p(dy), P, H, W, kh, kw, sh, sw, mode, _p(dx), _p(m)))
    return dx, m


def conv2d(x: np.ndarray, f: np.ndarray, sh: int = 1, sw: int = 1):
    """2-D single-channel sliding dot product (cross-correlation) of [planes, H, W] with f [kh, kw];
    returns (y double [planes, OH, OW], absmag)."""
    x = np.ascontiguousarray(x, np.float32)
    f = np.ascontiguousarray(f, np.float32)
    P, H, W = x.shape
    kh, kw = f.shape
    OH, OW = out_len(H, kh, sh), out_len(W, kw, sw)
    if OH < 0 or OW < 0:
        raise ValueError("window exceeds input")
    y = np.empty((P, OH, OW), np.float64)
    m = np.empty((P, OH, OW), np.float64)
    _check(lib().oracle_conv2d_f32(_p(x), P, H, W, _p(f), kh, kw, sh, sw, _p(y), _p(m)))
    return y, m


def conv2d_backward_input(dy: np.ndarray, f: np.ndarray, H: int, W: int, sh: int = 1, sw: int = 1):
    """dx of the 2-D sliding dot product (reading R21): [planes, H, W]; (dx, absmag)."""
    dy = np.ascontiguousarray(dy, np.float32)
    f = np.ascontiguousarray(f, np.float32)
    P = dy.shape[0]
    kh, kw = f.shape
    assert dy.shape[1:] == (out_len(H, kh, sh), out_len(W, kw, sw))
    dx = np.empty((P, H, W), np.float64)
    m = np.empty((P, H, W), np.float64)
    _check(lib().oracle_conv2d_backward_input_f32(_p(dy), P, H, W, _p(f), kh, kw, sh, sw, _p(dx), _p(m)))
    return dx, m


def conv2d_backward_filter(x: np.ndarray, dy: np.ndarray, kh: int, kw: int, sh: int = 1, sw: int = 1):
    """df [kh, kw] of the 2-D sliding dot product (reading R21); (df, absmag)."""
    x = np.ascontiguousarray(x, np.float32)
    dy = np.ascontiguousarray(dy, np.float32)
    P, H, W = x.shape
    assert dy.shape == (P, out_len(H, kh, sh), out_len(W, kw, sw))
    df = np.empty((kh, kw), np.float64)
    m = np.empty((kh, kw), np.float64)
    _check(lib().oracle_conv2d_backward_filter_f32(_p(x), _p(dy), P, H, W, kh, kw, sh, sw, _p(df), _p(m)))
    return df, m


def to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bfloat16 bit patterns (uint16)."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f32(h: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(h, np.uint16).astype(np.uint32) << 16).view(np.float32)


def conv1d_mc(x_bf16: np.ndarray, w_bf16: np.ndarray):
    """Multi-channel conv1d, channels-last: x [B, N, Cin] and w [Cout, Cin, k] as bf16 bit
    patterns (uint16); returns (y double [B, L, Cout], absmag)."""
    x = np.ascontiguousarray(x_bf16, np.uint16)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    B, N, cin = x.shape
    cout, cin2, k = w.shape
    assert cin2 == cin
    L = N - k + 1
    if L < 1:
        raise ValueError("window exceeds input")
    y = np.empty((B, L, cout), np.float64)
    m = np.empty((B, L, cout), np.float64)
    _check(lib().oracle_conv1d_mc_bf16(_p(x), _p(w), B, N, cin, cout, k, _p(y), _p(m)))
    return y, m


def conv2d_mc(x_bf16: np.ndarray, w_bf16: np.ndarray):
    """Multi-channel 2-D conv, NHWC: x [B, H, W, Cin] and w [Cout, Cin, kh, kw] as bf16 bit
    patterns (uint16); valid padding, stride 1; returns (y double [B, OH, OW, Cout], absmag)."""
    x = np.ascontiguousarray(x_bf16, np.uint16)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    B, H, W, cin = x.shape
    cout, cin2, kh, kw = w.shape
    assert cin2 == cin
    OH, OW = H - kh + 1, W - kw + 1
    if OH < 1 or OW < 1:
        raise ValueError("window exceeds input")
    y = np.empty((B, OH, OW, cout), np.float64)
    m = np.empty((B, OH, OW, cout), np.float64)
    _check(lib().oracle_conv2d_mc_bf16(_p(x), _p(w), B, H, W, cin, cout, kh, kw, _p(y), _p(m)))
    return y, m


def conv1d_mc_backward_input(dy_bf16: np.ndarray, w_bf16: np.ndarray, N: int):
    """dx [B, N, Cin] (double) of the multi-channel conv1d for bf16 dy [B, N-k+1, Cout] and
    w [Cout, Cin, k] (reading R23); returns (dx, absmag)."""
    dy = np.ascontiguousarray(dy_bf16, np.uint16)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    B, L, cout = dy.shape
    cout2, cin, k = w.shape
    assert cout2 == cout and L == N - k + 1
    dx = np.empty((B, N, cin), np.float64)
    m = np.empty((B, N, cin), np.float64)
    _check(lib().oracle_conv1d_mc_backward_input_bf16(_p(dy), _p(w), B, N, cin, cout, k, _p(dx), _p(m)))
    return dx, m


def conv1d_mc_backward_filter(dy_bf16: np.ndarray, x_bf16: np.ndarray, k: int):
    """dw [Cout, Cin, k] (double) of the multi-channel conv1d for bf16 dy [B, N-k+1, Cout] and
    x [B, N, Cin] (reading R25); returns (dw, absmag)."""
    dy = np.ascontiguousarray(dy_bf16, np.uint16)
    x = np.ascontiguousarray(x_bf16, np.uint16)
    B, L, cout = dy.shape
    B2, N, cin = x.shape
    assert B2 == B and L == N - k + 1
    dw = np.empty((cout, cin, k), np.float64)
    m = np.empty((cout, cin, k), np.float64)
    _check(lib().oracle_conv1d_mc_backward_filter_bf16(_p(dy), _p(x), B, N, cin, cout, k, _p(dw), _p(m)))
    return dw, m


def conv2d_mc_backward_input(dy_bf16: np.ndarray, w_bf16: np.ndarray, H: int, W: int):
    """dx [B, H, W, Cin] (double) of the multi-channel 2-D conv for bf16 dy [B, H-kh+1, W-kw+1, Cout]
    and w [Cout, Cin, kh, kw] (reading R26); returns (dx, absmag)."""
    dy = np.ascontiguousarray(dy_bf16, np.uint16)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    B, OH, OW, cout = dy.shape
    cout2, cin, kh, kw = w.shape
    assert cout2 == cout and OH == H - kh + 1 and OW == W - kw + 1
    dx = np.empty((B, H, W, cin), np.float64)
    m = np.empty((B, H, W, cin), np.float64)
    _check(lib().oracle_conv2d_mc_backward_input_bf16(_p(dy), _p(w), B, H, W, cin, cout, kh, kw, _p(dx), _p(m)))
    return dx, m


def conv2d_mc_backward_filter(dy_bf16: np.ndarray, x_bf16: np.ndarray, kh: int, kw: int):
    """dw [Cout, Cin, kh, kw] (double) of the multi-channel 2-D conv for bf16 dy [B, H-kh+1, W-kw+1, Cout]
    and x [B, H, W, Cin] (reading R27); returns (dw, absmag)."""
    dy = np.ascontiguousarray(dy_bf16, np.uint16)
    x = np.ascontiguousarray(x_bf16, np.uint16)
    B, OH, OW, cout = dy.shape
    B2, H, W, cin = x.shape
    assert B2 == B and OH == H - kh + 1 and OW == W - kw + 1
    dw = np.empty((cout, cin, kh, kw), np.float64)
    m = np.empty((cout, cin, kh, kw), np.float64)
    _check(lib().oracle_conv2d_mc_backward_filter_bf16(_p(dy), _p(x), B, H, W, cin, cout, kh, kw, _p(dw), _p(m)))
    return dw, m
