"""B200-native sliding-window-sum library (hot path of arXiv 2305.16513).

Thin Python binding over the C ABI in ``include/ss.h`` (``libss.so``, built
in-tree from ``csrc/`` for sm_100a).  This module only marshals arguments:
every step of the computation runs in the CUDA kernels.  There is no CPU
fallback -- importing this package without the built library raises.

Low-level names mirror the ABI (``ss_pool_sum``, ``ss_pool_max``,
``ss_conv1d``, ``ss_pool2d``, ``ss_out_len``...) and take raw device pointers;
the tensor helpers (``pool_sum``, ``pool_max``, ``conv1d``, ``pool2d``) take
CUDA torch tensors, allocate the output with torch, and launch on the current
torch stream.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libss.so")

SS_F32 = 0
SS_I32 = 1
SS_POOL_MAX = 0
SS_POOL_AVG = 1
SS_PAD_ZEROS = 0
SS_PAD_REFLECT = 1
SS_PAD_CIRCULAR = 2
SS_PAD_REPLICATE = 3
PAD_MODES = {"zeros": SS_PAD_ZEROS, "reflect": SS_PAD_REFLECT, "circular": SS_PAD_CIRCULAR,
             "replicate": SS_PAD_REPLICATE}
SS_OK = 0
SS_ERR_NULL = 1
SS_ERR_BAD_SIZE = 2
SS_ERR_WINDOW_EXCEEDS_INPUT = 3
SS_ERR_UNSUPPORTED = 4
SS_ERR_CUDA = 5
SS_ERR_OVERLAP = 6
SS_K_MAX = 1024
SS_AFFINE_W_MAX = 65536

EXPORTED = ("ss_abi_version", "ss_out_len", "ss_pool_sum", "ss_pool_max", "ss_pool_min", "ss_conv1d",
            "ss_pool2d", "ss_status_string", "ss_last_error", "ss_launch_count",
            "ss_out_len_ex", "ss_pool_sum_ex", "ss_pool_max_ex", "ss_pool_min_ex", "ss_conv1d_ex",
            "ss_affine_window", "ss_pool_sum_backward", "ss_pool_max_backward",
            "ss_conv1d_backward_input", "ss_conv1d_backward_filter_workspace", "ss_conv1d_backward_filter",
            "ss_pool2d_backward", "ss_conv2d", "ss_conv2d_backward_input", "ss_conv2d_backward_filter_workspace",
            "ss_conv2d_backward_filter", "ss_conv1d_mc", "ss_conv2d_mc", "ss_conv1d_mc_backward_input",
            "ss_conv1d_mc_backward_filter_workspace", "ss_conv1d_mc_backward_filter",
            "ss_conv2d_mc_backward_input", "ss_conv2d_mc_backward_filter_workspace", "ss_conv2d_mc_backward_filter")


class SSError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{ss_status_string(status)} -- {detail}")
        self.status = status


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i64, vp, i32 = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
    L.ss_abi_version.argtypes = []
    L.ss_abi_version.restype = i32
    L.ss_out_len.argtypes = [i64, i64, i64]
    L.ss_out_len.restype = i64
    for n in ("ss_pool_sum", "ss_pool_max", "ss_pool_min"):
        getattr(L, n).argtypes = [vp, vp, i64, i64, i64, i64, i32, vp]
        getattr(L, n).restype = i32
    L.ss_conv1d.argtypes = [vp, vp, i64, i64, ctypes.POINTER(ctypes.c_float), i64, i64, i32, vp]
    L.ss_conv1d.restype = i32
    L.ss_pool2d.argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, i32, i32, vp]
    L.ss_pool2d.restype = i32
    L.ss_out_len_ex.argtypes = [i64] * 6
    L.ss_out_len_ex.restype = i64
    for n in ("ss_pool_sum_ex", "ss_pool_max_ex", "ss_pool_min_ex"):
        getattr(L, n).argtypes = [vp, vp, i64, i64, i64, i64, i64, i64, i64, i32, i32, vp]
        getattr(L, n).restype = i32
    L.ss_conv1d_ex.argtypes = [vp, vp, i64, i64, ctypes.POINTER(ctypes.c_float), i64, i64, i64, i64, i64,
                               i32, i32, vp]
    L.ss_conv1d_ex.restype = i32
    L.ss_affine_window.argtypes = [vp, vp, vp, vp, i64, i64, i64, i64, vp]
    L.ss_affine_window.restype = i32
    L.ss_pool_sum_backward.argtypes = [vp, vp, i64, i64, i64, i64, i32, vp]
    L.ss_pool_sum_backward.restype = i32
    L.ss_pool_max_backward.argtypes = [vp, vp, vp, i64, i64, i64, i64, i32, vp]
    L.ss_pool_max_backward.restype = i32
    L.ss_conv1d_backward_input.argtypes = [vp, vp, i64, i64, ctypes.POINTER(ctypes.c_float), i64, i64, i32, vp]
    L.ss_conv1d_backward_input.restype = i32
    L.ss_conv1d_backward_filter_workspace.argtypes = [i64]
    L.ss_conv1d_backward_filter_workspace.restype = ctypes.c_size_t
    L.ss_conv1d_backward_filter.argtypes = [vp, vp, vp, i64, i64, i64, i64, vp, ctypes.c_size_t, vp]
    L.ss_conv1d_backward_filter.restype = i32
    L.ss_pool2d_backward.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i64, i32, i32, vp]
    L.ss_pool2d_backward.restype = i32
    L.ss_conv2d.argtypes = [vp, vp, i64, i64, i64, ctypes.POINTER(ctypes.c_float), i64, i64, i64, i64, i32, vp]
    L.ss_conv1d_mc.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, vp]
    L.ss_conv1d_mc.restype = i32
    L.ss_conv2d_mc.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i64, vp]
    L.ss_conv2d_mc.restype = i32
    L.ss_conv1d_mc_backward_input.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, vp]
    L.ss_conv1d_mc_backward_input.restype = i32
    L.ss_conv2d_mc_backward_input.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i64, vp]
    L.ss_conv2d_mc_backward_input.restype = i32
    L.ss_conv2d_mc_backward_filter_workspace.argtypes = [i64, i64, i64, i64]
    L.ss_conv2d_mc_backward_filter_workspace.restype = ctypes.c_size_t
    L.ss_conv2d_mc_backward_filter.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, ctypes.c_size_t, vp]
    L.ss_conv2d_mc_backward_filter.restype = i32
    L.ss_conv1d_mc_backward_filter_workspace.argtypes = [i64, i64, i64]
    L.ss_conv1d_mc_backward_filter_workspace.restype = ctypes.c_size_t
    L.ss_conv1d_mc_backward_filter.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, vp, ctypes.c_size_t, vp]
    L.ss_conv1d_mc_backward_filter.restype = i32
    L.ss_conv2d.restype = i32
    L.ss_conv2d_backward_input.argtypes = [vp, vp, i64, i64, i64, ctypes.POINTER(ctypes.c_float), i64, i64, i64, i64,
                                           i32, vp]
    L.ss_conv2d_backward_input.restype = i32
    L.ss_conv2d_backward_filter_workspace.argtypes = [i64, i64]
    L.ss_conv2d_backward_filter_workspace.restype = ctypes.c_size_t
    L.ss_conv2d_backward_filter.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, ctypes.c_size_t, vp]
    L.ss_conv2d_backward_filter.restype = i32
    L.ss_status_string.argtypes = [i32]
    L.ss_status_string.restype = ctypes.c_char_p
    L.ss_last_error.argtypes = []
    L.ss_last_error.restype = ctypes.c_char_p
    L.ss_launch_count.argtypes = []
    L.ss_launch_count.restype = ctypes.c_uint64
    return L


_lib = _load()
lib = _lib


# ------------------------------------------------------------ raw C-ABI names
def ss_abi_version() -> int:
    return _lib.ss_abi_version()


def ss_out_len(N: int, w: int, stride: int = 1) -> int:
    return int(_lib.ss_out_len(N, w, stride))


def ss_status_string(s: int) -> str:
    return _lib.ss_status_string(s).decode()


def ss_last_error() -> str:
    return _lib.ss_last_error().decode()


def ss_launch_count() -> int:
    return int(_lib.ss_launch_count())


def ss_pool_sum(x_ptr: int, y_ptr: int, N: int, batch: int, w: int, stride: int, dtype: int,
                stream: int = 0) -> int:
    return _lib.ss_pool_sum(x_ptr, y_ptr, N, batch, w, stride, dtype, stream)


def ss_pool_max(x_ptr: int, y_ptr: int, N: int, batch: int, w: int, stride: int, dtype: int,
                stream: int = 0) -> int:
    return _lib.ss_pool_max(x_ptr, y_ptr, N, batch, w, stride, dtype, stream)


def ss_pool_min(x_ptr: int, y_ptr: int, N: int, batch: int, w: int, stride: int, dtype: int,
                stream: int = 0) -> int:
    return _lib.ss_pool_min(x_ptr, y_ptr, N, batch, w, stride, dtype, stream)


def ss_conv1d(x_ptr: int, y_ptr: int, N: int, batch: int, filter_host, k: int, stride: int,
              dtype: int = SS_F32, stream: int = 0) -> int:
    if filter_host is None:
        fp = None
    else:
        fp = (ctypes.c_float * len(filter_host))(*[float(v) for v in filter_host])
    return _lib.ss_conv1d(x_ptr, y_ptr, N, batch, fp, k, stride, dtype, stream)


def ss_pool2d(x_ptr: int, y_ptr: int, planes: int, H: int, W: int, kh: int, kw: int, sh: int,
              sw: int, mode: int, dtype: int = SS_F32, stream: int = 0) -> int:
    return _lib.ss_pool2d(x_ptr, y_ptr, planes, H, W, kh, kw, sh, sw, mode, dtype, stream)


def ss_out_len_ex(N: int, w: int, stride: int = 1, dilation: int = 1, pad_left: int = 0,
                  pad_right: int = 0) -> int:
    return int(_lib.ss_out_len_ex(N, w, stride, dilation, pad_left, pad_right))


def ss_pool_sum_ex(x_ptr, y_ptr, N, batch, w, stride, dilation, pad_left, pad_right, pad_mode, dtype,
                   stream=0) -> int:
    return _lib.ss_pool_sum_ex(x_ptr, y_ptr, N, batch, w, stride, dilation, pad_left, pad_right, pad_mode, dtype,
                               stream)


def ss_pool_max_ex(x_ptr, y_ptr, N, batch, w, stride, dilation, pad_left, pad_right, pad_mode, dtype,
                   stream=0) -> int:
    return _lib.ss_pool_max_ex(x_ptr, y_ptr, N, batch, w, stride, dilation, pad_left, pad_right, pad_mode, dtype,
                               stream)


def ss_pool_min_ex(x_ptr, y_ptr, N, batch, w, stride, dilation, pad_left, pad_right, pad_mode, dtype,
                   stream=0) -> int:
    return _lib.ss_pool_min_ex(x_ptr, y_ptr, N, batch, w, stride, dilation, pad_left, pad_right, pad_mode, dtype,
                               stream)


def ss_conv1d_ex(x_ptr, y_ptr, N, batch, filter_host, k, stride, dilation, pad_left, pad_right, pad_mode,
                 dtype=SS_F32, stream=0) -> int:
    fp = None if filter_host is None else (ctypes.c_float * len(filter_host))(*[float(v) for v in filter_host])
    return _lib.ss_conv1d_ex(x_ptr, y_ptr, N, batch, fp, k, stride, dilation, pad_left, pad_right, pad_mode, dtype,
                             stream)


def ss_affine_window(u_ptr, v_ptr, U_ptr, V_ptr, N, batch, w, stride=1, stream=0) -> int:
    return _lib.ss_affine_window(u_ptr, v_ptr, U_ptr, V_ptr, N, batch, w, stride, stream)


def ss_pool_sum_backward(dy_ptr, dx_ptr, N, batch, w, stride, dtype, stream=0) -> int:
    return _lib.ss_pool_sum_backward(dy_ptr, dx_ptr, N, batch, w, stride, dtype, stream)


def ss_pool_max_backward(x_ptr, dy_ptr, dx_ptr, N, batch, w, stride, dtype=SS_F32, stream=0) -> int:
    return _lib.ss_pool_max_backward(x_ptr, dy_ptr, dx_ptr, N, batch, w, stride, dtype, stream)


def ss_conv1d_backward_input(dy_ptr, dx_ptr, N, batch, filter_host, k, stride, dtype=SS_F32, stream=0) -> int:
    fp = None if filter_host is None else (ctypes.c_float * len(filter_host))(*[float(v) for v in filter_host])
    return _lib.ss_conv1d_backward_input(dy_ptr, dx_ptr, N, batch, fp, k, stride, dtype, stream)


def ss_conv1d_backward_filter_workspace(k: int) -> int:
    return int(_lib.ss_conv1d_backward_filter_workspace(k))


def ss_conv1d_backward_filter(x_ptr, dy_ptr, df_ptr, N, batch, k, stride, ws_ptr, ws_bytes, stream=0) -> int:
    return _lib.ss_conv1d_backward_filter(x_ptr, dy_ptr, df_ptr, N, batch, k, stride, ws_ptr, ws_bytes, stream)


def ss_pool2d_backward(x_ptr, dy_ptr, dx_ptr, planes, H, W, kh, kw, sh, sw, mode, dtype=SS_F32, stream=0) -> int:
    return _lib.ss_pool2d_backward(x_ptr, dy_ptr, dx_ptr, planes, H, W, kh, kw, sh, sw, mode, dtype, stream)


def ss_conv2d(x_ptr, y_ptr, planes, H, W, filter_host, kh, kw, sh=1, sw=1, dtype=SS_F32, stream=0) -> int:
    fp = None if filter_host is None else (ctypes.c_float * len(filter_host))(*[float(v) for v in filter_host])
    return _lib.ss_conv2d(x_ptr, y_ptr, planes, H, W, fp, kh, kw, sh, sw, dtype, stream)


def ss_conv2d_backward_input(dy_ptr, dx_ptr, planes, H, W, filter_host, kh, kw, sh=1, sw=1, dtype=SS_F32,
                             stream=0) -> int:
    fp = None if filter_host is None else (ctypes.c_float * len(filter_host))(*[float(v) for v in filter_host])
    return _lib.ss_conv2d_backward_input(dy_ptr, dx_ptr, planes, H, W, fp, kh, kw, sh, sw, dtype, stream)


def ss_conv2d_backward_filter_workspace(kh: int, kw: int) -> int:
    return int(_lib.ss_conv2d_backward_filter_workspace(kh, kw))


def ss_conv2d_backward_filter(x_ptr, dy_ptr, df_ptr, planes, H, W, kh, kw, sh, sw, ws_ptr, ws_bytes, stream=0) -> int:
    return _lib.ss_conv2d_backward_filter(x_ptr, dy_ptr, df_ptr, planes, H, W, kh, kw, sh, sw, ws_ptr, ws_bytes,
                                          stream)


def ss_conv1d_mc(x_ptr, w_ptr, y_ptr, batch, N, cin, cout, k, stream=0) -> int:
    return _lib.ss_conv1d_mc(x_ptr, w_ptr, y_ptr, batch, N, cin, cout, k, stream)


def ss_conv2d_mc(x_ptr, w_ptr, y_ptr, batch, H, W, cin, cout, kh, kw, stream=0) -> int:
    return _lib.ss_conv2d_mc(x_ptr, w_ptr, y_ptr, batch, H, W, cin, cout, kh, kw, stream)


def ss_conv1d_mc_backward_input(dy_ptr, w_ptr, dx_ptr, batch, N, cin, cout, k, stream=0) -> int:
    return _lib.ss_conv1d_mc_backward_input(dy_ptr, w_ptr, dx_ptr, batch, N, cin, cout, k, stream)


def ss_conv2d_mc_backward_input(dy_ptr, w_ptr, dx_ptr, batch, H, W, cin, cout, kh, kw, stream=0) -> int:
    return _lib.ss_conv2d_mc_backward_input(dy_ptr, w_ptr, dx_ptr, batch, H, W, cin, cout, kh, kw, stream)


def ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw) -> int:
    return _lib.ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw)


def ss_conv2d_mc_backward_filter(dy_ptr, x_ptr, dw_ptr, batch, H, W, cin, cout, kh, kw, ws_ptr, ws_bytes,
                                 stream=0) -> int:
    return _lib.ss_conv2d_mc_backward_filter(dy_ptr, x_ptr, dw_ptr, batch, H, W, cin, cout, kh, kw, ws_ptr, ws_bytes,
                                             stream)


def ss_conv1d_mc_backward_filter_workspace(cin, cout, k) -> int:
    return _lib.ss_conv1d_mc_backward_filter_workspace(cin, cout, k)


def ss_conv1d_mc_backward_filter(dy_ptr, x_ptr, dw_ptr, batch, N, cin, cout, k, ws_ptr, ws_bytes, stream=0) -> int:
    return _lib.ss_conv1d_mc_backward_filter(dy_ptr, x_ptr, dw_ptr, batch, N, cin, cout, k, ws_ptr, ws_bytes, stream)


def check(status: int) -> None:
    if status != SS_OK:
        raise SSError(status, ss_last_error())


# ------------------------------------------------------------ tensor helpers
def _torch():
    import torch
    return torch


def _dtype_code(t) -> int:
    torch = _torch()
    if t.dtype == torch.float32:
        return SS_F32
    if t.dtype == torch.int32:
        return SS_I32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _stream(stream) -> int:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _dev(t, name, dtype=None, shape=None, device=None):
    """Argument check of a device tensor: CUDA, contiguous, and (if given) dtype,
    shape and device.  The kernels trust the sizes they are given, so a wrong
    tensor here would read or write out of bounds."""
    if not getattr(t, "is_cuda", False):
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if dtype is not None and t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    return t


def _alloc(out, shape, dtype, device, name="out"):
    """A fresh output, or the caller's `out` after checking it matches."""
    if out is None:
        return _torch().empty(tuple(shape), dtype=dtype, device=device)
    return _dev(out, name, dtype, shape, device)


def _rows(x, name="x"):
    _dev(x, name)
    if x.dim() == 1:
        return x.shape[0], 1
    if x.dim() == 2:
        return x.shape[1], x.shape[0]
    raise ValueError(f"{name} must be [N] or [batch, N]")


def _out(x, L, out):
    shape = (L,) if x.dim() == 1 else (x.shape[0], L)
    return _alloc(out, shape, x.dtype, x.device)


# a non-NULL stand-in for an output pointer in validation-only calls (the size
# checks fail before any pointer is used), so the C ABI reports the real status
_VALIDATE_ONLY = 16


def _plane_geom(x, name="x"):
    _dev(x, name)
    if x.dim() < 2:
        raise ValueError(f"{name} must be [..., H, W]")
    H, W = x.shape[-2], x.shape[-1]
    return H, W, (x.numel() // (H * W) if H * W else 0)


def _pads(padding):
    if isinstance(padding, (tuple, list)):
        return int(padding[0]), int(padding[1])
    return int(padding), int(padding)


def _pad_mode(pad_mode) -> int:
    return PAD_MODES[pad_mode] if isinstance(pad_mode, str) else int(pad_mode)


def _window(fn, x, w, stride, out, stream, dilation, padding, pad_mode):
    N, B = _rows(x)
    pl, pr = _pads(padding)
    L = ss_out_len_ex(N, w, stride, dilation, pl, pr)
    args = (N, B, w, stride, dilation, pl, pr, _pad_mode(pad_mode), _dtype_code(x), _stream(stream))
    if L < 0:
        check(fn(x.data_ptr(), _VALIDATE_ONLY, *args) or SS_ERR_BAD_SIZE)
    y = _out(x, L, out)
    check(fn(x.data_ptr(), y.data_ptr(), *args))
    return y


def pool_sum(x, w: int, stride: int = 1, out=None, stream=None, dilation: int = 1, padding=0,
             pad_mode="zeros"):
    """Eq. 3 with + (raw window sums) over the last dim of a CUDA [N] / [B, N] tensor;
    optional dilation and padding (int or (left, right); pad_mode zeros / reflect /
    circular / replicate)."""
    return _window(ss_pool_sum_ex, x, w, stride, out, stream, dilation, padding, pad_mode)


def pool_max(x, w: int, stride: int = 1, out=None, stream=None, dilation: int = 1, padding=0,
             pad_mode="zeros"):
    """Eq. 3 with max over the last dim of a CUDA [N] / [B, N] tensor; optional
    dilation and padding (zeros padding never wins)."""
    return _window(ss_pool_max_ex, x, w, stride, out, stream, dilation, padding, pad_mode)


def pool_min(x, w: int, stride: int = 1, out=None, stream=None, dilation: int = 1, padding=0,
             pad_mode="zeros"):
    """Eq. 3 with min (the sliding min of PAPER.md l.136) over the last dim of a CUDA
    [N] / [B, N] tensor; optional dilation and padding (zeros padding never wins)."""
    return _window(ss_pool_min_ex, x, w, stride, out, stream, dilation, padding, pad_mode)


def conv1d(x, filt, stride: int = 1, out=None, stream=None, dilation: int = 1, padding=0, pad_mode="zeros"):
    """Sliding dot product (cross-correlation) of a CUDA fp32 [N]/[B, N] tensor with
    a host filter (sequence of floats, numpy array or CPU tensor); optional
    dilation and padding."""
    N, B = _rows(x)
    f = [float(v) for v in (filt.tolist() if hasattr(filt, "tolist") else filt)]
    k = len(f)
    pl, pr = _pads(padding)
    L = ss_out_len_ex(N, k, stride, dilation, pl, pr)
    pm = _pad_mode(pad_mode)
    if L < 0:
        check(ss_conv1d_ex(x.data_ptr(), _VALIDATE_ONLY, N, B, f, k, stride, dilation, pl, pr, pm, _dtype_code(x),
                           _stream(stream)) or SS_ERR_BAD_SIZE)
    y = _out(x, L, out)
    check(ss_conv1d_ex(x.data_ptr(), y.data_ptr(), N, B, f, k, stride, dilation, pl, pr, pm, _dtype_code(x),
                       _stream(stream)))
    return y


def pool2d(x, kernel, stride, mode: str = "max", out=None, stream=None):
    """Separable 2-D max/avg pooling of a CUDA fp32 tensor [..., H, W] (e.g. NCHW)."""
    H, W, planes = _plane_geom(x)
    kh, kw = kernel
    sh, sw = stride
    OH, OW = ss_out_len(H, kh, sh), ss_out_len(W, kw, sw)
    m = SS_POOL_MAX if mode == "max" else SS_POOL_AVG
    if OH < 0 or OW < 0:
        check(ss_pool2d(x.data_ptr(), _VALIDATE_ONLY, planes, H, W, kh, kw, sh, sw, m, _dtype_code(x),
                        _stream(stream)) or SS_ERR_BAD_SIZE)
    y = _alloc(out, tuple(x.shape[:-2]) + (OH, OW), x.dtype, x.device)
    check(ss_pool2d(x.data_ptr(), y.data_ptr(), planes, H, W, kh, kw, sh, sw, m, _dtype_code(x), _stream(stream)))
    return y


def _filter2d(filt):
    f = filt.tolist() if hasattr(filt, "tolist") else [list(r) for r in filt]
    kh, kw = len(f), len(f[0])
    if any(len(r) != kw for r in f):
        raise ValueError("filter rows must have equal length")
    return kh, kw, [float(v) for row in f for v in row]


def conv2d(x, filt, stride=(1, 1), out=None, stream=None):
    """2-D single-channel sliding dot product of a CUDA fp32 [..., H, W] tensor with a host
    filter [kh, kw] (nested sequence, numpy array or CPU tensor); valid padding."""
    H, W, planes = _plane_geom(x)
    kh, kw, flat = _filter2d(filt)
    sh, sw = stride
    OH, OW = ss_out_len(H, kh, sh), ss_out_len(W, kw, sw)
    if OH < 0 or OW < 0:
        check(ss_conv2d(x.data_ptr(), _VALIDATE_ONLY, planes, H, W, flat, kh, kw, sh, sw, _dtype_code(x),
                        _stream(stream)) or SS_ERR_BAD_SIZE)
    y = _alloc(out, tuple(x.shape[:-2]) + (OH, OW), x.dtype, x.device)
    check(ss_conv2d(x.data_ptr(), y.data_ptr(), planes, H, W, flat, kh, kw, sh, sw, _dtype_code(x), _stream(stream)))
    return y


def affine_window(u, v, w: int, stride: int = 1, want_U: bool = True, out=None, stream=None):
    """Sliding window of gamma pairs (Eq. 8 operator, ss.h ss_affine_window) over the
    last dim of CUDA fp32 [N] / [B, N] tensors u, v.  Returns (U, V); U is None
    when want_U is False.  `out` = (U, V) preallocated (U may be None)."""
    N, B = _rows(u, "u")
    _dev(v, "v", u.dtype, u.shape, u.device)
    if _dtype_code(u) != SS_F32:
        raise TypeError("affine_window takes fp32 tensors")
    L = ss_out_len(N, w, stride)
    if L < 0:
        check(ss_affine_window(u.data_ptr(), v.data_ptr(), 0, _VALIDATE_ONLY, N, B, w, stride) or SS_ERR_BAD_SIZE)
    if out is None:
        V = _out(u, L, None)
        U = _out(u, L, None) if want_U else None
    else:
        U, V = out
        V = _out(u, L, V)
        U = _out(u, L, U) if U is not None else None
    check(ss_affine_window(u.data_ptr(), v.data_ptr(), 0 if U is None else U.data_ptr(), V.data_ptr(),
                           N, B, w, stride, _stream(stream)))
    return U, V


# ------------------------------------------------------------ backward passes
def _grad_out(dy, N, out):
    shape = (N,) if dy.dim() == 1 else (dy.shape[0], N)
    return _alloc(out, shape, dy.dtype, dy.device)


def _check_dy_1d(dy, N, w, stride):
    """dy must hold exactly the forward's out_len = (N - w) / stride + 1 outputs per row."""
    L = ss_out_len(N, w, stride)
    if L < 0:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT if N >= 1 and w > N else SS_ERR_BAD_SIZE,
                      f"invalid window: N={N} w={w} stride={stride}")
    if dy.shape[-1] != L:
        raise ValueError(f"dy must have {L} outputs per row (N={N}, w={w}, stride={stride}), got {dy.shape[-1]}")


def pool_sum_backward(dy, N: int, w: int, stride: int = 1, out=None, stream=None):
    """dx of pool_sum (valid padding): dx_t = sum of dy over the windows containing t."""
    L, B = _rows(dy, "dy")
    _check_dy_1d(dy, N, w, stride)
    dx = _grad_out(dy, N, out)
    check(ss_pool_sum_backward(dy.data_ptr(), dx.data_ptr(), N, B, w, stride, _dtype_code(dy), _stream(stream)))
    return dx


def pool_max_backward(x, dy, w: int, stride: int = 1, out=None, stream=None):
    """dx of pool_max: each window's dy goes to its first maximum in x."""
    N, B = _rows(x)
    _rows(dy, "dy")
    if dy.dim() != x.dim() or (x.dim() == 2 and dy.shape[0] != B) or dy.dtype != x.dtype or dy.device != x.device:
        raise ValueError("dy must match x's batch, dtype and device")
    _check_dy_1d(dy, N, w, stride)
    dx = _grad_out(dy, N, out)
    check(ss_pool_max_backward(x.data_ptr(), dy.data_ptr(), dx.data_ptr(), N, B, w, stride, _dtype_code(x),
                               _stream(stream)))
    return dx


def conv1d_backward_input(dy, filt, N: int, stride: int = 1, out=None, stream=None):
    """dx of conv1d (valid padding, cross-correlation) for a host filter."""
    L, B = _rows(dy, "dy")
    f = [float(v) for v in (filt.tolist() if hasattr(filt, "tolist") else filt)]
    _check_dy_1d(dy, N, len(f), stride)
    dx = _grad_out(dy, N, out)
    check(ss_conv1d_backward_input(dy.data_ptr(), dx.data_ptr(), N, B, f, len(f), stride, _dtype_code(dy),
                                   _stream(stream)))
    return dx


def _workspace(workspace, need, device):
    torch = _torch()
    if workspace is not None:
        _dev(workspace, "workspace", device=device)
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(max(need, 8), dtype=torch.uint8, device=device)
    return workspace


def conv1d_backward_filter(x, dy, k: int, stride: int = 1, out=None, workspace=None, stream=None):
    """df of conv1d: df_j = sum over rows and outputs of dy_i x_{i*stride+j} (device tensor of k floats)."""
    torch = _torch()
    N, B = _rows(x)
    _rows(dy, "dy")
    if dy.dim() != x.dim() or (x.dim() == 2 and dy.shape[0] != B) or dy.dtype != torch.float32 or \
            x.dtype != torch.float32 or dy.device != x.device:
        raise ValueError("x and dy must be fp32 on one device with the same batch")
    _check_dy_1d(dy, N, k, stride)
    df = _alloc(out, (k,), torch.float32, x.device)
    workspace = _workspace(workspace, ss_conv1d_backward_filter_workspace(k), x.device)
    check(ss_conv1d_backward_filter(x.data_ptr(), dy.data_ptr(), df.data_ptr(), N, B, k, stride,
                                    workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                                    _stream(stream)))
    return df


def _check_dy_2d(dy, H, W, kh, kw, sh, sw):
    OH, OW = ss_out_len(H, kh, sh), ss_out_len(W, kw, sw)
    if OH < 0 or OW < 0:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT, f"window {kh}x{kw} exceeds input {H}x{W}")
    if dy.dim() < 2 or tuple(dy.shape[-2:]) != (OH, OW):
        raise ValueError(f"dy must be [..., {OH}, {OW}] (H={H}, W={W}, window {kh}x{kw}, stride {sh}x{sw}), "
                         f"got {tuple(dy.shape)}")


def conv2d_backward_input(dy, filt, H: int, W: int, stride=(1, 1), out=None, stream=None):
    """dx of conv2d for a CUDA fp32 dy [..., OH, OW] and a host filter [kh, kw]: [..., H, W]."""
    torch = _torch()
    _dev(dy, "dy", torch.float32)
    kh, kw, flat = _filter2d(filt)
    sh, sw = stride
    _check_dy_2d(dy, H, W, kh, kw, sh, sw)
    planes = dy.numel() // (dy.shape[-2] * dy.shape[-1])
    dx = _alloc(out, tuple(dy.shape[:-2]) + (H, W), torch.float32, dy.device)
    check(ss_conv2d_backward_input(dy.data_ptr(), dx.data_ptr(), planes, H, W, flat, kh, kw, sh, sw,
                                   _dtype_code(dy), _stream(stream)))
    return dx


def conv2d_backward_filter(x, dy, kernel, stride=(1, 1), out=None, workspace=None, stream=None):
    """df [kh, kw] of conv2d: sum over planes and outputs of dy * the shifted x (device tensor)."""
    torch = _torch()
    kh, kw = kernel
    sh, sw = stride
    H, W, planes = _plane_geom(x)
    _dev(x, "x", torch.float32)
    _dev(dy, "dy", torch.float32, device=x.device)
    _check_dy_2d(dy, H, W, kh, kw, sh, sw)
    if dy.numel() // (dy.shape[-2] * dy.shape[-1]) != planes:
        raise ValueError("dy must have as many planes as x")
    df = _alloc(out, (kh, kw), torch.float32, x.device)
    workspace = _workspace(workspace, ss_conv2d_backward_filter_workspace(kh, kw), x.device)
    check(ss_conv2d_backward_filter(x.data_ptr(), dy.data_ptr(), df.data_ptr(), planes, H, W, kh, kw, sh, sw,
                                    workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                                    _stream(stream)))
    return df


def pool2d_backward(x, dy, kernel, stride, mode: str = "max", out=None, stream=None):
    """dx of pool2d for [..., H, W] tensors (for avg, x only sizes dx and is not read)."""
    if x is None:
        raise ValueError("pass x (or a tensor of its shape) to size dx")
    kh, kw = kernel
    sh, sw = stride
    H, W, planes = _plane_geom(x)
    _dev(dy, "dy", x.dtype, device=x.device)
    _check_dy_2d(dy, H, W, kh, kw, sh, sw)
    if dy.numel() // (dy.shape[-2] * dy.shape[-1]) != planes:
        raise ValueError("dy must have as many planes as x")
    dx = _alloc(out, x.shape, x.dtype, x.device)
    m = SS_POOL_MAX if mode == "max" else SS_POOL_AVG
    check(ss_pool2d_backward(x.data_ptr() if mode == "max" else 0, dy.data_ptr(), dx.data_ptr(), planes, H, W,
                             kh, kw, sh, sw, m, _dtype_code(dy), _stream(stream)))
    return dx


def conv1d_mc(x, w, out=None, stream=None):
    """Multi-channel conv1d, channels-last: x [B, N, Cin] bfloat16 (CUDA), w [Cout, Cin, k]
    bfloat16 (CUDA, torch conv1d weight order) -> y [B, N-k+1, Cout] float32."""
    torch = _torch()
    _dev(x, "x", torch.bfloat16)
    _dev(w, "w", torch.bfloat16, device=x.device)
    if x.dim() != 3 or w.dim() != 3:
        raise ValueError("x must be [B, N, Cin] and w [Cout, Cin, k]")
    B, N, cin = x.shape
    cout, cin2, k = w.shape
    if cin2 != cin:
        raise ValueError("w's Cin does not match x")
    if k > N:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT, f"window exceeds input: k={k} > N={N}")
    y = _alloc(out, (B, N - k + 1, cout), torch.float32, x.device)
    check(ss_conv1d_mc(x.data_ptr(), w.data_ptr(), y.data_ptr(), B, N, cin, cout, k, _stream(stream)))
    return y


def conv2d_mc(x, w, out=None, stream=None):
    """Multi-channel 2-D convolution, NHWC: x [B, H, W, Cin] bfloat16 (CUDA), w [Cout, Cin, kh, kw]
    bfloat16 (CUDA, torch conv2d weight order) -> y [B, H-kh+1, W-kw+1, Cout] float32 (valid, stride 1)."""
    torch = _torch()
    _dev(x, "x", torch.bfloat16)
    _dev(w, "w", torch.bfloat16, device=x.device)
    if x.dim() != 4 or w.dim() != 4:
        raise ValueError("x must be [B, H, W, Cin] and w [Cout, Cin, kh, kw]")
    B, H, W, cin = x.shape
    cout, cin2, kh, kw = w.shape
    if cin2 != cin:
        raise ValueError("w's Cin does not match x")
    if kh > H or kw > W:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT, f"window {kh}x{kw} exceeds input {H}x{W}")
    y = _alloc(out, (B, H - kh + 1, W - kw + 1, cout), torch.float32, x.device)
    check(ss_conv2d_mc(x.data_ptr(), w.data_ptr(), y.data_ptr(), B, H, W, cin, cout, kh, kw, _stream(stream)))
    return y


def conv1d_mc_backward_input(dy, w, N, out=None, stream=None):
    """Input gradient of conv1d_mc: dy [B, N-k+1, Cout] bfloat16 (CUDA), w [Cout, Cin, k] bfloat16
    (CUDA, the forward's weights) -> dx [B, N, Cin] float32."""
    torch = _torch()
    _dev(dy, "dy", torch.bfloat16)
    _dev(w, "w", torch.bfloat16, device=dy.device)
    if dy.dim() != 3 or w.dim() != 3:
        raise ValueError("dy must be [B, N-k+1, Cout] and w [Cout, Cin, k]")
    B, L, cout = dy.shape
    cout2, cin, k = w.shape
    if cout2 != cout:
        raise ValueError("w's Cout does not match dy")
    if k > N:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT, f"window exceeds input: k={k} > N={N}")
    if L != N - k + 1:
        raise ValueError(f"dy has {L} positions, expected N-k+1 = {N - k + 1}")
    dx = _alloc(out, (B, N, cin), torch.float32, dy.device)
    check(ss_conv1d_mc_backward_input(dy.data_ptr(), w.data_ptr(), dx.data_ptr(), B, N, cin, cout, k,
                                      _stream(stream)))
    return dx


def conv2d_mc_backward_input(dy, w, H, W, out=None, stream=None):
    """Input gradient of conv2d_mc: dy [B, H-kh+1, W-kw+1, Cout] bfloat16 (CUDA), w [Cout, Cin, kh, kw]
    bfloat16 (CUDA, the forward's weights) -> dx [B, H, W, Cin] float32."""
    torch = _torch()
    _dev(dy, "dy", torch.bfloat16)
    _dev(w, "w", torch.bfloat16, device=dy.device)
    if dy.dim() != 4 or w.dim() != 4:
        raise ValueError("dy must be [B, H-kh+1, W-kw+1, Cout] and w [Cout, Cin, kh, kw]")
    B, OH, OW, cout = dy.shape
    cout2, cin, kh, kw = w.shape
    if cout2 != cout:
        raise ValueError("w's Cout does not match dy")
    if kh > H or kw > W:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT, f"window {kh}x{kw} exceeds input {H}x{W}")
    if OH != H - kh + 1 or OW != W - kw + 1:
        raise ValueError(f"dy is {OH}x{OW}, expected {H - kh + 1}x{W - kw + 1}")
    dx = _alloc(out, (B, H, W, cin), torch.float32, dy.device)
    check(ss_conv2d_mc_backward_input(dy.data_ptr(), w.data_ptr(), dx.data_ptr(), B, H, W, cin, cout, kh, kw,
                                      _stream(stream)))
    return dx


def conv1d_mc_backward_filter(dy, x, k, out=None, workspace=None, stream=None):
    """Filter gradient of conv1d_mc: dy [B, N-k+1, Cout] and x [B, N, Cin] bfloat16 (CUDA) -> dw
    [Cout, Cin, k] float32 (torch conv1d weight order).  `workspace`: optional preallocated uint8 CUDA
    tensor of at least ss_conv1d_mc_backward_filter_workspace(Cin, Cout, k) bytes."""
    torch = _torch()
    _dev(dy, "dy", torch.bfloat16)
    _dev(x, "x", torch.bfloat16, device=dy.device)
    if dy.dim() != 3 or x.dim() != 3:
        raise ValueError("dy must be [B, N-k+1, Cout] and x [B, N, Cin]")
    B, L, cout = dy.shape
    B2, N, cin = x.shape
    if B2 != B:
        raise ValueError("dy and x batch sizes differ")
    if k > N:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT, f"window exceeds input: k={k} > N={N}")
    if L != N - k + 1:
        raise ValueError(f"dy has {L} positions, expected N-k+1 = {N - k + 1}")
    dw = _alloc(out, (cout, cin, k), torch.float32, dy.device)
    need = ss_conv1d_mc_backward_filter_workspace(cin, cout, k)
    ws = _workspace(workspace, need, dy.device) if need else None
    check(ss_conv1d_mc_backward_filter(dy.data_ptr(), x.data_ptr(), dw.data_ptr(), B, N, cin, cout, k,
                                       ws.data_ptr() if ws is not None else 0, need, _stream(stream)))
    return dw


def conv2d_mc_backward_filter(dy, x, kh, kw, out=None, workspace=None, stream=None):
    """Filter gradient of conv2d_mc: dy [B, H-kh+1, W-kw+1, Cout] and x [B, H, W, Cin] bfloat16 (CUDA) -> dw
    [Cout, Cin, kh, kw] float32 (torch conv2d weight order).  `workspace`: optional preallocated uint8 CUDA
    tensor of at least ss_conv2d_mc_backward_filter_workspace(Cin, Cout, kh, kw) bytes."""
    torch = _torch()
    _dev(dy, "dy", torch.bfloat16)
    _dev(x, "x", torch.bfloat16, device=dy.device)
    if dy.dim() != 4 or x.dim() != 4:
        raise ValueError("dy must be [B, H-kh+1, W-kw+1, Cout] and x [B, H, W, Cin]")
    B, OH, OW, cout = dy.shape
    B2, H, W, cin = x.shape
    if B2 != B:
        raise ValueError("dy and x batch sizes differ")
    if kh > H or kw > W:
        raise SSError(SS_ERR_WINDOW_EXCEEDS_INPUT, f"window {kh}x{kw} exceeds input {H}x{W}")
    if OH != H - kh + 1 or OW != W - kw + 1:
        raise ValueError(f"dy is {OH}x{OW}, expected {H - kh + 1}x{W - kw + 1}")
    dw = _alloc(out, (cout, cin, kh, kw), torch.float32, dy.device)
    need = ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw)
    ws = _workspace(workspace, need, dy.device) if need else None
    check(ss_conv2d_mc_backward_filter(dy.data_ptr(), x.data_ptr(), dw.data_ptr(), B, H, W, cin, cout, kh, kw,
                                       ws.data_ptr() if ws is not None else 0, need, _stream(stream)))
    return dw
