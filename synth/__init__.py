"""Seeded synthetic input generators shared by the oracle side and the GPU side.

This module holds NONE of the method's arithmetic (no window sums, no dot
products); it only turns (seed, element index) into input values.  Both sides
get identical bytes because the generator is counter-based: element i of a
stream depends only on (seed, i), so any shard or sampled slice can be
regenerated on its own, on the host (numpy, here) or on the device
(``synth.cu``, built into ``libsynth.so``), bit for bit.

Generator (bench.gen_input):
  z(seed, c) = splitmix64 output number c+1 of the stream started at `seed`:
      z = seed + (c+1) * 0x9E3779B97F4A7C15   (mod 2^64)
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
      z = (z ^ (z >> 27)) * 0x94D049BB133111EB
      z =  z ^ (z >> 31)
  z(0, 0) = 0xE220A8397B1DCDAF (pinned in tests).

Maps (all exact, so host and device agree bit for bit):
  uniform01  : u = (z(seed,i) >> 40) * 2^-24                  in [0, 1)
  uniform_pm1: 2u - 1                                         in [-1, 1)
  randint(lo, hi): lo + (((z >> 32) * (hi - lo + 1)) >> 32)   in {lo..hi}
  normal(sigma): Irwin-Hall(12) stand-in for N(0, 1): the twelve 16-bit lanes
      of z(seed, 3i), z(seed, 3i+1), z(seed, 3i+2) are summed as integers S;
      x = float32( ((S - 6*65536) * 2^-16) * sigma )  (one double multiply,
      one round-to-nearest to fp32; exact up to that final rounding).
      Mean 0, variance 1 (up to 2^-32), support [-6, 6).  DESIGN.md, input
      recipe, states why this stands in for the paper's N(0, sigma^2).
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, counters: np.ndarray) -> np.ndarray:
    """z(seed, c) for an array of counters c (uint64)."""
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (c + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
        z = z ^ (z >> np.uint64(31))
    return z


def _idx(start: int, n: int) -> np.ndarray:
    return np.arange(start, start + n, dtype=np.uint64)


def uniform01(seed: int, n: int, start: int = 0) -> np.ndarray:
    z = splitmix64(seed, _idx(start, n))
    return ((z >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)).astype(np.float32)


def uniform_pm1(seed: int, n: int, start: int = 0) -> np.ndarray:
    u = uniform01(seed, n, start)
    return (np.float32(2.0) * u - np.float32(1.0)).astype(np.float32)


def uab(seed: int, n: int, lo: float, hi: float, start: int = 0) -> np.ndarray:
    """Uniform on [lo, hi): fl(lo + fl((hi - lo) * u01)) in fp32 (device twin k_uab)."""
    u = uniform01(seed, n, start)
    span = np.float32(np.float32(hi) - np.float32(lo))
    return (np.float32(lo) + span * u).astype(np.float32)


def randint(seed: int, n: int, lo: int, hi: int, start: int = 0) -> np.ndarray:
    z = splitmix64(seed, _idx(start, n))
    span = np.uint64(hi - lo + 1)
    with np.errstate(over="ignore"):
        r = ((z >> np.uint64(32)) * span) >> np.uint64(32)
    return (r.astype(np.int64) + lo).astype(np.int32)


def normal(seed: int, n: int, sigma: float = 1.0, start: int = 0) -> np.ndarray:
    base = np.arange(start, start + n, dtype=np.uint64) * np.uint64(3)
    S = np.zeros(n, dtype=np.int64)
    for part in range(3):
        z = splitmix64(seed, base + np.uint64(part))
        for lane in range(4):
            S += ((z >> np.uint64(16 * lane)) & np.uint64(0xFFFF)).astype(np.int64)
    v = (S - 6 * 65536).astype(np.float64) * (2.0 ** -16)
    return (v * np.float64(sigma)).astype(np.float32)


# ---- BASELINE.json configs: the named streams --------------------------------
# (seed numbers are BASELINE.json's; the distributions its text names)

def cfg_sigma_filter(k: int) -> float:
    """f ~ N(0, 1/k): sigma = 1/sqrt(k) (SURVEY reading 13)."""
    return float(1.0 / np.sqrt(np.float64(k)))


def generate(dist: str, seed: int, n: int, start: int = 0, **kw) -> np.ndarray:
    if dist == "u01":
        return uniform01(seed, n, start)
    if dist == "upm1":
        return uniform_pm1(seed, n, start)
    if dist == "int":
        return randint(seed, n, kw["lo"], kw["hi"], start)
    if dist == "uab":
        return uab(seed, n, kw["lo"], kw["hi"], start)
    if dist == "normal":
        return normal(seed, n, kw.get("sigma", 1.0), start)
    raise ValueError(dist)


# ---- device twin (synth.cu -> libsynth.so) -----------------------------------
import ctypes as _ct
import os as _os
import subprocess as _sp

_SYN_DIR = _os.path.dirname(_os.path.abspath(__file__))
_SYN_SO = _os.path.join(_SYN_DIR, "libsynth.so")
_syn = None


def build_device(force: bool = False) -> str:
    src = _os.path.join(_SYN_DIR, "synth.cu")
    if force or not _os.path.exists(_SYN_SO) or _os.path.getmtime(_SYN_SO) < _os.path.getmtime(src):
        tmp = _SYN_SO + f".tmp{_os.getpid()}"
        _sp.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                        "-O3", "--fmad=false", "-Xcompiler", "-fPIC", "-shared", "-o", tmp, src])
        _os.replace(tmp, _SYN_SO)
    return _SYN_SO


def _dev():
    global _syn
    if _syn is None:
        build_device()
        L = _ct.CDLL(_SYN_SO)
        i64, u64, vp = _ct.c_int64, _ct.c_uint64, _ct.c_void_p
        L.synth_uniform01.argtypes = [vp, i64, u64, i64, vp]
        L.synth_uniform_pm1.argtypes = [vp, i64, u64, i64, vp]
        L.synth_randint.argtypes = [vp, i64, u64, i64, i64, i64, vp]
        L.synth_normal.argtypes = [vp, i64, u64, _ct.c_double, i64, vp]
        L.synth_uab.argtypes = [vp, i64, u64, _ct.c_float, _ct.c_float, i64, vp]
        _syn = L
    return _syn


def fill_device(t, dist: str, seed: int, start: int = 0, stream=None, **kw):
    """Fill the contiguous CUDA tensor `t` with elements [start, start+numel) of a stream."""
    import torch
    s = torch.cuda.current_stream().cuda_stream if stream is None else stream.cuda_stream
    n = t.numel()
    L = _dev()
    if dist == "u01":
        rc = L.synth_uniform01(t.data_ptr(), n, seed, start, s)
    elif dist == "upm1":
        rc = L.synth_uniform_pm1(t.data_ptr(), n, seed, start, s)
    elif dist == "int":
        rc = L.synth_randint(t.data_ptr(), n, seed, kw["lo"], kw["hi"], start, s)
    elif dist == "uab":
        span = float(np.float32(np.float32(kw["hi"]) - np.float32(kw["lo"])))
        rc = L.synth_uab(t.data_ptr(), n, seed, float(np.float32(kw["lo"])), span, start, s)
    elif dist == "normal":
        rc = L.synth_normal(t.data_ptr(), n, seed, float(kw.get("sigma", 1.0)), start, s)
    else:
        raise ValueError(dist)
    if rc != 0:
        raise RuntimeError(f"synth kernel launch failed: cuda error {rc}")
    return t
