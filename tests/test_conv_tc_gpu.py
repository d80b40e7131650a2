"""GPU parity of the tensor-core conv1d path (csrc/conv_tc.cu; SURVEY 8f NEXT #2,
the Conclusion's "small matrix multiplication"): every
33 <= k <= 64 at stride 1 runs a Toeplitz matrix product on tcgen05 (TF32 xh*fh
plus one bf16 correction MMA per K-step, fp32 accumulation in TMEM; 3xTF32 with
SS_CONV_TC_MIXED=0).  Checked against the oracle within the BASELINE.json
bound |y - y_ref| <= 1e-5 * sum|x f| + 1e-6, over batch rows, misaligned x / y,
ragged tails (the last CTA's direct-FMA tail) and padded outputs; integer
inputs (P8) stay bit-exact; a subprocess forces the path onto small k."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOL_REL, TOL_ABS = 1e-5, 1e-6


@pytest.fixture(scope="module")
def ss():
    import paper_2305_16513_b200 as ss
    return ss


def tc_launches(ss):
    ss.lib.ss_debug_conv_tc_launches.restype = __import__("ctypes").c_uint64
    return int(ss.lib.ss_debug_conv_tc_launches())


def run(ss, x, f, xoff=0, yoff=0, padding=0):
    B, N = x.shape
    pl, pr = (padding, padding) if isinstance(padding, int) else padding
    L = N + pl + pr - len(f) + 1
    xb = torch.zeros(B * N + xoff + 4, device="cuda")
    xb[xoff:xoff + B * N] = torch.from_numpy(np.ascontiguousarray(x).reshape(-1)).cuda()
    yb = torch.full((B * L + yoff + 5,), -555.0, device="cuda")
    y = yb[yoff:yoff + B * L].view(B, L)
    n0 = tc_launches(ss)
    ss.conv1d(xb[xoff:xoff + B * N].view(B, N), f, out=y, padding=(pl, pr))
    torch.cuda.synchronize()
    used = tc_launches(ss) - n0
    h = yb.cpu().numpy()
    assert np.all(h[:yoff] == -555.0) and np.all(h[yoff + B * L:] == -555.0), "canary overwritten"
    return y.cpu().numpy(), used


def check(y, ref, mag, what):
    err = np.abs(y.astype(np.float64) - ref)
    bound = TOL_REL * mag + TOL_ABS
    assert np.all(err <= bound), f"{what}: {(err > bound).sum()} out of bound, max err/bound {(err / bound).max():.3g}"
    return float((err / bound).max())


CASES = [  # (batch, N, k)
    (1, 70001, 33), (3, 30000, 40), (2, 65536, 48), (64, 4099, 56), (1, 200003, 63), (5, 12345, 64),
    (2, 1000, 63), (1, 9000, 64), (7, 8193, 63),
]


@pytest.mark.parametrize("B,N,k", CASES)
@pytest.mark.parametrize("xoff,yoff", [(0, 0), (1, 2), (3, 1)])
def test_tc_conv_parity(ss, B, N, k, xoff, yoff):
    x = synth.normal(3, B * N).reshape(B, N)
    f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
    y, used = run(ss, x, f, xoff, yoff)
    assert used == 1, "tensor-core path not taken"
    ref, mag = oracle.conv1d(x, f)
    check(y, ref, mag, f"B={B} N={N} k={k}")


def test_tc_conv_coherent_worst_case(ss):
    # Inputs whose truncated-away TF32 bits are all ones (the largest xl, fl: ~2^-10 of the
    # value) and all of one sign, so the bf16 rounding errors of the correction terms cannot
    # cancel across the window: the per-product bound ~2^-18 |x f| (tensor-core
    # conv) adds up coherently and must still stay inside 1e-5 sum|x f| + 1e-6.
    rng = np.random.default_rng(7)
    B, N, k = 2, 40000, 63
    def worst(n, scale):
        e = rng.integers(-3, 4, size=n)  # spread the exponents a little
        mant = (1 << 23) | (0x1FFF + (rng.integers(0, 1 << 10, size=n) << 13))  # low 13 bits all ones
        return (mant.astype(np.float64) * 2.0 ** (e - 23) * scale).astype(np.float32)
    x = worst(B * N, 1.0).reshape(B, N)
    f = worst(k, 0.1)
    y, used = run(ss, x, f)
    assert used == 1, "tensor-core path not taken"
    ref, mag = oracle.conv1d(x, f)
    ratio = check(y, ref, mag, "coherent worst case")
    print(f"coherent worst case: max err/bound {ratio:.3f}")
    assert ratio < 0.6, ratio  # measured margin; the analytical per-product bound gives ~0.38


def test_tc_conv_padded(ss):
    x = synth.normal(5, 3 * 20000).reshape(3, 20000)
    f = synth.normal(4, 63, sigma=synth.cfg_sigma_filter(63))
    y, used = run(ss, x, f, 1, 3, padding=(31, 31))
    assert used == 1
    ref, mag = oracle.conv1d_ex(x, f, 1, 1, 31, 31)
    check(y, ref, mag, "same-padded k=63")


def test_tc_conv_integer_exact(ss):
    # P8: integer inputs (|x| <= 1000, exact in TF32) and integer taps: every
    # product and partial sum is an integer < 2^24 -> bit-exact in any order
    x = synth.randint(8, 2 * 40000, -1000, 1000).reshape(2, 40000).astype(np.float32)
    for k in (33, 48, 63, 64):
        f = synth.randint(9, k, -3, 3).astype(np.float32)
        y, used = run(ss, x, f)
        assert used == 1
        ref, _ = oracle.conv1d(x, f)
        np.testing.assert_array_equal(y.astype(np.float64), ref)


def test_tc_conv_delta_filter(ss):
    # P3 on the tensor-core path: e_m picks x_{i+m}; 3xTF32 keeps xh + trunc11(xl),
    # i.e. |y - x| <= 2^-21 |x| (exact on the FFMA path, test_parity_gpu)
    x = synth.normal(3, 50000).reshape(1, -1)
    for k, m in ((33, 0), (63, 17), (64, 63)):
        f = np.zeros(k, np.float32)
        f[m] = 1.0
        y, used = run(ss, x, f)
        assert used == 1
        want = x[0, m:m + 50000 - k + 1].astype(np.float64)
        assert np.all(np.abs(y[0] - want) <= 2.0 ** -21 * np.abs(want))


def test_tc_conv_deterministic(ss):
    x = synth.normal(11, 2 * 100000).reshape(2, -1)
    f = synth.normal(4, 63, sigma=synth.cfg_sigma_filter(63))
    a, _ = run(ss, x, f)
    b, _ = run(ss, x, f)
    np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("mixed", ["1", "0"])
def test_tc_conv_forced_small_k(mixed):
    # SS_CONV_TC_MIN_K=1 routes every k <= 64 through the tensor cores (fresh process:
    # the threshold is read once); SS_CONV_TC_MIXED=0 checks the 3xTF32 mode as well
    env = dict(os.environ, SS_CONV_TC_MIN_K="1", SS_CONV_TC_MIXED=mixed)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "tc_conv_check.py"), "parity"], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "parity ok" in r.stdout


@pytest.mark.parametrize("k,d,pad", [(7, 4, 12), (5, 2, 0), (2, 63, 0), (16, 4, 30), (3, 7, 7)])
def test_tc_conv_dilated(ss, k, d, pad):
    # dilated filters with extent (k-1)d+1 <= 64 run on the tensor cores as the
    # zero-expanded filter (SURVEY 8f NEXT #1 x #2)
    B, N = 3, 30011
    x = synth.normal(41, B * N).reshape(B, N)
    f = synth.normal(42, k, sigma=synth.cfg_sigma_filter(k))
    xd = torch.from_numpy(x).cuda()
    n0 = tc_launches(ss)
    y = ss.conv1d(xd, f, dilation=d, padding=pad).cpu().numpy()
    assert tc_launches(ss) - n0 == 1
    ref, mag = oracle.conv1d_ex(x, f, 1, d, pad, pad)
    check(y, ref, mag, f"dilated k={k} d={d} pad={pad}")
