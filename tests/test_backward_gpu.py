"""GPU parity of the backward passes (csrc/backward.cu +
stride-1 reuse of the forward kernels) against the oracle's vector-Jacobian
products (tests/test_oracle_backward_pins.py pins those).  fp32 results within
1e-5 * sum|terms| + 1e-6 (BASELINE.json form; sum|terms| from the oracle, or
the max routing of |dy|), int32 sums bit-exact modulo 2^32; every dx element is
written (positions no window touches are 0) and canaries around dx survive."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
TOL_REL, TOL_ABS = 1e-5, 1e-6


@pytest.fixture(scope="module")
def ss():
    import paper_2305_16513_b200 as ss
    return ss


def dev(a, off=0):
    a = np.ascontiguousarray(a)
    buf = torch.zeros(a.size + off + 4, dtype=torch.from_numpy(a[:0]).dtype if a.size else torch.float32,
                      device="cuda")
    buf[off:off + a.size] = torch.from_numpy(a.reshape(-1)).cuda()
    return buf[off:off + a.size]


def out_buf(n, dtype=torch.float32, off=0, fill=-4321):
    buf = torch.full((n + off + 6,), fill, dtype=dtype, device="cuda")
    return buf, buf[off:off + n]


def canary_ok(buf, off, n, fill=-4321):
    h = buf.cpu().numpy()
    return np.all(h[:off] == fill) and np.all(h[off + n:] == fill)


def within(y, ref, mag, what):
    err = np.abs(y.astype(np.float64) - ref)
    bound = TOL_REL * mag + TOL_ABS
    assert np.all(err <= bound), f"{what}: {(err > bound).sum()} out of bound, max err/bound {(err / bound).max():.3g}"


POOL_CASES = [  # (B, N, w, s)
    (1, 1, 1, 1), (2, 9, 3, 1), (3, 1000, 8, 1), (2, 70001, 64, 1), (1, 40000, 257, 1), (2, 1001, 4, 2),
    (3, 999, 7, 3), (1, 5000, 2, 2), (2, 777, 9, 4), (1, 3000, 1, 5), (4, 20000, 33, 1),
    # unit-stride run kernel: tile edges (1984 / 3968 positions), R = 8 and R = 16 tiles
    (2, 5000, 16, 1), (1, 1984, 5, 1), (2, 3969, 64, 1), (1, 9000, 65, 1), (3, 7000, 128, 1), (1, 130, 129, 1),
]


@pytest.mark.parametrize("B,N,w,s", POOL_CASES)
@pytest.mark.parametrize("off", [0, 1])
def test_pool_sum_backward_f32(ss, B, N, w, s, off):
    L = (N - w) // s + 1
    dy = synth.normal(21, B * L).reshape(B, L)
    buf, dx = out_buf(B * N, off=off)
    dyd = dev(dy, off)  # keep the device copies alive until the launch has run
    ss.check(ss.ss_pool_sum_backward(dyd.data_ptr(), dx.data_ptr(), N, B, w, s, ss.SS_F32))
    torch.cuda.synchronize()
    assert canary_ok(buf, off, B * N)
    ref, mag = oracle.pool_sum_backward(dy, N, w, s)
    within(dx.cpu().numpy().reshape(B, N), ref, mag, f"sum bwd B={B} N={N} w={w} s={s}")


@pytest.mark.parametrize("B,N,w,s", POOL_CASES)
def test_pool_sum_backward_i32_exact(ss, B, N, w, s):
    L = (N - w) // s + 1
    dy = synth.randint(22, B * L, -1000, 1000).reshape(B, L)
    buf, dx = out_buf(B * N, torch.int32)
    dyd = dev(dy)
    ss.check(ss.ss_pool_sum_backward(dyd.data_ptr(), dx.data_ptr(), N, B, w, s, ss.SS_I32))
    torch.cuda.synchronize()
    assert canary_ok(buf, 0, B * N)
    ref, _ = oracle.pool_sum_backward(dy.astype(np.float32), N, w, s)  # |dy| <= 1000: exact in fp32 / double
    np.testing.assert_array_equal(dx.cpu().numpy().reshape(B, N).astype(np.int64), ref.astype(np.int64))


@pytest.mark.parametrize("B,N,w,s", POOL_CASES)
@pytest.mark.parametrize("ties", [False, True])
def test_pool_max_backward(ss, B, N, w, s, ties):
    L = (N - w) // s + 1
    x = (synth.randint(23, B * N, -2, 2).astype(np.float32) if ties else synth.normal(23, B * N)).reshape(B, N)
    dy = synth.normal(24, B * L).reshape(B, L)
    buf, dx = out_buf(B * N, off=1)
    xd, dyd = dev(x), dev(dy, 3)
    ss.check(ss.ss_pool_max_backward(xd.data_ptr(), dyd.data_ptr(), dx.data_ptr(), N, B, w, s))
    torch.cuda.synchronize()
    assert canary_ok(buf, 1, B * N)
    ref = oracle.pool_max_backward(x, dy, w, s)
    mag = oracle.pool_max_backward(x, np.abs(dy), w, s)  # same routing, |dy|
    within(dx.cpu().numpy().reshape(B, N), ref, mag, f"max bwd B={B} N={N} w={w} s={s} ties={ties}")
    if w <= s:  # windows disjoint: one dy per position -> exact
        np.testing.assert_array_equal(dx.cpu().numpy().reshape(B, N).astype(np.float64), ref)


# stride-1 TMA tile kernel (csrc/maxbwd.cu, w in {2,3,4,5,7,8,9,16,17,32,33,64}, 16-B aligned x / dy):
# T = 4094 - w stored positions per tile; rows of odd length (flat row starts at every
# alignment), N around T and 2T, N < w + 3, integer ties
S1_CASES = [  # (B, N, w)
    (3, 4092, 2), (2, 4091, 3), (5, 4090, 4), (1, 8179, 5), (3, 4087, 7), (2, 8173, 8), (4, 4085, 9),
    (3, 8157, 16), (2, 4077, 17), (2, 4061, 32), (2, 9000, 33), (3, 4030, 64), (2, 8061, 64), (7, 19, 16),
    (5, 10, 9), (1, 2, 2), (3, 1 << 16, 16), (2, 5000, 5),
]


@pytest.mark.parametrize("B,N,w", S1_CASES)
@pytest.mark.parametrize("ties", [False, True])
def test_pool_max_backward_s1_tile(ss, B, N, w, ties):
    L = N - w + 1
    x = (synth.randint(27, B * N, -3, 3).astype(np.float32) if ties else synth.normal(27, B * N)).reshape(B, N)
    dy = synth.normal(28, B * L).reshape(B, L)
    buf, dx = out_buf(B * N, off=4)
    xd, dyd = dev(x), dev(dy)
    ss.check(ss.ss_pool_max_backward(xd.data_ptr(), dyd.data_ptr(), dx.data_ptr(), N, B, w, 1))
    torch.cuda.synchronize()
    assert canary_ok(buf, 4, B * N)
    ref = oracle.pool_max_backward(x, dy, w, 1)
    mag = oracle.pool_max_backward(x, np.abs(dy), w, 1)
    within(dx.cpu().numpy().reshape(B, N), ref, mag, f"max bwd s1 tile B={B} N={N} w={w} ties={ties}")


@pytest.mark.parametrize("w", [3, 8, 9, 40, 64, 100, 128])
@pytest.mark.parametrize("pattern", ["spikes", "rising", "falling", "flat"])
def test_pool_max_backward_runs(ss, w, pattern):
    # long and short routing runs: a spike is the first maximum of up to w windows
    # (runs spanning several threads), rising / falling / flat inputs route every
    # window to its last / first / first element
    B, N = 2, 6000
    L = N - w + 1
    t = np.arange(B * N, dtype=np.float64)
    if pattern == "spikes":
        x = synth.normal(25, B * N).astype(np.float64)
        x[::97] = 50.0
    elif pattern == "rising":
        x = t
    elif pattern == "falling":
        x = -t
    else:
        x = np.zeros(B * N)
    x = x.astype(np.float32).reshape(B, N)
    dy = synth.normal(26, B * L).reshape(B, L)
    buf, dx = out_buf(B * N)
    xd, dyd = dev(x), dev(dy)
    ss.check(ss.ss_pool_max_backward(xd.data_ptr(), dyd.data_ptr(), dx.data_ptr(), N, B, w, 1))
    torch.cuda.synchronize()
    assert canary_ok(buf, 0, B * N)
    ref = oracle.pool_max_backward(x, dy, w, 1)
    mag = oracle.pool_max_backward(x, np.abs(dy), w, 1)
    within(dx.cpu().numpy().reshape(B, N), ref, mag, f"max bwd runs w={w} {pattern}")


CONV_CASES = [  # (B, N, k, s)
    (1, 10, 1, 1), (2, 1000, 3, 1), (3, 20001, 7, 1), (2, 70000, 31, 1), (2, 50000, 40, 1), (1, 80001, 63, 1),
    (3, 30000, 64, 1), (1, 9000, 100, 1), (2, 3001, 5, 2), (3, 4000, 9, 3), (1, 5000, 64, 4), (2, 999, 13, 7),
]


@pytest.mark.parametrize("B,N,k,s", CONV_CASES)
def test_conv_backward_input(ss, B, N, k, s):
    L = (N - k) // s + 1
    dy = synth.normal(25, B * L).reshape(B, L)
    f = synth.normal(26, k, sigma=synth.cfg_sigma_filter(k))
    buf, dx = out_buf(B * N, off=2)
    dyd = dev(dy, 1)
    ss.check(ss.ss_conv1d_backward_input(dyd.data_ptr(), dx.data_ptr(), N, B, f.tolist(), k, s))
    torch.cuda.synchronize()
    assert canary_ok(buf, 2, B * N)
    ref, mag = oracle.conv1d_backward_input(dy, f, N, s)
    within(dx.cpu().numpy().reshape(B, N), ref, mag, f"conv bwd input B={B} N={N} k={k} s={s}")


FILTER_CASES = CONV_CASES + [(1, 5000, 65, 1), (2, 3000, 130, 1), (1, 7000, 200, 3), (64, 4096, 63, 1),
                             (5, 1500, 1024, 1),
                             # tile-pair kernel: Q = 1 / 2 / 4 tap-group edges, odd tile counts, N < one tile
                             (2, 9000, 16, 1), (1, 12000, 17, 1), (3, 8200, 32, 1), (1, 300, 33, 1), (7, 1025, 2, 1)]


@pytest.mark.parametrize("B,N,k,s", FILTER_CASES)
def test_conv_backward_filter(ss, B, N, k, s):
    L = (N - k) // s + 1
    x = synth.normal(27, B * N).reshape(B, N)
    dy = synth.normal(28, B * L).reshape(B, L)
    df = ss.conv1d_backward_filter(dev(x, 1).view(B, N), dev(dy, 2).view(B, L), k, s).cpu().numpy()
    ref, mag = oracle.conv1d_backward_filter(x, dy, k, s)
    within(df, ref, mag, f"conv bwd filter B={B} N={N} k={k} s={s}")


# tensor-core filter gradient (csrc/fgrad_tc.cu): stride 1, k <= 64, N % 128 == 0, 16-B aligned x --
# chunks of 128 dy positions, units of 128 chunks, row tails (L % 128), one chunk per row, one unit per
# row and many, more units than CTAs; N % 128 != 0 cases take the FFMA kernels
FT_CASES = [  # (B, N, k)
    (1, 128, 1), (2, 128, 64), (3, 256, 3), (2, 384, 64), (5, 1280, 7), (4, 16384 + 128, 31), (2, 8192, 63),
    (3, 32768, 33), (64, 16384, 63), (2, 1 << 18, 17), (1, 70016, 64), (7, 20096, 2),
    (1, 4, 1), (3, 100, 7), (1, 132, 5), (3, 8196, 33),
]


@pytest.mark.parametrize("B,N,k", FT_CASES)
def test_conv_backward_filter_tc(ss, B, N, k):
    L = N - k + 1
    x = synth.normal(33, B * N).reshape(B, N)
    dy = synth.normal(34, B * L).reshape(B, L)
    df = ss.conv1d_backward_filter(dev(x).view(B, N), dev(dy).view(B, L), k, 1).cpu().numpy()
    ref, mag = oracle.conv1d_backward_filter(x, dy, k, 1)
    within(df, ref, mag, f"conv bwd filter (tensor cores) B={B} N={N} k={k}")


def test_conv_backward_filter_tc_integers_exact(ss):
    # small integers: the TF32 split is exact (lo = 0), every product and partial sum is an exact integer
    B, N, k = 3, 40064, 63
    L = N - k + 1
    x = synth.randint(35, B * N, -4, 4).astype(np.float32).reshape(B, N)
    dy = synth.randint(36, B * L, -4, 4).astype(np.float32).reshape(B, L)
    df = ss.conv1d_backward_filter(dev(x).view(B, N), dev(dy).view(B, L), k, 1).cpu().numpy()
    ref, _ = oracle.conv1d_backward_filter(x, dy, k, 1)
    np.testing.assert_array_equal(df.astype(np.float64), ref)


def test_conv_backward_filter_deterministic(ss):
    x = torch.from_numpy(synth.normal(29, 8 * 100000).reshape(8, -1)).cuda()
    dy = torch.from_numpy(synth.normal(30, 8 * (100000 - 62)).reshape(8, -1)).cuda()
    a = ss.conv1d_backward_filter(x, dy, 63)
    b = ss.conv1d_backward_filter(x, dy, 63)
    assert torch.equal(a, b)


P2_CASES = [(3, 16, 17, 3, 3, 1, 1), (2, 31, 30, 2, 2, 2, 2), (2, 20, 21, 3, 2, 2, 1), (1, 112, 112, 3, 3, 1, 1),
            (4, 9, 9, 9, 9, 1, 1), (2, 15, 40, 1, 5, 1, 3)]


@pytest.mark.parametrize("P,H,W,kh,kw,sh,sw", P2_CASES)
@pytest.mark.parametrize("mode", ["max", "avg"])
def test_pool2d_backward(ss, mode, P, H, W, kh, kw, sh, sw):
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    x = synth.uniform01(31, P * H * W).reshape(P, H, W)
    dy = synth.normal(32, P * OH * OW).reshape(P, OH, OW)
    m = ss.SS_POOL_MAX if mode == "max" else ss.SS_POOL_AVG
    buf, dx = out_buf(P * H * W, off=1)
    xd, dyd = dev(x), dev(dy)
    ss.check(ss.ss_pool2d_backward(xd.data_ptr() if mode == "max" else 0, dyd.data_ptr(), dx.data_ptr(),
                                   P, H, W, kh, kw, sh, sw, m))
    torch.cuda.synchronize()
    assert canary_ok(buf, 1, P * H * W)
    ref, mag = oracle.pool2d_backward(x, dy, H, W, kh, kw, sh, sw, oracle.POOL2D_MAX if mode == "max" else
                                      oracle.POOL2D_AVG)
    within(dx.cpu().numpy().reshape(P, H, W), ref, mag, f"pool2d bwd {mode} {(P, H, W, kh, kw, sh, sw)}")


def test_backward_matches_torch_autograd_cfg3_slice(ss):
    # a config-3-shaped slice (rows of 2^20, k = 63) end to end against torch
    # float64 autograd of F.conv1d (test-only library reference)
    B, N, k = 4, 1 << 20, 63
    x = torch.empty(B, N, device="cuda")
    synth.fill_device(x, "normal", 3)
    f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
    dy = torch.empty(B, N - k + 1, device="cuda")
    synth.fill_device(dy, "normal", 33)
    dx = ss.conv1d_backward_input(dy, f, N)
    df = ss.conv1d_backward_filter(x, dy, k)
    xt = x.double().requires_grad_(True)
    ft = torch.tensor(f, dtype=torch.float64, device="cuda", requires_grad=True)
    torch.nn.functional.conv1d(xt[:, None, :], ft[None, None, :])[:, 0, :].backward(dy.double())
    mag_x = torch.nn.functional.conv_transpose1d(dy.double().abs()[:, None, :], ft.detach().abs()[None, None, :])[:, 0, :]
    assert torch.all((dx.double() - xt.grad).abs() <= TOL_REL * mag_x + TOL_ABS)
    mag_f = (x.double().abs()[:, None, :].unfold(2, N - k + 1, 1)[:, 0] * dy.double().abs()[:, None, :]).sum((0, 2))
    assert torch.all((df.double() - ft.grad).abs() <= TOL_REL * mag_f + TOL_ABS)


STRIP_CASES = [(2, 3, 3), (1, 5, 31), (2, 40, 30), (1, 7, 61), (2, 200, 9), (3, 33, 59), (1, 130, 95), (4, 4, 32)]


@pytest.mark.parametrize("P,H,W", STRIP_CASES)
@pytest.mark.parametrize("ties", [False, True])
def test_pool2d_max_backward_3x3_strips(ss, ties, P, H, W):
    """3x3/1 max gradient (the plane kernel): widths around multiples of 30 and 32, narrow and short
    planes, tall planes, ties (first row-major maximum)."""
    OH, OW = H - 2, W - 2
    x = (synth.randint(35, P * H * W, 0, 2).astype(np.float32) if ties else
         synth.uniform01(35, P * H * W)).reshape(P, H, W)
    dy = synth.normal(36, P * OH * OW).reshape(P, OH, OW)
    dx = ss.pool2d_backward(torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda(), (3, 3), (1, 1), "max")
    ref, mag = oracle.pool2d_backward(x, dy, H, W, 3, 3, 1, 1, oracle.POOL2D_MAX)
    got = dx.cpu().numpy()
    within(got, ref, mag, f"pool2d max bwd strips ties={ties} {(P, H, W)}")
    np.testing.assert_array_equal(got.astype(np.float64) != 0, ref != 0)


@pytest.mark.parametrize("P,H,W,kh,kw,sh,sw", [(3, 16, 16, 2, 2, 2, 2), (2, 112, 112, 2, 2, 2, 2), (2, 10, 36, 2, 2, 2, 2),
                                                (2, 112, 112, 3, 3, 1, 1), (3, 37, 150, 3, 3, 1, 1),
                                                (2, 30, 140, 5, 5, 1, 1), (1, 20, 21, 7, 7, 1, 1)])
@pytest.mark.parametrize("mode", ["max", "avg"])
@pytest.mark.parametrize("ties", [False, True])
def test_pool2d_backward_fast_paths(ss, mode, ties, P, H, W, kh, kw, sh, sw):
    """16-B aligned buffers take the round-2 kernels: the 2x2/2 stream kernel (first-max routing,
    ties from integer-valued x) and, for avg at stride 1, the 2-D tile kernel (full correlation of
    dy with the 1/(kh kw) box)."""
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    x = (synth.randint(33, P * H * W, 0, 3).astype(np.float32) if ties else
         synth.uniform01(33, P * H * W)).reshape(P, H, W)
    dy = synth.normal(34, P * OH * OW).reshape(P, OH, OW)
    m = ss.SS_POOL_MAX if mode == "max" else ss.SS_POOL_AVG
    xd = torch.from_numpy(x).cuda()
    dyd = torch.from_numpy(dy).cuda()
    dx = ss.pool2d_backward(xd, dyd, (kh, kw), (sh, sw), mode)
    torch.cuda.synchronize()
    ref, mag = oracle.pool2d_backward(x, dy, H, W, kh, kw, sh, sw, oracle.POOL2D_MAX if mode == "max" else
                                      oracle.POOL2D_AVG)
    got = dx.cpu().numpy()
    within(got, ref, mag, f"pool2d bwd fast {mode} ties={ties} {(P, H, W, kh, kw, sh, sw)}")
    if mode == "max":  # routing is exact: each dy lands whole on one element
        np.testing.assert_array_equal(got.astype(np.float64) != 0, ref != 0)
