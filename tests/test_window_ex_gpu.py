"""GPU parity for the window-spec entry points (ss_*_ex: dilation + zero
padding) against the oracle's *_ex routines.  Covers the
stride-1 padded path (TMA tile kernel on the interior + direct kernel on the
edges), dilation / stride combinations (direct kernel), windows made only of
padding, misaligned pointers and canaries around y; the sliding min (SURVEY 8f
NEXT #3) on every path, and the reflect / circular / replicate padding modes
(8f NEXT #1, "padding, mirroring and periodicity")."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ss():
    import paper_2305_16513_b200 as ss
    return ss


SPECS = [  # (N, B, w, s, d, pl, pr)
    (20011, 3, 3, 1, 1, 1, 1), (20011, 2, 16, 1, 1, 5, 0), (30011, 2, 64, 1, 1, 0, 7),
    (30011, 1, 256, 1, 1, 100, 100), (9000, 2, 7, 1, 1, 6, 6), (9000, 2, 3, 2, 1, 1, 1),
    (9000, 2, 5, 1, 2, 0, 0), (9000, 3, 4, 2, 3, 2, 5), (5000, 1, 2, 1, 8, 3, 3),
    (100, 2, 8, 3, 4, 9, 9), (3, 1, 2, 1, 1, 4, 4), (1, 1, 1, 1, 1, 0, 2),
]


def run(ss, fn, x_np, extra, L, xoff=0, yoff=0, dt=torch.float32):
    B, N = x_np.shape
    xbuf = torch.empty(x_np.size + xoff + 3, dtype=torch.from_numpy(x_np[:0]).dtype, device="cuda")
    x = xbuf[xoff:xoff + x_np.size]
    x.copy_(torch.from_numpy(x_np.reshape(-1)).cuda())
    ybuf = torch.full((B * L + yoff + 5,), -77, dtype=dt, device="cuda")
    y = ybuf[yoff:yoff + B * L]
    ss.check(fn(x.data_ptr(), y.data_ptr(), N, B, *extra))
    torch.cuda.synchronize()
    h = ybuf.cpu().numpy()
    assert np.all(h[:yoff] == -77) and np.all(h[yoff + B * L:] == -77), "canary overwritten"
    return y.cpu().numpy().reshape(B, L)


@pytest.mark.parametrize("N,B,w,s,d,pl,pr", SPECS)
@pytest.mark.parametrize("off", [(0, 0), (1, 2)])
def test_pool_ex(ss, N, B, w, s, d, pl, pr, off):
    L = ss.ss_out_len_ex(N, w, s, d, pl, pr)
    if L < 0:
        pytest.skip("window exceeds padded input")
    assert L == oracle.out_len_ex(N, w, s, d, pl, pr)
    xi = synth.randint(2, B * N, -1000, 1000).reshape(B, N)
    ys = run(ss, ss.ss_pool_sum_ex, xi, (w, s, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_I32), L, *off, dt=torch.int32)
    np.testing.assert_array_equal(ys, (oracle.pool_sum_ex(xi, w, s, d, pl, pr) & 0xFFFFFFFF).astype(np.uint32).view(np.int32))
    ym = run(ss, ss.ss_pool_max_ex, xi, (w, s, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_I32), L, *off, dt=torch.int32)
    np.testing.assert_array_equal(ym, oracle.pool_max_ex(xi, w, s, d, pl, pr))
    yn = run(ss, ss.ss_pool_min_ex, xi, (w, s, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_I32), L, *off, dt=torch.int32)
    np.testing.assert_array_equal(yn, oracle.pool_min_ex(xi, w, s, d, pl, pr))
    xf = synth.uniform_pm1(0, B * N).reshape(B, N)
    ymf = run(ss, ss.ss_pool_max_ex, xf, (w, s, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L, *off)
    np.testing.assert_array_equal(ymf, oracle.pool_max_ex(xf, w, s, d, pl, pr))
    ysf = run(ss, ss.ss_pool_sum_ex, xf, (w, s, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L, *off)
    ref, mag = oracle.pool_sum_ex(xf, w, s, d, pl, pr)
    assert np.all(np.abs(ysf - ref) <= 1e-5 * mag + 1e-6)


@pytest.mark.parametrize("N,B,w,s,d,pl,pr", SPECS + [(40011, 2, 31, 1, 1, 15, 15), (40011, 2, 63, 1, 1, 31, 31),
                                                     (40011, 1, 63, 1, 1, 62, 0), (20000, 2, 15, 1, 3, 21, 21)])
def test_conv_ex(ss, N, B, w, s, d, pl, pr):
    L = ss.ss_out_len_ex(N, w, s, d, pl, pr)
    if L < 0:
        pytest.skip("window exceeds padded input")
    x = synth.normal(3, B * N).reshape(B, N)
    f = synth.normal(4, w, sigma=synth.cfg_sigma_filter(w))
    y = run(ss, lambda xp, yp, N_, B_, *a: ss.ss_conv1d_ex(xp, yp, N_, B_, f.tolist(), w, *a),
            x, (s, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L, 1, 1)
    ref, mag = oracle.conv1d_ex(x, f, s, d, pl, pr)
    err = np.abs(y.astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * mag + 1e-6), float((err / (1e-5 * mag + 1e-6)).max())


def test_padded_equals_valid_interior_bitwise(ss):
    # the padded call's interior equals the valid call bitwise (same kernels / association)
    x = torch.from_numpy(synth.normal(3, 2 * 50000).reshape(2, 50000)).cuda()
    f = synth.normal(4, 31, sigma=synth.cfg_sigma_filter(31))
    yv = ss.conv1d(x, f)
    yp = ss.conv1d(x, f, padding=(15, 15))
    assert torch.equal(yp[:, 15:15 + yv.shape[1]], yv)
    ym = ss.pool_max(x, 64, padding=3)
    assert torch.equal(ym[:, 3:3 + x.shape[1] - 63], ss.pool_max(x, 64))


def test_ex_validation(ss):
    FX, FY = 0x10000000, 0x20000000
    Z = ss.SS_PAD_ZEROS
    assert ss.ss_pool_sum_ex(FX, FY, 10, 1, 3, 1, 0, 0, 0, Z, ss.SS_F32) == ss.SS_ERR_BAD_SIZE  # dilation 0
    assert ss.ss_pool_sum_ex(FX, FY, 10, 1, 3, 1, 1, -1, 0, Z, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_max_ex(FX, FY, 3, 1, 3, 1, 2, 0, 0, Z, ss.SS_F32) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_pool_min_ex(FX, FY, 10, 1, 3, 1, 1, 10, 0, ss.SS_PAD_REFLECT, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_sum_ex(FX, FY, 10, 1, 3, 1, 1, 0, 11, ss.SS_PAD_CIRCULAR, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_sum_ex(FX, FY, 10, 1, 3, 1, 1, 1, 1, 7, ss.SS_F32) == ss.SS_ERR_UNSUPPORTED
    # (no valid call with fake pointers: it would launch)


DILATED = [  # (N, B, w, d, pl, pr): stride-1 dilated windows -> the phase-decomposed tile kernel
    (50011, 2, 8, 2, 0, 0), (50011, 3, 15, 8, 56, 56), (30000, 1, 32, 3, 0, 0), (40000, 2, 5, 16, 0, 9),
    (70001, 1, 3, 256, 0, 0), (9000, 2, 17, 7, 48, 64), (20000, 2, 2, 300, 0, 0), (5000, 2, 32, 33, 0, 0),
]


@pytest.mark.parametrize("N,B,w,d,pl,pr", DILATED)
def test_dilated_tile(ss, N, B, w, d, pl, pr):
    L = ss.ss_out_len_ex(N, w, 1, d, pl, pr)
    if L < 0:
        pytest.skip("window exceeds padded input")
    xf = synth.uniform_pm1(7, B * N).reshape(B, N)
    ymf = run(ss, ss.ss_pool_max_ex, xf, (w, 1, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L, 1, 2)
    np.testing.assert_array_equal(ymf, oracle.pool_max_ex(xf, w, 1, d, pl, pr))
    ynf = run(ss, ss.ss_pool_min_ex, xf, (w, 1, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L, 2, 1)
    np.testing.assert_array_equal(ynf, oracle.pool_min_ex(xf, w, 1, d, pl, pr))
    ysf = run(ss, ss.ss_pool_sum_ex, xf, (w, 1, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L, 3, 1)
    ref, mag = oracle.pool_sum_ex(xf, w, 1, d, pl, pr)
    assert np.all(np.abs(ysf - ref) <= 1e-5 * mag + 1e-6)
    f = synth.normal(4, w, sigma=synth.cfg_sigma_filter(w))
    y = run(ss, lambda xp, yp, N_, B_, *a: ss.ss_conv1d_ex(xp, yp, N_, B_, f.tolist(), w, *a),
            xf, (1, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L, 2, 3)
    ref, mag = oracle.conv1d_ex(xf, f, 1, d, pl, pr)
    assert np.all(np.abs(y.astype(np.float64) - ref) <= 1e-5 * mag + 1e-6)
    # integer-valued input (exact in fp32): the sum is exact in any order
    xi = synth.randint(8, B * N, -1000, 1000).reshape(B, N).astype(np.float32)
    ysi = run(ss, ss.ss_pool_sum_ex, xi, (w, 1, d, pl, pr, ss.SS_PAD_ZEROS, ss.SS_F32), L)
    refi, _ = oracle.pool_sum_ex(xi, w, 1, d, pl, pr)
    np.testing.assert_array_equal(ysi.astype(np.float64), refi)


MODE_SPECS = SPECS + [  # reflect / circular limits: pads up to N - 1 / N
    (40011, 2, 31, 1, 1, 15, 15), (40011, 1, 63, 1, 1, 62, 0), (20000, 2, 15, 1, 3, 21, 21),
    (50011, 2, 8, 1, 2, 7, 7), (64, 2, 9, 1, 1, 63, 63), (64, 2, 5, 2, 3, 64, 64), (7, 3, 3, 1, 1, 6, 2),
    (200003, 1, 256, 1, 1, 255, 255), (30000, 2, 1024, 1, 1, 600, 423),
]


def mode_ok(mode, N, pl, pr):
    lim = {"reflect": N - 1, "circular": N}.get(mode, 1 << 30)
    return pl <= lim and pr <= lim


@pytest.mark.parametrize("mode", ["reflect", "circular", "replicate"])
@pytest.mark.parametrize("N,B,w,s,d,pl,pr", MODE_SPECS)
def test_pad_modes(ss, mode, N, B, w, s, d, pl, pr):
    L = ss.ss_out_len_ex(N, w, s, d, pl, pr)
    if L < 0 or not mode_ok(mode, N, pl, pr):
        pytest.skip("window exceeds padded input / pad beyond the mode's limit")
    m = ss.PAD_MODES[mode]
    xi = synth.randint(12, B * N, -1000, 1000).reshape(B, N)
    ys = run(ss, ss.ss_pool_sum_ex, xi, (w, s, d, pl, pr, m, ss.SS_I32), L, 1, 2, dt=torch.int32)
    np.testing.assert_array_equal(ys, (oracle.pool_sum_ex(xi, w, s, d, pl, pr, mode) & 0xFFFFFFFF)
                                  .astype(np.uint32).view(np.int32))
    ym = run(ss, ss.ss_pool_max_ex, xi, (w, s, d, pl, pr, m, ss.SS_I32), L, dt=torch.int32)
    np.testing.assert_array_equal(ym, oracle.pool_max_ex(xi, w, s, d, pl, pr, mode))
    yn = run(ss, ss.ss_pool_min_ex, xi, (w, s, d, pl, pr, m, ss.SS_I32), L, 2, 1, dt=torch.int32)
    np.testing.assert_array_equal(yn, oracle.pool_min_ex(xi, w, s, d, pl, pr, mode))
    xf = synth.normal(13, B * N).reshape(B, N)
    ynf = run(ss, ss.ss_pool_min_ex, xf, (w, s, d, pl, pr, m, ss.SS_F32), L, 1, 1)
    np.testing.assert_array_equal(ynf, oracle.pool_min_ex(xf, w, s, d, pl, pr, mode))
    ysf = run(ss, ss.ss_pool_sum_ex, xf, (w, s, d, pl, pr, m, ss.SS_F32), L, 3, 0)
    ref, mag = oracle.pool_sum_ex(xf, w, s, d, pl, pr, mode)
    assert np.all(np.abs(ysf - ref) <= 1e-5 * mag + 1e-6)
    if w <= 64:
        f = synth.normal(14, w, sigma=synth.cfg_sigma_filter(w))
        y = run(ss, lambda xp, yp, N_, B_, *a: ss.ss_conv1d_ex(xp, yp, N_, B_, f.tolist(), w, *a),
                xf, (s, d, pl, pr, m, ss.SS_F32), L, 1, 3)
        ref, mag = oracle.conv1d_ex(xf, f, s, d, pl, pr, mode)
        err = np.abs(y.astype(np.float64) - ref)
        assert np.all(err <= 1e-5 * mag + 1e-6), float((err / (1e-5 * mag + 1e-6)).max())


MIN_SPECS = [  # (N, B, w, s): valid windows, every 1-D kernel family (tile, block, stride, tiny)
    (1 << 20, 1, 1, 1), (1 << 20, 1, 2, 1), (300001, 3, 16, 1), (300001, 2, 64, 1), (200003, 2, 300, 1),
    (100003, 2, 4096, 1), (100003, 1, 100003, 1), (300001, 2, 7, 3), (300001, 2, 64, 64), (1000, 5, 17, 2),
    (5, 2, 5, 1), (0, 1, 1, 1),
]


@pytest.mark.parametrize("N,B,w,s", MIN_SPECS)
def test_pool_min_valid(ss, N, B, w, s):
    if N == 0:  # empty input: rejected (N >= 1, ss.h), nothing launched
        with pytest.raises(Exception):
            ss.pool_min(torch.empty(0, dtype=torch.int32, device="cuda"), 1)
        return
    xi = torch.from_numpy(synth.randint(15, B * N, -(1 << 30), 1 << 30).reshape(B, N)).cuda()
    np.testing.assert_array_equal(ss.pool_min(xi, w, s).cpu().numpy(), oracle.pool_min(xi.cpu().numpy(), w, s))
    xf = torch.from_numpy(synth.normal(16, B * N).reshape(B, N)).cuda()
    np.testing.assert_array_equal(ss.pool_min(xf, w, s).cpu().numpy(), oracle.pool_min(xf.cpu().numpy(), w, s))
    # min(x) = -max(-x) bitwise on the device path too
    assert torch.equal(ss.pool_min(xf, w, s), -ss.pool_max(-xf, w, s))


def test_high_level_pad_mode_kwarg(ss):
    x = torch.from_numpy(synth.normal(17, 3 * 20001).reshape(3, 20001)).cuda()
    f = synth.normal(18, 9, sigma=synth.cfg_sigma_filter(9))
    for mode in ("reflect", "circular", "replicate"):
        y = ss.conv1d(x, f, padding=4, pad_mode=mode).cpu().numpy()
        ref, mag = oracle.conv1d_ex(x.cpu().numpy(), f, 1, 1, 4, 4, mode)
        assert np.all(np.abs(y - ref) <= 1e-5 * mag + 1e-6)
        ym = ss.pool_min(x, 9, padding=(8, 0), pad_mode=mode).cpu().numpy()
        np.testing.assert_array_equal(ym, oracle.pool_min_ex(x.cpu().numpy(), 9, 1, 1, 8, 0, mode))
    with pytest.raises(Exception):
        ss.pool_sum(x, 3, padding=20001, pad_mode="reflect")
