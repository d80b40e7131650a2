"""GPU parity of the 2-D convolution gradients (ss_conv2d_backward_input /
ss_conv2d_backward_filter, reading R21) against the
oracle (oracle_conv2d_backward_*_f32) on the same seeded inputs, element by
element within the BJ bound 1e-5 * sum|terms| + 1e-6.  Covers every kernel
variant (staged gather tile at stride 1 and strided, register / tap / direct
filter kernels), ragged tiles, uncovered edge elements (written 0), the
config-4 shape at full size, validation, and determinism."""
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


CASES = [  # (planes, H, W, kh, kw, sh, sw)
    (3, 37, 150, 3, 3, 1, 1), (2, 41, 259, 4, 2, 2, 3), (2, 30, 140, 5, 5, 1, 1), (2, 50, 301, 7, 7, 2, 2),
    (1, 17, 200, 1, 9, 1, 1), (2, 64, 33, 9, 1, 1, 1), (1, 80, 300, 31, 31, 1, 1), (1, 40, 40, 32, 32, 1, 1),
    (1, 1030, 3, 1024, 1, 1, 1), (1, 9, 700, 2, 300, 3, 5), (5, 8, 8, 8, 8, 1, 1), (4, 3, 3, 3, 3, 1, 1),
    (2, 23, 129, 3, 4, 3, 1), (1, 200, 1000, 6, 3, 7, 2),
]


def _grads(ss, x, f, dy, sh, sw):
    P, H, W = x.shape
    kh, kw = f.shape
    dxt = ss.conv2d_backward_input(torch.from_numpy(dy).cuda(), f, H, W, (sh, sw))
    dft = ss.conv2d_backward_filter(torch.from_numpy(x).cuda(), torch.from_numpy(dy).cuda(), (kh, kw), (sh, sw))
    torch.cuda.synchronize()
    return dxt.cpu().numpy(), dft.cpu().numpy()


def _check(got, ref, mag):
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * mag + 1e-6), float((err / (1e-5 * mag + 1e-6)).max())


@pytest.mark.parametrize("P,H,W,kh,kw,sh,sw", CASES)
def test_parity(ss, P, H, W, kh, kw, sh, sw):
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    x = synth.normal(90, P * H * W).reshape(P, H, W)
    f = synth.normal(91, kh * kw, sigma=synth.cfg_sigma_filter(kh * kw)).reshape(kh, kw)
    dy = synth.normal(92, P * OH * OW).reshape(P, OH, OW)
    dx, df = _grads(ss, x, f, dy, sh, sw)
    ref, mag = oracle.conv2d_backward_input(dy, f, H, W, sh, sw)
    _check(dx, ref, mag)
    assert np.all(dx[mag == 0] == 0)  # elements no window covers
    ref, mag = oracle.conv2d_backward_filter(x, dy, kh, kw, sh, sw)
    _check(df, ref, mag)


def test_config4_shape_full(ss):
    # BASELINE config 4's [32, 64, 112, 112] plane stack with a 3x3 filter, every element checked
    P, H, W = 32 * 64, 112, 112
    x = synth.uniform01(93, P * H * W).reshape(P, H, W)
    f = synth.normal(94, 9, sigma=synth.cfg_sigma_filter(9)).reshape(3, 3)
    dy = synth.normal(95, P * 110 * 110).reshape(P, 110, 110)
    dx, df = _grads(ss, x, f, dy, 1, 1)
    ref, mag = oracle.conv2d_backward_input(dy, f, H, W)
    _check(dx, ref, mag)
    ref, mag = oracle.conv2d_backward_filter(x, dy, 3, 3)
    _check(df, ref, mag)


def test_integer_exact_and_deterministic(ss):
    # small integers: every partial sum is exact in fp32 / fp64, so the result is exact and
    # repeated calls agree bitwise
    P, H, W = 6, 70, 260
    x = synth.randint(96, P * H * W, -8, 8).reshape(P, H, W).astype(np.float32)
    f = synth.randint(97, 25, -4, 4).reshape(5, 5).astype(np.float32)
    dy = synth.randint(98, P * 66 * 256, -8, 8).reshape(P, 66, 256).astype(np.float32)
    dx, df = _grads(ss, x, f, dy, 1, 1)
    np.testing.assert_array_equal(dx.astype(np.float64), oracle.conv2d_backward_input(dy, f, H, W)[0])
    np.testing.assert_array_equal(df.astype(np.float64), oracle.conv2d_backward_filter(x, dy, 5, 5)[0])
    for _ in range(3):
        dx2, df2 = _grads(ss, x, f, dy, 1, 1)
        assert np.array_equal(dx, dx2) and np.array_equal(df, df2)


def test_validation(ss):
    FX, FY = 0x10000000, 0x20000000
    f9 = [1.0] * 9
    assert ss.ss_conv2d_backward_input(FX, FY, 1, 2, 5, f9, 3, 3) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv2d_backward_input(FX, FY, 0, 5, 5, f9, 3, 3) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv2d_backward_input(FX, FY, 1, 5, 5, f9, 3, 3, dtype=ss.SS_I32) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_conv2d_backward_input(FX, FX, 1, 5, 5, f9, 3, 3) == ss.SS_ERR_OVERLAP
    need = ss.ss_conv2d_backward_filter_workspace(3, 3)
    assert need > 0 and ss.ss_conv2d_backward_filter_workspace(33, 32) == 0
    assert ss.ss_conv2d_backward_filter(FX, FY, 0x30000000, 1, 5, 5, 3, 3, 1, 1, 0x40000000, need - 8) == \
        ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv2d_backward_filter(FX, FY, 0x30000000, 1, 5, 5, 3, 3, 1, 1, 0, need) == ss.SS_ERR_NULL
