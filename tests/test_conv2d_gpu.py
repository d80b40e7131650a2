"""GPU parity of the 2-D single-channel sliding dot product (csrc/conv2d.cu;
SURVEY 8f NEXT #4, the multi-dimensional extension of PAPER.md l.226) against
oracle.conv2d: vector-kernel shapes (3x3 / 5x5 / 7x7 / 1x3 / 3x1 at stride 1,
column stride 2), the direct kernel (other strides, odd widths, misaligned x),
canaries, integer exactness and a config-4-sized sampled check."""
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


def run(ss, x, f, sh, sw, xoff=0):
    P, H, W = x.shape
    kh, kw = f.shape
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    xb = torch.zeros(x.size + xoff + 4, device="cuda")
    xb[xoff:xoff + x.size] = torch.from_numpy(x.reshape(-1)).cuda()
    yb = torch.full((P * OH * OW + 6,), -99.0, device="cuda")
    y = yb[1:1 + P * OH * OW]
    ss.check(ss.ss_conv2d(xb[xoff:].data_ptr(), y.data_ptr(), P, H, W, f.reshape(-1).tolist(), kh, kw, sh, sw))
    torch.cuda.synchronize()
    h = yb.cpu().numpy()
    assert h[0] == -99.0 and np.all(h[1 + P * OH * OW:] == -99.0), "canary overwritten"
    return y.cpu().numpy().reshape(P, OH, OW)


CASES = [  # (P, H, W, kh, kw, sh, sw)
    (3, 112, 112, 3, 3, 1, 1), (2, 112, 112, 5, 5, 1, 1), (2, 64, 96, 7, 7, 1, 1), (3, 40, 36, 1, 3, 1, 1),
    (2, 40, 36, 3, 1, 1, 1), (2, 112, 112, 3, 3, 1, 2), (2, 30, 44, 5, 5, 1, 2), (2, 112, 112, 3, 3, 2, 2),
    (3, 31, 29, 3, 3, 1, 1), (1, 17, 200, 4, 6, 3, 2), (2, 9, 9, 9, 9, 1, 1), (1, 5, 1000, 2, 33, 1, 1),
    # the round-2 FFMA2 tile kernel (stride-1 5x5 / 7x7): TMA mode (16-B rows), dense mode (even
    # rows of other widths), ragged units, a plane of one unit, an odd width (direct kernel)
    (3, 112, 112, 7, 7, 1, 1), (2, 50, 114, 7, 7, 1, 1), (2, 23, 58, 5, 5, 1, 1), (1, 7, 7, 7, 7, 1, 1),
    (2, 40, 113, 7, 7, 1, 1), (1, 250, 250, 5, 5, 1, 1), (3, 19, 36, 7, 7, 1, 1),
]


@pytest.mark.parametrize("P,H,W,kh,kw,sh,sw", CASES)
def test_conv2d(ss, P, H, W, kh, kw, sh, sw):
    x = synth.normal(60, P * H * W).reshape(P, H, W)
    f = synth.normal(61, kh * kw, sigma=(kh * kw) ** -0.5).reshape(kh, kw)
    y = run(ss, x, f, sh, sw)
    ref, mag = oracle.conv2d(x, f, sh, sw)
    err = np.abs(y.astype(np.float64) - ref)
    assert np.all(err <= TOL_REL * mag + TOL_ABS), float((err / (TOL_REL * mag + TOL_ABS)).max())


def test_conv2d_misaligned_and_integer_exact(ss):
    x = synth.randint(62, 2 * 112 * 112, -1000, 1000).astype(np.float32).reshape(2, 112, 112)
    f = synth.randint(63, 9, -3, 3).astype(np.float32).reshape(3, 3)
    ref, _ = oracle.conv2d(x, f)
    for xoff in (0, 1):  # 16-B aligned -> vector kernel; offset by 1 -> direct kernel
        np.testing.assert_array_equal(run(ss, x, f, 1, 1, xoff).astype(np.float64), ref)


def test_conv2d_cfg4_sampled(ss):
    x = torch.empty((32, 64, 112, 112), device="cuda")
    synth.fill_device(x, "u01", 5)
    f = synth.normal(64, 9, sigma=1 / 3).reshape(3, 3)
    y = ss.conv2d(x, f).cpu().numpy().reshape(2048, 110, 110)
    xh = synth.uniform01(5, 32 * 64 * 112 * 112).reshape(2048, 112, 112)
    for pl in (0, 1, 777, 2047):
        ref, mag = oracle.conv2d(xh[pl:pl + 1], f)
        assert np.all(np.abs(y[pl] - ref[0]) <= TOL_REL * mag[0] + TOL_ABS)
