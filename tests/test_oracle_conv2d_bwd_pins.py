"""Pins of the oracle's 2-D convolution gradients (oracle/oracle.c
oracle_conv2d_backward_input_f32 / _filter_f32; SURVEY 8f NEXT #4 "2-D
convolution and backward passes"; reading R21: the vector-Jacobian
products of the 2-D sliding dot product, PAPER.md l.226 multi-dimensional
extension of Sec. 2.5).

Independent of the oracle's code: a hand-worked case, torch float64 autograd of
F.conv2d (with stride), the adjoint identities <conv2d(x), dy> = <x, dx> and
<f, df> = <conv2d(x, f), dy>, finite differences, and the special case kh = 1
that reduces each image row to the 1-D gradients."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth


def test_hand_values():
    # x 3x3 = 1..9, f 2x2 = [[1, 2], [3, 4]], dy 2x2 = [[1, 0], [0, 0]] (only output (0,0))
    x = np.arange(1, 10, dtype=np.float32).reshape(1, 3, 3)
    f = np.array([[1, 2], [3, 4]], np.float32)
    dy = np.array([[[1, 0], [0, 0]]], np.float32)
    dx, _ = oracle.conv2d_backward_input(dy, f, 3, 3)
    np.testing.assert_array_equal(dx[0], [[1, 2, 0], [3, 4, 0], [0, 0, 0]])
    df, _ = oracle.conv2d_backward_filter(x, dy, 2, 2)
    np.testing.assert_array_equal(df, [[1, 2], [4, 5]])  # the window under output (0, 0)
    # all-ones dy: dx counts weighted taps; df = sum of each shifted window
    dy1 = np.ones((1, 2, 2), np.float32)
    dx, _ = oracle.conv2d_backward_input(dy1, f, 3, 3)
    np.testing.assert_array_equal(dx[0], [[1, 3, 2], [4, 10, 6], [3, 7, 4]])
    df, _ = oracle.conv2d_backward_filter(x, dy1, 2, 2)
    np.testing.assert_array_equal(df, [[1 + 2 + 4 + 5, 2 + 3 + 5 + 6], [4 + 5 + 7 + 8, 5 + 6 + 8 + 9]])


@pytest.mark.parametrize("P,H,W,kh,kw,sh,sw", [(2, 9, 11, 3, 3, 1, 1), (3, 16, 13, 5, 2, 2, 3),
                                               (1, 20, 20, 7, 7, 3, 2), (2, 6, 30, 1, 9, 1, 4),
                                               (1, 8, 8, 8, 8, 1, 1), (2, 12, 10, 4, 3, 5, 5)])
def test_against_torch_autograd(P, H, W, kh, kw, sh, sw):
    x = synth.normal(70, P * H * W).reshape(P, H, W)
    f = synth.normal(71, kh * kw).reshape(kh, kw)
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    dy = synth.normal(72, P * OH * OW).reshape(P, OH, OW)
    xt = torch.from_numpy(x.astype(np.float64)).view(P, 1, H, W).requires_grad_()
    ft = torch.from_numpy(f.astype(np.float64)).view(1, 1, kh, kw).requires_grad_()
    y = F.conv2d(xt, ft, stride=(sh, sw))
    y.backward(torch.from_numpy(dy.astype(np.float64)).view_as(y))
    dx, mx = oracle.conv2d_backward_input(dy, f, H, W, sh, sw)
    df, mf = oracle.conv2d_backward_filter(x, dy, kh, kw, sh, sw)
    np.testing.assert_allclose(dx, xt.grad.view(P, H, W).numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(df, ft.grad.view(kh, kw).numpy(), rtol=0, atol=1e-11)
    assert np.all(mx >= np.abs(dx) - 1e-12) and np.all(mf >= np.abs(df) - 1e-12)


def test_adjoint_identities():
    P, H, W, kh, kw, sh, sw = 3, 17, 23, 4, 5, 2, 3
    x = synth.normal(73, P * H * W).reshape(P, H, W)
    f = synth.normal(74, kh * kw).reshape(kh, kw)
    y, _ = oracle.conv2d(x, f, sh, sw)
    dy = synth.normal(75, y.size).reshape(y.shape)
    dx, _ = oracle.conv2d_backward_input(dy, f, H, W, sh, sw)
    df, _ = oracle.conv2d_backward_filter(x, dy, kh, kw, sh, sw)
    lhs = float(np.sum(y * dy.astype(np.float64)))
    assert abs(lhs - float(np.sum(x.astype(np.float64) * dx))) < 1e-9 * max(1.0, abs(lhs))
    assert abs(lhs - float(np.sum(f.astype(np.float64) * df))) < 1e-9 * max(1.0, abs(lhs))
    # rows/cols no window reaches (W - 1 > (OW - 1) sw + kw - 1) get exactly 0
    OW = y.shape[2]
    last = (OW - 1) * sw + kw
    assert np.all(dx[:, :, last:] == 0)


def test_finite_difference_filter():
    P, H, W, kh, kw = 1, 7, 8, 3, 2
    x = synth.normal(76, P * H * W).reshape(P, H, W).astype(np.float64)
    f = synth.normal(77, kh * kw).reshape(kh, kw).astype(np.float64)
    dy = synth.normal(78, P * 5 * 7).reshape(P, 5, 7).astype(np.float64)
    df, _ = oracle.conv2d_backward_filter(x, dy, kh, kw)
    # the loss is linear in f, so a unit step is exact: L(f + e_ab) - L(f) = df[a][b]
    base = float(np.sum(oracle.conv2d(x, f)[0] * dy))
    for a in range(kh):
        for b in range(kw):
            e = f.copy()
            e[a, b] += 1.0
            d = float(np.sum(oracle.conv2d(x, e)[0] * dy)) - base
            assert abs(d - df[a, b]) < 1e-5


def test_kh1_reduces_to_rows_of_1d():
    P, H, W, k, s = 2, 5, 40, 7, 3
    x = synth.normal(79, P * H * W).reshape(P, H, W)
    f = synth.normal(80, k)
    L = (W - k) // s + 1
    dy = synth.normal(81, P * H * L).reshape(P, H, L)
    dx, _ = oracle.conv2d_backward_input(dy, f.reshape(1, k), H, W, 1, s)
    dx1, _ = oracle.conv1d_backward_input(dy.reshape(P * H, L), f, W, s)
    np.testing.assert_allclose(dx.reshape(P * H, W), dx1, rtol=0, atol=1e-12)
    df, _ = oracle.conv2d_backward_filter(x, dy, 1, k, 1, s)
    df1, _ = oracle.conv1d_backward_filter(x.reshape(P * H, W), dy.reshape(P * H, L), k, s)
    np.testing.assert_allclose(df.reshape(k), df1, rtol=0, atol=1e-10)
