"""Pins of the oracle's tolerance magnitudes (the `absmag` output).

Every fp32 parity bound in the GPU tests is BASELINE.json's
|y - y_ref| <= 1e-5 * sum_j |term_j| + 1e-6 (Sec. 2.5 l.86-87 for the
dot product; the same form for sums, gradients and 2-D windows, R11,
R16-R18, R21).  The oracle emits sum_j |term_j| per output; these tests pin
that output against an independent computation: the same linear operator
evaluated by torch in float64 on the ABSOLUTE values of its operands (every term
is then non-negative, so the operator's value equals the sum of the term
magnitudes).  All inputs are signed, so a dropped fabs, a double-counted or a
missing term changes the result.  No GPU; torch is a test-only library routine.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F
from torch.nn import grad as tgrad

import oracle
import synth

TOL = dict(rtol=1e-12, atol=1e-12)
TORCH_MODE = {"reflect": "reflect", "circular": "circular", "replicate": "replicate", "zeros": "constant"}


def t64(a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(np.float64))


def signed(seed, n):
    return synth.normal(seed, n)


# ------------------------------------------------------------- 1-D forward, pad modes (oracle.c l.205-301)
@pytest.mark.parametrize("mode", ["zeros", "reflect", "circular", "replicate"])
@pytest.mark.parametrize("w,s,d,pl,pr", [(3, 1, 1, 2, 2), (7, 2, 1, 3, 1), (5, 1, 3, 4, 6), (1, 1, 1, 1, 0),
                                          (16, 3, 2, 9, 7)])
def test_pool_sum_ex_absmag(mode, w, s, d, pl, pr):
    n = 61
    x = signed(201, 2 * n).reshape(2, n)
    y, mag = oracle.pool_sum_ex(x, w, s=s, d=d, pl=pl, pr=pr, mode=mode)
    xp = F.pad(t64(x).abs().unsqueeze(1), (pl, pr), mode=TORCH_MODE[mode])
    ref = F.conv1d(xp, torch.ones(1, 1, w, dtype=torch.float64), stride=s, dilation=d).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    # and the value itself is the same operator on the signed input
    xs = F.pad(t64(x).unsqueeze(1), (pl, pr), mode=TORCH_MODE[mode])
    np.testing.assert_allclose(y, F.conv1d(xs, torch.ones(1, 1, w, dtype=torch.float64), stride=s,
                                           dilation=d).squeeze(1).numpy(), **TOL)
    assert np.all(mag >= np.abs(y) - 1e-12)
    if w > 1:  # several signed terms per output
        assert np.any(mag > np.abs(y) + 1e-9)


@pytest.mark.parametrize("mode", ["zeros", "reflect", "circular", "replicate"])
@pytest.mark.parametrize("k,s,d,pl,pr", [(3, 1, 1, 2, 2), (7, 2, 1, 3, 1), (5, 1, 3, 4, 6), (31, 1, 1, 15, 15)])
def test_conv1d_ex_absmag(mode, k, s, d, pl, pr):
    n = 97
    x = signed(202, 3 * n).reshape(3, n)
    f = signed(203, k)
    y, mag = oracle.conv1d_ex(x, f, s=s, d=d, pl=pl, pr=pr, mode=mode)
    xp = F.pad(t64(x).abs().unsqueeze(1), (pl, pr), mode=TORCH_MODE[mode])
    ref = F.conv1d(xp, t64(f).abs().view(1, 1, k), stride=s, dilation=d).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    if k > 1:
        assert np.any(mag > np.abs(y) + 1e-9)


# ------------------------------------------------------------- 2-D pooling (oracle.c l.123-155)
@pytest.mark.parametrize("kh,kw,sh,sw", [(3, 3, 1, 1), (2, 2, 2, 2), (3, 5, 2, 1), (4, 3, 3, 2)])
def test_pool2d_absmag_signed(kh, kw, sh, sw):
    x = signed(204, 3 * 23 * 19).reshape(3, 23, 19)
    y, mag = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_AVG)
    ref = F.avg_pool2d(t64(x).abs().unsqueeze(1), (kh, kw), (sh, sw)).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref, rtol=1e-13, atol=1e-15)
    assert np.any(mag > np.abs(y) + 1e-9)
    _, mag_max = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_MAX)
    assert np.all(mag_max == 0.0)  # max is exact: no rounding budget


# ------------------------------------------------------------- 2-D convolution (oracle.c l.529-547)
@pytest.mark.parametrize("kh,kw,sh,sw", [(3, 3, 1, 1), (5, 5, 1, 1), (7, 7, 2, 2), (1, 3, 1, 2), (3, 1, 3, 1)])
def test_conv2d_absmag(kh, kw, sh, sw):
    x = signed(205, 2 * 21 * 26).reshape(2, 21, 26)
    f = signed(206, kh * kw).reshape(kh, kw)
    y, mag = oracle.conv2d(x, f, sh, sw)
    ref = F.conv2d(t64(x).abs().unsqueeze(1), t64(f).abs().view(1, 1, kh, kw), stride=(sh, sw)).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    assert np.any(mag > np.abs(y) + 1e-9)


# ------------------------------------------------------------- 1-D gradients (oracle.c l.398-480)
@pytest.mark.parametrize("w,s", [(1, 1), (3, 1), (16, 1), (4, 3), (5, 2)])
def test_pool_sum_backward_absmag(w, s):
    N = 83
    L = (N - w) // s + 1
    dy = signed(207, 2 * L).reshape(2, L)
    dx, mag = oracle.pool_sum_backward(dy, N, w, s)
    ref = tgrad.conv1d_input((2, 1, N), torch.ones(1, 1, w, dtype=torch.float64), t64(dy).abs().unsqueeze(1),
                             stride=s).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    if w > 1:
        assert np.any(mag > np.abs(dx) + 1e-9)


@pytest.mark.parametrize("k,s", [(1, 1), (3, 1), (7, 2), (31, 1), (63, 1), (5, 4)])
def test_conv1d_backward_input_absmag(k, s):
    N = 150
    L = (N - k) // s + 1
    dy = signed(208, 2 * L).reshape(2, L)
    f = signed(209, k)
    dx, mag = oracle.conv1d_backward_input(dy, f, N, s)
    ref = tgrad.conv1d_input((2, 1, N), t64(f).abs().view(1, 1, k), t64(dy).abs().unsqueeze(1),
                             stride=s).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    if k > 1:
        assert np.any(mag > np.abs(dx) + 1e-9)


@pytest.mark.parametrize("k,s", [(1, 1), (3, 1), (7, 2), (31, 1), (63, 1), (5, 4)])
def test_conv1d_backward_filter_absmag(k, s):
    N = 150
    L = (N - k) // s + 1
    x = signed(210, 3 * N).reshape(3, N)
    dy = signed(211, 3 * L).reshape(3, L)
    df, mag = oracle.conv1d_backward_filter(x, dy, k, s)
    ref = tgrad.conv1d_weight(t64(x).abs().unsqueeze(1), (1, 1, k), t64(dy).abs().unsqueeze(1),
                              stride=s).view(k).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    assert np.any(mag > np.abs(df) + 1e-9)


# ------------------------------------------------------------- 2-D pooling gradient (oracle.c l.485-523)
@pytest.mark.parametrize("kh,kw,sh,sw", [(3, 3, 1, 1), (2, 2, 2, 2), (3, 2, 2, 1)])
def test_pool2d_backward_absmag(kh, kw, sh, sw):
    P, H, W = 2, 17, 14
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    x = signed(212, P * H * W).reshape(P, H, W)  # distinct values: one maximum per window
    dy = signed(213, P * OH * OW).reshape(P, OH, OW)
    # avg: the scatter of |dy|/(kh kw) over each window
    dx, mag = oracle.pool2d_backward(None, dy, H, W, kh, kw, sh, sw, oracle.POOL2D_AVG)
    xt = torch.zeros(P, 1, H, W, dtype=torch.float64, requires_grad=True)
    F.avg_pool2d(xt, (kh, kw), (sh, sw)).backward(t64(dy).abs().unsqueeze(1))
    np.testing.assert_allclose(mag, xt.grad.squeeze(1).numpy(), rtol=1e-13, atol=1e-15)
    if kh > sh or kw > sw:
        assert np.any(mag > np.abs(dx) + 1e-9)
    # max: |dy| routed to each window's maximum
    dx, mag = oracle.pool2d_backward(x, dy, H, W, kh, kw, sh, sw, oracle.POOL2D_MAX)
    xt = t64(x).unsqueeze(1).requires_grad_(True)
    F.max_pool2d(xt, (kh, kw), (sh, sw)).backward(t64(dy).abs().unsqueeze(1))
    np.testing.assert_allclose(mag, xt.grad.squeeze(1).numpy(), rtol=1e-13, atol=1e-15)
    if kh > sh or kw > sw:  # overlapping windows: some position collects signed dy of several windows
        assert np.any(mag > np.abs(dx) + 1e-9)


# ------------------------------------------------------------- 2-D convolution gradients (oracle.c l.554-594)
@pytest.mark.parametrize("kh,kw,sh,sw", [(3, 3, 1, 1), (5, 5, 1, 1), (7, 7, 2, 2), (1, 3, 1, 2), (3, 2, 3, 1)])
def test_conv2d_backward_absmag(kh, kw, sh, sw):
    P, H, W = 2, 19, 23
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    x = signed(214, P * H * W).reshape(P, H, W)
    dy = signed(215, P * OH * OW).reshape(P, OH, OW)
    f = signed(216, kh * kw).reshape(kh, kw)
    dx, mag = oracle.conv2d_backward_input(dy, f, H, W, sh, sw)
    ref = tgrad.conv2d_input((P, 1, H, W), t64(f).abs().view(1, 1, kh, kw), t64(dy).abs().unsqueeze(1),
                             stride=(sh, sw)).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    assert np.any(mag > np.abs(dx) + 1e-9)
    df, mag = oracle.conv2d_backward_filter(x, dy, kh, kw, sh, sw)
    ref = tgrad.conv2d_weight(t64(x).abs().unsqueeze(1), (1, 1, kh, kw), t64(dy).abs().unsqueeze(1),
                              stride=(sh, sw)).view(kh, kw).numpy()
    np.testing.assert_allclose(mag, ref, **TOL)
    assert np.any(mag > np.abs(df) + 1e-9)


# ------------------------------------------------------------- multi-channel conv (oracle.c l.609-627)
@pytest.mark.parametrize("cin,cout,k", [(4, 3, 3), (16, 8, 5), (64, 64, 1)])
def test_conv1d_mc_absmag(cin, cout, k):
    B, N = 2, 40
    xb = oracle.to_bf16_bits(signed(217, B * N * cin).reshape(B, N, cin))
    wb = oracle.to_bf16_bits(signed(218, cout * cin * k).reshape(cout, cin, k))
    y, mag = oracle.conv1d_mc(xb, wb)
    xf = t64(oracle.bf16_bits_to_f32(xb)).abs().permute(0, 2, 1)  # [B, Cin, N]
    wf = t64(oracle.bf16_bits_to_f32(wb)).abs()
    ref = F.conv1d(xf, wf).permute(0, 2, 1).numpy()  # [B, L, Cout]
    np.testing.assert_allclose(mag, ref, **TOL)
    assert np.any(mag > np.abs(y) + 1e-9)
