"""Pins of the backward-pass oracle (the abstract's "training",
PAPER.md l.7) against things other than itself:
  * the adjoint identity <A x, dy> = <x, A^T dy> (and <conv(x, f), dy> = <f, df>)
    with the FORWARD oracle supplying A x, exact in integers;
  * finite differences of sum_i dy_i max_i(x) on distinct values (max);
  * hand-worked values and closed forms (coverage counts, delta filters);
  * torch float64 autograd (a library routine, test-only).
No GPU."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth


def ints(seed, n, lo=-9, hi=9):
    return synth.randint(seed, n, lo, hi).astype(np.float32)


# ------------------------------------------------------------------ hand values
def test_hand_values():
    # dy = [1, 2, 3], N = 4, w = 2: dx = [1, 1+2, 2+3, 3]
    dx, mag = oracle.pool_sum_backward(np.array([1, 2, 3], np.float32), 4, 2)
    np.testing.assert_array_equal(dx, [1, 3, 5, 3])
    # max ties route to the FIRST maximum: x = [1, 1, 1], w = 2 -> windows' argmax 0, 1
    np.testing.assert_array_equal(oracle.pool_max_backward(np.ones(3, np.float32), np.array([5, 7], np.float32), 2),
                                  [5, 7, 0])
    # x = [1, 3, 2, 5, 4], w = 3 (SPEC.md l.186 forward: [3, 5, 5]) -> argmax 1, 3, 3
    np.testing.assert_array_equal(
        oracle.pool_max_backward(np.array([1, 3, 2, 5, 4], np.float32), np.array([1, 10, 100], np.float32), 3),
        [0, 1, 0, 110, 0])
    # conv [1,2,3,4] * [1,0,-1] -> [-2,-2]; dx = dy0 f shifted + dy1 f shifted
    dx, _ = oracle.conv1d_backward_input(np.array([1, 10], np.float32), np.array([1, 0, -1], np.float32), 4)
    np.testing.assert_array_equal(dx, [1, 10, -1, -10])
    # df_j = sum_i dy_i x_{i+j}: x = [1,2,3,4], dy = [1,1], k = 3 -> [3, 5, 7]
    df, _ = oracle.conv1d_backward_filter(np.array([1, 2, 3, 4], np.float32), np.array([1, 1], np.float32), 3)
    np.testing.assert_array_equal(df, [3, 5, 7])
    # stride 2: x = [1..6], w = 2, s = 2 -> windows {0,1},{2,3},{4,5}: dx = dy repeated
    dx, _ = oracle.pool_sum_backward(np.array([1, 2, 3], np.float32), 6, 2, 2)
    np.testing.assert_array_equal(dx, [1, 1, 2, 2, 3, 3])


# ------------------------------------------------------------------ adjoint identities (exact)
@pytest.mark.parametrize("N,B,w,s", [(1, 1, 1, 1), (7, 2, 3, 1), (40, 3, 5, 2), (33, 2, 33, 1), (100, 2, 9, 4),
                                     (64, 1, 1, 3)])
def test_pool_sum_adjoint(N, B, w, s):
    x = synth.randint(1, B * N, -50, 50).reshape(B, N)
    L = oracle.out_len(N, w, s)
    dy = ints(2, B * L).reshape(B, L)
    Ax = oracle.pool_sum(x, w, s)                      # forward oracle, exact int64
    dx, mag = oracle.pool_sum_backward(dy, N, w, s)
    lhs = int(np.sum(Ax * dy.astype(np.int64)))
    rhs = float(np.sum(x.astype(np.float64) * dx))
    assert lhs == rhs
    assert np.all(mag >= np.abs(dx))


@pytest.mark.parametrize("N,B,k,s", [(5, 1, 1, 1), (20, 2, 3, 1), (50, 3, 7, 2), (31, 1, 31, 1), (90, 2, 12, 5)])
def test_conv_adjoints(N, B, k, s):
    x = ints(3, B * N).reshape(B, N)
    f = ints(4, k, -5, 5)
    L = oracle.out_len(N, k, s)
    dy = ints(5, B * L).reshape(B, L)
    y, _ = oracle.conv1d(x, f, s)                       # forward oracle (exact: small integers)
    lhs = float(np.sum(y * dy))
    dx, _ = oracle.conv1d_backward_input(dy, f, N, s)
    assert lhs == float(np.sum(x.astype(np.float64) * dx))      # <A x, dy> = <x, A^T dy>
    df, _ = oracle.conv1d_backward_filter(x, dy, k, s)
    assert lhs == float(np.sum(f.astype(np.float64) * df))      # linear in f too


@pytest.mark.parametrize("P,H,W,kh,kw,sh,sw", [(2, 6, 7, 2, 2, 2, 2), (1, 9, 9, 3, 3, 1, 1), (3, 8, 10, 2, 4, 1, 3)])
def test_pool2d_avg_adjoint(P, H, W, kh, kw, sh, sw):
    x = ints(6, P * H * W).reshape(P, H, W)
    y, _ = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_AVG)
    dy = ints(7, y.size).reshape(y.shape)
    dx, _ = oracle.pool2d_backward(None, dy, H, W, kh, kw, sh, sw, oracle.POOL2D_AVG)
    lhs, rhs = float(np.sum(y * dy)), float(np.sum(x.astype(np.float64) * dx))
    assert abs(lhs - rhs) <= 1e-12 * (1 + abs(lhs))   # 1/(kh kw) not dyadic in general


# ------------------------------------------------------------------ finite differences (max)
@pytest.mark.parametrize("N,w,s", [(20, 3, 1), (31, 4, 2), (16, 16, 1), (25, 5, 3)])
def test_pool_max_finite_difference(N, w, s):
    rng = np.random.default_rng(N * 7 + w)
    x = rng.permutation(N).astype(np.float32)          # distinct values, gaps >= 1
    L = oracle.out_len(N, w, s)
    dy = ints(8, L)
    Fx = float(np.sum(oracle.pool_max(x, w, s).astype(np.float64) * dy))
    dx = oracle.pool_max_backward(x, dy, w, s)
    h = 0.25                                           # exact in fp32, below every gap
    for t in range(N):
        xp = x.copy()
        xp[t] += h
        Fp = float(np.sum(oracle.pool_max(xp, w, s).astype(np.float64) * dy))
        assert (Fp - Fx) / h == dx[t]


def test_pool2d_max_finite_difference():
    rng = np.random.default_rng(5)
    P, H, W, kh, kw, sh, sw = 2, 7, 8, 3, 2, 2, 1
    x = rng.permutation(P * H * W).astype(np.float32).reshape(P, H, W)
    y, _ = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_MAX)
    dy = ints(9, y.size).reshape(y.shape)
    dx, _ = oracle.pool2d_backward(x, dy, H, W, kh, kw, sh, sw, oracle.POOL2D_MAX)
    Fx = float(np.sum(y * dy))
    for t in range(x.size):
        xp = x.copy().reshape(-1)
        xp[t] += 0.25
        yp, _ = oracle.pool2d(xp.reshape(P, H, W), kh, kw, sh, sw, oracle.POOL2D_MAX)
        assert (float(np.sum(yp * dy)) - Fx) / 0.25 == dx.reshape(-1)[t]


# ------------------------------------------------------------------ closed forms
@pytest.mark.parametrize("N,w", [(10, 3), (10, 10), (7, 1), (50, 8)])
def test_pool_sum_backward_coverage_count(N, w):
    # dy = 1, stride 1: dx_t = number of windows covering t
    L = N - w + 1
    dx, _ = oracle.pool_sum_backward(np.ones(L, np.float32), N, w)
    t = np.arange(N)
    cover = np.minimum(t, L - 1) - np.maximum(0, t - w + 1) + 1
    np.testing.assert_array_equal(dx, cover)


def test_conv_backward_delta_filters():
    x = synth.normal(10, 60)
    L = 60 - 5 + 1
    dy = synth.normal(11, L)
    for m in range(5):
        f = np.zeros(5, np.float32)
        f[m] = 1.0
        dx, _ = oracle.conv1d_backward_input(dy, f, 60)
        want = np.zeros(60)
        want[m:m + L] = dy
        np.testing.assert_array_equal(dx, want)         # e_m: dy shifted by m
    for i in (0, 7, L - 1):
        e = np.zeros(L, np.float32)
        e[i] = 1.0
        df, _ = oracle.conv1d_backward_filter(x, e, 5)
        np.testing.assert_array_equal(df, x[i:i + 5].astype(np.float64))  # dy = e_i picks x's window i


# ------------------------------------------------------------------ torch float64 autograd (library routine)
def test_torch_autograd_cross_check():
    B, N, k, s = 3, 200, 9, 2
    x = synth.normal(12, B * N).reshape(B, N)
    f = synth.normal(13, k)
    L = oracle.out_len(N, k, s)
    dy = synth.normal(14, B * L).reshape(B, L)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    ft = torch.tensor(f, dtype=torch.float64, requires_grad=True)
    yt = F.conv1d(xt[:, None, :], ft[None, None, :], stride=s)[:, 0, :]
    yt.backward(torch.tensor(dy, dtype=torch.float64))
    dx, _ = oracle.conv1d_backward_input(dy, f, N, s)
    df, _ = oracle.conv1d_backward_filter(x, dy, k, s)
    np.testing.assert_allclose(dx, xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(df, ft.grad.numpy(), rtol=1e-12, atol=1e-11)
    # pooling: avg_pool1d * w is the sliding sum; max on distinct values
    w = 6
    L = oracle.out_len(N, w, s)
    dy = synth.normal(15, B * L).reshape(B, L)
    xt = torch.tensor(x, dtype=torch.float64, requires_grad=True)
    (F.avg_pool1d(xt[:, None, :], w, s)[:, 0, :] * w).backward(torch.tensor(dy, dtype=torch.float64))
    np.testing.assert_allclose(oracle.pool_sum_backward(dy, N, w, s)[0], xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    xd = np.random.default_rng(1).permutation(B * N).astype(np.float32).reshape(B, N)
    xt = torch.tensor(xd, dtype=torch.float64, requires_grad=True)
    F.max_pool1d(xt[:, None, :], w, s)[:, 0, :].backward(torch.tensor(dy, dtype=torch.float64))
    np.testing.assert_allclose(oracle.pool_max_backward(xd, dy, w, s), xt.grad.numpy(), rtol=1e-12, atol=1e-12)
    # 2-D
    x2 = np.random.default_rng(2).permutation(2 * 11 * 12).astype(np.float32).reshape(2, 11, 12)
    for mode, fn in ((oracle.POOL2D_MAX, F.max_pool2d), (oracle.POOL2D_AVG, F.avg_pool2d)):
        xt = torch.tensor(x2, dtype=torch.float64, requires_grad=True)
        yt = fn(xt[:, None], (3, 2), (2, 1))[:, 0]
        dy2 = synth.normal(16, yt.numel()).reshape(tuple(yt.shape))
        yt.backward(torch.tensor(dy2, dtype=torch.float64))
        dx, _ = oracle.pool2d_backward(x2, dy2, 11, 12, 3, 2, 2, 1, mode)
        np.testing.assert_allclose(dx, xt.grad.numpy(), rtol=1e-12, atol=1e-12)
