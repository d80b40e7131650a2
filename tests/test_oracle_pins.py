"""Pins for the CPU oracle (oracle/): each check ties an oracle routine to
something other than itself -- values printed in the spec written from the
paper (tests/golden/spec_examples.json), closed forms, invariants, brute force
on tiny inputs, and independent library routines (numpy cumsum, torch float64
pooling/conv) -- so that a dropped term, a wrong sign or index, or a transposed
operand in oracle.c fails at least one of them.

CPU only (no GPU marker)."""
import itertools
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- golden values
@pytest.mark.parametrize("case", GOLD["sliding_sum"], ids=lambda c: c["cite"])
def test_golden_sliding_sum(case):
    x = np.array(case["x"], np.int32)
    if case["op"] == "add":
        y = oracle.pool_sum(x, case["w"])
        np.testing.assert_array_equal(y, np.array(case["y"], np.int64))
        yf, _ = oracle.pool_sum(x.astype(np.float32), case["w"])
        np.testing.assert_array_equal(yf, np.array(case["y"], np.float64))
    else:
        np.testing.assert_array_equal(oracle.pool_max(x, case["w"]), np.array(case["y"], np.int32))
        np.testing.assert_array_equal(oracle.pool_max(x.astype(np.float32), case["w"]),
                                      np.array(case["y"], np.float32))


@pytest.mark.parametrize("case", GOLD["avg_pool"], ids=lambda c: c["cite"])
def test_golden_avg_pool(case):
    # SPEC avg_pool = sliding + divided by w (reading R5: ss_pool_sum is the raw sum;
    # the 1-D average is modelled here as a 1 x w 2-D average pool).
    x = np.array(case["x"], np.float32)
    y, _ = oracle.pool_sum(x, case["w"], case["stride"])
    np.testing.assert_array_equal(y / case["w"], np.array(case["y"]))
    y2, _ = oracle.pool2d(x.reshape(1, 1, -1), 1, case["w"], 1, case["stride"], oracle.POOL2D_AVG)
    np.testing.assert_array_equal(y2.reshape(-1), np.array(case["y"]))


@pytest.mark.parametrize("case", GOLD["conv1d"], ids=lambda c: c["cite"])
def test_golden_conv1d(case):
    y, _ = oracle.conv1d(np.array(case["x"], np.float32), np.array(case["f"], np.float32))
    np.testing.assert_array_equal(y, np.array(case["y"], np.float64))


@pytest.mark.parametrize("case", GOLD["gamma_combine"], ids=lambda c: c["cite"])
def test_golden_gamma_combine(case):
    assert oracle.gamma_combine(case["gi"], case["gj"]) == tuple(case["out"])


def test_gamma_combine_noncommutative_and_associative():
    # Eq. 8 is associative but not commutative.
    a, b, c = (2.0, 3.0), (0.5, -1.0), (4.0, 0.25)
    assert oracle.gamma_combine(a, b) != oracle.gamma_combine(b, a)
    lhs = oracle.gamma_combine(oracle.gamma_combine(a, b), c)
    rhs = oracle.gamma_combine(a, oracle.gamma_combine(b, c))
    assert lhs == rhs  # dyadic values: exact


@pytest.mark.parametrize("case", GOLD["gamma_sequence"], ids=lambda c: c["cite"])
def test_golden_gamma_sequence(case):
    u, v = oracle.gamma_sequence(np.array(case["a"]), np.array(case["b"]))
    np.testing.assert_array_equal(u, case["u"])
    np.testing.assert_array_equal(v, case["v"])


@pytest.mark.parametrize("case", GOLD["gamma_dot"], ids=lambda c: c["cite"])
def test_golden_gamma_dot(case):
    v, _ = oracle.gamma_dot(np.array(case["a"], float), np.array(case["b"], float))
    assert v == case["dot"]


def test_golden_splitmix64():
    case = GOLD["splitmix64"][0]
    z = synth.splitmix64(case["seed"], np.array([case["counter"]], np.uint64))[0]
    assert int(z) == int(case["z"], 16)


# ------------------------------------------- P5: dot product is a prefix sum (Eq. 9)
def test_gamma_dot_equals_direct_dot_product():
    rng = np.random.default_rng(11)
    for trial in range(300):
        M = int(rng.integers(1, 257))
        a = rng.uniform(0.25, 2.0, M) * rng.choice([-1.0, 1.0], M)
        a[rng.random(M) < 0.25] = 0.0  # Eq. 5 masking exercised
        b = rng.normal(size=M)
        v, u = oracle.gamma_dot(a, b)
        direct = float(np.dot(a, b))
        scale = float(np.abs(a * b).sum()) + 1e-300
        assert abs(v - direct) <= 1e-10 * scale, (M, v, direct)
        # u(delta_M) = prod u_i telescopes to alpha_0 (Eq. 7)
        alpha0 = 1.0 if a[0] == 0.0 else a[0]
        assert abs(u - alpha0) <= 1e-12 * abs(alpha0)


def test_gamma_masking_identity_eq6():
    # Eq. 6: sum alpha_i beta_i = sum a_i b_i (same order -> exact)
    rng = np.random.default_rng(5)
    a = rng.normal(size=64)
    a[rng.random(64) < 0.3] = 0.0
    b = rng.normal(size=64)
    u, v = oracle.gamma_sequence(a, b)
    alpha = np.where(a == 0.0, 1.0, a)
    beta = v[:-1]
    s1 = 0.0
    s2 = 0.0
    for i in range(64):
        s1 += alpha[i] * beta[i]
        s2 += a[i] * b[i]
    assert s1 == s2


# ------------------------------------------- P1: prefix-sum definition (Eq. 1, 2)
@pytest.mark.parametrize("w,s", [(1, 1), (2, 1), (3, 1), (16, 1), (64, 1), (256, 1), (5, 2), (7, 3), (3, 5)])
def test_pool_sum_i32_equals_prefix_difference(w, s):
    # Sliding sum (Eq. 3) = P_{is+w} - P_{is} with P the prefix sums of Eq. 1,
    # built here by numpy's cumsum (an independent library routine).
    x = synth.randint(2, 5000, -1000, 1000)
    P = np.concatenate([[0], np.cumsum(x.astype(np.int64))])
    L = (5000 - w) // s + 1
    i = np.arange(L) * s
    np.testing.assert_array_equal(oracle.pool_sum(x, w, s), P[i + w] - P[i])


def test_prefix_recurrence_eq2():
    # Eq. 2: the window starting at 0 with w = i+1 is the prefix y_i, and
    # y_{i+1} = y_i + x_{i+1}.
    x = synth.randint(9, 50, -1000, 1000)
    ys = [int(oracle.pool_sum(x[: i + 1], i + 1)[0]) for i in range(50)]
    for i in range(49):
        assert ys[i + 1] == ys[i] + int(x[i + 1])
    assert ys[0] == int(x[0])


# ------------------------------------------- P2: closed forms
@pytest.mark.parametrize("w,s", [(1, 1), (3, 1), (8, 1), (64, 1), (4, 3), (9, 2)])
def test_closed_forms_ramp_and_constant(w, s):
    N = 300
    L = (N - w) // s + 1
    i = np.arange(L, dtype=np.int64)
    ramp = np.arange(N, dtype=np.int32)
    np.testing.assert_array_equal(oracle.pool_sum(ramp, w, s), w * (i * s) + w * (w - 1) // 2)
    np.testing.assert_array_equal(oracle.pool_max(ramp, w, s), i * s + w - 1)
    np.testing.assert_array_equal(oracle.pool_max(-ramp, w, s), -(i * s))
    yf, mag = oracle.pool_sum(ramp.astype(np.float32), w, s)
    np.testing.assert_array_equal(yf, (w * (i * s) + w * (w - 1) // 2).astype(np.float64))
    np.testing.assert_array_equal(mag, yf)  # non-negative input: absmag = sum
    np.testing.assert_array_equal(oracle.pool_max(ramp.astype(np.float32), w, s), (i * s + w - 1).astype(np.float32))
    c = np.full(N, 7, np.int32)
    np.testing.assert_array_equal(oracle.pool_sum(c, w, s), np.full(L, 7 * w))
    np.testing.assert_array_equal(oracle.pool_max(c, w, s), np.full(L, 7))


def test_closed_forms_2d():
    P, H, W = 3, 17, 13
    r = np.arange(H)[:, None]
    c = np.arange(W)[None, :]
    x = np.broadcast_to((r * W + c).astype(np.float32), (P, H, W)).copy()
    for kh, kw, sh, sw in [(3, 3, 1, 1), (2, 2, 2, 2), (3, 2, 2, 3), (1, 1, 1, 1), (17, 13, 1, 1)]:
        OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
        orr = np.arange(OH)[:, None]
        occ = np.arange(OW)[None, :]
        ymax, _ = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_MAX)
        exp_max = (orr * sh + kh - 1) * W + occ * sw + kw - 1
        np.testing.assert_array_equal(ymax, np.broadcast_to(exp_max, (P, OH, OW)))
        yavg, mag = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_AVG)
        exp_avg = (orr * sh + (kh - 1) / 2) * W + occ * sw + (kw - 1) / 2
        np.testing.assert_allclose(yavg, np.broadcast_to(exp_avg, (P, OH, OW)), rtol=1e-15, atol=1e-12)
        np.testing.assert_array_equal(mag, yavg)


# ------------------------------------------- P3: delta and box filters
@pytest.mark.parametrize("k,m,s", [(1, 0, 1), (3, 0, 1), (3, 2, 1), (8, 5, 1), (31, 17, 1), (63, 62, 1), (5, 3, 2)])
def test_conv_delta_filter_is_shift(k, m, s):
    x = synth.normal(3, 1000)
    f = np.zeros(k, np.float32)
    f[m] = 1.0
    y, mag = oracle.conv1d(x, f, s)
    L = (1000 - k) // s + 1
    exp = x[np.arange(L) * s + m].astype(np.float64)
    np.testing.assert_array_equal(y, exp)  # orientation: cross-correlation, no flip
    np.testing.assert_array_equal(mag, np.abs(exp))


def test_conv_box_filter_is_sliding_sum():
    x = synth.uniform_pm1(0, 777)
    for k in (1, 2, 8, 33):
        y, mag = oracle.conv1d(x, np.ones(k, np.float32))
        ys, mags = oracle.pool_sum(x, k)
        np.testing.assert_array_equal(y, ys)
        np.testing.assert_array_equal(mag, mags)


def test_conv_asymmetric_filter_orientation():
    # [1,2,3,4] with f=[1,10]: cross-correlation gives x_i + 10 x_{i+1}
    y, _ = oracle.conv1d(np.array([1, 2, 3, 4], np.float32), np.array([1, 10], np.float32))
    np.testing.assert_array_equal(y, [21, 32, 43])


# ------------------------------------------- P4: brute force on tiny inputs
def test_brute_force_tiny_exhaustive():
    vals = [-2, -1, 0, 1, 2]
    for N in range(1, 6):
        for xs in itertools.product(vals, repeat=N):
            x = np.array(xs, np.int32)
            for w in range(1, N + 1):
                for s in (1, 2, 3):
                    L = (N - w) // s + 1
                    exp_sum = [sum(xs[i * s:i * s + w]) for i in range(L)]
                    exp_max = [max(xs[i * s:i * s + w]) for i in range(L)]
                    assert oracle.pool_sum(x, w, s).tolist() == exp_sum
                    assert oracle.pool_max(x, w, s).tolist() == exp_max
                    if s == 1 and L > 1:
                        y = oracle.pool_sum(x, w, 1)
                        # Eq. 3 identity: y_{i+1} - y_i = x_{i+w} - x_i
                        assert all(y[i + 1] - y[i] == xs[i + w] - xs[i] for i in range(L - 1))


# ------------------------------------------- P7: independent library routines (float64)
@pytest.mark.parametrize("w,s", [(1, 1), (3, 1), (8, 1), (16, 2), (64, 1), (5, 5)])
def test_pool_vs_torch(w, s):
    x = synth.normal(1, 3 * 1000).reshape(3, 1000)
    xt = torch.from_numpy(x.astype(np.float64)).unsqueeze(1)
    y, mag = oracle.pool_sum(x, w, s)
    ref = F.avg_pool1d(xt, w, s).squeeze(1).numpy() * w
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    ref_mag = F.avg_pool1d(xt.abs(), w, s).squeeze(1).numpy() * w
    np.testing.assert_allclose(mag, ref_mag, rtol=1e-12, atol=1e-12)
    np.testing.assert_array_equal(oracle.pool_max(x, w, s),
                                  F.max_pool1d(torch.from_numpy(x).unsqueeze(1), w, s).squeeze(1).numpy())
    xi = synth.randint(2, 3000, -1000, 1000).reshape(3, 1000)
    ref_i = F.max_pool1d(torch.from_numpy(xi.astype(np.float64)).unsqueeze(1), w, s).squeeze(1).numpy()
    np.testing.assert_array_equal(oracle.pool_max(xi, w, s), ref_i.astype(np.int32))


@pytest.mark.parametrize("k,s", [(1, 1), (3, 1), (5, 2), (8, 1), (31, 1), (63, 1), (7, 3)])
def test_conv_vs_torch(k, s):
    x = synth.normal(3, 2 * 2000).reshape(2, 2000)
    f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
    y, mag = oracle.conv1d(x, f, s)
    xt = torch.from_numpy(x.astype(np.float64)).unsqueeze(1)
    ft = torch.from_numpy(f.astype(np.float64)).view(1, 1, k)
    ref = F.conv1d(xt, ft, stride=s).squeeze(1).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    ref_mag = F.conv1d(xt.abs(), ft.abs(), stride=s).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref_mag, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("kh,kw,sh,sw", [(3, 3, 1, 1), (2, 2, 2, 2), (3, 5, 2, 1), (1, 1, 1, 1), (4, 3, 3, 2)])
def test_pool2d_vs_torch(kh, kw, sh, sw):
    x = synth.uniform01(5, 4 * 23 * 19).reshape(4, 23, 19)
    xt = torch.from_numpy(x.astype(np.float64)).unsqueeze(1)
    ymax, _ = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_MAX)
    np.testing.assert_array_equal(ymax, F.max_pool2d(xt, (kh, kw), (sh, sw)).squeeze(1).numpy())
    yavg, mag = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_AVG)
    ref = F.avg_pool2d(xt, (kh, kw), (sh, sw)).squeeze(1).numpy()
    np.testing.assert_allclose(yavg, ref, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(mag, ref, rtol=1e-13, atol=1e-15)  # x >= 0


# ------------------------------------------- P9: linearity, separability
def test_conv_linearity():
    x1 = synth.normal(21, 4000)
    x2 = synth.normal(22, 4000)
    f = synth.normal(4, 31, sigma=synth.cfg_sigma_filter(31))
    a = np.float32(0.5)  # exact scaling
    y1, m1 = oracle.conv1d(x1, f)
    y2, m2 = oracle.conv1d(x2, f)
    y12, _ = oracle.conv1d((a * x1 + x2).astype(np.float32), f)
    # inputs of (a x1 + x2) are rounded to fp32 once: allow that rounding
    bound = 1e-6 * (a * m1 + m2) + 1e-12
    assert np.all(np.abs(y12 - (a * y1 + y2)) <= bound)


def test_pool2d_max_separable_equals_direct():
    x = synth.normal(8, 5 * 31 * 29).reshape(5, 31, 29)
    for kh, kw, sh, sw in [(3, 3, 1, 1), (2, 2, 2, 2), (5, 3, 2, 3)]:
        ymax, _ = oracle.pool2d(x, kh, kw, sh, sw, oracle.POOL2D_MAX)
        rows = np.lib.stride_tricks.sliding_window_view(x, kw, axis=2)[:, :, ::sw].max(-1)
        cols = np.lib.stride_tricks.sliding_window_view(rows, kh, axis=1)[:, ::sh].max(-1)
        np.testing.assert_array_equal(ymax, cols.astype(np.float64))


# ------------------------------------------- argument checks
def test_oracle_rejects_window_exceeding_input():
    with pytest.raises(ValueError):
        oracle.pool_sum(np.zeros(3, np.int32), 4)
    with pytest.raises(ValueError):
        oracle.conv1d(np.zeros(3, np.float32), np.ones(5, np.float32))
    assert oracle.out_len(3, 4, 1) == -1
    assert oracle.out_len(10, 3, 4) == 2
    assert oracle.out_len(2 ** 32, 31, 1) == 2 ** 32 - 30


# ------------------------------------------- generator sanity (shared inputs)
def test_generator_counter_based_and_distributions():
    a = synth.normal(6, 1000, start=5000)
    b = synth.normal(6, 6000)[5000:]
    np.testing.assert_array_equal(a, b)
    z = synth.normal(3, 200000)
    assert abs(float(z.mean())) < 0.01 and abs(float(z.var()) - 1.0) < 0.02
    i = synth.randint(2, 200000, -1000, 1000)
    assert i.min() == -1000 and i.max() == 1000
    u = synth.uniform_pm1(0, 100000)
    assert u.min() >= -1.0 and u.max() < 1.0
    assert np.all((u * 2 ** 23) == np.round(u * 2 ** 23))


# ------------------------------------------- NEXT #1: zero padding + dilation (window spec)
@pytest.mark.parametrize("case", GOLD["window_ex"], ids=lambda c: c["cite"])
def test_golden_window_ex(case):
    x = np.array(case["x"], np.float32)
    a = (case["s"], case["d"], case["pl"], case["pr"])
    if case["op"] == "conv":
        y, _ = oracle.conv1d_ex(x, np.array(case["f"], np.float32), *a)
    else:
        y, _ = oracle.pool_sum_ex(x, case["w"], *a)
        if case["op"] == "avg":
            y = y / case["w"]
    np.testing.assert_array_equal(y, np.array(case["y"], np.float64))


EX_SPECS = [(1, 1, 0, 0), (2, 1, 0, 0), (1, 2, 0, 0), (1, 1, 2, 3), (3, 2, 1, 4), (2, 4, 5, 0), (1, 8, 7, 7)]


@pytest.mark.parametrize("s,d,pl,pr", EX_SPECS)
@pytest.mark.parametrize("w", [1, 2, 3, 7])
def test_window_ex_vs_torch(w, s, d, pl, pr):
    x = synth.normal(12, 3 * 500).reshape(3, 500)
    xt = torch.from_numpy(x.astype(np.float64)).unsqueeze(1)
    f = synth.normal(4, w, sigma=synth.cfg_sigma_filter(w))
    ft = torch.from_numpy(f.astype(np.float64)).view(1, 1, w)
    ref = F.conv1d(F.pad(xt, (pl, pr)), ft, stride=s, dilation=d).squeeze(1).numpy()
    y, mag = oracle.conv1d_ex(x, f, s, d, pl, pr)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
    ref_mag = F.conv1d(F.pad(xt.abs(), (pl, pr)), ft.abs(), stride=s, dilation=d).squeeze(1).numpy()
    np.testing.assert_allclose(mag, ref_mag, rtol=1e-12, atol=1e-12)
    ones = torch.ones(1, 1, w, dtype=torch.float64)
    ys, _ = oracle.pool_sum_ex(x, w, s, d, pl, pr)
    np.testing.assert_allclose(ys, F.conv1d(F.pad(xt, (pl, pr)), ones, stride=s, dilation=d).squeeze(1).numpy(),
                               rtol=1e-12, atol=1e-12)
    xm = F.pad(xt, (pl, pr), value=-np.inf)  # max padding never wins
    refm = F.max_pool1d(xm, w, s, dilation=d).squeeze(1).numpy()
    np.testing.assert_array_equal(oracle.pool_max_ex(x, w, s, d, pl, pr).astype(np.float64), refm)
    xi = synth.randint(2, 3 * 500, -1000, 1000).reshape(3, 500)
    yi = oracle.pool_sum_ex(xi, w, s, d, pl, pr)
    np.testing.assert_array_equal(yi, np.rint(F.conv1d(F.pad(torch.from_numpy(xi.astype(np.float64)).unsqueeze(1), (pl, pr)),
                                                       ones, stride=s, dilation=d).squeeze(1).numpy()).astype(np.int64))


def test_window_ex_reduces_to_valid_ops():
    x = synth.randint(3, 2 * 300, -1000, 1000).reshape(2, 300)
    xf = synth.normal(3, 2 * 300).reshape(2, 300)
    f = synth.normal(4, 5)
    for w, s in ((1, 1), (3, 1), (5, 2), (8, 3)):
        np.testing.assert_array_equal(oracle.pool_sum_ex(x, w, s), oracle.pool_sum(x, w, s))
        np.testing.assert_array_equal(oracle.pool_max_ex(x, w, s), oracle.pool_max(x, w, s))
        np.testing.assert_array_equal(oracle.pool_max_ex(xf, w, s), oracle.pool_max(xf, w, s))
    np.testing.assert_array_equal(oracle.conv1d_ex(xf, f, 2)[0], oracle.conv1d(xf, f, 2)[0])


def test_window_ex_brute_force_and_all_padding():
    vals = [-2, 0, 1, 2]
    for N in range(1, 5):
        for xs in itertools.product(vals, repeat=N):
            x = np.array(xs, np.int32)
            for w, s, d, pl, pr in ((1, 1, 1, 2, 1), (2, 1, 2, 1, 1), (3, 2, 1, 2, 2), (2, 3, 3, 3, 0)):
                L = oracle.out_len_ex(N, w, s, d, pl, pr)
                if L < 0:
                    continue
                xp = [None] * pl + list(xs) + [None] * pr
                exp_sum, exp_max = [], []
                for i in range(L):
                    win = [xp[i * s + j * d] for j in range(w)]
                    valid = [v for v in win if v is not None]
                    exp_sum.append(sum(valid))
                    exp_max.append(max(valid) if valid else -2 ** 31)
                assert oracle.pool_sum_ex(x, w, s, d, pl, pr).tolist() == exp_sum
                assert oracle.pool_max_ex(x, w, s, d, pl, pr).tolist() == exp_max
    # a window made only of padding: sum 0, max = identity
    assert oracle.pool_max_ex(np.array([5.0], np.float32), 1, 1, 1, 1, 0)[0] == -np.inf
    assert oracle.out_len_ex(3, 4, 1, 1, 0, 0) == -1 and oracle.out_len_ex(3, 4, 1, 1, 1, 0) == 1


# ------------------------------------------- NEXT #3: sliding window of gamma pairs (Eq. 8)
def test_affine_window_reduces_to_sliding_sum_and_product():
    v = synth.normal(13, 2000)
    u1 = np.ones(2000, np.float32)
    for w in (1, 2, 5, 33):
        U, V, M = oracle.affine_window(u1, v, w)
        ref, mag = oracle.pool_sum(v, w)  # u = 1: plain Eq. 3 sliding sum of v
        np.testing.assert_allclose(V, ref, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(M, mag, rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(U, np.ones_like(U))
    u = (0.5 + 0.5 * synth.uniform01(14, 2000)).astype(np.float32)
    for w in (1, 3, 8):
        U, V, _ = oracle.affine_window(u, np.zeros(2000, np.float32), w)
        np.testing.assert_array_equal(V, np.zeros_like(V))
        logp = np.convolve(np.log(u.astype(np.float64)), np.ones(w), mode="valid")  # sliding log-sum
        np.testing.assert_allclose(U, np.exp(logp), rtol=1e-12)


def test_affine_window_geometric_is_a_convolution():
    # u = c constant: V_i = sum_j v_{i+j} c^{w-1-j}  (an exponentially weighted window)
    c = np.float32(0.75)
    v = synth.normal(15, 3000)
    for w in (2, 7, 40):
        _, V, _ = oracle.affine_window(np.full(3000, c, np.float32), v, w)
        kern = np.array([float(c) ** (w - 1 - j) for j in range(w)])
        ref = np.convolve(v.astype(np.float64), kern[::-1], mode="valid")
        np.testing.assert_allclose(V, ref, rtol=1e-12, atol=1e-12)


def test_affine_window_exact_rationals_brute_force():
    from fractions import Fraction
    rng = np.random.default_rng(3)
    u = rng.integers(-4, 5, 12).astype(np.float32) / 4
    v = rng.integers(-8, 9, 12).astype(np.float32) / 8
    for w, s in ((1, 1), (3, 1), (4, 2), (12, 1), (5, 3)):
        U, V, _ = oracle.affine_window(u, v, w, s)
        for i in range(len(V)):
            acc_u, acc_v = Fraction(1), Fraction(0)
            for j in range(i * s, i * s + w):   # fold from the identity (1, 0), Eq. 8
                acc_u, acc_v = acc_u * Fraction(float(u[j])), Fraction(float(u[j])) * acc_v + Fraction(float(v[j]))
            assert Fraction(U[i]) == acc_u and Fraction(V[i]) == acc_v


def test_affine_window_is_order_sensitive_and_gives_the_dot_product():
    u = np.array([2.0, 0.5, 3.0], np.float32)
    v = np.array([1.0, 4.0, -2.0], np.float32)
    _, V, _ = oracle.affine_window(u, v, 3)
    _, Vr, _ = oracle.affine_window(u[::-1].copy(), v[::-1].copy(), 3)
    assert V[0] != Vr[0]  # non-commutative
    # Eq. 9: the window over the whole gamma sequence of (a, b) yields the dot product
    a = np.array([2.0, 0.0, 4.0, -1.0, 0.5])  # ratios of powers of two: exact in fp32
    b = np.array([1.0, 5.0, 7.0, 2.0, -3.0])
    gu, gv = oracle.gamma_sequence(a, b)
    _, Vd, _ = oracle.affine_window(gu.astype(np.float32), gv.astype(np.float32), len(gu))
    assert np.all(gu.astype(np.float32) == gu) and np.all(gv.astype(np.float32) == gv)
    assert Vd[0] == float(np.dot(a, b))


# ------------------------------------------- multi-dimensional extension: 2-D sliding dot product
def test_conv2d_separable_filter_is_row_then_column_conv():
    # f = u (x) v (outer product): the 2-D correlation equals the 1-D correlation of
    # every row with v followed by every column with u -- exact on integers
    x = synth.randint(50, 3 * 13 * 17, -9, 9).astype(np.float32).reshape(3, 13, 17)
    u = np.array([1, -2, 3], np.float32)
    v = np.array([2, 0, -1, 1], np.float32)
    y, _ = oracle.conv2d(x, np.outer(u, v))
    rows, _ = oracle.conv1d(x.reshape(-1, 17), v)                      # [3*13, 14]
    rows = rows.reshape(3, 13, 14).transpose(0, 2, 1).reshape(-1, 13)  # columns as rows
    cols, _ = oracle.conv1d(rows.astype(np.float32), u)                # exact: small integers
    np.testing.assert_array_equal(y, cols.reshape(3, 14, 11).transpose(0, 2, 1))


def test_conv2d_delta_and_box_filters():
    x = synth.uniform01(51, 2 * 9 * 10).reshape(2, 9, 10)
    for a, b in ((0, 0), (1, 2), (2, 1)):
        f = np.zeros((3, 3), np.float32)
        f[a, b] = 1.0
        y, _ = oracle.conv2d(x, f)
        np.testing.assert_array_equal(y, x[:, a:a + 7, b:b + 8].astype(np.float64))  # shifted plane, exact
    xi = synth.randint(52, 2 * 9 * 10, -50, 50).astype(np.float32).reshape(2, 9, 10)
    y, _ = oracle.conv2d(xi, np.ones((3, 2), np.float32), 2, 1)
    avg, _ = oracle.pool2d(xi, 3, 2, 2, 1, oracle.POOL2D_AVG)
    np.testing.assert_allclose(y, avg * 6, rtol=0, atol=1e-12)          # box filter = window sum


def test_conv2d_vs_torch_and_1d_reduction():
    x = synth.normal(53, 2 * 20 * 23).reshape(2, 20, 23)
    f = synth.normal(54, 15).reshape(3, 5)
    for sh, sw in ((1, 1), (2, 1), (2, 3)):
        y, _ = oracle.conv2d(x, f, sh, sw)
        ref = torch.nn.functional.conv2d(torch.tensor(x, dtype=torch.float64)[:, None],
                                         torch.tensor(f, dtype=torch.float64)[None, None], stride=(sh, sw))
        np.testing.assert_allclose(y, ref[:, 0].numpy(), rtol=1e-12, atol=1e-12)
    # kh = 1: every row is the 1-D sliding dot product
    f1 = synth.normal(55, 6).reshape(1, 6)
    y, _ = oracle.conv2d(x, f1)
    y1, _ = oracle.conv1d(x.reshape(-1, 23), f1[0])
    np.testing.assert_array_equal(y.reshape(-1, 18), y1)


# ------------------------------------------- multi-channel conv1d (channels-last, bf16 inputs)
def test_bf16_rounding_helper():
    # bf16 keeps 8 significant bits: spacing 2^-7 just above 1
    v = np.array([1.0, 1.0078125, 1.00390625, 1.01171875, -3.14159, 65504.0, 1e-30], np.float32)
    h = oracle.to_bf16_bits(v)
    back = oracle.bf16_bits_to_f32(h)
    np.testing.assert_array_equal(back[:2], [1.0, 1.0078125])                   # representable: exact
    assert back[2] == 1.0 and back[3] == 1.015625                                # ties -> even mantissa
    assert np.all(np.abs(back - v) <= np.abs(v) * 2.0 ** -8)                     # RN: half an ulp of 8 bits
    np.testing.assert_array_equal(oracle.to_bf16_bits(back), h)                  # idempotent


def test_conv1d_mc_reduces_to_single_channel_and_sums_channels():
    B, N, k = 2, 50, 5
    x = synth.randint(80, B * N * 3, -8, 8).astype(np.float32).reshape(B, N, 3)  # exact in bf16
    w = synth.randint(81, 2 * 3 * k, -4, 4).astype(np.float32).reshape(2, 3, k)
    y, _ = oracle.conv1d_mc(oracle.to_bf16_bits(x), oracle.to_bf16_bits(w))
    for co in range(2):  # = sum over input channels of the 1-D sliding dot product (oracle.conv1d)
        ref = sum(oracle.conv1d(np.ascontiguousarray(x[:, :, ci]), w[co, ci])[0] for ci in range(3))
        np.testing.assert_array_equal(y[:, :, co], ref)


def test_conv1d_mc_vs_torch():
    B, N, cin, cout, k = 2, 40, 8, 5, 3
    xf = synth.normal(82, B * N * cin).reshape(B, N, cin)
    wf = synth.normal(83, cout * cin * k).reshape(cout, cin, k)
    xb, wb = oracle.to_bf16_bits(xf), oracle.to_bf16_bits(wf)
    y, _ = oracle.conv1d_mc(xb, wb)
    xt = torch.tensor(oracle.bf16_bits_to_f32(xb), dtype=torch.float64).permute(0, 2, 1)  # NCW
    wt = torch.tensor(oracle.bf16_bits_to_f32(wb), dtype=torch.float64)
    ref = torch.nn.functional.conv1d(xt, wt).permute(0, 2, 1).numpy()
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)


# ------------------------------------------------ multi-channel 2-D conv (reading R22)
def test_conv2d_mc_sums_single_channel_2d_convs():
    # integer-valued (exact in bf16 and in double): every (co, ci) pair is the single-channel
    # 2-D correlation oracle.conv2d (pinned above against torch, separable filters, deltas)
    B, H, W, cin, cout, kh, kw = 2, 9, 11, 3, 2, 3, 4
    x = synth.randint(84, B * H * W * cin, -8, 8).astype(np.float32).reshape(B, H, W, cin)
    w = synth.randint(85, cout * cin * kh * kw, -4, 4).astype(np.float32).reshape(cout, cin, kh, kw)
    y, mag = oracle.conv2d_mc(oracle.to_bf16_bits(x), oracle.to_bf16_bits(w))
    for co in range(cout):
        ref = sum(oracle.conv2d(np.ascontiguousarray(x[..., ci]), w[co, ci])[0] for ci in range(cin))
        np.testing.assert_array_equal(y[..., co], ref)
        refm = sum(oracle.conv2d(np.abs(np.ascontiguousarray(x[..., ci])), np.abs(w[co, ci]))[0] for ci in range(cin))
        np.testing.assert_array_equal(mag[..., co], refm)


def test_conv2d_mc_vs_torch_and_reductions():
    B, H, W, cin, cout = 2, 7, 10, 8, 5
    xf = synth.normal(86, B * H * W * cin).reshape(B, H, W, cin)
    for kh, kw in ((3, 3), (1, 1), (2, 5)):
        wf = synth.normal(87, cout * cin * kh * kw).reshape(cout, cin, kh, kw)
        xb, wb = oracle.to_bf16_bits(xf), oracle.to_bf16_bits(wf)
        y, mag = oracle.conv2d_mc(xb, wb)
        xt = torch.tensor(oracle.bf16_bits_to_f32(xb), dtype=torch.float64).permute(0, 3, 1, 2)  # NCHW
        wt = torch.tensor(oracle.bf16_bits_to_f32(wb), dtype=torch.float64)
        ref = torch.nn.functional.conv2d(xt, wt).permute(0, 2, 3, 1).numpy()
        np.testing.assert_allclose(y, ref, rtol=1e-12, atol=1e-12)
        refm = torch.nn.functional.conv2d(xt.abs(), wt.abs()).permute(0, 2, 3, 1).numpy()
        np.testing.assert_allclose(mag, refm, rtol=1e-12, atol=1e-12)
    # H = kh = 1: the multi-channel 1-D convolution, row by row
    wb = oracle.to_bf16_bits(synth.normal(88, cout * cin * 3).reshape(cout, cin, 1, 3))
    xb = oracle.to_bf16_bits(xf)
    y, _ = oracle.conv2d_mc(xb, wb)
    for r in range(H):
        y1, _ = oracle.conv1d_mc(np.ascontiguousarray(xb[:, r]), np.ascontiguousarray(wb[:, :, 0, :]))
        np.testing.assert_array_equal(y[:, r], y1)


# ------------------------------------------------ multi-channel conv1d input gradient (reading R23)
def test_conv1d_mc_backward_input_adjoint_and_torch():
    B, N, cin, cout, k = 2, 30, 5, 4, 3
    # adjoint identity on integers (exact in bf16 and double): <conv1d_mc(x), dy> = <x, dx>
    x = synth.randint(104, B * N * cin, -5, 5).astype(np.float32).reshape(B, N, cin)
    w = synth.randint(105, cout * cin * k, -3, 3).astype(np.float32).reshape(cout, cin, k)
    dy = synth.randint(106, B * (N - k + 1) * cout, -4, 4).astype(np.float32).reshape(B, N - k + 1, cout)
    xb, wb, gb = oracle.to_bf16_bits(x), oracle.to_bf16_bits(w), oracle.to_bf16_bits(dy)
    y, _ = oracle.conv1d_mc(xb, wb)
    dx, mag = oracle.conv1d_mc_backward_input(gb, wb, N)
    assert float((y * dy).sum()) == float((x.astype(np.float64) * dx).sum())
    # torch float64 autograd of conv1d (NCW), signed values; magnitude = the same VJP on |w|, |dy|
    xf = synth.normal(107, B * N * cin).reshape(B, N, cin)
    wf = synth.normal(108, cout * cin * k).reshape(cout, cin, k)
    gf = synth.normal(109, B * (N - k + 1) * cout).reshape(B, N - k + 1, cout)
    wb, gb = oracle.to_bf16_bits(wf), oracle.to_bf16_bits(gf)
    dx, mag = oracle.conv1d_mc_backward_input(gb, wb, N)
    wt = torch.tensor(oracle.bf16_bits_to_f32(wb), dtype=torch.float64)
    gt = torch.tensor(oracle.bf16_bits_to_f32(gb), dtype=torch.float64).permute(0, 2, 1)
    ref = torch.nn.grad.conv1d_input((B, cin, N), wt, gt).permute(0, 2, 1).numpy()
    np.testing.assert_allclose(dx, ref, rtol=1e-12, atol=1e-12)
    refm = torch.nn.grad.conv1d_input((B, cin, N), wt.abs(), gt.abs()).permute(0, 2, 1).numpy()
    np.testing.assert_allclose(mag, refm, rtol=1e-12, atol=1e-12)
    assert np.any(mag > np.abs(dx) + 1e-9)
    # one channel each way: the single-channel input gradient oracle
    g1 = synth.normal(110, B * (N - k + 1)).reshape(B, N - k + 1, 1)
    w1 = synth.normal(111, k).reshape(1, 1, k)
    g1b, w1b = oracle.to_bf16_bits(g1), oracle.to_bf16_bits(w1)
    dx1, _ = oracle.conv1d_mc_backward_input(g1b, w1b, N)
    ref1, _ = oracle.conv1d_backward_input(oracle.bf16_bits_to_f32(g1b)[..., 0], oracle.bf16_bits_to_f32(w1b)[0, 0], N)
    np.testing.assert_allclose(dx1[..., 0], ref1, rtol=1e-12, atol=1e-12)


def test_conv1d_mc_backward_filter_adjoint_torch_and_single_channel():
    # reading R25: dw[co][ci][j] = sum_b sum_i dy[b][i][co] x[b][i+j][ci]
    B, N, cin, cout, k = 2, 30, 5, 4, 3
    L = N - k + 1
    # adjoint identity on integers (exact in bf16 and double): <conv1d_mc(x, w), dy> = <w, dw>
    x = synth.randint(112, B * N * cin, -5, 5).astype(np.float32).reshape(B, N, cin)
    w = synth.randint(113, cout * cin * k, -3, 3).astype(np.float32).reshape(cout, cin, k)
    dy = synth.randint(114, B * L * cout, -4, 4).astype(np.float32).reshape(B, L, cout)
    xb, wb, gb = oracle.to_bf16_bits(x), oracle.to_bf16_bits(w), oracle.to_bf16_bits(dy)
    y, _ = oracle.conv1d_mc(xb, wb)
    dw, _ = oracle.conv1d_mc_backward_filter(gb, xb, k)
    assert float((y * dy).sum()) == float((w.astype(np.float64) * dw).sum())
    # torch float64 autograd (NCW), signed values; magnitude = the same VJP on |x|, |dy|
    xf = synth.normal(115, B * N * cin).reshape(B, N, cin)
    gf = synth.normal(116, B * L * cout).reshape(B, L, cout)
    xb, gb = oracle.to_bf16_bits(xf), oracle.to_bf16_bits(gf)
    dw, mag = oracle.conv1d_mc_backward_filter(gb, xb, k)
    xt = torch.tensor(oracle.bf16_bits_to_f32(xb), dtype=torch.float64).permute(0, 2, 1)
    gt = torch.tensor(oracle.bf16_bits_to_f32(gb), dtype=torch.float64).permute(0, 2, 1)
    ref = torch.nn.grad.conv1d_weight(xt, (cout, cin, k), gt).numpy()
    np.testing.assert_allclose(dw, ref, rtol=1e-12, atol=1e-12)
    refm = torch.nn.grad.conv1d_weight(xt.abs(), (cout, cin, k), gt.abs()).numpy()
    np.testing.assert_allclose(mag, refm, rtol=1e-12, atol=1e-12)
    assert np.any(mag > np.abs(dw) + 1e-9)
    # one channel each way: the single-channel filter gradient oracle
    g1 = synth.normal(117, B * L).reshape(B, L, 1)
    x1 = synth.normal(118, B * N).reshape(B, N, 1)
    g1b, x1b = oracle.to_bf16_bits(g1), oracle.to_bf16_bits(x1)
    dw1, _ = oracle.conv1d_mc_backward_filter(g1b, x1b, k)
    ref1, _ = oracle.conv1d_backward_filter(oracle.bf16_bits_to_f32(x1b)[..., 0], oracle.bf16_bits_to_f32(g1b)[..., 0], k)
    np.testing.assert_allclose(dw1[0, 0], ref1, rtol=1e-12, atol=1e-12)


def test_conv2d_mc_backward_input_adjoint_torch_and_1d_reduction():
    # reading R26: dx[b][r+a][c+e][ci] += w[co][ci][a][e] dy[b][r][c][co]
    B, H, W, cin, cout, kh, kw = 2, 7, 9, 3, 4, 3, 2
    OH, OW = H - kh + 1, W - kw + 1
    x = synth.randint(130, B * H * W * cin, -4, 4).astype(np.float32).reshape(B, H, W, cin)
    w = synth.randint(131, cout * cin * kh * kw, -3, 3).astype(np.float32).reshape(cout, cin, kh, kw)
    dy = synth.randint(132, B * OH * OW * cout, -4, 4).astype(np.float32).reshape(B, OH, OW, cout)
    xb, wb, gb = oracle.to_bf16_bits(x), oracle.to_bf16_bits(w), oracle.to_bf16_bits(dy)
    y, _ = oracle.conv2d_mc(xb, wb)
    dx, _ = oracle.conv2d_mc_backward_input(gb, wb, H, W)
    assert float((y * dy).sum()) == float((x.astype(np.float64) * dx).sum())  # adjoint, exact on integers
    wf = synth.normal(133, cout * cin * kh * kw).reshape(cout, cin, kh, kw)
    gf = synth.normal(134, B * OH * OW * cout).reshape(B, OH, OW, cout)
    wb, gb = oracle.to_bf16_bits(wf), oracle.to_bf16_bits(gf)
    dx, mag = oracle.conv2d_mc_backward_input(gb, wb, H, W)
    wt = torch.tensor(oracle.bf16_bits_to_f32(wb), dtype=torch.float64)
    gt = torch.tensor(oracle.bf16_bits_to_f32(gb), dtype=torch.float64).permute(0, 3, 1, 2)
    ref = torch.nn.grad.conv2d_input((B, cin, H, W), wt, gt).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(dx, ref, rtol=1e-12, atol=1e-12)
    refm = torch.nn.grad.conv2d_input((B, cin, H, W), wt.abs(), gt.abs()).permute(0, 2, 3, 1).numpy()
    np.testing.assert_allclose(mag, refm, rtol=1e-12, atol=1e-12)
    # one image row (H = kh = 1): the 1-D multi-channel input gradient
    g1 = oracle.to_bf16_bits(synth.normal(135, B * 1 * (W - 2) * cout).reshape(B, 1, W - 2, cout))
    w1 = oracle.to_bf16_bits(synth.normal(136, cout * cin * 3).reshape(cout, cin, 1, 3))
    dx2, _ = oracle.conv2d_mc_backward_input(g1, w1, 1, W)
    dx1, _ = oracle.conv1d_mc_backward_input(g1[:, 0], w1[:, :, 0], W)
    np.testing.assert_array_equal(dx2[:, 0], dx1)


def test_conv2d_mc_backward_filter_adjoint_torch_and_1d_reduction():
    # reading R27: dw[co][ci][a][e] = sum_{b,r,c} dy[b][r][c][co] x[b][r+a][c+e][ci]
    B, H, W, cin, cout, kh, kw = 2, 7, 9, 3, 4, 3, 2
    OH, OW = H - kh + 1, W - kw + 1
    x = synth.randint(150, B * H * W * cin, -4, 4).astype(np.float32).reshape(B, H, W, cin)
    w = synth.randint(151, cout * cin * kh * kw, -3, 3).astype(np.float32).reshape(cout, cin, kh, kw)
    dy = synth.randint(152, B * OH * OW * cout, -4, 4).astype(np.float32).reshape(B, OH, OW, cout)
    xb, wb, gb = oracle.to_bf16_bits(x), oracle.to_bf16_bits(w), oracle.to_bf16_bits(dy)
    y, _ = oracle.conv2d_mc(xb, wb)
    dw, _ = oracle.conv2d_mc_backward_filter(gb, xb, kh, kw)
    assert float((y * dy).sum()) == float((w.astype(np.float64) * dw).sum())  # <y(w), dy> = <w, dw>, exact
    xf = synth.normal(153, B * H * W * cin).reshape(B, H, W, cin)
    gf = synth.normal(154, B * OH * OW * cout).reshape(B, OH, OW, cout)
    xb, gb = oracle.to_bf16_bits(xf), oracle.to_bf16_bits(gf)
    dw, mag = oracle.conv2d_mc_backward_filter(gb, xb, kh, kw)
    xt = torch.tensor(oracle.bf16_bits_to_f32(xb), dtype=torch.float64).permute(0, 3, 1, 2)
    gt = torch.tensor(oracle.bf16_bits_to_f32(gb), dtype=torch.float64).permute(0, 3, 1, 2)
    ref = torch.nn.grad.conv2d_weight(xt, (cout, cin, kh, kw), gt).numpy()
    np.testing.assert_allclose(dw, ref, rtol=1e-12, atol=1e-12)
    refm = torch.nn.grad.conv2d_weight(xt.abs(), (cout, cin, kh, kw), gt.abs()).numpy()
    np.testing.assert_allclose(mag, refm, rtol=1e-12, atol=1e-12)
    # one image row (H = kh = 1): the 1-D multi-channel filter gradient
    x1 = oracle.to_bf16_bits(synth.normal(155, B * 1 * W * cin).reshape(B, 1, W, cin))
    g1 = oracle.to_bf16_bits(synth.normal(156, B * 1 * (W - 2) * cout).reshape(B, 1, W - 2, cout))
    dw2, m2 = oracle.conv2d_mc_backward_filter(g1, x1, 1, 3)
    dw1, m1 = oracle.conv1d_mc_backward_filter(g1[:, 0], x1[:, 0], 3)
    np.testing.assert_array_equal(dw2[:, :, 0], dw1)
    np.testing.assert_array_equal(m2[:, :, 0], m1)
