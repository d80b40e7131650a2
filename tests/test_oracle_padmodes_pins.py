"""Pins of the oracle's padding modes and sliding min (oracle/oracle.c pad_source,
extremum_ex_*; SURVEY 8f NEXT #1 "zero/mirror/periodic padding" and NEXT #3
"sliding min"; PAPER.md l.158 names padding, mirroring and periodicity as the
boundary conditions, l.136 min as an associative operator).

Checked against what fixes them independently of the oracle's code: hand-worked
padded sequences, numpy's own padding (np.pad reflect / wrap / edge) with brute
force windows, torch float64 padding + conv1d / max_pool1d, and identities
(min = -max(-x), the circular full-period invariant)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth

NP_MODE = {"reflect": "reflect", "circular": "wrap", "replicate": "edge"}
TORCH_MODE = {"reflect": "reflect", "circular": "circular", "replicate": "replicate"}


def test_hand_values():
    x = np.array([1, 2, 3, 4], np.int32)
    # reflect: xp = 3 2 | 1 2 3 4 | 3 2 ; circular: 3 4 | 1 2 3 4 | 1 2 ; replicate: 1 1 | 1 2 3 4 | 4 4
    assert oracle.pool_sum_ex(x, 3, pl=2, pr=2, mode="reflect").tolist() == [6, 5, 6, 9, 10, 9]
    assert oracle.pool_max_ex(x, 3, pl=2, pr=2, mode="reflect").tolist() == [3, 2, 3, 4, 4, 4]
    assert oracle.pool_min_ex(x, 3, pl=2, pr=2, mode="reflect").tolist() == [1, 1, 1, 2, 3, 2]
    assert oracle.pool_sum_ex(x, 3, pl=2, pr=2, mode="circular").tolist() == [8, 7, 6, 9, 8, 7]
    assert oracle.pool_sum_ex(x, 3, pl=2, pr=2, mode="replicate").tolist() == [3, 4, 6, 9, 11, 12]
    assert oracle.pool_sum_ex(x, 3, pl=2, pr=2, mode="zeros").tolist() == [1, 3, 6, 9, 7, 4]
    # zeros: a window made only of padding is the identity of the operator
    # (pl = 3, w = 2: windows 0 and 1 are all padding, window 2 = [pad, 1])
    y = oracle.pool_max_ex(x, 2, pl=3, pr=0, mode="zeros")
    assert y[0] == y[1] == np.iinfo(np.int32).min and y[2] == 1
    y = oracle.pool_min_ex(x, 2, pl=3, pr=0, mode="zeros")
    assert y[0] == y[1] == np.iinfo(np.int32).max and y[2] == 1
    yf = oracle.pool_min_ex(x.astype(np.float32), 2, pl=3, pr=0)
    assert yf[0] == np.inf and yf[2] == 1.0
    # dilation 2, stride 2 on the reflected sequence: windows xp[2i], xp[2i+2]
    assert oracle.pool_sum_ex(x, 2, s=2, d=2, pl=2, pr=2, mode="reflect").tolist() == [3 + 1, 1 + 3, 3 + 3]


def _brute(x, w, s, d, pl, pr, mode, reduce):
    xp = np.pad(x.astype(np.float64), (pl, pr), mode=NP_MODE[mode])
    E = (w - 1) * d + 1
    L = (len(xp) - E) // s + 1
    return np.array([reduce(xp[i * s: i * s + E: d]) for i in range(L)])


@pytest.mark.parametrize("mode", ["reflect", "circular", "replicate"])
@pytest.mark.parametrize("N,w,s,d,pl,pr", [(17, 3, 1, 1, 1, 1), (40, 5, 2, 3, 4, 7), (9, 4, 1, 2, 8, 3),
                                           (31, 7, 3, 1, 6, 0), (12, 12, 1, 1, 11, 11)])
def test_against_numpy_padding(mode, N, w, s, d, pl, pr):
    if mode == "circular" and (pl > N or pr > N):
        pytest.skip("one period")
    xi = synth.randint(60, 2 * N, -50, 50).reshape(2, N)
    xf = synth.normal(61, 2 * N).reshape(2, N)
    for b in range(2):
        np.testing.assert_array_equal(oracle.pool_sum_ex(xi, w, s, d, pl, pr, mode)[b],
                                      _brute(xi[b], w, s, d, pl, pr, mode, np.sum).astype(np.int64))
        np.testing.assert_array_equal(oracle.pool_max_ex(xi, w, s, d, pl, pr, mode)[b],
                                      _brute(xi[b], w, s, d, pl, pr, mode, np.max))
        np.testing.assert_array_equal(oracle.pool_min_ex(xf, w, s, d, pl, pr, mode)[b],
                                      _brute(xf[b], w, s, d, pl, pr, mode, np.min).astype(np.float32))
        ysum, _ = oracle.pool_sum_ex(xf, w, s, d, pl, pr, mode)
        np.testing.assert_allclose(ysum[b], _brute(xf[b], w, s, d, pl, pr, mode, np.sum), rtol=0, atol=1e-12)


@pytest.mark.parametrize("mode", ["reflect", "circular", "replicate"])
@pytest.mark.parametrize("N,k,s,d,pl,pr", [(50, 7, 1, 1, 3, 3), (64, 5, 2, 2, 4, 4), (33, 9, 3, 1, 8, 2)])
def test_against_torch_padding(mode, N, k, s, d, pl, pr):
    x = synth.normal(62, 3 * N).reshape(3, N)
    f = synth.normal(63, k)
    xt = torch.from_numpy(x.astype(np.float64)).view(3, 1, N)
    xp = F.pad(xt, (pl, pr), mode=TORCH_MODE[mode])
    yc = F.conv1d(xp, torch.from_numpy(f.astype(np.float64)).view(1, 1, k), stride=s, dilation=d).view(3, -1)
    y, _ = oracle.conv1d_ex(x, f, s, d, pl, pr, mode)
    np.testing.assert_allclose(y, yc.numpy(), rtol=0, atol=1e-11)
    ym = F.max_pool1d(xp, k, stride=s, dilation=d).view(3, -1).numpy()
    np.testing.assert_array_equal(oracle.pool_max_ex(x, k, s, d, pl, pr, mode), ym.astype(np.float32))
    yn = -F.max_pool1d(-xp, k, stride=s, dilation=d).view(3, -1).numpy()
    np.testing.assert_array_equal(oracle.pool_min_ex(x, k, s, d, pl, pr, mode), yn.astype(np.float32))


def test_min_is_negated_max_of_negation():
    x = synth.normal(64, 4 * 333).reshape(4, 333)
    for w, s in ((1, 1), (5, 1), (64, 2), (333, 1)):
        np.testing.assert_array_equal(oracle.pool_min(x, w, s), -oracle.pool_max(-x, w, s))
    xi = synth.randint(65, 1000, -10 ** 6, 10 ** 6)
    np.testing.assert_array_equal(oracle.pool_min(xi, 17), -oracle.pool_max(-xi, 17))


def test_circular_full_period_invariant():
    # every window of length N over the periodic extension holds each element once
    x = synth.randint(66, 3 * 25, -100, 100).reshape(3, 25)
    y = oracle.pool_sum_ex(x, 25, pl=0, pr=24, mode="circular")
    assert y.shape == (3, 25)
    np.testing.assert_array_equal(y, np.repeat(x.astype(np.int64).sum(axis=1, keepdims=True), 25, axis=1))


def test_mode_limits_rejected():
    x = np.arange(5, dtype=np.int32)
    with pytest.raises(Exception):
        oracle.pool_sum_ex(x, 2, pl=5, mode="reflect")   # reflection needs pl <= N-1
    with pytest.raises(Exception):
        oracle.pool_sum_ex(x, 2, pr=6, mode="circular")  # one period
    oracle.pool_sum_ex(x, 2, pl=4, mode="reflect")
    oracle.pool_sum_ex(x, 2, pr=5, mode="circular")
