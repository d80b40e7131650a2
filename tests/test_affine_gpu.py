"""GPU parity for ss_affine_window (sliding window of the paper's gamma pairs,
Eq. 8 operator) against oracle.affine_window.

Tolerance (reading R15): every term v_j prod u_l of V passes through
at most 2w fp32 roundings in any (+) tree, so
    |V - V_ref| <= 2 w 2^-24 magV + 1e-6,   |U - U_ref| <= 2 w 2^-24 |U_ref| + 1e-30.
Exact cases (u = 1 or 1/2 with small-integer v) must match bit for bit."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -24


@pytest.fixture(scope="module")
def ss():
    import paper_2305_16513_b200 as ss
    return ss


def dev(a, off=0):
    """Copy a host array to a device buffer starting `off` elements in (misalignment)."""
    buf = torch.empty(a.size + off + 4, dtype=torch.float32, device="cuda")
    t = buf[off:off + a.size]
    t.copy_(torch.from_numpy(np.ascontiguousarray(a, np.float32).reshape(-1)).cuda())
    return t


def run(ss, u, v, w, s=1, want_U=True, uoff=0, yoff=0):
    B, N = u.shape
    L = ss.ss_out_len(N, w, s)
    ud, vd = dev(u, uoff), dev(v, uoff)
    Vb = torch.full((B * L + yoff + 5,), -77.0, device="cuda")
    Ub = torch.full((B * L + yoff + 5,), -77.0, device="cuda")
    V = Vb[yoff:yoff + B * L]
    U = Ub[yoff:yoff + B * L]
    ss.check(ss.ss_affine_window(ud.data_ptr(), vd.data_ptr(), U.data_ptr() if want_U else 0,
                                 V.data_ptr(), N, B, w, s))
    torch.cuda.synchronize()
    for buf in (Vb, Ub):
        h = buf.cpu().numpy()
        assert np.all(h[:yoff] == -77) and np.all(h[yoff + B * L:] == -77), "canary overwritten"
    if not want_U:
        assert torch.all(Ub == -77)
    return U.cpu().numpy().reshape(B, L), V.cpu().numpy().reshape(B, L)


def check_close(ss, u, v, w, s=1, **kw):
    U, V = run(ss, u, v, w, s, **kw)
    Ur, Vr, M = oracle.affine_window(u, v, w, s)
    tol = 2 * w * EPS
    assert np.all(np.abs(V - Vr) <= tol * M + 1e-6), np.max(np.abs(V - Vr) - tol * M)
    if kw.get("want_U", True):
        assert np.all(np.abs(U - Ur) <= tol * np.abs(Ur) + 1e-30)
    return U, V


def decay(seed, B, N, lo=0.5):
    return synth.uab(seed, B * N, lo, 1.0).reshape(B, N)


WS = [1, 2, 3, 7, 8, 9, 10, 16, 17, 23, 24, 25, 63, 64, 65, 130, 257, 520, 1000, 2049, 4097]


@pytest.mark.parametrize("w", WS)
@pytest.mark.parametrize("N,B", [(20011, 2), (2048 * 3 + 77, 1)])
def test_affine_decay(ss, w, N, B):
    if w > N:
        pytest.skip()
    lo = 0.5 if w <= 64 else 0.97  # keep U above fp32 underflow for long windows
    check_close(ss, decay(1, B, N, lo), synth.normal(2, B * N).reshape(B, N), w)


@pytest.mark.parametrize("w", [1, 5, 9, 40, 300])
def test_affine_signed_u_with_zeros(ss, w):
    # signed gains in [-1, 1) with exact zeros sprinkled (a zero resets the recurrence)
    N, B = 30011, 2
    u = synth.uniform_pm1(3, B * N).reshape(B, N)
    u[:, ::97] = 0.0
    check_close(ss, u, synth.normal(4, B * N).reshape(B, N), w)


@pytest.mark.parametrize("w,s", [(3, 2), (8, 3), (17, 5), (64, 64), (100, 7)])
def test_affine_strided(ss, w, s):
    N, B = 9001, 3
    check_close(ss, decay(5, B, N), synth.normal(6, B * N).reshape(B, N), w, s)


@pytest.mark.parametrize("w", [4, 12, 100])
@pytest.mark.parametrize("uoff,yoff", [(1, 0), (2, 3), (0, 1)])
def test_affine_misaligned_and_V_only(ss, w, uoff, yoff):
    N, B = 7001, 3
    u, v = decay(7, B, N), synth.normal(8, B * N).reshape(B, N)
    check_close(ss, u, v, w, uoff=uoff, yoff=yoff)
    check_close(ss, u, v, w, uoff=uoff, yoff=yoff, want_U=False)


@pytest.mark.parametrize("w", [1, 6, 9, 16, 33, 200])
def test_affine_exact_cases(ss, w):
    # u = 1: V is the plain sliding sum (Eq. 3, +) of small integers -> exact.
    N, B = 12007, 2
    v = synth.randint(9, B * N, -50, 50).reshape(B, N).astype(np.float32)
    U, V = run(ss, np.ones((B, N), np.float32), v, w)
    ref, _ = oracle.pool_sum(v, w)
    np.testing.assert_array_equal(V.astype(np.float64), ref)
    assert np.all(U == 1.0)
    # u = 1/2, |v| <= 8, w <= 16: every partial result is a dyadic number of < 24 bits -> exact.
    if w <= 16:
        v8 = synth.randint(10, B * N, -8, 8).reshape(B, N).astype(np.float32)
        U, V = run(ss, np.full((B, N), 0.5, np.float32), v8, w)
        Ur, Vr, _ = oracle.affine_window(np.full((B, N), 0.5, np.float32), v8, w)
        np.testing.assert_array_equal(V.astype(np.float64), Vr)
        np.testing.assert_array_equal(U.astype(np.float64), Ur)


def test_affine_edges(ss):
    for N, w in ((1, 1), (5, 5), (9, 9), (17, 9), (2048, 2048), (4100, 4097), (8, 1)):
        u, v = decay(11, 1, N), synth.normal(12, N).reshape(1, N)
        check_close(ss, u, v, w)


def test_affine_deterministic_and_binding(ss):
    N, B, w = 100003, 2, 77
    u = torch.from_numpy(decay(13, B, N)).cuda()
    v = torch.from_numpy(synth.normal(14, B * N).reshape(B, N)).cuda()
    U1, V1 = ss.affine_window(u, v, w)
    U2, V2 = ss.affine_window(u, v, w)
    assert torch.equal(U1, U2) and torch.equal(V1, V2)
    _, V3 = ss.affine_window(u, v, w, want_U=False)
    assert torch.equal(V1, V3)
    Ur, Vr, M = oracle.affine_window(u.cpu().numpy(), v.cpu().numpy(), w)
    assert np.all(np.abs(V1.cpu().numpy() - Vr) <= 2 * w * EPS * M + 1e-6)


def test_affine_full_size_sampled(ss):
    """bench.py's affine workload ([8][2^24], w = 64) in the timed launch config;
    sampled windows recomputed by the oracle one by one."""
    B, N, w = 8, 1 << 24, 64
    u = torch.empty(B, N, device="cuda")
    v = torch.empty(B, N, device="cuda")
    synth.fill_device(u, "uab", 31, lo=0.5, hi=1.0)
    synth.fill_device(v, "normal", 32)
    U, V = ss.affine_window(u, v, w)
    torch.cuda.synchronize()
    L = N - w + 1
    rng = np.random.default_rng(0)
    idx = np.concatenate([rng.integers(0, L, 2000), [0, 1, L - 1, L - 2, 2047, 2048, 2049]])
    for b in (0, 3, 7):
        uh = u[b].cpu().numpy()
        vh = v[b].cpu().numpy()
        Vd = V[b].cpu().numpy()
        Ud = U[b].cpu().numpy()
        for i in idx:
            Ur, Vr, M = oracle.affine_window(uh[i:i + w], vh[i:i + w], w)
            assert abs(Vd[i] - Vr[0]) <= 2 * w * EPS * M[0] + 1e-6
            assert abs(Ud[i] - Ur[0]) <= 2 * w * EPS * abs(Ur[0]) + 1e-30
