"""Exhaustive tiny cases on the GPU: every 1 <= w <= N <= 48,
stride in {1, 2, 3}, batch 3, int32 values in {-2..2} (many equal keys and
ties), against the oracle bit for bit; fp32 conv for every k <= N <= 40 within
the BASELINE.json bound; canaries around every output.  Inputs are packed so
that all (N, w, s) of one N share one host round trip."""
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


def launch_all(ss, fn, x_dev, N, B, jobs, dt, code, extra=None):
    """Run fn for every (w, s) of `jobs` into one canary-padded buffer; return host slices."""
    lens = [ss.ss_out_len(N, w, s) for (w, s) in jobs]
    offs, tot = [], 0
    for L in lens:
        offs.append(tot + 4)
        tot += B * L + 8
    fill = -7777
    y = torch.full((tot,), fill, dtype=dt, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for (w, s), o in zip(jobs, offs):
        yp = y[o:].data_ptr()
        if extra is None:
            ss.check(fn(x_dev.data_ptr(), yp, N, B, w, s, code, st))
        else:
            ss.check(fn(x_dev.data_ptr(), yp, N, B, extra[w], w, s, code, st))
    h = y.cpu().numpy()
    out = []
    for L, o in zip(lens, offs):
        assert np.all(h[o - 4:o] == fill) and np.all(h[o + B * L:o + B * L + 4] == fill), "canary overwritten"
        out.append(h[o:o + B * L].reshape(B, L))
    return out


@pytest.mark.parametrize("op", ["sum", "max"])
def test_pool_i32_exhaustive_tiny(ss, op):
    fn = ss.ss_pool_sum if op == "sum" else ss.ss_pool_max
    B = 3
    for N in range(1, 49):
        x = synth.randint(40 + N, B * N, -2, 2).reshape(B, N)
        xd = torch.from_numpy(x).cuda()
        jobs = [(w, s) for w in range(1, N + 1) for s in (1, 2, 3)]
        ys = launch_all(ss, fn, xd, N, B, jobs, torch.int32, ss.SS_I32)
        for (w, s), y in zip(jobs, ys):
            if op == "max":
                ref = oracle.pool_max(x, w, s)
            else:
                ref = oracle.pool_sum(x, w, s)
            np.testing.assert_array_equal(y.astype(np.int64), ref, err_msg=f"{op} N={N} w={w} s={s}")


def test_pool_f32_exhaustive_tiny(ss):
    B = 3
    for N in range(1, 49, 3):
        x = synth.uniform_pm1(90 + N, B * N).reshape(B, N)
        xd = torch.from_numpy(x).cuda()
        jobs = [(w, s) for w in range(1, N + 1) for s in (1, 2, 3)]
        ys = launch_all(ss, ss.ss_pool_max, xd, N, B, jobs, torch.float32, ss.SS_F32)
        for (w, s), y in zip(jobs, ys):
            np.testing.assert_array_equal(y.astype(np.float64), oracle.pool_max(x, w, s).astype(np.float64))
        ys = launch_all(ss, ss.ss_pool_sum, xd, N, B, jobs, torch.float32, ss.SS_F32)
        for (w, s), y in zip(jobs, ys):
            ref, mag = oracle.pool_sum(x, w, s)
            assert np.all(np.abs(y - ref) <= 1e-5 * mag + 1e-6), f"sum N={N} w={w} s={s}"


def test_conv_exhaustive_tiny(ss):
    B = 3
    for N in range(1, 41):
        x = synth.normal(130 + N, B * N).reshape(B, N)
        xd = torch.from_numpy(x).cuda()
        filters = {k: synth.normal(170 + k, k, sigma=synth.cfg_sigma_filter(k)) for k in range(1, N + 1)}
        jobs = [(k, s) for k in range(1, N + 1) for s in (1, 2, 3)]
        fl = {k: f.tolist() for k, f in filters.items()}
        ys = launch_all(ss, ss.ss_conv1d, xd, N, B, jobs, torch.float32, ss.SS_F32, extra=fl)
        for (k, s), y in zip(jobs, ys):
            ref, mag = oracle.conv1d(x, filters[k], s)
            assert np.all(np.abs(y - ref) <= 1e-5 * mag + 1e-6), f"conv N={N} k={k} s={s}"
