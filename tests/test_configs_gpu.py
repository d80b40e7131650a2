"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (device-generated inputs, whole-array launches).  Where the oracle
finishes in seconds the whole output is compared; otherwise sampled outputs
(random positions, both ends, every 8192-output tile boundary region, shard
boundaries) are recomputed one by one by the oracle on host-regenerated input
slices, plus properties that hold at any size."""
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


def sample_positions(L, n_rand=3000, seed=0, extra=()):
    rng = np.random.default_rng(seed)
    pos = set(rng.integers(0, L, n_rand).tolist())
    pos.update(range(0, min(L, 300)))
    pos.update(range(max(0, L - 300), L))
    for t in range(8192, L, 8192 * 97):  # tile edges (every 97th tile)
        pos.update(range(max(0, t - 3), min(L, t + 3)))
    for e in extra:
        pos.update(range(max(0, e - 70), min(L, e + 70)))
    return np.array(sorted(pos), dtype=np.int64)


def check_samples(y_dev, pos, w, gen_slice, op, f=None):
    """y_dev: 1-D device output; gen_slice(start, n) regenerates x on the host."""
    idx = torch.from_numpy(pos).to(y_dev.device)
    got = y_dev[idx].cpu().numpy()
    for j, i in enumerate(pos):
        xs = gen_slice(int(i), w)
        if op == "max":
            assert got[j] == oracle.pool_max(xs, w)[0], (i, got[j])
        elif op == "sum" and xs.dtype == np.int32:
            ref = int(oracle.pool_sum(xs, w)[0])
            assert int(got[j]) == ((ref + 2 ** 31) % 2 ** 32) - 2 ** 31, (i, got[j], ref)
        elif op == "sum":
            ref, mag = oracle.pool_sum(xs, w)
            assert abs(float(got[j]) - ref[0]) <= TOL_REL * mag[0] + TOL_ABS, (i, got[j], ref[0])
        else:
            ref, mag = oracle.conv1d(xs, f)
            assert abs(float(got[j]) - ref[0]) <= TOL_REL * mag[0] + TOL_ABS, (i, got[j], ref[0])


def test_cfg1_full(ss):
    x_h = synth.uniform_pm1(0, 65536)
    f = synth.uniform_pm1(1, 8)
    x = torch.empty(65536, device="cuda")
    synth.fill_device(x, "upm1", 0)
    assert np.array_equal(x.cpu().numpy(), x_h)
    ys, mag = oracle.pool_sum(x_h, 8)
    y = ss.pool_sum(x, 8).cpu().numpy()
    assert np.all(np.abs(y - ys) <= TOL_REL * mag + TOL_ABS)
    assert np.array_equal(ss.pool_max(x, 8).cpu().numpy(), oracle.pool_max(x_h, 8))
    yc, magc = oracle.conv1d(x_h, f)
    assert np.all(np.abs(ss.conv1d(x, f).cpu().numpy() - yc) <= TOL_REL * magc + TOL_ABS)


@pytest.fixture(scope="module")
def cfg2_x():
    x = torch.empty(1 << 26, dtype=torch.int32, device="cuda")
    synth.fill_device(x, "int", 2, lo=-1000, hi=1000)
    return x


@pytest.mark.parametrize("w", [3, 16, 64, 256])
@pytest.mark.parametrize("op", ["sum", "max"])
def test_cfg2_full_size(ss, cfg2_x, op, w):
    N = 1 << 26
    y = (ss.pool_sum if op == "sum" else ss.pool_max)(cfg2_x, w)
    assert y.shape[0] == N - w + 1
    # whole-array oracle on the first 2^22 outputs (several hundred tiles)
    n_head = 1 << 22
    x_head = synth.randint(2, n_head + w - 1, -1000, 1000)
    ref = oracle.pool_sum(x_head, w) if op == "sum" else oracle.pool_max(x_head, w)
    if op == "sum":
        ref = (ref & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    np.testing.assert_array_equal(y[:n_head].cpu().numpy(), ref)
    # sampled windows over the whole array
    pos = sample_positions(N - w + 1, seed=w)
    check_samples(y, pos, w, lambda i, n: synth.randint(2, n, -1000, 1000, start=i), op)
    if op == "sum":  # any-size property (Eq. 3): y[i+1] - y[i] = x[i+w] - x[i]  (mod 2^32)
        x64 = cfg2_x.long()
        d = (y[1:].long() - y[:-1].long()) - (x64[w:N] - x64[:N - w])
        assert int(torch.count_nonzero(d % (1 << 32))) == 0


@pytest.mark.parametrize("k", [3, 5, 7, 15, 31, 63])
def test_cfg3_full_size(ss, k):
    rows, N = 64, 1 << 20
    x = torch.empty((rows, N), device="cuda")
    synth.fill_device(x, "normal", 3)
    f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
    y = ss.conv1d(x, f)
    assert tuple(y.shape) == (rows, N - k + 1)
    for r in (0, 37, 63):  # whole rows against the oracle
        xr = synth.normal(3, N, start=r * N)
        ref, mag = oracle.conv1d(xr, f)
        err = np.abs(y[r].cpu().numpy().astype(np.float64) - ref)
        assert np.all(err <= TOL_REL * mag + TOL_ABS), (r, float((err / (TOL_REL * mag + TOL_ABS)).max()))
    yf = y.reshape(-1)
    L = N - k + 1
    rng = np.random.default_rng(k)
    flat = rng.integers(0, rows * L, 2000)
    check_samples(yf, np.sort(flat), k,
                  lambda o, n: synth.normal(3, n, start=(o // L) * N + (o % L)), "conv", f)


@pytest.mark.parametrize("mode", ["max", "avg"])
@pytest.mark.parametrize("kk,s", [(3, 1), (2, 2)])
def test_cfg4_full(ss, mode, kk, s):
    x = torch.empty((32, 64, 112, 112), device="cuda")
    synth.fill_device(x, "u01", 5)
    y = ss.pool2d(x, (kk, kk), (s, s), mode).cpu().numpy().reshape(2048, *([(112 - kk) // s + 1] * 2))
    xh = synth.uniform01(5, 32 * 64 * 112 * 112).reshape(2048, 112, 112)
    ref, mag = oracle.pool2d(xh, kk, kk, s, s, 0 if mode == "max" else 1)
    if mode == "max":
        np.testing.assert_array_equal(y.astype(np.float64), ref)
    else:
        assert np.all(np.abs(y - ref) <= TOL_REL * mag + TOL_ABS)


@pytest.mark.slow
def test_cfg5_full_size_and_shard_emulation(ss):
    """N = 2^32 fp32 (16 GiB): conv k=31 and max w=64 on one GPU, sampled parity,
    and the G=2/4/8 sequence sharding emulated on one device (each shard's
    buffer = its slice plus the next shard's first h elements, exactly what the
    NCCL halo delivers): outputs must be bitwise identical to the unsharded run."""
    N = 1 << 32
    x = torch.empty(N, device="cuda")
    synth.fill_device(x, "normal", 6)
    f = synth.normal(7, 31, sigma=synth.cfg_sigma_filter(31))
    for op, w in (("conv", 31), ("max", 64)):
        y = ss.conv1d(x, f) if op == "conv" else ss.pool_max(x, w)
        assert y.shape[0] == N - w + 1
        bounds = [N // g * r for g in (2, 4, 8) for r in range(1, g)]
        pos = sample_positions(N - w + 1, n_rand=1500, seed=w, extra=bounds)
        check_samples(y, pos, w, lambda i, n: synth.normal(6, n, start=i), op, f)
        for G in (2, 8):
            S = N // G
            ys = torch.empty_like(y)
            for r in range(G):
                s0 = r * S
                n_out = S if r < G - 1 else S - w + 1
                n_int = S - w + 1
                xv = x[s0:s0 + n_int + w - 1]   # interior: own shard only
                (ss.conv1d(xv, f, out=ys[s0:s0 + n_int]) if op == "conv"
                 else ss.pool_max(xv, w, out=ys[s0:s0 + n_int]))
                if n_out > n_int:               # tail: own last w-1 + halo w-1
                    xt = x[s0 + n_int:s0 + n_out + w - 1]
                    (ss.conv1d(xt, f, out=ys[s0 + n_int:s0 + n_out]) if op == "conv"
                     else ss.pool_max(xt, w, out=ys[s0 + n_int:s0 + n_out]))
            assert torch.equal(ys, y), (op, G)
            del ys
        del y
        torch.cuda.empty_cache()
