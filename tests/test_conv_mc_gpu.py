"""GPU parity of the multi-channel conv1d (csrc/conv_mc.cu; SURVEY 8f NEXT #4,
DESIGN.md reading R18): channels-last bf16 activations / weights, fp32 output,
against oracle.conv1d_mc (the same bf16 values in double) within
1e-5 * sum|terms| + 1e-6.  Tensor-core shapes (cin, cout in {64, 128}, k <= 9),
the direct kernel (other shapes, misaligned outputs), tiles crossing batch rows,
canaries, integer exactness."""
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


def bf16_dev(bits):
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).cuda().view(torch.bfloat16)


def run(ss, xb, wb, yoff=0):
    B, N, cin = xb.shape
    cout, _, k = wb.shape
    L = N - k + 1
    xd, wd = bf16_dev(xb), bf16_dev(wb)
    yb = torch.full((B * L * cout + yoff + 8,), -55.0, device="cuda")
    y = yb[yoff:yoff + B * L * cout]
    ss.check(ss.ss_conv1d_mc(xd.data_ptr(), wd.data_ptr(), y.data_ptr(), B, N, cin, cout, k))
    torch.cuda.synchronize()
    h = yb.cpu().numpy()
    assert np.all(h[:yoff] == -55.0) and np.all(h[yoff + B * L * cout:] == -55.0), "canary overwritten"
    return y.cpu().numpy().reshape(B, L, cout)


def check(y, ref, mag, what):
    err = np.abs(y.astype(np.float64) - ref)
    bound = TOL_REL * mag + TOL_ABS
    assert np.all(err <= bound), f"{what}: {(err > bound).sum()} out of bound, max err/bound {(err / bound).max():.3g}"


CASES = [  # (B, N, cin, cout, k)
    (2, 1000, 64, 64, 3), (3, 777, 128, 64, 5), (1, 4096, 64, 128, 9), (2, 300, 128, 128, 1),
    (5, 129, 64, 64, 2), (1, 20000, 128, 128, 3), (2, 200, 32, 48, 3), (1, 500, 3, 5, 7), (2, 400, 64, 64, 12),
    (1, 9, 64, 64, 9),
]


@pytest.mark.parametrize("B,N,cin,cout,k", CASES)
def test_conv1d_mc(ss, B, N, cin, cout, k):
    xb = oracle.to_bf16_bits(synth.normal(90, B * N * cin).reshape(B, N, cin))
    wb = oracle.to_bf16_bits(synth.normal(91, cout * cin * k, sigma=(cin * k) ** -0.5).reshape(cout, cin, k))
    y = run(ss, xb, wb)
    ref, mag = oracle.conv1d_mc(xb, wb)
    check(y, ref, mag, f"mc B={B} N={N} cin={cin} cout={cout} k={k}")


def test_conv1d_mc_direct_path_agrees(ss):
    # a 4-byte-offset output forces the direct kernel; both paths meet the same bound
    B, N, cin, cout, k = 2, 1000, 64, 64, 3
    xb = oracle.to_bf16_bits(synth.normal(92, B * N * cin).reshape(B, N, cin))
    wb = oracle.to_bf16_bits(synth.normal(93, cout * cin * k, sigma=0.1).reshape(cout, cin, k))
    ref, mag = oracle.conv1d_mc(xb, wb)
    check(run(ss, xb, wb, yoff=0), ref, mag, "tensor path")
    check(run(ss, xb, wb, yoff=1), ref, mag, "direct path")


def test_conv1d_mc_integer_exact(ss):
    # small integers are exact in bf16; every partial sum is an integer < 2^24 -> bit-exact
    B, N, cin, cout, k = 2, 700, 128, 64, 4
    xb = oracle.to_bf16_bits(synth.randint(94, B * N * cin, -8, 8).astype(np.float32).reshape(B, N, cin))
    wb = oracle.to_bf16_bits(synth.randint(95, cout * cin * k, -4, 4).astype(np.float32).reshape(cout, cin, k))
    ref, _ = oracle.conv1d_mc(xb, wb)
    np.testing.assert_array_equal(run(ss, xb, wb).astype(np.float64), ref)


def test_conv1d_mc_binding_vs_torch(ss):
    x = torch.randn(2, 513, 64, device="cuda").to(torch.bfloat16)
    w = (torch.randn(128, 64, 3, device="cuda") * 0.1).to(torch.bfloat16)
    y = ss.conv1d_mc(x, w)
    ref = torch.nn.functional.conv1d(x.double().permute(0, 2, 1), w.double()).permute(0, 2, 1)
    mag = torch.nn.functional.conv1d(x.double().abs().permute(0, 2, 1), w.double().abs()).permute(0, 2, 1)
    assert torch.all((y.double() - ref).abs() <= TOL_REL * mag + TOL_ABS)
