"""GPU parity of the multi-channel 2-D convolution (ss_conv2d_mc, csrc/conv_mc.cu;
SURVEY 8f NEXT #4, reading R22): NHWC bf16 activations, [Cout][Cin][kh][kw]
bf16 weights, fp32 output, against oracle.conv2d_mc (the same bf16 values in
double) within 1e-5 * sum|terms| + 1e-6.  Tensor-core shapes (cin, cout in
{64, 128}: tap (a, e) = the staged tile shifted by a W + e flat positions), tiles
crossing image rows and images, several TMA boxes per stage (wide images), the
direct kernel (other shapes), canaries, integer exactness, validation."""
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
    B, H, W, cin = xb.shape
    cout, _, kh, kw = wb.shape
    OH, OW = H - kh + 1, W - kw + 1
    n = B * OH * OW * cout
    xd, wd = bf16_dev(xb), bf16_dev(wb)
    yb = torch.full((n + yoff + 8,), -55.0, device="cuda")
    y = yb[yoff:yoff + n]
    ss.check(ss.ss_conv2d_mc(xd.data_ptr(), wd.data_ptr(), y.data_ptr(), B, H, W, cin, cout, kh, kw))
    torch.cuda.synchronize()
    h = yb.cpu().numpy()
    assert np.all(h[:yoff] == -55.0) and np.all(h[yoff + n:] == -55.0), "canary overwritten"
    return y.cpu().numpy().reshape(B, OH, OW, cout)


def check(y, ref, mag, what):
    err = np.abs(y.astype(np.float64) - ref)
    bound = TOL_REL * mag + TOL_ABS
    assert np.all(err <= bound), f"{what}: {(err > bound).sum()} out of bound, max err/bound {(err / bound).max():.3g}"


CASES = [  # (B, H, W, cin, cout, kh, kw)
    (2, 10, 12, 64, 64, 3, 3), (2, 9, 56, 64, 64, 3, 3), (1, 7, 30, 128, 64, 5, 5), (2, 6, 8, 64, 128, 1, 1),
    (3, 5, 40, 128, 128, 3, 3), (1, 12, 112, 64, 64, 3, 3), (1, 9, 200, 64, 64, 5, 5), (2, 4, 9, 64, 64, 4, 2),
    (1, 8, 8, 3, 16, 3, 3), (2, 5, 7, 32, 8, 2, 3), (1, 3, 3, 64, 64, 3, 3),
]


@pytest.mark.parametrize("B,H,W,cin,cout,kh,kw", CASES)
def test_conv2d_mc(ss, B, H, W, cin, cout, kh, kw):
    xb = oracle.to_bf16_bits(synth.normal(94, B * H * W * cin).reshape(B, H, W, cin))
    wb = oracle.to_bf16_bits(synth.normal(95, cout * cin * kh * kw, sigma=(cin * kh * kw) ** -0.5)
                             .reshape(cout, cin, kh, kw))
    y = run(ss, xb, wb)
    ref, mag = oracle.conv2d_mc(xb, wb)
    check(y, ref, mag, f"B={B} H={H} W={W} cin={cin} cout={cout} {kh}x{kw}")


def test_misaligned_output_uses_the_direct_kernel(ss):
    xb = oracle.to_bf16_bits(synth.normal(96, 2 * 6 * 10 * 64).reshape(2, 6, 10, 64))
    wb = oracle.to_bf16_bits(synth.normal(97, 64 * 64 * 9, sigma=(64 * 9) ** -0.5).reshape(64, 64, 3, 3))
    y = run(ss, xb, wb, yoff=1)
    ref, mag = oracle.conv2d_mc(xb, wb)
    check(y, ref, mag, "y offset by one float")


def test_integer_valued_inputs_are_exact(ss):
    # small integers: every bf16 product and every fp32 partial sum is exact
    B, H, W, cin, cout = 2, 8, 20, 64, 64
    xb = oracle.to_bf16_bits(synth.randint(98, B * H * W * cin, -3, 3).astype(np.float32).reshape(B, H, W, cin))
    wb = oracle.to_bf16_bits(synth.randint(99, cout * cin * 9, -2, 2).astype(np.float32).reshape(cout, cin, 3, 3))
    y = run(ss, xb, wb)
    ref, _ = oracle.conv2d_mc(xb, wb)
    np.testing.assert_array_equal(y.astype(np.float64), ref)


def test_resnet_layer_shape_sampled(ss):
    # a 56x56x64 -> 64, 3x3 layer (batch 8): full tensor-core run, sampled oracle outputs
    B, H, W, cin, cout = 8, 56, 56, 64, 64
    x = torch.empty(B, H, W, cin, device="cuda")
    synth.fill_device(x, "normal", 100)
    xd = x.to(torch.bfloat16)
    wb = oracle.to_bf16_bits(synth.normal(101, cout * cin * 9, sigma=(cin * 9) ** -0.5).reshape(cout, cin, 3, 3))
    wd = bf16_dev(wb)
    y = ss.conv2d_mc(xd, wd).cpu().numpy()
    xb = xd.view(torch.int16).cpu().numpy().view(np.uint16)
    for b in (0, B - 1):  # whole images (first / last: tiles crossing into and out of them)
        ref, mag = oracle.conv2d_mc(np.ascontiguousarray(xb[b:b + 1]), wb)
        check(y[b:b + 1], ref, mag, f"image {b}")


def test_validation(ss):
    x = torch.zeros(1, 4, 4, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(64, 64, 5, 3, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ss.SSError):
        ss.conv2d_mc(x, w)
    y = torch.empty(10, device="cuda")
    assert ss.ss_conv2d_mc(x.data_ptr(), w.data_ptr(), y.data_ptr(), 1, 4, 4, 64, 64, 5, 3) == \
        ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv2d_mc(0, w.data_ptr(), y.data_ptr(), 1, 4, 4, 64, 64, 3, 3) == ss.SS_ERR_NULL
