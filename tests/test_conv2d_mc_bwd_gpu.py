"""GPU parity of the multi-channel conv2d backward passes.  Filter gradient (ss_conv2d_mc_backward_filter,
csrc/mc_fgrad.cu 2-D mode, reading R27): bottom of the file.  Input gradient (ss_conv2d_mc_backward_input,
csrc/conv_mc.cu pad2d mode; reading R26): bf16 dy [B, H-kh+1, W-kw+1, Cout],
bf16 w [Cout, Cin, kh, kw], fp32 dx [B, H, W, Cin], against oracle.conv2d_mc_backward_input
(the same bf16 values in double) within 1e-5 * sum|terms| + 1e-6.  Tensor-core shapes
(cin, cout in {64, 128} whose weights and staged tiles fit shared memory: tiles of R dx
rows x Cw columns staged as one 5-D TMA box per atom starting kh-1 rows / kw-1 columns
outside dy), images narrower and wider than a tile (column tiles, W > 256), one-row and
one-column images, 1x1 and 1-D windows, the direct kernel (other shapes, misaligned dx),
canaries, integer exactness, a forward/backward adjoint check through the library,
validation."""
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


def run(ss, gb, wb, H, W, off=0):
    B, OH, OW, cout = gb.shape
    _, cin, kh, kw = wb.shape
    n = B * H * W * cin
    gd, wd = bf16_dev(gb), bf16_dev(wb)
    buf = torch.full((n + off + 8,), -55.0, device="cuda")
    dx = buf[off:off + n]
    ss.check(ss.ss_conv2d_mc_backward_input(gd.data_ptr(), wd.data_ptr(), dx.data_ptr(), B, H, W, cin, cout, kh, kw))
    torch.cuda.synchronize()
    h = buf.cpu().numpy()
    assert np.all(h[:off] == -55.0) and np.all(h[off + n:] == -55.0), "canary overwritten"
    return dx.cpu().numpy().reshape(B, H, W, cin)


def check(y, ref, mag, what):
    err = np.abs(y.astype(np.float64) - ref)
    bound = TOL_REL * mag + TOL_ABS
    assert np.all(err <= bound), f"{what}: {(err > bound).sum()} out of bound, max err/bound {(err / bound).max():.3g}"


def inputs(B, H, W, cin, cout, kh, kw, seed):
    OH, OW = H - kh + 1, W - kw + 1
    gb = oracle.to_bf16_bits(synth.normal(seed, B * OH * OW * cout).reshape(B, OH, OW, cout))
    wb = oracle.to_bf16_bits(
        synth.normal(seed + 1, cout * cin * kh * kw, sigma=(cout * kh * kw) ** -0.5).reshape(cout, cin, kh, kw))
    return gb, wb


CASES = [  # (B, H, W, cin, cout, kh, kw)
    (2, 20, 30, 64, 64, 3, 3), (1, 64, 64, 64, 64, 3, 3), (2, 40, 300, 64, 64, 3, 3), (1, 1, 500, 64, 64, 1, 3),
    (2, 300, 1, 64, 64, 3, 1), (2, 33, 65, 64, 64, 2, 4), (2, 9, 200, 64, 64, 1, 1), (2, 3, 3, 64, 64, 3, 3),
    (3, 50, 17, 128, 64, 3, 3), (1, 40, 40, 64, 128, 3, 3), (1, 30, 70, 128, 128, 2, 2), (2, 12, 260, 64, 64, 1, 7),
    (4, 5, 5, 64, 64, 5, 5), (2, 16, 16, 32, 48, 3, 3), (1, 11, 13, 3, 5, 4, 2), (1, 7, 300, 64, 64, 7, 1),
]


@pytest.mark.parametrize("B,H,W,cin,cout,kh,kw", CASES)
def test_conv2d_mc_backward_input(ss, B, H, W, cin, cout, kh, kw):
    gb, wb = inputs(B, H, W, cin, cout, kh, kw, 140)
    dx = run(ss, gb, wb, H, W)
    ref, mag = oracle.conv2d_mc_backward_input(gb, wb, H, W)
    check(dx, ref, mag, f"B={B} H={H} W={W} cin={cin} cout={cout} k={kh}x{kw}")


def test_misaligned_dx_uses_the_direct_kernel(ss):
    gb, wb = inputs(2, 20, 30, 64, 64, 3, 3, 142)
    dx = run(ss, gb, wb, 20, 30, off=1)
    ref, mag = oracle.conv2d_mc_backward_input(gb, wb, 20, 30)
    check(dx, ref, mag, "dx offset by one float")


def test_integer_valued_inputs_are_exact(ss):
    B, H, W, cin, cout, kh, kw = 2, 45, 70, 64, 64, 3, 3
    OH, OW = H - kh + 1, W - kw + 1
    gb = oracle.to_bf16_bits(synth.randint(144, B * OH * OW * cout, -3, 3).astype(np.float32).reshape(B, OH, OW, cout))
    wb = oracle.to_bf16_bits(synth.randint(145, cout * cin * kh * kw, -2, 2).astype(np.float32).reshape(cout, cin, kh, kw))
    dx = run(ss, gb, wb, H, W)
    ref, _ = oracle.conv2d_mc_backward_input(gb, wb, H, W)
    np.testing.assert_array_equal(dx.astype(np.float64), ref)


def test_adjoint_of_the_forward_kernel(ss):
    # <conv2d_mc(x, w), g> == <x, conv2d_mc_backward_input(g, w)>, both sides from the library's kernels
    B, H, W, cin, cout, kh, kw = 2, 56, 56, 64, 64, 3, 3
    x = torch.randn(B, H, W, cin, device="cuda").to(torch.bfloat16)
    w = (torch.randn(cout, cin, kh, kw, device="cuda") * (cin * kh * kw) ** -0.5).to(torch.bfloat16)
    g = torch.randn(B, H - kh + 1, W - kw + 1, cout, device="cuda").to(torch.bfloat16)
    y = ss.conv2d_mc(x, w)
    dx = ss.conv2d_mc_backward_input(g, w, H, W)
    lhs = (y.double() * g.double()).sum().item()
    rhs = (x.double() * dx.double()).sum().item()
    assert abs(lhs - rhs) <= 1e-4 * (y.double().abs() * g.double().abs()).sum().item()
    ref = torch.nn.grad.conv2d_input((B, cin, H, W), w.double(), g.double().permute(0, 3, 1, 2)).permute(0, 2, 3, 1)
    assert torch.allclose(dx.double(), ref, rtol=1e-4, atol=1e-4)


def test_validation(ss):
    g = torch.zeros(1, 4, 4, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(64, 64, 3, 3, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        ss.conv2d_mc_backward_input(g, w, 7, 6)       # dy height != H-kh+1
    with pytest.raises(ss.SSError):
        ss.conv2d_mc_backward_input(g, w, 2, 6)       # kh > H
    dx = torch.empty(10000, device="cuda")
    assert ss.ss_conv2d_mc_backward_input(0, w.data_ptr(), dx.data_ptr(), 1, 6, 6, 64, 64, 3, 3) == ss.SS_ERR_NULL
    assert ss.ss_conv2d_mc_backward_input(g.data_ptr(), w.data_ptr(), dx.data_ptr(), 1, 6, 2, 64, 64, 3, 3) == \
        ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv2d_mc_backward_input(g.data_ptr(), w.data_ptr(), g.data_ptr(), 1, 6, 6, 64, 64, 3, 3) == \
        ss.SS_ERR_OVERLAP
    assert ss.ss_conv2d_mc_backward_input(g.data_ptr(), w.data_ptr(), dx.data_ptr(), 0, 6, 6, 64, 64, 3, 3) == \
        ss.SS_ERR_BAD_SIZE


# ---- filter gradient (ss_conv2d_mc_backward_filter, csrc/mc_fgrad.cu 2-D mode, reading R27) ---------
# tensor cores: cin 64, cout 64 (kw <= 4) / 128 (kw <= 2), W <= 128 -- R = floor(128 / W) dy rows per
# tile, CTAs split over the kh tap rows; other shapes (W > 128, kw = 5, other channels): the direct kernel
FG_CASES = [  # (B, H, W, cin, cout, kh, kw)
    (2, 20, 30, 64, 64, 3, 3), (4, 56, 56, 64, 64, 3, 3), (2, 10, 128, 64, 64, 3, 3), (2, 9, 129, 64, 64, 3, 3),
    (3, 17, 9, 64, 128, 2, 2), (2, 30, 40, 64, 64, 1, 1), (2, 30, 40, 64, 64, 5, 1), (1, 7, 7, 64, 64, 7, 4),
    (2, 12, 16, 64, 64, 2, 5), (1, 1, 100, 64, 64, 1, 3), (2, 16, 16, 32, 48, 3, 3), (1, 11, 13, 3, 5, 4, 2),
    (3, 5, 127, 64, 128, 3, 1), (1, 70, 3, 64, 64, 3, 3),
]


def run_fg(ss, gb, xb, kh, kw, off=0):
    B, OH, OW, cout = gb.shape
    _, H, W, cin = xb.shape
    n = cout * cin * kh * kw
    gd, xd = bf16_dev(gb), bf16_dev(xb)
    need = ss.ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw)
    ws = torch.empty(max(need, 8), dtype=torch.uint8, device="cuda")
    buf = torch.full((n + off + 8,), -55.0, device="cuda")
    dw = buf[off:off + n]
    ss.check(ss.ss_conv2d_mc_backward_filter(gd.data_ptr(), xd.data_ptr(), dw.data_ptr(), B, H, W, cin, cout, kh, kw,
                                             ws.data_ptr(), need))
    torch.cuda.synchronize()
    h = buf.cpu().numpy()
    assert np.all(h[:off] == -55.0) and np.all(h[off + n:] == -55.0), "canary overwritten"
    return dw.cpu().numpy().reshape(cout, cin, kh, kw)


@pytest.mark.parametrize("B,H,W,cin,cout,kh,kw", FG_CASES)
def test_conv2d_mc_backward_filter(ss, B, H, W, cin, cout, kh, kw):
    OH, OW = H - kh + 1, W - kw + 1
    gb = oracle.to_bf16_bits(synth.normal(160, B * OH * OW * cout).reshape(B, OH, OW, cout))
    xb = oracle.to_bf16_bits(synth.normal(161, B * H * W * cin).reshape(B, H, W, cin))
    dw = run_fg(ss, gb, xb, kh, kw)
    ref, mag = oracle.conv2d_mc_backward_filter(gb, xb, kh, kw)
    check(dw, ref, mag, f"filter grad B={B} H={H} W={W} cin={cin} cout={cout} k={kh}x{kw}")


def test_conv2d_mc_backward_filter_integers_exact_many_runs(ss):
    # 1728 tiles over 49 CTAs per tap row: every CTA closes more than one 32-tile run (stored, then
    # added); small integers keep every fp32 partial sum exact
    B, H, W, cin, cout, kh, kw = 64, 56, 56, 64, 64, 3, 3
    OH, OW = H - kh + 1, W - kw + 1
    gb = oracle.to_bf16_bits(synth.randint(162, B * OH * OW * cout, -3, 3).astype(np.float32).reshape(B, OH, OW, cout))
    xb = oracle.to_bf16_bits(synth.randint(163, B * H * W * cin, -3, 3).astype(np.float32).reshape(B, H, W, cin))
    dw = run_fg(ss, gb, xb, kh, kw, off=1)
    ref, _ = oracle.conv2d_mc_backward_filter(gb, xb, kh, kw)
    np.testing.assert_array_equal(dw.astype(np.float64), ref)


def test_conv2d_mc_backward_filter_helper_and_validation(ss):
    B, H, W, cin, cout, kh, kw = 2, 40, 50, 64, 64, 3, 3
    g = torch.randn(B, H - kh + 1, W - kw + 1, cout, device="cuda").to(torch.bfloat16)
    x = torch.randn(B, H, W, cin, device="cuda").to(torch.bfloat16)
    a = ss.conv2d_mc_backward_filter(g, x, kh, kw)
    b2 = ss.conv2d_mc_backward_filter(g, x, kh, kw)
    assert torch.equal(a, b2)  # deterministic
    ref = torch.nn.grad.conv2d_weight(x.double().permute(0, 3, 1, 2), (cout, cin, kh, kw),
                                      g.double().permute(0, 3, 1, 2))
    assert torch.allclose(a.double(), ref, rtol=1e-4, atol=1e-3)
    with pytest.raises(ValueError):
        ss.conv2d_mc_backward_filter(g, x, kh + 1, kw)
    dw = torch.empty(cout * cin * kh * kw, device="cuda")
    need = ss.ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw)
    assert need > 0
    args = (B, H, W, cin, cout, kh, kw)
    assert ss.ss_conv2d_mc_backward_filter(g.data_ptr(), x.data_ptr(), dw.data_ptr(), *args, 0, 0) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv2d_mc_backward_filter(0, x.data_ptr(), dw.data_ptr(), *args, 0, 0) == ss.SS_ERR_NULL
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    assert ss.ss_conv2d_mc_backward_filter(g.data_ptr(), x.data_ptr(), dw.data_ptr(), B, 2, W, cin, cout, kh, kw,
                                           ws.data_ptr(), need) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv2d_mc_backward_filter(g.data_ptr(), x.data_ptr(), x.data_ptr(), *args, ws.data_ptr(), need) == \
        ss.SS_ERR_OVERLAP


def test_conv2d_mc_backward_filter_misaligned_dy_uses_the_direct_kernel(ss):
    B, H, W, cin, cout, kh, kw = 2, 12, 20, 64, 64, 3, 3
    OH, OW = H - kh + 1, W - kw + 1
    gb = oracle.to_bf16_bits(synth.normal(164, B * OH * OW * cout).reshape(B, OH, OW, cout))
    xb = oracle.to_bf16_bits(synth.normal(165, B * H * W * cin).reshape(B, H, W, cin))
    n = gb.size
    gbuf = torch.zeros(n + 8, dtype=torch.bfloat16, device="cuda")
    gbuf[1:1 + n] = bf16_dev(gb).reshape(-1)  # dy 2-B aligned, not 16-B
    xd = bf16_dev(xb)
    need = ss.ss_conv2d_mc_backward_filter_workspace(cin, cout, kh, kw)
    ws = torch.empty(max(need, 8), dtype=torch.uint8, device="cuda")
    dw = torch.empty(cout * cin * kh * kw, device="cuda")
    ss.check(ss.ss_conv2d_mc_backward_filter(gbuf[1:].data_ptr(), xd.data_ptr(), dw.data_ptr(), B, H, W, cin, cout,
                                             kh, kw, ws.data_ptr(), need))
    ref, mag = oracle.conv2d_mc_backward_filter(gb, xb, kh, kw)
    check(dw.cpu().numpy().reshape(cout, cin, kh, kw), ref, mag, "filter grad, dy offset by one element")
