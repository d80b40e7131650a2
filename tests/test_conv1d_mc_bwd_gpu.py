"""GPU parity of the multi-channel conv1d backward passes.  Filter gradient
(ss_conv1d_mc_backward_filter, csrc/mc_fgrad.cu, reading R25): tensor-core and direct
shapes, integer exactness, determinism, validation (bottom of the file).  Input gradient
(ss_conv1d_mc_backward_input, csrc/conv_mc.cu batched/transposed mode; SURVEY 8f NEXT #4,
DESIGN.md reading R23):
bf16 dy [B, N-k+1, Cout], bf16 w [Cout, Cin, k], fp32 dx [B, N, Cin], against
oracle.conv1d_mc_backward_input (the same bf16 values in double) within
1e-5 * sum|terms| + 1e-6.  Tensor-core shapes (cin, cout in {64, 128}, k <= 9:
per-row tiles whose TMA box starts k-1 positions before the row, zero-filled),
rows shorter than a tile, ragged row tails, k = 1, the direct kernel (other
shapes, misaligned dx), canaries, integer exactness, a forward/backward adjoint
check through the library, validation."""
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


def run(ss, gb, wb, N, off=0):
    B, L, cout = gb.shape
    _, cin, k = wb.shape
    n = B * N * cin
    gd, wd = bf16_dev(gb), bf16_dev(wb)
    buf = torch.full((n + off + 8,), -55.0, device="cuda")
    dx = buf[off:off + n]
    ss.check(ss.ss_conv1d_mc_backward_input(gd.data_ptr(), wd.data_ptr(), dx.data_ptr(), B, N, cin, cout, k))
    torch.cuda.synchronize()
    h = buf.cpu().numpy()
    assert np.all(h[:off] == -55.0) and np.all(h[off + n:] == -55.0), "canary overwritten"
    return dx.cpu().numpy().reshape(B, N, cin)


def check(y, ref, mag, what):
    err = np.abs(y.astype(np.float64) - ref)
    bound = TOL_REL * mag + TOL_ABS
    assert np.all(err <= bound), f"{what}: {(err > bound).sum()} out of bound, max err/bound {(err / bound).max():.3g}"


def inputs(B, N, cin, cout, k, seed):
    L = N - k + 1
    gb = oracle.to_bf16_bits(synth.normal(seed, B * L * cout).reshape(B, L, cout))
    wb = oracle.to_bf16_bits(synth.normal(seed + 1, cout * cin * k, sigma=(cout * k) ** -0.5).reshape(cout, cin, k))
    return gb, wb


CASES = [  # (B, N, cin, cout, k)
    (2, 1000, 64, 64, 3), (3, 777, 128, 64, 5), (1, 4096, 64, 128, 9), (2, 300, 128, 128, 1),
    (5, 129, 64, 64, 2), (1, 20000, 128, 128, 3), (4, 100, 64, 64, 7), (3, 128, 64, 64, 3), (2, 9, 64, 64, 9),
    (2, 200, 32, 48, 3), (1, 500, 3, 5, 7), (2, 400, 64, 64, 12),
]


@pytest.mark.parametrize("B,N,cin,cout,k", CASES)
def test_conv1d_mc_backward_input(ss, B, N, cin, cout, k):
    gb, wb = inputs(B, N, cin, cout, k, 110)
    dx = run(ss, gb, wb, N)
    ref, mag = oracle.conv1d_mc_backward_input(gb, wb, N)
    check(dx, ref, mag, f"B={B} N={N} cin={cin} cout={cout} k={k}")


def test_misaligned_dx_uses_the_direct_kernel(ss):
    gb, wb = inputs(2, 300, 64, 64, 5, 112)
    dx = run(ss, gb, wb, 300, off=1)
    ref, mag = oracle.conv1d_mc_backward_input(gb, wb, 300)
    check(dx, ref, mag, "dx offset by one float")


def test_integer_valued_inputs_are_exact(ss):
    B, N, cin, cout, k = 3, 700, 64, 128, 5
    L = N - k + 1
    gb = oracle.to_bf16_bits(synth.randint(114, B * L * cout, -3, 3).astype(np.float32).reshape(B, L, cout))
    wb = oracle.to_bf16_bits(synth.randint(115, cout * cin * k, -2, 2).astype(np.float32).reshape(cout, cin, k))
    dx = run(ss, gb, wb, N)
    ref, _ = oracle.conv1d_mc_backward_input(gb, wb, N)
    np.testing.assert_array_equal(dx.astype(np.float64), ref)


def test_adjoint_of_the_forward_kernel(ss):
    # <conv1d_mc(x, w), g> == <x, conv1d_mc_backward_input(g, w)>, both sides from the library's kernels
    B, N, cin, cout, k = 2, 2000, 64, 64, 7
    x = torch.randn(B, N, cin, device="cuda").to(torch.bfloat16)
    w = (torch.randn(cout, cin, k, device="cuda") * (cin * k) ** -0.5).to(torch.bfloat16)
    g = torch.randn(B, N - k + 1, cout, device="cuda").to(torch.bfloat16)
    y = ss.conv1d_mc(x, w)
    dx = ss.conv1d_mc_backward_input(g, w, N)
    lhs = (y.double() * g.double()).sum().item()
    rhs = (x.double() * dx.double()).sum().item()
    assert abs(lhs - rhs) <= 1e-4 * (y.double().abs() * g.double().abs()).sum().item()


def test_validation(ss):
    g = torch.zeros(1, 4, 64, dtype=torch.bfloat16, device="cuda")
    w = torch.zeros(64, 64, 3, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        ss.conv1d_mc_backward_input(g, w, 7)        # dy length != N-k+1
    with pytest.raises(ss.SSError):
        ss.conv1d_mc_backward_input(g, w, 2)        # k > N
    dx = torch.empty(1000, device="cuda")
    assert ss.ss_conv1d_mc_backward_input(0, w.data_ptr(), dx.data_ptr(), 1, 6, 64, 64, 3) == ss.SS_ERR_NULL
    assert ss.ss_conv1d_mc_backward_input(g.data_ptr(), w.data_ptr(), dx.data_ptr(), 1, 2, 64, 64, 3) == \
        ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv1d_mc_backward_input(g.data_ptr(), w.data_ptr(), g.data_ptr(), 1, 6, 64, 64, 3) == \
        ss.SS_ERR_OVERLAP


# ---- filter gradient (ss_conv1d_mc_backward_filter, csrc/mc_fgrad.cu, reading R25) -----------------
# tensor cores: cin 64, cout 64 (k <= 4) / 128 (k <= 2) -- tiles of 128 positions per row (row tails,
# rows shorter than a tile, more tiles than CTAs, runs of 16 tiles); other shapes: the direct kernel
FG_CASES = [  # (B, N, cin, cout, k)
    (2, 1000, 64, 64, 3), (3, 777, 64, 64, 1), (1, 4096, 64, 64, 4), (2, 300, 64, 128, 2), (5, 129, 64, 64, 2),
    (1, 20000, 64, 128, 1), (4, 100, 64, 64, 3), (64, 2050, 64, 64, 3), (1, 9, 64, 64, 4),
    (2, 200, 32, 48, 3), (1, 500, 3, 5, 7), (2, 60, 128, 128, 3), (2, 50, 64, 64, 9),
]


def run_fg(ss, gb, xb, k, off=0):
    B, L, cout = gb.shape
    _, N, cin = xb.shape
    n = cout * cin * k
    gd, xd = bf16_dev(gb), bf16_dev(xb)
    need = ss.ss_conv1d_mc_backward_filter_workspace(cin, cout, k)
    ws = torch.empty(max(need, 8), dtype=torch.uint8, device="cuda")
    buf = torch.full((n + off + 8,), -55.0, device="cuda")
    dw = buf[off:off + n]
    ss.check(ss.ss_conv1d_mc_backward_filter(gd.data_ptr(), xd.data_ptr(), dw.data_ptr(), B, N, cin, cout, k,
                                             ws.data_ptr(), need))
    torch.cuda.synchronize()
    h = buf.cpu().numpy()
    assert np.all(h[:off] == -55.0) and np.all(h[off + n:] == -55.0), "canary overwritten"
    return dw.cpu().numpy().reshape(cout, cin, k)


@pytest.mark.parametrize("B,N,cin,cout,k", FG_CASES)
def test_conv1d_mc_backward_filter(ss, B, N, cin, cout, k):
    L = N - k + 1
    gb = oracle.to_bf16_bits(synth.normal(120, B * L * cout).reshape(B, L, cout))
    xb = oracle.to_bf16_bits(synth.normal(121, B * N * cin).reshape(B, N, cin))
    dw = run_fg(ss, gb, xb, k)
    ref, mag = oracle.conv1d_mc_backward_filter(gb, xb, k)
    check(dw, ref, mag, f"filter grad B={B} N={N} cin={cin} cout={cout} k={k}")


def test_conv1d_mc_backward_filter_integers_exact(ss):
    # small integers: bf16 products exact, every partial sum an exact integer in fp32
    B, N, cin, cout, k = 3, 2000, 64, 64, 3
    L = N - k + 1
    gb = oracle.to_bf16_bits(synth.randint(122, B * L * cout, -3, 3).astype(np.float32).reshape(B, L, cout))
    xb = oracle.to_bf16_bits(synth.randint(123, B * N * cin, -3, 3).astype(np.float32).reshape(B, N, cin))
    dw = run_fg(ss, gb, xb, k, off=1)
    ref, _ = oracle.conv1d_mc_backward_filter(gb, xb, k)
    np.testing.assert_array_equal(dw.astype(np.float64), ref)


def test_conv1d_mc_backward_filter_helper_and_validation(ss):
    B, N, cin, cout, k = 2, 500, 64, 64, 3
    g = torch.randn(B, N - k + 1, cout, device="cuda").to(torch.bfloat16)
    x = torch.randn(B, N, cin, device="cuda").to(torch.bfloat16)
    a = ss.conv1d_mc_backward_filter(g, x, k)
    b2 = ss.conv1d_mc_backward_filter(g, x, k)
    assert torch.equal(a, b2)  # deterministic
    ref = torch.nn.grad.conv1d_weight(x.double().permute(0, 2, 1), (cout, cin, k), g.double().permute(0, 2, 1))
    assert torch.allclose(a.double(), ref, rtol=1e-4, atol=1e-3)
    with pytest.raises(ValueError):
        ss.conv1d_mc_backward_filter(g, x, k + 1)
    dw = torch.empty(cout * cin * k, device="cuda")
    need = ss.ss_conv1d_mc_backward_filter_workspace(cin, cout, k)
    assert need > 0
    assert ss.ss_conv1d_mc_backward_filter(g.data_ptr(), x.data_ptr(), dw.data_ptr(), B, N, cin, cout, k, 0, 0) == \
        ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv1d_mc_backward_filter(0, x.data_ptr(), dw.data_ptr(), B, N, cin, cout, k, 0, 0) == ss.SS_ERR_NULL
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    assert ss.ss_conv1d_mc_backward_filter(g.data_ptr(), x.data_ptr(), dw.data_ptr(), B, 2, cin, cout, k,
                                           ws.data_ptr(), need) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
