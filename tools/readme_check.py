"""Runs the README usage snippet (extracted verbatim) on a GPU: python tools/readme_check.py"""
import sys, os; sys.path.insert(0, os.getcwd()); import torch, paper_2305_16513_b200 as ss      # build first: python -c 'import __graft_entry__ as g; g.build()'
x = torch.randn(64, 1 << 20, device="cuda")
y_max = ss.pool_max(x, 64)                      # Eq. 3 with max, window 64
y_sum = ss.pool_sum(x, 8, stride=2, padding=3)  # raw window sums, zero padding
y_min = ss.pool_min(x, 16, padding=(8, 7), pad_mode="circular")  # periodic boundary
y_cnv = ss.conv1d(x, torch.randn(63))           # cross-correlation, k = 63 (tensor cores)
dx = ss.conv1d_backward_input(torch.randn_like(y_cnv), torch.randn(63), x.shape[1])
x4 = torch.rand(32, 64, 112, 112, device="cuda"); f3 = torch.randn(3, 3)
g4 = torch.randn(32, 64, 110, 110, device="cuda")      # dL/dy of ss.conv2d(x4, f3)
dx4 = ss.conv2d_backward_input(g4, f3, 112, 112); df3 = ss.conv2d_backward_filter(x4, g4, (3, 3))
xm = torch.randn(8, 56, 56, 64, device="cuda").to(torch.bfloat16)      # NHWC, multi-channel (tcgen05)
wm = (torch.randn(64, 64, 3, 3, device="cuda") / 24).to(torch.bfloat16)
ym = ss.conv2d_mc(xm, wm)                                               # fp32 [8, 54, 54, 64]
gm = torch.randn_like(ym).to(torch.bfloat16)
dxm = ss.conv2d_mc_backward_input(gm, wm, 56, 56); dwm = ss.conv2d_mc_backward_filter(gm, xm, 3, 3)

torch.cuda.synchronize(); print('readme ok', y_cnv.shape, dxm.shape, dwm.shape)
