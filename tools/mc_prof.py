"""Launch the multi-channel conv kernels on their bench shapes (for ncu captures):
    python tools/mc_prof.py [2d|1d9|dx|dw|dw128|dx2d|dw2d] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_16513_b200 as ss  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "2d"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
torch.manual_seed(0)
if which == "2d":
    x = torch.randn(128, 56, 56, 64, device="cuda").to(torch.bfloat16)
    w = (torch.randn(64, 64, 3, 3, device="cuda") / 24).to(torch.bfloat16)
    f = lambda: ss.conv2d_mc(x, w)  # noqa: E731
elif which == "1d9":
    x = torch.randn(16, 65536, 64, device="cuda").to(torch.bfloat16)
    w = (torch.randn(64, 64, 9, device="cuda") / 24).to(torch.bfloat16)
    f = lambda: ss.conv1d_mc(x, w)  # noqa: E731
elif which == "dw":
    g = torch.randn(16, 65534, 64, device="cuda").to(torch.bfloat16)
    x = torch.randn(16, 65536, 64, device="cuda").to(torch.bfloat16)
    dw = torch.empty(64, 64, 3, device="cuda")
    wsb = torch.empty(ss.ss_conv1d_mc_backward_filter_workspace(64, 64, 3), dtype=torch.uint8, device="cuda")
    f = lambda: ss.conv1d_mc_backward_filter(g, x, 3, out=dw, workspace=wsb)  # noqa: E731
elif which == "dw128":
    g = torch.randn(16, 65535, 128, device="cuda").to(torch.bfloat16)
    x = torch.randn(16, 65536, 64, device="cuda").to(torch.bfloat16)
    dw = torch.empty(128, 64, 2, device="cuda")
    wsb = torch.empty(ss.ss_conv1d_mc_backward_filter_workspace(64, 128, 2), dtype=torch.uint8, device="cuda")
    f = lambda: ss.conv1d_mc_backward_filter(g, x, 2, out=dw, workspace=wsb)  # noqa: E731
elif which == "dw2d":
    g = torch.randn(128, 54, 54, 64, device="cuda").to(torch.bfloat16)
    x = torch.randn(128, 56, 56, 64, device="cuda").to(torch.bfloat16)
    dw = torch.empty(64, 64, 3, 3, device="cuda")
    wsb = torch.empty(ss.ss_conv2d_mc_backward_filter_workspace(64, 64, 3, 3), dtype=torch.uint8, device="cuda")
    f = lambda: ss.conv2d_mc_backward_filter(g, x, 3, 3, out=dw, workspace=wsb)  # noqa: E731
elif which == "dx2d":
    g = torch.randn(128, 54, 54, 64, device="cuda").to(torch.bfloat16)
    w = (torch.randn(64, 64, 3, 3, device="cuda") / 24).to(torch.bfloat16)
    f = lambda: ss.conv2d_mc_backward_input(g, w, 56, 56)  # noqa: E731
else:
    g = torch.randn(16, 65534, 64, device="cuda").to(torch.bfloat16)
    w = (torch.randn(64, 64, 3, device="cuda") / 24).to(torch.bfloat16)
    f = lambda: ss.conv1d_mc_backward_input(g, w, 65536)  # noqa: E731
for _ in range(reps):
    f()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    f()
e.record()
torch.cuda.synchronize()
print(which, "avg us", s.elapsed_time(e) / 20 * 1e3)
