"""Launch the stride-1 filter gradient on the bench shape (64 x 2^20, k) for ncu captures:
    python tools/fgrad_prof.py [k] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_16513_b200 as ss  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 63
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N = 1 << 20
x = torch.randn(64, N, device="cuda")
dy = torch.randn(64, N - k + 1, device="cuda")
for _ in range(reps):
    df = ss.conv1d_backward_filter(x, dy, k)
torch.cuda.synchronize()
print("df[0:3]", df[:3].tolist())
