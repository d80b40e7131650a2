"""Launch the stride-1 max-pool gradient on the backward workload's shape, w = 16 (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_16513_b200 as ss  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 16
x = torch.randn(64, 1 << 20, device="cuda")
dy = torch.randn(64, (1 << 20) - w + 1, device="cuda")
for _ in range(2):
    ss.pool_max_backward(x, dy, w)
torch.cuda.synchronize()
