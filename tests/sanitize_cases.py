"""Small cases through every kernel family, checked against the oracle; meant to
run under compute-sanitizer (one --tool per invocation):
    compute-sanitizer --tool memcheck python tests/sanitize_cases.py
Exits non-zero on a parity failure."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2305_16513_b200 as ss  # noqa: E402
import synth  # noqa: E402

bad = 0


def chk(name, ok):
    global bad
    if not ok:
        bad += 1
        print("FAIL", name)


for N, B, w in ((20011, 3, 3), (20011, 2, 8), (30011, 2, 16), (30011, 1, 40), (40011, 2, 64), (40011, 1, 256),
                (1000, 2, 2), (300, 1, 1000 if False else 100)):
    x = synth.randint(2, B * N, -1000, 1000).reshape(B, N)
    xt = torch.from_numpy(x).cuda()
    ys = ss.pool_sum(xt, w).cpu().numpy()
    ym = ss.pool_max(xt, w).cpu().numpy()
    ref = oracle.pool_sum(x, w)
    chk(f"sum {N} {B} {w}", np.array_equal(ys, (ref & 0xFFFFFFFF).astype(np.uint32).view(np.int32)))
    chk(f"max {N} {B} {w}", np.array_equal(ym, oracle.pool_max(x, w)))
for N, B, k in ((20011, 3, 3), (30011, 2, 31), (30011, 1, 63), (5000, 1, 100)):
    x = synth.normal(3, B * N).reshape(B, N)
    f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
    y = ss.conv1d(torch.from_numpy(x).cuda(), f).cpu().numpy()
    ref, mag = oracle.conv1d(x, f)
    chk(f"conv {N} {B} {k}", bool(np.all(np.abs(y - ref) <= 1e-5 * mag + 1e-6)))
for P, H, W, kk, s in ((3, 112, 112, 3, 1), (3, 112, 112, 2, 2), (2, 31, 45, 3, 2)):
    x = synth.uniform01(5, P * H * W).reshape(P, H, W)
    y = ss.pool2d(torch.from_numpy(x).cuda(), (kk, kk), (s, s), "max").cpu().numpy()
    ref, _ = oracle.pool2d(x, kk, kk, s, s, 0)
    chk(f"pool2d {P} {H} {W} {kk} {s}", np.array_equal(y.astype(np.float64), ref))
torch.cuda.synchronize()
print("sanitize cases done, failures:", bad)
sys.exit(1 if bad else 0)
