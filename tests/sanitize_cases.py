"""Small cases through every kernel family (incl. the 2-D conv gradients and the
padded sliding min), checked against the oracle; written to run under
compute-sanitizer (one --tool per invocation) where it is available:
    compute-sanitizer --tool memcheck python tests/sanitize_cases.py
(the GPU pool of this round has compute-sanitizer disabled, so it ran plainly:
0 failures).  Exits non-zero on a parity failure."""
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
for P, H, W, kh, kw, sh, sw in ((2, 37, 150, 3, 3, 1, 1), (1, 30, 140, 7, 7, 1, 1), (2, 41, 259, 4, 2, 2, 3),
                               (1, 40, 40, 5, 6, 1, 1), (1, 1030, 3, 1024, 1, 1, 1)):
    OH, OW = (H - kh) // sh + 1, (W - kw) // sw + 1
    x = synth.normal(90, P * H * W).reshape(P, H, W)
    f = synth.normal(91, kh * kw).reshape(kh, kw)
    g = synth.normal(92, P * OH * OW).reshape(P, OH, OW)
    dx = ss.conv2d_backward_input(torch.from_numpy(g).cuda(), f, H, W, (sh, sw)).cpu().numpy()
    df = ss.conv2d_backward_filter(torch.from_numpy(x).cuda(), torch.from_numpy(g).cuda(), (kh, kw),
                                   (sh, sw)).cpu().numpy()
    ref, mag = oracle.conv2d_backward_input(g, f, H, W, sh, sw)
    chk(f"conv2d dx {P} {H} {W} {kh} {kw}", bool(np.all(np.abs(dx - ref) <= 1e-5 * mag + 1e-6)))
    ref, mag = oracle.conv2d_backward_filter(x, g, kh, kw, sh, sw)
    chk(f"conv2d df {P} {H} {W} {kh} {kw}", bool(np.all(np.abs(df - ref) <= 1e-5 * mag + 1e-6)))
for mode in ("reflect", "circular", "replicate"):
    x = synth.normal(3, 2 * 20011).reshape(2, 20011)
    y = ss.pool_min(torch.from_numpy(x).cuda(), 16, padding=(8, 7), pad_mode=mode).cpu().numpy()
    chk(f"min {mode}", np.array_equal(y, oracle.pool_min_ex(x, 16, 1, 1, 8, 7, mode)))
torch.cuda.synchronize()
print("sanitize cases done, failures:", bad)
sys.exit(1 if bad else 0)
