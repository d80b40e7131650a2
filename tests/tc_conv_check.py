"""Quick GPU check of the tensor-core conv path (csrc/conv_tc.cu): parity against
the oracle over shapes / alignments, forced onto the TC path with
SS_CONV_TC_MIN_K=1, then per-NC timing of BASELINE config 3 (64 x 2^20,
k in {31, 48, 63}) against the FFMA2 tile kernel.  Usage (GPU box):
    SS_CONV_TC_MIN_K=1 python tests/tc_conv_check.py [parity|time|trace]
(test infrastructure: imports oracle/; tests/test_conv_tc_gpu.py runs the parity mode)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2305_16513_b200 as ss  # noqa: E402
import synth  # noqa: E402


def parity():
    cases = [(1, 200, 1), (1, 5000, 8), (3, 1000, 33), (2, 70001, 63), (1, 65536, 64), (5, 9999, 40),
             (64, 4096, 63), (7, 333, 64), (1, 1 << 18, 48), (4, 12345, 17), (2, 190, 63), (3, 130, 64)]
    worst = 0.0
    for (B, N, k) in cases:
        for xoff in (0, 1, 3):
            x = synth.normal(3, B * N).reshape(B, N)
            f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
            buf = torch.zeros(B * N + 8, device="cuda")
            buf[xoff:xoff + B * N] = torch.from_numpy(x.reshape(-1)).cuda()
            xd = buf[xoff:xoff + B * N].view(B, N)
            L = N - k + 1
            ybuf = torch.full((B * L + 9,), -777.0, device="cuda")
            y = ybuf[1:1 + B * L].view(B, L)
            n0 = ss.ss_launch_count()
            ss.conv1d(xd, f, out=y)
            torch.cuda.synchronize()
            h = ybuf.cpu().numpy()
            assert h[0] == -777.0 and np.all(h[1 + B * L:] == -777.0), "canary"
            ref, mag = oracle.conv1d(x, f)
            err = np.abs(y.cpu().numpy().astype(np.float64) - ref)
            ratio = float((err / (1e-5 * mag + 1e-6)).max())
            worst = max(worst, ratio)
            bad = int((err > 1e-5 * mag + 1e-6).sum())
            print(f"B={B} N={N} k={k} xoff={xoff}: launches {ss.ss_launch_count() - n0} max err/bound {ratio:.3g} bad {bad}",
                  flush=True)
            assert bad == 0
    print("parity ok, worst err/bound", worst)


def timing():
    B, N = 64, 1 << 20
    x = torch.empty(B, N, device="cuda")
    synth.fill_device(x, "normal", 3)
    ks = [int(v) for v in os.environ.get("KS", "31,48,63").split(",")]
    reps = int(os.environ.get("REPS", "12"))
    for k in ks:
        f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
        y = torch.empty(B, N - k + 1, device="cuda")
        flush = torch.empty(64 << 20, device="cuda")
        ts = []
        for it in range(reps):
            flush.fill_(1.0)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ss.conv1d(x, f, out=y)
            b.record()
            torch.cuda.synchronize()
            if it >= min(2, reps - 1):
                ts.append(a.elapsed_time(b))
        t = sorted(ts)[len(ts) // 2]
        outs = B * (N - k + 1)
        print(f"k={k}: {t * 1e3:.1f} us  {outs / t / 1e6:.1f} GElem/s  {8 * outs / t / 1e6:.0f} GB/s", flush=True)


def trace():
    import ctypes
    B, N, k = 64, 1 << 20, int(os.environ.get("KS", "63"))
    x = torch.empty(B, N, device="cuda")
    synth.fill_device(x, "normal", 3)
    f = synth.normal(4, k, sigma=synth.cfg_sigma_filter(k))
    y = torch.empty(B, N - k + 1, device="cuda")
    tbuf = torch.zeros(1024, dtype=torch.int64, device="cuda")  # caller-owned trace buffer
    ss.lib.ss_debug_conv_tc_set_trace(ctypes.c_void_p(tbuf.data_ptr()))
    for _ in range(int(os.environ.get("REPS", "3"))):
        ss.conv1d(x, f, out=y)
    torch.cuda.synchronize()
    ss.lib.ss_debug_conv_tc_set_trace(ctypes.c_void_p(0))
    allv = tbuf.cpu().numpy()
    t = allv[:512].reshape(64, 8)

    t0 = t[0, 0]
    names = ["P.iss0", "P.iss1", "S.full0", "M.data0", "M.issued", "S.full1", "M.data1", "E.dfull"]
    print("tile " + " ".join(f"{n:>9s}" for n in names))
    n = 0
    for i in range(t.shape[0]):
        if t[i, 0] == 0:
            break
        n = i + 1
        if i < 6 or i >= int(os.environ.get("TAIL", "50")):
            print(f"{i:4d} " + " ".join(f"{v - t0:9d}" for v in t[i]))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ss.conv1d(x, f, out=y)
    b.record()
    torch.cuda.synchronize()
    g = allv[63 * 8: 63 * 8 + 6]
    if g[0]:
        print(f"CTA 0 globaltimer: setup {(g[2] - g[0]) / 1e3:.1f} us, setup->exit {(g[4] - g[2]) / 1e3:.1f} us; "
              f"clock {(g[5] - g[1]) / ((g[4] - g[0]) / 1e3):.0f} MHz; first tile start at +{(t0 - g[1])} clk")
    ce = allv[512:].reshape(256, 2)
    ce = ce[ce[:, 0] > 0]
    if len(ce):
        g0 = ce[:, 0].min()
        print(f"{len(ce)} CTAs: entry spread {(ce[:, 0].max() - g0) / 1e3:.1f} us, exit min / median / max "
              f"{(ce[:, 1].min() - g0) / 1e3:.1f} / {(np.median(ce[:, 1]) - g0) / 1e3:.1f} / "
              f"{(ce[:, 1].max() - g0) / 1e3:.1f} us after the first entry")
        allce = allv[512:].reshape(256, 2)
        order = np.argsort(allce[:, 1])[::-1]
        print("slowest CTAs (index: exit us):",
              ", ".join(f"{i}: {(allce[i, 1] - g0) / 1e3:.1f}" for i in order[:8] if allce[i, 1] > 0))
    span = t[n - 1, 7] - t0
    print(f"CTA 0: {n} tiles, span {span} clk; event time of one call {a.elapsed_time(b) * 1e3:.1f} us "
          f"-> {span / (a.elapsed_time(b) * 1e3):.0f} MHz if the span were the whole kernel")
    d = np.diff(t[5:40, 4])
    print("MMA issue-done period (clk): median", np.median(d))


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "parity"
    if what == "parity":
        parity()
    elif what == "trace":
        trace()
    else:
        timing()
