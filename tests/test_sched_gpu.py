"""Dynamic work claims of the persistent kernels by cluster launch control
(ss_device.cuh ClcSmem): the grid has one CTA
per tile / plane and running CTAs cancel not-yet-launched CTAs to take their
units, so the claim state lives in the hardware scheduler -- the library keeps
no device memory and no state between launches (include/ss.h ownership).
Which SM computes a unit must not change any output; calls on concurrent
streams, graph replays (including two captured graphs replayed concurrently,
and a capture that is the very first call of the process) must not disturb
each other.  Covers the 1-D TMA tile kernel (sum / max / conv k <= 32), the
tensor-core conv (k = 63), the 2-D pooling and 2-D conv vector kernels and the
multi-channel conv, against eager single-stream results (bit for bit) and
against the static schedule (SS_DYNAMIC_TILES=0, subprocess)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ss():
    import paper_2305_16513_b200 as ss
    return ss


def workload(ss, seed=0):
    """[(name, fn)]: one call of each persistent kernel on fixed synthetic inputs."""
    xi = torch.from_numpy(synth.randint(40 + seed, 3 << 20, -1000, 1000)).cuda()
    xf = torch.from_numpy(synth.normal(41 + seed, 8 * 300001).reshape(8, 300001)).cuda()
    x4 = torch.from_numpy(synth.uniform01(42 + seed, 2 * 64 * 112 * 112).reshape(2, 64, 112, 112)).cuda()
    f7 = synth.normal(43, 7, sigma=synth.cfg_sigma_filter(7))
    f63 = synth.normal(44, 63, sigma=synth.cfg_sigma_filter(63))
    f2 = synth.normal(45, 9).reshape(3, 3)
    xm = torch.from_numpy(synth.normal(46, 4 * 5000 * 64).reshape(4, 5000, 64)).cuda().to(torch.bfloat16)
    wm = torch.from_numpy(synth.normal(47, 64 * 64 * 3, sigma=0.1).reshape(64, 64, 3)).cuda().to(torch.bfloat16)
    return [
        ("sum_i32_w16", lambda: ss.pool_sum(xi, 16)),
        ("max_i32_w64", lambda: ss.pool_max(xi, 64)),
        ("conv_k7", lambda: ss.conv1d(xf, f7)),
        ("conv_k63_tc", lambda: ss.conv1d(xf, f63)),
        ("pool2d_max_3x3", lambda: ss.pool2d(x4, (3, 3), (1, 1), "max")),
        ("pool2d_avg_2x2", lambda: ss.pool2d(x4, (2, 2), (2, 2), "avg")),
        ("conv2d_3x3", lambda: ss.conv2d(x4.reshape(-1, 112, 112), f2)),
        ("conv1d_mc", lambda: ss.conv1d_mc(xm, wm)),
    ]


def test_repeated_calls_and_concurrent_streams_bitwise(ss):
    calls = workload(ss)
    ref = {n: fn().clone() for n, fn in calls}
    torch.cuda.synchronize()
    for _ in range(3):
        for n, fn in calls:
            assert torch.equal(fn(), ref[n]), n
    # two streams, interleaved
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs = []
    for rep in range(4):
        for i, (n, fn) in enumerate(calls):
            st = s1 if (i + rep) % 2 == 0 else s2
            with torch.cuda.stream(st):
                outs.append((n, fn()))
    torch.cuda.synchronize()
    for n, y in outs:
        assert torch.equal(y, ref[n]), n


def test_graph_replays_bitwise(ss):
    calls = workload(ss, seed=1)
    ref = {n: fn().clone() for n, fn in calls}
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        outs = [(n, fn()) for n, fn in calls]
    for _ in range(5):
        g.replay()
        torch.cuda.synchronize()
        for n, y in outs:
            assert torch.equal(y, ref[n]), n


_CHILD = r"""
import sys, torch, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import paper_2305_16513_b200 as ss
from test_sched_gpu import workload
np.savez({out!r}, **{{n: fn().float().cpu().numpy() for n, fn in workload(ss)}})
"""


def test_static_and_dynamic_schedules_agree(tmp_path):
    res = {}
    for dyn in ("0", "1"):
        out = str(tmp_path / f"sched{dyn}.npz")
        env = dict(os.environ, SS_DYNAMIC_TILES=dyn)
        code = _CHILD.format(root=ROOT, tests=os.path.join(ROOT, "tests"), out=out)
        subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=ROOT, timeout=600)
        res[dyn] = np.load(out)
    for n in res["0"].files:
        np.testing.assert_array_equal(res["0"][n], res["1"][n], err_msg=n)


def test_concurrent_graph_replays_and_eager_bitwise(ss):
    """Two graphs of the same launches, replayed at the same time on two streams
    while eager calls run on a third: no claim of one launch may leak into another."""
    calls = workload(ss, seed=2)
    ref = {n: fn().clone() for n, fn in calls}
    torch.cuda.synchronize()
    graphs = []
    for _ in range(2):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            outs = [(n, fn()) for n, fn in calls]
        graphs.append((g, outs))
    streams = [torch.cuda.Stream() for _ in range(3)]
    torch.cuda.synchronize()
    for _ in range(4):
        eager = []
        for (g, _), st in zip(graphs, streams):
            with torch.cuda.stream(st):
                g.replay()
        with torch.cuda.stream(streams[2]):
            eager = [(n, fn()) for n, fn in calls]
        torch.cuda.synchronize()
        for _, outs in graphs:
            for n, y in outs:
                assert torch.equal(y, ref[n]), n
        for n, y in eager:
            assert torch.equal(y, ref[n]), n


_CAPTURE_FIRST = r"""
import sys, torch, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import paper_2305_16513_b200 as ss
from test_sched_gpu import workload
calls = workload(ss, seed=3)
torch.cuda.synchronize()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):   # the first libss calls of this process
    outs = [(n, fn()) for n, fn in calls]
g.replay(); g.replay()
torch.cuda.synchronize()
cap = {{n: y.float().cpu().numpy() for n, y in outs}}
ref = {{n: fn().float().cpu().numpy() for n, fn in calls}}
for n in ref:
    assert np.array_equal(cap[n], ref[n]), n
print("capture-first ok")
"""


def test_first_call_inside_capture():
    code = _CAPTURE_FIRST.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ), cwd=ROOT, timeout=600,
                       capture_output=True, text=True)
    assert r.returncode == 0 and "capture-first ok" in r.stdout, r.stdout + r.stderr
