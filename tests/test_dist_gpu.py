"""Multi-rank run of the sharded hot path with the real kernels, several ranks
on the one available GPU (gloo, host-staged halo: no rank's kernel ever waits
on another rank).  Sharded outputs must equal the unsharded run bitwise."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nproc", [2, 3])
def test_sharded_suite_equals_unsharded(nproc):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + nproc),
           os.path.join(ROOT, "tools", "dist_check.py"), "--backend", "gloo"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "DIST_CHECK PASS" in out, out[-4000:]


def _bench_line(stdout: str) -> dict:
    import json
    lines = [ln for ln in stdout.splitlines() if ln.startswith("{") and '"metric"' in ln]
    assert lines, stdout[-4000:]
    return json.loads(lines[-1])


def test_bench_self_launch_two_ranks_gloo():
    """`bench.py --gpus 2` without WORLD_SIZE re-launches itself with 2 ranks (here
    both on the one GPU, gloo host-staged halo); the line reports n_gpus 2, the
    same graph launch mode as N = 1, and sharded == unsharded outputs bitwise for
    the suite (sequence-sharded cfg2 with its halo, batch-sharded cfg3 / cfg4) and
    the strong-scaled config-5 sub-record (2^28 elements here)."""
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--dist-backend", "gloo", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline", "--verify", "--cfg5-log2n", "28", "--cfg5-steps", "3", "--cell-reps", "2",
           "--e2e-steps", "2"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    line = _bench_line(r.stdout)
    assert line["n_gpus"] == 2 and line["impl"] == "ours"
    assert line["gpu_launches"] > 0
    assert "CUDA graphs at every N" in line["config"]["launch_mode"]
    v = line["verify"]
    assert v["compared"] > 0 and v["mismatches"] == 0, v
    c5 = line["cfg5"]
    assert c5["n_gpus"] == 2 and c5["scaling"] == "strong"
    assert c5["verify"]["compared"] > 0 and c5["verify"]["mismatches"] == 0, c5["verify"]
    assert line["e2e"]["h2d_bytes_per_step"] > 0
