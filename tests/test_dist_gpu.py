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
