"""Multi-rank check of the sharded hot path with the real kernels:
    torchrun --nproc-per-node 2 tools/dist_check.py [--backend gloo|nccl]
Each rank runs bench.Runner on its share of configs 2 (sequence-sharded with
the halo exchange), 3 and 4 (batch-sharded) at reduced sizes, gathers its
outputs to rank 0, and rank 0 compares them bitwise with an unsharded
single-process run of the same kernels (max, int32 sums and FFMA conv
(k <= 32) are shard-invariant bitwise; the tensor-core conv (33 <= k <= 64)
rounds by position, so those cells are compared within twice the
BASELINE.json bound 1e-5 * sum|x f| + 1e-6)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402


def small(inputs, cells):
    """Shrink the BASELINE shapes (keep structure: ragged shards, batch rows)."""
    for k, sp in inputs.items():
        if "n" in sp and sp.get("shard") == "seq":
            sp["n"] = 3 * 1_000_003
        if sp.get("shard") == "batch":
            sp["rows"], sp["n"] = 6, 70_001
        if sp.get("shard") == "image":
            sp["images"], sp["C"] = 3, 4
    return inputs, cells


def tc_cell(c):
    return c.op == "conv" and 33 <= c.w <= 64 and c.stride == 1 and c.dilation == 1 and tuple(c.pads) == (0, 0)


def close_within_bound(a, b, R1, c):
    """|a - b| <= 2 (1e-5 sum_j |x_{i+j} f_j| + 1e-6), magnitudes from the unsharded input."""
    import torch.nn.functional as F
    x = R1.x[c.inp].float()
    x = x.reshape(-1, x.shape[-1])
    f = torch.tensor(list(c.f), dtype=torch.float32, device=x.device)
    mag = F.conv1d(x.abs()[:, None, :].double(), f.abs().double()[None, None, :]).reshape(-1).cpu()
    d = (a.double() - b.double()).abs()
    return bool((d <= 2 * (1e-5 * mag[:d.numel()] + 1e-6)).all())


def outputs(R):
    return {c.name: R.y[c.name].reshape(-1)[:max(c.n_out, 0)].clone() for c in R.cells}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="gloo")
    ap.add_argument("--workload", default="suite")
    a = ap.parse_args()
    world, rank, local = bench.dist_env()
    dev = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group(a.backend)
    orig = bench.cfg_cells
    bench.cfg_cells = lambda w, *extra: small(*orig(w, *extra))
    R = bench.Runner(a.workload, world, rank, dev)
    R.step_eager()
    torch.cuda.synchronize()
    mine = outputs(R)
    gathered = {}
    for name, t in mine.items():
        parts = [None] * world
        dist.all_gather_object(parts, t.cpu())
        gathered[name] = torch.cat(parts)
    ok = True
    if rank == 0:
        R1 = bench.Runner(a.workload, 1, 0, dev)
        R1.step_eager()
        torch.cuda.synchronize()
        ref = outputs(R1)
        cells = {c.name: c for c in R1.cells}
        for name in ref:
            c = cells[name]
            if tc_cell(c):
                same = close_within_bound(gathered[name], ref[name].cpu(), R1, c)
                how = "within bound"
            else:
                same = torch.equal(gathered[name], ref[name].cpu())
                how = "bitwise"
            print(f"{name:18s} sharded x{world} == unsharded ({how}): {same} ({ref[name].numel()} outputs)")
            ok &= same
        print("DIST_CHECK", "PASS" if ok else "FAIL")
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
