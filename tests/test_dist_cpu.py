"""World-size-2 (and 3) gloo tests of the multi-GPU plumbing on CPU:
sequence sharding with the (w-1)-element halo exchanged by send/recv
(paper_2305_16513_b200/dist.py) and batch sharding.  The window arithmetic in
these CPU tests is the oracle's (the GPU path plugs ss_* kernels into the same
`compute` slot); what is tested here is shard geometry and the halo exchange:
the concatenated per-rank outputs must equal the unsharded result exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2305_16513_b200.dist import SeqShard, even_split, halo_start, run_interior, run_tail, \
    sliding_sharded, wait_all


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, ws, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = SeqShard(n_total, world, rank, max(ws))
        xbuf = torch.zeros(sh.size + sh.halo, dtype=torch.int32)
        xbuf[:sh.size] = torch.from_numpy(synth.randint(2, sh.size, -1000, 1000, start=sh.start))
        outs = {}
        ops = []
        for w in ws:
            y = torch.full((max(sh.n_outputs(w), 1),), -99, dtype=torch.int64)
            outs[w] = y

            def compute(xv, yv, w=w):
                yv.copy_(torch.from_numpy(oracle.pool_sum(xv.numpy(), w)))
            ops.append((w, compute, y))
        sliding_sharded(xbuf, sh, ops)
        # second form: explicit phases, max op
        works = halo_start(xbuf, sh)
        ymax = torch.full((max(sh.n_outputs(ws[-1]), 1),), -99, dtype=torch.int32)

        def cmax(xv, yv):
            yv.copy_(torch.from_numpy(oracle.pool_max(xv.numpy(), ws[-1])))
        run_interior(xbuf, sh, ws[-1], cmax, ymax)
        wait_all(works)
        run_tail(xbuf, sh, ws[-1], cmax, ymax)
        q.put((rank, {w: outs[w][:sh.n_outputs(w)].numpy() for w in ws},
               ymax[:sh.n_outputs(ws[-1])].numpy(), sh.start, sh.size))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_total,ws", [(2, 10007, (3, 16, 64, 256)), (3, 5000, (2, 31)),
                                              (2, 300, (1, 64))])
def test_sequence_shard_halo_gloo(world, n_total, ws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_total, ws, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = synth.randint(2, n_total, -1000, 1000)
    for w in ws:
        got = np.concatenate([r[1][w] for r in res])
        np.testing.assert_array_equal(got, oracle.pool_sum(x, w))
    np.testing.assert_array_equal(np.concatenate([r[2] for r in res]), oracle.pool_max(x, ws[-1]))
    # shards tile the sequence
    assert res[0][3] == 0 and sum(r[4] for r in res) == n_total


def test_even_split_partitions():
    for total in (1, 7, 64, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            parts = [even_split(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_seq_shard_output_counts():
    for n, world, w in ((1 << 26, 8, 256), (1 << 32, 8, 64), (1000, 3, 7)):
        shards = [SeqShard(n, world, r, w) for r in range(world)]
        assert sum(s.n_outputs(w) for s in shards) == n - w + 1
        for s in shards[:-1]:
            assert s.n_outputs(w) == s.size and s.halo == w - 1
        assert shards[-1].halo == 0


def test_seq_shard_rejects_shards_shorter_than_halo():
    # rank r's halo must come from rank r+1 alone: every shard needs >= w_max-1 elements
    SeqShard(126, 2, 0, 64)  # 63 per shard = w_max-1: fine
    with pytest.raises(ValueError):
        SeqShard(125, 2, 0, 64)
    with pytest.raises(ValueError):
        SeqShard(100, 8, 3, 31)
    SeqShard(10, 1, 0, 64 + 1)  # one rank: no halo, the window check is the kernel's
