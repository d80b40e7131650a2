"""Multi-GPU plumbing for the sliding-window hot path (one process per GPU).

Two partitionings:

* batch sharding -- independent rows / images are split evenly over ranks;
  no collective on the data path.
* sequence sharding -- one long sequence is split into contiguous shards.
  Rank r owns x[g0, g0+S) and the outputs of the windows that START in its
  shard.  The windows that start in the last w-1 positions need the first
  h = w-1 elements of rank r+1's shard (the "halo"; "each
  range is extended by w-1 elements of overlap").  The halo is the method's
  only inter-GPU exchange: one NCCL send/recv pair per rank per step
  (``halo_start``), overlapped with the interior kernels, then a short tail
  launch computes the last w-1 outputs once the halo has landed.

Everything here is index arithmetic and torch.distributed calls; the window
arithmetic runs in the CUDA kernels (or, in the CPU gloo tests, in whatever
``compute`` callable the test passes).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist


def even_split(total: int, world: int, rank: int) -> tuple[int, int]:
    """[start, end) of rank's contiguous share of `total` units (first ranks get +1)."""
    base, rem = divmod(total, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


@dataclass
class SeqShard:
    """Geometry of one rank's contiguous shard of a sequence of length n_total
    for windows of up to w_max elements (halo h = w_max - 1)."""
    n_total: int
    world: int
    rank: int
    w_max: int

    def __post_init__(self):
        # the halo of rank r is the first w_max-1 elements of rank r+1 ALONE: every
        # shard must hold at least that many, or windows would need rank r+2's data
        if self.world < 1 or not 0 <= self.rank < self.world or self.w_max < 1 or self.n_total < 1:
            raise ValueError(f"bad shard geometry {self}")
        if self.world > 1 and self.n_total // self.world < self.w_max - 1:
            raise ValueError(f"sequence of {self.n_total} over {self.world} ranks: shards of "
                             f"{self.n_total // self.world} < w_max-1 = {self.w_max - 1}; shard fewer ranks")

    @property
    def start(self) -> int:
        return even_split(self.n_total, self.world, self.rank)[0]

    @property
    def size(self) -> int:
        a, b = even_split(self.n_total, self.world, self.rank)
        return b - a

    @property
    def halo(self) -> int:
        return self.w_max - 1 if self.rank < self.world - 1 else 0

    @property
    def is_last(self) -> bool:
        return self.rank == self.world - 1

    def n_outputs(self, w: int) -> int:
        """Windows of length w that start inside this shard (global count sums to n_total-w+1)."""
        last_start = self.n_total - w  # last valid global window start
        a, b = self.start, min(self.start + self.size, last_start + 1)
        return max(0, b - a)

    def interior_outputs(self, w: int) -> int:
        """Windows fully inside the local shard (no halo needed)."""
        return max(0, min(self.size - w + 1, self.n_outputs(w)))


def halo_start(xbuf: torch.Tensor, shard: SeqShard, group=None):
    """Post the halo exchange for a local buffer laid out as
    [shard.size own elements | shard.halo received elements]: send our first
    h elements to rank-1, receive rank+1's first h elements into the tail.
    Returns the list of work handles (wait on them before the tail launch)."""
    h_send = shard.w_max - 1 if shard.rank > 0 else 0
    ops = []
    if shard.rank > 0 and h_send > 0:
        ops.append(dist.P2POp(dist.isend, xbuf[:h_send], shard.rank - 1, group))
    if not shard.is_last and shard.halo > 0:
        ops.append(dist.P2POp(dist.irecv, xbuf[shard.size:shard.size + shard.halo], shard.rank + 1, group))
    if not ops:
        return []
    if xbuf.is_cuda and dist.get_backend(group) == "gloo":
        return _halo_gloo_staged(xbuf, shard, h_send, group)
    return dist.batch_isend_irecv(ops)


def _halo_gloo_staged(xbuf: torch.Tensor, shard: SeqShard, h_send: int, group=None):
    """Blocking host-staged exchange for CUDA buffers under the gloo backend
    (used to exercise the multi-rank path with several ranks on one device;
    the production path is NCCL).  Sends go first on even ranks to avoid a
    cycle of blocking sends."""
    def send():
        if shard.rank > 0 and h_send > 0:
            dist.send(xbuf[:h_send].cpu(), shard.rank - 1, group)

    def recv():
        if not shard.is_last and shard.halo > 0:
            t = torch.empty(shard.halo, dtype=xbuf.dtype)
            dist.recv(t, shard.rank + 1, group)
            xbuf[shard.size:shard.size + shard.halo].copy_(t)
    if shard.rank % 2 == 0:
        send()
        recv()
    else:
        recv()
        send()
    return []


def run_interior(xbuf: torch.Tensor, shard: SeqShard, w: int, compute, y: torch.Tensor) -> None:
    """Outputs whose windows lie inside the local shard (needs no halo).
    compute(x_view, y_view) evaluates the op on a contiguous input view,
    writing len(x_view) - w + 1 outputs."""
    n_int = shard.interior_outputs(w)
    if n_int > 0:
        compute(xbuf[: n_int + w - 1], y[:n_int])


def run_tail(xbuf: torch.Tensor, shard: SeqShard, w: int, compute, y: torch.Tensor) -> None:
    """Outputs whose windows reach into the halo (call after the exchange completed)."""
    n_out, n_int = shard.n_outputs(w), shard.interior_outputs(w)
    if n_out > n_int:
        compute(xbuf[n_int: n_out + w - 1], y[n_int:n_out])


def wait_all(works) -> None:
    for wk in works:
        wk.wait()


def sliding_sharded(xbuf: torch.Tensor, shard: SeqShard, ops, group=None):
    """Run several window ops [(w, compute, y), ...] over one sequence shard with
    a single halo exchange: post the exchange, run every interior (overlapping
    the transfer), wait, then run every tail."""
    works = halo_start(xbuf, shard, group)
    for w, compute, y in ops:
        run_interior(xbuf, shard, w, compute, y)
    wait_all(works)
    for w, compute, y in ops:
        run_tail(xbuf, shard, w, compute, y)
