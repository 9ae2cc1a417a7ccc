"""Multi-GPU plumbing: one process per GPU, torch.distributed over NCCL.

* Walks shard with no communication: rank r computes the contiguous slice of
  the root-major work list repeat(roots, walk_number) (walks.py:166) covering
  its entity range; every walker derives its shard, row and stream position
  from its global work index, so the union over ranks is byte-identical to
  a single-process corpus.
* SGNS is data-parallel with the reference's local-replica contract
  (w2v.py:662-746): rank r trains the r-th contiguous span of each epoch's
  permutation with its own Adam state; every sync round the per-row deltas
  and touch counts are summed with one all-reduce and each rank applies
  shared += delta_sum / count (_merge_bundles, w2v.py:642-659).
"""

from __future__ import annotations

import os


def rank_slice(total: int, rank: int, world: int, granule: int = 1) -> tuple[int, int]:
    """Contiguous [begin, end) share of ``total`` units, boundaries on ``granule`` multiples."""
    units = -(-total // granule)
    per = -(-units // world)
    b = min(rank * per, units) * granule
    e = min((rank + 1) * per, units) * granule
    return min(b, total), min(e, total)


def walk_work_range(n_roots: int, walk_number: int, rank: int, world: int) -> tuple[int, int]:
    """Walker range of a rank: whole root groups (duplicate_free needs them, walks.py:188-194)."""
    rb, re_ = rank_slice(n_roots, rank, world)
    return rb * walk_number, re_ * walk_number


class RankExchange:
    """The collective step of multi-GPU SGNS (sums across ranks)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world_size = dist.get_world_size(group)

    def all_reduce_(self, *tensors):
        for t in tensors:
            self.dist.all_reduce(t, group=self.group)

    def reduce_epoch(self, loss_sum: float, count: int, diverged):
        import torch

        dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
        div_e, div_b = (diverged if diverged is not None else (-1, -1))
        buf = torch.tensor([loss_sum, float(count)], dtype=torch.float64, device=dev)
        self.dist.all_reduce(buf, group=self.group)
        # first diverged (epoch, batch) over ranks; -1 means none
        big = 1 << 62
        d = torch.tensor([div_e if div_e >= 0 else big, div_b if div_b >= 0 else big], dtype=torch.int64,
                         device=dev)
        self.dist.all_reduce(d, op=self.dist.ReduceOp.MIN, group=self.group)
        div = None if int(d[0]) == big else (int(d[0]), int(d[1]))
        return float(buf[0]), int(buf[1]), div

    def or_flags_(self, *flags):
        for f in flags:
            self.dist.all_reduce(f, op=self.dist.ReduceOp.MAX, group=self.group)


def env_rank() -> tuple[int, int, int]:
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
