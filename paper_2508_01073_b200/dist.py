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

    @property
    def _staged(self) -> bool:
        # gloo (multi-process tests on one GPU / CPU): collectives on host copies
        return self.dist.get_backend(self.group) != "nccl"

    def _all_reduce(self, t, op=None):
        op = op if op is not None else self.dist.ReduceOp.SUM
        if self._staged and t.is_cuda:
            h = t.cpu()
            self.dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, op=op, group=self.group)
        return t

    def _all_gather(self, out, local):
        if self._staged and local.is_cuda:
            parts = list(out.cpu().chunk(self.world_size))
            self.dist.all_gather(parts, local.cpu().contiguous(), group=self.group)
            import torch

            out.copy_(torch.cat(parts))
        else:
            self.dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)

    def all_reduce_(self, *tensors):
        for t in tensors:
            self._all_reduce(t)

    def merge_deltas_(self, deltas, counts, dim: int, sparse_fraction: float = 0.5):
        """Sum per-row deltas ([V*d] each) and touch counts ([V] each) across ranks, in place.

        A rank's delta is non-zero only on the rows it touched this round
        (count > 0 before the reduction).  Per matrix: when every rank touched
        few rows (world * max touched < sparse_fraction * V) only those rows
        travel -- their ids and rows are all-gathered and summed in rank order
        (the same order on every rank, so all replicas stay identical);
        otherwise one dense all-reduce.  Returns the path per matrix, e.g.
        "sparse,dense".
        """
        import torch

        V = int(counts[0].numel())
        touched = [torch.nonzero(c > 0).flatten() for c in counts]
        nmax = torch.tensor([int(t.numel()) for t in touched], dtype=torch.int64, device=counts[0].device)
        self._all_reduce(nmax, self.dist.ReduceOp.MAX)
        nmax = nmax.tolist()
        for c in counts:
            self._all_reduce(c)
        W = self.world_size
        modes = []
        for dlt, rows, n in zip(deltas, touched, nmax):
            if W * n >= sparse_fraction * V:
                self._all_reduce(dlt)
                modes.append("dense")
                continue
            dv = dlt.view(V, dim)
            ids = torch.full((n,), -1, dtype=torch.int64, device=dlt.device)
            ids[: rows.numel()] = rows
            vals = torch.zeros((n, dim), dtype=dlt.dtype, device=dlt.device)
            vals[: rows.numel()] = dv[rows]
            all_ids = torch.empty((W * n,), dtype=torch.int64, device=dlt.device)
            all_vals = torch.empty((W * n, dim), dtype=dlt.dtype, device=dlt.device)
            self._all_gather(all_ids, ids)
            self._all_gather(all_vals, vals)
            dv.zero_()
            for r in range(W):  # rank order: a row's ids are unique within one rank
                ir = all_ids[r * n:(r + 1) * n]
                ok = ir >= 0
                dv.index_put_((ir[ok],), all_vals[r * n:(r + 1) * n][ok], accumulate=True)
            modes.append("sparse")
        return ",".join(modes)

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


def bfs_walks_rank(graph, start_vertices=None, walk_depth: int = 5, *, max_walks_per_root: int | None = None,
                   rank: int | None = None, world: int | None = None, group=None):
    """BFS walks of this rank's contiguous root range with GLOBAL walk ids (BFS row).

    Roots are independent (walks.py:261-310: each root's walks depend on that
    root only), so rank r walks ``rank_slice(len(roots), r, world)`` with no
    communication; the one exchange is an all-gather of the ranks' walk counts,
    whose exclusive prefix is this rank's first global walk id.  The
    PathTable's walk ids are shifted by it, so concatenating the ranks'
    outputs in rank order gives exactly the single-process
    ``bfs_walks(graph, roots, walk_depth)``.  Returns (corpus, table, first_walk_id).
    """
    import torch
    import torch.distributed as dist

    from .walks import _resolve_roots, as_device_graph, bfs_walks

    if rank is None or world is None:
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    g = as_device_graph(graph)
    roots = _resolve_roots(g, start_vertices)
    rb, re_ = rank_slice(len(roots), rank, world)
    if re_ > rb:
        corpus, table = bfs_walks(g, roots[rb:re_], walk_depth, max_walks_per_root=max_walks_per_root)
        n = len(corpus)
    else:
        corpus, table, n = None, None, 0
    counts = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    if world > 1:
        dist.all_gather(counts, torch.tensor([n], dtype=torch.int64), group=group)
    else:
        counts[0][0] = n
    base = int(sum(int(c.item()) for c in counts[:rank]))
    if table is not None:
        table.walk_ids = table.walk_ids + base
    if corpus is not None:
        corpus.first_walk_id = base
    return corpus, table, base
