"""Row-sharded SGNS / CBOW training across ranks.

When the parameter + RowAdam state (6 x V x d floats: 480 GB at 100M x 200
fp32) cannot be replicated on every GPU, rank r of N owns the rows
``row % N == r`` of both matrices and their optimizer state.  Each global
batch (the reference's batch rule over the whole corpus, w2v.py:437-497):

1. every rank decodes the whole batch (Feistel/Philox streams or the
   replayed numpy streams) and groups the contribution slots of its own rows
   (``wv_shard_decode_group``);
2. the rank's share of pairs requests its rows from their owners
   (``wv_shard_requests``, all-to-all, ``wv_shard_serve``, all-to-all back,
   ``wv_shard_place``);
3. ``wv_shard_gather`` computes the loss terms, coefficients and U/G rows of
   the rank's pairs, normalised by the global batch (w2v.py:276-299);
4. U, G and the coefficients are all-gathered in global pair order;
5. ``wv_shard_update`` sums each owned row's contributions in the
   reference's slot order and applies RowAdam (w2v.py:364-434).

Every step is deterministic and the owner-side slot lists are those of the
single-GPU batch, so the result equals single-GPU training with the same
global batch (``tests/test_shard_gpu.py`` checks bit-equality).  The corpus
index is replicated (every rank decodes every pair).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from .w2v import TrainingDiverged, _Params, _Trainer, CBOW


class ShardExchange:
    """all-to-all / all-gather over a torch.distributed group (NCCL on device tensors;
    gloo via host staging, for multi-process tests on one GPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def all_to_all(self, send, send_counts, recv_counts, row_elems: int = 1):
        """Variable-size all-to-all of ``send`` (grouped by destination), counts in rows."""
        import torch

        out_n = int(sum(recv_counts))
        tail = send.shape[1:] if send.dim() > 1 else ()
        if self.nccl:
            recv = torch.empty((out_n, *tail), dtype=send.dtype, device=send.device)
            self.dist.all_to_all_single(recv, send[: int(sum(send_counts))].contiguous(), list(map(int, recv_counts)),
                                        list(map(int, send_counts)), group=self.group)
            return recv
        src = send[: int(sum(send_counts))].cpu().contiguous()
        recv = torch.empty((out_n, *tail), dtype=send.dtype)
        self.dist.all_to_all_single(recv, src, list(map(int, recv_counts)), list(map(int, send_counts)),
                                    group=self.group)
        return recv.to(send.device)

    def exchange_counts(self, counts):
        import torch

        c = counts.to(torch.int64)
        if not self.nccl:
            c = c.cpu()
        out = torch.empty_like(c)
        self.dist.all_to_all_single(out, c, group=self.group)
        return out.cpu().tolist()

    def all_gather(self, out, local):
        """out [world * n, ...] <- every rank's local [n, ...] in rank order."""
        if self.nccl:
            self.dist.all_gather_into_tensor(out, local.contiguous(), group=self.group)
            return
        parts = [p for p in out.cpu().chunk(self.world)]
        self.dist.all_gather(parts, local.cpu().contiguous(), group=self.group)
        out.copy_(self.dist_cat(parts).to(out.device))

    @staticmethod
    def dist_cat(parts):
        import torch

        return torch.cat(parts)

    def sum_(self, t):
        if self.nccl:
            self.dist.all_reduce(t, group=self.group)
            return t
        h = t.cpu()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h.to(t.device))
        return t


def train_row_sharded(corpus, vocab_size: int, config, rng_seed: int, exchange: ShardExchange | None = None, *,
                      precision: str = "fp32", pairs: str = "device"):
    """Row-sharded ``train``: returns (local _Params of this rank, per-epoch losses).

    The rank's store holds global rows ``l * N + rank`` at local row ``l``.
    """
    if not config.use_sparse:
        raise NotImplementedError("row-sharded training implements sparse RowAdam")
    ex = exchange or ShardExchange()
    N, r = ex.world, ex.rank
    tr = _Trainer(corpus, vocab_size, config, rng_seed, lambda *a, **k: None, precision, pairs, 1)
    torch = tr.torch
    dev = tr.dev
    V = tr.V
    p = _Params(torch, dev, V, config.vector_size, tr.seed, precision, True, config.learning_rate, shard=(N, r))
    d = p.d
    B, Npairs = tr.batch_size, tr.N
    R = (2 * tr.cbow_window + 1 + tr.k) if tr.cbow_window else (2 + tr.k)
    ws = torch.empty(_lib.query("wv_sgns_batch_workspace_bytes", p.V, d, tr.k, B, p.precision, tr.cbow_window),
                     dtype=torch.uint8, device=dev)
    st = _lib.stream_ptr()
    _lib.call("wv_sgns_workspace_init", _lib.ptr(ws), ws.numel(), p.V, d, tr.k, B, p.precision, tr.cbow_window, st)
    bl_max = -(-B // N)
    dt = p.dtype
    keys = torch.empty(max(bl_max * R, 1), dtype=torch.int64, device=dev)
    items = torch.empty(max(bl_max * R, 1), dtype=torch.int32, device=dev)
    ident = torch.empty(max(bl_max * R, 1), dtype=torch.int32, device=dev)
    cursor = torch.empty(N, dtype=torch.int32, device=dev)
    counts = torch.empty(N, dtype=torch.int64, device=dev)
    itemrows = torch.empty((max(bl_max * R, 1), d), dtype=dt, device=dev)
    U_l = torch.zeros((bl_max, d), dtype=dt, device=dev)
    G_l = torch.zeros((bl_max, d), dtype=dt, device=dev)
    c_l = torch.zeros((bl_max, tr.k + 1), dtype=dt, device=dev)
    U_g = torch.empty((N * bl_max, d), dtype=dt, device=dev)
    G_g = torch.empty((N * bl_max, d), dtype=dt, device=dev)
    c_g = torch.empty((N * bl_max, tr.k + 1), dtype=dt, device=dev)
    bs = tr.batch_struct
    model = C.byref(p.struct)
    if pairs == "numpy":
        shuffle_rng = np.random.default_rng(np.random.SeedSequence([tr.seed, 1, 1]))
        neg_rng = np.random.default_rng(np.random.SeedSequence([tr.seed, 1, 2, 0]))
    # skip-gram: every split size of a batch's all-to-alls is computed on the device one batch
    # ahead (wv_shard_count_requests) and copied to pinned host memory asynchronously, so no
    # batch waits on a device -> host round trip; CBOW reads its counts synchronously
    lookahead = tr.cbow_window == 0 and not os.environ.get("WV_SHARD_SYNC_COUNTS")
    check = bool(os.environ.get("WV_SHARD_CHECK"))
    if lookahead:
        scratch = torch.empty(max(B * R, 1), dtype=torch.int32, device=dev)
        cnt_dev = torch.empty(N * N, dtype=torch.int64, device=dev)
        cnt_host = [torch.empty(N * N, dtype=torch.int64, pin_memory=torch.cuda.is_available()) for _ in range(2)]
        cnt_evt = [torch.cuda.Event() for _ in range(2)]

    def issue_counts(epoch, lo, slot):
        _lib.call("wv_shard_count_requests", C.byref(bs), epoch, lo, min(B, Npairs - lo), N, _lib.ptr(scratch),
                  _lib.ptr(cnt_dev), st)
        cnt_host[slot].copy_(cnt_dev, non_blocking=True)
        cnt_evt[slot].record()

    losses = []
    for epoch in range(config.epochs):
        if pairs == "numpy":
            order = shuffle_rng.permutation(Npairs)
            tr._upload_epoch_streams(order, [(lo, min(B, Npairs - lo), neg_rng) for lo in range(0, Npairs, B)])
        _lib.call("wv_sgns_epoch_begin", _lib.ptr(p.state), epoch, 0, st)
        starts = list(range(0, Npairs, B))
        if lookahead:
            issue_counts(epoch, 0, 0)
        for bi, lo in enumerate(starts):
            rows = min(B, Npairs - lo)
            bs.batch_rows = rows
            _lib.call("wv_shard_decode_group", model, C.byref(bs), _lib.ptr(ws), ws.numel(), V, N, r, st)
            if lookahead and bi + 1 < len(starts):
                issue_counts(epoch, starts[bi + 1], (bi + 1) % 2)
            bl = -(-rows // N)
            pb = min(r * bl, rows)
            pc = min(rows, pb + bl) - pb
            _lib.call("wv_shard_requests", model, C.byref(bs), _lib.ptr(ws), ws.numel(), V, N, r, pb * R, pc * R,
                      _lib.ptr(cursor), _lib.ptr(keys), _lib.ptr(items), _lib.ptr(ident), _lib.ptr(counts), st)
            if lookahead:
                cnt_evt[bi % 2].synchronize()  # recorded a batch ago: already complete
                M = cnt_host[bi % 2].view(N, N).tolist()
                send_counts = M[r]
                recv_counts = [M[s_][r] for s_ in range(N)]
                if check:
                    assert send_counts == counts.cpu().tolist(), (send_counts, counts.cpu().tolist())
                    assert recv_counts == ex.exchange_counts(counts), "request counts differ across ranks"
            else:
                send_counts = counts.cpu().tolist()
                recv_counts = ex.exchange_counts(counts)
            req = ex.all_to_all(keys, send_counts, recv_counts)
            served = torch.empty((max(len(req), 1), d), dtype=dt, device=dev)
            _lib.call("wv_shard_serve", model, _lib.ptr(req), len(req), V, N, _lib.ptr(served), st)
            back = ex.all_to_all(served, recv_counts, send_counts)
            _lib.call("wv_shard_place", _lib.ptr(back), _lib.ptr(items), int(sum(send_counts)), d, p.precision,
                      _lib.ptr(itemrows), st)
            _lib.call("wv_shard_gather", model, C.byref(bs), _lib.ptr(ws), ws.numel(), V, N, r, _lib.ptr(itemrows),
                      _lib.ptr(ident), pc, _lib.ptr(U_l), _lib.ptr(G_l), _lib.ptr(c_l), st)
            ex.all_gather(U_g[: N * bl], U_l[:bl])
            ex.all_gather(G_g[: N * bl], G_l[:bl])
            ex.all_gather(c_g[: N * bl], c_l[:bl])
            # the global batch's pair b sits at row b of the gathered arrays
            _lib.call("wv_shard_update", model, C.byref(bs), _lib.ptr(ws), ws.numel(), V, N, r, _lib.ptr(U_g),
                      _lib.ptr(G_g), _lib.ptr(c_g), st)
        s = p.read_state()
        agg = torch.tensor([s.epoch_loss_sum, float(s.epoch_count),
                            float(s.diverged_batch if s.diverged_batch >= 0 else 1 << 50)], dtype=torch.float64,
                           device=dev)
        div = torch.tensor([agg[2].item()], dtype=torch.float64, device=dev)
        ex.sum_(agg[:2])
        if ex.nccl:
            ex.dist.all_reduce(div, op=ex.dist.ReduceOp.MIN, group=ex.group)
        else:
            h = div.cpu()
            ex.dist.all_reduce(h, op=ex.dist.ReduceOp.MIN, group=ex.group)
            div = h
        if div.item() < (1 << 50):
            raise TrainingDiverged(epoch, int(div.item()))
        losses.append(float(agg[0] / agg[1]))
    return p, losses
