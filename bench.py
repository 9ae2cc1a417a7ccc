#!/usr/bin/env python
"""RDF2vec hot-path benchmark (walks -> SGNS) on B200, BASELINE.json config 2.

Workload: synthetic power-law KG, Barabasi-Albert
n=1,000,000 m=10 with 200 predicates (9,999,945 triples), generated on the
device (csrc/synth.cu); uniform random walks depth 8 x 100 walks per entity
on the reference's own PCG64 streams (walks.py:144-204, byte-identical
corpus); SGNS d=200, window 5, 5 negatives, lr 0.01, batch by the
reference's 1 GiB rule (23,933 pairs, w2v.py:437-497), fp32 parameter store.

A step = one RDF2vec pass over a block of ``--roots`` entities (default 8192)
per GPU: the walk kernel over the block's 100 x roots walkers (the exact
slice of the full cfg2 corpus), compaction, pair index, then one SGNS epoch
over the block's ~1.03e8 pairs continuing the same resident parameters
(SkipGramSession).  122 blocks = one full cfg2 epoch.

value = SGNS pairs trained per second through the whole step (walk time
included), summed over ranks.  e2e = the same through the public API with a
host root block (pinned H2D) and the block's entity vectors read back (D2H).
cpu_baseline / --impl reference = the numpy oracle (oracle/, a restatement
of the reference's algorithm) on the host cores, on a bounded sample.

Multi-GPU (torchrun): weak scaling; rank r takes blocks r, r+N, ...; the
walks need no communication, SGNS replicas are averaged once per step with
one NCCL all-reduce of per-row deltas (the reference's _merge_bundles).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "walk hops/s + SGNS pairs/s at 1/2/4/8 B200; end-to-end RDF2vec sec vs CPU ref"
N_ENT, M_BA, N_PRED, GEN_SEED = 1_000_000, 10, 200, 7
DEPTH, WALKS, DIM, WINDOW, NEG, LR, SEED = 8, 100, 200, 5, 5, 0.01, 42
BUDGET = 1 << 30


def workload(roots_per_step: int, precision: str = "fp64") -> dict:
    return {
        "workload": "cfg2: BA(1M entities, m=10) -> 9,999,945 triples, 200 predicates; random walks depth 8 x 100/entity "
                    "(reference PCG64 streams, bit-exact corpus); SGNS d200 w5 k5 lr0.01, reference 1 GiB batch rule "
                    f"(23,933 pairs); step = {roots_per_step}-entity root block per GPU, 1 SGNS epoch over its pairs",
        "graph": {"model": "barabasi", "entities": N_ENT, "m": M_BA, "predicates": N_PRED, "gen_seed": GEN_SEED},
        "walks": {"depth": DEPTH, "walks_per_entity": WALKS, "rng": "pcg64"},
        "sgns": {"dim": DIM, "window": WINDOW, "negatives": NEG, "lr": LR, "batch_rule": "1 GiB", "precision": precision},
        "roots_per_step": roots_per_step,
        "l2": "no flush: per-step working set (SGNS state 4.8 GB, corpus ~55 MB) exceeds the 126 MB L2; "
              "the 88 MB CSR is L2-resident by design",
    }


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if os.environ.get("BENCH_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=5)

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ distributed --
def dist_setup():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world > 1:
        import torch.distributed as dist

        # BENCH_DIST_BACKEND=gloo exercises the multi-rank path on a single GPU
        # (ranks share device local % device_count); NCCL is the real path
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        import torch

        if torch.cuda.is_available():
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return rank, world, local


def max_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int, device) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


# ------------------------------------------------------------- the graph ----
def make_graph():
    """cfg2 graph on the device: (Graph, vocab_size, entity tokens (device int64))."""
    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import synth

    edges, V, ents, _ = synth.device_synthetic_kg("barabasi", N_ENT, m=M_BA, predicates=N_PRED, seed=GEN_SEED)
    g = wv.build_graph(edges, V)
    del edges
    return g, V, ents


# ------------------------------------------------------- CPU reference ----
REF_DIR = ROOT / "baseline" / "_ref"  # pip-installed, unmodified reference (git-ignored, travels to the box)


def load_reference():
    """The reference's walkvec package from baseline/_ref, or None if it was not installed."""
    if not (REF_DIR / "walkvec" / "__init__.py").exists():
        return None
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import walkvec  # noqa: F401
    import walkvec.w2v
    import walkvec.walks

    return walkvec


class RefPipeline:
    """The reference's own RDF2vec hot path, one replica (a _train_multi worker, w2v.py:579-746).

    A step trains one block of the cfg2 work list end to end with the
    reference's functions: ``walks._walk_shard`` over the block's walks
    (walks.py:117-141, the block's shard stream SeedSequence([seed, 0, s])),
    ``w2v.generate_pairs`` (:161-191), a fresh ``permutation`` of the block's
    pairs, then every batch of 23,933 pairs (the 1 GiB rule at d 200) through
    ``_draw_negatives`` -> ``_BatchData.batch_grads`` (= sgns_batch_grads) ->
    ``apply_sparse_update`` (RowAdam) -- the loop body of _train_single
    (:547-576).  Parameters and RowAdam state persist across steps.  With
    the oracle port (``ref=None``) the same steps run oracle/ instead.
    """

    def __init__(self, ref, graph, roots, V, wid):
        self.ref, self.graph, self.roots, self.V = ref, graph, roots, V
        self.B = 23_933
        if ref is not None:
            w2v = ref.w2v
            self.cfg = w2v.TrainConfig(vector_size=DIM, window_size=WINDOW, negative_samples=NEG, learning_rate=LR,
                                       min_count=0, epochs=1, batch_size=self.B)
            self.model = w2v.init_embeddings(V, DIM, SEED)
            self.model.touched_input = np.zeros(V, dtype=bool)
            self.model.touched_output = np.zeros(V, dtype=bool)
            self.opt_in = w2v.RowAdam(self.model.input_matrix.shape, LR)
            self.opt_out = w2v.RowAdam(self.model.output_matrix.shape, LR)
        else:
            from oracle import w2v as ow2v

            self.inp, self.out = ow2v.init(V, DIM, SEED)
            self.opt_in, self.opt_out = ow2v.RowAdam(self.inp.shape, LR), ow2v.RowAdam(self.out.shape, LR)
        self.candidates = np.arange(V)  # min_count 10 keeps every token at cfg2
        self.shuffle_rng = np.random.default_rng(np.random.SeedSequence([SEED, 1, 1, wid]))
        self.neg_rng = np.random.default_rng(np.random.SeedSequence([SEED, 1, 2, wid]))
        self.loss = None

    def step(self, walk_begin: int, n_walks: int) -> dict:
        t0 = time.perf_counter()
        work = self.roots[(walk_begin + np.arange(n_walks)) // WALKS]
        shard_rng = np.random.default_rng(np.random.SeedSequence([SEED, 0, walk_begin // 8192]))
        if self.ref is not None:
            tok, lens = self.ref.walks._walk_shard(self.graph, work, DEPTH, shard_rng)
        else:
            from oracle import walks as owalks

            rows = owalks.walk_rows(*self.graph, work, DEPTH, shard_rng)
            keep = rows != -1
            tok, lens = rows[keep], keep.sum(axis=1)
        offs = np.zeros(n_walks + 1, dtype=np.int64)
        np.cumsum(lens, out=offs[1:])
        t1 = time.perf_counter()
        if self.ref is not None:
            w2v = self.ref.w2v
            pairs, _ = w2v.generate_pairs(w2v._Corpus(tok, offs), WINDOW, 0, self.V)
            data = w2v._BatchData(w2v.SKIPGRAM, pairs=pairs)
        else:
            from oracle import w2v as ow2v

            pairs = ow2v.pairs(tok, offs, WINDOW)
        n = len(pairs)
        order = self.shuffle_rng.permutation(n)
        loss_sum = 0.0
        for lo in range(0, n, self.B):
            index = order[lo:lo + self.B]
            if self.ref is not None:
                negs = w2v._draw_negatives(data, self.cfg, self.neg_rng, self.candidates, len(index), self.V)
                loss, ir, ig, orr, og = data.batch_grads(self.model, index, negs)
                uin, uout = w2v.apply_sparse_update(self.model, ir, ig, orr, og, self.opt_in, self.opt_out)
                self.model.touched_input[uin] = True
                self.model.touched_output[uout] = True
            else:
                from oracle import w2v as ow2v

                negs = self.candidates[self.neg_rng.integers(0, len(self.candidates), size=len(index) * NEG)]
                sel = pairs[index]
                loss, ir, ig, orr, og = ow2v.sgns_step(self.inp, self.out, sel[:, 0], sel[:, 1],
                                                      negs.reshape(len(index), NEG))
                self.opt_in.update(self.inp, *ow2v.coalesce(ir, ig))
                self.opt_out.update(self.out, *ow2v.coalesce(orr, og))
            loss_sum += loss * len(index)
        t2 = time.perf_counter()
        self.loss = loss_sum / n
        hops = (len(tok) - n_walks) // 2
        return {"s": t2 - t0, "walk_s": t1 - t0, "pairs": n, "hops": hops, "batches": -(-n // self.B)}


def ref_graph(ref, off, tgt, prd, V):
    """The reference's Graph (graph.py:31-41) over given CSR arrays, or the oracle's tuple."""
    if ref is None:
        return off, tgt, prd
    return ref.graph.Graph(row_offsets=off, col_targets=tgt, col_predicates=prd, vertex_count=V)


def host_csr(g):
    return g.row_offsets, g.col_targets, g.col_predicates


def _ref_kind(ref) -> str:
    return "reference" if ref is not None else "port"


_REF = {}  # inherited by forked reference workers (graph, roots)


def _ref_worker(job):
    """One reference worker (own replica, own blocks); returns per-step timings."""
    wid, n_workers, warmup, steps, walks_per_step = job
    ref = load_reference() if _REF["use_ref"] else None
    pipe = RefPipeline(ref, _REF["graph"], _REF["roots"], _REF["V"], wid)
    total_walks = len(_REF["roots"]) * WALKS
    rows = []
    for i in range(warmup + steps):
        blk = (i * n_workers + wid) * walks_per_step % total_walks
        r = pipe.step(blk, min(walks_per_step, total_walks - blk))
        if i >= warmup:
            rows.append(r)
    return rows, pipe.loss


def ref_sample_text(cores, walks_per_step):
    return (f"{cores} forked worker(s), one per host core, each a replica of the reference trainer (own parameters, "
            f"RowAdam, negative stream, as a _train_multi worker) over its own blocks of the cfg2 work list; "
            f"a step = {walks_per_step} walks of depth 8 (the reference's _walk_shard), generate_pairs, a permutation "
            f"and every 23,933-pair batch over the block's pairs (sgns_batch_grads + apply_sparse_update, float64); "
            f"value = pairs trained by all workers / the slowest worker's summed step time; the replica merge "
            f"(every 64 batches in reproducible mode) is not reached within the run")


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation on all host cores (rank 0 only)."""
    if rank != 0:
        return
    import multiprocessing as mp

    from oracle import synth as osy

    ref = load_reference()
    # cfg2 input without the product library: the numpy restatement of the device generator
    # (bit-identical graph, tests/test_gpu_synth.py), CSR by the reference's own build_graph
    t0 = time.perf_counter()
    edges, V, ents, _ = osy.barabasi_kg(N_ENT, M_BA, N_PRED, GEN_SEED)
    if ref is not None:
        graph = ref.graph.build_graph(edges, V)
    else:
        from oracle import walks as owalks

        graph = owalks.csr(edges, V)
    del edges
    setup_s = time.perf_counter() - t0
    try:
        import psutil

        mem_cap = max(1, int(0.6 * psutil.virtual_memory().available / 10.5e9))
    except ImportError:
        mem_cap = 8
    cores = int(args.ref_cores) if args.ref_cores else min(len(os.sched_getaffinity(0)), mem_cap)
    _REF.update(graph=graph, roots=ents, V=V, use_ref=ref is not None)
    jobs = [(w, cores, args.warmup, args.steps, args.ref_walks) for w in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        results = pool.map(_ref_worker, jobs)
    per_worker_s = [sum(r["s"] for r in rows) for rows, _ in results]
    pairs = sum(r["pairs"] for rows, _ in results for r in rows)
    hops = sum(r["hops"] for rows, _ in results for r in rows)
    walk_s = max(sum(r["walk_s"] for r in rows) for rows, _ in results)
    tot = max(per_worker_s)
    value = pairs / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (oracle/synth.py restatement of the device BA graph)",
        "config": workload(args.roots, "fp64"),
        "walk_hops_per_s": hops / walk_s if walk_s else None,
        "last_loss": results[0][1], "setup_s": setup_s,
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": _ref_kind(ref),
                         "sample": ref_sample_text(cores, args.ref_walks)},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(args, off, tgt, prd, roots, V) -> dict:
    """Our arm's cpu_baseline: the same reference pipeline on one core, a bounded sample."""
    ref = load_reference()
    pipe = RefPipeline(ref, ref_graph(ref, off, tgt, prd, V), roots, V, 0)
    pipe.step(0, args.ref_walks)  # warm-up (page faults of the state)
    rows = [pipe.step((i + 1) * args.ref_walks, args.ref_walks) for i in range(args.cpu_steps)]
    tot = sum(r["s"] for r in rows)
    pairs = sum(r["pairs"] for r in rows)
    return {"value": pairs / tot, "unit": "pairs/s", "cores": 1, "kind": _ref_kind(ref),
            "sample": ref_sample_text(1, args.ref_walks).replace("forked worker(s), one per host core", "process")
            + f"; {args.cpu_steps} timed steps after 1 warm-up",
            "walk_hops_per_s": sum(r["hops"] for r in rows) / sum(r["walk_s"] for r in rows),
            "last_loss": pipe.loss}


# ------------------------------------------------------------------- ours ---
def run_ours(args, rank, world, local):
    import torch

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import _lib, walks as wmod
    from paper_2508_01073_b200.dist import RankExchange

    _lib.require_cuda()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    t_setup = time.perf_counter()
    g, V, ents = make_graph()
    n_roots = int(ents.numel())
    R = int(args.roots)
    n_blocks = -(-n_roots // R)
    cfg = wv.TrainConfig(vector_size=DIM, window_size=WINDOW, negative_samples=NEG, learning_rate=LR, epochs=1)
    sess = wv.SkipGramSession(V, cfg, SEED, precision=args.precision)
    if world > 1:
        sess.attach_exchange(RankExchange())
    stream = torch.cuda.current_stream()
    setup_s = time.perf_counter() - t_setup

    def block_range(step):
        b = (step * world + rank) % n_blocks
        return b * R, min((b + 1) * R, n_roots)

    stats = {"last_loss": None, "walk_ms": [], "hops": 0, "walks": 0, "pairs": 0, "batches": 0, "sgns_ms": [], "phase_ms": {}}

    def one_step(step, timed, profile=False):
        rb, re_ = block_range(step)
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        # keep the device busy (~0.5 ms) while the host prepares the walk launch,
        # so e0 -> e1 brackets the walk kernel and not host-side launch overhead
        torch.cuda._sleep(1_000_000)
        e0.record(stream)
        corpus, lengths, width = wmod.random_walks_fixed(g, ents, DEPTH, WALKS, SEED, "pcg64",
                                                         work_begin=rb * WALKS, work_count=(re_ - rb) * WALKS)
        e1.record(stream)
        n_w = (re_ - rb) * WALKS
        wc = wmod._compact(torch, dev, corpus, lengths, n_w, width, wmod.RANDOM)
        losses = sess.fit(wc, 1, profile=profile)
        stats["last_loss"] = losses[-1]
        sess.sync()
        e2.record(stream)
        if timed:
            e2.synchronize()
            if os.environ.get("BENCH_DEBUG"):
                print(f"step {step}: walk {e0.elapsed_time(e1):.1f} ms, rest {e1.elapsed_time(e2):.1f} ms, "
                      f"pairs {sess.last_pairs}", file=sys.stderr)
            stats["walk_ms"].append(e0.elapsed_time(e1))
            stats["sgns_ms"].append(e1.elapsed_time(e2))
            stats["hops"] += (wc.total_tokens - n_w) // 2
            stats["walks"] += n_w
            stats["pairs"] += sess.last_pairs
            stats["batches"] += -(-sess.last_pairs // sess.last_batch_size)
        if profile:
            e2.synchronize()
            from paper_2508_01073_b200.w2v import PHASE_NAMES

            for sample in sess.last_replica.profile_samples:
                for name, v in zip(PHASE_NAMES, sample):
                    stats["phase_ms"].setdefault(name, []).append(v)
            sess.last_replica.profile_samples.clear()
        return sess.last_pairs

    for i in range(args.warmup):
        one_step(i, False)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    rows0 = sess.rows_updated()
    launches0 = _lib.launch_count()
    pairs = 0
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        t_start.record(stream)
        for i in range(args.steps):
            pairs += one_step(args.warmup + i, True)
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    rows_updated = sess.rows_updated() - rows0
    # kernel breakdown: one extra step after the timed region with device timestamps inside
    # the CUDA graphs (kept out of the timed steps so they carry no event-record nodes)
    rows_p0 = sess.rows_updated()
    prof_t0 = time.perf_counter()
    one_step(args.warmup + args.steps, False, profile=True)
    prof_batches = -(-sess.last_pairs // sess.last_batch_size)
    rows_per_batch_prof = (sess.rows_updated() - rows_p0) / max(prof_batches, 1)
    prof_wall = time.perf_counter() - prof_t0
    ms = t_start.elapsed_time(t_end)
    ms_max = max_over_ranks(ms, world, dev)
    total_pairs = sum_over_ranks(float(pairs), world, dev)
    value = total_pairs / (ms_max / 1e3)

    # ---- e2e: public API, host root block in pinned memory, entity vectors back to the host
    e2e_ms, h2d, d2h, e2e_pairs = 0.0, 0, 0, 0
    if args.e2e_steps > 0:
        roots_host = ents.cpu().numpy()
        pinned = torch.empty(R, dtype=torch.int64).pin_memory()
        out_host = torch.empty((R, DIM), dtype=torch.float32).pin_memory()
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.e2e_steps):
            rb, re_ = block_range(args.warmup + args.steps + i)
            n = re_ - rb
            pinned[:n].copy_(torch.from_numpy(roots_host[rb:re_]))
            block = pinned[:n].numpy()
            wc = wv.random_walks(g, block, walk_depth=DEPTH, walk_number=WALKS, rng_seed=SEED)
            sess.fit(wc, 1)
            sess.sync()
            idx = torch.from_numpy(block).to(dev, non_blocking=True)
            out_host[:n].copy_(sess.params.inp.view(V, DIM).index_select(0, idx), non_blocking=True)
            torch.cuda.current_stream().synchronize()
            h2d += n * 8
            d2h += n * DIM * 4 + 8  # entity rows + the epoch loss
            e2e_pairs += sess.last_pairs
        e2e_ms = (time.perf_counter() - t0) * 1e3
    e2e_ms = max_over_ranks(e2e_ms, world, dev)
    e2e_pairs = sum_over_ranks(float(e2e_pairs), world, dev)

    # ---- kernel roofline (events on the launching stream, inside the timed steps)
    peaks_path = ROOT / "MEASURED_PEAKS.json"
    if peaks_path.exists():
        peak, peak_src = float(json.loads(peaks_path.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    else:
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    es = 8 if args.precision == "fp64" else 4
    B = sess.last_batch_size
    n_batches = max(stats["batches"], 1)
    U = rows_per_batch_prof  # unique (row, matrix) updates per batch (profiled step)
    walk_ms = float(np.mean(stats["walk_ms"]))
    walk_bytes = 24 * stats["hops"] / args.steps + 8 * stats["walks"] / args.steps
    ph = {k_: float(np.mean(v_)) for k_, v_ in stats["phase_ms"].items()}
    pair_bytes = (2 + NEG) * DIM * es * B  # gathers of the 2+k rows (SURVEY §8d pair phase, first half)
    owner_bytes = (2 + NEG) * DIM * es * B + 8 * DIM * es * U  # scatter half + RowAdam rows
    per = n_batches / args.steps
    kern = {
        "walk": {"ms": walk_ms, "bytes": walk_bytes, "per_step": 1},
        "sgns_decode": {"ms": ph.get("decode", float("nan")), "bytes": None, "per_step": per},
        "sgns_gather": {"ms": ph.get("gather", float("nan")), "bytes": pair_bytes, "per_step": per},
        "sgns_grouping(side stream, overlaps gather)": {"ms": ph.get("group", float("nan")), "bytes": None,
                                                         "per_step": per},
        "sgns_owner_adam(flat light rows + heavy pieces)": {"ms": ph.get("owner", float("nan")), "bytes": owner_bytes,
                                                            "per_step": per},
    }
    for k_, v_ in kern.items():
        v_["share_of_step"] = v_["ms"] * v_["per_step"] / (ms / args.steps)
        v_["gbs"] = v_["bytes"] / (v_["ms"] * 1e-3) / 1e9 if v_["bytes"] else None
        v_["frac"] = v_["gbs"] / peak if v_["gbs"] else None
    dom = max((k_ for k_ in kern if kern[k_]["bytes"]), key=lambda k_: kern[k_]["share_of_step"])
    batch_bytes = pair_bytes + owner_bytes
    batch_ms = ph.get("batch", float("nan"))
    # ncu DRAM traffic per launch of the owner phase's kernels (same batch geometry), newest capture
    traffic, traffic_src, batch_traffic = None, None, None
    tfs = sorted((ROOT / "profiles").glob("traffic_*.json"))
    if tfs:
        t_ = json.loads(tfs[-1].read_text())
        owner_parts = [k_ for k_ in t_ if k_.startswith("sgns_owner") or k_.startswith("heavy_piece")]
        if owner_parts:
            traffic = sum(t_[k_]["dram_bytes"] for k_ in owner_parts)
            traffic_src = (f"{tfs[-1].relative_to(ROOT)}: ncu --set full dram__bytes_read+write of "
                           f"{' + '.join(sorted(owner_parts))}")
        batch_traffic = sum(v_["dram_bytes"] for k_, v_ in t_.items() if k_ != "random_walk_kernel")
        if "random_walk_kernel" in t_:  # CSR lookups: ncu DRAM bytes and L2 hit rate of the walk kernel
            kern["walk"]["ncu_dram_bytes"] = t_["random_walk_kernel"]["dram_bytes"]
            kern["walk"]["ncu_l2_hit_rate_pct"] = t_["random_walk_kernel"].get("l2_hit_rate_pct")
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak, "unit": "GB/s",
        "frac": kern[dom]["frac"], "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
        "algorithmic_bytes_per_launch": kern[dom]["bytes"], "avg_launch_ms": kern[dom]["ms"],
        "kernels": kern,
        "sgns_batch": {"bytes": batch_bytes, "ms": batch_ms, "gbs": batch_bytes / (batch_ms * 1e-3) / 1e9,
                       "frac": batch_bytes / (batch_ms * 1e-3) / 1e9 / peak, "batch_pairs": B,
                       "unique_rows_per_batch": U,
                       "dram_traffic": batch_traffic,
                       "frac_of_measured_traffic": (batch_traffic / (batch_ms * 1e-3) / 1e9 / peak
                                                    if batch_traffic else None)},
        # the same kernel against its measured DRAM bytes (the algorithmic figure counts a row
        # gathered by the pair phase and then updated by the Adam phase twice)
        "frac_of_measured_traffic": (traffic / (kern[dom]["ms"] * 1e-3) / 1e9 / peak if traffic else None),
        "note": "achieved = SURVEY §8d algorithmic bytes per launch / mean CUDA-event launch time. walk: events "
                "around the walk kernel in the timed steps; SGNS phases: CUDA events around the phases of every 16th "
                "batch of one extra step right after the timed region, run eagerly (event nodes inside CUDA graphs "
                "would distort the graph-replayed timing). traffic: see profiles/",
        "timed_unique_rows_per_batch": rows_updated / n_batches, "profiled_step_wall_s": prof_wall,
    }
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        off, tgt, prd = host_csr(g)
        cpu = cpu_baseline_leg(args, off, tgt, prd, ents.cpu().numpy(), V)
    walk_hops = sum_over_ranks(float(stats["hops"]), world, dev)
    walk_ms_tot = max_over_ranks(float(sum(stats["walk_ms"])), world, dev)
    sgns_ms_tot = max_over_ranks(float(sum(stats["sgns_ms"])), world, dev)
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64" if args.precision == "fp64" else "f32",
        "data": "synthetic (device-generated BA graph, seed 7)",
        "config": workload(R, args.precision),
        "walk_hops_per_s": walk_hops / (walk_ms_tot / 1e3),
        "sgns_pairs_per_s": total_pairs / (sgns_ms_tot / 1e3),
        "e2e_cfg2_epoch_s_extrapolated": (ms_max / args.steps) * n_blocks / world / 1e3,
        "e2e": {"value": e2e_pairs / (e2e_ms / 1e3) if e2e_ms else None, "unit": "pairs/s",
                "h2d_bytes_per_step": h2d // max(args.e2e_steps, 1), "d2h_bytes_per_step": d2h // max(args.e2e_steps, 1),
                "steps": args.e2e_steps, "api": "random_walks(graph, host roots) -> SkipGramSession.fit -> vectors .cpu()"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "setup_s": setup_s,
        "last_loss": stats["last_loss"],  # epoch-mean SGNS loss of the last block (rank 0)
    }
    if rank == 0:
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--roots", type=int, default=8192, help="entities per GPU per step")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-walks", type=int, default=384,
                    help="walks per reference step (~48k pairs: two full 23,933-pair batches + a remainder)")
    ap.add_argument("--cpu-steps", type=int, default=3, help="timed steps of our arm's one-core cpu_baseline leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-cores", type=int, default=0, help="reference-arm workers (default: all host cores)")
    ap.add_argument("--precision", choices=["fp64", "fp32"], default="fp64",
                    help="parameter store (the reference computes in float64, w2v.py:127-130, 379-380)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        # CPU only: rank 0 runs the reference on the host cores, other ranks exit without work
        run_reference(args, int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)))
        return
    rank, world, local = dist_setup()
    if world != args.gpus and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    try:
        run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
