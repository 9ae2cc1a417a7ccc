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



# ------------------------------------------------- fp32 store, other configs --
def fp32_leg(args, wv, wmod, g, ents, V, block_range, torch, dev):
    """The fp32 parameter store beside the fp64 headline: throughput over the same
    blocks, and its max |fp32 - fp64| after one block's epoch from the same init."""
    cfg = wv.TrainConfig(vector_size=DIM, window_size=WINDOW, negative_samples=NEG, learning_rate=LR, epochs=1)

    def block(step):
        rb, re_ = block_range(step)
        corpus, lengths, width = wmod.random_walks_fixed(g, ents, DEPTH, WALKS, SEED, "pcg64",
                                                         work_begin=rb * WALKS, work_count=(re_ - rb) * WALKS)
        n_w = (re_ - rb) * WALKS
        return wmod._compact(torch, dev, corpus, lengths, n_w, width, wmod.RANDOM)

    sess = wv.SkipGramSession(V, cfg, SEED, precision="fp32")
    for i in range(args.warmup):
        sess.fit(block(i), 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pairs = 0
    e0.record()
    for i in range(args.fp32_steps):
        sess.fit(block(args.warmup + i), 1)
        pairs += sess.last_pairs
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    del sess
    # deviation: one block's epoch (all its batches) in both stores from the same init and streams
    wc = block(0)
    s64 = wv.SkipGramSession(V, cfg, SEED, precision="fp64")
    l64 = s64.fit(wc, 1)
    s32 = wv.SkipGramSession(V, cfg, SEED, precision="fp32")
    l32 = s32.fit(wc, 1)
    dev_in = float((s64.params.inp - s32.params.inp.double()).abs().max())
    dev_out = float((s64.params.out - s32.params.out.double()).abs().max())
    mag = float(s64.params.inp.abs().max())
    n_b = -(-s64.last_pairs // s64.last_batch_size)
    del s64, s32
    torch.cuda.empty_cache()
    return {"value": pairs / (ms / 1e3), "unit": "pairs/s", "dtype": "f32", "steps": args.fp32_steps,
            "ms_per_step": ms / args.fp32_steps,
            "max_abs_dev_vs_fp64": max(dev_in, dev_out), "max_abs_param_fp64": mag,
            "loss_fp64": l64[0], "loss_fp32": l32[0], "dev_batches": n_b,
            "note": f"fp32 store (FMA, approximate sqrt/divide) vs the fp64 store after the {n_b} batches of one "
                    f"block's epoch from the same init and device streams"}


def _ref_train_sample(ref, corpus_ref, V, d, B, n_batches, min_count=10):
    """Reference SGNS on the host: generate_pairs + n_batches batches of _train_single's loop body."""
    w2v = ref.w2v
    t0 = time.perf_counter()
    pairs, freq = w2v.generate_pairs(corpus_ref, WINDOW, min_count, V)
    t1 = time.perf_counter()
    cfg = w2v.TrainConfig(vector_size=d, window_size=WINDOW, negative_samples=NEG, learning_rate=LR,
                          min_count=min_count, epochs=1, batch_size=B)
    model = w2v.init_embeddings(V, d, SEED)
    opt_in, opt_out = w2v.RowAdam(model.input_matrix.shape, LR), w2v.RowAdam(model.output_matrix.shape, LR)
    data = w2v._BatchData(w2v.SKIPGRAM, pairs=pairs)
    cand = np.flatnonzero(freq >= min_count)
    rng = np.random.default_rng(np.random.SeedSequence([SEED, 1, 2, 0]))
    order = np.random.default_rng(np.random.SeedSequence([SEED, 1, 1])).permutation(len(pairs))
    t2 = time.perf_counter()
    for b in range(n_batches):
        index = order[b * B:(b + 1) * B]
        negs = w2v._draw_negatives(data, cfg, rng, cand, len(index), V)
        _, ir, ig, orr, og = data.batch_grads(model, index, negs)
        w2v.apply_sparse_update(model, ir, ig, orr, og, opt_in, opt_out)
    t3 = time.perf_counter()
    return {"pairs": len(pairs), "pairs_s": t1 - t0, "batch_s": (t3 - t2) / n_batches, "batches_timed": n_batches}


def _ref_e2e_estimate(walk_s, tr, epochs, B):
    """Reference seconds for the whole config from its measured pieces (walks, pair generation, per-batch time)."""
    n_batches = -(-tr["pairs"] // B) * epochs
    return walk_s + tr["pairs_s"] + n_batches * tr["batch_s"]


def cfg_sgns_e2e(args, wv, synth, torch, name, gen, depth, number, d, epochs, ref):
    """cfg1 / cfg4: device graph -> walks -> SGNS (fp64) -> vectors to the host, end to end."""
    res = None
    for rep in range(2):  # the first (one-epoch) pass pays one-time CUDA / graph-capture costs
        run_epochs = epochs if rep else 1
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        edges, V, ents, _ = gen()
        g = wv.build_graph(edges, V)
        roots = ents.cpu().numpy()
        corpus = wv.random_walks(g, roots, walk_depth=depth, walk_number=number, rng_seed=SEED)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        cfg = wv.TrainConfig(vector_size=d, window_size=WINDOW, negative_samples=NEG, learning_rate=LR,
                             epochs=run_epochs, min_count=10)
        model, losses = wv.train(corpus, V, cfg, SEED, precision=args.precision)
        vec = model.input_matrix  # float64 host matrix (the EmbeddingTable's vectors)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        pairs = model.n_pairs * epochs
        res = {"value": t2 - t0, "unit": "s", "higher_is_better": False, "dtype": "f64" if args.precision == "fp64"
               else "f32", "graph_and_walks_s": t1 - t0, "train_and_export_s": t2 - t1,
               "sgns_pairs_per_s": pairs / (t2 - t1), "pairs": pairs, "batch": model.batch_size,
               "walks": len(corpus), "triples": g.edge_count, "vocab": V, "losses": losses,
               "vectors": list(vec.shape)}
    es = 8 if args.precision == "fp64" else 4
    state_mb = 6 * res["vocab"] * d * es / 1e6
    res["roofline"] = {"bound": "l2" if state_mb < 100 else "hbm", "unit": "GB/s",
                       "achieved": res["sgns_pairs_per_s"] * 2 * (2 + NEG) * d * es / 1e9,
                       "note": f"SGNS pair-phase algorithmic bytes (SURVEY §8d, 2(2+k)d·s per pair) / train time; "
                               f"the parameter + Adam state is {state_mb:.0f} MB, "
                               + ("L2-resident (126 MB L2): not an HBM-roofline case" if state_mb < 100 else "")}
    if ref is not None and not args.no_cpu_baseline:
        off, tgt, prd = g.row_offsets, g.col_targets, g.col_predicates
        rgraph = ref_graph(ref, off, tgt, prd, V)
        # bounded: the first 1/frac of the root list (walks + generate_pairs scale linearly with it)
        frac = max(1, -(-len(roots) * number * (2 * depth + 1) // 20_000_000))
        t0 = time.perf_counter()
        rc = ref.walks.random_walks(rgraph, roots[: -(-len(roots) // frac)], walk_depth=depth, walk_number=number,
                                    rng_seed=SEED)
        walk_s = (time.perf_counter() - t0) * frac
        tr = _ref_train_sample(ref, rc, V, d, res["batch"], 3)
        tr["pairs"] = res["pairs"] // epochs
        tr["pairs_s"] *= frac
        est = _ref_e2e_estimate(walk_s, tr, epochs, res["batch"])
        res["cpu_baseline"] = {"value": est, "unit": "s", "cores": 1, "kind": "reference",
                               "sample": f"the reference's random_walks + generate_pairs over 1/{frac} of the "
                                         f"{name} root list, scaled x{frac} ({walk_s:.2f} s + {tr['pairs_s']:.2f} s), "
                                         f"and 3 timed "
                                         f"batches of _train_single's loop ({tr['batch_s']:.2f} s each), "
                                         f"value = walks + pairs + all {epochs} epoch(s) of batches at that rate "
                                         f"(estimate; the reference's own init and export excluded)",
                               "pairs_per_s": res["batch"] / tr["batch_s"]}
    return res


def cfg3_bfs(args, wv, torch, g, ents, ref):
    """cfg3: BFS walks depth 4, at most 250 per entity, over every entity of the cfg2 graph."""
    roots = ents.cpu().numpy()
    R = 1 << 18
    wv.bfs_walks(g, roots[:4096], 4, max_walks_per_root=250, with_table=False)  # warm-up
    walks = tokens = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for rb in range(0, len(roots), R):
        c, _ = wv.bfs_walks(g, roots[rb:rb + R], 4, max_walks_per_root=250, with_table=False)
        walks += len(c)
        tokens += c.total_tokens
        del c
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res = {"value": len(roots) / dt, "unit": "roots/s", "seconds": dt, "walks": walks, "tokens": tokens,
           "walks_per_s": walks / dt,
           "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": tokens * 4 / dt / 1e9,
                        "note": "output bytes only (compacted int32 tokens): a lower bound of the traffic; "
                                "the BFS frontier work (CSR reads, first-occurrence tables) is not counted"}}
    if ref is not None and not args.no_cpu_baseline:
        rgraph = ref_graph(ref, g.row_offsets, g.col_targets, g.col_predicates, g.vertex_count)
        sample = roots[:: len(roots) // 100][:100]
        t0 = time.perf_counter()
        ref.walks.bfs_walks(rgraph, sample, 4)
        rdt = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": len(sample) / rdt, "unit": "roots/s", "cores": 1, "kind": "reference",
                               "sample": "the reference's bfs_walks (uncapped: the cap is a prefix of its output "
                                         "and saves it no work) on 100 uniformly spaced roots of the cfg2 graph"}
    return res


def cfg5_walks(args, wv, wmod, synth, torch, ref, peak):
    """cfg5 walks on one GPU: BA(1e8, m=10), 200 predicates, depth 4 x 20 per entity (SGNS needs >= 4 GPUs)."""
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    edges, V, ents, _ = synth.device_synthetic_kg("barabasi", 100_000_000, m=10, predicates=200, seed=GEN_SEED)
    g = wv.build_graph(edges, V)
    del edges
    torch.cuda.synchronize()
    graph_s = time.perf_counter() - t0
    n_roots = int(ents.numel())
    R = 1 << 22
    stream = torch.cuda.current_stream()
    kern_ms, hops, walks = 0.0, 0, 0
    t1 = time.perf_counter()
    for rb in range(0, n_roots, R):
        re_ = min(rb + R, n_roots)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1_000_000)
        e0.record(stream)
        corpus, lengths, width = wmod.random_walks_fixed(g, ents, 4, 20, SEED, "pcg64", work_begin=rb * 20,
                                                         work_count=(re_ - rb) * 20)
        e1.record(stream)
        e1.synchronize()
        kern_ms += e0.elapsed_time(e1)
        nw = (re_ - rb) * 20
        hops += int((lengths[:nw].sum().item() - nw) // 2)
        walks += nw
        del corpus, lengths
    wall = time.perf_counter() - t1
    byt = 24 * hops + 8 * walks
    res = {"value": hops / (kern_ms / 1e3), "unit": "hops/s", "graph_build_s": graph_s, "walks": walks,
           "hops": hops, "walk_kernel_s": kern_ms / 1e3, "walks_wall_s": wall,
           "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
           "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": byt / (kern_ms * 1e-3) / 1e9, "peak": peak, "frac": byt / (kern_ms * 1e-3) / 1e9 / peak,
                        "note": "SURVEY §8d walk bytes (24 B/hop + 8 B/walk) / summed walk-kernel time "
                                "(CUDA events); CSR 8.8 GB: not L2-resident"},
           "note": "cfg5's SGNS state (6 x 1e8 x 200 values) needs the row-sharded mode over >= 4 GPUs"}
    # the same kernel against its measured DRAM traffic (ncu --set full of one cfg5 launch, committed):
    # random 8-byte reads cost 64-byte fetches, so the algorithmic 24 B/hop undercounts what moves
    cap = sorted((ROOT / "profiles" / "r02").glob("prof_random_walk_kernel_cfg5_*.raw.csv.gz"))
    if cap:
        import csv
        import gzip

        rows = list(csv.reader(gzip.open(cap[-1], "rt")))
        dd = dict(zip(rows[0], zip(rows[2], rows[1])))
        unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        byt_ncu = sum(float(dd[m][0].replace(",", "")) * unit.get(dd[m][1], 1)
                      for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        dur = float(dd["gpu__time_duration.sum"][0].replace(",", "")) * (
            1e-9 if dd["gpu__time_duration.sum"][1] == "nsecond" else 1e-6 if dd["gpu__time_duration.sum"][1] ==
            "usecond" else 1e-3)
        res["roofline"]["ncu_dram_gbs"] = byt_ncu / dur / 1e9
        res["roofline"]["frac_of_measured_traffic"] = byt_ncu / dur / 1e9 / peak
        res["roofline"]["ncu_source"] = str(cap[-1].relative_to(ROOT))
    if ref is not None and not args.no_cpu_baseline:
        off = g.row_offsets
        tgt, prd = g.col_targets, g.col_predicates
        rgraph = ref_graph(ref, off, tgt, prd, V)
        roots = ents[:2 * 8192 // 20 + 1].cpu().numpy()
        work = np.repeat(roots, 20)[:2 * 8192]
        t0 = time.perf_counter()
        tok, lens = ref.walks._walk_shard(rgraph, work[:8192], 4, np.random.default_rng(
            np.random.SeedSequence([SEED, 0, 0])))
        tok2, lens2 = ref.walks._walk_shard(rgraph, work[8192:], 4, np.random.default_rng(
            np.random.SeedSequence([SEED, 0, 1])))
        rdt = time.perf_counter() - t0
        rh = (len(tok) + len(tok2) - len(work)) // 2
        res["cpu_baseline"] = {"value": rh / rdt, "unit": "hops/s", "cores": 1, "kind": "reference",
                               "sample": "the reference's _walk_shard over the first two 8192-walk shards of the "
                                         "cfg5 work list on the cfg5 CSR (host copy)"}
        del off, tgt, prd, rgraph
    del g, ents
    torch.cuda.empty_cache()
    return res


def extra_configs(args, wv, wmod, synth, torch, g2, ents2, peak) -> dict:
    """BASELINE.json configs 1, 3, 4, 5 on the driver's clock (rank 0, one GPU)."""
    ref = load_reference() if not args.no_cpu_baseline else None
    want = [c for c in args.configs.split(",") if c]
    out = {}
    if "cfg1" in want:
        out["cfg1"] = cfg_sgns_e2e(args, wv, synth, torch, "cfg1", lambda: synth.device_synthetic_kg(
            "barabasi", 10_000, m=5, predicates=20, seed=GEN_SEED), 4, 10, 100, 1, ref)
        out["cfg1"]["workload"] = ("cfg1: BA(10k, m=5), 20 predicates; walks depth 4 x 10; SGNS d100 w5 k5, 1 epoch; "
                                   "end to end (graph, walks, training, float64 vectors on the host)")
    if "cfg3" in want:
        out["cfg3"] = cfg3_bfs(args, wv, torch, g2, ents2, ref)
        out["cfg3"]["workload"] = "cfg3: BFS walks depth 4, <= 250 per entity, all 1M entities of the cfg2 graph"
    if "cfg4" in want:
        out["cfg4"] = cfg_sgns_e2e(args, wv, synth, torch, "cfg4", lambda: synth.device_synthetic_kg(
            "erdos_renyi", 15_000, p=0.001378, predicates=237, seed=GEN_SEED), 16, 500, 100, args.cfg4_epochs, ref)
        out["cfg4"]["workload"] = (f"cfg4: ER(15k, p=0.001378), 237 predicates (~310k triples); walks depth 16 x 500; "
                                   f"SGNS d100 w5 k5, {args.cfg4_epochs} epochs; end to end")
    if "cfg5" in want:
        out["cfg5_walks"] = cfg5_walks(args, wv, wmod, synth, torch, ref, peak)
        out["cfg5_walks"]["workload"] = "cfg5: BA(1e8, m=10) -> ~1e9 triples, 200 predicates; walks depth 4 x 20"
    return out

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
    # the update phase's required DRAM bytes: RowAdam read-modify-write of p, m, v for each unique
    # row (this design keeps no gradient accumulator, so §8d's g read + zeroing is not moved) + one
    # read of the batch's U/G rows the contributions come from
    owner_bytes = 6 * DIM * es * U + 2 * DIM * es * B
    owner_bytes_8d = (2 + NEG) * DIM * es * B + 8 * DIM * es * U  # scatter half + 8 d s per row
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
    frac_8d = owner_bytes_8d / (kern["sgns_owner_adam(flat light rows + heavy pieces)"]["ms"] * 1e-3) / 1e9 / peak
    batch_ms = ph.get("batch", float("nan"))
    batch_ms_timed = (ms / args.steps - walk_ms) / per
    # ncu DRAM traffic per launch of the owner phase's kernels (same batch geometry), newest capture
    traffic, traffic_src, batch_traffic = None, None, None
    # newest capture: tags grow in length through a round (r02y < r02ac < r02ai_full), then by name
    tfs = sorted((ROOT / "profiles").glob("traffic_*.json"), key=lambda p_: (p_.stem[:11], len(p_.stem), p_.stem))
    if tfs:
        t_ = json.loads(tfs[-1].read_text())
        owner_parts = [k_ for k_ in t_ if k_.startswith("sgns_owner") or k_.startswith("heavy_piece")]
        if owner_parts:
            traffic = sum(t_[k_]["dram_bytes"] for k_ in owner_parts)
            traffic_src = (f"{tfs[-1].relative_to(ROOT)}: ncu dram__bytes_read+write per launch of "
                           f"{' + '.join(sorted(owner_parts))}")
        batch_traffic = sum(v_["dram_bytes"] for k_, v_ in t_.items() if k_ != "random_walk_kernel")
        if "random_walk_kernel" in t_:  # CSR lookups: ncu DRAM bytes and L2 hit rate of the walk kernel
            kern["walk"]["ncu_dram_bytes"] = t_["random_walk_kernel"]["dram_bytes"]
            kern["walk"]["ncu_l2_hit_rate_pct"] = t_["random_walk_kernel"].get("l2_hit_rate_pct")
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": kern[dom]["gbs"], "peak": peak, "unit": "GB/s",
        "frac": kern[dom]["frac"], "frac_survey_8d_bytes": frac_8d, "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
        "algorithmic_bytes_per_launch": kern[dom]["bytes"], "avg_launch_ms": kern[dom]["ms"],
        "kernels": kern,
        "sgns_batch": {"bytes": batch_bytes, "ms": batch_ms, "gbs": batch_bytes / (batch_ms * 1e-3) / 1e9,
                       "frac": batch_bytes / (batch_ms * 1e-3) / 1e9 / peak, "batch_pairs": B,
                       "unique_rows_per_batch": U,
                       "dram_traffic": batch_traffic,
                       "frac_of_measured_traffic": (batch_traffic / (batch_ms * 1e-3) / 1e9 / peak
                                                    if batch_traffic else None),
                       # the batch period on the timed region's own clock (graph-replayed, no phase
                       # events): (step time - walk kernel) / batches per step
                       "timed": {"ms": batch_ms_timed, "gbs": batch_bytes / (batch_ms_timed * 1e-3) / 1e9,
                                 "frac": batch_bytes / (batch_ms_timed * 1e-3) / 1e9 / peak,
                                 "frac_of_measured_traffic": (batch_traffic / (batch_ms_timed * 1e-3) / 1e9 / peak
                                                              if batch_traffic else None)}},
        # the same kernel against its measured DRAM bytes (the algorithmic figure counts a row
        # gathered by the pair phase and then updated by the Adam phase twice)
        "frac_of_measured_traffic": (traffic / (kern[dom]["ms"] * 1e-3) / 1e9 / peak if traffic else None),
        "note": "achieved = required bytes per launch / mean CUDA-event launch time; update phase: 6 d s per unique "
                "row (p, m, v read + write) + 2 B d s (the U/G rows read once); gather: (2+k) d s per pair; "
                "frac_survey_8d_bytes uses SURVEY §8d's figure (8 d s per row + (2+k) d s per pair), which counts "
                "a gradient accumulator this design does not have. walk: events "
                "around the walk kernel in the timed steps; SGNS phases: CUDA events around the phases of every 16th "
                "batch of one extra step right after the timed region, run eagerly (event nodes inside CUDA graphs "
                "would distort the graph-replayed timing). traffic: see profiles/",
        "timed_unique_rows_per_batch": rows_updated / n_batches, "profiled_step_wall_s": prof_wall,
    }
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        off, tgt, prd = host_csr(g)
        cpu = cpu_baseline_leg(args, off, tgt, prd, ents.cpu().numpy(), V)
    fp32 = None
    if args.precision == "fp64" and args.fp32_steps > 0 and world == 1:
        fp32 = fp32_leg(args, wv, wmod, g, ents, V, block_range, torch, dev)
    configs = None
    if rank == 0 and world == 1 and args.configs not in ("", "none"):
        from paper_2508_01073_b200 import synth

        configs = extra_configs(args, wv, wmod, synth, torch, g, ents, peak)
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
        "fp32_store": fp32,
        "configs": configs,
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
    ap.add_argument("--fp32-steps", type=int, default=3, help="timed steps of the fp32-store leg (0: skip)")
    ap.add_argument("--configs", default="cfg1,cfg3,cfg4,cfg5",
                    help="other BASELINE configs timed after the headline (rank 0, N=1; '' to skip)")
    ap.add_argument("--cfg4-epochs", type=int, default=5)
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
