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


def workload(roots_per_step: int) -> dict:
    return {
        "workload": "cfg2: BA(1M entities, m=10) -> 9,999,945 triples, 200 predicates; random walks depth 8 x 100/entity "
                    "(reference PCG64 streams, bit-exact corpus); SGNS d200 w5 k5 lr0.01, reference 1 GiB batch rule "
                    f"(23,933 pairs); step = {roots_per_step}-entity root block per GPU, 1 SGNS epoch over its pairs",
        "graph": {"model": "barabasi", "entities": N_ENT, "m": M_BA, "predicates": N_PRED, "gen_seed": GEN_SEED},
        "walks": {"depth": DEPTH, "walks_per_entity": WALKS, "rng": "pcg64"},
        "sgns": {"dim": DIM, "window": WINDOW, "negatives": NEG, "lr": LR, "batch_rule": "1 GiB", "precision": "fp32"},
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


# ------------------------------------------------------------ CPU oracle ----
def cpu_sample(off, tgt, prd, roots_np, V, shards, batches: int, state=None):
    """Oracle (numpy restatement of the reference) on a bounded sample.

    Walks: the given 8192-walk shards of the cfg2 corpus (walks.py:117-204);
    SGNS: ``batches`` reference batches (23,933 pairs) drawn from those walks'
    pairs, continuing ``state`` (init + RowAdam).  Returns timings + counts.
    """
    from oracle import w2v as ow2v
    from oracle import walks as owalks

    if state is None:
        inp, out = ow2v.init(V, DIM, SEED)
        state = {"inp": inp, "out": out, "ai": ow2v.RowAdam(inp.shape, LR), "ao": ow2v.RowAdam(out.shape, LR),
                 "rng": np.random.default_rng(np.random.SeedSequence([SEED, 1, 2, 0]))}
    t0 = time.perf_counter()
    pieces, lens = [], []
    for s in shards:  # walks.py:168-173: shard s = work[8192 s : 8192 (s+1)] on SeedSequence([seed, 0, s])
        w = np.arange(s * owalks.SHARD, min((s + 1) * owalks.SHARD, len(roots_np) * WALKS))
        rows = owalks.walk_rows(off, tgt, prd, roots_np[w // WALKS], DEPTH, owalks._shard_rng(SEED, s, "pcg64"))
        keep = rows != -1
        pieces.append(rows[keep])
        lens.append(keep.sum(axis=1))
    tok = np.concatenate(pieces)
    offs = np.concatenate([[0], np.cumsum(np.concatenate(lens))]).astype(np.int64)
    t1 = time.perf_counter()
    pr = ow2v.pairs(tok, offs, WINDOW)
    t2 = time.perf_counter()
    B = ow2v.batch_size(len(pr), DIM, NEG, BUDGET)
    order = np.random.default_rng(np.random.SeedSequence([SEED, 1, 1])).permutation(len(pr))
    t3 = time.perf_counter()
    trained = 0
    for b in range(batches):
        idx = order[b * B:(b + 1) * B]
        if len(idx) == 0:
            break
        negs = state["rng"].integers(0, V, size=len(idx) * NEG).reshape(len(idx), NEG)
        loss, ir, ig, orr, og = ow2v.sgns_step(state["inp"], state["out"], pr[idx, 0], pr[idx, 1], negs)
        ur, ug = ow2v.coalesce(ir, ig)
        state["ai"].update(state["inp"], ur, ug)
        ur, ug = ow2v.coalesce(orr, og)
        state["ao"].update(state["out"], ur, ug)
        trained += len(idx)
    t4 = time.perf_counter()
    hops = (len(tok) - (len(offs) - 1)) // 2
    res = {"walk_s": t1 - t0, "pairs_s": t2 - t1, "shuffle_s": t3 - t2, "sgns_s": t4 - t3, "pairs_generated": len(pr),
           "pairs_trained": trained, "hops": hops, "batch": B}
    # pipeline seconds per trained pair: walk + pair generation scaled to the trained share, + SGNS
    frac = trained / max(len(pr), 1)
    res["pipeline_s"] = (res["walk_s"] + res["pairs_s"] + res["shuffle_s"]) * frac + res["sgns_s"]
    res["pairs_per_s"] = trained / res["pipeline_s"]
    res["hops_per_s"] = hops / res["walk_s"]
    return res, state


def host_csr(g):
    return g.row_offsets, g.col_targets, g.col_predicates


# ------------------------------------------------------------- reference ----
_REF = {}  # inherited by forked reference workers (CSR, roots, initial state)


def _ref_worker(job):
    """One reference worker: its own replica (init + RowAdam + negative stream, as a
    _train_multi worker, w2v.py:579-746) over its own walk shards."""
    wid, n_workers, warmup, steps, batches = job
    from oracle import w2v as ow2v

    inp, out = _REF["init"]  # forked: the replica's pages are copied on first write
    state = {"inp": inp, "out": out, "ai": ow2v.RowAdam(inp.shape, LR), "ao": ow2v.RowAdam(out.shape, LR),
             "rng": np.random.default_rng(np.random.SeedSequence([SEED, 1, 2, wid]))}
    rows = []
    for i in range(warmup + steps):
        shard = (i * n_workers + wid) % _REF["n_shards"]
        res, state = cpu_sample(_REF["off"], _REF["tgt"], _REF["prd"], _REF["roots"], _REF["V"], [shard], batches, state)
        if i >= warmup:
            rows.append((res["pipeline_s"], res["pairs_trained"], res["hops"], res["walk_s"]))
    return rows


def run_reference(args, rank, world):
    """--impl reference: the oracle port of the reference on all host cores (rank 0 only).

    One forked worker per core, each a replica of the reference's multi-worker
    trainer (own Adam state and negative stream, w2v.py:579-746) walking its own
    8192-walk shards (walks.py:168-173) and training reference batches from them;
    the replica merge every 64 batches (_merge_bundles) is not timed.  value =
    pairs trained by all workers / the slowest worker's time.
    """
    if rank != 0:
        return
    import multiprocessing as mp

    import torch

    from oracle import w2v as ow2v

    g, V, ents = make_graph()  # synthetic input only; the timed path below is pure numpy
    off, tgt, prd = host_csr(g)
    roots_np = ents.cpu().numpy()
    del g
    torch.cuda.empty_cache()
    # one replica per core; each holds its own parameters + Adam state (~10.5 GB at cfg2 once its
    # touched pages are copied), so the worker count is also capped by 60% of the available RAM
    try:
        import psutil

        mem_cap = max(1, int(0.6 * psutil.virtual_memory().available / 10.5e9))
    except ImportError:
        mem_cap = 8
    cores = int(args.ref_cores) if args.ref_cores else min(len(os.sched_getaffinity(0)), mem_cap)
    _REF.update(off=off, tgt=tgt, prd=prd, roots=roots_np, V=V, n_shards=-(-len(roots_np) * WALKS // 8192),
                init=ow2v.init(V, DIM, SEED))
    jobs = [(w, cores, args.warmup, args.steps, args.ref_batches) for w in range(cores)]
    with mp.get_context("fork").Pool(cores) as pool:
        results = pool.map(_ref_worker, jobs)
    per_worker_s = [sum(r[0] for r in rows) for rows in results]
    trained = sum(r[1] for rows in results for r in rows)
    hops = sum(r[2] for rows in results for r in rows)
    walk_s = max(sum(r[3] for r in rows) for rows in results)
    tot = max(per_worker_s)
    value = trained / tot
    sample = (f"{cores} forked workers (one per host core), each per step: one 8192-walk shard of the cfg2 corpus "
              f"(oracle walks) + {args.ref_batches} SGNS batches of 23,933 pairs from its pairs (oracle fp64 numpy, "
              f"own replica as in _train_multi; merge not timed); walk/pair time scaled to the trained share; "
              f"value = all pairs / slowest worker")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": workload(args.roots),
        "walk_hops_per_s": hops / walk_s if walk_s else None,
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    sess = wv.SkipGramSession(V, cfg, SEED, precision="fp32")
    if world > 1:
        sess.attach_exchange(RankExchange())
    stream = torch.cuda.current_stream()
    setup_s = time.perf_counter() - t_setup

    def block_range(step):
        b = (step * world + rank) % n_blocks
        return b * R, min((b + 1) * R, n_roots)

    stats = {"walk_ms": [], "hops": 0, "walks": 0, "pairs": 0, "batches": 0, "sgns_ms": [], "phase_ms": {}}

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
        sess.fit(wc, 1, profile=profile)
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
    es = 4
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
        res, _ = cpu_sample(off, tgt, prd, ents.cpu().numpy(), V, [0], args.ref_batches)
        cpu = {"value": res["pairs_per_s"], "unit": "pairs/s", "cores": 1, "kind": "port",
               "sample": f"oracle (numpy restatement, fp64): shard 0 of the cfg2 corpus (8192 walks, {res['hops']} hops, "
                         f"{res['pairs_generated']} pairs) + {args.ref_batches} SGNS batches of {res['batch']} pairs; "
                         f"walk+pair time scaled to the trained share",
               "walk_hops_per_s": res["hops_per_s"], "sgns_pairs_per_s": res["pairs_trained"] / res["sgns_s"]}
    walk_hops = sum_over_ranks(float(stats["hops"]), world, dev)
    walk_ms_tot = max_over_ranks(float(sum(stats["walk_ms"])), world, dev)
    sgns_ms_tot = max_over_ranks(float(sum(stats["sgns_ms"])), world, dev)
    line = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic (device-generated BA graph, seed 7)",
        "config": workload(R),
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
        "last_loss": None,
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
    ap.add_argument("--ref-batches", type=int, default=2, help="SGNS batches per CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-cores", type=int, default=0, help="reference-arm workers (default: all host cores)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank, world, local = dist_setup()
    if world != args.gpus and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
