"""north_star target end to end on ONE B200: synthetic KG of 10M entities / 100M triples
(BA(1e7, m=10), 200 predicates, generated and encoded on the device), random walks
depth 4 x 20 per entity (cfg5 walk parameters), one SGNS epoch at d=200 (window 5,
5 negatives, the reference's 1 GiB batch rule), streamed over root blocks through
SkipGramSession (parameters resident: 10M x 200 x 6 fp64 = 96 GB; fp32 halves it).

    python profiles/northstar_e2e.py [n_entities] [roots_per_block, 0 = all] [fp64|fp32]


Prints one JSON line: seconds for graph build, walks, SGNS, and the totals.
"""
import json
import sys
import time

sys.path.insert(0, ".")


def main():
    import torch

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import synth, walks as wmod

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    # roots per block; default (0) = all entities in one block: one global permutation over the
    # whole corpus per epoch, exactly the reference's epoch (a 2e8-walk corpus fits in HBM)
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    depth, number, dim = 4, 20, 200
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    t0 = time.perf_counter()
    edges, V, ents, _ = synth.device_synthetic_kg("barabasi", n, m=10, predicates=200, seed=7)
    g = wv.build_graph(edges, V)
    del edges
    torch.cuda.synchronize()
    t_graph = time.perf_counter() - t0
    cfg = wv.TrainConfig(vector_size=dim, window_size=5, negative_samples=5, learning_rate=0.01, epochs=1)
    prec = sys.argv[3] if len(sys.argv) > 3 else "fp64"  # the reference computes in float64
    sess = wv.SkipGramSession(V, cfg, 42, precision=prec)
    n_roots = int(ents.numel())
    R = R or n_roots
    walk_s = sgns_s = 0.0
    hops = pairs = walks = 0
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for rb in range(0, n_roots, R):
        re_ = min(rb + R, n_roots)
        a = time.perf_counter()
        corpus, lengths, width = wmod.random_walks_fixed(g, ents, depth, number, 42, "pcg64",
                                                         work_begin=rb * number, work_count=(re_ - rb) * number)
        nw = (re_ - rb) * number
        wc = wmod._compact(torch, dev, corpus, lengths, nw, width, wmod.RANDOM)
        del corpus, lengths
        torch.cuda.synchronize()
        b = time.perf_counter()
        sess.fit(wc, 1)
        torch.cuda.synchronize()
        c = time.perf_counter()
        walk_s += b - a
        sgns_s += c - b
        walks += nw
        hops += (wc.total_tokens - nw) // 2
        pairs += sess.last_pairs
    total = time.perf_counter() - t1
    print(json.dumps({
        "workload": f"BA({n}, m=10) -> {g.edge_count} triples, 200 predicates; random walks depth {depth} x {number} "
                    f"per entity; SGNS d{dim} w5 k5, 1 GiB batch rule ({sess.last_batch_size} pairs), 1 epoch; "
                    f"{R}-root blocks; one B200",
        "vocab": V, "walks": walks, "hops": hops, "pairs": pairs,
        "graph_build_s": t_graph, "walks_s": walk_s, "sgns_s": sgns_s, "walks_plus_sgns_s": total,
        "end_to_end_s": t_graph + total, "walk_hops_per_s": hops / walk_s, "sgns_pairs_per_s": pairs / sgns_s,
        "precision": prec,
        "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
    }), flush=True)


if __name__ == "__main__":
    main()
