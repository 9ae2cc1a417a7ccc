"""BASELINE cfg5 graph + walks on one B200: BA(1e8, m=10) with 200 predicates (~1e9
triples) generated, encoded and built into a CSR on the device, then random walks
depth 4 x 20 per entity (2e9 walks) in root blocks.  (cfg5's SGNS state, 6 x 1e8 x
200 fp32 = 480 GB, needs the row-sharded mode over >= 4 GPUs: shard.py.)

    python profiles/cfg5_walks.py [n_entities] [roots_per_block]
"""
import json
import sys
import time

sys.path.insert(0, ".")


def main():
    import torch

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import synth, walks as wmod

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 22
    torch.cuda.set_device(0)
    t0 = time.perf_counter()
    edges, V, ents, _ = synth.device_synthetic_kg("barabasi", n, m=10, predicates=200, seed=7)
    g = wv.build_graph(edges, V)
    del edges
    torch.cuda.synchronize()
    t_graph = time.perf_counter() - t0
    mem_graph = torch.cuda.max_memory_allocated() / 1e9
    n_roots = int(ents.numel())
    stream = torch.cuda.current_stream()
    kern_ms = 0.0
    hops = walks = 0
    t1 = time.perf_counter()
    for rb in range(0, n_roots, R):
        re_ = min(rb + R, n_roots)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(1_000_000)
        e0.record(stream)
        corpus, lengths, width = wmod.random_walks_fixed(g, ents, 4, 20, 42, "pcg64", work_begin=rb * 20,
                                                         work_count=(re_ - rb) * 20)
        e1.record(stream)
        e1.synchronize()
        kern_ms += e0.elapsed_time(e1)
        nw = (re_ - rb) * 20
        hops += int((lengths[:nw].sum().item() - nw) // 2)
        walks += nw
        del corpus, lengths
    total = time.perf_counter() - t1
    print(json.dumps({"workload": f"cfg5: BA({n}, m=10) -> {g.edge_count} triples, 200 predicates; walks depth 4 x 20",
                      "graph_build_s": t_graph, "graph_peak_mem_gb": mem_graph, "walks": walks, "hops": hops,
                      "walk_kernel_s": kern_ms / 1e3, "walk_hops_per_s": hops / (kern_ms / 1e3),
                      "walks_wall_s": total, "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)


if __name__ == "__main__":
    main()
