"""BASELINE cfg3 on one B200: BFS-enumerated walks, depth 4, at most 250 walks per
entity, over every entity of the cfg2 graph (BA(1M, m=10), 200 predicates, generated
on the device).  Prints one JSON line with roots/s, walks/s and tokens/s; the
reference's Python BFS runs ~31 uniform roots/s on one core.

    python profiles/cfg3_bfs.py [n_entities] [roots_per_call]
"""
import json
import sys
import time

sys.path.insert(0, ".")


def main():
    import numpy as np
    import torch

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import synth

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
    torch.cuda.set_device(0)
    edges, V, ents, _ = synth.device_synthetic_kg("barabasi", n, m=10, predicates=200, seed=7)
    g = wv.build_graph(edges, V)
    roots = ents.cpu().numpy()
    # warm-up on a small slice
    wv.bfs_walks(g, roots[:1024], 4, max_walks_per_root=250, with_table=False)
    torch.cuda.synchronize()
    walks = tokens = 0
    t0 = time.perf_counter()
    for rb in range(0, len(roots), R):
        c, _ = wv.bfs_walks(g, roots[rb:rb + R], 4, max_walks_per_root=250, with_table=False)
        walks += len(c)
        tokens += c.total_tokens
        del c
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(json.dumps({"workload": f"cfg3: BFS depth 4, cap 250 walks/root, all {len(roots)} entities of BA({n}, m=10)",
                      "seconds": dt, "roots_per_s": len(roots) / dt, "walks": walks, "walks_per_s": walks / dt,
                      "tokens": tokens, "tokens_per_s": tokens / dt,
                      "reference_roots_per_s_1core": 31.0,
                      "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
    del np


if __name__ == "__main__":
    main()
