"""cfg5 walk kernel on one B200 for ncu: BA(1e8, m=10), 200 predicates (~1e9 triples, 8.8 GB CSR),
random walks depth 4 x 20 per entity over three 2^22-root blocks (the bench's block size).
    ncu --set full -k regex:random_walk_kernel -s 1 -c 1 python profiles/cfg5_walk_prof.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import synth, walks as wmod

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    torch.cuda.set_device(0)
    edges, V, ents, _ = synth.device_synthetic_kg("barabasi", n, m=10, predicates=200, seed=7)
    g = wv.build_graph(edges, V)
    del edges
    torch.cuda.empty_cache()
    R = 1 << 22
    for b in range(3):
        rb = b * R * 37 % int(ents.numel())  # blocks spread over the id range (young and old vertices)
        rb = min(rb, int(ents.numel()) - R)
        c, l, w = wmod.random_walks_fixed(g, ents, 4, 20, 42, "pcg64", work_begin=rb * 20, work_count=R * 20)
        torch.cuda.synchronize()
        del c, l
    print("done", V, g.edge_count)


if __name__ == "__main__":
    main()
