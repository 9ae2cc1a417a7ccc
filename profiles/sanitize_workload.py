"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Every kernel family of the path at a cfg1-like shape cut down so the tools
finish in minutes: device BA graph + encoding, CSR, random walks (PCG64 and
Philox), duplicate-free, BFS (+ cap), projection, pair index, SGNS training in
both stores and both pair sources, pipelined batches on two workspace halves
(eager and CUDA-graph replayed), CBOW, replica merge, the fp64 export.

    compute-sanitizer --tool memcheck python profiles/sanitize_workload.py
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import synth

    torch.cuda.set_device(0)
    edges, V, ents, _ = synth.device_synthetic_kg("barabasi", 3000, m=5, predicates=20, seed=7)
    g = wv.build_graph(edges, V)
    roots = ents.cpu().numpy()
    c1 = wv.random_walks(g, roots, walk_depth=4, walk_number=10, rng_seed=42)
    c2 = wv.random_walks(g, roots[:500], walk_depth=6, walk_number=4, rng_seed=1, rng="philox", duplicate_free=True)
    b, table = wv.bfs_walks(g, roots[:200], 3, max_walks_per_root=50)
    wv.project_corpus(c1, "entity")
    for precision in ("fp32", "fp64"):
        for pairs in ("device", "numpy"):
            cfg = wv.TrainConfig(vector_size=100, window_size=5, negative_samples=5, min_count=2, epochs=1,
                                 batch_size=4096)
            model, losses = wv.train(c1, V, cfg, 42, precision=precision, pairs=pairs, graph_batches=1)
            model.input_matrix
    cfg = wv.TrainConfig(vector_size=200, window_size=5, negative_samples=5, min_count=1, epochs=1, batch_size=2000)
    sess = wv.SkipGramSession(V, cfg, 3, precision="fp32", graph_batches=4)
    sess.fit(c2, 1)
    cb = wv.TrainConfig(model="cbow", vector_size=64, window_size=3, min_count=1, epochs=1, batch_size=1024)
    wv.train(c2, V, cb, 5, graph_batches=1)
    multi = wv.TrainConfig(vector_size=32, window_size=3, negative_samples=3, min_count=1, epochs=1,
                           batch_size=512, workers=2, reproducible=True)
    wv.train(c2, V, multi, 9, graph_batches=1)
    torch.cuda.synchronize()
    print("sanitize workload done", len(c1), len(c2), len(b), len(table), losses)


if __name__ == "__main__":
    main()
