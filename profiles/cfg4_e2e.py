"""BASELINE cfg4 on one B200: FB15k-237-shaped synthetic KG (Erdos-Renyi(15,000,
p=0.001378) with 237 predicates, ~310k triples), random walks depth 16 x
500 per entity (7.5e6 walks), SGNS 5 epochs (d=100, window 5, 5 negatives, the
reference's 1 GiB batch rule).  Prints one JSON line.

    python profiles/cfg4_e2e.py [epochs]
"""
import json
import sys
import time

sys.path.insert(0, ".")


def main():
    import torch

    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200 import synth

    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    torch.cuda.set_device(0)
    t0 = time.perf_counter()
    edges, V, ents, _ = synth.device_synthetic_kg("erdos_renyi", 15_000, p=0.001378, predicates=237, seed=7)
    g = wv.build_graph(edges, V)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    corpus = wv.random_walks(g, ents.cpu().numpy(), walk_depth=16, walk_number=500, rng_seed=42)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cfg = wv.TrainConfig(vector_size=100, window_size=5, negative_samples=5, learning_rate=0.01, epochs=epochs,
                         min_count=10)
    model, losses = wv.train(corpus, V, cfg, 42)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    pairs = model.n_pairs * epochs
    print(json.dumps({"workload": f"cfg4: ER(15000, p=0.001378) -> {g.edge_count} triples, 237 predicates; walks depth "
                                  f"16 x 500 ({len(corpus)} walks); SGNS d100 w5 k5, batch {model.batch_size}, "
                                  f"{epochs} epochs",
                      "graph_s": t1 - t0, "walks_s": t2 - t1, "train_s": t3 - t2, "total_s": t3 - t0,
                      "pairs": pairs, "sgns_pairs_per_s": pairs / (t3 - t2), "losses": losses}), flush=True)


if __name__ == "__main__":
    main()
