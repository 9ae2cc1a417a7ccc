"""GPU ingest throughput on a synthetic N-Triples document.

    python profiles/ingest_bench.py [n_entities]          # GPU box: device ingest
    python profiles/ingest_bench.py [n_entities] --ref    # build container: the reference parser

Document: BA(n, m=10) edges with 200 predicates as <http://kg/e{u}> <http://kg/p{k}> <http://kg/e{v}> .
lines.  GPU time covers the whole call (pinned H2D of the bytes, parse,
interning, edges and vocabulary back to the host).
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")


def document(n: int) -> bytes:
    from paper_2508_01073_b200.synth import barabasi_edges, predicate_picks

    e = barabasi_edges(n, 10, 7)
    pk = predicate_picks(len(e), 200, 7)
    lines = [f"<http://kg/e{u}> <http://kg/p{k}> <http://kg/e{v}> .\n"
             for u, k, v in zip(e[:, 0].tolist(), pk.tolist(), e[:, 1].tolist())]
    return "".join(lines).encode()


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 100_000
    doc = document(n)
    lines = doc.count(b"\n")
    if "--ref" in sys.argv:
        import io

        sys.path.insert(0, "/root/reference/pkg/src")
        from walkvec.ingest import build_vocabulary, parse_ntriples

        t0 = time.perf_counter()
        vocab, edges = build_vocabulary(parse_ntriples(io.BytesIO(doc)))
        dt = time.perf_counter() - t0
        print(f"reference (1 core): {lines} triples, {len(doc) / 1e6:.1f} MB in {dt:.2f} s -> "
              f"{lines / dt / 1e6:.3f} M triples/s, {len(doc) / dt / 1e6:.1f} MB/s; vocab {len(vocab)}")
        return
    import torch

    from paper_2508_01073_b200.ingest import load_triples_device

    for _ in range(3):
        load_triples_device(doc)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        vocab, edges = load_triples_device(doc)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    dt = float(np.median(ts))
    print(f"GPU ingest: {lines} triples, {len(doc) / 1e6:.1f} MB in {dt * 1e3:.1f} ms -> "
          f"{lines / dt / 1e6:.2f} M triples/s, {len(doc) / dt / 1e9:.2f} GB/s; vocab {len(vocab)}, edges {len(edges)}")


if __name__ == "__main__":
    main()
