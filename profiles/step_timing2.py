"""Compare SkipGramSession.fit per-batch time vs a fresh replica per step."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench
import paper_2508_01073_b200 as wv
from paper_2508_01073_b200 import walks as wmod, w2v as w2vmod, _lib

g, V, ents = bench.make_graph()
cfg = wv.TrainConfig(vector_size=200, window_size=5, negative_samples=5, learning_rate=0.01, epochs=1)
sess = wv.SkipGramSession(V, cfg, 42)
dev = torch.device("cuda", 0)
R = 8192
def t(): torch.cuda.synchronize(); return time.perf_counter()
mode = sys.argv[1] if len(sys.argv) > 1 else "session"
orig_run = w2vmod._Replica.run
def timed_run(self, count, rows):
    t0 = t(); orig_run(self, count, rows); t1 = t()
    print(f"   run({count}, {rows}) {1e3*(t1-t0):.1f} ms = {1e3*(t1-t0)/max(count,1):.3f} ms/batch, graphs={len(self.graphs)}")
w2vmod._Replica.run = timed_run
for step in range(6):
    rb, re_ = (step + 3) * R, (step + 4) * R
    corpus, lengths, width = wmod.random_walks_fixed(g, ents, 8, 100, 42, "pcg64", work_begin=rb * 100, work_count=(re_ - rb) * 100)
    wc = wmod._compact(torch, dev, corpus, lengths, (re_ - rb) * 100, width, wmod.RANDOM)
    t0 = t()
    if mode == "fresh":
        sess.last_replica = None
    sess.fit(wc, 1)
    t1 = t()
    print(f"step {step} [{mode}]: fit {1e3*(t1-t0):.1f} ms, pairs {sess.last_pairs}")
