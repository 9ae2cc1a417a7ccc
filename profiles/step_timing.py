"""Host-side anatomy of one bench step (where the GPU idles between SGNS batches)."""
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
for step in range(4):
    rb, re_ = step * R + 3 * R, (step + 1) * R + 3 * R
    t0 = t()
    corpus, lengths, width = wmod.random_walks_fixed(g, ents, 8, 100, 42, "pcg64", work_begin=rb * 100, work_count=(re_ - rb) * 100)
    t1 = t()
    wc = wmod._compact(torch, dev, corpus, lengths, (re_ - rb) * 100, width, wmod.RANDOM)
    t2 = t()
    tr = w2vmod._Trainer(wc, V, cfg, 42, lambda *a, **k: None, "fp32", "device", 64, device=dev)
    t3 = t()
    rep = w2vmod._Replica(tr, 0, sess.params)
    t4 = t()
    B, N = tr.batch_size, tr.N
    full, rem = divmod(N, B)
    _lib.call("wv_sgns_epoch_begin", _lib.ptr(sess.params.state), 100 + step, 0, _lib.stream_ptr())
    rep.run(64, B)  # includes capture
    t5 = t()
    rep.run(full - 64, B)
    t6 = t()
    st = sess.params.read_state()
    t7 = t()
    print(f"step {step}: walks {1e3*(t1-t0):.1f} ms, compact {1e3*(t2-t1):.1f}, trainer/corpus {1e3*(t3-t2):.1f}, "
          f"replica+ws {1e3*(t4-t3):.1f}, capture+64 batches {1e3*(t5-t4):.1f}, {full-64} batches {1e3*(t6-t5):.1f} "
          f"({1e3*(t6-t5)/(full-64):.3f} ms/batch), state {1e3*(t7-t6):.1f}; N={N} batches={full}")
