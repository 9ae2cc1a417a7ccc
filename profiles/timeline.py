"""Timeline of pipelined SGNS batches on the cfg2 workload: per batch, device timestamps of
the side stream (decode + grouping) and of the gather / update on the main stream, with the
light-row owner and the concurrent heavy pieces ended separately.

    python profiles/timeline.py [fp64|fp32]     (on the GPU box)
"""
import ctypes as C
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

import bench
import paper_2508_01073_b200 as wv
from paper_2508_01073_b200 import _lib, walks as wmod

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
g, V, ents = bench.make_graph()
dev = torch.device('cuda', 0)
cfg = wv.TrainConfig(vector_size=200, window_size=5, negative_samples=5, learning_rate=0.01, epochs=1)
sess = wv.SkipGramSession(V, cfg, 42, precision=prec)
for blk in range(2):
    corpus, lengths, width = wmod.random_walks_fixed(g, ents, 8, 100, 42, "pcg64", work_begin=blk * 819200,
                                                     work_count=819200)
    wc = wmod._compact(torch, dev, corpus, lengths, 819200, width, wmod.RANDOM)
    sess.fit(wc, 1)
torch.cuda.synchronize()
rep = sess.last_replica
n, S = 24, 7
timer = _lib.DeviceTimer(S * n)
bs = rep.t.batch_struct
bs.batch_rows = rep.batch_size
bs.timer, bs.timer_base = timer.h, 0
_lib.call("wv_sgns_batches", C.byref(rep.p.struct), C.byref(bs), _lib.ptr(rep.ws), rep.ws.numel(), n, _lib.stream_ptr())
bs.timer, bs.timer_base = None, 0
torch.cuda.synchronize()
t = np.array([[timer.elapsed(0, S * i + j) for j in range(S)] for i in range(n)]) * 1e3
print(f"{prec}: batch  side0   side1   g0      g1      upd1  light1  heavy1 | side  gather upd  light heavy gap")
for i in range(n):
    gap = t[i, 2] - t[i - 1, 4] if i else 0
    print(f"{i:3d} " + " ".join(f"{x:7.1f}" for x in t[i]) +
          f" | {t[i,1]-t[i,0]:5.1f} {t[i,3]-t[i,2]:5.1f} {t[i,4]-t[i,3]:5.1f} {t[i,5]-t[i,3]:5.1f} {t[i,6]-t[i,3]:5.1f}"
          f" {gap:6.1f}")
m = t[4:]
print("mean batch period us", (t[-1, 4] - t[4, 4]) / (n - 5))
print("means (batches 4..): side %.1f gather %.1f update %.1f light %.1f heavy %.1f" % (
    np.mean(m[:, 1] - m[:, 0]), np.mean(m[:, 3] - m[:, 2]), np.mean(m[:, 4] - m[:, 3]), np.mean(m[:, 5] - m[:, 3]),
    np.mean(m[:, 6] - m[:, 3])))
