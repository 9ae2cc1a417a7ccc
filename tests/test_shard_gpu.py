"""Row-sharded SGNS / CBOW (SURVEY §8e, cfg5 mode) on one GPU: two ranks (processes)
over gloo with host staging; each rank's rows must equal single-GPU training with
the same global batch, bit for bit (fp32 device streams and fp64 numpy replay)."""

import json
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out_dir):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    os.environ["WV_SHARD_CHECK"] = "1"  # lookahead split sizes == the exchanged device counts, every batch
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    import paper_2508_01073_b200 as wv
    from paper_2508_01073_b200.shard import train_row_sharded

    g = np.load(os.path.join(ROOT, "tests", "golden", case["golden"]))
    corpus = wv.WalkCorpus(g["train_tokens"], g["train_offsets"])
    V = int(g["train_V"])
    cfg = wv.TrainConfig(**case["cfg"])
    p, losses = train_row_sharded(corpus, V, cfg, 42, precision=case["precision"], pairs=case["pairs"])
    inp = p.inp.view(p.V, p.d).double().cpu().numpy()
    out = p.out.view(p.V, p.d).double().cpu().numpy()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), inp=inp, out=out, losses=np.array(losses))
    dist.barrier()
    dist.destroy_process_group()


CASES = {
    "sgns_fp32_device": dict(golden="w2v.npz", precision="fp32", pairs="device",
                             cfg=dict(min_count=1, vector_size=16, epochs=2, window_size=3, negative_samples=5,
                                      batch_size=96)),
    "sgns_fp64_replay": dict(golden="w2v.npz", precision="fp64", pairs="numpy",
                             cfg=dict(min_count=2, vector_size=12, epochs=2, window_size=3, negative_samples=4,
                                      learning_rate=0.02, batch_size=64)),
    "cbow_fp32_device": dict(golden="cbow.npz", precision="fp32", pairs="device",
                             cfg=dict(model="cbow", min_count=1, vector_size=16, epochs=2, window_size=2,
                                      batch_size=80)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_row_sharded_equals_single_gpu(tmp_path, name):
    import torch.multiprocessing as mp

    import paper_2508_01073_b200 as wv

    case = CASES[name]
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    g = np.load(os.path.join(ROOT, "tests", "golden", case["golden"]))
    corpus = wv.WalkCorpus(g["train_tokens"], g["train_offsets"])
    V = int(g["train_V"])
    model, losses = wv.train(corpus, V, wv.TrainConfig(**case["cfg"]), 42, precision=case["precision"],
                             pairs=case["pairs"])
    ref_in, ref_out = model.input_matrix, model.output_matrix
    if case["precision"] == "fp32":  # the fp32 store as it is on the device (untouched rows re-exported in fp64)
        ref_in = model.device_input.double().cpu().numpy().reshape(V, -1)
        ref_out = model.device_output.double().cpu().numpy().reshape(V, -1)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        rows = np.arange(r, V, world)
        n = len(rows)
        assert np.array_equal(got["inp"][:n], ref_in[rows]), f"rank {r} input rows"
        assert np.array_equal(got["out"][:n], ref_out[rows]), f"rank {r} output rows"
        np.testing.assert_allclose(got["losses"], losses, rtol=1e-12)
