"""N > 1 data-parallel path on CPU (gloo, world_size 2): the LPT shard assignment every
rank computes is identical and disjoint, and the SUM all-reduced parameter gradients of
the shards equal the single-process gradients of the whole batch (gradients are sums
over tokens).  Per-shard gradients come from the fp64 oracle, standing in for the GPU
layer (which the -m gpu tests check against the same oracle)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2602_16986_b200 import dist as D
from paper_2602_16986_b200 import synth
from paper_2602_16986_b200 import uhstu as U

LENGTHS = [40, 7, 33, 64, 5, 18, 51, 9]
H, DH, K1, K2 = 2, 4, 6, 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    d = H * DH
    cfg = synth.Config("dp", LENGTHS, H=H, dh=DH, K1=K1, K2=K2, N=64.0, seed=21, pos_len=16, ts_len=8)
    p = synth.layer_params(d, cfg.seed)
    prm = O.LayerParams(**{k: np.asarray(v, np.float64) for k, v in p.items()})
    x, dout = synth.layer_inputs(cfg)
    pos, ts = synth.rab_tables(cfg)
    t = synth.timestamps(cfg.seed, cfg.lengths)
    return cfg, prm, x, dout, pos, ts, t


def _oracle_grads(cfg, prm, x, dout, pos, ts, t, ids):
    off = cfg.offsets()
    rows = np.concatenate([np.arange(off[i], off[i + 1]) for i in ids]) if ids else np.zeros(0, int)
    lens = [cfg.lengths[i] for i in ids]
    o2 = np.zeros(len(lens) + 1, np.int32)
    o2[1:] = np.cumsum(lens)
    spec = O.AttnSpec(K1=K1, K2=K2, alpha=1.0, N=cfg.N, pos_w=pos, ts_w=ts, timestamps=t[rows])
    _, g = O.layer_backward(dout[rows], o2, prm, H, spec, x=x[rows])
    return g


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg, prm, x, dout, pos, ts, t = _problem()
    ids, lens, cost = D.shard(cfg.lengths, world, rank, U.mask(K1, K2), cfg.d, H)
    g = _oracle_grads(cfg, prm, x, dout, pos, ts, t, ids)
    shapes = {k: (g["pos_w"].shape if k == "pos_bias" else g["ts_w"].shape if k == "time_bias" else g[k].shape)
              for k in D.GRAD_NAMES}
    bucket = D.GradBucket(shapes, "cpu")
    for k in D.GRAD_NAMES:
        src = g["pos_w"] if k == "pos_bias" else g["ts_w"] if k == "time_bias" else g[k]
        bucket.views[k].copy_(torch.from_numpy(np.asarray(src, np.float32)))
    bucket.allreduce_()
    q.put((rank, ids, bucket.flat.numpy().copy(), cost.tolist()))
    dist.destroy_process_group()


def test_dp_world2_allreduce_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids0, ids1 = res[0][1], res[1][1]
    assert sorted(ids0 + ids1) == list(range(len(LENGTHS))) and not set(ids0) & set(ids1)
    assert res[0][3] == res[1][3]                       # every rank computed the same assignment
    assert np.array_equal(res[0][2], res[1][2])         # all-reduced buckets are identical
    cfg, prm, x, dout, pos, ts, t = _problem()
    g = _oracle_grads(cfg, prm, x, dout, pos, ts, t, list(range(len(LENGTHS))))
    shapes = {k: (g["pos_w"].shape if k == "pos_bias" else g["ts_w"].shape if k == "time_bias" else g[k].shape)
              for k in D.GRAD_NAMES}
    full = D.GradBucket(shapes, "cpu")
    for k in D.GRAD_NAMES:
        src = g["pos_w"] if k == "pos_bias" else g["ts_w"] if k == "time_bias" else g[k]
        full.views[k].copy_(torch.from_numpy(np.asarray(src, np.float32)))
    f = full.flat.numpy()
    assert np.max(np.abs(res[0][2] - f)) <= 1e-5 * max(np.max(np.abs(f)), 1.0)


def test_bucket_views_aligned_and_disjoint():
    shapes = {"ln1_w": (6,), "w1": (6, 24), "b1": (24,), "w2": (6, 6), "pos_bias": (5,), "time_bias": (3,)}
    b = D.GradBucket(shapes, "cpu")
    seen = set()
    for k, v in b.views.items():
        if v is None:
            continue
        assert (v.data_ptr() - b.flat.data_ptr()) % 16 == 0
        rng = set(range((v.data_ptr() - b.flat.data_ptr()) // 4, (v.data_ptr() - b.flat.data_ptr()) // 4 + v.numel()))
        assert not rng & seen
        seen |= rng
