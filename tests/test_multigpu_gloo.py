"""World-size-2 gloo test (CPU) of the C5 multi-view step's host logic: views[r::N] sharding, the flat
gradient layout and the single SUM allreduce.  Per-view gradients come from the oracle here (the
device kernels need a GPU); the check is that the sharded+allreduced gradient equals the
single-process sum over all views and is identical on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2501_16312_b200 import scenegen, train
from tests.helpers import oscene

N_VIEWS = 4


def _scene():
    scene, cams = scenegen.make_scene("C5", seed=3, n=400)
    cams = [dict(c, width=40, height=32, cx=np.float32(20), cy=np.float32(16), fx=np.float32(34.6),
                 fy=np.float32(34.6)) for c in cams[:N_VIEWS]]
    return scene, cams


def _flat_grad(scene, cams, views):
    n, kind, deg = scene["pos"].shape[1], scene["kind"], scene["sh_degree"]
    off = train.flat_offsets(kind, n, deg)
    flat = np.zeros(max(e for _, e in off.values()), np.float64)
    for v in views:
        G = scenegen.upstream_grad(40, 32, seed=v)[0]
        _, g = oracle.forward_backward(oscene(scene), cams[v], G)
        for name in ("pos", "rot", "dist", "opacity", "sh"):
            b, e = off[name]
            flat[b:e] += getattr(g, name).reshape(-1)
    return flat


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cams = _scene()
    views = train.shard_views(N_VIEWS, rank, world)
    g = torch.from_numpy(_flat_grad(scene, cams, views))
    train.allreduce_gradients(g, world)
    np.save(os.path.join(out_dir, f"g{rank}.npy"), g.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_views():
    assert train.shard_views(8, 0, 1) == list(range(8))
    assert train.shard_views(8, 1, 2) == [1, 3, 5, 7]
    assert sorted(sum((train.shard_views(8, r, 4) for r in range(4)), [])) == list(range(8))
    with pytest.raises(ValueError):
        train.shard_views(8, 2, 2)


def test_lr_groups_cover_every_parameter_once():
    off = train.flat_offsets(0, 100, 3)
    groups = train.lr_groups(off, 100)
    cover = np.zeros(max(e for _, e in off.values()), np.int32)
    for b, e, lr in groups:
        cover[b:e] += 1
        assert lr > 0
    assert np.all(cover == 1)


def test_two_rank_gloo_allreduce_matches_single_process(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g0 = np.load(tmp_path / "g0.npy")
    g1 = np.load(tmp_path / "g1.npy")
    assert np.array_equal(g0, g1)                          # every rank holds the same sum
    scene, cams = _scene()
    ref = _flat_grad(scene, cams, range(N_VIEWS))
    assert np.allclose(g0, ref, rtol=1e-12, atol=1e-18)    # == the single-process sum over all views
    assert np.abs(ref).max() > 0
