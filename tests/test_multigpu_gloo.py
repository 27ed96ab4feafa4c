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


def _spawn(fn, world, out_dir, tries=3):
    """mp.spawn on a fresh rendezvous port; a port taken between probing and binding (a race with any
    other process on the host) is retried on a new one."""
    for attempt in range(tries):
        try:
            mp.spawn(fn, args=(world, _free_port(), out_dir), nprocs=world, join=True)
            return
        except mp.ProcessRaisedException:
            if attempt == tries - 1:
                raise


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
    _spawn(_worker, world, str(tmp_path))
    g0 = np.load(tmp_path / "g0.npy")
    g1 = np.load(tmp_path / "g1.npy")
    assert np.array_equal(g0, g1)                          # every rank holds the same sum
    scene, cams = _scene()
    ref = _flat_grad(scene, cams, range(N_VIEWS))
    assert np.allclose(g0, ref, rtol=1e-12, atol=1e-18)    # == the single-process sum over all views
    assert np.abs(ref).max() > 0


# ---------------------------------------------------------------- sharded optimizer (N > 1)

def _adam_ref(p, g, m, v, groups, step, b1=0.9, b2=0.999, eps=1e-15):
    """Plain per-element Adam with bias correction over the listed groups (test reference)."""
    bc1, bc2 = 1 - b1 ** step, 1 - b2 ** step
    for b, e, lr in groups:
        m[b:e] = b1 * m[b:e] + (1 - b1) * g[b:e]
        v[b:e] = b2 * v[b:e] + (1 - b2) * g[b:e] * g[b:e]
        p[b:e] = p[b:e] - lr * (m[b:e] / bc1) / (torch.sqrt(v[b:e] / bc2) + eps)


@pytest.mark.parametrize("total,world", [(1000, 2), (1003, 2), (7, 4), (4096, 8), (13, 3)])
def test_shard_range_partitions_the_buffer(total, world):
    seen = np.zeros(total, np.int32)
    chunks = set()
    for r in range(world):
        lo, hi, chunk = train.shard_range(total, r, world)
        assert chunk % 4 == 0 and world * chunk >= total
        assert lo == min(r * chunk, total) and hi - lo <= chunk
        seen[lo:hi] += 1
        chunks.add(chunk)
    assert len(chunks) == 1 and np.all(seen == 1)


def test_shard_groups_clip_and_rebase():
    groups = [(0, 10, 1.0), (10, 25, 2.0), (25, 40, 3.0)]
    assert train.shard_groups(groups, 8, 20) == [(0, 2, 1.0), (2, 12, 2.0)]
    assert train.shard_groups(groups, 30, 32) == [(0, 2, 3.0)]
    assert train.shard_groups(groups, 40, 48) == []


def _zero_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cams = _scene()
    n, kind, deg = scene["pos"].shape[1], scene["kind"], scene["sh_degree"]
    off = train.flat_offsets(kind, n, deg)
    total = max(e for _, e in off.values())
    lo, hi, chunk = train.shard_range(total, rank, world)
    g = torch.zeros(world * chunk, dtype=torch.float32)
    g[:total] = torch.from_numpy(_flat_grad(scene, cams, train.shard_views(N_VIEWS, rank, world))).float()
    p = torch.zeros(world * chunk, dtype=torch.float32)
    p[:total] = torch.linspace(-1, 1, total)
    gs = torch.zeros(chunk, dtype=torch.float32)
    train.reduce_scatter_gradients(g, gs, world)
    m, v = torch.zeros(chunk), torch.zeros(chunk)
    groups = train.shard_groups(train.lr_groups(off, n), lo, hi)
    _adam_ref(p[rank * chunk:(rank + 1) * chunk], gs, m, v, groups, step=1)
    train.all_gather_params(p, rank, chunk)
    np.save(os.path.join(out_dir, f"p{rank}.npy"), p[:total].numpy())
    dist.destroy_process_group()


def test_two_rank_sharded_adam_matches_allreduce_adam(tmp_path):
    """reduce-scatter + Adam on the rank's shard + all-gather == allreduce + replicated Adam."""
    world = 2
    _spawn(_zero_worker, world, str(tmp_path))
    p0, p1 = np.load(tmp_path / "p0.npy"), np.load(tmp_path / "p1.npy")
    assert np.array_equal(p0, p1)
    scene, cams = _scene()
    n, kind, deg = scene["pos"].shape[1], scene["kind"], scene["sh_degree"]
    off = train.flat_offsets(kind, n, deg)
    total = max(e for _, e in off.values())
    g = torch.zeros(total, dtype=torch.float32)
    for r in range(world):   # the float32 sum of the two ranks' gradients, as the collective forms it
        g += torch.from_numpy(_flat_grad(scene, cams, train.shard_views(N_VIEWS, r, world))).float()
    p = torch.linspace(-1, 1, total)
    m, v = torch.zeros(total), torch.zeros(total)
    _adam_ref(p, g, m, v, train.lr_groups(off, n), step=1)
    assert np.array_equal(p0, p.numpy())
    assert np.abs(p0 - np.linspace(-1, 1, total)).max() > 1e-4   # the step moved the parameters


def _chunked_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cams = _scene()
    n, kind, deg = scene["pos"].shape[1], scene["kind"], scene["sh_degree"]
    off = train.flat_offsets(kind, n, deg)
    total = max(e for _, e in off.values())
    g = torch.from_numpy(_flat_grad(scene, cams, train.shard_views(N_VIEWS, rank, world))).float()
    p = torch.linspace(-1, 1, total)
    m, v = torch.zeros(total), torch.zeros(total)
    groups = train.lr_groups(off, n)
    bounds = train.chunk_bounds(total, 4)
    works = train.allreduce_gradients_chunked(g, world, bounds)
    for (lo, hi), work in zip(bounds, works):   # TrainStep.run's order: wait chunk k, Adam on chunk k
        work.wait()
        _adam_ref(p[lo:hi], g[lo:hi], m[lo:hi], v[lo:hi], train.shard_groups(groups, lo, hi), step=1)
    np.save(os.path.join(out_dir, f"c{rank}.npy"), p.numpy())
    dist.destroy_process_group()


def test_chunk_bounds_cover_the_buffer():
    for total, parts in ((0, 4), (1, 4), (7, 4), (1000, 4), (1001, 3), (59 * 1000, 4)):
        b = train.chunk_bounds(total, parts)
        assert [x for lo, hi in b for x in range(lo, hi)] == list(range(total))
        assert all(lo % 4 == 0 and hi > lo for lo, hi in b) and len(b) <= parts


def test_two_rank_chunked_allreduce_adam_matches_single(tmp_path):
    """The chunked allreduce (one async collective per chunk) with Adam per chunk on groups clipped to
    the chunk == one allreduce + Adam over the whole buffer (TrainStep's N > 1 default)."""
    world = 2
    _spawn(_chunked_worker, world, str(tmp_path))
    c0, c1 = np.load(tmp_path / "c0.npy"), np.load(tmp_path / "c1.npy")
    assert np.array_equal(c0, c1)
    scene, cams = _scene()
    n, kind, deg = scene["pos"].shape[1], scene["kind"], scene["sh_degree"]
    off = train.flat_offsets(kind, n, deg)
    total = max(e for _, e in off.values())
    g = torch.zeros(total, dtype=torch.float32)
    for r in range(world):
        g += torch.from_numpy(_flat_grad(scene, cams, train.shard_views(N_VIEWS, r, world))).float()
    p = torch.linspace(-1, 1, total)
    m, v = torch.zeros(total), torch.zeros(total)
    _adam_ref(p, g, m, v, train.lr_groups(off, n), step=1)
    assert np.array_equal(c0, p.numpy())
