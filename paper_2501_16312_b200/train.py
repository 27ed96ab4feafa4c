"""Host-side logic of the C5 multi-view training step (row a13): view sharding, the flat gradient
layout, the single gradient allreduce and the paper's per-group learning rates.

The device work of a step is liblinprim (preprocess / bin_sort / render_fwd / l1 / raster_bwd per
local view, one fused preprocess_bwd, one Adam); this module only decides WHICH views a rank
renders and HOW the per-rank gradients are combined, so it is testable on CPU with gloo
(tests/test_multigpu_gloo.py).
"""
from __future__ import annotations


def section_sizes(kind, n, sh_degree):
    """Sections of the flat feature / gradient buffer (same SoA layout as lp_prims)."""
    K = 3 if kind == 0 else 4
    return [("pos", 3 * n), ("rot", 4 * n), ("dist", K * n), ("opacity", n), ("sh", (sh_degree + 1) ** 2 * 3 * n)]


def shard_views(n_views: int, rank: int, world: int) -> list:
    """views[r::N] on rank r: strong scaling of a fixed global batch (north_star: 8 views, 1/2/4/8 GPUs)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return list(range(rank, n_views, world))


def flat_offsets(kind: int, n: int, sh_degree: int) -> dict:
    """[begin, end) of each feature section in the flat buffer [pos | rot | dist | opacity | sh]."""
    out, o = {}, 0
    for name, size in section_sizes(kind, n, sh_degree):
        out[name] = (o, o + size)
        o += size
    return out


def lr_groups(offsets: dict, n: int, extent: float = 4.0) -> list:
    """Adam groups (begin, end, lr): colour (SH DC) 2.5e-3, SH rest 1.25e-4, opacity 2.5e-2,
    rotation 1e-3, distance 2.6^-1 1e-4 x extent; position 1.6e-4 x extent (3DGS)."""
    return [(offsets["pos"][0], offsets["pos"][1], 1.6e-4 * extent),
            (offsets["rot"][0], offsets["rot"][1], 1e-3),
            (offsets["dist"][0], offsets["dist"][1], 1e-4 / 2.6 * extent),
            (offsets["opacity"][0], offsets["opacity"][1], 2.5e-2),
            (offsets["sh"][0], offsets["sh"][0] + 3 * n, 2.5e-3),
            (offsets["sh"][0] + 3 * n, offsets["sh"][1], 1.25e-4)]


def allreduce_gradients(flat_grad, world: int):
    """The step's single exchange: SUM-allreduce of the flat fp32 gradient (NCCL on GPUs, gloo in tests)."""
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(flat_grad, op=dist.ReduceOp.SUM)
    return flat_grad


def chunk_bounds(total: int, parts: int, align: int = 4) -> list:
    """[(lo, hi)] covering [0, total) in `parts` contiguous pieces of about equal size, every lo a
    multiple of `align` (float4 Adam path); empty pieces dropped."""
    per = -(-total // max(1, parts))
    per = -(-per // align) * align
    return [(lo, min(lo + per, total)) for lo in range(0, total, per)] if total > 0 else []


def allreduce_gradients_chunked(flat_grad, world: int, bounds):
    """The same SUM-allreduce as `allreduce_gradients`, issued as one asynchronous collective per
    chunk of `bounds` (in order); returns the works.  The caller waits chunk k's work before its
    optimizer step on chunk k, so Adam on chunk k overlaps the transfer of chunk k + 1."""
    import torch.distributed as dist
    return [dist.all_reduce(flat_grad[lo:hi], op=dist.ReduceOp.SUM, async_op=True) for lo, hi in bounds]


# ---------------------------------------------------------------------------------------------
# sharded optimizer (N > 1): reduce-scatter the flat gradient, Adam on the rank's shard only,
# all-gather the parameters -- the allreduce's wire bytes, 1/N of the Adam work and Adam state
# per rank (SURVEY §8e variant).
# ---------------------------------------------------------------------------------------------
def shard_range(total: int, rank: int, world: int, align: int = 4):
    """(lo, hi, chunk): the rank's [lo, hi) of a flat buffer of `total` elements split into `world`
    equal chunks of `chunk` elements (a multiple of `align`, so the float4 Adam path applies); the
    buffer is padded to world * chunk, the padding belongs to the last ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    per = -(-total // world)
    chunk = -(-per // align) * align
    lo = min(rank * chunk, total)
    hi = min(lo + chunk, total)
    return lo, hi, chunk


def shard_groups(groups, lo: int, hi: int) -> list:
    """Adam groups (begin, end, lr) clipped to [lo, hi) and re-based to the shard start."""
    out = []
    for b, e, lr in groups:
        b2, e2 = max(int(b), lo), min(int(e), hi)
        if b2 < e2:
            out.append((b2 - lo, e2 - lo, lr))
    return out


def reduce_scatter_gradients(flat_grad_padded, grad_shard, world: int):
    """grad_shard (chunk elements) <- this rank's chunk of the SUM over ranks of flat_grad_padded."""
    import torch.distributed as dist
    dist.reduce_scatter_tensor(grad_shard, flat_grad_padded, op=dist.ReduceOp.SUM)
    return grad_shard


def all_gather_params(flat_padded, rank: int, chunk: int):
    """Every rank's updated chunk into every rank's padded parameter buffer (in place: the input is
    this rank's chunk of the output)."""
    import torch.distributed as dist
    dist.all_gather_into_tensor(flat_padded, flat_padded[rank * chunk:(rank + 1) * chunk])
    return flat_padded
