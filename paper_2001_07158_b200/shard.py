"""Sieve-point sharding across GPUs.

The 2^k sieve points of one evaluation are independent and the
accumulators are XOR sums over points (/root/reference/proj/core/src/
sieve.cpp:297-303), so rank r of N evaluates the contiguous point range
``point_range(P, r, N)`` over the full graph it holds, and the per-vertex
partial accumulators are combined once per evaluation by an exclusive-or.
NCCL has no XOR reduction: the combine is an all-gather followed by the
engine's XOR kernel (on CUDA tensors) or torch.bitwise_xor (CPU / gloo).
There is no other data-path communication.
"""
from __future__ import annotations


def point_range(P: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous share [begin, end) of P sieve points for `rank` of `world`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return rank * P // world, (rank + 1) * P // world


def work_units(reps: int, P: int, rank: int, world: int) -> list[tuple[int, int, int]]:
    """Share of one decide over `reps` repetitions x P sieve points.

    The (repetition, point) units are split into contiguous ranges, so a rank
    keeps whole repetitions while world <= reps (every batch stays as wide as
    a single-GPU run) and splits a repetition's points only beyond that.
    Returns [(rep, p_begin, p_end), ...]."""
    u0, u1 = point_range(reps * P, rank, world)
    out = []
    for r in range(u0 // P, (u1 + P - 1) // P if u1 > u0 else u0 // P):
        a, b = max(u0, r * P) - r * P, min(u1, (r + 1) * P) - r * P
        if a < b:
            out.append((r, a, b))
    return out


def plan_units(reps: int, P: int, k: int, rank: int, world: int) -> list[tuple[int, int, int]]:
    """Work of `rank` for one decide, choosing between the two engines.

    A unit covering all P points of a repetition runs the coefficient engine
    (DESIGN.md 2b), which costs about as much as the point engine on P / r
    points, r ~ 4 at k = 6 (C2: 0.71 vs 2.87 ms per evaluation) and ~1.3 at
    k = 5 (C5, whose point engine multiplies by y tables).  Fixing some of the
    k variables per rank does not shrink the coefficient form, so when there
    are more ranks than repetitions and a rank's point share would still be
    >= P / 4 (k >= 6), the repetitions stay whole on ranks 0..reps-1 and the
    other ranks idle; otherwise the points are split (work_units)."""
    if k >= 6 and world > reps and reps * P >= world * (P // 4):
        return [(rank, 0, P)] if rank < reps else []
    return work_units(reps, P, rank, world)


def xor_allreduce(t, group=None, out=None):
    """XOR-combine an int64 tensor across ranks; every rank receives the result.

    CUDA tensors: NCCL all-gather into one buffer + tsv_xor_combine_device;
    CPU tensors (gloo): all_gather + torch.bitwise_xor."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return t if out is None else out.copy_(t)
    if t.is_cuda:
        from .sieve import xor_combine_device
        gathered = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(gathered.view(-1), t.contiguous().view(-1), group=group)
        res = out if out is not None else torch.empty_like(t)
        xor_combine_device(gathered.data_ptr(), world, t.numel(), res.data_ptr(),
                           torch.cuda.current_stream(t.device).cuda_stream)
        return res
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous(), group=group)
    res = parts[0].clone()
    for p in parts[1:]:
        torch.bitwise_xor(res, p, out=res)
    if out is not None:
        out.copy_(res)
        return out
    return res
