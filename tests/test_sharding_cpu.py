"""Multi-rank sieve-point sharding on CPU (gloo, world_size 2): every rank
evaluates its contiguous share of the sieve points (CPU oracle standing in
for the device), the partial accumulators are XOR-combined with
shard.xor_allreduce, and the result equals the single-process evaluation
and the reference's golden accumulators."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2001_07158_b200.shard import point_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2001_07158_b200 import sieve as S
        from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
        from paper_2001_07158_b200.shard import xor_allreduce
        c = case
        cu, cv, ct = O.canonical_edges(c["n"], c["u"], c["v"], c["ts"], c["directed"])
        sh = S.build_shades(MotifQuery.from_multiset(c["motif"]),
                            VertexColoring(c["colors"], max(c["colors"])),
                            S.SieveConfig(seed=c["seed"]))
        k = len(c["motif"])
        p0, p1 = point_range(1 << k, rank, world)
        t = c["t"] or int(ct.max())
        part = O.eval_points(c["n"], cu, cv, ct, c["directed"], k, c["max_ts"] or t,
                             sh.vertex_off, sh.vertex_shades, c["seed"], c["anchor"][0], p0, p1)
        acc = xor_allreduce(torch.from_numpy(part.view(np.int64).copy()))
        if rank == 0:
            q.put(acc.numpy().view(np.uint64).tolist())
    finally:
        dist.barrier()
        dist.destroy_process_group()


def test_work_units_cover_every_rep_point_once():
    from paper_2001_07158_b200.shard import work_units
    for reps, P in ((4, 64), (1, 32), (3, 8), (1, 4096)):
        for world in (1, 2, 3, 4, 8):
            seen = {}
            for r in range(world):
                for rep, a, b in work_units(reps, P, r, world):
                    assert 0 <= a < b <= P
                    for p in range(a, b):
                        assert (rep, p) not in seen
                        seen[(rep, p)] = r
            assert len(seen) == reps * P
    # C2 (4 reps x 64 points): up to 4 GPUs every rank keeps whole 64-point reps
    assert work_units(4, 64, 1, 4) == [(1, 0, 64)]
    assert work_units(4, 64, 5, 8) == [(2, 32, 64)]


def test_plan_units_keeps_coefficient_reps_whole():
    from paper_2001_07158_b200.shard import plan_units
    for reps, P, k in ((4, 64, 6), (1, 32, 5), (1, 256, 8), (1, 4096, 12), (3, 64, 6)):
        for world in (1, 2, 4, 8):
            seen = set()
            for r in range(world):
                for rep, a, b in plan_units(reps, P, k, r, world):
                    for p in range(a, b):
                        assert (rep, p) not in seen
                        seen.add((rep, p))
            assert len(seen) == reps * P
    # C2 at 8 GPUs: four whole repetitions, four idle ranks
    assert plan_units(4, 64, 6, 3, 8) == [(3, 0, 64)]
    assert plan_units(4, 64, 6, 5, 8) == []
    # C5 (k = 5, one repetition): points split over the ranks
    assert plan_units(1, 32, 5, 1, 2) == [(0, 16, 32)]


def test_point_ranges_partition():
    for P in (2, 32, 64, 4096):
        for world in (1, 2, 3, 4, 8):
            rs = [point_range(P, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == P
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    with pytest.raises(ValueError):
        point_range(8, 2, 2)


@pytest.mark.parametrize("name", ["C1 k-TempPath k=5", "fig2 pathmotif {1,1,2,3}", "random 7"])
def test_two_rank_gloo_sharding_reproduces_golden(golden, name):
    case = next(c for c in golden["sieve"] if c["name"] == name)
    if not case["feasible"]:
        pytest.skip("infeasible case")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    acc = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    from oracle import oracle as O
    acc_fin, nflag, cs = O.finalize(np.array(acc, np.uint64), case["anchor"][1])
    assert f"{cs:016x}" == case["checksum"]
    if "acc" in case:
        assert [f"{int(x):016x}" for x in acc_fin] == case["acc"]


def _xor_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2001_07158_b200.shard import xor_allreduce
        rng = np.random.default_rng(1000 + rank)
        part = rng.integers(-2**63, 2**63 - 1, size=(3, n), dtype=np.int64)
        res = xor_allreduce(torch.from_numpy(part))
        out = torch.zeros(3, n, dtype=torch.int64)
        xor_allreduce(torch.from_numpy(part), out=out)
        q.put((rank, res.numpy().tolist(), out.numpy().tolist()))
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1), (2, 1001), (4, 7), (4, 4096), (3, 10)])
def test_xor_reduce_scatter_combine(world, n):
    """shard.xor_allreduce (all-to-all of slices + XOR + all-gather) returns
    on EVERY rank the XOR of all ranks' tensors, for sizes that do not split
    evenly and tensors smaller than the world."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xor_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    want = np.zeros((3, n), np.int64)
    for r in range(world):
        want ^= np.random.default_rng(1000 + r).integers(-2**63, 2**63 - 1, size=(3, n),
                                                         dtype=np.int64)
    for rank, res, out in got:
        assert np.array_equal(np.array(res, np.int64), want), rank
        assert np.array_equal(np.array(out, np.int64), want), rank


def _vertex_worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2001_07158_b200 import sieve as S
        from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
        from paper_2001_07158_b200.shard import vertex_partitioned_eval
        c = case
        n = c["n"]
        cu, cv, ct = O.canonical_edges(n, c["u"], c["v"], c["ts"], c["directed"])
        sh = S.build_shades(MotifQuery.from_multiset(c["motif"]),
                            VertexColoring(c["colors"], max(c["colors"])),
                            S.SieveConfig(seed=c["seed"]))
        k = len(c["motif"])
        t = c["t"] or int(ct.max())
        G = O.BigGraph(n, cu, cv, ct, c["directed"], c["max_ts"] or t)
        P = 1 << k
        W = min(P, 16)
        total = np.zeros(n, np.uint64)
        bounds = [(n * r // world, n * (r + 1) // world) for r in range(world)]
        runs = [G.run_range(a, b) for a, b in bounds]
        for base in range(0, P, W):      # the oracle stands in for the device, W points a pass
            prev = torch.zeros(max(G.runs, 1) * W, dtype=torch.int64)
            cur = torch.zeros_like(prev)
            acc = torch.zeros(n, dtype=torch.int64)
            v_lo, v_hi = bounds[rank]

            def level_fn(ell, pv, cr, a):
                G.level(k, ell, sh.vertex_off, sh.vertex_shades, c["seed"], c["anchor"][0],
                        base, W, v_lo, v_hi, pv.numpy().view(np.uint64),
                        cr.numpy().view(np.uint64), a.numpy().view(np.uint64))

            res = vertex_partitioned_eval(level_fn, k, lambda ell: [(a * W, b * W) for a, b in runs],
                                          prev, cur, acc)
            total ^= res.numpy().view(np.uint64)
        if rank == 0:
            q.put(total.tolist())
    finally:
        dist.barrier()
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("name", ["C1 k-TempPath k=5", "fig2 pathmotif {1,1,2,3}", "random 7"])
def test_vertex_partitioned_gloo_reproduces_golden(golden, name, world):
    """The multi-GPU algorithm of the coefficient engine (shard.vertex_partitioned_eval):
    each rank computes the levels of its head-vertex range, the ranks'
    state rows are all-gathered after every level, the readouts are
    XOR-combined -- with the oracle's per-level form (tsvo_big_level)
    standing in for the device kernel, on gloo; equals the reference's golden
    accumulators."""
    case = next(c for c in golden["sieve"] if c["name"] == name)
    if not case["feasible"] or len(case["motif"]) < 2:
        pytest.skip("infeasible or k < 2")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vertex_worker, args=(r, world, port, case, q))
             for r in range(world)]
    for p in procs:
        p.start()
    acc = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    from oracle import oracle as O
    acc_fin, nflag, cs = O.finalize(np.array(acc, np.uint64), case["anchor"][1])
    assert f"{cs:016x}" == case["checksum"]
    if "acc" in case:
        assert [f"{int(x):016x}" for x in acc_fin] == case["acc"]
