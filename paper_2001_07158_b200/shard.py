"""Sieve-point sharding across GPUs.

The 2^k sieve points of one evaluation are independent and the
accumulators are XOR sums over points (/root/reference/proj/core/src/
sieve.cpp:297-303), so rank r of N evaluates the contiguous point range
``point_range(P, r, N)`` over the full graph it holds, and the per-vertex
partial accumulators are combined once per evaluation by an exclusive-or.
NCCL has no XOR reduction: the combine is a reduce-scatter built from an
all-to-all, the engine's XOR kernel (CUDA tensors; torch.bitwise_xor on
CPU / gloo) and an all-gather (xor_allreduce).  There is no other data-path
communication.
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


def _xor_parts(parts, out):
    """out = XOR of the rows of parts ([N, L]); CUDA: tsv_xor_combine_device."""
    import torch
    if parts.is_cuda:
        from .sieve import xor_combine_device
        xor_combine_device(parts.data_ptr(), parts.shape[0], parts.shape[1], out.data_ptr(),
                           torch.cuda.current_stream(parts.device).cuda_stream)
        return out
    out.copy_(parts[0])
    for i in range(1, parts.shape[0]):
        torch.bitwise_xor(out, parts[i], out=out)
    return out


def xor_allreduce(t, group=None, out=None):
    """XOR-combine an int64 tensor across ranks; every rank receives the result.

    NCCL (and gloo) have no XOR reduction, so this is a reduce-scatter /
    all-gather built from primitives: the flattened tensor is cut into
    `world` slices, an all-to-all sends slice j of every rank to rank j,
    rank j XORs the `world` copies of its slice (tsv_xor_combine_device on
    the device), and an all-gather returns the combined slices.  Each rank
    moves 2 (world-1)/world of the tensor (an all-gather of whole tensors
    moves world-1 of it and needs world copies in memory)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return t if out is None else out.copy_(t)
    flat = t.contiguous().view(-1)
    L = flat.numel()
    sl = (L + world - 1) // world
    if sl * world != L:
        src = torch.zeros(sl * world, dtype=flat.dtype, device=flat.device)
        src[:L] = flat
    else:
        src = flat
    recv = torch.empty(world, sl, dtype=flat.dtype, device=flat.device)
    dist.all_to_all_single(recv.view(-1), src, group=group)
    mine = torch.empty(sl, dtype=flat.dtype, device=flat.device)
    _xor_parts(recv, mine)
    full = torch.empty(world * sl, dtype=flat.dtype, device=flat.device)
    if flat.is_cuda:
        dist.all_gather_into_tensor(full, mine, group=group)
    else:
        dist.all_gather(list(full.view(world, sl).unbind(0)), mine, group=group)
    res = full[:L].view(t.shape)
    if out is not None:
        out.copy_(res)
        return out
    return res


def vertex_partitioned_eval(level_fn, k, ranges, prev, cur, acc, group=None, exchange=None):
    """One evaluation split by HEAD VERTEX across the ranks:
    the multi-GPU form of the coefficient engine.

    Rank r owns the heads [n r/N, n (r+1)/N).  Level l of the sieve needs
    the level l-1 state rows of every tail, so after each level the ranks'
    rows are made visible to all: `ranges(l)` gives, per rank, the element
    range of `cur` holding its level-l rows (contiguous: state rows are in
    vertex-major run order), and every range is broadcast from its owner
    (an all-gather, in place, into the full-size buffers every rank holds).
    `level_fn(l, prev, cur, acc)` computes this rank's share of level l;
    at l = k it XORs its vertices' readout into acc, which the ranks
    XOR-combine at the end (each vertex's word comes from its owner).
    `exchange(level, cur)`, when given, replaces the all-gather (the targeted
    exchange of eval_vertex_partitioned_device)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    for level in range(2, k + 1):
        level_fn(level, prev, cur, acc)
        if level < k and world > 1 and exchange is not None:
            exchange(level, cur)
        elif level < k and world > 1:
            works = []
            for q, (lo, hi) in enumerate(ranges(level)):
                if hi > lo:
                    src = dist.get_global_rank(group, q) if group is not None else q
                    works.append(dist.broadcast(cur[lo:hi], src=src, group=group, async_op=True))
            for w in works:
                w.wait()
        prev, cur = cur, prev
    return xor_allreduce(acc, group) if world > 1 else acc


class PeerStateBuffers:
    """The two state buffers of a vertex-partitioned evaluation in symmetric
    memory (torch.distributed._symmetric_memory): every rank's buffer is
    mapped on every GPU of the NVLink domain.  Built once per (graph size,
    group) -- the allocation and the handle exchange are collective -- and
    reused by every evaluation."""

    def __init__(self, words, device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        grp = group if group is not None else dist.group.WORLD
        self.bufs = [symm.empty(int(words), dtype=torch.int64, device=device) for _ in range(2)]
        self.hdls = [symm.rendezvous(b, grp) for b in self.bufs]


def eval_vertex_partitioned_peer(g, ds, k, max_ts, cfg, anchor_source, acc, rank, world,
                                 group=None, stream=None, peer_bufs=None):
    """The vertex-partitioned evaluation with the row exchange INSIDE the
    level kernel (tsv_eval_vertex_level_peer): the two state buffers live in
    symmetric memory (PeerStateBuffers), a rank stores each row it forms
    into its own buffer and into the buffers of the ranks whose arcs read
    it, and the only step between levels is a barrier -- which also guards
    the ping-pong: level l+1 overwrites, on the peers too, the buffer level l
    read.  No pack / all-to-all / unpack, and the transfer overlaps the
    level's products row by row.  Checked on one GPU by
    eval_vertex_simulated_peer (tests); opt-in for N > 1 (bench.py
    --exchange peer): the pool had no multi-GPU box to run it on."""
    import torch
    from .sieve import eval_vertex_level, vertex_partition
    parts = [vertex_partition(g, ds, k, q, world) for q in range(world)]
    if not all(p.applicable for p in parts):
        raise ValueError("vertex partition not applicable")
    if world > 8:
        raise ValueError("peer stores take at most 8 ranks (one NVLink domain)")
    st = stream or torch.cuda.current_stream(acc.device)
    with torch.cuda.stream(st):
        if peer_bufs is None:
            peer_bufs = PeerStateBuffers(parts[0].state_words, acc.device, group)
        bufs, hdls = peer_bufs.bufs, peer_bufs.hdls
        hdls[0].barrier()   # the previous evaluation's readers are done with both buffers
        cur_i = 1
        for level in range(2, k + 1):
            prev, cur = bufs[1 - cur_i], bufs[cur_i]
            peers = [int(p) for p in hdls[cur_i].buffer_ptrs] if level < k else None
            eval_vertex_level(g, ds, k, level, max_ts, cfg, anchor_source, rank, world,
                              prev.data_ptr(), cur.data_ptr(), acc.data_ptr(), st.cuda_stream,
                              peer_cur=peers)
            if level < k:
                hdls[cur_i].barrier()   # every rank's level-l rows are in place everywhere
            cur_i = 1 - cur_i
    return xor_allreduce(acc, group) if world > 1 else acc


def eval_vertex_partitioned_device(g, ds, k, max_ts, cfg, anchor_source, acc, rank, world,
                                   group=None, bufs=None, stream=None, targeted=True):
    """vertex_partitioned_eval with the device engine (tsv_eval_vertex_level)
    on this rank's GPU; acc: int64 CUDA tensor of n words (XORed into).

    targeted=True: between levels each rank sends a peer only the rows some
    arc of that peer reads (tsv_vertex_exchange_pack -> all_to_all_single ->
    tsv_vertex_exchange_unpack; at C5 ~1.5 readers per row, so ~1.5/(N-1)
    of the all-gather's bytes); else the all-gather of row ranges."""
    import torch
    import torch.distributed as dist
    from .sieve import (eval_vertex_level, vertex_exchange_move, vertex_exchange_plan,
                        vertex_partition)
    parts = [vertex_partition(g, ds, k, q, world) for q in range(world)]
    if not all(p.applicable for p in parts):
        raise ValueError("vertex partition not applicable")
    words = parts[0].state_words
    if bufs is None:
        bufs = (torch.empty(words, dtype=torch.int64, device=acc.device),
                torch.empty(words, dtype=torch.int64, device=acc.device))
    sp = (stream or torch.cuda.current_stream(acc.device)).cuda_stream

    def level_fn(level, prev, cur, a):
        eval_vertex_level(g, ds, k, level, max_ts, cfg, anchor_source, rank, world,
                          prev.data_ptr(), cur.data_ptr(), a.data_ptr(), sp)

    def ranges(level):
        rw = parts[0].row_words[level]
        return [(p.slot_lo * rw, p.slot_hi * rw) for p in parts]

    exchange = None
    if targeted and world > 1:
        plan = vertex_exchange_plan(g, ds, k, rank, world)
        fmax = max(parts[0].row_words[lv] for lv in range(2, k))
        sbuf = torch.empty(max(plan.send_total * fmax, 1), dtype=torch.int64, device=acc.device)
        rbuf = torch.empty(max(plan.recv_total * fmax, 1), dtype=torch.int64, device=acc.device)

        def exchange(level, cur):
            F = parts[0].row_words[level]
            vertex_exchange_move(g, rank, world, F, cur.data_ptr(), sbuf.data_ptr(), True, sp)
            dist.all_to_all_single(rbuf[:plan.recv_total * F], sbuf[:plan.send_total * F],
                                   output_split_sizes=[plan.recv_rows[q] * F for q in range(world)],
                                   input_split_sizes=[plan.send_rows[q] * F for q in range(world)],
                                   group=group)
            vertex_exchange_move(g, rank, world, F, rbuf.data_ptr(), cur.data_ptr(), False, sp)

    return vertex_partitioned_eval(level_fn, k, ranges, bufs[0], bufs[1], acc, group, exchange)


def eval_vertex_simulated(g, ds, k, max_ts, cfg, anchor_source, acc, world, bufs=None,
                          timed=False, peer_store=False):
    """The `world`-rank vertex-partitioned evaluation run on ONE device: at
    every level the ranks' shares run one after the other on the same
    full-size buffers, so the all-gather between levels is the identity.
    Returns acc and, with timed=True, the CUDA-event time of every
    (level, rank) share in ms -- the per-rank compute of an N-GPU run
    (bench.py --simulate-world).  peer_store=True runs the peer-store kernel
    with the shared buffer standing in for every peer's: each row is stored
    again once per reading rank (same value, same address), which times the
    kernel's share WITH its exchange stores issued."""
    import torch
    from .sieve import eval_vertex_level, vertex_partition
    parts = [vertex_partition(g, ds, k, q, world) for q in range(world)]
    if not all(p.applicable for p in parts):
        raise ValueError("vertex partition not applicable")
    words = parts[0].state_words
    if bufs is None:
        bufs = (torch.empty(words, dtype=torch.int64, device=acc.device),
                torch.empty(words, dtype=torch.int64, device=acc.device))
    st = torch.cuda.current_stream(acc.device)
    prev, cur = bufs
    times = {}
    for level in range(2, k + 1):
        for q in range(world):
            if timed:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
            peers = [cur.data_ptr()] * world if peer_store and level < k and world > 1 else None
            eval_vertex_level(g, ds, k, level, max_ts, cfg, anchor_source, q, world,
                              prev.data_ptr(), cur.data_ptr(), acc.data_ptr(), st.cuda_stream,
                              peer_cur=peers)
            if timed:
                e1.record(st)
                times[(level, q)] = (e0, e1)
        prev, cur = cur, prev
    if timed:
        torch.cuda.synchronize(acc.device)
        times = {key: a.elapsed_time(b) for key, (a, b) in times.items()}
    return acc, times, parts


def eval_vertex_simulated_peer(g, ds, k, max_ts, cfg, anchor_source, n, world, timed=False):
    """Test form of the peer-store levels on ONE device: every simulated rank
    has its own zeroed state buffers; at a level the ranks run one after the
    other, each storing its rows into its own buffer and -- through the
    kernel's reader bytes -- into the buffers of the ranks that read them
    (the other ranks' buffers stand in for NVLink peer mappings).  A row a
    reader does not receive stays zero, so equality with the single-GPU
    result checks the masks and the stores.  timed=True also returns the
    CUDA-event time of every (level, rank) share, peer stores included."""
    import torch
    from .sieve import eval_vertex_level, vertex_partition
    parts = [vertex_partition(g, ds, k, q, world) for q in range(world)]
    words = parts[0].state_words
    stream = torch.cuda.current_stream()
    st = stream.cuda_stream
    bufs = [[torch.zeros(words, dtype=torch.int64, device="cuda") for _ in range(2)]
            for _ in range(world)]
    accs = [torch.zeros(n, dtype=torch.int64, device="cuda") for _ in range(world)]
    cur_i = 1
    times = {}
    for level in range(2, k + 1):
        peers = [bufs[r][cur_i].data_ptr() for r in range(world)] if level < k else None
        for q in range(world):
            if timed:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            eval_vertex_level(g, ds, k, level, max_ts, cfg, anchor_source, q, world,
                              bufs[q][1 - cur_i].data_ptr(), bufs[q][cur_i].data_ptr(),
                              accs[q].data_ptr(), st, peer_cur=peers)
            if timed:
                e1.record(stream)
                times[(level, q)] = (e0, e1)
        cur_i = 1 - cur_i
    out = accs[0]
    for a in accs[1:]:
        torch.bitwise_xor(out, a, out=out)
    if timed:
        torch.cuda.synchronize()
        return out, {key: a.elapsed_time(b) for key, (a, b) in times.items()}
    return out


def eval_vertex_simulated_private(g, ds, k, max_ts, cfg, anchor_source, n, world):
    """Test form of the targeted exchange on ONE device: every simulated rank
    has its own full-size state buffers and accumulators, computes only its
    vertices' rows, and receives only the rows its exchange lists name (the
    all-to-all done as copies between the ranks' packed buffers).  A row
    missing from the lists leaves a zero where a reader needs it, so equality
    with the single-GPU result checks the lists."""
    import torch
    from .sieve import (eval_vertex_level, vertex_exchange_move, vertex_exchange_plan,
                        vertex_partition)
    parts = [vertex_partition(g, ds, k, q, world) for q in range(world)]
    plans = [vertex_exchange_plan(g, ds, k, q, world) for q in range(world)]
    words = parts[0].state_words
    st = torch.cuda.current_stream().cuda_stream
    bufs = [[torch.zeros(words, dtype=torch.int64, device="cuda") for _ in range(2)]
            for _ in range(world)]
    accs = [torch.zeros(n, dtype=torch.int64, device="cuda") for _ in range(world)]
    cur_i = 1
    for level in range(2, k + 1):
        for q in range(world):
            eval_vertex_level(g, ds, k, level, max_ts, cfg, anchor_source, q, world,
                              bufs[q][1 - cur_i].data_ptr(), bufs[q][cur_i].data_ptr(),
                              accs[q].data_ptr(), st)
        if level < k and world > 1:
            F = parts[0].row_words[level]
            sends = []
            for q in range(world):
                sb = torch.zeros(max(plans[q].send_total * F, 1), dtype=torch.int64, device="cuda")
                vertex_exchange_move(g, q, world, F, bufs[q][cur_i].data_ptr(), sb.data_ptr(),
                                     True, st)
                sends.append(sb)
            for q in range(world):   # q receives from every r: r's segment for q
                segs = []
                for r in range(world):
                    off = sum(plans[r].send_rows[p] for p in range(q)) * F
                    segs.append(sends[r][off:off + plans[r].send_rows[q] * F])
                    assert plans[r].send_rows[q] == plans[q].recv_rows[r]
                rb = torch.cat(segs) if segs else torch.zeros(1, dtype=torch.int64, device="cuda")
                if rb.numel():
                    vertex_exchange_move(g, q, world, F, rb.data_ptr(), bufs[q][cur_i].data_ptr(),
                                         False, st)
        cur_i = 1 - cur_i
    out = accs[0]
    for a in accs[1:]:
        torch.bitwise_xor(out, a, out=out)
    return out
