"""Benchmark of the temporal-sieve hot path on B200 (contract: see DESIGN.md).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one DECIDE of the configured BASELINE workload: every repetition
seed evaluates all 2^k_eff sieve points over the whole synthetic graph
(default config 2 = BASELINE configs[1]: PathMotif k=6, n=1e5, m=1e6,
4 repetitions).  Metric: GF(2^64) edge x level x sieve-point updates per
second, updates = A * (k_eff - 1) * 2^k_eff per repetition.

With N > 1 (torchrun) the (repetition, sieve point) units of the decide are
split into contiguous ranges (shard.work_units: whole repetitions while
N <= reps, halves of one beyond), with no data-path collective; the
per-vertex partial accumulators are XOR-combined once per step (NCCL
all-gather + XOR kernel; NCCL has no XOR reduction).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REPS = {1: 1, 2: 4, 3: 1, 4: 1, 5: 1}
BYTES_PER_UPDATE = 16  # 8 B predecessor-state read + 8 B state write


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled during the timed
    region, in-process through NVML (nvidia_ml_py) every 5 ms.  NVML is
    initialised when the sampler is created (before the warm-up): starting an
    `nvidia-smi` process inside the timed region stalled the GPU submissions
    of this process by up to 0.6 s (runs of 2.4 vs 14.6 ms per step).
    Falls back to `nvidia-smi -lms 100` when NVML is unavailable."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples = []          # (sm_mhz, max_mhz, [reason names])
        self.stop = threading.Event()
        self.proc = None
        self.nv = None
        if os.environ.get("BENCH_NO_CLOCKS"):   # (diagnosis only: no sampling)
            return
        try:
            import pynvml as nv
            nv.nvmlInit()
            try:
                import torch
                phys = torch.cuda._get_nvml_device_index(index)
            except Exception:
                phys = index
            self.h = nv.nvmlDeviceGetHandleByIndex(phys)
            self.bits = [nv.nvmlClocksEventReasonHwSlowdown,
                         nv.nvmlClocksEventReasonHwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwThermalSlowdown,
                         nv.nvmlClocksEventReasonSwPowerCap]
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM))
            self.nv = nv
        except Exception:
            self.nv = None

    def _sample_nvml(self):
        nv = self.nv
        sm = float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
        try:
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((sm, self.max_mhz,
                             [n for n, b in zip(self.NAMES, self.bits) if r & b]))

    def __enter__(self):
        self.stop.clear()
        if self.nv is not None:
            def poll():
                while True:
                    self._sample_nvml()
                    if self.stop.wait(0.005):
                        break
            self.th = threading.Thread(target=poll, daemon=True)
            self.th.start()
            return self
        if shutil.which("nvidia-smi") is None or os.environ.get("BENCH_NO_CLOCKS"):
            return self
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        self.proc = subprocess.Popen(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
             "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)

        def reader():
            for line in self.proc.stdout:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) == 6 and parts[0].replace(".", "").isdigit():
                    self.samples.append((float(parts[0]), float(parts[1]),
                                         [self.NAMES[i] for i in range(4)
                                          if parts[2 + i].lower().startswith("active")]))
        self.th = threading.Thread(target=reader, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.nv is not None:
            self.th.join(timeout=5)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted({n for s in self.samples for n in s[2]}),
                "samples": len(self.samples),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local




# ------------------------------------------------------------------ CPU legs


def cpu_sample(inst, k, colors, motif, anchor, seed=1, frac=0.1, threads=None):
    """The reference's own eval_temporal_sieve (oracle/_ref) on a bounded
    sample of the workload: the time prefix ts <= frac * t of the same graph
    (all 2^k points, all levels).  Returns (updates/s, seconds, sample, kind, cores)."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    max_ts = max(1, int(inst.t * frac))
    arcs = int(np.count_nonzero(inst.ts <= max_ts)) * (1 if inst.directed else 2)
    upd = arcs * (k - 1) * (1 << k)
    sample = (f"ts <= {max_ts} of t={inst.t} ({arcs} arcs, all {1 << k} points, "
              f"{k - 1} levels, seed {seed})")
    # The reference's dense layers (2 n W (max_ts+1) words, sieve.cpp:188-192)
    # only fit for configs 1-2; beyond that the validated sparse restatement
    # (oracle port) stands in, on 2 of the sieve points.
    dense_bytes = 2 * inst.n * 8 * (max_ts + 1) * 8
    if O.ref_available() and dense_bytes < 24e9:
        os.environ.setdefault("OMP_WAIT_POLICY", "active")
        r = O.ref_eval(inst.n, inst.u, inst.v, inst.ts, inst.directed, colors, motif,
                       max_ts=max_ts, seed=seed, lanes=8, threads=threads, anchor=anchor,
                       t=inst.t, repeats=2)
        return upd / r["seconds"], r["seconds"], sample, "reference", threads
    # port: the time-prefix subgraph itself, bounded to ~2e6 arcs
    max_ts = max(1, min(max_ts, int(inst.t * 2e6 / max(arcs / max(frac, 1e-9), 1))))
    sel = inst.ts <= max_ts
    arcs = int(np.count_nonzero(sel)) * (1 if inst.directed else 2)
    cu, cv, ct = O.canonical_edges(inst.n, inst.u[sel], inst.v[sel], inst.ts[sel], inst.directed)
    from paper_2001_07158_b200.sieve import SieveConfig, build_shades
    from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
    sh = build_shades(MotifQuery.from_multiset(motif), VertexColoring(colors, int(colors.max())),
                      SieveConfig(seed=seed))
    npts = min(2, 1 << k)
    upd = arcs * (k - 1) * npts
    sample = (f"ts <= {max_ts} of t={inst.t} ({arcs} arcs, sieve points 0..{npts - 1}, "
              f"{k - 1} levels, seed {seed}; sparse oracle port)")
    t0 = time.perf_counter()
    O.eval_points(inst.n, cu, cv, ct, inst.directed, k, max_ts, sh.vertex_off, sh.vertex_shades,
                  seed, anchor[0], 0, npts)
    s = time.perf_counter() - t0
    return upd / s, s, sample, "port", 1


def run_reference(args, rank, world):
    """--impl reference: the reference CPU implementation on the host cores."""
    if rank != 0:
        return
    from paper_2001_07158_b200 import synth
    inst = synth.make_config(args.config, scale=args.scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    times, rates = [], []
    info = None
    for i in range(args.warmup + args.steps):
        rate, sec, sample, kind, cores = cpu_sample(inst, k, colors, motif, anchor,
                                                    frac=args.ref_frac)
        info = (sample, kind, cores)
        if i >= args.warmup:
            times.append(sec)
            rates.append(rate)
    value = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": config_json(inst, world, args, cpu=True),
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": info[2],
                             "kind": info[1], "sample": info[0]},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "GF(2^64) edge x level x sieve-pt updates/s (decide)"


def config_json(inst, world, args, cpu=False):
    k_eff = inst.k_eff
    l2 = ("host arm: the reference's CPU code, no device cache involved" if cpu else
          "flushed before every step: a 256 MB buffer (2x the 126 MB L2) is "
          "zeroed on the bench stream inside the timed region")
    return {"workload": f"BASELINE configs[{args.config - 1}]: {inst.name}"
                        + ("" if args.scale == 1.0 else f" (scaled x{args.scale})"), "n": inst.n,
            "m": inst.m, "t": inst.t, "directed": inst.directed, "k_eff": k_eff,
            "sieve_points": 1 << k_eff, "repetitions": REPS[args.config],
            "updates_per_step": inst.updates() * REPS[args.config],
            "parallelism": (f"repetitions / sieve points over {world} GPU(s) (shard.plan_units)"
                            if not cpu else
                            "reference CPU code on all host threads (rank 0)"),
            "l2": l2}


# ---------------------------------------------------------------- our arm



def coef_alg_bytes(g, sh, k):
    """Algorithmic bytes of one full evaluation by the coefficient engine, per
    kernel family ("Roofline"), from the graph and the
    shade classes: a vertex with no shade is dead, one shade d keeps the
    (l-1)-subsets without d (frame C(k-1, l-1)), several shades keep all
    C(k, l-1).
      coef_arcs, middle levels 3 <= l < k: 8 B per (live arc with a
        predecessor run, entry it carries) read -- C(k-2, l-2) for single ->
        single shades d_t != d_h, C(k-1, l-2) single -> multi, C(k-1, l-1)
        multi -> single, C(k, l-1) multi -> multi -- plus 8 B per (referenced
        run of a live head, frame entry) written, plus 12 B per arc and 4 B
        per run of the shaded subgraph (graph metadata);
      coef_ztrans, levels 2 <= l < k: 8 B per (referenced run of a
        multi-shade head, C(k, l-1) entry) read + C(k, l) written."""
    from math import comb
    n = g.n()
    cu, cv, ct = (np.asarray(x, dtype=np.int64) for x in g.edges())
    if not g.directed():
        cu, cv, ct = np.concatenate([cu, cv]), np.concatenate([cv, cu]), np.concatenate([ct, ct])
    cnt = np.diff(np.asarray(sh.vertex_off, dtype=np.int64))
    d1 = np.full(n, -1, np.int64)
    one = cnt == 1
    d1[one] = np.asarray(sh.vertex_shades, dtype=np.int64)[np.asarray(sh.vertex_off)[:-1][one]]
    multi = cnt >= 2
    # predecessor run: the tail has an in-arc with an earlier timestamp
    first_in = np.full(n, np.iinfo(np.int64).max, np.int64)
    np.minimum.at(first_in, cv, ct)
    live = (cnt[cu] > 0) & (cnt[cv] > 0) & (first_in[cu] < ct)
    tu, hv = cu[live], cv[live]
    ss = one[tu] & one[hv] & (d1[tu] != d1[hv])
    sm = one[tu] & multi[hv]
    ms = multi[tu] & one[hv]
    mm = multi[tu] & multi[hv]
    n_ss, n_sm, n_ms, n_mm = (int(x.sum()) for x in (ss, sm, ms, mm))
    # referenced runs (tail, its last in-timestamp < ts) of live heads
    key_in = np.unique(cv * (1 << 32) + ct)          # runs (head, ts), sorted
    q = cu * (1 << 32) + ct                           # an arc's source lies before (tail, ts)
    pos = np.searchsorted(key_in, q, side="left") - 1
    ok = (pos >= 0) & (cnt[cu] > 0)
    src = key_in[np.clip(pos, 0, None)]
    ok &= (src >> 32) == cu
    ref = np.unique(src[ok])
    rh = ref >> 32
    r_single, r_multi = int(one[rh].sum()), int(multi[rh].sum())
    # + the graph itself at every middle level: 12 B per arc (edge id,
    # predecessor slot, tail) and 4 B per run (head) of the shaded subgraph
    # the engine walks (arcs with both endpoints shaded)
    kept = (cnt[cu] > 0) & (cnt[cv] > 0)
    runs_kept = len(np.unique(cv[kept] * (1 << 32) + ct[kept]))
    meta = 12 * int(kept.sum()) + 4 * runs_kept
    arcs = sum(8 * (n_ss * comb(k - 2, l - 2) + n_sm * comb(k - 1, l - 2) +
                    n_ms * comb(k - 1, l - 1) + n_mm * comb(k, l - 1) +
                    r_single * comb(k - 1, l - 1) + r_multi * comb(k, l - 1)) + meta
               for l in range(3, k))
    ztrans = sum(8 * r_multi * (comb(k, l - 1) + comb(k, l)) for l in range(2, k))
    return {"coef_arcs": arcs, "coef_ztrans": ztrans}


def coef_roofline(coef, k, alg1, evals, hbm, peak_kind, args, world, sm_mhz):
    """Roofline of the coefficient engine's dominant kernel.

    alg1 = coef_alg_bytes() of one evaluation; achieved = those bytes x the
    evaluations of the profile pass / the kernel family's CUDA-event time in
    that pass; int_pipe from the committed ncu capture of the same kernel."""
    alg = {nm: evals * b for nm, b in alg1.items()}
    name = max(coef, key=lambda nm: coef[nm][1])
    n_launch, tot_ms = coef[name]
    if not n_launch or not alg[name]:
        return None
    achieved = alg[name] / (tot_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "peak_kind": peak_kind,
            "kernel": {"coef_arcs": "k_coef_items / k_coef_arcs (3 <= l < k)",
                       "coef_ztrans": "k_coef_ztrans_tab (2 <= l < k)"}[name],
            "engine": "coefficient (top-degree) form on the shaded subgraph, DESIGN.md 2b",
            "avg_launch_ms": tot_ms / n_launch,
            "alg_bytes_per_launch": alg[name] / n_launch,
            "kernel_ms_per_eval": {nm: coef[nm][1] / max(evals, 1) for nm in coef}}
    try:
        with open(os.path.join(ROOT, "profiles", f"coef_kernels_c{args.config}.json")) as f:
            prof = json.load(f)
        if prof["config"] != args.config or args.scale != 1.0 or world != 1:
            prof = None
        else:
            prof = dict(prof["kernels"][name], capture=prof["capture"])
    except Exception:
        prof = None
    if prof is not None:
        roof["traffic"] = prof["traffic_bytes_per_launch"]
        clk = sm_mhz or prof["sm_clock_ghz"] * 1e3
        peak_issue = 148 * 4 * clk * 1e6
        ach = prof["warp_inst_per_launch"] / (roof["avg_launch_ms"] * 1e-3)
        roof["int_pipe"] = {"bound": "issue", "unit": "warp-inst/s", "achieved": ach,
                            "peak": peak_issue, "frac": ach / peak_issue,
                            "alu_pipe_frac_ncu": prof["alu_pipe_pct_active"] / 100,
                            "capture": prof["capture"]}
    return roof


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0,
                    help="shrink n and m of the config (not a bench line unless 1.0)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-frac", type=float, default=0.1)
    ap.add_argument("--points-per-batch", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--streams", type=int, default=4,
                    help="concurrent CUDA streams for the repetitions of a step "
                         "(at most one per work unit)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    import paper_2001_07158_b200 as T
    from paper_2001_07158_b200 import _native, synth
    from paper_2001_07158_b200.shard import plan_units, xor_allreduce

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = local
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    inst = synth.make_config(args.config, scale=args.scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    reps = REPS[args.config]
    seeds = [1 + r for r in range(reps)]
    P = 1 << k
    work = plan_units(reps, P, k, rank, world)   # [(rep, p_begin, p_end)]
    my_points = sum(b - a for _, a, b in work)

    g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, dev)
    col = T.VertexColoring(colors, int(colors.max()))
    # the reference's default cap (2^31 words) sizes ITS dense layers; the
    # engine's batch width is bounded by device memory instead
    cfgs = [T.SieveConfig(seed=s, points_per_batch=args.points_per_batch,
                          memory_cap_words=1 << 62) for s in seeds]
    sh = T.build_shades(T.MotifQuery.from_multiset(motif), col, cfgs[0])
    ds = T.DeviceShades(g, k, sh)
    n = g.n()
    acc = torch.zeros((reps, n), dtype=torch.int64, device="cuda")
    total = torch.zeros((reps, n), dtype=torch.int64, device="cuda")

    # repetitions (independent evaluations) may run on concurrent streams so
    # one evaluation's tail wave overlaps the next one's launches
    side = [torch.cuda.Stream() for _ in range(max(1, min(args.streams, len(work))) - 1)]

    # L2 flush between steps (inside the timed region, counted against us):
    # the coefficient engine's working set at C2 (~70 MB per evaluation,
    # ~15 MB of graph) would otherwise partly survive in L2 across steps
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(concurrent=True):
        l2_flush.zero_()
        acc.zero_()
        if not side or not concurrent:
            for r, a, b in work:
                T.eval_points_device(g, ds, k, g.t(), cfgs[r], anchor[0], a, b,
                                     acc[r].data_ptr(), sp)
        else:
            lanes = [stream] + side
            for s in side:
                s.wait_stream(stream)
            for i, (r, a, b) in enumerate(work):
                T.eval_points_device(g, ds, k, g.t(), cfgs[r], anchor[0], a, b,
                                     acc[r].data_ptr(), lanes[i % len(lanes)].cuda_stream)
            for s in side:
                stream.wait_stream(s)
        if world > 1:
            return xor_allreduce(acc, out=total)
        return acc

    clk = ClockSampler(dev)   # NVML initialised outside the timed region
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _native.Profile.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clk:
        e0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            res = step()
        host_ms = (time.perf_counter() - h0) * 1e3 / args.steps   # enqueue time per step
        e1.record(stream)
        torch.cuda.synchronize()
    launches = _native.Profile.launches() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    # Per-kernel CUDA-event timing (roofline) from a separate single-stream
    # pass after the timed region: with concurrent streams a launch's events
    # would also cover the other stream's kernels.
    prof_steps = max(1, min(args.steps, 3))
    _native.Profile.reset()
    _native.Profile.enable(True)
    for _ in range(prof_steps):
        step(concurrent=False)
    torch.cuda.synchronize()
    lvl_n, lvl_ms = _native.Profile.get("level")
    last_n, _ = _native.Profile.get("level_last")
    grouped = False
    if not lvl_n:  # W < 32: the grouped kernel
        lvl_n, lvl_ms = _native.Profile.get("level_grouped")
        grouped = bool(lvl_n)
    coef = {nm: _native.Profile.get(nm) for nm in ("coef_arcs", "coef_ztrans")}
    all_n, all_ms = _native.Profile.get(None)
    _native.Profile.enable(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    upd_step = inst.updates() * reps
    value = upd_step / (ms * 1e-3)

    # decision / checksum of the last step (finalize on the host)
    host = res.cpu().numpy().view(np.uint64)
    sink = anchor[1]
    decisions, checksums = [], []
    for r in range(reps):
        a, nflag, cs = T.finalize(host[r], sink)
        decisions.append(bool(nflag))
        checksums.append(f"{cs:016x}")

    # roofline of the dominant kernel
    hbm, peak_kind = peaks()
    roof = None
    # full-range evaluations in the profile pass (the coefficient engine's)
    evals = sum(1 for _, a, b in work if a == 0 and b == P) * prof_steps
    if any(c for c, _ in coef.values()):
        roof = coef_roofline(coef, k, coef_alg_bytes(g, sh, k), evals, hbm, peak_kind, args, world,
                             clk.summary().get("sm_mhz"))
    elif lvl_n:
        # updates executed by the middle-level launches (3 <= l < k when level
        # k is fused with the readout, else 3 <= l <= k) of this rank in the
        # timed region
        # algorithmic bytes: 16 B per (arc, point) update --
        # one 8-B predecessor-state read plus one 8-B state write -- times the
        # updates of one middle-level launch.  The engine moves less (no state
        # for runs no arc reads, no read for arcs without a predecessor): that
        # shows as ncu `traffic` below the algorithmic figure.
        mid_levels = (k - 2) - (1 if last_n else 0)
        upd_launch = g.info.arcs * mid_levels * my_points * prof_steps / lvl_n
        alg_bytes = BYTES_PER_UPDATE * upd_launch
        avg_ms = lvl_ms / lvl_n
        achieved = alg_bytes / (avg_ms * 1e-3) / 1e9
        # per-launch DRAM traffic and instruction counts of the same kernel on
        # the same workload, from the committed ncu capture (tools/ncu_level_json.py)
        traffic, prof = None, None
        try:
            with open(os.path.join(ROOT, "profiles", f"level_kernel_c{args.config}.json")) as f:
                prof = json.load(f)
            if prof["config"] != args.config or args.scale != 1.0 or world != 1 or grouped:
                prof = None
            else:
                traffic = prof["traffic_bytes_per_launch"]
        except Exception:
            prof = None
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
                "kernel": ("k_level (grouped, W < 32, 3 <= l < k)" if grouped
                           else "k_level_wide (3 <= l < k)"), "avg_launch_ms": avg_ms,
                "launch_share_of_step": lvl_ms / max(all_ms, 1e-9),
                "alg_bytes_per_launch": alg_bytes}
        # The kernel is integer-pipe bound (GF(2^64) carry-less products), so
        # the binding roofline is instruction issue: 4 warp-instructions per
        # clock per SM.  achieved = the capture's executed warp-instructions
        # per launch / this run's launch time; ALU-pipe utilization is the
        # capture's own counter.
        if prof is not None:
            sm_mhz = clk.summary().get("sm_mhz") or prof["sm_clock_ghz"] * 1e3
            peak_issue = 148 * 4 * sm_mhz * 1e6
            ach = prof["warp_inst_per_launch"] / (avg_ms * 1e-3)
            roof["int_pipe"] = {"bound": "issue", "unit": "warp-inst/s", "achieved": ach,
                                "peak": peak_issue, "frac": ach / peak_issue,
                                "alu_pipe_frac_ncu": prof["alu_pipe_pct_active"] / 100,
                                "thread_inst_per_update": 32 * prof["warp_inst_per_launch"] /
                                upd_launch,
                                "capture": prof["capture"]}

    # e2e through the public API with host buffers (graph build + shades +
    # eval + accumulator read-back), same metric
    e2e = None
    if args.e2e_steps > 0:
        # the step's inputs live in pinned host memory; every step copies them
        # to the device, builds, evaluates and reads the accumulators back
        pinned = tuple(torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
                       for a in (inst.u, inst.v, inst.ts))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            g2 = T.TemporalGraph.build(inst.n, pinned, inst.directed, 0, dev)
            ds2 = T.DeviceShades(g2, k, sh)
            a2 = torch.zeros((reps, n), dtype=torch.int64, device="cuda")
            lanes = [stream] + side
            for s in side:
                s.wait_stream(stream)
            for i, (r, a, b) in enumerate(work):
                T.eval_points_device(g2, ds2, k, g2.t(), cfgs[r], anchor[0], a, b,
                                     a2[r].data_ptr(), lanes[i % len(lanes)].cuda_stream)
            for s in side:
                stream.wait_stream(s)
            if world > 1:
                a2 = xor_allreduce(a2, out=total)
            h = a2.cpu()
            del g2, ds2
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([sec], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
        e2e = {"value": upd_step / sec, "unit": "updates/s",
               "h2d_bytes_per_step": int(inst.m * 12 + sh.vertex_off.nbytes +
                                         sh.vertex_shades.nbytes),
               "d2h_bytes_per_step": int(reps * n * 8), "ms_per_step": sec * 1e3}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            rate, sec, sample, kind, cores = cpu_sample(inst, k, colors, motif, anchor,
                                                        frac=args.ref_frac)
            cpu = {"value": rate, "unit": "updates/s", "cores": cores, "kind": kind,
                   "sample": sample, "seconds": sec}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "updates/s", "cores": 0, "kind": "unavailable",
                   "sample": str(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u64", "data": "synthetic",
                "config": config_json(inst, world, args), "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "host_enqueue_ms_per_step": host_ms, "clocks": clk.summary(),
                "decision": decisions, "checksums": checksums,
                "graph": {"arcs": g.info.arcs, "runs": g.info.runs, "chunks": g.info.chunks,
                          "arcs_with_src": g.info.arcs_with_src,
                          "runs_referenced": g.info.runs_referenced,
                          "split_chunks": g.info.split_chunks,
                          "device_bytes": g.info.device_bytes},
                "engine": "coefficient" if any(c for c, _ in coef.values()) else "points",
                "kernel_ms_per_step": {"level": lvl_ms / prof_steps,
                                       "coef_arcs": coef["coef_arcs"][1] / prof_steps,
                                       "coef_ztrans": coef["coef_ztrans"][1] / prof_steps,
                                       "all": all_ms / prof_steps,
                                       "source": f"{prof_steps}-step single-stream profile pass"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
