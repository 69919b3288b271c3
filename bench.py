"""Benchmark of the temporal-sieve hot path on B200 (contract: see DESIGN.md).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is one DECIDE of the configured BASELINE workload: every repetition
seed evaluates all 2^k_eff sieve points over the whole synthetic graph.
Default: config 5 = BASELINE configs[4], the config the metric is quoted on
(k-TempPath k=5, n=1e8, m=1e9, ts in [1,1e6], one repetition).  Metric:
GF(2^64) edge x level x sieve-point updates per second, updates =
A * (k_eff - 1) * 2^k_eff per repetition, and the decide wall time.  The
coefficient engine computes the same sieve sums without visiting points,
so for it the rate is an EQUIVALENT point-form rate (`value_kind`).

Every run checks its decide against the committed full-size golden
(tests/golden/full_size.json) and reports `parity`.

With N > 1 (torchrun) the (repetition, sieve point) units of the decide are
split (shard.plan_units), with no data-path collective; the per-vertex
partial accumulators are XOR-combined once per step (shard.xor_allreduce).
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
    cnt = np.diff(np.asarray(sh.vertex_off, dtype=np.int64))
    if n and int(cnt.min()) >= 2:
        # every vertex carries several shades (k-TempPath: all k): every
        # arc with a predecessor run is live and carries C(k, l-1) entries,
        # every referenced run is a multi-shade row -- closed form from the
        # graph's own counts (no host pass over 1e9 edges)
        a_src, S = g.info.arcs_with_src, g.info.runs_referenced
        meta = 12 * g.info.arcs + 4 * g.info.runs
        arcs = sum(8 * (a_src + S) * comb(k, l - 1) + meta for l in range(3, k))
        ztrans = sum(8 * S * (comb(k, l - 1) + comb(k, l)) for l in range(2, k))
        # vertex-lane engine (z map fused): per middle level 8 B per (live
        # arc, input entry) + 8 B per (referenced run, output entry) + 8 B of
        # metadata per arc (edge id, source slot) + 4 B per run (slot)
        vertex = sum(8 * (a_src * comb(k, l - 1) + S * comb(k, l)) + 8 * g.info.arcs +
                     4 * g.info.runs for l in range(3, k))
        # GF(2^64) products of the vertex-lane middle levels: C(k, l-1) per
        # live arc (y times its source row) + C(k, l-1) + C(k, l) per
        # referenced run (the paired z map, coef_vertex.cu)
        p_arc = sum(a_src * comb(k, l - 1) for l in range(3, k))
        p_z = sum(S * (comb(k, l - 1) + comb(k, l)) for l in range(3, k))
        return {"coef_arcs": arcs, "coef_ztrans": ztrans, "coef_vertex": vertex,
                "_products": {"coef_vertex": p_arc + p_z},
                "_products_split": {"coef_vertex": {"lane_table": p_arc, "holes": p_z}}}
    cu, cv, ct = (np.asarray(x, dtype=np.int64) for x in g.edges())
    if not g.directed():
        cu, cv, ct = np.concatenate([cu, cv]), np.concatenate([cv, cu]), np.concatenate([ct, ct])
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
    products = alg1.get("_products", {})
    alg = {nm: evals * b for nm, b in alg1.items() if nm in coef}
    name = max(coef, key=lambda nm: coef[nm][1])
    n_launch, tot_ms = coef[name]
    if not n_launch or not alg.get(name):
        return None
    achieved = alg[name] / (tot_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": None, "peak_kind": peak_kind,
            "kernel": {"coef_arcs": "k_coef_items / k_coef_arcs (3 <= l < k)",
                       "coef_ztrans": "k_coef_ztrans_direct (2 <= l < k)",
                       "coef_vertex": "k_coef_vertex (3 <= l < k; z map fused)"}[name],
            "engine": "coefficient (top-degree) form on the shaded subgraph, DESIGN.md 2b",
            "family": name,
            "avg_launch_ms": tot_ms / n_launch,
            "alg_bytes_per_launch": alg[name] / n_launch,
            "kernel_ms_per_eval": {nm: coef[nm][1] / max(evals, 1) for nm in coef}}
    try:
        with open(os.path.join(ROOT, "profiles", f"coef_kernels_c{args.config}.json")) as f:
            prof = json.load(f)
        cscale = prof.get("capture_scale", 1.0)
        if prof["config"] != args.config or world != 1:
            prof = None
        else:
            prof = dict(prof["kernels"][name], capture=prof["capture"], capture_scale=cscale)
    except Exception:
        prof = None
    if prof is not None:
        # a capture at another scale of the same config: per-launch DRAM
        # bytes and instructions scaled by the arc count (both are per arc)
        f = args.scale / prof["capture_scale"]
        roof["traffic"] = prof["traffic_bytes_per_launch"] * f
        if f != 1.0:
            roof["traffic_source"] = (f"ncu --set full at scale {prof['capture_scale']:g} "
                                      f"({prof['capture']}), x{f:g} by arcs")
        clk = sm_mhz or prof["sm_clock_ghz"] * 1e3
        peak_issue = 148 * 4 * clk * 1e6
        ach = prof["warp_inst_per_launch"] * f / (roof["avg_launch_ms"] * 1e-3)
        roof["int_pipe"] = {"bound": "issue", "unit": "warp-inst/s", "achieved": ach,
                            "peak": peak_issue, "frac": ach / peak_issue,
                            "alu_pipe_frac_ncu": prof["alu_pipe_pct_active"] / 100,
                            "capture": prof["capture"]}
        if "fmaheavy_pipe_pct_elapsed" in prof:
            # the carry-less products' IMAD.WIDE run on the FMA-heavy pipe
            roof["int_pipe"]["fmaheavy_pipe_frac_ncu"] = prof["fmaheavy_pipe_pct_elapsed"] / 100
    if name in products:
        # GF(2^64) products per second of the family against the measured
        # throughput of the same multiply alone (tsv_gf_bench, holes +
        # Karatsuba, full grid: profiles/int_pipe_peaks.json)
        # (arc products: lane table, 10 per build; z map: holes + Karatsuba;
        # the peak is the time-weighted blend of the two microbenchmarks)
        rate = evals * products[name] / (tot_ms * 1e-3)
        split = alg1.get("_products_split", {}).get(name)
        try:
            with open(os.path.join(ROOT, "profiles", "int_pipe_peaks.json")) as f:
                peaks = json.load(f)
            holes = peaks["GF product, holes + Karatsuba"]
            table = peaks.get("GF product, lane table, 10 per build")
            if split and table:
                gpeak = products[name] / (split["lane_table"] / table + split["holes"] / holes)
                kind = ("measured microbenchmarks blended by product count (tsv_gf_bench "
                        "variant 12, lane table, for the arc products; variant 2, holes + "
                        "Karatsuba, for the z map)")
            else:
                gpeak = holes
                kind = "measured microbenchmark (tsv_gf_bench variant 2)"
        except Exception:
            gpeak, kind = None, None
        roof["gf_products"] = {"unit": "products/s", "achieved": rate, "peak": gpeak,
                               "frac": rate / gpeak if gpeak else None,
                               "peak_kind": kind,
                               "per_launch": products[name] * evals / n_launch}
        if split:
            roof["gf_products"]["split_per_eval"] = split
    return roof


def e2e_api_leg(inst, reps, steps, upd_step, gold):
    """The same decide through the C++ drop-in API a reference user calls
    (libtsieve: TemporalGraph::build from host vectors + solve() in decide
    mode, --preprocess none, one call per repetition seed), host arrays in,
    host outcome out.  The host vectors are staged outside the timed region
    (a caller owns them); graph canonicalization, upload, shades, evaluation
    and finalize are inside."""
    import ctypes as C
    lib = C.CDLL(os.path.join(ROOT, "paper_2001_07158_b200", "lib", "libtsieve.so"))
    i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    lib.tsieve_last_error.restype = C.c_char_p
    lib.tsieve_e2e_stage.restype = C.c_int64
    lib.tsieve_e2e_stage.argtypes = [C.c_int32, C.c_int64, i32p, i32p, i32p, C.c_int, i32p]
    lib.tsieve_e2e_decide.restype = C.c_int64
    lib.tsieve_e2e_decide.argtypes = [C.c_char_p, i32p, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_uint64, C.c_int32,
                                      np.ctypeslib.ndpointer(np.int32), np.ctypeslib.ndpointer(
                                          np.uint64), np.ctypeslib.ndpointer(np.int64)]
    a = lambda x: np.ascontiguousarray(np.asarray(x), dtype=np.int32)  # noqa: E731
    u, v, ts = a(inst.u), a(inst.v), a(inst.ts)
    colors = a(inst.colors) if inst.colors is not None else np.ones(max(inst.n, 1), np.int32)
    motif = a(inst.motif) if inst.motif else np.zeros(1, np.int32)
    dec = np.zeros(reps, np.int32)
    cs = np.zeros(reps, np.uint64)
    fl = np.zeros(reps, np.int64)
    total = 0.0
    for _ in range(steps):
        if lib.tsieve_e2e_stage(inst.n, len(u), u, v, ts, int(inst.directed), colors) < 0:
            raise RuntimeError(lib.tsieve_last_error().decode())
        t0 = time.perf_counter()
        r = lib.tsieve_e2e_decide(inst.problem.encode(), motif, len(inst.motif or []), inst.k,
                                  inst.source, inst.dest, 1, reps, dec, cs, fl)
        total += time.perf_counter() - t0
        if r < 0:
            raise RuntimeError(lib.tsieve_last_error().decode())
    sec = total / steps
    out = {"value": upd_step / sec, "unit": "updates/s", "ms_per_step": sec * 1e3,
           "h2d_bytes_per_step": int(u.nbytes + v.nbytes + ts.nbytes),
           "d2h_bytes_per_step": int(reps * inst.n * 8),
           "path": ("C++ drop-in (libtsieve): TemporalGraph::build + solve(decide, "
                    "--preprocess none, memory_cap_words 2^62 as the other legs) per "
                    "repetition seed"),
           "checksums": [f"{int(x):016x}" for x in cs]}
    if gold is not None:
        out["parity"] = all(f"{int(cs[r]):016x}" == gold[1][r]["checksum"] and
                            int(fl[r]) == gold[1][r]["nflagged"] for r in range(reps))
    return out


# ------------------------------------------------------------------ CPU legs

METRIC = "GF(2^64) edge x level x sieve-pt updates/s (decide)"
GOLDEN_FULL = os.path.join(ROOT, "tests", "golden", "full_size.json")
DEFAULT_STEPS = {1: 50, 2: 20, 3: 10, 4: 3, 5: 5}
DEFAULT_E2E = {1: 5, 2: 5, 3: 3, 4: 1, 5: 2}
# CPU sample per config: the time prefix ts <= frac * t (10-30 s of host work)
CPU_FRAC = {1: 1.0, 2: 0.1, 3: 0.1, 4: 0.002, 5: 0.01}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_sample(inst, k, colors, motif, anchor, seed=1, frac=None, threads=None, gpu_check=None):
    """The reference's CPU implementation of the path on a BOUNDED sample of
    the workload (the time prefix ts <= frac * t of the same graph, all 2^k
    points, all levels), on all host threads.  Returns a dict.

    Configs 1-2: the reference's own eval_temporal_sieve (oracle/_ref, the
    unmodified core compiled by oracle/Makefile; kind "reference").  Configs
    3-5: its dense layers (2 n W (t+1) words, sieve.cpp:188-192) cannot be
    allocated, so the validated multi-threaded restatement stands in
    (oracle/tsv_oracle_big.c; kind "port").  gpu_check(max_ts) -> the GPU's
    accumulators on the same window, compared word for word."""
    from oracle import oracle as O
    threads = threads or os.cpu_count() or 1
    if frac is None:
        frac = CPU_FRAC[inst_cfg(inst)]
    max_ts = max(1, int(inst.t * frac))
    sel = inst.ts <= max_ts
    arcs = int(np.count_nonzero(sel)) * (1 if inst.directed else 2)
    upd = arcs * (k - 1) * (1 << k)
    dense_bytes = 2 * inst.n * 8 * (max_ts + 1) * 8
    res = {"threads": threads, "max_ts": max_ts, "arcs": arcs, "updates": upd}
    if O.ref_available() and dense_bytes < 24e9:
        os.environ.setdefault("OMP_WAIT_POLICY", "active")
        r = O.ref_eval(inst.n, inst.u, inst.v, inst.ts, inst.directed, colors, motif,
                       max_ts=max_ts, seed=seed, lanes=8, threads=threads, anchor=anchor,
                       t=inst.t, repeats=2)
        res.update(seconds=r["seconds"], kind="reference", acc=r["acc"],
                   sample=f"ts <= {max_ts} of t={inst.t} ({arcs} arcs, all {1 << k} points, "
                          f"{k - 1} levels, seed {seed}; reference eval_temporal_sieve, "
                          f"best of 2)")
    else:
        from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
        from paper_2001_07158_b200.sieve import SieveConfig, build_shades
        u = np.ascontiguousarray(inst.u[sel], dtype=np.int32)
        v = np.ascontiguousarray(inst.v[sel], dtype=np.int32)
        ts = np.ascontiguousarray(inst.ts[sel], dtype=np.int32)
        O.set_threads(threads)
        w = O.canonicalize_inplace(inst.n, u, v, ts, inst.directed)
        G = O.BigGraph(inst.n, u[:w], v[:w], ts[:w], inst.directed, max_ts)
        sh = build_shades(MotifQuery.from_multiset(motif),
                          VertexColoring(colors, int(colors.max())), SieveConfig(seed=seed))
        t0 = time.perf_counter()
        acc = G.eval(k, sh.vertex_off, sh.vertex_shades, seed, anchor[0], lanes=16)
        sec = time.perf_counter() - t0
        G.close()
        res.update(seconds=sec, kind="port", acc=acc,
                   sample=f"ts <= {max_ts} of t={inst.t} ({arcs} arcs, all {1 << k} points, "
                          f"{k - 1} levels, seed {seed}; oracle/tsv_oracle_big.c, the "
                          f"reference's dense layers do not fit at this size)")
    res["value"] = upd / res["seconds"]
    if gpu_check is not None:
        try:
            res["window_parity"] = bool(np.array_equal(gpu_check(max_ts), res["acc"]))
        except Exception as e:  # reported, never fatal
            res["window_parity"] = f"unchecked: {e}"
    return res


def inst_cfg(inst):
    return int(inst.name[1])


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on the host cores
    (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    from paper_2001_07158_b200 import synth
    inst = synth.make_config(args.config, scale=args.scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    times, rates = [], []
    info = None
    steps = args.steps or DEFAULT_STEPS[args.config]
    for i in range(args.warmup + steps):
        r = cpu_sample(inst, k, colors, motif, anchor, frac=args.ref_frac)
        info = r
        if i >= args.warmup:
            times.append(r["seconds"])
            rates.append(r["value"])
    value = statistics.median(rates)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "updates/s",
            "n_gpus": world, "steps": steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": config_json(inst, world, args, cpu=True),
            "cpu_baseline": {"value": value, "unit": "updates/s", "cores": info["threads"],
                             "kind": info["kind"], "sample": info["sample"],
                             "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_json(inst, world, args, cpu=False):
    k_eff = inst.k_eff
    reps = REPS[args.config]
    l2 = ("host arm: the reference's CPU code, no device cache involved" if cpu else
          "flushed before every step: a 256 MB buffer (2x the 126 MB L2) is "
          "zeroed on the bench stream inside the timed region")
    return {"workload": f"BASELINE configs[{args.config - 1}]: {inst.name}"
                        + ("" if args.scale == 1.0 else f" (scaled x{args.scale})"), "n": inst.n,
            "m": inst.m, "t": inst.t, "directed": inst.directed, "k_eff": k_eff,
            "sieve_points": 1 << k_eff, "repetitions": reps,
            "updates_per_step": inst.updates() * reps,
            "parallelism": (f"head-vertex partition of every evaluation over {world} GPU(s) "
                            "(shard.vertex_partitioned_eval) when the vertex-lane engine applies, "
                            "else repetitions / sieve points (shard.plan_units)"
                            + (f"; rows between levels: {args.exchange}" if world > 1 else "")
                            if not cpu else
                            "reference CPU code on all host threads (rank 0)"),
            "l2": l2}


def golden_for(args, reps):
    """Committed full-size golden decide outputs for this config (seed 1+r,
    max_ts = t), or None."""
    if args.scale != 1.0 and not (args.config == 5 and args.scale == 0.1):
        return None
    key = f"C{args.config}" + ("x0.1" if args.scale != 1.0 else "")
    try:
        with open(GOLDEN_FULL) as f:
            rec = json.load(f).get(key)
    except Exception:
        return None
    if not rec or "evals" not in rec:
        return None
    want = {}
    for e in rec["evals"]:
        if e["max_ts"] == rec["t_canonical"]:
            want[e["seed"]] = e
    if not all((1 + r) in want for r in range(reps)):
        return None
    return key, [want[1 + r] for r in range(reps)]


# ---------------------------------------------------------------- our arm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0, help="0 = per-config default")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=float, default=1.0,
                    help="shrink n and m of the config (not a bench line unless 1.0)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-frac", type=float, default=None,
                    help="CPU sample: time prefix ts <= frac * t (default per config)")
    ap.add_argument("--points-per-batch", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=-1, help="-1 = per-config default")
    ap.add_argument("--simulate-world", default="",
                    help="N list (2,4,8 or 2+4+8): time each rank's share of the vertex-partitioned "
                         "evaluation on this one GPU and project the N-GPU step (DESIGN.md 6)")
    ap.add_argument("--nvlink-gbs", type=float, default=720.0,
                    help="all-gather bandwidth per GPU assumed by the --simulate-world model")
    ap.add_argument("--exchange", default=os.environ.get("TSV_EXCHANGE", "alltoall"),
                    choices=["alltoall", "peer"],
                    help="N > 1, vertex partition: rows between levels by pack / all_to_all / "
                         "unpack (default), or stored into the peers' buffers by the level "
                         "kernel over symmetric memory (NVLink peer stores)")
    ap.add_argument("--streams", type=int, default=4,
                    help="concurrent CUDA streams for the repetitions of a step "
                         "(at most one per work unit)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    steps = args.steps or DEFAULT_STEPS[args.config]
    e2e_steps = DEFAULT_E2E[args.config] if args.e2e_steps < 0 else args.e2e_steps

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

    g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, dev)
    col = T.VertexColoring(colors, int(colors.max()))
    # the reference's default cap (2^31 words) sizes ITS dense layers; the
    # engine's working set is bounded by device memory instead
    cfgs = [T.SieveConfig(seed=s, points_per_batch=args.points_per_batch,
                          memory_cap_words=1 << 62) for s in seeds]
    sh = T.build_shades(T.MotifQuery.from_multiset(motif), col, cfgs[0])
    ds = T.DeviceShades(g, k, sh)
    n = g.n()
    graph_info = {"arcs": g.info.arcs, "runs": g.info.runs, "chunks": g.info.chunks,
                  "arcs_with_src": g.info.arcs_with_src,
                  "runs_referenced": g.info.runs_referenced,
                  "split_chunks": g.info.split_chunks, "device_bytes": g.info.device_bytes}
    acc = torch.zeros((reps, n), dtype=torch.int64, device="cuda")
    total = torch.zeros((reps, n), dtype=torch.int64, device="cuda") if world > 1 else None
    # N > 1 and a query the vertex-lane engine takes (k <= 5, every shaded
    # vertex multi-shade, no hubs; C5): every repetition is split by head
    # vertex over the ranks (shard.vertex_partitioned_eval), else the
    # (repetition, point) units of plan_units
    vertex_mode = False
    if world > 1:
        from paper_2001_07158_b200.shard import eval_vertex_partitioned_device
        from paper_2001_07158_b200.sieve import vertex_partition
        ok = torch.tensor([1 if vertex_partition(g, ds, k, rank, world).applicable else 0],
                          device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        vertex_mode = bool(ok.item())
    vbufs = peer_bufs = None
    if vertex_mode:
        words = vertex_partition(g, ds, k, rank, world).state_words
        if args.exchange == "peer":
            from paper_2001_07158_b200.shard import PeerStateBuffers, eval_vertex_partitioned_peer
            peer_bufs = PeerStateBuffers(words, torch.device("cuda", torch.cuda.current_device()))
        else:
            vbufs = (torch.empty(words, dtype=torch.int64, device="cuda"),
                     torch.empty(words, dtype=torch.int64, device="cuda"))

    def vertex_eval(gg, dd, cfg_r, acc_r, bufs):
        if peer_bufs is not None:
            return eval_vertex_partitioned_peer(gg, dd, k, gg.t(), cfg_r, anchor[0], acc_r, rank,
                                                world, peer_bufs=peer_bufs)
        return eval_vertex_partitioned_device(gg, dd, k, gg.t(), cfg_r, anchor[0], acc_r, rank,
                                              world, bufs=bufs)

    # repetitions (independent evaluations) may run on concurrent streams so
    # one evaluation's tail wave overlaps the next one's launches
    side = [torch.cuda.Stream() for _ in range(max(1, min(args.streams, len(work))) - 1)]

    # L2 flush between steps (inside the timed region, counted against us)
    l2_flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step(concurrent=True):
        l2_flush.zero_()
        acc.zero_()
        if vertex_mode:
            for r in range(reps):
                total[r] = vertex_eval(g, ds, cfgs[r], acc[r], vbufs)
            return total
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
        for _ in range(steps):
            res = step()
        host_ms = (time.perf_counter() - h0) * 1e3 / steps   # enqueue time per step
        e1.record(stream)
        torch.cuda.synchronize()
    launches = _native.Profile.launches() - launches0
    ms = e0.elapsed_time(e1) / steps
    # Per-kernel CUDA-event timing (roofline) from a separate single-stream
    # pass after the timed region: with concurrent streams a launch's events
    # would also cover the other stream's kernels.
    prof_steps = max(1, min(steps, 3))
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
    # the vertex-lane engine (coef_vertex.cu) fuses the z map into the level:
    # one family, "coef_vertex" (middle levels)
    vx = _native.Profile.get("coef_vertex")
    if vx[0]:
        coef = {"coef_vertex": vx}
    all_n, all_ms = _native.Profile.get(None)
    _native.Profile.enable(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    upd_step = inst.updates() * reps
    value = upd_step / (ms * 1e-3)

    # decision / checksum of the last timed step, finalized on the device
    decisions, checksums, nflagged = [], [], []
    for r in range(reps):
        f, cs = _native.finalize_device(res[r].data_ptr(), n, anchor[1], sp)
        decisions.append(f > 0)
        checksums.append(f"{cs:016x}")
        nflagged.append(f)
    gold = golden_for(args, reps)
    parity = None
    if gold is not None:
        key, evals = gold
        parity = {"golden": f"tests/golden/full_size.json {key}",
                  "source": evals[0]["source"],
                  "match": all(checksums[r] == evals[r]["checksum"] and
                               nflagged[r] == evals[r]["nflagged"] for r in range(reps))}

    # roofline of the dominant kernel
    hbm, peak_kind = peaks()
    roof = None
    # full-range evaluations in the profile pass (the coefficient engine's)
    evals = sum(1 for _, a, b in work if a == 0 and b == P) * prof_steps
    if any(c for c, _ in coef.values()):
        roof = coef_roofline(coef, k, coef_alg_bytes(g, sh, k), evals, hbm, peak_kind, args,
                             world, clk.summary().get("sm_mhz"))
        if roof is not None:
            roof["launch_share_of_step"] = coef[roof["family"]][1] / max(all_ms, 1e-9)
    elif lvl_n:
        mid_levels = (k - 2) - (1 if last_n else 0)
        my_points = sum(b - a for _, a, b in work)
        upd_launch = g.info.arcs * mid_levels * my_points * prof_steps / lvl_n
        alg_bytes = BYTES_PER_UPDATE * upd_launch
        avg_ms = lvl_ms / lvl_n
        achieved = alg_bytes / (avg_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                "frac": achieved / hbm, "traffic": None, "peak_kind": peak_kind,
                "kernel": ("k_level (grouped, W < 32, 3 <= l < k)" if grouped
                           else "k_level_wide (3 <= l < k)"), "avg_launch_ms": avg_ms,
                "launch_share_of_step": lvl_ms / max(all_ms, 1e-9),
                "alg_bytes_per_launch": alg_bytes}

    # --simulate-world: every rank's share of the vertex-partitioned
    # evaluation timed on this GPU, the N-GPU step projected from it
    simulated = None
    if args.simulate_world and world == 1:
        from paper_2001_07158_b200.shard import eval_vertex_simulated
        simulated = {"model": ("per level: max over ranks of the rank's measured share + the "
                               "targeted row exchange (the largest rank's rows sent or received, "
                               "from its exchange lists) at --nvlink-gbs per GPU (modeled: one "
                               "GPU here); + XOR combine of n words.  peer_store: the "
                               "exchange rides inside the level kernel (NVLink peer stores, "
                               "tsv_eval_vertex_level_peer): per level max(the rank's share "
                               "measured WITH its peer stores issued -- to local HBM here -- , "
                               "the same exchange bytes at --nvlink-gbs) + a barrier"),
                     "nvlink_gbs": args.nvlink_gbs, "worlds": {}}
        ref_acc = res[0].clone()
        sim_bufs = None   # one pair of state buffers for every simulated world and pass
        for N in (int(x) for x in args.simulate_world.replace("+", ",").split(",") if x):
            a = torch.zeros(n, dtype=torch.int64, device="cuda")
            try:
                if sim_bufs is None:
                    from paper_2001_07158_b200.sieve import vertex_partition
                    words = vertex_partition(g, ds, k, 0, 1).state_words
                    sim_bufs = (torch.empty(words, dtype=torch.int64, device="cuda"),
                                torch.empty(words, dtype=torch.int64, device="cuda"))
                eval_vertex_simulated(g, ds, k, g.t(), cfgs[0], anchor[0], a, N,
                                      bufs=sim_bufs)  # warm-up
                a.zero_()
                a, times, parts = eval_vertex_simulated(g, ds, k, g.t(), cfgs[0], anchor[0], a, N,
                                                        bufs=sim_bufs, timed=True)
                if N > 1:   # the exchange lists / reader bytes are built on first use
                    from paper_2001_07158_b200.sieve import vertex_exchange_plan
                    for q in range(N):
                        vertex_exchange_plan(g, ds, k, q, N)
                a2 = torch.zeros(n, dtype=torch.int64, device="cuda")
                a2, times_p, _ = eval_vertex_simulated(g, ds, k, g.t(), cfgs[0], anchor[0], a2, N,
                                                       bufs=sim_bufs, timed=True, peer_store=True)
            except ValueError as e:
                simulated["worlds"][str(N)] = {"unavailable": str(e)}
                continue
            if anchor[1] >= 0:
                _native.finalize_device(a.data_ptr(), n, anchor[1], sp)
            S = parts[0].slots
            # targeted exchange: rows per rank from the exchange lists
            from paper_2001_07158_b200.sieve import vertex_exchange_plan
            rows_max = 0
            if N > 1:
                plans = [vertex_exchange_plan(g, ds, k, q, N) for q in range(N)]
                rows_max = max(max(p.send_total, p.recv_total) for p in plans)
            lv = {}
            total_ms = total_peer_ms = 0.0
            for level in range(2, k + 1):
                per = [times[(level, q)] for q in range(N)]
                per_p = [times_p[(level, q)] for q in range(N)]
                xch = xch_ag = 0.0
                if level < k and N > 1:
                    F = parts[0].row_words[level]
                    xch = rows_max * F * 8 / (args.nvlink_gbs * 1e9) * 1e3
                    xch_ag = (N - 1) / N * S * F * 8 / (args.nvlink_gbs * 1e9) * 1e3
                lv[str(level)] = {"rank_ms": per, "max_ms": max(per), "exchange_ms": xch,
                                  "allgather_exchange_ms": xch_ag,
                                  "peer_store_max_ms": max(per_p)}
                total_ms += max(per) + xch
                total_peer_ms += max(max(per_p), xch) + (0.02 if level < k and N > 1 else 0.0)
            comb = 2 * (N - 1) / N * n * 8 / (args.nvlink_gbs * 1e9) * 1e3 if N > 1 else 0.0
            total_ms += comb
            total_peer_ms += comb
            if anchor[1] >= 0:
                _native.finalize_device(a2.data_ptr(), n, anchor[1], sp)
            simulated["worlds"][str(N)] = {
                "levels": lv, "combine_ms": comb, "projected_ms_per_step": total_ms * reps,
                "peer_store": {"projected_ms_per_step": total_peer_ms * reps,
                               "projected_value": upd_step / (total_peer_ms * reps * 1e-3),
                               "barrier_ms_assumed": 0.02,
                               "parity_vs_n1": bool(torch.equal(a2, ref_acc))},
                "projected_value": upd_step / (total_ms * reps * 1e-3),
                "exchange_rows_per_rank_max": rows_max, "slots": S,
                "parity_vs_n1": bool(torch.equal(a, ref_acc))}

    # the GPU's accumulators on the CPU sample's window (horizon max_ts on the
    # same graph), checked word for word against the CPU arm below
    gpu_window = None
    want_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
    if want_cpu:
        frac = args.ref_frac if args.ref_frac is not None else CPU_FRAC[args.config]
        wts = max(1, int(inst.t * frac))
        if wts <= g.t():
            o = T.eval_temporal_sieve(g, k, wts, sh, cfgs[0], T.AnchorSpec(*anchor))
            gpu_window = (wts, o.accumulators)

    # e2e through the C-ABI with HOST buffers: every step copies the edge
    # arrays from pinned host memory (tsv_graph_build: device canonicalize +
    # layout), uploads the host shade CSR, evaluates, finalizes and copies the
    # accumulators back into a host buffer (tsv_eval_temporal_sieve).  The
    # timed graph is freed first so both fit in HBM.
    del ds, g
    sim_bufs = None
    acc = total = vbufs = None
    torch.cuda.synchronize()
    e2e = None
    e2e_parity = None
    if e2e_steps > 0:
        import ctypes as C
        pinned = tuple(torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).pin_memory()
                       for a in (inst.u, inst.v, inst.ts))
        pu, pv, pt = (x.numpy() for x in pinned)
        host_acc = np.zeros((reps, max(n, 1)), np.uint64)
        vs = sh.vertex_shades if len(sh.vertex_shades) else np.zeros(1, np.int32)
        voff = np.ascontiguousarray(sh.vertex_off, np.int32)
        L = _native.lib()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        outs = []

        def e2e_step():
            h = C.c_void_p()
            _native.check(L.tsv_graph_build(inst.n, len(pu), pu, pv, pt, int(inst.directed), 0,
                                             dev, C.byref(h)))
            info = _native.GraphInfo()
            _native.check(L.tsv_graph_get_info(h, C.byref(info)))
            outs = []
            if world == 1:
                for r in range(reps):
                    o = _native.Outcome()
                    cfg = cfgs[r].to_native()
                    _native.check(L.tsv_eval_temporal_sieve(
                        h, k, info.t, voff, vs, C.byref(cfg), anchor[0], anchor[1],
                        host_acc[r], C.byref(o)))
                    outs.append((int(o.flagged), f"{o.checksum:016x}"))
            else:
                g2 = T.TemporalGraph(h, info)
                ds2 = T.DeviceShades(g2, k, sh)
                a2 = torch.zeros((reps, n), dtype=torch.int64, device="cuda")
                if vertex_mode:
                    for r in range(reps):
                        a2[r] = vertex_eval(g2, ds2, cfgs[r], a2[r], None)
                else:
                    for r, a, b in work:
                        T.eval_points_device(g2, ds2, k, g2.t(), cfgs[r], anchor[0], a, b,
                                             a2[r].data_ptr(), sp)
                    a2 = xor_allreduce(a2)
                host_acc[:] = a2.cpu().numpy().view(np.uint64)
                del ds2, g2
                h = None
            if h is not None:
                L.tsv_graph_free(h)
            return outs

        # one untimed step first (first-use allocations of the build and the
        # staging buffers), then the timed ones
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            outs = e2e_step()
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / e2e_steps
        if world > 1:
            t = torch.tensor([sec], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
        if gold is not None and outs:
            e2e_parity = all(outs[r] == (gold[1][r]["nflagged"], gold[1][r]["checksum"])
                             for r in range(reps))
        e2e = {"value": upd_step / sec, "unit": "updates/s", "steps": e2e_steps, "warmup": 1,
               "h2d_bytes_per_step": int(pu.nbytes + pv.nbytes + pt.nbytes + voff.nbytes +
                                         (vs.nbytes if len(sh.vertex_shades) else 0)),
               "d2h_bytes_per_step": int(reps * n * 8), "ms_per_step": sec * 1e3,
               "path": ("C-ABI: tsv_graph_build (pinned host edges) + tsv_eval_temporal_sieve "
                        "(host shade CSR, host accumulators, device finalize) per repetition"
                        if world == 1 else "tsv_graph_build + tsv_eval_points_device + "
                        "XOR combine + D2H"),
               "parity": e2e_parity}
        del pinned, pu, pv, pt
        if world == 1:
            e2e["api"] = e2e_api_leg(inst, reps, e2e_steps, upd_step, gold)

    cpu = None
    if want_cpu:
        def gpu_check(mt):
            if gpu_window is None or gpu_window[0] != mt:
                raise ValueError("no GPU evaluation at this horizon")
            return gpu_window[1]
        try:
            r = cpu_sample(inst, k, colors, motif, anchor, frac=args.ref_frac,
                           gpu_check=gpu_check)
            cpu = {"value": r["value"], "unit": "updates/s", "cores": r["threads"],
                   "kind": r["kind"], "sample": r["sample"], "seconds": r["seconds"],
                   "cpu_model": cpu_model(), "window_parity": r.get("window_parity")}
            # calibration of the sampled rate: the whole evaluation's CPU time
            # when the full-size golden was made (reference or OpenMP port,
            # tests/golden/full_size.json; the build container's cores)
            if gold is not None:
                e0 = gold[1][0]
                secs = e0.get("reference_seconds") or e0.get("oracle_seconds")
                if secs:
                    thr = e0.get("reference_threads") or e0.get("oracle_threads")
                    cpu["full_run_calibration"] = {
                        "seconds": secs, "threads": thr, "source": e0.get("source"),
                        "updates_per_s": inst.updates() / secs,
                        "note": "one whole evaluation on the golden-making host"}
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "updates/s", "cores": 0, "kind": "unavailable",
                   "sample": str(e)}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "updates/s", "n_gpus": world,
                "steps": steps, "warmup": args.warmup, "ms_per_step": ms,
                "decide_ms": ms / reps if reps > 1 else ms,
                "value_kind": ("equivalent point-form updates/s: A*(k_eff-1)*2^k_eff per decide "
                               "/ decide time; the coefficient engine computes the same sieve "
                               "sums without visiting points (DESIGN.md 2b)"
                               if any(c for c, _ in coef.values()) else
                               "point-form updates/s (point engine)"),
                "higher_is_better": True, "scaling": "weak" if world > 1 else "strong",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": config_json(inst, world, args), "parity": parity,
                "simulated_world": simulated,
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": e2e, "gpu_launches": launches, "host_enqueue_ms_per_step": host_ms,
                "clocks": clk.summary(), "decision": decisions, "checksums": checksums,
                "nflagged": nflagged, "graph": graph_info,
                "engine": "coefficient" if any(c for c, _ in coef.values()) else "points",
                "kernel_ms_per_step": {"level": lvl_ms / prof_steps,
                                       **{nm: c[1] / prof_steps for nm, c in coef.items()},
                                       "all": all_ms / prof_steps,
                                       "source": f"{prof_steps}-step single-stream profile pass"}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
