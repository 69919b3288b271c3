"""Summarize an `ncu --set full` capture of one evaluation's coefficient-engine
launches (tools/gpu_profile_coef.sh) into profiles/coef_kernels_c<config>.json,
which bench.py reads for the roofline `traffic` and instruction-issue figures.
Per kernel family (middle-level k_coef_arcs, k_coef_ztrans_tab, ...): launches,
mean duration, DRAM bytes, executed warp instructions, pipe utilizations.
Usage: python tools/ncu_coef_json.py gpurun_out/prof_<tag>.ncu-rep <config> <tag> [OUT.json] [SCALE]
(SCALE: the config scale the capture ran at; bench.py scales per-launch
traffic and instructions by arcs when it runs at another scale)"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6,
         "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
         "inst": 1.0, "%": 1.0, "register/thread": 1.0, "Ghz": 1.0, "cycle/second": 1e-9,
         "Mhz": 1e-3}
KEYS = {"ncu_duration_ms": "gpu__time_duration.sum",
        "dram_read_bytes": "dram__bytes_read.sum",
        "dram_write_bytes": "dram__bytes_write.sum",
        "warp_inst_per_launch": "smsp__inst_executed.sum",
        "alu_pipe_pct_active": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "fma_pipe_pct_active": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "fmaheavy_pipe_pct_elapsed": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lsu_pipe_pct_active": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "issue_pct_active": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1_shared_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second"}


def family(name):
    m = re.search(r"k_coef_vertex<(\d+), (\d+), (\w+), (\w+)>", name)
    if m:
        first = m.group(3) in ("1", "true")
        last = m.group(4) in ("1", "true")
        return "coef_vertex_first" if first else "coef_vertex_last" if last else "coef_vertex"
    m = re.search(r"k_coef_arcs<(\d+), (\d+), (\w+), (\w+)>", name)
    if m:
        first = m.group(3) in ("1", "true")
        last = m.group(4) in ("1", "true")
        return "coef_arcs_first" if first else "coef_arcs_last" if last else "coef_arcs"
    m = re.search(r"k_coef_items(?:_reg)?<(\w+), (\w+), (\d+)>", name)
    if m:
        first = m.group(1) in ("1", "true")
        last = m.group(2) in ("1", "true")
        return "coef_arcs_first" if first else "coef_arcs_last" if last else "coef_arcs"
    for f in ("k_coef_ztrans_tab", "k_coef_ztrans", "k_coef_readout", "k_coef_fixup"):
        if f in name:
            return {"k_coef_ztrans_tab": "coef_ztrans"}.get(f, f[2:])
    return None


def main():
    rep, config, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    dest = sys.argv[4] if len(sys.argv) > 4 and sys.argv[4] != "-" else None
    scale = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    fams = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        f = family(d["Kernel Name"])
        if f:
            fams.setdefault(f, []).append(d)
    res = {"config": config, "capture": os.path.basename(rep), "tag": tag, "capture_scale": scale,
           "kernels": {}}
    for f, ds in fams.items():
        e = {"launches": len(ds), "kernel": ds[0]["Kernel Name"],
             "registers_per_thread": int(float(ds[0]["launch__registers_per_thread"]))}
        for k, m in KEYS.items():
            if m in hdr:
                e[k] = sum(float(d[m]) for d in ds) / len(ds) * SCALE.get(units[m], 1.0)
        e["traffic_bytes_per_launch"] = e.get("dram_read_bytes", 0) + e.get("dram_write_bytes", 0)
        res["kernels"][f] = e
    path = dest or os.path.join(ROOT, "profiles", f"coef_kernels_c{config}.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
