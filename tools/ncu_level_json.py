"""Summarize the middle-level launches of an `ncu --set full` capture
(tools/gpu_profile.sh) into profiles/level_kernel_c<config>.json, which
bench.py reads for the roofline `traffic` and the instruction-issue figures.
Usage: python tools/ncu_level_json.py gpurun_out/prof_<tag>.ncu-rep <config> <tag>"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, config, tag = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6,
             "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6,
             "inst": 1.0, "%": 1.0, "register/thread": 1.0, "Ghz": 1.0, "cycle/second": 1e-9,
             "Mhz": 1e-3}
    mids = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d["Kernel Name"]
        # middle levels: not FIRST (2nd template arg 0) and not LAST (4th 0)
        if "k_level_wide<" in name and ", 0, 1, 0>" in name:
            mids.append(d)
    if not mids:
        sys.exit("no middle-level launch in the capture")

    def avg(key):
        return sum(float(d[key]) for d in mids) / len(mids) * scale[units[key]]

    prof = {
        "config": config,
        "capture": os.path.basename(rep),
        "tag": tag,
        "kernel": mids[0]["Kernel Name"],
        "launches": len(mids),
        "ncu_duration_ms": avg("gpu__time_duration.sum"),
        "traffic_bytes_per_launch": avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum"),
        "dram_read_bytes": avg("dram__bytes_read.sum"),
        "dram_write_bytes": avg("dram__bytes_write.sum"),
        "warp_inst_per_launch": avg("smsp__inst_executed.sum"),
        "alu_pipe_pct_active": avg("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "fma_pipe_pct_active": avg("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_pct_active": avg("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": avg("sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": int(float(mids[0]["launch__registers_per_thread"])),
        "sm_clock_ghz": avg("sm__cycles_elapsed.avg.per_second"),
    }
    path = os.path.join(ROOT, "profiles", f"level_kernel_c{config}.json")
    with open(path, "w") as f:
        json.dump(prof, f, indent=1)
    print(json.dumps(prof, indent=1))


if __name__ == "__main__":
    main()
