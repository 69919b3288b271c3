"""Where the end-to-end step goes: graph build from host arrays (pageable vs
pinned), shade upload, the sieve, accumulator read-back, the synchronous
C-ABI call (tsv_eval_temporal_sieve: shade cache check/upload, sieve, device
finalize, staged D2H) and the graph free.  TSV_TRACE_BUILD=1 adds the device
build's phase times on stderr.  `python tools/e2e_breakdown.py --config 5`."""
import argparse

import numpy as np
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--kinds", default="pageable,pinned")
    args = ap.parse_args()
    import torch
    import paper_2001_07158_b200 as T
    from paper_2001_07158_b200 import synth
    inst = synth.make_config(args.config, scale=args.scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    col = T.VertexColoring(colors, int(colors.max()))
    cfg = T.SieveConfig(seed=1, memory_cap_words=1 << 62)
    sh = T.build_shades(T.MotifQuery.from_multiset(motif), col, cfg)
    pin = [torch.from_numpy(a).pin_memory() for a in (inst.u, inst.v, inst.ts)]
    arrs = {"pageable": (inst.u, inst.v, inst.ts), "pinned": tuple(p.numpy() for p in pin)}
    acc = torch.zeros(inst.n, dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream

    import ctypes as C
    from paper_2001_07158_b200 import _native
    host = np.zeros(max(inst.n, 1), np.uint64)
    vs = np.ascontiguousarray(sh.vertex_shades, np.int32)
    voff = np.ascontiguousarray(sh.vertex_off, np.int32)

    def api(g):
        o = _native.Outcome()
        c = cfg.to_native()
        _native.check(_native.lib().tsv_eval_temporal_sieve(
            g.handle, k, g.t(), voff, vs, C.byref(c), anchor[0], anchor[1], host, C.byref(o)))

    def t(f):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        return r, (time.perf_counter() - t0) * 1e3

    for kind in args.kinds.replace("+", ",").split(","):
        a = arrs[kind]
        rows = []
        for _ in range(args.iters):
            g, tb = t(lambda: T.TemporalGraph.build(inst.n, a, inst.directed, 0, 0))
            ds, ts_ = t(lambda: T.DeviceShades(g, k, sh))
            _, te = t(lambda: T.eval_points_device(g, ds, k, g.t(), cfg, anchor[0], 0, 1 << k,
                                                   acc.data_ptr(), sp))
            _, te2 = t(lambda: T.eval_points_device(g, ds, k, g.t(), cfg, anchor[0], 0, 1 << k,
                                                    acc.data_ptr(), sp))
            print(f"  eval first {te:.1f} ms, again {te2:.1f} ms", flush=True)
            _, td = t(lambda: acc.cpu())
            del ds
            _, tapi = t(lambda: api(g))
            _, tapi2 = t(lambda: api(g))
            _, tf = t(lambda: g.__del__())
            rows.append((tb, ts_, te, td, tapi, tapi2, tf))
            del g
        for r in rows:
            print(f"  {kind} iter: " + " ".join(f"{x:.1f}" for x in r) +
                  f"  free GB {torch.cuda.mem_get_info()[0] / 1e9:.1f}", flush=True)
        best = [min(r[i] for r in rows) for i in range(7)]
        print(f"{kind:9s} build {best[0]:.2f} ms  shades {best[1]:.2f}  eval(1 rep) {best[2]:.2f}"
              f"  d2h {best[3]:.2f}  C-ABI eval (shade upload) {best[4]:.2f}"
              f"  C-ABI eval (cached shades) {best[5]:.2f}  graph free {best[6]:.2f}", flush=True)


if __name__ == "__main__":
    main()
