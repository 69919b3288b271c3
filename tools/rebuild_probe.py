"""Does an evaluation slow down once graphs have been built and freed?
Builds the C5 graph `--rounds` times (freeing the previous one), evaluates it
twice each, prints per-kernel times and device memory; --trim calls
cudaMemPoolTrimTo(0) on the default pool after every free.
`python tools/rebuild_probe.py [--config 5] [--rounds 4] [--trim]`"""
import argparse
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--trim", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_2001_07158_b200 as T
    from paper_2001_07158_b200 import _native, synth
    inst = synth.make_config(args.config, scale=args.scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    cfg = T.SieveConfig(seed=1, memory_cap_words=1 << 62)
    sh = T.build_shades(T.MotifQuery.from_multiset(motif),
                        T.VertexColoring(colors, int(colors.max())), cfg)
    acc = torch.zeros(inst.n, dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    cudart = C.CDLL("libcudart.so.12") if args.trim else None
    for r in range(args.rounds):
        g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, 0)
        ds = T.DeviceShades(g, k, sh)
        for i in range(2):
            _native.Profile.reset()
            _native.Profile.enable(True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            T.eval_points_device(g, ds, k, g.t(), cfg, anchor[0], 0, 1 << k, acc.data_ptr(), sp)
            torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) * 1e3
            prof = {nm: round(_native.Profile.get(nm)[1], 1) for nm in
                    ("coef_vertex_first", "coef_vertex", "coef_vertex_last", "zj")}
            _native.Profile.enable(False)
            print(f"round {r} eval {i}: {wall:.1f} ms {prof} free GB "
                  f"{torch.cuda.mem_get_info()[0] / 1e9:.1f}", flush=True)
        del ds, g
        torch.cuda.synchronize()
        if cudart is not None:
            pool = C.c_void_p()
            cudart.cudaDeviceGetDefaultMemPool(C.byref(pool), 0)
            cudart.cudaMemPoolTrimTo(pool, C.c_size_t(0))
            print(f"  trimmed; free GB {torch.cuda.mem_get_info()[0] / 1e9:.1f}", flush=True)


if __name__ == "__main__":
    main()
