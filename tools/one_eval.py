"""N full evaluations of one BASELINE config on cuda:0 (the command ncu
captures): `python tools/one_eval.py CONFIG [SCALE] [EVALS]`.  The graph and
shades are built first; each evaluation is one tsv_eval_points_device over
all 2^k points, synchronized, timed with CUDA events."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    cfgno = int(sys.argv[1])
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    evals = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    import torch
    import paper_2001_07158_b200 as T
    from paper_2001_07158_b200 import synth
    inst = synth.make_config(cfgno, scale=scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, 0)
    cfg = T.SieveConfig(seed=1, memory_cap_words=1 << 62)
    sh = T.build_shades(T.MotifQuery.from_multiset(motif),
                        T.VertexColoring(colors, int(colors.max())), cfg)
    ds = T.DeviceShades(g, k, sh)
    acc = torch.zeros(inst.n, dtype=torch.int64, device="cuda")
    sp = torch.cuda.current_stream().cuda_stream
    for i in range(evals):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        T.eval_points_device(g, ds, k, g.t(), cfg, anchor[0], 0, 1 << k, acc.data_ptr(), sp)
        e1.record()
        torch.cuda.synchronize()
        print(f"eval {i}: {e0.elapsed_time(e1):.2f} ms", flush=True)


if __name__ == "__main__":
    main()
