"""Host enqueue cost of eval_points_device calls (C5 by default; TSV_TRACE_COEF
phase marks on stderr): `python tools/host_probe.py [SCALE]`."""
import os, sys, time
os.environ["TSV_TRACE_COEF"] = "1"
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import paper_2001_07158_b200 as T
from paper_2001_07158_b200 import synth
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
inst = synth.make_config(5, scale=scale)
k, colors, motif, anchor = synth.effective_query(inst)
g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, 0)
cfg = T.SieveConfig(seed=1, memory_cap_words=1 << 62)
sh = T.build_shades(T.MotifQuery.from_multiset(motif), T.VertexColoring(colors, int(colors.max())), cfg)
ds = T.DeviceShades(g, k, sh)
acc = torch.zeros(inst.n, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream()
sp = st.cuda_stream
for i in range(3):
    T.eval_points_device(g, ds, k, g.t(), cfg, anchor[0], 0, 1 << k, acc.data_ptr(), sp)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h = []
for i in range(4):
    t0 = time.perf_counter()
    T.eval_points_device(g, ds, k, g.t(), cfg, anchor[0], 0, 1 << k, acc.data_ptr(), sp)
    h.append((time.perf_counter() - t0) * 1e3)
e1.record()
torch.cuda.synchronize()
print("host ms per call", [round(x, 2) for x in h], "gpu ms per call", e0.elapsed_time(e1) / 4, flush=True)
