"""One solve() through the C++ drop-in on a BASELINE config with a chosen
preprocessing level, phase marks of the solver (TSIEVE_TRACE), the C-ABI
(TSV_TRACE_API) and the static sieve on stderr:
`python tools/preprocess_probe.py CONFIG [PREPROCESS 0-3] [MODE 0 decide|2 extract] [SCALE]`."""
import ctypes as C
import json
import os
import sys
import time

os.environ.setdefault("TSIEVE_TRACE", "1")
os.environ.setdefault("TSV_TRACE_API", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    from paper_2001_07158_b200 import synth
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    pre = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    mode = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    scale = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    inst = synth.make_config(cfg, scale=scale)
    lib = C.CDLL(os.path.join(ROOT, "paper_2001_07158_b200", "lib", "libtsieve.so"))
    i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
    lib.tsieve_last_error.restype = C.c_char_p
    lib.tsieve_solve_json.restype = C.c_int64
    lib.tsieve_solve_json.argtypes = [C.c_int32, C.c_int64, i32p, i32p, i32p, C.c_int, C.c_int32,
                                      i32p, C.c_char_p, i32p, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                      C.c_char_p, C.c_int64]
    a = lambda x: np.ascontiguousarray(np.asarray(x), dtype=np.int32)  # noqa: E731
    motif = a(inst.motif) if inst.motif else np.zeros(1, np.int32)
    buf = C.create_string_buffer(1 << 24)
    t0 = time.perf_counter()
    r = lib.tsieve_solve_json(inst.n, inst.m, a(inst.u), a(inst.v), a(inst.ts),
                              int(inst.directed), 0, a(inst.colors), inst.problem.encode(), motif,
                              len(inst.motif or []), inst.k, inst.source, inst.dest, 1, mode, 0,
                              pre, buf, len(buf))
    wall = time.perf_counter() - t0
    if r < 0:
        print("error:", lib.tsieve_last_error().decode())
        return
    rec = json.loads(buf.value.decode())
    rec.pop("flagged", None)
    print(json.dumps({"wall_s": round(wall, 3), **rec})[:800], flush=True)


if __name__ == "__main__":
    main()
