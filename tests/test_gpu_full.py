"""Bit-exact parity at the BASELINE sizes: one named test per config, both
engines, against tests/golden/full_size.json (make_golden_full.py).

* C2 (n=1e5, m=1e6, k=6): the UNMODIFIED reference's outputs, seeds 1-4 at
  max_ts = t and one binary-search horizon (t/2).
* C3 full, C5 x0.1: the multi-threaded oracle over the whole point range.
* C4 full (k_eff = 12): sampled blocks of sieve points (the XOR over points
  is exact, so every block is independently checkable; SURVEY.md section 7,
  hard part 6), through the point engine.
* C5 full (n=1e8, m=1e9): the oracle over all 32 points, and every point's
  own partial sum for the point engine.

Engines: the coefficient engine serves every full-range call; the point
engine (`TSV_ENGINE=points`, and every partial range) is the multi-GPU path.
`tsv_profile_get` confirms which kernels ran.
"""
import json
import os

import numpy as np
import pytest

import paper_2001_07158_b200 as T
from paper_2001_07158_b200 import _native, synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu

FULL = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "full_size.json")


@pytest.fixture(scope="module")
def full_golden():
    with open(FULL) as f:
        return json.load(f)


class Cfg:
    """A BASELINE config on the device: graph, shades per seed."""

    def __init__(self, cfgno, scale=1.0):
        inst = synth.make_config(cfgno, scale=scale)
        self.k, self.colors, self.motif, self.anchor = synth.effective_query(inst)
        self.n, self.directed, self.planted = inst.n, inst.directed, inst.planted
        self.g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, 0)
        del inst
        self._sh = {}

    def shades(self, seed):
        if seed not in self._sh:
            cfg = T.SieveConfig(seed=seed, memory_cap_words=1 << 62)
            sh = T.build_shades(T.MotifQuery.from_multiset(self.motif),
                                T.VertexColoring(self.colors, int(self.colors.max())), cfg)
            self._sh[seed] = (cfg, sh, T.DeviceShades(self.g, self.k, sh))
        return self._sh[seed]

    def decide(self, seed, max_ts):
        cfg, sh, _ = self.shades(seed)
        return T.eval_temporal_sieve(self.g, self.k, max_ts, sh, cfg, T.AnchorSpec(*self.anchor))

    def points(self, seed, p0, p1, max_ts=None):
        """Raw per-vertex XOR of sieve points [p0, p1) (no finalize)."""
        import torch
        cfg, _, ds = self.shades(seed)
        acc = torch.zeros(self.n, dtype=torch.int64, device="cuda")
        T.eval_points_device(self.g, ds, self.k, max_ts or self.g.t(), cfg, self.anchor[0], p0,
                             p1, acc.data_ptr(), torch.cuda.current_stream().cuda_stream)
        return acc.cpu().numpy().view(np.uint64)


def summary(acc, sink=-1):
    a, nflag, cs = O.finalize(acc, sink)
    return {"checksum": f"{cs:016x}", "nflagged": nflag,
            "xor_total": f"{int(np.bitwise_xor.reduce(a)) if len(a) else 0:016x}"}


def outcome(out):
    return {"checksum": f"{out.checksum:016x}", "nflagged": len(out.flagged),
            "xor_total": f"{int(np.bitwise_xor.reduce(out.accumulators)):016x}"}


def want(e):
    return {key: e[key] for key in ("checksum", "nflagged", "xor_total")}


def engine_ran(name):
    return _native.Profile.get(name)[0] > 0


def check_header(c, rec):
    assert c.g.n() == rec["n"] and c.g.m() == rec["m_canonical"] and c.g.t() == rec["t_canonical"]
    assert c.k == rec["k"] and list(c.anchor) == rec["anchor"]


def run_engines(c, seed, max_ts, expect, monkeypatch):
    """Coefficient engine, then the point engine, both == expect."""
    _native.Profile.reset()
    _native.Profile.enable(True)
    try:
        got = outcome(c.decide(seed, max_ts))
        assert engine_ran("coef_arcs_last") or engine_ran("coef_vertex_last")
        assert got == expect, ("coefficient engine", seed, max_ts)
        monkeypatch.setenv("TSV_ENGINE", "points")
        _native.Profile.reset()
        got = outcome(c.decide(seed, max_ts))
        assert not engine_ran("coef_arcs_last") and not engine_ran("coef_vertex_last")
        assert engine_ran("level_last")
        assert got == expect, ("point engine", seed, max_ts)
    finally:
        monkeypatch.delenv("TSV_ENGINE", raising=False)
        _native.Profile.enable(False)


def test_full_c2_pathmotif_vs_reference(cuda_device, full_golden, monkeypatch):
    """C2 at full size: per seed and horizon, checksum / flagged / XOR equal
    the reference's own eval_temporal_sieve (sieve.cpp:170-307,35-49)."""
    rec = full_golden["C2"]
    c = Cfg(2)
    check_header(c, rec)
    for e in rec["evals"]:
        run_engines(c, e["seed"], e["max_ts"], want(e), monkeypatch)


def test_full_c3_colorfulpath_vs_oracle(cuda_device, full_golden, monkeypatch):
    rec = full_golden["C3"]
    c = Cfg(3)
    check_header(c, rec)
    e = rec["evals"][0]
    run_engines(c, e["seed"], e["max_ts"], want(e), monkeypatch)


def test_full_c5_scaled_ktemppath_vs_oracle(cuda_device, full_golden, monkeypatch):
    rec = full_golden["C5x0.1"]
    c = Cfg(5, 0.1)
    check_header(c, rec)
    e = rec["evals"][0]
    run_engines(c, e["seed"], e["max_ts"], want(e), monkeypatch)


def test_full_c4_sd_colorful_sampled_points(cuda_device, full_golden):
    """C4 at full size (k_eff = 12, 4096 points): sampled point blocks of the
    point engine against the oracle's; the planted s->d path is found."""
    rec = full_golden["C4"]
    c = Cfg(4)
    check_header(c, rec)
    for p in rec["points"]:
        got = summary(c.points(p["seed"], p["p_begin"], p["p_end"]))
        assert got == want(p), (p["p_begin"], p["p_end"])
    _native.Profile.reset()
    _native.Profile.enable(True)
    out = c.decide(1, c.g.t())
    assert engine_ran("coef_win_carry")  # the coefficient engine in time windows
    _native.Profile.enable(False)
    assert out.global_nonzero and out.flagged.tolist() == [c.n - 1]


def test_full_c4_windows_equal_point_engine(cuda_device, monkeypatch):
    """C4 at full size: the windowed coefficient engine (coef_window.cu; its
    state rows do not fit at once) and the point engine over all 4096
    points (pinned by the sampled blocks above) give the same accumulators
    and checksum, at t and at a binary-search horizon."""
    c = Cfg(4)
    for mt in (c.g.t(), c.g.t() // 2):
        coef = c.decide(1, mt)
        monkeypatch.setenv("TSV_ENGINE", "points")
        pts = c.decide(1, mt)
        monkeypatch.delenv("TSV_ENGINE")
        assert np.array_equal(coef.accumulators, pts.accumulators), mt
        assert coef.checksum == pts.checksum


def test_full_c5_ktemppath_vs_oracle(cuda_device, full_golden, monkeypatch):
    """C5 at full size (n=1e8, m=1e9): the coefficient engine's decide equals
    the oracle over all 32 points; sampled single points of the point engine
    equal the oracle's per-point partial sums; their XOR is the whole."""
    rec = full_golden["C5"]
    c = Cfg(5)
    check_header(c, rec)
    e = rec["evals"][0]
    _native.Profile.reset()
    _native.Profile.enable(True)
    got = outcome(c.decide(e["seed"], e["max_ts"]))
    assert engine_ran("coef_vertex_last")       # the vertex-lane engine (coef_vertex.cu)
    _native.Profile.enable(False)
    assert got == want(e)
    # and the arc-parallel coefficient kernels (TSV_VERTEX=0)
    monkeypatch.setenv("TSV_VERTEX", "0")
    assert outcome(c.decide(e["seed"], e["max_ts"])) == want(e)
    monkeypatch.delenv("TSV_VERTEX")
    pts = {p["p_begin"]: p for p in rec["points"]}
    for p0 in (0, 7, 31):
        got = summary(c.points(1, p0, p0 + 1))
        assert got == want(pts[p0]), p0


@pytest.mark.parametrize("n,density,sink", [(1, 1.0, -1), (1000, 0.5, -1), (8192, 1.0, -1),
                                            (8193, 0.3, -1), (100_003, 0.9, -1),
                                            (3_000_001, 0.01, -1), (3_000_001, 1.0, -1),
                                            (50_000, 1.0, 777), (50_000, 0.0, 5), (10, 1.0, 12)])
def test_device_finalize_matches_host(cuda_device, n, density, sink):
    """tsv_finalize_device (parallel FNV-1a: per-range low-byte permutations,
    then per-range hashes with the carry correction) == the reference's
    sequential finalize (sieve.cpp:136-159, 35-49)."""
    import torch
    rng = np.random.default_rng(n + int(density * 100))
    acc = rng.integers(0, 2**64 - 1, n, dtype=np.uint64, endpoint=True)
    acc[rng.random(n) >= density] = 0
    if n > 2:
        acc[1] = 0xff                       # bytes that exercise every low-byte path
        acc[2] = 1 << 63
    d = torch.from_numpy(acc.view(np.int64).copy()).cuda()
    flagged, cs = _native.finalize_device(d.data_ptr(), n, sink)
    a, nflag, cs_host = O.finalize(acc, sink)
    assert (flagged, cs) == (nflag, cs_host)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), a)
