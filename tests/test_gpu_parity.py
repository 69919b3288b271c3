"""GPU parity tests proper: the CUDA engine through the C-ABI (libtsv.so)
against the golden vectors (reference outputs) and the CPU oracle.  Bit-exact
everywhere: field arithmetic is integer work."""
import numpy as np
import pytest

import paper_2001_07158_b200 as T
from paper_2001_07158_b200 import _native, synth
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def u64(h):
    return int(h, 16)


def run_case(c, **cfgkw):
    g = T.TemporalGraph.build(c["n"], (c["u"], c["v"], c["ts"]), c["directed"], c["t"])
    col = T.VertexColoring(c["colors"], max(c["colors"]))
    cfg = T.SieveConfig(seed=c["seed"], **cfgkw)
    sh = T.build_shades(T.MotifQuery.from_multiset(c["motif"]), col, cfg)
    if not sh.feasible:
        return None
    max_ts = c["max_ts"] or g.t()
    return T.eval_temporal_sieve(g, len(c["motif"]), max_ts, sh, cfg,
                                 T.AnchorSpec(*c["anchor"]))


def test_gf_mul_device_matches_reference(cuda_device, golden):
    a = np.array([u64(x[0]) for x in golden["gf_mul"]], np.uint64)
    b = np.array([u64(x[1]) for x in golden["gf_mul"]], np.uint64)
    want = [u64(x[2]) for x in golden["gf_mul"]]
    for variant in (0, 1, 2, 3, 10):   # production, bit-serial, holes (2 forms), lane table
        assert _native.gf_mul_device(a, b, variant).tolist() == want, variant
    assert _native.gf_mul_device([1 << 63], [2]).tolist() == [0x1B]


def test_gf_mul_device_random_vs_oracle(cuda_device):
    rng = np.random.default_rng(5)
    a = rng.integers(0, 2**64 - 1, 200_000, dtype=np.uint64, endpoint=True)
    b = rng.integers(0, 2**64 - 1, 200_000, dtype=np.uint64, endpoint=True)
    a[:64] = 1 << np.arange(64, dtype=np.uint64)   # every single-bit operand
    b[:64] = np.uint64(2**64 - 1)
    got = _native.gf_mul_device(a, b)
    idx = rng.choice(len(a), 3000, replace=False).tolist() + list(range(64))
    for i in idx:
        assert int(got[i]) == O.gf_mul(int(a[i]), int(b[i]))
    # the lane-table product (gf_device.cuh LaneTable: the vertex-lane engine's
    # arc products) and the holes forms, on every pair
    for variant in (2, 3, 10):
        assert np.array_equal(_native.gf_mul_device(a, b, variant), got), variant
    assert _native.gf_mul_device([1 << 63], [2], 10).tolist() == [0x1B]
    assert _native.gf_mul_device([2**64 - 1], [2**64 - 1], 10).tolist() == \
        [O.gf_mul(2**64 - 1, 2**64 - 1)]


def test_edge_y_draws_device(cuda_device):
    edges = np.arange(0, 5000, 7, dtype=np.int32)
    for seed, level in ((1, 2), (99, 5)):
        got = _native.draw_edge_y_device(seed, level, edges)
        for e, y in zip(edges.tolist()[:200], got.tolist()[:200]):
            assert y == O.draw_nonzero(seed, 3, e, level - 1, 0)


def test_golden_sieve_cases(cuda_device, golden):
    nz = 0
    for c in golden["sieve"]:
        out = run_case(c)
        if out is None:
            assert not c["feasible"]
            continue
        assert f"{out.checksum:016x}" == c["checksum"], c["name"]
        assert out.flagged.tolist() == c["flagged"], c["name"]
        assert out.global_nonzero == c["global"], c["name"]
        if "acc" in c:
            assert [f"{int(x):016x}" for x in out.accumulators] == c["acc"], c["name"]
        nz += len(c["flagged"]) > 0
    assert nz >= 20


def level_kernels_ran():
    """Launches of the point engine's level kernels since the last reset."""
    return sum(_native.Profile.get(nm)[0] for nm in
               ("level", "level_first", "level_last", "level_grouped", "level_grouped_first"))


@pytest.fixture
def point_engine(monkeypatch):
    """Full-range calls on the point engine (TSV_ENGINE=points), with the
    per-kernel profile on so a test can assert which kernels ran."""
    monkeypatch.setenv("TSV_ENGINE", "points")
    _native.Profile.reset()
    _native.Profile.enable(True)
    yield
    _native.Profile.enable(False)


@pytest.mark.parametrize("ppb", [1, 2, 4, 8, 16, 32, 64, 128])
def test_results_independent_of_batch_width(cuda_device, golden, ppb, point_engine):
    """test_sieve.cpp:291-308 (lane/thread invariance) for every kernel shape
    of the point engine (grouped W < 32, wide W >= 32)."""
    by = {c["name"]: c for c in golden["sieve"]}
    for name in ("fig2 seed5", "C1 k-TempPath k=5", "random 3", "random 7", "random 11"):
        c = by[name]
        out = run_case(c, points_per_batch=ppb)
        if out is None:
            continue
        assert f"{out.checksum:016x}" == c["checksum"], (name, ppb)
        if "acc" in c:
            assert [f"{int(x):016x}" for x in out.accumulators] == c["acc"], (name, ppb)
    assert level_kernels_ran() > 0
    assert _native.Profile.get("coef_arcs_last")[0] == 0
    assert _native.Profile.get("level_last")[0] > 0


def test_decreasing_timestamps_no_for_every_seed(cuda_device):
    # test_sieve.cpp:92-104: soundness holds for every seed
    g = T.TemporalGraph.build(3, [(0, 1, 2), (1, 2, 1)], True)
    col = T.VertexColoring([1, 2, 3], 3)
    for seed in range(1, 21):
        cfg = T.SieveConfig(seed=seed)
        sh = T.build_shades(T.MotifQuery.from_multiset([1, 2, 3]), col, cfg)
        assert not T.eval_temporal_sieve(g, 3, g.t(), sh, cfg).global_nonzero


def _oracle_vs_gpu(n, u, v, ts, d, colors, motif, seed, anchor=(-1, -1), max_ts=None, ppb=0):
    g = T.TemporalGraph.build(n, (u, v, ts), d)
    col = T.VertexColoring(colors, int(max(colors)))
    cfg = T.SieveConfig(seed=seed, points_per_batch=ppb)
    sh = T.build_shades(T.MotifQuery.from_multiset(motif), col, cfg)
    if not sh.feasible:
        return None
    mt = max_ts or g.t()
    out = T.eval_temporal_sieve(g, len(motif), mt, sh, cfg, T.AnchorSpec(*anchor))
    cu, cv, ct = g.edges()
    acc, nf, cs = O.oracle_eval(n, cu, cv, ct, d, len(motif), mt, sh.vertex_off,
                                sh.vertex_shades, seed, anchor)
    assert np.array_equal(out.accumulators, acc)
    assert out.checksum == cs
    return nf


def test_random_sweep_vs_oracle(cuda_device):
    rng = np.random.default_rng(123)
    nz = 0
    for i in range(120):
        n, u, v, ts, d, colors, motif = synth.random_small(rng, n_max=30, m_max=120, t_max=10,
                                                           k_max=7)
        anchor = (-1, -1)
        if i % 3 == 0:
            s, dd = rng.choice(n, 2, replace=False)
            anchor = (int(s), int(dd))
        cu, _, ct = O.canonical_edges(n, u, v, ts, d)
        tmax = int(ct.max()) if len(ct) else 1
        nf = _oracle_vs_gpu(n, u, v, ts, d, colors, motif, int(rng.integers(1, 1 << 40)), anchor,
                            int(rng.integers(1, tmax + 1)), ppb=int(rng.choice([0, 1, 4, 32])))
        nz += bool(nf)
    assert nz > 15


def test_hub_vertices_split_across_chunks(cuda_device):
    """A head with far more in-arcs than a chunk holds is split into pieces
    whose per-vertex prefix is repaired by the carry fix-up kernel."""
    rng = np.random.default_rng(9)
    n, m, t = 300, 12000, 60
    u = rng.integers(0, n, m)
    v = np.where(rng.random(m) < 0.5, 0, rng.integers(0, n, m))   # vertex 0 is a hub
    v = np.where(rng.random(m) < 0.2, 1, v)                        # vertex 1 too
    ts = rng.integers(1, t + 1, m)
    colors = rng.integers(1, 4, n)
    g = T.TemporalGraph.build(n, (u, v, ts), True)
    assert g.info.split_chunks > 0
    for motif in ([1, 1, 2, 3], [1, 2, 3, 1, 2]):
        for seed in (1, 77):
            assert _oracle_vs_gpu(n, u, v, ts, True, colors, motif, seed) >= 0
    assert _oracle_vs_gpu(n, u, v, ts, False, colors, [1, 2, 3], 5) >= 0


@pytest.mark.parametrize("env", [{}, {"TSV_YMUL": "holes"}])
@pytest.mark.parametrize("ppb", [4, 16, 64])
def test_engine_paths_agree(cuda_device, monkeypatch, env, ppb, point_engine):
    """Grouped and wide kernels of the point engine (and the wide kernel's
    holes product for y instead of the tables) give the oracle's
    accumulators with hub vertices split across chunks (carry fix-up into
    state slots), horizons below t (fused readout of the last run <= max_ts)
    and compacted state rows."""
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(31)
    n, m, t = 200, 6000, 40
    u = rng.integers(0, n, m)
    v = np.where(rng.random(m) < 0.4, 0, rng.integers(0, n, m))
    ts = rng.integers(1, t + 1, m)
    colors = rng.integers(1, 4, n)
    for motif, seed, mt in (([1, 1, 2, 3], 3, None), ([1, 2, 3, 1, 2], 8, 25),
                            ([1, 2, 3, 1, 2, 3], 11, 33)):
        _oracle_vs_gpu(n, u, v, ts, True, colors, motif, seed, max_ts=mt, ppb=ppb)
    _oracle_vs_gpu(n, u, v, ts, False, colors, [1, 2, 3], 5, max_ts=20, ppb=ppb)
    assert _native.Profile.get("level_grouped" if ppb < 32 else "level")[0] > 0
    assert _native.Profile.get("fixup")[0] > 0


@pytest.mark.parametrize("ppb", [1, 2, 4, 8, 16, 32, 64, 128])
def test_partial_point_ranges_vs_oracle(cuda_device, ppb):
    """The multi-GPU path: partial sieve-point ranges [a, b) (every call on
    the point engine) equal the oracle's partial sums for the same range, at
    every batch width; hubs split across chunks, anchors, horizons below t,
    undirected graphs.  Ranges that are not multiples of the width exercise
    the idle lanes of the last batch."""
    import torch
    rng = np.random.default_rng(100 + ppb)
    n, m, t = 160, 5000, 30
    u = rng.integers(0, n, m)
    v = np.where(rng.random(m) < 0.35, 0, rng.integers(0, n, m))     # hub
    ts = rng.integers(1, t + 1, m)
    colors = rng.integers(1, 5, n)
    _native.Profile.reset()
    _native.Profile.enable(True)
    try:
        for directed, motif, seed, mt, anchor in (
                (True, [1, 1, 2, 3, 4], 3, None, (-1, -1)),
                (True, [1, 2, 3, 4, 1, 2], 5, 22, (-1, -1)),
                (True, [1, 2, 3, 4, 4, 3, 2], 7, None, (4, 9)),
                (False, [1, 2, 3, 1], 9, 17, (-1, -1))):
            g = T.TemporalGraph.build(n, (u, v, ts), directed)
            col = T.VertexColoring(colors, int(colors.max()))
            cfg = T.SieveConfig(seed=seed, points_per_batch=ppb)
            sh = T.build_shades(T.MotifQuery.from_multiset(motif), col, cfg)
            ds = T.DeviceShades(g, len(motif), sh)
            k = len(motif)
            P = 1 << k
            cu, cv, ct = g.edges()
            mt = mt or g.t()
            for a, b in ((0, 1), (3, min(P, 3 + ppb)), (1, P // 2 + 3), (P // 2, P), (P - 1, P),
                         (5, P - 2)):
                acc = torch.zeros(n, dtype=torch.int64, device="cuda")
                T.eval_points_device(g, ds, k, mt, cfg, anchor[0], a, b, acc.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream)
                got = acc.cpu().numpy().view(np.uint64)
                want = O.eval_points(n, cu, cv, ct, directed, k, mt, sh.vertex_off,
                                     sh.vertex_shades, seed, anchor[0], a, b)
                assert np.array_equal(got, want), (directed, motif, a, b)
        assert level_kernels_ran() > 0
        assert _native.Profile.get("coef_arcs_last")[0] == 0
    finally:
        _native.Profile.enable(False)


@pytest.mark.parametrize("env", [{"TSV_ENGINE": "points"}, {"TSV_ITEMS": "0"}, {"TSV_VERTEX": "0"},
                                 {"TSV_ITEMS": "1", "TSV_ITEMS_REG": "0"}, {"TSV_ITEMS": "1"},
                                 {"TSV_ZTRANS": "tab"}, {"TSV_SUBGRAPH": "0"},
                                 {"TSV_PERSIST": "0"}, {"TSV_WALK_SPLIT": "0"}])
def test_coefficient_engine_kernels_agree(cuda_device, monkeypatch, env):
    """Every arc kernel of the coefficient engine (k_coef_arcs, the item
    stream k_coef_items, its register-walk form k_coef_items_reg for frames
    <= 64 words, one and two entries per lane), both z maps of multi-shade
    rows (direct and table), with and without the shaded subgraph (arcs
    touching shadeless vertices dropped, edge ids kept) and the persistent
    chunk loop, with and without the half-warp split walk (frames <= 16),
    and the point engine give the
    oracle's accumulators: single-shade, multi-shade and shadeless vertices,
    hubs split across chunks, horizons below t, (s,d) anchors, undirected
    graphs, k = 2..8."""
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(47)
    n, m, t = 200, 6000, 40
    u = rng.integers(0, n, m)
    v = np.where(rng.random(m) < 0.3, 0, rng.integers(0, n, m))
    ts = rng.integers(1, t + 1, m)
    colors = rng.integers(1, 6, n)            # color 5 is in no motif: shadeless vertices
    nz = 0
    for motif, seed, mt, anchor in (([1, 2], 2, None, (-1, -1)),
                                     ([1, 2, 3], 4, 30, (-1, -1)),
                                     ([1, 1, 2, 3], 3, None, (-1, -1)),
                                     ([1, 2, 3, 4, 1], 8, 25, (-1, -1)),
                                     ([1, 1, 2, 3, 4, 2], 11, None, (-1, -1)),
                                     ([1, 2, 3, 4, 1, 2, 3], 13, 35, (-1, -1)),
                                     ([1, 2, 3, 4, 1, 2, 3, 4], 17, None, (-1, -1)),
                                     ([1, 2, 3, 4], 19, None, (3, 0)),
                                     ([1, 2, 3, 4, 2, 3], 23, 31, (5, 7))):
        nz += bool(_oracle_vs_gpu(n, u, v, ts, True, colors, motif, seed, anchor, mt))
    # every vertex carries every shade (k-TempPath): multi-shade frames only
    one = np.ones(n, np.int64)
    for k_ in (5, 6, 7):
        nz += bool(_oracle_vs_gpu(n, u, v, ts, True, one, [1] * k_, 29 + k_))
    nz += bool(_oracle_vs_gpu(n, u, v, ts, False, colors, [1, 1, 2, 3, 4, 2], 31, max_ts=20))
    assert nz >= 8


@pytest.mark.parametrize("rows,env", [(300, {}), (1200, {}), (700, {"TSV_ITEMS": "0"}),
                                      (900, {"TSV_ITEMS": "1", "TSV_ITEMS_REG": "0"}),
                                      (500, {"TSV_SUBGRAPH": "0"})])
def test_time_windows_vs_oracle(cuda_device, monkeypatch, rows, env):
    """The coefficient engine in time windows (coef_window.cu: arcs in
    windows of consecutive timestamps, per-vertex carries of every level,
    carry slots for sources before the window, ulast accumulated over the
    windows) equals the oracle: single-, multi-shade and shadeless
    vertices, horizons below t, (s,d) anchors, undirected graphs, k = 2..8,
    item-stream and k_coef_arcs paths.  TSV_WINDOW_ROWS caps the arcs per
    window (the engine windows by itself when the rows do not fit)."""
    monkeypatch.setenv("TSV_WINDOW_ROWS", str(rows))
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(rows)
    n, m, t = 150, 5000, 60
    u = rng.integers(0, n, m)
    v = np.where(rng.random(m) < 0.2, 0, rng.integers(0, n, m))
    ts = rng.integers(1, t + 1, m)
    colors = rng.integers(1, 6, n)            # color 5: shadeless vertices
    _native.Profile.reset()
    _native.Profile.enable(True)
    try:
        nz = 0
        for motif, seed, mt, anchor, d in (([1, 2], 2, None, (-1, -1), True),
                                           ([1, 2, 3], 4, 45, (-1, -1), True),
                                           ([1, 1, 2, 3], 3, None, (-1, -1), True),
                                           ([1, 2, 3, 4, 1], 8, 33, (-1, -1), True),
                                           ([1, 1, 2, 3, 4, 2], 11, None, (-1, -1), True),
                                           ([1, 2, 3, 4, 1, 2, 3, 4], 17, None, (-1, -1), True),
                                           ([1, 2, 3, 4], 19, None, (3, 0), True),
                                           ([1, 2, 3, 4, 2, 3], 23, 50, (5, 7), True),
                                           ([1, 1, 2, 3, 4, 2], 31, 40, (-1, -1), False),
                                           ([1, 2, 3, 4, 1], 37, None, (-1, -1), False)):
            nz += bool(_oracle_vs_gpu(n, u, v, ts, d, colors, motif, seed, anchor, mt))
        assert nz >= 6
        assert _native.Profile.get("coef_win_carry")[0] > 0
    finally:
        _native.Profile.enable(False)


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_vertex_engine_vs_oracle(cuda_device, k):
    """The vertex-lane coefficient engine (coef_vertex.cu; every shaded vertex
    multi-shade, k <= 5 -- k-TempPath, C5's query): oracle accumulators for
    directed and undirected graphs, (s,d) anchors, horizons below t, shadeless
    vertices, and a graph with a hub above the engine's in-degree bound
    (which must fall back to the arc-parallel kernels)."""
    rng = np.random.default_rng(70 + k)
    n, m, t = 300, 5000, 50
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    ts = rng.integers(1, t + 1, m)
    ones = np.ones(n, np.int64)
    two = rng.integers(1, 4, n)              # colors 1, 2 shaded twice; 3 shadeless
    _native.Profile.reset()
    _native.Profile.enable(True)
    try:
        nz = 0
        for d, colors, motif, seed, mt, anchor in (
                (True, ones, [1] * k, 3, None, (-1, -1)),
                (False, ones, [1] * k, 5, 31, (-1, -1)),
                (True, ones, [1] * k, 7, None, (4, 11)),
                (True, two, {2: [1, 1], 3: [1, 1, 1], 4: [1, 1, 2, 2], 5: [1, 1, 2, 2, 2]}[k],
                 9, 40, (-1, -1))):
            nz += bool(_oracle_vs_gpu(n, u, v, ts, d, colors, motif, seed, anchor, mt))
        assert nz >= 2
        assert _native.Profile.get("coef_vertex_last")[0] > 0
        # every kind of horizon (a probe below t stops each vertex at its first
        # arc past it): the first timestamp, the middle, t - 1, with an anchor
        for mt, anchor in ((1, (-1, -1)), (2, (-1, -1)), (t // 3, (-1, -1)), (t // 2, (4, 11)),
                           (t - 1, (-1, -1)), (t, (4, 11))):
            _oracle_vs_gpu(n, u, v, ts, True, ones, [1] * k, 21 + mt, anchor, mt)
            _oracle_vs_gpu(n, u, v, ts, False, ones, [1] * k, 22 + mt, anchor, mt)
        # hub above the in-degree bound (4096 arcs): the arc kernels take over
        hv = np.concatenate([v, np.zeros(5000, np.int64)])
        hu = np.concatenate([u, rng.integers(1, n, 5000)])
        hts = np.concatenate([ts, rng.integers(1, t + 1, 5000)])
        _native.Profile.reset()
        _oracle_vs_gpu(n, hu, hv, hts, True, ones, [1] * k, 13)
        assert _native.Profile.get("coef_vertex_last")[0] == 0
    finally:
        _native.Profile.enable(False)


@pytest.mark.parametrize("env", [{}, {"TSV_ENGINE": "points"}])
def test_coefficient_engine_large_k_vs_oracle(cuda_device, monkeypatch, env):
    """k = 9..12 (C4's k_eff is 12): frames above 64 words take the shared-
    memory item kernel, multi-shade rows the direct z map with up to 924
    entries per row; colorful, repeated-color and anchored queries, hubs."""
    for k_, v_ in env.items():
        monkeypatch.setenv(k_, v_)
    rng = np.random.default_rng(61)
    n, m, t = 90, 2500, 60
    u = rng.integers(0, n, m)
    v = np.where(rng.random(m) < 0.25, 0, rng.integers(0, n, m))
    ts = rng.integers(1, t + 1, m)
    colors = rng.integers(1, 13, n)                # 12 colors; 13+ absent
    nz = 0
    for motif, seed, mt, anchor in ((list(range(1, 10)), 3, None, (-1, -1)),
                                     ([1, 1, 2, 3, 4, 5, 6, 7, 8, 9], 5, 50, (-1, -1)),
                                     (list(range(1, 12)), 7, None, (2, 5)),
                                     ([1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12], 9, None, (-1, -1)),
                                     ([1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6], 11, 45, (-1, -1))):
        nz += bool(_oracle_vs_gpu(n, u, v, ts, True, colors, motif, seed, anchor, mt))
    assert nz == 5


def test_c2_shape_small_scale_vs_oracle(cuda_device):
    inst = synth.make_config(2, scale=0.01)   # n=1e3, m=1e4, k=6 PathMotif
    k, col, motif, anchor = synth.effective_query(inst)
    nf = _oracle_vs_gpu(inst.n, inst.u, inst.v, inst.ts, True, col, motif, 1)
    assert nf > 0  # the planted path is found


def test_sd_anchor_vs_oracle(cuda_device):
    inst = synth.make_config(4, scale=0.0001)  # n=100, m=1e4, k_eff=12
    k, col, motif, anchor = synth.effective_query(inst)
    nf = _oracle_vs_gpu(inst.n, inst.u, inst.v, inst.ts, True, col, motif, 3, anchor)
    assert nf == 1  # only the sink is kept


def test_memory_cap_raises(cuda_device):
    # test_sieve.cpp:364-371: cap -> std::runtime_error
    rng = np.random.default_rng(5)
    g = T.TemporalGraph.build(60, (rng.integers(0, 60, 240), rng.integers(0, 60, 240),
                                   rng.integers(1, 13, 240)), False)
    col = T.VertexColoring(rng.integers(1, 4, 60), 3)
    cfg = T.SieveConfig(memory_cap_words=100)
    sh = T.build_shades(T.MotifQuery.from_multiset([1, 2, 3]), col, cfg)
    with pytest.raises(MemoryError, match="memory cap exceeded"):
        T.eval_temporal_sieve(g, 3, g.t(), sh, cfg)


def test_argument_errors(cuda_device):
    g = T.TemporalGraph.build(3, [(0, 1, 1), (1, 2, 2)], True)
    col = T.VertexColoring([1, 2, 3], 3)
    sh = T.build_shades(T.MotifQuery.from_multiset([1, 2, 3]), col, T.SieveConfig())
    with pytest.raises(ValueError, match="max_ts outside"):
        T.eval_temporal_sieve(g, 3, 5, sh, T.SieveConfig())
    with pytest.raises(ValueError, match="field_bits"):
        T.eval_temporal_sieve(g, 3, 2, sh, T.SieveConfig(field_bits=12))
    with pytest.raises(ValueError, match="endpoint out of range"):
        T.TemporalGraph.build(3, [(0, 4, 1)], True)


@pytest.mark.parametrize("bits", [8, 16, 32])
def test_small_fields_vs_reference(cuda_device, bits):
    """GF(2^8 / 2^16 / 2^32) (small_field.cu; the reference's --field-bits,
    tools/main.cpp:70) against the reference's own eval_temporal_sieve at the
    same width (oracle/_ref, temporal_impl<Word> through sieve.cpp:637-649):
    accumulators, checksum and the false-negative bound (2k-1)/2^b; small
    fields do produce false negatives, so zero accumulators must agree too."""
    assert O.ref_available()
    rng = np.random.default_rng(bits)
    nz = 0
    try:
        for i in range(40):
            n, u, v, ts, d, colors, motif = synth.random_small(rng, n_max=40, m_max=200,
                                                               t_max=12, k_max=6)
            cu, _, ct = O.canonical_edges(n, u, v, ts, d)
            if len(cu) == 0:
                continue
            tmax = int(ct.max())
            mt = int(rng.integers(1, tmax + 1)) if i % 2 else tmax
            anchor = (-1, -1)
            if i % 4 == 1:
                s_, dd = rng.choice(n, 2, replace=False)
                anchor = (int(s_), int(dd))
            seed = int(rng.integers(1, 1 << 40))
            ref = O.ref_eval(n, u, v, ts, d, colors, motif, max_ts=mt, seed=seed, anchor=anchor,
                             field_bits=bits)
            if ref is None:
                continue
            g = T.TemporalGraph.build(n, (u, v, ts), d)
            cfg = T.SieveConfig(seed=seed, field_bits=bits)
            sh = T.build_shades(T.MotifQuery.from_multiset(motif),
                                T.VertexColoring(colors, int(max(colors))), cfg)
            out = T.eval_temporal_sieve(g, len(motif), mt, sh, cfg, T.AnchorSpec(*anchor))
            assert np.array_equal(out.accumulators, ref["acc"]), (i, bits)
            assert out.checksum == ref["checksum"]
            assert out.fn_bound == (2 * len(motif) - 1) / 2.0 ** bits
            assert int(out.accumulators.max(initial=0)) < (1 << bits)
            nz += ref["nflagged"] > 0
    finally:
        O.ref_lib().ref_set_field_bits(64)
    assert nz >= 5


@pytest.mark.parametrize("directed", [True, False])
def test_device_static_projection_matches_host_grouping(cuda_device, directed):
    """tsv_graph_static_edges (the radix-sorted projection the C++
    StaticProjection::project uses from 2^22 edges on) equals the
    reference's grouping (graph.cpp:148-199: stable sort of the canonical
    edges by their oriented (u, v), pairs ascending, edge ids increasing
    within a pair) -- here restated with numpy on the same canonical list;
    repeated pairs (few vertices, many timestamps) and self-loops dropped by
    the build."""
    rng = np.random.default_rng(5 if directed else 6)
    n, m = 300, 200_000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    ts = rng.integers(1, 5000, m)
    g = T.TemporalGraph.build(n, (u, v, ts), directed)
    a, b, off, back = g.static_projection()
    cu, cv, _ = g.edges()
    cu, cv = cu.astype(np.int64), cv.astype(np.int64)
    if not directed:
        cu, cv = np.minimum(cu, cv), np.maximum(cu, cv)
    key = cu * n + cv
    order = np.argsort(key, kind="stable")
    uk, first = np.unique(key[order], return_index=True)
    assert np.array_equal(a, uk // n) and np.array_equal(b, uk % n)
    assert np.array_equal(off, np.append(first, len(key)))
    assert np.array_equal(back, order)
    assert len(uk) < g.m()  # repeated pairs were grouped


@pytest.mark.parametrize("junction", [1, 0])
def test_static_coefficient_engine_equals_point_engine(cuda_device, monkeypatch, junction):
    """The junction / static sieves on the projection in coefficient form
    (coef_static.cu: walks-ending and walks-starting families as top-degree
    rows, readout XOR_b E_{k+1-b} * S_b on complementary subsets) equal the
    point form (static_kernels.cu, every sieve point; pinned against the
    reference through test_default_preprocessing_matches_reference):
    single-, multi-shade and shadeless vertices, directed and undirected
    projections with repeated vertices, k = 1..12."""
    import ctypes as C
    L = _native.lib()
    rng = np.random.default_rng(41 + junction)
    nz = 0
    for i in range(24):
        n = int(rng.integers(3, 60))
        ms = int(rng.integers(1, 400))
        a = rng.integers(0, n, ms).astype(np.int32)
        b = rng.integers(0, n, ms).astype(np.int32)
        keep = a != b
        a, b = a[keep], b[keep]
        directed = int(i % 2)
        k = int(rng.integers(1, 9)) if i < 18 else int(rng.integers(9, 13))  # up to C4's 12
        q = int(rng.integers(1, 5))
        colors = rng.integers(1, q + 2, n).astype(np.int32)  # color q+1: no shade
        motif = sorted(int(x) for x in rng.integers(1, q + 1, k))
        cfg = T.SieveConfig(seed=int(rng.integers(1, 1 << 30)), memory_cap_words=1 << 62)
        sh = T.build_shades(T.MotifQuery.from_multiset(motif), T.VertexColoring(colors, q + 1),
                            cfg)
        vs = np.ascontiguousarray(sh.vertex_shades if len(sh.vertex_shades) else
                                  np.zeros(1, np.int32), np.int32)
        voff = np.ascontiguousarray(sh.vertex_off, np.int32)
        res = []
        for engine in ("coef", "points"):
            if engine == "points":
                monkeypatch.setenv("TSV_STATIC_ENGINE", "points")
            acc = np.zeros(n, np.uint64)
            o = _native.Outcome()
            c = cfg.to_native()
            _native.check(L.tsv_eval_static_projection(n, len(a), np.ascontiguousarray(a),
                                                       np.ascontiguousarray(b), directed,
                                                       junction, k, voff, vs, C.byref(c), 0,
                                                       acc, C.byref(o)))
            res.append((acc, o.checksum))
            monkeypatch.delenv("TSV_STATIC_ENGINE", raising=False)
        assert np.array_equal(res[0][0], res[1][0]), (i, k, directed, motif)
        assert res[0][1] == res[1][1]
        nz += int(res[0][0].any())
    assert nz >= 8


def test_device_points_api_shards_xor_to_full(cuda_device, golden):
    """tsv_eval_points_device over disjoint point ranges + tsv_xor_combine_device
    reproduces the full evaluation (the multi-GPU sieve-point sharding path)."""
    import torch
    c = next(c for c in golden["sieve"] if c["name"] == "C1 k-TempPath k=5")
    g = T.TemporalGraph.build(c["n"], (c["u"], c["v"], c["ts"]), True)
    cfg = T.SieveConfig(seed=1)
    sh = T.build_shades(T.MotifQuery.from_multiset(c["motif"]),
                        T.VertexColoring(c["colors"], 1), cfg)
    ds = T.DeviceShades(g, 5, sh)
    parts = torch.zeros((4, g.n()), dtype=torch.int64, device="cuda")
    bounds = [0, 5, 16, 17, 32]
    stream = torch.cuda.current_stream().cuda_stream
    for i in range(4):
        T.eval_points_device(g, ds, 5, g.t(), cfg, -1, bounds[i], bounds[i + 1],
                             parts[i].data_ptr(), stream)
    total = torch.zeros(g.n(), dtype=torch.int64, device="cuda")
    T.xor_combine_device(parts.data_ptr(), 4, g.n(), total.data_ptr(), stream)
    acc = total.cpu().numpy().view(np.uint64)
    acc, nflag, cs = T.finalize(acc)
    assert f"{cs:016x}" == c["checksum"]
    assert [f"{int(x):016x}" for x in acc] == c["acc"]


def test_device_build_matches_host_build(cuda_device):
    """The on-device graph build (CUB sort + own kernels) yields the same
    canonical edge ids, drop counts and sieve results as the host layout."""
    import os
    rng = np.random.default_rng(21)
    for directed in (True, False):
        n, m, t = 500, 6000, 30
        u = rng.integers(0, n, m)
        v = np.where(rng.random(m) < 0.3, 7, rng.integers(0, n, m))   # a hub + loops + dups
        ts = rng.integers(1, t + 1, m)
        u[:50], v[:50], ts[:50] = u[50:100], v[50:100], ts[50:100]    # duplicates
        graphs = {}
        for mode in ("0", "1"):
            os.environ["TSV_HOST_BUILD"] = mode
            try:
                graphs[mode] = T.TemporalGraph.build(n, (u, v, ts), directed)
            finally:
                os.environ.pop("TSV_HOST_BUILD", None)
        gd, gh = graphs["0"], graphs["1"]
        for a, b in zip(gd.edges(), gh.edges()):
            assert np.array_equal(a, b)
        for f in ("m", "arcs", "runs", "dropped_self_loops", "dropped_duplicates", "t"):
            assert getattr(gd.info, f) == getattr(gh.info, f), f
        col = T.VertexColoring(rng.integers(1, 4, n), 3)
        cfg = T.SieveConfig(seed=4)
        sh = T.build_shades(T.MotifQuery.from_multiset([1, 2, 3, 1]), col, cfg)
        od = T.eval_temporal_sieve(gd, 4, gd.t(), sh, cfg)
        oh = T.eval_temporal_sieve(gh, 4, gh.t(), sh, cfg)
        assert np.array_equal(od.accumulators, oh.accumulators) and od.checksum == oh.checksum
        assert od.global_nonzero
    with pytest.raises(ValueError, match="timestamp below 1"):
        T.TemporalGraph.build(3, [(0, 1, 1), (1, 2, 0)], True)
    g0 = T.TemporalGraph.build(4, np.zeros((0, 3), np.int64), True)
    assert g0.m() == 0 and g0.info.arcs == 0


def test_device_restrict_matches_reference_renumbering(cuda_device):
    """tsv_graph_restrict (device, order-preserving) equals rebuilding the
    kept edges from scratch (restrict_to, graph.cpp:483-494), and the sieve on
    it equals the oracle on the restricted edge list."""
    rng = np.random.default_rng(33)
    for directed in (True, False):
        n, m, t = 80, 900, 12
        u, v, ts = rng.integers(0, n, m), rng.integers(0, n, m), rng.integers(1, t + 1, m)
        g = T.TemporalGraph.build(n, (u, v, ts), directed)
        keep = rng.random(n) < 0.7
        for max_ts in (t, 7):
            r = T.restrict_to(g, keep, max_ts)
            cu, cv, ct = g.edges()
            sel = (ct <= max_ts) & keep[cu] & keep[cv]
            ref = T.TemporalGraph.build(n, (cu[sel], cv[sel], ct[sel]), directed, min(max_ts, g.t()))
            for a, b in zip(r.edges(), ref.edges()):
                assert np.array_equal(a, b)
            assert r.t() == ref.t() and r.info.runs == ref.info.runs
            col = T.VertexColoring(rng.integers(1, 3, n), 2)
            cfg = T.SieveConfig(seed=9)
            sh = T.build_shades(T.MotifQuery.from_multiset([1, 2, 1]), col, cfg)
            o1 = T.eval_temporal_sieve(r, 3, r.t(), sh, cfg)
            acc, nf, cs = O.oracle_eval(n, *r.edges(), directed, 3, r.t(), sh.vertex_off,
                                        sh.vertex_shades, 9)
            assert np.array_equal(o1.accumulators, acc) and o1.checksum == cs


def _decide_points(g, ds, k, cfg, anchor_src, p0, p1):
    import torch
    acc = torch.zeros(g.n(), dtype=torch.int64, device="cuda")
    T.eval_points_device(g, ds, k, g.t(), cfg, anchor_src, p0, p1, acc.data_ptr(),
                         torch.cuda.current_stream().cuda_stream)
    return acc.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("cfgno,scale", [(2, 1.0), (5, 0.01)])
def test_full_size_properties(cuda_device, monkeypatch, cfgno, scale):
    """Size-independent properties at BASELINE sizes (the bit-exact full-size
    goldens are test_gpu_full.py's): (1) the point engine's accumulators do
    not depend on the batch width (wide W=64/32 and grouped W=8/4 kernels
    agree bit for bit) and equal the coefficient engine's;
    (2) sieve points are independent: XOR of disjoint point ranges = whole;
    (3) the planted path is found; (4) restricted to the planted path's
    vertices the engine equals the oracle exactly."""
    inst = synth.make_config(cfgno, scale=scale)
    k, col, motif, anchor = synth.effective_query(inst)
    g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed)
    cfg = T.SieveConfig(seed=3, memory_cap_words=1 << 62)
    sh = T.build_shades(T.MotifQuery.from_multiset(motif), T.VertexColoring(col, int(col.max())),
                        cfg)
    ds = T.DeviceShades(g, k, sh)
    P = 1 << k
    ref = None
    monkeypatch.setenv("TSV_ENGINE", "points")      # the width loop is the point engine's
    for ppb in (64, 32, 8, 4):
        c = T.SieveConfig(seed=3, points_per_batch=ppb, memory_cap_words=1 << 62)
        acc = _decide_points(g, ds, k, c, anchor[0], 0, P)
        if ref is None:
            ref = acc
        assert np.array_equal(acc, ref), ppb
    monkeypatch.delenv("TSV_ENGINE")
    # the coefficient engine (full range) equals the point engine
    assert np.array_equal(_decide_points(g, ds, k, cfg, anchor[0], 0, P), ref)
    parts = [_decide_points(g, ds, k, cfg, anchor[0], a, b)
             for a, b in ((0, 5), (5, P // 2), (P // 2, P - 1), (P - 1, P))]
    assert np.array_equal(parts[0] ^ parts[1] ^ parts[2] ^ parts[3], ref)
    fin, nflag, cs = T.finalize(ref, anchor[1])
    assert nflag > 0
    keep = np.zeros(inst.n, bool)
    keep[inst.planted] = True
    r = T.restrict_to(g, keep, g.t())
    out = T.eval_temporal_sieve(r, k, r.t(), sh, cfg, T.AnchorSpec(*anchor))
    acc, nf, cs2 = O.oracle_eval(inst.n, *r.edges(), inst.directed, k, r.t(), sh.vertex_off,
                                 sh.vertex_shades, 3, anchor)
    assert np.array_equal(out.accumulators, acc) and out.checksum == cs2
    assert int(inst.planted[-1]) in out.flagged.tolist()


@pytest.mark.parametrize("model", ["transition", "delay", "transition_delay", "instant"])
def test_edge_models_vs_reference(cuda_device, model):
    """Transition-time and vertex-delay models (sieve.cpp:257-291) against the
    reference itself (oracle/_ref): an arc departing at ts lands at
    ts + eps - 1 and reads its tail's state at ts - delta(tail); every kernel
    shape, anchors, horizons below t, duplicates and self loops."""
    rng = np.random.default_rng({"transition": 1, "delay": 2, "transition_delay": 3,
                                 "instant": 4}[model])
    nz = 0
    for i in range(60):
        n = int(rng.integers(3, 25))
        m = int(rng.integers(1, 90))
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        ts = rng.integers(1, 12, m)
        eps = rng.integers(1, 4, m)
        delays = rng.integers(0, 4, n) if i % 4 else None
        directed = bool(rng.integers(0, 2))
        k = int(rng.integers(1, 6))
        q = int(rng.integers(1, 4))
        colors = rng.integers(1, q + 1, n)
        motif = sorted(rng.integers(1, q + 1, k).tolist())
        anchor = (-1, -1)
        if i % 5 == 0:
            s, d = rng.choice(n, 2, replace=False)
            anchor = (int(s), int(d))
        seed = int(rng.integers(1, 1 << 30))
        ppb = int(rng.choice([0, 1, 4, 32, 64]))
        want = O.ref_eval_temporal_model(n, u, v, ts, eps, delays, directed, colors, motif,
                                         T.EDGE_MODELS[model], seed=seed, anchor=anchor)
        if want is None:
            continue
        tmax = int(want["ts"].max()) if len(want["ts"]) else 1
        max_ts = int(rng.integers(1, tmax + 1))
        want = O.ref_eval_temporal_model(n, u, v, ts, eps, delays, directed, colors, motif,
                                         T.EDGE_MODELS[model], seed=seed, anchor=anchor,
                                         max_ts=max_ts)
        g = T.TemporalGraph.build_model(n, (u, v, ts), directed, model, eps=eps, delays=delays)
        cfg = T.SieveConfig(seed=seed, edge_model=model, points_per_batch=ppb)
        sh = T.build_shades(T.MotifQuery.from_multiset(motif), T.VertexColoring(colors, q), cfg)
        out = T.eval_temporal_sieve(g, k, max_ts, sh, cfg, T.AnchorSpec(*anchor))
        assert np.array_equal(out.accumulators, want["acc"]), (model, i)
        assert out.checksum == want["checksum"], (model, i)
        nz += bool(out.global_nonzero)
    assert nz > 5


def test_edge_model_mismatch_is_rejected(cuda_device):
    g = T.TemporalGraph.build_model(3, [(0, 1, 1), (1, 2, 3)], True, "transition", eps=[2, 1])
    col = T.VertexColoring([1, 2, 3], 3)
    cfg = T.SieveConfig()
    sh = T.build_shades(T.MotifQuery.from_multiset([1, 2, 3]), col, cfg)
    with pytest.raises(ValueError, match="edge model"):
        T.eval_temporal_sieve(g, 3, g.t(), sh, cfg)
    with pytest.raises(ValueError, match="transition time below 1"):
        T.TemporalGraph.build_model(3, [(0, 1, 1)], True, "transition", eps=[0])


def test_edges_rebuilt_from_layout(cuda_device, monkeypatch):
    """Large device-built graphs keep no canonical edge list (neither in HBM
    nor on the host): edges(), restriction and the EC engine rebuild it from
    the arc layout.  Forced here on small graphs (TSV_EDGES_IN_LAYOUT=1) and
    compared with the stored-list build."""
    rng = np.random.default_rng(44)
    for directed in (True, False):
        n, m, t = 300, 5000, 40
        u = rng.integers(0, n, m)
        v = np.where(rng.random(m) < 0.3, 3, rng.integers(0, n, m))
        ts = rng.integers(1, t + 1, m)
        ref = T.TemporalGraph.build(n, (u, v, ts), directed)
        monkeypatch.setenv("TSV_EDGES_IN_LAYOUT", "1")
        g = T.TemporalGraph.build(n, (u, v, ts), directed)
        monkeypatch.delenv("TSV_EDGES_IN_LAYOUT")
        for a, b in zip(g.edges(), ref.edges()):
            assert np.array_equal(a, b)
        keep = rng.random(n) < 0.8
        r1 = T.restrict_to(g, keep, 30)
        r2 = T.restrict_to(ref, keep, 30)
        for a, b in zip(r1.edges(), r2.edges()):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_vertex_partitioned_simulated_equals_single(cuda_device, world):
    """The multi-GPU form of the vertex-lane engine (tsv_vertex_partition +
    tsv_eval_vertex_level per rank; shard.eval_vertex_simulated runs the ranks
    one after the other on this device, so the row all-gather is the identity)
    gives the single-GPU accumulators and the oracle's, with anchors and
    horizons; the ranks' state-row ranges tile [0, slots)."""
    import torch
    from paper_2001_07158_b200.shard import eval_vertex_simulated
    rng = np.random.default_rng(90 + world)
    n, m, t = 500, 8000, 60
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    ts = rng.integers(1, t + 1, m)
    for k, seed, mt, anchor, directed in ((5, 3, None, (-1, -1), True), (4, 5, 40, (7, 9), True),
                                          (3, 9, None, (-1, -1), False)):
        g = T.TemporalGraph.build(n, (u, v, ts), directed)
        cfg = T.SieveConfig(seed=seed)
        sh = T.build_shades(T.MotifQuery.from_multiset([1] * k), T.VertexColoring.uniform(n),
                            cfg)
        ds = T.DeviceShades(g, k, sh)
        mt = mt or g.t()
        acc = torch.zeros(n, dtype=torch.int64, device="cuda")
        acc, _, parts = eval_vertex_simulated(g, ds, k, mt, cfg, anchor[0], acc, world)
        got = acc.cpu().numpy().view(np.uint64)
        assert parts[0].slot_lo == 0 and parts[-1].slot_hi == parts[0].slots
        assert all(a.slot_hi == b.slot_lo for a, b in zip(parts, parts[1:]))
        cu, cv, ct = g.edges()
        want = O.eval_points(n, cu, cv, ct, directed, k, mt, sh.vertex_off, sh.vertex_shades, seed,
                             anchor[0])
        assert np.array_equal(got, want), (k, world)
        if world > 1:   # targeted exchange: private buffers per simulated rank
            from paper_2001_07158_b200.shard import eval_vertex_simulated_private
            acc2 = eval_vertex_simulated_private(g, ds, k, mt, cfg, anchor[0], n, world)
            assert np.array_equal(acc2.cpu().numpy().view(np.uint64), want), ("targeted", k, world)
            # peer stores: the exchange inside the level kernel
            # (tsv_eval_vertex_level_peer), zeroed private buffers per rank
            from paper_2001_07158_b200.shard import eval_vertex_simulated_peer
            acc3 = eval_vertex_simulated_peer(g, ds, k, mt, cfg, anchor[0], n, world)
            assert np.array_equal(acc3.cpu().numpy().view(np.uint64), want), ("peer", k, world)
