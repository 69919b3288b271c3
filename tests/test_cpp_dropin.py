"""The C++ drop-in (tsieve API + CLI, paper_2001_07158_b200/cpp) against the
reference: solver decisions, flagged sets, checksums, optimum horizons and
witnesses from the golden sweep, and the CLI surface of test_cli.cpp."""
import ctypes as C
import json
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2001_07158_b200", "lib")
CLI = os.path.join(LIB, "tsieve")
FIG2_EDGES = "u1 u2 3\nu2 u3 1\nu3 u4 3\nu4 u5 1\nu5 u1 2\nu2 u5 4\nu3 u5 5\n"
FIG2_COLORS = "u1 1\nu2 3\nu3 4\nu4 1\nu5 2\n"

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def dropin():
    lib = C.CDLL(os.path.join(LIB, "libtsieve.so"))
    lib.tsieve_last_error.restype = C.c_char_p
    lib.tsieve_solve_json.restype = C.c_int64
    lib.tsieve_solve_json.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                      C.c_int32, _i32p, C.c_char_p, _i32p, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
                                      C.c_int32, C.c_char_p, C.c_int64]
    return lib


def solve(c):
    a = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.int32))  # noqa: E731
    buf = C.create_string_buffer(1 << 16)
    motif = a(c["motif"]) if c["motif"] else np.zeros(1, np.int32)
    u = a(c["u"]) if c["u"] else np.zeros(1, np.int32)
    v = a(c["v"]) if c["v"] else np.zeros(1, np.int32)
    ts = a(c["ts"]) if c["ts"] else np.zeros(1, np.int32)
    lib = dropin()
    r = lib.tsieve_solve_json(c["n"], len(c["u"]), u, v, ts, int(c["directed"]), 0, a(c["colors"]),
                              c["problem"].encode(), motif, len(c["motif"]), c["k"], c["source"],
                              c["dest"], c["seed"], c["mode"], c["extraction"], c["preprocess"],
                              buf, len(buf))
    if r < 0:
        raise ValueError(lib.tsieve_last_error().decode())
    return json.loads(buf.value.decode())


def cli(args, cwd=None):
    p = subprocess.run([CLI] + args, capture_output=True, text=True, cwd=cwd)
    return p.returncode, p.stdout + p.stderr


@pytest.fixture
def fig2(tmp_path):
    (tmp_path / "fig2.edges").write_text(FIG2_EDGES)
    (tmp_path / "fig2.colors").write_text(FIG2_COLORS)
    return ["--graph", str(tmp_path / "fig2.edges"), "--colors", str(tmp_path / "fig2.colors")]


# ------------------------------------------------------------------ CPU


def test_cli_usage_errors_exit_2_naming_the_flag(fig2):
    # test_cli.cpp:52-63
    rc, out = cli(["decide"] + fig2 + ["--problem", "ktemppath", "--k", "0"])
    assert rc == 2 and "--k" in out
    rc, out = cli(["decide", "--problem", "pathmotif", "--motif", "1,2"])
    assert rc == 2 and "--graph" in out
    rc, out = cli(["decide", "--graph", "/nonexistent.edges", "--problem", "pathmotif",
                   "--motif", "1,2"])
    assert rc == 2
    rc, out = cli(["decide"] + fig2 + ["--bogus"])
    assert rc == 2 and "--bogus" in out
    rc, out = cli(["frobnicate"])
    assert rc == 2
    assert cli(["--help"])[0] == 0


def test_cli_certain_no_without_device(fig2):
    # infeasible queries are decided on the host before any evaluation
    rc, out = cli(["decide"] + fig2 + ["--problem", "pathmotif", "--motif", "1,9",
                                       "--preprocess", "none", "--format", "json"])
    assert rc == 1
    rec = json.loads(out)
    assert rec["decision"] == "NO" and rec["certain"] is True
    assert rec["note"] == "query color 9 absent from the graph"
    rc, out = cli(["decide"] + fig2 + ["--problem", "ktemppath", "--k", "6",
                                       "--preprocess", "none", "--format", "json"])
    assert rc == 1 and json.loads(out)["note"] == "k exceeds vertex count"


def test_dropin_exports():
    lib = dropin()
    assert hasattr(lib, "tsieve_solve_json")
    assert hasattr(lib, "tsieve_load_graph_text")


def dropin_load(edge_text, color_text, directed):
    lib = dropin()
    f = lib.tsieve_load_graph_text
    f.restype = C.c_int64
    f.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                  _i32p, _i32p, _i32p, C.c_int64, _i32p, C.c_int32, C.c_char_p, C.c_int64]
    cap = edge_text.count("\n") + 2
    ou, ov, ot = (np.empty(cap, np.int32) for _ in range(3))
    n, t = C.c_int32(0), C.c_int32(0)
    cols = np.empty(2 * cap + 2, np.int32)
    names = C.create_string_buffer(1 << 22)
    m = f(edge_text.encode(), None if color_text is None else color_text.encode(), int(directed),
          C.byref(n), C.byref(t), ou, ov, ot, cap, cols, len(cols), names, len(names))
    if m < 0:
        raise ValueError(lib.tsieve_last_error().decode())
    nm = names.value.decode().split("\n") if n.value else []
    return {"n": n.value, "t": t.value, "u": ou[:m].copy(), "v": ov[:m].copy(),
            "ts": ot[:m].copy(), "colors": cols[:n.value].copy(), "names": nm}


def _random_text(rng):
    """Edge/colour text exercising the tokenizer: numeric and symbolic names
    (including non-canonical decimals like '007' and '+7'), comments, blank
    lines, tabs, CRLF, sparse and dense timestamp spans, a missing final
    newline, duplicates and self loops."""
    pool = ["7", "007", "+7", "a", "b", "x_1", "12", "0", "00", "1073741824", "99999999999",
            "-3", "v9", "3"]
    names = [pool[i] for i in rng.choice(len(pool), size=rng.integers(2, len(pool)),
                                         replace=False)]
    span = int(rng.choice([5, 1000, 10**12]))
    lines = []
    for _ in range(int(rng.integers(0, 40))):
        a, b = rng.choice(names), rng.choice(names)
        ts = int(rng.integers(0, span))
        sep = rng.choice([" ", "\t", "  "])
        line = f"{a}{sep}{b}{sep}{ts}"
        r = rng.random()
        if r < 0.1:
            line += " # comment"
        elif r < 0.2:
            line += "\r"
        elif r < 0.25:
            line += " 1"
        lines.append(line)
        if rng.random() < 0.1:
            lines.append(rng.choice(["", "   ", "# only a comment"]))
    text = "\n".join(lines) + ("\n" if rng.random() < 0.7 else "")
    colors = None
    if rng.random() < 0.7:
        colors = "".join(f"{rng.choice(names + ['ghost'])} {int(rng.integers(1, 6))}\n"
                         for _ in range(int(rng.integers(0, 10))))
    return text, colors


def test_load_graph_matches_reference_loader():
    """load_graph (graph.cpp) against the reference's own load_graph
    (oracle/_ref, graph.cpp:376-448): names, rank-normalized timestamps,
    canonical edges, colours, and error messages on malformed lines."""
    from oracle import oracle
    try:
        oracle.ref_lib()
    except Exception as e:  # pragma: no cover
        pytest.skip(f"oracle/_ref not built: {e}")
    rng = np.random.default_rng(7)
    for _ in range(300):
        text, colors = _random_text(rng)
        directed = bool(rng.integers(0, 2))
        want = oracle.ref_load_graph(text, colors, directed)
        got = dropin_load(text, colors, directed)
        assert got["n"] == want["n"] and got["t"] == want["t"], text
        assert got["names"] == want["names"]
        for key in ("u", "v", "ts", "colors"):
            assert got[key].tolist() == want[key].tolist(), (key, text)
    for bad in ["a b 3x\n", "a b\n", "a b 1\nb c -1\n", "a b 1 0\n", "a b 99999999999999999999\n",
                "a b 1\n\n# c\na b 0x5\n", "a b --1\n", "a b +\n"]:
        with pytest.raises(ValueError) as ref_err:
            oracle.ref_load_graph(bad, None, False)
        with pytest.raises(ValueError) as our_err:
            dropin_load(bad, None, False)
        assert str(our_err.value) == str(ref_err.value), bad
    with pytest.raises(ValueError) as ref_err:
        oracle.ref_load_graph("a b 1\n", "a 0\n", False)
    with pytest.raises(ValueError) as our_err:
        dropin_load("a b 1\n", "a 0\n", False)
    assert str(our_err.value) == str(ref_err.value)


def dropin_load_file(path, color_text, directed, cache):
    lib = dropin()
    f = lib.tsieve_load_graph_file
    f.restype = C.c_int64
    f.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_char_p, C.POINTER(C.c_int32),
                  C.POINTER(C.c_int32), C.POINTER(C.c_int32), _i32p, _i32p, _i32p, C.c_int64,
                  _i32p, C.c_int32, C.c_char_p, C.c_int64,
                  np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")]
    with open(path) as fh:
        cap = fh.read().count("\n") + 2
    ou, ov, ot = (np.empty(cap, np.int32) for _ in range(3))
    n, t, hit = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    cols = np.empty(2 * cap + 2, np.int32)
    names = C.create_string_buffer(1 << 22)
    stats = np.zeros(3, np.int64)
    m = f(str(path).encode(), None if color_text is None else color_text.encode(), int(directed),
          None if cache is None else str(cache).encode(), C.byref(hit), C.byref(n), C.byref(t),
          ou, ov, ot, cap, cols, len(cols), names, len(names), stats)
    if m < 0:
        raise ValueError(lib.tsieve_last_error().decode())
    nm = names.value.decode().split("\n") if n.value else []
    return {"n": n.value, "t": t.value, "u": ou[:m].copy(), "v": ov[:m].copy(),
            "ts": ot[:m].copy(), "colors": cols[:n.value].copy(), "names": nm,
            "stats": stats.tolist()}, bool(hit.value)


def _same_load(a, b):
    return (a["n"] == b["n"] and a["t"] == b["t"] and a["names"] == b["names"] and
            all(np.array_equal(a[k], b[k]) for k in ("u", "v", "ts", "colors")))


def test_ingest_cache_reproduces_the_text_load(tmp_path):
    """Binary ingest cache (graph.cpp): a load that hits the
    cache equals the text parse (which test_load_graph_matches_reference_loader
    pins to the reference's load_graph, graph.cpp:376-448) -- canonical edges,
    names, colors, drop counts, for either directedness; a changed, truncated
    or foreign cache file is a miss and is rewritten."""
    import os
    rng = np.random.default_rng(23)
    hits = 0
    for case in range(40):
        text, colors = _random_text(rng)
        nl = "" if not text or text.endswith("\n") else "\n"
        if case % 4 == 0:  # transition times ride through the cache
            text += nl + "a b 3 2\nb c 4 5\n"
            nl = ""
        src = tmp_path / f"g{case}.edges"
        cache = tmp_path / f"g{case}.ingest"
        src.write_text(text)
        try:
            want = dropin_load(text, colors, False)
        except ValueError as e:
            with pytest.raises(ValueError) as ei:
                dropin_load_file(src, colors, False, cache)
            assert str(ei.value) == str(e)
            assert not cache.exists()        # a file that fails to parse leaves no cache
            continue
        plain, hit = dropin_load_file(src, colors, False, None)
        assert not hit and _same_load(want, plain)
        first, hit = dropin_load_file(src, colors, False, cache)
        assert not hit and cache.exists()
        assert _same_load(want, first) and first["stats"] == plain["stats"]
        again, hit = dropin_load_file(src, colors, False, cache)
        assert hit and _same_load(want, again) and again["stats"] == plain["stats"]
        hits += 1
        # the cache holds raw records: the other directedness is served from it too
        wd = dropin_load(text, colors, True)
        gd, hit = dropin_load_file(src, colors, True, cache)
        assert hit and _same_load(wd, gd)
        # a truncated cache is a miss (and is rewritten)
        blob = cache.read_bytes()
        cache.write_bytes(blob[:-1])
        got, hit = dropin_load_file(src, colors, False, cache)
        assert not hit and _same_load(want, got)
        assert cache.read_bytes() == blob
        # a changed source invalidates it
        st = os.stat(src)
        src.write_text(text + nl + "zz yy 7\n")
        os.utime(src, ns=(st.st_atime_ns, st.st_mtime_ns + 5_000_000_000))
        w2 = dropin_load(text + nl + "zz yy 7\n", colors, False)
        g2, hit = dropin_load_file(src, colors, False, cache)
        assert not hit and _same_load(w2, g2)
        g3, hit = dropin_load_file(src, colors, False, cache)
        assert hit and _same_load(w2, g3)
    assert hits >= 20


def test_load_graph_multi_chunk_matches_reference_loader():
    """A multi-megabyte edge file is parsed in parallel line-aligned chunks:
    interning order, ranks and the line number of a late error must still be
    those of the reference's sequential loader."""
    from oracle import oracle
    try:
        oracle.ref_lib()
    except Exception as e:  # pragma: no cover
        pytest.skip(f"oracle/_ref not built: {e}")
    rng = np.random.default_rng(11)
    L = 160_000
    names = np.array([str(i) for i in range(3000)] + [f"n{i}" for i in range(500)] +
                     ["007", "+3", "00"])
    a = names[rng.integers(0, len(names), L)]
    b = names[rng.integers(0, len(names), L)]
    ts = rng.integers(0, 10**9, L)
    lines = [f"{x} {y} {t}" for x, y, t in zip(a.tolist(), b.tolist(), ts.tolist())]
    for i in rng.choice(L, 500, replace=False).tolist():
        lines[i] = lines[i] + (" # note" if i % 2 else "\t1")
    for i in rng.choice(L, 300, replace=False).tolist():
        lines[i] = ""
    text = "\n".join(lines) + "\n"
    assert len(text) > 2 << 20  # several 1 MiB chunks
    want = oracle.ref_load_graph(text, None, False)
    got = dropin_load(text, None, False)
    assert got["n"] == want["n"] and got["t"] == want["t"] and got["names"] == want["names"]
    for key in ("u", "v", "ts"):
        assert np.array_equal(got[key], want[key]), key
    bad = lines[:]
    bad[140_001] = "x y zz"
    bad[150_000] = "x y"
    text = "\n".join(bad) + "\n"
    with pytest.raises(ValueError) as ref_err:
        oracle.ref_load_graph(text, None, False)
    with pytest.raises(ValueError) as our_err:
        dropin_load(text, None, False)
    assert str(our_err.value) == str(ref_err.value) == "line 140002: malformed integer 'zz'"


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
def test_solver_sweep_matches_reference(cuda_device, golden):
    """Decisions, certainty, flagged sets, checksums, optimum horizons, probe
    counts and the extracted witnesses equal the reference's on the golden
    sweep (four problems x decide/optimum/extract x both strategies x
    preprocess none/colors)."""
    for c in golden["solve_sweep"]:
        got, want = solve(c), c["result"]
        for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "witness",
                    "extraction_failed", "oracle_calls", "preprocessed_n", "preprocessed_m"):
            assert got[key] == want[key], (key, c["problem"], c["mode"], got, want)


@pytest.mark.gpu
def test_fig2_solver_cases(cuda_device, golden):
    fig = {"n": 5, "u": [0, 1, 2, 3, 4, 1, 2], "v": [1, 2, 3, 4, 0, 4, 4],
           "ts": [3, 1, 3, 1, 2, 4, 5], "directed": False, "colors": [1, 3, 4, 1, 2],
           "extraction": 0, "preprocess": 0, "seed": 1}
    for s in golden["solve_fig2"]:
        c = dict(fig, problem=s["problem"], motif=s["motif"], k=s["k"], mode=s["mode"],
                 source=s.get("source", -1), dest=s.get("dest", -1))
        got = solve(c)
        for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "witness"):
            assert got[key] == s["result"][key], (key, s)


@pytest.mark.gpu
def test_cli_decide_extract_verify_optimum(cuda_device, fig2, tmp_path, golden):
    # test_cli.cpp:41-84 with --preprocess none / colors
    for pre in ("none", "colors"):
        rc, out = cli(["decide"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                           "--preprocess", pre, "--format", "json"])
        assert rc == 0 and '"decision": "YES"' in out
        rc, _ = cli(["decide"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,1,3",
                                         "--preprocess", pre])
        assert rc == 1
    rc, out = cli(["decide"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                       "--preprocess", "none", "--format", "json"])
    rec = json.loads(out)
    want = next(s for s in golden["solve_fig2"] if s["problem"] == "pathmotif" and s["mode"] == 0)
    assert rec["accumulator_checksum"] == want["result"]["checksum"]
    assert rec["flagged"] == want["result"]["flagged"]
    # the same record from the binary ingest cache (written by the first run, hit by the second)
    cache = tmp_path / "fig2.ingest"
    for _ in range(2):
        rc, out = cli(["decide"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                           "--preprocess", "none", "--format", "json",
                                           "--ingest-cache", str(cache)])
        assert rc == 0 and cache.exists()
        again = json.loads(out)
        assert again["accumulator_checksum"] == rec["accumulator_checksum"]
        assert again["flagged"] == rec["flagged"]

    rc, out = cli(["extract"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                        "--preprocess", "none", "--format", "json"])
    assert rc == 0 and '"witness"' in out
    wfile = tmp_path / "w.json"
    wfile.write_text(out)
    rc, out2 = cli(["verify"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                        "--witness", str(wfile)])
    assert rc == 0 and "witness OK" in out2
    rec = json.loads(out)
    assert rec["witness"]["vertex_names"] == ["u4", "u5", "u1", "u2"]

    rc, out = cli(["optimum"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                        "--preprocess", "none", "--format", "json"])
    assert rc == 0 and '"optimum_ts": 3' in out

    # (s,d) by vertex name, self-reducible extraction
    rc, out = cli(["extract"] + fig2 + ["--problem", "sdcolorful", "--k", "2", "--source", "u4",
                                        "--dest", "u2", "--preprocess", "none",
                                        "--extraction", "self-reducible", "--format", "json"])
    assert rc == 0
    assert json.loads(out)["witness"]["vertex_names"][0] == "u4"


@pytest.mark.gpu
def test_default_preprocessing_matches_reference(cuda_device, golden):
    """--preprocess both / static: the junction sieve on the static
    projection runs on the GPU; the kept-vertex set (preprocessed_n/m), and
    through the renumbered edge ids every checksum, equal the reference's."""
    for c in golden["solve_sweep_preprocess"]:
        got, want = solve(c), c["result"]
        for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "witness",
                    "extraction_failed", "oracle_calls", "preprocessed_n", "preprocessed_m"):
            assert got[key] == want[key], (key, c["problem"], c["preprocess"], got, want)


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [8, 16, 32])
def test_solver_small_fields_match_reference(cuda_device, golden, bits):
    """SieveConfig::field_bits 8 / 16 / 32 (the reference CLI's --field-bits,
    tools/main.cpp:70): solve() records -- decisions, checksums, probes,
    witnesses -- equal the reference's at the same width, with the default
    preprocessing (junction sieve on the projection) and without; small
    fields give false negatives, which must agree too."""
    from oracle import oracle as O
    lib = dropin()
    lib.tsieve_set_field_bits(bits)
    try:
        for c in golden["solve_sweep_preprocess"][:32]:
            want = O.ref_solve(c["n"], c["u"], c["v"], c["ts"], c["directed"], c["colors"],
                               c["problem"], c["motif"], c["k"], c["source"], c["dest"],
                               seed=c["seed"], mode=c["mode"], extraction=c["extraction"],
                               preprocess=c["preprocess"], field_bits=bits)
            got = solve(c)
            for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "witness",
                        "extraction_failed", "oracle_calls", "preprocessed_n", "preprocessed_m"):
                assert got[key] == want[key], (key, bits, c["problem"], got, want)
    finally:
        lib.tsieve_set_field_bits(64)
        O.ref_lib().ref_set_field_bits(64)


@pytest.mark.gpu
def test_default_preprocessing_large_graph_matches_reference(cuda_device):
    """--preprocess both on a graph above 2^22 edges, where the C++
    StaticProjection::project groups on the device (radix sort) and
    TemporalGraph::build canonicalizes there: the solve() record equals the
    reference's (its host stable_sort and build)."""
    from oracle import oracle as O
    rng = np.random.default_rng(23)
    n, m = 3000, (1 << 22) + 5000
    u = rng.integers(0, n, m).astype(np.int32)
    v = rng.integers(0, n, m).astype(np.int32)
    ts = rng.integers(1, 40, m).astype(np.int32)
    colors = rng.integers(1, 6, n).astype(np.int32)
    c = {"n": n, "u": u.tolist(), "v": v.tolist(), "ts": ts.tolist(), "directed": True,
         "colors": colors,
         "problem": "pathmotif", "motif": [1, 2, 2, 3], "k": 4, "source": -1, "dest": -1,
         "seed": 3, "mode": 1, "extraction": 0, "preprocess": 3}
    want = O.ref_solve(n, u, v, ts, True, colors, "pathmotif", [1, 2, 2, 3], 4, seed=3, mode=1,
                       preprocess=3)
    got = solve(c)
    for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "oracle_calls",
                "preprocessed_n", "preprocessed_m"):
        assert got[key] == want[key], (key, got[key], want[key])


@pytest.mark.gpu
def test_cli_reference_defaults(cuda_device, fig2, golden):
    """The reference CLI tests (test_cli.cpp:41-84) with DEFAULT flags
    (preprocess both, optimize on)."""
    rc, out = cli(["decide"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                       "--format", "json"])
    assert rc == 0 and '"decision": "YES"' in out
    rc, _ = cli(["decide"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,1,3"])
    assert rc == 1
    rc, out = cli(["optimum"] + fig2 + ["--problem", "pathmotif", "--motif", "1,1,2,3",
                                        "--format", "json"])
    assert rc == 0 and '"optimum_ts": 3' in out
    for case in golden["solve_fig2_default"]:
        args = ["extract"] + fig2 + ["--problem", case["problem"], "--format", "json"]
        args += ["--motif", ",".join(map(str, case["motif"]))] if case["motif"] else \
            ["--k", str(case["k"])]
        rc, out = cli(args)
        rec = json.loads(out)
        want = case["result"]
        assert rec["decision"] == ("YES" if want["decision"] else "NO")
        assert rec["accumulator_checksum"] == want["checksum"]
        assert rec["preprocessed"]["n"] == want["preprocessed_n"]
        got_w = None if rec["witness"] is None else {"vertices": rec["witness"]["vertices"],
                                                     "edges": rec["witness"]["edges"]}
        assert got_w == want["witness"]


@pytest.mark.gpu
def test_large_build_canonicalizes_on_device_like_host(cuda_device):
    """TemporalGraph::build sorts inputs of >= 2^22 edges on device 0 (and
    keeps that HBM mirror); the canonical list must equal the host
    canonicalizer's (TSV_HOST_BUILD=1), duplicates and self loops included."""
    rng = np.random.default_rng(5)
    m = (1 << 22) + 12345
    u = rng.integers(0, 50_000, m)
    v = rng.integers(0, 50_000, m)
    ts = rng.integers(1, 3_000, m)
    v[:1000] = u[:1000]                      # self loops
    u[1000:3000], v[1000:3000], ts[1000:3000] = u[3000:5000], v[3000:5000], ts[3000:5000]
    text = "".join(f"{a} {b} {t}\n" for a, b, t in zip(u.tolist(), v.tolist(), ts.tolist()))
    for directed in (False, True):
        os.environ["TSV_HOST_BUILD"] = "1"
        try:
            host = dropin_load(text, None, directed)
        finally:
            del os.environ["TSV_HOST_BUILD"]
        dev = dropin_load(text, None, directed)
        assert dev["n"] == host["n"] and dev["t"] == host["t"]
        for key in ("u", "v", "ts"):
            assert np.array_equal(dev[key], host[key]), key


def solve_ex(c, eps, delays, model, times=(), order=()):
    lib = dropin()
    f = lib.tsieve_solve_json_ex
    f.restype = C.c_int64
    f.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_void_p, C.c_void_p, C.c_int32,
                  C.c_int, C.c_int32, _i32p, C.c_char_p, _i32p, C.c_int32, C.c_int32, C.c_int32,
                  C.c_int32, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, C.c_char_p, C.c_int64,
                  C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]
    a = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.int32))  # noqa: E731
    e = a(eps) if eps is not None else None
    d = a(delays) if delays is not None else None
    tm = a(times) if len(times) else None
    od = a(order) if len(order) else None
    buf = C.create_string_buffer(1 << 16)
    motif = a(c["motif"]) if c["motif"] else np.zeros(1, np.int32)
    r = f(c["n"], len(c["u"]), a(c["u"]), a(c["v"]), a(c["ts"]),
          None if e is None else e.ctypes.data, None if d is None else d.ctypes.data, model,
          int(c["directed"]), 0, a(c["colors"]), c["problem"].encode(), motif, len(c["motif"]),
          c["k"], c["source"], c["dest"], c["seed"], c["mode"], c["extraction"], c["preprocess"],
          buf, len(buf), None if tm is None else tm.ctypes.data, len(times),
          None if od is None else od.ctypes.data, len(order))
    if r < 0:
        raise ValueError(lib.tsieve_last_error().decode())
    return json.loads(buf.value.decode())


@pytest.mark.gpu
@pytest.mark.parametrize("model", [1, 2, 3])
def test_solver_edge_models_match_reference(cuda_device, model):
    """solve() under the transition / delay / transition-delay models: the
    sieve probes run on model-specific device layouts, the DFS uses the
    reference's eps/delta gaps, self-reduction restricts on the host; every
    field of the record equals the reference's."""
    from oracle import oracle as O
    from paper_2001_07158_b200 import synth
    rng = np.random.default_rng(100 + model)
    problems = ["pathmotif", "ktemppath", "colorfulpath", "sdcolorful"]
    found = 0
    for i in range(32):
        n, u, v, ts, d, colors, motif = synth.random_small(rng, n_max=16, m_max=70, t_max=9,
                                                           k_max=4, q_max=3)
        eps = rng.integers(1, 3, len(u))
        delays = rng.integers(0, 3, n) if i % 3 else None
        prob = problems[i % 4]
        k, src, dst = 0, -1, -1
        if prob == "ktemppath":
            motif, k = [], int(rng.integers(1, 4))
        elif prob == "colorfulpath":
            motif = sorted(set(motif)) or [1]
        elif prob == "sdcolorful":
            motif, k = [], int(rng.integers(1, 3))
            src, dst = (int(x) for x in rng.choice(n, 2, replace=False))
        c = {"n": n, "u": u.tolist(), "v": v.tolist(), "ts": ts.tolist(), "directed": d,
             "colors": colors.tolist(), "problem": prob, "motif": motif, "k": k, "source": src,
             "dest": dst, "seed": int(rng.integers(1, 1000)), "mode": [0, 1, 2, 3][(i // 4) % 4],
             "extraction": (i // 16) % 2, "preprocess": [0, 1][(i // 8) % 2]}
        want = O.ref_solve_model(n, u, v, ts, eps, delays, model, d, colors, prob, motif, k,
                                 source=src, dest=dst, seed=c["seed"], mode=c["mode"],
                                 extraction=c["extraction"], preprocess=c["preprocess"])
        got = solve_ex(c, eps, delays, model)
        for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "witness",
                    "extraction_failed", "oracle_calls", "preprocessed_n", "preprocessed_m"):
            assert got[key] == want[key], (key, model, i, got, want)
        found += got["witness"] is not None
    assert found > 3


@pytest.mark.gpu
def test_cli_edge_models_from_files(cuda_device, tmp_path):
    """The CLI reads transition times (4th column) and --delays files and
    picks the model like the reference's --edge-model auto; results equal
    the reference's solve() under the same model."""
    from oracle import oracle as O
    rng = np.random.default_rng(8)
    n, m = 12, 60
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    ts, eps = rng.integers(1, 8, m), rng.integers(1, 3, m)
    delays = rng.integers(0, 3, n)
    colors = rng.integers(1, 3, n)
    (tmp_path / "g.edges").write_text("".join(f"{a} {b} {t} {e}\n" for a, b, t, e in
                                              zip(u.tolist(), v.tolist(), ts.tolist(),
                                                  eps.tolist())))
    (tmp_path / "g.colors").write_text("".join(f"{i} {c}\n" for i, c in enumerate(colors)))
    (tmp_path / "g.delays").write_text("".join(f"{i} {d}\n" for i, d in enumerate(delays)))
    # file tokens "0".."11" intern in first-appearance order: map ids
    order = []
    for a, b in zip(u.tolist(), v.tolist()):
        for x in (a, b):
            if x not in order:
                order.append(x)
    idx = {x: i for i, x in enumerate(order)}
    nn = len(order)
    uu = np.array([idx[x] for x in u.tolist()])
    vv = np.array([idx[x] for x in v.tolist()])
    col2 = np.array([colors[x] for x in order])
    del2 = np.array([delays[x] for x in order])
    for extra, model, dl in (([], 1, None), (["--delays", str(tmp_path / "g.delays")], 3, del2)):
        args = ["decide", "--graph", str(tmp_path / "g.edges"), "--colors",
                str(tmp_path / "g.colors"), "--problem", "pathmotif", "--motif", "1,2,1",
                "--directed", "--preprocess", "none", "--format", "json"] + extra
        rc, out = cli(args)
        rec = json.loads(out)
        want = O.ref_solve_model(nn, uu, vv, ts, eps, dl, model, True, col2, "pathmotif",
                                 [1, 1, 2], 0, seed=1, mode=0)
        assert rec["decision"] == ("YES" if want["decision"] else "NO"), (model, rec, want)
        assert rec["accumulator_checksum"] == want["checksum"]
        assert rec["config"]["edge_model"] == {1: "transition", 3: "transition-delay"}[model]


@pytest.mark.gpu
@pytest.mark.parametrize("problem", ["ectemppath", "ecpathmotif", "vcpathmotif",
                                     "vccolorfulpath"])
def test_solver_ec_vc_problems_match_reference(cuda_device, problem):
    """Edge-constrained (prescribed timestamps) and vertex-ordered (position
    colors) problems: the EC and VC sieves and the VC-ColorfulPath exact DP on
    the device, the DFS with timed / ordered constraints; every record field
    equals the reference's (decide / optimum / extract, both strategies,
    preprocess none / colors / both)."""
    from oracle import oracle as O
    from paper_2001_07158_b200 import synth
    rng = np.random.default_rng(sum(map(ord, problem)))
    found = 0
    for i in range(28):
        n, u, v, ts, d, colors, _ = synth.random_small(rng, n_max=14, m_max=60, t_max=8,
                                                       k_max=4, q_max=3)
        k = int(rng.integers(2, 5))
        times, order, motif = [], [], []
        if problem.startswith("ec"):
            # prescribed stamps: often those of an existing increasing walk
            if i % 3 and len(ts):
                cand = sorted(set(ts.tolist()))
                pick = sorted(rng.choice(cand, min(k - 1, len(cand)), replace=False).tolist())
                times = pick
            else:
                times = sorted(rng.choice(np.arange(1, 9), k - 1, replace=False).tolist())
            k = len(times) + 1
            if problem == "ecpathmotif":
                motif = sorted(rng.integers(1, int(colors.max()) + 1, k).tolist())
        else:
            q = int(colors.max())
            if problem == "vccolorfulpath":
                k = min(k, q)
                order = rng.permutation(np.arange(1, q + 1))[:k].tolist()
            else:
                order = rng.integers(1, q + 1, k).tolist()
        c = {"n": n, "u": u.tolist(), "v": v.tolist(), "ts": ts.tolist(), "directed": d,
             "colors": colors.tolist(), "problem": problem, "motif": motif, "k": 0,
             "source": -1, "dest": -1, "seed": int(rng.integers(1, 1000)),
             "mode": [0, 1, 2, 3][i % 4], "extraction": (i // 4) % 2,
             "preprocess": [0, 1, 3][(i // 8) % 3]}
        want = O.ref_solve_query(n, u, v, ts, times, order, d, colors, problem, motif, 0,
                                 seed=c["seed"], mode=c["mode"], extraction=c["extraction"],
                                 preprocess=c["preprocess"])
        got = solve_ex(c, None, None, 0, times=times, order=order)
        for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "witness",
                    "extraction_failed", "oracle_calls", "preprocessed_n", "preprocessed_m"):
            assert got[key] == want[key], (key, problem, i, times, order, got, want)
        found += got["witness"] is not None
    assert found >= 2


@pytest.mark.gpu
def test_solver_larger_instances_match_reference(cuda_device):
    """Solver records on larger random graphs (hubs split across warp chunks,
    several batches per evaluation, both extraction strategies, default
    junction preprocessing) against the reference."""
    from oracle import oracle as O
    rng = np.random.default_rng(2024)
    for i in range(6):
        n, m, t = 400, 6000, 25
        u = rng.integers(0, n, m)
        v = np.where(rng.random(m) < 0.2, 7, rng.integers(0, n, m))   # a hub head
        ts = rng.integers(1, t + 1, m)
        d = bool(i % 2)
        colors = rng.integers(1, 4, n)
        prob, motif, k = [("pathmotif", [1, 1, 2, 3, 1], 0), ("ktemppath", [], 6),
                          ("colorfulpath", [1, 2, 3], 0)][i % 3]
        c = {"n": n, "u": u.tolist(), "v": v.tolist(), "ts": ts.tolist(), "directed": d,
             "colors": colors.tolist(), "problem": prob, "motif": motif, "k": k,
             "source": -1, "dest": -1, "seed": 7 + i, "mode": 3, "extraction": i // 3,
             "preprocess": 3}
        want = O.ref_solve(n, u, v, ts, d, colors, prob, motif, k, seed=c["seed"], mode=3,
                           extraction=c["extraction"], preprocess=3)
        got = solve(c)
        for key in ("decision", "certain", "optimum_ts", "checksum", "flagged", "witness",
                    "extraction_failed", "oracle_calls", "preprocessed_n", "preprocessed_m"):
            assert got[key] == want[key], (key, i, got, want)
