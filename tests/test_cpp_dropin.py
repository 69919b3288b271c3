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
