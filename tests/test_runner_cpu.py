"""CPU: the runner layer's host-only pieces (config files, bench matrices,
output writers, the CLI's argument handling) against the compiled reference
(proj/core/src/config_file.cpp, runner.cpp:215-414, proj/tools/sdns.cpp).
Outputs are compared byte for byte; error paths by status and message.
"""
import os
import subprocess

import numpy as np
import pytest

import paper_1607_00850_b200 as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1607_00850_b200", "sdns_cuda")

CONFIG_CASES = [
    ("", []),
    ("n = 64\ndecomp = slab\np = 4\nnu = 0.01\ndt = 0.01\nt_end = 1\n", []),
    ("# comment line\n  n=32   # trailing comment\n\nre = 1600\nt_end = 0.5\n", []),
    ("n = 64\ndecomp = pencil\np = 8\nt_end = 0.1\n", []),
    ("n = 64\ndecomp = pencil\np = 4\np1 = 4\np2 = 1\n", []),
    ("n = 16\ndealias = off\ncase = isotropic\nout_every = 3\n", [("dealias", "yes")]),
    ("n = 16\n", [("n", "32"), ("p", "2"), ("t_end", "0.2")]),
    ("n = 16\nt_end = 0\n", []),
]

CONFIG_ERRORS = [
    "n = 16\nbogus = 1\n",
    "n = sixteen\n",
    "n = 16x\n",
    "nu = abc\n",
    "nu = inf\n",
    "dealias = maybe\n",
    "re = 0\n",
    "n = 16\njust text\n",
    "decomp = cube\n",
    "n = 16\np = 3\n",
    "n = 16\ndt = 0\n",
    "n = 16\nout_every = 0\n",
    "n = 16\ndecomp = pencil\np = 4\np1 = 3\np2 = 2\n",
    "n = 16\ndecomp = pencil\np = 34\n",
    "case = \n",
]


@pytest.mark.parametrize("text,over", CONFIG_CASES)
def test_parse_config_matches_reference(ref, text, over):
    want, want_notes = ref.parse_config(text, over)
    got = S.parse_config_text(text, over)
    c = got.cfg
    assert dict(n=c.n, decomp=c.decomp, p=c.p, p1=c.p1, p2=c.p2, dealias=c.dealias,
                out_every=c.out_every, nu=c.nu, dt=c.dt, t_end=c.t_end,
                initial_case=c.initial_case) == want
    assert got.notices == want_notes


@pytest.mark.parametrize("text", CONFIG_ERRORS)
def test_parse_config_errors_match_reference(ref, text):
    with pytest.raises(ref.RefError) as r:
        ref.parse_config(text)
    with pytest.raises(S.SdnsError) as g:
        S.parse_config_text(text)
    assert r.value.code == g.value.code == 1
    assert str(g.value) == str(r.value)


def test_parse_config_file(ref, tmp_path):
    p = tmp_path / "case.cfg"
    p.write_text("n = 32\nt_end = 0.25\n")
    got = S.parse_config_file(str(p), [("out_every", "5")])
    assert (got.cfg.n, got.cfg.t_end, got.cfg.out_every) == (32, 0.25, 5)
    with pytest.raises(S.IoError, match="cannot open config file"):
        S.parse_config_file(str(tmp_path / "missing.cfg"))


@pytest.mark.parametrize("n,p", [(64, 1), (64, 2), (64, 4), (64, 8), (64, 6), (16, 12),
                                 (32, 64), (8, 7)])
def test_default_pencil_grid_matches_reference(ref, n, p):
    try:
        want = ref.parse_config(f"n = {n}\ndecomp = pencil\np = {p}\n")[0]
        want = (want["p1"], want["p2"])
    except ref.RefError:
        want = None
    if want is None:
        with pytest.raises(S.ConfigError):
            S.parse_config_text(f"n = {n}\ndecomp = pencil\np = {p}\n")
    else:
        assert S.default_pencil_grid(n, p) == want


MATRICES = [
    "16 slab 1\n32, slab, 8\n# comment\n\n64 pencil 4 2 2\n64 pencil 8  # default grid\n",
    "",
    "  8 slab 2 ,\n",
]
MATRIX_ERRORS = ["16 slab\n", "16 cube 1\n", "16 pencil 4 2\n", "x slab 1\n", "16 slab 1 1 1 9\n"]


@pytest.mark.parametrize("text", MATRICES)
def test_bench_matrix_matches_reference(ref, text):
    want = ref.parse_bench_matrix(text)
    got = [(e.n, 0 if e.decomp == "slab" else 1, e.p, e.p1, e.p2)
           for e in S.parse_bench_matrix_text(text)]
    assert got == want


@pytest.mark.parametrize("text", MATRIX_ERRORS)
def test_bench_matrix_errors_match_reference(ref, text):
    with pytest.raises(ref.RefError) as r:
        ref.parse_bench_matrix(text)
    with pytest.raises(S.ConfigError) as g:
        S.parse_bench_matrix_text(text)
    assert str(g.value) == str(r.value)


def test_diagnostics_csv_byte_identical(ref, tmp_path):
    rng = np.random.default_rng(7)
    shells = 12
    steps = np.array([0, 10, 20, 25], dtype=np.int64)
    rows = rng.standard_normal((4, 5 + shells)) * 10.0 ** rng.integers(-20, 5, (4, 5 + shells))
    rows[0, 4] = 0.0
    rows[1, 1] = 1e-300
    ref.write_diagnostics_csv(tmp_path / "ref.csv", steps, rows, shells)
    samples = [(int(s), S.FlowStats(*r[:5], r[5:])) for s, r in zip(steps, rows)]
    S.write_diagnostics_csv(str(tmp_path / "ours.csv"), samples, shells)
    assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()


def test_bench_csv_byte_identical(ref, tmp_path):
    entries = [(16, 0, 1, 0, 0), (64, 1, 8, 2, 4), (32, 0, 4, 0, 0)]
    nodes = [4096, 32768, 8192]
    secs = [0.0123456789, 1.5e-5, 0.0]
    statuses = ["ok", "ok", "failed: a, b\nc"]
    ref.write_bench_csv(tmp_path / "ref.csv", entries, nodes, secs, statuses)
    rows = [S.BenchRow(S.BenchEntry(e[0], "slab" if e[1] == 0 else "pencil", *e[2:]), nd, sc, st)
            for e, nd, sc, st in zip(entries, nodes, secs, statuses)]
    S.write_bench_csv(str(tmp_path / "sub" / "ours.csv"), rows)
    assert (tmp_path / "sub" / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()


def test_manifest_identical_but_version(ref, tmp_path):
    cfg = S.SolverConfig(n=64, decomp="pencil", p=8, p1=2, p2=4, nu=1 / 1600, dt=1e-3,
                         t_end=0.3, dealias=False, initial_case="taylor_green", out_every=7)
    res = S.RunResult(cfg, "inprocess", "diverged at step 12", 11,
                      {"min_s": 0.01, "mean_s": 0.0125, "max_s": 0.02, "timed_steps": 6}, [],
                      "out/diagnostics.csv", "out/checkpoint.sdns", "out/manifest.txt")
    S.write_manifest(str(tmp_path / "ours.txt"), res)
    ref.write_manifest(tmp_path / "ref.txt", [64, 1, 8, 2, 4, 0, 7],
                       [1 / 1600, 1e-3, 0.3, 0.01, 0.0125, 0.02], "taylor_green", "inprocess",
                       "diverged at step 12", 11, 6, "out/diagnostics.csv", "out/checkpoint.sdns")
    ours = (tmp_path / "ours.txt").read_text().splitlines()
    theirs = (tmp_path / "ref.txt").read_text().splitlines()
    assert len(ours) == len(theirs) == 22
    for a, b in zip(ours, theirs):
        if a.startswith("version = "):
            assert b.startswith("version = ")
        else:
            assert a == b


def test_writers_raise_io_error(tmp_path):
    with pytest.raises(S.IoError, match="cannot open"):
        S.write_diagnostics_csv(str(tmp_path / "no" / "such" / "d.csv"), [], 3)


def _cli(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=120)


def test_cli_host_paths():
    """Argument handling and config errors need no device (sdns.cpp:102-161)."""
    assert os.path.exists(CLI), "build() makes paper_1607_00850_b200/sdns_cuda"
    r = _cli("--version")
    assert r.returncode == 0 and r.stdout.startswith("sdns-b200")
    assert _cli().returncode != 0
    r = _cli("run", "--n", "16", "--p", "3")
    assert r.returncode == 1
    assert "error: slab requires p to divide n, got p=3 n=16" in r.stderr
    assert r.stdout == ""  # parse and validate precede any output (sdns.cpp:37-41)
    r = _cli("run", "--n", "8", "--t-end", "0.002", "--out", "/tmp/sdns-cli-host-test")
    assert r.stdout.startswith("running taylor_green: n=8 slab p=1 nu=0.000625 dt=0.001 "
                               "t_end=0.002\n")
    assert r.returncode in (0, 1)  # 1 without a device: the context cannot be created
    r = _cli("run", "--nope")
    assert r.returncode != 0 and "--nope" in r.stderr
    r = _cli("bench", "--steps", "2")
    assert r.returncode != 0 and "--matrix" in r.stderr
    r = _cli("run", "--config", "/nonexistent/x.cfg")
    assert r.returncode == 1 and "cannot open config file" in r.stderr
