"""GPU: the runner layer (run / bench / CLI / acceptance suite) on the device
pipeline against the compiled reference's own run() (proj/core/src/runner.cpp:
67-213): the same diagnostics.csv rows (within the fp64 tolerances of
north_star), manifest lines, checkpoint contents, divergence handling and
bench.csv schema.
"""
import csv
import os
import struct
import subprocess

import numpy as np
import pytest

import paper_1607_00850_b200 as S

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1607_00850_b200", "sdns_cuda")


def read_csv(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    return rows[0], np.array([[float(x) for x in r] for r in rows[1:]])


def read_manifest(path):
    out = {}
    for line in open(path):
        k, v = line.rstrip("\n").split(" = ", 1)
        out[k] = v
    return out


def read_checkpoint(path):
    raw = open(path, "rb").read()
    magic, ver, n, comps, t, step = struct.unpack("<4sIIIdQ", raw[:32])
    u = np.frombuffer(raw[32:], dtype="<f8").reshape(comps, n, n, n)
    return dict(magic=magic, version=ver, n=n, t=t, step=step), u


def config_text(n, decomp="slab", p=1, p1=1, p2=1, t_end=0.05, out_every=5, nu=None, dt=None,
                case="taylor_green"):
    s = f"n = {n}\ndecomp = {decomp}\np = {p}\nt_end = {t_end}\nout_every = {out_every}\n"
    if decomp == "pencil":
        s += f"p1 = {p1}\np2 = {p2}\n"
    if nu is not None:
        s += f"nu = {nu}\n"
    if dt is not None:
        s += f"dt = {dt}\n"
    return s + f"case = {case}\n"


def compare_runs(ours_dir, ref_dir, tol=1e-12):
    h1, a = read_csv(os.path.join(ours_dir, "diagnostics.csv"))
    h2, b = read_csv(os.path.join(ref_dir, "diagnostics.csv"))
    assert h1 == h2
    assert a.shape == b.shape
    np.testing.assert_array_equal(a[:, 0], b[:, 0])  # steps
    np.testing.assert_array_equal(a[:, 1], b[:, 1])  # t, bitwise (t = k*dt)
    for col in (2, 3, 4):  # E, Z, eps
        np.testing.assert_allclose(a[:, col], b[:, col], rtol=tol, atol=0)
    assert np.all(a[:, 5] <= 1e-10) and np.all(b[:, 5] <= 1e-10)  # div_max
    e0 = b[0, 2]
    assert np.max(np.abs(a[:, 6:] - b[:, 6:])) <= tol * e0  # spectrum shells
    m1 = read_manifest(os.path.join(ours_dir, "manifest.txt"))
    m2 = read_manifest(os.path.join(ref_dir, "manifest.txt"))
    assert list(m1) == list(m2)
    for k in m1:
        if k in ("version", "step_seconds_min", "step_seconds_mean", "step_seconds_max",
                 "csv", "checkpoint"):
            continue
        assert m1[k] == m2[k], k
    c1, u1 = read_checkpoint(os.path.join(ours_dir, "checkpoint.sdns"))
    c2, u2 = read_checkpoint(os.path.join(ref_dir, "checkpoint.sdns"))
    assert c1 == c2
    assert np.linalg.norm(u1 - u2) <= 1e-11 * np.linalg.norm(u2)
    return m1


@pytest.mark.parametrize("geom", [dict(p=1), dict(p=4), dict(decomp="pencil", p=4, p1=2, p2=2)])
def test_run_matches_reference_run(ref, tmp_path, geom):
    text = config_text(32, **geom)
    ref.run_files(text, str(tmp_path / "ref"))
    parsed = S.parse_config_text(text)
    res = S.run(parsed.cfg, S.RunOptions(out_dir=str(tmp_path / "ours"), collective_timeout_s=300))
    assert res.status == "ok" and res.steps == 50
    assert len(res.samples) == 11
    assert res.backend == ("loopback" if geom["p"] == 1 else "inprocess")
    m = compare_runs(str(tmp_path / "ours"), str(tmp_path / "ref"))
    assert m["backend"] == res.backend and m["status"] == "ok"
    assert int(m["timed_steps"]) == 45 and float(m["step_seconds_mean"]) > 0


def test_run_isotropic_and_baseline_cases(tmp_path):
    for case in ("isotropic", "taylor_green_baseline"):
        cfg = S.SolverConfig(n=32, t_end=0.01, out_every=5, initial_case=case)
        res = S.run(cfg, S.RunOptions(out_dir=str(tmp_path / case)))
        assert res.status == "ok" and len(res.samples) == 3
        if case == "isotropic":
            assert abs(res.samples[0][1].energy - 0.5) < 1e-12
        else:
            assert abs(res.samples[0][1].energy - 0.125) < 1e-12
    with pytest.raises(S.ConfigError, match="unknown initial case 'vortex'"):
        S.run(S.SolverConfig(n=16, initial_case="vortex"), S.RunOptions(out_dir=str(tmp_path / "x")))


def test_run_divergence_matches_reference(ref, tmp_path):
    """Blow-up: the last sampled state is checkpointed, the manifest records
    the step and DivergenceError is raised (runner.cpp:113-146)."""
    text = config_text(16, t_end=100.0, out_every=2, nu=0.0, dt=5.0)
    with pytest.raises(ref.RefError) as r:
        ref.run_files(text, str(tmp_path / "ref"))
    assert r.value.code == 4
    parsed = S.parse_config_text(text)
    with pytest.raises(S.DivergenceError) as g:
        S.run(parsed.cfg, S.RunOptions(out_dir=str(tmp_path / "ours")))
    assert "checkpointed to" in str(g.value)
    m1 = read_manifest(tmp_path / "ours" / "manifest.txt")
    m2 = read_manifest(tmp_path / "ref" / "manifest.txt")
    assert m1["status"] == m2["status"] and m1["steps"] == m2["steps"]
    assert g.value.step == int(m2["status"].rsplit(" ", 1)[-1])
    c1, _ = read_checkpoint(tmp_path / "ours" / "checkpoint.sdns")
    c2, _ = read_checkpoint(tmp_path / "ref" / "checkpoint.sdns")
    assert (c1["t"], c1["step"]) == (c2["t"], c2["step"])


def test_bench_rows_and_csv(tmp_path):
    entries = S.parse_bench_matrix_text("16 slab 1\n32 slab 2\n32 pencil 4\n64 slab 1\n")
    rows = S.bench(entries, 3)
    assert [r.status for r in rows] == ["ok"] * 4
    assert all(np.isfinite(r.sec_per_step) and r.sec_per_step > 0 for r in rows)
    assert (rows[2].entry.p1, rows[2].entry.p2) == (2, 2)
    assert [r.nodes_per_rank for r in rows] == [4096, 16384, 8192, 262144]
    bad = S.bench([S.BenchEntry(2048, "slab", 1)], 2)
    assert bad[0].status.startswith("the sm_100a path supports n <= 1024")
    S.write_bench_csv(str(tmp_path / "b.csv"), rows + bad)
    lines = open(tmp_path / "b.csv").read().splitlines()
    assert lines[0] == "n,decomp,p,p1,p2,nodes_per_rank,sec_per_step,status"
    assert lines[3].startswith("32,pencil,4,2,2,8192,") and lines[3].endswith(",ok")


def test_cli_run_bench_verify(tmp_path):
    out = tmp_path / "run"
    r = subprocess.run([CLI, "run", "--n", "16", "--t-end", "0.02", "--out-every", "5",
                        "--out", str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == "running taylor_green: n=16 slab p=1 nu=0.000625 dt=0.001 t_end=0.02"
    assert lines[1].startswith("completed 20 steps; E=")
    assert lines[2].startswith("mean step time ") and lines[2].endswith(" s over 15 timed steps")
    assert lines[3] == f"wrote {out}/diagnostics.csv, {out}/checkpoint.sdns, {out}/manifest.txt"
    # divergence exits 2
    r = subprocess.run([CLI, "run", "--n", "16", "--nu", "0", "--dt", "5", "--t-end", "100",
                        "--out", str(tmp_path / "div")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 2 and "error: solution diverged:" in r.stderr
    m = tmp_path / "m.txt"
    m.write_text("16 slab 1\n16 slab 2\n")
    r = subprocess.run([CLI, "bench", "--matrix", str(m), "--steps", "2", "--out",
                        str(tmp_path / "b.csv")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.splitlines()[0] == "benchmarking 2 entries, 2 timed steps each"
    r = subprocess.run([CLI, "verify"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.splitlines()[-1] == "ALL CRITERIA PASSED"
    assert sum(l.startswith("[PASS] ") for l in r.stdout.splitlines()) == 9


def test_acceptance_suite_python():
    res = S.run_acceptance_suite(verbose=False)
    assert [r.index for r in res] == list(range(1, 10))
    assert all(r.passed for r in res), [(r.name, r.detail) for r in res if not r.passed]


def test_run_rank_matches_run(tmp_path):
    """run_worker for one rank of a caller-made group (sdns_run_rank: one
    process per GPU over NCCL in production) equals run() of the same config."""
    cfg = S.SolverConfig(n=32, p=2, t_end=0.02, out_every=5)
    S.run(cfg, S.RunOptions(out_dir=str(tmp_path / "run")))
    results = S.run_group(2, lambda rank, comm: S.run(
        cfg, S.RunOptions(out_dir=str(tmp_path / "rank")), comm=comm, rank=rank))
    assert results[0].backend == "inprocess" and results[0].status == "ok"
    a = open(tmp_path / "run" / "diagnostics.csv").read()
    b = open(tmp_path / "rank" / "diagnostics.csv").read()
    assert a == b
    assert (tmp_path / "run" / "checkpoint.sdns").read_bytes() == \
        (tmp_path / "rank" / "checkpoint.sdns").read_bytes()


def test_run_reruns_byte_identical_and_decomposition_invariant(tmp_path):
    """test_app.cpp pins: a rerun writes byte-identical diagnostics and
    checkpoint; p = 2 agrees with p = 1 to <= 1e-13."""
    cfg = S.SolverConfig(n=32, t_end=0.03, out_every=3)
    for d in ("a", "b"):
        S.run(cfg, S.RunOptions(out_dir=str(tmp_path / d)))
    for f in ("diagnostics.csv", "checkpoint.sdns"):
        assert (tmp_path / "a" / f).read_bytes() == (tmp_path / "b" / f).read_bytes()
    S.run(S.SolverConfig(n=32, p=2, t_end=0.03, out_every=3), S.RunOptions(out_dir=str(tmp_path / "p2")))
    _, a = read_csv(tmp_path / "a" / "diagnostics.csv")
    _, b = read_csv(tmp_path / "p2" / "diagnostics.csv")
    np.testing.assert_allclose(b[:, 2:5], a[:, 2:5], rtol=1e-13, atol=0)
    _, u1 = read_checkpoint(tmp_path / "a" / "checkpoint.sdns")
    _, u2 = read_checkpoint(tmp_path / "p2" / "checkpoint.sdns")
    assert np.max(np.abs(u1 - u2)) <= 1e-13 * np.max(np.abs(u1))
