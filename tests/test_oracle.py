"""CPU: pin the oracles before trusting them.

* The compiled reference (oracle/_ref, unmodified sources + FFTW shim) must
  pass the reference's own 8 doctest suites and 9-criterion acceptance gate
  (proj/tests/*.cpp, proj/core/src/verification.cpp:548-614).
* The numpy restatement (oracle/sdns_np.py) must agree with the compiled
  reference and with the committed golden fixtures (tests/golden/), and
  reproduce the reference's known answers.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import sdns_np as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "golden_ref.npz"))


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300)


@pytest.mark.parametrize("suite", ["grid", "transport", "serial_fft", "fft", "ns", "rk4",
                                   "diagnostics", "app"])
def test_reference_unit_suites_pass_on_shim(ref, suite, tmp_path):
    exe = os.path.join(ROOT, "oracle", "_ref", "sdns_tests")
    r = subprocess.run([exe, f"-ts={suite}"], cwd=tmp_path, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "Status: SUCCESS" in r.stdout


def test_reference_acceptance_gate(ref, tmp_path):
    exe = os.path.join(ROOT, "oracle", "_ref", "sdns_acceptance")
    r = subprocess.run([exe], cwd=tmp_path, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL CRITERIA PASSED (9 total)" in r.stdout


# --- numpy restatement vs golden fixtures (no reference needed) -------------

def test_np_fft_matches_golden():
    u = GOLD["fft8_u"]
    fu = O.forward(u)
    assert np.abs(fu - GOLD["fft8_slab1"]).max() <= 1e-12 * np.abs(fu).max()
    # every decomposition of the reference agrees (test_fft.cpp:73-110)
    for k in ("fft8_slab2", "fft8_slab4", "fft8_pencil22", "fft8_pencil24"):
        assert np.abs(GOLD[k] - GOLD["fft8_slab1"]).max() <= 1e-11
    assert np.abs(O.inverse(fu, 8) - u).max() <= 1e-13
    assert np.abs(GOLD["fft8_inverse"] - u).max() <= 1e-13


def test_np_pointwise_match_golden_bitwise():
    wm = O.Wavenumbers(8)
    uh = GOLD["pw8_uh"]
    assert np.array_equal(O.curl_hat(uh, wm), GOLD["pw8_curl"])
    assert np.array_equal(O.project(uh, wm), GOLD["pw8_project"])
    assert np.array_equal(O.pressure_hat(uh, wm), GOLD["pw8_pressure"])
    assert np.array_equal(O.cross(GOLD["pw8_a"], GOLD["pw8_b"]), GOLD["pw8_cross"])


def test_np_rhs_and_rk4_match_golden():
    wm = O.Wavenumbers(16)
    assert rel(O.compute_rhs(GOLD["rnd16_uh"], wm, 1e-3), GOLD["rnd16_rhs"]) < 1e-12
    st = O.Rk4State(GOLD["rnd16_uh"])
    rhs = lambda u: O.compute_rhs(u, wm, 1e-3)  # noqa: E731
    for _ in range(3):
        O.rk4_step_finite(st, 1e-3, rhs)
        st.u_hat = O.project(st.u_hat, wm)
    assert rel(st.u_hat, GOLD["rnd16_rk3"]) < 1e-12
    s = O.collect_stats(GOLD["rnd16_uh"], wm, 1e-3)
    g = GOLD["rnd16_stats"]
    assert abs(s["energy"] - g[1]) <= 1e-13 * g[1]
    assert abs(s["enstrophy"] - g[2]) <= 1e-13 * g[2]
    assert abs(s["divergence_max"] - g[4]) <= 1e-12
    assert np.allclose(s["spectrum"], g[5:], rtol=1e-12, atol=1e-300)


def test_np_taylor_green_trajectory_matches_golden():
    n = 16
    wm = O.Wavenumbers(n)
    uh0 = O.project(O.forward(O.taylor_green_baseline(n)), wm)
    assert rel(uh0, O.project(GOLD["tg16_uh0"], wm)) < 1e-14
    rows = []
    st = O.Rk4State(uh0)
    O.advance(st, wm, 0.01, 0.01, 0.1, 1,
              sample=lambda k, t: rows.append(O.collect_stats(st.u_hat, wm, 0.01, t)))
    g = GOLD["tg16_stats"]
    assert len(rows) == g.shape[0] == 11
    for r, gr in zip(rows, g):
        assert r["t"] == gr[0]
        assert abs(r["energy"] - gr[1]) <= 1e-12 * gr[1]
        assert abs(r["enstrophy"] - gr[2]) <= 1e-12 * gr[2]
    assert rel(st.u_hat, GOLD["tg16_final"]) < 1e-11


def test_known_answers():
    """proj/tests/test_diagnostics.cpp:45-66, test_ns.cpp:68-76."""
    assert [O.spectrum_shells(n) for n in (8, 16, 32, 64)] == [8, 15, 29, 56]
    a = np.array([1.0, 2.0, 3.0]).reshape(3, 1, 1, 1)
    b = np.array([4.0, 5.0, 6.0]).reshape(3, 1, 1, 1)
    assert O.cross(a, b).ravel().tolist() == [-3.0, 6.0, -3.0]
    for n in (8, 16):
        wm = O.Wavenumbers(n)
        for init in (O.taylor_green_reference, O.taylor_green_baseline):
            s = O.collect_stats(O.forward(init(n)), wm, 0.01)
            assert abs(s["energy"] - 0.125) <= 1e-13 * 0.125
            assert abs(s["enstrophy"] - 0.375) <= 1e-13 * 0.375
            assert s["spectrum"].argmax() == 2  # shell round(sqrt(3))
    assert O.step_count(0.1, 1e-3) == 100
    assert O.step_count(0.1, 0.03) == 4
    lo = O.build_layout(8, "pencil", 4, 2, 2, 3)
    assert lo["stages"][0][0] == [48, 32] and lo["stages"][0][1] == [32, 32]  # test_grid.cpp


# --- numpy restatement vs compiled reference on fresh inputs ------------------

@pytest.mark.parametrize("n", [8, 16, 32])
def test_np_vs_reference_rhs(ref, n):
    rng = np.random.default_rng(n)
    u = rng.uniform(-1, 1, (3, n, n, n))
    wm = O.Wavenumbers(n)
    uh = O.project(O.forward(u), wm) / n**3
    a = O.compute_rhs(uh, wm, 0.01)
    b = ref.compute_rhs(uh, n, 0.01)
    assert rel(a, b) < 1e-12


def test_np_vs_reference_pencil_and_slab_run(ref):
    n = 16
    wm = O.Wavenumbers(n)
    uh0 = ref.forward(O.taylor_green_baseline(n), n)
    s1, f1 = ref.run(uh0, n, 0.01, 0.01, 4)
    s2, f2 = ref.run(uh0, n, 0.01, 0.01, 4, decomp="slab", p=4)
    s3, f3 = ref.run(uh0, n, 0.01, 0.01, 4, decomp="pencil", p=4, p1=2, p2=2)
    assert rel(f2, f1) < 1e-12 and rel(f3, f1) < 1e-12
    st = O.Rk4State(O.project(uh0, wm))
    O.advance(st, wm, 0.01, 0.01, 0.04)
    assert rel(st.u_hat, f1) < 1e-11


def test_reference_checkpoint_decomposition_independent(ref, tmp_path):
    """Pins the checkpoint format the product writes: the compiled reference
    reads across decompositions bit-exactly (checkpoint.hpp:11-15)."""
    n = 8
    u = np.random.default_rng(11).uniform(-1, 1, (3, n, n, n))
    path = str(tmp_path / "c.ck")
    ref.checkpoint_write(path, u, n, 0.75, 4, decomp="pencil", p=4, p1=2, p2=2)
    raw = open(path, "rb").read()
    assert raw[:4] == b"SDNS" and len(raw) == 32 + 3 * n ** 3 * 8
    assert np.frombuffer(raw[:16], dtype="<u4")[1:].tolist() == [1, n, 3]
    assert np.frombuffer(raw[16:24], dtype="<f8")[0] == 0.75
    assert np.frombuffer(raw[24:32], dtype="<u8")[0] == 4
    assert np.array_equal(np.frombuffer(raw[32:], dtype="<f8").reshape(3, n, n, n), u)
    v, t, step = ref.checkpoint_read(path, n, decomp="slab", p=2)
    assert np.array_equal(v, u) and (t, step) == (0.75, 4)
