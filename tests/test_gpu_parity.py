"""GPU parity: the sm_100a path (through the C ABI) against the oracles.

Bars (BASELINE.json north_star): FFT vs reference <= 1e-11 * max|X| and
round trip <= 1e-13 relative L2; pointwise operators bitwise; velocity field
relative L2 <= 1e-11 after 10 RK4 steps; energy and enstrophy <= 1e-12
relative per sampled step.
"""
import os

import numpy as np
import pytest

import paper_1607_00850_b200 as S
from oracle import sdns_np as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "golden_ref.npz"))


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300)


def ctx_for(n, nu=0.01, dt=0.01, steps=10, out_every=1, dealias=True):
    cfg = S.SolverConfig(n=n, nu=nu, dt=dt, t_end=steps * dt, dealias=dealias,
                         out_every=out_every)
    return S.Context(cfg)


# --- transforms ------------------------------------------------------------------

@pytest.mark.parametrize("n", [4, 8, 16, 32, 64, 128, 256])
def test_fft_forward_inverse_vs_numpy(n):
    rng = np.random.default_rng(42 + n)
    u = rng.uniform(-1, 1, (3, n, n, n))
    with ctx_for(n) as c:
        fft = S.DistributedFFT(c)
        fu_d, u_d = c.spectral_field(), c.real_field()
        u_d.upload(u)
        fft.forward(u_d, fu_d)
        fu = fu_d.download()
        ref = O.forward(u)
        assert np.abs(fu - ref).max() <= 1e-11 * np.abs(ref).max()
        back = c.real_field()
        fft.inverse(fu_d, back)
        assert rel(back.download(), u) <= 1e-13


def test_fft_matches_reference_golden():
    u = GOLD["fft8_u"]
    with ctx_for(8) as c:
        fft = S.DistributedFFT(c)
        ud, fd = c.real_field().upload(u), c.spectral_field()
        fft.forward(ud, fd)
        fu = fd.download()
        g = GOLD["fft8_slab1"]
        assert np.abs(fu - g).max() <= 1e-11 * np.abs(g).max()


def test_fft_constant_field_and_cosine_spike():
    """proj/tests/test_fft.cpp:112-175: DC of a constant = 2.5 n^3, cos(x)
    spike = n^3/2, inverse of the DC spike recovers 2.5 everywhere."""
    n = 16
    with ctx_for(n) as c:
        fft = S.DistributedFFT(c)
        u = np.full((3, n, n, n), 2.5)
        fd = c.spectral_field()
        fft.forward(c.real_field().upload(u), fd)
        fu = fd.download()
        assert abs(fu[0, 0, 0, 0] - 2.5 * n**3) <= 1e-9
        fu0 = fu.copy()
        fu0[:, 0, 0, 0] = 0
        assert np.abs(fu0).max() <= 1e-9
        back = c.real_field()
        fft.inverse(fd, back)
        assert np.allclose(back.download(), 2.5, rtol=0, atol=1e-13)
        x = O.physical_axis(n)
        u = np.broadcast_to(np.cos(x)[:, None, None], (3, n, n, n)).copy()
        fft.forward(c.real_field().upload(u), fd)
        fu = fd.download()
        assert abs(fu[0, 1, 0, 0] - n**3 / 2) <= 1e-9
        assert abs(fu[0, n - 1, 0, 0] - n**3 / 2) <= 1e-9


def test_c2r_ignores_imaginary_dc_and_nyquist():
    """FFTW c2r semantics: Im of the kz = 0 and kz = n/2
    bins does not reach the real output, exactly as the reference."""
    n = 16
    rng = np.random.default_rng(7)
    u = rng.uniform(-1, 1, (3, n, n, n))
    uh = O.forward(u)
    bad = uh.copy()
    bad[:, 3, 5, 0] += 0.25j
    bad[:, 2, 1, n // 2] -= 0.5j
    with ctx_for(n) as c:
        fft = S.DistributedFFT(c)
        out = c.real_field()
        fft.inverse(c.spectral_field().upload(bad), out)
        got = out.download()
    expect = O.inverse(bad, n)  # pocketfft c2r also drops them
    assert np.abs(got - expect).max() <= 1e-14 * max(1.0, np.abs(expect).max())


# --- pointwise operators: bitwise ---------------------------------------------------

def test_pointwise_ops_bitwise_vs_reference():
    uh = GOLD["pw8_uh"]
    with ctx_for(8) as c:
        u = c.spectral_field().upload(uh)
        w = c.spectral_field()
        S.curl_hat(c, u, w)
        assert np.array_equal(w.download(), GOLD["pw8_curl"])
        p = c.spectral_field(1)
        S.pressure_hat(c, u, p)
        assert np.array_equal(p.download()[0], GOLD["pw8_pressure"])
        S.project(c, u)
        assert np.array_equal(u.download(), GOLD["pw8_project"])
        a = c.real_field().upload(GOLD["pw8_a"])
        b = c.real_field().upload(GOLD["pw8_b"])
        o = c.real_field()
        S.cross(c, a, b, o)
        assert np.array_equal(o.download(), GOLD["pw8_cross"])


# --- compute_rhs -------------------------------------------------------------------

def test_compute_rhs_matches_reference_golden():
    for key_in, key_out, n, nu in (("rnd16_uh", "rnd16_rhs", 16, 1e-3),):
        with ctx_for(n) as c:
            u = c.spectral_field().upload(GOLD[key_in])
            du = c.spectral_field()
            S.compute_rhs(c, u, nu, du)
            assert rel(du.download(), GOLD[key_out]) <= 1e-12


@pytest.mark.parametrize("n", [4, 16, 32, 64])
def test_compute_rhs_vs_numpy_oracle(n):
    rng = np.random.default_rng(n)
    wm = O.Wavenumbers(n)
    uh = O.project(O.forward(rng.uniform(-1, 1, (3, n, n, n))), wm) / n**3
    expect = O.compute_rhs(uh, wm, 0.01)
    with ctx_for(n) as c:
        du = c.spectral_field()
        S.compute_rhs(c, c.spectral_field().upload(uh), 0.01, du)
        assert rel(du.download(), expect) <= 1e-12


@pytest.mark.parametrize("dealias", [False, True])
def test_compute_rhs_dealias_switch(dealias):
    """dealias = false disables the 2/3 rule (and the forward pruning)."""
    n = 32
    rng = np.random.default_rng(5)
    wm = O.Wavenumbers(n, dealias=dealias)
    uh = O.project(O.forward(rng.uniform(-1, 1, (3, n, n, n))), wm) / n**3
    expect = O.compute_rhs(uh, wm, 0.02)
    with ctx_for(n, dealias=dealias) as c:
        du = c.spectral_field()
        S.compute_rhs(c, c.spectral_field().upload(uh), 0.02, du)
        got = du.download()
    assert rel(got, expect) <= 1e-12
    if not dealias:  # the masked band carries the nonlinear term when the rule is off
        band = ~O.Wavenumbers(n, dealias=True).mask
        assert np.abs(got[:, band]).max() > 1e-6


def test_compute_rhs_solenoidal_and_linear_in_nu():
    """proj/tests/test_ns.cpp:170-214: k . du = 0, d(du)/d(nu) = -k^2 u."""
    n = 16
    wm = O.Wavenumbers(n)
    uh = O.project(O.forward(O.taylor_green_baseline(n)), wm)
    with ctx_for(n) as c:
        u = c.spectral_field().upload(uh)
        d0, d1 = c.spectral_field(), c.spectral_field()
        S.compute_rhs(c, u, 0.0, d0)
        S.compute_rhs(c, u, 0.1, d1)
        a, b = d0.download(), d1.download()
    kd = (wm.KX * a[0] + wm.KY * a[1]) + wm.KZ * a[2]
    assert np.abs(kd).max() <= 1e-9 * max(1.0, np.abs(a).max())
    assert np.abs((b - a) / 0.1 + wm.k2[None] * uh).max() <= 1e-10 * np.abs(wm.k2[None] * uh).max()


# --- RK4 trajectories -----------------------------------------------------------

def spectrum_close(a, b, energy, rtol=1e-11, eps=1e-15):
    """Shell spectra agree to rtol, or to the roundoff of the shell's modes:
    a velocity error of eps * sqrt(E) moves a shell holding E_k by at most
    2 sqrt(E_k) eps sqrt(E) (deep cascade shells, E_k / E ~ 1e-18, sit at
    that level after a few steps whatever the FFT's rounding)."""
    a, b = np.asarray(a), np.asarray(b)
    tol = rtol * np.abs(b) + 2.0 * np.sqrt(np.abs(b)) * eps * np.sqrt(energy) + 1e-300
    return bool(np.all(np.abs(a - b) <= tol))


def run_gpu(n, uh0, nu, dt, steps, out_every=1, project_init=True):
    cfg = S.SolverConfig(n=n, nu=nu, dt=dt, t_end=steps * dt, out_every=out_every)
    with S.Context(cfg) as c:
        u = c.spectral_field().upload(uh0)
        if project_init:
            S.project(c, u)
        st = S.Rk4State(c)
        st.set(u)
        rows = []
        st.advance(lambda k, t: rows.append(S.collect_stats(c, st.u_hat, nu, t)))
        final = st.u_hat.download()
        st.close()
    return rows, final


def test_taylor_green_16_matches_reference_golden():
    rows, final = run_gpu(16, GOLD["tg16_uh0"], 0.01, 0.01, 10)
    g = GOLD["tg16_stats"]
    assert len(rows) == g.shape[0]
    for r, gr in zip(rows, g):
        assert r.t == gr[0]
        assert abs(r.energy - gr[1]) <= 1e-12 * gr[1]
        assert abs(r.enstrophy - gr[2]) <= 1e-12 * gr[2]
        assert spectrum_close(r.spectrum, gr[5:], gr[1])
    assert rel(final, GOLD["tg16_final"]) <= 1e-11


def test_config1_taylor_green_64_100_steps_vs_reference(ref):
    """BASELINE config 1: TG n=64, nu=0.01, dt=0.01, 100 steps, E and Z every step."""
    n, nu, dt, steps = 64, 0.01, 0.01, 100
    uh0 = ref.forward(O.taylor_green_baseline(n), n)
    gs, gf = ref.run(uh0, n, nu, dt, steps, out_every=1, decomp="slab", p=8)
    rows, final = run_gpu(n, uh0, nu, dt, steps)
    assert len(rows) == gs.shape[0] == steps + 1
    for r, gr in zip(rows, gs):
        assert abs(r.energy - gr[1]) <= 1e-12 * gr[1]
        assert abs(r.enstrophy - gr[2]) <= 1e-12 * gr[2]
        assert r.divergence_max <= 1e-10
    assert rel(final, gf) <= 1e-11


def test_smallest_mesh_n4_10_steps_vs_reference(ref):
    """n = 4, the smallest mesh the reference accepts (config.cpp:18-19):
    10 RK4 steps of a random solenoidal field against the compiled reference."""
    n, nu, dt = 4, 1e-2, 1e-2
    rng = np.random.default_rng(44)
    wm = O.Wavenumbers(n)
    uh0 = O.project(O.forward(rng.uniform(-1, 1, (3, n, n, n))), wm) / n**3
    gs, gf = ref.run(uh0, n, nu, dt, 10, out_every=1, init_project=False, p=2)
    rows, final = run_gpu(n, uh0, nu, dt, 10, project_init=False)
    for r, gr in zip(rows, gs):
        assert abs(r.energy - gr[1]) <= 1e-12 * gr[1]
        assert abs(r.enstrophy - gr[2]) <= 1e-12 * gr[2]
    assert rel(final, gf) <= 1e-11


def test_smallest_mesh_n4_decompositions_agree(tmp_path):
    """n = 4 over slab p = 1, 2, 4 and pencil 2x2 (ranks as threads): the
    same Taylor-Green samples."""
    got = []
    for i, geom in enumerate([dict(), dict(p=2), dict(p=4), dict(decomp="pencil", p=4, p1=2, p2=2)]):
        cfg = S.SolverConfig(n=4, nu=1e-2, dt=1e-2, t_end=0.05, out_every=1, **geom)
        r = S.run(cfg, S.RunOptions(out_dir=str(tmp_path / str(i))))
        got.append([(st.energy, st.enstrophy) for _, st in r.samples])
    for g in got[1:]:
        assert np.allclose(g, got[0], rtol=1e-13, atol=0)


@pytest.mark.parametrize("n", [32, 64])
def test_iso_10_steps_vs_reference(ref, n):
    """Configs 2-4 construction at test size: iso field, 10 RK4 steps."""
    cfg = S.SolverConfig(n=n)
    lo = S.build_layout(cfg, 0)
    uh0 = S.iso_init(n, lo, seed=1607)
    nu, dt = 1e-3, 1e-3
    gs, gf = ref.run(uh0, n, nu, dt, 10, out_every=1, init_project=False, p=8)
    rows, final = run_gpu(n, uh0, nu, dt, 10, project_init=False)
    assert abs(rows[0].energy - 0.5) <= 1e-13
    for r, gr in zip(rows, gs):
        assert abs(r.energy - gr[1]) <= 1e-12 * gr[1]
        assert abs(r.enstrophy - gr[2]) <= 1e-12 * gr[2]
    assert rel(final, gf) <= 1e-11


def test_rk4_steps_match_reference_golden():
    n = 16
    cfg = S.SolverConfig(n=n, nu=1e-3, dt=1e-3)
    with S.Context(cfg) as c:
        st = S.Rk4State(c)
        st.set(c.spectral_field().upload(GOLD["rnd16_uh"]))
        for _ in range(3):
            st.rk4_step(1e-3, post_project=True)
        assert rel(st.u_hat.download(), GOLD["rnd16_rk3"]) <= 1e-12
        assert st.step == 3
        st.close()


def test_stats_match_reference():
    n = 16
    with ctx_for(n) as c:
        s = S.collect_stats(c, c.spectral_field().upload(GOLD["rnd16_uh"]), 1e-3)
    g = GOLD["rnd16_stats"]
    assert abs(s.energy - g[1]) <= 1e-13 * g[1]
    assert abs(s.enstrophy - g[2]) <= 1e-13 * g[2]
    assert abs(s.dissipation - g[3]) <= 1e-13 * g[3]
    assert abs(s.divergence_max - g[4]) <= 1e-12 * max(g[4], 1e-300) + 1e-15
    assert np.allclose(s.spectrum, g[5:], rtol=1e-12, atol=1e-300)


def test_stats_deterministic_bitwise():
    n = 32
    lo = S.build_layout(S.SolverConfig(n=n), 0)
    uh = S.iso_init(n, lo)
    with ctx_for(n) as c:
        u = c.spectral_field().upload(uh)
        a = S.collect_stats(c, u, 1e-3)
        b = S.collect_stats(c, u, 1e-3)
    assert a.energy == b.energy and a.enstrophy == b.enstrophy
    assert np.array_equal(a.spectrum, b.spectrum)


@pytest.mark.parametrize("n", [16, 64])
def test_sampled_stats_fused_into_last_stage(n):
    """advance() accumulates the diagnostics of each sampled step's final state
    inside the last stage update. Inside the hook they must
    equal, bit for bit, collect_stats of a copy of that state, and sampling must
    not change the trajectory."""
    lo = S.build_layout(S.SolverConfig(n=n), 0)
    uh0 = S.iso_init(n, lo, seed=3)
    nu, dt, steps = 2e-3, 2e-3, 4

    def run(every, check):
        cfg = S.SolverConfig(n=n, nu=nu, dt=dt, t_end=steps * dt, out_every=every)
        with S.Context(cfg) as c:
            st = S.Rk4State(c)
            st.set(c.spectral_field().upload(uh0))
            seen = []

            def hook(k, t):
                fused = S.collect_stats(c, st.u_hat, nu, t)
                copy = c.spectral_field().upload(st.u_hat.download())
                plain = S.collect_stats(c, copy, nu, t)
                seen.append((k, fused, plain))

            st.advance(hook if check else None)
            final = st.u_hat.download()
            st.close()
        return final, seen

    final_s, seen = run(1, True)
    final_n, _ = run(steps, False)
    assert np.array_equal(final_s, final_n)
    assert [k for k, _, _ in seen] == list(range(steps + 1))
    for _, f, p in seen:
        assert f.energy == p.energy and f.enstrophy == p.enstrophy
        assert f.divergence_max == p.divergence_max
        assert np.array_equal(f.spectrum, p.spectrum)


# --- advance semantics and errors ------------------------------------------------

def test_advance_schedule_and_shortened_last_step():
    """rk4.cpp:86-107: t_end = 0.1, dt = 0.03 -> 4 steps, last dt = 0.01."""
    n = 8
    cfg = S.SolverConfig(n=n, nu=0.01, dt=0.03, t_end=0.1, out_every=2)
    with S.Context(cfg) as c:
        u = c.spectral_field().upload(GOLD["pw8_uh"] * 1e-3)
        S.project(c, u)
        st = S.Rk4State(c)
        st.set(u)
        seen = []
        st.advance(lambda k, t: seen.append((k, t)))
        assert seen == [(0, 0.0), (2, 0.06), (4, 0.1)]
        assert st.t == 0.1 and st.step == 4
        st.close()


def test_divergence_error_on_nonfinite():
    n = 8
    cfg = S.SolverConfig(n=n, nu=0.01, dt=0.01, t_end=0.02)
    with S.Context(cfg) as c:
        uh = GOLD["pw8_uh"].copy()
        uh[0, 1, 1, 1] = np.nan
        st = S.Rk4State(c)
        st.set(c.spectral_field().upload(uh))
        with pytest.raises(S.DivergenceError) as ei:
            st.advance()
        assert ei.value.step == 1
        st.close()


@pytest.mark.parametrize("geom", [dict(p=2), dict(decomp="pencil", p=4, p1=2, p2=2)])
def test_divergence_detection_is_collective(geom):
    """test_rk4.cpp:164-189: one rank goes non-finite, every rank raises
    DivergenceError at the same step."""
    n = 16
    cfg = S.SolverConfig(n=n, nu=0.01, dt=0.01, t_end=0.05, **geom)
    uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=5)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            uh = _scatter_spec(uh0, c.layout).copy()
            if rank == 0:
                uh[1, 0, 0, 1] = np.inf
            st = S.Rk4State(c)
            st.set(c.spectral_field().upload(uh))
            try:
                st.advance()
            except S.DivergenceError as e:
                return e.step
            finally:
                st.close()
            return None

    assert S.run_group(cfg.p, body) == [1] * cfg.p


@pytest.mark.parametrize("geom", [dict(), dict(p=4), dict(decomp="pencil", p=4, p1=2, p2=2)])
def test_vector_transforms_equal_component_calls(geom):
    """test_fft.cpp:129-156: the 3-component forward equals three
    single-component calls bit for bit; the round trip is <= 1e-13."""
    n = 16
    cfg = S.SolverConfig(n=n, **geom)
    u0 = np.random.default_rng(900).uniform(-1, 1, (3, n, n, n))

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            fft = S.DistributedFFT(c)
            u = c.real_field().upload(_scatter_real(u0, c.layout))
            fu = c.spectral_field()
            fft.forward(u, fu)
            whole = fu.download()
            ok = True
            for comp in range(3):
                one_r = c.real_field(1).upload(_scatter_real(u0, c.layout)[comp:comp + 1])
                one = c.spectral_field(1)
                fft.forward(one_r, one)
                ok &= np.array_equal(one.download()[0], whole[comp])
            back = c.real_field()
            fft.inverse(fu, back)
            err = np.max(np.abs(back.download() - _scatter_real(u0, c.layout)))
            return ok, err

    for ok, err in S.run_group(cfg.p, body):
        assert ok and err <= 1e-13


def test_l2_diff_and_shells_of_taylor_green():
    """test_diagnostics.cpp:80-145: TG energy lies in shell 2 and the shells
    sum to E; l2_diff(u, 0) = sqrt(2E) = 0.5, l2_diff(u, u) = 0."""
    n = 16
    with S.Context(S.SolverConfig(n=n)) as c:
        u = c.real_field().upload(O.taylor_green_reference(n))
        uh = c.spectral_field()
        S.DistributedFFT(c).forward(u, uh)
        st = S.collect_stats(c, uh, 0.0)
        assert abs(st.energy - 0.125) <= 1e-13
        assert abs(st.spectrum[2] - st.energy) <= 1e-13
        assert abs(st.spectrum.sum() - st.energy) <= 1e-13
        zero = c.real_field().upload(np.zeros((3, n, n, n)))
        assert abs(S.l2_diff(c, u, zero) - 0.5) <= 0.5e-13
        assert S.l2_diff(c, u, u) == 0.0


def test_config_errors():
    with pytest.raises(S.ConfigError):
        S.Context(S.SolverConfig(n=2048))  # beyond the z pass's shared memory
    with pytest.raises(S.ConfigError):
        S.Context(S.SolverConfig(n=7))
    with pytest.raises(S.ConfigError):
        S.Context(S.SolverConfig(n=2))  # the reference's own minimum is 4
    with ctx_for(8) as c:
        u = c.spectral_field()
        with pytest.raises(S.ConfigError):
            S.compute_rhs(c, u, 0.01, u)


# --- multi-rank decomposition on one GPU (threads-as-ranks) ------------------------

def _scatter_spec(g, lo):
    (s0, s1, s2), (o0, o1, o2) = lo.spec_shape, lo.spec_offset
    return g[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2]


def _scatter_real(g, lo):
    (s0, s1, s2), (o0, o1, o2) = lo.real_shape, lo.real_offset
    return g[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2]


@pytest.mark.parametrize("p", [2, 4, 8])
def test_inprocess_slab_fft_matches_single_rank(p):
    n = 32
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, (3, n, n, n))
    expect = O.forward(u)
    cfg = S.SolverConfig(n=n, p=p)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            fft = S.DistributedFFT(c)
            lo = c.layout
            ud = c.real_field().upload(_scatter_real(u, lo))
            fd = c.spectral_field()
            fft.forward(ud, fd)
            back = c.real_field()
            fft.inverse(fd, back)
            return lo, fd.download(), back.download()

    out = S.run_group(p, body)
    for lo, fu, back in out:
        e = _scatter_spec(expect, lo)
        assert np.abs(fu - e).max() <= 1e-11 * np.abs(expect).max()
        assert rel(back, _scatter_real(u, lo)) <= 1e-13


@pytest.mark.parametrize("p", [2, 4])
def test_inprocess_slab_rk4_matches_single_rank(p):
    n = 32
    lo1 = S.build_layout(S.SolverConfig(n=n), 0)
    uh0 = S.iso_init(n, lo1)
    _, f1 = run_gpu(n, uh0, 1e-3, 1e-3, 5, project_init=False)
    cfg = S.SolverConfig(n=n, p=p, nu=1e-3, dt=1e-3, t_end=5e-3, out_every=1)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            lo = c.layout
            uh = S.iso_init(n, lo)
            assert np.array_equal(uh, _scatter_spec(uh0, lo))
            st = S.Rk4State(c)
            st.set(c.spectral_field().upload(uh))
            rows = []
            st.advance(lambda k, t: rows.append(S.collect_stats(c, st.u_hat, 1e-3, t)))
            out = (lo, st.u_hat.download(), rows)
            st.close()
            return out

    res = S.run_group(p, body)
    for lo, f, rows in res:
        assert rel(f, _scatter_spec(f1, lo)) <= 1e-12
    for r in range(1, p):
        for a, b in zip(res[0][2], res[r][2]):
            assert a.energy == b.energy and a.enstrophy == b.enstrophy


@pytest.mark.parametrize("geom", [dict(p=2), dict(p=4), dict(p=8),
                                  dict(decomp="pencil", p=2, p1=2, p2=1),
                                  dict(decomp="pencil", p=2, p1=1, p2=2),
                                  dict(decomp="pencil", p=4, p1=2, p2=2),
                                  dict(decomp="pencil", p=8, p1=2, p2=4),
                                  dict(decomp="pencil", p=8, p1=4, p2=2)])
def test_inprocess_transpose_modes_bitwise(geom):
    """Slab p > 1 and the pencil transposes (column group p1 > 1: P1 / P4;
    row group p2 > 1: P2 / the z pass) run fused into the producing passes by
    default (stores straight into the owning rank's buffer, a stream barrier
    after each: peer-direct), else as
    all-to-alls -- overlapped with the next group's transforms for slab
    (context option all_to_all), else serial (all_to_all + serial). The transforms and
    arithmetic are the same, so one RHS and two RK4 steps must agree bit for
    bit across the modes."""
    n = 32
    p = geom["p"]
    lo1 = S.build_layout(S.SolverConfig(n=n), 0)
    uh0 = S.iso_init(n, lo1, seed=9)
    cfg = S.SolverConfig(n=n, nu=1e-3, dt=1e-3, t_end=1e-3, **geom)

    def run():
        def body(rank, comm):
            with S.Context(cfg, rank=rank, comm=comm) as c:
                u = c.spectral_field().upload(_scatter_spec(uh0, c.layout))
                du = c.spectral_field()
                S.compute_rhs(c, u, 1e-3, du)
                st = S.Rk4State(c)
                st.set(u)
                st.rk4_step(1e-3)
                st.rk4_step(1e-3)
                out = c.spectral_field()
                st.get(out)
                # the distributed FFT API (slab: fused transposes too)
                fft = S.DistributedFFT(c)
                ur = c.real_field()
                fft.inverse(out, ur)
                fu = c.spectral_field()
                fft.forward(ur, fu)
                return du.download(), out.download(), ur.download(), fu.download()
        return S.run_group(p, body)

    modes = {}
    for name, opt in (("peer", {}), ("overlap", {"all_to_all": 1}),
                      ("serial", {"all_to_all": 1, "serial": 1})):
        with S.context_options(**opt):
            modes[name] = run()
    for name in ("overlap", "serial"):
        for a, b in zip(modes["peer"], modes[name]):
            for x, y in zip(a, b):
                assert np.array_equal(x, y), name


@pytest.mark.gpu
@pytest.mark.parametrize("n,geom", [(128, dict(p=1)), (256, dict(p=1)), (256, dict(p=2)),
                                    (128, dict(decomp="pencil", p=4, p1=2, p2=2)),
                                    (512, dict(p=1))])
def test_p1_single_transform_items(n, geom):
    """The x inverse pass (P1) as five single-transform items on one tile
    buffer -- what n = 1024 runs, where two 128 B-row tiles plus a scratch
    tile do not fit -- forced at smaller n (context option p1_single) against
    the default three-item kernel: the same transforms and operations, so one
    RHS must agree to rounding (the compiler contracts the kx products into
    FMAs differently in the two kernels: bitwise at 256, 512 and 1024, 3e-16
    at 128) at p = 1 (chunk-major and plain layouts), slab and pencil with
    peer-direct stores, and with all-to-all transposes; the variants of the
    single-item kernel itself (TMA / LDGSTS tiles, layouts, transposes) must
    agree bit for bit."""
    p = geom["p"]
    uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=11)
    cfg = S.SolverConfig(n=n, nu=1e-3, dt=1e-3, t_end=1e-3, **geom)

    def run():
        def body(rank, comm):
            with S.Context(cfg, rank=rank, comm=comm) as c:
                u = c.spectral_field().upload(_scatter_spec(uh0, c.layout))
                du = c.spectral_field()
                S.compute_rhs(c, u, 1e-3, du)
                return du.download()
        return S.run_group(p, body)

    base = run()
    variants = [dict(p1_single=1), dict(p1_single=1, ldgsts_tiles=1)]
    variants.append(dict(p1_single=1, plain_layout=1) if p == 1 else dict(p1_single=1, all_to_all=1))
    first = None
    for opt in variants:
        with S.context_options(**opt):
            got = run()
        # one scale for all ranks: a pencil rank that owns only high kz holds
        # values ~1e-13 of the field's largest modes, and the rounding noise
        # of the unnormalised transforms is absolute, not relative to them
        scale = max(np.abs(a).max() for a in base)
        for a, b in zip(base, got):
            assert np.abs(a - b).max() <= 4e-15 * scale, opt
        if first is None:
            first = got
        for a, b in zip(first, got):
            assert np.array_equal(a, b), opt


# --- pencil decomposition (fft.cpp:130-227) on one GPU ---------------------------

PENCILS = [(2, 1), (1, 2), (2, 2), (2, 4), (4, 2)]


@pytest.mark.parametrize("p1,p2", PENCILS)
def test_inprocess_pencil_fft_matches_reference_golden_rule(p1, p2):
    """Distributed forward/inverse on a p1 x p2 pencil grid vs the global FFT
    (proj/tests/test_fft.cpp:73-110 runs pencil 1, 2x2, 2x4 at n = 8)."""
    n = 16
    rng = np.random.default_rng(9)
    u = rng.uniform(-1, 1, (3, n, n, n))
    expect = O.forward(u)
    cfg = S.SolverConfig(n=n, decomp="pencil", p=p1 * p2, p1=p1, p2=p2)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            fft = S.DistributedFFT(c)
            lo = c.layout
            fd = c.spectral_field()
            fft.forward(c.real_field().upload(_scatter_real(u, lo)), fd)
            back = c.real_field()
            fft.inverse(fd, back)
            return lo, fd.download(), back.download()

    for lo, fu, back in S.run_group(p1 * p2, body):
        assert np.abs(fu - _scatter_spec(expect, lo)).max() <= 1e-11 * np.abs(expect).max()
        assert rel(back, _scatter_real(u, lo)) <= 1e-13


def test_pencil_fft_golden_n8_2x4():
    """The reference's own pencil 2x4 result at n = 8 (tests/golden)."""
    n = 8
    u = GOLD["fft8_u"]
    cfg = S.SolverConfig(n=n, decomp="pencil", p=8, p1=2, p2=4)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            fd = c.spectral_field()
            S.DistributedFFT(c).forward(c.real_field().upload(_scatter_real(u, c.layout)), fd)
            return c.layout, fd.download()

    g = GOLD["fft8_pencil24"]
    for lo, fu in S.run_group(8, body):
        assert np.abs(fu - _scatter_spec(g, lo)).max() <= 1e-11 * np.abs(g).max()


@pytest.mark.parametrize("p1,p2", [(2, 2), (2, 4)])
def test_inprocess_pencil_rk4_matches_single_rank(p1, p2):
    """Configs 4 construction at test size: iso field, pencil p1 x p2 vs p = 1."""
    n = 32
    lo1 = S.build_layout(S.SolverConfig(n=n), 0)
    uh0 = S.iso_init(n, lo1)
    _, f1 = run_gpu(n, uh0, 1e-3, 1e-3, 4, project_init=False)
    cfg = S.SolverConfig(n=n, decomp="pencil", p=p1 * p2, p1=p1, p2=p2, nu=1e-3, dt=1e-3,
                         t_end=4e-3, out_every=1)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            lo = c.layout
            st = S.Rk4State(c)
            st.set(c.spectral_field().upload(S.iso_init(n, lo)))
            rows = []
            st.advance(lambda k, t: rows.append(S.collect_stats(c, st.u_hat, 1e-3, t)))
            out = (lo, st.u_hat.download(), rows)
            st.close()
            return out

    res = S.run_group(p1 * p2, body)
    for lo, f, rows in res:
        assert rel(f, _scatter_spec(f1, lo)) <= 1e-12
    for r in range(1, p1 * p2):
        for a, b in zip(res[0][2], res[r][2]):
            assert a.energy == b.energy and a.enstrophy == b.enstrophy


def test_pencil_compute_rhs_vs_reference_pencil(ref):
    """compute_rhs on the reference's own pencil 2x2 decomposition."""
    n = 16
    uh = GOLD["rnd16_uh"]
    expect = ref.compute_rhs(uh, n, 1e-3, decomp="pencil", p=4, p1=2, p2=2)
    cfg = S.SolverConfig(n=n, decomp="pencil", p=4, p1=2, p2=2)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            du = c.spectral_field()
            S.compute_rhs(c, c.spectral_field().upload(_scatter_spec(uh, c.layout)), 1e-3, du)
            return c.layout, du.download()

    for lo, du in S.run_group(4, body):
        e = _scatter_spec(expect, lo)
        assert np.linalg.norm(du - e) <= 1e-12 * np.linalg.norm(expect)


# --- checkpoints (checkpoint.cpp:64-187) ----------------------

def test_checkpoint_round_trip_with_reference(ref, tmp_path):
    """Our file is the reference's format: the reference reads what we write
    and we read what it writes, bit for bit, header included."""
    n = 16
    u = np.random.default_rng(5).uniform(-1, 1, (3, n, n, n))
    ours = str(tmp_path / "ours.ck")
    theirs = str(tmp_path / "sub" / "theirs.ck")
    with ctx_for(n) as c:
        S.write_checkpoint(c, ours, c.real_field().upload(u), 0.25, 12)
        v, t, step = ref.checkpoint_read(ours, n)
        assert np.array_equal(v, u) and t == 0.25 and step == 12
        ref.checkpoint_write(theirs, u[::-1].copy(), n, 1.5, 3)
        back = c.real_field()
        t2, s2 = S.read_checkpoint(c, theirs, back)
        assert np.array_equal(back.download(), u[::-1]) and (t2, s2) == (1.5, 3)


@pytest.mark.parametrize("decomp,p,p1,p2", [("slab", 2, 1, 1), ("pencil", 4, 2, 2)])
def test_checkpoint_decomposition_independent(ref, tmp_path, decomp, p, p1, p2):
    """A file written by p ranks is read by any other decomposition (here the
    reference at p = 1 and our own ranks again) bit-exactly."""
    n = 16
    u = np.random.default_rng(6).uniform(-1, 1, (3, n, n, n))
    path = str(tmp_path / "multi.ck")
    cfg = S.SolverConfig(n=n, decomp=decomp, p=p, p1=p1, p2=p2)

    def write(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            S.write_checkpoint(c, path, c.real_field().upload(_scatter_real(u, c.layout)), 2.0, 9)

    S.run_group(p, write)
    v, t, step = ref.checkpoint_read(path, n)
    assert np.array_equal(v, u) and (t, step) == (2.0, 9)

    def read(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            f = c.real_field()
            meta = S.read_checkpoint(c, path, f)
            return c.layout, f.download(), meta

    for lo, blk, meta in S.run_group(p, read):
        assert np.array_equal(blk, _scatter_real(u, lo)) and meta == (2.0, 9)


def test_checkpoint_errors(tmp_path):
    """IoError on every failure the reference checks (checkpoint.cpp:139-160)."""
    n = 8
    with ctx_for(n) as c:
        f = c.real_field()
        with pytest.raises(S.IoError, match="cannot open"):
            S.read_checkpoint(c, str(tmp_path / "missing.ck"), f)
        bad = tmp_path / "bad.ck"
        bad.write_bytes(b"NOPE" + bytes(60))
        with pytest.raises(S.IoError, match="bad magic"):
            S.read_checkpoint(c, str(bad), f)
        good = str(tmp_path / "good.ck")
        S.write_checkpoint(c, good, c.real_field(), 0.0, 0)
        raw = open(good, "rb").read()
        open(str(tmp_path / "short.ck"), "wb").write(raw[:-8])
        with pytest.raises(S.IoError, match="truncated"):
            S.read_checkpoint(c, str(tmp_path / "short.ck"), f)
        with S.Context(S.SolverConfig(n=16)) as c16:
            with pytest.raises(S.IoError, match="does not match configured n=16"):
                S.read_checkpoint(c16, good, c16.real_field())
        (tmp_path / "dir.ck").mkdir()
        with pytest.raises(S.IoError, match="for writing"):
            S.write_checkpoint(c, str(tmp_path / "dir.ck"), f, 0.0, 0)
