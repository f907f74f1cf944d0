"""GPU: even n that is not a power of two (the reference accepts any even
n >= 4, proj/core/src/config.cpp:17-19; its suites use lengths 3, 5 and 6,
proj/tests/test_serial_fft.cpp:71-166). These lengths run the generic
mixed-radix kernels (csrc/kernels_gen.cu) behind the same launchers,
geometries and transposes as the tuned lengths. Same bars as the tuned path:
FFT <= 1e-11 max|X| and round trip <= 1e-13 (proj/tests/test_fft.cpp:73-110),
RHS <= 1e-12 relative, 10 RK4 steps <= 1e-11 relative L2 with E and Z
<= 1e-12 per step, against the compiled reference."""
import os

import numpy as np
import pytest

import paper_1607_00850_b200 as S
from oracle import sdns_np as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(np.asarray(b).ravel()), 1e-300)


def _blk(g, shape, off):
    (s0, s1, s2), (o0, o1, o2) = shape, off
    return g[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2]


GEOMS = [dict(), dict(p=2), dict(p=3), dict(decomp="pencil", p=6, p1=2, p2=3),
         dict(decomp="pencil", p=4, p1=2, p2=2)]


def _valid(n, geom):
    p = geom.get("p", 1)
    if geom.get("decomp") == "pencil":
        return n % geom["p1"] == 0 and n % geom["p2"] == 0 and geom["p2"] <= n // 2
    return n % p == 0


@pytest.mark.parametrize("n", [6, 10, 12, 14, 18, 20, 24, 30, 36, 48, 96, 100])
def test_fft_generic_length_vs_numpy(n):
    u = np.random.default_rng(7 + n).uniform(-1, 1, (3, n, n, n))
    with S.Context(S.SolverConfig(n=n)) as c:
        fft = S.DistributedFFT(c)
        ud, fd = c.real_field().upload(u), c.spectral_field()
        fft.forward(ud, fd)
        fu = fd.download()
        ref = O.forward(u)
        assert np.abs(fu - ref).max() <= 1e-11 * np.abs(ref).max()
        back = c.real_field()
        fft.inverse(fd, back)
        assert rel(back.download(), u) <= 1e-13


@pytest.mark.parametrize("n", [12, 18, 24])
@pytest.mark.parametrize("gi", range(len(GEOMS)))
@pytest.mark.parametrize("a2a", [0, 1])
def test_fft_generic_length_decompositions(n, gi, a2a):
    """Slab and pencil with blocks that are not powers of two (n/p = 9, 6, 4;
    pencil kz blocks 4/3/3 of n/2+1 = 10), peer-direct and all-to-all."""
    geom = GEOMS[gi]
    if not _valid(n, geom):
        pytest.skip("p does not divide n")
    u = np.random.default_rng(n).uniform(-1, 1, (3, n, n, n))
    expect = O.forward(u)
    cfg = S.SolverConfig(n=n, **geom)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm, options={"all_to_all": a2a}) as c:
            lo = c.layout
            fd = c.spectral_field()
            fft = S.DistributedFFT(c)
            fft.forward(c.real_field().upload(_blk(u, lo.real_shape, lo.real_offset)), fd)
            back = c.real_field()
            fft.inverse(fd, back)
            return lo, fd.download(), back.download()

    for lo, fu, back in S.run_group(cfg.p, body):
        assert np.abs(fu - _blk(expect, lo.spec_shape, lo.spec_offset)).max() <= \
            1e-11 * np.abs(expect).max()
        assert rel(back, _blk(u, lo.real_shape, lo.real_offset)) <= 1e-13


@pytest.mark.parametrize("n,geom", [(12, dict()), (18, dict()), (24, dict(p=3)),
                                    (20, dict(decomp="pencil", p=4, p1=2, p2=2)),
                                    (30, dict(p=2))])
def test_compute_rhs_generic_length_vs_reference(ref, n, geom):
    uh = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=11)
    expect = ref.compute_rhs(uh, n, 1e-3, decomp=geom.get("decomp", "slab"), p=geom.get("p", 1),
                             p1=geom.get("p1", 1), p2=geom.get("p2", 1))
    cfg = S.SolverConfig(n=n, **geom)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            lo = c.layout
            du = c.spectral_field()
            S.compute_rhs(c, c.spectral_field().upload(_blk(uh, lo.spec_shape, lo.spec_offset)),
                          1e-3, du)
            return lo, du.download()

    for lo, du in S.run_group(cfg.p, body):
        e = _blk(expect, lo.spec_shape, lo.spec_offset)
        assert np.linalg.norm(du - e) <= 1e-12 * np.linalg.norm(expect)


@pytest.mark.parametrize("n,geom", [(12, dict()), (24, dict()), (48, dict()), (36, dict(p=3)),
                                    (24, dict(decomp="pencil", p=6, p1=2, p2=3))])
def test_ten_rk4_steps_generic_length_vs_reference(ref, n, geom):
    nu, dt, steps = 1e-3, 1e-3, 10
    uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=1607)
    gs, gf = ref.run(uh0, n, nu, dt, steps, out_every=1, init_project=False)
    cfg = S.SolverConfig(n=n, nu=nu, dt=dt, t_end=steps * dt, out_every=1, **geom)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            lo = c.layout
            st = S.Rk4State(c)
            st.set(c.spectral_field().upload(_blk(uh0, lo.spec_shape, lo.spec_offset)))
            rows = []
            st.advance(lambda k, t: rows.append(S.collect_stats(c, st.u_hat, nu, t)))
            out = (lo, st.u_hat.download(), rows)
            st.close()
            return out

    res = S.run_group(cfg.p, body)
    final = np.empty_like(gf)
    for lo, blk, _ in res:
        (s0, s1, s2), (o0, o1, o2) = lo.spec_shape, lo.spec_offset
        final[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2] = blk
    rows = res[0][2]
    assert len(rows) == gs.shape[0] == steps + 1
    for r, g in zip(rows, gs):
        assert abs(r.energy - g[1]) <= 1e-12 * g[1]
        assert abs(r.enstrophy - g[2]) <= 1e-12 * g[2]
    assert rel(final, gf) <= 1e-11


def test_taylor_green_generic_length_energy_balance():
    """n = 48 Taylor-Green: E0 = 0.125 (test_diagnostics.cpp:52-66 for the
    BASELINE variant), dissipative and divergence-free over 5 steps."""
    n, nu, dt = 48, 0.01, 0.01
    cfg = S.SolverConfig(n=n, nu=nu, dt=dt, t_end=5 * dt, out_every=1)
    with S.Context(cfg) as c:
        uh = c.spectral_field()
        S.DistributedFFT(c).forward(c.real_field().upload(O.taylor_green_baseline(n)), uh)
        S.project(c, uh)
        st = S.Rk4State(c)
        st.set(uh)
        rows = []
        st.advance(lambda k, t: rows.append(S.collect_stats(c, st.u_hat, nu, t)))
        st.close()
    assert abs(rows[0].energy - 0.125) <= 1e-14
    assert all(b.energy < a.energy for a, b in zip(rows, rows[1:]))
    assert max(r.divergence_max for r in rows) <= 1e-10
