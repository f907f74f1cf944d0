"""TEST INFRASTRUCTURE — numpy restatement of the reference's hot path.

This module is the CPU oracle used only by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` leg. It is never imported by the product
package. It restates, function by function, the reference C++ solver
(``/root/reference/proj/core``) on GLOBAL arrays (the p = 1 view):

* spectral fields: ``(3, n, n, n//2+1)`` complex128, axis order (kx, ky, kz)
  with kz fastest — the reference's slab spectral layout at p = 1
  (proj/core/src/layout.cpp:30-44);
* real fields: ``(3, n, n, n)`` float64 (x, y, z), z fastest.

numpy's pocketfft stands in for FFTW (unnormalised forward, inverse scaled
once by 1/n^3 exactly like DistributedFFT, proj/core/src/fft.cpp:26-27,125).
Parity of this restatement is pinned by tests/test_oracle.py against the
compiled reference (oracle/_ref/libsdns_ref.so) and the golden fixtures in
tests/golden/.
"""
from __future__ import annotations

import math

import numpy as np

EPS = np.finfo(np.float64).eps


# --- layout (proj/core/src/layout.cpp) -------------------------------------

def block_size(total: int, parts: int, index: int) -> int:
    """proj/core/src/layout.cpp:7-10 — first (total mod parts) blocks get the ceiling."""
    base = total // parts
    return base + (1 if index < total % parts else 0)


def block_start(total: int, parts: int, index: int) -> int:
    """proj/core/src/layout.cpp:12-15."""
    base = total // parts
    return index * base + min(index, total % parts)


def validate(n, decomp="slab", p=1, p1=1, p2=1, nu=0.0, dt=1.0, t_end=0.0, out_every=1):
    """SolverConfig::validate, proj/core/src/config.cpp:17-50. Raises ValueError."""
    if n < 4:
        raise ValueError(f"n must be >= 4, got {n}")
    if n % 2:
        raise ValueError(f"n must be even, got {n}")
    if p < 1:
        raise ValueError(f"p must be >= 1, got {p}")
    if decomp == "slab":
        if p > n:
            raise ValueError(f"slab requires p <= n, got p={p} n={n}")
        if n % p:
            raise ValueError(f"slab requires p to divide n, got p={p} n={n}")
    else:
        if p1 < 1 or p2 < 1:
            raise ValueError("pencil requires p1 >= 1 and p2 >= 1")
        if p != p1 * p2:
            raise ValueError(f"pencil requires p = p1*p2, got p={p} p1={p1} p2={p2}")
        if n % p1:
            raise ValueError(f"pencil requires p1 to divide n, got p1={p1} n={n}")
        if n % p2:
            raise ValueError(f"pencil requires p2 to divide n, got p2={p2} n={n}")
        if p2 > n // 2:
            raise ValueError(f"pencil requires p2 <= n/2, got p2={p2} n={n}")
    if nu < 0:
        raise ValueError("nu must be >= 0")
    if not dt > 0:
        raise ValueError("dt must be > 0")
    if t_end < 0:
        raise ValueError("t_end must be >= 0")
    if out_every < 1:
        raise ValueError("out_every must be >= 1")


def build_layout(n, decomp, p, p1, p2, rank):
    """build_layout, proj/core/src/layout.cpp:17-76, as a dict."""
    validate(n, decomp, p, p1, p2)
    nf = n // 2 + 1
    lo = {"rank": rank, "p": p, "n": n, "nf": nf}
    if decomp == "slab":
        np_ = n // p
        lo.update(p1=p, p2=1, coord1=rank, coord2=0,
                  real_shape=(np_, n, n), real_offset=(rank * np_, 0, 0),
                  spec_shape=(n, np_, nf), spec_offset=(0, rank * np_, 0),
                  stages=[([np_ * np_ * nf] * p, [np_ * np_ * nf] * p)])
    else:
        c1, c2 = rank // p2, rank % p2
        xl, yl, yl2 = n // p1, n // p2, n // p1
        b = block_size(nf, p2, c2)
        s0 = ([xl * yl * block_size(nf, p2, q) for q in range(p2)], [xl * yl * b] * p2)
        s1 = ([xl * yl2 * b] * p1, [xl * yl2 * b] * p1)
        lo.update(p1=p1, p2=p2, coord1=c1, coord2=c2,
                  real_shape=(xl, yl, n), real_offset=(c1 * xl, c2 * yl, 0),
                  spec_shape=(n, yl2, b), spec_offset=(0, c1 * yl2, block_start(nf, p2, c2)),
                  stages=[s0, s1])
    return lo


# --- mesh (proj/core/src/mesh.cpp) -----------------------------------------

def axis_wavenumber(j, n):
    """proj/core/include/sdns/mesh.hpp:19-21."""
    j = np.asarray(j)
    return np.where(j <= n // 2 - 1, j, j - n)


class Wavenumbers:
    """WavenumberMesh for the global spectral block (mesh.cpp:23-89)."""

    def __init__(self, n: int, dealias: bool = True):
        self.n = n
        nf = n // 2 + 1
        self.kx = axis_wavenumber(np.arange(n), n).astype(np.float64)
        self.ky = self.kx.copy()
        self.kz = np.arange(nf, dtype=np.float64)
        KX = self.kx[:, None, None]
        KY = self.ky[None, :, None]
        KZ = self.kz[None, None, :]
        # k2 = kx*kx + ky*ky + kz*kz in that order (mesh.cpp:57)
        self.k2 = (KX * KX + KY * KY) + KZ * KZ
        inv = np.where(self.k2 > 0, 1.0 / np.where(self.k2 > 0, self.k2, 1.0), 0.0)
        self.kx_over_k2 = KX * inv
        self.ky_over_k2 = KY * inv
        self.kz_over_k2 = KZ * inv
        if dealias:
            kmax = n / 3.0
            self.mask = ((np.abs(KX) < kmax) & (np.abs(KY) < kmax) & (np.abs(KZ) < kmax))
        else:
            self.mask = np.ones(self.k2.shape, dtype=bool)
        self.KX, self.KY, self.KZ = KX, KY, KZ


def physical_axis(n):
    """physical_mesh, proj/core/src/mesh.cpp:8-21: x_i = (2 pi / n) * i."""
    h = 2.0 * math.pi / n
    return h * np.arange(n, dtype=np.float64)


# --- transforms (proj/core/src/fft.cpp) -------------------------------------

def forward(u):
    """DistributedFFT::forward (unnormalised r2c over x, y, z)."""
    return np.fft.rfftn(u, axes=(-3, -2, -1))


def inverse(uh, n):
    """DistributedFFT::inverse, normalised once by 1/n^3 (fft.cpp:125)."""
    return np.fft.irfftn(uh, s=(n, n, n), axes=(-3, -2, -1))


# --- navier-stokes (proj/core/src/navier_stokes.cpp) -------------------------

def taylor_green_baseline(n):
    """BASELINE.json config 1 / PAPER.md:243-247 variant:
    u = sin x cos y cos z, v = -cos x sin y cos z, w = 0 (the reference code
    uses the pi/2-shifted variant, navier_stokes.cpp:18-20)."""
    x = physical_axis(n)
    sx, cx = np.sin(x), np.cos(x)
    u = np.zeros((3, n, n, n))
    u[0] = sx[:, None, None] * cx[None, :, None] * cx[None, None, :]
    u[1] = -(cx[:, None, None] * sx[None, :, None] * cx[None, None, :])
    return u


def taylor_green_reference(n):
    """taylor_green_init, proj/core/src/navier_stokes.cpp:7-25."""
    x = physical_axis(n)
    s, c = np.sin(x), np.cos(x)
    u = np.zeros((3, n, n, n))
    u[0] = (c[:, None, None] * s[None, :, None]) * s[None, None, :]
    u[1] = (-s[:, None, None] * c[None, :, None]) * s[None, None, :]
    return u


def cross(a, b):
    """proj/core/src/navier_stokes.cpp:34-50 (same operation order)."""
    o = np.empty_like(a)
    o[0] = a[1] * b[2] - a[2] * b[1]
    o[1] = a[2] * b[0] - a[0] * b[2]
    o[2] = a[0] * b[1] - a[1] * b[0]
    return o


def _imul(z):
    """Complex(0,1) * z  ->  (-Im z, Re z)."""
    return -z.imag + 1j * z.real


def curl_hat(uh, wm):
    """omega_hat = i k x u_hat, proj/core/src/navier_stokes.cpp:52-72."""
    o = np.empty_like(uh)
    o[0] = _imul(wm.KY * uh[2] - wm.KZ * uh[1])
    o[1] = _imul(wm.KZ * uh[0] - wm.KX * uh[2])
    o[2] = _imul(wm.KX * uh[1] - wm.KY * uh[0])
    return o


def pressure_hat(nl, wm):
    """proj/core/src/navier_stokes.cpp:74-83: -i (k/k^2 . nl_hat)."""
    kd = (wm.kx_over_k2 * nl[0] + wm.ky_over_k2 * nl[1]) + wm.kz_over_k2 * nl[2]
    return kd.imag - 1j * kd.real


def project(uh, wm):
    """u_hat -= (k/k^2) (k . u_hat), proj/core/src/navier_stokes.cpp:85-102."""
    kd = (wm.KX * uh[0] + wm.KY * uh[1]) + wm.KZ * uh[2]
    out = np.empty_like(uh)
    out[0] = uh[0] - wm.kx_over_k2 * kd
    out[1] = uh[1] - wm.ky_over_k2 * kd
    out[2] = uh[2] - wm.kz_over_k2 * kd
    return out


def compute_rhs(uh, wm, nu):
    """proj/core/src/navier_stokes.cpp:104-139 (rotational form)."""
    n = wm.n
    vel = inverse(uh, n)
    vor = inverse(curl_hat(uh, wm), n)
    c = forward(cross(vel, vor))
    c = np.where(wm.mask[None], c, 0.0)
    kd = (wm.KX * c[0] + wm.KY * c[1]) + wm.KZ * c[2]
    c[0] = c[0] - wm.kx_over_k2 * kd
    c[1] = c[1] - wm.ky_over_k2 * kd
    c[2] = c[2] - wm.kz_over_k2 * kd
    visc = nu * wm.k2
    return c - visc[None] * uh


# --- RK4 (proj/core/src/rk4.cpp) -------------------------------------------

def _two_sum_err(a, b, s):
    """Neumaier branch of TwoSum, proj/core/src/rk4.cpp:21-23."""
    return np.where(np.abs(a) >= np.abs(b), (a - s) + b, (b - s) + a)


class Rk4State:
    """proj/core/include/sdns/rk4.hpp:18-30."""

    def __init__(self, uh):
        self.u_hat = uh.copy()
        self.carry = np.zeros_like(uh)
        self.t = 0.0
        self.step = 0


def rk4_step_finite(st, dt, rhs):
    """proj/core/src/rk4.cpp:27-71: low-storage classical RK4 + Neumaier carry."""
    W = (1.0, 2.0, 2.0)
    B = (0.5, 0.5, 1.0)
    u0 = st.u_hat.copy()
    acc = np.zeros_like(u0)
    for stage in range(4):
        du = rhs(st.u_hat)
        if stage < 3:
            acc = acc + W[stage] * du
            st.u_hat = u0 + (B[stage] * dt) * du
        else:
            sixth = dt / 6.0
            delta = sixth * (acc + du) + st.carry
            unew = u0 + delta
            st.carry = (_two_sum_err(u0.real, delta.real, unew.real)
                        + 1j * _two_sum_err(u0.imag, delta.imag, unew.imag))
            st.u_hat = unew
    st.t += dt
    st.step += 1
    return bool(np.all(np.isfinite(st.u_hat)))


def step_count(t_end, dt):
    """proj/core/src/rk4.cpp:79-84."""
    if t_end <= 0:
        return 0
    return max(0, int(math.ceil(t_end / dt - 1e-9)))


def advance(st, wm, nu, dt, t_end, out_every=1, sample=None, post_project=True):
    """advance, proj/core/src/rk4.cpp:86-107 with the runner's hooks
    (post_step = project, proj/core/src/runner.cpp:107)."""
    n_steps = step_count(t_end, dt)
    rhs = lambda u: compute_rhs(u, wm, nu)  # noqa: E731
    if sample:
        sample(0, st.t)
    for k in range(1, n_steps + 1):
        last = k == n_steps
        target = t_end if last else float(k) * dt
        dtk = target - st.t
        finite = rk4_step_finite(st, dtk, rhs)
        if post_project:
            st.u_hat = project(st.u_hat, wm)
        st.t = target
        if not finite:
            raise FloatingPointError(f"non-finite values in solution update at step {k}")
        if sample and (k % out_every == 0 or last):
            sample(k, st.t)


# --- diagnostics (proj/core/src/diagnostics.cpp) ----------------------------

def spectrum_shells(n):
    """proj/core/src/diagnostics.cpp:66-69 (llround = half away from zero)."""
    half = float(n // 2)
    return int(math.floor(math.sqrt(3.0 * half * half) + 0.5)) + 1


def collect_stats(uh, wm, nu, t=0.0):
    """collect_stats, proj/core/src/diagnostics.cpp:24-91 (sums in numpy order)."""
    n = wm.n
    w = np.where((wm.KZ == 0.0) | (wm.KZ == float(n // 2)), 1.0, 2.0)
    e = (np.abs(uh[0]) ** 2 + np.abs(uh[1]) ** 2) + np.abs(uh[2]) ** 2
    c0 = wm.KY * uh[2] - wm.KZ * uh[1]
    c1 = wm.KZ * uh[0] - wm.KX * uh[2]
    c2 = wm.KX * uh[1] - wm.KY * uh[0]
    z = (np.abs(c0) ** 2 + np.abs(c1) ** 2) + np.abs(c2) ** 2
    we = np.broadcast_to(w, e.shape) * e
    wz = np.broadcast_to(w, z.shape) * z
    shells = spectrum_shells(n)
    knorm = np.sqrt(wm.k2)
    shell = np.floor(knorm + 0.5).astype(np.int64)
    spec = np.bincount(shell.ravel(), weights=(0.5 * we).ravel(), minlength=shells)[:shells]
    kd = (wm.KX * uh[0] + wm.KY * uh[1]) + wm.KZ * uh[2]
    ratio = np.abs(kd) / (knorm * np.sqrt(e) + EPS)
    n3 = float(n) ** 3
    n6 = n3 * n3
    E = 0.5 * we.sum() / n6
    Z = 0.5 * wz.sum() / n6
    return {"t": t, "energy": E, "enstrophy": Z, "dissipation": 2.0 * nu * Z,
            "divergence_max": float(ratio.max()), "spectrum": spec / n6}


def l2_diff(a, b, n):
    """proj/core/src/diagnostics.cpp:113-127."""
    d = (a - b).ravel()
    return math.sqrt(float(np.dot(d, d)) / float(n) ** 3)
