"""Generates the golden fixtures in tests/golden/ from the compiled reference.

Run in the build container (needs oracle/_ref, i.e. /root/reference):
    python tests/golden/make_golden.py
Every array is produced by the UNMODIFIED reference library through
oracle/ref.py; inputs are seeded synthetic fields (no external data).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402
from oracle import sdns_np as O  # noqa: E402


def random_field(n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(3, n, n, n))


def random_spec(n, seed):
    rng = np.random.default_rng(seed)
    s = (3, n, n, n // 2 + 1)
    return rng.uniform(-1, 1, s) + 1j * rng.uniform(-1, 1, s)


def main():
    out = {}
    # 1. distributed FFT at n = 8 under every decomposition the reference tests
    #    use (proj/tests/test_fft.cpp:73-110); forward of 3 random components.
    n = 8
    u = random_field(n, 50)
    out["fft8_u"] = u
    out["fft8_slab1"] = R.forward(u, n, "slab", 1)
    out["fft8_slab2"] = R.forward(u, n, "slab", 2)
    out["fft8_slab4"] = R.forward(u, n, "slab", 4)
    out["fft8_pencil22"] = R.forward(u, n, "pencil", 4, 2, 2)
    out["fft8_pencil24"] = R.forward(u, n, "pencil", 8, 2, 4)
    out["fft8_inverse"] = R.inverse(out["fft8_slab1"], n)
    # 2. pointwise operators at n = 8
    uh = random_spec(n, 51)
    out["pw8_uh"] = uh
    out["pw8_curl"] = R.spectral_op("curl", uh, n)
    out["pw8_project"] = R.spectral_op("project", uh, n)
    out["pw8_pressure"] = R.spectral_op("pressure", uh, n)[0]
    a, b = random_field(n, 52), random_field(n, 53)
    out["pw8_a"], out["pw8_b"] = a, b
    out["pw8_cross"] = R.cross(a, b)
    # 3. Taylor-Green (BASELINE config-1 formula) at n = 16: init + 10 steps
    n = 16
    u0 = O.taylor_green_baseline(n)
    uh0 = R.forward(u0, n)
    stats, uhf = R.run(uh0, n, nu=0.01, dt=0.01, steps=10, out_every=1)
    out["tg16_uh0"] = uh0
    out["tg16_stats"] = stats
    out["tg16_final"] = uhf
    out["tg16_rhs"] = R.compute_rhs(O.project(uh0, O.Wavenumbers(n)), n, 0.01)
    # 4. random solenoidal-ish spectrum at n = 16: compute_rhs + 3 RK4 steps
    uh = random_spec(n, 54) * 1e-3
    out["rnd16_uh"] = uh
    out["rnd16_rhs"] = R.compute_rhs(uh, n, 1e-3)
    out["rnd16_rk3"] = R.rk4_steps(uh, n, 1e-3, 1e-3, 3, post_project=True)
    out["rnd16_stats"] = R.collect_stats(uh, n, 1e-3)
    np.savez_compressed(os.path.join(HERE, "golden_ref.npz"), **out)
    print("wrote", os.path.join(HERE, "golden_ref.npz"), {k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
