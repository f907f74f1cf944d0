"""TEST INFRASTRUCTURE — ctypes binding of the compiled reference oracle.

``oracle/_ref/libsdns_ref.so`` is the UNMODIFIED reference library
(/root/reference/proj/core) built by ``oracle/Makefile`` against the
self-written FFTW subset in ``oracle/fftw_shim``, plus ``oracle/ref_driver.cpp``
(a small extern "C" driver over the reference's public API). Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arm use it.

All arrays are GLOBAL: spectral (3, n, n, n//2+1) complex128, real
(3, n, n, n) float64, exactly the reference's p = 1 block layout.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libsdns_ref.so")
_lib = None

DECOMP = {"slab": 0, "pencil": 1}


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB} missing: build with `make -C oracle`")
        # The oracle's g++ links libstdc++ statically; its formatted stream
        # output (the reference's CSV/manifest writers) needs the locale of
        # an initialised libstdc++, so load the system one globally first.
        ctypes.CDLL("libstdc++.so.6", mode=ctypes.RTLD_GLOBAL)
        L = ctypes.CDLL(LIB)
        I, D, P = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        L.sdns_ref_last_error.restype = ctypes.c_char_p
        L.sdns_ref_spectrum_shells.argtypes = [I]
        L.sdns_ref_forward.argtypes = [I, I, I, I, I, P, P]
        L.sdns_ref_inverse.argtypes = [I, I, I, I, I, P, P]
        L.sdns_ref_forward_scalar.argtypes = [I, I, I, I, I, I, P, P]
        L.sdns_ref_inverse_scalar.argtypes = [I, I, I, I, I, I, P, P]
        L.sdns_ref_iso_init.argtypes = [I, ctypes.c_ulonglong, D, D, P]
        L.sdns_ref_compute_rhs.argtypes = [I, I, I, I, I, D, I, P, P]
        L.sdns_ref_spectral_op.argtypes = [I, I, I, P, P]
        L.sdns_ref_cross.argtypes = [ctypes.c_int64, P, P, P]
        L.sdns_ref_collect_stats.argtypes = [I, I, I, I, I, D, P, P]
        L.sdns_ref_run.argtypes = [I, I, I, I, I, D, D, I, I, I, I, P, P,
                                   ctypes.POINTER(I), P]
        L.sdns_ref_rk4_steps.argtypes = [I, I, I, I, I, D, D, I, I, P]
        L.sdns_ref_bench.argtypes = [I, I, I, I, I, I, ctypes.POINTER(D)]
        L.sdns_ref_time_units.argtypes = [I, I, I, I, I, D, D, I, I, I, P, ctypes.POINTER(D)]
        L.sdns_ref_checkpoint_write.argtypes = [I, I, I, I, I, P, ctypes.c_char_p, D,
                                                ctypes.c_int64]
        L.sdns_ref_checkpoint_read.argtypes = [I, I, I, I, I, ctypes.c_char_p, P,
                                               ctypes.POINTER(D), ctypes.POINTER(ctypes.c_int64)]
        CP = ctypes.c_char_p
        I64 = ctypes.c_int64
        L.sdns_ref_parse_config.argtypes = [CP, P, P, I, P, P, P, I, P, I]
        L.sdns_ref_parse_bench_matrix.argtypes = [CP, P, I, ctypes.POINTER(I)]
        L.sdns_ref_write_diagnostics_csv.argtypes = [CP, P, P, I64, I]
        L.sdns_ref_write_bench_csv.argtypes = [CP, P, P, P, P, I]
        L.sdns_ref_write_manifest.argtypes = [CP, P, P, CP, CP, CP, I64, I64, CP, CP]
        L.sdns_ref_run_files.argtypes = [CP, CP, P, I]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"reference oracle error {rc}: "
                           f"{lib().sdns_ref_last_error().decode(errors='replace')}")


def _p(a):
    return ctypes.c_void_p(a.ctypes.data)


def shells(n):
    return lib().sdns_ref_spectrum_shells(n)


def forward(u, n, decomp="slab", p=1, p1=1, p2=1):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros((3, n, n, n // 2 + 1), dtype=np.complex128)
    _check(lib().sdns_ref_forward(n, DECOMP[decomp], p, p1, p2, _p(u), _p(out)))
    return out


def inverse(uh, n, decomp="slab", p=1, p1=1, p2=1):
    uh = np.ascontiguousarray(uh, dtype=np.complex128)
    out = np.zeros((3, n, n, n), dtype=np.float64)
    _check(lib().sdns_ref_inverse(n, DECOMP[decomp], p, p1, p2, _p(uh), _p(out)))
    return out


def iso_init(n, seed=1607, k0=4.0, energy=0.5):
    """The seeded isotropic field, GLOBAL (3, n, n, n//2+1), restated in the
    oracle (ref_driver.cpp sdns_ref_iso_init)."""
    out = np.empty((3, n, n, n // 2 + 1), dtype=np.complex128)
    _check(lib().sdns_ref_iso_init(n, seed, k0, energy, _p(out)))
    return out


def forward_scalar(u, n, decomp="slab", p=1, p1=1, p2=1):
    """Component-wise forward through the scalar DistributedFFT overload
    (fft.cpp:59-63); u is (ncomp, n, n, n)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    ncomp = u.shape[0]
    out = np.empty((ncomp, n, n, n // 2 + 1), dtype=np.complex128)
    _check(lib().sdns_ref_forward_scalar(n, DECOMP[decomp], p, p1, p2, ncomp, _p(u), _p(out)))
    return out


def inverse_scalar(uh, n, decomp="slab", p=1, p1=1, p2=1):
    """Component-wise normalised inverse through the scalar overload
    (fft.cpp:65-69); uh is (ncomp, n, n, n//2+1)."""
    uh = np.ascontiguousarray(uh, dtype=np.complex128)
    ncomp = uh.shape[0]
    out = np.empty((ncomp, n, n, n), dtype=np.float64)
    _check(lib().sdns_ref_inverse_scalar(n, DECOMP[decomp], p, p1, p2, ncomp, _p(uh), _p(out)))
    return out


def compute_rhs(uh, n, nu, dealias=True, decomp="slab", p=1, p1=1, p2=1):
    uh = np.ascontiguousarray(uh, dtype=np.complex128)
    out = np.zeros_like(uh)
    _check(lib().sdns_ref_compute_rhs(n, DECOMP[decomp], p, p1, p2, nu, int(dealias),
                                      _p(uh), _p(out)))
    return out


def spectral_op(op, uh, n, dealias=True):
    """op: 'curl' | 'project' | 'pressure' (component 0 of the result)."""
    uh = np.ascontiguousarray(uh, dtype=np.complex128)
    out = np.zeros_like(uh)
    _check(lib().sdns_ref_spectral_op(n, {"curl": 0, "project": 1, "pressure": 2}[op],
                                      int(dealias), _p(uh), _p(out)))
    return out


def cross(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    count = a[0].size
    out = np.zeros_like(a)
    _check(lib().sdns_ref_cross(count, _p(a), _p(b), _p(out)))
    return out


def collect_stats(uh, n, nu, decomp="slab", p=1, p1=1, p2=1):
    uh = np.ascontiguousarray(uh, dtype=np.complex128)
    row = np.zeros(5 + shells(n))
    _check(lib().sdns_ref_collect_stats(n, DECOMP[decomp], p, p1, p2, nu, _p(uh), _p(row)))
    return row


def run(uh0, n, nu, dt, steps, out_every=1, dealias=True, init_project=True,
        decomp="slab", p=1, p1=1, p2=1):
    """advance() with post_step = project and a stats sample every out_every
    steps (run_worker, proj/core/src/runner.cpp:67-111). Returns
    (stats rows [t,E,Z,eps,div,spectrum...], final u_hat)."""
    uh0 = np.ascontiguousarray(uh0, dtype=np.complex128)
    nrows = steps // out_every + 2
    stats = np.zeros((nrows, 5 + shells(n)))
    nsamp = ctypes.c_int(0)
    out = np.zeros_like(uh0)
    _check(lib().sdns_ref_run(n, DECOMP[decomp], p, p1, p2, nu, dt, steps, out_every,
                              int(dealias), int(init_project), _p(uh0), _p(stats),
                              ctypes.byref(nsamp), _p(out)))
    return stats[: nsamp.value], out


def rk4_steps(uh, n, nu, dt, steps, post_project=True, decomp="slab", p=1, p1=1, p2=1):
    uh = np.ascontiguousarray(uh, dtype=np.complex128).copy()
    _check(lib().sdns_ref_rk4_steps(n, DECOMP[decomp], p, p1, p2, nu, dt, steps,
                                    int(post_project), _p(uh)))
    return uh


def time_units(n, p=1, nu=5e-4, dt=5e-4, warmup=0, units=1, unit="step", uhat0=None,
               decomp="slab", p1=1, p2=1):
    """Mean seconds per unit ('step' = rk4_step + project, 'rhs' = one
    compute_rhs) of the reference on p threads-as-ranks (runner.cpp:336-373)."""
    s = ctypes.c_double()
    ptr = None if uhat0 is None else _p(np.ascontiguousarray(uhat0, dtype=np.complex128))
    _check(lib().sdns_ref_time_units(n, DECOMP[decomp], p, p1, p2, nu, dt, warmup, units,
                                     0 if unit == "step" else 1, ptr, ctypes.byref(s)))
    return s.value


def bench(n, p=1, steps=2, decomp="slab", p1=0, p2=0):
    """sdns::bench (proj/core/src/runner.cpp:336-397): seconds per step."""
    s = ctypes.c_double()
    _check(lib().sdns_ref_bench(n, DECOMP[decomp], p, p1, p2, steps, ctypes.byref(s)))
    return s.value


def checkpoint_write(path, u, n, t, step, decomp="slab", p=1, p1=1, p2=1):
    """write_checkpoint of the global real field u (3, n, n, n)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    _check(lib().sdns_ref_checkpoint_write(n, DECOMP[decomp], p, p1, p2, _p(u),
                                           os.fsencode(path), float(t), int(step)))


def checkpoint_read(path, n, decomp="slab", p=1, p1=1, p2=1):
    """read_checkpoint -> (u (3, n, n, n), t, step)."""
    u = np.zeros((3, n, n, n))
    t = ctypes.c_double()
    step = ctypes.c_int64()
    _check(lib().sdns_ref_checkpoint_read(n, DECOMP[decomp], p, p1, p2, os.fsencode(path), _p(u),
                                          ctypes.byref(t), ctypes.byref(step)))
    return u, t.value, step.value


# --- runner layer (config_file.hpp, runner.hpp) --------------------------------

class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _check_coded(rc):
    if rc != 0:
        raise RefError(rc, lib().sdns_ref_last_error().decode(errors="replace"))


def parse_config(text, overrides=()):
    """parse_config_text -> (dict of SolverConfig fields, notices list)."""
    items = list(overrides)
    keys = (ctypes.c_char_p * max(1, len(items)))(*[k.encode() for k, _ in items])
    vals = (ctypes.c_char_p * max(1, len(items)))(*[str(v).encode() for _, v in items])
    iv = np.zeros(7, dtype=np.int32)
    dv = np.zeros(3)
    case = ctypes.create_string_buffer(256)
    notes = ctypes.create_string_buffer(4096)
    _check_coded(lib().sdns_ref_parse_config(text.encode(), keys, vals, len(items), _p(iv),
                                             _p(dv), case, 256, notes, 4096))
    cfg = dict(n=int(iv[0]), decomp=["slab", "pencil"][iv[1]], p=int(iv[2]), p1=int(iv[3]),
               p2=int(iv[4]), dealias=bool(iv[5]), out_every=int(iv[6]), nu=float(dv[0]),
               dt=float(dv[1]), t_end=float(dv[2]), initial_case=case.value.decode())
    return cfg, [x for x in notes.value.decode().split("\n") if x]


def parse_bench_matrix(text):
    cnt = ctypes.c_int()
    out = np.zeros(5 * 256, dtype=np.int32)
    _check_coded(lib().sdns_ref_parse_bench_matrix(text.encode(), _p(out), 256,
                                                   ctypes.byref(cnt)))
    return [tuple(int(v) for v in out[5 * i:5 * i + 5]) for i in range(cnt.value)]


def write_diagnostics_csv(path, steps, rows, shells):
    steps = np.ascontiguousarray(steps, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    _check_coded(lib().sdns_ref_write_diagnostics_csv(os.fsencode(path), _p(steps), _p(rows),
                                                      len(steps), shells))


def write_bench_csv(path, entries, nodes, secs, statuses):
    ent = np.ascontiguousarray(np.array(entries, dtype=np.int32).reshape(-1))
    nodes = np.ascontiguousarray(nodes, dtype=np.int64)
    secs = np.ascontiguousarray(secs, dtype=np.float64)
    st = (ctypes.c_char_p * max(1, len(statuses)))(*[x.encode() for x in statuses])
    _check_coded(lib().sdns_ref_write_bench_csv(os.fsencode(path), _p(ent), _p(nodes), _p(secs),
                                                st, len(statuses)))


def write_manifest(path, ints, doubles, icase, backend, status, steps, timed_steps, csv, ckpt):
    iv = np.ascontiguousarray(ints, dtype=np.int32)
    dv = np.ascontiguousarray(doubles, dtype=np.float64)
    _check_coded(lib().sdns_ref_write_manifest(os.fsencode(path), _p(iv), _p(dv), icase.encode(),
                                               backend.encode(), status.encode(), steps,
                                               timed_steps, csv.encode(), ckpt.encode()))


def run_files(config_text, out_dir):
    """The reference's run() (runner.cpp:197-213) into out_dir; returns status."""
    st = ctypes.create_string_buffer(256)
    _check_coded(lib().sdns_ref_run_files(config_text.encode(), os.fsencode(out_dir), st, 256))
    return st.value.decode()
