"""CPU: the C-ABI library loads, exports every declared entry point, and its
host-only setup logic (no device needed) matches the reference's rules and
the oracle restatement.
"""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_1607_00850_b200 as S
from oracle import sdns_np as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sdns_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sdns_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = S.load_library()
    syms = header_symbols()
    assert len(syms) >= 50
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.sdns_version().startswith(b"sdns-b200")


def test_library_is_sm100a_only():
    """The product .so carries sm_100a SASS (cross-compiled here)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", S.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out


@pytest.mark.parametrize("kw,ok", [
    (dict(n=8), True), (dict(n=7), False), (dict(n=2), False), (dict(n=8, p=0), False),
    (dict(n=8, p=3), False), (dict(n=8, p=16), False), (dict(n=8, p=8), True),
    (dict(n=8, decomp="pencil", p=4, p1=2, p2=2), True),
    (dict(n=8, decomp="pencil", p=8, p1=2, p2=4), True),
    (dict(n=8, decomp="pencil", p=8, p1=1, p2=8), False),   # p2 > n/2
    (dict(n=8, decomp="pencil", p=6, p1=2, p2=3), False),   # p2 does not divide n
    (dict(n=8, decomp="pencil", p=4, p1=2, p2=3), False),   # p != p1 p2
    (dict(n=8, nu=-1.0), False), (dict(n=8, dt=0.0), False), (dict(n=8, t_end=-1.0), False),
    (dict(n=8, out_every=0), False),
])
def test_validate_rules(kw, ok):
    """SolverConfig::validate, proj/core/src/config.cpp:17-50 (and test_grid.cpp)."""
    cfg = S.SolverConfig(**kw)
    args = dict(n=cfg.n, decomp=cfg.decomp, p=cfg.p, p1=cfg.p1, p2=cfg.p2, nu=cfg.nu,
                dt=cfg.dt, t_end=cfg.t_end, out_every=cfg.out_every)
    if ok:
        S.validate(cfg)
        O.validate(**args)
    else:
        with pytest.raises(S.ConfigError):
            S.validate(cfg)
        with pytest.raises(ValueError):
            O.validate(**args)


CASES = [(8, "slab", 1, 1, 1), (8, "slab", 4, 4, 1), (16, "slab", 8, 8, 1),
         (8, "pencil", 4, 2, 2), (8, "pencil", 8, 2, 4), (16, "pencil", 8, 4, 2),
         (64, "pencil", 8, 2, 4), (1024, "pencil", 8, 2, 4), (1024, "slab", 8, 8, 1)]


@pytest.mark.parametrize("n,decomp,p,p1,p2", CASES)
def test_build_layout_matches_reference_rule(n, decomp, p, p1, p2):
    for rank in range(p):
        cfg = S.SolverConfig(n=n, decomp=decomp, p=p, p1=p1, p2=p2)
        lo = S.build_layout(cfg, rank)
        ref = O.build_layout(n, decomp, p, p1, p2, rank)
        assert lo.real_shape == ref["real_shape"] and lo.real_offset == ref["real_offset"]
        assert lo.spec_shape == ref["spec_shape"] and lo.spec_offset == ref["spec_offset"]
        assert (lo.coord1, lo.coord2) == (ref["coord1"], ref["coord2"])
        assert [list(map(list, s)) for s in lo.stages] == [list(map(list, s)) for s in ref["stages"]]


def test_layout_pins_from_reference_tests():
    """proj/tests/test_grid.cpp: slab n=8 p=4 r=2; pencil n=8 2x2 rank 3; 1024 2x4 kz blocks."""
    lo = S.build_layout(S.SolverConfig(n=8, p=4), 2)
    assert lo.real_shape == (2, 8, 8) and lo.spec_shape == (8, 2, 5)
    lo = S.build_layout(S.SolverConfig(n=8, decomp="pencil", p=4, p1=2, p2=2), 3)
    assert lo.stages[0][0] == [48, 32] and lo.stages[0][1] == [32, 32]
    assert [S.block_size(513, 4, q) for q in range(4)] == [129, 128, 128, 128]
    assert [S.block_start(513, 4, q) for q in range(4)] == [0, 129, 257, 385]


def test_step_count_and_shells():
    assert S.step_count(0.1, 1e-3) == 100 == O.step_count(0.1, 1e-3)
    assert S.step_count(0.1, 0.03) == 4
    assert S.step_count(0.0, 0.1) == 0
    assert S.step_count(1.0, 0.01) == 100  # 100 steps of config 1
    assert [S.spectrum_shells(n) for n in (8, 16, 32, 64, 256, 512, 1024)] == \
        [O.spectrum_shells(n) for n in (8, 16, 32, 64, 256, 512, 1024)] == [8, 15, 29, 56, 223, 444, 888]


def test_device_layout_pads_rows_and_kz():
    d = S.device_layout(S.SolverConfig(n=512), 0)
    assert d["pitch"] == 264 and d["prow"] == 513 and d["np"] == 512
    # the x-plane stride is an odd multiple of 128 B
    assert (d["prow"] * d["pitch"] * 16) % 128 == 0 and ((d["prow"] * d["pitch"] * 16) // 128) % 2 == 1
    d = S.device_layout(S.SolverConfig(n=16, p=2), 1)
    assert d == {"pitch": 16, "prow": 9, "np": 8, "spec_cs": 16 * 9 * 16, "real_cs": 8 * 16 * 16}


def test_exchange_plan_is_peer_blocks():
    cfg = S.SolverConfig(n=32, p=4)
    for rank in range(4):
        d = S.device_layout(cfg, rank)
        for inv in (True, False):
            plan = S.exchange_plan(cfg, rank, inv, 3)
            assert plan.shape == (12, 4)
            blk = d["np"] * d["prow"] * d["pitch"]
            for i, (peer, so, do, cnt) in enumerate(plan):
                f, q = divmod(i, 4)
                assert peer == q and cnt == blk and so == do == f * d["spec_cs"] + q * blk


# --- isotropic initial field (BASELINE configs 2-4) ---------------------------

def _global_iso(n, seed=1607):
    lo = S.build_layout(S.SolverConfig(n=n), 0)
    return S.iso_init(n, lo, seed=seed)


def test_iso_field_properties():
    n = 32
    uh = _global_iso(n)
    wm = O.Wavenumbers(n)
    s = O.collect_stats(uh, wm, 1e-3)
    assert abs(s["energy"] - 0.5) <= 1e-13
    kd = (wm.KX * uh[0] + wm.KY * uh[1]) + wm.KZ * uh[2]
    assert np.abs(kd).max() <= 1e-15 * np.abs(uh).max() * n
    assert np.all(uh[:, 0, 0, 0] == 0)
    assert np.all(uh[:, n // 2] == 0) and np.all(uh[:, :, n // 2] == 0) and np.all(uh[:, :, :, n // 2] == 0)
    # Hermitian symmetry on kz = 0: u(-kx,-ky,0) = conj u(kx,ky,0)
    p0 = uh[:, :, :, 0]
    mirror = np.conj(p0[:, (-np.arange(n)) % n][:, :, (-np.arange(n)) % n])
    assert np.array_equal(p0, mirror)
    # spectrum peaks near k0 = 4 (E(k) ~ k^4 exp(-2 (k/4)^2) peaks at k = 4)
    assert 3 <= int(np.argmax(s["spectrum"])) <= 5
    # it is a real field: irfftn(uh) round trips
    u = O.inverse(uh, n)
    assert np.abs(O.forward(u) - uh).max() <= 1e-13 * np.abs(uh).max() * n**3


@pytest.mark.parametrize("decomp,p,p1,p2", [("slab", 2, 2, 1), ("slab", 4, 4, 1),
                                             ("pencil", 4, 2, 2), ("pencil", 8, 2, 4)])
def test_iso_field_is_decomposition_independent(decomp, p, p1, p2):
    n = 16
    g = _global_iso(n)
    for r in range(p):
        lo = S.build_layout(S.SolverConfig(n=n, decomp=decomp, p=p, p1=p1, p2=p2), r)
        (s0, s1, s2), (o0, o1, o2) = lo.spec_shape, lo.spec_offset
        assert np.array_equal(S.iso_init(n, lo), g[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2])


@pytest.mark.parametrize("n,seed", [(8, 1607), (16, 3), (64, 1607)])
def test_iso_field_matches_oracle_restatement(ref, n, seed):
    """The product's iso_init (csrc/iso_init.cpp) and the oracle's independent
    restatement of SURVEY §8(d)'s recipe (oracle/ref_driver.cpp) agree bit
    for bit; the reference arm of bench.py builds its input from the latter."""
    assert np.array_equal(_global_iso(n, seed), ref.iso_init(n, seed=seed))


def test_iso_field_is_seeded():
    a, b = _global_iso(16, 1), _global_iso(16, 2)
    assert not np.array_equal(a, b) and np.array_equal(a, _global_iso(16, 1))


def test_errors_map_to_reference_exception_types():
    with pytest.raises(S.ConfigError):
        S.build_layout(S.SolverConfig(n=8, p=2), 5)
    with pytest.raises(S.ConfigError):
        S.SolverConfig(n=8, decomp="cube").to_c()
    lib = S.load_library()
    rc = lib.sdns_build_layout(ctypes.byref(S.SolverConfig(n=9).to_c()), 0,
                               ctypes.byref(S._Layout()))
    assert rc == 1 and b"even" in lib.sdns_last_error()


def test_context_options_are_explicit():
    """Execution choices are API options (sdns_ctx_options), not environment
    variables: unknown names are rejected, and the library reads no
    environment (no getenv in the product sources)."""
    with pytest.raises(S.ConfigError):
        with S.context_options(bogus=1):
            pass
    with S.context_options(all_to_all=1):
        assert S._ctx_options(None).all_to_all == 1
        assert S._ctx_options({"serial": 1}).serial == 1
    assert S._ctx_options(None).all_to_all == 0
    csrc = os.path.join(os.path.dirname(S.__file__), "csrc")
    for f in os.listdir(csrc):
        if f.endswith((".cu", ".cuh", ".cpp", ".h")):
            assert "getenv" not in open(os.path.join(csrc, f)).read(), f
    assert "os.environ" not in open(S.__file__).read()
