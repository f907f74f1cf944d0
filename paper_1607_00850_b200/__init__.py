"""B200-native hot path of the triply periodic Fourier-Galerkin Navier-Stokes
solver (arXiv 1607.00850), behind the reference solver's operator API.

This package is a thin Python mirror of the reference C++ API
(``sdns``: SolverConfig, build_layout, DistributedFFT, curl_hat, cross,
project, pressure_hat, compute_rhs, Rk4State / rk4_step / advance,
collect_stats, l2_diff) over the C ABI declared in ``include/sdns_cuda.h``
and implemented by ``libsdns_cuda.so`` (sm_100a CUDA kernels + C++ host
orchestration + NCCL). Every compute call runs on the GPU; there is no CPU
fallback: if the library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import contextlib
import ctypes
import os
import threading
import weakref
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

__all__ = [
    "SolverConfig", "Layout", "ConfigError", "ProtocolError", "CollectiveTimeout",
    "DivergenceError", "IoError", "CudaError", "SdnsError", "load_library", "validate",
    "build_layout", "device_layout", "exchange_plan", "block_size", "block_start", "step_count", "spectrum_shells",
    "iso_init", "Comm", "Context", "Field", "DistributedFFT", "curl_hat", "cross",
    "project", "pressure_hat", "compute_rhs", "Rk4State", "FlowStats", "collect_stats",
    "l2_diff", "write_checkpoint", "read_checkpoint", "run_group",
    "ParsedConfig", "parse_config_text", "parse_config_file", "default_pencil_grid",
    "RunOptions", "RunResult", "run", "BenchEntry", "BenchRow", "parse_bench_matrix_text",
    "parse_bench_matrix_file", "bench", "write_bench_csv", "write_diagnostics_csv",
    "write_manifest", "CriterionResult", "run_acceptance_suite",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsdns_cuda.so")


# --- errors (proj/core/include/sdns/types.hpp:28-62) ------------------------

class SdnsError(RuntimeError):
    code = 9


class ConfigError(SdnsError):
    code = 1


class ProtocolError(SdnsError):
    code = 2


class CollectiveTimeout(SdnsError):
    code = 3


class DivergenceError(SdnsError):
    code = 4

    def __init__(self, msg, step=0):
        super().__init__(msg)
        self.step = step


class IoError(SdnsError):
    code = 5


class CudaError(SdnsError):
    code = 6


# the reference's name (types.hpp:41-44); CollectiveTimeout does not shadow
# the builtin inside this module
TimeoutError = CollectiveTimeout  # noqa: A001

_ERRORS = {1: ConfigError, 2: ProtocolError, 3: CollectiveTimeout, 4: DivergenceError,
           5: IoError, 6: CudaError}


# --- C structs ----------------------------------------------------------------

class _Config(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("decomp", ctypes.c_int), ("p", ctypes.c_int),
                ("p1", ctypes.c_int), ("p2", ctypes.c_int), ("nu", ctypes.c_double),
                ("dt", ctypes.c_double), ("t_end", ctypes.c_double),
                ("dealias", ctypes.c_int), ("out_every", ctypes.c_int)]


MAX_PEERS = 64


class _Layout(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("p", ctypes.c_int), ("p1", ctypes.c_int),
                ("p2", ctypes.c_int), ("coord1", ctypes.c_int), ("coord2", ctypes.c_int),
                ("n", ctypes.c_int64), ("nf", ctypes.c_int64),
                ("real_shape", ctypes.c_int64 * 3), ("real_offset", ctypes.c_int64 * 3),
                ("spec_shape", ctypes.c_int64 * 3), ("spec_offset", ctypes.c_int64 * 3),
                ("nstages", ctypes.c_int), ("stage_peers", ctypes.c_int * 2),
                ("send_counts", (ctypes.c_int64 * MAX_PEERS) * 2),
                ("recv_counts", (ctypes.c_int64 * MAX_PEERS) * 2)]


class _DevLayout(ctypes.Structure):
    _fields_ = [("pitch", ctypes.c_int), ("prow", ctypes.c_int), ("np", ctypes.c_int),
                ("spec_cs", ctypes.c_int64), ("real_cs", ctypes.c_int64)]


PASS_NAMES = ["x_inv_curl", "y_inv", "z_fused", "y_fwd", "x_fwd_tail", "x_fwd_rk0",
              "x_fwd_rk12", "x_fwd_rk3", "a2a_inv", "a2a_fwd", "x_fwd_fft"]
NPASS = len(PASS_NAMES)

class _ParsedConfig(ctypes.Structure):
    _fields_ = [("cfg", _Config), ("initial_case", ctypes.c_char * 64),
                ("notices", ctypes.c_char * 512)]


class _CtxOptions(ctypes.Structure):
    _fields_ = [("all_to_all", ctypes.c_int), ("serial", ctypes.c_int),
                ("ldgsts_tiles", ctypes.c_int), ("plain_layout", ctypes.c_int),
                ("no_graph", ctypes.c_int), ("p1_single", ctypes.c_int)]


class _RunOptions(ctypes.Structure):
    _fields_ = [("out_dir", ctypes.c_char_p), ("backend", ctypes.c_char_p),
                ("collective_timeout_s", ctypes.c_double), ("device", ctypes.c_int),
                ("seed", ctypes.c_uint64), ("ctx", _CtxOptions)]


class _RunResult(ctypes.Structure):
    _fields_ = [("backend", ctypes.c_char * 16), ("status", ctypes.c_char * 256),
                ("steps", ctypes.c_int64), ("step_min_s", ctypes.c_double),
                ("step_mean_s", ctypes.c_double), ("step_max_s", ctypes.c_double),
                ("timed_steps", ctypes.c_int64), ("shells", ctypes.c_int),
                ("n_samples", ctypes.c_int64), ("sample_cap", ctypes.c_int64),
                ("sample_steps", ctypes.POINTER(ctypes.c_int64)),
                ("sample_rows", ctypes.POINTER(ctypes.c_double)),
                ("csv_path", ctypes.c_char * 512), ("checkpoint_path", ctypes.c_char * 512),
                ("manifest_path", ctypes.c_char * 512)]


class _BenchEntry(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("decomp", ctypes.c_int), ("p", ctypes.c_int),
                ("p1", ctypes.c_int), ("p2", ctypes.c_int)]


class _BenchRow(ctypes.Structure):
    _fields_ = [("entry", _BenchEntry), ("nodes_per_rank", ctypes.c_int64),
                ("sec_per_step", ctypes.c_double), ("status", ctypes.c_char * 256)]


class _CriterionResult(ctypes.Structure):
    _fields_ = [("index", ctypes.c_int), ("name", ctypes.c_char * 64), ("passed", ctypes.c_int),
                ("detail", ctypes.c_char * 512), ("seconds", ctypes.c_double)]


SAMPLE_FN = ctypes.CFUNCTYPE(None, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                ctypes.c_void_p)
GROUP_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                            ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p))

_lib = None
_lib_lock = threading.Lock()


def use_library(path: str):
    """Selects another build of the library (A/B variants from
    tools/build_variant.sh) before the first call loads one."""
    global LIB_PATH
    if _lib is not None and os.path.abspath(path) != os.path.abspath(LIB_PATH):
        raise CudaError("the library is already loaded; call use_library first")
    LIB_PATH = path


def load_library(path: Optional[str] = None):
    """Loads libsdns_cuda.so (built by __graft_entry__.build()). Raises if absent."""
    global _lib
    path = path or LIB_PATH
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise CudaError(f"{path} is missing: run __graft_entry__.build() first")
        lib = ctypes.CDLL(path)
        P, I, D, I64, V = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64, None
        PP = ctypes.POINTER(ctypes.c_void_p)
        sig = {
            "sdns_last_error": (ctypes.c_char_p, []),
            "sdns_version": (ctypes.c_char_p, []),
            "sdns_config_validate": (I, [ctypes.POINTER(_Config)]),
            "sdns_build_layout": (I, [ctypes.POINTER(_Config), I, ctypes.POINTER(_Layout)]),
            "sdns_block_size": (I64, [I64, I, I]),
            "sdns_block_start": (I64, [I64, I, I]),
            "sdns_step_count": (I64, [D, D]),
            "sdns_spectrum_shells": (I, [I64]),
            "sdns_iso_init_host": (I, [I64, ctypes.c_uint64, D, D, ctypes.POINTER(_Layout), P]),
            "sdns_comm_loopback": (I, [PP]),
            "sdns_comm_inprocess_group": (I, [I, I, D, PP]),
            "sdns_comm_nccl_unique_id": (I, [ctypes.c_char_p]),
            "sdns_comm_nccl_init": (I, [ctypes.c_char_p, I, I, I, PP]),
            "sdns_comm_rank": (I, [P]),
            "sdns_comm_size": (I, [P]),
            "sdns_comm_barrier": (I, [P]),
            "sdns_comm_allreduce": (I, [P, P, I, I]),
            "sdns_comm_broadcast_bytes": (I, [P, P, ctypes.c_int64, I]),
            "sdns_comm_destroy": (I, [P]),
            "sdns_ctx_create": (I, [ctypes.POINTER(_Config), I, I, P, P, PP]),
            "sdns_ctx_create_ex": (I, [ctypes.POINTER(_Config), I, I, P, P, P, PP]),
            "sdns_ctx_destroy": (I, [P]),
            "sdns_ctx_layout": (I, [P, ctypes.POINTER(_Layout)]),
            "sdns_ctx_stream": (P, [P]),
            "sdns_ctx_sync": (I, [P]),
            "sdns_ctx_device_bytes": (I64, [P]),
            "sdns_field_alloc": (I, [P, I, I, PP]),
            "sdns_field_free": (I, [P]),
            "sdns_field_upload": (I, [P, P, P]),
            "sdns_field_download": (I, [P, P, P]),
            "sdns_field_copy": (I, [P, P, P]),
            "sdns_fft_forward": (I, [P, P, P]),
            "sdns_fft_inverse": (I, [P, P, P]),
            "sdns_curl_hat": (I, [P, P, P]),
            "sdns_cross": (I, [P, P, P, P]),
            "sdns_project": (I, [P, P]),
            "sdns_pressure_hat": (I, [P, P, P]),
            "sdns_compute_rhs": (I, [P, P, D, P]),
            "sdns_state_create": (I, [P, PP]),
            "sdns_state_destroy": (I, [P]),
            "sdns_state_set": (I, [P, P, P, D, I64]),
            "sdns_state_get": (I, [P, P, P]),
            "sdns_state_u_hat": (P, [P]),
            "sdns_state_time": (I, [P, ctypes.POINTER(D), ctypes.POINTER(I64)]),
            "sdns_rk4_step": (I, [P, P, D, I, ctypes.POINTER(I)]),
            "sdns_advance": (I, [P, P, SAMPLE_FN, P, ctypes.POINTER(I64)]),
            "sdns_rk4_step_host": (I, [P, P, P, D, I]),
            "sdns_collect_stats": (I, [P, P, D, D, P]),
            "sdns_l2_diff": (I, [P, P, P, ctypes.POINTER(D)]),
            "sdns_checkpoint_write": (I, [P, P, ctypes.c_char_p, D, ctypes.c_int64]),
            "sdns_checkpoint_read": (I, [P, ctypes.c_char_p, P, ctypes.POINTER(D),
                                         ctypes.POINTER(ctypes.c_int64)]),
            "sdns_ctx_timing": (I, [P, I]),
            "sdns_ctx_timing_read": (I, [P, P, P]),
            "sdns_device_layout": (I, [ctypes.POINTER(_Config), I, ctypes.POINTER(_DevLayout)]),
            "sdns_exchange_plan": (I, [ctypes.POINTER(_Config), I, I, I, P, ctypes.POINTER(I)]),
            "sdns_comm_split": (I, [P, I, I, PP]),
            "sdns_comm_poison": (I, [P, ctypes.c_char_p]),
            "sdns_comm_host_init": (I, [I, I, I, ALLGATHER_FN, GROUP_FN, P, PP]),
            "sdns_comm_set_timeout": (I, [P, D]),
            "sdns_ctx_transposes": (I, [P]),
            "sdns_comm_all_to_all_bytes": (I, [P, P, P, P, P, P]),
            "sdns_config_defaults": (V, [ctypes.POINTER(_Config)]),
            "sdns_parse_config_text": (I, [ctypes.c_char_p, P, P, I,
                                           ctypes.POINTER(_ParsedConfig)]),
            "sdns_parse_config_file": (I, [ctypes.c_char_p, P, P, I,
                                           ctypes.POINTER(_ParsedConfig)]),
            "sdns_default_pencil_grid": (I, [I, I, ctypes.POINTER(I), ctypes.POINTER(I)]),
            "sdns_run": (I, [ctypes.POINTER(_Config), ctypes.c_char_p,
                             ctypes.POINTER(_RunOptions), ctypes.POINTER(_RunResult)]),
            "sdns_run_rank": (I, [ctypes.POINTER(_Config), ctypes.c_char_p,
                                  ctypes.POINTER(_RunOptions), I, P,
                                  ctypes.POINTER(_RunResult)]),
            "sdns_parse_bench_matrix_text": (I, [ctypes.c_char_p, P, I, ctypes.POINTER(I)]),
            "sdns_parse_bench_matrix_file": (I, [ctypes.c_char_p, P, I, ctypes.POINTER(I)]),
            "sdns_bench": (I, [P, I, I, ctypes.POINTER(_RunOptions), P]),
            "sdns_write_bench_csv": (I, [ctypes.c_char_p, P, I]),
            "sdns_write_diagnostics_csv": (I, [ctypes.c_char_p, P, P, I64, I]),
            "sdns_write_manifest": (I, [ctypes.c_char_p, ctypes.POINTER(_Config),
                                        ctypes.c_char_p, ctypes.POINTER(_RunResult)]),
            "sdns_acceptance_suite": (I, [I, I, P, ctypes.POINTER(I)]),
            "sdns_advance_hooks_run": (I, [P, P, P, ctypes.POINTER(I64)]),
            "sdns_host_alloc": (P, [ctypes.c_size_t]),
            "sdns_host_free": (V, [P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def _check(rc: int, step: int = 0):
    if rc == 0:
        return
    msg = load_library().sdns_last_error().decode(errors="replace")
    cls = _ERRORS.get(rc, SdnsError)
    if cls is DivergenceError:
        raise DivergenceError(msg, step)
    raise cls(msg)


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


# --- config and layout (config.hpp, layout.hpp) --------------------------------

@dataclass
class SolverConfig:
    """SolverConfig, proj/core/include/sdns/config.hpp:14-30."""
    n: int = 32
    decomp: str = "slab"
    p: int = 1
    p1: int = 1
    p2: int = 1
    nu: float = 1.0 / 1600.0
    dt: float = 1e-3
    t_end: float = 0.1
    dealias: bool = True
    initial_case: str = "taylor_green"
    out_every: int = 10

    def to_c(self) -> _Config:
        if self.decomp not in ("slab", "pencil"):
            raise ConfigError(f"unknown decomposition '{self.decomp}' (expected slab|pencil)")
        slab = self.decomp == "slab"
        return _Config(self.n, 0 if slab else 1, self.p, 1 if slab else self.p1,
                       1 if slab else self.p2, self.nu, self.dt, self.t_end,
                       1 if self.dealias else 0, self.out_every)

    def validate(self):
        validate(self)


@dataclass
class Layout:
    """RankLayout, proj/core/include/sdns/layout.hpp:24-41."""
    rank: int
    p: int
    p1: int
    p2: int
    coord1: int
    coord2: int
    n: int
    nf: int
    real_shape: tuple
    real_offset: tuple
    spec_shape: tuple
    spec_offset: tuple
    stages: list = field(default_factory=list)  # [(send_counts, recv_counts)]

    @staticmethod
    def _from_c(c: _Layout) -> "Layout":
        stages = []
        for s in range(c.nstages):
            k = c.stage_peers[s]
            stages.append(([c.send_counts[s][q] for q in range(k)],
                           [c.recv_counts[s][q] for q in range(k)]))
        return Layout(c.rank, c.p, c.p1, c.p2, c.coord1, c.coord2, c.n, c.nf,
                      tuple(c.real_shape), tuple(c.real_offset), tuple(c.spec_shape),
                      tuple(c.spec_offset), stages)

    def _to_c(self) -> _Layout:
        c = _Layout()
        c.rank, c.p, c.p1, c.p2 = self.rank, self.p, self.p1, self.p2
        c.coord1, c.coord2, c.n, c.nf = self.coord1, self.coord2, self.n, self.nf
        for i in range(3):
            c.real_shape[i] = self.real_shape[i]
            c.real_offset[i] = self.real_offset[i]
            c.spec_shape[i] = self.spec_shape[i]
            c.spec_offset[i] = self.spec_offset[i]
        c.nstages = len(self.stages)
        for s, (sc, rc) in enumerate(self.stages):
            c.stage_peers[s] = len(sc)
            for q in range(len(sc)):
                c.send_counts[s][q] = sc[q]
                c.recv_counts[s][q] = rc[q]
        return c


def validate(cfg: SolverConfig):
    """SolverConfig::validate, proj/core/src/config.cpp:17-50."""
    c = cfg.to_c()
    _check(load_library().sdns_config_validate(ctypes.byref(c)))


def build_layout(cfg: SolverConfig, rank: int) -> Layout:
    """build_layout, proj/core/src/layout.cpp:17-76."""
    c = cfg.to_c()
    out = _Layout()
    _check(load_library().sdns_build_layout(ctypes.byref(c), rank, ctypes.byref(out)))
    return Layout._from_c(out)


def device_layout(cfg: SolverConfig, rank: int) -> dict:
    """Device field layout of a rank (include/sdns_cuda.h sdns_device_layout)."""
    c = cfg.to_c()
    out = _DevLayout()
    _check(load_library().sdns_device_layout(ctypes.byref(c), rank, ctypes.byref(out)))
    return {"pitch": out.pitch, "prow": out.prow, "np": out.np, "spec_cs": out.spec_cs,
            "real_cs": out.real_cs}


def exchange_plan(cfg: SolverConfig, rank: int, inverse: bool, nfields: int) -> np.ndarray:
    """The transpose plan a context executes: rows (peer, src_off, dst_off, count)."""
    c = cfg.to_c()
    cnt = ctypes.c_int(0)
    lib = load_library()
    _check(lib.sdns_exchange_plan(ctypes.byref(c), rank, int(inverse), nfields, None,
                                  ctypes.byref(cnt)))
    out = np.zeros((cnt.value, 4), dtype=np.int64)
    _check(lib.sdns_exchange_plan(ctypes.byref(c), rank, int(inverse), nfields, _ptr(out),
                                  ctypes.byref(cnt)))
    return out


def block_size(total: int, parts: int, index: int) -> int:
    return load_library().sdns_block_size(total, parts, index)


def block_start(total: int, parts: int, index: int) -> int:
    return load_library().sdns_block_start(total, parts, index)


def step_count(t_end: float, dt: float) -> int:
    """proj/core/src/rk4.cpp:79-84."""
    return load_library().sdns_step_count(t_end, dt)


def spectrum_shells(n: int) -> int:
    """proj/core/src/diagnostics.cpp:66-69."""
    return load_library().sdns_spectrum_shells(n)


def iso_init(n: int, layout: Layout, seed: int = 1607, k0: float = 4.0,
             energy: float = 0.5) -> np.ndarray:
    """Seeded isotropic initial u_hat for the rank's spectral block,
    shape (3, *spec_shape) complex128 (BASELINE configs 2-4)."""
    out = np.empty((3,) + tuple(layout.spec_shape), dtype=np.complex128)
    lc = layout._to_c()
    _check(load_library().sdns_iso_init_host(n, seed, k0, energy, ctypes.byref(lc), _ptr(out)))
    return out


# --- communicators (transport.hpp:46-131) ---------------------------------------

class Comm:
    """Communicator handle: loopback, in-process group or NCCL."""

    def __init__(self, handle):
        self._h = handle
        self._lib = load_library()

    @staticmethod
    def loopback() -> "Comm":
        h = ctypes.c_void_p()
        _check(load_library().sdns_comm_loopback(ctypes.byref(h)))
        return Comm(h)

    @staticmethod
    def inprocess_group(size: int, device: int = 0, timeout_s: float = 600.0) -> List["Comm"]:
        arr = (ctypes.c_void_p * size)()
        _check(load_library().sdns_comm_inprocess_group(size, device, timeout_s, arr))
        return [Comm(ctypes.c_void_p(arr[i])) for i in range(size)]

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load_library().sdns_comm_nccl_unique_id(buf))
        return buf.raw

    @staticmethod
    def nccl(uid: bytes, size: int, rank: int, device: int) -> "Comm":
        h = ctypes.c_void_p()
        _check(load_library().sdns_comm_nccl_init(uid, size, rank, device, ctypes.byref(h)))
        return Comm(h)

    @staticmethod
    def host(size: int, rank: int, device: int, allgather: Callable,
             new_group: Optional[Callable] = None) -> "Comm":
        """One process per rank over a host all-gather: `allgather(data,
        group)` returns every member's `data` (bytes) in rank order for the
        group handle `group` (None = the world); `new_group(ranks)` (world
        ranks, called on every rank for every group, as
        torch.distributed.new_group requires) returns a handle and enables
        split() for the pencil row/column groups. CUDA IPC memory and events
        carry the peer-direct transposes; several ranks may share a GPU."""
        groups = {0: (None, list(range(size)))}

        def cb(send, nbytes, recv, user):
            try:
                g, members = groups[user or 0]
                parts = allgather(ctypes.string_at(send, nbytes), g)
                buf = b"".join(parts)
                if len(buf) != nbytes * len(members):
                    return 1
                ctypes.memmove(recv, buf, len(buf))
                return 0
            except BaseException as e:  # noqa: BLE001
                # a peer that stalled or died surfaces as the caller's
                # transport timeout (gloo: "Timed out waiting ... ms")
                m = str(e).lower()
                return 2 if ("timed out" in m or "timeout" in m) else 1

        def gcb(ranks, n, user, child):
            try:
                _, members = groups[user or 0]
                world = [members[ranks[i]] for i in range(n)]
                key = len(groups)
                groups[key] = (new_group(world), world)
                child[0] = key
                return 0
            except BaseException:  # noqa: BLE001
                return 1

        fn = ALLGATHER_FN(cb)
        gfn = GROUP_FN(gcb) if new_group else GROUP_FN()
        h = ctypes.c_void_p()
        _check(load_library().sdns_comm_host_init(size, rank, device, fn, gfn, None,
                                                  ctypes.byref(h)))
        c = Comm(h)
        c._keep = (fn, gfn, groups)  # the callbacks must outlive the communicator
        return c

    def set_timeout(self, seconds: float) -> "Comm":
        """Collective deadline (reference collective_timeout, default 30 s):
        past it a host wait raises TimeoutError and the communicator is
        aborted; later collectives fail fast with the same error."""
        _check(self._lib.sdns_comm_set_timeout(self._h, float(seconds)))
        return self

    @property
    def rank(self) -> int:
        return self._lib.sdns_comm_rank(self._h)

    @property
    def size(self) -> int:
        return self._lib.sdns_comm_size(self._h)

    def barrier(self):
        _check(self._lib.sdns_comm_barrier(self._h))

    def allreduce(self, values, op: str = "sum") -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.float64).copy()
        _check(self._lib.sdns_comm_allreduce(self._h, _ptr(v), v.size,
                                             {"sum": 0, "max": 1, "min": 2}[op]))
        return v

    def broadcast_bytes(self, data, root: int = 0) -> bytes:
        """broadcast_bytes, transport.hpp:62: the root's bytes on every rank
        (`data`: bytes-like of the agreed length; the root's content is sent)."""
        buf = ctypes.create_string_buffer(bytes(data), len(data))
        _check(self._lib.sdns_comm_broadcast_bytes(self._h, buf, len(data), root))
        return buf.raw

    def split(self, color: int, key: int) -> "Comm":
        """split, transport.hpp:66-67: members ordered by (key, rank)."""
        h = ctypes.c_void_p()
        _check(self._lib.sdns_comm_split(self._h, color, key, ctypes.byref(h)))
        return Comm(h)

    def poison(self, reason: str):
        """InProcessBackend::poison, transport.hpp:125-128."""
        _check(self._lib.sdns_comm_poison(self._h, reason.encode()))

    def all_to_all_bytes(self, send_ptr: int, send_bytes, recv_ptr: int, recv_bytes,
                         stream: int = 0):
        """all_to_all_bytes (transport.hpp:55-58) on DEVICE buffers; block q
        of send goes to peer q (displacements = prefix sums of the counts)."""
        sb = np.ascontiguousarray(send_bytes, dtype=np.int64)
        rb = np.ascontiguousarray(recv_bytes, dtype=np.int64)
        _check(self._lib.sdns_comm_all_to_all_bytes(self._h, ctypes.c_void_p(send_ptr), _ptr(sb),
                                                    ctypes.c_void_p(recv_ptr), _ptr(rb),
                                                    ctypes.c_void_p(stream) if stream else None))

    def close(self):
        if self._h:
            self._lib.sdns_comm_destroy(self._h)
            self._h = None


def run_group(size: int, body: Callable[[int, Comm], object], device: int = 0,
              timeout_s: float = 600.0) -> list:
    """run_group, proj/core/src/transport.cpp:397-424: runs body(rank, comm)
    on one host thread per rank over an in-process group sharing `device`;
    rethrows the lowest-rank exception."""
    comms = [Comm.loopback()] if size == 1 else Comm.inprocess_group(size, device, timeout_s)
    results: list = [None] * size
    errors: list = [None] * size

    def worker(r):
        try:
            results[r] = body(r, comms[r])
        except BaseException as e:  # noqa: BLE001
            errors[r] = e

    if size == 1:
        worker(0)
    else:
        ts = [threading.Thread(target=worker, args=(r,)) for r in range(size)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    for c in comms:
        c.close()
    for e in errors:
        if e is not None:
            raise e
    return results


# --- context and fields -----------------------------------------------------------

_OPTION_KEYS = ("all_to_all", "serial", "ldgsts_tiles", "plain_layout", "no_graph", "p1_single")
_default_options: dict = {}


@contextlib.contextmanager
def context_options(**kw):
    """Default execution options of the Contexts created inside the block
    (sdns_ctx_options: all_to_all, serial, ldgsts_tiles, plain_layout,
    no_graph, p1_single); none changes a result bit. The library reads no environment."""
    global _default_options
    bad = set(kw) - set(_OPTION_KEYS)
    if bad:
        raise ConfigError(f"unknown context options {sorted(bad)}")
    old = _default_options
    _default_options = {**old, **kw}
    try:
        yield
    finally:
        _default_options = old


def set_default_options(**kw) -> None:
    """Execution options of every Context created from now on (A/B runs)."""
    global _default_options
    bad = set(kw) - set(_OPTION_KEYS)
    if bad:
        raise ConfigError(f"unknown context options {sorted(bad)}")
    _default_options = {**_default_options, **kw}


def _ctx_options(options: Optional[dict]) -> _CtxOptions:
    opt = {**_default_options, **(options or {})}
    bad = set(opt) - set(_OPTION_KEYS)
    if bad:
        raise ConfigError(f"unknown context options {sorted(bad)}")
    return _CtxOptions(*[int(opt.get(k, 0)) for k in _OPTION_KEYS])


class Context:
    """One rank's device context: DistributedFFT + WavenumberMesh + RhsWorkspace
    (proj/core/src/fft.cpp:15-57, mesh.cpp:23-72, navier_stokes.hpp:32-41).
    `options`: execution choices (see context_options)."""

    def __init__(self, cfg: SolverConfig, rank: int = 0, device: int = 0,
                 comm: Optional[Comm] = None, stream: Optional[int] = None,
                 options: Optional[dict] = None):
        self.cfg = cfg
        self._lib = load_library()
        self._own_comm = comm is None
        self.comm = comm if comm is not None else Comm.loopback()
        c = cfg.to_c()
        h = ctypes.c_void_p()
        copt = _ctx_options(options)
        _check(self._lib.sdns_ctx_create_ex(ctypes.byref(c), rank, device, self.comm._h,
                                            ctypes.c_void_p(stream) if stream else None,
                                            ctypes.byref(copt), ctypes.byref(h)))
        self._h = h
        # fields and states allocated under this context: freed before it
        self._children = weakref.WeakSet()
        lo = _Layout()
        self._lib.sdns_ctx_layout(h, ctypes.byref(lo))
        self.layout = Layout._from_c(lo)

    @property
    def stream(self) -> int:
        return self._lib.sdns_ctx_stream(self._h) or 0

    @property
    def device_bytes(self) -> int:
        return self._lib.sdns_ctx_device_bytes(self._h)

    @property
    def transposes(self) -> str:
        """How the RHS pipeline's transposes run: "peer-direct" (all),
        "peer-direct (column)" / "peer-direct (row)" (pencil, one group) or
        "all-to-all"."""
        f = self._lib.sdns_ctx_transposes(self._h)
        if self.cfg.decomp == "pencil" and self.cfg.p > 1:
            need = (1 if self.cfg.p1 > 1 else 0) | (2 if self.cfg.p2 > 1 else 0)
            if f and f != need:
                return "peer-direct (column)" if f == 1 else "peer-direct (row)"
        return "peer-direct" if f else "all-to-all"

    def sync(self):
        _check(self._lib.sdns_ctx_sync(self._h))

    def timing(self, enable: bool = True):
        """Enables (and resets) CUDA-event timing of every pipeline launch."""
        _check(self._lib.sdns_ctx_timing(self._h, 1 if enable else 0))

    def timing_read(self):
        """Returns {pass: (total_ms, launches)} since the last enable/read."""
        ms = np.zeros(NPASS)
        cnt = np.zeros(NPASS, dtype=np.int64)
        _check(self._lib.sdns_ctx_timing_read(self._h, _ptr(ms), _ptr(cnt)))
        return {PASS_NAMES[i]: (float(ms[i]), int(cnt[i])) for i in range(NPASS)}

    def real_field(self, ncomp: int = 3) -> "Field":
        return Field(self, 0, ncomp)

    def spectral_field(self, ncomp: int = 3) -> "Field":
        return Field(self, 1, ncomp)

    def close(self):
        if self._h:
            # device fields and states reference the context: release them
            # first (sdns_field_free / sdns_state_destroy use its device)
            kids = list(self._children)
            for k in kids:
                if isinstance(k, Field):
                    k.free()
            for k in kids:
                if isinstance(k, Rk4State):
                    k.close()
            self._lib.sdns_ctx_destroy(self._h)
            self._h = None
        if self._own_comm:
            self.comm.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Field:
    """Device-resident field (Field3d / VectorField3, fields.hpp:10-49)."""

    def __init__(self, ctx: Context, kind: int, ncomp: int, handle=None, owned=True):
        self.ctx = ctx
        self.kind = kind
        self.ncomp = ncomp
        self._owned = owned
        if handle is None:
            h = ctypes.c_void_p()
            _check(ctx._lib.sdns_field_alloc(ctx._h, kind, ncomp, ctypes.byref(h)))
            handle = h
        self._h = handle
        ctx._children.add(self)

    def __del__(self):
        try:
            if self._h and self._owned and self.ctx._h:
                self.free()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass

    @property
    def shape(self) -> tuple:
        lo = self.ctx.layout
        return (self.ncomp,) + tuple(lo.real_shape if self.kind == 0 else lo.spec_shape)

    @property
    def dtype(self):
        return np.float64 if self.kind == 0 else np.complex128

    def upload(self, host: np.ndarray) -> "Field":
        a = np.ascontiguousarray(host, dtype=self.dtype).reshape(self.shape)
        _check(self.ctx._lib.sdns_field_upload(self.ctx._h, self._h, _ptr(a)))
        return self

    def download(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype)
        _check(self.ctx._lib.sdns_field_download(self.ctx._h, self._h, _ptr(out)))
        return out

    def copy_from(self, other: "Field"):
        _check(self.ctx._lib.sdns_field_copy(self.ctx._h, other._h, self._h))

    def free(self):
        if self._h and self._owned:
            self.ctx._lib.sdns_field_free(self._h)
        self._h = None


# --- operators ---------------------------------------------------------------------

class DistributedFFT:
    """DistributedFFT, proj/core/include/sdns/fft.hpp:26-62 (collective)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def forward(self, u: Field, fu: Field):
        _check(self.ctx._lib.sdns_fft_forward(self.ctx._h, u._h, fu._h))

    def inverse(self, fu: Field, u: Field):
        _check(self.ctx._lib.sdns_fft_inverse(self.ctx._h, fu._h, u._h))


def curl_hat(ctx: Context, u_hat: Field, omega_hat: Field):
    """navier_stokes.cpp:52-72."""
    _check(ctx._lib.sdns_curl_hat(ctx._h, u_hat._h, omega_hat._h))


def cross(ctx: Context, a: Field, b: Field, out: Field):
    """navier_stokes.cpp:34-50."""
    _check(ctx._lib.sdns_cross(ctx._h, a._h, b._h, out._h))


def project(ctx: Context, u_hat: Field):
    """navier_stokes.cpp:85-102 (in place)."""
    _check(ctx._lib.sdns_project(ctx._h, u_hat._h))


def pressure_hat(ctx: Context, nl_hat: Field, p_hat: Field):
    """navier_stokes.cpp:74-83."""
    _check(ctx._lib.sdns_pressure_hat(ctx._h, nl_hat._h, p_hat._h))


def compute_rhs(ctx: Context, u_hat: Field, nu: float, du_hat: Field):
    """navier_stokes.cpp:104-139."""
    _check(ctx._lib.sdns_compute_rhs(ctx._h, u_hat._h, nu, du_hat._h))


class Rk4State:
    """Rk4State + rk4_step + advance (proj/core/include/sdns/rk4.hpp:18-62)."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        h = ctypes.c_void_p()
        _check(ctx._lib.sdns_state_create(ctx._h, ctypes.byref(h)))
        self._h = h
        self.u_hat = Field(ctx, 1, 3, handle=ctypes.c_void_p(ctx._lib.sdns_state_u_hat(h)),
                           owned=False)
        ctx._children.add(self)

    def __del__(self):
        try:
            if self._h and self.ctx._h:
                self.close()
        except Exception:  # noqa: BLE001  (interpreter shutdown)
            pass

    def set(self, u_hat: Field, t: float = 0.0, step: int = 0):
        _check(self.ctx._lib.sdns_state_set(self.ctx._h, self._h, u_hat._h, t, step))

    def get(self, out: Field):
        _check(self.ctx._lib.sdns_state_get(self.ctx._h, self._h, out._h))

    @property
    def t(self) -> float:
        t = ctypes.c_double()
        s = ctypes.c_int64()
        self.ctx._lib.sdns_state_time(self._h, ctypes.byref(t), ctypes.byref(s))
        return t.value

    @property
    def step(self) -> int:
        t = ctypes.c_double()
        s = ctypes.c_int64()
        self.ctx._lib.sdns_state_time(self._h, ctypes.byref(t), ctypes.byref(s))
        return s.value

    def rk4_step(self, dt: float, post_project: bool = True, check: bool = True) -> bool:
        """rk4_step (rk4.cpp:73-77) with the runner's post-step projection
        fused in; raises DivergenceError on a non-finite update if check."""
        fin = ctypes.c_int(1)
        _check(self.ctx._lib.sdns_rk4_step(self.ctx._h, self._h, dt, 1 if post_project else 0,
                                            ctypes.byref(fin) if check else None))
        if check and not fin.value:
            raise DivergenceError(f"non-finite values in solution update at step {self.step}",
                                  self.step)
        return bool(fin.value)

    def advance(self, sample: Optional[Callable[[int, float], None]] = None):
        """advance, rk4.cpp:86-107 (post_step = project, runner.cpp:107)."""
        err: list = []

        def cb(step, t, _user):
            try:
                sample(int(step), float(t))
            except BaseException as e:  # noqa: BLE001
                err.append(e)

        fn = SAMPLE_FN(cb) if sample else SAMPLE_FN()
        fail = ctypes.c_int64(0)
        rc = self.ctx._lib.sdns_advance(self.ctx._h, self._h, fn, None, ctypes.byref(fail))
        if err:
            raise err[0]
        _check(rc, fail.value)

    def step_host(self, host_u_hat: np.ndarray, dt: float, steps: int = 1):
        """Host-buffer tier: upload, `steps` fused steps, download (in place)."""
        _check(self.ctx._lib.sdns_rk4_step_host(self.ctx._h, self._h, _ptr(host_u_hat), dt,
                                                 steps))

    def close(self):
        if self._h:
            self.ctx._lib.sdns_state_destroy(self._h)
            self._h = None


@dataclass
class FlowStats:
    """FlowStats, proj/core/include/sdns/diagnostics.hpp:12-19."""
    t: float
    energy: float
    enstrophy: float
    dissipation: float
    divergence_max: float
    spectrum: np.ndarray


def collect_stats(ctx: Context, u_hat: Field, nu: float, t: float = 0.0) -> FlowStats:
    """diagnostics.cpp:71-91 (deterministic device reduction + rank-order fold)."""
    shells = spectrum_shells(ctx.cfg.n)
    row = np.zeros(5 + shells)
    _check(ctx._lib.sdns_collect_stats(ctx._h, u_hat._h, nu, t, _ptr(row)))
    return FlowStats(row[0], row[1], row[2], row[3], row[4], row[5:].copy())


def write_checkpoint(ctx: Context, path: str, u: Field, t: float, step: int):
    """write_checkpoint, checkpoint.cpp:64-121 (collective; u = this rank's
    real velocity block). The reference's file format and error behaviour."""
    _check(ctx._lib.sdns_checkpoint_write(ctx._h, u._h, os.fsencode(path), float(t), int(step)))


def read_checkpoint(ctx: Context, path: str, u: Field):
    """read_checkpoint, checkpoint.cpp:123-187: fills u (this rank's block),
    returns (t, step)."""
    t = ctypes.c_double()
    step = ctypes.c_int64()
    _check(ctx._lib.sdns_checkpoint_read(ctx._h, os.fsencode(path), u._h, ctypes.byref(t),
                                         ctypes.byref(step)))
    return t.value, step.value


def l2_diff(ctx: Context, a: Field, b: Field) -> float:
    """diagnostics.cpp:113-127."""
    out = ctypes.c_double()
    _check(ctx._lib.sdns_l2_diff(ctx._h, a._h, b._h, ctypes.byref(out)))
    return out.value


# --- config files, runner and bench harness (config_file.hpp, runner.hpp) ------

_DECOMP = {"slab": 0, "pencil": 1}
_DECOMP_NAME = {0: "slab", 1: "pencil"}


@dataclass
class ParsedConfig:
    """ParsedConfig, proj/core/include/sdns/config_file.hpp:14-17."""
    cfg: SolverConfig
    notices: List[str]


def _from_c_config(c: _Config, initial_case: str = "taylor_green") -> SolverConfig:
    return SolverConfig(n=c.n, decomp=_DECOMP_NAME[c.decomp], p=c.p, p1=c.p1, p2=c.p2, nu=c.nu,
                        dt=c.dt, t_end=c.t_end, dealias=bool(c.dealias),
                        initial_case=initial_case, out_every=c.out_every)


def _overrides(overrides):
    items = list(overrides.items()) if isinstance(overrides, dict) else list(overrides or [])
    keys = (ctypes.c_char_p * max(1, len(items)))(*[k.encode() for k, _ in items])
    vals = (ctypes.c_char_p * max(1, len(items)))(*[str(v).encode() for _, v in items])
    return keys, vals, len(items)


def _parsed(out: _ParsedConfig) -> ParsedConfig:
    notes = [x for x in out.notices.decode().split("\n") if x]
    return ParsedConfig(_from_c_config(out.cfg, out.initial_case.decode()), notes)


def parse_config_text(text: str, overrides=()) -> ParsedConfig:
    """parse_config_text, config_file.cpp:57-136 (ordered overrides applied last)."""
    L = load_library()
    keys, vals, n = _overrides(overrides)
    out = _ParsedConfig()
    _check(L.sdns_parse_config_text(text.encode(), keys, vals, n, ctypes.byref(out)))
    return _parsed(out)


def parse_config_file(path: str, overrides=()) -> ParsedConfig:
    """parse_config_file, config_file.cpp:138-145 (IoError on a missing file)."""
    L = load_library()
    keys, vals, n = _overrides(overrides)
    out = _ParsedConfig()
    _check(L.sdns_parse_config_file(os.fsencode(path), keys, vals, n, ctypes.byref(out)))
    return _parsed(out)


def default_pencil_grid(n: int, p: int):
    """default_pencil_grid, config_file.cpp:43-55."""
    a, b = ctypes.c_int(), ctypes.c_int()
    _check(load_library().sdns_default_pencil_grid(n, p, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


@dataclass
class RunOptions:
    """RunOptions, proj/core/include/sdns/runner.hpp:11-15 (+ device, iso seed)."""
    out_dir: str = "out"
    backend: str = "auto"
    collective_timeout_s: float = 30.0
    device: int = 0
    seed: int = 1607
    options: Optional[dict] = None  # context execution options (context_options)

    def to_c(self) -> _RunOptions:
        return _RunOptions(os.fsencode(self.out_dir), self.backend.encode(),
                           self.collective_timeout_s, self.device, self.seed,
                           _ctx_options(self.options))


@dataclass
class RunResult:
    """RunResult, proj/core/include/sdns/runner.hpp:28-36."""
    cfg: SolverConfig
    backend: str
    status: str
    steps: int
    timing: dict
    samples: list          # [(step, FlowStats)]
    csv_path: str
    checkpoint_path: str
    manifest_path: str


def _run_result(cfg, r: _RunResult, steps, rows) -> RunResult:
    w = 5 + r.shells
    samples = []
    for i in range(min(r.n_samples, len(steps))):
        row = rows[i * w:(i + 1) * w]
        samples.append((int(steps[i]), FlowStats(row[0], row[1], row[2], row[3], row[4],
                                                 row[5:].copy())))
    return RunResult(cfg, r.backend.decode(), r.status.decode(), r.steps,
                     {"min_s": r.step_min_s, "mean_s": r.step_mean_s, "max_s": r.step_max_s,
                      "timed_steps": r.timed_steps},
                     samples, r.csv_path.decode(), r.checkpoint_path.decode(),
                     r.manifest_path.decode())


def _result_buffers(cfg: SolverConfig):
    cap = step_count(cfg.t_end, cfg.dt) // cfg.out_every + 2
    steps = np.zeros(cap, dtype=np.int64)
    rows = np.zeros(cap * (5 + spectrum_shells(cfg.n)))
    r = _RunResult()
    r.sample_cap = cap
    r.sample_steps = steps.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    r.sample_rows = rows.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    return r, steps, rows


def run(cfg: SolverConfig, opts: Optional[RunOptions] = None,
        comm: Optional["Comm"] = None, rank: int = 0) -> RunResult:
    """run(), runner.cpp:197-213: ranks as threads on one device (comm None),
    or, with `comm`, one rank of a caller-made group (run_worker,
    runner.cpp:67-146; e.g. one process per GPU over NCCL). Writes
    diagnostics.csv, checkpoint.sdns and manifest.txt into opts.out_dir.
    DivergenceError after the last-good checkpoint, like the reference."""
    L = load_library()
    opts = opts or RunOptions()
    r, steps, rows = _result_buffers(cfg)
    c = cfg.to_c()
    o = opts.to_c()
    if comm is None:
        rc = L.sdns_run(ctypes.byref(c), cfg.initial_case.encode(), ctypes.byref(o),
                        ctypes.byref(r))
    else:
        rc = L.sdns_run_rank(ctypes.byref(c), cfg.initial_case.encode(), ctypes.byref(o), rank,
                             comm._h, ctypes.byref(r))
    if rc == DivergenceError.code:
        msg = L.sdns_last_error().decode(errors="replace")
        st = r.status.decode()
        step = int(st.rsplit(" ", 1)[-1]) if st.startswith("diverged at step") else 0
        raise DivergenceError(msg, step)
    _check(rc)
    return _run_result(cfg, r, steps, rows)


@dataclass
class BenchEntry:
    """BenchEntry, runner.hpp:40-45 (p1 = p2 = 0: near-square pencil grid)."""
    n: int = 32
    decomp: str = "slab"
    p: int = 1
    p1: int = 0
    p2: int = 0


@dataclass
class BenchRow:
    """BenchRow, runner.hpp:47-52."""
    entry: BenchEntry
    nodes_per_rank: int
    sec_per_step: float
    status: str


def _entries(arr, count) -> List[BenchEntry]:
    return [BenchEntry(e.n, _DECOMP_NAME[e.decomp], e.p, e.p1, e.p2) for e in arr[:count]]


def parse_bench_matrix_text(text: str) -> List[BenchEntry]:
    """parse_bench_matrix_text, runner.cpp:249-289."""
    L = load_library()
    n = ctypes.c_int()
    _check(L.sdns_parse_bench_matrix_text(text.encode(), None, 0, ctypes.byref(n)))
    arr = (_BenchEntry * max(1, n.value))()
    _check(L.sdns_parse_bench_matrix_text(text.encode(), arr, n.value, ctypes.byref(n)))
    return _entries(arr, n.value)


def parse_bench_matrix_file(path: str) -> List[BenchEntry]:
    """parse_bench_matrix_file, runner.cpp:291-297."""
    L = load_library()
    n = ctypes.c_int()
    _check(L.sdns_parse_bench_matrix_file(os.fsencode(path), None, 0, ctypes.byref(n)))
    arr = (_BenchEntry * max(1, n.value))()
    _check(L.sdns_parse_bench_matrix_file(os.fsencode(path), arr, n.value, ctypes.byref(n)))
    return _entries(arr, n.value)


def _c_entries(entries):
    arr = (_BenchEntry * max(1, len(entries)))()
    for i, e in enumerate(entries):
        if e.decomp not in _DECOMP:
            raise ConfigError(f"unknown decomposition '{e.decomp}' (expected slab|pencil)")
        arr[i] = _BenchEntry(e.n, _DECOMP[e.decomp], e.p, e.p1, e.p2)
    return arr


def bench(entries: List[BenchEntry], steps: int,
          opts: Optional[RunOptions] = None) -> List[BenchRow]:
    """bench(), runner.cpp:375-397: per entry the Taylor-Green case, 5 warm-up
    steps, then `steps` timed steps (fused RK4 + projection) between barriers."""
    L = load_library()
    o = (opts or RunOptions()).to_c()
    arr = _c_entries(entries)
    rows = (_BenchRow * max(1, len(entries)))()
    _check(L.sdns_bench(arr, len(entries), steps, ctypes.byref(o), rows))
    return [BenchRow(BenchEntry(r.entry.n, _DECOMP_NAME[r.entry.decomp], r.entry.p, r.entry.p1,
                                r.entry.p2), r.nodes_per_rank, r.sec_per_step,
                     r.status.decode()) for r in rows[:len(entries)]]


def write_bench_csv(path: str, rows: List[BenchRow]):
    """write_bench_csv, runner.cpp:399-414."""
    arr = (_BenchRow * max(1, len(rows)))()
    for i, r in enumerate(rows):
        e = r.entry
        arr[i] = _BenchRow(_BenchEntry(e.n, _DECOMP[e.decomp], e.p, e.p1, e.p2),
                           r.nodes_per_rank, r.sec_per_step, r.status.encode())
    _check(load_library().sdns_write_bench_csv(os.fsencode(path), arr, len(rows)))


def write_diagnostics_csv(path: str, samples, shells: int):
    """write_diagnostics_csv, runner.cpp:215-231; samples = [(step, FlowStats)]."""
    steps = np.array([s for s, _ in samples], dtype=np.int64)
    rows = np.array([[f.t, f.energy, f.enstrophy, f.dissipation, f.divergence_max,
                      *list(f.spectrum)] for _, f in samples], dtype=np.float64).reshape(-1)
    _check(load_library().sdns_write_diagnostics_csv(os.fsencode(path), _ptr(steps), _ptr(rows),
                                                     len(samples), shells))


def write_manifest(path: str, result: RunResult):
    """write_manifest, runner.cpp:233-247."""
    r = _RunResult()
    r.backend = result.backend.encode()
    r.status = result.status.encode()
    r.steps = result.steps
    r.step_min_s = result.timing["min_s"]
    r.step_mean_s = result.timing["mean_s"]
    r.step_max_s = result.timing["max_s"]
    r.timed_steps = result.timing["timed_steps"]
    r.csv_path = result.csv_path.encode()
    r.checkpoint_path = result.checkpoint_path.encode()
    c = result.cfg.to_c()
    _check(load_library().sdns_write_manifest(os.fsencode(path), ctypes.byref(c),
                                              result.cfg.initial_case.encode(), ctypes.byref(r)))


@dataclass
class CriterionResult:
    """CriterionResult, proj/core/include/sdns/verification.hpp:9-15."""
    index: int
    name: str
    passed: bool
    detail: str
    seconds: float


def run_acceptance_suite(device: int = 0, verbose: bool = True) -> List[CriterionResult]:
    """run_acceptance_suite, verification.cpp:548-614, on the device pipeline."""
    arr = (_CriterionResult * 9)()
    ok = ctypes.c_int()
    _check(load_library().sdns_acceptance_suite(device, 1 if verbose else 0, arr,
                                                ctypes.byref(ok)))
    return [CriterionResult(r.index, r.name.decode(), bool(r.passed), r.detail.decode(),
                            r.seconds) for r in arr]
