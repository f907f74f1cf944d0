#!/usr/bin/env python
"""Benchmark of the B200-native RK4 step (BASELINE.json metric).

Workload (default): BASELINE configs[2] -- seeded isotropic field at n = 512^3
fp64, nu = 5e-4, dt = 5e-4, slab decomposition along x over N GPUs (N = 1
fits one B200: ~21 GB). `--n 1024 --decomp pencil` is configs[3] (1024^3,
pencil 2x4 at 8 GPUs; `--decomp slab` for its slab 1x8 comparison). One
"step" = one classical RK4 step (4 fused RHS evaluations) plus the post-step
projection, exactly the reference's bench step
(proj/core/src/runner.cpp:356-359).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--size 512]
                  [--decomp slab|pencil] [--p1 P1 --p2 P2]
  python bench.py --gpus 2          # re-launches itself under torch.distributed.run
  python bench.py --impl reference  # the reference C++ solver on host cores

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback
NVL_FALLBACK = 900.0   # GB/s per direction, NVLink 5 spec (no measured figure)
NU_DT = {64: (0.01, 0.01), 256: (1e-3, 1e-3), 512: (5e-4, 5e-4), 1024: (2.5e-4, 2.5e-4)}


def peaks():
    """(HBM GB/s, its source, NVLink GB/s per direction, its source)."""
    hbm, hsrc = HBM_FALLBACK, "fallback (B200_PROFILING.md)"
    nvl, nsrc = NVL_FALLBACK, "fallback: NVLink 5 spec 900 GB/s per direction (no measured figure)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        hbm, hsrc = float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        for k in ("nvlink_gbs", "nvlink_gbs_per_dir", "p2p_gbs"):
            if k in d:
                nvl, nsrc = float(d[k]), f"measured (MEASURED_PEAKS.json {k})"
                break
    except Exception:  # noqa: BLE001
        pass
    return hbm, hsrc, nvl, nsrc


def spectral_bytes(n, p):
    """C = one half-spectrum complex128 component per rank."""
    return 16.0 * n * n * (n // 2 + 1) / p


def a2a_fraction(decomp, p, p1, p2):
    """Share of a rank's transposed bytes that leave the GPU."""
    if p <= 1:
        return 0.0
    if decomp == "slab":
        return (p - 1) / p
    return (p1 - 1) / p1 + (p2 - 1) / p2


def step_roofline(n, decomp, p, p1, p2, hbm_gbs, nvl_gbs):
    """BASELINE.md §3 / SURVEY §8(d): per GPU and step, HBM = 213 C/p bytes,
    all-to-all egress = 36 (C/p) f; roofline = the slower of the two."""
    C = spectral_bytes(n, p)
    hbm = 213.0 * C
    a2a = 36.0 * C * a2a_fraction(decomp, p, p1, p2)
    t_h = hbm / hbm_gbs / 1e6
    t_n = a2a / nvl_gbs / 1e6
    return {"hbm_bytes_per_step": hbm, "a2a_bytes_per_step": a2a, "t_hbm_ms": t_h,
            "t_nvlink_ms": t_n, "roofline_ms": max(t_h, t_n),
            "bound": "nvlink" if t_n > t_h else "hbm"}


# Algorithmic HBM bytes per launch, in units of C.
PASS_BYTES_C = {"x_inv_curl": 8, "y_inv": 11, "z_fused": 9, "y_fwd": 6, "x_fwd_fft": 6, "x_fwd_rk0": 12,
                "x_fwd_rk12": 18, "x_fwd_rk3": 21, "x_fwd_tail": 12}


def pass_a2a_c(name, decomp, p, p1, p2):
    """Fields a pass stores into peers' buffers (peer-direct transposes,
    DESIGN §5) times the fraction that leaves the GPU, in units of C."""
    if p <= 1:
        return 0.0
    if decomp == "slab":
        f = (p - 1) / p
        return {"x_inv_curl": 5 * f, "y_fwd": 3 * f}.get(name, 0.0)
    f1, f2 = (p1 - 1) / p1, (p2 - 1) / p2
    return {"x_inv_curl": 5 * f1, "y_inv": 6 * f2, "z_fused": 3 * f2, "y_fwd": 3 * f1}.get(name, 0.0)


def default_grid(world):
    """Pencil grids of the reference's bench matrix (config_file.cpp:51-61)."""
    return {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}.get(world, (1, world))


class ClockSampler:
    """Samples nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def pow2_floor(x):
    p = 1
    while p * 2 <= x:
        p *= 2
    return p


def resolve(args, world):
    """Decomposition of the GPU job and the config dict both arms print."""
    n = args.n
    decomp = args.decomp or "slab"
    p1, p2 = 1, 1
    if decomp == "pencil":
        p1, p2 = (args.p1, args.p2) if args.p1 and args.p2 else default_grid(world)
        if p1 * p2 != world:
            raise SystemExit(f"pencil grid {p1}x{p2} does not match {world} ranks")
    nu, dt = NU_DT.get(n, (5e-4, 5e-4))
    if n == 1024:
        wl = f"configs[3]: isotropic 1024^3 fp64, nu={nu:g}, dt={dt:g}, " + (
            f"pencil {p1}x{p2}" if decomp == "pencil" else f"slab 1x{world}")
    elif n == 512:
        wl = f"configs[2]: isotropic 512^3 fp64, nu={nu:g}, dt={dt:g}, " + (
            f"pencil {p1}x{p2}" if decomp == "pencil" else f"slab x {world}")
    else:
        wl = f"isotropic {n}^3 fp64, nu={nu:g}, dt={dt:g}, {decomp} x {world}"
    C = spectral_bytes(n, world)
    config = {"workload": wl, "n": n, "decomp": decomp, "p": world, "p1": p1, "p2": p2,
              "nu": nu, "dt": dt, "seed": 1607, "global_points": n**3,
              "l2": "inputs larger than L2 (u_hat alone is %.2f GB per rank)" % (3 * C / 1e9)}
    return config


def relaunch(args):
    """`bench.py --gpus N` without torchrun: re-exec under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)]
    # torch.distributed.run would read "--n" as an abbreviation of its own options
    cmd += ["--size" if a == "--n" else ("--size=" + a[4:] if a.startswith("--n=") else a)
            for a in sys.argv[1:]]
    return subprocess.call(cmd)


# --- reference arm -------------------------------------------------------------

REF_BUDGET_S = 300.0


def run_reference(args):
    """The UNMODIFIED reference (oracle/_ref: proj/core compiled against the
    FFTW shim) timed on the host's cores with the reference's own bench method
    (rk4_step + project per step between barriers, runner.cpp:336-373), on the
    same seeded isotropic input (restated in the oracle), threads-as-ranks."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    config = resolve(args, world)
    n, nu, dt = config["n"], config["nu"], config["dt"]
    from oracle import ref
    threads = cpu_threads()
    p = min(pow2_floor(max(1, threads)), n)
    base = {"metric": "RK4 steps/s", "unit": "steps/s", "impl": "reference", "n_gpus": world,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded isotropic field, BASELINE configs[2] construction)",
            "config": config}
    if not ref.available():
        print(json.dumps({**base, "unavailable": "oracle/_ref/libsdns_ref.so not built"}))
        return
    if n > 512:
        # ~36 C of host RAM (310 GB at 1024^3): beyond the box
        print(json.dumps({**base, "value": None, "steps": 0, "warmup": 0,
                          "unavailable": f"reference at {n}^3 needs ~{36 * spectral_bytes(n, 1) / 1e9:.0f} GB "
                                         "of host RAM (SURVEY §8(d))"}))
        return
    uh0 = ref.iso_init(n, seed=1607)
    # size the run: one compute_rhs (a quarter of a step's transforms) probes
    probe = ref.time_units(n, p=p, nu=nu, dt=dt, warmup=0, units=1, unit="rhs", uhat0=uh0)
    est = 4.2 * probe
    warm, steps = args.warmup, args.steps
    if (warm + steps) * est > REF_BUDGET_S:
        warm = min(warm, 1)
        steps = max(1, min(steps, int((REF_BUDGET_S - warm * est) / est)))
    sec = ref.time_units(n, p=p, nu=nu, dt=dt, warmup=warm, units=steps, unit="step", uhat0=uh0)
    value = 1.0 / sec
    line = {**base, "value": value, "steps": steps, "warmup": warm, "ms_per_step": sec * 1e3,
            "requested": {"steps": args.steps, "warmup": args.warmup},
            "ns_per_gridpoint_step": sec * 1e9 / n**3,
            "cpu_baseline": {"value": value, "unit": "steps/s", "cores": p, "kind": "reference",
                             "sample": f"{steps} whole RK4 steps (rk4_step + project) at {n}^3 on the "
                                       f"iso field after {warm} warm-up step(s), {p} threads-as-ranks "
                                       "(slab), the reference's bench method (runner.cpp:336-373)",
                             "fft": "self-written FFTW guru64 shim (no libfftw3 in image)"},
            "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    if not args.no_cpu1:
        s1 = ref.time_units(n, p=1, nu=nu, dt=dt, warmup=0, units=1, unit="rhs", uhat0=uh0)
        line["cpu_p1"] = {"sec_per_rhs": s1, "est_sec_per_step": 4 * s1, "cores": 1,
                          "sample": f"one compute_rhs at {n}^3 on 1 thread (p_cpu = 1), "
                                    "x4 for a step (RK4 vector updates excluded)"}
    try:
        line["host"] = {"threads": threads, "nproc": os.cpu_count(),
                        "mem_gb": os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9}
    except Exception:  # noqa: BLE001
        pass
    print(json.dumps(line), flush=True)


def cpu_baseline_leg(config):
    """Our arm's cpu_baseline (rank 0, N = 1): whole reference steps on the
    same iso input, bounded (1 warm-up + 2 timed steps at 512^3, ~30 s)."""
    from oracle import ref
    n, nu, dt = config["n"], config["nu"], config["dt"]
    if not ref.available() or n > 512:
        raise RuntimeError("reference unavailable at this size")
    p = min(pow2_floor(cpu_threads()), n)
    uh0 = ref.iso_init(n, seed=1607)
    steps = 2 if n >= 512 else 5
    sec = ref.time_units(n, p=p, nu=nu, dt=dt, warmup=1, units=steps, unit="step", uhat0=uh0)
    return {"value": 1.0 / sec, "unit": "steps/s", "cores": p, "kind": "reference",
            "sample": f"{steps} whole RK4 steps (rk4_step + project) at {n}^3 on the iso field "
                      f"after 1 warm-up step, {p} threads-as-ranks (slab)",
            "fft": "self-written FFTW guru64 shim (no libfftw3 in image)"}


# --- our arm -------------------------------------------------------------------

def other_configs(S, ctx, peak):
    """The other BASELINE configs, measured quickly beside the headline line
    (informational; each on seeded synthetic fields of the config's shape):
    config 5 round trip at 512^3 (3 comps) against its HBM roofline
    3*(2R + 10C) bytes, config 1 (TG 64^3, 100 steps, E and Z
    every step) and config 2 (iso 256^3, 50 steps)."""
    import numpy as np
    import torch

    out = {}
    n = ctx.cfg.n
    stream = torch.cuda.ExternalStream(ctx.stream)
    fft = S.DistributedFFT(ctx)
    ur, ub, fu = ctx.real_field(), ctx.real_field(), ctx.spectral_field()
    ur.upload(np.random.default_rng(42 + n).uniform(-1.0, 1.0, (3, n, n, n)))
    fft.forward(ur, fu)
    fft.inverse(fu, ub)
    ctx.sync()
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fft.forward(ur, fu)
        fft.inverse(fu, ub)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    R, C = 8.0 * n**3, spectral_bytes(n, 1)
    rt_bytes = 3 * (2 * R + 10 * C)
    out["config5_round_trip_512"] = {
        "ms": ms, "roofline_ms": rt_bytes / peak / 1e6, "frac": rt_bytes / (ms * 1e-3) / 1e9 / peak,
        "rel_l2": S.l2_diff(ctx, ub, ur) / S.l2_diff(ctx, ur, ctx.real_field())}
    for f in (ur, ub, fu):
        f.free()
    for key, (m, steps, every, nu, dt, tg) in {
            "config1_tg64_sampled": (64, 100, 1, 0.01, 0.01, True),
            "config2_iso256": (256, 50, 50, 1e-3, 1e-3, False)}.items():
        cfg = S.SolverConfig(n=m, nu=nu, dt=dt, t_end=steps * dt, out_every=every)
        with S.Context(cfg) as c:
            lo = c.layout
            if tg:
                x = 2 * np.pi * np.arange(m) / m
                X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
                u = np.stack([np.sin(X) * np.cos(Y) * np.cos(Z),
                              -np.cos(X) * np.sin(Y) * np.cos(Z), np.zeros_like(X)])
                uh = c.spectral_field()
                S.DistributedFFT(c).forward(c.real_field().upload(u), uh)
                S.project(c, uh)
            else:
                uh = c.spectral_field().upload(S.iso_init(m, lo, seed=1607))
            st = S.Rk4State(c)
            rows = []
            hook = lambda k, t: rows.append(S.collect_stats(c, st.u_hat, nu, t))  # noqa: E731
            st.set(uh)
            st.advance(hook)  # warm (captures the step graph)
            st.set(uh)
            rows.clear()
            c.sync()
            t0 = time.perf_counter()
            st.advance(hook)
            c.sync()
            sec = time.perf_counter() - t0
            rf = step_roofline(m, "slab", 1, 1, 1, peak, NVL_FALLBACK)
            out[key] = {"steps_per_s": steps / sec, "ms_per_step": sec / steps * 1e3,
                        "step_roofline_frac": rf["roofline_ms"] / (sec / steps * 1e3),
                        "samples": len(rows), "energy_last": rows[-1].energy}
            st.close()
    return out


def other_configs_1024(S, peak):
    """n = 1024 on one GPU (informational): config 5's 3-component round trip
    (rfftn + irfftn) against 3*(2R + 10C) bytes, and one RK4 step of the
    configs[3] field (state + work ~155 GB) against the 213 C step roofline.
    The round trip's real input is the inverse transform of that field
    (timing is data-independent; its parity is pinned by the tests)."""
    import torch

    out = {}
    n = 1024
    R, C = 8.0 * n**3, spectral_bytes(n, 1)
    nu, dt = NU_DT[n]
    lo = S.build_layout(S.SolverConfig(n=n), 0)
    t0 = time.time()
    uh0 = S.iso_init(n, lo, seed=1607)
    out["iso_init_s"] = time.time() - t0
    with S.Context(S.SolverConfig(n=n)) as c:
        stream = torch.cuda.ExternalStream(c.stream)
        fft = S.DistributedFFT(c)
        ur, ub, fu = c.real_field(), c.real_field(), c.spectral_field()
        fu.upload(uh0)
        fft.inverse(fu, ur)
        fft.forward(ur, fu)
        fft.inverse(fu, ub)
        c.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(2):
            fft.forward(ur, fu)
            fft.inverse(fu, ub)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        rt = 3 * (2 * R + 10 * C)
        out["config5_round_trip_1024"] = {
            "ms": ms, "roofline_ms": rt / peak / 1e6, "frac": rt / (ms * 1e-3) / 1e9 / peak,
            "rel_l2": S.l2_diff(c, ub, ur) / S.l2_diff(c, ur, c.real_field())}
        for f in (ur, ub, fu):
            f.free()
    with S.Context(S.SolverConfig(n=n, nu=nu, dt=dt, t_end=dt)) as c:
        stream = torch.cuda.ExternalStream(c.stream)
        st = S.Rk4State(c)
        u = c.spectral_field().upload(uh0)
        st.set(u)
        u.free()
        del uh0
        st.rk4_step(dt, post_project=True, check=True)  # warm
        c.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(2):
            st.rk4_step(dt, post_project=True, check=False)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 2
        rf = step_roofline(n, "slab", 1, 1, 1, peak, NVL_FALLBACK)
        out["config4_size_step_1024_one_gpu"] = {
            "ms_per_step": ms, "roofline_ms": rf["roofline_ms"], "frac": rf["roofline_ms"] / ms}
        st.close()
    return out


def run_ours(args):
    import numpy as np
    import torch

    import paper_1607_00850_b200 as S

    if args.lib:
        S.use_library(args.lib)
    if args.opt:  # A/B only: the defaults are what the line reports
        S.set_default_options(**{k: int(v) for k, v in (kv.split("=") for kv in args.opt.split(","))})
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    config = resolve(args, world)
    n, nu, dt = config["n"], config["nu"], config["dt"]
    decomp, p1, p2 = config["decomp"], config["p1"], config["p2"]
    # --transport host (a harness check, not a bench): ranks share the GPUs
    # present round-robin over the host-callback transport (gloo all-gathers,
    # CUDA IPC), e.g. 2 ranks on one GPU
    device = local if args.transport == "nccl" else local % torch.cuda.device_count()
    torch.cuda.set_device(device)
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist
        if args.transport == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # the communicator log names every rank
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")  # ... at init only
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
            uid = [S.Comm.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = S.Comm.nccl(uid[0], world, rank, device)
            # the deadline catches dead peers, not slow ones (host-side setup
            # such as the 1024^3 iso field can desynchronise ranks by minutes)
            comm.set_timeout(900.0)
        else:
            dist.init_process_group("gloo")
            red_dev = "cpu"

            def allgather(data, group):
                t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
                parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
                dist.all_gather(parts, t, group=group)
                return [x.numpy().tobytes() for x in parts]
            comm = S.Comm.host(world, rank, device, allgather, new_group=dist.new_group)
            comm.set_timeout(900.0)
    else:
        comm = S.Comm.loopback()

    cfg = S.SolverConfig(n=n, decomp=decomp, p=world, p1=p1, p2=p2, nu=nu, dt=dt,
                         t_end=args.steps * dt)
    ctx = S.Context(cfg, rank=rank, device=device, comm=comm)
    transposes = ctx.transposes if world > 1 else "none (p = 1)"
    lo = ctx.layout
    t0 = time.time()
    uh0 = S.iso_init(n, lo, seed=1607)
    init_s = time.time() - t0
    state = S.Rk4State(ctx)
    u = ctx.spectral_field().upload(uh0)
    state.set(u)
    u.free()
    del uh0
    stream = torch.cuda.ExternalStream(ctx.stream)
    if dist is not None:
        dist.barrier()  # every rank's host setup done before the first collective

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        state.rk4_step(dt, post_project=True, check=True)
    ctx.sync()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.timing(True)
    with ClockSampler(device) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            state.rk4_step(dt, post_project=True, check=False)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    passes = ctx.timing_read()
    ctx.timing(False)
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    finite = state.rk4_step(dt, post_project=True, check=True)
    stats = S.collect_stats(ctx, state.u_hat, nu)

    # --- e2e: reference-facing host-buffer API (pinned host u_hat in/out) ---
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    shape = (3,) + tuple(lo.spec_shape)
    nbytes = int(np.prod(shape)) * 16
    pinned = S.load_library().sdns_host_alloc(nbytes)
    hbuf = np.ctypeslib.as_array((S.ctypes.c_double * (nbytes // 8)).from_address(pinned))
    hbuf[:] = state.u_hat.download().view(np.float64).ravel()
    hview = hbuf.view(np.complex128).reshape(shape)
    state.step_host(hview, dt, 1)  # warm
    barrier()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        state.step_host(hview, dt, 1)
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - te) / e2e_steps)
    S.load_library().sdns_host_free(pinned)

    if rank != 0:
        state.close()
        ctx.close()
        if dist is not None:
            dist.barrier()  # rank 0 has printed its line: no log output can cut into it
            dist.destroy_process_group()
        return

    hbm_peak, hbm_src, nvl_peak, nvl_src = peaks()
    C = spectral_bytes(n, world)
    ncu_bytes = {}
    tfile = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if world == 1 and os.path.exists(tfile):
        try:
            with open(tfile) as f:
                ncu_bytes = json.load(f).get(str(n), {})
        except Exception:  # noqa: BLE001
            ncu_bytes = {}
    per_pass = {k: {"avg_ms": v[0] / v[1], "launches": v[1], "share": None}
                for k, v in passes.items() if v[1] > 0}
    kernel_total = sum(v[0] for k, v in passes.items() if not k.startswith("a2a"))
    for k, v in passes.items():
        if v[1] > 0:
            per_pass[k]["share"] = v[0] / max(kernel_total, 1e-30) if not k.startswith("a2a") else None
            if k in PASS_BYTES_C:
                per_pass[k]["hbm_frac_alg"] = PASS_BYTES_C[k] * C / (v[0] / v[1] * 1e-3) / 1e9 / hbm_peak
            if k in ncu_bytes:  # DRAM bytes per launch (ncu) / live launch time
                gbs = ncu_bytes[k] / (v[0] / v[1] * 1e-3) / 1e9
                per_pass[k]["dram_gbs"] = gbs
                per_pass[k]["dram_frac"] = gbs / hbm_peak
    launches = sum(v[1] for k, v in passes.items() if not k.startswith("a2a"))
    dom = max((k for k in per_pass if k in PASS_BYTES_C), key=lambda k: passes[k][0])
    dom_ms = per_pass[dom]["avg_ms"]
    dom_bytes = PASS_BYTES_C[dom] * C
    dom_nvl = pass_a2a_c(dom, decomp, world, p1, p2) * C
    t_hbm, t_nvl = dom_bytes / hbm_peak, dom_nvl / nvl_peak
    if t_nvl > t_hbm:
        roof = {"bound": "nvlink", "achieved": dom_nvl / (dom_ms * 1e-3) / 1e9, "peak": nvl_peak,
                "unit": "GB/s", "peak_source": nvl_src, "algorithmic_bytes_per_launch": dom_nvl,
                "hbm_bytes_per_launch": dom_bytes}
    else:
        roof = {"bound": "hbm", "achieved": dom_bytes / (dom_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "peak_source": hbm_src, "algorithmic_bytes_per_launch": dom_bytes,
                "nvlink_bytes_per_launch": dom_nvl}
    roof["frac"] = roof["achieved"] / roof["peak"]
    roof["traffic"] = ncu_bytes.get(dom)
    roof["kernel"] = dom
    sr = step_roofline(n, decomp, world, p1, p2, hbm_peak, nvl_peak)
    sr["frac"] = sr["roofline_ms"] / ms
    sr["achieved_hbm_gbs"] = sr["hbm_bytes_per_step"] / (ms * 1e-3) / 1e9
    sr["peaks"] = {"hbm_gbs": hbm_peak, "hbm_source": hbm_src, "nvlink_gbs": nvl_peak,
                   "nvlink_source": nvl_src}
    value = 1e3 / ms  # steps/s of the whole job (strong scaling: one problem on N GPUs)
    line = {
        "metric": "RK4 steps/s", "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded isotropic field, BASELINE configs[2] construction)",
        "config": config,
        "transposes": transposes,
        "transport": args.transport if world > 1 else "loopback",
        "ns_per_gridpoint_step": ms * 1e6 / n**3,
        "roofline": roof,
        "step_roofline": sr,
        "passes": per_pass,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "e2e": {"value": 1.0 / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": nbytes * world,
                "d2h_bytes_per_step": nbytes * world,
                "api": "sdns_rk4_step_host (host u_hat in/out, pinned)"},
        "check": {"finite": bool(finite), "energy": stats.energy, "enstrophy": stats.enstrophy,
                  "div_max": stats.divergence_max},
        "init_s": init_s,
    }
    if world == 1 and n == 512 and not args.no_other_configs:
        state.close()
        try:
            line["other_configs"] = other_configs(S, ctx, hbm_peak)
        except Exception as e:  # noqa: BLE001  (informational lines never cost the headline)
            line["other_configs"] = {"error": f"not run: {e}"}
    state.close()
    ctx.close()
    if world == 1 and n == 512 and not args.no_other_configs and not args.no_1024:
        try:
            line.setdefault("other_configs", {}).update(other_configs_1024(S, hbm_peak))
        except Exception as e:  # noqa: BLE001
            line.setdefault("other_configs", {})["n1024"] = f"not run: {e}"
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_leg(config)
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "steps/s", "cores": 0,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--size", "--n", dest="n", type=int, default=512,
                    help="grid points per axis (512: configs[2], 1024: configs[3])")
    ap.add_argument("--decomp", choices=["slab", "pencil"], default=None)
    ap.add_argument("--p1", type=int, default=0)
    ap.add_argument("--p2", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu1", action="store_true", help="reference arm: skip the p_cpu = 1 sample")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--no-1024", action="store_true", help="skip the n = 1024 one-GPU lines")
    ap.add_argument("--lib", default=None, help="A/B: another build of the product library")
    ap.add_argument("--opt", default="", help="A/B: context options, e.g. p1_single=1,plain_layout=1")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="N > 1: NCCL (one GPU per rank) or the host-callback transport "
                         "(harness check; ranks may share a GPU)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
