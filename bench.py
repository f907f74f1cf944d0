#!/usr/bin/env python
"""Benchmark of the B200-native RK4 step (BASELINE.json metric).

Workload: BASELINE configs[2] -- seeded isotropic field at n = 512^3 fp64,
nu = 5e-4, dt = 5e-4, slab decomposition along x over N GPUs (N = 1 fits one
B200: ~21 GB). One "step" = one classical RK4 step (4 fused RHS evaluations)
plus the post-step projection, exactly the reference's bench step
(proj/core/src/runner.cpp:356-359).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 512]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference   # the reference C++ solver on host cores

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return HBM_FALLBACK, "fallback"


def spectral_bytes(n, p):
    """C = one half-spectrum complex128 component per rank."""
    return 16.0 * n * n * (n // 2 + 1) / p


# Algorithmic HBM bytes per launch, in units of C.
PASS_BYTES_C = {"x_inv_curl": 8, "y_inv": 11, "z_fused": 9, "y_fwd": 6, "x_fwd_fft": 6, "x_fwd_rk0": 12,
                "x_fwd_rk12": 18, "x_fwd_rk3": 21, "x_fwd_tail": 12}
STEP_BYTES_C = 213


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
                 "--format=csv,noheader,nounits", "-lms", "200"],
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


def reference_timing(n, nu, dt, warmup, units, unit, threads):
    """Times the UNMODIFIED reference (oracle/_ref) on `threads` host cores."""
    from oracle import ref
    if not ref.available():
        raise RuntimeError("oracle/_ref/libsdns_ref.so not built")
    p = min(pow2_floor(max(1, threads)), n)
    sec = ref.time_units(n, p=p, nu=nu, dt=dt, warmup=warmup, units=units, unit=unit)
    return sec, p


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n, nu, dt = args.n, 5e-4, 5e-4
    threads = cpu_threads()
    # Bounded sample per step: one compute_rhs (1/4 of the RK4 step's RHS
    # work) at the full size, scaled to steps/s by x4 -- the step's 36 FFTs
    # are 4 identical RHS evaluations; RK4 updates are excluded (optimistic
    # for the reference).
    unit = "rhs" if n >= 256 else "step"
    # One untimed unit sizes the run: K units are timed, capped so the whole
    # reference arm stays within a few minutes of host time.
    warm_s, p = reference_timing(n, nu, dt, 0, 1, unit, threads)
    units = max(1, min(args.steps, int(150.0 / max(warm_s, 1e-3))))
    sec, p = reference_timing(n, nu, dt, 0, units, unit, threads)
    step_s = sec * (4.0 if unit == "rhs" else 1.0)
    value = 1.0 / step_s
    line = {
        "metric": "RK4 steps/s", "value": value, "unit": "steps/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference Taylor-Green init)",
        "config": {"workload": f"configs[2]: iso/TG {n}^3 fp64 RK4, slab", "n": n,
                   "decomp": "slab", "p_cpu": p},
        "ns_per_gridpoint_step": step_s * 1e9 / n**3,
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": p, "kind": "reference",
                         "sample": (f"{units} x one compute_rhs at {n}^3 (x4 per step), "
                                    f"after 1 untimed unit" if unit == "rhs"
                                    else f"{units} RK4 steps at {n}^3"),
                         "fft": "self-written FFTW guru64 shim (no libfftw3 in image)"},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
            out[key] = {"steps_per_s": steps / sec, "ms_per_step": sec / steps * 1e3,
                        "samples": len(rows), "energy_last": rows[-1].energy}
            st.close()
    return out


def run_ours(args):
    import numpy as np
    import torch

    import paper_1607_00850_b200 as S

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
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
            dist.init_process_group("nccl", device_id=torch.device("cuda", device))
            uid = [S.Comm.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = S.Comm.nccl(uid[0], world, rank, device)
        else:
            dist.init_process_group("gloo")
            red_dev = "cpu"

            def allgather(data, group):
                t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
                parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
                dist.all_gather(parts, t, group=group)
                return [x.numpy().tobytes() for x in parts]
            comm = S.Comm.host(world, rank, device, allgather, new_group=dist.new_group)
    else:
        comm = S.Comm.loopback()
    local = device

    n, nu, dt = args.n, 5e-4, 5e-4
    cfg = S.SolverConfig(n=n, p=world, nu=nu, dt=dt, t_end=args.steps * dt)
    ctx = S.Context(cfg, rank=rank, device=local, comm=comm)
    transposes = ctx.transposes if world > 1 else "none (p = 1)"
    lo = ctx.layout
    t0 = time.time()
    uh0 = S.iso_init(n, lo, seed=1607)
    init_s = time.time() - t0
    state = S.Rk4State(ctx)
    u = ctx.spectral_field().upload(uh0)
    state.set(u)
    u.free()
    stream = torch.cuda.ExternalStream(ctx.stream)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        state.rk4_step(dt, post_project=True, check=True)
    ctx.sync()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.timing(True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            state.rk4_step(dt, post_project=True, check=False)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    passes = ctx.timing_read()
    ctx.timing(False)
    ms = ev0.elapsed_time(ev1) / args.steps
    finite = state.rk4_step(dt, post_project=True, check=True)
    stats = S.collect_stats(ctx, state.u_hat, nu)
    if dist is not None:
        t = torch.tensor([ms], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # --- e2e: reference-facing host-buffer API (pinned host u_hat in/out) ---
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    host = np.empty((3,) + tuple(lo.spec_shape), dtype=np.complex128)
    nbytes = host.nbytes
    pinned = S.load_library().sdns_host_alloc(nbytes)
    hbuf = np.ctypeslib.as_array((S.ctypes.c_double * (nbytes // 8)).from_address(pinned))
    hbuf[:] = state.u_hat.download().view(np.float64).ravel()
    hview = hbuf.view(np.complex128).reshape(host.shape)
    state.step_host(hview, dt, 1)  # warm
    barrier()
    te = time.perf_counter()
    for _ in range(e2e_steps):
        state.step_host(hview, dt, 1)
    barrier()
    e2e_s = (time.perf_counter() - te) / e2e_steps
    if dist is not None:
        t = torch.tensor([e2e_s], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    S.load_library().sdns_host_free(pinned)

    if rank != 0:
        state.close()
        ctx.close()
        if dist is not None:
            dist.destroy_process_group()
        return

    peak, peak_kind = peaks()
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
            if k in ncu_bytes:  # DRAM bytes per launch (ncu) / live launch time
                gbs = ncu_bytes[k] / (v[0] / v[1] * 1e-3) / 1e9
                per_pass[k]["dram_gbs"] = gbs
                per_pass[k]["dram_frac"] = gbs / peak
    launches = sum(v[1] for k, v in passes.items() if not k.startswith("a2a"))
    dom = max((k for k in per_pass if k in PASS_BYTES_C), key=lambda k: passes[k][0])
    dom_ms = per_pass[dom]["avg_ms"]
    dom_bytes = PASS_BYTES_C[dom] * C
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = ncu_bytes.get(dom)
    step_bytes = STEP_BYTES_C * C
    step_gbs = step_bytes / (ms * 1e-3) / 1e9
    value = 1e3 / ms  # steps/s of the whole job (strong scaling: one problem on N GPUs)
    line = {
        "metric": "RK4 steps/s", "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded isotropic field, BASELINE configs[2] construction)",
        "config": {"workload": f"configs[2]: isotropic {n}^3 fp64, nu=5e-4, dt=5e-4, slab x {world}",
                   "n": n, "decomp": "slab", "p": world, "global_points": n**3,
                   "transposes": transposes, "transport": args.transport if world > 1 else "loopback",
                   "l2": "inputs larger than L2 (u_hat alone is %.1f GB per rank)" % (3 * C / 1e9)},
        "ns_per_gridpoint_step": ms * 1e6 / n**3,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": dom,
                     "algorithmic_bytes_per_launch": dom_bytes,
                     "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)"},
        "step_roofline": {"bytes_per_step": step_bytes, "achieved_gbs": step_gbs,
                          "frac": step_gbs / peak, "roofline_ms": step_bytes / peak / 1e6},
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
        line["other_configs"] = other_configs(S, ctx, peak)
    state.close()
    ctx.close()
    if world == 1 and not args.no_cpu_baseline:
        try:
            threads = cpu_threads()
            unit = "rhs" if n >= 256 else "step"
            sec, p = reference_timing(n, nu, dt, 0, 1, unit, threads)
            step_s = sec * (4.0 if unit == "rhs" else 1.0)
            line["cpu_baseline"] = {
                "value": 1.0 / step_s, "unit": "steps/s", "cores": p, "kind": "reference",
                "sample": (f"one compute_rhs at {n}^3 on {p} threads-as-ranks, x4 per RK4 step"
                           if unit == "rhs" else f"one RK4 step at {n}^3"),
                "fft": "self-written FFTW guru64 shim (no libfftw3 in image)"}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": "steps/s", "cores": 0,
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=512)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-other-configs", action="store_true")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "host"],
                    help="N > 1: NCCL (one GPU per rank) or the host-callback transport "
                         "(harness check; ranks may share a GPU)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
