"""One rank of the stalled-peer test (tests/test_gpu_multiprocess.py): slab
p = 2 over the host-callback transport with a 5 s gloo timeout. Rank 1 builds
its context and then stalls (never enters another collective); rank 0 runs
RK4 steps, must see TimeoutError (the reference's collective deadline,
transport.cpp:105-140), and every later collective on the communicator must
fail fast with the same error. Rank 0 writes <out>/stall.txt.

    python tests/helpers/mp_stall_worker.py <rank> <port> <out>"""
import datetime
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1607_00850_b200 as S  # noqa: E402


def main():
    rank, port, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=2, timeout=datetime.timedelta(seconds=5))

    def allgather(data: bytes, group):
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(parts, t, group=group)
        return [p.numpy().tobytes() for p in parts]

    comm = S.Comm.host(2, rank, 0, allgather).set_timeout(10.0)
    n = 16
    cfg = S.SolverConfig(n=n, p=2, nu=1e-3, dt=1e-3, t_end=1e-3)
    ctx = S.Context(cfg, rank=rank, device=0, comm=comm)
    lo = ctx.layout
    uh0 = S.iso_init(n, lo, seed=9)
    st = S.Rk4State(ctx)
    st.set(ctx.spectral_field().upload(uh0))
    st.rk4_step(1e-3)  # both ranks: a healthy step first
    if rank == 1:
        time.sleep(120)  # stalls: the test kills this process
        return
    lines = []
    t0 = time.time()
    try:
        for _ in range(100):
            st.rk4_step(1e-3)
        lines.append("no error")
    except S.TimeoutError as e:
        lines.append(f"TimeoutError after {time.time() - t0:.1f} s: {e}")
    except Exception as e:  # noqa: BLE001
        lines.append(f"{type(e).__name__}: {e}")
    t1 = time.time()
    try:
        comm.barrier()
        lines.append("barrier: no error")
    except S.TimeoutError as e:
        lines.append(f"barrier TimeoutError after {time.time() - t1:.1f} s: {e}")
    except Exception as e:  # noqa: BLE001
        lines.append(f"barrier {type(e).__name__}: {e}")
    with open(os.path.join(out, "stall.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    os._exit(0)  # the communicator is dead; skip teardown collectives


if __name__ == "__main__":
    main()
