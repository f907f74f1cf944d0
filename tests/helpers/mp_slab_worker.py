"""One rank of the multi-process test (tests/test_gpu_multiprocess.py): slab
or pencil p = world over the host-callback transport (gloo all-gathers and
groups, CUDA IPC memory and events), several ranks sharing GPU 0. Saves this
rank's RHS, two-step state and stats to <out>/r<rank>.npz.

    python tests/helpers/mp_slab_worker.py <rank> <world> <port> <out> <n> [p1 p2]"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1607_00850_b200 as S  # noqa: E402

if os.environ.get("AB_LIB"):  # debugging: another build of the library
    S.use_library(os.environ["AB_LIB"])


def main():
    rank, world, port, out, n = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]),
                                 sys.argv[4], int(sys.argv[5]))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)

    def allgather(data: bytes, group):
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8)
        size = dist.get_world_size(group)
        parts = [torch.empty_like(t) for _ in range(size)]
        dist.all_gather(parts, t, group=group)
        return [p.numpy().tobytes() for p in parts]

    comm = S.Comm.host(world, rank, 0, allgather, new_group=dist.new_group)
    bc = comm.broadcast_bytes(bytes([rank + 1]) * 24, root=world - 1)
    geom = {}
    if len(sys.argv) > 7:
        geom = dict(decomp="pencil", p1=int(sys.argv[6]), p2=int(sys.argv[7]))
    cfg = S.SolverConfig(n=n, p=world, nu=1e-3, dt=1e-3, t_end=1e-3, **geom)
    with S.Context(cfg, rank=rank, device=0, comm=comm) as c:
        lo = c.layout
        uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=9)
        (s0, s1, s2), (o0, o1, o2) = lo.spec_shape, lo.spec_offset
        u = c.spectral_field().upload(uh0[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2])
        du = c.spectral_field()
        S.compute_rhs(c, u, 1e-3, du)
        st = S.Rk4State(c)
        st.set(u)
        st.rk4_step(1e-3)
        st.rk4_step(1e-3)
        uo = c.spectral_field()
        st.get(uo)
        stats = S.collect_stats(c, uo, 1e-3)
        fft = S.DistributedFFT(c)  # the API transforms fuse their transposes too
        ur = c.real_field()
        fft.inverse(uo, ur)
        fu = c.spectral_field()
        fft.forward(ur, fu)
        # checkpoints over this transport (the gathers/scatters go through the
        # host all-gather): write, then read back into a fresh field
        ck = os.path.join(out, "ck.sdns")
        S.write_checkpoint(c, ck, ur, 0.25, 7)
        back = c.real_field()
        tt, stp = S.read_checkpoint(c, ck, back)
        ck_ok = bool(np.array_equal(back.download(), ur.download())) and (tt, stp) == (0.25, 7)
        np.savez(os.path.join(out, f"r{rank}.npz"), du=du.download(), u=uo.download(), ck_ok=ck_ok,
                 ur=ur.download(), fu=fu.download(), e=stats.energy, z=stats.enstrophy,
                 transposes=c.transposes, bcast=np.frombuffer(bc, dtype=np.uint8))
        st.close()
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
