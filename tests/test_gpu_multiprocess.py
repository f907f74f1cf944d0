"""GPU: the multi-process peer-direct path (slab and pencil). Ranks are separate processes
(one CUDA context each, sharing the one GPU here) over the host-callback
transport: their buffers are mapped with CUDA IPC and the stream barriers
wait on IPC events -- the same mapping code (ipc_map_peers) the NCCL backend
uses across GPUs. One RHS and two RK4 steps must equal the single-process
result bit for bit; the checkpoint gathers and scatters run over the same
transport (its all-to-all goes through the host all-gather), and the file
is the reference's format (compared with the threads-as-ranks file)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import paper_1607_00850_b200 as S

if os.environ.get("AB_LIB"):  # debugging: another build of the library
    S.use_library(os.environ["AB_LIB"])

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "helpers", "mp_slab_worker.py")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,grid", [(2, None), (4, None), (2, (1, 2)), (4, (2, 2))])
def test_multiprocess_peer_direct_bitwise(tmp_path, world, grid):
    """slab p = 2, 4 and pencil 1x2, 2x2 (row / column sub-communicators
    split through the transport's group callback)."""
    n = 32
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    extra = [str(grid[0]), str(grid[1])] if grid else []
    procs = [subprocess.Popen([sys.executable, WORKER, str(r), str(world), str(port),
                               str(tmp_path), str(n)] + extra, env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=300)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    assert all(p.returncode == 0 for p in procs), "\n".join(outs)

    # the same decomposition as threads in this process (same kernels, the
    # peers' buffers addressed directly): bitwise
    geom = dict(decomp="pencil", p1=grid[0], p2=grid[1]) if grid else {}
    cfg = S.SolverConfig(n=n, p=world, nu=1e-3, dt=1e-3, t_end=1e-3, **geom)
    uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=9)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            (s0, s1, s2), (o0, o1, o2) = c.layout.spec_shape, c.layout.spec_offset
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
            fft = S.DistributedFFT(c)
            ur = c.real_field()
            fft.inverse(uo, ur)
            fu = c.spectral_field()
            fft.forward(ur, fu)
            res = (du.download(), uo.download(), stats.energy, stats.enstrophy, ur.download(),
                   fu.download())
            st.close()
            return res

    ref = S.run_group(world, body)
    for r in range(world):
        d = np.load(tmp_path / f"r{r}.npz")
        assert str(d["transposes"]) == "peer-direct"
        assert bool(d["ck_ok"])  # checkpoint round trip over the host transport
        assert d["bcast"].tolist() == [world] * 24  # broadcast_bytes from the last rank
        assert np.array_equal(d["du"], ref[r][0])
        assert np.array_equal(d["u"], ref[r][1])
        assert float(d["e"]) == ref[r][2] and float(d["z"]) == ref[r][3]
        assert np.array_equal(d["ur"], ref[r][4]) and np.array_equal(d["fu"], ref[r][5])
    # the multi-process checkpoint equals one written by the threads-as-ranks run
    with S.Context(S.SolverConfig(n=n)) as c1:
        u1 = c1.real_field()
        t1, s1 = S.read_checkpoint(c1, str(tmp_path / "ck.sdns"), u1)
        g = u1.download()
    assert (t1, s1) == (0.25, 7)
    for r in range(world):
        lo = S.build_layout(cfg, r)
        (a0, a1, a2), (b0, b1, b2) = lo.real_shape, lo.real_offset
        assert np.array_equal(g[:, b0:b0 + a0, b1:b1 + a1, b2:b2 + a2], ref[r][4])


def test_stalled_peer_raises_timeout_error(tmp_path):
    """A rank whose peer stalls inside the step sees TimeoutError (the
    reference's collective deadline, transport.cpp:105-140) instead of
    hanging, and the communicator is poisoned: the next collective fails
    at once with the same error."""
    worker = os.path.join(ROOT, "tests", "helpers", "mp_stall_worker.py")
    port = _free_port()
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(port), str(tmp_path)], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(2)]
    try:
        out0 = procs[0].communicate(timeout=240)[0]
    finally:
        procs[1].kill()
        procs[1].communicate()
    assert procs[0].returncode == 0, out0
    lines = (tmp_path / "stall.txt").read_text().splitlines()
    assert lines[0].startswith("TimeoutError"), lines
    assert lines[1].startswith("barrier TimeoutError"), lines
    assert float(lines[1].split("after ")[1].split(" s")[0]) < 1.0, lines  # fails fast
