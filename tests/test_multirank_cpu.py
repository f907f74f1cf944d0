"""CPU, world_size > 1 over gloo: the multi-rank host logic of the slab path.

Each process is one rank. It takes its layout, device layout and transpose
plan from the product library (host-only C-ABI calls; the same code the
device context executes), runs the distributed 3-D transform with numpy
standing in for the per-axis device FFT passes but with the EXACT device
buffer layouts (pitched rows, pad rows, the [peer][x_l][y_l] receive layout)
and moves the plan's blocks with torch.distributed.all_to_all_single. The
result must equal the global transform (forward and inverse), and the block
tables of all ranks must pair up (transport.cpp:271-304 validation).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange(buf_src, buf_dst, plan):
    """Executes a plan (peer, src_off, dst_off, count) with all_to_all_single;
    blocks are grouped by peer in plan order (the k-th block sent to q is the
    k-th block q receives from me, as for the NCCL grouped send/recv)."""
    p = int(plan[:, 0].max()) + 1
    order = [i for q in range(p) for i in range(len(plan)) if plan[i, 0] == q]
    send_by_peer = np.concatenate([buf_src[plan[i, 1]:plan[i, 1] + plan[i, 3]] for i in order]).view(np.float64)
    split = [int(2 * sum(plan[i, 3] for i in range(len(plan)) if plan[i, 0] == q)) for q in range(p)]
    out = torch.empty(sum(split), dtype=torch.float64)
    dist.all_to_all_single(out, torch.from_numpy(send_by_peer.copy()), split, split)
    got = out.numpy().view(np.complex128)
    pos = 0
    for i in order:
        c = int(plan[i, 3])
        buf_dst[plan[i, 2]:plan[i, 2] + c] = got[pos:pos + c]
        pos += c


def _worker(rank, world, port, n, result_dir):
    import sys
    sys.path.insert(0, ROOT)
    import paper_1607_00850_b200 as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = S.SolverConfig(n=n, p=world)
        lo = S.build_layout(cfg, rank)
        d = S.device_layout(cfg, rank)
        # block tables pair up across ranks
        tables = [None] * world
        dist.all_gather_object(tables, lo.stages)
        for q in range(world):
            assert lo.stages[0][0][q] == tables[q][0][1][rank]
        rng = np.random.default_rng(11)
        u = rng.uniform(-1, 1, (n, n, n))
        ref = np.fft.rfftn(u)
        np_, pitch, prow, cs = d["np"], d["pitch"], d["prow"], d["spec_cs"]
        nf = n // 2 + 1
        x0 = lo.real_offset[0]
        # forward: z r2c + y c2c on the real slab -> receive layout (wb)
        a = np.fft.fft(np.fft.rfft(u[x0:x0 + np_], axis=2), axis=1)  # (x_l, y, kz)
        wb = np.zeros(cs, dtype=np.complex128)
        for xl in range(np_):
            for y in range(n):
                plane = (y // np_) * np_ + xl
                off = (plane * prow + y % np_) * pitch
                wb[off:off + nf] = a[xl, y]
        wa = np.zeros(cs, dtype=np.complex128)
        _exchange(wb, wa, S.exchange_plan(cfg, rank, False, 1))
        # x layout: (x, y_l, kz) at (x*prow + y_l)*pitch + kz -> x c2c
        X = np.empty((n, np_, nf), dtype=np.complex128)
        for x in range(n):
            for yl in range(np_):
                off = (x * prow + yl) * pitch
                X[x, yl] = wa[off:off + nf]
        spec = np.fft.fft(X, axis=0)
        y0 = lo.spec_offset[1]
        fwd_err = np.abs(spec - ref[:, y0:y0 + np_, :]).max() / np.abs(ref).max()
        # inverse: x c2c back -> x layout -> plan (wa -> wb) -> y, z back
        Xi = np.fft.ifft(spec, axis=0)
        wa[:] = 0
        for x in range(n):
            for yl in range(np_):
                off = (x * prow + yl) * pitch
                wa[off:off + nf] = Xi[x, yl]
        wb[:] = 0
        _exchange(wa, wb, S.exchange_plan(cfg, rank, True, 1))
        B = np.empty((np_, n, nf), dtype=np.complex128)
        for xl in range(np_):
            for y in range(n):
                plane = (y // np_) * np_ + xl
                off = (plane * prow + y % np_) * pitch
                B[xl, y] = wb[off:off + nf]
        back = np.fft.irfft(np.fft.ifft(B, axis=1), n=n, axis=2)
        inv_err = np.abs(back - u[x0:x0 + np_]).max()
        # iso field blocks agree with the single-rank field
        g = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0))
        mine = S.iso_init(n, lo)
        iso_ok = np.array_equal(mine, g[:, :, y0:y0 + np_, :])
        np.save(os.path.join(result_dir, f"r{rank}.npy"), np.array([fwd_err, inv_err, float(iso_ok)]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [16])
def test_slab_transpose_plan_world2_gloo(tmp_path, n):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        fwd_err, inv_err, iso_ok = np.load(tmp_path / f"r{r}.npy")
        assert fwd_err <= 1e-13, fwd_err
        assert inv_err <= 1e-13, inv_err
        assert iso_ok == 1.0
