"""GPU: the in-process transport (threads-as-ranks on one device) against
the reference's transport suite (proj/tests/test_transport.cpp:15-219):
split ordering, rank-ordered bit-deterministic reductions, all-to-all with
empty and unequal blocks on device buffers, and the fault paths -- mismatched
collectives and inconsistent tables raise ProtocolError on every rank, an
absent rank times out, a poisoned group fails fast and stays failed."""
import time

import numpy as np
import pytest
import torch

import paper_1607_00850_b200 as S

pytestmark = pytest.mark.gpu


def test_split_orders_subgroups_by_key_then_rank():  # test_transport.cpp:104-117
    def body(rank, comm):
        sub = comm.split(rank % 2, -rank)
        try:
            assert sub.size == 2
            assert sub.rank == (0 if rank >= 2 else 1)
            return float(sub.allreduce([float(rank)])[0])
        finally:
            sub.close()
    assert S.run_group(4, body) == [2.0, 4.0, 2.0, 4.0]


def test_allreduce_rank_order_and_bit_deterministic():
    rng = np.random.default_rng(3)
    vals = rng.standard_normal((5, 16)) * 10.0 ** rng.integers(-8, 8, (5, 16))

    def body(rank, comm):
        outs = [comm.allreduce(vals[rank], op) for op in ("sum", "max", "min")]
        again = [comm.allreduce(vals[rank], "sum") for _ in range(3)]
        return outs, again
    res = S.run_group(5, body)
    want = vals[0].copy()
    for q in range(1, 5):
        want = want + vals[q]  # ascending rank order (transport.cpp:319-329)
    for outs, again in res:
        assert np.array_equal(outs[0], want)
        assert np.array_equal(outs[1], vals.max(axis=0))
        assert np.array_equal(outs[2], vals.min(axis=0))
        assert all(np.array_equal(a, want) for a in again)


def _a2a(comm, send_counts, recv_counts, send_vals):
    s = torch.tensor(send_vals if len(send_vals) else [0.0], dtype=torch.float64, device="cuda")
    r = torch.full((max(1, int(sum(recv_counts))),), -1.0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    comm.all_to_all_bytes(s.data_ptr(), [8 * c for c in send_counts], r.data_ptr(),
                          [8 * c for c in recv_counts])
    return r.cpu().numpy()[:int(sum(recv_counts))]


def test_all_to_all_empty_and_unequal_blocks():  # test_transport.cpp:199-219
    def body(rank, comm):
        torch.cuda.set_device(0)
        if rank == 0:
            return _a2a(comm, [1, 3], [1, 0], [1.0, 2.0, 3.0, 4.0])
        return _a2a(comm, [0, 0], [3, 0], [])
    r0, r1 = S.run_group(2, body)
    assert list(r0) == [1.0] and list(r1) == [2.0, 3.0, 4.0]


def test_all_to_all_random_tables_round_trip():
    rng = np.random.default_rng(11)
    p = 4
    counts = rng.integers(0, 9, (p, p))

    def body(rank, comm):
        torch.cuda.set_device(0)
        send = [1000.0 * rank + 10.0 * q + i for q in range(p) for i in range(counts[rank][q])]
        return _a2a(comm, list(counts[rank]), [counts[q][rank] for q in range(p)], send)
    res = S.run_group(p, body)
    for r in range(p):
        want = [1000.0 * q + 10.0 * r + i for q in range(p) for i in range(counts[q][r])]
        assert list(res[r]) == want


def test_broadcast_from_a_non_zero_root():  # test_transport.cpp:95-103
    want = np.arange(10, 15, dtype=np.int32).tobytes()

    def body(rank, comm):
        buf = want if rank == 2 else bytes(len(want))
        return comm.broadcast_bytes(buf, root=2)
    assert S.run_group(4, body) == [want] * 4


def test_broadcast_argument_mismatch_raises_everywhere():  # transport.cpp:332-349
    errors = []

    def body(rank, comm):
        try:
            comm.broadcast_bytes(bytes(8 if rank == 0 else 16), root=0)
        except S.ProtocolError as e:
            errors.append(str(e))
            raise
    with pytest.raises(S.ProtocolError):
        S.run_group(3, body, timeout_s=10.0)
    assert len(errors) == 3 and all("broadcast argument mismatch" in e for e in errors)

    def bad_root(rank, comm):
        comm.broadcast_bytes(b"x", root=5)
    with pytest.raises(S.ProtocolError, match="out of range"):
        S.run_group(2, bad_root, timeout_s=10.0)


def test_mismatched_collectives_raise_protocol_error_everywhere():  # :119-137
    errors = []

    def body(rank, comm):
        try:
            if rank == 0:
                comm.allreduce([1.0])
            else:
                comm.barrier()
        except S.ProtocolError as e:
            errors.append(str(e))
            raise
    with pytest.raises(S.ProtocolError):
        S.run_group(2, body, timeout_s=10.0)
    assert len(errors) == 2 and all("mismatched collectives" in e for e in errors)


def test_inconsistent_all_to_all_tables_raise_protocol_error():  # :139-156
    def body(rank, comm):
        torch.cuda.set_device(0)
        if rank == 0:
            _a2a(comm, [0, 2], [1, 1], [1.0, 1.0])
        else:
            _a2a(comm, [1, 0], [2, 0], [1.0])
    t0 = time.monotonic()
    with pytest.raises(S.ProtocolError):
        S.run_group(2, body, timeout_s=30.0)
    assert time.monotonic() - t0 < 10.0  # the detecting rank poisons the group


def test_absent_rank_times_out_the_peers():  # :158-170
    def body(rank, comm):
        if rank == 1:
            return
        comm.barrier()
    t0 = time.monotonic()
    with pytest.raises(S.CollectiveTimeout):
        S.run_group(2, body, timeout_s=0.2)
    assert time.monotonic() - t0 < 10.0


def test_poisoned_group_fails_with_the_reason_and_stays_failed():  # :172-197
    def body(rank, comm):
        if rank == 2:
            comm.poison("rank 2 failed: boom at rank 2")
            raise RuntimeError("boom at rank 2")
        comm.barrier()
        comm.barrier()
    with pytest.raises((S.ProtocolError, RuntimeError), match="boom at rank 2"):
        S.run_group(3, body, timeout_s=30.0)
    comms = S.Comm.inprocess_group(2, 0, 0.5)
    try:
        comms[0].poison("manual poison")
        with pytest.raises(S.ProtocolError, match="manual poison"):
            comms[0].barrier()
        with pytest.raises(S.ProtocolError):
            comms[0].allreduce([1.0])
    finally:
        for c in comms:
            c.close()


def test_loopback_transport():  # :40-58
    c = S.Comm.loopback()
    try:
        assert (c.rank, c.size) == (0, 1)
        assert list(c.allreduce([1.5, -2.0], "max")) == [1.5, -2.0]
        torch.cuda.set_device(0)
        assert list(_a2a(c, [3], [3], [1.0, 2.0, 3.0])) == [1.0, 2.0, 3.0]
        b = np.array([7.0, 8.0]).tobytes()
        assert c.broadcast_bytes(b, root=0) == b
        with pytest.raises(S.ProtocolError, match="root must be 0"):
            c.broadcast_bytes(b, root=1)
    finally:
        c.close()
