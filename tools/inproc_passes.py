"""Per-pass times of one rank (rank 0) of an in-process run (ranks as threads
on one GPU): python tools/inproc_passes.py [n] [p] [decomp p1 p2]   (GPU box)"""
import sys

sys.path.insert(0, ".")
import paper_1607_00850_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
p = int(sys.argv[2]) if len(sys.argv) > 2 else 2
geom = dict(decomp=sys.argv[3], p1=int(sys.argv[4]), p2=int(sys.argv[5])) if len(sys.argv) > 5 else {}
cfg = S.SolverConfig(n=n, p=p, nu=5e-4, dt=5e-4, t_end=5e-4, **geom)
uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=1607)


def body(rank, comm):
    with S.Context(cfg, rank=rank, comm=comm) as c:
        (s0, s1, s2), (o0, o1, o2) = c.layout.spec_shape, c.layout.spec_offset
        st = S.Rk4State(c)
        st.set(c.spectral_field().upload(uh0[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2]))
        for _ in range(2):
            st.rk4_step(5e-4, check=False)
        c.sync()
        c.timing(True)
        for _ in range(3):
            st.rk4_step(5e-4, check=False)
        res = c.timing_read()
        c.timing(False)
        st.close()
        return c.transposes, res


tr, res = S.run_group(p, body)[0]
print(f"n={n} p={p} {geom} transposes={tr}")
tot = 0.0
for k, (ms, cnt) in res.items():
    if cnt:
        print(f"  {k:12s} {ms / cnt:8.3f} ms x {cnt}")
        tot += ms
print(f"  total {tot / 3:.2f} ms/step (rank 0, sum of timed launches)")
