"""Small device-path workload for compute-sanitizer (tools/sanitize.sh):
n = 16 and 32 RK4 steps with fused stats at p = 1, slab p = 2 threads-as-ranks
(peer-direct transposes) and pencil 2x2, plus the API transforms. Every
kernel family of the step runs (column passes with TMA/LDGSTS rings, the
fused z pass, the RK4 updates, the sampled-stats stage, reductions)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_00850_b200 as S  # noqa: E402


def one(n, geom):
    cfg = S.SolverConfig(n=n, nu=1e-3, dt=1e-3, t_end=2e-3, out_every=1, **geom)
    uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=3)

    def body(rank, comm):
        with S.Context(cfg, rank=rank, comm=comm) as c:
            (s0, s1, s2), (o0, o1, o2) = c.layout.spec_shape, c.layout.spec_offset
            st = S.Rk4State(c)
            u = c.spectral_field().upload(uh0[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2])
            st.set(u)
            rows = []
            st.advance(lambda k, t: rows.append(S.collect_stats(c, st.u_hat, 1e-3, t)))
            fft = S.DistributedFFT(c)
            ur = c.real_field()
            fft.inverse(st.u_hat, ur)
            fft.forward(ur, u)
            st.close()
            return rows[-1].energy

    e = S.run_group(cfg.p, body)
    print(n, geom, e[0], flush=True)


if __name__ == "__main__":
    for n in (16, 32):
        one(n, {})
        one(n, dict(p=2))
        one(n, dict(decomp="pencil", p=4, p1=2, p2=2))
    if len(sys.argv) > 1 and sys.argv[1] == "big":
        one(512 if len(sys.argv) < 3 else int(sys.argv[2]), {})
