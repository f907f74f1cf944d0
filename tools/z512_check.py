"""One RHS at 512^3 (iso field) with the current library; saves du to
gpurun_out/rhs_<tag>.npy so two library variants can be compared."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_00850_b200 as S  # noqa: E402

if os.environ.get("AB_LIB"):  # tool-level A/B: another build of the library
    S.use_library(os.environ["AB_LIB"])

tag = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 512
geom = {}
if len(sys.argv) > 3 and sys.argv[3] == "pencil":
    geom = dict(decomp="pencil", p=4, p1=2, p2=2)
cfg = S.SolverConfig(n=n, nu=5e-4, dt=5e-4, t_end=5e-4, **geom)
uh = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=1607)


def body(rank, comm):
    with S.Context(cfg, rank=rank, comm=comm) as c:
        lo = c.layout
        (s0, s1, s2), (o0, o1, o2) = lo.spec_shape, lo.spec_offset
        u = c.spectral_field().upload(uh[:, o0:o0 + s0, o1:o1 + s1, o2:o2 + s2])
        du = c.spectral_field()
        S.compute_rhs(c, u, cfg.nu, du)
        return (o1, s1, o2, s2), du.download()


out = np.empty_like(uh)
for (o1, s1, o2, s2), blk in S.run_group(cfg.p, body):
    out[:, :, o1:o1 + s1, o2:o2 + s2] = blk
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/rhs_{tag}.npy", out)
print(tag, "saved", np.linalg.norm(out))
