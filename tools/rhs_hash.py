"""sha256 of one compute_rhs of the seeded iso field (A/B: two builds of the
library must print the same hash): python tools/rhs_hash.py N [LIB]   (GPU box)"""
import hashlib
import sys

sys.path.insert(0, ".")
import paper_1607_00850_b200 as S  # noqa: E402

n = int(sys.argv[1])
if len(sys.argv) > 2:
    S.use_library(sys.argv[2])
nu = {512: 5e-4, 1024: 2.5e-4}.get(n, 1e-3)
uh = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=1607)
cfg = S.SolverConfig(n=n, nu=nu, dt=nu, t_end=nu)
with S.Context(cfg) as c:
    u = c.spectral_field().upload(uh)
    du = c.spectral_field()
    S.compute_rhs(c, u, cfg.nu, du)
    a = du.download()
print(n, sys.argv[2] if len(sys.argv) > 2 else "default", hashlib.sha256(a.tobytes()).hexdigest())
