"""A few captured RK4 steps at n = 64 (the launch list of config 1's step
under ncu: which kernels, how long each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_00850_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = S.SolverConfig(n=n, nu=0.01, dt=0.01, t_end=0.01)
with S.Context(cfg) as c:
    st = S.Rk4State(c)
    st.set(c.spectral_field().upload(S.iso_init(n, c.layout, seed=1)))
    for _ in range(3):
        st.rk4_step(0.01, post_project=True, check=False)
    c.sync()
    st.close()
