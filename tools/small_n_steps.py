"""Steps/s of advance() at small n (config 1 is TG 64^3 sampled every step):
   python tools/small_n_steps.py      (GPU box; DT=... overrides dt)"""
import time, sys, os
DT = float(os.environ.get("DT", "0.01"))
sys.path.insert(0, '.')
import numpy as np
import paper_1607_00850_b200 as S
from oracle import sdns_np as O
for n, steps, every in [(64, 100, 1), (64, 100, 0), (128, 50, 1), (256, 20, 1)]:
    lo = S.build_layout(S.SolverConfig(n=n), 0)
    cfg = S.SolverConfig(n=n, nu=0.01, dt=DT, t_end=steps * DT, out_every=max(every, 1))
    with S.Context(cfg) as c:
        u = c.spectral_field().upload(S.iso_init(n, lo, seed=1))
        st = S.Rk4State(c); st.set(u)
        rows = []
        cb = (lambda k, t: rows.append(S.collect_stats(c, st.u_hat, 0.01, t))) if every else None
        st.advance(cb); c.sync()
        st.set(u)
        t0 = time.perf_counter(); st.advance(cb); c.sync(); dt = time.perf_counter() - t0
        print(f"n={n} steps={steps} sample_every={every}: {dt*1e3:.1f} ms total, {dt/steps*1e3:.3f} ms/step, {steps/dt:.0f} steps/s")
        st.close()
