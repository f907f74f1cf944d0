"""Where config 1's step time goes (TG-like iso 64^3): advance with a stats
sample every step, advance without samples, and back-to-back captured steps
with no host synchronisation (the GPU-side floor)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_00850_b200 as S  # noqa: E402

if os.environ.get("AB_LIB"):  # tool-level A/B: another build of the library
    S.use_library(os.environ["AB_LIB"])

for n in (32, 64, 128):
    steps = 200
    lo = S.build_layout(S.SolverConfig(n=n), 0)
    cfg = S.SolverConfig(n=n, nu=0.01, dt=0.01, t_end=steps * 0.01, out_every=1)
    with S.Context(cfg) as c:
        u = c.spectral_field().upload(S.iso_init(n, lo, seed=1))
        st = S.Rk4State(c)
        res = {}
        for mode in ("advance+sample", "advance"):
            cb = (lambda k, t: S.collect_stats(c, st.u_hat, 0.01, t)) if mode != "advance" else None
            st.set(u)
            st.advance(cb)
            c.sync()
            st.set(u)
            t0 = time.perf_counter()
            st.advance(cb)
            c.sync()
            res[mode] = (time.perf_counter() - t0) / steps * 1e3
        st.set(u)
        for _ in range(3):
            st.rk4_step(0.01, post_project=True, check=False)
        c.sync()
        stream = torch.cuda.ExternalStream(c.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            st.rk4_step(0.01, post_project=True, check=False)
        e1.record(stream)
        torch.cuda.synchronize()
        res["graph-only"] = e0.elapsed_time(e1) / steps
        import hashlib
        res["sha"] = hashlib.sha1(st.u_hat.download().tobytes()).hexdigest()[:12]
        st.close()
        print(n, {k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()},
              "ms/step", flush=True)
