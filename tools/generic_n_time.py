"""RK4 step time at generic (non-power-of-two) n beside the tuned lengths:
   python tools/generic_n_time.py [n ...]        (GPU box)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_00850_b200 as S  # noqa: E402

sizes = [int(a) for a in sys.argv[1:]] or [96, 128, 192, 256, 384, 512]
for n in sizes:
    cfg = S.SolverConfig(n=n, nu=1e-3, dt=1e-3, t_end=1e-3)
    with S.Context(cfg) as c:
        st = S.Rk4State(c)
        st.set(c.spectral_field().upload(S.iso_init(n, c.layout, seed=1)))
        for _ in range(2):
            st.rk4_step(1e-3, post_project=True, check=False)
        c.sync()
        s = torch.cuda.ExternalStream(c.stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        k = 3
        for _ in range(k):
            st.rk4_step(1e-3, post_project=True, check=False)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / k
        c3 = 16.0 * n * n * (n // 2 + 1)
        print(f"n={n}: {ms:.3f} ms/step, {213 * c3 / (ms * 1e-3) / 1e9:.0f} GB/s (213 C)", flush=True)
        st.close()
