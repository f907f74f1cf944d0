"""Times the distributed FFT API (config 5 round trip) at n^3, 3 components:
   python tools/fft_api_time.py [n]      (GPU box)"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1607_00850_b200 as S  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
with S.Context(S.SolverConfig(n=n)) as c:
    fft = S.DistributedFFT(c)
    ur, ub, fu = c.real_field(), c.real_field(), c.spectral_field()
    ur.upload(np.random.default_rng(1).uniform(-1, 1, (3, n, n, n)))
    st = torch.cuda.ExternalStream(c.stream)
    for _ in range(2):
        fft.forward(ur, fu)
        fft.inverse(fu, ub)
    c.sync()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record(st)
    fft.forward(ur, fu)
    ev[1].record(st)
    fft.inverse(fu, ub)
    ev[2].record(st)
    torch.cuda.synchronize()
    print(f"n={n}: forward {ev[0].elapsed_time(ev[1]):.3f} ms, inverse {ev[1].elapsed_time(ev[2]):.3f} ms")
