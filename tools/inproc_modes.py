"""Slab transpose modes at p > 1, ranks as threads on one GPU (sdns_bench:
5 warm-up + K timed RK4 steps, wall time): peer-direct (default), all-to-all
overlapped (context option all_to_all), serial (all_to_all + serial).
   python tools/inproc_modes.py [K]      (GPU box)"""
import os
import sys

sys.path.insert(0, ".")
import paper_1607_00850_b200 as S

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
entries = [S.BenchEntry(n, "slab", p) for n in (256, 512) for p in (1, 2, 4, 8)]
entries += [S.BenchEntry(n, "pencil", p, p1, p2) for n in (256, 512)
            for p, p1, p2 in ((4, 2, 2), (8, 2, 4), (8, 4, 2))]
for name, opt in (("peer", {}), ("overlap", {"all_to_all": 1}),
                  ("serial", {"all_to_all": 1, "serial": 1})):
    rows = S.bench(entries, K, S.RunOptions(collective_timeout_s=600, options=opt))
    for r in rows:
        print(f"{name:8s} n={r.entry.n} {r.entry.decomp} p={r.entry.p} ({r.entry.p1}x{r.entry.p2}): "
              f"{r.sec_per_step * 1e3:8.2f} ms/step "
              f"{r.status}", flush=True)
