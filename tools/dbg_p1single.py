"""Debug: P1 single-item kernel vs default on a pencil grid (where do they differ?)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1607_00850_b200 as S



def scatter(uh0, lo):
    o, s = lo.spec_offset, lo.spec_shape
    return np.ascontiguousarray(uh0[:, o[0]:o[0]+s[0], o[1]:o[1]+s[1], o[2]:o[2]+s[2]])

def main(n, geom, reps):
    p = geom["p"]
    uh0 = S.iso_init(n, S.build_layout(S.SolverConfig(n=n), 0), seed=11)
    cfg = S.SolverConfig(n=n, nu=1e-3, dt=1e-3, t_end=1e-3, **geom)
    def run():
        def body(rank, comm):
            with S.Context(cfg, rank=rank, comm=comm) as c:
                u = c.spectral_field().upload(scatter(uh0, c.layout))
                du = c.spectral_field()
                S.compute_rhs(c, u, 1e-3, du)
                return du.download()
        return S.run_group(p, body)
    base = run()
    for opt in (dict(), dict(p1_single=1), dict(p1_single=1, ldgsts_tiles=1), dict(p1_single=1, all_to_all=1), dict(all_to_all=1)):
        for r in range(reps):
            with S.context_options(**opt):
                got = run()
            msg = []
            for rk, (a, b) in enumerate(zip(base, got)):
                d = np.abs(a - b)
                if d.max() > 4e-15 * np.abs(a).max():
                    idx = np.argwhere(d > 4e-15 * np.abs(a).max())
                    msg.append("rank %d: %d bad, max %.3e, comps %s, x %s..%s y %s..%s kz %s..%s" % (
                        rk, len(idx), d.max(), sorted(set(idx[:, 0])), idx[:, 1].min(), idx[:, 1].max(),
                        idx[:, 2].min(), idx[:, 2].max(), idx[:, 3].min(), idx[:, 3].max()))
            print(n, geom, opt, r, "OK" if not msg else msg, flush=True)

if __name__ == "__main__":
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    main(128, dict(decomp="pencil", p=4, p1=2, p2=2), reps)
    main(128, dict(decomp="pencil", p=2, p1=2, p2=1), reps)
    main(128, dict(decomp="pencil", p=2, p1=1, p2=2), reps)
    main(128, dict(p=2), reps)
    main(256, dict(decomp="pencil", p=4, p1=2, p2=2), 1)
