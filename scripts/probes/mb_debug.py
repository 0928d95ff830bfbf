import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1201_2118_b200 as sfb
ext = (48, 40, 36)
for workers in (2,):
    for maxs in (1, 2, 3):
        res = {}
        for fused in (1, 3):
            cfg = sfb.SolverConfig(extents=ext, tolerance=1e-30, max_sweeps=maxs, symmetry_z=False)
            s = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), workers=workers, ghost=2, fused=fused)
            s.init_cavity()
            rng = np.random.default_rng(1)
            for f in ("vx", "vy", "vz"):
                s.scatter(f, rng.uniform(-0.5, 0.5, size=ext[::-1]))
            st = s.step()
            res[fused] = (st, {f: s.gather(f) for f in ("vx", "vy", "vz", "p", "divu")})
        print("workers", workers, "maxs", maxs, res[1][0].residual, res[3][0].residual)
        for f in ("vx", "vy", "vz", "p", "divu"):
            a, b = res[1][1][f], res[3][1][f]
            d = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
            if len(d):
                print("  ", f, len(d), "first (z,y,x):", d[:4].tolist(), "x range", d[:, 2].min(), d[:, 2].max(), "y", d[:, 1].min(), d[:, 1].max(), "z", d[:, 0].min(), d[:, 0].max())
