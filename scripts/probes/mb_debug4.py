import sys, itertools
sys.path.insert(0, ".")
import numpy as np
import paper_1201_2118_b200 as sfb
def run(ext, workers, maxs, facemode):
    rng = np.random.default_rng(5)
    vel = {f: rng.uniform(-0.5, 0.5, size=ext[::-1]) for f in ("vx", "vy", "vz")}
    out = {}
    for fused in (1, 3):
        cfg = sfb.SolverConfig(extents=ext, tolerance=1e-30, max_sweeps=maxs, symmetry_z=False, omega=1.5)
        s = sfb.Simulation(cfg, sfb.FluidParams(viscosity=0.02, lid_speed=0.0), workers=workers, ghost=2, fused=fused)
        s.init_cavity()
        if facemode == "sym":
            for a in range(3):
                for sd in range(2):
                    s.set_face_bc(a, sd, "symmetry")
        for f, arr in vel.items():
            s.scatter(f, arr)
        st = s.step()
        out[fused] = (st.residual, {f: s.gather(f) for f in ("vx", "vy", "vz", "p", "divu")})
    bad = []
    for f in out[1][1]:
        a, b = out[1][1][f], out[3][1][f]
        dd = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
        if len(dd): bad.append((f, len(dd), dd[0].tolist(), 'z', (dd[:,0].min(), dd[:,0].max()), 'y', (dd[:,1].min(), dd[:,1].max()), 'x', (dd[:,2].min(), dd[:,2].max())))
    return out[1][0] == out[3][0], bad
for ext, workers in [((77, 43, 63), 3), ((77, 43, 20), 3), ((77, 20, 20), 3), ((60, 20, 20), 2), ((52, 20, 20), 2)]:
    d = sfb.decompose(ext, workers, 2, (False, False, False))
    for maxs in (4,):
        print(ext, workers, [(tuple(d.lo[w]), d.size(w)) for w in range(workers)][:2], maxs, run(ext, workers, maxs, "walls"))
