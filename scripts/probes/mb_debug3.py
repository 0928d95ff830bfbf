import sys, itertools
sys.path.insert(0, ".")
import numpy as np
import paper_1201_2118_b200 as sfb
ext = (54, 59, 14)
def run(workers, maxs, facemode, steps):
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
        elif facemode == "wallvel":
            for a in range(3):
                for sd in range(2):
                    s.set_face_bc(a, sd, "wall", (0.1, -0.2, 0.15))
        elif facemode.startswith("one"):
            fi = int(facemode[3:])
            s.set_face_bc(fi // 2, fi % 2, "wall", (0.1, -0.2, 0.15))
        for f, arr in vel.items():
            s.scatter(f, arr)
        for _ in range(steps):
            s.step()
        out[fused] = {f: s.gather(f) for f in ("vx", "vy", "vz", "p", "divu")}
    bad = []
    for f in out[1]:
        a, b = out[1][f], out[3][f]
        dd = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
        if len(dd): bad.append((f, len(dd), dd[0].tolist()))
    return bad
for workers, maxs, fm, steps in itertools.product((2, 4), (13,), ["one%d" % i for i in range(6)], (1,)):
    print(workers, maxs, fm, steps, run(workers, maxs, fm, steps))
