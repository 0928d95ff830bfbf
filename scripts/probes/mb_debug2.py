import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1201_2118_b200 as sfb
seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
rng = np.random.default_rng(200 + seed)
ext = (int(rng.integers(40, 90)), int(rng.integers(24, 60)), int(rng.integers(6, 70)))
workers = int(rng.choice([2, 3, 4, 6]))
kinds = ["wall", "symmetry"]
faces = [(a, sd, kinds[int(rng.integers(0, 2))], tuple(rng.uniform(-0.3, 0.3, 3))) for a in range(3) for sd in range(2)]
tol, maxs, omega = float(rng.choice([1e-30, 1e-3])), int(rng.integers(1, 25)), float(rng.uniform(1.0, 1.95))
vel = {f: rng.uniform(-0.5, 0.5, size=ext[::-1]) for f in ("vx", "vy", "vz")}
if len(sys.argv) > 2: workers = int(sys.argv[2])
if len(sys.argv) > 3: maxs = int(sys.argv[3])
if len(sys.argv) > 4: tol = float(sys.argv[4])
if len(sys.argv) > 5: faces = [(a, sd, k if sys.argv[5] == "keep" else sys.argv[5], v if sys.argv[5] == "keep" else (0, 0, 0)) for a, sd, k, v in faces]
print(ext, workers, tol, maxs, [(a, sd, k) for a, sd, k, v in faces])
sims = {}
for fused in (1, 3):
    cfg = sfb.SolverConfig(extents=ext, tolerance=tol, max_sweeps=maxs, symmetry_z=False, omega=omega)
    s = sfb.Simulation(cfg, sfb.FluidParams(viscosity=0.02, lid_speed=0.0), workers=workers, ghost=2, fused=fused)
    s.init_cavity()
    for a, sd, k, v in faces:
        s.set_face_bc(a, sd, k, v)
    for f, arr in vel.items():
        s.scatter(f, arr)
    sims[fused] = s
d = sfb.decompose(ext, workers, 2, (False, False, False))
print("blocks", [(tuple(d.lo[w]), d.size(w)) for w in range(workers)])
for step in range(1):
    st = {f: sims[f].step() for f in (1, 3)}
    print("step", step, [(x.sweeps, x.residual) for x in st.values()])
    for f in ("vx", "vy", "vz", "p", "divu"):
        a, b = sims[1].gather(f), sims[3].gather(f)
        dd = np.argwhere(a.view(np.uint64) != b.view(np.uint64))
        if len(dd):
            print("  ", f, len(dd), "first (z,y,x):", dd[:6].tolist(), "max abs diff", np.abs(a - b).max())
