# per-half-sweep time of the pressure loop vs grid size (env selects the path:
# SF_PERSIST=0/1, SF_PZC); fixed 200 half-sweeps per step (tolerance 1e-300)
import os, sys, time
sys.path.insert(0, ".")
import paper_1201_2118_b200 as sfb
sizes = [tuple(int(v) for v in s.split("x")) for s in (sys.argv[1] if len(sys.argv) > 1 else "129x129x3,64x64x64,96x96x96,128x128x128,192x192x192,256x256x256").split(",")]
fused = int(os.environ.get("FUSED", "1"))
par = sfb.FluidParams(viscosity=0.01, lid_speed=1.0)
out = []
for ext in sizes:
    cfg = sfb.SolverConfig(extents=ext, reynolds=100.0, sigma=0.9, omega=1.9525, tolerance=1e-300, max_sweeps=200,
                           symmetry_z=ext[2] <= 4)
    sim = sfb.Simulation(cfg, par, fused=fused)
    sim.init_cavity()
    for _ in range(3): sim.step()
    n = 20
    t = time.perf_counter()
    for _ in range(n): st = sim.step()
    dt = (time.perf_counter() - t) / n
    out.append("%s %.2f us/sweep" % ("x".join(map(str, ext)), dt * 1e6 / st.sweeps))
print("PERSIST=%s PZC=%s ZC2=%s fused=%d: %s" % (os.environ.get("SF_PERSIST", "auto"), os.environ.get("SF_PZC", "auto"), os.environ.get("SF_ZC2", "auto"), fused, " | ".join(out)))
