# temporal pass with processor faces on one device: 512^3 in 2 or 4 grid components, ghost 2
import sys, time
sys.path.insert(0, ".")
import paper_1201_2118_b200 as sfb
workers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = sfb.SolverConfig(extents=(512, 512, 512), symmetry_z=False, tolerance=1e-30, max_sweeps=200, omega=1.9525)
s = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), workers=workers, ghost=2)
s.init_cavity()
s.step()
s.synchronize()
t = time.perf_counter()
for _ in range(2):
    s.step()
s.synchronize()
print("workers", workers, "ms/step %.1f" % ((time.perf_counter() - t) / 2 * 1e3))
