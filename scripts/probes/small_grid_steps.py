# a few re100-sized steps (for an ncu launch list of the small-grid regime)
import sys
sys.path.insert(0, ".")
import paper_1201_2118_b200 as sfb
cfg = sfb.SolverConfig(extents=(129, 129, 3), reynolds=100.0, sigma=0.9, omega=1.9525, tolerance=1e-6,
                       max_sweeps=3000, symmetry_z=True)
sim = sfb.Simulation(cfg, sfb.FluidParams(viscosity=0.01, lid_speed=1.0), fused=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
sim.init_cavity()
for _ in range(3):
    sim.step()
