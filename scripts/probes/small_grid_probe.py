# small-grid regime: where a re100 step's time goes (wall clock, after warm-up)
import time, sys
sys.path.insert(0, ".")
import paper_1201_2118_b200 as sfb
from paper_1201_2118_b200.cavity import run_cavity
cfg = sfb.SolverConfig(extents=(129, 129, 3), reynolds=100.0, sigma=0.9, omega=1.9525, tolerance=1e-6,
                       max_sweeps=3000, symmetry_z=True)
par = sfb.FluidParams(viscosity=0.01, lid_speed=1.0)
for fused in ([int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else (1, 3)):
    sim = sfb.Simulation(cfg, par, fused=fused)
    sim.init_cavity()
    for _ in range(200): sim.step()
    n = 500
    t = time.perf_counter(); sw = 0
    for _ in range(n):
        st = sim.step(); sw += st.sweeps
    t_step = (time.perf_counter() - t) / n
    t = time.perf_counter()
    for _ in range(n): sim.steady_delta()
    t_sd = (time.perf_counter() - t) / n
    t = time.perf_counter()
    for _ in range(n): sim.compute_dt()
    t_dt = (time.perf_counter() - t) / n
    print("fused=%d step %.1f us (%.1f sweeps, %.2f us/sweep) steady_delta %.1f us compute_dt %.1f us" %
          (fused, t_step * 1e6, sw / n, t_step * 1e6 / (sw / n), t_sd * 1e6, t_dt * 1e6))
