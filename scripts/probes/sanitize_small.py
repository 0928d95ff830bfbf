# small temporal + single runs for compute-sanitizer (racecheck / memcheck)
import sys
sys.path.insert(0, ".")
import paper_1201_2118_b200 as sfb
for fused in (1, 3):
    cfg = sfb.SolverConfig(extents=(40, 24, 20), tolerance=1e-30, max_sweeps=5, symmetry_z=False)
    s = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), fused=fused)
    s.init_cavity()
    for _ in range(3):
        s.step()
    print(fused, s.checksum())
