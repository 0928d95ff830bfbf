# where the end-to-end step time goes (512^3 cavity, async block transfers)
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1201_2118_b200 as sfb
cfg = sfb.SolverConfig(extents=(512, 512, 512), symmetry_z=False, tolerance=1e-30, max_sweeps=200, omega=1.9525)
sim = sfb.Simulation(cfg, sfb.cavity_fluid(cfg))
sim.init_cavity()
names = ("vx", "vy", "vz", "p")
hin = {f: torch.from_numpy(sim.gather_block(f)).reshape(-1).pin_memory() for f in names}
hout = {f: torch.empty(512 ** 3, dtype=torch.float64).pin_memory() for f in names}
sim.step()
def t(): sim.synchronize(); return time.perf_counter()
for rep in range(2):
    a = t()
    for f in names: sim.scatter_block(f, hin[f], wait=False)
    b = time.perf_counter()
    sim.step()
    c = time.perf_counter()
    for f in names: sim.gather_block(f, out=hout[f], wait=False)
    d = time.perf_counter()
    e = t()
    print("scatter enqueue %.1f ms, step %.1f ms, gather enqueue %.1f ms, final sync %.1f ms, total %.1f" % ((b-a)*1e3, (c-b)*1e3, (d-c)*1e3, (e-d)*1e3, (e-a)*1e3))
a = t(); sim.step(); b = t(); print("step alone %.1f ms" % ((b - a) * 1e3))
# step while the previous step's downloads run in the background
for f in names: sim.gather_block(f, out=hout[f], wait=False)
a = time.perf_counter(); sim.step(); b = time.perf_counter(); sim.synchronize(); c = time.perf_counter()
print("step with background downloads %.1f ms (+%.1f to drain)" % ((b - a) * 1e3, (c - b) * 1e3))
# the bench's loop: no per-iteration synchronisation
sim.synchronize()
a = time.perf_counter()
marks = []
for _ in range(3):
    m0 = time.perf_counter()
    for f in names: sim.scatter_block(f, hin[f], wait=False)
    m1 = time.perf_counter()
    sim.step()
    m2 = time.perf_counter()
    for f in names: sim.gather_block(f, out=hout[f], wait=False)
    m3 = time.perf_counter()
    marks.append(((m1 - m0) * 1e3, (m2 - m1) * 1e3, (m3 - m2) * 1e3))
sim.synchronize()
b = time.perf_counter()
print("bench loop: %.1f ms/step" % ((b - a) / 3 * 1e3), ["scatter %.1f step %.1f gather %.1f" % m for m in marks])
