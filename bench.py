#!/usr/bin/env python
"""bench.py -- headline benchmark of the B200 stencil hot path.

Workload (BASELINE.json configs[1]): the 3D lid-driven cavity at 512^3, fp64,
ghost width 1, on one B200.  One bench "step" is one full cfd::simulation::step
(cfd.hpp:307-316): compute_dt + ghost refresh + UPDATE_VELOCITY + 200
red-black pressure half-sweeps (each: PRESSURE_SWEEP + velocity refresh +
DIVERGENCE + max|div|) + refresh(p).  Fixed work per step as in
proj/runs/bench128.cfg: tolerance 1e-30, max_sweeps 200, omega 1.9525.

metric: grid-point updates/sec = cells x steps / second (the reference bench
unit, bench.hpp:87-89), reported in Mcells/s.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified stencilforge compiled in place) on this box's host cores on a
bounded sample of the same workload, projected to the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_HALF_SWEEP = 80  # fused half-sweep: read divu,p,vx,vy,vz; write p,vx,vy,vz,divu' (fp64)
BYTES_UV = 56              # UPDATE_VELOCITY: read vx,vy,vz,p; write vx,vy,vz
BYTES_DIV = 32             # DIVERGENCE: read vx,vy,vz; write divu
METRIC = "grid-point updates/sec"
UNIT = "Mcells/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=512, help="cells per axis per GPU")
    ap.add_argument("--sweeps", type=int, default=200, help="pressure half-sweeps per step")
    ap.add_argument("--variant", default="tma", choices=["tma", "tma1", "ldg", "unfused"],
                    help="tma: TMA pipeline with the temporal pass (two half-sweeps per launch) where it "
                         "applies (default); tma1: one TMA half-sweep per launch; ldg: fused with plain "
                         "loads; unfused: the reference's dataflow")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--strong", type=int, default=0, metavar="N",
                    help="strong scaling (BASELINE.json configs[3]): a fixed N^3 global grid block-decomposed "
                         "over the ranks (default: weak scaling, --n^3 per rank)")
    ap.add_argument("--force-dist", action="store_true",
                    help="take the multi-rank (NCCL) path even at one rank (a check of that path on one GPU)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--ref-budget", type=float, default=1200.0,
                    help="--impl reference: wall seconds of timed reference steps (at least one step runs)")
    ap.add_argument("--workload", default="cavity", choices=["cavity", "stencil"],
                    help="cavity = configs[1] (headline); stencil = configs[4], a descriptor-declared "
                         "high-order Laplacian (radius 2 or 3) JIT-compiled from its point function")
    ap.add_argument("--radius", type=int, default=2)
    ap.add_argument("--config", default="c1", choices=["c1", "c0"],
                    help="c1: BASELINE.json configs[1] fixed-work cavity (default); c0: configs[0], the 64^3 "
                         "reference oracle run with the default solver config (tolerance 1e-6, up to 500 "
                         "half-sweeps per step), timed from rest over --steps steps")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="field storage: --workload stencil fields; --workload cavity: f32 = the fp32 variant of the "
                         "CFD fields (fused TMA half-sweep in fp32; tolerance-checked, not bitwise)")
    ap.add_argument("--tile", default="32,16,64", help="descriptor TILE for --workload stencil")
    return ap.parse_args()


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def kernel_source_sha() -> str:
    """sha256 (16 hex) over the library's CUDA sources (scripts/ncu_summary.py
    records the same hash with each capture)."""
    import hashlib
    h = hashlib.sha256()
    src = os.path.join(ROOT, "paper_1201_2118_b200", "csrc")
    for n in sorted(os.listdir(src)):
        if n.endswith((".cu", ".cuh", ".hpp")):
            with open(os.path.join(src, n), "rb") as f:
                h.update(n.encode() + f.read())
    return h.hexdigest()[:16]


def ncu_traffic(kernel="sweep_div", algo_bytes=None):
    """DRAM bytes per launch of the dominant kernel from its committed ncu
    capture (profiles/ncu_<kernel>.json), with the capture's provenance: the
    traffic is marked stale when the kernel sources changed since, and is not
    reported for another workload (the capture's algorithmic bytes per launch
    differ from this run's)."""
    p = os.path.join(ROOT, "profiles", f"ncu_{kernel}.json")
    try:
        with open(p) as f:
            d = json.load(f)
        sha = d.get("kernel_source_sha")
        src = {"file": os.path.relpath(p, ROOT), "captured_from": d.get("captured_from"),
               "kernel_source_sha": sha, "stale": sha != kernel_source_sha()}
        cap = d.get("algo_bytes_per_launch")
        if algo_bytes is not None and cap is not None and int(cap) != int(algo_bytes):
            src["not_applicable"] = "captured on a workload of %d algorithmic bytes per launch, this run has %d" % (
                int(cap), int(algo_bytes))
            return None, src
        return d.get("dram_bytes_per_launch"), src
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.TemporaryFile(mode="w+")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.device)], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
                pw.append(float(r[3]))
            except ValueError:
                continue
            for nm, v in zip(names, r[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s, p in zip(sm, pw) if p > 200.0] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def cavity_cfg(sfb, n, sweeps, c0=False):
    if c0:  # configs[0]: the reference oracle run, cli::run_config defaults (config.hpp:51-94)
        return sfb.SolverConfig(extents=(n, n, n), reynolds=100.0, symmetry_z=False)
    return sfb.SolverConfig(extents=(n, n, n), reynolds=100.0, sigma=0.5, omega=1.9525,
                            tolerance=1e-30, max_sweeps=sweeps, symmetry_z=False)


def golden_checksums(n, sweeps, c0):
    """FNV checksums (bench.hpp:24-39) the reference produced for this
    configuration from rest, by step count (tests/golden/golden.json, made by
    tests/golden/make_golden.py from oracle/_ref)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
            g = json.load(f)
    except Exception:
        return {}, None
    key = "cavity64" if (c0 and n == 64) else ("cavity512_s200" if (n == 512 and sweeps == 200 and not c0) else None)
    if key is None or key not in g:
        return {}, None
    return {int(k): v for k, v in g[key]["checksums"].items()}, key


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------
# CPU baseline: the reference compiled in place, bounded sample
# ---------------------------------------------------------------------------
def reference_steps(n, sweeps, threads, steps, warmup=0, budget_s=None, log=None, c0=False):
    """Times the reference's own implementation (oracle/_ref/libsfref.so, the
    unmodified stencilforge compiled in place) on full steps of the workload:
    each timed unit is one complete cfd::simulation::step (cfd.hpp:307-316;
    compute_dt, provisional, the whole pressure loop of `sweeps` half-sweeps,
    refresh(p)) through the reference executor with `threads` worker threads,
    as the reference's own bench times sim.advance (bench.hpp:68-80).  Nothing
    is projected.  `budget_s` caps the timed steps (at least one) so a slow
    host still ends within the driver's step limit; the steps actually timed
    are returned."""
    from oracle.oracle import Oracle, available, cavity_case
    kind = "reference" if available("ref") else "port"
    t0 = time.time()
    wk = threads if kind == "reference" else 1
    case = (cavity_case(n, symmetry_z=False, workers=wk) if c0 else
            cavity_case(n, symmetry_z=False, omega=1.9525, tolerance=1e-30, max_sweeps=sweeps, workers=wk))
    o = Oracle(case, "ref" if kind == "reference" else "port")
    o.init_cavity()
    setup = time.time() - t0
    for q in range(warmup):
        t1 = time.perf_counter()
        o.step()
        if log:
            log(f"reference warm-up step {q}: {time.perf_counter() - t1:.2f}s")
    per_step = []
    t_start = time.perf_counter()
    for q in range(steps):
        t1 = time.perf_counter()
        _, sw, _ = o.step()
        per_step.append(time.perf_counter() - t1)
        if log:
            log(f"reference step {q}: {per_step[-1]:.2f}s, {sw} half-sweeps")
        if budget_s and q + 1 < steps:
            mean = (time.perf_counter() - t_start) / (q + 1)
            if time.perf_counter() - t_start + mean > budget_s:
                break
    o.close()
    return kind, per_step, setup


def cpu_threads(args):
    if args.cpu_threads:
        return args.cpu_threads
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def weak_extents(n, world):
    """Global grid with an n^3 block per rank: double x, y, z in turn per factor
    of two (2: 2n x n x n, 4: 2n x 2n x n, 8: (2n)^3), the weak-scaling configs
    of BASELINE.json configs[2]; grid::decompose then picks exactly that grid."""
    p, w, a = [1, 1, 1], world, 0
    while w % 2 == 0:
        p[a % 3] *= 2
        w //= 2
        a += 1
    p[0] *= w
    return tuple(n * q for q in p)


def run_ours(args):
    import torch

    import paper_1201_2118_b200 as sfb

    rank, world, local = dist_env()
    dev = local
    torch.cuda.set_device(dev)
    c0 = args.config == "c0"
    if c0:
        args.n, args.sweeps = (64 if args.n == 512 else args.n), 500
    n, S = args.n, args.sweeps
    fused = {"tma": 1, "tma1": 3, "ldg": 2, "unfused": 0}[args.variant]
    dist = None
    if world > 1 or args.force_dist:  # one rank per GPU over NCCL, weak scaling: n^3 per rank
        import torch.distributed as dist
        if "RANK" not in os.environ:  # --force-dist without a launcher: a one-rank job
            os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        uid = [sfb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ext = (args.strong,) * 3 if args.strong else weak_extents(n, world)
        # the temporal pass reads 2-deep halos across processor faces
        ghost = 2 if fused == 1 else 1
        d = sfb.decompose(ext, world, ghost)
        if not args.strong:
            assert all(d.size(w) == (n, n, n) for w in range(world)), d
        cfg = cavity_cfg(sfb, n, S)
        cfg.extents = ext
        sim = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), device=dev, fused=fused, rank=rank, world=world,
                             nccl_id=uid[0], ghost=ghost)
    else:
        ghost = 1
        if args.strong:
            n = args.strong
        cfg = cavity_cfg(sfb, n, S, c0)
        sim = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), workers=1, device=dev, fused=fused, precision=args.dtype)
    if args.strong:  # this rank's block of the fixed global grid
        cells = 1
        for a in sim.block_shape():
            cells *= a
        total_cells = args.strong ** 3
    else:
        cells = n * n * n          # per rank
        total_cells = cells * world
    sim.init_cavity()
    stream = torch.cuda.ExternalStream(sim.stream, device=dev)

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if dist is not None:
            dist.barrier()

    # ---- parity: the first steps from rest against the reference's checksums --
    golden, gkey = (golden_checksums(n, S, c0) if (world == 1 and not args.strong and args.dtype == "f64")
                    else ({}, None))
    parity = {"ok": None, "golden": gkey,
              "note": ("fp32 variant: compared with the fp64 reference under stated per-field tolerances "
                       "(tests/test_gpu_fp32.py), not by checksum" if args.dtype == "f32" else
                       "no reference checksum for this configuration (multi-rank and strong-scaling grids are "
                       "pinned by tests/test_gpu_*: grid components, cross-process transport, path equivalence)")}
    done = 0
    if golden and not c0:  # warm-up steps 1 and 2 are checked (untimed)
        got = {}
        for k in sorted(golden):
            while done < k:
                sim.step()
                done += 1
            got[k] = sim.checksum()
        parity = {"ok": all(got[k] == golden[k] for k in golden), "golden": gkey,
                  "checked": {str(k): {"checksum": got[k], "reference": golden[k]} for k in sorted(golden)}}
    for _ in range(max(0, args.warmup - done)):
        sim.step()
    if c0:  # configs[0] is timed from rest: the warm-up ran on the same grid, start over
        sim.init_cavity()

    # ---- device-timed region: K full steps, inputs resident in HBM -------------
    clocks = ClockSampler(dev)
    # per-launch CUDA events around the dominant kernel, except on small grids:
    # there the persistent pressure loop (one launch per loop)
    # is what runs, and per-launch timing would swap in the launch-per-sweep path
    small = cells <= 4.0e5
    sim.set_kernel_timing(not small)
    sim.launch_count(reset=True)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    stats = [sim.step() for _ in range(args.steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    launches = sim.launch_count()
    # the dominant kernel: the temporal pass where it ran, else the half-sweep;
    # both move 80 algorithmic bytes per cell per launch (read S0, write S2)
    kname = "sweep2" if sim.kernel_timing("sweep2")[1] > 0 else ("loop" if small else "sweep_div")
    k_ms, k_n = sim.kernel_timing(kname) if not small else (0.0, 0)
    k_ms = max_over_ranks(k_ms)
    sim.set_kernel_timing(False)
    ms_per_step = ms_total / args.steps
    value = total_cells * args.steps / (ms_total / 1e3) / 1e6
    sweeps_done = sum(s.sweeps for s in stats)
    if c0:
        if args.steps in golden:  # the timed steps themselves, from rest
            got = sim.checksum()
            parity = {"ok": got == golden[args.steps], "golden": gkey,
                      "checked": {str(args.steps): {"checksum": got, "reference": golden[args.steps]}}}
    else:
        assert sweeps_done == S * args.steps, "fixed-work config must run exactly max_sweeps per step"

    peak, peak_src = measured_peaks()
    avg_launch_s = (k_ms / k_n) / 1e3 if k_n else None
    # 80 algorithmic bytes per cell per half-sweep; a temporal
    # pass processes two half-sweeps per launch (its DRAM traffic is half of
    # that: the first sweep's state never leaves the SM, see dram_* below)
    units = 2 if kname == "sweep2" else 1
    es = 4 if args.dtype == "f32" else 8
    algo_launch = BYTES_PER_HALF_SWEEP * es // 8 * units * cells
    achieved = (algo_launch / avg_launch_s / 1e9) if avg_launch_s else None
    traffic, traffic_src = ncu_traffic(kname, algo_launch)
    step_bytes = (BYTES_UV + BYTES_DIV + BYTES_PER_HALF_SWEEP * sweeps_done / args.steps) * es / 8 * cells
    if small:  # the whole step stands in for the kernel (L2-resident, launch/latency-bound regime)
        achieved = step_bytes / (ms_per_step / 1e3) / 1e9
    roofline = {
        "bound": "hbm",
        "kernel": ("temporal pass, two fused half-sweeps per pass (one walled component in one process: k_sweep2i "
                   "over the interior tiles beside k_sweep2 over the z / y slabs and its x-slab form over the x "
                   "slabs, concurrent; else k_sweep2)" if kname == "sweep2"
                   else "whole step: persistent pressure loop k_pressure_loop (grid L2-resident; achieved = "
                        "step algorithmic bytes / step time)" if small
                   else "k_sweep_div (fused half-sweep)"),
        "achieved": round(achieved, 1) if achieved else None, "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4) if achieved else None,
        "traffic": traffic,
        "traffic_source": traffic_src,
        "half_sweeps_per_launch": units,
        "algorithmic_bytes_per_launch": algo_launch,
        "avg_launch_ms": round(k_ms / k_n, 4) if k_n else None, "launches_timed": k_n,
        "peak_source": peak_src,
        # bytes the kernel actually moves (ncu DRAM traffic per launch) over the same time
        "dram_gbs": round(traffic / avg_launch_s / 1e9, 1) if (traffic and avg_launch_s) else None,
        "dram_frac": round(traffic / avg_launch_s / 1e9 / peak, 4) if (traffic and avg_launch_s) else None,
        "step_achieved_gbs": round(step_bytes / (ms_per_step / 1e3) / 1e9, 1),
        "step_frac": round(step_bytes / (ms_per_step / 1e3) / 1e9 / peak, 4),
    }

    # ---- end to end through the public API with host buffers -------------------
    e2e = None
    if not args.no_e2e:
        # each rank moves its own block (sf_sim_scatter_block / gather_block);
        # at N=1 the block is the whole grid
        names = ("vx", "vy", "vz", "p")
        host_in = {f: torch.from_numpy(sim.gather_block(f)).reshape(-1).pin_memory() for f in names}
        host_out = {f: torch.empty(cells, dtype=torch.float64).pin_memory() for f in names}
        # asynchronous transfers: step k+1's inputs are staged (H2D into the
        # fields' upload buffers, sf_sim_stage_block_async) while step k
        # computes and installed in stream order when step k+1 begins
        # (sf_sim_install_staged); step k's results are snapshotted on the
        # device and drain to the host while step k+1 computes
        # (sf_sim_gather_block_async). PCIe is full duplex.
        for f in names:  # one untimed warm trip
            sim.scatter_block(f, host_in[f], wait=False)
        sim.step()
        for f in names:
            sim.gather_block(f, out=host_out[f], wait=False)
        sim.synchronize()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(stream)
        for f in names:  # step 0's inputs
            sim.stage_block(f, host_in[f])
        for k in range(args.steps):
            for f in names:
                sim.install_staged(f)
            if k + 1 < args.steps:
                for f in names:
                    sim.stage_block(f, host_in[f])
            sim.step()
            for f in names:
                sim.gather_block(f, out=host_out[f], wait=False)
        sim.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e_ms = max(e0.elapsed_time(e1), 0.0)
        e_ms = max_over_ranks(max(e_ms, wall * 1e3))  # host-side copies can run outside the events
        e2e = {"value": round(total_cells * args.steps / (e_ms / 1e3) / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * total_cells * 8, "d2h_bytes_per_step": 4 * total_cells * 8,
               "ms_per_step": round(e_ms / args.steps, 3),
               "path": "per rank and step: sf_sim_install_staged(vx,vy,vz,p) -> sf_sim_stage_block_async(next step's vx,vy,vz,p from pinned host) -> sf_sim_step -> sf_sim_gather_block_async(vx,vy,vz,p to pinned host); uploads cross PCIe during the previous step and are installed by a kernel, downloads are device snapshots drained while the next step computes"}

    # ---- CPU baseline (rank 0, N=1): the reference on this host, one full step --
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        th = cpu_threads(args)
        kind, per, setup = reference_steps(n, S, th, steps=1, c0=c0)
        cpu = {"value": round(cells / per[0] / 1e6, 4), "unit": UNIT, "cores": th,
               "kind": "reference" if kind == "reference" else "port",
               "sample": (f"one full step of the same {n}^3 cavity ({S} half-sweeps) from rest through the "
                          f"reference executor with {th} worker threads, measured: {per[0]:.1f}s"),
               "ms_per_step": round(per[0] * 1e3, 1)}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None,
        "dtype": args.dtype if args.workload == "cavity" else "f64",
        "data": "synthetic (lid-driven cavity from rest, init_cavity)",
        "config": {"workload": (f"configs[0]: 3D lid-driven cavity {n}^3 fp64, ghost 1, the reference oracle run "
                                f"(default solver config: tolerance 1e-6, up to 500 half-sweeps per step), "
                                f"{args.steps} steps from rest" if c0 else
                                f"3D lid-driven cavity {args.strong}^3 fp64 global grid, strong scaling over {world} B200 (BASELINE.json configs[3]), {S} half-sweeps per step"
                                if args.strong else
                                f"3D lid-driven cavity {n}^3 {'fp64' if es == 8 else 'fp32'}, {S} pressure half-sweeps per step (BASELINE.json configs[1]{'' if es == 8 else '-shaped'}; runs/bench128.cfg fixed-work pattern)"
                                if world == 1 else
                                f"3D lid-driven cavity, {n}^3 per GPU weak scaling, global {list(cfg.extents)} block-decomposed over {world} B200 with NCCL ghost exchange (BASELINE.json configs[2]), {S} half-sweeps per step"),
                   "grid": list(cfg.extents), "ghost": ghost, "sweeps_per_step": S,
                   "parallelism": "1 GPU" if world == 1 else f"{world} ranks, block decomposition (grid::decompose), NCCL halo + allreduce",
                   "path": {"tma": "TMA pipeline, temporal pass (two half-sweeps per launch)" if kname == "sweep2"
                            else "fused half-sweep, TMA pipeline",
                            "tma1": "fused half-sweep, TMA pipeline", "ldg": "fused half-sweep, plain loads",
                            "unfused": "unfused (reference dataflow)"}[args.variant],
                   "l2": "inputs larger than L2: 9 resident %s arrays of %.2f GB" % (args.dtype, cells * es / 1e9)},
        "half_sweep_rate": round(total_cells * sweeps_done / (ms_total / 1e3) / 1e6, 1),
        "parity": parity,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        sim.close()
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    c0 = args.config == "c0"
    if c0:
        args.n, args.sweeps = (64 if args.n == 512 else args.n), 500
    n, S = args.n, args.sweeps
    cells = n * n * n
    th = cpu_threads(args)
    # full steps, nothing projected; one warm-up step (a CPU has no clocks or
    # caches to settle beyond first touch, which init_cavity already did) and a
    # wall budget so K steps of ~35 s each end inside the driver's step limit
    warm = min(args.warmup, 1)
    log = (lambda m: print(m, file=sys.stderr, flush=True))
    kind, tsteps, setup = reference_steps(n, S, th, steps=args.steps, warmup=warm, budget_s=args.ref_budget, log=log,
                                         c0=c0)
    ms = 1e3 * sum(tsteps) / len(tsteps)
    value = cells * len(tsteps) / sum(tsteps) / 1e6
    sample = (f"{len(tsteps)} full steps (of {args.steps} requested) of the {n}^3 cavity, {S} half-sweeps each, "
              f"through the reference executor ({th} worker threads), after {warm} warm-up step; each step "
              f"timed whole (cfd::simulation::step), nothing projected")
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
        "steps": len(tsteps), "warmup": warm, "ms_per_step": round(ms, 1),
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (lid-driven cavity from rest, init_cavity)",
        "config": {"workload": (f"configs[0]: 3D lid-driven cavity {n}^3 fp64, ghost 1, the reference oracle run "
                                f"(default solver config: tolerance 1e-6, up to 500 half-sweeps per step)" if c0 else
                                f"3D lid-driven cavity {n}^3 fp64, {S} pressure half-sweeps per step (BASELINE.json configs[1]; runs/bench128.cfg fixed-work pattern)"),
                   "grid": [n, n, n], "ghost": 1, "sweeps_per_step": S, "parallelism": f"{th} CPU worker threads",
                   "build": "oracle/Makefile: g++ -std=c++20 -O3 -march=x86-64-v3 -ffp-contract=off -pthread (the "
                            "reference CMake uses -march=native; x86-64-v3 so the library built here runs on the "
                            "bench host)"},
        "impl": "reference",
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": th,
                         "kind": "reference" if kind == "reference" else "port", "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": round(setup, 1),
    }
    print(json.dumps(line), flush=True)


LAP_BODIES = {  # written against sf_real: fp64, or fp32 when both fields are fp32 (--dtype f32)
    2: """
  const auto& f = c.field(0);
  const sf_real c0 = -2.5, c1 = (sf_real)(4.0 / 3.0), c2 = (sf_real)(-1.0 / 12.0);
  sf_real sx = c1 * (f(-1, 0, 0) + f(1, 0, 0)) + c2 * (f(-2, 0, 0) + f(2, 0, 0));
  sf_real sy = c1 * (f(0, -1, 0) + f(0, 1, 0)) + c2 * (f(0, -2, 0) + f(0, 2, 0));
  sf_real sz = c1 * (f(0, 0, -1) + f(0, 0, 1)) + c2 * (f(0, 0, -2) + f(0, 0, 2));
  c.field(1).store(((sf_real)3 * c0) * f.load() + ((sx + sy) + sz));
""",
    3: """
  const auto& f = c.field(0);
  const sf_real c0 = (sf_real)(-49.0 / 18.0), c1 = 1.5, c2 = (sf_real)(-0.15), c3 = (sf_real)(1.0 / 90.0);
  sf_real s[3];
  for (int a = 0; a < 3; ++a) {
    const int x = a == 0, y = a == 1, z = a == 2;
    s[a] = c1 * (f(-x, -y, -z) + f(x, y, z)) + c2 * (f(-2 * x, -2 * y, -2 * z) + f(2 * x, 2 * y, 2 * z))
         + c3 * (f(-3 * x, -3 * y, -3 * z) + f(3 * x, 3 * y, 3 * z));
  }
  c.field(1).store(((sf_real)3 * c0) * f.load() + ((s[0] + s[1]) + s[2]));
""",
}


def run_stencil(args):
    """configs[4]: a ghost-width-2/3 stencil declared as an execution plan +
    point-function body (the reference's user-kernel path, executor.hpp:484),
    JIT-compiled for sm_100a.  One step = exchange(u) + run_kernel over the grid.
    Algorithmic bytes: read u, write lu = 16 B/cell in fp64, 8 in fp32
    (--dtype f32: fields stored in fp32, point function computes in fp64)."""
    import numpy as np
    import torch

    import paper_1201_2118_b200 as sfb

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    n = args.n if args.n != 512 else 768
    r = args.radius
    tile = tuple(int(x) for x in args.tile.split(","))
    cfg = sfb.SolverConfig(extents=(n, n, n), periodic=(True, True, True))
    sim = sfb.Simulation(cfg, sfb.FluidParams(), workers=1, ghost=r, device=local)
    es = 4 if args.dtype == "f32" else 8
    sim.create_field("u", dtype=args.dtype)
    sim.create_field("lu", dtype=args.dtype)
    sim.scatter("u", np.random.default_rng(1).uniform(-1, 1, size=(n, n, n)))
    name = f"LAP{2 * r}"
    sim.register_kernel(sfb.ExecutionPlan(name, tile, (r,) * 6, [("u", "IN", True), ("lu", "OUT")]),
                        (["u", "lu"], []), LAP_BODIES[r])
    stream = torch.cuda.ExternalStream(sim.stream, device=local)
    for _ in range(args.warmup):
        sim.exchange(["u"])
        sim.run_kernel(name)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local)
    clocks.start()
    sim.launch_count(reset=True)
    e0.record(stream)
    kms = 0.0
    for _ in range(args.steps):
        sim.exchange(["u"])
        k0.record(stream)
        sim.run_kernel(name)
        k1.record(stream)
        k1.synchronize()
        kms += k0.elapsed_time(k1)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    cells = n ** 3
    peak, src = measured_peaks()
    ach = 2.0 * es * cells / (kms / args.steps / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": round(cells * args.steps / (ms / 1e3) / 1e6, 2), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (uniform random field)",
        "config": {"workload": f"configs[4]: radius-{r} Laplacian ({6 * r + 1}-point, order {2 * r}) at {n}^3 {'fp32' if es == 4 else 'fp64'}, "
                               f"ghost width {r}, descriptor TILE {tile}, periodic, exchange + run_kernel per step",
                   "grid": [n, n, n], "ghost": r, "tile": list(tile)},
        "roofline": {"bound": "hbm", "kernel": f"sf_user_kernel ({name}, NVRTC)", "achieved": round(ach, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": None,
                     "algorithmic_bytes_per_launch": 2 * es * cells, "avg_launch_ms": round(kms / args.steps, 4),
                     "peak_source": src},
        "gpu_launches": sim.launch_count(), "clocks": clk,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.workload == "stencil":
        run_stencil(args)
        return
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
