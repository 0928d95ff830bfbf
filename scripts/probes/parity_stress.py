"""Randomised parity stress run: the device (every pressure-loop path the
configuration selects: persistent loop, temporal pass, fused half-sweeps,
unfused dataflow) against the reference compiled in place, bitwise, on random
cavities (extents, periodicity, ghost width, grid components, random initial
velocities, tolerance- and cap-driven stops). Test infrastructure: uses
oracle/ (the checker). Prints one line per case and a summary.

  python scripts/probes/parity_stress.py [n_cases] [seed] [max_seconds] [case_index | bc]

"bc": random face conditions (moving walls, symmetry, outflow), the fused
paths against the unfused dataflow.
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1201_2118_b200 as sfb  # noqa: E402
from oracle.oracle import Case, Oracle  # noqa: E402


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def gen(rng):
    """All random draws of one case (so a case can be replayed by index)."""
    per = tuple(bool(rng.integers(0, 2)) for _ in range(3)) if rng.random() < 0.3 else (False,) * 3
    workers = int(rng.choice([1, 1, 1, 2, 3, 4]))
    ghost = int(rng.choice([1, 1, 2, 3]))
    lo = 2 * ghost + 2
    top = int(os.environ.get("PS_MAXEXT", "48"))  # larger grids reach the interior/boundary split of the pass
    ext = tuple(int(rng.integers(max(lo, 5), top)) for _ in range(2)) + (int(rng.integers(max(lo, 3), max(top * 5 // 6, 4))),)
    fused = int(rng.choice([1, 1, 3, 2, 0]))
    tol = float(rng.choice([1e-2, 1e-3, 1e-5, 1e-30]))
    maxs = int(rng.integers(1, 80))
    kw = dict(viscosity=float(rng.uniform(0.005, 0.05)))
    kw["lid"] = 0.0 if any(per) else float(rng.uniform(0.2, 1.5))  # drawn only for walled boxes
    kw.update(omega=float(rng.uniform(1.0, 1.95)), sigma=float(rng.uniform(0.2, 0.9)), symz=bool(rng.integers(0, 2)))
    fields = {f: rng.uniform(-0.5, 0.5, size=ext[::-1]) for f in ("vx", "vy", "vz")} if rng.random() < 0.7 else None
    steps = int(rng.integers(1, 4))
    return dict(per=per, workers=workers, ghost=ghost, ext=ext, fused=fused, tol=tol, maxs=maxs, fields=fields,
                steps=steps, **kw)


def run(p, fused=None, detail=False):
    ext, per, workers, ghost = p["ext"], p["per"], p["workers"], p["ghost"]
    fused = p["fused"] if fused is None else fused
    lid = p["lid"]
    c = Case(extents=ext, periodic=per, tolerance=p["tol"], max_sweeps=p["maxs"], viscosity=p["viscosity"],
             lid_speed=lid, workers=workers, ghost=ghost, omega=p["omega"], sigma=p["sigma"], symmetry_z=p["symz"])
    o = Oracle(c, "ref")
    cfg = sfb.SolverConfig(extents=ext, periodic=per, tolerance=p["tol"], max_sweeps=p["maxs"], omega=p["omega"],
                           sigma=p["sigma"], symmetry_z=p["symz"])
    d = sfb.Simulation(cfg, sfb.FluidParams(viscosity=p["viscosity"], lid_speed=lid), workers=workers,
                       ghost=ghost, fused=fused)
    o.init_cavity()
    d.init_cavity()
    if p["fields"]:
        for f, a in p["fields"].items():
            o.scatter(f, a)
            d.scatter(f, a)
        o.invalidate_all_ghosts()
        d.invalidate_all_ghosts()
    so = o.advance(p["steps"])
    dd = [d.step() for _ in range(p["steps"])]
    st_d = [[x.dt, x.sweeps, x.residual] for x in dd]
    st_o = [[float(a), int(b), float(r)] for a, b, r in zip(*so)]
    ok = st_d == st_o
    diff = {}
    for f in ("vx", "vy", "vz", "p"):
        a, b = d.gather(f), o.gather(f)
        e = not np.array_equal(bits(a), bits(b))
        ok = ok and not e
        if e and detail:
            w = np.argwhere(bits(a) != bits(b))
            diff[f] = (len(w), w[:3].tolist(), float(np.nanmax(np.abs(a - b))))
    ok = ok and d.pending_color == o.pending_color
    desc = "ext=%s per=%s w=%d g=%d fused=%d tol=%g maxs=%d steps=%d sweeps=%s" % (
        ext, "".join("1" if q else "0" for q in per), workers, ghost, fused, p["tol"], p["maxs"], p["steps"],
        [x.sweeps for x in dd])
    if detail:
        desc += "\n   device %s\n   oracle %s\n   fields %s" % (st_d, st_o, diff)
    d.close()
    return ok, desc


def run_bc(rng):
    """Random face conditions (moving walls, symmetry, outflow) on random
    velocities: the fused, TMA and temporal paths against the unfused
    reference dataflow (fused=0, itself bitwise with the reference), since the
    reference's simulation fixes its own boundary spec."""
    top = int(os.environ.get("PS_BCMAX", "44"))  # larger grids reach the interior form of the pass
    ext = tuple(int(rng.integers(6, top)) for _ in range(3))
    workers = int(rng.choice([1, 1, 2, 3]))
    ghost = int(rng.choice([1, 2]))
    kinds = ["wall", "symmetry", "outflow"]
    faces = [(a, sd, kinds[int(rng.integers(0, 3))], tuple(rng.uniform(-0.3, 0.3, 3))) for a in range(3)
             for sd in range(2)]
    tol = float(rng.choice([1e-3, 1e-4, 1e-30]))
    maxs = int(rng.integers(1, 40))
    vel = {f: rng.uniform(-0.5, 0.5, size=ext[::-1]) for f in ("vx", "vy", "vz")}
    out = {}
    for fused in (0, 1, 3, 2):
        cfg = sfb.SolverConfig(extents=ext, tolerance=tol, max_sweeps=maxs, symmetry_z=False)
        d = sfb.Simulation(cfg, sfb.FluidParams(viscosity=0.02, lid_speed=0.0), workers=workers, ghost=ghost,
                           fused=fused)
        d.init_cavity()
        for a, sd, k, v in faces:
            d.set_face_bc(a, sd, k, v)
        for f, arr in vel.items():
            d.scatter(f, arr)
        st = [d.step() for _ in range(2)]
        out[fused] = ([[x.dt, x.sweeps, x.residual] for x in st], d.checksum(), d.pending_color)
        d.close()
    ok = out[1] == out[0] and out[3] == out[0] and out[2] == out[0]
    desc = "bc ext=%s w=%d g=%d faces=%s tol=%g maxs=%d sweeps=%s" % (
        ext, workers, ghost, "".join(k[0] for _, _, k, _ in faces), tol, maxs, [r[1] for r in out[0][0]])
    return ok, desc


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2026
    budget = float(sys.argv[3]) if len(sys.argv) > 3 else 900.0
    only = int(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[4] != "bc" else None  # replay one case
    mode = "bc" if "bc" in sys.argv[4:] else "ref"
    rng = np.random.default_rng(seed)
    t0 = time.time()
    good = bad = 0
    for k in range(n):
        if time.time() - t0 > budget:
            break
        if mode == "bc":
            try:
                ok, desc = run_bc(rng)
            except Exception as e:  # noqa: BLE001
                print("%4d SKIP %s: %s" % (k, type(e).__name__, e), flush=True)
                continue
            good += ok
            bad += not ok
            print("%4d %s %s" % (k, "OK  " if ok else "DIFF", desc), flush=True)
            continue
        p = gen(rng)
        if only is not None and k != only:
            continue
        try:
            if only is not None:
                for fz in (p["fused"], 3, 2, 0):
                    print("fused=%d" % fz, run(p, fz, True))
            ok, desc = run(p)
        except Exception as e:  # noqa: BLE001 -- e.g. blocks thinner than the ghost width: rejected at setup
            print("%4d SKIP %s: %s" % (k, type(e).__name__, e), flush=True)
            continue
        good += ok
        bad += not ok
        print("%4d %s %s" % (k, "OK  " if ok else "DIFF", desc), flush=True)
    print("summary: %d cases, %d bitwise equal, %d differ, %.0f s, seed %d" % (good + bad, good, bad,
                                                                             time.time() - t0, seed))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
