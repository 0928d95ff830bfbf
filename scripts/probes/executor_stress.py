"""Randomised stress of the plugin path: random descriptor-style kernels (a
weighted sum over random axis-aligned offsets within a random per-face halo),
random TILE, CACHED on/off, fp64 or fp32 fields, 1-4 grid components with
ghost width 1-3 on a periodic box, against numpy doing the same operations in
the same order (bitwise). Test infrastructure only.

  python scripts/probes/executor_stress.py [n_cases] [seed] [max_seconds]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1201_2118_b200 as sfb  # noqa: E402


def one(rng, k):
    g = int(rng.integers(1, 4))
    workers = int(rng.choice([1, 1, 2, 3, 4]))
    ext = tuple(int(rng.integers(2 * g + 4, 40)) for _ in range(3))
    halo = tuple(int(rng.integers(0, g + 1)) for _ in range(6))  # -x +x -y +y -z +z
    offs = [(0, 0, 0)]
    for a in range(3):
        for sd, sign in ((0, -1), (1, 1)):
            for r in range(1, halo[2 * a + sd] + 1):
                if rng.random() < 0.8:
                    o = [0, 0, 0]
                    o[a] = sign * r
                    offs.append(tuple(o))
    rng.shuffle(offs)
    w = [float(rng.uniform(-1, 1)) for _ in offs]
    tile = tuple(int(x) for x in rng.choice([(32, 8, 64), (32, 4, 16), (16, 16, 8), (8, 8, 8), (32, 8, 5), (4, 4, 4),
                                             (64, 2, 32)]))
    cached = bool(rng.integers(0, 2))
    f32 = bool(rng.random() < 0.3)
    dt = np.float32 if f32 else np.float64
    body = "  const auto& f = c.field(0);\n  sf_real s = (sf_real)0;\n"
    for (di, dj, dk), wk in zip(offs, w):
        body += "  s += (sf_real)(%s) * f(%d, %d, %d);\n" % (float.hex(wk), di, dj, dk)
    body += "  c.field(1).store(s);\n"
    cfg = sfb.SolverConfig(extents=ext, periodic=(True, True, True))
    s = sfb.Simulation(cfg, sfb.FluidParams(), workers=workers, ghost=g)
    s.create_field("u", dtype="f32" if f32 else "f64")
    s.create_field("v", dtype="f32" if f32 else "f64")
    data = rng.uniform(-1.0, 1.0, size=ext[::-1]).astype(dt).astype(np.float64)
    s.scatter("u", data)
    s.register_kernel(sfb.ExecutionPlan("K%d" % k, tile, halo, [("u", "IN", cached), ("v", "OUT")]), (["u", "v"], []),
                      body)
    s.exchange(["u"])
    s.run_kernel("K%d" % k)
    got = s.gather("v")
    u = data.astype(dt)
    acc = np.zeros_like(u)
    for (di, dj, dk), wk in zip(offs, w):
        sh = np.roll(u, shift=(-dk, -dj, -di), axis=(0, 1, 2))
        acc = acc + dt(wk) * sh
    want = acc.astype(np.float64)
    ok = np.array_equal(got.view(np.uint64), want.view(np.uint64))
    desc = "ext=%s w=%d g=%d halo=%s tile=%s cached=%d %s offsets=%d" % (ext, workers, g, halo, tile, cached,
                                                                         "f32" if f32 else "f64", len(offs))
    s.close()
    return ok, desc


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    budget = float(sys.argv[3]) if len(sys.argv) > 3 else 600.0
    rng = np.random.default_rng(seed)
    t0 = time.time()
    good = bad = 0
    for k in range(n):
        if time.time() - t0 > budget:
            break
        try:
            ok, desc = one(rng, k)
        except Exception as e:  # noqa: BLE001 -- configurations both sides reject (e.g. blocks vs ghost)
            print("%4d SKIP %s: %s" % (k, type(e).__name__, str(e)[:200]), flush=True)
            continue
        good += ok
        bad += not ok
        print("%4d %s %s" % (k, "OK  " if ok else "DIFF", desc), flush=True)
    print("summary: %d cases, %d bitwise equal, %d differ, %.0f s, seed %d" % (good + bad, good, bad,
                                                                             time.time() - t0, seed))
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
