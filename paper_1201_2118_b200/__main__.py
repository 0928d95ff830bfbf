"""Command-line front end: ``python -m paper_1201_2118_b200 <command>``, the
``sforge`` commands on the path (proj/tools/sforge.cpp):

  gen <file.ccl> -o <dir>            descriptors -> <kernel>.h.generated + plans.txt
  cavity --config <file> [--workers N] [--mode plain|overlap] [--tile tx,ty,tz]
                                     the lid-driven cavity to steady state on the GPU
  validate --profiles <csv> --reference <csv> --tol <t>
                                     centerline profiles against a reference table
  bench --config <file> [--workers 1,2,4] [--modes plain,overlap] [--steps N] [--out bench.csv]
                                     the fixed-step benchmark table and CSV

Same output lines, files and exit status (0 ok, 1 run or validation failure,
2 usage error) as the reference's CLI. ``--mode`` and ``--tile`` select the
reference's CPU execution strategy; they are accepted and do not change the
device run (results are mode- and tile-invariant in the reference too).
"""
from __future__ import annotations

import bisect
import os
import sys

EXIT_OK, EXIT_FAILURE, EXIT_USAGE = 0, 1, 2

SYNOPSIS = """usage: sforge <command> [options]

commands:
  gen <file.ccl> -o <dir>
      parse kernel descriptors, write <kernel>.h.generated files and plans.txt
  cavity --config <file> [--workers N] [--mode plain|overlap] [--tile tx,ty,tz]
      run the lid-driven cavity to steady state, write profile and residual CSVs
  validate --profiles <csv> --reference <csv> --tol <t>
      compare centerline profiles against a reference table
  bench --config <file> [--workers 1,2,4] [--modes plain,overlap] [--steps N]
        [--out bench.csv]
      fixed-step strong-scaling benchmark

exit status: 0 success, 1 run or validation failure, 2 usage error
"""


class UsageError(Exception):
    pass


class ValidateError(Exception):
    """cli::validate_error (validate.hpp:24-27)."""


def _flag_value(args, i, flag):
    if i + 1 >= len(args):
        raise UsageError(flag + " needs a value")
    return args[i + 1]


def _parse_long(v, what):
    from .config import _INT
    m = _INT.fullmatch(v.lstrip(" \t\n\v\f\r"))
    if not m or not -2 ** 63 <= int(v) < 2 ** 63:
        raise UsageError("bad %s '%s'" % (what, v))
    return int(v)


def _parse_double(v, what):
    from .config import _strtod_prefix
    val, used = _strtod_prefix(v)
    if val is None or val == "range" or used != len(v):
        raise UsageError("bad %s '%s'" % (what, v))
    return val


def cmd_gen(args):
    from . import descriptor as D
    inp, outdir = "", ""
    i = 0
    while i < len(args):
        a = args[i]
        if a in ("-o", "--out"):
            outdir = _flag_value(args, i, a)
            i += 1
        elif a.startswith("-"):
            raise UsageError("unknown option '%s'" % a)
        elif not inp:
            inp = a
        else:
            raise UsageError("unexpected argument '%s'" % a)
        i += 1
    if not inp:
        raise UsageError("gen needs a descriptor file")
    if not outdir:
        raise UsageError("gen needs -o <dir>")
    try:
        with open(inp, "rb") as f:
            text = f.read().decode("latin-1")
    except OSError:
        sys.stderr.write("sforge: cannot open '%s'\n" % inp)
        return EXIT_FAILURE
    raw = D.parse_descriptors(text)
    fields = {n for k in raw for g in k.groups if not g.parameter for n in g.names}
    kernels = D.validate_all(raw, fields)
    written = D.write_generated(kernels, outdir)
    for p in written:
        print("wrote " + p)
    print("%d kernel%s, %d files" % (len(kernels), "" if len(kernels) == 1 else "s", len(written)))
    return EXIT_OK


def cmd_cavity(args):
    from .cavity import centerline_profiles, dump_fields, run_to_steady, write_profiles, write_residuals
    from .config import load_run_config
    from .sim import Simulation
    config_path, workers, mode, tile = "", 0, None, None
    i = 0
    while i < len(args):
        a = args[i]
        if a == "--config":
            config_path = _flag_value(args, i, a)
        elif a == "--workers":
            workers = _parse_long(_flag_value(args, i, a), "--workers")
            if workers < 1:
                raise UsageError("--workers must be at least 1")
        elif a == "--mode":
            mode = _flag_value(args, i, a)
            if mode not in ("plain", "overlap"):
                raise UsageError("mode must be plain or overlap, got '%s'" % mode)
        elif a == "--tile":
            parts = _flag_value(args, i, a).split(",")
            if len(parts) != 3:
                raise UsageError("--tile needs tx,ty,tz")
            tile = tuple(_parse_long(p, "tile extent") for p in parts)
            if any(t < 0 for t in tile):
                raise UsageError("tile extents must be non-negative")
        else:
            raise UsageError("unknown option '%s'" % a)
        i += 2 if a in ("--config", "--workers", "--mode", "--tile") else 1
    if not config_path:
        raise UsageError("cavity needs --config <file>")
    rc = load_run_config(config_path)
    if workers:
        rc.workers = workers
    if mode:
        rc.mode = mode
    if tile:
        rc.tile = tile
    sim = Simulation(rc.solver(), rc.fluid(), workers=rc.workers, ghost=rc.ghost)
    sim.init_cavity()
    print("cavity %dx%dx%d  Re=%g  workers=%d  mode=%s" % (rc.nx, rc.ny, rc.nz, rc.re, rc.workers, rc.mode))
    rows = []
    stop_rate = rc.steady_tol * rc.lid_speed

    def on_step(n, st, rate):
        rows.append((n, st))
        if rc.output_cadence > 0 and n % rc.output_cadence == 0:
            print("  step %d  t=%.4f  dt=%.3e  sweeps=%d  div=%.3e  rate=%.3e" % (
                n, sim.time, st.dt, st.sweeps, st.residual, rate))

    summary = run_to_steady(sim, rc.max_steps, stop_rate, on_step)
    with open(rc.residuals_out, "w", newline="") as f:
        f.write(write_residuals(rows))
    print("wrote " + rc.residuals_out)
    u, v = centerline_profiles(sim, rc.lid_speed)
    comment = "lid-driven cavity centerline profiles: %dx%dx%d, Re=%g, t=%.6g, steps=%d" % (
        rc.nx, rc.ny, rc.nz, rc.re, sim.time, summary.steps)
    with open(rc.profiles_out, "w", newline="") as f:
        f.write(write_profiles(u, v, [comment]))
    print("wrote " + rc.profiles_out)
    if rc.fields_out:
        for p in dump_fields(sim, rc.fields_out):
            print("wrote " + p)
    last = rows[-1][1].residual if rows else 0.0
    print("steps=%d  t=%.6g  rate=%.3e  max|div|=%.3e" % (summary.steps, summary.time, summary.rate, last))
    sys.stdout.flush()
    if not summary.converged:
        sys.stderr.write("sforge: not steady after %d steps (rate %s > %s)\n" % (
            summary.steps, _ostream_double(summary.rate), _ostream_double(stop_rate)))
        return EXIT_FAILURE
    print("steady state reached")
    return EXIT_OK


def _ostream_double(x: float) -> str:
    """std::ostream << double (default precision 6, %g style)."""
    return "%g" % x


def read_profiles(text: str, what: str):
    """cli::read_profiles (validate.hpp:31-79), with its error texts."""
    u, v, sec = [], [], None
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines = lines[:-1]
    for n, raw in enumerate(lines, start=1):
        if raw.endswith("\r"):
            raw = raw[:-1]
        t = raw.strip(" \t")
        if not t or t.startswith("#"):
            continue
        if t == "y,u":
            sec = u
            continue
        if t == "x,v":
            sec = v
            continue

        def fail(why):
            raise ValidateError("%s, line %d: %s" % (what, n, why))

        if sec is None:
            fail("expected a 'y,u' or 'x,v' header before data rows")
        comma = t.find(",")
        if comma < 0:
            fail("expected 'coordinate,value'")
        from .config import _strtod_prefix
        first, second = t[:comma], t[comma + 1:]
        c, used = _strtod_prefix(first)
        if c is None or c == "range":
            fail("malformed number in '%s'" % t)
        if used != len(first):
            fail("trailing characters in coordinate")
        val, used = _strtod_prefix(second)
        if val is None or val == "range":
            fail("malformed number in '%s'" % t)
        if used != len(second):
            fail("trailing characters in value")
        if sec and not c > sec[-1][0]:
            fail("coordinates must be strictly increasing")
        sec.append((c, val))
    if len(u) < 2 or len(v) < 2:
        raise ValidateError(what + ": each section needs at least two rows")
    return u, v


def compare_profiles(computed, reference):
    """cli::compare_profiles (validate.hpp:137-157): rows (section, coord,
    computed, reference, |diff|) and the max deviation."""
    rows, worst = [], 0.0
    for comp, ref, tag, what in ((computed[0], reference[0], "u", "u(y) section"),
                                 (computed[1], reference[1], "v", "v(x) section")):
        xs = [r[0] for r in comp]
        for x, want in ref:
            if x < xs[0] or x > xs[-1]:
                raise ValidateError("%s: reference coordinate %f is outside the computed profile range" % (what, x))
            k = bisect.bisect_left(xs, x)
            if xs[k] == x:
                got = comp[k][1]
            else:
                lo, hi = comp[k - 1], comp[k]
                t = (x - lo[0]) / (hi[0] - lo[0])
                got = lo[1] + t * (hi[1] - lo[1])
            d = abs(got - want)
            worst = max(worst, d)
            rows.append((tag, x, got, want, d))
    return rows, worst


def cmd_validate(args):
    prof, ref, tol = "", "", -1.0
    i = 0
    while i < len(args):
        a = args[i]
        if a == "--profiles":
            prof = _flag_value(args, i, a)
        elif a == "--reference":
            ref = _flag_value(args, i, a)
        elif a == "--tol":
            tol = _parse_double(_flag_value(args, i, a), "--tol")
            if not tol >= 0.0:
                raise UsageError("--tol must be non-negative")
        else:
            raise UsageError("unknown option '%s'" % a)
        i += 2
    if not prof or not ref or tol < 0.0:
        raise UsageError("validate needs --profiles, --reference, and --tol")

    def load(path):
        try:
            with open(path, newline="") as f:
                text = f.read()
        except OSError:
            raise ValidateError("cannot open profile file '%s'" % path) from None
        return read_profiles(text, path)

    rows, worst = compare_profiles(load(prof), load(ref))
    out = ["section,coord,computed,reference,abs_deviation\n"]
    out += ["%s,%.6g,%.9g,%.9g,%.9g\n" % r for r in rows]
    out.append("max abs deviation: %.9g\n" % worst)
    out.append("tolerance: %g\n" % tol)
    sys.stdout.write("".join(out))
    if worst <= tol:
        print("PASS")
        return EXIT_OK
    print("FAIL")
    return EXIT_FAILURE


def cmd_bench(args):
    """sforge bench (sforge.cpp:296-349, bench.hpp:46-143) on the device:
    `workers` grid components on one GPU, each (workers, mode) run timed over
    advance(steps) after a device synchronisation on both sides. The
    reference's `bytes_staged` column (its executor's tile-staging ledger) is
    the device path's algorithmic HBM traffic, 56 + 32 + 80 * sweeps bytes per
    cell and step."""
    import time

    from .config import load_run_config
    from .sim import Simulation
    config_path, out_path, steps = "", "bench.csv", 20
    workers, modes = [1, 2, 4], ["plain", "overlap"]
    i = 0
    while i < len(args):
        a = args[i]
        if a == "--config":
            config_path = _flag_value(args, i, a)
        elif a == "--workers":
            workers = []
            for part in _flag_value(args, i, a).split(","):
                w = _parse_long(part, "--workers")
                if w < 1:
                    raise UsageError("--workers entries must be at least 1")
                workers.append(w)
        elif a == "--modes":
            modes = []
            for part in _flag_value(args, i, a).split(","):
                if part not in ("plain", "overlap"):
                    raise UsageError("mode must be plain or overlap, got '%s'" % part)
                modes.append(part)
        elif a == "--steps":
            steps = _parse_long(_flag_value(args, i, a), "--steps")
            if steps < 1:
                raise UsageError("--steps must be at least 1")
        elif a == "--out":
            out_path = _flag_value(args, i, a)
        else:
            raise UsageError("unknown option '%s'" % a)
        i += 2
    if not config_path:
        raise UsageError("bench needs --config <file>")
    rc = load_run_config(config_path)
    rows = []
    for w in workers:
        for mode in modes:
            sim = Simulation(rc.solver(), rc.fluid(), workers=w, mode=mode, ghost=rc.ghost)
            sim.init_cavity()
            sim.synchronize()
            sweeps = 0
            t0 = time.perf_counter()
            for _ in range(steps):
                sweeps += sim.step().sweeps
            sim.synchronize()
            wall = time.perf_counter() - t0
            cells = rc.nx * rc.ny * rc.nz
            rows.append({"workers": w, "mode": mode, "ext": (rc.nx, rc.ny, rc.nz), "steps": steps, "wall": wall,
                         "ups": cells * steps / wall if wall > 0 else 0.0,
                         "bytes": cells * ((56 + 32) * steps + 80 * sweeps), "checksum": sim.checksum()})
            sim.close()
    for r in rows:
        base = min((o for o in rows if o["mode"] == r["mode"]), key=lambda o: o["workers"])
        r["speedup"] = 1.0 if base is r else (base["wall"] / r["wall"] if r["wall"] > 0 else 1.0)
    print("%8s %8s %14s %7s %10s %14s %8s %14s  %s" % ("workers", "mode", "grid", "steps", "wall[s]", "updates/s",
                                                       "speedup", "bytes staged", "checksum"))
    for r in rows:
        print("%8d %8s %14s %7d %10.3f %14.4g %8.2f %14d  %s" % (
            r["workers"], r["mode"], "%dx%dx%d" % r["ext"], r["steps"], r["wall"], r["ups"], r["speedup"],
            r["bytes"], r["checksum"]))
    with open(out_path, "w", newline="") as f:
        f.write("workers,mode,nx,ny,nz,steps,wall_seconds,updates_per_second,speedup,bytes_staged,checksum\n")
        for r in rows:
            f.write("%d,%s,%d,%d,%d,%d,%.6f,%.6g,%.4f,%d,%s\n" % (
                r["workers"], r["mode"], r["ext"][0], r["ext"][1], r["ext"][2], r["steps"], r["wall"], r["ups"],
                r["speedup"], r["bytes"], r["checksum"]))
    print("wrote " + out_path)
    sys.stdout.flush()
    mismatch = False
    for a in rows:
        for b in rows:
            if a["workers"] == b["workers"] and a["checksum"] != b["checksum"]:
                sys.stderr.write("sforge: checksum mismatch at %d workers: %s=%s vs %s=%s\n" % (
                    a["workers"], a["mode"], a["checksum"], b["mode"], b["checksum"]))
                mismatch = True
    return EXIT_FAILURE if mismatch else EXIT_OK


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    if not argv:
        sys.stderr.write(SYNOPSIS)
        return EXIT_USAGE
    cmd, args = argv[0], argv[1:]
    try:
        if cmd == "gen":
            return cmd_gen(args)
        if cmd == "cavity":
            return cmd_cavity(args)
        if cmd == "validate":
            return cmd_validate(args)
        if cmd == "bench":
            return cmd_bench(args)
        if cmd in ("-h", "--help", "help"):
            sys.stdout.write(SYNOPSIS)
            return EXIT_OK
        raise UsageError("unknown command '%s'" % cmd)
    except UsageError as e:
        sys.stderr.write("sforge: %s\n\n" % e)
        sys.stderr.write(SYNOPSIS)
        return EXIT_USAGE
    except Exception as e:  # noqa: BLE001 -- every other error is a run failure, as in sforge.cpp
        sys.stderr.write("sforge: %s\n" % e)
        return EXIT_FAILURE


if __name__ == "__main__":
    sys.exit(main())
