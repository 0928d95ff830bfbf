"""Lid-driven cavity harness on the device simulation: the host-side parts of
``sforge cavity`` (proj/tools/sforge.cpp:188-259) around the hot path --
run_to_steady (cfd.hpp:323-338), centerline_profiles (cfd.hpp:403-440) and the
profile / residual CSV formats (validate.hpp:88-102, sforge.cpp:156-174).
The step loop, reductions and gathers run in the CUDA library; this module only
evaluates the same host arithmetic the reference does on the gathered fields.
"""
from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np

from .sim import FluidParams, Simulation, SolverConfig


@dataclass
class RunSummary:  # cfd.hpp:92-97
    steps: int = 0
    time: float = 0.0
    rate: float = 0.0
    converged: bool = False


def run_to_steady(sim: Simulation, max_steps: int, steady_tol: float, on_step=None) -> RunSummary:
    """cfd::simulation::run_to_steady (cfd.hpp:324-338): step until
    steady_delta / dt <= steady_tol."""
    r = RunSummary()
    for _ in range(int(max_steps)):
        st = sim.step()
        r.steps = sim.step_count
        r.time = sim.time
        r.rate = sim.steady_delta() / st.dt
        if on_step:
            on_step(r.steps, st, r.rate)
        if r.rate <= steady_tol:
            r.converged = True
            break
    return r


def centerline_profiles(sim: Simulation, lid_speed: float = 1.0):
    """cfd::simulation::centerline_profiles (cfd.hpp:405-440), same float64 ops."""
    nx, ny, nz = sim.extents
    if nz % 2 == 0:
        raise ValueError("profiles need an odd z extent for an exact mid plane")
    km = nz // 2
    sp = sim.cfg.spacing or [1.0 / float(n) for n in sim.extents]
    gu, gv = sim.gather("vx"), sim.gather("vy")
    u_at = lambda i, j: float(gu[km, j, i])  # noqa: E731
    v_at = lambda i, j: float(gv[km, j, i])  # noqa: E731
    u_of_y = [(0.0, 0.0)]
    for j in range(ny):
        y = (float(j) + 0.5) * sp[1]
        u = u_at(nx // 2 - 1, j) if nx % 2 == 0 else 0.5 * (u_at(nx // 2 - 1, j) + u_at(nx // 2, j))
        u_of_y.append((y, u))
    u_of_y.append((1.0, lid_speed))
    v_of_x = [(0.0, 0.0)]
    for i in range(nx):
        x = (float(i) + 0.5) * sp[0]
        v = v_at(i, ny // 2 - 1) if ny % 2 == 0 else 0.5 * (v_at(i, ny // 2 - 1) + v_at(i, ny // 2))
        v_of_x.append((x, v))
    v_of_x.append((1.0, 0.0))
    return u_of_y, v_of_x


def _g17(x: float) -> str:
    """printf("%.17g") (validate.hpp:94)."""
    return "%.17g" % x


def write_profiles(u_of_y, v_of_x, comments=()) -> str:
    """cli::write_profiles (validate.hpp:88-102)."""
    out = io.StringIO()
    for c in comments:
        out.write("# " + c + "\n")
    out.write("y,u\n")
    for y, u in u_of_y:
        out.write(_g17(y) + "," + _g17(u) + "\n")
    out.write("x,v\n")
    for x, v in v_of_x:
        out.write(_g17(x) + "," + _g17(v) + "\n")
    return out.getvalue()


def write_residuals(rows) -> str:
    """residual_log::write (sforge.cpp:161-173): step,dt,max_div,sweeps."""
    out = io.StringIO()
    out.write("step,dt,max_div,sweeps\n")
    for step, st in rows:
        out.write("%d,%s,%s,%d\n" % (step, _g17(st.dt), _g17(st.residual), st.sweeps))
    return out.getvalue()


SFG1_MAGIC = b"SFG1"


def write_sfg1(out, extents, data) -> None:
    """grid::write_sfg1 (io.hpp:66-84): "SFG1", nx ny nz as little-endian
    int64, then nx*ny*nz little-endian float64 values, x fastest. ``out`` is a
    binary stream or a path."""
    import numpy as np
    from ._lib import GridError
    a = np.ascontiguousarray(data, dtype="<f8").reshape(-1)
    if a.size != int(extents[0]) * int(extents[1]) * int(extents[2]):
        raise GridError(2, "SFG1 write: data size does not match extents")
    blob = SFG1_MAGIC + np.asarray([int(e) for e in extents], dtype="<i8").tobytes() + a.tobytes()
    if isinstance(out, (str, bytes)) or hasattr(out, "__fspath__"):
        with open(out, "wb") as f:
            f.write(blob)
    else:
        out.write(blob)


def read_sfg1(src):
    """grid::read_sfg1 (io.hpp:86-101): returns (extents, values as a
    (nz, ny, nx) float64 array); the same error texts."""
    import numpy as np
    from ._lib import GridError
    if isinstance(src, (str, bytes)) or hasattr(src, "__fspath__"):
        with open(src, "rb") as f:
            blob = f.read()
    else:
        blob = src.read()
    if blob[:4] != SFG1_MAGIC:
        raise GridError(2, "not an SFG1 stream")
    ext = []
    for a in range(3):
        raw = blob[4 + 8 * a:12 + 8 * a]
        v = int(np.frombuffer(raw, dtype="<i8")[0]) if len(raw) == 8 else 0
        if v < 1:
            raise GridError(2, "SFG1 read: bad extents")
        ext.append(v)
    n = ext[0] * ext[1] * ext[2]
    payload = blob[28:28 + 8 * n]
    if len(payload) != 8 * n:
        raise GridError(2, "SFG1 read: truncated payload")
    return tuple(ext), np.frombuffer(payload, dtype="<f8").reshape(ext[2], ext[1], ext[0]).astype(np.float64)


def dump_fields(sim: Simulation, directory: str) -> list:
    """sforge.cpp dump_fields (:176-185): vx, vy, vz, p gathered to <dir>/<name>.sfg1."""
    import os
    os.makedirs(directory, exist_ok=True)
    written = []
    for name in ("vx", "vy", "vz", "p"):
        path = os.path.join(directory, name + ".sfg1")
        write_sfg1(path, sim.extents, sim.gather(name))
        written.append(path)
    return written


def run_cavity(nx=129, ny=129, nz=3, re=100.0, sigma=0.9, omega=1.9525, tolerance=1e-6, max_sweeps=3000,
               alpha=0.0, lid_speed=1.0, symmetry_z=True, steady_tol=1e-6, max_steps=200000, workers=1,
               device=0, fused=1, progress=None):
    """The ``sforge cavity`` flow (sforge.cpp:223-259) with runs/re100.cfg as defaults.
    Returns (summary, profiles_csv_text, residuals_csv_text, sim)."""
    cfg = SolverConfig(extents=(nx, ny, nz), reynolds=re, sigma=sigma, omega=omega, tolerance=tolerance,
                       max_sweeps=max_sweeps, symmetry_z=symmetry_z)
    par = FluidParams(viscosity=lid_speed * 1.0 / re, lid_speed=lid_speed, blend=alpha)
    sim = Simulation(cfg, par, workers=workers, device=device, fused=fused)
    sim.init_cavity()
    rows = []

    def on_step(n, st, rate):
        rows.append((n, st))
        if progress:
            progress(n, st, rate)

    summary = run_to_steady(sim, max_steps, steady_tol * lid_speed, on_step)
    u, v = centerline_profiles(sim, lid_speed)
    comment = "lid-driven cavity centerline profiles: %dx%dx%d, Re=%s, t=%s, steps=%d" % (
        nx, ny, nz, "%g" % re, "%.6g" % sim.time, summary.steps)
    return summary, write_profiles(u, v, [comment]), write_residuals(rows), sim


def read_profiles(text: str):
    """cli::read_profiles (validate.hpp:31-79): `y,u` and `x,v` sections, '#' comments."""
    u, v, sec = [], [], None
    for raw in text.splitlines():
        t = raw.strip()
        if not t or t.startswith("#"):
            continue
        if t == "y,u":
            sec = u
            continue
        if t == "x,v":
            sec = v
            continue
        if sec is None:
            raise ValueError("expected a 'y,u' or 'x,v' header before data rows")
        a, b = t.split(",")
        sec.append((float(a), float(b)))
    return u, v


def compare_profiles(computed, reference):
    """cli::compare_profiles (validate.hpp:137-157): piecewise-linear sample of the
    computed profile at every reference coordinate; returns the max |deviation|."""
    import bisect

    def interp(table, x):
        xs = [r[0] for r in table]
        k = bisect.bisect_left(xs, x)
        if xs[k] == x:
            return table[k][1]
        lo, hi = table[k - 1], table[k]
        t = (x - lo[0]) / (hi[0] - lo[0])
        return lo[1] + t * (hi[1] - lo[1])

    worst = 0.0
    for comp, ref in ((computed[0], reference[0]), (computed[1], reference[1])):
        for x, want in ref:
            worst = max(worst, abs(interp(comp, x) - want))
    return worst
