"""The fp32 variant of the CFD fields (precision="f32": storage and arithmetic
in fp32 on the fused TMA path -- the temporal pass with fused = 1, the single
half-sweep with fused = 3) against the fp64 reference after N steps.

fp32 cannot reach the default pressure tolerance (max|div| 1e-6: roundoff x
1/dx is ~6e-6 at 64^3; SURVEY.md §7 hard part 6), so the comparison uses the
fixed-work configurations (tolerance 1e-30, max_sweeps S: the
runs/bench128.cfg pattern): both runs do exactly the same sweeps, and each
field is compared by its relative error against the reference,

    err(f) = max |f_fp32 - f_ref| / max |f_ref|     over the owned cells,

which must stay within the stated per-field tolerance (TOL below), where the
scale of the three velocity components is the flow's velocity scale
max(|vx|, |vy|, |vz|) of the reference (vz of a cavity is orders of magnitude
smaller than the lid-driven vx, vy: its own maximum is not a meaningful
scale) and the scale of p is max |p|.  dt per step is compared the same way.
"""
import json
import os

import numpy as np
import pytest

import paper_1201_2118_b200 as sfb
from oracle.oracle import Oracle, cavity_case

pytestmark = pytest.mark.gpu

# stated tolerances (relative to the field's max magnitude) after the steps below
# (measured on B200: ~4e-7 .. 9e-7 for every field after 3 steps at 64^3 and
# 2 steps at 128^3, i.e. a few fp32 ulps of the field scale; dt exact)
TOL = {"vx": 1e-5, "vy": 1e-5, "vz": 1e-5, "p": 1e-5, "dt": 1e-6}


def _fixed_work(n, sweeps):
    return dict(symmetry_z=False, omega=1.9525, tolerance=1e-30, max_sweeps=sweeps)


def rel_err(a, b, scale=None):
    s = float(np.max(np.abs(b))) if scale is None else scale
    return float(np.max(np.abs(a - b)) / max(s, 1e-300))


def field_errors(d, o):
    ref = {f: o.gather(f) for f in ("vx", "vy", "vz", "p")}
    vscale = max(float(np.max(np.abs(ref[f]))) for f in ("vx", "vy", "vz"))
    return {f: rel_err(d.gather(f), ref[f], vscale if f != "p" else None) for f in ref}


def _compare(n, sweeps, steps, fused=3, workers=8):
    c = cavity_case(n, workers=workers, **_fixed_work(n, sweeps))
    o = Oracle(c, "ref")
    o.init_cavity()
    dts, sw, _ = o.advance(steps)
    ext = (n, n, n) if isinstance(n, int) else tuple(n)
    cfg = sfb.SolverConfig(extents=ext, reynolds=100.0, **_fixed_work(n, sweeps))
    d = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), fused=fused, precision="f32")
    d.init_cavity()
    st = [d.step() for _ in range(steps)]
    assert [s.sweeps for s in st] == [int(x) for x in sw]
    errs = field_errors(d, o)
    errs["dt"] = max(abs(s.dt - float(t)) / float(t) for s, t in zip(st, dts))
    d.close()
    return errs


@pytest.mark.parametrize("fused", [3, 1])
def test_fp32_cavity64_fixed_work_within_stated_tolerance(ref_available, fused):
    errs = _compare(64, 200, 3, fused=fused)
    print("fp32 64^3 x 3 steps:", json.dumps(errs))
    for f, e in errs.items():
        assert e <= TOL[f], (f, e, TOL[f])


@pytest.mark.parametrize("fused", [1, 3])
def test_fp32_cavity64_ten_steps_within_stated_tolerance(ref_available, fused):
    # a longer horizon: fp32 roundoff must not grow past the tolerance
    errs = _compare(64, 200, 10, fused=fused)
    print("fp32 64^3 x 10 steps:", json.dumps(errs))
    for f, e in errs.items():
        assert e <= TOL[f], (f, e, TOL[f])


@pytest.mark.parametrize("fused", [1, 3])
def test_fp32_bench128_config_within_stated_tolerance(ref_available, fused):
    # runs/bench128.cfg: 128^3, omega 1.9525, 200 half-sweeps per step, 2 steps
    errs = _compare(128, 200, 2, fused=fused)
    print("fp32 128^3 x 2 steps:", json.dumps(errs))
    for f, e in errs.items():
        assert e <= TOL[f], (f, e, TOL[f])


def test_fp32_odd_extents_and_refresh_paths(ref_available):
    # uneven tiles, symmetry faces, two grid components on the device (the
    # temporal pass with the fused exchange between them), an odd sweep cap
    # (the redo of a pass's first sweep)
    n = (45, 37, 11)
    c = cavity_case(n, workers=2, symmetry_z=True, omega=1.7, tolerance=1e-30, max_sweeps=61)
    o = Oracle(c, "ref")
    o.init_cavity()
    o.advance(4)
    cfg = sfb.SolverConfig(extents=n, reynolds=100.0, symmetry_z=True, omega=1.7, tolerance=1e-30, max_sweeps=61)
    d = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), workers=2, ghost=2, fused=1, precision="f32")
    d.init_cavity()
    d.advance(4)
    for f, e in field_errors(d, o).items():
        assert e <= TOL[f], (f, e)


def test_fp32_rejects_the_fp64_only_paths():
    cfg = sfb.SolverConfig(extents=(16, 16, 16), symmetry_z=False)
    with pytest.raises(sfb.SfError, match="fused TMA"):
        sfb.Simulation(cfg, sfb.cavity_fluid(cfg), fused=0, precision="f32")
    d = sfb.Simulation(cfg, sfb.cavity_fluid(cfg), fused=3, precision="f32")
    with pytest.raises(sfb.SfError, match="fp64"):
        d.run_kernel("DIVERGENCE", {})
