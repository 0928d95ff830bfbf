"""GPU tests of the plugin path: descriptor-declared kernels JIT-compiled for
sm_100a and run through the executor operations, mirroring the reference's
tests/test_executor.cpp case by case.  Oracles are numpy restatements that keep
the reference's evaluation order (the reference's own "untiled oracle" style,
test_executor.cpp:150-194), so results must match bitwise."""
import numpy as np
import pytest

import paper_1201_2118_b200 as sfb
from paper_1201_2118_b200 import ExecutionPlan as Plan
from paper_1201_2118_b200 import ScheduleStep as Step

pytestmark = pytest.mark.gpu


def rig(ext, workers, ghost, periodic, bc="unset", lid=None):
    """test_executor.cpp:38-50: decomposition + store + executor; bc "unset"
    is the reference's empty boundary_spec."""
    cfg = sfb.SolverConfig(extents=ext, periodic=periodic)
    s = sfb.Simulation(cfg, sfb.FluidParams(), workers=workers, ghost=ghost)
    s.set_boundary_uniform(bc)
    if lid is not None:
        s.set_face_bc(1, 1, "wall", lid)
    return s


def random_global(ext, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=tuple(ext)[::-1])


def same(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint64), np.ascontiguousarray(b).view(np.uint64))


SMOOTH_BODY = """
  const auto& f = c.field(0);
  double sum = f(-1, 0, 0) + f(1, 0, 0);
  sum += f(0, -1, 0) + f(0, 1, 0);
  sum += f(0, 0, -1) + f(0, 0, 1);
  c.field(1).store(0.25 * f.load() + 0.125 * sum);
"""


def smooth_np(data):
    """smooth_expr (test_executor.cpp:141-148) over a periodic global array."""
    r = lambda di, dj, dk: np.roll(data, shift=(-dk, -dj, -di), axis=(0, 1, 2))  # noqa: E731
    s = r(-1, 0, 0) + r(1, 0, 0)
    s = s + (r(0, -1, 0) + r(0, 1, 0))
    s = s + (r(0, 0, -1) + r(0, 0, 1))
    return 0.25 * data + 0.125 * s


def test_identity_kernel_copies_input_to_output():
    s = rig((8, 6, 5), 2, 1, (False, False, False))
    s.create_field("in")
    s.create_field("out")
    data = random_global((8, 6, 5), 1)
    s.scatter("in", data)
    s.register_kernel(Plan("IDENT", (4, 4, 4), (0,) * 6, [("in", "IN"), ("out", "OUT")]), (["in", "out"], []),
                      "c.field(1).store(c.field(0).load());")
    s.run_kernel("IDENT")
    assert same(s.gather("out"), data)


LAP_BODY = """
  const auto& v = c.field(0);
  double s = v(-1, 0, 0) + v(1, 0, 0);
  s += v(0, -1, 0) + v(0, 1, 0);
  s += v(0, 0, -1) + v(0, 0, 1);
  c.field(1).store(s - 6.0 * v.load());
"""


def quadratic():
    i = np.arange(8, dtype=np.float64)
    return np.broadcast_to(i * i, (8, 8, 8)).copy()


def test_seven_point_laplacian_is_exact_on_a_quadratic_interior():
    s = rig((8, 8, 8), 1, 1, (False, False, False))
    s.create_field("f")
    s.create_field("lap")
    s.scatter("f", quadratic())
    s.register_kernel(Plan("LAP", (16, 16, 16), (1,) * 6, [("f", "IN", True), ("lap", "OUT")]), (["f", "lap"], []),
                      LAP_BODY)
    s.run_kernel("LAP", region="interior")
    out = s.gather("lap")
    inner = out[1:7, 1:7, 1:7]
    assert np.all(inner == 2.0)
    shell = out.copy()
    shell[1:7, 1:7, 1:7] = 0.0
    assert np.all(shell == 0.0)


def test_seven_point_laplacian_across_an_exchanged_seam():
    s = rig((8, 8, 8), 2, 1, (False, False, False))
    s.create_field("f")
    s.create_field("lap")
    s.scatter("f", quadratic())
    s.register_kernel(Plan("LAP", (16, 16, 16), (1,) * 6, [("f", "IN", True), ("lap", "OUT")]), (["f", "lap"], []),
                      LAP_BODY)
    s.exchange(["f"])
    s.run_kernel("LAP")
    assert np.all(s.gather("lap")[1:7, 1:7, 1:7] == 2.0)


@pytest.mark.parametrize("tile,workers", [((16, 16, 16), 1), ((4, 4, 4), 1), ((5, 3, 7), 4), ((1, 1, 1), 2),
                                          ((16, 16, 16), 4), ((12, 12, 12), 8), ((32, 8, 4), 2)])
def test_tiling_and_worker_count_are_transparent_bitwise(tile, workers):
    n = 12
    data = random_global((n, n, n), 2)
    want = smooth_np(data)
    s = rig((n, n, n), workers, 1, (True, True, True))
    s.create_field("src")
    s.create_field("dst")
    s.scatter("src", data)
    s.register_kernel(Plan("SMOOTH", tile, (1,) * 6, [("src", "IN", True), ("dst", "OUT", True)]),
                      (["src", "dst"], []), SMOOTH_BODY)
    s.exchange(["src"])
    s.run_kernel("SMOOTH")
    assert same(s.gather("dst"), want)


@pytest.mark.parametrize("shape,workers,tile", [((13, 11, 9), 1, (32, 8, 4)), ((17, 15, 7), 2, (16, 6, 5)),
                                                ((9, 7, 13), 4, (8, 2, 3)), ((40, 9, 6), 1, (32, 16, 64))])
def test_two_rows_per_thread_on_ragged_tiles_bitwise(shape, workers, tile):
    """The TMA template sweeps two adjacent rows per thread with the stores
    deferred to the end of the pair (sf_jit.hpp SF_RPT, the default for an even
    tile height).  Odd block heights leave a lone last row, a body that stores
    twice keeps the last value (executor.hpp:173-184 store semantics), and a
    second output and an uncached input are written/read per row."""
    data = random_global(shape, 3)
    extra = random_global(shape, 4)
    s = rig(shape, workers, 1, (True, True, True))
    for f in ("src", "dst", "aux", "w"):
        s.create_field(f)
    s.scatter("src", data)
    s.scatter("w", extra)
    body = SMOOTH_BODY + """
  c.field(2).store(-1.0);
  c.field(2).store((c.field(0)(0, 1, 0) - c.field(0)(0, -1, 0)) * c.field(3)(0, 1, 0));
"""
    s.register_kernel(Plan("SMOOTH2", tile, (1,) * 6,
                           [("src", "IN", True), ("dst", "OUT"), ("aux", "OUT"), ("w", "IN")]),
                      (["src", "dst", "aux", "w"], []), body)
    s.exchange(["src", "w"])
    s.run_kernel("SMOOTH2")
    r = lambda a, dj: np.roll(a, shift=-dj, axis=1)  # noqa: E731
    assert same(s.gather("dst"), smooth_np(data))
    assert same(s.gather("aux"), (r(data, 1) - r(data, -1)) * r(extra, 1))


@pytest.mark.parametrize("tile", [(2, 2, 2), (8, 8, 8), (3, 1, 5)])
def test_separate_inout_reads_the_pre_kernel_state(tile):
    s = rig((8, 4, 4), 2, 1, (True, False, False), bc="outflow")
    s.create_field("v")
    i = np.arange(8, dtype=np.float64)
    s.scatter("v", np.broadcast_to(i, (4, 4, 8)).copy())
    s.register_kernel(Plan("SHIFT", tile, (0, 1, 0, 0, 0, 0), [("v", "SEPARATEINOUT")]), (["v"], []),
                      "c.field(0).store(c.field(0)(1, 0, 0));")
    s.refresh(["v"])
    s.run_kernel("SHIFT")
    out = s.gather("v")
    assert np.all(out == np.broadcast_to((i + 1) % 8, (4, 4, 8)))
    s.refresh(["v"])
    s.run_kernel("SHIFT")
    assert s.gather("v")[0, 0, 0] == 2.0


def test_interior_and_boundary_regions_partition_the_block():
    for ext in [(8, 8, 8)]:
        s = rig(ext, 2, 2, (False, False, False))
        s.create_field("count")
        s.register_kernel(Plan("INC", (3, 3, 3), (2,) * 6, [("count", "INOUT")]), (["count"], []),
                          "c.field(0).store(c.field(0).load() + 1.0);")
        s.run_kernel("INC", region="interior")
        s.run_kernel("INC", region="boundary")
        assert np.all(s.gather("count") == 1.0)
        d = sfb.decompose(ext, 2, 2)
        assert d.size(0)[0] == 4  # no interior with a (2,2) halo: boundary covers all


def test_schedule_dry_run_demands_an_exchange_before_ghost_reads():
    s = rig((8, 8, 8), 1, 1, (True, True, True))
    s.create_field("a")
    s.create_field("b")
    s.register_kernel(Plan("STEP", (8, 8, 8), (1,) * 6, [("a", "IN"), ("b", "SEPARATEINOUT")]), (["a", "b"], []),
                      "c.field(1).store(c.field(0)(1, 0, 0) + c.field(1)(0, 1, 0));")
    s.invalidate_all_ghosts()
    with pytest.raises(sfb.ExecError, match="never exchanged"):
        s.run_schedule([Step.run("STEP")], passes=1)
    s.run_schedule([Step.exchange(["a", "b"]), Step.run("STEP")], passes=3)
    s.exchange(["a", "b"])
    s.run_schedule([Step.run("STEP")], passes=1)
    s.exchange(["a", "b"])
    with pytest.raises(sfb.ExecError, match="ghosts of 'b'"):
        s.run_schedule([Step.run("STEP")], passes=2)
    with pytest.raises(sfb.ExecError, match="unknown kernel"):
        s.run_schedule([Step.run("NOPE")], passes=1)
    with pytest.raises(sfb.ExecError, match="unknown field 'zz'"):
        s.run_schedule([Step.exchange(["zz"])], passes=1)
    s.create_field("c")
    s.register_kernel(Plan("LOCAL", (8, 8, 8), (0,) * 6, [("c", "INOUT")]), (["c"], []),
                      "c.field(0).store(c.field(0).load() * 2.0);")
    s.run_schedule([Step.run("LOCAL")], passes=2)


def test_an_empty_schedule_changes_nothing():
    s = rig((6, 6, 6), 2, 1, (False, False, False))
    s.create_field("f")
    data = random_global((6, 6, 6), 3)
    s.scatter("f", data)
    s.run_schedule([], passes=5)
    assert same(s.gather("f"), data)


SMOOTH_INPLACE = """
  const auto& f = c.field(0);
  double sum = f(-1, 0, 0) + f(1, 0, 0);
  sum += f(0, -1, 0) + f(0, 1, 0);
  sum += f(0, 0, -1) + f(0, 0, 1);
  c.field(0).store(0.25 * f.load() + 0.125 * sum);
"""


def test_schedules_execute_refreshes_kernels_and_reductions_in_order():
    data = random_global((10, 8, 6), 4)

    def setup(workers):
        s = rig((10, 8, 6), workers, 1, (False, False, False), bc="wall")
        s.create_field("v")
        s.scatter("v", data)
        s.register_kernel(Plan("SMOOTH", (4, 4, 4), (1,) * 6, [("v", "SEPARATEINOUT", True)]), (["v"], []),
                          SMOOTH_INPLACE)
        return s

    r, ref = setup(2), setup(1)
    results = {}
    r.run_schedule([Step.refresh(["v"]), Step.run("SMOOTH"), Step.reduce("v", "max_abs", "vmax")], passes=3,
                   results=results)
    want_max = 0.0
    for _ in range(3):
        ref.refresh(["v"])
        ref.run_kernel("SMOOTH")
        want_max = ref.reduce("v", "max_abs")
    assert same(r.gather("v"), ref.gather("v"))
    assert results["vmax"] == want_max and r.result("vmax") == want_max


BLUR_BODY = """
  const auto& f = c.field(0);
  double sum = f(-1, 0, 0) + f(1, 0, 0);
  sum += f(0, -1, 0) + f(0, 1, 0);
  sum += f(0, 0, -1) + f(0, 0, 1);
  const double mixed = 0.25 * f.load() + 0.125 * sum;
  c.field(0).store(mixed + 0.01 * c.field(1)(0, 1, 0));
"""


def test_overlap_mode_matches_plain_mode_bitwise():
    ext = (12, 10, 8)
    dv, ds = random_global(ext, 5), random_global(ext, 6)

    def build(workers):
        s = rig(ext, workers, 1, (False, False, True), bc="wall", lid=(1.0, 0.0, 0.0))
        s.create_field("vx_", "x")
        s.create_field("s")
        s.scatter("vx_", dv)
        s.scatter("s", ds)
        s.register_kernel(Plan("BLUR", (4, 4, 4), (1,) * 6, [("vx_", "SEPARATEINOUT", True), ("s", "IN")]),
                          (["vx_", "s"], []), BLUR_BODY)
        return s

    sched = [Step.refresh(["vx_", "s"]), Step.run("BLUR")]
    p1 = build(1)
    p1.run_schedule(sched, passes=10)
    want = p1.gather("vx_")
    for workers in (1, 2, 4):
        for mode in ("overlap", "plain"):
            q = build(workers)
            q.run_schedule(sched, passes=10, mode=mode)
            assert same(q.gather("vx_"), want), (workers, mode)


def test_overlap_with_an_in_place_comm_field_matches_plain():
    ext = (10, 10, 6)
    dv, da = random_global(ext, 7), random_global(ext, 8)
    outs = []
    for mode in ("plain", "overlap"):
        s = rig(ext, 2, 1, (False, False, False), bc="wall")
        s.create_field("v")
        s.create_field("a")
        s.scatter("v", dv)
        s.scatter("a", da)
        s.register_kernel(Plan("ACC", (4, 4, 4), (0, 1, 0, 0, 0, 0), [("v", "INOUT"), ("a", "IN")]), (["v", "a"], []),
                          "c.field(0).store(c.field(0).load() + 0.5 * c.field(1)(1, 0, 0));")
        s.run_schedule([Step.refresh(["v", "a"]), Step.run("ACC")], passes=5, mode=mode)
        outs.append(s.gather("v"))
    assert same(outs[0], outs[1])


def test_debug_mode_polices_reads_writes_and_ghost_validity(monkeypatch):
    monkeypatch.setenv("SF_DEBUG_BOUNDS", "1")
    s = rig((8, 8, 8), 1, 1, (True, True, True))
    s.create_field("a")
    s.create_field("b")
    cases = [
        ("REACH", (0,) * 6, [("a", "IN"), ("b", "OUT")], "c.field(1).store(c.field(0)(1, 0, 0));",
         "outside the declared stencil"),
        ("WREAD", (0,) * 6, [("a", "IN"), ("b", "OUT")], "c.field(1).store(c.field(1).load());",
         "write-only binding 'b'"),
        ("WRST", (0,) * 6, [("a", "IN"), ("b", "OUT")], "c.field(0).store(1.0);", "store to read-only binding 'a'"),
    ]
    for name, halo, binds, body, msg in cases:
        s.register_kernel(Plan(name, (8, 8, 8), halo, binds), ([b[0] for b in binds], []), body)
        with pytest.raises(sfb.ExecError, match=msg):
            s.run_kernel(name)
    s.register_kernel(Plan("INPL", (8, 8, 8), (1,) * 6, [("a", "INOUT")]), (["a"], []),
                      "c.field(0).store(c.field(0)(1, 0, 0));")
    s.exchange(["a"])
    with pytest.raises(sfb.ExecError, match="non-center read"):
        s.run_kernel("INPL")
    s.register_kernel(Plan("NEEDS", (8, 8, 8), (1,) * 6, [("b", "IN"), ("a", "INOUT")]), (["b", "a"], []),
                      "c.field(1).store(c.field(0)(0, 1, 0));")
    s.invalidate_ghosts("b")
    with pytest.raises(sfb.ExecError, match="never exchanged"):
        s.run_kernel("NEEDS")
    s.exchange(["b", "a"])
    s.run_kernel("NEEDS")


def test_debug_mode_stays_quiet_for_disciplined_kernels_and_matches_numpy(monkeypatch):
    monkeypatch.setenv("SF_DEBUG_BOUNDS", "1")
    ext = (8, 6, 6)
    data = random_global(ext, 9)
    s = rig(ext, 2, 2, (True, True, True))
    s.create_field("v")
    s.scatter("v", data)
    s.register_kernel(Plan("OK", (4, 4, 4), (2, 1, 0, 2, 1, 1), [("v", "SEPARATEINOUT", True)]), (["v"], []),
                      """const auto& f = c.field(0);
                         c.field(0).store(f(-2, 0, 0) + f(1, 0, 0) + f(0, 2, 0) + f(0, 0, -1) + f(0, 0, 1));""")
    s.exchange(["v"])
    s.run_kernel("OK")
    r = lambda di, dj, dk: np.roll(data, shift=(-dk, -dj, -di), axis=(0, 1, 2))  # noqa: E731
    want = (((r(-2, 0, 0) + r(1, 0, 0)) + r(0, 2, 0)) + r(0, 0, -1)) + r(0, 0, 1)
    assert same(s.gather("v"), want)


def test_parameters_reach_the_point_function_by_slot():
    s = rig((4, 4, 4), 1, 1, (False, False, False))
    s.create_field("out")
    s.register_kernel(Plan("PARAMS", (4, 4, 4), (0,) * 6, [("out", "OUT")], ["alpha", "beta"]),
                      (["out"], ["alpha", "beta"]), "c.field(0).store(c.param(0) * 10.0 + c.param(1));")
    s.run_kernel("PARAMS", {"alpha": 3.0, "beta": 0.5, "extra": 9.0})
    assert np.all(s.gather("out") == 30.5)


def test_global_indices_reach_the_point_function():
    s = rig((9, 7, 5), 4, 1, (False, False, False))
    s.create_field("gi")
    s.register_kernel(Plan("IDX", (3, 3, 3), (0,) * 6, [("gi", "OUT")]), (["gi"], []),
                      "c.field(0).store((double)c.i + 100.0 * (double)c.j + 10000.0 * (double)c.k);")
    s.run_kernel("IDX")
    k, j, i = np.meshgrid(np.arange(5), np.arange(7), np.arange(9), indexing="ij")
    assert np.array_equal(s.gather("gi"), i + 100.0 * j + 10000.0 * k)


def test_registration_rejects_bad_signatures_naming_the_offender():
    s = rig((8, 8, 8), 1, 1, (False, False, False))
    s.create_field("vx2", "x")
    s.create_field("q")
    plan = Plan("K", (4, 4, 4), (1,) * 6, [("vx2", "SEPARATEINOUT", True), ("q", "IN", True)], ["density"])
    body = "(void)c;"
    with pytest.raises(sfb.ExecError, match="missing parameter 'density'"):
        s.register_kernel(plan, (["vx2", "q"], []), body)
    with pytest.raises(sfb.ExecError, match="slot 0 binds 'vx2'"):
        s.register_kernel(plan, (["q", "vx2"], ["density"]), body)
    with pytest.raises(sfb.ExecError, match="missing binding 'q'"):
        s.register_kernel(plan, (["vx2"], ["density"]), body)
    with pytest.raises(sfb.ExecError, match="unknown binding 'z'"):
        s.register_kernel(plan, (["vx2", "q", "z"], ["density"]), body)
    s.register_kernel(plan, (["vx2", "q"], ["density"]), body)
    with pytest.raises(sfb.ExecError, match="already registered"):
        s.register_kernel(plan, (["vx2", "q"], ["density"]), body)
    with pytest.raises(sfb.ExecError, match="ghost layers"):
        s.register_kernel(Plan("G", (4, 4, 4), (2,) * 6, [("q", "IN")]), (["q"], []), body)
    with pytest.raises(sfb.ExecError, match="unknown field 'nope'"):
        s.register_kernel(Plan("M", (4, 4, 4), (0,) * 6, [("nope", "IN")]), (["nope"], []), body)
    with pytest.raises(sfb.ExecError):
        s.run_kernel("K")  # density not supplied
    with pytest.raises(sfb.ExecError):
        s.run_kernel("NOSUCH")
    with pytest.raises(sfb.ExecError, match="device compilation failed"):
        s.register_kernel(Plan("BAD", (4, 4, 4), (0,) * 6, [("q", "IN")]), (["q"], []), "this is not C++;")


# ---- config C5: higher-order stencils, ghost width 2-3 ----------------------
LAP4 = """
  const auto& f = c.field(0);
  const double c0 = -2.5, c1 = 4.0 / 3.0, c2 = -1.0 / 12.0;
  double sx = c1 * (f(-1, 0, 0) + f(1, 0, 0)) + c2 * (f(-2, 0, 0) + f(2, 0, 0));
  double sy = c1 * (f(0, -1, 0) + f(0, 1, 0)) + c2 * (f(0, -2, 0) + f(0, 2, 0));
  double sz = c1 * (f(0, 0, -1) + f(0, 0, 1)) + c2 * (f(0, 0, -2) + f(0, 0, 2));
  c.field(1).store((3.0 * c0) * f.load() + ((sx + sy) + sz));
"""
LAP6 = """
  const auto& f = c.field(0);
  const double c0 = -49.0 / 18.0, c1 = 1.5, c2 = -0.15, c3 = 1.0 / 90.0;
  double s[3];
  for (int a = 0; a < 3; ++a) {
    const int x = a == 0, y = a == 1, z = a == 2;
    s[a] = c1 * (f(-x, -y, -z) + f(x, y, z)) + c2 * (f(-2 * x, -2 * y, -2 * z) + f(2 * x, 2 * y, 2 * z))
         + c3 * (f(-3 * x, -3 * y, -3 * z) + f(3 * x, 3 * y, 3 * z));
  }
  c.field(1).store((3.0 * c0) * f.load() + ((s[0] + s[1]) + s[2]));
"""


def lap_np(data, radius):
    r = lambda di, dj, dk: np.roll(data, shift=(-dk, -dj, -di), axis=(0, 1, 2))  # noqa: E731
    if radius == 2:
        c0, c1, c2 = -2.5, 4.0 / 3.0, -1.0 / 12.0
        s = [c1 * (r(*[-(a == q) for q in range(3)]) + r(*[(a == q) for q in range(3)]))
             + c2 * (r(*[-2 * (a == q) for q in range(3)]) + r(*[2 * (a == q) for q in range(3)])) for a in range(3)]
    else:
        c0, c1, c2, c3 = -49.0 / 18.0, 1.5, -0.15, 1.0 / 90.0
        s = [c1 * (r(*[-(a == q) for q in range(3)]) + r(*[(a == q) for q in range(3)]))
             + c2 * (r(*[-2 * (a == q) for q in range(3)]) + r(*[2 * (a == q) for q in range(3)]))
             + c3 * (r(*[-3 * (a == q) for q in range(3)]) + r(*[3 * (a == q) for q in range(3)])) for a in range(3)]
    return (3.0 * c0) * data + ((s[0] + s[1]) + s[2])


@pytest.mark.parametrize("radius,ghost,workers,tile", [(2, 2, 1, (32, 4, 16)), (2, 3, 2, (64, 4, 8)),
                                                       (3, 3, 1, (128, 2, 8)), (3, 3, 4, (32, 8, 4))])
def test_higher_order_stencils_match_numpy_bitwise(radius, ghost, workers, tile):
    ext = (20, 18, 16)
    data = random_global(ext, 11)
    s = rig(ext, workers, ghost, (True, True, True))
    s.create_field("u")
    s.create_field("lu")
    s.scatter("u", data)
    s.register_kernel(Plan(f"LAP{2 * radius}", tile, (radius,) * 6, [("u", "IN", True), ("lu", "OUT")]),
                      (["u", "lu"], []), LAP4 if radius == 2 else LAP6)
    s.exchange(["u"])
    s.run_kernel(f"LAP{2 * radius}")
    assert same(s.gather("lu"), lap_np(data, radius))


# the same stencils written against sf_real: float in a kernel whose bindings
# are all fp32, double otherwise (the fp64 results equal LAP4 / LAP6 bitwise)
LAP4R = """
  const auto& f = c.field(0);
  const sf_real c0 = -2.5, c1 = (sf_real)(4.0 / 3.0), c2 = (sf_real)(-1.0 / 12.0);
  sf_real sx = c1 * (f(-1, 0, 0) + f(1, 0, 0)) + c2 * (f(-2, 0, 0) + f(2, 0, 0));
  sf_real sy = c1 * (f(0, -1, 0) + f(0, 1, 0)) + c2 * (f(0, -2, 0) + f(0, 2, 0));
  sf_real sz = c1 * (f(0, 0, -1) + f(0, 0, 1)) + c2 * (f(0, 0, -2) + f(0, 0, 2));
  c.field(1).store(((sf_real)3 * c0) * f.load() + ((sx + sy) + sz));
"""
LAP6R = """
  const auto& f = c.field(0);
  const sf_real c0 = (sf_real)(-49.0 / 18.0), c1 = 1.5, c2 = (sf_real)(-0.15), c3 = (sf_real)(1.0 / 90.0);
  sf_real s[3];
  for (int a = 0; a < 3; ++a) {
    const int x = a == 0, y = a == 1, z = a == 2;
    s[a] = c1 * (f(-x, -y, -z) + f(x, y, z)) + c2 * (f(-2 * x, -2 * y, -2 * z) + f(2 * x, 2 * y, 2 * z))
         + c3 * (f(-3 * x, -3 * y, -3 * z) + f(3 * x, 3 * y, 3 * z));
  }
  c.field(1).store(((sf_real)3 * c0) * f.load() + ((s[0] + s[1]) + s[2]));
"""


def lap_np32(data32, radius):
    """lap_np in IEEE single precision, operation for operation (sf_real = float)."""
    f = np.float32
    r = lambda di, dj, dk: np.roll(data32, shift=(-dk, -dj, -di), axis=(0, 1, 2))  # noqa: E731
    ax = lambda a, m: [m * (a == q) for q in range(3)]  # noqa: E731
    if radius == 2:
        c0, c1, c2 = f(-2.5), f(4.0 / 3.0), f(-1.0 / 12.0)
        s = [c1 * (r(*ax(a, -1)) + r(*ax(a, 1))) + c2 * (r(*ax(a, -2)) + r(*ax(a, 2))) for a in range(3)]
    else:
        c0, c1, c2, c3 = f(-49.0 / 18.0), f(1.5), f(-0.15), f(1.0 / 90.0)
        s = [c1 * (r(*ax(a, -1)) + r(*ax(a, 1))) + c2 * (r(*ax(a, -2)) + r(*ax(a, 2)))
             + c3 * (r(*ax(a, -3)) + r(*ax(a, 3))) for a in range(3)]
    return (f(3) * c0) * data32 + ((s[0] + s[1]) + s[2])


@pytest.mark.parametrize("no_tma", [False, True])
@pytest.mark.parametrize("radius,ghost,workers,tile", [(2, 2, 1, (32, 4, 16)), (2, 3, 2, (64, 4, 8)),
                                                       (3, 3, 4, (32, 8, 4))])
def test_fp32_fields_in_descriptor_stencils(radius, ghost, workers, tile, no_tma, monkeypatch):
    # configs[4] in fp32: both fields fp32, so the kernel computes in fp32
    # (sf_real = float); the exchange moves fp32 values between components.
    # numpy repeats every single-precision operation.
    if no_tma:
        monkeypatch.setenv("SF_JIT_NO_TMA", "1")
    ext = (20, 18, 16)
    data = random_global(ext, 21).astype(np.float32).astype(np.float64)
    s = rig(ext, workers, ghost, (True, True, True))
    s.create_field("u", dtype="f32")
    s.create_field("lu", dtype="f32")
    s.scatter("u", data)
    assert same(s.gather("u"), data)
    s.register_kernel(Plan(f"LAP{2 * radius}F", tile, (radius,) * 6, [("u", "IN", True), ("lu", "OUT")]),
                      (["u", "lu"], []), LAP4R if radius == 2 else LAP6R)
    s.exchange(["u"])
    s.run_kernel(f"LAP{2 * radius}F")
    want = lap_np32(data.astype(np.float32), radius).astype(np.float64)
    assert same(s.gather("lu"), want)
    assert s.reduce("lu", "max_abs") == float(np.max(np.abs(want)))
    assert s.reduce("lu", "sum") == pytest.approx(float(np.sum(want)), rel=1e-12)


# configs[4] in fp32 against the fp64 result (the stated tolerance of the fp32
# variant): inputs rounded to fp32, every operation in fp32; the error is a few
# fp32 ulps of the result's scale
FP32_STENCIL_TOL = 1e-6  # max |lu_fp32 - lu_fp64| / max |lu_fp64|


@pytest.mark.parametrize("radius", [2, 3])
def test_fp32_stencil_within_the_stated_tolerance_of_fp64(radius):
    ext = (48, 40, 36)
    data = random_global(ext, 31)  # fp64 data: the fp32 run also rounds its inputs
    s = rig(ext, 2, radius, (True, True, True))
    s.create_field("u", dtype="f32")
    s.create_field("lu", dtype="f32")
    s.scatter("u", data)
    s.register_kernel(Plan(f"LAP{2 * radius}T", (32, 16, 64), (radius,) * 6, [("u", "IN", True), ("lu", "OUT")]),
                      (["u", "lu"], []), LAP4R if radius == 2 else LAP6R)
    s.exchange(["u"])
    s.run_kernel(f"LAP{2 * radius}T")
    want = lap_np(data, radius)
    err = float(np.max(np.abs(s.gather("lu") - want)) / np.max(np.abs(want)))
    print(f"fp32 radius {radius} stencil: relative error {err:.3g}")
    assert err <= FP32_STENCIL_TOL, err


@pytest.mark.parametrize("radius", [2, 3])
def test_mixed_precision_kernel_computes_in_fp64(radius):
    # an fp32 input with an fp64 output: accessors widen, the body runs in fp64;
    # with every binding fp64 the sf_real bodies equal LAP4 / LAP6 bitwise
    ext = (20, 18, 16)
    data = random_global(ext, 22).astype(np.float32).astype(np.float64)
    s = rig(ext, 1, radius, (True, True, True))
    s.create_field("u", dtype="f32")
    s.create_field("lu")
    s.create_field("u64")
    s.create_field("lu64")
    s.scatter("u", data)
    s.scatter("u64", data)
    body = LAP4R if radius == 2 else LAP6R
    s.register_kernel(Plan("MIX", (32, 4, 16), (radius,) * 6, [("u", "IN", True), ("lu", "OUT")]), (["u", "lu"], []),
                      body)
    s.register_kernel(Plan("F64", (32, 4, 16), (radius,) * 6, [("u64", "IN", True), ("lu64", "OUT")]),
                      (["u64", "lu64"], []), body)
    s.exchange(["u", "u64"])
    s.run_kernel("MIX")
    s.run_kernel("F64")
    want = lap_np(data, radius)
    assert same(s.gather("lu"), want)
    assert same(s.gather("lu64"), want)


SMOOTH_CCL = """# a user kernel declared in the descriptor language
CCTK_CUDA_KERNEL SMOOTH TYPE=3DBLOCK STENCIL="1,1,1,1,1,1" TILE="8,4,4"
{
  CCTK_CUDA_KERNEL_VARIABLE CACHED=YES INTENT=IN { src } "SOURCE"
  CCTK_CUDA_KERNEL_VARIABLE INTENT=OUT { dst } "RESULT"
}
"""


@pytest.mark.parametrize("workers", [1, 4])
def test_descriptor_file_drives_a_device_kernel(workers):
    # .ccl text -> parse -> validate against the store's fields -> plan ->
    # register_kernel -> run: the plugin path from the descriptor front end on
    from paper_1201_2118_b200.descriptor import load_plans
    n = 12
    data = random_global((n, n, n), 7)
    s = rig((n, n, n), workers, 1, (True, True, True))
    s.create_field("src")
    s.create_field("dst")
    s.scatter("src", data)
    plan = load_plans(SMOOTH_CCL, sfb.FIELDS + ("src", "dst"))["SMOOTH"]
    s.register_kernel(plan, (["src", "dst"], []), SMOOTH_BODY)
    s.exchange(["src"])
    s.run_kernel("SMOOTH")
    assert same(s.gather("dst"), smooth_np(data))
