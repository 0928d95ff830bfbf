"""Level-2 C ABI (``sf_launch_*``, include/sforge_b200.h) against the reference.

This is the executor-plugin path of INTEGRATION.md §2: a maintainer keeps the
reference's own ``exec::executor`` / ``exchanger`` and sends each
(kernel, region box list) of ``executor::run_region_worker``
(executor.hpp:759-767), each ``bc_face`` (exchange.hpp:231-480) and each
``pack_axis`` / ``unpack`` (exchange.hpp:165-224) to one ``sf_launch_*`` call on
device arrays it owns.  Every test below drives the device the way that
plugin would -- caller-owned buffers in the ``sf_make_layout`` padded layout,
region boxes computed as ``detail::region_boxes`` (executor.hpp:81-109) does --
and compares with the reference (oracle/_ref/libsfref.so) running the same
operation through its own executor.  fp64 results are bitwise equal.
"""
import ctypes as C

import numpy as np
import pytest

import paper_1201_2118_b200 as sfb
from paper_1201_2118_b200 import _lib as L
from oracle.oracle import Case, Oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIELDS5 = ("vx", "vy", "vz", "p", "divu")
STAGGER = {"vx": 0, "vy": 1, "vz": 2, "p": -1, "divu": -1}
BC_WALL, BC_SYMMETRY = 1, 2
SCOPE_ALL = 0
MAX_ABS, MAX_ABS_DIFF = 0, 3


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


# ---- the plugin's host side ---------------------------------------------------
def layout(dims, lo, g):
    out = L.Layout()
    d = (C.c_int64 * 3)(*dims)
    l0 = (C.c_int64 * 3)(*lo)
    L.check(L.lib().sf_make_layout(d, l0, int(g), C.byref(out)))
    return out


def _xo(lay):
    g = lay.ghost
    return lay.base - (g * lay.sy + g) * lay.sx


def to_dev(lay, padded):
    """reference local_block (ld = dims + 2g, field.hpp:39-44) -> sf_layout device array"""
    g, n = lay.ghost, lay.dims
    a = np.zeros(lay.sx * lay.sy * lay.sz)
    v = a.reshape(lay.sz, lay.sy, lay.sx)
    xo = _xo(lay)
    v[:, :, xo - g:xo + n[0] + g] = padded
    return torch.from_numpy(a).cuda()


def from_dev(lay, t):
    g, n = lay.ghost, lay.dims
    v = t.cpu().numpy().reshape(lay.sz, lay.sy, lay.sx)
    xo = _xo(lay)
    return v[:, :, xo - g:xo + n[0] + g].copy()


def owned(lay, padded):
    g, n = lay.ghost, lay.dims
    return padded[g:g + n[2], g:g + n[1], g:g + n[0]]


def region_boxes(dims, halo, region):
    """detail::region_boxes (executor.hpp:81-109)"""
    allb = [(0, 0, 0, dims[0], dims[1], dims[2])]
    if region == "all":
        return allb
    il = [min(halo[2 * a], dims[a]) for a in range(3)]
    ih = [max(il[a], dims[a] - halo[2 * a + 1]) for a in range(3)]
    have = all(il[a] < ih[a] for a in range(3))
    if region == "interior":
        return [(il[0], il[1], il[2], ih[0], ih[1], ih[2])] if have else []
    if not have:
        return allb
    shell = [(0, 0, 0, dims[0], dims[1], il[2]), (0, 0, ih[2], dims[0], dims[1], dims[2]),
             (0, 0, il[2], dims[0], il[1], ih[2]), (0, ih[1], il[2], dims[0], dims[1], ih[2]),
             (0, il[1], il[2], il[0], ih[1], ih[2]), (ih[0], il[1], il[2], dims[0], ih[1], ih[2])]
    return [b for b in shell if b[3] > b[0] and b[4] > b[1] and b[5] > b[2]]


def boxes_c(boxes):
    arr = (L.Box * max(1, len(boxes)))()
    for q, b in enumerate(boxes):
        for a in range(3):
            arr[q].lo[a], arr[q].hi[a] = b[a], b[3 + a]
    return arr, len(boxes)


def consts_for(case, dt):
    cfg = sfb.SolverConfig(extents=tuple(case.extents), periodic=tuple(case.periodic), reynolds=case.reynolds,
                           sigma=case.sigma, tolerance=case.tolerance, omega=case.omega,
                           max_sweeps=case.max_sweeps, symmetry_z=case.symmetry_z)
    par = sfb.FluidParams(viscosity=case.viscosity, density=case.density, body_force=tuple(case.body_force),
                          lid_speed=case.lid_speed, blend=case.blend)
    c = L.CfdConsts()
    L.check(L.lib().sf_make_cfd_consts(C.byref(cfg.to_c()), C.byref(par.to_c()), C.byref(c)))
    c.dt = dt
    return c


def ptr(t):
    return C.c_void_p(t.data_ptr())


def stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def face_bc(case, axis, side):
    """cfd::simulation::make_bc (cfd.hpp:500-512) for one physical face"""
    bc = L.FaceBC()
    bc.kind = BC_WALL
    if axis == 1 and side == 1:
        bc.velocity[0] = case.lid_speed
    if axis == 2 and case.symmetry_z:
        bc.kind = BC_SYMMETRY
    return bc


def random_oracle(case, seed, fields=FIELDS5):
    rng = np.random.default_rng(seed)
    o = Oracle(case, "ref")
    shape = tuple(case.extents)[::-1]
    for f in fields:
        o.scatter(f, rng.uniform(-1.0, 1.0, size=shape))
    o.invalidate_all_ghosts()
    return o


def block_of(case, w=0):
    d = sfb.decompose(case.extents, case.workers, case.ghost, case.periodic)
    return d, d.size(w), d.lo[w]


# ---- kernels over region boxes ----------------------------------------------------
@pytest.mark.parametrize("split", [False, True])
def test_launch_update_velocity_over_region_boxes_matches_provisional(ref_available, split):
    # UPDATE_VELOCITY over all owned cells as the plugin issues it: either the
    # interior box and the boundary shell in one call, or one call each
    c = Case(extents=(19, 11, 7), symmetry_z=False, lid_speed=1.0, blend=0.3, viscosity=0.02,
             body_force=(0.1, -0.2, 0.3))
    o = random_oracle(c, 11, ("vx", "vy", "vz", "p"))
    o.refresh(["vx", "vy", "vz", "p"])
    _, n, lo = block_of(c)
    lay = layout(n, lo, c.ghost)
    dev = {f: to_dev(lay, o.local_front(f)) for f in ("vx", "vy", "vz", "p")}
    out = {f: torch.zeros_like(dev[f]) for f in ("vx", "vy", "vz")}
    dt = 0.0123
    k = consts_for(c, dt)
    halo = (1, 1, 1, 1, 1, 1)
    calls = [region_boxes(n, halo, "interior"), region_boxes(n, halo, "boundary")]
    if not split:
        calls = [calls[0] + calls[1]]
    for bx in calls:
        arr, nb = boxes_c(bx)
        L.check(L.lib().sf_launch_update_velocity(C.byref(lay), ptr(dev["vx"]), ptr(dev["vy"]), ptr(dev["vz"]),
                                                  ptr(dev["p"]), ptr(out["vx"]), ptr(out["vy"]), ptr(out["vz"]),
                                                  C.byref(k), arr, nb, stream()))
    torch.cuda.synchronize()
    o.provisional(dt)  # refresh + UPDATE_VELOCITY + swap (cfd.hpp:275-282)
    for f in ("vx", "vy", "vz"):
        assert same(owned(lay, from_dev(lay, out[f])), owned(lay, o.local_front(f))), f


@pytest.mark.parametrize("region", ["all", "interior", "boundary"])
def test_launch_divergence_and_pressure_sweep_match_run_kernel(ref_available, region):
    c = Case(extents=(21, 13, 9), symmetry_z=False, lid_speed=0.8)
    o = random_oracle(c, 12)
    o.provisional(0.017)  # sets the step constants' dt both kernels use
    o.refresh(list(FIELDS5))
    _, n, lo = block_of(c)
    lay = layout(n, lo, c.ghost)
    k = consts_for(c, 0.017)
    dev = {f: to_dev(lay, o.local_front(f)) for f in FIELDS5}
    arr, nb = boxes_c(region_boxes(n, (1, 0, 1, 0, 1, 0), region))
    if nb:
        L.check(L.lib().sf_launch_divergence(C.byref(lay), ptr(dev["vx"]), ptr(dev["vy"]), ptr(dev["vz"]),
                                             ptr(dev["divu"]), C.byref(k), arr, nb, stream()))
    o.run_kernel("DIVERGENCE", {}, region)
    torch.cuda.synchronize()
    assert same(from_dev(lay, dev["divu"]), o.local_front("divu"))
    o.refresh(["divu"])
    dev["divu"] = to_dev(lay, o.local_front("divu"))
    arr, nb = boxes_c(region_boxes(n, (0, 1, 0, 1, 0, 1), region))
    if nb:
        L.check(L.lib().sf_launch_pressure_sweep(C.byref(lay), ptr(dev["divu"]), ptr(dev["p"]), ptr(dev["vx"]),
                                                 ptr(dev["vy"]), ptr(dev["vz"]), C.byref(k), C.c_double(0.37), 1,
                                                 arr, nb, stream()))
    o.run_kernel("PRESSURE_SWEEP", {"beta": 0.37, "color": 1}, region)
    torch.cuda.synchronize()
    for f in ("p", "vx", "vy", "vz"):
        assert same(from_dev(lay, dev[f]), o.local_front(f)), f


# ---- the refresh as exchanger::refresh_worker issues it ------------------------------
def device_refresh(case, decomp, lays, dev, fields):
    """exchanger::refresh (exchange.hpp:98-119) through level-2 calls: per axis
    phase, every processor face (or periodic self-wrap) is one copy of the
    neighbour's g owned layers, widened over the earlier axes' ghosts
    (sf_launch_copy_box: the pack + unpack of one message between two blocks
    on one device), then every physical face is one sf_launch_bc_face."""
    g = case.ghost
    lib = L.lib()
    for axis in range(3):
        for f in fields:
            for w in range(decomp.workers):
                n = decomp.size(w)
                for side in (0, 1):
                    nb = decomp.neighbor(w, axis, side)
                    if nb < 0:
                        continue
                    m = decomp.size(nb)
                    dims = [n[a] + 2 * g if a < axis else n[a] for a in range(3)]
                    dims[axis] = g
                    src = [-g if a < axis else 0 for a in range(3)]
                    dst = list(src)
                    src[axis] = m[axis] - g if side == 0 else 0
                    dst[axis] = -g if side == 0 else n[axis]
                    a64 = lambda v: (C.c_int64 * 3)(*v)  # noqa: E731
                    L.check(lib.sf_launch_copy_box(C.byref(lays[nb]), ptr(dev[nb][f]), C.byref(lays[w]),
                                                   ptr(dev[w][f]), a64(src), a64(dims), a64(dst), stream()))
            for w in range(decomp.workers):
                for side in (0, 1):
                    if decomp.neighbor(w, axis, side) >= 0:
                        continue
                    bc = face_bc(case, axis, side)
                    L.check(lib.sf_launch_bc_face(C.byref(lays[w]), ptr(dev[w][f]), STAGGER[f], axis, side,
                                                  C.byref(bc), SCOPE_ALL, stream()))
    torch.cuda.synchronize()


@pytest.mark.parametrize("workers", [1, 2, 4])
@pytest.mark.parametrize("ghost", [1, 2])
@pytest.mark.parametrize("per", [(False, False, False), (True, False, False), (False, True, True)])
def test_launch_bc_face_and_copy_box_reproduce_the_reference_refresh(ref_available, workers, ghost, per):
    # every ghost cell of every field (normal pins, tangential reflection of a
    # moving lid, scalar mirrors, symmetry planes, self-wraps, processor faces)
    c = Case(extents=(14, 11, 9), periodic=per, symmetry_z=not per[2], lid_speed=0.7, ghost=ghost,
             workers=workers)
    try:
        o = random_oracle(c, 13)
    except Exception:
        pytest.skip("infeasible decomposition")
    d = sfb.decompose(c.extents, workers, ghost, per)
    lays, dev = [], []
    for w in range(workers):
        lays.append(layout(d.size(w), d.lo[w], ghost))
        dev.append({f: to_dev(lays[w], o.local_front(f, w)) for f in FIELDS5})
    device_refresh(c, d, lays, dev, FIELDS5)
    o.refresh(list(FIELDS5))
    for w in range(workers):
        for f in FIELDS5:
            assert same(from_dev(lays[w], dev[w][f]), o.local_front(f, w)), (f, w)


def test_launch_bc_face_rejects_an_unset_face():
    lay = layout((8, 8, 8), (0, 0, 0), 1)
    t = torch.zeros(lay.sx * lay.sy * lay.sz, dtype=torch.float64, device="cuda")
    bc = L.FaceBC()
    with pytest.raises(sfb.GridError, match="no boundary condition on axis 1 high face"):
        L.check(L.lib().sf_launch_bc_face(C.byref(lay), ptr(t), -1, 1, 1, C.byref(bc), SCOPE_ALL, stream()))


def test_launch_bc_face_allocates_nothing_per_call():
    # the task travels as a kernel parameter: no device allocation, so the
    # call is legal inside stream capture (an allocation would break it)
    lay = layout((16, 12, 10), (0, 0, 0), 2)
    t = torch.randn(lay.sx * lay.sy * lay.sz, dtype=torch.float64, device="cuda")
    bc = L.FaceBC()
    bc.kind = BC_WALL
    bc.velocity[0] = 0.5
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        L.check(L.lib().sf_launch_bc_face(C.byref(lay), ptr(t), 0, 1, 1, C.byref(bc), SCOPE_ALL,
                                          C.c_void_p(s.cuda_stream)))
    ref = t.clone()
    L.check(L.lib().sf_launch_bc_face(C.byref(lay), ptr(ref), 0, 1, 1, C.byref(bc), SCOPE_ALL, stream()))
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(t, ref)


# ---- messages ----------------------------------------------------------------------
def test_launch_pack_and_unpack_move_boxes_bitwise():
    g = 2
    lay = layout((37, 13, 11), (5, 0, 3), g)
    rng = np.random.default_rng(3)
    padded = rng.standard_normal((11 + 2 * g, 13 + 2 * g, 37 + 2 * g))
    src = to_dev(lay, padded)
    lib = L.lib()
    for lo, dims in [((-2, 0, 0), (2, 13, 11)), ((0, -2, -2), (37, 2, 15)), ((3, 4, 5), (33, 7, 2)),
                     ((-2, -2, -2), (41, 17, 15))]:
        cnt = dims[0] * dims[1] * dims[2]
        buf = torch.full((cnt,), np.nan, dtype=torch.float64, device="cuda")
        a64 = lambda v: (C.c_int64 * 3)(*v)  # noqa: E731
        L.check(lib.sf_launch_pack_box(C.byref(lay), ptr(src), a64(lo), a64(dims), ptr(buf), stream()))
        sl = (slice(lo[2] + g, lo[2] + g + dims[2]), slice(lo[1] + g, lo[1] + g + dims[1]),
              slice(lo[0] + g, lo[0] + g + dims[0]))
        torch.cuda.synchronize()
        assert same(buf.cpu().numpy(), padded[sl].reshape(-1))
        dst = torch.zeros_like(src)
        L.check(lib.sf_launch_unpack_box(C.byref(lay), ptr(dst), a64(lo), a64(dims), ptr(buf), stream()))
        torch.cuda.synchronize()
        want = np.zeros_like(padded)
        want[sl] = padded[sl]
        assert same(from_dev(lay, dst), want)


# ---- reductions ----------------------------------------------------------------------
def test_launch_reduce_max_matches_the_reference_and_accumulates(ref_available):
    c = Case(extents=(23, 9, 6), symmetry_z=False)
    o = random_oracle(c, 14)
    _, n, lo = block_of(c)
    lay = layout(n, lo, c.ghost)
    lib = L.lib()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    for f in ("vx", "vy", "vz"):
        out.zero_()
        t = to_dev(lay, o.local_front(f))
        L.check(lib.sf_launch_reduce_max(C.byref(lay), ptr(t), None, MAX_ABS, ptr(out), stream()))
        torch.cuda.synchronize()
        assert same(out.cpu().numpy(), np.array([o.reduce(f, "max_abs")])), f
    # accumulation over calls (worker-order combine, reductions.hpp:75-88) and NaN stickiness
    a = to_dev(lay, o.local_front("vx"))
    b = to_dev(lay, o.local_front("vy"))
    out.zero_()
    for t in (a, b):
        L.check(lib.sf_launch_reduce_max(C.byref(lay), ptr(t), None, MAX_ABS, ptr(out), stream()))
    torch.cuda.synchronize()
    assert out.item() == max(o.reduce("vx", "max_abs"), o.reduce("vy", "max_abs"))
    L.check(lib.sf_launch_reduce_max(C.byref(lay), ptr(a), ptr(b), MAX_ABS_DIFF, ptr(out.zero_()), stream()))
    torch.cuda.synchronize()
    want = np.abs(owned(lay, from_dev(lay, a)) - owned(lay, from_dev(lay, b))).max()
    assert out.item() == want
    pa = from_dev(lay, a)
    pa[3, 4, 5] = np.nan
    L.check(lib.sf_launch_reduce_max(C.byref(lay), ptr(to_dev(lay, pa)), None, MAX_ABS, ptr(out.zero_()),
                                     stream()))
    torch.cuda.synchronize()
    assert np.isnan(out.item())
    with pytest.raises(sfb.GridError, match="no back buffer"):
        L.check(lib.sf_launch_reduce_max(C.byref(lay), ptr(a), None, MAX_ABS_DIFF, ptr(out), stream()))


def test_launch_box_lists_are_checked():
    lay = layout((8, 8, 8), (0, 0, 0), 1)
    c = Case(extents=(8, 8, 8))
    k = consts_for(c, 0.01)
    t = torch.zeros(lay.sx * lay.sy * lay.sz, dtype=torch.float64, device="cuda")
    arr, nb = boxes_c([(0, 0, 0, 9, 8, 8)])
    with pytest.raises(sfb.SfError, match="box outside the block"):
        L.check(L.lib().sf_launch_divergence(C.byref(lay), ptr(t), ptr(t), ptr(t), ptr(t), C.byref(k), arr, nb,
                                             stream()))
    arr, nb = boxes_c([(0, 0, 0, 1, 1, 1)] * 9)
    with pytest.raises(sfb.SfError, match="nbox must lie in"):
        L.check(L.lib().sf_launch_divergence(C.byref(lay), ptr(t), ptr(t), ptr(t), ptr(t), C.byref(k), arr, nb,
                                             stream()))
