"""ctypes bindings for the CPU oracles -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this module; the product package never does.

Two checkers live behind the same Python surface (``Oracle``):

* ``kind="ref"``  -- ``oracle/_ref/libsfref.so``: the unmodified reference
  (stencilforge, header-only C++20) compiled in place by ``oracle/Makefile``
  and driven through ``oracle/ref_shim.cpp``.  Supports every worker count,
  run mode, tile and kernel form of ``cfd::simulation`` (cfd.hpp:175-222).
* ``kind="port"`` -- ``oracle/build/libsforacle.so``: our plain-C restatement
  ``oracle/sf_oracle.c`` (single worker; results are decomposition-invariant,
  which the reference's own tests pin: tests/test_cfd.cpp:231-273, 436-461).

Fields are exchanged as global x-fastest float64 arrays of shape (nz, ny, nx),
the layout of grid::gather / grid::scatter (io.hpp:25-65).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field as dfield
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsfref.so")
PORT_SO = os.path.join(HERE, "build", "libsforacle.so")

FIELDS = ("vx", "vy", "vz", "p", "divu")
REDUCE_OPS = {"max_abs": 0, "sum": 1, "sum_sq": 2, "max_abs_diff": 3}
REGIONS = {"all": 0, "interior": 1, "boundary": 2}


class OracleError(RuntimeError):
    pass


class _Params(C.Structure):
    _fields_ = [
        ("extents", C.c_int64 * 3),
        ("spacing", C.c_double * 3),
        ("periodic", C.c_int * 3),
        ("reynolds", C.c_double),
        ("sigma", C.c_double),
        ("tolerance", C.c_double),
        ("omega", C.c_double),
        ("max_sweeps", C.c_int),
        ("symmetry_z", C.c_int),
        ("viscosity", C.c_double),
        ("density", C.c_double),
        ("body_force", C.c_double * 3),
        ("lid_speed", C.c_double),
        ("blend", C.c_double),
        ("workers", C.c_int),
        ("mode", C.c_int),
        ("tile", C.c_int * 3),
        ("ghost", C.c_int),
        ("form", C.c_int),
    ]


@dataclass
class Case:
    """Flat solver_config + fluid_params (cfd.hpp:29-67) plus driver options."""

    extents: Sequence[int] = (8, 8, 8)
    spacing: Sequence[float] | None = None  # default: unit box, 1/n
    periodic: Sequence[bool] = (False, False, False)
    reynolds: float = 100.0
    sigma: float = 0.5
    tolerance: float = 1e-6
    omega: float = 1.7
    max_sweeps: int = 500
    symmetry_z: bool = True
    viscosity: float = 0.01
    density: float = 1.0
    body_force: Sequence[float] = (0.0, 0.0, 0.0)
    lid_speed: float = 1.0
    blend: float = 0.0
    workers: int = 1
    mode: str = "plain"
    tile: Sequence[int] = (0, 0, 0)
    ghost: int = 1
    form: str = "rows"

    def params(self) -> _Params:
        p = _Params()
        sp = self.spacing or [1.0 / n for n in self.extents]
        for a in range(3):
            p.extents[a] = int(self.extents[a])
            p.spacing[a] = float(sp[a])
            p.periodic[a] = 1 if self.periodic[a] else 0
            p.body_force[a] = float(self.body_force[a])
            p.tile[a] = int(self.tile[a])
        p.reynolds, p.sigma, p.tolerance, p.omega = self.reynolds, self.sigma, self.tolerance, self.omega
        p.max_sweeps = int(self.max_sweeps)
        p.symmetry_z = 1 if self.symmetry_z else 0
        p.viscosity, p.density = self.viscosity, self.density
        p.lid_speed, p.blend = self.lid_speed, self.blend
        p.workers = int(self.workers)
        p.mode = 1 if self.mode == "overlap" else 0
        p.ghost = int(self.ghost)
        p.form = 1 if self.form == "points" else 0
        return p


def cavity_case(n: int | Sequence[int], **kw) -> Case:
    """cli::run_config defaults (config.hpp:51-94) for a unit-box cavity:
    viscosity = lid_speed / re."""
    ext = (n, n, n) if isinstance(n, int) else tuple(n)
    re = kw.pop("reynolds", 100.0)
    lid = kw.pop("lid_speed", 1.0)
    return Case(extents=ext, reynolds=re, lid_speed=lid, viscosity=lid * 1.0 / re, **kw)


_libs: dict[str, C.CDLL] = {}


def _load(kind: str) -> C.CDLL:
    if kind in _libs:
        return _libs[kind]
    path = REF_SO if kind == "ref" else PORT_SO
    if not os.path.exists(path):
        raise OracleError(f"oracle library {path} not built (run `make -C oracle`)")
    lib = C.CDLL(path)
    pre = "sfref_" if kind == "ref" else "sfo_"
    vp, d, i, i64 = C.c_void_p, C.c_double, C.c_int, C.c_int64
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
    sigs = {
        "last_error": ([], C.c_char_p),
        "create": ([C.POINTER(_Params)], vp),
        "destroy": ([vp], None),
        "init_cavity": ([vp], i),
        "init_uniform": ([vp, d, d, d], i),
        "init_taylor_green": ([vp], i),
        "scatter": ([vp, C.c_char_p, dp, i64], i),
        "gather": ([vp, C.c_char_p, dp], i),
        "local_front": ([vp, C.c_char_p, i, dp, C.POINTER(i64), C.POINTER(i64)], i),
        "compute_dt": ([vp, dp], i),
        "provisional": ([vp, d], i),
        "pressure_iteration": ([vp, d, ip, dp], i),
        "step": ([vp, dp, ip, dp], i),
        "advance": ([vp, i, dp, ip, dp], i),
        "checksum": ([vp], C.c_uint64),
        "time": ([vp], d),
        "step_count": ([vp], C.c_long),
        "pending_color": ([vp], i),
        "reduce": ([vp, C.c_char_p, i, dp], i),
        "refresh": ([vp, C.c_char_p], i),
        "exchange": ([vp, C.c_char_p], i),
        "run_kernel": ([vp, C.c_char_p, C.c_char_p, i], i),
        "invalidate_all_ghosts": ([vp], None),
        "diag": ([vp, dp, dp, dp], i),
        "taylor_green_error": ([vp, d, dp], i),
        "time_phases": ([vp, dp, dp, ip], i),
        "time_half_sweeps": ([vp, i, d, dp], i),
        "time_provisional": ([vp, dp, dp], i),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(lib, pre + name, None)
        if fn is None:
            continue
        fn.argtypes = args
        fn.restype = res
    lib._pre = pre  # type: ignore[attr-defined]
    _libs[kind] = lib
    return lib


def available(kind: str) -> bool:
    try:
        _load(kind)
        return True
    except OracleError:
        return False


def ref_ccl(text: str, fields: Sequence[str] | None = None, directory: str | None = None) -> tuple[int, str]:
    """The reference's descriptor front end (descriptor.hpp / codegen.hpp) on
    `text`: without `fields`, parse + canonical render; with them, parse +
    validate_all + the concatenated rendered headers, and write_generated into
    `directory`. Returns (0, result) or (1 parse_error | 2 descriptor_error |
    3 other, message)."""
    lib = _load("ref")
    buf = C.create_string_buffer(1 << 20)
    if fields is None:
        f = lib.sfref_ccl_render
        f.argtypes, f.restype = [C.c_char_p, C.c_char_p, C.c_size_t], C.c_int
        rc = f(text.encode(), buf, len(buf))
    else:
        f = lib.sfref_ccl_generate
        f.argtypes, f.restype = [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p, C.c_size_t], C.c_int
        rc = f(text.encode(), ",".join(fields).encode(), (directory or ".").encode(), buf, len(buf))
    if rc == 0:
        return 0, buf.value.decode()
    err = lib.sfref_last_error
    err.restype = C.c_char_p
    return rc, err().decode()


def ref_parse_config(text: str) -> tuple[int, str]:
    """The reference's cli::parse_run_config on `text`: (0, key=value lines) or
    (1 config_error | 2 cfd_error | 3 other, message)."""
    lib = _load("ref")
    buf = C.create_string_buffer(1 << 16)
    f = lib.sfref_parse_config
    f.argtypes, f.restype = [C.c_char_p, C.c_char_p, C.c_size_t], C.c_int
    rc = f(text.encode(), buf, len(buf))
    if rc == 0:
        return 0, buf.value.decode()
    err = lib.sfref_last_error
    err.restype = C.c_char_p
    return rc, err().decode()


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Oracle:
    """One CPU simulation (reference or restatement) with the cfd::simulation API."""

    def __init__(self, case: Case, kind: str = "ref"):
        self.kind = kind
        self.case = case
        self._lib = _load(kind)
        self._f = lambda n: getattr(self._lib, self._lib._pre + n)
        p = case.params()
        h = self._f("create")(C.byref(p))
        if not h:
            raise OracleError(self._err())
        self._h = h
        self.extents = tuple(int(x) for x in case.extents)

    def _err(self) -> str:
        return self._f("last_error")().decode()

    def _ck(self, rc: int) -> None:
        if rc != 0:
            raise OracleError(self._err())

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._f("destroy")(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- initial states ---------------------------------------------------
    def init_cavity(self):
        self._ck(self._f("init_cavity")(self._h))

    def init_uniform(self, c):
        self._ck(self._f("init_uniform")(self._h, *map(float, c)))

    def init_taylor_green(self):
        self._ck(self._f("init_taylor_green")(self._h))

    # -- data movement ----------------------------------------------------
    def scatter(self, name: str, data: np.ndarray):
        a = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        self._ck(self._f("scatter")(self._h, name.encode(), _dp(a), a.size))

    def gather(self, name: str) -> np.ndarray:
        nx, ny, nz = self.extents
        out = np.empty((nz, ny, nx), dtype=np.float64)
        self._ck(self._f("gather")(self._h, name.encode(), _dp(out)))
        return out

    def local_front(self, name: str, worker: int = 0) -> np.ndarray:
        """Worker's padded front array incl. ghosts, shape (nz+2g, ny+2g, nx+2g)."""
        g = self.case.ghost
        # the largest block cannot exceed the domain
        nx, ny, nz = self.extents
        buf = np.empty((nz + 2 * g) * (ny + 2 * g) * (nx + 2 * g), dtype=np.float64)
        dims = (C.c_int64 * 3)()
        lo = (C.c_int64 * 3)()
        self._ck(self._f("local_front")(self._h, name.encode(), worker, _dp(buf), dims, lo))
        d = [dims[0] + 2 * g, dims[1] + 2 * g, dims[2] + 2 * g]
        return buf[: d[0] * d[1] * d[2]].reshape(d[2], d[1], d[0]).copy()

    # -- the time step ----------------------------------------------------
    def compute_dt(self) -> float:
        v = C.c_double()
        self._ck(self._f("compute_dt")(self._h, C.byref(v)))
        return v.value

    def provisional(self, dt: float):
        self._ck(self._f("provisional")(self._h, float(dt)))

    def pressure_iteration(self, dt: float):
        s, r = C.c_int(), C.c_double()
        self._ck(self._f("pressure_iteration")(self._h, float(dt), C.byref(s), C.byref(r)))
        return s.value, r.value

    def step(self):
        dt, s, r = C.c_double(), C.c_int(), C.c_double()
        self._ck(self._f("step")(self._h, C.byref(dt), C.byref(s), C.byref(r)))
        return dt.value, s.value, r.value

    def advance(self, n: int):
        dts = np.zeros(max(n, 1))
        sw = np.zeros(max(n, 1), dtype=np.int32)
        res = np.zeros(max(n, 1))
        self._ck(self._f("advance")(self._h, int(n), _dp(dts), sw.ctypes.data_as(C.POINTER(C.c_int)), _dp(res)))
        return dts[:n], sw[:n], res[:n]

    def checksum(self) -> str:
        return "%016x" % self._f("checksum")(self._h)

    @property
    def time(self) -> float:
        return self._f("time")(self._h)

    @property
    def step_count(self) -> int:
        return self._f("step_count")(self._h)

    @property
    def pending_color(self) -> int:
        return self._f("pending_color")(self._h)

    def reduce(self, name: str, op: str = "max_abs") -> float:
        v = C.c_double()
        self._ck(self._f("reduce")(self._h, name.encode(), REDUCE_OPS[op], C.byref(v)))
        return v.value

    def refresh(self, names: Sequence[str]):
        self._ck(self._f("refresh")(self._h, ",".join(names).encode()))

    def exchange(self, names: Sequence[str]):
        self._ck(self._f("exchange")(self._h, ",".join(names).encode()))

    def run_kernel(self, name: str, params: dict | None = None, region: str = "all"):
        ps = ",".join(f"{k}={float(v)!r}" for k, v in (params or {}).items())
        self._ck(self._f("run_kernel")(self._h, name.encode(), ps.encode(), REGIONS[region]))

    def invalidate_all_ghosts(self):
        self._f("invalidate_all_ghosts")(self._h)

    def max_divergence(self) -> float:
        v = C.c_double()
        self._ck(self._f("diag")(self._h, C.byref(v), None, None))
        return v.value

    def steady_delta(self) -> float:
        v = C.c_double()
        self._ck(self._f("diag")(self._h, None, C.byref(v), None))
        return v.value

    def kinetic_energy(self) -> float:
        v = C.c_double()
        self._ck(self._f("diag")(self._h, None, None, C.byref(v)))
        return v.value

    def taylor_green_error(self, t: float) -> float:
        v = C.c_double()
        self._ck(self._f("taylor_green_error")(self._h, float(t), C.byref(v)))
        return v.value

    def time_half_sweeps(self, k: int, beta: float) -> float:
        t = C.c_double()
        self._ck(self._f("time_half_sweeps")(self._h, int(k), float(beta), C.byref(t)))
        return t.value

    def time_provisional(self):
        t, dt = C.c_double(), C.c_double()
        self._ck(self._f("time_provisional")(self._h, C.byref(t), C.byref(dt)))
        return t.value, dt.value

    def time_phases(self):
        tp, ti, s = C.c_double(), C.c_double(), C.c_int()
        self._ck(self._f("time_phases")(self._h, C.byref(tp), C.byref(ti), C.byref(s)))
        return tp.value, ti.value, s.value


def fnv1a_checksum(fields: dict) -> str:
    """FNV-1a over name bytes + gathered float64 bytes of vx, vy, vz, p
    (bench.hpp:24-39).  numpy restatement used to checksum device gathers."""
    h = 1469598103934665603
    prime = 1099511628211
    mask = (1 << 64) - 1
    for name in ("vx", "vy", "vz", "p"):
        for b in name.encode():
            h = ((h ^ b) * prime) & mask
        data = np.ascontiguousarray(fields[name], dtype="<f8").view(np.uint8).reshape(-1)
        h = _fnv_bytes(h, data)
    return "%016x" % h


def _fnv_bytes(h: int, data: np.ndarray) -> int:
    # vectorised FNV-1a is inherently sequential; use the C oracle when built
    try:
        lib = _load("port")
        fn = getattr(lib, "sfo_fnv1a", None)
        if fn is not None:
            fn.argtypes = [C.c_uint64, C.c_void_p, C.c_int64]
            fn.restype = C.c_uint64
            return int(fn(h, data.ctypes.data, data.size))
    except OracleError:
        pass
    prime = 1099511628211
    mask = (1 << 64) - 1
    for b in data.tolist():
        h = ((h ^ b) * prime) & mask
    return h
