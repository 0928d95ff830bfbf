"""Python face of the device simulation: the cfd::simulation API (cfd.hpp:173-766)
and the exec::executor operations on its fields (executor.hpp:477-862), over
the C ABI.  All compute runs in the CUDA library; this module only marshals.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _lib as L

FIELDS = ("vx", "vy", "vz", "p", "divu")
REGIONS = {"all": 0, "interior": 1, "boundary": 2}
REDUCE_OPS = {"max_abs": 0, "sum": 1, "sum_sq": 2, "max_abs_diff": 3}


@dataclass
class SolverConfig:
    """cfd::solver_config (cfd.hpp:43-67)."""

    extents: Sequence[int] = (33, 33, 3)
    spacing: Sequence[float] | None = None  # default: unit box (cfd::unit_box, cfd.hpp:69-74)
    periodic: Sequence[bool] = (False, False, False)
    reynolds: float = 100.0
    sigma: float = 0.5
    tolerance: float = 1e-6
    omega: float = 1.7
    max_sweeps: int = 500
    symmetry_z: bool = True
    output_cadence: int = 0

    def to_c(self) -> L.SolverConfig:
        c = L.SolverConfig()
        sp = self.spacing or [1.0 / float(n) for n in self.extents]
        for a in range(3):
            c.extents[a] = int(self.extents[a])
            c.spacing[a] = float(sp[a])
            c.origin[a] = 0.0
            c.periodic[a] = 1 if self.periodic[a] else 0
        c.reynolds, c.sigma, c.tolerance, c.omega = self.reynolds, self.sigma, self.tolerance, self.omega
        c.max_sweeps = int(self.max_sweeps)
        c.symmetry_z = 1 if self.symmetry_z else 0
        c.output_cadence = int(self.output_cadence)
        return c


@dataclass
class FluidParams:
    """cfd::fluid_params (cfd.hpp:29-41)."""

    viscosity: float = 0.01
    density: float = 1.0
    body_force: Sequence[float] = (0.0, 0.0, 0.0)
    lid_speed: float = 1.0
    blend: float = 0.0

    def to_c(self) -> L.FluidParams:
        p = L.FluidParams()
        p.viscosity, p.density = self.viscosity, self.density
        for a in range(3):
            p.body_force[a] = float(self.body_force[a])
        p.lid_speed, p.blend = self.lid_speed, self.blend
        return p


def cavity_fluid(cfg: SolverConfig, alpha: float = 0.0) -> FluidParams:
    """cfd::cavity_fluid (cfd.hpp:78-84)."""
    return FluidParams(viscosity=1.0 * 1.0 / cfg.reynolds, lid_speed=1.0, blend=alpha)


INTENTS = {"IN": 0, "OUT": 1, "INOUT": 2, "SEPARATEINOUT": 3}
STAGGER = {"none": -1, "x": 0, "y": 1, "z": 2}


@dataclass
class ExecutionPlan:
    """codegen::execution_plan (codegen.hpp:41-57): kernel name, TILE, per-face
    halo (-x,+x,-y,+y,-z,+z), bindings [(field, intent, cached)] in declaration
    order, parameter names."""

    kernel: str
    tile: Sequence[int] = (16, 16, 16)
    halo: Sequence[int] = (0, 0, 0, 0, 0, 0)
    bindings: Sequence[tuple] = ()
    parameters: Sequence[str] = ()


BC_KINDS = {"unset": 0, "wall": 1, "symmetry": 2, "outflow": 3}
STEP_KINDS = {"run": 0, "exchange": 1, "physical_bc": 2, "refresh": 3, "reduce": 4}


@dataclass
class ScheduleStep:
    """exec::schedule_step (executor.hpp:422-466)."""

    kind: str
    kernel: str = ""
    region: str = "all"
    fields: Sequence[str] = ()
    source: str = ""
    op: str = "max_abs"
    target: str = ""

    @staticmethod
    def run(kernel, region="all"):
        return ScheduleStep("run", kernel=kernel, region=region)

    @staticmethod
    def exchange(fields):
        return ScheduleStep("exchange", fields=tuple(fields))

    @staticmethod
    def physical_bc(fields):
        return ScheduleStep("physical_bc", fields=tuple(fields))

    @staticmethod
    def refresh(fields):
        return ScheduleStep("refresh", fields=tuple(fields))

    @staticmethod
    def reduce(source, op, target):
        return ScheduleStep("reduce", source=source, op=op, target=target)


@dataclass
class StepStats:
    dt: float
    sweeps: int
    residual: float


def _host_f64(buf, what: str, pinned: bool = False):
    """(pointer, element count) of a contiguous float64 host buffer (numpy
    array or CPU torch tensor); the C side reads or writes 8 bytes per
    element, so any other dtype or a strided view is rejected."""
    if hasattr(buf, "data_ptr"):  # torch tensor
        import torch
        if buf.is_cuda:
            raise ValueError(f"{what}: expected a host buffer, got a CUDA tensor")
        if buf.dtype != torch.float64 or not buf.is_contiguous():
            raise ValueError(f"{what}: expected a contiguous float64 tensor, got {buf.dtype}"
                             f"{'' if buf.is_contiguous() else ' (non-contiguous)'}")
        if pinned and not buf.is_pinned():
            raise ValueError(f"{what}: an asynchronous transfer needs a pinned tensor")
        return buf.data_ptr(), buf.numel()
    if pinned:
        raise ValueError(f"{what}: an asynchronous transfer needs a pinned tensor")
    if not isinstance(buf, np.ndarray) or buf.dtype != np.float64 or not buf.flags.c_contiguous:
        raise ValueError(f"{what}: expected a C-contiguous float64 array")
    return buf.ctypes.data, buf.size


def _device_f64(t, what: str):
    import torch
    if t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous float64 CUDA tensor, got {t.dtype}")
    return t


def _cstrs(names: Iterable[str]):
    ns = [n.encode() for n in names]
    arr = (C.c_char_p * max(1, len(ns)))(*ns)
    return arr, len(ns)


class Simulation:
    """Device-resident cfd::simulation.  ``workers`` grid components of
    grid::decompose() live on ``device``.  ``fused``: 1/True = fused half-sweep,
    TMA-pipelined, with the temporal pass (two half-sweeps per launch) wherever
    every face is a wall, a symmetry plane or a processor face and, with
    processor faces, ``ghost`` >= 2 (default); 3 = TMA half-sweeps only; 2 =
    fused half-sweep with plain loads; 0/False = the reference's unfused
    dataflow (refresh, SWEEP, refresh, DIV, reduce)."""

    def __init__(self, cfg: SolverConfig, par: FluidParams, workers: int = 1, mode: str = "plain",
                 tile: Sequence[int] = (0, 0, 0), ghost: int = 1, form: str = "rows",
                 device: int = 0, fused: int | bool = True, rank: int | None = None,
                 world: int | None = None, nccl_id: bytes | None = None, transport: str | None = None,
                 group=None, precision: str = "f64"):
        """With ``nccl_id`` (from :func:`nccl_unique_id` on rank 0, broadcast to all
        ranks) the simulation is the rank-``rank`` component of a ``world``-rank
        decomposition and exchanges ghosts over NCCL.
        With ``transport="ipc"`` it exchanges them through CUDA IPC instead
        (peers' device buffers mapped into this process); the host side of that
        transport (handles, residual maxima, barriers) runs over the
        ``torch.distributed`` process group ``group`` (default: the world
        group, e.g. gloo). Ranks may then share one device.
        ``precision="f32"`` stores the five CFD fields in fp32 and runs the
        fused TMA half-sweep and UPDATE_VELOCITY in fp32 arithmetic (the fp32
        variant; compared with the fp64 reference under per-field tolerances,
        tests/test_gpu_fp32.py)."""
        self._h = None
        self.cfg, self.par = cfg, par
        self._lib = L.lib()
        opt = L.SimOptions()
        self._lib.sf_sim_options_default(C.byref(opt))
        opt.workers, opt.mode = int(workers), (1 if mode == "overlap" else 0)
        for a in range(3):
            opt.tile[a] = int(tile[a])
        opt.ghost, opt.form, opt.device, opt.fused = int(ghost), (1 if form == "points" else 0), int(device), int(fused)
        if precision not in ("f64", "f32"):
            raise ValueError("precision must be 'f64' or 'f32'")
        opt.precision = 8 if precision == "f64" else 4  # f32: the fp32 variant of the CFD fields
        self._ccfg, self._cpar, self._opt = cfg.to_c(), par.to_c(), opt
        h = C.c_void_p()
        if transport == "ipc":
            self._transport = _TorchHostTransport(group)
            L.check(self._lib.sf_sim_create_ipc(C.byref(self._ccfg), C.byref(self._cpar), C.byref(opt),
                                                int(rank or 0), int(world or 1), C.byref(self._transport.c),
                                                C.byref(h)))
        elif transport not in (None, "nccl"):
            raise ValueError("transport must be 'nccl' or 'ipc'")
        elif nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
            L.check(self._lib.sf_sim_create_distributed(C.byref(self._ccfg), C.byref(self._cpar), C.byref(opt),
                                                        int(rank or 0), int(world or 1), idbuf, C.byref(h)))
        else:
            L.check(self._lib.sf_sim_create(C.byref(self._ccfg), C.byref(self._cpar), C.byref(opt), C.byref(h)))
        self._h = h
        self._async_keep = []  # host buffers of queued transfers, held until synchronize()
        self.rank = int(rank or 0)
        self.world = int(world or 1)
        self.extents = tuple(int(x) for x in cfg.extents)
        self.workers = int(workers)

    # -- lifetime ----------------------------------------------------------
    def close(self) -> None:
        if self._h:
            self._lib.sf_sim_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- initial states (cfd.hpp:229-257) -----------------------------------
    def init_cavity(self):
        L.check(self._lib.sf_sim_init_cavity(self._h))

    def init_uniform(self, c):
        L.check(self._lib.sf_sim_init_uniform(self._h, *map(float, c)))

    def init_taylor_green(self):
        L.check(self._lib.sf_sim_init_taylor_green(self._h))

    # -- the time step (cfd.hpp:264-321) ------------------------------------
    def compute_dt(self) -> float:
        v = C.c_double()
        L.check(self._lib.sf_sim_compute_dt(self._h, C.byref(v)))
        return v.value

    def provisional(self, dt: float):
        L.check(self._lib.sf_sim_provisional(self._h, float(dt)))

    def pressure_iteration(self, dt: float):
        s, r = C.c_int(), C.c_double()
        L.check(self._lib.sf_sim_pressure_iteration(self._h, float(dt), C.byref(s), C.byref(r)))
        return s.value, r.value

    def step(self) -> StepStats:
        st = L.StepStats()
        L.check(self._lib.sf_sim_step(self._h, C.byref(st)))
        return StepStats(st.dt, st.sweeps, st.residual)

    def advance(self, n: int) -> StepStats:
        st = L.StepStats()
        L.check(self._lib.sf_sim_advance(self._h, int(n), C.byref(st)))
        return StepStats(st.dt, st.sweeps, st.residual)

    @property
    def time(self) -> float:
        return self._lib.sf_sim_time(self._h)

    @property
    def step_count(self) -> int:
        return self._lib.sf_sim_step_count(self._h)

    @property
    def pending_color(self) -> int:
        return self._lib.sf_sim_pending_color(self._h)

    # -- diagnostics (cfd.hpp:342-363) --------------------------------------
    def max_divergence(self) -> float:
        v = C.c_double()
        L.check(self._lib.sf_sim_max_divergence(self._h, C.byref(v)))
        return v.value

    def steady_delta(self) -> float:
        v = C.c_double()
        L.check(self._lib.sf_sim_steady_delta(self._h, C.byref(v)))
        return v.value

    def taylor_green_error(self, t: float) -> float:
        """RMS distance to the decayed analytic vortex (cfd.hpp:367-401), bitwise the reference's."""
        v = C.c_double()
        L.check(self._lib.sf_sim_taylor_green_error(self._h, float(t), C.byref(v)))
        return v.value

    def kinetic_energy(self) -> float:
        v = C.c_double()
        L.check(self._lib.sf_sim_kinetic_energy(self._h, C.byref(v)))
        return v.value

    # -- data movement (io.hpp:25-65, bench.hpp:24-39) -----------------------
    @property
    def cells(self) -> int:
        nx, ny, nz = self.extents
        return nx * ny * nz

    def scatter(self, name: str, data) -> None:
        if hasattr(data, "is_cuda") and data.is_cuda:
            import torch
            t = data.to(torch.float64).contiguous()
            cur, ext = self._torch_order()
            ext.wait_stream(cur)  # the data was produced on torch's stream
            L.check(self._lib.sf_sim_scatter_device(self._h, name.encode(), C.c_void_p(t.data_ptr()), t.numel()))
            # torch's stream waits for the copy: a temporary from .to()/.contiguous()
            # goes back to the caching allocator on that stream, so no later torch
            # work can reuse it before the copy ran (no record_stream on the
            # library's stream, which may be destroyed before the tensor)
            cur.wait_stream(ext)
            return
        if hasattr(data, "data_ptr"):
            import torch
            data = data.to(torch.float64).contiguous()
            ptr, n = data.data_ptr(), data.numel()
        else:
            data = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
            ptr, n = data.ctypes.data, data.size
        L.check(self._lib.sf_sim_scatter(self._h, name.encode(), C.c_void_p(ptr), n))

    def gather(self, name: str, out=None) -> np.ndarray:
        nx, ny, nz = self.extents
        if out is not None and hasattr(out, "is_cuda") and out.is_cuda:
            _device_f64(out, "gather(out=)")
            cur, ext = self._torch_order()
            ext.wait_stream(cur)  # torch may still use `out`
            L.check(self._lib.sf_sim_gather_device(self._h, name.encode(), C.c_void_p(out.data_ptr()), out.numel()))
            cur.wait_stream(ext)  # later torch work sees the gathered values
            return out
        if out is not None:
            ptr, n = _host_f64(out, "gather(out=)")
            L.check(self._lib.sf_sim_gather(self._h, name.encode(), C.c_void_p(ptr), n))
            return out
        a = np.empty((nz, ny, nx), dtype=np.float64)
        L.check(self._lib.sf_sim_gather(self._h, name.encode(), C.c_void_p(a.ctypes.data), a.size))
        return a

    def block_shape(self, worker: int | None = None):
        d = decompose(self.extents, self.world if self.world > 1 else self.workers, int(self._opt.ghost),
                      tuple(bool(x) for x in self.cfg.periodic))
        return d.size(self.rank if worker is None else worker)

    def gather_block(self, name: str, worker: int | None = None, out=None, wait: bool = True):
        """Owned block -> dense host array. ``wait=False`` queues the download
        (``out`` must be pinned, e.g. a pinned torch tensor) and returns; call
        ``synchronize()`` before reading it."""
        w = self.rank if worker is None else worker
        if out is None:
            if not wait:
                raise ValueError("an asynchronous gather needs a pinned `out` buffer")
            nx, ny, nz = self.block_shape(w)
            out = np.empty((nz, ny, nx), dtype=np.float64)
        ptr, n = _host_f64(out, "gather_block(out=)", pinned=not wait)
        fn = self._lib.sf_sim_gather_block if wait else self._lib.sf_sim_gather_block_async
        L.check(fn(self._h, name.encode(), int(w), C.c_void_p(ptr), n))
        if not wait:
            self._async_keep.append(out)
        return out

    def scatter_block(self, name: str, data, worker: int | None = None, wait: bool = True):
        """Dense host array -> owned block. ``wait=False`` queues the upload
        (``data`` must be pinned and unchanged until ``synchronize()``)."""
        w = self.rank if worker is None else worker
        if wait and not hasattr(data, "data_ptr"):
            data = np.ascontiguousarray(data, dtype=np.float64)
        ptr, n = _host_f64(data, "scatter_block", pinned=not wait)
        fn = self._lib.sf_sim_scatter_block if wait else self._lib.sf_sim_scatter_block_async
        L.check(fn(self._h, name.encode(), int(w), C.c_void_p(ptr), n))
        if not wait:
            self._async_keep.append(data)

    def stage_block(self, name: str, data, worker: int | None = None):
        """First half of an asynchronous scatter: queue the upload of ``data``
        (pinned, unchanged until ``synchronize()``) into the field's device
        buffer. ``install_staged`` later copies it into the field in stream
        order, so staging step k+1's inputs before ``step()`` overlaps the
        transfer with step k."""
        w = self.rank if worker is None else worker
        ptr, n = _host_f64(data, "stage_block", pinned=True)
        L.check(self._lib.sf_sim_stage_block_async(self._h, name.encode(), int(w), C.c_void_p(ptr), n))
        self._async_keep.append(data)

    def install_staged(self, name: str, worker: int | None = None):
        w = self.rank if worker is None else worker
        L.check(self._lib.sf_sim_install_staged(self._h, name.encode(), int(w)))

    def checksum(self) -> str:
        v = C.c_uint64()
        L.check(self._lib.sf_sim_checksum(self._h, C.byref(v)))
        return "%016x" % v.value

    def local_front(self, name: str, worker: int = 0) -> np.ndarray:
        g = int(self._opt.ghost)
        nx, ny, nz = self.extents
        buf = np.empty((nx + 2 * g) * (ny + 2 * g) * (nz + 2 * g), dtype=np.float64)
        dims = (C.c_int64 * 3)()
        lo = (C.c_int64 * 3)()
        L.check(self._lib.sf_sim_local_front(self._h, name.encode(), int(worker), C.c_void_p(buf.ctypes.data),
                                             buf.size, dims, lo))
        d = [dims[0] + 2 * g, dims[1] + 2 * g, dims[2] + 2 * g]
        return buf[: d[0] * d[1] * d[2]].reshape(d[2], d[1], d[0]).copy()

    # -- executor operations (executor.hpp:500-527) -------------------------
    def refresh(self, names: Sequence[str]):
        arr, n = _cstrs(names)
        L.check(self._lib.sf_sim_refresh(self._h, arr, n))

    def exchange(self, names: Sequence[str]):
        arr, n = _cstrs(names)
        L.check(self._lib.sf_sim_exchange(self._h, arr, n))

    def run_kernel(self, name: str, params: dict | None = None, region: str = "all"):
        params = params or {}
        arr, n = _cstrs(params.keys())
        vals = (C.c_double * max(1, n))(*[float(v) for v in params.values()])
        L.check(self._lib.sf_sim_run_kernel(self._h, name.encode(), arr, vals, n, REGIONS[region]))

    def reduce(self, name: str, op: str = "max_abs") -> float:
        v = C.c_double()
        L.check(self._lib.sf_sim_reduce(self._h, name.encode(), REDUCE_OPS[op], C.byref(v)))
        return v.value

    def create_field(self, name: str, stagger: str | int = "none", dtype: str = "f64"):
        """field_store::create (field.hpp:108-112). ``dtype`` "f32" stores the
        field in fp32 (values still cross the API as fp64)."""
        st = STAGGER[stagger] if isinstance(stagger, str) else int(stagger)
        if dtype not in ("f64", "f32"):
            raise ValueError("dtype must be 'f64' or 'f32'")
        L.check(self._lib.sf_sim_create_field_typed(self._h, name.encode(), st, 8 if dtype == "f64" else 4))

    def register_kernel(self, plan: ExecutionPlan, signature: tuple, body: str):
        """executor::register_kernel (executor.hpp:484-488, 650-692).  ``signature``
        = (fields, params) as kernel_signature; ``body`` is the CUDA C++ body of
        the point function over point_ctx ``c`` (c.field(s)(di,dj,dk), .load(),
        .store(v), c.param(s), c.i/c.j/c.k), JIT-compiled for sm_100a."""
        binds = (L.Binding * max(1, len(plan.bindings)))()
        keep = []
        for i, b in enumerate(plan.bindings):
            name, intent = b[0], b[1]
            cached = b[2] if len(b) > 2 else False
            keep.append(name.encode())
            binds[i].field = keep[-1]
            binds[i].intent = INTENTS[intent] if isinstance(intent, str) else int(intent)
            binds[i].cached = 1 if cached else 0
        params, npar = _cstrs(plan.parameters)
        cp = L.Plan()
        cp.kernel = plan.kernel.encode()
        for a in range(3):
            cp.tile[a] = int(plan.tile[a])
        for a in range(6):
            cp.halo[a] = int(plan.halo[a])
        cp.bindings = binds
        cp.n_bindings = len(plan.bindings)
        cp.params = params
        cp.n_params = npar
        sf, nsf = _cstrs(signature[0])
        sp, nsp = _cstrs(signature[1] if len(signature) > 1 else ())
        L.check(self._lib.sf_sim_register_kernel(self._h, C.byref(cp), sf, nsf, sp, nsp, body.encode()))

    def set_face_bc(self, axis: int, side: int, kind: str, velocity=(0.0, 0.0, 0.0)):
        """executor::boundary() at (axis, side) (exchange.hpp:18-42)."""
        v = (C.c_double * 3)(*map(float, velocity))
        L.check(self._lib.sf_sim_set_face_bc(self._h, int(axis), int(side), BC_KINDS[kind], v))

    def set_boundary_uniform(self, kind: str, velocity=(0.0, 0.0, 0.0)):
        """boundary_spec::uniform (exchange.hpp:37-41)."""
        for a in range(3):
            for sd in range(2):
                self.set_face_bc(a, sd, kind, velocity)

    def physical_bc(self, names: Sequence[str]):
        arr, n = _cstrs(names)
        L.check(self._lib.sf_sim_physical_bc(self._h, arr, n))

    def run_schedule(self, steps: Sequence[ScheduleStep], params: dict | None = None, passes: int = 1,
                     mode: str = "plain", results: dict | None = None):
        """executor::run_schedule (executor.hpp:533-553) with its dry run."""
        cs = (L.ScheduleStep * max(1, len(steps)))()
        keep = []
        for i, st in enumerate(steps):
            fl, nf = _cstrs(st.fields)
            keep.append(fl)
            cs[i].kind = STEP_KINDS[st.kind]
            cs[i].kernel = st.kernel.encode()
            cs[i].region = REGIONS[st.region]
            cs[i].fields = fl
            cs[i].n_fields = nf
            cs[i].source = st.source.encode()
            cs[i].op = REDUCE_OPS[st.op]
            cs[i].target = st.target.encode()
        params = params or {}
        pn, npn = _cstrs(params.keys())
        pv = (C.c_double * max(1, npn))(*[float(v) for v in params.values()])
        L.check(self._lib.sf_sim_run_schedule(self._h, cs, len(steps), pn, pv, npn, int(passes),
                                              1 if mode == "overlap" else 0))
        if results is not None:
            for st in steps:
                if st.kind == "reduce":
                    results[st.target] = self.result(st.target)

    def result(self, name: str) -> float:
        v = C.c_double()
        L.check(self._lib.sf_sim_result(self._h, name.encode(), C.byref(v)))
        return v.value

    def invalidate_ghosts(self, name: str):
        L.check(self._lib.sf_sim_invalidate_ghosts(self._h, name.encode()))

    def invalidate_all_ghosts(self):
        L.check(self._lib.sf_sim_invalidate_all_ghosts(self._h))

    def ghosts_valid(self, name: str) -> bool:
        return bool(self._lib.sf_sim_ghosts_valid(self._h, name.encode()))

    # -- device plumbing -----------------------------------------------------
    def set_direct_exchange(self, mode: int | bool):
        """Temporal-pass exchange across ranks, where the peers' buffers map:
        1/True (default) = fused into the pass (boundary cells store straight
        into the neighbours' ghost shells), 2 = one separate launch of the
        same direct stores after each pass, 0/False = pack / send / unpack
        phases overlapped with the interior."""
        L.check(self._lib.sf_sim_set_direct_exchange(self._h, int(mode)))

    @property
    def direct_exchange(self) -> int:
        """The direct-exchange mode in use (0 = phases; collective on first use)."""
        return int(self._lib.sf_sim_direct_exchange(self._h))

    def synchronize(self):
        L.check(self._lib.sf_sim_synchronize(self._h))
        self._async_keep.clear()

    def _torch_order(self):
        """(torch's current stream, the simulation's stream as a torch stream):
        device-pointer transfers are ordered against torch's work in both
        directions."""
        import torch
        return torch.cuda.current_stream(), torch.cuda.ExternalStream(self.stream)

    @property
    def stream(self) -> int:
        return self._lib.sf_sim_stream(self._h) or 0

    def launch_count(self, reset: bool = False) -> int:
        return int(self._lib.sf_sim_launch_count(self._h, 1 if reset else 0))

    def set_kernel_timing(self, on: bool):
        L.check(self._lib.sf_sim_set_kernel_timing(self._h, 1 if on else 0))

    def kernel_timing(self, kernel: str = "sweep_div"):
        ms, n = C.c_double(), C.c_int64()
        L.check(self._lib.sf_sim_kernel_timing(self._h, kernel.encode(), C.byref(ms), C.byref(n)))
        return ms.value, n.value


class _TorchHostTransport:
    """sf_host_transport over a torch.distributed process group: the
    allgather and barrier callbacks the CUDA-IPC transport calls (from the
    thread that drives the simulation)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self._torch, self._dist, self._group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.error = None
        self._ag = L.ALLGATHER_FN(self._allgather)  # referenced for the simulation's lifetime
        self._bar = L.BARRIER_FN(self._barrier)
        self.c = L.HostTransport(None, self._ag, self._bar)

    def _allgather(self, ctx, send, recv, nbytes):
        try:
            torch = self._torch
            mine = torch.frombuffer(bytearray(C.string_at(send, nbytes)), dtype=torch.uint8) if nbytes else \
                torch.empty(0, dtype=torch.uint8)
            out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(self.world)]
            self._dist.all_gather(out, mine, group=self._group)
            C.memmove(recv, b"".join(bytes(t.numpy()) for t in out), nbytes * self.world)
            return 0
        except Exception as e:  # pragma: no cover - reported through the C status
            self.error = e
            return 1

    def _barrier(self, ctx):
        try:
            self._dist.barrier(group=self._group)
            return 0
        except Exception as e:  # pragma: no cover
            self.error = e
            return 1


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (rank 0 calls it, then broadcasts)."""
    buf = C.create_string_buffer(128)
    L.check(L.lib().sf_nccl_unique_id(buf))
    return buf.raw


@dataclass
class Decomposition:
    """grid::decomposition (grid.hpp:52-86) as computed by the library."""

    extents: tuple
    workers: int
    ghost: int
    proc_grid: tuple
    periodic: tuple
    lo: list = field(default_factory=list)
    hi: list = field(default_factory=list)

    def coords_of(self, w: int):
        pz, py = self.proc_grid[2], self.proc_grid[1]
        return (w // (py * pz), (w // pz) % py, w % pz)

    def neighbor(self, w: int, axis: int, side: int) -> int:
        pg = (C.c_int * 3)(*self.proc_grid)
        per = (C.c_int * 3)(*[1 if p else 0 for p in self.periodic])
        return L.lib().sf_decomp_neighbor(pg, per, int(w), int(axis), int(side))

    def face_physical(self, w: int, axis: int, side: int) -> bool:
        return self.neighbor(w, axis, side) < 0

    def size(self, w: int):
        return tuple(self.hi[w][a] - self.lo[w][a] for a in range(3))


def decompose(extents, workers: int, ghost: int, periodic=(False, False, False), spacing=None) -> Decomposition:
    """grid::decompose (grid.hpp:92-163) -- host logic, no GPU needed."""
    lib = L.lib()
    ext = (C.c_int64 * 3)(*[int(x) for x in extents])
    sp = (C.c_double * 3)(*(spacing or [1.0 / float(n) if n else 1.0 for n in extents]))
    per = (C.c_int * 3)(*[1 if p else 0 for p in periodic])
    pg = (C.c_int * 3)()
    n = max(1, int(workers))
    lo = (C.c_int64 * (3 * n))()
    hi = (C.c_int64 * (3 * n))()
    L.check(lib.sf_decompose(ext, sp, int(workers), int(ghost), per, pg, lo, hi))
    return Decomposition(tuple(int(x) for x in extents), int(workers), int(ghost), tuple(pg),
                         tuple(bool(p) for p in periodic),
                         [tuple(lo[3 * w + a] for a in range(3)) for w in range(workers)],
                         [tuple(hi[3 * w + a] for a in range(3)) for w in range(workers)])
