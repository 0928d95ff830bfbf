"""ctypes binding of the in-tree CUDA library (include/sforge_b200.h).

The library is required: there is no CPU fallback.  Importing the package
without ``_lib/libsfb200.so`` raises immediately; calls that need a GPU fail
with the CUDA error text when none is present.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

LIB_PATH = _build.LIB

SF_OK = 0
STATUS = {1: "config", 2: "grid", 3: "exec", 4: "cfd", 5: "cuda", 6: "arg"}


class SfError(RuntimeError):
    """Raised for a non-zero sf_status; ``kind`` names the reference error type."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code
        self.kind = STATUS.get(code, "unknown")


class ConfigError(SfError):  # cfd_error from validate()
    pass


class GridError(SfError):  # grid::grid_error
    pass


class ExecError(SfError):  # exec::exec_error
    pass


class CfdError(SfError):  # cfd::cfd_error at run time
    pass


_ERRS = {1: ConfigError, 2: GridError, 3: ExecError, 4: CfdError}


class SolverConfig(C.Structure):
    _fields_ = [
        ("extents", C.c_int64 * 3),
        ("spacing", C.c_double * 3),
        ("origin", C.c_double * 3),
        ("periodic", C.c_int * 3),
        ("reynolds", C.c_double),
        ("sigma", C.c_double),
        ("tolerance", C.c_double),
        ("omega", C.c_double),
        ("max_sweeps", C.c_int),
        ("symmetry_z", C.c_int),
        ("output_cadence", C.c_int),
    ]


class FluidParams(C.Structure):
    _fields_ = [
        ("viscosity", C.c_double),
        ("density", C.c_double),
        ("body_force", C.c_double * 3),
        ("lid_speed", C.c_double),
        ("blend", C.c_double),
    ]


class SimOptions(C.Structure):
    _fields_ = [
        ("workers", C.c_int),
        ("mode", C.c_int),
        ("tile", C.c_int * 3),
        ("ghost", C.c_int),
        ("form", C.c_int),
        ("device", C.c_int),
        ("fused", C.c_int),
        ("precision", C.c_int),
    ]


class StepStats(C.Structure):
    _fields_ = [("dt", C.c_double), ("sweeps", C.c_int), ("residual", C.c_double)]


class Layout(C.Structure):
    _fields_ = [
        ("dims", C.c_int64 * 3),
        ("lo", C.c_int64 * 3),
        ("ghost", C.c_int),
        ("sx", C.c_int64),
        ("sy", C.c_int64),
        ("sz", C.c_int64),
        ("base", C.c_int64),
    ]


class Box(C.Structure):
    _fields_ = [("lo", C.c_int64 * 3), ("hi", C.c_int64 * 3)]


class FaceBC(C.Structure):
    _fields_ = [("kind", C.c_int), ("velocity", C.c_double * 3)]


class Binding(C.Structure):
    _fields_ = [("field", C.c_char_p), ("intent", C.c_int), ("cached", C.c_int)]


class Plan(C.Structure):
    _fields_ = [
        ("kernel", C.c_char_p),
        ("tile", C.c_int * 3),
        ("halo", C.c_int * 6),
        ("bindings", C.POINTER(Binding)),
        ("n_bindings", C.c_int),
        ("params", C.POINTER(C.c_char_p)),
        ("n_params", C.c_int),
    ]


class ScheduleStep(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("kernel", C.c_char_p),
        ("region", C.c_int),
        ("fields", C.POINTER(C.c_char_p)),
        ("n_fields", C.c_int),
        ("source", C.c_char_p),
        ("op", C.c_int),
        ("target", C.c_char_p),
    ]


# sf_host_transport (include/sforge_b200.h): host callbacks of the CUDA-IPC transport
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)
BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)


class HostTransport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", ALLGATHER_FN), ("barrier", BARRIER_FN)]


class CfdConsts(C.Structure):
    _fields_ = [
        ("dt", C.c_double), ("nu", C.c_double), ("alpha", C.c_double),
        ("fx", C.c_double), ("fy", C.c_double), ("fz", C.c_double),
        ("ix", C.c_double), ("iy", C.c_double), ("iz", C.c_double),
        ("ix2", C.c_double), ("iy2", C.c_double), ("iz2", C.c_double),
        ("bscale", C.c_double * 8),
        ("nxm1", C.c_int64), ("nym1", C.c_int64), ("nzm1", C.c_int64),
        ("px", C.c_int), ("py", C.c_int), ("pz", C.c_int),
    ]


# (name, argtypes, restype) -- every symbol include/sforge_b200.h declares
_vp, _i, _d, _i64 = C.c_void_p, C.c_int, C.c_double, C.c_int64
_dp, _ip, _i64p = C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_int64)
_cp, _cpp = C.c_char_p, C.POINTER(C.c_char_p)
SIGNATURES = [
    ("sf_abi_version", [], _i),
    ("sf_last_error", [], _cp),
    ("sf_device_count", [], _i),
    ("sf_decompose", [_i64p, _dp, _i, _i, _ip, _ip, _i64p, _i64p], _i),
    ("sf_decomp_neighbor", [_ip, _ip, _i, _i, _i], _i),
    ("sf_sim_options_default", [C.POINTER(SimOptions)], None),
    ("sf_sim_create", [C.POINTER(SolverConfig), C.POINTER(FluidParams), C.POINTER(SimOptions), C.POINTER(_vp)], _i),
    ("sf_sim_destroy", [_vp], None),
    ("sf_sim_init_cavity", [_vp], _i),
    ("sf_sim_init_uniform", [_vp, _d, _d, _d], _i),
    ("sf_sim_init_taylor_green", [_vp], _i),
    ("sf_sim_compute_dt", [_vp, _dp], _i),
    ("sf_sim_provisional", [_vp, _d], _i),
    ("sf_sim_pressure_iteration", [_vp, _d, _ip, _dp], _i),
    ("sf_sim_step", [_vp, C.POINTER(StepStats)], _i),
    ("sf_sim_advance", [_vp, _i, C.POINTER(StepStats)], _i),
    ("sf_sim_time", [_vp], _d),
    ("sf_sim_step_count", [_vp], C.c_long),
    ("sf_sim_pending_color", [_vp], _i),
    ("sf_sim_max_divergence", [_vp, _dp], _i),
    ("sf_sim_steady_delta", [_vp, _dp], _i),
    ("sf_sim_kinetic_energy", [_vp, _dp], _i),
    ("sf_sim_taylor_green_error", [_vp, _d, _dp], _i),
    ("sf_sim_scatter", [_vp, _cp, _vp, _i64], _i),
    ("sf_sim_gather", [_vp, _cp, _vp, _i64], _i),
    ("sf_sim_scatter_device", [_vp, _cp, _vp, _i64], _i),
    ("sf_sim_gather_device", [_vp, _cp, _vp, _i64], _i),
    ("sf_sim_checksum", [_vp, C.POINTER(C.c_uint64)], _i),
    ("sf_sim_local_front", [_vp, _cp, _i, _vp, _i64, _i64p, _i64p], _i),
    ("sf_sim_refresh", [_vp, _cpp, _i], _i),
    ("sf_sim_exchange", [_vp, _cpp, _i], _i),
    ("sf_sim_run_kernel", [_vp, _cp, _cpp, _dp, _i, _i], _i),
    ("sf_sim_reduce", [_vp, _cp, _i, _dp], _i),
    ("sf_sim_create_field", [_vp, _cp, _i], _i),
    ("sf_sim_create_field_typed", [_vp, _cp, _i, _i], _i),
    ("sf_sim_register_kernel", [_vp, C.POINTER(Plan), _cpp, _i, _cpp, _i, _cp], _i),
    ("sf_sim_set_face_bc", [_vp, _i, _i, _i, _dp], _i),
    ("sf_sim_physical_bc", [_vp, _cpp, _i], _i),
    ("sf_sim_run_schedule", [_vp, C.POINTER(ScheduleStep), _i, _cpp, _dp, _i, _i, _i], _i),
    ("sf_sim_result", [_vp, _cp, _dp], _i),
    ("sf_sim_invalidate_ghosts", [_vp, _cp], _i),
    ("sf_sim_invalidate_all_ghosts", [_vp], _i),
    ("sf_sim_ghosts_valid", [_vp, _cp], _i),
    ("sf_nccl_unique_id", [_vp], _i),
    ("sf_sim_create_distributed", [C.POINTER(SolverConfig), C.POINTER(FluidParams), C.POINTER(SimOptions),
                                   _i, _i, _vp, C.POINTER(_vp)], _i),
    ("sf_direct_plan", [_i64p, _i, _i, C.POINTER(_i), _i, _i, _i64p, C.POINTER(_i)], _i),
    ("sf_sim_create_ipc", [C.POINTER(SolverConfig), C.POINTER(FluidParams), C.POINTER(SimOptions), _i, _i,
                           C.POINTER(HostTransport), C.POINTER(_vp)], _i),
    ("sf_sim_set_direct_exchange", [_vp, _i], _i),
    ("sf_sim_direct_exchange", [_vp], _i),
    ("sf_sim_rank", [_vp], _i),
    ("sf_sim_world", [_vp], _i),
    ("sf_sim_gather_block", [_vp, _cp, _i, _vp, _i64], _i),
    ("sf_sim_scatter_block", [_vp, _cp, _i, _vp, _i64], _i),
    ("sf_sim_gather_block_async", [_vp, _cp, _i, _vp, _i64], _i),
    ("sf_sim_scatter_block_async", [_vp, _cp, _i, _vp, _i64], _i),
    ("sf_sim_stage_block_async", [_vp, _cp, _i, _vp, _i64], _i),
    ("sf_sim_install_staged", [_vp, _cp, _i], _i),
    ("sf_exchange_plan", [_i64p, _i, _i, _ip, _i, C.c_uint, _i, _i, _i64p, _ip], _i),
    ("sf_sim_synchronize", [_vp], _i),
    ("sf_sim_stream", [_vp], _vp),
    ("sf_sim_launch_count", [_vp, _i], _i64),
    ("sf_sim_set_kernel_timing", [_vp, _i], _i),
    ("sf_sim_kernel_timing", [_vp, _cp, _dp, _i64p], _i),
    ("sf_make_layout", [_i64p, _i64p, _i, C.POINTER(Layout)], _i),
    ("sf_layout_elems", [C.POINTER(Layout)], _i64),
    ("sf_make_cfd_consts", [C.POINTER(SolverConfig), C.POINTER(FluidParams), C.POINTER(CfdConsts)], _i),
    ("sf_launch_update_velocity", [C.POINTER(Layout), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                   C.POINTER(CfdConsts), C.POINTER(Box), _i, _vp], _i),
    ("sf_launch_divergence", [C.POINTER(Layout), _vp, _vp, _vp, _vp, C.POINTER(CfdConsts),
                              C.POINTER(Box), _i, _vp], _i),
    ("sf_launch_pressure_sweep", [C.POINTER(Layout), _vp, _vp, _vp, _vp, _vp, C.POINTER(CfdConsts),
                                  _d, _i, C.POINTER(Box), _i, _vp], _i),
    ("sf_launch_bc_face", [C.POINTER(Layout), _vp, _i, _i, _i, C.POINTER(FaceBC), _i, _vp], _i),
    ("sf_launch_copy_box", [C.POINTER(Layout), _vp, C.POINTER(Layout), _vp, _i64p, _i64p, _i64p, _vp], _i),
    ("sf_launch_pack_box", [C.POINTER(Layout), _vp, _i64p, _i64p, _vp, _vp], _i),
    ("sf_launch_unpack_box", [C.POINTER(Layout), _vp, _i64p, _i64p, _vp, _vp], _i),
    ("sf_launch_reduce_max", [C.POINTER(Layout), _vp, _vp, _i, _vp, _vp], _i),
]

_lib = None


def _pin_nccl() -> None:
    """Point the library's run-time NCCL load (SF_NCCL_LIB) at the libnccl.so.2
    torch links against (the nvidia-nccl wheel), so a later `import torch` finds
    the same library instead of clashing with an older system copy."""
    if os.environ.get("SF_NCCL_LIB"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations or []) if spec else []:
            cand = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["SF_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def lib() -> C.CDLL:
    """Load the library (building it first if sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) or _build._stale():
        try:
            _build.build()
        except Exception as e:  # no nvcc on the box: a prebuilt .so must exist
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"CUDA library {LIB_PATH} is missing and could not be built: {e}") from e
    _pin_nccl()
    L = C.CDLL(LIB_PATH)
    for name, args, res in SIGNATURES:
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != SF_OK:
        msg = lib().sf_last_error().decode()
        raise _ERRS.get(rc, SfError)(rc, msg)
