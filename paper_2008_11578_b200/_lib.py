"""ctypes binding of liborca_b200.so (the C ABI in include/orca_b200.h).

There is no CPU fallback: `load()` raises if the shared library has not been
built (`python -c "import __graft_entry__ as g; g.build()"` or
`make -C paper_2008_11578_b200/csrc`), and every entry point fails with
OrcaError if no CUDA device is usable.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ORCA_B200_LIB: load another build of the same ABI (kernel experiments)
LIB_PATH = os.environ.get("ORCA_B200_LIB") or os.path.join(_HERE, "liborca_b200.so")

ORCA_F32, ORCA_F64, ORCA_MIXED, ORCA_CERT32 = 0, 1, 2, 3
ORCA_MAX_NEIGHBORS = 32
ORCA_N_STAGES = 6
STAGE_NAMES = ["bins", "gather", "solve", "fallback", "finish", "metrics"]
ORCA_EINVAL, ORCA_ECUDA = -1, -2
ORCA_ECOINCIDENT, ORCA_ERANGE = -3, -4
ORCA_ECAPACITY, ORCA_EUNSUPPORTED, ORCA_ETIMEOUT = -5, -6, -7
ORCA_IPC_HANDLE_BYTES = 64

# every symbol include/orca_b200.h declares (checked by tests/test_abi.py)
SYMBOLS = [
    "orca_abi_version", "orca_create", "orca_destroy", "orca_set_stream", "orca_set_params",
    "orca_last_error", "orca_upload", "orca_download", "orca_download_pv", "orca_upload_pv",
    "orca_download_last_step_pv", "orca_download_last_step_kept",
    "orca_step", "orca_run", "orca_run_logged", "orca_sync", "orca_get_info", "orca_step_host", "orca_advance_host", "orca_reorder_rows",
    "orca_profile_stages", "orca_get_stage_ms",
    "orca_debug_last_step", "orca_lp_solve_batch", "orca_lp_release_scratch", "orca_lp_batch_create",
    "orca_lp_batch_set_stream", "orca_lp_batch_solve", "orca_lp_batch_download",
    "orca_lp_batch_destroy", "orca_vo_exit_batch", "orca_shuffle_order", "orca_problem_seed",
    "orca_least_penetration", "orca_neighbor_query", "orca_neighbor_query_all",
    "orca_strip_pack", "orca_strip_append", "orca_strip_drop_ghosts",
    "orca_strip_halo_record_bytes", "orca_strip_configure", "orca_strip_pack_halo",
    "orca_strip_append_slab", "orca_strip_step", "orca_strip_stats",
    "orca_strip_window_create", "orca_strip_window_open", "orca_strip_window_push",
    "orca_strip_window_wait", "orca_strip_window_close",
]

RECORD_BYTES = 96   # sizeof(orca_agent_record)
RECORD_DTYPE = np.dtype([("x", "f8"), ("y", "f8"), ("vx", "f8"), ("vy", "f8"), ("radius", "f8"),
                         ("pref_speed", "f8"), ("max_speed", "f8"), ("goal_tol", "f8"),
                         ("goal_x", "f8"), ("goal_y", "f8"), ("id", "i8"), ("class_code", "i8")])


# orca_frame_record (orca_run_logged)
FRAME_RECORD_DTYPE = np.dtype([("frame", "i8"), ("active_agents", "i8"), ("rows_before", "i8"),
                               ("lp_fallbacks", "i8"), ("removed_agents", "i8"), ("collision_count", "i8"),
                               ("min_separation", "f8")])

# slabs of the device-side exchange protocol (orca_slab_header + records)
SLAB_HEADER_BYTES = 32
SLAB_HEADER_DTYPE = np.dtype([("count", "i4"), ("overflow", "i4"), ("reserved", "i8", (3,))])
HALO_DTYPE_F32 = np.dtype([("x", "f4"), ("y", "f4"), ("vx", "f4"), ("vy", "f4"), ("radius", "f4"),
                           ("class_code", "u4"), ("id", "i8")])                      # 32 bytes
HALO_DTYPE_F64 = np.dtype([("x", "f8"), ("y", "f8"), ("vx", "f8"), ("vy", "f8"), ("radius", "f8"),
                           ("id", "i8"), ("class_code", "i8"), ("pad", "i8")])       # 64 bytes


class OrcaError(RuntimeError):
    """A C-ABI call failed; .code is the ORCA_E* value."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[orca_b200 rc={code}] {message}")
        self.code = code
        self.message = message


class OrcaParams(C.Structure):
    _fields_ = [("dt", C.c_double), ("tau", C.c_double), ("neighbor_radius", C.c_double),
                ("avoidance_margin", C.c_double), ("fmat", C.c_double * 4),
                ("max_neighbors", C.c_int32), ("remove_arrivals", C.c_int32),
                ("compute_metrics", C.c_int32), ("reserved", C.c_int32)]


class OrcaInfo(C.Structure):
    _fields_ = [("frame", C.c_int64), ("active_agents", C.c_int64), ("lp_fallbacks", C.c_int64),
                ("removed_agents", C.c_int64), ("collision_count", C.c_int64),
                ("min_separation", C.c_double), ("grid_nx", C.c_int32), ("grid_ny", C.c_int32),
                ("grid_cell", C.c_double), ("kernel_launches", C.c_int64),
                ("gather_queue", C.c_int64), ("solve_queue", C.c_int64)]


_lib = None


def load():
    """Load liborca_b200.so and declare its prototypes. Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: the CUDA extension has not been built. Run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (needs nvcc). "
            "paper_2008_11578_b200 has no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp, i64, f64, u64, ci = C.c_void_p, C.c_int64, C.c_double, C.c_uint64, C.c_int
    P = C.POINTER
    L.orca_abi_version.restype = ci
    L.orca_create.argtypes = [P(vp), ci, i64, ci]
    L.orca_destroy.argtypes = [vp]
    L.orca_destroy.restype = None
    L.orca_set_stream.argtypes = [vp, vp]
    L.orca_set_params.argtypes = [vp, P(OrcaParams)]
    L.orca_last_error.argtypes = [vp]
    L.orca_last_error.restype = C.c_char_p
    L.orca_upload.argtypes = [vp, i64, i64] + [vp] * 9
    L.orca_download.argtypes = [vp] + [vp] * 9
    L.orca_download_pv.argtypes = [vp, vp, vp]
    L.orca_download_last_step_pv.argtypes = [vp, i64, vp, vp]
    L.orca_download_last_step_kept.argtypes = [vp, i64, vp]
    L.orca_upload_pv.argtypes = [vp, i64, i64, vp, vp]
    L.orca_step.argtypes = [vp]
    L.orca_run.argtypes = [vp, i64]
    L.orca_run_logged.argtypes = [vp, i64, vp, P(i64), vp, i64, P(i64), vp, vp, i64, P(i64)]
    L.orca_sync.argtypes = [vp]
    L.orca_get_info.argtypes = [vp, P(OrcaInfo)]
    L.orca_step_host.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp]
    L.orca_advance_host.argtypes = [vp, i64, i64, vp, vp, vp, vp, C.POINTER(OrcaInfo)]
    L.orca_reorder_rows.argtypes = [vp]
    L.orca_profile_stages.argtypes = [vp, ci]
    L.orca_get_stage_ms.argtypes = [vp, P(C.c_double), P(i64)]
    L.orca_debug_last_step.argtypes = [vp, i64] + [vp] * 8
    L.orca_lp_solve_batch.argtypes = [ci, ci, i64] + [vp] * 9
    L.orca_lp_release_scratch.argtypes = []
    L.orca_lp_batch_create.argtypes = [P(vp), ci, ci, i64] + [vp] * 6
    L.orca_lp_batch_set_stream.argtypes = [vp, vp]
    L.orca_lp_batch_solve.argtypes = [vp]
    L.orca_lp_batch_download.argtypes = [vp, vp, vp, vp]
    L.orca_lp_batch_destroy.argtypes = [vp]
    L.orca_lp_batch_destroy.restype = None
    L.orca_vo_exit_batch.argtypes = [ci, ci, i64, vp, vp]
    L.orca_least_penetration.argtypes = [ci, ci, i64, vp, vp, f64, i64, f64, f64, vp]
    L.orca_neighbor_query.argtypes = [ci, i64, vp, vp, f64, C.c_int32, vp, vp]
    L.orca_neighbor_query_all.argtypes = [ci, i64, vp, vp, f64, i64, vp, vp, P(i64)]
    L.orca_shuffle_order.argtypes = [ci, i64, u64, vp]
    L.orca_problem_seed.argtypes = [ci, i64, i64, P(u64)]
    L.orca_strip_pack.argtypes = [vp, f64, f64, ci, vp, i64, P(i64)]
    L.orca_strip_append.argtypes = [vp, vp, i64, ci]
    L.orca_strip_drop_ghosts.argtypes = [vp]
    L.orca_strip_halo_record_bytes.argtypes = [vp]
    L.orca_strip_configure.argtypes = [vp, f64, f64, f64, i64]
    L.orca_strip_pack_halo.argtypes = [vp, f64, vp, vp, i64]
    L.orca_strip_append_slab.argtypes = [vp, vp, i64, ci]
    L.orca_strip_step.argtypes = [vp, vp, vp, i64]
    L.orca_strip_stats.argtypes = [vp, P(i64), P(i64)]
    L.orca_strip_window_create.argtypes = [vp, i64, vp, P(vp)]
    L.orca_strip_window_open.argtypes = [vp, ci, vp, vp]
    L.orca_strip_window_push.argtypes = [vp, ci, vp, i64, i64, i64]
    L.orca_strip_window_wait.argtypes = [vp, ci, i64, P(vp)]
    L.orca_strip_window_close.argtypes = [vp]
    for name in SYMBOLS:
        fn = getattr(L, name)
        if name == "orca_strip_halo_record_bytes":
            fn.restype = i64
        elif name not in ("orca_destroy", "orca_last_error", "orca_lp_batch_destroy"):
            fn.restype = ci
    _lib = L
    return L


def check(rc: int, handle=None):
    if rc == 0:
        return
    msg = load().orca_last_error(handle)
    raise OrcaError(rc, msg.decode("utf-8", "replace") if msg else "unknown error")


def ptr(a):
    """void* of a C-contiguous numpy array (or NULL for None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


_PRECISIONS = {"f32": ORCA_F32, "float32": ORCA_F32, "f64": ORCA_F64, "float64": ORCA_F64,
               "mixed": ORCA_MIXED, "cert32": ORCA_CERT32, ORCA_F32: ORCA_F32, ORCA_F64: ORCA_F64,
               ORCA_MIXED: ORCA_MIXED, ORCA_CERT32: ORCA_CERT32}


def precision_code(precision) -> int:
    """'mixed' (FP32 state, FP64 arithmetic; default), 'f32' or 'f64' -> ORCA_* code."""
    try:
        return _PRECISIONS[precision]
    except (KeyError, TypeError):
        raise ValueError(f"unknown precision {precision!r} (use 'f64', 'mixed', 'cert32' or 'f32')") from None


def precision_name(code: int) -> str:
    return {ORCA_F32: "f32", ORCA_F64: "f64", ORCA_MIXED: "mixed", ORCA_CERT32: "cert32"}[code]
