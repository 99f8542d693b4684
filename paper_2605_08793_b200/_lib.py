"""ctypes binding of libregot_b200.so (the C ABI declared in include/regot_b200.h).

There is no fallback: if the CUDA library is missing this module raises at
load time, and every compute entry point runs sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libregot_b200.so")

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_int64_p = C.POINTER(C.c_int64)
c_float_p = C.POINTER(C.c_float)


class SplrConfigC(C.Structure):
    """regot_splr_config == SplrConfig (splr.h:22-60) + PCG extensions."""

    _fields_ = [
        ("tau_max", C.c_double),
        ("S", C.c_int64),
        ("J", C.c_int64),
        ("density", C.c_double),
        ("c1", C.c_double),
        ("c2", C.c_double),
        ("max_iter", C.c_int64),
        ("tol", C.c_double),
        ("max_ls_trials", C.c_int64),
        ("record_every", C.c_int64),
        ("overlap", C.c_int32),
        ("tile_rows", C.c_int32),
        ("tile_cols", C.c_int32),
        ("cg_max_iter", C.c_int32),
        ("cg_rtol", C.c_double),
    ]


class SinkhornConfigC(C.Structure):
    """regot_sinkhorn_config == SinkhornConfig (sinkhorn.h:16-31)."""

    _fields_ = [("max_iter", C.c_int64), ("record_every", C.c_int64), ("tol", C.c_double)]


class TraceRowC(C.Structure):
    """regot_trace_row == TraceRow (trace.h:11-18)."""

    _fields_ = [
        ("iter", C.c_int64),
        ("wall_ms", C.c_double),
        ("f", C.c_double),
        ("marginal_error", C.c_double),
        ("duality_gap", C.c_double),
    ]


class StepRecordC(C.Structure):
    """regot_step_record == SplrStepRecord (splr.h:294-312) + cg_iters."""

    _fields_ = [
        ("iter", C.c_int64),
        ("refresh", C.c_int32),
        ("sinkhorn_selected", C.c_int32),
        ("f_before", C.c_double),
        ("f_after", C.c_double),
        ("f_cand_sinkhorn", C.c_double),
        ("f_cand_qn", C.c_double),
        ("gamma", C.c_double),
        ("g_dot_d", C.c_double),
        ("gnew_dot_d", C.c_double),
        ("curvature_ok", C.c_int32),
        ("ls_failed", C.c_int32),
        ("lowrank_active", C.c_int32),
        ("factor_retries", C.c_int32),
        ("tau", C.c_double),
        ("ls_evals", C.c_int32),
        ("cg_iters", C.c_int32),
    ]


class ResultC(C.Structure):
    """regot_result == SplrResult / SinkhornResult."""

    _fields_ = [
        ("status", C.c_int32),
        ("reserved", C.c_int32),
        ("n", C.c_int64),
        ("m", C.c_int64),
        ("alpha", c_double_p),
        ("beta", c_double_p),
        ("trace", C.POINTER(TraceRowC)),
        ("n_trace", C.c_int64),
        ("steps", C.POINTER(StepRecordC)),
        ("n_steps", C.c_int64),
        ("eta", C.c_double),
        ("algo", C.c_char * 16),
        ("config_hash", C.c_char * 24),
        ("message", C.c_char * 256),
        ("device_ms", C.c_double),
        ("gradient_passes", C.c_int64),
        ("lse_passes", C.c_int64),
        ("kernel_launches", C.c_int64),
    ]


class GradientInfoC(C.Structure):
    _fields_ = [
        ("f", C.c_double),
        ("marginal_error", C.c_double),
        ("duality_gap", C.c_double),
        ("grad_norm2", C.c_double),
        ("total_mass", C.c_double),
    ]


# every symbol include/regot_b200.h declares: name -> (restype, argtypes)
_vp = C.c_void_p
PROTOTYPES = {
    "regot_b200_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "regot_b200_destroy": (None, [_vp]),
    "regot_b200_last_error": (C.c_char_p, [_vp]),
    "regot_b200_status_name": (C.c_char_p, [C.c_int]),
    "regot_b200_version": (C.c_char_p, []),
    "regot_b200_comm_unique_id": (C.c_int, [_vp]),
    "regot_b200_comm_init": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "regot_b200_set_problem": (C.c_int, [_vp, C.c_int64, C.c_int64, _vp, C.c_int, C.c_int64, _vp, _vp, C.c_double]),
    "regot_b200_set_problem_rows": (
        C.c_int,
        [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _vp, C.c_int, C.c_int64, _vp, _vp, C.c_double],
    ),
    "regot_b200_set_problem_device": (
        C.c_int,
        [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _vp, C.c_int64, _vp, _vp, C.c_double],
    ),
    "regot_b200_set_pointcloud": (
        C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int32, _vp, _vp, _vp, _vp, C.c_double, C.c_int32]),
    "regot_b200_set_pointcloud_rows": (
        C.c_int,
        [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int32, _vp, _vp, _vp, _vp, C.c_double, C.c_int32],
    ),
    "regot_b200_get_cost": (C.c_int, [_vp, _vp]),
    "regot_b200_validate_problem": (C.c_int, [_vp]),
    "regot_b200_set_eta": (C.c_int, [_vp, C.c_double]),
    "regot_b200_fused_gradient": (C.c_int, [_vp, _vp, _vp, C.POINTER(GradientInfoC), _vp, _vp, _vp]),
    "regot_b200_plan": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int]),
    "regot_b200_optimal_alpha": (C.c_int, [_vp, _vp, _vp, _vp]),
    "regot_b200_optimal_beta": (C.c_int, [_vp, _vp, _vp]),
    "regot_b200_sinkhorn_step": (C.c_int, [_vp, _vp, _vp]),
    "regot_b200_run_sinkhorn": (C.c_int, [_vp, _vp, _vp, C.POINTER(SinkhornConfigC), C.POINTER(ResultC)]),
    "regot_b200_select_topk_dense": (
        C.c_int,
        [_vp, C.c_int64, C.c_int64, _vp, C.c_int, C.c_int64, _vp, C.c_int64, c_int64_p],
    ),
    "regot_b200_topk_budget": (C.c_int64, [C.c_int64, C.c_int64, C.c_double]),
    "regot_b200_assemble_topk": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_double, _vp, _vp, C.POINTER(_vp)]),
    "regot_b200_assemble": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, C.c_double, _vp, _vp, C.POINTER(_vp)]),
    "regot_b200_update_values": (C.c_int, [_vp, _vp, _vp, _vp, C.c_double, _vp, _vp]),
    "regot_b200_matvec": (C.c_int, [_vp, _vp, _vp, _vp]),
    "regot_b200_sparse_info": (C.c_int, [_vp, c_int32_p, c_int64_p, c_int64_p, C.POINTER(C.c_uint64)]),
    "regot_b200_sparse_export": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "regot_b200_sparse_export_local": (C.c_int, [_vp, _vp, _vp, _vp, C.c_int64, c_int64_p]),
    "regot_b200_sparse_free": (None, [_vp]),
    "regot_b200_compute_direction": (
        C.c_int,
        [_vp, _vp, _vp, _vp, _vp, C.c_double, C.c_double, C.c_double, C.c_int32, _vp, c_int32_p],
    ),
    "regot_b200_run_splr": (C.c_int, [_vp, _vp, _vp, C.POINTER(SplrConfigC), C.POINTER(ResultC)]),
    "regot_b200_splr_init": (C.c_int, [_vp, _vp, _vp, C.POINTER(SplrConfigC), C.POINTER(_vp)]),
    "regot_b200_splr_step": (C.c_int, [_vp, _vp, C.POINTER(SplrConfigC), C.POINTER(StepRecordC)]),
    "regot_b200_splr_state_info": (C.c_int, [_vp, _vp, c_int64_p, c_int32_p, C.POINTER(GradientInfoC)]),
    "regot_b200_splr_state_point": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "regot_b200_splr_state_matrix": (_vp, [_vp]),
    "regot_b200_splr_state_free": (None, [_vp]),
    "regot_b200_splr_config_default": (None, [C.POINTER(SplrConfigC)]),
    "regot_b200_sinkhorn_config_default": (None, [C.POINTER(SinkhornConfigC)]),
    "regot_b200_splr_config_validate": (C.c_int, [C.POINTER(SplrConfigC)]),
    "regot_b200_sinkhorn_config_validate": (C.c_int, [C.POINTER(SinkhornConfigC)]),
    "regot_b200_splr_config_hash": (None, [C.POINTER(SplrConfigC), C.c_char_p]),
    "regot_b200_sinkhorn_config_hash": (None, [C.POINTER(SinkhornConfigC), C.c_char_p]),
    "regot_b200_result_free": (None, [C.POINTER(ResultC)]),
    "regot_b200_host_row_block": (None, [C.c_int64, C.c_int, C.c_int, c_int64_p, c_int64_p]),
    "regot_b200_host_pick_bucket": (None, [C.POINTER(C.c_uint64), C.c_int, C.c_int64, C.POINTER(C.c_int), c_int64_p]),
    "regot_b200_time_kernel": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int, c_float_p]),
    "regot_b200_launch_count": (C.c_int64, [_vp]),
    "regot_b200_set_pattern_reuse": (C.c_int, [_vp, C.c_double, C.c_int]),
    "regot_b200_pattern_counts": (None, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "regot_b200_set_profiling": (C.c_int, [_vp, C.c_int]),
    "regot_b200_get_profile": (C.c_int, [_vp, C.c_int, c_int64_p, c_double_p]),
}

_lib = None


def load() -> C.CDLL:
    """Load the CUDA library (once).  Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_2605_08793_b200/csrc).  There is no CPU fallback."
        )
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, (res, args) in PROTOTYPES.items():
        fn = getattr(lib, name)  # AttributeError here == header and library disagree
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
