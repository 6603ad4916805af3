"""ctypes binding of libbal.so (include/bal.h).  Argument marshalling only: every step of the hot
path runs inside the CUDA library; this module never computes any part of the method.
The library is mandatory -- importing this module fails loudly when libbal.so is missing."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BAL_LIB_PATH") or os.path.join(HERE, "libbal.so")  # override: build variants

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libbal.so not built at {LIB_PATH}: run `python -m paper_2407_00046_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

c_double_p = C.POINTER(C.c_double)
c_int_p = C.POINTER(C.c_int32)
c_u8_p = C.POINTER(C.c_uint8)

BAL_OK = 0
STATUS = {0: "OK", -1: "INVALID_ARG", -2: "BAD_MESH", -3: "INFEASIBLE", -4: "NOT_CONVERGED",
          -5: "CONSTRAINT_BUDGET", -6: "CUDA", -7: "NCCL", -8: "OOM", -9: "NAN"}
BAL_NO_WARMSTART = 1
BAL_NO_AUGLAG = 2
BAL_FRICTION_LAGGED = 4
BAL_SIGMA_CAP = 8
BAL_SIGMA_MIN = 16
BAL_FRICTION_NO_FREEZE = 32
BAL_CCD_LITERAL = 64
BAL_PCG_LITERAL_STALL = 128
BAL_FP32_MATRIX = 256
BAL_ADDITIVE_PRECOND = 512
BAL_PCG_CRIT_I = 1024
BAL_PCG_CRIT_II = 2048
BAL_PCG_CRIT_III = 4096


class bal_mesh(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("n_tets", C.c_int32), ("rest_x", c_double_p), ("tets", c_int_p),
                ("node_fixed", c_u8_p), ("tet_material", c_int_p), ("n_obstacle_tris", C.c_int32),
                ("obstacle_tris", c_int_p)]


class bal_material(C.Structure):
    _fields_ = [("E", C.c_double), ("nu", C.c_double), ("rho", C.c_double), ("model", C.c_int32)]


class bal_params(C.Structure):
    _fields_ = [("h", C.c_double), ("gravity", C.c_double * 3), ("dhat", C.c_double), ("eps_v", C.c_double),
                ("chi", C.c_double), ("newton_rel_tol", C.c_double), ("pcg_rel_tol", C.c_double),
                ("pcg_stall_window", C.c_int32), ("pcg_resume_iters", C.c_int32), ("alpha_min", C.c_double),
                ("ws_rel_tol", C.c_double), ("ws_max_iters", C.c_int32), ("max_newton", C.c_int32),
                ("max_pcg", C.c_int32), ("max_constraints", C.c_int64), ("flags", C.c_uint32)]


class bal_step_stats(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("pcg_iters", C.c_int64), ("ws_iters", C.c_int64),
                ("max_constraints", C.c_int32), ("max_aprime", C.c_int32), ("sigma0", C.c_double),
                ("sigma_final", C.c_double), ("min_distance", C.c_double), ("last_rel_grad", C.c_double),
                ("ms_total", C.c_double), ("ms_collision", C.c_double), ("ms_assembly", C.c_double),
                ("ms_warmstart", C.c_double), ("ms_pcg", C.c_double), ("ms_linesearch", C.c_double)]


class bal_contact_state(C.Structure):
    _fields_ = [("n_active", C.c_int32), ("active_keys", c_int_p), ("n_aprime", C.c_int32),
                ("aprime_keys", c_int_p), ("aprime_mu", c_double_p), ("aprime_s", c_double_p),
                ("sigma", C.c_double), ("n_friction", C.c_int32), ("friction_keys", c_int_p),
                ("friction_gamma", c_double_p), ("friction_n", c_double_p), ("friction_lambda", c_double_p),
                ("x_t", c_double_p), ("y", c_double_p)]


class bal_system_view(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nnzb_static", C.c_int32), ("static_row_ptr", C.c_void_p),
                ("static_col", C.c_void_p), ("static_val", C.c_void_p), ("nnzb_contact", C.c_int32),
                ("contact_row_ptr", C.c_void_p), ("contact_col", C.c_void_p), ("contact_val", C.c_void_p),
                ("diag_inv", C.c_void_p), ("grad", C.c_void_p), ("e_node", C.c_void_p), ("group", C.c_void_p),
                ("n_elastic", C.c_int32), ("elastic_blocks", C.c_void_p), ("elastic_lbar", C.c_void_p),
                ("n_contact_stencils", C.c_int32), ("contact_blocks", C.c_void_p), ("contact_lbar", C.c_void_p),
                ("contact_stencil_nodes", C.c_void_p), ("n_friction_stencils", C.c_int32),
                ("contact_grad", C.c_void_p)]


class bal_pcg_opts(C.Structure):
    _fields_ = [("warm_start", C.c_int32), ("rel_tol", C.c_double), ("stall_window", C.c_int32),
                ("max_iters", C.c_int32), ("ws_rel_tol", C.c_double), ("ws_max_iters", C.c_int32)]


class bal_pcg_stats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("stop_reason", C.c_int32), ("ws_iters_max", C.c_int32),
                ("n_groups", C.c_int32), ("rel_residual", C.c_double)]


HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int32, c_double_p, C.c_int32, C.c_void_p)
HOST_EXCHANGE = C.CFUNCTYPE(C.c_int32, c_double_p, c_int_p, c_double_p, c_int_p, C.c_void_p)


class bal_dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("host_allreduce", HOST_ALLREDUCE), ("host_exchange", HOST_EXCHANGE), ("user", C.c_void_p)]


class bal_bsr_host(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("nnzb", C.c_int32), ("row_ptr", c_int_p), ("col", c_int_p),
                ("val", c_double_p), ("group", c_int_p)]


_sig = {
    "bal_init": (C.c_int, [C.POINTER(bal_mesh), C.POINTER(bal_material), C.c_int32, C.POINTER(bal_params),
                           C.POINTER(bal_dist), C.POINTER(C.c_void_p)]),
    "bal_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "bal_dist_info": (C.c_int, [C.c_void_p, c_int_p, c_int_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "bal_halo_plan": (C.c_int32, [C.c_int32, c_int_p, c_int_p, C.c_int32, c_int_p, C.c_int32, c_int_p, c_int_p,
                                  c_int_p, c_int_p, C.c_int32]),
    "bal_halo_pack": (C.c_int, [C.c_int32, c_int_p, c_double_p, c_double_p]),
    "bal_halo_unpack": (C.c_int, [C.c_int32, c_int_p, c_double_p, c_double_p]),
    "bal_spmv_rows": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "bal_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bal_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(bal_step_stats)]),
    "bal_step_host": (C.c_int, [C.c_void_p, c_double_p, c_double_p, c_double_p, c_double_p,
                                C.POINTER(bal_step_stats)]),
    "bal_frame_begin": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "bal_frame_iterate": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]),
    "bal_frame_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(bal_step_stats)]),
    "bal_frame_peek": (C.c_int, [C.c_void_p, C.POINTER(bal_step_stats)]),
    "bal_assemble": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(bal_contact_state), C.POINTER(bal_system_view)]),
    "bal_get_system": (C.c_int, [C.c_void_p, C.POINTER(bal_system_view)]),
    "bal_detect": (C.c_int, [C.c_void_p, C.c_void_p, c_int_p, c_double_p, C.c_int32, C.POINTER(C.c_int32)]),
    "bal_spmv": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "bal_pcg": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(bal_pcg_opts),
                          C.POINTER(bal_pcg_stats)]),
    "bal_load_bsr": (C.c_int, [C.c_void_p, C.POINTER(bal_bsr_host)]),
    "bal_bench_spmv": (C.c_int, [C.c_void_p, C.c_int32, c_double_p]),
    "bal_get_trace": (C.c_int32, [C.c_void_p, c_double_p, C.c_int32]),
    "bal_spmv_counters": (C.c_int, [C.c_void_p, c_double_p]),
    "bal_pcg_history": (C.c_int32, [C.c_void_p, c_double_p, C.c_int32]),
    "bal_pcg_objective_history": (C.c_int32, [C.c_void_p, c_double_p, C.c_int32]),
    "bal_kernel_launches": (C.c_int64, [C.c_void_p]),
    "bal_partition_rows": (C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.c_int32, c_int_p]),
    "bal_ghost_columns": (C.c_int32, [C.c_int32, c_int_p, c_int_p, C.c_int32, C.c_int32, c_int_p, C.c_int32]),
    "bal_last_error": (C.c_char_p, [C.c_void_p]),
    "bal_destroy": (None, [C.c_void_p]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTS = tuple(_sig)


def ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))
