"""ctypes binding of libadmm_b200.so (the C ABI declared in include/admm_b200.h).

There is deliberately no fallback: if the shared library is missing the import of
this module raises, and every compute call returns ADMM_E_CUDA without a device.
"""
from __future__ import annotations

import ctypes
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ADMM_B200_LIB", os.path.join(PKG_DIR, "libadmm_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a).  There is no CPU fallback.")

_u64, _dbl, _ptr, _i32, _u32 = (ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p, ctypes.c_int,
                                ctypes.c_uint32)


class SolverConfigC(ctypes.Structure):
    _fields_ = [("rho", _dbl), ("lambda_", _dbl), ("scl", _dbl), ("max_iters", _u64),
                ("eps_pri", _dbl), ("eps_dual", _dbl), ("seed", _u64)]


class PlanOptionsC(ctypes.Structure):
    _fields_ = [("method", _i32), ("M", _u64), ("N", _u64), ("ragged", _i32), ("dtype", _i32),
                ("device", _i32), ("trace_objective", _i32), ("schedule", _i32), ("batch", _u64),
                ("noise_sigma", _dbl)]


class SnapshotC(ctypes.Structure):
    _fields_ = [("iteration", _u64), ("n_pix", _u64), ("v", ctypes.POINTER(_dbl)),
                ("v_prev", ctypes.POINTER(_dbl)), ("n_workers", _u64),
                ("replica_u", ctypes.POINTER(ctypes.POINTER(_dbl))),
                ("replica_len", ctypes.POINTER(_u64)), ("primal", _dbl), ("dual", _dbl)]


class PlanInfoC(ctypes.Structure):
    _fields_ = [("n_blocks", _u64), ("h_bytes", _u64), ("k_bytes", _u64),
                ("h_stream_bytes_per_iter", _u64), ("bytes_per_iter", _u64),
                ("launches_per_iter", _u64), ("grid_gemv_n", _u64), ("grid_gemv_h", _u64),
                ("setup_seconds", _dbl), ("inner_dim_max", _u64), ("schedule", _u64),
                ("grid_sweep", _u64), ("hbm_bytes_per_iter", _u64), ("sweep_variant", _u64),
                ("slab_cluster", _u64), ("slab_row_bytes", _u64), ("slab_rows", _u64),
                ("grid_pr", _u64), ("grid_pc", _u64), ("n_ranks", _u64), ("exchange_bytes_per_iter", _u64),
                ("setup_phase_s", _dbl * 4), ("gram_device_s", _dbl), ("gram_flops", _dbl),
                ("inverse_device_s", _dbl), ("inverse_flops", _dbl)]


class ShardC(ctypes.Structure):
    _fields_ = [("Pr", _u64), ("Pc", _u64), ("pr", _u64), ("pc", _u64)]


OBSERVER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.POINTER(SnapshotC), ctypes.c_void_p)

lib = ctypes.CDLL(LIB_PATH)
ABI_VERSION = 3
if lib.admm_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH}: ABI {lib.admm_abi_version()} != {ABI_VERSION}; rebuild (__graft_entry__.build())")

_SIGS = {
    "admm_abi_version": ([], _i32),
    "admm_last_error": ([], ctypes.c_char_p),
    "admm_last_good_iteration": ([], _u64),
    "admm_plan_create": ([ctypes.POINTER(PlanOptionsC), ctypes.POINTER(SolverConfigC), _u64, _u64,
                          _ptr, _i32, _ptr, ctypes.POINTER(_ptr)], _i32),
    "admm_plan_create_sharded": ([ctypes.POINTER(PlanOptionsC), ctypes.POINTER(SolverConfigC), _u64, _u64,
                                  _ptr, _i32, _ptr, ctypes.POINTER(ShardC), ctypes.POINTER(_ptr)], _i32),
    "admm_nccl_unique_id": ([_ptr], _i32),
    "admm_choose_grid": ([_i32, _i32, _u64, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64)], _i32),
    "admm_plan_create_dist": ([ctypes.POINTER(PlanOptionsC), ctypes.POINTER(SolverConfigC), _u64, _u64,
                               _ptr, _i32, _ptr, ctypes.c_char_p, _i32, _i32, ctypes.POINTER(_ptr)], _i32),
    "admm_plan_create_multi": ([ctypes.POINTER(PlanOptionsC), ctypes.POINTER(SolverConfigC), _u64, _u64,
                                _ptr, _i32, _ptr, _i32, _ptr, ctypes.POINTER(_ptr)], _i32),
    "admm_plan_exchange_info": ([_ptr, _i32, ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                                 ctypes.POINTER(_u64)], _i32),
    "admm_plan_attach": ([_ptr, _i32, _ptr], _i32),
    "admm_plan_run_phase": ([_ptr, _i32], _i32),
    "admm_plan_schedule": ([_ptr, ctypes.POINTER(_i32)], _i32),
    "admm_plan_set_g": ([_ptr, _ptr], _i32),
    "admm_plan_set_lambda": ([_ptr, _dbl], _i32),
    "admm_plan_set_lambdas": ([_ptr, _ptr], _i32),
    "admm_plan_max_abs_adjoint_batched": ([_ptr, _ptr], _i32),
    "admm_plan_max_abs_adjoint": ([_ptr, ctypes.POINTER(_dbl)], _i32),
    "admm_plan_solve": ([_ptr, _ptr, _ptr, ctypes.POINTER(_u64), ctypes.POINTER(_dbl), OBSERVER,
                         _ptr], _i32),
    "admm_plan_reset": ([_ptr], _i32),
    "admm_plan_enqueue": ([_ptr, _u64], _i32),
    "admm_plan_sync": ([_ptr], _i32),
    "admm_plan_stream": ([_ptr], _ptr),
    "admm_plan_set_stream": ([_ptr, _ptr], _i32),
    "admm_plan_kernel_count": ([_ptr], _u32),
    "admm_plan_profile": ([_ptr, _u64, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(_dbl)], _i32),
    "admm_plan_get_info": ([_ptr, ctypes.POINTER(PlanInfoC)], _i32),
    "admm_plan_read": ([_ptr, _i32, _ptr, _u64], _i32),
    "admm_plan_destroy": ([_ptr], None),
    "admm_matvec": ([_ptr, _u64, _u64, _ptr, _ptr, _i32], _i32),
    "admm_adjoint_matvec": ([_ptr, _u64, _u64, _ptr, _ptr, _i32], _i32),
    "admm_soft_threshold": ([_ptr, _u64, _dbl, _ptr, _i32], _i32),
    "admm_gram_solve": ([_ptr, _u64, _u64, _dbl, _ptr, _ptr, _i32], _i32),
    "admm_gram_create": ([_ptr, _u64, _u64, _dbl, _i32, _i32, ctypes.POINTER(_ptr)], _i32),
    "admm_gram_apply": ([_ptr, _ptr, _ptr], _i32),
    "admm_gram_info": ([_ptr, ctypes.POINTER(_i32), ctypes.POINTER(_u64)], _i32),
    "admm_gram_destroy": ([_ptr], None),
    "admm_gen_problem": ([_u64, _u64, _u64, _dbl, _u64, _i32, _ptr, _i32, _ptr, _ptr, _ptr], _i32),
    "admm_cmat_info": ([ctypes.c_char_p, ctypes.POINTER(_u64), ctypes.POINTER(_u64), ctypes.POINTER(_i32)], _i32),
    "admm_cmat_read": ([ctypes.c_char_p, _ptr, _u64, _i32], _i32),
    "admm_cmat_write": ([ctypes.c_char_p, _ptr, _u64, _u64, _i32, _i32], _i32),
    "admm_cmat_error_offset": ([], _u64),
    "admm_gen_cra": ([_u64, _u64, _u64, _dbl, _dbl, _dbl, _dbl, _dbl, _u64, _u64, _ptr, _i32], _i32),
}
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)
