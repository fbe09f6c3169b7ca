"""ctypes binding of libdho2gpu.so (include/dho2gpu.h).

The shared library is the product: every numeric call below runs hand-written sm_100a CUDA.
There is no CPU fallback — a missing or unloadable library raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DHO2G_LIB") or os.path.join(_HERE, "libdho2gpu.so")  # override: A/B experiments

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` at the repo root (or __graft_entry__.build()). "
        "The DHO2 B200 path has no CPU fallback.")

lib = C.CDLL(LIB_PATH)

dp = C.POINTER(C.c_double)
up = C.POINTER(C.c_uint64)
sp = C.POINTER(C.c_size_t)
ip = C.POINTER(C.c_int)
i64p = C.POINTER(C.c_int64)
vp = C.c_void_p


class LanczosOpts(C.Structure):
    _fields_ = [("reorth_safeguard", C.c_int), ("safeguard_ratio", C.c_double), ("breakdown_rtol", C.c_double)]


class BaseCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("lr", C.c_double), ("weight_decay", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("momentum", C.c_double)]


class TrainCfg(C.Structure):
    _fields_ = [("trainer", C.c_int), ("base", BaseCfg), ("k", C.c_size_t), ("l", C.c_size_t),
                ("alpha", C.c_double), ("eigval_floor", C.c_double), ("refresh_interval", C.c_size_t),
                ("curvature_batch", C.c_size_t), ("reorth_safeguard", C.c_int), ("safeguard_ratio", C.c_double),
                ("breakdown_rtol", C.c_double), ("sigma", C.c_double), ("outer_rounds", C.c_size_t),
                ("inner_epochs", C.c_size_t), ("sigma_zero_reduction", C.c_int), ("epochs", C.c_size_t),
                ("batch_size", C.c_size_t), ("seed", C.c_uint64), ("lanczos_m", C.c_size_t),
                ("model_bandwidth_gbps", C.c_double), ("model_gflops", C.c_double), ("debug_hash_checks", C.c_int)]


HOST_HVP = C.CFUNCTYPE(None, vp, dp, dp, C.c_size_t)
HOST_ALLGATHER = C.CFUNCTYPE(C.c_int, vp, vp, vp, C.c_size_t)  # dho2g_host_allgather

_SIGS = {
    "dho2g_last_error": ([], C.c_char_p),
    "dho2g_ctx_create": ([C.c_int, C.POINTER(vp)], C.c_int),
    "dho2g_ctx_destroy": ([vp], C.c_int),
    "dho2g_ctx_set_option": ([vp, C.c_char_p, C.c_double], C.c_int),
    "dho2g_ctx_get_stat": ([vp, C.c_char_p, dp], C.c_int),
    "dho2g_synchronize": ([vp], C.c_int),
    "dho2g_timer_mark": ([vp, C.c_int], C.c_int),
    "dho2g_timer_ms": ([vp, C.c_int, C.c_int, dp], C.c_int),
    "dho2g_ctx_kernel_name": ([vp, C.c_int, C.c_char_p, C.c_size_t], C.c_int),
    "dho2g_nccl_unique_id": ([vp], C.c_int),
    "dho2g_comm_init": ([vp, vp, C.c_int, C.c_int], C.c_int),
    "dho2g_comm_rank": ([vp, ip, ip], C.c_int),
    "dho2g_local_fabric_create": ([C.c_int, C.POINTER(vp)], C.c_int),
    "dho2g_local_fabric_destroy": ([vp], C.c_int),
    "dho2g_comm_init_local": ([vp, vp, C.c_int], C.c_int),
    "dho2g_comm_init_host": ([vp, C.c_int, C.c_int, HOST_ALLGATHER, vp], C.c_int),
    "dho2g_ctx_ledger_rows": ([vp], C.c_size_t),
    "dho2g_ctx_ledger_row": ([vp, C.c_size_t, i64p, C.c_char_p, C.c_size_t, i64p, ip, i64p, i64p], C.c_int),
    "dho2g_ctx_memory_count": ([vp], C.c_size_t),
    "dho2g_ctx_memory_entry": ([vp, C.c_size_t, C.c_char_p, C.c_size_t, i64p], C.c_int),
    "dho2g_ctx_accounting_reset": ([vp], C.c_int),
    "dho2g_ctx_allgather_host": ([vp, dp, C.c_size_t, dp], C.c_int),
    "dho2g_test_collectives": ([vp, dp], C.c_int),
    "dho2g_test_collectives_graph": ([vp, dp], C.c_int),
    "dho2g_test_gemm_trace": ([vp, C.c_int, C.POINTER(C.c_uint64), C.c_size_t], C.c_int),
    "dho2g_rng_u64": ([C.c_uint64, C.c_size_t, up], None),
    "dho2g_rng_normal": ([C.c_uint64, C.c_size_t, dp], None),
    "dho2g_shuffle_iota": ([C.c_uint64, C.c_size_t, up], None),
    "dho2g_mix_seed": ([C.c_uint64, C.c_uint64], C.c_uint64),
    "dho2g_shard": ([C.c_size_t, C.c_int, C.c_int, sp, sp], C.c_int),
    "dho2g_lanczos_budget": ([C.c_size_t, C.c_size_t, C.c_size_t, sp], C.c_int),
    "dho2g_epoch_permutation": ([C.c_size_t, C.c_uint64, C.c_uint64, up], None),
    "dho2g_init_params": ([C.POINTER(C.c_size_t), C.c_int, C.c_uint64, dp, C.POINTER(C.c_size_t)], C.c_int),
    "dho2g_synthetic_dataset": ([C.c_char_p, C.c_size_t, C.c_uint64, dp, dp, C.POINTER(C.c_size_t),
                                 C.POINTER(C.c_size_t)], C.c_int),
    "dho2g_curvature_indices": ([C.c_size_t, C.c_size_t, C.c_uint64, C.c_uint64, up], None),
    "dho2g_batch_indices": ([up, C.c_size_t, C.c_int, C.c_int, C.c_size_t, C.c_size_t, up], C.c_int),
    "dho2g_blobs_dataset": ([C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, dp, dp], None),
    "dho2g_mlp_create": ([vp, sp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)], C.c_int),
    "dho2g_mlp_destroy": ([vp], C.c_int),
    "dho2g_mlp_dim": ([vp], C.c_size_t),
    "dho2g_mlp_init_params": ([vp, C.c_uint64, dp], C.c_int),
    "dho2g_mlp_value": ([vp, dp, dp, dp, C.c_size_t, C.c_size_t, dp], C.c_int),
    "dho2g_mlp_grad": ([vp, dp, dp, dp, C.c_size_t, C.c_size_t, dp], C.c_int),
    "dho2g_mlp_hvp": ([vp, dp, dp, dp, dp, C.c_size_t, C.c_size_t, dp], C.c_int),
    "dho2g_mlp_accuracy": ([vp, dp, dp, dp, C.c_size_t, C.c_size_t, dp], C.c_int),
    "dho2g_op_mlp": ([vp, vp, dp, dp, dp, C.c_size_t, C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_op_diag": ([vp, dp, C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_op_dense": ([vp, dp, C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_op_quadratic": ([vp, dp, C.c_size_t, C.c_uint64, C.POINTER(vp)], C.c_int),
    "dho2g_op_apply": ([vp, dp, dp, dp], C.c_int),
    "dho2g_op_host": ([vp, HOST_HVP, vp, C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_op_destroy": ([vp], C.c_int),
    "dho2g_lanczos_run": ([vp, vp, C.c_size_t, C.c_uint64, C.POINTER(LanczosOpts), C.POINTER(vp)], C.c_int),
    "dho2g_lanczos_result": ([vp, dp, dp, sp, ip, sp, sp, sp], C.c_int),
    "dho2g_lanczos_basis": ([vp, dp], C.c_int),
    "dho2g_lanczos_destroy": ([vp], C.c_int),
    "dho2g_extract_ese": ([vp, vp, C.c_size_t, C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_ese_count": ([vp], C.c_size_t),
    "dho2g_ese_eigvals": ([vp, dp], C.c_int),
    "dho2g_ese_eigvecs": ([vp, dp], C.c_int),
    "dho2g_ese_gather": ([vp, dp], C.c_int),
    "dho2g_ese_eigvecs_device": ([vp, vp, C.c_size_t], C.c_int),
    "dho2g_ese_from_host": ([vp, dp, dp, C.c_size_t, C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_ese_from_device": ([vp, dp, vp, C.c_size_t, C.c_size_t, C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_ese_destroy": ([vp], C.c_int),
    "dho2g_opt_create": ([vp, C.POINTER(BaseCfg), C.c_size_t, C.POINTER(vp)], C.c_int),
    "dho2g_opt_destroy": ([vp], C.c_int),
    "dho2g_opt_step": ([vp, dp, dp, dp], C.c_int),
    "dho2g_deltas": ([vp, vp, dp, dp, dp, C.c_double, C.c_double, C.c_double, dp, dp], C.c_int),
    "dho2g_admm_w_update": ([vp, C.c_size_t, C.c_double, dp, dp, dp], C.c_int),
    "dho2g_admm_dual_update": ([vp, C.c_size_t, C.c_double, dp, dp, dp], C.c_int),
    "dho2g_trainer_create": ([vp, C.POINTER(TrainCfg), vp, dp, dp, C.c_size_t, C.c_size_t, C.c_uint64, dp, C.c_int,
                              C.c_int, C.POINTER(vp)], C.c_int),
    "dho2g_trainer_create_quadratic": ([vp, C.POINTER(TrainCfg), vp, C.c_size_t, dp, C.c_int, C.POINTER(vp)], C.c_int),
    "dho2g_trainer_destroy": ([vp], C.c_int),
    "dho2g_trainer_step": ([vp, C.c_size_t, C.c_int], C.c_int),
    "dho2g_trainer_run": ([vp], C.c_int),
    "dho2g_trainer_params": ([vp, dp], C.c_int),
    "dho2g_trainer_rows": ([vp], C.c_size_t),
    "dho2g_trainer_metrics": ([vp, C.c_size_t, dp, dp, dp, i64p, ip], C.c_int),
    "dho2g_trainer_metrics_ex": ([vp, C.c_size_t, i64p, i64p, dp], C.c_int),
    "dho2g_trainer_last_loss": ([vp, dp], C.c_int),
    "dho2g_trainer_stat": ([vp, C.c_char_p, dp], C.c_int),
    "dho2g_trainer_eigvals": ([vp, dp, sp], C.c_int),
    "dho2g_test_gemm": ([vp, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_float),
                         C.POINTER(C.c_float), C.c_int], C.c_int),
    "dho2g_test_gemm_seg": ([vp, C.c_int, C.c_int, C.c_int, C.c_int] + [C.POINTER(C.c_float)] * 5 +
                            [C.c_int, C.c_int, C.c_int], C.c_int),
}

for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)
