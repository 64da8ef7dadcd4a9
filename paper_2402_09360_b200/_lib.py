"""ctypes binding of libhire_cuda.so (include/hire_cuda.h).

The product path has no fallback: if the in-tree library is missing or a
call fails, this raises. Nothing here imports oracle/.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, os.environ.get("HIRE_LIB_VARIANT", "libhire_cuda.so"))  # variant: A/B experiments only

OK, ERR_INVALID, ERR_IO, ERR_RUNTIME = 0, 1, 2, 3
F32, BF16 = 0, 1
PHI = {"identity": 0, "relu": 1, "squared-relu": 2}
SCORER_LOWRANK, SCORER_Q4 = 1, 2
X_FP32, X_INT8 = 0, 1
SELECT_EXACT, SELECT_BUCKETED = 0, 1
MERGE_PER_SHARD, MERGE_GLOBAL = 0, 1
STAGES = ["proxy", "select", "recompute", "final", "down", "comm", "prep_x", "ffn_fused"]

# Every symbol include/hire_cuda.h declares (checked by tests/test_lib_symbols.py).
EXPORTS = [
    "hire_last_error", "hire_abi_version", "hire_experiments_built",
    "hire_ctx_create", "hire_ctx_destroy", "hire_ctx_stream", "hire_ctx_synchronize",
    "hire_ctx_launch_count", "hire_ctx_set_profiling", "hire_ctx_profile_read", "hire_ctx_read_trace", "hire_debug_ktrace",
    "hire_ctx_select_fallbacks",
    "hire_device_alloc", "hire_device_free", "hire_copy",
    "hire_matrix_create", "hire_matrix_view", "hire_matrix_slice", "hire_matrix_destroy",
    "hire_matrix_info",
    "hire_scorer_create_q4_codes", "hire_scorer_create_q4_hirq", "hire_scorer_quantize",
    "hire_scorer_create_lowrank", "hire_scorer_slice", "hire_scorer_export_q4",
    "hire_scorer_info", "hire_scorer_destroy",
    "hire_scores", "hire_matvec", "hire_topk_select",
    "hire_topk_run", "hire_topk_host",
    "hire_ffn_run", "hire_ffn_host", "hire_ffn_dense_run", "hire_ffn_union_select", "hire_ffn_common_path_run",
    "hire_comm_unique_id", "hire_comm_create", "hire_comm_destroy",
    "hire_da_topk_run", "hire_da_topk_emulated", "hire_da_ffn_run", "hire_da_ffn_emulated",
    "hire_da_topk_slots", "hire_da_topk_local", "hire_da_topk_merge",
    "hire_da_ffn_slots", "hire_da_ffn_local", "hire_da_ffn_merge",
    "hire_gather_bench", "hire_derive_seed", "hire_gen_vector", "hire_gen_instance",
]


class HireError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class HireInvalidArgument(HireError, ValueError):
    """The reference's std::invalid_argument."""


class TopkParams(C.Structure):
    _fields_ = [("k", C.c_int64), ("k_prime", C.c_int64), ("phi", C.c_int32),
                ("x_mode", C.c_int32), ("select", C.c_int32), ("strict", C.c_int32),
                ("n_buckets", C.c_int64), ("bucket_t", C.c_int64)]


class FfnParams(C.Structure):
    _fields_ = [("k", C.c_int64), ("k_prime", C.c_int64), ("group_size", C.c_int64),
                ("phi", C.c_int32), ("x_mode", C.c_int32), ("strict", C.c_int32),
                ("reserved", C.c_int32)]


class GatherBenchConfig(C.Structure):
    """hire_gather_bench_config (GatherBenchConfig, gather_bench.hpp:18-25)."""
    _fields_ = [("n_groups", C.c_int64), ("g", C.c_int64), ("d", C.c_int64), ("fraction_selected", C.c_double),
                ("repeats", C.c_int64), ("seed", C.c_uint64)]


class GatherBenchResult(C.Structure):
    """hire_gather_bench_result (GatherBenchResult, gather_bench.hpp:38-46)."""
    _fields_ = [("sparse_ns", C.c_double), ("dense_ns", C.c_double), ("efficiency_paper", C.c_double),
                ("efficiency_ratio", C.c_double), ("bytes_moved", C.c_int64), ("groups_selected", C.c_int64),
                ("checksum_ok", C.c_int32), ("reserved", C.c_int32)]


_vp, _i64, _i32, _p = C.c_void_p, C.c_int64, C.c_int, C.POINTER
_lib = None


def _sig(L):
    L.hire_last_error.restype = C.c_char_p
    L.hire_last_error.argtypes = []
    L.hire_abi_version.restype = _i32
    L.hire_experiments_built.restype = _i32
    L.hire_experiments_built.argtypes = []
    L.hire_derive_seed.restype = C.c_uint64
    L.hire_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
    L.hire_ctx_launch_count.restype = _i64
    L.hire_ctx_launch_count.argtypes = [_vp]
    sigs = {
        "hire_ctx_create": [_i32, _vp, _i32, _p(_vp)],
        "hire_ctx_destroy": [_vp],
        "hire_ctx_stream": [_vp, _p(_vp)],
        "hire_ctx_synchronize": [_vp],
        "hire_ctx_set_profiling": [_vp, _i32],
        "hire_ctx_read_trace": [_vp, _vp, _i32],
        "hire_ctx_select_fallbacks": [_vp, _vp],
        "hire_debug_ktrace": [_vp, _i32, _vp, _i32],
        "hire_ctx_profile_read": [_vp, _vp, _vp, _i32],
        "hire_device_alloc": [_i64, _p(_vp)],
        "hire_device_free": [_vp],
        "hire_copy": [_vp, _vp, _vp, _i64, _i32, _i32],
        "hire_matrix_create": [_vp, _i64, _i64, _i32, _i32, _p(_vp)],
        "hire_matrix_view": [_vp, _i64, _i64, _i32, _p(_vp)],
        "hire_matrix_slice": [_vp, _i64, _i64, _p(_vp)],
        "hire_matrix_destroy": [_vp],
        "hire_matrix_info": [_vp, _p(_i64), _p(_i64), _p(_i32)],
        "hire_scorer_create_q4_codes": [_vp, _vp, _i64, _i64, _p(_vp)],
        "hire_scorer_create_q4_hirq": [_vp, _vp, _i64, _i64, _p(_vp)],
        "hire_scorer_quantize": [_vp, _vp, _p(_vp)],
        "hire_scorer_create_lowrank": [_vp, _vp, _i64, _i64, _i64, _i32, _i32, _p(_vp)],
        "hire_scorer_slice": [_vp, _i64, _i64, _p(_vp)],
        "hire_scorer_export_q4": [_vp, _vp, _vp],
        "hire_scorer_info": [_vp, _p(_i32), _p(_i64), _p(_i64), _p(_i64)],
        "hire_scorer_destroy": [_vp],
        "hire_scores": [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _vp],
        "hire_matvec": [_vp, _vp, _vp, _i64, _i32, _i32, _vp],
        "hire_topk_select": [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _p(_i32)],
        "hire_topk_run": [_vp, _vp, _vp, _vp, _i64, _p(TopkParams), _vp, _vp, _vp, _vp,
                          _p(_i64), _p(_i64), _p(_i32)],
        "hire_topk_host": [_vp, _vp, _vp, _vp, _i64, _p(TopkParams), _vp, _vp, _vp, _vp,
                           _p(_i64), _p(_i64), _p(_i32)],
        "hire_ffn_run": [_vp, _vp, _vp, _vp, _vp, _i64, _p(FfnParams), _vp, _vp],
        "hire_ffn_host": [_vp, _vp, _vp, _vp, _vp, _i64, _p(FfnParams), _vp, _vp],
        "hire_ffn_dense_run": [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp],
        "hire_ffn_union_select": [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _p(_i64)],
        "hire_ffn_common_path_run": [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp],
        "hire_comm_unique_id": [_vp],
        "hire_comm_create": [_vp, _i32, _i32, _p(_vp)],
        "hire_comm_destroy": [_vp],
        "hire_da_topk_run": [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _i64, _p(TopkParams),
                             _i32, _i32, _vp, _vp, _p(_i64), _p(_i32)],
        "hire_da_topk_emulated": [_vp, _vp, _vp, _i32, _vp, _i64, _p(TopkParams), _i32, _i32,
                                  _vp, _vp, _p(_i64), _p(_i32)],
        "hire_da_ffn_run": [_vp, _vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _i64, _p(FfnParams),
                            _i32, _vp, _vp],
        "hire_da_ffn_emulated": [_vp, _vp, _vp, _vp, _i32, _vp, _i64, _p(FfnParams), _i32,
                                 _vp, _vp],
        "hire_da_topk_slots": [_p(TopkParams), _i32, _i32, _p(_i64)],
        "hire_da_topk_local": [_vp, _vp, _vp, _i64, _i32, _i32, _vp, _i64, _p(TopkParams), _i32, _i32, _vp],
        "hire_da_topk_merge": [_vp, _vp, _i64, _i32, _i64, _p(TopkParams), _i32, _i32, _vp, _vp, _p(_i64),
                               _p(_i32)],
        "hire_da_ffn_slots": [_p(FfnParams), _i32, _p(_i64)],
        "hire_da_ffn_local": [_vp, _vp, _vp, _vp, _i64, _i32, _i32, _vp, _i64, _p(FfnParams), _i32, _vp, _vp],
        "hire_da_ffn_merge": [_vp, _vp, _vp, _i64, _i64, _i32, _i64, _p(FfnParams), _i32, _vp, _vp],
        "hire_gather_bench": [_vp, _p(GatherBenchConfig), _p(GatherBenchResult)],
        "hire_gen_vector": [C.c_uint64, _i64, _vp],
        "hire_gen_instance": [_i64, _i64, C.c_uint64, _i32, _vp],
    }
    for name, args in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = _i32


def lib():
    """Load the in-tree library (building it if the sources are newer)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from . import build as _b
            _b.build()
        _lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        _sig(_lib)
        if _lib.hire_abi_version() != 1:
            raise HireError(ERR_RUNTIME, "libhire_cuda.so ABI version mismatch")
    return _lib


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().hire_last_error().decode(errors="replace")
        if rc == ERR_INVALID:
            raise HireInvalidArgument(rc, msg)
        raise HireError(rc, msg)
