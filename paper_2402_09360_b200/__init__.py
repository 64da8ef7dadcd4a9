"""B200-native (sm_100a) HiRE approximate top-k path.

Drop-in for the hot path of the reference's `hire::` operator API
(/root/reference/proj/include/hire): compressed-proxy scoring, exact /
bucketed top-k' selection, row-gather exact recompute + top-k (+ softmax),
the sparse FFN down-projection, and DA-TOP-k over NCCL. All compute runs in
libhire_cuda.so (csrc/), reached through the C ABI in include/hire_cuda.h.
"""
from ._lib import (BF16, F32, MERGE_GLOBAL, MERGE_PER_SHARD, SELECT_BUCKETED, SELECT_EXACT,
                   X_FP32, X_INT8, HireError, HireInvalidArgument, lib)
from .api import (ApproxScorer, CommonPathFFN, Context, CostReport, GatherBenchConfig, GatherBenchResult, GroupedFFN,
                  HireConfig, HireResult, ScoreMatrix, run_gather_bench,
                  da_group_sparse_emulated, da_topk_emulated, default_context, exact_topk,
                  ffn_common_path, ffn_dense, ffn_group_sparse, hire_topk, matvec, overlap_ratio, param_bytes, recall,
                  roofline_bytes,
                  shard_range, softmax_topk, topk_select, union_group_select)

__all__ = [
    "ApproxScorer", "Context", "GroupedFFN", "HireConfig", "HireResult", "ScoreMatrix",
    "hire_topk", "softmax_topk", "topk_select", "exact_topk", "matvec", "ffn_group_sparse",
    "ffn_dense", "union_group_select", "CommonPathFFN", "ffn_common_path", "overlap_ratio", "da_topk_emulated", "da_group_sparse_emulated", "recall", "shard_range",
    "CostReport", "param_bytes", "roofline_bytes", "GatherBenchConfig", "GatherBenchResult", "run_gather_bench",
    "F32", "BF16", "X_FP32", "X_INT8", "SELECT_EXACT", "SELECT_BUCKETED", "MERGE_PER_SHARD",
    "MERGE_GLOBAL", "HireError", "HireInvalidArgument", "lib",
]
