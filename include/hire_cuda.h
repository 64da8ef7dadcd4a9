/*
 * hire_cuda.h — C ABI of libhire_cuda.so, the B200 (sm_100a) HiRE
 * approximate top-k path.
 *
 * The reference (/root/reference/proj/include/hire/*.hpp) is a header-only
 * C++20 library with no FFI; its operator API is the `hire::` functions.
 * Each entry point below replaces the hot-path body of one of them; the
 * C++ drop-in wrapper (include/hire_b200.hpp) keeps the `hire::` names and
 * calls these. Conventions:
 *   - plain pointers and sizes only; no C++ or torch types;
 *   - every function returns a status: 0 ok, 1 invalid argument (the
 *     reference's std::invalid_argument), 2 I/O, 3 numeric / CUDA failure;
 *     hire_last_error() gives the thread-local message;
 *   - matrices are row-major [rows][d] == the reference's column-major d x l
 *     ScoreMatrix (linalg.hpp:40-43): "column j" of the reference is row j;
 *   - *_run functions take DEVICE pointers and are asynchronous on the
 *     context's stream; *_host functions take HOST pointers and return after
 *     the results are on the host (copies included);
 *   - selection order everywhere is the reference's ranks_before
 *     (linalg.hpp:129-133): value descending, index ascending.
 */
#ifndef HIRE_CUDA_H_
#define HIRE_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HIRE_ABI_VERSION 1

#if defined(__GNUC__)
#define HIRE_API __attribute__((visibility("default")))
#else
#define HIRE_API
#endif

enum { HIRE_OK = 0, HIRE_ERR_INVALID = 1, HIRE_ERR_IO = 2, HIRE_ERR_RUNTIME = 3 };
enum { HIRE_F32 = 0, HIRE_BF16 = 1 };
/* linalg.hpp:20 Activation */
enum { HIRE_PHI_IDENTITY = 0, HIRE_PHI_RELU = 1, HIRE_PHI_SQUARED_RELU = 2 };
/* approx.hpp:307-312 ScorerKind numbering */
enum { HIRE_SCORER_LOWRANK = 1, HIRE_SCORER_Q4 = 2 };
/* int4 proxy activation mode: FP32 = the reference's scorer
 * (approx.hpp:395-403); INT8 = BASELINE's int4 x int8 -> int32 mode. */
enum { HIRE_X_FP32 = 0, HIRE_X_INT8 = 1 };
/* candidate rule: EXACT = topk_select (linalg.hpp:157-176);
 * BUCKETED = per-bucket top-t then top-k' of the survivors. */
enum { HIRE_SELECT_EXACT = 0, HIRE_SELECT_BUCKETED = 1 };
/* DA-TOP-k merge: PER_SHARD = distributed.hpp:94-131 (top-(k/s) per shard,
 * concatenated, globally sorted); GLOBAL = all k' exact pairs gathered, global
 * top-k. */
enum { HIRE_MERGE_PER_SHARD = 0, HIRE_MERGE_GLOBAL = 1 };

typedef struct hire_ctx_s* hire_ctx;
typedef struct hire_matrix_s* hire_matrix;
typedef struct hire_scorer_s* hire_scorer;
typedef struct hire_comm_s* hire_comm;

/* HireConfig (hire.hpp:16-20) plus the B200 path's knobs. */
typedef struct {
  int64_t k;          /* final count, 1 <= k <= k_prime */
  int64_t k_prime;    /* candidate count (clamped to rows, flagged) */
  int32_t phi;        /* HIRE_PHI_* */
  int32_t x_mode;     /* HIRE_X_* (int4 proxy only) */
  int32_t select;     /* HIRE_SELECT_* */
  int32_t strict;     /* 1: every fp reduction in the reference's sequential
                         order, no FMA contraction — bit-identical to the
                         reference; 0: fast tree reductions (tolerance) */
  int64_t n_buckets;  /* 0 = auto (EXACT); required for BUCKETED */
  int64_t bucket_t;   /* survivors per bucket; 0 = auto (EXACT) / 1 (BUCKETED) */
} hire_topk_params;

/* GroupedFFN (ffn.hpp:19-28) + select_groups quotas (ffn.hpp:175-201). */
typedef struct {
  int64_t k;           /* final units, g | k */
  int64_t k_prime;     /* candidate units, g | k_prime, k <= k_prime <= m */
  int64_t group_size;  /* g */
  int32_t phi;
  int32_t x_mode;
  int32_t strict;
  int32_t reserved;
} hire_ffn_params;

HIRE_API const char* hire_last_error(void);
HIRE_API int hire_abi_version(void);
/* 1 when the library was built with -DHIRE_EXPERIMENTS=1: the measured
 * negative-result kernels (single-launch FFN layer, bulk-copy recompute
 * ring, cluster / shared-memory selectors, post-proxy single launch) are
 * then selectable through their environment switches; 0 in the product. */
HIRE_API int hire_experiments_built(void);

/* ---- context: device, stream, workspace -------------------------------- */
/* own_stream = 1: the context creates (and owns) a non-blocking stream and
 * ignores cuda_stream; otherwise kernels go to cuda_stream (NULL = the
 * legacy default stream).
 * Threading: a context serves one call at a time (its workspaces, host-call
 * graphs and input slot belong to that call). Matrix and scorer handles are
 * read-only after construction and may be shared by any number of contexts.
 * For several calls in flight give each host thread its own context; the
 * *_host calls bind the context's device on a thread's first call
 * (tests/test_gpu_host_calls.py: two threads, two contexts, shared handles). */
HIRE_API int hire_ctx_create(int device, void* cuda_stream, int own_stream, hire_ctx* out);
HIRE_API int hire_ctx_destroy(hire_ctx ctx);
HIRE_API int hire_ctx_stream(hire_ctx ctx, void** cuda_stream);
HIRE_API int hire_ctx_synchronize(hire_ctx ctx);
/* number of kernels this context launched so far (bench accounting) */
HIRE_API int64_t hire_ctx_launch_count(hire_ctx ctx);
/* Stage profiling: when on, every stage of every run is bracketed by CUDA
 * events on the context stream. profile_read synchronises, returns the
 * summed milliseconds and the number of timed intervals per stage
 * (0 proxy scores, 1 candidate select, 2 gather recompute, 3 final top-k,
 * 4 FFN down-projection, 5 NCCL collective, 6 int8 x quantisation,
 * 7 the fused single-launch HiRE-FFN layer), and clears the record. */
HIRE_API int hire_ctx_set_profiling(hire_ctx ctx, int on);
/* Phase timestamps (%globaltimer, ns) of the last fused-kernel launch, when the
 * context was created with HIRE_FUSED_TRACE=1 in the environment. */
HIRE_API int hire_ctx_read_trace(hire_ctx ctx, long long* out, int n);
/* Debug: per-kernel %globaltimer window (min CTA start, max CTA end) for the
 * kernels launched while enabled. op 1 enable+reset, 2 read n words
 * (pairs per kernel id, see common.cuh KtId), 0 disable. */
HIRE_API int hire_debug_ktrace(hire_ctx ctx, int op, unsigned long long* out, int n);
HIRE_API int hire_ctx_profile_read(hire_ctx ctx, double* ms, int64_t* counts, int n_stages);
/* Queries whose exact top-k' selection took the slow whole-row path since the
 * context was created (a sampled bound missed, a list segment overflowed, a
 * sorted or constant score row): results are exact either way, this counts
 * the time cliff. Synchronises the context stream. */
HIRE_API int hire_ctx_select_fallbacks(hire_ctx ctx, long long* count);

/* ---- device buffers (for wrappers that start from host data) ------------ */
HIRE_API int hire_device_alloc(int64_t bytes, void** out);
HIRE_API int hire_device_free(void* p);
/* kind: 0 host->device, 1 device->host, 2 device->device; ordered on the
 * context stream; returns after the copy completes when sync != 0 */
HIRE_API int hire_copy(hire_ctx ctx, void* dst, const void* src, int64_t bytes, int kind, int sync);

/* ---- dense matrices (ScoreMatrix, linalg.hpp:44-90) --------------------- */
/* Copies src (host or device) into an owned device buffer; dtype HIRE_F32 or
 * HIRE_BF16 (the device storage type; src has the same type). */
HIRE_API int hire_matrix_create(const void* src, int64_t rows, int64_t d, int dtype,
                       int src_on_device, hire_matrix* out);
/* Non-owning view of an existing device buffer. */
HIRE_API int hire_matrix_view(void* device_ptr, int64_t rows, int64_t d, int dtype, hire_matrix* out);
/* Rows [first, first+count) as a view (ScoreMatrix::slice_cols, linalg.hpp:78-84). */
HIRE_API int hire_matrix_slice(hire_matrix m, int64_t first, int64_t count, hire_matrix* out);
HIRE_API int hire_matrix_destroy(hire_matrix m);
HIRE_API int hire_matrix_info(hire_matrix m, int64_t* rows, int64_t* d, int* dtype);

/* ---- proxies (ApproxScorer, approx.hpp:327-541) ------------------------- */
/* int4 from one code per byte (QuantizedMatrix::codes, approx.hpp:28-37). */
HIRE_API int hire_scorer_create_q4_codes(const int8_t* codes_host, const float* scales_host,
                                int64_t rows, int64_t d, hire_scorer* out);
/* int4 from a HIRQ payload (approx.hpp:551-564: continuous, low nibble first). */
HIRE_API int hire_scorer_create_q4_hirq(const uint8_t* payload_host, const float* scales_host,
                               int64_t rows, int64_t d, hire_scorer* out);
/* int4 built on the device from a dense matrix (quantize_int4, approx.hpp:49-65). */
HIRE_API int hire_scorer_quantize(hire_ctx ctx, hire_matrix w, hire_scorer* out);
/* low-rank: z1 [r][d] (reference z1 columns), z2 [rows][r]; dtype of both. */
HIRE_API int hire_scorer_create_lowrank(const void* z1, const void* z2, int64_t d, int64_t rows,
                               int64_t r, int dtype, int src_on_device, hire_scorer* out);
/* rows [first, first+count) (ApproxScorer::slice_cols, approx.hpp:415-445). */
HIRE_API int hire_scorer_slice(hire_scorer a, int64_t first, int64_t count, hire_scorer* out);
HIRE_API int hire_scorer_export_q4(hire_scorer a, int8_t* codes_host, float* scales_host);
HIRE_API int hire_scorer_info(hire_scorer a, int* kind, int64_t* rows, int64_t* d, int64_t* rank);
HIRE_API int hire_scorer_destroy(hire_scorer a);

/* ---- primitives ---------------------------------------------------------- */
/* ApproxScorer::scores for B queries: out [B][rows] (phi applied). */
HIRE_API int hire_scores(hire_ctx ctx, hire_scorer a, const float* x, int64_t B, int phi,
                int x_mode, int strict, float* out);
/* matvec (linalg.hpp:148-154) for B queries: out [B][rows]. */
HIRE_API int hire_matvec(hire_ctx ctx, hire_matrix w, const float* x, int64_t B, int phi, int strict,
                float* out);
/* topk_select (linalg.hpp:157-176) of B score vectors v [B][n]:
 * idx/val [B][min(k,n)] in rank order; *clamped = k > n. */
HIRE_API int hire_topk_select(hire_ctx ctx, const float* v, int64_t B, int64_t n, int64_t k,
                     uint32_t* idx, float* val, int* clamped);

/* ---- hire_topk / softmax_topk (hire.hpp:50-86, :123-144) ---------------- */
/* Output rows have fixed strides: cand [B][k_prime] (first n_cand valid,
 * ascending — the CandidateSet), top_idx/top_val/top_prob [B][k] (first
 * n_top valid, rank order). top_prob (nullable; phi must be identity) is the
 * renormalised top-k softmax. cand may be NULL. */
HIRE_API int hire_topk_run(hire_ctx ctx, hire_matrix w, hire_scorer a, const float* x, int64_t B,
                  const hire_topk_params* p, uint32_t* cand, uint32_t* top_idx,
                  float* top_val, float* top_prob, int64_t* n_cand, int64_t* n_top,
                  int* clamped);
HIRE_API int hire_topk_host(hire_ctx ctx, hire_matrix w, hire_scorer a, const float* x_host,
                   int64_t B, const hire_topk_params* p, uint32_t* cand_host,
                   uint32_t* top_idx_host, float* top_val_host, float* top_prob_host,
                   int64_t* n_cand, int64_t* n_top, int* clamped);

/* ---- HiRE-FFN: ffn_group_sparse (ffn.hpp:211-219) ----------------------- */
/* sel [B][k/g] selected group ids ascending; out [B][d]. */
HIRE_API int hire_ffn_run(hire_ctx ctx, hire_matrix u, hire_matrix v, hire_scorer a, const float* x,
                 int64_t B, const hire_ffn_params* p, uint32_t* sel, float* out);
HIRE_API int hire_ffn_host(hire_ctx ctx, hire_matrix u, hire_matrix v, hire_scorer a,
                  const float* x_host, int64_t B, const hire_ffn_params* p,
                  uint32_t* sel_host, float* out_host);
/* dense FFN (ffn.hpp:65-76), the baseline */
HIRE_API int hire_ffn_dense_run(hire_ctx ctx, hire_matrix u, hire_matrix v, const float* x, int64_t B,
                       int phi, int strict, float* out);
/* union_group_select (ffn.hpp:237-253): the sorted union of the B per-sample
 * select_groups results. ids: device, capacity m / g; *n_ids = |union|
 * (host, the call synchronises). */
HIRE_API int hire_ffn_union_select(hire_ctx ctx, hire_matrix u, hire_scorer a, const float* x, int64_t B,
                                   const hire_ffn_params* p, uint32_t* ids, int64_t* n_ids);
/* ffn_common_path (ffn.hpp:223-234): ffn_dense over the dense part (du, dv;
 * both NULL or 0 rows = none) plus ffn_group_sparse over the sparse part. */
HIRE_API int hire_ffn_common_path_run(hire_ctx ctx, hire_matrix du, hire_matrix dv, hire_matrix u, hire_matrix v,
                                      hire_scorer a, const float* x, int64_t B, const hire_ffn_params* p,
                                      float* out);

/* ---- DA-TOP-k (distributed.hpp:73-206) ----------------------------------- */
HIRE_API int hire_comm_unique_id(uint8_t id[128]);
HIRE_API int hire_comm_create(const uint8_t id[128], int world, int rank, hire_comm* out);
HIRE_API int hire_comm_destroy(hire_comm c);

/* One rank's share: w_shard / a_shard are rows [first, first+width) of the
 * full matrix under the shard width rule (distributed.hpp:53-57); total_rows
 * is l. uneven = 1 allows quotas that s does not divide (first k % s shards
 * take one more). Every rank gets the merged top_idx/top_val [B][k] (row
 * stride k, first n_top valid).
 * hire_da_topk_run = hire_da_topk_local -> one ncclAllGather of the B x slots
 * rank keys -> hire_da_topk_merge. comm NULL (world must be 1) runs
 * hire_topk directly (the reference's s = 1 equivalence); a 1-rank
 * communicator runs the full local -> all-gather -> merge chain. */
HIRE_API int hire_da_topk_run(hire_ctx ctx, hire_comm comm, hire_matrix w_shard, hire_scorer a_shard,
                     int64_t total_rows, int world, int rank, const float* x, int64_t B,
                     const hire_topk_params* p, int merge, int uneven, uint32_t* top_idx,
                     float* top_val, int64_t* n_top, int* clamped);
/* The two halves of hire_da_topk_run, for callers that move the keys
 * themselves (another transport, or tests driving the exchange):
 * local writes this rank's keys (8-byte rank keys of (exact value, global
 * index), distributed.hpp:94-125; padding slots 0) into send [B][slots];
 * merge takes the gathered [world][B][slots] keys (rank-major) and writes
 * the merged top-k (distributed.hpp:127-131 for PER_SHARD; the global
 * exact top-k for GLOBAL). slots = ceil(k/world) (PER_SHARD) or
 * ceil(k_prime/world) (GLOBAL). */
HIRE_API int hire_da_topk_slots(const hire_topk_params* p, int world, int merge, int64_t* slots);
HIRE_API int hire_da_topk_local(hire_ctx ctx, hire_matrix w_shard, hire_scorer a_shard, int64_t total_rows,
                                int world, int rank, const float* x, int64_t B, const hire_topk_params* p,
                                int merge, int uneven, uint64_t* send);
HIRE_API int hire_da_topk_merge(hire_ctx ctx, const uint64_t* gathered, int64_t total_rows, int world,
                                int64_t B, const hire_topk_params* p, int merge, int uneven,
                                uint32_t* top_idx, float* top_val, int64_t* n_top, int* clamped);
/* All `world` shards on this one device, no collective (the per-shard local
 * stages write straight into the gathered buffer): the single-GPU
 * emulation of hire_da_topk_run used for parity at D > 1. */
HIRE_API int hire_da_topk_emulated(hire_ctx ctx, hire_matrix w, hire_scorer a, int world,
                          const float* x, int64_t B, const hire_topk_params* p, int merge,
                          int uneven, uint32_t* top_idx, float* top_val, int64_t* n_top,
                          int* clamped);
/* da_group_sparse: local select with local quotas, local partial
 * down-projection; one grouped NCCL all-gather of the selected group ids and
 * the partial outputs; out [B][d] = the partials summed in rank order (the
 * same bits on every rank and topology); sel gets the union [B][k/g] of
 * selected groups (ascending). comm NULL: world must be 1. */
HIRE_API int hire_da_ffn_run(hire_ctx ctx, hire_comm comm, hire_matrix u_shard, hire_matrix v_shard,
                    hire_scorer a_shard, int64_t total_units, int world, int rank,
                    const float* x, int64_t B, const hire_ffn_params* p, int uneven,
                    uint32_t* sel, float* out);
/* The halves of hire_da_ffn_run: local writes this rank's selected group
 * ids (global, ascending) into sel_send [B][slots] and its partial output
 * into partial [B][d]; merge takes the gathered ids [world][B][slots] and
 * partials [world][B][d] and writes sel [B][k/g] and out [B][d].
 * slots = ceil((k/g)/world). */
HIRE_API int hire_da_ffn_slots(const hire_ffn_params* p, int world, int64_t* slots);
HIRE_API int hire_da_ffn_local(hire_ctx ctx, hire_matrix u_shard, hire_matrix v_shard, hire_scorer a_shard,
                               int64_t total_units, int world, int rank, const float* x, int64_t B,
                               const hire_ffn_params* p, int uneven, uint32_t* sel_send, float* partial);
HIRE_API int hire_da_ffn_merge(hire_ctx ctx, const uint32_t* gathered_sel, const float* gathered_parts,
                               int64_t total_units, int64_t d, int world, int64_t B, const hire_ffn_params* p,
                               int uneven, uint32_t* sel, float* out);
/* Single-GPU emulation of hire_da_ffn_run over `world` shards (strict: the
 * reference's one ascending sum over the union; else the rank-order sum
 * hire_da_ffn_run computes). */
HIRE_API int hire_da_ffn_emulated(hire_ctx ctx, hire_matrix u, hire_matrix v, hire_scorer a, int world,
                         const float* x, int64_t B, const hire_ffn_params* p, int uneven,
                         uint32_t* sel, float* out);

/* ---- seeded instances (host; rng.hpp:20-67, instance.hpp:16-83) --------- */
/* The reference's Rng stream, derive_seed, gen_vector and gen_instance with
 * the same arithmetic (bit-identical inputs for the experiment runner).
 * gen_instance writes [l][d] row-major (= the reference's d x l column-
 * major ScoreMatrix); spectrum 0 flat (iid Gaussian), 1 decaying (1/i). */
HIRE_API uint64_t hire_derive_seed(uint64_t seed, uint64_t stream);
HIRE_API int hire_gen_vector(uint64_t seed, int64_t n, float* out);
HIRE_API int hire_gen_instance(int64_t d, int64_t l, uint64_t seed, int spectrum, float* out);

/* ---- gather microbenchmark (gather_bench.hpp:18-152 on the GPU) --------- */
/* GatherBenchConfig (gather_bench.hpp:18-25): n_groups groups of g vectors
 * of dimension d; a seeded random fraction of the groups is gathered. */
typedef struct {
  int64_t n_groups;
  int64_t g;
  int64_t d;
  double fraction_selected; /* (0, 1] */
  int64_t repeats;          /* >= 3 */
  uint64_t seed;
} hire_gather_bench_config;
/* GatherBenchResult (gather_bench.hpp:38-46). */
typedef struct {
  double sparse_ns;         /* median over repeats, CUDA events */
  double dense_ns;
  double efficiency_paper;  /* sparse / dense */
  double efficiency_ratio;  /* dense / sparse */
  int64_t bytes_moved;
  int64_t groups_selected;
  int32_t checksum_ok;
  int32_t reserved;
} hire_gather_bench_result;
/* run_gather_bench (gather_bench.hpp:71-150): the selection is the
 * reference's seeded partial Fisher-Yates (its Rng stream, rng.hpp:20-61, at
 * the same counter position), kept in draw order; the sparse gather (one
 * warp per group, 128-bit loads) and a dense copy of the same bytes are timed
 * on the context stream; the gathered groups are checked against the source
 * with the reference's FNV-1a checksum. The buffers are device memory
 * (the reference times host memcpy). */
HIRE_API int hire_gather_bench(hire_ctx ctx, const hire_gather_bench_config* cfg, hire_gather_bench_result* out);

#ifdef __cplusplus
}
#endif
#endif /* HIRE_CUDA_H_ */
