// hire_cuda.cu — C ABI (include/hire_cuda.h) and host orchestration of the
// HiRE approximate top-k path on B200 (sm_100a).
//
// One call = a fixed chain of stream-ordered kernels, no host sync:
//   [prep_x] -> proxy scores (K1/K2) -> [bucket survivors] -> candidate
//   select (K3) -> gather + exact recompute (K4) -> final top-k / softmax (K5)
//   [-> FFN down-projection (K6)] [-> NCCL all-gather/all-reduce + merge (K7)]
// Reference orchestration replaced: hire_topk hire.hpp:50-86, softmax_topk
// hire.hpp:123-144, ffn_group_sparse ffn.hpp:211-219 (select_groups :175-201,
// ffn_apply_groups :154-171), da_topk distributed.hpp:73-134,
// da_group_sparse distributed.hpp:145-206.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/hire_cuda.h"
#include "common.cuh"
#include "exact.cuh"
#if HIRE_EXPERIMENTS
#include "ffn_fused.cuh"
#endif
#include "score.cuh"
#include "select.cuh"
#include "select2.cuh"
#include "fsel.cuh"
#include "score_umma.cuh"
#include "gather_bench.cuh"

using namespace hire_dev;

// ------------------------------------------------------------ plumbing --
namespace {
thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int invalid(const std::string& msg) { return set_err(HIRE_ERR_INVALID, msg); }

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return set_err(HIRE_ERR_RUNTIME, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define CKN(call)                                                                  \
  do {                                                                             \
    ncclResult_t r_ = (call);                                                      \
    if (r_ != ncclSuccess)                                                         \
      return set_err(HIRE_ERR_RUNTIME, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

#define RET(call)             \
  do {                        \
    int rc_ = (call);         \
    if (rc_ != HIRE_OK) return rc_; \
  } while (0)

constexpr size_t kAlign = 256;
size_t align_up(size_t v, size_t a = kAlign) { return (v + a - 1) / a * a; }
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace

struct hire_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int num_sms = 148;
  void* ws = nullptr;
  size_t ws_cap = 0;
  void* io_dev = nullptr;
  size_t io_dev_cap = 0;
  void* io_host = nullptr;
  size_t io_host_cap = 0;
  int64_t launches = 0;
  bool pdl = true;
  bool force_dp4a = false;
  bool ffn_fused = false;  // the kernel chain is faster since the grid-wide selector (HIRE_FFN_FUSED=1 opts in)
  bool trace = false;
  int* counters = nullptr;  // zeroed hand-off counters of the fused kernels
  unsigned* selc = nullptr;  // zeroed selection counters (select2.cuh qc / agg)
  unsigned* tickets = nullptr;  // [B] S3 chunk tickets, zero at rest (the last claimer resets)
  size_t tickets_cap = 0;
  size_t selc_cap = 0;
  void* fzero = nullptr;     // zero-at-rest sample slots + bounds of the fused selector (fsel.cuh)
  size_t fzero_cap = 0;
  unsigned long long* umask = nullptr;  // zero-at-rest row masks of the batch-union gather (exact.cuh K4U)
  size_t umask_cap = 0;                 // rows
  void* upart = nullptr;                // its per-slice partial sums [B][rows][slices]
  size_t upart_cap = 0;
  // host-buffer calls (*_host): after one eager call per shape, the whole
  // call — H2D copy, kernel chain, D2H copy — replays as one CUDA graph on
  // gstream. An entry is valid while every buffer it captured is unchanged.
  // The input-fetch kernel of a host call reads its source address from
  // fetch_slot (one word of mapped host memory the host stores before every
  // launch: the caller's own pinned buffer when it has a device alias, else
  // the context's staging buffer), so one captured graph serves every input
  // buffer and a replay never edits the executable graph. (Round 2e: the
  // earlier scheme re-pointed the fetch node with
  // cudaGraphExecKernelNodeSetParams per call; two contexts replaying their
  // graphs from two host threads then hit illegal-address faults — see
  // tools/probes/concurrent_host_calls.py.)
  unsigned long long* fetch_slot = nullptr;      // host view
  unsigned long long* fetch_slot_dev = nullptr;  // device alias
  bool fetch_by_slot = false;                    // set by fetch_inputs when it launched the slot kernel
  struct HostGraph {
    std::vector<int64_t> key;
    std::vector<const void*> bufs;
    cudaGraphExec_t exec = nullptr;
    int64_t out[4] = {0, 0, 0, 0};
    bool uses_slot = false;  // its fetch kernel reads the input address from fetch_slot
  };
  static constexpr size_t kMaxHostGraphs = 64;
  std::vector<HostGraph> hgraphs;  // least recently used first
  std::vector<std::vector<int64_t>> hseen;
  bool host_graphs = true;
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev = nullptr;
  std::vector<const void*> buf_snapshot() const { return {ws, io_dev, io_host, selc, fzero, counters, tickets, umask, upart}; }
  // stage profiling (hire_ctx_set_profiling): event pairs around each stage
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
  cudaEvent_t get_event() {
    if (ev_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = ev_pool.back();
    ev_pool.pop_back();
    return e;
  }
};

namespace {
// Stage ids for hire_ctx_profile_read.
enum Stage { kStageProxy = 0, kStageSelect = 1, kStageRecompute = 2, kStageFinal = 3, kStageDown = 4,
             kStageComm = 5, kStagePrep = 6, kStageFused = 7, kNumStages = 8 };

struct StageScope {
  hire_ctx c;
  int stage;
  cudaEvent_t e0 = nullptr;
  // Inside stream capture the records become external event nodes, so the
  // pairs time the replayed graph.
  static void record(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &st);
    if (st == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    else cudaEventRecord(e, s);
  }
  StageScope(hire_ctx ctx, int st) : c(ctx), stage(st) {
    if (c->prof) {
      e0 = c->get_event();
      record(e0, c->stream);
    }
  }
  ~StageScope() {
    if (c->prof) {
      cudaEvent_t e1 = c->get_event();
      record(e1, c->stream);
      c->marks.push_back({stage, {e0, e1}});
    }
  }
};
}  // namespace

namespace {
// Process-wide handle ids: host-call graphs are keyed on these, never on a
// handle's address (a freed handle's address can be reused by a new one).
std::atomic<uint64_t> g_next_uid{1};
uint64_t next_uid() { return g_next_uid.fetch_add(1, std::memory_order_relaxed); }
}  // namespace

struct hire_matrix_s {
  uint64_t uid = next_uid();
  void* ptr = nullptr;
  int64_t rows = 0, d = 0;
  int dtype = HIRE_F32;
  bool owned = false;
};

struct hire_scorer_s {
  uint64_t uid = next_uid();
  int kind = HIRE_SCORER_Q4;
  int64_t rows = 0, d = 0, r = 0;
  // int4
  uint8_t* codes = nullptr;
  int64_t pitch = 0;
  float* scales = nullptr;
  uint4* mma = nullptr;        // MMA-tiled copy for the tensor-core proxy (lazy)
  bool mma_owned = false;
  uint32_t* umma = nullptr;    // tcgen05 layout (128-row blocks) for B >= 9 (lazy)
  bool umma_owned = false;
  CUtensorMap umap;            // TMA descriptor of `umma` (built with it)
  bool umap_ok = false;
  // low-rank
  void* z1 = nullptr;
  void* z2 = nullptr;
  int dtype = HIRE_F32;
  bool owned = false;
};

struct hire_comm_s {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
};

namespace {

size_t dtype_size(int dt) { return dt == HIRE_BF16 ? 2 : 4; }

// Every launch goes through here: programmatic stream serialization (PDL)
// so each kernel's launch overlaps its predecessor's tail (kernels call
// griddepcontrol.wait before consuming). Counted for bench accounting.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(hire_ctx ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx->pdl ? 1 : 0;
  ++ctx->launches;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// launch_k with a thread-block cluster of cluster_x CTAs along x
template <typename... KArgs, typename... Args>
cudaError_t launch_k_cluster(hire_ctx ctx, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             unsigned cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster_x;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = ctx->pdl ? 2 : 1;
  ++ctx->launches;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

int ensure(void** buf, size_t* cap, size_t need, cudaStream_t s) {
  if (need <= *cap) return HIRE_OK;
  if (*buf) {
    CK(cudaStreamSynchronize(s));
    CK(cudaFree(*buf));
    *buf = nullptr;
  }
  size_t n = std::max(need, *cap * 2);
  CK(cudaMalloc(buf, n));
  *cap = n;
  return HIRE_OK;
}

int ensure_host(void** buf, size_t* cap, size_t need, cudaStream_t s) {
  if (need <= *cap) return HIRE_OK;
  if (*buf) {
    CK(cudaStreamSynchronize(s));
    CK(cudaFreeHost(*buf));
    *buf = nullptr;
  }
  size_t n = std::max(need, *cap * 2);
  // mapped: the kernels read the inputs and write the results straight
  // through PCIe (a copy-engine transfer costs ~10 us of setup latency)
  CK(cudaHostAlloc(buf, n, cudaHostAllocMapped | cudaHostAllocPortable));
  *cap = n;
  return HIRE_OK;
}

// Zero-at-rest counters for select2.cuh (the kernels restore the zeros).
int ensure_selc(hire_ctx ctx, size_t words) {
  if (words <= ctx->selc_cap) return HIRE_OK;
  if (ctx->selc) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaFree(ctx->selc));
    ctx->selc = nullptr;
  }
  const size_t n = std::max<size_t>(words, 4096);
  CK(cudaMalloc(&ctx->selc, n * sizeof(unsigned)));
  CK(cudaMemsetAsync(ctx->selc, 0, n * sizeof(unsigned), ctx->stream));
  ctx->selc_cap = n;
  return HIRE_OK;
}

// Zero-at-rest sample slots / bounds / list counts of the fused and list
// selectors (fsel.cuh): [B][kFselSampleMax] samples, lo[B], cnt[B], ctr.
// Per-query chunk tickets of the ordered emit (zero at rest; a separate
// buffer: the selc regions move with the call shape)
int ensure_tickets(hire_ctx ctx, int64_t B) {
  if (static_cast<size_t>(B) <= ctx->tickets_cap) return HIRE_OK;
  if (ctx->tickets) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaFree(ctx->tickets));
    ctx->tickets = nullptr;
  }
  const size_t n = std::max<size_t>(static_cast<size_t>(B), 256);
  CK(cudaMalloc(&ctx->tickets, n * sizeof(unsigned)));
  CK(cudaMemsetAsync(ctx->tickets, 0, n * sizeof(unsigned), ctx->stream));
  ctx->tickets_cap = n;
  return HIRE_OK;
}

int ensure_fzero(hire_ctx ctx, int64_t B) {
  const size_t need = static_cast<size_t>(B) * (hire_dev::kFselSampleMax + 2) * 8 + hire_dev::kFselCtr * 32 * 4 +
                      static_cast<size_t>(B) * 8;
  if (need <= ctx->fzero_cap) return HIRE_OK;
  if (ctx->fzero) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaFree(ctx->fzero));
    ctx->fzero = nullptr;
  }
  const size_t nb = std::max(need, ctx->fzero_cap * 2);
  CK(cudaMalloc(&ctx->fzero, nb));
  CK(cudaMemsetAsync(ctx->fzero, 0, nb, ctx->stream));
  ctx->fzero_cap = nb;
  return HIRE_OK;
}

int ensure_umask(hire_ctx ctx, int64_t rows) {
  if (static_cast<size_t>(rows) <= ctx->umask_cap) return HIRE_OK;
  if (ctx->umask) {
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaFree(ctx->umask));
    ctx->umask = nullptr;
  }
  const size_t n = std::max<size_t>(static_cast<size_t>(rows), 2 * ctx->umask_cap);
  CK(cudaMalloc(&ctx->umask, n * 8));
  CK(cudaMemsetAsync(ctx->umask, 0, n * 8, ctx->stream));
  ctx->umask_cap = n;
  return HIRE_OK;
}

void fzero_layout(hire_ctx ctx, int64_t B, hire_dev::FuseSel* fs) {
  fs->samp = static_cast<uint64_t*>(ctx->fzero);
  fs->lo = static_cast<unsigned long long*>(ctx->fzero) + static_cast<size_t>(B) * hire_dev::kFselSampleMax;
  fs->cnt = reinterpret_cast<unsigned*>(fs->lo + B);
  fs->ctr = reinterpret_cast<unsigned*>(fs->lo + 2 * B);
}

// Bump allocator over the context workspace. Offsets first, then one
// ensure(); pointers are only valid for the current call.
struct Arena {
  size_t off = 0;
  std::vector<std::pair<void**, size_t>> reqs;
  template <typename T>
  void take(T** p, size_t count) {
    reqs.push_back({reinterpret_cast<void**>(p), off});
    off += align_up(std::max<size_t>(count, 1) * sizeof(T));
  }
  int commit(hire_ctx ctx) {
    RET(ensure(&ctx->ws, &ctx->ws_cap, off, ctx->stream));
    for (auto& r : reqs) *r.first = static_cast<char*>(ctx->ws) + r.second;
    return HIRE_OK;
  }
};

template <typename K>
int max_blocks(K kernel, int threads, size_t smem) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, threads, smem) != cudaSuccess) n = 1;
  return std::max(n, 1);
}

// ----------------------------------------------------- selection policy --
// context counter buffer: fused-kernel barriers, per-query counters, trace
constexpr int kQcntOff = 8 * 16 * 32;  // the fused FFN kernel's barrier counters (ffn_fused.cuh kCntInts)
constexpr int kTraceOff = kQcntOff + 64;
constexpr int kFallbackOff = kTraceOff + 128;  // selection fallbacks since the context was created
constexpr int kCtxCounterInts = kFallbackOff + 16;

constexpr int64_t kSelGridChunks = 4 * 160;  // S2/S3 CTAs over a whole batch (workspace bound; 4 per SM used)

struct SelPlan {
  int mode = 0;          // 0 direct, 1 bucket, 2 grid-wide pivot/window/emit (select2.cuh)
  int n_buckets = 0, t = 0;
  int exact_fix = 1;
  int64_t k_eff = 0;     // candidates produced
  bool clamped = false;
  int64_t wcap = 0;      // mode 2: window capacity per chunk
  int64_t wseg = 0;      // mode 2: window segment (keys) per chunk
  // u64 workspace words for B queries ("surv" buffer); mode 2: pivots,
  // thresholds and one window segment per chunk (<= kSelGridChunks chunks
  // over the whole batch)
  int64_t surv_words(int64_t B) const {
    // piv, thr, 8 x 256-bin hists, 8 x 256 x 32 bin lists, chunk windows
    if (mode == 2) return 5 * B + B * 1024 + B * 65536 + wseg * kSelGridChunks;
    return B * std::max(n_buckets * t, 1);
  }
};

// Prime multiplier coprime with nblk for the S1 sample permutation.
uint32_t sample_perm(uint64_t nblk) {
  auto is_prime = [](uint64_t v) {
    if (v < 2) return false;
    for (uint64_t f = 2; f * f <= v; ++f)
      if (v % f == 0) return false;
    return true;
  };
  uint64_t p = std::max<uint64_t>(3, static_cast<uint64_t>(0.6180339887 * static_cast<double>(nblk)));
  while (!is_prime(p) || nblk % p == 0) ++p;
  const uint32_t r = static_cast<uint32_t>(p % std::max<uint64_t>(nblk, 1));
  return r ? r : 1u;
}

int plan_select(int64_t n, int64_t k_prime, int sel_mode, int64_t nb_req, int64_t t_req,
                SelPlan* sp) {
  if (k_prime < 1) return invalid("topk_select: k must be >= 1");
  if (n < 1) return invalid("selection over an empty score vector");
  if (n > 0xFFFFFFFELL) return invalid("selection: more than 2^32-2 scores");
  if (sel_mode == HIRE_SELECT_BUCKETED) {
    if (nb_req < 1 || nb_req > n) return invalid("bucketed select: n_buckets must be in [1, rows]");
    const int64_t t = t_req > 0 ? t_req : 1;
    if (ceil_div(n, nb_req) > kBucketMaxWidth)
      return invalid("bucketed select: bucket width exceeds " + std::to_string(kBucketMaxWidth));
    // valid survivors = sum_b min(t, width_b)
    const int64_t base = n / nb_req, extra = n % nb_req;
    const int64_t valid = extra * std::min(t, base + 1) + (nb_req - extra) * std::min(t, base);
    if (nb_req * t > kPoolKeys) return invalid("bucketed select: n_buckets * t exceeds the pool");
    sp->mode = 1;
    sp->n_buckets = static_cast<int>(nb_req);
    sp->t = static_cast<int>(t);
    sp->exact_fix = 0;
    sp->k_eff = std::min(k_prime, valid);
    sp->clamped = k_prime > valid;
    return HIRE_OK;
  }
  sp->k_eff = std::min(k_prime, n);
  sp->clamped = k_prime > n;
  if (nb_req == 0 && std::getenv("HIRE_SELECT_V1") == nullptr) {
    sp->mode = 2;
    if (n > kSel2Exact) {
      // window segment per chunk: the chunk width, capped (a chunk holding
      // more window keys than its segment falls back to the slow path)
      sp->wseg = std::min<int64_t>(n, 1024);
    }
    return HIRE_OK;
  }
  if (n <= kDirectMax && nb_req == 0) {
    sp->mode = 0;
    return HIRE_OK;
  }
  sp->mode = 1;
  sp->exact_fix = 1;
  int64_t width = 256;
  for (;;) {
    const int64_t nb = nb_req > 0 ? nb_req : std::max<int64_t>(1, ceil_div(n, width));
    const int64_t w = ceil_div(n, nb);
    const double mean = static_cast<double>(sp->k_eff) / static_cast<double>(nb);
    int64_t t = t_req > 0 ? t_req : static_cast<int64_t>(std::ceil(mean + 4.0 * std::sqrt(mean) + 2.0));
    t = std::min(t, w);
    if (w > kBucketMaxWidth) return invalid("selection: bucket width exceeds " + std::to_string(kBucketMaxWidth));
    if ((nb * t <= kPoolKeys / 2 && nb * t >= sp->k_eff) || nb_req > 0) {
      if (nb * t > kPoolKeys) return invalid("selection: n_buckets * t exceeds the pool");
      if (nb * t < sp->k_eff) return invalid("selection: n_buckets * t < k_prime");
      sp->n_buckets = static_cast<int>(nb);
      sp->t = static_cast<int>(t);
      return HIRE_OK;
    }
    width *= 2;
    if (width > kBucketMaxWidth) {
      // very large k': fall back to the global-memory exact path via a
      // single huge "overflow" (select kernel handles it)
      sp->n_buckets = static_cast<int>(std::max<int64_t>(1, ceil_div(n, kBucketMaxWidth)));
      sp->t = static_cast<int>(std::min<int64_t>(kBucketMaxWidth, kPoolKeys / 2 / sp->n_buckets));
      if (static_cast<int64_t>(sp->n_buckets) * sp->t < sp->k_eff)
        return invalid("selection: k_prime too large for the on-chip selector");
      return HIRE_OK;
    }
  }
}

// Stream path plan (sel_stream_kernel): C chunks per query, seg list slots per
// chunk, and the sample rank r_s of the query's bound. r_s is the smallest
// rank with P[Binomial(S, k'/n) >= r_s] <= 1e-7 (S = the sampler's sample
// size): the chance that the bound lies above the true k'-th key. C is the
// largest chunk count (up to one wave of CTAs) for which the modelled chance
// of an overflow (a CTA's 1024-key stage, or the query's 8192-key list) stays
// below 1e-6 per query; failing that the safest C if below 1e-4 (cfg4, k' =
// 2048 of 256000: 4e-6, the list is small for the bound's spread), else the
// pivot + list kernels. Either event only costs the finisher's slow path,
// never exactness.
struct StreamPlan {
  int C = 0, seg = 0;
  int64_t r_s = 0;
};

int64_t binom_tail_rank(int64_t S, double p, double eps) {
  // smallest r with P[X >= r] <= eps, X ~ Binomial(S, p)
  if (p <= 0.0) return 1;
  if (p >= 1.0) return S + 1;
  const double lp = std::log(p), lq = std::log1p(-p);
  auto logpmf = [&](int64_t x) {
    return std::lgamma(static_cast<double>(S) + 1.0) - std::lgamma(static_cast<double>(x) + 1.0) -
           std::lgamma(static_cast<double>(S - x) + 1.0) + static_cast<double>(x) * lp + static_cast<double>(S - x) * lq;
  };
  double tail = 0.0;
  int64_t r = S + 1;
  for (int64_t x = S; x >= 0; --x) {
    tail += std::exp(logpmf(x));
    if (tail > eps) break;
    r = x;
  }
  return r;
}

// P[X >= r], X ~ Binomial(n, p) (pmf recurrence from x = r).
double binom_sf_ge(int n, double p, int r) {
  if (r <= 0) return 1.0;
  if (r > n || p <= 0.0) return 0.0;
  if (p >= 1.0) return 1.0;
  double pmf = std::exp(std::lgamma(n + 1.0) - std::lgamma(r + 1.0) - std::lgamma(n - r + 1.0) + r * std::log(p) +
                        (n - r) * std::log1p(-p));
  const double ratio = p / (1.0 - p);
  double sum = 0.0;
  for (int x = r; x <= n; ++x) {
    sum += pmf;
    pmf *= ratio * static_cast<double>(n - x) / static_cast<double>(x + 1);
  }
  return std::min(sum, 1.0);
}

inline double normal_sf(double z) { return 0.5 * std::erfc(z / std::sqrt(2.0)); }

// Probability that a query of the stream selector ends on the finisher's slow
// path because a list segment (or the whole list) overflows. The bound tau is
// the r_s-th largest of 256 per-thread maxima of kpt sample keys each, so the
// fraction Q of the row above tau has the distribution P[Q <= q] =
// P[Binomial(256, 1 - (1 - q)^kpt) >= r_s] — wider than an order statistic of
// the sample itself (measured: cfg4, k' = 2048, C = 19 chunks, 6.6e-5 per
// query against this model's 7.8e-5). Given Q = q a chunk lists about
// Binomial(chunk, q) keys; integrate over q.
double stream_overflow_prob(int64_t n, int64_t r_s, int kpt, int64_t C, int64_t chunk, int64_t seg, int64_t cap) {
  const double S = 256.0 * kpt;
  const double q0 = 0.4 * static_cast<double>(r_s) / S, q1 = std::min(0.5, 8.0 * static_cast<double>(r_s) / S);
  constexpr int N = 240;
  double pf = 0.0, prev = 0.0;
  for (int i = 0; i <= N; ++i) {
    const double q = q0 * std::pow(q1 / q0, static_cast<double>(i) / N);
    const double pt = 1.0 - std::pow(1.0 - q, static_cast<double>(kpt));
    const double F = binom_sf_ge(256, pt, static_cast<int>(r_s));
    const double dF = std::max(F - prev, 0.0);
    prev = std::max(prev, F);
    const double mc = q * static_cast<double>(chunk), sd = std::sqrt(mc * (1.0 - q));
    const double tot = q * static_cast<double>(n);
    const double g = static_cast<double>(C) * normal_sf((static_cast<double>(seg) + 0.5 - mc) / sd) +
                     normal_sf((static_cast<double>(cap) + 0.5 - tot) / std::sqrt(tot));
    pf += dF * std::min(1.0, g);
  }
  return pf + (1.0 - prev);
}

bool plan_stream(hire_ctx ctx, int64_t n, uint32_t K, int64_t B, StreamPlan* st) {
  using namespace hire_dev;
  static const int occ = max_blocks(sel_stream_kernel, kStrThreads, 0);
  const char* ce = std::getenv("HIRE_STREAM_C");
  int64_t C = std::min<int64_t>({ceil_div(n, kStrSample), std::max<int64_t>(1, static_cast<int64_t>(ctx->num_sms) * occ / B),
                                 static_cast<int64_t>(kStrMaxChunks)});
  if (ce) C = std::max<int64_t>(1, std::min<int64_t>(std::atoi(ce), kStrMaxChunks));
  const int64_t G = ceil_div(n, 128);
  // the plan of a shape is computed once (the overflow model costs ~1 ms)
  using Key = std::tuple<int64_t, uint32_t, int64_t>;
  static thread_local std::map<Key, StreamPlan> memo;
  const Key key{n, K, C};
  auto it = memo.find(key);
  if (it != memo.end()) {
    *st = it->second;
    return st->C > 0;
  }
  StreamPlan plan;  // C == 0: the stream path does not apply
  // the largest C with at most one query in a million on the slow path; else
  // the safest C if that is at most one in 10^4 (the slow path costs ~150 us
  // for the step it hits: below 0.1 us per step on average)
  double best = 1e-4;
  for (; C >= 1; C = C > 1 ? (C + 1) / 2 : 0) {
    const int64_t chunk = ceil_div(G, C) * 128;                 // keys of a full chunk
    const int64_t S = std::min<int64_t>(kStrSample, chunk);     // its sample
    const int64_t r_s = binom_tail_rank(S, static_cast<double>(K) / static_cast<double>(n), 1e-7);
    if (r_s > S || r_s > kStrFastRank) break;  // larger ranks: pivot + list kernels
    const int64_t seg = kStrSegMax;  // keys a CTA can stage; the query's list holds kFinCap
    const int kpt = static_cast<int>(std::max<int64_t>(1, S / kStrThreads));
    const double pf = stream_overflow_prob(n, r_s, kpt, C, chunk, seg, kFinCap);
    if (pf < best) {
      best = pf;
      plan.C = static_cast<int>(C);
      plan.seg = static_cast<int>(seg);
      plan.r_s = r_s;
    }
    if (pf <= 1e-6) break;
  }
  if (memo.size() > 256) memo.clear();
  memo.emplace(key, plan);
  *st = plan;
  return plan.C > 0;
}

// Candidate selection over scores [B][n] -> cand [B][cand_stride] ascending.
int run_select(hire_ctx ctx, const float* scores, int64_t score_stride, int64_t n, int64_t B,
               const SelPlan& sp, uint64_t* surv, uint32_t* cand, int64_t cand_stride,
               int* status, bool ordered = true) {
  StageScope scope(ctx, kStageSelect);
  status = ctx->counters + kFallbackOff;  // context-lifetime count (hire_ctx_select_fallbacks)
  if (sp.mode == 2) {
    const uint32_t nn = static_cast<uint32_t>(n), K = static_cast<uint32_t>(sp.k_eff);
#if HIRE_EXPERIMENTS
    // opt-in: one thread-block cluster per query (select2.cuh
    // sel_cluster_kernel). Measured slower than the paths below on B200
    // (a cluster barrier per pass costs more than the counting it splits).
    if (std::getenv("HIRE_SEL_CLUSTER")) {
#define HIRE_SC(NT_, KPT_)                                                                                    \
      if (n <= 16 * NT_ * KPT_) {                                                                             \
        const unsigned cl = static_cast<unsigned>(std::max<int64_t>(1, ceil_div(n, NT_ * KPT_)));           \
        CK(launch_k_cluster(ctx, sel_cluster_kernel<NT_, KPT_>, dim3(cl, static_cast<unsigned>(B)), NT_, 0, cl, \
                            scores, score_stride, nn, K, cand, cand_stride));                                 \
        CK(cudaGetLastError());                                                                               \
        return HIRE_OK;                                                                                       \
      }
      HIRE_SC(256, 4) HIRE_SC(256, 8) HIRE_SC(256, 16) HIRE_SC(512, 16) HIRE_SC(512, 32)
#undef HIRE_SC
    }
#endif
    if (n <= kSel2Exact) {
      // fewer warps per CTA: the per-pass cost of the order statistic is
      // per-warp overhead, the key counting is cheap
      const char* v = std::getenv("HIRE_SEL_EXACT");
      // mid ranks over long rows: the histogram select (variant 4) needs ~10
      // barriers whatever the rank; the 16-way range select wins near the top
      const int variant = v ? std::atoi(v) : (n <= 4096 ? 1 : (K * 64 >= nn ? 4 : 0));
      if (variant == 4 && K <= nn) {
        CK(launch_k(ctx, hire_dev::sel_exact_fast_kernel, static_cast<unsigned>(B), hire_dev::kFinThreads, 0, scores,
                    score_stride, nn, K, cand, cand_stride));
        CK(cudaGetLastError());
        return HIRE_OK;
      }
      if (variant == 1)
        CK(launch_k(ctx, sel_exact_kernel<256, 16>, static_cast<unsigned>(B), 256, 0, scores, score_stride, nn, K,
                    cand, cand_stride));
      else if (variant == 2 && n <= 8192)
        CK(launch_k(ctx, sel_exact_kernel<256, 32>, static_cast<unsigned>(B), 256, 0, scores, score_stride, nn, K,
                    cand, cand_stride));
      else if (variant == 3 && n <= 8192)
        CK(launch_k(ctx, sel_exact_kernel<1024, 8>, static_cast<unsigned>(B), 1024, 0, scores, score_stride, nn, K,
                    cand, cand_stride));
      else
        CK(launch_k(ctx, sel_exact_kernel<512, 16>, static_cast<unsigned>(B), 512, 0, scores, score_stride, nn, K,
                    cand, cand_stride));
      CK(cudaGetLastError());
      return HIRE_OK;
    }
#if HIRE_EXPERIMENTS
    static const bool smem_sel = std::getenv("HIRE_SEL_SMEM") != nullptr;
    if (n <= kSmemRowMax && smem_sel) {
      // opt-in: one CTA per query with the row in shared memory (measured
      // 29 us at n = 32768 against 19 us for the grid-wide chain below)
      CK(launch_k(ctx, sel_smem_kernel, static_cast<unsigned>(B), 1024, static_cast<size_t>(n) * 4, scores,
                  score_stride, nn, K, cand, cand_stride));
      CK(cudaGetLastError());
      return HIRE_OK;
    }
#endif
    const char* nolist = std::getenv("HIRE_SEL_NOLIST");
    if (!(nolist && nolist[0] == '1') && n <= hire_dev::kFinMaxRows && K <= static_cast<uint32_t>(hire_dev::kFinCap)) {
      // list path: sampled exact lower bound -> every key >= lo appended to
      // a per-query list -> sel_fin_kernel (exact k'-th key, emit)
      RET(ensure_fzero(ctx, B));
      hire_dev::FuseSel fs{};
      fs.n = nn;
      fs.K = K;
      fs.n_samp = 0;
      fzero_layout(ctx, B, &fs);
      uint64_t* piv = surv;                                              // [B][4]
      uint64_t* lists = surv + 5 * B + B * kWinBins * kWinGroups / 2;    // [B][kFinCap] (>= B x 65536 words)
      fs.lists = lists;
      // stream path: sample bound + list scan in one launch (sel_stream_kernel)
      {
        const char* se = std::getenv("HIRE_SEL_STREAM");
        const bool aligned = (reinterpret_cast<uintptr_t>(scores) & 15) == 0 && (score_stride & 3) == 0;
        StreamPlan st;
        // whenever the planner accepts the shape: one launch instead of pivot +
        // list scan is 2.5-4.5 us faster from 9000-key rows up at every batch
        // (tools/bench_select.py; cfg1, 32768 keys, B=1: step 28.5 -> 25.7 us)
        if (!(se && se[0] == '0') && aligned && plan_stream(ctx, n, K, B, &st)) {
          fs.stream = 1;
          RET(ensure_tickets(ctx, B));
          CK(launch_k(ctx, sel_stream_kernel, dim3(static_cast<unsigned>(st.C), static_cast<unsigned>(B)), kStrThreads,
                      0, scores, score_stride, nn, static_cast<uint32_t>(st.r_s), static_cast<uint32_t>(st.seg), fs.cnt,
                      fs.lo, lists, static_cast<int64_t>(hire_dev::kFinCap), ctx->tickets));
          CK(launch_k(ctx, sel_fin_kernel, static_cast<unsigned>(B), hire_dev::kFinThreads,
                      static_cast<size_t>((n + 31) / 32) * 4, scores, score_stride, fs, cand, cand_stride,
                      ordered ? 1 : 0, status));
          CK(cudaGetLastError());
          return HIRE_OK;
        }
      }
      // (32 instead of 8 CTAs per SM over the batch: measured the same)
      const int64_t CL = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kWinThreads * kScanBatch),
                                                                std::max<int64_t>(1, 8 * ctx->num_sms / B)));
      const uint32_t perm = sample_perm(static_cast<uint64_t>(n) / 4);
      // sample select on 256 / 512 threads (8-16 keys each; 128 threads: cfg1
      // pivot 7.0 -> 4.3 us); the 2048-key sample in 4-key blocks caps NT at 512
      const char* pe = std::getenv("HIRE_PIV_NT");
      const int pnt = pe ? std::atoi(pe) : (B >= 8 ? 512 : 256);
      auto pk = pnt >= 512 ? sel_pivot_kernel<512> : pnt >= 256 ? sel_pivot_kernel<256> : sel_pivot_kernel<128>;
      CK(launch_k(ctx, pk, static_cast<unsigned>(B), pnt >= 512 ? 512 : pnt >= 256 ? 256 : 128, 0,
                  scores, score_stride, nn, K, perm, piv, reinterpret_cast<unsigned*>(surv + 5 * B), 1));
      CK(launch_k(ctx, sel_wlist_kernel, dim3(static_cast<unsigned>(CL), static_cast<unsigned>(B)), kWinThreads, 0,
                  scores, score_stride, nn, static_cast<const uint64_t*>(piv), fs.cnt, lists, hire_dev::kFinCap));
      CK(launch_k(ctx, sel_fin_kernel, static_cast<unsigned>(B), hire_dev::kFinThreads,
                  static_cast<size_t>((n + 31) / 32) * 4, scores, score_stride, fs, cand, cand_stride, ordered ? 1 : 0,
                  status));
      CK(cudaGetLastError());
      return HIRE_OK;
    }
    // chunks per query: every S3 CTA of the grid must be co-resident (the
    // look-back waits on lower chunks), 4 x 256-thread CTAs per SM
    const int64_t C = std::max<int64_t>(
        1, std::min<int64_t>({std::min<int64_t>(4 * ctx->num_sms, kSelGridChunks) / B,
                              ceil_div(n, kWinThreads * kScanBatch), kWselMaxChunks}));
    if (C * B > std::min<int64_t>(4 * ctx->num_sms, kSelGridChunks))
      return invalid("selection: batch too large for the grid-wide selector");
    const uint32_t seg = static_cast<uint32_t>(sp.wseg);
    RET(ensure_selc(ctx, static_cast<size_t>(B * 3 * C)));
    RET(ensure_tickets(ctx, B));
    unsigned* cnt = ctx->selc;
    unsigned* agg = ctx->selc + B * 2 * C;
    uint64_t* piv = surv;                                        // [B][4]
    uint64_t* thr = surv + 4 * B;                                // [B]
    unsigned* gh = reinterpret_cast<unsigned*>(surv + 5 * B);    // [B][kWinGroups][kWinBins]
    uint64_t* lists = surv + 5 * B + B * kWinBins * kWinGroups / 2;  // [B][groups][bins][cap]
    uint64_t* win = lists + B * kWinGroups * kWinBins * kBinCap;      // [B][C][seg]
    const uint32_t perm = sample_perm(static_cast<uint64_t>(n) / 4);
    CK(launch_k(ctx, sel_pivot_kernel<kPivThreads>, static_cast<unsigned>(B), kPivThreads, 0, scores, score_stride,
                nn, K, perm, piv, gh, 0));
    CK(launch_k(ctx, sel_window_kernel, dim3(static_cast<unsigned>(C), static_cast<unsigned>(B)), kWinThreads, 0,
                scores, score_stride, nn, static_cast<const uint64_t*>(piv), win, seg, cnt, agg, gh, lists));
    CK(launch_k(ctx, sel_wselect_kernel, static_cast<unsigned>(B), kWselThreads, 0, scores, score_stride, nn, K,
                static_cast<int>(C), static_cast<const uint64_t*>(piv), static_cast<const uint64_t*>(win), seg,
                static_cast<const unsigned*>(cnt), static_cast<const unsigned*>(gh),
                static_cast<const uint64_t*>(lists), thr, status));
    CK(launch_k(ctx, sel_emit_kernel, dim3(static_cast<unsigned>(C), static_cast<unsigned>(B)), kEmitThreads, 0,
                scores, score_stride, nn, static_cast<const uint64_t*>(thr), agg, cand, cand_stride,
                ctx->tickets));
    CK(cudaGetLastError());
    return HIRE_OK;
  }
  if (sp.mode == 1) {
    CK(launch_k(ctx, bucket_topt_kernel, dim3(sp.n_buckets, static_cast<unsigned>(B)), 256,
                static_cast<size_t>(ceil_div(n, sp.n_buckets)) * 8, 
        scores, score_stride, n, sp.n_buckets, sp.t, surv));
    CK(cudaGetLastError());
  }
  const size_t smem = sp.mode == 0 ? static_cast<size_t>(n) * 4 : static_cast<size_t>(kPoolKeys) * 8;
  CK(launch_k(ctx, select_candidates_kernel, static_cast<unsigned>(B), kSelectThreads, smem, 
      sp.mode, scores, score_stride, n, surv, sp.n_buckets, sp.t, static_cast<int>(sp.k_eff),
      sp.exact_fix, cand, cand_stride, status));
  CK(cudaGetLastError());
  return HIRE_OK;
}

int check_phi(int phi) {
  if (phi < 0 || phi > 2) return invalid("unknown activation");
  return HIRE_OK;
}

// ---------------------------------------------------------- proxy scores --
struct ScoreWs {
  int8_t* xq = nullptr;
  int8_t* xperm = nullptr;
  float* sx = nullptr;
  int* sumxq = nullptr;
  float* t = nullptr;
};

void take_score_ws(Arena& ar, ScoreWs* w, const hire_scorer_s* a, int64_t B) {
  ar.take(&w->xq, static_cast<size_t>(B * a->d));
  ar.take(&w->xperm, static_cast<size_t>((B + 15) / 16 * 16 * a->d));  // + zero padding queries (tcgen05 B layout)
  ar.take(&w->sx, static_cast<size_t>(B));
  ar.take(&w->sumxq, static_cast<size_t>(B));
  ar.take(&w->t, static_cast<size_t>(B * std::max<int64_t>(a->r, 1)));
}

template <int QB, int CPL>
int launch_q4_int8(hire_ctx ctx, const hire_scorer_s* a, const ScoreWs& w, int64_t b0, int phi,
                   float* out, int64_t stride) {
  auto k = q4_score_fast_int8<QB, CPL>;
  static int bps = 0;
  if (!bps) bps = max_blocks(k, 256, 0);
  const int64_t want = ceil_div(a->rows, 16);
  const int grid = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(bps) * ctx->num_sms));
  CK(launch_k(ctx, k, grid, 256, 0, a->codes, a->pitch, a->scales, a->rows, static_cast<int>(a->d),
                                    w.xperm + b0 * a->d, w.sx + b0, w.sumxq + b0, phi,
                                    out + b0 * stride, stride));
  CK(cudaGetLastError());
  return HIRE_OK;
}

template <int CPL>
int launch_q4_int8_cpl(hire_ctx ctx, const hire_scorer_s* a, const ScoreWs& w, int64_t B, int phi,
                       float* out, int64_t stride) {
  constexpr int QBMAX = CPL <= 2 ? 4 : (CPL == 4 ? 2 : 1);
  int64_t b0 = 0;
  while (b0 < B) {
    const int64_t left = B - b0;
    if (QBMAX >= 4 && left >= 4) { RET((launch_q4_int8<(QBMAX >= 4 ? 4 : 1), CPL>(ctx, a, w, b0, phi, out, stride))); b0 += 4; }
    else if (QBMAX >= 2 && left >= 2) { RET((launch_q4_int8<(QBMAX >= 2 ? 2 : 1), CPL>(ctx, a, w, b0, phi, out, stride))); b0 += 2; }
    else { RET((launch_q4_int8<1, CPL>(ctx, a, w, b0, phi, out, stride))); b0 += 1; }
  }
  return HIRE_OK;
}

template <int CPL>
int launch_q4_fpx(hire_ctx ctx, const hire_scorer_s* a, const float* x, int64_t B, int phi,
                  float* out, int64_t stride) {
  auto k = q4_score_fast_fpx<CPL>;
  static int bps = 0;
  if (!bps) bps = max_blocks(k, 256, 0);
  const int64_t want = ceil_div(a->rows, 8);
  const int grid = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(bps) * ctx->num_sms));
  for (int64_t b = 0; b < B; ++b) {
    CK(launch_k(ctx, k, grid, 256, 0, a->codes, a->pitch, a->scales, a->rows, static_cast<int>(a->d),
                                      x + b * a->d, phi, out + b * stride));
  }
  CK(cudaGetLastError());
  return HIRE_OK;
}

int ensure_mma_layout(hire_ctx ctx, hire_scorer_s* a) {
  if (a->mma) return HIRE_OK;
  const int64_t n_rb = ceil_div(a->rows, 16);
  const int64_t n_words = n_rb * (a->d / 64) * 128;
  CK(cudaMalloc(&a->mma, static_cast<size_t>(n_words) * 4));
  a->mma_owned = true;
  CK(launch_k(ctx, q4_to_mma_layout, static_cast<unsigned>(ceil_div(n_words, 256)), 256, 0, a->codes,
              a->pitch, a->rows, static_cast<int>(a->d), reinterpret_cast<uint32_t*>(a->mma), n_words));
  return HIRE_OK;
}

// ---- tcgen05 proxy (score_umma.cuh) ----
bool umma_shape_ok(const hire_scorer_s* a, int64_t nb) {
  if (a->d % 256 != 0 || nb < 1 || nb > 64) return false;
  const int nq = static_cast<int>((nb + 15) / 16 * 16);
  return UmmaSmem::bytes(4, nq, static_cast<int>(a->d)) <= 227 * 1024;  // at least a 4-stage ring
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

int ensure_umma_layout(hire_ctx ctx, hire_scorer_s* a) {
  if (!a->umma) {
    const int64_t n_rb = ceil_div(a->rows, kUmmaRows);
    const int64_t n_words = n_rb * (a->d / 32) * 512;
    CK(cudaMalloc(&a->umma, static_cast<size_t>(n_words) * 4));
    a->umma_owned = true;
    CK(launch_k(ctx, q4_to_umma_layout, static_cast<unsigned>(ceil_div(n_words, 256)), 256, 0, a->codes,
                a->pitch, a->rows, static_cast<int>(a->d), a->umma, n_words));
  }
  if (!a->umap_ok) {
    auto enc = tensor_map_encoder();
    if (!enc) return set_err(HIRE_ERR_RUNTIME, "cuTensorMapEncodeTiled is unavailable");
    // 2-D u64 view: inner dim = one k chunk of a row block (128 rows x 16 B
    // = 256 x 8 B), outer dim = (row block, k chunk) pairs
    const cuuint64_t dims[2] = {256, static_cast<cuuint64_t>(ceil_div(a->rows, kUmmaRows) * (a->d / 32))};
    const cuuint64_t strides[1] = {2048};
    const cuuint32_t box[2] = {256, static_cast<cuuint32_t>(kUmmaStageChunks)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = enc(&a->umap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, a->umma, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return set_err(HIRE_ERR_RUNTIME, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    a->umap_ok = true;
  }
  return HIRE_OK;
}

int launch_q4_umma(hire_ctx ctx, hire_scorer_s* a, const ScoreWs& w, int64_t b0, int64_t nb, int phi, float* out,
                   int64_t stride) {
  RET(ensure_umma_layout(ctx, a));
  const int d = static_cast<int>(a->d);
  const int nq = static_cast<int>((nb + 15) / 16 * 16);
  const int stages = UmmaSmem::stages_for(nq, d, 227 * 1024);
  const size_t smem = UmmaSmem::bytes(stages, nq, d);  // attribute set in hire_ctx_create
  const int64_t n_rb = ceil_div(a->rows, kUmmaRows);
  const int grid = static_cast<int>(std::min<int64_t>(n_rb, ctx->num_sms));
  // x operand of this chunk: groups of 8 queries, 8d bytes each (b0 % 64 == 0)
  CK(launch_k(ctx, q4_score_umma, grid, kUmmaThreads, smem, a->umap, a->rows, d, a->scales, w.xperm + b0 * d,
              w.sx + b0, w.sumxq + b0, static_cast<int>(nb), nq, stages, phi, out + b0 * stride, stride));
  return HIRE_OK;
}

// the tcgen05 proxy from this many queries per launch up (HIRE_UMMA_MIN_B
// overrides; 0 = off): 9, or 5 when the score row is long enough to keep
// every SM streaming (>= 4 row blocks of 128 per SM). Measured at cfg3
// (V = 256000): the fused IMMA kernel takes 54 / 58 / 63 us at B = 1 / 4 / 8,
// the tcgen05 proxy ~50 us at any batch but needs the stream selector after
// it: B = 8 step 83.9 -> 77.7 us, B = 6 80.1 -> 75.9, B = 5 78.8 -> 75.5, B = 4 about equal (74.3).
int64_t umma_min_batch(int64_t rows = 0, int num_sms = 1 << 30) {
  static const int64_t env = [] {
    const char* e = std::getenv("HIRE_UMMA_MIN_B");
    return e ? static_cast<int64_t>(std::atoi(e)) : static_cast<int64_t>(-1);
  }();
  if (env >= 0) return env;
  return rows >= static_cast<int64_t>(4) * 128 * num_sms ? 5 : 9;
}

template <int NT, int KS>
int launch_q4_mma_t(hire_ctx ctx, const hire_scorer_s* a, const ScoreWs& w, int64_t b0, int64_t nb,
                    int phi, float* out, int64_t stride) {
  auto k = q4_score_mma<NT, KS>;
  const int d = static_cast<int>(a->d);
  const size_t smem = static_cast<size_t>(NT) * 8 * (d + 16) + (KS > 1 ? 8 * NT * 4 * 32 * 4 : 0);
  static int bps = 0;
  if (!bps) {
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    bps = max_blocks(k, 256, smem);
  }
  const int64_t n_rb = ceil_div(a->rows, 16);
  const int64_t want = ceil_div(n_rb, 8 / KS);
  static const int mult = std::getenv("HIRE_MMA_CTAS_PER_SM") ? std::atoi(std::getenv("HIRE_MMA_CTAS_PER_SM")) : 0;
  const int per_sm = mult > 0 ? std::min(mult, bps) : bps;
  const int grid = static_cast<int>(std::min<int64_t>(want, static_cast<int64_t>(per_sm) * ctx->num_sms));
  CK(launch_k(ctx, k, grid, 256, smem, a->mma, a->rows, d, a->scales, w.xq + b0 * d, w.sx + b0,
              w.sumxq + b0, static_cast<int>(nb), phi, out + b0 * stride, stride));
  return HIRE_OK;
}

template <int NT>
int launch_q4_mma_nt(hire_ctx ctx, const hire_scorer_s* a, const ScoreWs& w, int64_t b0, int64_t nb,
                     int phi, float* out, int64_t stride) {
  // split k across warps until the grid has ~32 warps per SM
  const int64_t n_rb = ceil_div(a->rows, 16);
  const int64_t nkb = a->d / 64;
  int ks = 1;
  while (ks < 8 && n_rb * ks < 32LL * ctx->num_sms && nkb >= 2 * ks) ks *= 2;
  switch (ks) {
    case 1: return launch_q4_mma_t<NT, 1>(ctx, a, w, b0, nb, phi, out, stride);
    case 2: return launch_q4_mma_t<NT, 2>(ctx, a, w, b0, nb, phi, out, stride);
    case 4: return launch_q4_mma_t<NT, 4>(ctx, a, w, b0, nb, phi, out, stride);
    default: return launch_q4_mma_t<NT, 8>(ctx, a, w, b0, nb, phi, out, stride);
  }
}

int launch_q4_mma(hire_ctx ctx, const hire_scorer_s* a, const ScoreWs& w, int64_t b0, int64_t nb,
                  int phi, float* out, int64_t stride) {
  if (nb <= 8) return launch_q4_mma_nt<1>(ctx, a, w, b0, nb, phi, out, stride);
  if (nb <= 16) return launch_q4_mma_nt<2>(ctx, a, w, b0, nb, phi, out, stride);
  if (nb <= 32) return launch_q4_mma_nt<4>(ctx, a, w, b0, nb, phi, out, stride);
  return launch_q4_mma_nt<8>(ctx, a, w, b0, nb, phi, out, stride);
}

// phi(Z_approx^T x) for B queries into out [B][stride].
int run_scores(hire_ctx ctx, const hire_scorer_s* a, const float* x, int64_t B, int phi,
               int x_mode, int strict, const ScoreWs& w, float* out, int64_t stride) {
  const int d = static_cast<int>(a->d);
  // the tcgen05 proxy takes every 64-query chunk of >= umma_min_batch()
  // queries; its x operand is prep's grouped layout (xperm, xg_mode 1)
  const bool umma = a->kind == HIRE_SCORER_Q4 && x_mode == HIRE_X_INT8 && d % 64 == 0 && !ctx->force_dp4a &&
                    umma_min_batch() > 0 && std::min<int64_t>(B, 64) >= umma_min_batch(a->rows, ctx->num_sms) &&
                    umma_shape_ok(a, std::min<int64_t>(B, 64));
  if (a->kind == HIRE_SCORER_Q4 && x_mode == HIRE_X_INT8) {
    StageScope pscope(ctx, kStagePrep);
    const int64_t grid = umma ? (B + 15) / 16 * 16 : B;
    CK(launch_k(ctx, prep_x_int8_kernel, static_cast<unsigned>(grid), 256, 0, x, d, w.xq, w.xperm, w.sx, w.sumxq,
                umma ? 1 : 0, static_cast<int>(B)));
    CK(cudaGetLastError());
  }
  StageScope scope(ctx, kStageProxy);
  if (a->kind == HIRE_SCORER_Q4) {
    if (x_mode == HIRE_X_INT8 && d % 64 == 0 && !ctx->force_dp4a) {
      int64_t b0 = 0;
      while (b0 < B) {
        const int64_t nb = std::min<int64_t>(64, B - b0);
        if (umma && nb >= umma_min_batch(a->rows, ctx->num_sms)) {
          RET(launch_q4_umma(ctx, const_cast<hire_scorer_s*>(a), w, b0, nb, phi, out, stride));
        } else {
          RET(ensure_mma_layout(ctx, const_cast<hire_scorer_s*>(a)));
          RET(launch_q4_mma(ctx, a, w, b0, nb, phi, out, stride));
        }
        b0 += nb;
      }
      return HIRE_OK;
    }
    const bool fast_shape = (d % 1024 == 0) && a->pitch == d / 2 && d <= 8192;
    if (fast_shape && x_mode == HIRE_X_INT8) {
      switch (d / 1024) {
        case 1: return launch_q4_int8_cpl<1>(ctx, a, w, B, phi, out, stride);
        case 2: return launch_q4_int8_cpl<2>(ctx, a, w, B, phi, out, stride);
        case 4: return launch_q4_int8_cpl<4>(ctx, a, w, B, phi, out, stride);
        case 8: return launch_q4_int8_cpl<8>(ctx, a, w, B, phi, out, stride);
        default: break;
      }
    }
    if (fast_shape && x_mode == HIRE_X_FP32 && !strict) {
      switch (d / 1024) {
        case 1: return launch_q4_fpx<1>(ctx, a, x, B, phi, out, stride);
        case 2: return launch_q4_fpx<2>(ctx, a, x, B, phi, out, stride);
        case 4: return launch_q4_fpx<4>(ctx, a, x, B, phi, out, stride);
        default: break;
      }
    }
    const size_t smem = static_cast<size_t>(d) * 5 + 16;
    CK(launch_k(ctx, q4_score_seq, dim3(static_cast<unsigned>(ceil_div(a->rows, 128)), static_cast<unsigned>(B)), 128, smem, 
        a->codes, a->pitch, a->scales, a->rows, d, x, w.xq, w.sx, x_mode == HIRE_X_INT8, phi, out, stride));
    CK(cudaGetLastError());
    return HIRE_OK;
  }
  // low-rank
  const int r = static_cast<int>(a->r);
  const bool bf = a->dtype == HIRE_BF16;
  if (!strict && d % 8 == 0 && (r == 32 || r == 64 || r == 128) && B <= 64 && !std::getenv("HIRE_LR_SIMT")) {
    const dim3 gt(static_cast<unsigned>(r), static_cast<unsigned>(ceil_div(B, 4)));
    if (bf) CK(launch_k(ctx, lr_t_fast<__nv_bfloat16>, gt, 256, 0, static_cast<const __nv_bfloat16*>(a->z1), d, x, static_cast<int>(B), r, w.t));
    else CK(launch_k(ctx, lr_t_fast<float>, gt, 256, 0, static_cast<const float*>(a->z1), d, x, static_cast<int>(B), r, w.t));
    const int64_t tiles = ceil_div(a->rows, 16);
    const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(tiles, kLrThreads / 32), 3 * ctx->num_sms)));
#define LRM(TT, RR, NN)                                                                                    \
    CK(launch_k(ctx, lr_score_mma<TT, RR, NN>, grid, kLrThreads, 0, static_cast<const TT*>(a->z2), a->rows, \
                static_cast<const float*>(w.t), static_cast<int>(B), static_cast<int>(b0), phi, out, stride))
#define LRR(TT, NN) \
    { if (r == 32) LRM(TT, 32, NN); else if (r == 64) LRM(TT, 64, NN); else LRM(TT, 128, NN); }
    for (int64_t b0 = 0; b0 < B; b0 += 16) {
      const bool one = B - b0 <= 8;
      if (bf) { if (one) LRR(__nv_bfloat16, 1) else LRR(__nv_bfloat16, 2) }
      else { if (one) LRR(float, 1) else LRR(float, 2) }
    }
#undef LRR
#undef LRM
    CK(cudaGetLastError());
    return HIRE_OK;
  }
  {
    const int64_t items = static_cast<int64_t>(r) * B;
    const unsigned grid = static_cast<unsigned>(strict ? ceil_div(items, 256) : ceil_div(items * 32, 256));
    if (bf) CK(launch_k(ctx, lr_t_kernel<__nv_bfloat16>, grid, 256, 0, static_cast<const __nv_bfloat16*>(a->z1), r, d, x, static_cast<int>(B), strict, w.t));
    else CK(launch_k(ctx, lr_t_kernel<float>, grid, 256, 0, static_cast<const float*>(a->z1), r, d, x, static_cast<int>(B), strict, w.t));
    CK(cudaGetLastError());
  }
  const size_t smem = static_cast<size_t>(r) * B * 4;
  const unsigned grid = static_cast<unsigned>(ceil_div(a->rows, 128));
  auto setsm = [&](const void*) -> int { return HIRE_OK; };  // attributes set at ctx creation
  if (smem > 200 * 1024) return invalid("low-rank scores: rank * batch too large");
  if (r == 64 && B * r * 4 <= 200 * 1024) {
    if (bf && strict) { RET(setsm((const void*)lr_score_kernel<__nv_bfloat16, 64, true>)); CK(launch_k(ctx, lr_score_kernel<__nv_bfloat16, 64, true>, grid, 128, smem, static_cast<const __nv_bfloat16*>(a->z2), a->rows, w.t, static_cast<int>(B), phi, out, stride)); }
    else if (bf) { RET(setsm((const void*)lr_score_kernel<__nv_bfloat16, 64, false>)); CK(launch_k(ctx, lr_score_kernel<__nv_bfloat16, 64, false>, grid, 128, smem, static_cast<const __nv_bfloat16*>(a->z2), a->rows, w.t, static_cast<int>(B), phi, out, stride)); }
    else if (strict) { RET(setsm((const void*)lr_score_kernel<float, 64, true>)); CK(launch_k(ctx, lr_score_kernel<float, 64, true>, grid, 128, smem, static_cast<const float*>(a->z2), a->rows, w.t, static_cast<int>(B), phi, out, stride)); }
    else { RET(setsm((const void*)lr_score_kernel<float, 64, false>)); CK(launch_k(ctx, lr_score_kernel<float, 64, false>, grid, 128, smem, static_cast<const float*>(a->z2), a->rows, w.t, static_cast<int>(B), phi, out, stride)); }
  } else {
    if (bf && strict) { RET(setsm((const void*)lr_score_generic<__nv_bfloat16, true>)); CK(launch_k(ctx, lr_score_generic<__nv_bfloat16, true>, grid, 128, smem, static_cast<const __nv_bfloat16*>(a->z2), a->rows, r, w.t, static_cast<int>(B), phi, out, stride)); }
    else if (bf) { RET(setsm((const void*)lr_score_generic<__nv_bfloat16, false>)); CK(launch_k(ctx, lr_score_generic<__nv_bfloat16, false>, grid, 128, smem, static_cast<const __nv_bfloat16*>(a->z2), a->rows, r, w.t, static_cast<int>(B), phi, out, stride)); }
    else if (strict) { RET(setsm((const void*)lr_score_generic<float, true>)); CK(launch_k(ctx, lr_score_generic<float, true>, grid, 128, smem, static_cast<const float*>(a->z2), a->rows, r, w.t, static_cast<int>(B), phi, out, stride)); }
    else { RET(setsm((const void*)lr_score_generic<float, false>)); CK(launch_k(ctx, lr_score_generic<float, false>, grid, 128, smem, static_cast<const float*>(a->z2), a->rows, r, w.t, static_cast<int>(B), phi, out, stride)); }
  }
  CK(cudaGetLastError());
  return HIRE_OK;
}

// ------------------------------------------------------------- recompute --
template <typename T, int CPL>
int launch_recompute_fast(hire_ctx ctx, const void* w, int d, const uint32_t* cand,
                          int64_t cand_stride, int64_t n_cand, const float* x, int64_t B, int phi,
                          float* out, int64_t out_stride) {
  const size_t smem = static_cast<size_t>(d) * 4;
  auto k = recompute_fast<T, CPL>;
  // one wave of 2 CTAs/SM (8 warps each); warps stride over the rows
  // (CPL >= 16: one CTA/SM, the long rows need more than 128 registers)
  const int per_sm = CPL >= 16 ? 1 : 2;
  const int64_t tiles = std::max<int64_t>(1, std::min<int64_t>(ceil_div(n_cand, 8), std::max<int64_t>(1, per_sm * ctx->num_sms / B)));
  CK(launch_k(ctx, k, dim3(static_cast<unsigned>(tiles), static_cast<unsigned>(B)), 256, smem,
      static_cast<const T*>(w), d, cand, cand_stride, static_cast<int>(n_cand), x, phi, out, out_stride));
  CK(cudaGetLastError());
  return HIRE_OK;
}

#if HIRE_EXPERIMENTS
// Bulk-copy ring variant (exact.cuh recompute_tma); *done = false when the
// rows do not fit two groups of slots.
template <typename T, int G>
int launch_recompute_tma_g(hire_ctx ctx, const void* w, int d, const uint32_t* cand, int64_t cand_stride,
                           int64_t n_cand, const float* x, int64_t B, int phi, float* out, int64_t out_stride) {
  const size_t row_bytes = static_cast<size_t>(d) * sizeof(T);
  const size_t smem = ((static_cast<size_t>(d) * 4 + 4 * 2 * G * 8 + 127) & ~static_cast<size_t>(127)) +
                      4 * 2 * G * row_bytes;
  static bool attr = false;
  if (!attr) {
    CK(cudaFuncSetAttribute(recompute_tma<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  const int64_t per_q = std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms / std::max<int64_t>(B, 1), ceil_div(n_cand, 8)));
  CK(launch_k(ctx, recompute_tma<T, G>, dim3(static_cast<unsigned>(per_q), static_cast<unsigned>(B)), 128, smem,
              static_cast<const T*>(w), d, cand, cand_stride, static_cast<int>(n_cand), x, phi, out, out_stride));
  CK(cudaGetLastError());
  return HIRE_OK;
}

template <typename T>
int launch_recompute_tma(hire_ctx ctx, const void* w, int d, const uint32_t* cand, int64_t cand_stride,
                         int64_t n_cand, const float* x, int64_t B, int phi, float* out, int64_t out_stride,
                         bool* done) {
  *done = false;
  const size_t row_bytes = static_cast<size_t>(d) * sizeof(T);
  const size_t fixed = static_cast<size_t>(d) * 4 + 1024;
  const size_t budget = 224 * 1024;
  auto fits = [&](int g) { return fixed + 4 * 2 * static_cast<size_t>(g) * row_bytes <= budget; };
  if (fits(4)) { RET((launch_recompute_tma_g<T, 4>(ctx, w, d, cand, cand_stride, n_cand, x, B, phi, out, out_stride))); }
  else if (fits(3)) { RET((launch_recompute_tma_g<T, 3>(ctx, w, d, cand, cand_stride, n_cand, x, B, phi, out, out_stride))); }
  else if (fits(2)) { RET((launch_recompute_tma_g<T, 2>(ctx, w, d, cand, cand_stride, n_cand, x, B, phi, out, out_stride))); }
  else return HIRE_OK;
  *done = true;
  return HIRE_OK;
}

// phi(<W_row, x_b>) for rows cand[b][i] (or i when cand == nullptr).
#endif

#if HIRE_EXPERIMENTS
// Batch-union gather (exact.cuh K4U), opt-in with HIRE_UNION=1: measured
// slower than the per-query gather at every batch (see exact.cuh).
bool union_gather_pays(hire_ctx ctx, const hire_matrix_s* m, int64_t n_cand, int64_t B) {
  (void)ctx;
  (void)n_cand;
  const int64_t nct = m->d * static_cast<int64_t>(dtype_size(m->dtype)) / 512;
  if (B < 2 || B > 64 || nct < 1 || B * m->rows * nct * 4 > (int64_t{64} << 20)) return false;
  const char* e = std::getenv("HIRE_UNION");
  return e && e[0] == '1';
}

int run_recompute_union(hire_ctx ctx, const hire_matrix_s* m, const uint32_t* cand, int64_t cand_stride,
                        int64_t n_cand, const float* x, int64_t B, int phi, float* out, int64_t out_stride) {
  using namespace hire_dev;
  const int d = static_cast<int>(m->d);
  const bool bf = m->dtype == HIRE_BF16;
  const int nct = static_cast<int>(m->d * static_cast<int64_t>(dtype_size(m->dtype)) / 512);
  const int dc = bf ? 256 : 128;
  RET(ensure_umask(ctx, m->rows));
  // the partial sums live behind the caller's arena allocations: a
  // context-owned grow-only buffer of their own
  const size_t need = static_cast<size_t>(B) * m->rows * nct * 4;
  RET(ensure(&ctx->upart, &ctx->upart_cap, need, ctx->stream));
  float* part = static_cast<float*>(ctx->upart);
  const unsigned pairs_blocks = static_cast<unsigned>(ceil_div(B * n_cand, 256));
  CK(launch_k(ctx, union_mark_kernel, pairs_blocks, 256, 0, cand, cand_stride, static_cast<int>(n_cand),
              static_cast<int>(B), ctx->umask));
  // row tiles: about 4 CTAs per SM over the nct slices, at least 64 rows each
  const int64_t tiles = std::max<int64_t>(1, std::min<int64_t>(ceil_div(m->rows, 64), 4 * ctx->num_sms / nct));
  const int rows_per_cta = static_cast<int>(ceil_div(m->rows, tiles));
  const size_t smem = static_cast<size_t>(B) * dc * 4;
  if (bf) {
    static bool attr = false;
    if (!attr) {
      CK(cudaFuncSetAttribute(union_dot_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 256 * 4));
      attr = true;
    }
    CK(launch_k(ctx, union_dot_kernel<__nv_bfloat16>, dim3(static_cast<unsigned>(nct), static_cast<unsigned>(ceil_div(m->rows, rows_per_cta))),
                256, smem, static_cast<const __nv_bfloat16*>(m->ptr), d, m->rows,
                static_cast<const unsigned long long*>(ctx->umask), x, static_cast<int>(B), rows_per_cta, part));
  } else {
    CK(launch_k(ctx, union_dot_kernel<float>, dim3(static_cast<unsigned>(nct), static_cast<unsigned>(ceil_div(m->rows, rows_per_cta))),
                256, smem, static_cast<const float*>(m->ptr), d, m->rows,
                static_cast<const unsigned long long*>(ctx->umask), x, static_cast<int>(B), rows_per_cta, part));
  }
  CK(launch_k(ctx, union_gather_kernel, pairs_blocks, 256, 0, static_cast<const float*>(part), m->rows, nct, cand,
              cand_stride, static_cast<int>(n_cand), static_cast<int>(B), phi, out, out_stride, ctx->umask));
  CK(cudaGetLastError());
  return HIRE_OK;
}
#endif  // HIRE_EXPERIMENTS

int run_recompute(hire_ctx ctx, const hire_matrix_s* m, const uint32_t* cand, int64_t cand_stride,
                  int64_t n_cand, const float* x, int64_t B, int phi, int strict, float* out,
                  int64_t out_stride) {
  if (n_cand <= 0) return HIRE_OK;
  StageScope scope(ctx, kStageRecompute);
  const int d = static_cast<int>(m->d);
  const size_t es = dtype_size(m->dtype);
  const int64_t bytes = static_cast<int64_t>(d) * static_cast<int64_t>(es);
#if HIRE_EXPERIMENTS
  // bulk-copy ring: opt-in (HIRE_RECOMPUTE_TMA=1). Measured on B200 the
  // register path is faster at every batch (cfg3 B=8: 8.0 vs 12.6 us, B=32:
  // 23 vs 46 us; cfg4: 61 vs 63 us)
  const bool tma = std::getenv("HIRE_RECOMPUTE_TMA") != nullptr;
  if (!strict && bytes % 512 == 0 && n_cand * B >= 8192 && tma) {
    bool done = false;
    if (m->dtype == HIRE_BF16)
      RET(launch_recompute_tma<__nv_bfloat16>(ctx, m->ptr, d, cand, cand_stride, n_cand, x, B, phi, out, out_stride, &done));
    else
      RET(launch_recompute_tma<float>(ctx, m->ptr, d, cand, cand_stride, n_cand, x, B, phi, out, out_stride, &done));
    if (done) return HIRE_OK;
  }
#endif
#if HIRE_EXPERIMENTS
  if (!strict && bytes % 512 == 0 && cand && union_gather_pays(ctx, m, n_cand, B))
    return run_recompute_union(ctx, m, cand, cand_stride, n_cand, x, B, phi, out, out_stride);
#endif
  if (!strict && bytes % 512 == 0) {
    const int cpl = static_cast<int>(bytes / 512);
    const bool bf = m->dtype == HIRE_BF16;
#define RC(C)                                                                                              \
  case C:                                                                                                 \
    return bf ? launch_recompute_fast<__nv_bfloat16, C>(ctx, m->ptr, d, cand, cand_stride, n_cand, x, B, phi, out, out_stride) \
              : launch_recompute_fast<float, C>(ctx, m->ptr, d, cand, cand_stride, n_cand, x, B, phi, out, out_stride);
    switch (cpl) {
      RC(1) RC(2) RC(4) RC(8) RC(16)
      default: break;
    }
#undef RC
  }
  const size_t smem = static_cast<size_t>(d) * 4;
  const dim3 grid(static_cast<unsigned>(ceil_div(n_cand, 128)), static_cast<unsigned>(B));
  if (m->dtype == HIRE_BF16) {
    CK(launch_k(ctx, recompute_seq<__nv_bfloat16>, grid, 128, smem, static_cast<const __nv_bfloat16*>(m->ptr), d, cand, cand_stride, static_cast<int>(n_cand), x, phi, out, out_stride));
  } else {
    CK(launch_k(ctx, recompute_seq<float>, grid, 128, smem, static_cast<const float*>(m->ptr), d, cand, cand_stride, static_cast<int>(n_cand), x, phi, out, out_stride));
  }
  CK(cudaGetLastError());
  return HIRE_OK;
}

int run_final(hire_ctx ctx, const float* vals, int64_t vs, const uint32_t* idx, int64_t is,
              const uint64_t* src_keys, int64_t n_per, int64_t part_stride, int64_t n, int64_t K,
              int64_t B, int out_mode, uint32_t* out_idx, float* out_val, float* out_prob,
              uint64_t* out_keys, int64_t out_stride) {
  if (K < 1 || n < 1) return HIRE_OK;
  StageScope scope(ctx, kStageFinal);
  if (out_mode == 0 && K > kFinalMax) return invalid("final top-k: k exceeds " + std::to_string(kFinalMax));
  int64_t P = 1;
  while (P < K) P <<= 1;
  const size_t smem = out_mode == 0 ? static_cast<size_t>(P) * 8 : 0;
  // ranked top-k of a small pool, a few queries: per-warp register sort +
  // merge tree (final3_kernel). Measured (cfg3, n = 1024, K = 64): B = 1 step
  // 67.7 -> 65.5 us, but B = 8 83.9 -> 85.7 and B = 32 107.5 -> 109.3 (the
  // shuffle pipe of 16 sorting warps per SM); K = 128 of 2048 (cfg4) loses 9 us.
  const char* f3 = std::getenv("HIRE_FINAL3");
  if (out_mode == 0 && K <= 64 && n <= 2048 && (f3 ? f3[0] == '1' : B <= 4)) {
    const int np = static_cast<int>(std::max<int64_t>(n_per, 1));
#define HIRE_F3(NT_, SL_)                                                                                   \
    if (K <= 32 * SL_ && n <= (NT_ / 32) * 32 * SL_) {                                                      \
      CK(launch_k(ctx, final3_kernel<NT_, SL_>, static_cast<unsigned>(B), NT_, 0, vals, vs, idx, is, src_keys, np, \
                  part_stride, static_cast<int>(n), static_cast<int>(K), out_idx, out_val, out_prob, out_stride)); \
      CK(cudaGetLastError());                                                                               \
      return HIRE_OK;                                                                                       \
    }
    HIRE_F3(32, 1) HIRE_F3(64, 1) HIRE_F3(128, 1) HIRE_F3(256, 1)
    HIRE_F3(128, 2) HIRE_F3(256, 2) HIRE_F3(512, 2) HIRE_F3(1024, 2)
#undef HIRE_F3
  }
  if (n <= kFinal2Max && !std::getenv("HIRE_SELECT_V1")) {
    const int np = static_cast<int>(std::max<int64_t>(n_per, 1));
    // the K-th key by the histogram select (HIRE_F2_FAST=0: 16-way range
    // splits). Measured: cfg4 (128 of 2048) step 86.5 -> 84.7 us, cfg2 (410
    // of 820) 36.7 -> 36.0, cfg3 B=32 (64 of 1024) 99.6 -> 99.2
    const char* f2e = std::getenv("HIRE_F2_FAST");
    const int f2_fast = f2e ? std::atoi(f2e) : 1;
#define HIRE_F2(NT_, KPT)                                                                               \
    if (n <= NT_ * KPT) {                                                                               \
      CK(launch_k(ctx, final2_kernel<NT_, KPT>, static_cast<unsigned>(B), NT_, smem, vals, vs, idx, is, \
                  src_keys, np, part_stride, static_cast<int>(n), static_cast<int>(K), out_mode, out_idx,   \
                  out_val, out_prob, out_keys, out_stride, f2_fast));                                   \
      CK(cudaGetLastError());                                                                           \
      return HIRE_OK;                                                                                   \
    }
    // batches of >= 8 queries: 2 keys per thread (up to 1024 threads) — the
    // range-select passes are shorter (cfg4 final 12.7 -> 9.9 us, cfg3 B=32
    // 10.4 -> 7.1); a single query is faster on the narrow CTA
    const char* wide = std::getenv("HIRE_F2_WIDE");
    if ((wide ? wide[0] == '1' : B >= 8) && n > 256) {
      HIRE_F2(256, 2) HIRE_F2(512, 2) HIRE_F2(1024, 2)
    }
    HIRE_F2(128, 1) HIRE_F2(128, 2) HIRE_F2(128, 4) HIRE_F2(128, 8) HIRE_F2(128, 16)
    HIRE_F2(256, 16) HIRE_F2(256, 32) HIRE_F2(512, 32)
#undef HIRE_F2
  }
  CK(launch_k(ctx, final_select_kernel, static_cast<unsigned>(B), kSelectThreads, smem, 
      vals, vs, idx, is, src_keys, static_cast<int>(std::max<int64_t>(n_per, 1)), part_stride,
      static_cast<int>(n), static_cast<int>(K), out_mode, out_idx, out_val, out_prob, out_keys, out_stride));
  CK(cudaGetLastError());
  return HIRE_OK;
}

// Host-call inputs: pinned (mapped) host memory -> device, 16 B per thread,
// read straight over PCIe (no copy-engine transfer in the call's graph).
__global__ void fetch_host_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, int64_t n16) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

constexpr int kFetchCtas = 64;         // grid bound of the fetch kernels
constexpr int kFetchSlotStride = 16;   // u64 words between the CTAs' copies of the slot (128 B)

// The same copy with the source address read from a word of mapped host
// memory (hire_ctx_s::fetch_slot): system-scope load, never a cached copy.
__global__ void fetch_host_slot_kernel(const unsigned long long* __restrict__ slot, uint4* __restrict__ dst,
                                       int64_t n16) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  // one PCIe read per CTA, each CTA from a line of its own: system-scope loads
  // of one address are served one after the other (~0.8 us each: 64 CTAs on
  // one word cost 52 us, a load per thread ~450 us)
  __shared__ unsigned long long s_src;
  if (threadIdx.x == 0) {
    unsigned long long p;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(p) : "l"(slot + blockIdx.x * kFetchSlotStride) : "memory");
    s_src = p;
  }
  __syncthreads();
  // read-only path (ld.global.nc, as the compiler picks for a const __restrict__
  // parameter): whole lines per request over PCIe. Plain generic loads through a
  // pointer the compiler cannot classify took 60 us for 256 KB instead of 10.
  const uint4* src = reinterpret_cast<const uint4*>(s_src);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    dst[i] = __ldg(src + i);
}

// A host thread that has made no CUDA call yet has no current device: its
// first cudaPointerGetAttributes fails (found with two threads calling
// hire_topk_host on two contexts: the input then had "no device alias"). Every
// entry point that takes host buffers binds the context's device once per thread.
void bind_thread(hire_ctx ctx) {
  static thread_local int bound = -1;
  if (bound != ctx->device) {
    cudaSetDevice(ctx->device);
    bound = ctx->device;
  }
}

void store_fetch_slot(hire_ctx ctx, const void* dsrc) {
  volatile unsigned long long* sl = ctx->fetch_slot;
  for (int c = 0; c < kFetchCtas; ++c) sl[c * kFetchSlotStride] = reinterpret_cast<unsigned long long>(dsrc);
}

// H2D of a host call's inputs: the fetch kernel when aligned (source address
// through the context's slot), else a copy.
int fetch_inputs(hire_ctx ctx, void* dst, const void* host_src, size_t bytes) {
  void* dsrc = nullptr;
  if (ctx->fetch_slot && bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(host_src) & 15) == 0 &&
      cudaHostGetDevicePointer(&dsrc, const_cast<void*>(host_src), 0) == cudaSuccess && dsrc) {
    const int64_t n16 = static_cast<int64_t>(bytes / 16);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(n16, 256), kFetchCtas));
    store_fetch_slot(ctx, dsrc);
    ctx->fetch_by_slot = true;
    CK(launch_k(ctx, fetch_host_slot_kernel, grid, 256, 0, static_cast<const unsigned long long*>(ctx->fetch_slot_dev),
                static_cast<uint4*>(dst), n16));
    return HIRE_OK;
  }
  cudaGetLastError();
  CK(cudaMemcpyAsync(dst, host_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return HIRE_OK;
}

// union_group_select (ffn.hpp:237-253): sorted union of the B per-sample
// selections. One CTA: group bitmap in shared memory, OR of every selected id,
// popcount prefix, ascending emit. *count = |union|.
__global__ void __launch_bounds__(1024) group_union_kernel(const uint32_t* __restrict__ sel, int64_t stride, int kg,
                                                           int B, int ng, uint32_t* __restrict__ out,
                                                           int64_t* __restrict__ count) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  extern __shared__ unsigned u_bm[];
  __shared__ int s_scan[40];
  const int nw = (ng + 31) / 32;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) u_bm[i] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < B * kg; i += blockDim.x) {
    const uint32_t id = sel[static_cast<int64_t>(i / kg) * stride + i % kg];
    atomicOr(u_bm + (id >> 5), 1u << (id & 31));
  }
  __syncthreads();
  const int W = (nw + 1023) / 1024, w0 = threadIdx.x * W;
  int mine = 0;
  for (int i = 0; i < W; ++i)
    if (w0 + i < nw) mine += __popc(u_bm[w0 + i]);
  int total;
  int pos = hire_dev::block_scan_excl<1024>(mine, s_scan, &total);
  for (int i = 0; i < W && w0 + i < nw; ++i) {
    unsigned word = u_bm[w0 + i];
    while (word) {
      out[pos++] = static_cast<uint32_t>((w0 + i) * 32 + __ffs(word) - 1);
      word &= word - 1u;
    }
  }
  if (threadIdx.x == 0) *count = total;
}

// out[i] += add[i] (ffn_common_path's dense + sparse sum, ffn.hpp:232)
__global__ void add_f32_kernel(float* __restrict__ out, const float* __restrict__ add, int64_t n) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = __fadd_rn(out[i], add[i]);
}

// A caller buffer the kernels can address directly (pinned / registered host
// memory, 16-byte aligned): its device alias; nullptr for pageable memory.
void* host_alias(const void* p, size_t bytes) {
  if (!p || bytes % 16 != 0 || (reinterpret_cast<uintptr_t>(p) & 15) != 0) return nullptr;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

__global__ void add_offset_kernel(uint32_t* idx, int64_t n, uint32_t off) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) idx[i] += off;
}

__global__ void add_offset_strided_kernel(uint32_t* s, int64_t stride, int64_t n, int64_t B, uint32_t off) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n * B) s[(i / n) * stride + i % n] += off;
}

__global__ void iota_mod_kernel(uint32_t* u, int64_t m, int64_t n) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) u[i] = static_cast<uint32_t>(i % m);
}

__global__ void gather_values_kernel(const float* v, int64_t n, const uint32_t* c, int64_t kk, int64_t B, float* o) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  KTrace kt_(hire_dev::kKtGather);
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < kk * B) o[i] = v[(i / kk) * n + c[i]];
}

// FFN helpers for g > 1 -------------------------------------------------------
__global__ void group_proxy_kernel(const float* scores, int64_t ss, int64_t ngroups, int g, int B,
                                   float* proxy) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (id >= ngroups * B) return;
  const int64_t b = id / ngroups, j = id % ngroups;
  float acc = 0.0f;  // ffn.hpp:115-118, ascending t
  for (int t = 0; t < g; ++t) acc = __fadd_rn(acc, fabsf(scores[b * ss + j * g + t]));
  proxy[b * ngroups + j] = acc;
}

__global__ void expand_groups_kernel(const uint32_t* groups, int64_t gs, int64_t n, int g, int B,
                                     uint32_t* units) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (id >= n * g * B) return;
  const int64_t b = id / (n * g), r = id % (n * g);
  units[b * n * g + r] = groups[b * gs + r / g] * g + static_cast<uint32_t>(r % g);
}

__global__ void group_sum_kernel(const float* act, int64_t n, int g, int B, float* out) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t id = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (id >= n * B) return;
  const int64_t b = id / n, j = id % n;
  float acc = 0.0f;  // ffn.hpp:127-129
  for (int t = 0; t < g; ++t) acc = __fadd_rn(acc, fabsf(act[b * n * g + j * g + t]));
  out[b * n + j] = acc;
}

int run_down(hire_ctx ctx, const hire_matrix_s* v, const uint32_t* units, const float* act,
             int64_t stride, int64_t n_units, int64_t B, int strict, float* partial, float* out) {
  StageScope scope(ctx, kStageDown);
  const int d = static_cast<int>(v->d);
  const bool bf = v->dtype == HIRE_BF16;
  if (n_units == 0) {
    CK(cudaMemsetAsync(out, 0, static_cast<size_t>(B) * d * 4, ctx->stream));
    return HIRE_OK;
  }
  if (strict || (static_cast<int64_t>(d) * static_cast<int64_t>(dtype_size(v->dtype))) % 16 != 0) {
    const dim3 grid(static_cast<unsigned>(ceil_div(d, 256)), static_cast<unsigned>(B));
    if (bf) CK(launch_k(ctx, ffn_down_seq<__nv_bfloat16>, grid, 256, 0, static_cast<const __nv_bfloat16*>(v->ptr), d, units, act, stride, static_cast<int>(n_units), out));
    else CK(launch_k(ctx, ffn_down_seq<float>, grid, 256, 0, static_cast<const float*>(v->ptr), d, units, act, stride, static_cast<int>(n_units), out));
    CK(cudaGetLastError());
    return HIRE_OK;
  }
  const int ch = 8;
  const int64_t nch = ceil_div(n_units, ch);
  const dim3 grid(static_cast<unsigned>(nch), static_cast<unsigned>(B));
  if (bf) CK(launch_k(ctx, ffn_down_partial<__nv_bfloat16>, grid, 256, 0, static_cast<const __nv_bfloat16*>(v->ptr), d, units, act, stride, static_cast<int>(n_units), ch, partial));
  else CK(launch_k(ctx, ffn_down_partial<float>, grid, 256, 0, static_cast<const float*>(v->ptr), d, units, act, stride, static_cast<int>(n_units), ch, partial));
  CK(cudaGetLastError());
  CK(launch_k(ctx, ffn_down_reduce, static_cast<unsigned>(ceil_div(B * d, 256)), 256, 0, partial, static_cast<int>(nch), d, static_cast<int>(B), out));
  CK(cudaGetLastError());
  return HIRE_OK;
}

int validate_topk(const hire_matrix_s* w, const hire_scorer_s* a, int64_t B, const hire_topk_params* p) {
  if (!w || !a || !p) return invalid("null handle");
  if (p->k < 1) return invalid("HireConfig: k must be >= 1");
  if (p->k > p->k_prime)
    return invalid("HireConfig: k (" + std::to_string(p->k) + ") must be <= k_prime (" + std::to_string(p->k_prime) + ")");
  RET(check_phi(p->phi));
  if (a->d != w->d || a->rows != w->rows)
    return invalid("hire_topk: scorer is " + std::to_string(a->d) + "x" + std::to_string(a->rows) +
                   " but Z is " + std::to_string(w->d) + "x" + std::to_string(w->rows));
  if (B < 1) return invalid("hire_topk: batch must be >= 1");
  if (p->x_mode != HIRE_X_FP32 && p->x_mode != HIRE_X_INT8) return invalid("unknown x_mode");
  if (p->x_mode == HIRE_X_INT8 && a->kind != HIRE_SCORER_Q4) return invalid("x_mode int8 needs an int4 proxy");
  return HIRE_OK;
}

// The local stage of hire_topk: scores -> candidates -> exact values.
// ------------------------------------------- proxy + fused selection --
// fsel.cuh: the int4 tensor-core proxy kernel filters its own scores against
// a sampled lower bound; sel_fin_kernel finishes the exact top-k'.
struct FselPlan {
  bool on = false;
  int nt = 1, ks = 1, G = 0, nbrk = 1, samp_step = 1, n_samp = 0, r_lo = 0;
  size_t smem = 0;
};

template <int NT, int KS>
size_t fsel_smem(int d) {
  return static_cast<size_t>(NT) * 8 * (d + 16) + (KS > 1 ? static_cast<size_t>(8) * NT * 4 * 32 * 4 : 0);
}

template <int NT, int KS>
int fsel_bps(size_t smem) {
  static size_t last = ~size_t(0);
  static int bps = 0;
  if (smem != last) {
    auto k = q4_score_mma_sel<NT, KS>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024) != cudaSuccess) return 0;
    bps = max_blocks(k, 256, smem);
    last = smem;
  }
  return bps;
}

template <int NT>
int fsel_bps_ks(int ks, int d, size_t* smem) {
  if (ks == 1) { *smem = fsel_smem<NT, 1>(d); return fsel_bps<NT, 1>(*smem); }
  *smem = fsel_smem<NT, 2>(d);
  return fsel_bps<NT, 2>(*smem);
}

// Decide whether the fused path applies and size it: one full wave of
// streaming CTAs (same count on every SM) + bracket CTAs, list capacity,
// sample rank of the bracket.
void plan_fsel(hire_ctx ctx, const hire_scorer_s* a, int64_t B, const hire_topk_params* p, const SelPlan& sp,
               FselPlan* f) {
  f->on = false;
  const char* env = std::getenv("HIRE_FSEL");
  if (env && env[0] == '0') return;
  if (sp.mode != 2 || a->rows <= kSel2Exact || a->kind != HIRE_SCORER_Q4 || p->x_mode != HIRE_X_INT8) return;
  // B <= 8 (one MMA n-tile): at larger batches the in-flight filter's
  // registers spill and the fused kernel loses to the unfused chain (measured)
  if (a->d % 64 != 0 || ctx->force_dp4a || B < 1 || B > 8) return;
  // from umma_min_batch() queries up the tcgen05 proxy + stream selector win
  if (umma_min_batch() != 0 && B >= umma_min_batch(a->rows, ctx->num_sms) && umma_shape_ok(a, B)) return;
  const int64_t n = a->rows, K = sp.k_eff, n_rb = ceil_div(n, 16);
  f->nt = B <= 8 ? 1 : B <= 16 ? 2 : B <= 32 ? 4 : 8;
  f->ks = n_rb < 32LL * ctx->num_sms ? 2 : 1;
  int bps = 0;
  switch (f->nt) {
    case 1: bps = fsel_bps_ks<1>(f->ks, static_cast<int>(a->d), &f->smem); break;
    case 2: bps = fsel_bps_ks<2>(f->ks, static_cast<int>(a->d), &f->smem); break;
    case 4: bps = fsel_bps_ks<4>(f->ks, static_cast<int>(a->d), &f->smem); break;
    default: bps = fsel_bps_ks<8>(f->ks, static_cast<int>(a->d), &f->smem); break;
  }
  if (bps < 1) return;
  const int64_t resident = static_cast<int64_t>(bps) * ctx->num_sms;
  f->nbrk = static_cast<int>(std::min<int64_t>(B, 8));
  const int64_t rpc = 8 / f->ks;
  const int64_t G = std::min<int64_t>(resident - f->nbrk, ceil_div(n_rb, rpc));
  if (G < 1 || n > kFinMaxRows) return;
  // sample: round-0 row-blocks of every samp_step-th CTA (rpc * 16 keys each)
  const int64_t per = rpc * 16;
  const int64_t want = std::min<int64_t>(G, kFselSampleMax / per);
  f->samp_step = static_cast<int>(ceil_div(G, want));
  f->n_samp = static_cast<int>(std::min<int64_t>(ceil_div(G, f->samp_step) * per, std::min<int64_t>(n, kFselSampleMax)));
  // bracket: sample rank ~ mean + 4 sigma
  const double S = f->n_samp, pr = static_cast<double>(K) / static_cast<double>(n);
  const double mu = pr * S, sd = std::sqrt(S * pr * (1.0 - pr));
  f->r_lo = static_cast<int>(std::ceil(mu + 4.0 * sd + 1.0));
  if (f->r_lo > S / 2) return;
  const double listed = f->r_lo / S * static_cast<double>(n) + 4.0 * std::sqrt(static_cast<double>(f->r_lo) / S * n);
  if (listed > 0.9 * kFinCap) return;
  f->G = static_cast<int>(G);
  f->on = true;
}

template <int NT, int KS>
int launch_fsel_t(hire_ctx ctx, const hire_scorer_s* a, const ScoreWs& w, int64_t B, int phi, float* out,
                  const FselPlan& f, const FuseSel& fs) {
  CK(launch_k(ctx, q4_score_mma_sel<NT, KS>, f.G + f.nbrk, 256, f.smem, a->mma, a->rows, static_cast<int>(a->d), a->scales,
              w.xq, w.sx, w.sumxq, static_cast<int>(B), phi, out, a->rows, fs));
  return HIRE_OK;
}

struct TopkWs {
  ScoreWs sw;
  float* scores = nullptr;
  uint64_t* surv = nullptr;
  uint32_t* cand = nullptr;
  float* vals = nullptr;
  int* status = nullptr;
  FselPlan fz;
  uint64_t* fz_lists = nullptr;
};

void take_topk_ws(Arena& ar, TopkWs* t, const hire_scorer_s* a, int64_t B, const SelPlan& sp,
                  bool need_cand, hire_ctx ctx = nullptr, const hire_topk_params* p = nullptr) {
  take_score_ws(ar, &t->sw, a, B);
  ar.take(&t->scores, static_cast<size_t>(B * a->rows));
  if (ctx && p) plan_fsel(ctx, a, B, p, sp, &t->fz);
  if (t->fz.on) {
    ar.take(&t->fz_lists, static_cast<size_t>(B) * kFinCap);
  } else {
    ar.take(&t->surv, static_cast<size_t>(sp.surv_words(B)));
  }
  if (need_cand) ar.take(&t->cand, static_cast<size_t>(B * sp.k_eff));
  ar.take(&t->vals, static_cast<size_t>(B * sp.k_eff));
  ar.take(&t->status, 1);
}

// prep_x -> fused proxy/filter kernel -> sel_fin_kernel
// Everything after the proxy kernel in one launch (fsel_post_kernel): the
// finisher, the exact recompute and the final top-k + softmax.
struct FselPost {
  const hire_matrix_s* w = nullptr;  // non-null: use the post kernel
  int64_t k = 0;
  uint32_t* top_idx = nullptr;
  float* top_val = nullptr;
  float* top_prob = nullptr;
  int64_t out_stride = 0;
};

bool fsel_post_ok(const hire_matrix_s* w, const hire_topk_params* p, const SelPlan& sp, int64_t B, int num_sms) {
  // opt-in (HIRE_FSEL_POST=1): measured slower than fin -> K4 -> K5 on B200
  // (the recompute workers are latency-bound at 1024 threads / 64 registers)
#if !HIRE_EXPERIMENTS
  (void)w; (void)p; (void)sp; (void)B; (void)num_sms;
  return false;
#else
  const char* e = std::getenv("HIRE_FSEL_POST");
  if (!e || e[0] != '1' || p->strict) return false;
  const int64_t es = w->dtype == HIRE_BF16 ? 2 : 4;
  const int64_t bytes = w->d * es;
  if (bytes % 512 != 0) return false;
  const int64_t cpl = bytes / 512;
  if (cpl != 4 && cpl != 8 && cpl != 16) return false;
  if (p->k > kPostMaxK || sp.k_eff > kFinCap || w->d * 4 > 64 * 1024) return false;
  return B + 8 <= num_sms;
#endif
}

#if HIRE_EXPERIMENTS
template <typename T, int CPL>
int launch_post_t(hire_ctx ctx, const float* scores, int64_t stride, const FuseSel& fs, uint32_t* cand,
                  int64_t cand_stride, int ordered, int* status, const void* w, int d, const float* x, int phi,
                  float* vals, int kp, int K, const FselPost& po, unsigned* post, int B, int R, size_t smem) {
  auto k = fsel_post_kernel<T, CPL>;
  static size_t set = 0;
  if (smem > set) {
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    set = smem;
  }
  CK(launch_k(ctx, k, static_cast<unsigned>(B + R), kFinThreads, smem, scores, stride, fs, cand, cand_stride, ordered,
              status, static_cast<const T*>(w), d, x, phi, vals, kp, K, po.top_idx, po.top_val, po.top_prob,
              po.out_stride, post, R));
  return HIRE_OK;
}
#endif

int run_scores_fsel(hire_ctx ctx, const hire_scorer_s* a, const float* x, int64_t B, int phi, const SelPlan& sp,
                    const TopkWs& t, uint32_t* cand, bool ordered, const FselPost* po = nullptr) {
  const FselPlan& f = t.fz;
  const int d = static_cast<int>(a->d);
  RET(ensure_mma_layout(ctx, const_cast<hire_scorer_s*>(a)));
  // B <= 2: the proxy kernel quantises x itself (one launch fewer)
  const bool fold = B <= 2 && !std::getenv("HIRE_FSEL_NOFOLD");
  if (!fold) {
    StageScope pscope(ctx, kStagePrep);
    CK(launch_k(ctx, prep_x_int8_kernel, static_cast<unsigned>(B), 256, 0, x, d, t.sw.xq, t.sw.xperm, t.sw.sx,
                t.sw.sumxq, 0, static_cast<int>(B)));
  }
  FuseSel fs{};
  fs.xf = fold ? x : nullptr;
  fs.n = static_cast<uint32_t>(a->rows);
  fs.K = static_cast<uint32_t>(sp.k_eff);
  fs.g_stream = f.G;
  fs.nbrk = f.nbrk;
  fs.samp_step = f.samp_step;
  fs.n_samp = f.n_samp;
  fs.r_lo = f.r_lo;
  RET(ensure_fzero(ctx, B));  // dedicated zero-at-rest buffer (the arena is shared with other ops)
  fzero_layout(ctx, B, &fs);
  {
    const int64_t U = static_cast<int64_t>(f.G) * (8 / f.ks);
    const int64_t full = a->rows / 16 / U;  // complete rounds
    // static round-robin for every round by default; HIRE_FSEL_STATIC=k
    // claims the row-blocks after round k dynamically (measured: no gain —
    // the proxy stream is bandwidth-bound to the end)
    fs.n_static = 1 << 30;
    (void)full;
    if (const char* e = std::getenv("HIRE_FSEL_STATIC")) fs.n_static = std::max(1, std::atoi(e));
  }
  fs.lists = t.fz_lists;
  {
    StageScope scope(ctx, kStageProxy);
#define HIRE_FS(NT_)                                                                   \
    if (f.nt == NT_) {                                                                 \
      if (f.ks == 1) RET((launch_fsel_t<NT_, 1>(ctx, a, t.sw, B, phi, t.scores, f, fs))); \
      else RET((launch_fsel_t<NT_, 2>(ctx, a, t.sw, B, phi, t.scores, f, fs)));           \
    }
    HIRE_FS(1) else HIRE_FS(2) else HIRE_FS(4) else HIRE_FS(8)
#undef HIRE_FS
  }
  const size_t bm = static_cast<size_t>((a->rows + 31) / 32) * 4;
#if HIRE_EXPERIMENTS
  if (po && po->w) {
    StageScope scope(ctx, kStageSelect);
    const hire_matrix_s* w = po->w;
    const int dd = static_cast<int>(w->d);
    const int64_t kp = sp.k_eff;
    const int R = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ctx->num_sms - B, ceil_div(B * kp, 32))));
    const size_t smem = std::max(bm, static_cast<size_t>(dd) * 4);
    unsigned* post = fs.ctr + kFselCtr * 32;
    const int cpl = static_cast<int>(dd * (w->dtype == HIRE_BF16 ? 2 : 4) / 512);
    const int K = static_cast<int>(std::min<int64_t>(po->k, kp));
#define HIRE_PO(TT, C)                                                                                           \
    RET((launch_post_t<TT, C>(ctx, t.scores, a->rows, fs, cand, kp, ordered ? 1 : 0, t.status, w->ptr, dd, x, phi, \
                              t.vals, static_cast<int>(kp), K, *po, post, static_cast<int>(B), R, smem)))
    if (w->dtype == HIRE_BF16) {
      if (cpl == 4) HIRE_PO(__nv_bfloat16, 4); else if (cpl == 8) HIRE_PO(__nv_bfloat16, 8); else HIRE_PO(__nv_bfloat16, 16);
    } else {
      if (cpl == 4) HIRE_PO(float, 4); else if (cpl == 8) HIRE_PO(float, 8); else HIRE_PO(float, 16);
    }
#undef HIRE_PO
  } else
#endif
  {
    StageScope scope(ctx, kStageSelect);
    CK(launch_k(ctx, sel_fin_kernel, static_cast<unsigned>(B), kFinThreads, bm, static_cast<const float*>(t.scores),
                a->rows, fs, cand, sp.k_eff, ordered ? 1 : 0, ctx->counters + kFallbackOff));
  }
  CK(cudaGetLastError());
  return HIRE_OK;
}

// ordered: the candidate list is returned to the caller (ascending indices,
// hire.hpp:65-67); otherwise any order (recompute and final top-k do not care)
int local_candidates(hire_ctx ctx, const hire_matrix_s* w, const hire_scorer_s* a, const float* x,
                     int64_t B, const hire_topk_params* p, const SelPlan& sp, const TopkWs& t,
                     uint32_t* cand, bool ordered = true) {
  if (t.fz.on) {
    RET(run_scores_fsel(ctx, a, x, B, p->phi, sp, t, cand, ordered));
  } else {
    RET(run_scores(ctx, a, x, B, p->phi, p->x_mode, p->strict, t.sw, t.scores, a->rows));
    RET(run_select(ctx, t.scores, a->rows, a->rows, B, sp, t.surv, cand, sp.k_eff, t.status, ordered));
  }
  RET(run_recompute(ctx, w, cand, sp.k_eff, sp.k_eff, x, B, p->phi, p->strict, t.vals, sp.k_eff));
  return HIRE_OK;
}

}  // namespace

namespace {
// ------------------------------------------------------- host-call graphs --
// body(stream) issues the whole host call (copies + kernels) on ctx->stream
// and fills out[4]. First call per key: eager. Second: captured on gstream,
// instantiated, launched. Later: launched. The caller synchronises.
// *done_on = the stream the caller synchronises on.
template <class Body>
int run_host_graph(hire_ctx ctx, const std::vector<int64_t>& key, int64_t* out, cudaStream_t* done_on,
                   const void* fetch_src, Body body) {
  *done_on = ctx->stream;
  if (!ctx->host_graphs || ctx->prof) return body(out);
  const auto bufs = ctx->buf_snapshot();
  for (size_t gi = 0; gi < ctx->hgraphs.size(); ++gi)
    if (ctx->hgraphs[gi].key == key && ctx->hgraphs[gi].bufs == bufs) {
      if (gi + 1 != ctx->hgraphs.size())  // most recently used goes last
        std::rotate(ctx->hgraphs.begin() + static_cast<long>(gi), ctx->hgraphs.begin() + static_cast<long>(gi) + 1,
                    ctx->hgraphs.end());
      auto& g = ctx->hgraphs.back();
      // order after earlier work on the context stream only if there is any
      if (cudaStreamQuery(ctx->stream) != cudaSuccess) {
        cudaGetLastError();
        CK(cudaEventRecord(ctx->gev, ctx->stream));
        CK(cudaStreamWaitEvent(ctx->gstream, ctx->gev, 0));
      }
      // this call's input buffer (read by the fetch kernel through the slot);
      // without a device address for it the call runs eagerly
      if (g.uses_slot) {
        if (!fetch_src) return body(out);
        store_fetch_slot(ctx, fetch_src);
      }
      CK(cudaGraphLaunch(g.exec, ctx->gstream));
      *done_on = ctx->gstream;  // the host call blocks on it: no event back
      for (int i = 0; i < 4; ++i) out[i] = g.out[i];
      return HIRE_OK;
    }
  bool seen = false;
  for (auto& k : ctx->hseen) seen |= k == key;
  if (!seen) {  // eager first call: allocations, lazy layouts, static state
    if (ctx->hseen.size() >= hire_ctx_s::kMaxHostGraphs * 4) ctx->hseen.erase(ctx->hseen.begin());
    ctx->hseen.push_back(key);
    return body(out);
  }
  if (!ctx->gstream) {
    CK(cudaStreamCreateWithFlags(&ctx->gstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ctx->gev, cudaEventDisableTiming));
  }
  // drop stale entries of this key (a buffer moved)
  for (size_t i = 0; i < ctx->hgraphs.size();)
    if (ctx->hgraphs[i].key == key) {
      cudaGraphExecDestroy(ctx->hgraphs[i].exec);
      ctx->hgraphs.erase(ctx->hgraphs.begin() + static_cast<long>(i));
    } else {
      ++i;
    }
  CK(cudaStreamSynchronize(ctx->stream));
  cudaStream_t user = ctx->stream;
  ctx->stream = ctx->gstream;
  CK(cudaStreamBeginCapture(ctx->gstream, cudaStreamCaptureModeThreadLocal));
  const int64_t launches0 = ctx->launches;
  ctx->fetch_by_slot = false;
  const int rc = body(out);
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(ctx->gstream, &graph);
  ctx->stream = user;
  ctx->launches = launches0;
  if (rc != HIRE_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ec != cudaSuccess || ctx->buf_snapshot() != bufs) {  // not capturable as is: stay eager
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    ctx->host_graphs = ec == cudaSuccess;
    return body(out);
  }
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  CK(ei);
  if (ctx->hgraphs.size() >= hire_ctx_s::kMaxHostGraphs) {  // bounded: evict the least recently used
    cudaGraphExecDestroy(ctx->hgraphs.front().exec);
    ctx->hgraphs.erase(ctx->hgraphs.begin());
  }
  ctx->hgraphs.push_back({key, bufs, exec, {out[0], out[1], out[2], out[3]}, ctx->fetch_by_slot});
  CK(cudaGraphLaunch(exec, ctx->gstream));
  *done_on = ctx->gstream;
  return HIRE_OK;
}
}  // namespace

// ====================================================================== ABI
extern "C" {

const char* hire_last_error(void) { return g_err.c_str(); }
int hire_abi_version(void) { return HIRE_ABI_VERSION; }
int hire_experiments_built(void) { return HIRE_EXPERIMENTS; }
#if HIRE_EXPERIMENTS
static_assert(kQcntOff >= hire_dev::kCntInts, "context counters overlap the fused FFN barriers");
#endif

int hire_ctx_create(int device, void* stream, int own_stream, hire_ctx* out) {
  if (!out) return invalid("null out");
  CK(cudaSetDevice(device));
  auto* c = new hire_ctx_s();
  c->device = device;
  if (!own_stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      return set_err(HIRE_ERR_RUNTIME, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
    }
    c->own_stream = true;
  }
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  // opt-in shared memory for the selectors
  CK(cudaFuncSetAttribute(select_candidates_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kPoolKeys * 8));
#if HIRE_EXPERIMENTS
  for (const void* kf : {(const void*)sel_cluster_kernel<256, 4>, (const void*)sel_cluster_kernel<256, 8>,
                         (const void*)sel_cluster_kernel<256, 16>, (const void*)sel_cluster_kernel<512, 16>,
                         (const void*)sel_cluster_kernel<512, 32>})
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
#endif
  {
    const int f2 = kFinalMax * 8;
    CK(cudaFuncSetAttribute(final2_kernel<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<128, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<128, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<128, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<256, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<256, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<512, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
    CK(cudaFuncSetAttribute(final2_kernel<1024, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, f2));
  }
  CK(cudaFuncSetAttribute(final_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kFinalMax * 8));
  CK(cudaFuncSetAttribute(sel_fin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFinMaxRows / 8));
#if HIRE_EXPERIMENTS
  CK(cudaFuncSetAttribute(sel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemRowMax * 4));
#endif
  CK(cudaFuncSetAttribute(bucket_topt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          kBucketMaxWidth * 8));
  // every other kernel with dynamic shared memory: allow up to 200 KB once,
  // here, so no attribute call ever happens inside a captured graph
  {
    const int mx = 200 * 1024;
    const void* ks[] = {
        (const void*)q4_score_seq,
        (const void*)recompute_fast<float, 1>, (const void*)recompute_fast<float, 2>,
        (const void*)recompute_fast<float, 4>, (const void*)recompute_fast<float, 8>,
        (const void*)recompute_fast<float, 16>, (const void*)recompute_fast<__nv_bfloat16, 1>,
        (const void*)recompute_fast<__nv_bfloat16, 2>, (const void*)recompute_fast<__nv_bfloat16, 4>,
        (const void*)recompute_fast<__nv_bfloat16, 8>, (const void*)recompute_fast<__nv_bfloat16, 16>,
        (const void*)recompute_seq<float>, (const void*)recompute_seq<__nv_bfloat16>,
        (const void*)lr_score_kernel<float, 64, true>, (const void*)lr_score_kernel<float, 64, false>,
        (const void*)lr_score_kernel<__nv_bfloat16, 64, true>,
        (const void*)lr_score_kernel<__nv_bfloat16, 64, false>,
        (const void*)lr_score_generic<float, true>, (const void*)lr_score_generic<float, false>,
        (const void*)lr_score_generic<__nv_bfloat16, true>,
        (const void*)lr_score_generic<__nv_bfloat16, false>};
    for (const void* k : ks) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    CK(cudaFuncSetAttribute(q4_score_umma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  }
  if (const char* e = getenv("HIRE_PROXY_KERNEL")) c->force_dp4a = std::strcmp(e, "dp4a") == 0;
  if (const char* e = getenv("HIRE_FFN_FUSED")) c->ffn_fused = std::strcmp(e, "1") == 0;
  if (const char* e = getenv("HIRE_FUSED_TRACE")) c->trace = std::strcmp(e, "1") == 0;
  {
    void* hp = nullptr;
    void* dp = nullptr;
    if (cudaHostAlloc(&hp, kFetchCtas * kFetchSlotStride * 8, cudaHostAllocMapped | cudaHostAllocPortable) == cudaSuccess &&
        cudaHostGetDevicePointer(&dp, hp, 0) == cudaSuccess && dp) {
      c->fetch_slot = static_cast<unsigned long long*>(hp);
      c->fetch_slot_dev = static_cast<unsigned long long*>(dp);
      std::memset(hp, 0, kFetchCtas * kFetchSlotStride * 8);
    } else {  // no mapped memory: host calls stage their inputs with a copy
      if (hp) cudaFreeHost(hp);
      cudaGetLastError();
    }
  }
  CK(cudaMalloc(&c->counters, kCtxCounterInts * sizeof(int)));
  CK(cudaMemset(c->counters, 0, kCtxCounterInts * sizeof(int)));
  if (const char* e = getenv("HIRE_NO_PDL")) c->pdl = std::strcmp(e, "1") != 0;
  if (const char* e = getenv("HIRE_HOST_GRAPHS")) c->host_graphs = std::strcmp(e, "0") != 0;
  *out = c;
  return HIRE_OK;
}

int hire_ctx_destroy(hire_ctx c) {
  if (!c) return HIRE_OK;
  cudaStreamSynchronize(c->stream);
  if (c->ws) cudaFree(c->ws);
  if (c->counters) cudaFree(c->counters);
  if (c->selc) cudaFree(c->selc);
  if (c->tickets) cudaFree(c->tickets);
  if (c->fzero) cudaFree(c->fzero);
  if (c->umask) cudaFree(c->umask);
  if (c->upart) cudaFree(c->upart);
  if (c->io_dev) cudaFree(c->io_dev);
  if (c->io_host) cudaFreeHost(c->io_host);
  if (c->fetch_slot) cudaFreeHost(c->fetch_slot);
  for (auto& g : c->hgraphs) cudaGraphExecDestroy(g.exec);
  if (c->gstream) cudaStreamDestroy(c->gstream);
  if (c->gev) cudaEventDestroy(c->gev);
  for (auto& m : c->marks) { cudaEventDestroy(m.second.first); cudaEventDestroy(m.second.second); }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return HIRE_OK;
}

int hire_ctx_stream(hire_ctx c, void** s) {
  if (!c || !s) return invalid("null handle");
  *s = c->stream;
  return HIRE_OK;
}

int hire_ctx_synchronize(hire_ctx c) {
  if (!c) return invalid("null handle");
  CK(cudaStreamSynchronize(c->stream));
  return HIRE_OK;
}

int64_t hire_ctx_launch_count(hire_ctx c) { return c ? c->launches : 0; }

int hire_ctx_read_trace(hire_ctx c, long long* out, int n) {
  if (!c || !out || n > 64) return invalid("bad trace request");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(out, c->counters + kTraceOff, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
  return HIRE_OK;
}

int hire_ctx_select_fallbacks(hire_ctx c, long long* count) {
  if (!c || !count) return invalid("null argument");
  CK(cudaStreamSynchronize(c->stream));
  int v = 0;
  CK(cudaMemcpy(&v, c->counters + kFallbackOff, sizeof(int), cudaMemcpyDeviceToHost));
  *count = v;
  return HIRE_OK;
}

int hire_debug_ktrace(hire_ctx c, int op, unsigned long long* out, int n) {
  // op 1: enable + reset, 2: read n (<= 96) words, 0: disable
  if (!c) return invalid("null handle");
  static unsigned long long* buf = nullptr;
  constexpr int kWords = 2 * hire_dev::kKtNum + 32;  // + 32 ad hoc probe words (g_ktrace[64..95])
  CK(cudaStreamSynchronize(c->stream));
  if (op == 1) {
    if (!buf) CK(cudaMalloc(&buf, kWords * sizeof(unsigned long long)));
    unsigned long long init[kWords];
    for (int i = 0; i < kWords; ++i) init[i] = (((i & 1) || i >= 24) && i != 54 && i != 83) ? 0ull : ~0ull;
    CK(cudaMemcpy(buf, init, sizeof(init), cudaMemcpyHostToDevice));
    CK(cudaMemcpyToSymbol(hire_dev::g_ktrace, &buf, sizeof(buf)));
  } else if (op == 2) {
    if (!buf || !out || n > kWords) return invalid("ktrace not enabled / bad size");
    CK(cudaMemcpy(out, buf, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost));
  } else {
    unsigned long long* z = nullptr;
    CK(cudaMemcpyToSymbol(hire_dev::g_ktrace, &z, sizeof(z)));
  }
  return HIRE_OK;
}

int hire_ctx_set_profiling(hire_ctx c, int on) {
  if (!c) return invalid("null handle");
  c->prof = on != 0;
  return HIRE_OK;
}

int hire_ctx_profile_read(hire_ctx c, double* ms, int64_t* counts, int n_stages) {
  if (!c || !ms || !counts) return invalid("null argument");
  CK(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < n_stages; ++i) { ms[i] = 0.0; counts[i] = 0; }
  cudaError_t err = cudaSuccess;
  for (auto& m : c->marks) {
    float t = 0.0f;
    const cudaError_t e = cudaEventElapsedTime(&t, m.second.first, m.second.second);
    if (e != cudaSuccess) err = e;
    else if (m.first < n_stages) { ms[m.first] += t; counts[m.first] += 1; }
    c->ev_pool.push_back(m.second.first);
    c->ev_pool.push_back(m.second.second);
  }
  c->marks.clear();
  if (err != cudaSuccess) {
    cudaGetLastError();
    return set_err(HIRE_ERR_RUNTIME, std::string("cudaEventElapsedTime: ") + cudaGetErrorString(err));
  }
  return HIRE_OK;
}

// ------------------------------------------------------- device buffers --
int hire_device_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return invalid("bad allocation request");
  *out = nullptr;
  if (bytes == 0) return HIRE_OK;
  CK(cudaMalloc(out, static_cast<size_t>(bytes)));
  return HIRE_OK;
}

int hire_device_free(void* p) {
  if (p) CK(cudaFree(p));
  return HIRE_OK;
}

int hire_copy(hire_ctx ctx, void* dst, const void* src, int64_t bytes, int kind, int sync) {
  if (!ctx || (!dst && bytes) || (!src && bytes) || bytes < 0) return invalid("bad copy request");
  if (bytes == 0) return HIRE_OK;
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                     : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  CK(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), k, ctx->stream));
  if (sync) CK(cudaStreamSynchronize(ctx->stream));
  return HIRE_OK;
}

// ------------------------------------------------------------- matrices --
int hire_matrix_create(const void* src, int64_t rows, int64_t d, int dtype, int src_on_device,
                       hire_matrix* out) {
  if (!out || !src) return invalid("null argument");
  if (rows < 1 || d < 1) return invalid("ScoreMatrix: rows must be >= 1");
  if (dtype != HIRE_F32 && dtype != HIRE_BF16) return invalid("unknown dtype");
  auto* m = new hire_matrix_s();
  m->rows = rows;
  m->d = d;
  m->dtype = dtype;
  m->owned = true;
  const size_t bytes = static_cast<size_t>(rows) * d * dtype_size(dtype);
  cudaError_t e = cudaMalloc(&m->ptr, bytes);
  if (e == cudaSuccess)
    e = cudaMemcpy(m->ptr, src, bytes, src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    if (m->ptr) cudaFree(m->ptr);
    delete m;
    return set_err(HIRE_ERR_RUNTIME, std::string("hire_matrix_create: ") + cudaGetErrorString(e));
  }
  *out = m;
  return HIRE_OK;
}

int hire_matrix_view(void* ptr, int64_t rows, int64_t d, int dtype, hire_matrix* out) {
  if (!out || !ptr) return invalid("null argument");
  if (rows < 1 || d < 1) return invalid("ScoreMatrix: rows must be >= 1");
  if (dtype != HIRE_F32 && dtype != HIRE_BF16) return invalid("unknown dtype");
  auto* m = new hire_matrix_s();
  m->ptr = ptr;
  m->rows = rows;
  m->d = d;
  m->dtype = dtype;
  m->owned = false;
  *out = m;
  return HIRE_OK;
}

int hire_matrix_slice(hire_matrix m, int64_t first, int64_t count, hire_matrix* out) {
  if (!m || !out) return invalid("null argument");
  if (first < 0 || count < 1 || first + count > m->rows) return invalid("ScoreMatrix::slice_cols: out of range");
  return hire_matrix_view(static_cast<char*>(m->ptr) + first * m->d * dtype_size(m->dtype), count, m->d,
                          m->dtype, out);
}

int hire_matrix_destroy(hire_matrix m) {
  if (!m) return HIRE_OK;
  if (m->owned && m->ptr) cudaFree(m->ptr);
  delete m;
  return HIRE_OK;
}

int hire_matrix_info(hire_matrix m, int64_t* rows, int64_t* d, int* dtype) {
  if (!m) return invalid("null handle");
  if (rows) *rows = m->rows;
  if (d) *d = m->d;
  if (dtype) *dtype = m->dtype;
  return HIRE_OK;
}

// -------------------------------------------------------------- scorers --
static int64_t q4_pitch(int64_t d) { return (((d + 1) / 2) + 15) / 16 * 16; }

static int make_q4(const std::vector<uint8_t>& packed_rows, const float* scales, int64_t rows,
                   int64_t d, hire_scorer* out) {
  auto* a = new hire_scorer_s();
  a->kind = HIRE_SCORER_Q4;
  a->rows = rows;
  a->d = d;
  a->pitch = q4_pitch(d);
  a->owned = true;
  cudaError_t e = cudaMalloc(&a->codes, static_cast<size_t>(rows) * a->pitch);
  if (e == cudaSuccess) e = cudaMalloc(&a->scales, static_cast<size_t>(rows) * 4);
  if (e == cudaSuccess) e = cudaMemcpy(a->codes, packed_rows.data(), packed_rows.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(a->scales, scales, static_cast<size_t>(rows) * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(a->codes);
    cudaFree(a->scales);
    delete a;
    return set_err(HIRE_ERR_RUNTIME, std::string("q4 upload: ") + cudaGetErrorString(e));
  }
  if (d % 64 == 0) {
    hire_ctx_s tmp;
    tmp.stream = nullptr;
    tmp.pdl = false;
    const int rc = ensure_mma_layout(&tmp, a);
    if (rc == HIRE_OK) CK(cudaStreamSynchronize(nullptr));
    if (rc != HIRE_OK) { hire_scorer_destroy(a); return rc; }
  }
  *out = a;
  return HIRE_OK;
}

int hire_scorer_create_q4_codes(const int8_t* codes, const float* scales, int64_t rows, int64_t d,
                                hire_scorer* out) {
  if (!codes || !scales || !out) return invalid("null argument");
  if (rows < 1 || d < 1) return invalid("quantized matrix: dims must be positive");
  const int64_t pitch = q4_pitch(d);
  std::vector<uint8_t> buf(static_cast<size_t>(rows * pitch), 0);
  for (int64_t j = 0; j < rows; ++j)
    for (int64_t i = 0; i < d; ++i) {
      const int8_t c = codes[j * d + i];
      if (c < -7 || c > 7) return invalid("quantized matrix: code outside [-7, 7]");
      const uint8_t nib = static_cast<uint8_t>(c) & 0x0F;
      buf[j * pitch + i / 2] |= (i & 1) ? static_cast<uint8_t>(nib << 4) : nib;
    }
  return make_q4(buf, scales, rows, d, out);
}

int hire_scorer_create_q4_hirq(const uint8_t* payload, const float* scales, int64_t rows, int64_t d,
                               hire_scorer* out) {
  if (!payload || !scales || !out) return invalid("null argument");
  if (rows < 1 || d < 1) return invalid("quantized matrix: dims must be positive");
  const int64_t pitch = q4_pitch(d);
  std::vector<uint8_t> buf(static_cast<size_t>(rows * pitch), 0);
  if (d % 2 == 0) {
    for (int64_t j = 0; j < rows; ++j) std::memcpy(&buf[j * pitch], payload + j * (d / 2), d / 2);
  } else {
    for (int64_t j = 0; j < rows; ++j)
      for (int64_t i = 0; i < d; ++i) {
        const int64_t s = j * d + i;  // continuous HIRQ stream position
        const uint8_t nib = (s & 1) ? (payload[s / 2] >> 4) : (payload[s / 2] & 0x0F);
        buf[j * pitch + i / 2] |= (i & 1) ? static_cast<uint8_t>(nib << 4) : nib;
      }
  }
  return make_q4(buf, scales, rows, d, out);
}

int hire_scorer_quantize(hire_ctx ctx, hire_matrix w, hire_scorer* out) {
  if (!ctx || !w || !out) return invalid("null argument");
  auto* a = new hire_scorer_s();
  a->kind = HIRE_SCORER_Q4;
  a->rows = w->rows;
  a->d = w->d;
  a->pitch = q4_pitch(w->d);
  a->owned = true;
  cudaError_t e = cudaMalloc(&a->codes, static_cast<size_t>(a->rows) * a->pitch);
  if (e == cudaSuccess) e = cudaMalloc(&a->scales, static_cast<size_t>(a->rows) * 4);
  if (e != cudaSuccess) {
    cudaFree(a->codes);
    delete a;
    return set_err(HIRE_ERR_RUNTIME, std::string("hire_scorer_quantize: ") + cudaGetErrorString(e));
  }
  const unsigned grid = static_cast<unsigned>(ceil_div(w->rows * 32, 256));
  if (w->dtype == HIRE_BF16)
    CK(launch_k(ctx, quantize_q4_kernel<__nv_bfloat16>, grid, 256, 0, static_cast<const __nv_bfloat16*>(w->ptr), w->rows, static_cast<int>(w->d), a->codes, a->pitch, a->scales));
  else
    CK(launch_k(ctx, quantize_q4_kernel<float>, grid, 256, 0, static_cast<const float*>(w->ptr), w->rows, static_cast<int>(w->d), a->codes, a->pitch, a->scales));
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFree(a->codes);
    cudaFree(a->scales);
    delete a;
    return set_err(HIRE_ERR_RUNTIME, std::string("quantize_q4_kernel: ") + cudaGetErrorString(e));
  }
  if (a->d % 64 == 0) {
    const int rc = ensure_mma_layout(ctx, a);
    if (rc != HIRE_OK) { hire_scorer_destroy(a); return rc; }
  }
  *out = a;
  return HIRE_OK;
}

int hire_scorer_create_lowrank(const void* z1, const void* z2, int64_t d, int64_t rows, int64_t r,
                               int dtype, int src_on_device, hire_scorer* out) {
  if (!z1 || !z2 || !out) return invalid("null argument");
  if (d < 1 || rows < 1 || r < 1) return invalid("ApproxScorer: low-rank factors do not match rank " + std::to_string(r));
  if (dtype != HIRE_F32 && dtype != HIRE_BF16) return invalid("unknown dtype");
  auto* a = new hire_scorer_s();
  a->kind = HIRE_SCORER_LOWRANK;
  a->rows = rows;
  a->d = d;
  a->r = r;
  a->dtype = dtype;
  a->owned = true;
  const size_t es = dtype_size(dtype);
  const auto kind = src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaError_t e = cudaMalloc(&a->z1, static_cast<size_t>(r) * d * es);
  if (e == cudaSuccess) e = cudaMalloc(&a->z2, static_cast<size_t>(rows) * r * es);
  if (e == cudaSuccess) e = cudaMemcpy(a->z1, z1, static_cast<size_t>(r) * d * es, kind);
  if (e == cudaSuccess) e = cudaMemcpy(a->z2, z2, static_cast<size_t>(rows) * r * es, kind);
  if (e != cudaSuccess) {
    cudaFree(a->z1);
    cudaFree(a->z2);
    delete a;
    return set_err(HIRE_ERR_RUNTIME, std::string("low-rank upload: ") + cudaGetErrorString(e));
  }
  *out = a;
  return HIRE_OK;
}

int hire_scorer_slice(hire_scorer a, int64_t first, int64_t count, hire_scorer* out) {
  if (!a || !out) return invalid("null argument");
  if (first < 0 || count < 1 || first + count > a->rows) return invalid("ApproxScorer::slice_cols: out of range");
  auto* s = new hire_scorer_s(*a);
  s->uid = next_uid();
  s->owned = false;
  s->rows = count;
  s->mma = nullptr;
  s->mma_owned = false;
  if (a->kind == HIRE_SCORER_Q4) {
    s->codes = a->codes + first * a->pitch;
    s->scales = a->scales + first;
    if (a->mma && first % 16 == 0) s->mma = a->mma + (first / 16) * (a->d / 64) * 32;
    s->umma = nullptr;
    s->umma_owned = false;
    s->umap_ok = false;
    if (a->umma && first % kUmmaRows == 0) s->umma = a->umma + (first / kUmmaRows) * (a->d / 32) * 512;
  } else {
    s->z2 = static_cast<char*>(a->z2) + first * a->r * dtype_size(a->dtype);
  }
  *out = s;
  return HIRE_OK;
}

int hire_scorer_export_q4(hire_scorer a, int8_t* codes, float* scales) {
  if (!a || !codes || !scales) return invalid("null argument");
  if (a->kind != HIRE_SCORER_Q4) return invalid("not an int4 scorer");
  std::vector<uint8_t> buf(static_cast<size_t>(a->rows * a->pitch));
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(buf.data(), a->codes, buf.size(), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(scales, a->scales, static_cast<size_t>(a->rows) * 4, cudaMemcpyDeviceToHost));
  for (int64_t j = 0; j < a->rows; ++j)
    for (int64_t i = 0; i < a->d; ++i) {
      const uint8_t b = buf[j * a->pitch + i / 2];
      const uint8_t nib = (i & 1) ? (b >> 4) : (b & 0x0F);
      codes[j * a->d + i] = static_cast<int8_t>((nib & 0x08) ? (nib | 0xF0) : nib);
    }
  return HIRE_OK;
}

int hire_scorer_info(hire_scorer a, int* kind, int64_t* rows, int64_t* d, int64_t* rank) {
  if (!a) return invalid("null handle");
  if (kind) *kind = a->kind;
  if (rows) *rows = a->rows;
  if (d) *d = a->d;
  if (rank) *rank = a->r;
  return HIRE_OK;
}

int hire_scorer_destroy(hire_scorer a) {
  if (!a) return HIRE_OK;
  if (a->owned) {
    cudaFree(a->codes);
    cudaFree(a->scales);
    cudaFree(a->z1);
    cudaFree(a->z2);
  }
  if (a->mma_owned) cudaFree(a->mma);
  if (a->umma_owned) cudaFree(a->umma);
  delete a;
  return HIRE_OK;
}

// ----------------------------------------------------------- primitives --
int hire_scores(hire_ctx ctx, hire_scorer a, const float* x, int64_t B, int phi, int x_mode,
                int strict, float* out) {
  if (!ctx || !a || !x || !out) return invalid("null argument");
  if (B < 1) return invalid("batch must be >= 1");
  RET(check_phi(phi));
  if (x_mode == HIRE_X_INT8 && a->kind != HIRE_SCORER_Q4) return invalid("x_mode int8 needs an int4 proxy");
  Arena ar;
  ScoreWs w;
  take_score_ws(ar, &w, a, B);
  RET(ar.commit(ctx));
  return run_scores(ctx, a, x, B, phi, x_mode, strict, w, out, a->rows);
}

int hire_matvec(hire_ctx ctx, hire_matrix w, const float* x, int64_t B, int phi, int strict, float* out) {
  if (!ctx || !w || !x || !out) return invalid("null argument");
  RET(check_phi(phi));
  return run_recompute(ctx, w, nullptr, 0, w->rows, x, B, phi, strict, out, w->rows);
}

int hire_topk_select(hire_ctx ctx, const float* v, int64_t B, int64_t n, int64_t k, uint32_t* idx,
                     float* val, int* clamped) {
  if (!ctx || !v || !idx || !val) return invalid("null argument");
  if (k < 1) return invalid("topk_select: k must be >= 1");
  SelPlan sp;
  RET(plan_select(n, k, HIRE_SELECT_EXACT, 0, 0, &sp));
  Arena ar;
  uint64_t* surv;
  uint32_t* cand;
  int* status;
  float* cv;
  ar.take(&surv, static_cast<size_t>(sp.surv_words(B)));
  ar.take(&cand, static_cast<size_t>(B * sp.k_eff));
  ar.take(&status, 1);
  ar.take(&cv, static_cast<size_t>(B * sp.k_eff));
  RET(ar.commit(ctx));
  RET(run_select(ctx, v, n, n, B, sp, surv, cand, sp.k_eff, status));
  CK(launch_k(ctx, gather_values_kernel, static_cast<unsigned>(ceil_div(B * sp.k_eff, 256)), 256, 0, v, n, cand, sp.k_eff, B, cv));
  CK(cudaGetLastError());
  RET(run_final(ctx, cv, sp.k_eff, cand, sp.k_eff, nullptr, 0, 0, sp.k_eff, sp.k_eff, B, 0, idx, val,
                nullptr, nullptr, sp.k_eff));
  if (clamped) *clamped = sp.clamped;
  return HIRE_OK;
}


// ------------------------------------------------------------ hire_topk --
int hire_topk_run(hire_ctx ctx, hire_matrix w, hire_scorer a, const float* x, int64_t B,
                  const hire_topk_params* p, uint32_t* cand, uint32_t* top_idx, float* top_val,
                  float* top_prob, int64_t* n_cand, int64_t* n_top, int* clamped) {
  if (!ctx || !x || !top_idx || !top_val) return invalid("null argument");
  RET(validate_topk(w, a, B, p));
  if (top_prob && p->phi != HIRE_PHI_IDENTITY) return invalid("softmax_topk: phi must be identity");
  SelPlan sp;
  RET(plan_select(w->rows, p->k_prime, p->select, p->n_buckets, p->bucket_t, &sp));
  Arena ar;
  TopkWs t;
  take_topk_ws(ar, &t, a, B, sp, true, ctx, p);
  RET(ar.commit(ctx));
  const int64_t take = std::min<int64_t>(p->k, sp.k_eff);
  if (t.fz.on && fsel_post_ok(w, p, sp, B, ctx->num_sms)) {
    // one launch after the proxy kernel: finisher + recompute + final top-k
    FselPost po;
    po.w = w;
    po.k = p->k;
    po.top_idx = top_idx;
    po.top_val = top_val;
    po.top_prob = top_prob;
    po.out_stride = p->k;
    RET(run_scores_fsel(ctx, a, x, B, p->phi, sp, t, t.cand, cand != nullptr, &po));
  } else {
    RET(local_candidates(ctx, w, a, x, B, p, sp, t, t.cand, cand != nullptr));
    RET(run_final(ctx, t.vals, sp.k_eff, t.cand, sp.k_eff, nullptr, 0, 0, sp.k_eff, take, B, 0, top_idx,
                  top_val, top_prob, nullptr, p->k));
  }
  if (cand) CK(cudaMemcpy2DAsync(cand, p->k_prime * 4, t.cand, sp.k_eff * 4, sp.k_eff * 4, B,
                                 cudaMemcpyDefault, ctx->stream));
  if (n_cand) *n_cand = sp.k_eff;
  if (n_top) *n_top = take;
  if (clamped) *clamped = sp.clamped || take < p->k;
  return HIRE_OK;
}

int hire_topk_host(hire_ctx ctx, hire_matrix w, hire_scorer a, const float* x_host, int64_t B,
                   const hire_topk_params* p, uint32_t* cand_host, uint32_t* top_idx_host,
                   float* top_val_host, float* top_prob_host, int64_t* n_cand, int64_t* n_top,
                   int* clamped) {
  if (!ctx || !x_host || !top_idx_host || !top_val_host) return invalid("null argument");
  bind_thread(ctx);
  RET(validate_topk(w, a, B, p));
  SelPlan sp;
  RET(plan_select(w->rows, p->k_prime, p->select, p->n_buckets, p->bucket_t, &sp));
  const int64_t take = std::min<int64_t>(p->k, sp.k_eff);
  const size_t xb = static_cast<size_t>(B * w->d) * 4;
  const size_t cb = cand_host ? static_cast<size_t>(B * p->k_prime) * 4 : 0;
  const size_t tb = static_cast<size_t>(B * p->k) * 4;
  const size_t pb = top_prob_host ? tb : 0;
  const size_t in_bytes = align_up(xb);
  const size_t out_bytes = align_up(cb) + align_up(tb) * 2 + align_up(pb);
  RET(ensure(&ctx->io_dev, &ctx->io_dev_cap, in_bytes + out_bytes, ctx->stream));
  RET(ensure_host(&ctx->io_host, &ctx->io_host_cap, in_bytes + out_bytes, ctx->stream));
  char* dv = static_cast<char*>(ctx->io_dev);
  char* hs = static_cast<char*>(ctx->io_host);
  // the input: read in place when the caller's buffer is pinned (the graph's
  // fetch node is pointed at it per call), else staged into the context's
  // mapped buffer; results are written into the mapped buffer and copied
  // out after the synchronise
  const void* xa = host_alias(x_host, xb);
  if (!xa) std::memcpy(hs, x_host, xb);
  const void* xsrc = xa ? static_cast<const void*>(x_host) : hs;
  const void* xdev = xa ? xa : host_alias(hs, align_up(xb));
  const std::vector<int64_t> key = {1, static_cast<int64_t>(w->uid), static_cast<int64_t>(a->uid), B, p->k, p->k_prime,
                                    p->phi, p->x_mode, p->select, p->strict, p->n_buckets, p->bucket_t,
                                    cb ? 1 : 0, pb ? 1 : 0};
  int64_t res[4];
  cudaStream_t done_on = nullptr;
  RET(run_host_graph(ctx, key, res, &done_on, xdev, [&](int64_t* r) -> int {
    RET(fetch_inputs(ctx, dv, xsrc, xb));
    // results are written straight into mapped host memory (through its device alias)
    char* o = hs + in_bytes;  // results are written straight into mapped host memory
    uint32_t* dcand = cb ? reinterpret_cast<uint32_t*>(o) : nullptr;
    o += align_up(cb);
    uint32_t* didx = reinterpret_cast<uint32_t*>(o);
    o += align_up(tb);
    float* dval = reinterpret_cast<float*>(o);
    o += align_up(tb);
    float* dprob = pb ? reinterpret_cast<float*>(o) : nullptr;
    int cl = 0;
    RET(hire_topk_run(ctx, w, a, reinterpret_cast<const float*>(dv), B, p, dcand, didx, dval, dprob, &r[0], &r[1],
                      &cl));
    r[2] = cl;
    return HIRE_OK;
  }));
  if (n_cand) *n_cand = res[0];
  if (n_top) *n_top = res[1];
  if (clamped) *clamped = static_cast<int>(res[2]);
  CK(cudaStreamSynchronize(done_on));
  const char* ho = hs + in_bytes;
  (void)take;
  if (cb) std::memcpy(cand_host, ho, cb);
  ho += align_up(cb);
  std::memcpy(top_idx_host, ho, tb);
  ho += align_up(tb);
  std::memcpy(top_val_host, ho, tb);
  ho += align_up(tb);
  if (pb) std::memcpy(top_prob_host, ho, pb);
  return HIRE_OK;
}

// ------------------------------------------------------------------ FFN --
namespace {
int validate_ffn(const hire_matrix_s* u, const hire_matrix_s* v, const hire_scorer_s* a, int64_t B,
                 const hire_ffn_params* p) {
  if (!u || !v || !a || !p) return invalid("null handle");
  if (u->rows != v->rows || u->d != v->d) return invalid("GroupedFFN: U and V must both be d x m");
  const int64_t g = p->group_size, m = u->rows;
  if (g < 1) return invalid("GroupedFFN: group size must be >= 1");
  if (m % g != 0) return invalid("GroupedFFN: g = " + std::to_string(g) + " must divide m = " + std::to_string(m));
  if (p->k < 1 || p->k % g != 0) return invalid("ffn_group_sparse: g = " + std::to_string(g) + " must divide k = " + std::to_string(p->k));
  if (p->k_prime % g != 0) return invalid("ffn_group_sparse: g = " + std::to_string(g) + " must divide k_prime = " + std::to_string(p->k_prime));
  if (p->k > p->k_prime || p->k_prime > m)
    return invalid("ffn_group_sparse: need k <= k_prime <= m, got k = " + std::to_string(p->k) +
                   ", k_prime = " + std::to_string(p->k_prime) + ", m = " + std::to_string(m));
  if (a->rows != m || a->d != u->d)
    return invalid("group_proxy: scorer covers " + std::to_string(a->rows) + " units but FFN has " + std::to_string(m));
  RET(check_phi(p->phi));
  if (B < 1) return invalid("batch must be >= 1");
  if (p->x_mode == HIRE_X_INT8 && a->kind != HIRE_SCORER_Q4) return invalid("x_mode int8 needs an int4 proxy");
  return HIRE_OK;
}

struct FfnWs {
  TopkWs t;
  float* proxy = nullptr;
  uint32_t* cand = nullptr;
  uint32_t* units = nullptr;
  float* act = nullptr;
  float* gval = nullptr;
  uint32_t* selg = nullptr;
  float* selv = nullptr;
  uint32_t* selu = nullptr;
  float* selact = nullptr;
  float* partial = nullptr;
};

// Local select_groups + the exact activations of the selected units. Writes
// selected group ids (ascending) into `sel` [B][kg] (stride kg) and returns
// units/activations for the down-projection in fw.selu/fw.selact [B][kg*g].
int ffn_select(hire_ctx ctx, const hire_matrix_s* u, const hire_scorer_s* a, const float* x,
               int64_t B, int64_t g, int64_t kg, int64_t kpg, int phi, int x_mode, int strict,
               const SelPlan& sp, FfnWs& fw, uint32_t* sel, int64_t sel_stride) {
  const int64_t m = u->rows, ng = m / g;
  RET(run_scores(ctx, a, x, B, phi, x_mode, strict, fw.t.sw, fw.t.scores, m));
  const float* proxy = fw.t.scores;
  if (g > 1) {
    CK(launch_k(ctx, group_proxy_kernel, static_cast<unsigned>(ceil_div(ng * B, 256)), 256, 0, fw.t.scores, m, ng, static_cast<int>(g), static_cast<int>(B), fw.proxy));
    CK(cudaGetLastError());
    proxy = fw.proxy;
  }
  RET(run_select(ctx, proxy, g > 1 ? ng : m, ng, B, sp, fw.t.surv, fw.cand, kpg, fw.t.status));
  if (g == 1) {
    RET(run_recompute(ctx, u, fw.cand, kpg, kpg, x, B, phi, strict, fw.act, kpg));
    // top-k by exact activation, emitted in ascending unit order with values
    RET(run_final(ctx, fw.act, kpg, fw.cand, kpg, nullptr, 0, 0, kpg, kg, B, 1, sel, fw.selact,
                  nullptr, nullptr, sel_stride));
    return HIRE_OK;
  }
  CK(launch_k(ctx, expand_groups_kernel, static_cast<unsigned>(ceil_div(kpg * g * B, 256)), 256, 0, fw.cand, kpg, kpg, static_cast<int>(g), static_cast<int>(B), fw.units));
  CK(cudaGetLastError());
  RET(run_recompute(ctx, u, fw.units, kpg * g, kpg * g, x, B, phi, strict, fw.act, kpg * g));
  CK(launch_k(ctx, group_sum_kernel, static_cast<unsigned>(ceil_div(kpg * B, 256)), 256, 0, fw.act, kpg, static_cast<int>(g), static_cast<int>(B), fw.gval));
  CK(cudaGetLastError());
  RET(run_final(ctx, fw.gval, kpg, fw.cand, kpg, nullptr, 0, 0, kpg, kg, B, 1, sel, fw.selv, nullptr,
                nullptr, sel_stride));
  CK(launch_k(ctx, expand_groups_kernel, static_cast<unsigned>(ceil_div(kg * g * B, 256)), 256, 0, sel, sel_stride, kg, static_cast<int>(g), static_cast<int>(B), fw.selu));
  CK(cudaGetLastError());
  RET(run_recompute(ctx, u, fw.selu, kg * g, kg * g, x, B, phi, strict, fw.selact, kg * g));
  return HIRE_OK;
}

void take_ffn_ws(Arena& ar, FfnWs* fw, const hire_scorer_s* a, int64_t B, int64_t m, int64_t d,
                 int64_t g, int64_t kg, int64_t kpg, const SelPlan& sp, int64_t max_chunks) {
  take_score_ws(ar, &fw->t.sw, a, B);
  ar.take(&fw->t.scores, static_cast<size_t>(B * m));
  ar.take(&fw->t.surv, static_cast<size_t>(sp.surv_words(B)));
  ar.take(&fw->t.status, 1);
  ar.take(&fw->proxy, static_cast<size_t>(B * (m / g)));
  ar.take(&fw->cand, static_cast<size_t>(B * kpg));
  ar.take(&fw->units, static_cast<size_t>(B * kpg * g));
  ar.take(&fw->act, static_cast<size_t>(B * kpg * g));
  ar.take(&fw->gval, static_cast<size_t>(B * kpg));
  ar.take(&fw->selv, static_cast<size_t>(B * kg));
  ar.take(&fw->selu, static_cast<size_t>(B * kg * g));
  ar.take(&fw->selact, static_cast<size_t>(B * kg * g));
  ar.take(&fw->partial, static_cast<size_t>(B * std::max<int64_t>(max_chunks, 1) * d));
}
}  // namespace

}  // extern "C"

namespace {
#if HIRE_EXPERIMENTS
template <typename T, int NT, int KS>
int launch_ffn_fused_t(hire_ctx ctx, const FusedFfnArgs& args, size_t smem) {
  auto k = ffn_fused_kernel<T, NT, KS>;
  static int max_dyn = 0;
  if (!max_dyn) {
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, k));
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
    max_dyn = optin - static_cast<int>(fa.sharedSizeBytes);
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn));
  }
  if (static_cast<int>(smem) > max_dyn) return 1;  // not taken: fall back to the kernel chain
  const int bps = max_blocks(k, kFusedThreads, smem);
  if (bps < 1) return invalid("fused FFN: does not fit one CTA per SM");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(ctx->num_sms);
  cfg.blockDim = dim3(kFusedThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++ctx->launches;
  CK(cudaLaunchKernelEx(&cfg, k, args));
  return HIRE_OK;
}

template <typename T>
int launch_ffn_fused_nt(hire_ctx ctx, const FusedFfnArgs& args, size_t smem, int nt, int ks) {
  if (nt == 1) {
    if (ks == 8) return launch_ffn_fused_t<T, 1, 8>(ctx, args, smem);
    if (ks == 4) return launch_ffn_fused_t<T, 1, 4>(ctx, args, smem);
    if (ks == 2) return launch_ffn_fused_t<T, 1, 2>(ctx, args, smem);
    return launch_ffn_fused_t<T, 1, 1>(ctx, args, smem);
  }
  if (ks == 8) return launch_ffn_fused_t<T, 2, 8>(ctx, args, smem);
  if (ks == 4) return launch_ffn_fused_t<T, 2, 4>(ctx, args, smem);
  if (ks == 2) return launch_ffn_fused_t<T, 2, 2>(ctx, args, smem);
  return launch_ffn_fused_t<T, 2, 1>(ctx, args, smem);
}

// One cooperative launch for the whole layer (ffn_fused.cuh) when the shape
// allows it; returns 1 (not taken) otherwise.
#endif

int try_ffn_fused(hire_ctx ctx, const hire_matrix_s* u, const hire_matrix_s* v, hire_scorer_s* a,
                  const float* x, int64_t B, const hire_ffn_params* p, uint32_t* sel, float* out) {
#if !HIRE_EXPERIMENTS
  (void)ctx; (void)u; (void)v; (void)a; (void)x; (void)B; (void)p; (void)sel; (void)out;
  return 1;  // the kernel chain (the single-launch layer is an experiments-build kernel)
#else
  if (!ctx->ffn_fused || p->group_size != 1 || p->x_mode != HIRE_X_INT8 || p->strict) return 1;
  if (a->kind != HIRE_SCORER_Q4 || B < 1 || B > 16 || u->d % 64 != 0 || u->d > 8192) return 1;
  if (u->rows > 16384 || p->k_prime > u->rows || p->k > p->k_prime) return 1;
  if (u->dtype != v->dtype) return 1;
  RET(ensure_mma_layout(ctx, a));
  const int64_t m = u->rows, d = u->d, kp = p->k_prime, k = p->k;
  const int nt = B <= 8 ? 1 : 2;
  const int64_t nkb = d / 64, n_rb = ceil_div(m, 16);
  int ks = 1;
  while (ks < 8 && n_rb * ks < static_cast<int64_t>(ctx->num_sms) * kFusedWarps && nkb >= 2 * ks) ks *= 2;
  const size_t xq_acc = static_cast<size_t>(nt) * 8 * (d + 16) + (ks > 1 ? static_cast<size_t>(kFusedWarps) * nt * 4 * 32 * 4 : 0);
  if (kp > 1024 || ctx->num_sms > 255) return 1;  // P4: 128 threads x 8 pairs, u8 slot ids
  if (ceil_div(m, ctx->num_sms) > 2048) return 1;  // P2b prefetch bitmap
  if (d * static_cast<int64_t>(dtype_size(u->dtype)) > 4096) return 1;  // P3: one register pass per row
  const int64_t G = ctx->num_sms;
  const int64_t wrow = ceil_div(m, G);
  const size_t pool = std::max({xq_acc, static_cast<size_t>(B * wrow) * 8 + static_cast<size_t>(wrow) * 8 + 8,
                                static_cast<size_t>((m + 31) / 32) * 4 + static_cast<size_t>(m) * 4 +
                                    static_cast<size_t>(G) * 4 + static_cast<size_t>(kp)});
  const size_t smem = static_cast<size_t>(B) * d * 4 + pool;
  if (smem > 200 * 1024) return 1;
  const int64_t nch = ceil_div(k, kFusedCh);
  Arena ar;
  FusedFfnArgs args{};
  ar.take(&args.scores, static_cast<size_t>(B * m));
  ar.take(&args.piv, static_cast<size_t>(4 * B));
  ar.take(&args.thr, static_cast<size_t>(B));
  ar.take(&args.acnt, static_cast<size_t>(B * G));
  ar.take(&args.pcnt, static_cast<size_t>(B * G));
  ar.take(&args.gh, static_cast<size_t>(B) * kWinGroups * kWinBins);
  ar.take(&args.lists, static_cast<size_t>(B) * kWinGroups * kWinBins * kBinCap);
  ar.take(&args.pairs, static_cast<size_t>(B * G * wrow));
  ar.take(&args.selact, static_cast<size_t>(B * k));
  ar.take(&args.partial, static_cast<size_t>(B * nch * d));
  RET(ar.commit(ctx));
  args.u_mma = a->mma;
  args.scales = a->scales;
  args.u = u->ptr;
  args.v = v->ptr;
  args.x = x;
  args.B = static_cast<int>(B);
  args.m = static_cast<int>(m);
  args.d = static_cast<int>(d);
  args.kp = static_cast<int>(kp);
  args.k = static_cast<int>(k);
  args.phi = p->phi;
  args.wmax = static_cast<int>(wrow);
  args.qcnt = nullptr;
  args.sel = sel;
  args.out = out;
  args.counters = ctx->counters;
  args.trace = ctx->trace ? reinterpret_cast<long long*>(ctx->counters + kTraceOff) : nullptr;
  StageScope scope(ctx, kStageFused);
  if (u->dtype == HIRE_BF16) return launch_ffn_fused_nt<__nv_bfloat16>(ctx, args, smem, nt, ks);
  return launch_ffn_fused_nt<float>(ctx, args, smem, nt, ks);
#endif
}
}  // namespace

extern "C" {

int hire_ffn_run(hire_ctx ctx, hire_matrix u, hire_matrix v, hire_scorer a, const float* x, int64_t B,
                 const hire_ffn_params* p, uint32_t* sel, float* out) {
  if (!ctx || !x || !sel || !out) return invalid("null argument");
  RET(validate_ffn(u, v, a, B, p));
  {
    const int rc = try_ffn_fused(ctx, u, v, a, x, B, p, sel, out);
    if (rc != 1) return rc;
  }
  const int64_t g = p->group_size, m = u->rows, kg = p->k / g, kpg = p->k_prime / g;
  SelPlan sp;
  RET(plan_select(m / g, kpg, HIRE_SELECT_EXACT, 0, 0, &sp));
  Arena ar;
  FfnWs fw;
  take_ffn_ws(ar, &fw, a, B, m, u->d, g, kg, kpg, sp, ceil_div(kg * g, 8));
  RET(ar.commit(ctx));
  RET(ffn_select(ctx, u, a, x, B, g, kg, kpg, p->phi, p->x_mode, p->strict, sp, fw, sel, kg));
  const uint32_t* units = g == 1 ? sel : fw.selu;
  RET(run_down(ctx, v, units, fw.selact, kg * g, kg * g, B, p->strict, fw.partial, out));
  return HIRE_OK;
}

int hire_ffn_host(hire_ctx ctx, hire_matrix u, hire_matrix v, hire_scorer a, const float* x_host,
                  int64_t B, const hire_ffn_params* p, uint32_t* sel_host, float* out_host) {
  if (!ctx || !x_host || !out_host) return invalid("null argument");
  bind_thread(ctx);
  RET(validate_ffn(u, v, a, B, p));
  const int64_t kg = p->k / p->group_size;
  const size_t xb = static_cast<size_t>(B * u->d) * 4;
  const size_t sb = static_cast<size_t>(B * kg) * 4;
  const size_t ob = static_cast<size_t>(B * u->d) * 4;
  const size_t in_bytes = align_up(xb), out_bytes = align_up(sb) + align_up(ob);
  RET(ensure(&ctx->io_dev, &ctx->io_dev_cap, in_bytes + out_bytes, ctx->stream));
  RET(ensure_host(&ctx->io_host, &ctx->io_host_cap, in_bytes + out_bytes, ctx->stream));
  char* dv = static_cast<char*>(ctx->io_dev);
  char* hs = static_cast<char*>(ctx->io_host);
  // results go straight into caller buffers in pinned memory (no staging;
  // the graph key then holds those addresses, and the cache is bounded);
  // the input is always staged: a graph keyed on every caller input buffer
  // would be re-captured for each new buffer
  void* od = host_alias(out_host, ob);
  void* sd = sel_host ? host_alias(sel_host, sb) : nullptr;
  // the input: in place when pinned (the fetch node follows it per call), else staged
  const void* xa = host_alias(x_host, xb);
  if (!xa) std::memcpy(hs, x_host, xb);
  const void* xsrc = xa ? static_cast<const void*>(x_host) : hs;
  const void* xdev = xa ? xa : host_alias(hs, align_up(xb));
  // the output rows are written straight into mapped host memory; the unit
  // ids stay on the device (the down-projection reads them) and are stored
  // to the host by a small kernel at the end
  uint32_t* dsel = reinterpret_cast<uint32_t*>(dv + in_bytes);
  uint32_t* hsel = sd ? static_cast<uint32_t*>(sd) : reinterpret_cast<uint32_t*>(hs + in_bytes);
  float* dout = od ? static_cast<float*>(od) : reinterpret_cast<float*>(hs + in_bytes + align_up(sb));
  const std::vector<int64_t> key = {2, static_cast<int64_t>(u->uid), static_cast<int64_t>(v->uid),
                                    static_cast<int64_t>(a->uid), B, p->k, p->k_prime, p->group_size, p->phi,
                                    p->x_mode, p->strict, reinterpret_cast<int64_t>(od),
                                    reinterpret_cast<int64_t>(sd), sel_host ? 1 : 0};
  int64_t res[4];
  cudaStream_t done_on = nullptr;
  RET(run_host_graph(ctx, key, res, &done_on, xdev, [&](int64_t*) -> int {
    RET(fetch_inputs(ctx, dv, xsrc, xb));
    RET(hire_ffn_run(ctx, u, v, a, reinterpret_cast<const float*>(dv), B, p, dsel, dout));
    if (sel_host) {
      if (sb % 16 == 0) {
        const int64_t n16 = static_cast<int64_t>(sb / 16);
        CK(launch_k(ctx, fetch_host_kernel, static_cast<unsigned>(std::min<int64_t>(ceil_div(n16, 256), 64)), 256, 0,
                    reinterpret_cast<const uint4*>(dsel), reinterpret_cast<uint4*>(hsel), n16));
      } else {
        CK(cudaMemcpyAsync(hsel, dsel, sb, cudaMemcpyDefault, ctx->stream));
      }
    }
    return HIRE_OK;
  }));
  CK(cudaStreamSynchronize(done_on));
  if (sel_host && !sd) std::memcpy(sel_host, hs + in_bytes, sb);
  if (!od) std::memcpy(out_host, hs + in_bytes + align_up(sb), ob);
  return HIRE_OK;
}

int hire_ffn_dense_run(hire_ctx ctx, hire_matrix u, hire_matrix v, const float* x, int64_t B, int phi,
                       int strict, float* out) {
  if (!ctx || !u || !v || !x || !out) return invalid("null argument");
  if (u->rows != v->rows || u->d != v->d) return invalid("GroupedFFN: U and V must both be d x m");
  RET(check_phi(phi));
  const int64_t m = u->rows;
  Arena ar;
  float* act;
  uint32_t* units;
  float* partial;
  ar.take(&act, static_cast<size_t>(B * m));
  ar.take(&units, static_cast<size_t>(B * m));
  ar.take(&partial, static_cast<size_t>(B * ceil_div(m, 8) * u->d));
  RET(ar.commit(ctx));
  RET(run_recompute(ctx, u, nullptr, 0, m, x, B, phi, strict, act, m));
  CK(launch_k(ctx, iota_mod_kernel, static_cast<unsigned>(ceil_div(B * m, 256)), 256, 0, units, m, B * m));
  CK(cudaGetLastError());
  return run_down(ctx, v, units, act, m, m, B, strict, partial, out);
}

int hire_ffn_union_select(hire_ctx ctx, hire_matrix u, hire_scorer a, const float* x, int64_t B,
                          const hire_ffn_params* p, uint32_t* ids, int64_t* n_ids) {
  if (!ctx || !x || !ids || !n_ids) return invalid("null argument");
  if (B < 1) return invalid("union_group_select: no input samples");
  RET(validate_ffn(u, u, a, B, p));
  const int64_t g = p->group_size, m = u->rows, kg = p->k / g, kpg = p->k_prime / g, ng = m / g;
  if ((ng + 31) / 32 * 4 > 48 * 1024) return invalid("union_group_select: more than 393216 groups");
  SelPlan sp;
  RET(plan_select(ng, kpg, HIRE_SELECT_EXACT, 0, 0, &sp));
  Arena ar;
  FfnWs fw;
  take_ffn_ws(ar, &fw, a, B, m, u->d, g, kg, kpg, sp, 1);
  uint32_t* sel;
  int64_t* cnt;
  ar.take(&sel, static_cast<size_t>(B * kg));
  ar.take(&cnt, 1);
  RET(ar.commit(ctx));
  RET(ffn_select(ctx, u, a, x, B, g, kg, kpg, p->phi, p->x_mode, p->strict, sp, fw, sel, kg));
  CK(launch_k(ctx, group_union_kernel, 1u, 1024, static_cast<size_t>((ng + 31) / 32) * 4, static_cast<const uint32_t*>(sel),
              kg, static_cast<int>(kg), static_cast<int>(B), static_cast<int>(ng), ids, cnt));
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(n_ids, cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return HIRE_OK;
}

int hire_ffn_common_path_run(hire_ctx ctx, hire_matrix du, hire_matrix dv, hire_matrix u, hire_matrix v,
                             hire_scorer a, const float* x, int64_t B, const hire_ffn_params* p, float* out) {
  if (!ctx || !x || !out || !u || !v || !p) return invalid("null argument");
  // CommonPathFFN validate (ffn.hpp:49-56)
  if (du && dv && (du->rows != dv->rows || du->d != dv->d)) return invalid("GroupedFFN: U and V must both be d x m");
  if (du && du->d != u->d) return invalid("CommonPathFFN: parts disagree on d");
  if (u->rows < p->group_size) return invalid("CommonPathFFN: sparse part needs m2 >= g");
  RET(validate_ffn(u, v, a, B, p));
  const size_t n = static_cast<size_t>(B * u->d);
  if (du && dv && du->rows > 0) {
    RET(hire_ffn_dense_run(ctx, du, dv, x, B, p->phi, p->strict, out));
  } else {
    CK(cudaMemsetAsync(out, 0, n * 4, ctx->stream));
  }
  // the sparse part's output in io_dev (out stays untouched until the add)
  RET(ensure(&ctx->io_dev, &ctx->io_dev_cap, n * 4 + static_cast<size_t>(B * p->k) * 4 + 512, ctx->stream));
  float* sp_out = static_cast<float*>(ctx->io_dev);
  uint32_t* sp_sel = reinterpret_cast<uint32_t*>(static_cast<char*>(ctx->io_dev) + align_up(n * 4));
  RET(hire_ffn_run(ctx, u, v, a, x, B, p, sp_sel, sp_out));
  CK(launch_k(ctx, add_f32_kernel, static_cast<unsigned>(ceil_div(static_cast<int64_t>(n), 256)), 256, 0, out,
              static_cast<const float*>(sp_out), static_cast<int64_t>(n)));
  CK(cudaGetLastError());
  return HIRE_OK;
}

// ------------------------------------------------------------------- DA --
int hire_comm_unique_id(uint8_t id[128]) {
  ncclUniqueId u;
  CKN(ncclGetUniqueId(&u));
  std::memcpy(id, u.internal, 128);
  return HIRE_OK;
}

int hire_comm_create(const uint8_t id[128], int world, int rank, hire_comm* out) {
  if (!out || world < 1 || rank < 0 || rank >= world) return invalid("bad communicator arguments");
  ncclUniqueId u;
  std::memcpy(u.internal, id, 128);
  auto* c = new hire_comm_s();
  c->world = world;
  c->rank = rank;
  ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return set_err(HIRE_ERR_RUNTIME, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *out = c;
  return HIRE_OK;
}

int hire_comm_destroy(hire_comm c) {
  if (!c) return HIRE_OK;
  ncclCommDestroy(c->comm);
  delete c;
  return HIRE_OK;
}

namespace {
int64_t quota(int64_t k, int64_t s, int64_t i) { return k / s + (i < k % s ? 1 : 0); }

struct DaPlan {
  int64_t kl = 0, kpl = 0;     // this shard's quotas
  int64_t kq_max = 0;          // per-rank send slots
  SelPlan sp;
};

int plan_da(const hire_topk_params* p, int64_t width, int world, int rank, int merge, int uneven,
            DaPlan* dp) {
  if (world < 1) return invalid("da_topk: no shards");
  if (!uneven && p->k % world != 0)
    return invalid("da_topk: s = " + std::to_string(world) + " must divide k = " + std::to_string(p->k));
  if (!uneven && p->k_prime % world != 0)
    return invalid("da_topk: s = " + std::to_string(world) + " must divide k_prime = " + std::to_string(p->k_prime));
  dp->kl = quota(p->k, world, rank);
  dp->kpl = quota(p->k_prime, world, rank);
  if (dp->kl > width)
    return invalid("da_topk: per-shard quota k/s = " + std::to_string(dp->kl) + " exceeds shard width " + std::to_string(width));
  RET(plan_select(width, dp->kpl, p->select, p->n_buckets, p->bucket_t, &dp->sp));
  dp->kq_max = merge == HIRE_MERGE_PER_SHARD ? ceil_div(p->k, world) : ceil_div(p->k_prime, world);
  return HIRE_OK;
}

// One shard's local stage; writes keys (global indices) into send [B][kq_max].
int da_local(hire_ctx ctx, const hire_matrix_s* w, const hire_scorer_s* a, int64_t offset,
             const float* x, int64_t B, const hire_topk_params* p, const DaPlan& dp, int merge,
             uint64_t* send) {
  Arena ar;
  TopkWs t;
  take_topk_ws(ar, &t, a, B, dp.sp, true, ctx, p);
  RET(ar.commit(ctx));
  RET(local_candidates(ctx, w, a, x, B, p, dp.sp, t, t.cand, false));
  if (offset) {
    CK(launch_k(ctx, add_offset_kernel, static_cast<unsigned>(ceil_div(B * dp.sp.k_eff, 256)), 256, 0, t.cand, B * dp.sp.k_eff, static_cast<uint32_t>(offset)));
    CK(cudaGetLastError());
  }
  const int64_t K = merge == HIRE_MERGE_PER_SHARD ? std::min(dp.kl, dp.sp.k_eff) : dp.sp.k_eff;
  if (K < 1) {
    CK(cudaMemsetAsync(send, 0, static_cast<size_t>(B * dp.kq_max) * 8, ctx->stream));
    return HIRE_OK;
  }
  return run_final(ctx, t.vals, dp.sp.k_eff, t.cand, dp.sp.k_eff, nullptr, 0, 0, dp.sp.k_eff, K, B, 2,
                   nullptr, nullptr, nullptr, send, dp.kq_max);
}

int64_t da_total_k(const hire_topk_params* p, int64_t total_rows, int world, int merge, int uneven,
                   bool* clamped) {
  int64_t tot = 0, kp_tot = 0;
  *clamped = false;
  for (int r = 0; r < world; ++r) {
    int64_t f, wdt;
    part_range(total_rows, world, r, &f, &wdt);
    const int64_t kpl = quota(p->k_prime, world, r), kl = quota(p->k, world, r);
    const int64_t keff = std::min(kpl, wdt);
    if (kpl > wdt) *clamped = true;
    kp_tot += keff;
    tot += std::min(kl, keff);
  }
  (void)uneven;
  if (merge == HIRE_MERGE_GLOBAL) {
    if (kp_tot < p->k) *clamped = true;
    return std::min(p->k, kp_tot);
  }
  return tot;
}
}  // namespace

namespace {
// Checks shared by the DA-TOP-k entry points: this rank's shard against the
// width rule (distributed.hpp:53-57) and its quotas; fills the plan.
int da_prepare(const hire_matrix_s* w, const hire_scorer_s* a, int64_t total_rows, int world, int rank,
               int64_t B, const hire_topk_params* p, int merge, int uneven, int64_t* first, DaPlan* dp) {
  if (!p) return invalid("null argument");
  if (world < 1 || rank < 0 || rank >= world) return invalid("da_topk: bad world/rank");
  if (merge != HIRE_MERGE_PER_SHARD && merge != HIRE_MERGE_GLOBAL) return invalid("da_topk: unknown merge mode");
  hire_topk_params lp = *p;
  lp.k = std::max<int64_t>(1, quota(p->k, world, rank));
  lp.k_prime = std::max(lp.k, quota(p->k_prime, world, rank));
  RET(validate_topk(w, a, B, &lp));
  int64_t width;
  part_range(total_rows, world, rank, first, &width);
  if (w->rows != width) return invalid("da_topk: shard has " + std::to_string(w->rows) + " rows, width rule says " + std::to_string(width));
  return plan_da(p, width, world, rank, merge, uneven, dp);
}

int da_merge(hire_ctx ctx, const uint64_t* gathered, int64_t slots, int64_t total_rows, int world, int64_t B,
             const hire_topk_params* p, int merge, int uneven, uint32_t* top_idx, float* top_val, int64_t* n_top,
             int* clamped) {
  bool cl = false;
  const int64_t K = da_total_k(p, total_rows, world, merge, uneven, &cl);
  RET(run_final(ctx, nullptr, 0, nullptr, 0, gathered, slots, B * slots, world * slots, K, B, 0, top_idx, top_val,
                nullptr, nullptr, p->k));
  if (n_top) *n_top = K;
  if (clamped) *clamped = cl;
  return HIRE_OK;
}
}  // namespace

int hire_da_topk_slots(const hire_topk_params* p, int world, int merge, int64_t* slots) {
  if (!p || !slots) return invalid("null argument");
  if (world < 1) return invalid("da_topk: no shards");
  *slots = merge == HIRE_MERGE_PER_SHARD ? ceil_div(p->k, world) : ceil_div(p->k_prime, world);
  return HIRE_OK;
}

int hire_da_topk_local(hire_ctx ctx, hire_matrix w, hire_scorer a, int64_t total_rows, int world, int rank,
                       const float* x, int64_t B, const hire_topk_params* p, int merge, int uneven, uint64_t* send) {
  if (!ctx || !x || !send) return invalid("null argument");
  int64_t first = 0;
  DaPlan dp;
  RET(da_prepare(w, a, total_rows, world, rank, B, p, merge, uneven, &first, &dp));
  return da_local(ctx, w, a, first, x, B, p, dp, merge, send);
}

int hire_da_topk_merge(hire_ctx ctx, const uint64_t* gathered, int64_t total_rows, int world, int64_t B,
                       const hire_topk_params* p, int merge, int uneven, uint32_t* top_idx, float* top_val,
                       int64_t* n_top, int* clamped) {
  if (!ctx || !gathered || !top_idx || !top_val || !p) return invalid("null argument");
  if (world < 1 || B < 1) return invalid("da_topk: bad world or batch");
  int64_t slots = 0;
  RET(hire_da_topk_slots(p, world, merge, &slots));
  return da_merge(ctx, gathered, slots, total_rows, world, B, p, merge, uneven, top_idx, top_val, n_top, clamped);
}

int hire_da_topk_run(hire_ctx ctx, hire_comm comm, hire_matrix w, hire_scorer a, int64_t total_rows,
                     int world, int rank, const float* x, int64_t B, const hire_topk_params* p,
                     int merge, int uneven, uint32_t* top_idx, float* top_val, int64_t* n_top,
                     int* clamped) {
  if (!ctx || !x || !top_idx || !top_val) return invalid("null argument");
  if (comm && (comm->world != world || comm->rank != rank)) return invalid("communicator does not match world/rank");
  if (!comm && world != 1) return invalid("da_topk: world > 1 needs a communicator");
  int64_t first = 0;
  DaPlan dp;
  RET(da_prepare(w, a, total_rows, world, rank, B, p, merge, uneven, &first, &dp));
  if (!comm) {
    // one shard, no communicator: DA-TOP-k is hire_topk itself
    // (distributed.hpp:94-131 with s = 1; the reference's s = 1 equivalence,
    // test_distributed.cpp:104-117) — no key hand-off, no second selection
    int64_t nc = 0;
    return hire_topk_run(ctx, w, a, x, B, p, nullptr, top_idx, top_val, nullptr, &nc, n_top, clamped);
  }
  // local stage -> one ncclAllGather of B x slots rank keys -> merge
  const size_t sendb = align_up(static_cast<size_t>(B * dp.kq_max) * 8);
  const size_t recvb = align_up(static_cast<size_t>(world * B * dp.kq_max) * 8);
  RET(ensure(&ctx->io_dev, &ctx->io_dev_cap, sendb + recvb, ctx->stream));
  uint64_t* send = static_cast<uint64_t*>(ctx->io_dev);
  uint64_t* recv = reinterpret_cast<uint64_t*>(static_cast<char*>(ctx->io_dev) + sendb);
  RET(da_local(ctx, w, a, first, x, B, p, dp, merge, send));
  {
    StageScope scope(ctx, kStageComm);
    CKN(ncclAllGather(send, recv, static_cast<size_t>(B * dp.kq_max), ncclUint64, comm->comm, ctx->stream));
  }
  return da_merge(ctx, recv, dp.kq_max, total_rows, world, B, p, merge, uneven, top_idx, top_val, n_top, clamped);
}

int hire_da_topk_emulated(hire_ctx ctx, hire_matrix w, hire_scorer a, int world, const float* x,
                          int64_t B, const hire_topk_params* p, int merge, int uneven,
                          uint32_t* top_idx, float* top_val, int64_t* n_top, int* clamped) {
  if (!ctx || !x || !top_idx || !top_val) return invalid("null argument");
  RET(validate_topk(w, a, B, p));
  if (world < 1 || world > w->rows) return invalid("shard: s = " + std::to_string(world) + " exceeds l = " + std::to_string(w->rows));
  int64_t kq_max = 0;
  std::vector<DaPlan> plans(world);
  for (int r = 0; r < world; ++r) {
    int64_t f, wd;
    part_range(w->rows, world, r, &f, &wd);
    RET(plan_da(p, wd, world, r, merge, uneven, &plans[r]));
    kq_max = plans[r].kq_max;
  }
  const size_t recvb = align_up(static_cast<size_t>(world * B * kq_max) * 8);
  RET(ensure(&ctx->io_dev, &ctx->io_dev_cap, recvb, ctx->stream));
  uint64_t* recv = static_cast<uint64_t*>(ctx->io_dev);
  // shard slices share the parent's tensor-core layouts (built here once)
  if (a->kind == HIRE_SCORER_Q4 && p->x_mode == HIRE_X_INT8 && !p->strict && umma_min_batch() > 0 &&
      B >= 5 && umma_shape_ok(a, std::min<int64_t>(B, 64)))
    RET(ensure_umma_layout(ctx, a));
  for (int r = 0; r < world; ++r) {
    int64_t f, wd;
    part_range(w->rows, world, r, &f, &wd);
    hire_matrix ws;
    hire_scorer as;
    RET(hire_matrix_slice(w, f, wd, &ws));
    RET(hire_scorer_slice(a, f, wd, &as));
    const int rc = da_local(ctx, ws, as, f, x, B, p, plans[r], merge, recv + static_cast<int64_t>(r) * B * kq_max);
    hire_matrix_destroy(ws);
    hire_scorer_destroy(as);
    RET(rc);
  }
  return da_merge(ctx, recv, kq_max, w->rows, world, B, p, merge, uneven, top_idx, top_val, n_top, clamped);
}

// DA FFN ------------------------------------------------------------------
namespace {
struct DaFfnPlan {
  int64_t kgl = 0, kpl = 0, kg_max = 0;
  SelPlan sp;
};

int plan_da_ffn(const hire_ffn_params* p, int64_t total_units, int64_t width_groups, int world, int rank,
                int uneven, DaFfnPlan* fp) {
  const int64_t g = p->group_size;
  const int64_t kg = p->k / g, kpg = p->k_prime / g;
  if (world < 1) return invalid("da_group_sparse: s must be >= 1");
  if (world > total_units / g)
    return invalid("da_group_sparse: s = " + std::to_string(world) + " exceeds group count " + std::to_string(total_units / g));
  if (!uneven && kg % world != 0)
    return invalid("da_group_sparse: s = " + std::to_string(world) + " must divide the group quota k/g = " + std::to_string(kg));
  if (!uneven && kpg % world != 0)
    return invalid("da_group_sparse: s = " + std::to_string(world) + " must divide the candidate quota k_prime/g = " + std::to_string(kpg));
  fp->kgl = quota(kg, world, rank);
  fp->kpl = std::min(quota(kpg, world, rank), width_groups);  // distributed.hpp:192
  if (fp->kgl > width_groups)
    return invalid("da_group_sparse: per-shard quota " + std::to_string(fp->kgl) + " exceeds shard group count " + std::to_string(width_groups));
  fp->kg_max = ceil_div(kg, world);
  return plan_select(width_groups, fp->kpl, HIRE_SELECT_EXACT, 0, 0, &fp->sp);
}

// Union of the per-rank selections (distributed.hpp:196-201): rank r
// contributed min(quota(kg, s, r), width_r) ascending shard-local group ids
// (already global); the rank-major concatenation is globally ascending.
__global__ void concat_sel_kernel(const uint32_t* recv, int world, int64_t B, int64_t kg_max, int64_t ng,
                                  int64_t kg, int64_t total, uint32_t* sel) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t b = blockIdx.x;
  int64_t pos = 0;
  for (int r = 0; r < world; ++r) {
    const int64_t width = ng / world + (r < ng % world ? 1 : 0);
    const int64_t q = kg / world + (r < kg % world ? 1 : 0);
    const int64_t c = q < width ? q : width;
    for (int64_t i = threadIdx.x; i < c; i += blockDim.x)
      sel[b * total + pos + i] = recv[(r * B + b) * kg_max + i];
    pos += c;
  }
}

// local stage of da_group_sparse: selection with local quotas on this
// shard, global group ids, partial down-projection into out_partial.
int da_ffn_local(hire_ctx ctx, const hire_matrix_s* u, const hire_matrix_s* v, const hire_scorer_s* a,
                 int64_t first_group, const float* x, int64_t B, const hire_ffn_params* p,
                 const DaFfnPlan& fp, uint32_t* sel_out, int64_t sel_stride, float* out_partial) {
  const int64_t g = p->group_size, m = u->rows;
  Arena ar;
  FfnWs fw;
  take_ffn_ws(ar, &fw, a, B, m, u->d, g, fp.kgl, fp.kpl, fp.sp, ceil_div(fp.kgl * g, 8));
  uint32_t* sel_local;
  ar.take(&sel_local, static_cast<size_t>(B * std::max<int64_t>(fp.kgl, 1)));
  RET(ar.commit(ctx));
  if (fp.kgl == 0 || fp.kpl == 0) {
    CK(cudaMemsetAsync(out_partial, 0, static_cast<size_t>(B * u->d) * 4, ctx->stream));
    return HIRE_OK;
  }
  RET(ffn_select(ctx, u, a, x, B, g, fp.kgl, fp.kpl, p->phi, p->x_mode, p->strict, fp.sp, fw, sel_local, fp.kgl));
  const uint32_t* units = g == 1 ? sel_local : fw.selu;
  RET(run_down(ctx, v, units, fw.selact, fp.kgl * g, fp.kgl * g, B, p->strict, fw.partial, out_partial));
  // global group ids into the send slots (padded rows untouched)
  CK(cudaMemcpy2DAsync(sel_out, sel_stride * 4, sel_local, fp.kgl * 4, fp.kgl * 4, B, cudaMemcpyDeviceToDevice, ctx->stream));
  if (first_group) {
    CK(launch_k(ctx, add_offset_strided_kernel, static_cast<unsigned>(ceil_div(fp.kgl * B, 256)), 256, 0, sel_out, sel_stride, fp.kgl, B, static_cast<uint32_t>(first_group)));
    CK(cudaGetLastError());
  }
  return HIRE_OK;
}

// out = sum over ranks of the partial outputs, added in rank order
// (deterministic: the same bits whatever the collective topology)
__global__ void sum_parts_kernel(const float* parts, int world, int64_t n, float* out) {
  hire_dev::griddep_wait();
  hire_dev::griddep_launch();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.0f;
  for (int r = 0; r < world; ++r) s = __fadd_rn(s, parts[r * n + i]);
  out[i] = s;
}

int64_t da_ffn_total(int64_t ng, int64_t kg, int world) {
  int64_t total = 0;
  for (int r = 0; r < world; ++r) {
    int64_t f2, w2;
    part_range(ng, world, r, &f2, &w2);
    total += std::min(quota(kg, world, r), w2);
  }
  return total;
}

int da_ffn_prepare(const hire_matrix_s* u, const hire_matrix_s* v, const hire_scorer_s* a, int64_t total_units,
                   int world, int rank, int64_t B, const hire_ffn_params* p, int uneven, int64_t* first_group,
                   DaFfnPlan* fp) {
  if (!u || !v || !a || !p) return invalid("null argument");
  if (world < 1 || rank < 0 || rank >= world) return invalid("da_group_sparse: bad world/rank");
  const int64_t g = p->group_size;
  if (g < 1 || total_units % g != 0) return invalid("GroupedFFN: g must divide m");
  const int64_t ng = total_units / g;
  int64_t wg;
  part_range(ng, world, rank, first_group, &wg);
  if (u->rows != wg * g) return invalid("da_group_sparse: shard unit count does not match the width rule");
  RET(plan_da_ffn(p, total_units, wg, world, rank, uneven, fp));
  hire_ffn_params lp = *p;
  lp.k = std::max<int64_t>(1, fp->kgl) * g;
  lp.k_prime = std::max<int64_t>(lp.k, fp->kpl * g);
  if (fp->kgl > 0) RET(validate_ffn(u, v, a, B, &lp));
  return HIRE_OK;
}

int da_ffn_merge(hire_ctx ctx, const uint32_t* gsel, int64_t kg_max, const float* parts, int64_t d,
                 int64_t total_units, int world, int64_t B, const hire_ffn_params* p, uint32_t* sel, float* out) {
  const int64_t g = p->group_size, ng = total_units / g, kg = p->k / g;
  const int64_t total = da_ffn_total(ng, kg, world);
  CK(launch_k(ctx, concat_sel_kernel, static_cast<unsigned>(B), 128, 0, gsel, world, B, kg_max, ng, kg, total, sel));
  CK(cudaGetLastError());
  if (parts) {
    CK(launch_k(ctx, sum_parts_kernel, static_cast<unsigned>(ceil_div(B * d, 256)), 256, 0, parts, world, B * d, out));
    CK(cudaGetLastError());
  }
  return HIRE_OK;
}
}  // namespace

int hire_da_ffn_slots(const hire_ffn_params* p, int world, int64_t* slots) {
  if (!p || !slots) return invalid("null argument");
  if (world < 1 || p->group_size < 1) return invalid("da_group_sparse: bad world or group size");
  *slots = ceil_div(p->k / p->group_size, world);
  return HIRE_OK;
}

int hire_da_ffn_local(hire_ctx ctx, hire_matrix u, hire_matrix v, hire_scorer a, int64_t total_units, int world,
                      int rank, const float* x, int64_t B, const hire_ffn_params* p, int uneven, uint32_t* sel_send,
                      float* partial) {
  if (!ctx || !x || !sel_send || !partial) return invalid("null argument");
  int64_t fg = 0;
  DaFfnPlan fp;
  RET(da_ffn_prepare(u, v, a, total_units, world, rank, B, p, uneven, &fg, &fp));
  return da_ffn_local(ctx, u, v, a, fg, x, B, p, fp, sel_send, fp.kg_max, partial);
}

int hire_da_ffn_merge(hire_ctx ctx, const uint32_t* gathered_sel, const float* gathered_parts, int64_t total_units,
                      int64_t d, int world, int64_t B, const hire_ffn_params* p, int uneven, uint32_t* sel,
                      float* out) {
  if (!ctx || !gathered_sel || !gathered_parts || !sel || !out || !p) return invalid("null argument");
  if (world < 1 || B < 1 || d < 1) return invalid("da_group_sparse: bad world, batch or d");
  if (p->group_size < 1 || total_units % p->group_size != 0) return invalid("GroupedFFN: g must divide m");
  (void)uneven;
  int64_t slots = 0;
  RET(hire_da_ffn_slots(p, world, &slots));
  return da_ffn_merge(ctx, gathered_sel, slots, gathered_parts, d, total_units, world, B, p, sel, out);
}

int hire_da_ffn_run(hire_ctx ctx, hire_comm comm, hire_matrix u, hire_matrix v, hire_scorer a,
                    int64_t total_units, int world, int rank, const float* x, int64_t B,
                    const hire_ffn_params* p, int uneven, uint32_t* sel, float* out) {
  if (!ctx || !x || !sel || !out) return invalid("null argument");
  if (comm && (comm->world != world || comm->rank != rank)) return invalid("communicator does not match world/rank");
  if (!comm && world != 1) return invalid("da_group_sparse: world > 1 needs a communicator");
  int64_t fg = 0;
  DaFfnPlan fp;
  RET(da_ffn_prepare(u, v, a, total_units, world, rank, B, p, uneven, &fg, &fp));
  const int64_t d = u->d;
  // send: [B][kg_max] ids + [B][d] partial; recv: [world][B][kg_max] + [world][B][d]
  const size_t sselb = align_up(static_cast<size_t>(B * fp.kg_max) * 4);
  const size_t spartb = align_up(static_cast<size_t>(B * d) * 4);
  const size_t rselb = align_up(static_cast<size_t>(world * B * fp.kg_max) * 4);
  const size_t rpartb = align_up(static_cast<size_t>(world * B * d) * 4);
  RET(ensure(&ctx->io_dev, &ctx->io_dev_cap, sselb + spartb + rselb + rpartb, ctx->stream));
  char* base = static_cast<char*>(ctx->io_dev);
  uint32_t* ssel = reinterpret_cast<uint32_t*>(base);
  float* spart = reinterpret_cast<float*>(base + sselb);
  uint32_t* rsel = reinterpret_cast<uint32_t*>(base + sselb + spartb);
  float* rpart = reinterpret_cast<float*>(base + sselb + spartb + rselb);
  RET(da_ffn_local(ctx, u, v, a, fg, x, B, p, fp, comm ? ssel : rsel, fp.kg_max, comm ? spart : out));
  if (!comm) {  // one shard: the partial is the output
    return da_ffn_merge(ctx, rsel, fp.kg_max, nullptr, d, total_units, 1, B, p, sel, out);
  }
  {
    // the partial outputs are all-gathered and summed in rank order, not
    // all-reduced: NCCL's reduction order depends on the topology, the
    // rank-order sum gives the same bits on every rank and every machine
    StageScope scope(ctx, kStageComm);
    CKN(ncclGroupStart());
    CKN(ncclAllGather(ssel, rsel, static_cast<size_t>(B * fp.kg_max), ncclUint32, comm->comm, ctx->stream));
    CKN(ncclAllGather(spart, rpart, static_cast<size_t>(B * d), ncclFloat32, comm->comm, ctx->stream));
    CKN(ncclGroupEnd());
  }
  return da_ffn_merge(ctx, rsel, fp.kg_max, rpart, d, total_units, world, B, p, sel, out);
}

int hire_da_ffn_emulated(hire_ctx ctx, hire_matrix u, hire_matrix v, hire_scorer a, int world,
                         const float* x, int64_t B, const hire_ffn_params* p, int uneven, uint32_t* sel,
                         float* out) {
  if (!ctx || !u || !v || !a || !p || !x || !sel || !out) return invalid("null argument");
  RET(validate_ffn(u, v, a, B, p));
  const int64_t g = p->group_size, ng = u->rows / g, kg = p->k / g;
  std::vector<DaFfnPlan> plans(world);
  for (int r = 0; r < world; ++r) {
    int64_t f, w;
    part_range(ng, world, r, &f, &w);
    RET(plan_da_ffn(p, u->rows, w, world, r, uneven, &plans[r]));
  }
  const int64_t kg_max = plans[0].kg_max;
  const size_t recvb = align_up(static_cast<size_t>(world * B * kg_max) * 4);
  const size_t partb = align_up(static_cast<size_t>(world * B * u->d) * 4);
  RET(ensure(&ctx->io_dev, &ctx->io_dev_cap, recvb + partb, ctx->stream));
  uint32_t* recv = static_cast<uint32_t*>(ctx->io_dev);
  float* parts = reinterpret_cast<float*>(static_cast<char*>(ctx->io_dev) + recvb);
  for (int r = 0; r < world; ++r) {
    int64_t fgr, wg;
    part_range(ng, world, r, &fgr, &wg);
    hire_matrix us, vs;
    hire_scorer as;
    RET(hire_matrix_slice(u, fgr * g, wg * g, &us));
    RET(hire_matrix_slice(v, fgr * g, wg * g, &vs));
    RET(hire_scorer_slice(a, fgr * g, wg * g, &as));
    const int rc = da_ffn_local(ctx, us, vs, as, fgr, x, B, p, plans[r],
                                recv + static_cast<int64_t>(r) * B * kg_max, kg_max,
                                parts + static_cast<int64_t>(r) * B * u->d);
    hire_matrix_destroy(us);
    hire_matrix_destroy(vs);
    hire_scorer_destroy(as);
    RET(rc);
  }
  const int64_t total = da_ffn_total(ng, kg, world);
  if (p->strict) {
    // the reference's own order: one ascending sum over the union
    // (distributed.hpp:203-204 -> ffn_apply_groups, ffn.hpp:160-169)
    RET(da_ffn_merge(ctx, recv, kg_max, nullptr, u->d, u->rows, world, B, p, sel, out));
    Arena ar;
    uint32_t* units;
    float* act;
    ar.take(&units, static_cast<size_t>(B * total * g));
    ar.take(&act, static_cast<size_t>(B * total * g));
    RET(ar.commit(ctx));
    CK(launch_k(ctx, expand_groups_kernel, static_cast<unsigned>(ceil_div(total * g * B, 256)), 256, 0, sel, total, total, static_cast<int>(g), static_cast<int>(B), units));
    RET(run_recompute(ctx, u, units, total * g, total * g, x, B, p->phi, 1, act, total * g));
    RET(run_down(ctx, v, units, act, total * g, total * g, B, 1, nullptr, out));
  } else {
    // what hire_da_ffn_run computes across ranks: rank-order sum of the partials
    RET(da_ffn_merge(ctx, recv, kg_max, parts, u->d, u->rows, world, B, p, sel, out));
  }
  return HIRE_OK;
}

// ------------------------------------------------ seeded host instances --
// The reference's input generators (host code: the experiment runner's
// instances are generated on the host in the reference too): Rng
// (rng.hpp:20-61, splitmix64 counter stream, Box-Muller with a cached
// spare, libm log1p / sin / cos), derive_seed (rng.hpp:64-67), gen_vector
// and gen_instance (instance.hpp:16-83, Gram-Schmidt in double for the
// decaying spectrum) — the same arithmetic, so the same bits.
namespace {
struct HostRng {
  uint64_t seed, counter = 0;
  double spare = 0.0;
  bool has_spare = false;
  explicit HostRng(uint64_t s) : seed(s) {}
  uint64_t next_u64() { return rng_mix64(seed, ++counter); }
  double next_uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_gaussian() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    const double u1 = next_uniform(), u2 = next_uniform();
    const double radius = std::sqrt(-2.0 * std::log1p(-u1));
    const double angle = 2.0 * 3.141592653589793238462643383279502884 * u2;
    spare = radius * std::sin(angle);
    has_spare = true;
    return radius * std::cos(angle);
  }
};

// orthonormal columns (instance.hpp:26-50): q[c][0..rows)
int orthonormal_columns(int64_t rows, int64_t cols, HostRng& rng, std::vector<std::vector<double>>* q) {
  q->assign(static_cast<size_t>(cols), std::vector<double>(static_cast<size_t>(rows)));
  for (int64_t c = 0; c < cols; ++c) {
    auto& qc = (*q)[static_cast<size_t>(c)];
    for (int attempt = 0;; ++attempt) {
      for (int64_t i = 0; i < rows; ++i) qc[i] = rng.next_gaussian();
      for (int64_t p = 0; p < c; ++p) {
        const auto& qp = (*q)[static_cast<size_t>(p)];
        double proj = 0.0;
        for (int64_t i = 0; i < rows; ++i) proj += qc[i] * qp[i];
        for (int64_t i = 0; i < rows; ++i) qc[i] -= proj * qp[i];
      }
      double norm = 0.0;
      for (double x : qc) norm += x * x;
      norm = std::sqrt(norm);
      if (norm > 1e-8) {
        for (int64_t i = 0; i < rows; ++i) qc[i] /= norm;
        break;
      }
      if (attempt > 16) return set_err(HIRE_ERR_RUNTIME, "orthonormal_columns: degenerate draw");
    }
  }
  return HIRE_OK;
}
}  // namespace

uint64_t hire_derive_seed(uint64_t seed, uint64_t stream) {
  HostRng r(seed ^ (0xA5A5A5A55A5A5A5AULL + stream));
  return r.next_u64();
}

int hire_gen_vector(uint64_t seed, int64_t n, float* out) {
  if (!out || n < 0) return invalid("null argument");
  HostRng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = static_cast<float>(r.next_gaussian());
  return HIRE_OK;
}

int hire_gen_instance(int64_t d, int64_t l, uint64_t seed, int spectrum, float* out) {
  if (!out) return invalid("null argument");
  if (d < 1 || l < 1) return invalid("gen_instance: dims must be positive");
  HostRng rng(seed);
  if (spectrum == 0) {  // flat: column j (row j here) entries i, j-major
    for (int64_t j = 0; j < l; ++j)
      for (int64_t i = 0; i < d; ++i) out[j * d + i] = static_cast<float>(rng.next_gaussian());
    return HIRE_OK;
  }
  const int64_t rank = std::min(d, l);
  std::vector<std::vector<double>> left, right;
  RET(orthonormal_columns(d, rank, rng, &left));
  RET(orthonormal_columns(l, rank, rng, &right));
  for (int64_t j = 0; j < l; ++j)
    for (int64_t i = 0; i < d; ++i) {
      double acc = 0.0;
      for (int64_t q = 0; q < rank; ++q)
        acc += left[static_cast<size_t>(q)][i] * right[static_cast<size_t>(q)][j] / static_cast<double>(q + 1);
      out[j * d + i] = static_cast<float>(acc);
    }
  return HIRE_OK;
}

// ------------------------------------------------------ gather benchmark --
int hire_gather_bench(hire_ctx ctx, const hire_gather_bench_config* cfg, hire_gather_bench_result* out) {
  if (!ctx || !cfg || !out) return invalid("null argument");
  // validate (gather_bench.hpp:27-36), the reference's messages
  if (cfg->n_groups < 1 || cfg->g < 1 || cfg->d < 1) return invalid("GatherBenchConfig: dims must be >= 1");
  if (!(cfg->fraction_selected > 0.0) || cfg->fraction_selected > 1.0)
    return invalid("GatherBenchConfig: fraction_selected must be in (0, 1]");
  if (cfg->repeats < 3) return invalid("GatherBenchConfig: repeats must be >= 3");
  const int64_t group_elems = cfg->g * cfg->d, total = cfg->n_groups * group_elems;
  const int64_t n_sel = static_cast<int64_t>(std::ceil(cfg->fraction_selected * static_cast<double>(cfg->n_groups)));
  // seeded partial Fisher-Yates in draw order (gather_bench.hpp:84-93): the
  // Rng has produced total Gaussians = 2 * ceil(total / 2) uniforms first
  std::vector<uint32_t> ids(static_cast<size_t>(cfg->n_groups));
  for (int64_t i = 0; i < cfg->n_groups; ++i) ids[i] = static_cast<uint32_t>(i);
  uint64_t counter = 2 * static_cast<uint64_t>((total + 1) / 2);
  for (int64_t i = 0; i < n_sel; ++i) {
    const uint64_t r = rng_mix64(cfg->seed, ++counter);
    const int64_t j = i + static_cast<int64_t>(r % static_cast<uint64_t>(cfg->n_groups - i));
    std::swap(ids[i], ids[j]);
  }
  ids.resize(static_cast<size_t>(n_sel));
  const int64_t sel_elems = n_sel * group_elems;
  float *src = nullptr, *dst = nullptr;
  uint32_t* dids = nullptr;
  uint64_t* sums = nullptr;
  auto release = [&] {
    cudaFree(src);
    cudaFree(dst);
    cudaFree(dids);
    cudaFree(sums);
  };
  cudaError_t e = cudaMalloc(&src, static_cast<size_t>(total) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dst, static_cast<size_t>(sel_elems) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dids, static_cast<size_t>(n_sel) * 4);
  if (e == cudaSuccess) e = cudaMalloc(&sums, static_cast<size_t>(n_sel) * 16);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dids, ids.data(), static_cast<size_t>(n_sel) * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (e != cudaSuccess) {
    release();
    return set_err(HIRE_ERR_RUNTIME, std::string("hire_gather_bench: ") + cudaGetErrorString(e));
  }
  gb_fill_kernel<<<static_cast<unsigned>(ceil_div(total, 256)), 256, 0, ctx->stream>>>(src, total, cfg->seed);
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(sel_elems / 4 + 1, 256), 16LL * ctx->num_sms));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch_copy = [&](const uint32_t* sel) {
    if (sel) {
      gb_gather_kernel<<<grid, 256, 0, ctx->stream>>>(src, sel, n_sel, group_elems, dst);
    } else if (sel_elems % 4 == 0) {  // dense: one contiguous copy of the same bytes
      gb_copy_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(sel_elems / 4, 256), 16LL * ctx->num_sms)), 256, 0,
                       ctx->stream>>>(reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), sel_elems / 4);
    } else {
      cudaMemcpyAsync(dst, src, static_cast<size_t>(sel_elems) * 4, cudaMemcpyDeviceToDevice, ctx->stream);
    }
  };
  auto time_copy = [&](const uint32_t* sel, std::vector<double>* ts) {
    launch_copy(sel);  // warm-up, discarded
    for (int64_t r = 0; r < cfg->repeats; ++r) {
      cudaEventRecord(e0, ctx->stream);
      launch_copy(sel);
      cudaEventRecord(e1, ctx->stream);
      cudaEventSynchronize(e1);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, e0, e1);
      ts->push_back(static_cast<double>(ms) * 1e6);
    }
  };
  auto median = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    const size_t n = v.size();
    return n % 2 == 1 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
  };
  std::vector<double> sparse_t, dense_t;
  time_copy(dids, &sparse_t);
  // verify the gather before the dense baseline reuses the buffer (gather_bench.hpp:116-127)
  const unsigned cg = static_cast<unsigned>(ceil_div(n_sel, 128));
  gb_checksum_kernel<<<cg, 128, 0, ctx->stream>>>(dst, nullptr, n_sel, group_elems, sums);
  gb_checksum_kernel<<<cg, 128, 0, ctx->stream>>>(src, dids, n_sel, group_elems, sums + n_sel);
  std::vector<uint64_t> hs(static_cast<size_t>(2 * n_sel));
  e = cudaMemcpyAsync(hs.data(), sums, static_cast<size_t>(2 * n_sel) * 8, cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  uint64_t gathered = 0, expected = 0;
  for (int64_t i = 0; i < n_sel; ++i) {
    gathered = gathered * 31 + hs[static_cast<size_t>(i)];
    expected = expected * 31 + hs[static_cast<size_t>(n_sel + i)];
  }
  if (e == cudaSuccess) time_copy(nullptr, &dense_t);
  if (e == cudaSuccess) e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  release();
  if (e != cudaSuccess) return set_err(HIRE_ERR_RUNTIME, std::string("hire_gather_bench: ") + cudaGetErrorString(e));
  out->sparse_ns = median(sparse_t);
  out->dense_ns = median(dense_t);
  out->efficiency_paper = out->sparse_ns / out->dense_ns;
  out->efficiency_ratio = out->dense_ns / out->sparse_ns;
  out->bytes_moved = sel_elems * 4;
  out->groups_selected = n_sel;
  out->checksum_ok = gathered == expected ? 1 : 0;
  out->reserved = 0;
  return HIRE_OK;
}

}  // extern "C"
