// ref_shim.cpp — C-ABI shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle/hire_oracle.c). Compiled by
// oracle/Makefile with -I/root/reference/proj/include into
// oracle/_ref/libhire_ref.so; no reference source is copied into this repo.
// This library is "the reference itself run here": it validates the C
// restatement, generates the golden fixtures in tests/golden/, and is the
// CPU baseline timed by bench.py (cpu_baseline.kind = "reference").
//
// Pointer layout: a row-major float W[l][d] is byte-identical to the
// reference's column-major d x l ScoreMatrix (linalg.hpp:40-43).
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "hire/approx.hpp"
#include "hire/instance.hpp"
#include "hire/distributed.hpp"
#include "hire/ffn.hpp"
#include "hire/hire.hpp"
#include "hire/linalg.hpp"
#include "hire/metrics.hpp"
#include "hire/rng.hpp"

#define REF_EXPORT extern "C" __attribute__((visibility("default")))

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

hire::ScoreMatrix to_matrix(const float* w, uint64_t cols, uint64_t d) {
  return hire::ScoreMatrix(d, cols, std::vector<float>(w, w + cols * d));
}

hire::Activation act(int phi) { return static_cast<hire::Activation>(phi); }

// Scorer kinds: 0 exact copy of W, 1 low-rank (z1 [r][d], z2 [l][r]),
// 2 int4 quantized (codes [l][d], scales [l]), 3 low-rank quantized.
struct Scorer {
  hire::ApproxScorer a;
};
}  // namespace

REF_EXPORT const char* ref_last_error() { return g_err.c_str(); }

// ------------------------------------------------------------------ rng --
REF_EXPORT void ref_rng_u64(uint64_t seed, uint64_t n, uint64_t* out) {
  hire::Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
REF_EXPORT void ref_rng_uniform(uint64_t seed, uint64_t n, double* out) {
  hire::Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.next_uniform();
}
REF_EXPORT uint64_t ref_derive_seed(uint64_t seed, uint64_t stream) {
  return hire::derive_seed(seed, stream);
}
REF_EXPORT void ref_gen_vector(uint64_t dim, uint64_t seed, float* out) {
  hire::Rng r(seed);
  for (uint64_t i = 0; i < dim; ++i) out[i] = r.next_gaussian_f();
}

// gen_instance (instance.hpp:58-83) into [l][d] (column j of Z = row j)
REF_EXPORT int ref_gen_instance(uint64_t d, uint64_t l, uint64_t seed, int decaying, float* out) {
  try {
    const hire::ScoreMatrix z =
        hire::gen_instance(d, l, seed, decaying ? hire::Spectrum::kDecaying : hire::Spectrum::kFlat);
    for (uint64_t j = 0; j < l; ++j) {
      const auto c = z.col(j);
      std::memcpy(out + j * d, c.data(), d * sizeof(float));
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ------------------------------------------------------------- objects --
REF_EXPORT void* ref_matrix_create(const float* w, uint64_t cols, uint64_t d) {
  try {
    return new hire::ScoreMatrix(to_matrix(w, cols, d));
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
REF_EXPORT void ref_matrix_destroy(void* m) {
  delete static_cast<hire::ScoreMatrix*>(m);
}

REF_EXPORT void* ref_scorer_create(int kind, const void* m_exact,
                                   const float* z1, const float* z2,
                                   const int8_t* codes, const float* scales,
                                   uint64_t cols, uint64_t d, uint64_t r) {
  try {
    switch (kind) {
      case 0:
        return new Scorer{hire::ApproxScorer::exact_copy(
            *static_cast<const hire::ScoreMatrix*>(m_exact))};
      case 1:
      case 3: {
        hire::LowRankApprox lr;
        lr.rank = r;
        lr.z1 = hire::ScoreMatrix(d, r, std::vector<float>(z1, z1 + d * r));
        lr.z2 = hire::ScoreMatrix(cols, r);
        for (uint64_t j = 0; j < cols; ++j)
          for (uint64_t q = 0; q < r; ++q) lr.z2.at(j, q) = z2[j * r + q];
        return new Scorer{kind == 1 ? hire::ApproxScorer::low_rank(std::move(lr))
                                    : hire::ApproxScorer::low_rank_quantized(lr)};
      }
      case 2: {
        hire::QuantizedMatrix q;
        q.rows = d;
        q.cols = cols;
        q.codes.assign(codes, codes + cols * d);
        q.scales.assign(scales, scales + cols);
        return new Scorer{hire::ApproxScorer::quantized(std::move(q))};
      }
    }
    throw std::invalid_argument("ref_scorer_create: bad kind");
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
REF_EXPORT void ref_scorer_destroy(void* s) { delete static_cast<Scorer*>(s); }

// ----------------------------------------------------------- primitives --
REF_EXPORT int ref_quantize_int4(const float* w, uint64_t cols, uint64_t d,
                                 int8_t* codes, float* scales) {
  try {
    const hire::QuantizedMatrix q = hire::quantize_int4(to_matrix(w, cols, d));
    std::memcpy(codes, q.codes.data(), q.codes.size());
    std::memcpy(scales, q.scales.data(), q.scales.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// HIRQ bytes (approx.hpp:551-564); returns the byte count written.
REF_EXPORT uint64_t ref_write_quantized(const int8_t* codes, const float* scales,
                                        uint64_t cols, uint64_t d, uint8_t* out,
                                        uint64_t cap) {
  hire::QuantizedMatrix q;
  q.rows = d;
  q.cols = cols;
  q.codes.assign(codes, codes + cols * d);
  q.scales.assign(scales, scales + cols);
  std::stringstream ss;
  hire::write_quantized(ss, q);
  const std::string b = ss.str();
  if (b.size() <= cap) std::memcpy(out, b.data(), b.size());
  return b.size();
}

REF_EXPORT float ref_round_bf16(float f) { return hire::round_bf16(f); }

REF_EXPORT int ref_scores(const void* scorer, const float* x, uint64_t d,
                          int phi, float* out) {
  try {
    const auto v = static_cast<const Scorer*>(scorer)->a.scores(
        std::span<const float>(x, d), act(phi));
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_EXPORT int ref_matvec(const void* m, const float* x, uint64_t d, int phi,
                          float* out) {
  try {
    const auto v = hire::matvec(*static_cast<const hire::ScoreMatrix*>(m),
                                std::span<const float>(x, d), act(phi));
    std::memcpy(out, v.data(), v.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_EXPORT int ref_topk_select(const float* v, uint64_t n, uint64_t k,
                               uint32_t* idx, float* val, uint64_t* n_out,
                               int* clamped) {
  try {
    const hire::TopKSet t = hire::topk_select(std::span<const float>(v, n), k);
    for (size_t i = 0; i < t.entries.size(); ++i) {
      idx[i] = t.entries[i].index;
      val[i] = t.entries[i].value;
    }
    *n_out = t.entries.size();
    *clamped = t.clamped;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// --------------------------------------------------------------- hire --
REF_EXPORT int ref_hire_topk(const void* m, const void* scorer, const float* x,
                             uint64_t d, uint64_t k, uint64_t k_prime, int phi,
                             uint32_t* cand, uint64_t* n_cand, uint32_t* idx,
                             float* val, uint64_t* n_top, int* clamped) {
  try {
    const hire::HireResult r = hire::hire_topk(
        std::span<const float>(x, d), *static_cast<const hire::ScoreMatrix*>(m),
        static_cast<const Scorer*>(scorer)->a, hire::HireConfig{k, k_prime, act(phi)});
    std::memcpy(cand, r.candidates.indices.data(),
                r.candidates.indices.size() * sizeof(uint32_t));
    *n_cand = r.candidates.indices.size();
    for (size_t i = 0; i < r.topk.entries.size(); ++i) {
      idx[i] = r.topk.entries[i].index;
      val[i] = r.topk.entries[i].value;
    }
    *n_top = r.topk.entries.size();
    *clamped = r.topk.clamped;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_EXPORT int ref_softmax_topk(const void* m, const void* scorer,
                                const float* x, uint64_t d, uint64_t k,
                                uint64_t k_prime, uint32_t* idx, float* prob,
                                uint64_t* n_out) {
  try {
    const hire::SparseDistribution s = hire::softmax_topk(
        *static_cast<const hire::ScoreMatrix*>(m), std::span<const float>(x, d),
        static_cast<const Scorer*>(scorer)->a,
        hire::HireConfig{k, k_prime, hire::Activation::kIdentity});
    for (size_t i = 0; i < s.entries.size(); ++i) {
      idx[i] = s.entries[i].index;
      prob[i] = s.entries[i].value;
    }
    *n_out = s.entries.size();
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Batched hire_topk over B queries on `threads` host threads (pure and
// reentrant per SPEC.md:90). Used as the CPU baseline; outputs only the
// top-k (k entries per query).
REF_EXPORT int ref_hire_topk_batch(const void* m, const void* scorer,
                                   const float* x, uint64_t batch, uint64_t d,
                                   uint64_t k, uint64_t k_prime, int phi,
                                   uint32_t* idx, float* val, int threads) {
  std::vector<std::thread> pool;
  std::vector<int> rc(threads > 0 ? threads : 1, 0);
  const int nt = threads > 0 ? threads : 1;
  for (int t = 0; t < nt; ++t) {
    pool.emplace_back([&, t] {
      try {
        for (uint64_t b = t; b < batch; b += nt) {
          const hire::HireResult r = hire::hire_topk(
              std::span<const float>(x + b * d, d),
              *static_cast<const hire::ScoreMatrix*>(m),
              static_cast<const Scorer*>(scorer)->a,
              hire::HireConfig{k, k_prime, act(phi)});
          for (size_t i = 0; i < r.topk.entries.size(); ++i) {
            idx[b * k + i] = r.topk.entries[i].index;
            val[b * k + i] = r.topk.entries[i].value;
          }
        }
      } catch (const std::exception& e) {
        rc[t] = fail(e);
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int v : rc)
    if (v) return v;
  return 0;
}

// ---------------------------------------------------------------- ffn --
namespace {
struct Ffn {
  hire::GroupedFFN f;
};
}  // namespace

REF_EXPORT void* ref_ffn_create(const float* u, const float* v, uint64_t m,
                                uint64_t d, uint64_t g, int phi) {
  try {
    auto* p = new Ffn{hire::GroupedFFN{to_matrix(u, m, d), to_matrix(v, m, d),
                                       g, act(phi)}};
    hire::validate(p->f);
    return p;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}
REF_EXPORT void ref_ffn_destroy(void* f) { delete static_cast<Ffn*>(f); }

REF_EXPORT int ref_ffn_group_sparse(const void* ffn, const void* scorer,
                                    const float* x, uint64_t d, uint64_t k,
                                    uint64_t k_prime, uint32_t* ids,
                                    uint64_t* n_ids, float* out) {
  try {
    const auto r = hire::ffn_group_sparse(static_cast<const Ffn*>(ffn)->f,
                                          std::span<const float>(x, d),
                                          static_cast<const Scorer*>(scorer)->a,
                                          k, k_prime);
    std::memcpy(ids, r.selected.ids.data(), r.selected.ids.size() * 4);
    *n_ids = r.selected.ids.size();
    std::memcpy(out, r.output.data(), r.output.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_EXPORT int ref_ffn_group_sparse_batch(const void* ffn, const void* scorer,
                                          const float* x, uint64_t batch,
                                          uint64_t d, uint64_t k,
                                          uint64_t k_prime, float* out,
                                          int threads) {
  const int nt = threads > 0 ? threads : 1;
  std::vector<std::thread> pool;
  std::vector<int> rc(nt, 0);
  for (int t = 0; t < nt; ++t) {
    pool.emplace_back([&, t] {
      try {
        for (uint64_t b = t; b < batch; b += nt) {
          const auto r = hire::ffn_group_sparse(
              static_cast<const Ffn*>(ffn)->f,
              std::span<const float>(x + b * d, d),
              static_cast<const Scorer*>(scorer)->a, k, k_prime);
          std::memcpy(out + b * d, r.output.data(), d * 4);
        }
      } catch (const std::exception& e) {
        rc[t] = fail(e);
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int v : rc)
    if (v) return v;
  return 0;
}

REF_EXPORT int ref_ffn_dense(const void* ffn, const float* x, uint64_t d,
                             float* out) {
  try {
    const auto o = hire::ffn_dense(static_cast<const Ffn*>(ffn)->f,
                                   std::span<const float>(x, d));
    std::memcpy(out, o.data(), o.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// -------------------------------------------------------- distributed --
REF_EXPORT int ref_da_topk(const void* m, const void* scorer, const float* x,
                           uint64_t d, uint64_t s, uint64_t k, uint64_t k_prime,
                           int phi, uint32_t* idx, float* val, uint64_t* n_out,
                           int* clamped, uint64_t* bytes_gathered) {
  try {
    const hire::ShardedScorer sh =
        hire::shard(*static_cast<const hire::ScoreMatrix*>(m),
                    static_cast<const Scorer*>(scorer)->a, s);
    const hire::DaTopkResult r = hire::da_topk(
        sh, std::span<const float>(x, d), hire::HireConfig{k, k_prime, act(phi)});
    for (size_t i = 0; i < r.topk.entries.size(); ++i) {
      idx[i] = r.topk.entries[i].index;
      val[i] = r.topk.entries[i].value;
    }
    *n_out = r.topk.entries.size();
    *clamped = r.topk.clamped;
    *bytes_gathered = r.comm.bytes_gathered;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

REF_EXPORT int ref_da_group_sparse(const void* ffn, const void* scorer,
                                   const float* x, uint64_t d, uint64_t k,
                                   uint64_t k_prime, uint64_t s, uint32_t* ids,
                                   uint64_t* n_ids, float* out) {
  try {
    const auto r = hire::da_group_sparse(
        static_cast<const Ffn*>(ffn)->f, std::span<const float>(x, d),
        static_cast<const Scorer*>(scorer)->a, k, k_prime, s);
    std::memcpy(ids, r.selected.ids.data(), r.selected.ids.size() * 4);
    *n_ids = r.selected.ids.size();
    std::memcpy(out, r.output.data(), r.output.size() * 4);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ------------------------------------------------------------ metrics --
REF_EXPORT double ref_recall(const uint32_t* cand_sorted, uint64_t n_cand,
                             const uint32_t* exact_idx, const float* exact_val,
                             uint64_t n_exact, uint64_t* hits, int* top1) {
  hire::CandidateSet c;
  c.indices.assign(cand_sorted, cand_sorted + n_cand);
  hire::TopKSet t;
  for (uint64_t i = 0; i < n_exact; ++i) t.entries.push_back({exact_idx[i], exact_val[i]});
  const hire::RecallReport r = hire::recall(c, t);
  *hits = r.intersection_k;
  *top1 = r.top1_agree;
  return r.recall;
}

REF_EXPORT void ref_param_bytes(uint64_t d, uint64_t l, uint64_t r,
                                uint64_t k_prime, uint64_t out[4]) {
  const hire::CostReport c = hire::param_bytes(d, l, r, k_prime);
  out[0] = c.bytes_baseline;
  out[1] = c.bytes_lr;
  out[2] = c.bytes_q;
  out[3] = c.bytes_lrq;
}
