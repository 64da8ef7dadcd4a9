// hire_b200.hpp — drop-in replacement for the hot path of the reference's
// C++ operator API (/root/reference/proj/include/hire/*.hpp), backed by
// libhire_cuda.so through the C ABI in hire_cuda.h.
//
//   swap  #include "hire/hire.hpp" (+ approx / linalg / ffn / distributed /
//         metrics)   for   #include "hire_b200.hpp"   and link -lhire_cuda.
//
// Same namespace, type names, function names, argument meaning and error
// behaviour: std::invalid_argument with the reference's messages, clamping
// flagged rather than thrown, CUDA failures as hire::NumericError (the
// reference's exit-code-3 class). ScoreMatrix keeps the reference layout —
// d x l column-major (linalg.hpp:40-43), byte-identical to the [l][d]
// row-major matrix the device holds. Device mirrors are built on first use
// and rebuilt after any mutation through a non-const accessor.
//
// Proxies: int4 (ApproxScorer::quantized), low-rank (::low_rank) and both
// combined (::low_rank_quantized); exact_copy throws std::invalid_argument
// (not accelerated). Extensions are defaulted so
// reference call sites compile unchanged: HireConfig::{x_mode, select,
// strict, n_buckets, bucket_t}, ScoreMatrix::set_device_bf16, batched
// hire_topk_batch.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <iterator>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "hire_cuda.h"

namespace hire {

struct NumericError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class Activation : std::uint8_t { kIdentity, kRelu, kSquaredRelu };
enum class ScorerKind : std::uint8_t { kExactCopy, kLowRank, kQuantized, kLowRankQuantized };

namespace detail {

inline void throw_status(int rc) {
  if (rc == HIRE_OK) return;
  const std::string msg = hire_last_error();
  if (rc == HIRE_ERR_INVALID) throw std::invalid_argument(msg);
  throw NumericError(msg);
}

// One context (own stream + workspace) per thread: the API is reentrant.
inline hire_ctx thread_ctx() {
  struct Holder {
    hire_ctx c = nullptr;
    ~Holder() {
      if (c) hire_ctx_destroy(c);
    }
  };
  thread_local Holder h;
  if (!h.c) throw_status(hire_ctx_create(0, nullptr, 1, &h.c));
  return h.c;
}

// Device buffer with host staging helpers.
struct DevBuf {
  void* p = nullptr;
  std::int64_t n = 0;
  explicit DevBuf(std::int64_t bytes) : n(bytes) { throw_status(hire_device_alloc(bytes, &p)); }
  DevBuf(const void* host, std::int64_t bytes) : DevBuf(bytes) {
    throw_status(hire_copy(thread_ctx(), p, host, bytes, 0, 0));
  }
  ~DevBuf() { hire_device_free(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void to_host(void* dst, std::int64_t bytes) const { throw_status(hire_copy(thread_ctx(), dst, p, bytes, 1, 1)); }
};

struct MatrixHandle {
  hire_matrix h = nullptr;
  ~MatrixHandle() { hire_matrix_destroy(h); }
};
struct ScorerHandle {
  hire_scorer h = nullptr;
  std::shared_ptr<ScorerHandle> parent;  // keeps the owner alive for slices
  ~ScorerHandle() { hire_scorer_destroy(h); }
};

inline void check_dims(std::size_t matrix_rows, std::size_t x_dim, const char* op) {
  if (matrix_rows != x_dim)
    throw std::invalid_argument(std::string(op) + ": matrix has " + std::to_string(matrix_rows) +
                                " rows but x has dim " + std::to_string(x_dim));
}

// round-to-nearest-even to bf16 (approx.hpp:76-81 semantics), as raw bits
inline std::uint16_t bf16_bits(float f) {
  std::uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u += 0x7FFFu + ((u >> 16) & 1u);
  return static_cast<std::uint16_t>(u >> 16);
}

}  // namespace detail

// -------------------------------------------------------------- linalg ----
class ScoreMatrix {
 public:
  ScoreMatrix() = default;
  ScoreMatrix(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), v_(rows * cols, 0.0f) {
    if (rows == 0) throw std::invalid_argument("ScoreMatrix: rows must be >= 1");
  }
  ScoreMatrix(std::size_t rows, std::size_t cols, std::vector<float> values)
      : rows_(rows), cols_(cols), v_(std::move(values)) {
    if (rows == 0) throw std::invalid_argument("ScoreMatrix: rows must be >= 1");
    if (v_.size() != rows * cols)
      throw std::invalid_argument("ScoreMatrix: values size " + std::to_string(v_.size()) + " != " +
                                  std::to_string(rows * cols));
  }

  std::size_t rows() const { return rows_; }
  std::size_t cols() const { return cols_; }
  float at(std::size_t i, std::size_t j) const { return v_[j * rows_ + i]; }
  float& at(std::size_t i, std::size_t j) {
    ++version_;
    return v_[j * rows_ + i];
  }
  std::span<const float> col(std::size_t j) const { return {v_.data() + j * rows_, rows_}; }
  std::span<float> col(std::size_t j) {
    ++version_;
    return {v_.data() + j * rows_, rows_};
  }
  const std::vector<float>& values() const { return v_; }
  std::vector<float>& values() {
    ++version_;
    return v_;
  }
  ScoreMatrix slice_cols(std::size_t first, std::size_t count) const {
    if (first + count > cols_) throw std::invalid_argument("ScoreMatrix::slice_cols: out of range");
    ScoreMatrix s(rows_, count,
                  std::vector<float>(v_.begin() + static_cast<std::ptrdiff_t>(first * rows_),
                                     v_.begin() + static_cast<std::ptrdiff_t>((first + count) * rows_)));
    s.bf16_ = bf16_;
    return s;
  }

  // Extension: keep the device mirror in bf16 (RNE rounding) instead of fp32.
  void set_device_bf16(bool on) {
    bf16_ = on;
    ++version_;
  }

  hire_matrix device() const {
    if (!dev_ || dev_version_ != version_) {
      auto d = std::make_shared<detail::MatrixHandle>();
      const auto l = static_cast<std::int64_t>(cols_), d_ = static_cast<std::int64_t>(rows_);
      if (bf16_) {
        std::vector<std::uint16_t> b(v_.size());
        for (std::size_t i = 0; i < v_.size(); ++i) b[i] = detail::bf16_bits(v_[i]);
        detail::throw_status(hire_matrix_create(b.data(), l, d_, HIRE_BF16, 0, &d->h));
      } else {
        detail::throw_status(hire_matrix_create(v_.data(), l, d_, HIRE_F32, 0, &d->h));
      }
      dev_ = std::move(d);
      dev_version_ = version_;
    }
    return dev_->h;
  }

 private:
  std::size_t rows_ = 1, cols_ = 0;
  std::vector<float> v_;
  bool bf16_ = false;
  std::uint64_t version_ = 0;
  mutable std::uint64_t dev_version_ = ~0ull;
  mutable std::shared_ptr<detail::MatrixHandle> dev_;
};

struct TopKEntry {
  std::uint32_t index = 0;
  float value = 0.0f;
  friend bool operator==(const TopKEntry&, const TopKEntry&) = default;
};

struct TopKSet {
  std::vector<TopKEntry> entries;
  std::size_t k = 0;
  bool clamped = false;
  std::vector<std::uint32_t> indices() const {
    std::vector<std::uint32_t> out;
    out.reserve(entries.size());
    for (const auto& e : entries) out.push_back(e.index);
    return out;
  }
  friend bool operator==(const TopKSet&, const TopKSet&) = default;
};

inline std::vector<float> matvec(const ScoreMatrix& z, std::span<const float> x, Activation phi) {
  detail::check_dims(z.rows(), x.size(), "matvec");
  detail::DevBuf dx(x.data(), static_cast<std::int64_t>(x.size() * 4));
  detail::DevBuf dout(static_cast<std::int64_t>(z.cols() * 4));
  detail::throw_status(hire_matvec(detail::thread_ctx(), z.device(), dx.as<float>(), 1, static_cast<int>(phi), 0,
                                   dout.as<float>()));
  std::vector<float> out(z.cols());
  dout.to_host(out.data(), dout.n);
  return out;
}

inline TopKSet topk_select(std::span<const float> v, std::size_t k) {
  if (k == 0) throw std::invalid_argument("topk_select: k must be >= 1");
  const std::size_t kk = std::min(k, v.size());
  detail::DevBuf dv(v.data(), static_cast<std::int64_t>(v.size() * 4));
  detail::DevBuf di(static_cast<std::int64_t>(std::max<std::size_t>(kk, 1) * 4));
  detail::DevBuf dval(static_cast<std::int64_t>(std::max<std::size_t>(kk, 1) * 4));
  int cl = 0;
  detail::throw_status(hire_topk_select(detail::thread_ctx(), dv.as<float>(), 1, static_cast<std::int64_t>(v.size()),
                                        static_cast<std::int64_t>(k), di.as<std::uint32_t>(), dval.as<float>(), &cl));
  std::vector<std::uint32_t> idx(kk);
  std::vector<float> val(kk);
  di.to_host(idx.data(), static_cast<std::int64_t>(kk * 4));
  dval.to_host(val.data(), static_cast<std::int64_t>(kk * 4));
  TopKSet t;
  t.k = k;
  t.clamped = cl != 0;
  for (std::size_t i = 0; i < kk; ++i) t.entries.push_back({idx[i], val[i]});
  return t;
}

inline TopKSet topk_select(const std::vector<float>& v, std::size_t k) {
  return topk_select(std::span<const float>(v), k);
}

inline TopKSet exact_topk(const ScoreMatrix& z, std::span<const float> x, std::size_t k, Activation phi) {
  detail::check_dims(z.rows(), x.size(), "exact_topk");
  return topk_select(matvec(z, x, phi), k);
}

// -------------------------------------------------------------- approx ----
struct LowRankApprox {
  ScoreMatrix z1;  // d x r
  ScoreMatrix z2;  // l x r
  std::size_t rank = 0;
};

struct QuantizedMatrix {
  std::size_t rows = 0, cols = 0;
  std::vector<std::int8_t> codes;  // column-major, one code per entry
  std::vector<float> scales;       // one per column
  float entry(std::size_t i, std::size_t j) const { return static_cast<float>(codes[j * rows + i]) * scales[j]; }
};

// approx.hpp:49-65, computed by the device proxy build (K9) and read back.
inline QuantizedMatrix quantize_int4(const ScoreMatrix& z) {
  hire_scorer s = nullptr;
  detail::throw_status(hire_scorer_quantize(detail::thread_ctx(), z.device(), &s));
  QuantizedMatrix q;
  q.rows = z.rows();
  q.cols = z.cols();
  q.codes.resize(q.rows * q.cols);
  q.scales.resize(q.cols);
  const int rc = hire_scorer_export_q4(s, q.codes.data(), q.scales.data());
  hire_scorer_destroy(s);
  detail::throw_status(rc);
  return q;
}

class ApproxScorer {
 public:
  static ApproxScorer quantized(QuantizedMatrix q) {
    ApproxScorer a(ScorerKind::kQuantized, q.rows, q.cols, 0);
    detail::throw_status(hire_scorer_create_q4_codes(q.codes.data(), q.scales.data(),
                                                     static_cast<std::int64_t>(q.cols),
                                                     static_cast<std::int64_t>(q.rows), &a.h_->h));
    return a;
  }
  static ApproxScorer quantized(const ScoreMatrix& z) {
    ApproxScorer a(ScorerKind::kQuantized, z.rows(), z.cols(), 0);
    detail::throw_status(hire_scorer_quantize(detail::thread_ctx(), z.device(), &a.h_->h));
    return a;
  }
  static ApproxScorer low_rank(LowRankApprox lr) {
    if (lr.z1.cols() != lr.rank || lr.z2.cols() != lr.rank)
      throw std::invalid_argument("ApproxScorer: low-rank factors do not match rank " + std::to_string(lr.rank));
    ApproxScorer a(ScorerKind::kLowRank, lr.z1.rows(), lr.z2.rows(), lr.rank);
    std::vector<float> z2t(a.l_ * a.r_);  // device layout [l][r]
    for (std::size_t j = 0; j < a.l_; ++j)
      for (std::size_t q = 0; q < a.r_; ++q) z2t[j * a.r_ + q] = lr.z2.at(j, q);
    detail::throw_status(hire_scorer_create_lowrank(lr.z1.values().data(), z2t.data(),
                                                    static_cast<std::int64_t>(a.d_),
                                                    static_cast<std::int64_t>(a.l_),
                                                    static_cast<std::int64_t>(a.r_), HIRE_F32, 0, &a.h_->h));
    return a;
  }
  static ApproxScorer exact_copy(const ScoreMatrix&) {
    throw std::invalid_argument("ApproxScorer::exact_copy: not accelerated on the B200 path");
  }
  // approx.hpp:342-347: both factors through the int4 rule (per column, the
  // device K9 build), scored over the dequantized entries — the reference's
  // arithmetic (approx.hpp:500-516), bit-identical in strict mode.
  static ApproxScorer low_rank_quantized(const LowRankApprox& lr) {
    if (lr.z1.cols() != lr.rank || lr.z2.cols() != lr.rank)
      throw std::invalid_argument("ApproxScorer: low-rank factors do not match rank " + std::to_string(lr.rank));
    auto dequant = [](const ScoreMatrix& z) {
      const QuantizedMatrix q = quantize_int4(z);
      std::vector<float> v(q.rows * q.cols);
      for (std::size_t j = 0; j < q.cols; ++j)
        for (std::size_t i = 0; i < q.rows; ++i) v[j * q.rows + i] = q.entry(i, j);
      return ScoreMatrix(q.rows, q.cols, std::move(v));
    };
    ApproxScorer a = low_rank(LowRankApprox{dequant(lr.z1), dequant(lr.z2), lr.rank});
    a.kind_ = ScorerKind::kLowRankQuantized;
    return a;
  }

  ScorerKind kind() const { return kind_; }
  std::size_t input_dim() const { return d_; }
  std::size_t output_dim() const { return l_; }
  hire_scorer device() const { return h_->h; }

  // approx.hpp:382-411 (fp32 x, the reference's scorer)
  std::vector<float> scores(std::span<const float> x, Activation phi) const {
    if (x.size() != d_)
      throw std::invalid_argument("ApproxScorer::scores: scorer expects dim " + std::to_string(d_) +
                                  " but x has dim " + std::to_string(x.size()));
    detail::DevBuf dx(x.data(), static_cast<std::int64_t>(d_ * 4));
    detail::DevBuf dout(static_cast<std::int64_t>(l_ * 4));
    detail::throw_status(hire_scores(detail::thread_ctx(), h_->h, dx.as<float>(), 1, static_cast<int>(phi),
                                     HIRE_X_FP32, 0, dout.as<float>()));
    std::vector<float> out(l_);
    dout.to_host(out.data(), dout.n);
    return out;
  }

  // approx.hpp:415-445 — a view of outputs [first, first+count)
  ApproxScorer slice_cols(std::size_t first, std::size_t count) const {
    if (first + count > l_) throw std::invalid_argument("ApproxScorer::slice_cols: out of range");
    ApproxScorer s(kind_, d_, count, r_);
    s.h_->parent = h_;
    detail::throw_status(hire_scorer_slice(h_->h, static_cast<std::int64_t>(first),
                                           static_cast<std::int64_t>(count), &s.h_->h));
    return s;
  }

 private:
  ApproxScorer(ScorerKind k, std::size_t d, std::size_t l, std::size_t r)
      : kind_(k), d_(d), l_(l), r_(r), h_(std::make_shared<detail::ScorerHandle>()) {}
  ScorerKind kind_;
  std::size_t d_, l_, r_;
  std::shared_ptr<detail::ScorerHandle> h_;
};

// ---------------------------------------------------------------- hire ----
struct HireConfig {
  std::size_t k = 1;
  std::size_t k_prime = 1;
  Activation phi = Activation::kIdentity;
  // B200 extensions (defaults reproduce the reference's semantics)
  int x_mode = HIRE_X_FP32;        // HIRE_X_INT8: int4 x int8 -> int32 proxy
  int select = HIRE_SELECT_EXACT;  // HIRE_SELECT_BUCKETED: literal bucket rule
  bool strict = true;              // sequential fp32 like the reference
  std::size_t n_buckets = 0, bucket_t = 0;

  hire_topk_params params() const {
    hire_topk_params p{};
    p.k = static_cast<std::int64_t>(k);
    p.k_prime = static_cast<std::int64_t>(k_prime);
    p.phi = static_cast<int>(phi);
    p.x_mode = x_mode;
    p.select = select;
    p.strict = strict ? 1 : 0;
    p.n_buckets = static_cast<std::int64_t>(n_buckets);
    p.bucket_t = static_cast<std::int64_t>(bucket_t);
    return p;
  }
};

inline void validate(const HireConfig& cfg) {
  if (cfg.k < 1) throw std::invalid_argument("HireConfig: k must be >= 1");
  if (cfg.k > cfg.k_prime)
    throw std::invalid_argument("HireConfig: k (" + std::to_string(cfg.k) + ") must be <= k_prime (" +
                                std::to_string(cfg.k_prime) + ")");
}

struct CandidateSet {
  std::vector<std::uint32_t> indices;
  ScorerKind origin = ScorerKind::kExactCopy;
  bool contains(std::uint32_t idx) const { return std::binary_search(indices.begin(), indices.end(), idx); }
};

struct HireResult {
  TopKSet topk;
  CandidateSet candidates;
};

// Batched hire_topk: B queries x [B*d] -> B results (one device call).
inline std::vector<HireResult> hire_topk_batch(std::span<const float> x, std::size_t B, const ScoreMatrix& z,
                                               const ApproxScorer& a, const HireConfig& cfg) {
  validate(cfg);
  if (B == 0 || x.size() != B * z.rows()) detail::check_dims(z.rows(), B ? x.size() / B : 0, "hire_topk");
  const hire_topk_params p = cfg.params();
  std::vector<std::uint32_t> cand(B * cfg.k_prime), idx(B * cfg.k);
  std::vector<float> val(B * cfg.k);
  std::int64_t nc = 0, nt = 0;
  int cl = 0;
  detail::throw_status(hire_topk_host(detail::thread_ctx(), z.device(), a.device(), x.data(),
                                      static_cast<std::int64_t>(B), &p, cand.data(), idx.data(), val.data(), nullptr,
                                      &nc, &nt, &cl));
  std::vector<HireResult> out(B);
  for (std::size_t b = 0; b < B; ++b) {
    out[b].candidates.origin = a.kind();
    out[b].candidates.indices.assign(cand.begin() + static_cast<std::ptrdiff_t>(b * cfg.k_prime),
                                     cand.begin() + static_cast<std::ptrdiff_t>(b * cfg.k_prime + nc));
    out[b].topk.k = cfg.k;
    out[b].topk.clamped = cl != 0;
    for (std::int64_t i = 0; i < nt; ++i) out[b].topk.entries.push_back({idx[b * cfg.k + i], val[b * cfg.k + i]});
  }
  return out;
}

// hire.hpp:50-86
inline HireResult hire_topk(std::span<const float> x, const ScoreMatrix& z, const ApproxScorer& a,
                            const HireConfig& cfg) {
  validate(cfg);
  detail::check_dims(z.rows(), x.size(), "hire_topk");
  if (a.input_dim() != z.rows() || a.output_dim() != z.cols())
    throw std::invalid_argument("hire_topk: scorer is " + std::to_string(a.input_dim()) + "x" +
                                std::to_string(a.output_dim()) + " but Z is " + std::to_string(z.rows()) + "x" +
                                std::to_string(z.cols()));
  return hire_topk_batch(x, 1, z, a, cfg).front();
}

struct SparseDistribution {
  std::vector<TopKEntry> entries;  // value = probability
  double total() const {
    double s = 0.0;
    for (const auto& e : entries) s += e.value;
    return s;
  }
};

// hire.hpp:123-144
inline SparseDistribution softmax_topk(const ScoreMatrix& w, std::span<const float> x, const ApproxScorer& a,
                                       const HireConfig& cfg) {
  if (cfg.phi != Activation::kIdentity) throw std::invalid_argument("softmax_topk: phi must be identity");
  validate(cfg);
  detail::check_dims(w.rows(), x.size(), "hire_topk");
  const hire_topk_params p = cfg.params();
  std::vector<std::uint32_t> idx(cfg.k);
  std::vector<float> val(cfg.k), prob(cfg.k);
  std::int64_t nc = 0, nt = 0;
  int cl = 0;
  detail::throw_status(hire_topk_host(detail::thread_ctx(), w.device(), a.device(), x.data(), 1, &p, nullptr,
                                      idx.data(), val.data(), prob.data(), &nc, &nt, &cl));
  SparseDistribution d;
  for (std::int64_t i = 0; i < nt; ++i) d.entries.push_back({idx[i], prob[i]});
  return d;
}

// ----------------------------------------------------------------- ffn ----
struct GroupedFFN {
  ScoreMatrix u;  // d x m
  ScoreMatrix v;  // d x m
  std::size_t group_size = 1;
  Activation phi = Activation::kRelu;
  std::size_t dim() const { return u.rows(); }
  std::size_t hidden() const { return u.cols(); }
  std::size_t num_groups() const { return hidden() / group_size; }
};

struct GroupIndexSet {
  std::vector<std::uint32_t> ids;
  friend bool operator==(const GroupIndexSet&, const GroupIndexSet&) = default;
};

struct GroupSparseResult {
  std::vector<float> output;
  GroupIndexSet selected;
};

// ffn.hpp:211-219. x_mode / strict extensions default to the reference.
inline GroupSparseResult ffn_group_sparse(const GroupedFFN& f, std::span<const float> x, const ApproxScorer& a,
                                          std::size_t k, std::size_t k_prime, int x_mode = HIRE_X_FP32,
                                          bool strict = true) {
  detail::check_dims(f.dim(), x.size(), "group_proxy");
  hire_ffn_params p{};
  p.k = static_cast<std::int64_t>(k);
  p.k_prime = static_cast<std::int64_t>(k_prime);
  p.group_size = static_cast<std::int64_t>(f.group_size);
  p.phi = static_cast<int>(f.phi);
  p.x_mode = x_mode;
  p.strict = strict ? 1 : 0;
  const std::size_t kg = f.group_size ? k / f.group_size : 0;
  GroupSparseResult r;
  r.output.resize(f.dim());
  r.selected.ids.resize(kg);
  detail::throw_status(hire_ffn_host(detail::thread_ctx(), f.u.device(), f.v.device(), a.device(), x.data(), 1, &p,
                                     r.selected.ids.data(), r.output.data()));
  return r;
}

// ffn.hpp:65-76: every unit, ascending (strict = the reference's arithmetic).
inline std::vector<float> ffn_dense(const GroupedFFN& f, std::span<const float> x, bool strict = true) {
  detail::check_dims(f.dim(), x.size(), "ffn_dense");
  detail::DevBuf dx(x.data(), static_cast<std::int64_t>(x.size() * 4));
  detail::DevBuf dout(static_cast<std::int64_t>(f.dim() * 4));
  detail::throw_status(hire_ffn_dense_run(detail::thread_ctx(), f.u.device(), f.v.device(), dx.as<float>(), 1,
                                          static_cast<int>(f.phi), strict ? 1 : 0, dout.as<float>()));
  std::vector<float> out(f.dim());
  dout.to_host(out.data(), dout.n);
  return out;
}

// ffn.hpp:44-47
struct CommonPathFFN {
  GroupedFFN dense_part;
  GroupedFFN sparse_part;
};

// ffn.hpp:223-234: ffn_dense(dense part) + ffn_group_sparse(sparse part).
inline std::vector<float> ffn_common_path(const CommonPathFFN& c, std::span<const float> x, const ApproxScorer& a,
                                          std::size_t k, std::size_t k_prime, int x_mode = HIRE_X_FP32,
                                          bool strict = true) {
  detail::check_dims(c.sparse_part.dim(), x.size(), "ffn_common_path");
  hire_ffn_params p{};
  p.k = static_cast<std::int64_t>(k);
  p.k_prime = static_cast<std::int64_t>(k_prime);
  p.group_size = static_cast<std::int64_t>(c.sparse_part.group_size);
  p.phi = static_cast<int>(c.sparse_part.phi);
  p.x_mode = x_mode;
  p.strict = strict ? 1 : 0;
  detail::DevBuf dx(x.data(), static_cast<std::int64_t>(x.size() * 4));
  detail::DevBuf dout(static_cast<std::int64_t>(c.sparse_part.dim() * 4));
  const bool has_dense = c.dense_part.hidden() > 0;
  detail::throw_status(hire_ffn_common_path_run(detail::thread_ctx(), has_dense ? c.dense_part.u.device() : nullptr,
                                                has_dense ? c.dense_part.v.device() : nullptr,
                                                c.sparse_part.u.device(), c.sparse_part.v.device(), a.device(),
                                                dx.as<float>(), 1, &p, dout.as<float>()));
  std::vector<float> out(c.sparse_part.dim());
  dout.to_host(out.data(), dout.n);
  return out;
}

// ffn.hpp:237-253: union of the per-sample selections (dynamic overlap).
inline GroupIndexSet union_group_select(const GroupedFFN& f, std::span<const std::vector<float>> xs,
                                        const ApproxScorer& a, std::size_t k, std::size_t k_prime,
                                        int x_mode = HIRE_X_FP32, bool strict = true) {
  if (xs.empty()) throw std::invalid_argument("union_group_select: no input samples");
  std::vector<float> flat;
  for (const auto& x : xs) {
    detail::check_dims(f.dim(), x.size(), "union_group_select");
    flat.insert(flat.end(), x.begin(), x.end());
  }
  hire_ffn_params p{};
  p.k = static_cast<std::int64_t>(k);
  p.k_prime = static_cast<std::int64_t>(k_prime);
  p.group_size = static_cast<std::int64_t>(f.group_size);
  p.phi = static_cast<int>(f.phi);
  p.x_mode = x_mode;
  p.strict = strict ? 1 : 0;
  detail::DevBuf dx(flat.data(), static_cast<std::int64_t>(flat.size() * 4));
  detail::DevBuf dids(static_cast<std::int64_t>(std::max<std::size_t>(f.num_groups(), 1) * 4));
  std::int64_t n = 0;
  detail::throw_status(hire_ffn_union_select(detail::thread_ctx(), f.u.device(), a.device(), dx.as<float>(),
                                             static_cast<std::int64_t>(xs.size()), &p, dids.as<std::uint32_t>(), &n));
  GroupIndexSet r;
  r.ids.resize(static_cast<std::size_t>(n));
  if (n) dids.to_host(r.ids.data(), n * 4);
  return r;
}

// metrics.hpp:68-88: |union| / (s * k_groups).
inline double overlap_ratio(const std::vector<GroupIndexSet>& per_sample_sets, std::size_t k_groups) {
  if (per_sample_sets.empty()) throw std::invalid_argument("overlap_ratio: no sample sets");
  if (k_groups < 1) throw std::invalid_argument("overlap_ratio: k_groups must be >= 1");
  std::vector<std::uint32_t> merged;
  for (const auto& s : per_sample_sets) {
    if (s.ids.size() != k_groups)
      throw std::invalid_argument("overlap_ratio: sample selected " + std::to_string(s.ids.size()) +
                                  " groups, expected " + std::to_string(k_groups));
    std::vector<std::uint32_t> next;
    std::set_union(merged.begin(), merged.end(), s.ids.begin(), s.ids.end(), std::back_inserter(next));
    merged.swap(next);
  }
  return static_cast<double>(merged.size()) / (static_cast<double>(per_sample_sets.size()) * k_groups);
}

// ----------------------------------------------------------- distributed --
struct Shard {
  ScoreMatrix z;
  ApproxScorer a;
  std::size_t offset = 0;
};

struct ShardedScorer {
  std::vector<Shard> shards;
  std::size_t input_dim = 0;
  std::size_t total_cols = 0;
  std::size_t num_shards() const { return shards.size(); }
  // the unsharded handles the single-GPU emulation runs on
  std::shared_ptr<ScoreMatrix> whole_z;
  std::shared_ptr<ApproxScorer> whole_a;
};

struct CommReport {
  std::size_t bytes_gathered = 0;
  std::vector<std::size_t> candidates_per_shard;
  std::size_t values_concatenated = 0;
};

struct DaTopkResult {
  TopKSet topk;
  CommReport comm;
};

// distributed.hpp:41-63 (width rule: first l % s shards one wider)
inline ShardedScorer shard(const ScoreMatrix& z, const ApproxScorer& a, std::size_t s) {
  if (s < 1) throw std::invalid_argument("shard: s must be >= 1");
  if (s > z.cols())
    throw std::invalid_argument("shard: s = " + std::to_string(s) + " exceeds l = " + std::to_string(z.cols()));
  if (a.input_dim() != z.rows() || a.output_dim() != z.cols())
    throw std::invalid_argument("shard: scorer shape does not match Z");
  ShardedScorer out;
  out.input_dim = z.rows();
  out.total_cols = z.cols();
  out.whole_z = std::make_shared<ScoreMatrix>(z);
  out.whole_a = std::make_shared<ApproxScorer>(a);
  const std::size_t base = z.cols() / s, extra = z.cols() % s;
  std::size_t offset = 0;
  for (std::size_t i = 0; i < s; ++i) {
    const std::size_t width = base + (i < extra ? 1 : 0);
    out.shards.push_back({z.slice_cols(offset, width), a.slice_cols(offset, width), offset});
    offset += width;
  }
  return out;
}

// distributed.hpp:73-134, all shards on this GPU (the single-process
// simulation the reference performs; one device call, no host loop).
inline DaTopkResult da_topk(const ShardedScorer& sh, std::span<const float> x, const HireConfig& cfg) {
  validate(cfg);
  detail::check_dims(sh.input_dim, x.size(), "da_topk");
  const std::size_t s = sh.num_shards();
  if (s == 0) throw std::invalid_argument("da_topk: no shards");
  const hire_topk_params p = cfg.params();
  detail::DevBuf dx(x.data(), static_cast<std::int64_t>(x.size() * 4));
  detail::DevBuf di(static_cast<std::int64_t>(cfg.k * 4)), dv(static_cast<std::int64_t>(cfg.k * 4));
  std::int64_t n = 0;
  int cl = 0;
  detail::throw_status(hire_da_topk_emulated(detail::thread_ctx(), sh.whole_z->device(), sh.whole_a->device(),
                                             static_cast<int>(s), dx.as<float>(), 1, &p, HIRE_MERGE_PER_SHARD, 0,
                                             di.as<std::uint32_t>(), dv.as<float>(), &n, &cl));
  std::vector<std::uint32_t> idx(static_cast<std::size_t>(n));
  std::vector<float> val(static_cast<std::size_t>(n));
  di.to_host(idx.data(), n * 4);
  dv.to_host(val.data(), n * 4);
  DaTopkResult r;
  r.topk.k = cfg.k;
  r.topk.clamped = cl != 0;
  for (std::int64_t i = 0; i < n; ++i) r.topk.entries.push_back({idx[i], val[i]});
  for (const auto& shd : sh.shards) {
    const std::size_t c = std::min(cfg.k_prime / s, shd.z.cols());
    r.comm.candidates_per_shard.push_back(c);
    r.comm.bytes_gathered += c * sh.input_dim * 4;  // distributed.hpp:124
  }
  r.comm.values_concatenated = r.topk.entries.size();
  return r;
}

struct DaGroupSparseResult {
  std::vector<float> output;
  GroupIndexSet selected;
  std::vector<std::size_t> groups_per_shard;
};

// distributed.hpp:145-206 (single-GPU emulation of the sharded FFN).
inline DaGroupSparseResult da_group_sparse(const GroupedFFN& f, std::span<const float> x, const ApproxScorer& a,
                                           std::size_t k, std::size_t k_prime, std::size_t s,
                                           int x_mode = HIRE_X_FP32, bool strict = true) {
  detail::check_dims(f.dim(), x.size(), "group_proxy");
  hire_ffn_params p{};
  p.k = static_cast<std::int64_t>(k);
  p.k_prime = static_cast<std::int64_t>(k_prime);
  p.group_size = static_cast<std::int64_t>(f.group_size);
  p.phi = static_cast<int>(f.phi);
  p.x_mode = x_mode;
  p.strict = strict ? 1 : 0;
  const std::size_t kg = f.group_size ? k / f.group_size : 0;
  detail::DevBuf dx(x.data(), static_cast<std::int64_t>(x.size() * 4));
  detail::DevBuf dsel(static_cast<std::int64_t>(std::max<std::size_t>(kg, 1) * 4));
  detail::DevBuf dout(static_cast<std::int64_t>(f.dim() * 4));
  detail::throw_status(hire_da_ffn_emulated(detail::thread_ctx(), f.u.device(), f.v.device(), a.device(),
                                            static_cast<int>(s), dx.as<float>(), 1, &p, 0,
                                            dsel.as<std::uint32_t>(), dout.as<float>()));
  DaGroupSparseResult r;
  r.output.resize(f.dim());
  r.selected.ids.resize(kg);
  dout.to_host(r.output.data(), static_cast<std::int64_t>(f.dim() * 4));
  dsel.to_host(r.selected.ids.data(), static_cast<std::int64_t>(kg * 4));
  r.groups_per_shard.assign(s, kg / s);
  return r;
}

// ------------------------------------------------------------- metrics ----
struct RecallReport {
  double recall = 0.0;
  std::size_t intersection_k = 0;
  bool top1_agree = false;
};

// metrics.hpp:23-34 (host set arithmetic over index sets)
inline RecallReport recall(const CandidateSet& candidates, const TopKSet& exact) {
  RecallReport r;
  if (exact.entries.empty()) return r;
  for (const auto& e : exact.entries) r.intersection_k += candidates.contains(e.index);
  r.recall = static_cast<double>(r.intersection_k) / static_cast<double>(exact.entries.size());
  r.top1_agree = candidates.contains(exact.entries.front().index);
  return r;
}

// gather_bench.hpp:18-152 — the group-gather microbenchmark, on the GPU
// (device buffers, CUDA-event timing; same selection, checksum and messages)
struct GatherBenchConfig {
  std::size_t n_groups = 4096;
  std::size_t g = 8;
  std::size_t d = 128;
  double fraction_selected = 0.25;
  std::size_t repeats = 9;
  std::uint64_t seed = 0;
};

struct GatherBenchResult {
  double sparse_ns = 0.0;
  double dense_ns = 0.0;
  double efficiency_paper = 0.0;
  double efficiency_ratio = 0.0;
  std::size_t bytes_moved = 0;
  std::size_t groups_selected = 0;
  bool checksum_ok = false;
};

inline GatherBenchResult run_gather_bench(const GatherBenchConfig& cfg) {
  hire_gather_bench_config c{static_cast<std::int64_t>(cfg.n_groups), static_cast<std::int64_t>(cfg.g),
                             static_cast<std::int64_t>(cfg.d), cfg.fraction_selected,
                             static_cast<std::int64_t>(cfg.repeats), cfg.seed};
  hire_gather_bench_result r{};
  detail::throw_status(hire_gather_bench(detail::thread_ctx(), &c, &r));
  GatherBenchResult o;
  o.sparse_ns = r.sparse_ns;
  o.dense_ns = r.dense_ns;
  o.efficiency_paper = r.efficiency_paper;
  o.efficiency_ratio = r.efficiency_ratio;
  o.bytes_moved = static_cast<std::size_t>(r.bytes_moved);
  o.groups_selected = static_cast<std::size_t>(r.groups_selected);
  o.checksum_ok = r.checksum_ok != 0;
  return o;
}

// metrics.hpp:43-64 — the paper's parameter-bytes cost model (host integer
// arithmetic; like the reference, the int4 term leaves out the scales)
struct CostReport {
  std::uint64_t bytes_baseline = 0;
  std::uint64_t bytes_lr = 0;
  std::uint64_t bytes_q = 0;
  std::uint64_t bytes_lrq = 0;
  bool lr_no_saving = false;
  bool q_no_saving = false;
  bool lrq_no_saving = false;
};

inline CostReport param_bytes(std::uint64_t d, std::uint64_t l, std::uint64_t r, std::uint64_t k_prime) {
  if (d < 1 || l < 1 || r < 1) throw std::invalid_argument("param_bytes: dims must be positive");
  CostReport c;
  c.bytes_baseline = 2 * d * l;
  c.bytes_lr = 2 * (d * r + r * l + d * k_prime);
  c.bytes_q = (d * l + 1) / 2 + 2 * d * k_prime;
  c.bytes_lrq = (d * r + r * l + 1) / 2 + 2 * d * k_prime;
  c.lr_no_saving = c.bytes_lr >= c.bytes_baseline;
  c.q_no_saving = c.bytes_q >= c.bytes_baseline;
  c.lrq_no_saving = c.bytes_lrq >= c.bytes_baseline;
  return c;
}

}  // namespace hire
