// Drop-in check: reference-style call sites compiled against hire_b200.hpp.
// Reads an instance from argv[1] (raw little-endian: u32 V, u32 d, u32 k,
// u32 kp, f32 W[V*d] row-major (= column-major d x V), f32 x[d]) and prints
// the results as whitespace-separated text for tests/test_cpp_dropin.py.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "hire_b200.hpp"

int main(int argc, char** argv) {
  // 1) hand trace of test_hire.cpp:60-75 with a prescribed scorer built as a
  //    rank-1 low-rank proxy: t = <(1,0), x> = 2, z2_j = s_j / 2.
  {
    hire::ScoreMatrix z(2, 4, {1, 0, 0, 1, 1, 1, -1, -1});
    const std::vector<float> x = {2, 1};
    hire::LowRankApprox lr{hire::ScoreMatrix(2, 1, {1, 0}),
                           hire::ScoreMatrix(4, 1, {2.1f / 2, 0.9f / 2, 2.9f / 2, 0.0f}), 1};
    const auto a = hire::ApproxScorer::low_rank(lr);
    const auto r = hire::hire_topk(x, z, a, hire::HireConfig{2, 3, hire::Activation::kRelu});
    std::printf("trace %zu %u %u %u | %u %g %u %g\n", r.candidates.indices.size(), r.candidates.indices[0],
                r.candidates.indices[1], r.candidates.indices[2], r.topk.entries[0].index, r.topk.entries[0].value,
                r.topk.entries[1].index, r.topk.entries[1].value);
    try {
      hire::hire_topk(x, z, a, hire::HireConfig{5, 4});
      std::printf("validate none\n");
    } catch (const std::invalid_argument& e) {
      std::printf("validate %s\n", e.what());
    }
  }
  if (argc < 2) return 0;
  std::ifstream in(argv[1], std::ios::binary);
  uint32_t hdr[4];
  in.read(reinterpret_cast<char*>(hdr), 16);
  const uint32_t V = hdr[0], d = hdr[1], k = hdr[2], kp = hdr[3];
  std::vector<float> w(static_cast<size_t>(V) * d), x(d);
  in.read(reinterpret_cast<char*>(w.data()), w.size() * 4);
  in.read(reinterpret_cast<char*>(x.data()), x.size() * 4);
  const hire::ScoreMatrix z(d, V, w);
  // 2) int4 proxy: quantize_int4 (device) + hire_topk + softmax_topk
  const hire::QuantizedMatrix q = hire::quantize_int4(z);
  const auto a = hire::ApproxScorer::quantized(q);
  const auto r = hire::hire_topk(x, z, a, hire::HireConfig{k, kp, hire::Activation::kIdentity});
  std::printf("cand");
  for (auto c : r.candidates.indices) std::printf(" %u", c);
  std::printf("\ntop");
  for (auto& e : r.topk.entries) std::printf(" %u:%.9g", e.index, e.value);
  const auto dist = hire::softmax_topk(z, x, a, hire::HireConfig{k, kp});
  std::printf("\nprob");
  for (auto& e : dist.entries) std::printf(" %u:%.9g", e.index, e.value);
  // 3) DA-TOP-k over 2 shards
  const auto sh = hire::shard(z, a, 2);
  const auto da = hire::da_topk(sh, x, hire::HireConfig{k - k % 2, kp - kp % 2});
  std::printf("\nda");
  for (auto& e : da.topk.entries) std::printf(" %u:%.9g", e.index, e.value);
  std::printf("\nbytes %zu\n", da.comm.bytes_gathered);
  // 4) FFN on the same matrix as U and V
  hire::GroupedFFN f{z, z, 1, hire::Activation::kRelu};
  const auto fr = hire::ffn_group_sparse(f, x, a, k, kp);
  std::printf("ffn");
  for (auto id : fr.selected.ids) std::printf(" %u", id);
  std::printf("\nffnout");
  for (float o : fr.output) std::printf(" %.9g", o);
  std::printf("\nrecall %.6f\n", hire::recall(r.candidates, hire::exact_topk(z, x, k, hire::Activation::kIdentity)).recall);
  // batch-level FFN levers: dense, common path (dense = sparse = f), union over {x, -x}
  const auto dense = hire::ffn_dense(f, x);
  std::printf("dense");
  for (float o : dense) std::printf(" %.9g", o);
  const auto cp = hire::ffn_common_path(hire::CommonPathFFN{f, f}, x, a, k, kp);
  std::printf("\ncommon");
  for (float o : cp) std::printf(" %.9g", o);
  std::vector<float> xn(x.size());
  for (size_t i = 0; i < x.size(); ++i) xn[i] = -x[i];
  const std::vector<std::vector<float>> xs = {x, xn};
  const auto un = hire::union_group_select(f, xs, a, k, kp);
  std::printf("\nunion");
  for (auto id : un.ids) std::printf(" %u", id);
  const auto s2 = hire::ffn_group_sparse(f, xn, a, k, kp).selected;
  std::printf("\noverlap %.9g\n", hire::overlap_ratio({fr.selected, s2}, k));
  return 0;
}
