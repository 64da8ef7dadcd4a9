/*
 * hire_oracle.c — CPU restatement of the HiRE approximate top-k hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker for the CUDA
 * path in paper_2402_09360_b200/csrc. It may be loaded only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg; the product path
 * never links, loads or calls it.
 *
 * Every function restates the algorithm of the reference header-only
 * library (/root/reference/proj/include/hire/*.hpp, cited file:line) in
 * plain C, or — where BASELINE.json asks for semantics the reference does
 * not have — states the extension explicitly (marked EXTENSION).
 *
 * Pinning: tests/test_oracle.py checks this restatement against the
 * reference's own known-answer tests (restated), against golden vectors in
 * tests/golden/ produced by the compiled reference (oracle/_ref, built from
 * the unmodified headers by oracle/Makefile), and, when oracle/_ref is
 * present, against the reference directly on seeded random instances.
 *
 * Build with -ffp-contract=off: the reference's CMake build uses no -march,
 * so GCC never contracts `acc += a*b` into an FMA there; neither may we.
 *
 * Layout convention: the reference's ScoreMatrix Z is d x l column-major
 * (linalg.hpp:40-43,65-73); column j is contiguous. That is byte-identical
 * to a row-major W[l][d], which is what every pointer here is.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EXPORT __attribute__((visibility("default")))

enum { PHI_IDENTITY = 0, PHI_RELU = 1, PHI_SQRELU = 2 };

/* ---------------------------------------------------------------- rng -- */
/* rng.hpp:20-40 — counter-based splitmix64: out_i = mix64(seed+(i+1)*G). */
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* The counter-th output (counter counts from 1, rng.hpp:25). */
ORC_EXPORT uint64_t orc_rng_u64(uint64_t seed, uint64_t counter) {
  return mix64(seed + counter * 0x9E3779B97F4A7C15ULL);
}

/* rng.hpp:32-34 — uniform from the high 53 bits. */
ORC_EXPORT double orc_rng_uniform(uint64_t seed, uint64_t counter) {
  return (double)(orc_rng_u64(seed, counter) >> 11) * 0x1.0p-53;
}

/* rng.hpp:64-67 */
ORC_EXPORT uint64_t orc_derive_seed(uint64_t seed, uint64_t stream) {
  return orc_rng_u64(seed ^ (0xA5A5A5A55A5A5A5AULL + stream), 1);
}

/* instance.hpp:16-21 (gen_vector) over rng.hpp:38-50 (Box-Muller, cos then
 * sin of each pair). Gaussian number n uses uniforms 2*(n/2)+1, +2. The
 * range [first, first+count) lets callers fill huge arrays in parallel. */
ORC_EXPORT void orc_gen_gaussian_range(uint64_t seed, uint64_t first,
                                       uint64_t count, float* out) {
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (uint64_t n = first; n < first + count; ++n) {
    const uint64_t pair = n / 2;
    const double u1 = orc_rng_uniform(seed, 2 * pair + 1);
    const double u2 = orc_rng_uniform(seed, 2 * pair + 2);
    const double radius = sqrt(-2.0 * log1p(-u1));
    const double angle = two_pi * u2;
    const double g = (n & 1) ? radius * sin(angle) : radius * cos(angle);
    out[n - first] = (float)g;
  }
}

ORC_EXPORT void orc_gen_vector(uint64_t dim, uint64_t seed, float* out) {
  orc_gen_gaussian_range(seed, 0, dim, out);
}

/* ------------------------------------------------------------- linalg -- */
/* linalg.hpp:31-38 */
static inline float apply_phi(int phi, float z) {
  switch (phi) {
    case PHI_RELU: return z > 0.0f ? z : 0.0f;
    case PHI_SQRELU: return z > 0.0f ? z * z : 0.0f;
    default: return z;
  }
}
ORC_EXPORT float orc_apply_phi(int phi, float z) { return apply_phi(phi, z); }

/* linalg.hpp:129-133 — value descending, index ascending. */
static inline int ranks_before(float va, uint32_t ia, float vb, uint32_t ib) {
  if (va != vb) return va > vb;
  return ia < ib;
}

typedef struct { uint32_t index; float value; } orc_entry;

static int cmp_rank(const void* a, const void* b) {
  const orc_entry* p = (const orc_entry*)a;
  const orc_entry* q = (const orc_entry*)b;
  if (ranks_before(p->value, p->index, q->value, q->index)) return -1;
  if (ranks_before(q->value, q->index, p->value, p->index)) return 1;
  return 0;
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return (x > y) - (x < y);
}

/* linalg.hpp:140-146 — phi(<W_j, x>), sequential ascending fp32. */
ORC_EXPORT float orc_column_score(const float* w_row, const float* x,
                                  uint64_t d, int phi) {
  float acc = 0.0f;
  for (uint64_t i = 0; i < d; ++i) acc += w_row[i] * x[i];
  return apply_phi(phi, acc);
}

/* linalg.hpp:148-154 */
ORC_EXPORT void orc_matvec(const float* w, uint64_t rows, uint64_t d,
                           const float* x, int phi, float* out) {
  for (uint64_t j = 0; j < rows; ++j)
    out[j] = orc_column_score(w + j * d, x, d, phi);
}

/* linalg.hpp:157-176 — top-k by ranks_before; k > n clamps and flags.
 * Any correct selection under this total order (unique indices) equals
 * std::partial_sort's result. Returns the number of entries written, or
 * (uint64_t)-1 for k == 0 (the reference throws invalid_argument). */
ORC_EXPORT uint64_t orc_topk_select(const float* v, uint64_t n, uint64_t k,
                                    uint32_t* out_idx, float* out_val,
                                    int* clamped) {
  if (k == 0) return (uint64_t)-1;
  *clamped = 0;
  if (k > n) { k = n; *clamped = 1; }
  orc_entry* order = (orc_entry*)malloc(sizeof(orc_entry) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) { order[i].index = (uint32_t)i; order[i].value = v[i]; }
  qsort(order, n, sizeof(orc_entry), cmp_rank);
  for (uint64_t i = 0; i < k; ++i) {
    out_idx[i] = order[i].index;
    if (out_val) out_val[i] = order[i].value;
  }
  free(order);
  return k;
}

/* ------------------------------------------------------------- approx -- */
/* approx.hpp:41-45 — round half away from zero, clamped to [-7, 7]. */
static inline int rhaz_clamp(float v, int lim) {
  const float r = v >= 0.0f ? floorf(v + 0.5f) : ceilf(v - 0.5f);
  const int c = (int)r;
  return c < -lim ? -lim : (c > lim ? lim : c);
}

/* approx.hpp:49-65 — per-column (= per W row) absmax/7 scale, 1 for an
 * all-zero column; code = RHAZ(w / scale) clamped to [-7, 7]. */
ORC_EXPORT void orc_quantize_int4(const float* w, uint64_t rows, uint64_t d,
                                  int8_t* codes, float* scales) {
  for (uint64_t j = 0; j < rows; ++j) {
    const float* c = w + j * d;
    float max_abs = 0.0f;
    for (uint64_t i = 0; i < d; ++i) {
      const float a = fabsf(c[i]);
      max_abs = max_abs > a ? max_abs : a;  /* std::max(max_abs, a) */
    }
    const float scale = max_abs > 0.0f ? max_abs / 7.0f : 1.0f;
    scales[j] = scale;
    for (uint64_t i = 0; i < d; ++i)
      codes[j * d + i] = (int8_t)rhaz_clamp(c[i] / scale, 7);
  }
}

/* approx.hpp:551-564 (HIRQ payload) — two codes per byte, low nibble first,
 * in storage order; an odd trailing code gets a zero high nibble. */
ORC_EXPORT void orc_pack_int4(const int8_t* codes, uint64_t n, uint8_t* out) {
  for (uint64_t i = 0; i < n; i += 2) {
    const uint8_t lo = (uint8_t)codes[i] & 0x0F;
    const uint8_t hi = i + 1 < n ? ((uint8_t)codes[i + 1] & 0x0F) : 0;
    out[i / 2] = (uint8_t)(lo | (hi << 4));
  }
}

/* approx.hpp:575-585 — sign-extending unpack. */
ORC_EXPORT void orc_unpack_int4(const uint8_t* in, uint64_t n, int8_t* codes) {
  for (uint64_t i = 0; i < n; ++i) {
    const uint8_t nib = (i & 1) ? (in[i / 2] >> 4) : (in[i / 2] & 0x0F);
    codes[i] = (int8_t)(nib & 0x08 ? (nib | 0xF0) : nib);
  }
}

/* approx.hpp:76-81 — bf16 round-to-nearest-even, widened back to f32. */
ORC_EXPORT float orc_round_bf16(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return f;
  u += 0x7FFFu + ((u >> 16) & 1u);
  u &= 0xFFFF0000u;
  float r;
  memcpy(&r, &u, 4);
  return r;
}

ORC_EXPORT void orc_round_bf16_array(const float* in, uint64_t n, float* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = orc_round_bf16(in[i]);
}

/* approx.hpp:395-403 — quantized scorer, fp32 x ("fp-x" mode):
 * s_j = phi(sum_i (code_ji * scale_j) * x_i), ascending i. */
ORC_EXPORT void orc_q4_scores_fpx(const int8_t* codes, const float* scales,
                                  uint64_t rows, uint64_t d, const float* x,
                                  int phi, float* out) {
  for (uint64_t j = 0; j < rows; ++j) {
    const int8_t* c = codes + j * d;
    const float s = scales[j];
    float acc = 0.0f;
    for (uint64_t i = 0; i < d; ++i) acc += ((float)c[i] * s) * x[i];
    out[j] = apply_phi(phi, acc);
  }
}

/* EXTENSION (BASELINE.json cfg2: "scored against an int8-quantised x"; the
 * reference has no int8 path). x is quantised with the same
 * symmetric absmax/RHAZ rule as quantize_int4 (approx.hpp:41-65) but to
 * [-127, 127]: sx = max|x|/127 (1 if x == 0), xq = RHAZ(x / sx). */
ORC_EXPORT void orc_quantize_x_int8(const float* x, uint64_t d, int8_t* xq,
                                    float* sx_out) {
  float max_abs = 0.0f;
  for (uint64_t i = 0; i < d; ++i) {
    const float a = fabsf(x[i]);
    max_abs = max_abs > a ? max_abs : a;
  }
  const float sx = max_abs > 0.0f ? max_abs / 127.0f : 1.0f;
  for (uint64_t i = 0; i < d; ++i) xq[i] = (int8_t)rhaz_clamp(x[i] / sx, 127);
  *sx_out = sx;
}

/* EXTENSION — integer-mode score: acc_j = sum_i code_ji * xq_i exactly in
 * int32 (order-free), s_j = phi(float(acc_j) * (scale_j * sx)). The two fp32
 * multiplies happen in exactly this order on the GPU too, so scores — and
 * therefore candidate sets — are bit-exact. */
ORC_EXPORT void orc_q4_scores_int8(const int8_t* codes, const float* scales,
                                   uint64_t rows, uint64_t d, const float* x,
                                   int phi, float* out) {
  int8_t* xq = (int8_t*)malloc(d ? d : 1);
  float sx;
  orc_quantize_x_int8(x, d, xq, &sx);
  for (uint64_t j = 0; j < rows; ++j) {
    const int8_t* c = codes + j * d;
    int32_t acc = 0;
    for (uint64_t i = 0; i < d; ++i) acc += (int32_t)c[i] * (int32_t)xq[i];
    const float cs = scales[j] * sx;
    out[j] = apply_phi(phi, (float)acc * cs);
  }
  free(xq);
}

/* approx.hpp:477-496 — low-rank scores: t_q = sum_i Z1[i,q] x_i ascending i,
 * then s_j = phi(sum_q Z2[j,q] t_q) ascending q. z1 is stored [r][d] (each
 * reference column z1.col(q) contiguous — byte-identical to the reference's
 * column-major d x r); z2 is stored [rows][r] (row j = the r coefficients of
 * output j, i.e. the transpose of the reference's column-major l x r). */
ORC_EXPORT void orc_lowrank_t(const float* z1, uint64_t d, uint64_t r,
                              const float* x, float* t) {
  for (uint64_t q = 0; q < r; ++q) {
    const float* c = z1 + q * d;
    float acc = 0.0f;
    for (uint64_t i = 0; i < d; ++i) acc += c[i] * x[i];
    t[q] = acc;
  }
}

ORC_EXPORT void orc_lowrank_scores_from_t(const float* z2, uint64_t rows,
                                          uint64_t r, const float* t, int phi,
                                          float* out) {
  for (uint64_t j = 0; j < rows; ++j) {
    float acc = 0.0f;
    for (uint64_t q = 0; q < r; ++q) acc += z2[j * r + q] * t[q];
    out[j] = apply_phi(phi, acc);
  }
}

ORC_EXPORT void orc_lowrank_scores(const float* z1, const float* z2, uint64_t d,
                                   uint64_t rows, uint64_t r, const float* x,
                                   int phi, float* out) {
  float* t = (float*)malloc(sizeof(float) * (r ? r : 1));
  orc_lowrank_t(z1, d, r, x, t);
  orc_lowrank_scores_from_t(z2, rows, r, t, phi, out);
  free(t);
}

/* ------------------------------------------------------ bucket rules -- */
/* Contiguous partition of [0, n) into `parts`, the first n % parts one
 * wider — the shard width rule of distributed.hpp:53-57. */
ORC_EXPORT void orc_partition(uint64_t n, uint64_t parts, uint64_t i,
                              uint64_t* first, uint64_t* width) {
  const uint64_t base = n / parts, extra = n % parts;
  *first = i * base + (i < extra ? i : extra);
  *width = base + (i < extra ? 1 : 0);
}

/* EXTENSION — BASELINE.json cfg3's literal bucketed rule ("approx top-k'
 * with n buckets"): per bucket (distributed.hpp:53-57 width rule, the
 * per-shard candidate step of da_topk at :101-102) keep the top-t by
 * ranks_before, then take the top-k' of the pooled survivors. Writes the
 * selected indices sorted ascending; returns their count. *clamped is set
 * when k' exceeds the survivor count. */
ORC_EXPORT uint64_t orc_bucketed_select(const float* s, uint64_t n,
                                        uint64_t n_buckets, uint64_t t,
                                        uint64_t k_prime, uint32_t* out_idx,
                                        int* clamped) {
  orc_entry* pool = (orc_entry*)malloc(sizeof(orc_entry) * (n_buckets * t + 1));
  orc_entry* tmp = (orc_entry*)malloc(sizeof(orc_entry) * (n + 1));
  uint64_t np = 0;
  for (uint64_t b = 0; b < n_buckets; ++b) {
    uint64_t first, width;
    orc_partition(n, n_buckets, b, &first, &width);
    for (uint64_t i = 0; i < width; ++i) {
      tmp[i].index = (uint32_t)(first + i);
      tmp[i].value = s[first + i];
    }
    qsort(tmp, width, sizeof(orc_entry), cmp_rank);
    const uint64_t take = t < width ? t : width;
    for (uint64_t i = 0; i < take; ++i) pool[np++] = tmp[i];
  }
  *clamped = 0;
  uint64_t k = k_prime;
  if (k > np) { k = np; *clamped = 1; }
  qsort(pool, np, sizeof(orc_entry), cmp_rank);
  for (uint64_t i = 0; i < k; ++i) out_idx[i] = pool[i].index;
  qsort(out_idx, k, sizeof(uint32_t), cmp_u32);
  free(pool);
  free(tmp);
  return k;
}

/* --------------------------------------------------------- hire core -- */
/* Selection modes for the candidate step. */
enum { SEL_EXACT = 0, SEL_BUCKETED = 1 };

/* hire.hpp:50-86 (hire_topk) given the approximate scores (already phi'd,
 * approx.hpp:382): candidates = top-k' (exact rule: linalg.hpp:157-176, or
 * the bucketed EXTENSION above), sorted ascending (hire.hpp:65-67); exact
 * rescoring of each candidate row (hire.hpp:69-72 -> linalg.hpp:140-146);
 * top-k by ranks_before (hire.hpp:74-80); clamp flag (hire.hpp:84).
 * Returns 0, or 1 on an invalid config (validate, hire.hpp:22-29). */
ORC_EXPORT int orc_hire_topk(const float* w, uint64_t rows, uint64_t d,
                             const float* x, const float* approx, uint64_t k,
                             uint64_t k_prime, int phi, int sel_mode,
                             uint64_t n_buckets, uint64_t bucket_t,
                             uint32_t* cand_idx, uint64_t* n_cand,
                             uint32_t* top_idx, float* top_val,
                             uint64_t* n_top, int* clamped) {
  if (k < 1 || k > k_prime) return 1;
  int cl = 0;
  uint64_t nc;
  if (sel_mode == SEL_BUCKETED) {
    nc = orc_bucketed_select(approx, rows, n_buckets, bucket_t, k_prime,
                             cand_idx, &cl);
  } else {
    float* tmpv = (float*)malloc(sizeof(float) * (k_prime < rows ? k_prime : rows) + 4);
    nc = orc_topk_select(approx, rows, k_prime, cand_idx, tmpv, &cl);
    free(tmpv);
    qsort(cand_idx, nc, sizeof(uint32_t), cmp_u32);
  }
  orc_entry* rescored = (orc_entry*)malloc(sizeof(orc_entry) * (nc + 1));
  for (uint64_t i = 0; i < nc; ++i) {
    rescored[i].index = cand_idx[i];
    rescored[i].value = orc_column_score(w + (uint64_t)cand_idx[i] * d, x, d, phi);
  }
  const uint64_t take = k < nc ? k : nc;
  qsort(rescored, nc, sizeof(orc_entry), cmp_rank);
  for (uint64_t i = 0; i < take; ++i) {
    top_idx[i] = rescored[i].index;
    top_val[i] = rescored[i].value;
  }
  *n_cand = nc;
  *n_top = take;
  *clamped = cl || take < k;
  free(rescored);
  return 0;
}

/* hire.hpp:123-144 — softmax over the retained top-k exact logits:
 * p_i = exp((double)v_i - v_max) as double, stored as float; sum of the
 * double p_i; renormalised value = float(float(p_i) / sum). */
ORC_EXPORT void orc_softmax_topk_probs(const float* top_val, uint64_t n,
                                       float* probs) {
  if (n == 0) return;
  const float max_logit = top_val[0];
  double sum = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double p = exp((double)top_val[i] - max_logit);
    probs[i] = (float)p;
    sum += p;
  }
  for (uint64_t i = 0; i < n; ++i) probs[i] = (float)((double)probs[i] / sum);
}

/* metrics.hpp:23-34 — recall of the exact top-k inside the (ascending)
 * candidate set; top-1 agreement. */
ORC_EXPORT double orc_recall(const uint32_t* cand_sorted, uint64_t n_cand,
                             const uint32_t* exact_idx, uint64_t n_exact,
                             uint64_t* hits, int* top1) {
  uint64_t h = 0;
  *top1 = 0;
  for (uint64_t e = 0; e < n_exact; ++e) {
    const uint32_t key = exact_idx[e];
    const int found = bsearch(&key, cand_sorted, n_cand, sizeof(uint32_t), cmp_u32) != NULL;
    h += found;
    if (e == 0) *top1 = found;
  }
  *hits = h;
  return n_exact ? (double)h / (double)n_exact : 0.0;
}

/* --------------------------------------------------------------- ffn -- */
/* ffn.hpp:102-121 (group_proxy): Phi_j = sum_{t<g} |s_{jg+t}| over the
 * phi'd approximate scores, ascending t. */
ORC_EXPORT void orc_group_proxy(const float* scores, uint64_t m, uint64_t g,
                                float* proxy) {
  for (uint64_t j = 0; j < m / g; ++j) {
    float acc = 0.0f;
    for (uint64_t t = 0; t < g; ++t) acc += fabsf(scores[j * g + t]);
    proxy[j] = acc;
  }
}

/* ffn.hpp:175-201 (select_groups) with ffn.hpp:125-131 (exact_group_proxy)
 * and the checks of ffn.hpp:133-149. scores are the phi'd approximate
 * scores of U's m units. Writes the selected group ids ascending.
 * Returns 0 or 1 (invalid argument). */
ORC_EXPORT int orc_select_groups(const float* u, uint64_t m, uint64_t d,
                                 uint64_t g, int phi, const float* x,
                                 const float* scores, uint64_t k,
                                 uint64_t k_prime, uint32_t* out_ids,
                                 uint64_t* n_out) {
  if (g < 1 || m % g != 0) return 1;
  if (k < 1 || k % g != 0 || k_prime % g != 0 || k > k_prime || k_prime > m)
    return 1;
  const uint64_t ng = m / g;
  float* proxy = (float*)malloc(sizeof(float) * ng);
  orc_group_proxy(scores, m, g, proxy);
  const uint64_t kpg = k_prime / g;
  uint32_t* cidx = (uint32_t*)malloc(sizeof(uint32_t) * (kpg + 1));
  float* cval = (float*)malloc(sizeof(float) * (kpg + 1));
  int cl;
  const uint64_t nc = orc_topk_select(proxy, ng, kpg, cidx, cval, &cl);
  orc_entry* ex = (orc_entry*)malloc(sizeof(orc_entry) * (nc + 1));
  for (uint64_t i = 0; i < nc; ++i) {  /* candidates in rank order, :185-186 */
    float acc = 0.0f;
    for (uint64_t t = 0; t < g; ++t)
      acc += fabsf(orc_column_score(u + (cidx[i] * g + t) * d, x, d, phi));
    ex[i].index = cidx[i];
    ex[i].value = acc;
  }
  const uint64_t take = (k / g) < nc ? (k / g) : nc;
  qsort(ex, nc, sizeof(orc_entry), cmp_rank);
  for (uint64_t i = 0; i < take; ++i) out_ids[i] = ex[i].index;
  qsort(out_ids, take, sizeof(uint32_t), cmp_u32);
  *n_out = take;
  free(proxy); free(cidx); free(cval); free(ex);
  return 0;
}

/* ffn.hpp:154-171 (ffn_apply_groups): out = sum over groups ascending, units
 * ascending within the group, of phi(<U_u, x>) * V_u, accumulated
 * elementwise in fp32 (out[i] += act * v[i]). */
ORC_EXPORT void orc_ffn_apply_groups(const float* u, const float* v,
                                     uint64_t d, uint64_t g, int phi,
                                     const float* x, const uint32_t* ids,
                                     uint64_t n_ids, float* out) {
  for (uint64_t i = 0; i < d; ++i) out[i] = 0.0f;
  for (uint64_t n = 0; n < n_ids; ++n) {
    for (uint64_t t = 0; t < g; ++t) {
      const uint64_t unit = (uint64_t)ids[n] * g + t;
      const float act = orc_column_score(u + unit * d, x, d, phi);
      const float* vu = v + unit * d;
      for (uint64_t i = 0; i < d; ++i) out[i] += act * vu[i];
    }
  }
}

/* ffn.hpp:211-219 */
ORC_EXPORT int orc_ffn_group_sparse(const float* u, const float* v, uint64_t m,
                                    uint64_t d, uint64_t g, int phi,
                                    const float* x, const float* scores,
                                    uint64_t k, uint64_t k_prime,
                                    uint32_t* out_ids, uint64_t* n_out,
                                    float* out) {
  const int rc = orc_select_groups(u, m, d, g, phi, x, scores, k, k_prime,
                                   out_ids, n_out);
  if (rc) return rc;
  orc_ffn_apply_groups(u, v, d, g, phi, x, out_ids, *n_out, out);
  return 0;
}

/* ffn.hpp:65-76 — dense FFN (the dense baseline). */
ORC_EXPORT void orc_ffn_dense(const float* u, const float* v, uint64_t m,
                              uint64_t d, int phi, const float* x, float* out) {
  for (uint64_t i = 0; i < d; ++i) out[i] = 0.0f;
  for (uint64_t j = 0; j < m; ++j) {
    const float act = orc_column_score(u + j * d, x, d, phi);
    for (uint64_t i = 0; i < d; ++i) out[i] += act * v[j * d + i];
  }
}

/* ------------------------------------------------------- distributed -- */
/* Quota of shard i: the reference requires s | k (distributed.hpp:79-85) and
 * then uses k/s everywhere. EXTENSION for s not dividing k (cfg2/cfg5's
 * k = 410 at s = 4, 8): the first k % s shards take one more, mirroring the
 * width rule of distributed.hpp:53-57. Identical to k/s when s | k. */
ORC_EXPORT uint64_t orc_quota(uint64_t k, uint64_t s, uint64_t i) {
  return k / s + (i < k % s ? 1 : 0);
}

enum { MERGE_PER_SHARD = 0, MERGE_GLOBAL = 1 };

/* distributed.hpp:73-134 (da_topk). scores = the full phi'd approximate
 * score vector; shard i's scores are its slice (ApproxScorer::slice_cols,
 * approx.hpp:415-445, pinned equal to the score slice by the reference
 * test test_approx.cpp:344-361).
 *  MERGE_PER_SHARD (reference): per shard top-(k'_i) candidates, exact
 *    rescoring with global indices, local top-(k_i); pooled and sorted.
 *  MERGE_GLOBAL (EXTENSION, BASELINE.json cfg4): per shard top-(k'_i)
 *    candidates and exact rescoring; all k' exact pairs pooled; global
 *    top-k of the pool.
 * `uneven` = 0 reproduces the reference's divisibility errors; 1 enables the
 * orc_quota rule. Returns 0 or 1 (invalid argument). bytes_gathered follows
 * distributed.hpp:124 (candidates * d * 4). */
ORC_EXPORT int orc_da_topk(const float* w, uint64_t rows, uint64_t d,
                           const float* x, const float* scores, uint64_t s,
                           uint64_t k, uint64_t k_prime, int phi,
                           int merge_mode, int uneven, uint32_t* top_idx,
                           float* top_val, uint64_t* n_top, int* clamped,
                           uint64_t* bytes_gathered) {
  if (k < 1 || k > k_prime || s < 1 || s > rows) return 1;
  if (!uneven && (k % s != 0 || k_prime % s != 0)) return 1;
  orc_entry* pooled = (orc_entry*)malloc(sizeof(orc_entry) * (k_prime + k + 1));
  uint64_t np = 0;
  *clamped = 0;
  *bytes_gathered = 0;
  for (uint64_t i = 0; i < s; ++i) {
    uint64_t first, width;
    orc_partition(rows, s, i, &first, &width);
    const uint64_t kl = orc_quota(k, s, i), kpl = orc_quota(k_prime, s, i);
    if (kl > width) { free(pooled); return 1; }
    uint32_t* cidx = (uint32_t*)malloc(sizeof(uint32_t) * (kpl + 1));
    int cl = 0;
    const uint64_t nc = orc_topk_select(scores + first, width, kpl, cidx, NULL, &cl);
    if (cl) *clamped = 1;
    qsort(cidx, nc, sizeof(uint32_t), cmp_u32);
    orc_entry* rs = (orc_entry*)malloc(sizeof(orc_entry) * (nc + 1));
    for (uint64_t c = 0; c < nc; ++c) {
      rs[c].index = (uint32_t)(first + cidx[c]);
      rs[c].value = orc_column_score(w + (first + cidx[c]) * d, x, d, phi);
    }
    uint64_t take = nc;
    if (merge_mode == MERGE_PER_SHARD) {
      take = kl < nc ? kl : nc;
      qsort(rs, nc, sizeof(orc_entry), cmp_rank);
    }
    for (uint64_t c = 0; c < take; ++c) pooled[np++] = rs[c];
    *bytes_gathered += nc * d * 4;
    free(cidx);
    free(rs);
  }
  qsort(pooled, np, sizeof(orc_entry), cmp_rank);
  uint64_t out_n = np;
  if (merge_mode == MERGE_GLOBAL && out_n > k) out_n = k;
  if (merge_mode == MERGE_GLOBAL && np < k) *clamped = 1;
  for (uint64_t c = 0; c < out_n; ++c) {
    top_idx[c] = pooled[c].index;
    top_val[c] = pooled[c].value;
  }
  *n_top = out_n;
  free(pooled);
  return 0;
}

/* distributed.hpp:145-206 (da_group_sparse): groups sharded contiguously,
 * per-shard quotas k/(s g) and k'/(s g) (candidate quota clamped to the
 * shard width, :192), local select_groups on the shard's slice of U and of
 * the scores, union of the selections (sorted), exact FFN over the union.
 * `uneven` as in orc_da_topk. Returns 0 or 1. */
ORC_EXPORT int orc_da_group_sparse(const float* u, const float* v, uint64_t m,
                                   uint64_t d, uint64_t g, int phi,
                                   const float* x, const float* scores,
                                   uint64_t k, uint64_t k_prime, uint64_t s,
                                   int uneven, uint32_t* out_ids,
                                   uint64_t* n_out, float* out) {
  if (g < 1 || m % g != 0) return 1;
  if (k < 1 || k % g != 0 || k_prime % g != 0 || k > k_prime || k_prime > m)
    return 1;
  const uint64_t ng = m / g;
  if (s < 1 || s > ng) return 1;
  const uint64_t kg = k / g, kpg = k_prime / g;
  if (!uneven && (kg % s != 0 || kpg % s != 0)) return 1;
  uint64_t n = 0;
  for (uint64_t i = 0; i < s; ++i) {
    uint64_t fg, width;
    orc_partition(ng, s, i, &fg, &width);
    const uint64_t kgl = orc_quota(kg, s, i);
    uint64_t kpl = orc_quota(kpg, s, i);
    if (kgl > width) return 1;
    if (kpl > width) kpl = width;
    uint64_t nl = 0;
    const int rc = orc_select_groups(u + fg * g * d, width * g, d, g, phi, x,
                                     scores + fg * g, kgl * g, kpl * g,
                                     out_ids + n, &nl);
    if (rc) return rc;
    for (uint64_t c = 0; c < nl; ++c) out_ids[n + c] += (uint32_t)fg;
    n += nl;
  }
  qsort(out_ids, n, sizeof(uint32_t), cmp_u32);
  *n_out = n;
  orc_ffn_apply_groups(u, v, d, g, phi, x, out_ids, n, out);
  return 0;
}

/* metrics.hpp:51-64 — the paper's paramsize cost model. */
ORC_EXPORT void orc_param_bytes(uint64_t d, uint64_t l, uint64_t r,
                                uint64_t k_prime, uint64_t out[4]) {
  out[0] = 2 * d * l;
  out[1] = 2 * (d * r + r * l + d * k_prime);
  out[2] = (d * l + 1) / 2 + 2 * d * k_prime;
  out[3] = (d * r + r * l + 1) / 2 + 2 * d * k_prime;
}
