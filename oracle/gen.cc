// Host restatement of the synthetic-graph generator (csrc/gns_gen.cu).
//
// TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py): the CPU arm of
// bench.py builds its graph with this file so that the reference-side process
// never loads libgns.so or touches the GPU, and the GPU tests check the device
// generator against it bit for bit.
//
// Contract (the reference's build_csr, graph.py:142-169): symmetric CSR, no
// self loops, no duplicate edges, rows ascending.  Pair e draws two endpoint
// ranks from Philox4x32-10 with P(rank x) ~ (x + offset)^-alpha through a
// closed-form inverse CDF evaluated with the deterministic IEEE op sequence of
// gns_common.cuh (det_log / det_exp: correctly rounded +,-,*,/ only; built
// with -ffp-contract=off so no FMA contraction), then maps ranks to ids with
// the Feistel bijection.  Node attributes (labels, masks, class-mean + noise
// features) are pure functions of (seed, node) with the same Philox streams
// as gns_gen_node_attrs / gns_gen_features.
//
// Build: oracle/Makefile (g++ -O3 -fopenmp -ffp-contract=off).
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

namespace {

struct U4 {
  uint32_t x, y, z, w;
};

inline U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0, p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

inline uint32_t stream_word(uint32_t tag) { return (tag & 0xffu) << 24; }

inline uint64_t feistel_once(uint64_t x, int h, uint32_t seed, uint32_t epoch) {
  const uint64_t hmask = (1ull << h) - 1;
  uint64_t left = x >> h, right = x & hmask;
  for (int r = 0; r < 4; ++r) {
    U4 w = philox((uint32_t)right, (uint32_t)r, stream_word(31), 0u, seed, epoch);
    uint64_t f = (uint64_t)w.x & hmask;
    uint64_t nl = right;
    right = left ^ f;
    left = nl;
  }
  return (left << h) | right;
}

const double kAtanhC[12] = {0x1p+0,
                            0x1.5555555555555p-2,
                            0x1.999999999999ap-3,
                            0x1.2492492492492p-3,
                            0x1.c71c71c71c71cp-4,
                            0x1.745d1745d1746p-4,
                            0x1.3b13b13b13b14p-4,
                            0x1.1111111111111p-4,
                            0x1.e1e1e1e1e1e1ep-5,
                            0x1.af286bca1af28p-5,
                            0x1.8618618618618p-5,
                            0x1.642c8590b2164p-5};
const double kExpC[18] = {0x1p+0,
                          0x1p-1,
                          0x1.5555555555555p-3,
                          0x1.5555555555555p-5,
                          0x1.1111111111111p-7,
                          0x1.6c16c16c16c17p-10,
                          0x1.a01a01a01a01ap-13,
                          0x1.a01a01a01a01ap-16,
                          0x1.71de3a556c734p-19,
                          0x1.27e4fb7789f5cp-22,
                          0x1.ae64567f544e4p-26,
                          0x1.1eed8eff8d898p-29,
                          0x1.6124613a86d09p-33,
                          0x1.93974a8c07c9dp-37,
                          0x1.ae7f3e733b81fp-41,
                          0x1.ae7f3e733b81fp-45,
                          0x1.952c77030ad4ap-49,
                          0x1.6827863b97d97p-53};
const double LN2_HI = 0x1.62e42fee00000p-1, LN2_LO = 0x1.a39ef35793c76p-33;
const double INV_LN2 = 0x1.71547652b82fep+0, SQRT_HALF = 0x1.6a09e667f3bcdp-1;

// gns_common.cuh det_log (12-term atanh series)
inline double det_log(double x) {
  int e;
  double f = frexp(x, &e);
  if (f < SQRT_HALF) {
    f = f * 2.0;
    e -= 1;
  }
  double s = (f - 1.0) / (f + 1.0);
  double z = s * s;
  double p = kAtanhC[11];
  for (int i = 10; i >= 0; --i) p = p * z + kAtanhC[i];
  double poly = (s * p) * 2.0;
  double ed = (double)e;
  return ed * LN2_HI + (ed * LN2_LO + poly);
}

// gns_common.cuh det_exp (range reduction + 18-term Taylor expm1)
inline double det_exp(double y) {
  double k = rint(y * INV_LN2);
  double r = (y - k * LN2_HI) - k * LN2_LO;
  double p = kExpC[17];
  for (int i = 16; i >= 0; --i) p = p * r + kExpC[i];
  return ldexp(r * p + 1.0, (int)k);
}

struct Params {
  int64_t n;
  double alpha, offset, a0, span;
  int h;
  uint32_t seed;
};

Params make_params(int64_t n, double alpha, double offset, uint32_t seed) {
  Params P;
  P.n = n;
  P.alpha = alpha;
  P.offset = offset;
  P.a0 = pow(offset, 1.0 - alpha);  // host libm, as gns_gen.cu make_params
  P.span = pow((double)n + offset, 1.0 - alpha) - P.a0;
  int bits = 2;
  while ((1ll << bits) < n) ++bits;
  bits += bits & 1;
  P.h = bits / 2;
  P.seed = seed;
  return P;
}

// Branch-free det_log/det_exp for batches (frexp / rint / ldexp as exact bit
// operations on positive normal inputs; same values as the scalar versions),
// so the compiler can vectorise the pair draw.
inline double bits_d(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}
inline uint64_t d_bits(double d) {
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
}

inline double det_log_v(double x) {
  const uint64_t b = d_bits(x);
  double e = (double)((int64_t)((b >> 52) & 0x7ff) - 1022);
  double f = bits_d((b & 0x000fffffffffffffull) | 0x3fe0000000000000ull);
  const bool small = f < SQRT_HALF;
  f = small ? f * 2.0 : f;
  e = small ? e - 1.0 : e;
  double s = (f - 1.0) / (f + 1.0);
  double z = s * s;
  double p = kAtanhC[11];
  for (int i = 10; i >= 0; --i) p = p * z + kAtanhC[i];
  double poly = (s * p) * 2.0;
  return e * LN2_HI + (e * LN2_LO + poly);
}

inline double det_exp_v(double y) {
  const double shift = 0x1.8p52;
  double t = y * INV_LN2;
  double k = (t + shift) - shift;  // rint (round half even), |t| < 2^51
  double r = (y - k * LN2_HI) - k * LN2_LO;
  double p = kExpC[17];
  for (int i = 16; i >= 0; --i) p = p * r + kExpC[i];
  return (r * p + 1.0) * bits_d((uint64_t)((int64_t)k + 1023) << 52);
}

__attribute__((target_clones("avx2", "default"))) void rank_batch(double* a, int cnt, double a0, double span,
                                                                  double inv, double offset) {
#pragma omp simd
  for (int i = 0; i < cnt; ++i) a[i] = det_exp_v(inv * det_log_v(a0 + a[i] * span)) - offset;
}

inline int64_t gen_rank(double u, const Params& P) {
  const double oma = 1.0 - P.alpha;
  double x = det_exp((1.0 / oma) * det_log(P.a0 + u * P.span)) - P.offset;
  int64_t r = (int64_t)x;
  if (r < 0) r = 0;
  if (r >= P.n) r = P.n - 1;
  return r;
}

inline int32_t rank_to_id(uint64_t x, const Params& P) {
  uint64_t y = feistel_once(x, P.h, P.seed, 0x47454eu);
  while (y >= (uint64_t)P.n) y = feistel_once(y, P.h, P.seed, 0x47454eu);
  return (int32_t)y;
}

inline void gen_pair(int64_t e, const Params& P, int32_t& u, int32_t& v) {
  U4 w = philox((uint32_t)e, (uint32_t)(e >> 32), stream_word(40), 0u, P.seed, 0x5041u);
  double u1 = (double)(((((uint64_t)w.x) << 32) | w.y) >> 11) * 0x1p-53;
  double u2 = (double)(((((uint64_t)w.z) << 32) | w.w) >> 11) * 0x1p-53;
  u = rank_to_id(gen_rank(u1, P), P);
  v = rank_to_id(gen_rank(u2, P), P);
}

// CSR from endpoint pairs (us[e], vs[e]), e < m.  Each of T threads owns a
// static chunk of pairs and private per-row counters (no atomics, so the
// random accesses overlap): count -> per-row exclusive scan over threads ->
// row offsets -> scatter both directions -> per-row sort + unique -> scan ->
// in-place ascending compaction.
int64_t csr(const int32_t* us, const int32_t* vs, int64_t n, int64_t m, int64_t* indptr, int32_t* raw,
            int threads) {
  const int T = threads < 1 ? 1 : threads;
  std::vector<int64_t> ptr0(n + 1, 0);
  std::vector<int32_t> cnt((size_t)T * n, 0);
  double T0 = omp_get_wtime();
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    int32_t* c = cnt.data() + (size_t)t * n;
    for (int64_t e = m * t / T; e < m * (t + 1) / T; ++e) {
      const int32_t u = us[e], v = vs[e];
      if (u == v) continue;
      ++c[u];
      ++c[v];
    }
  }
  double T1 = omp_get_wtime();
  std::vector<int32_t> deg(n);
#pragma omp parallel for schedule(static) num_threads(T)
  for (int64_t r = 0; r < n; ++r) {
    int32_t s = 0;
    for (int t = 0; t < T; ++t) {
      int32_t x = cnt[(size_t)t * n + r];
      cnt[(size_t)t * n + r] = s;
      s += x;
    }
    deg[r] = s;
  }
  for (int64_t i = 0; i < n; ++i) ptr0[i + 1] = ptr0[i] + deg[i];
  double T2 = omp_get_wtime();
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    int32_t* c = cnt.data() + (size_t)t * n;
    for (int64_t e = m * t / T; e < m * (t + 1) / T; ++e) {
      const int32_t u = us[e], v = vs[e];
      if (u == v) continue;
      raw[ptr0[u] + c[u]++] = v;
      raw[ptr0[v] + c[v]++] = u;
    }
  }
  std::vector<int32_t>().swap(cnt);
  double T3 = omp_get_wtime();
#pragma omp parallel for schedule(dynamic, 4096) num_threads(T)
  for (int64_t r = 0; r < n; ++r) {
    int32_t* a = raw + ptr0[r];
    int64_t L = ptr0[r + 1] - ptr0[r];
    std::sort(a, a + L);
    deg[r] = (int32_t)(std::unique(a, a + L) - a);
  }
  double T4 = omp_get_wtime();
  indptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) indptr[i + 1] = indptr[i] + deg[i];
  for (int64_t r = 0; r < n; ++r)  // destination <= source: ascending order is safe
    if (indptr[r] != ptr0[r]) memmove(raw + indptr[r], raw + ptr0[r], (size_t)deg[r] * sizeof(int32_t));
  if (getenv("OG_VERBOSE"))
    fprintf(stderr, "csr: count %.2fs scan %.2fs scatter %.2fs sort %.2fs compact %.2fs\n", T1 - T0, T2 - T1,
            T3 - T2, T4 - T3, omp_get_wtime() - T4);
  return indptr[n];
}

constexpr uint32_t kAttrKey = 0x4e4f4445u;
constexpr float kSqrt3f = 0x1.bb67aep+0f;

inline float ih4_normal(uint32_t a, uint32_t b) {
  uint32_t s = (a & 0xffffu) + (a >> 16) + (b & 0xffffu) + (b >> 16);
  return ((float)s * 0x1p-16f - 2.0f) * kSqrt3f;
}

}  // namespace

extern "C" {

// Power-law graph: raw = caller buffer of 2 * num_pairs int32; on return
// raw[0:nnz] holds the indices of the CSR whose indptr[num_nodes + 1] is
// written.  Returns nnz.  The rank -> id bijection is tabulated once (n
// Feistel walks instead of two per pair; same values by construction) and
// the pairs are drawn once into host memory (8 B per pair).
int64_t og_gen_powerlaw(int64_t n, int64_t m, double alpha, double offset, uint32_t seed, int64_t* indptr,
                        int32_t* raw, int threads) {
  Params P = make_params(n, alpha, offset, seed);
  double T0 = omp_get_wtime();
  std::vector<int32_t> id_of(n);
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t r = 0; r < n; ++r) id_of[r] = rank_to_id((uint64_t)r, P);
  std::vector<int32_t> us(m), vs(m);
  const double oma = 1.0 - P.alpha, inv = 1.0 / oma;
  constexpr int B = 64;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t e0 = 0; e0 < m; e0 += B) {
    const int cnt = (int)std::min<int64_t>(B, m - e0);
    double a[2 * B];
    for (int i = 0; i < cnt; ++i) {
      const int64_t e = e0 + i;
      U4 w = philox((uint32_t)e, (uint32_t)(e >> 32), stream_word(40), 0u, P.seed, 0x5041u);
      a[2 * i] = (double)(((((uint64_t)w.x) << 32) | w.y) >> 11) * 0x1p-53;
      a[2 * i + 1] = (double)(((((uint64_t)w.z) << 32) | w.w) >> 11) * 0x1p-53;
    }
    rank_batch(a, 2 * cnt, P.a0, P.span, inv, P.offset);
    for (int i = 0; i < cnt; ++i) {
      int64_t r0 = (int64_t)a[2 * i], r1 = (int64_t)a[2 * i + 1];
      r0 = r0 < 0 ? 0 : (r0 >= n ? n - 1 : r0);
      r1 = r1 < 0 ? 0 : (r1 >= n ? n - 1 : r1);
      us[e0 + i] = id_of[r0];
      vs[e0 + i] = id_of[r1];
    }
  }
  if (getenv("OG_VERBOSE")) fprintf(stderr, "pairs: %.2fs\n", omp_get_wtime() - T0);
  std::vector<int32_t>().swap(id_of);
  return csr(us.data(), vs.data(), n, m, indptr, raw, threads);
}

// build_csr from endpoint arrays (graph.py:142-169), same contract.
int64_t og_build_csr(int64_t n, const int32_t* us, const int32_t* vs, int64_t m, int64_t* indptr, int32_t* raw,
                     int threads) {
  return csr(us, vs, n, m, indptr, raw, threads);
}

// The endpoint ids of pairs [e0, e0 + cnt) (for tests).
void og_gen_pairs(int64_t n, double alpha, double offset, uint32_t seed, int64_t e0, int64_t cnt, int32_t* u,
                  int32_t* v) {
  Params P = make_params(n, alpha, offset, seed);
  for (int64_t i = 0; i < cnt; ++i) gen_pair(e0 + i, P, u[i], v[i]);
}

void og_gen_node_attrs(int64_t n, int32_t classes, double train_frac, uint32_t seed, int32_t* labels,
                       uint8_t* train, uint8_t* val, uint8_t* test, int threads) {
  const float t1 = (float)train_frac;
  const float t2 = (float)(train_frac + (1.0 - train_frac) / 2);
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t v = 0; v < n; ++v) {
    U4 w = philox((uint32_t)v, (uint32_t)(v >> 32), stream_word(41), 0u, seed, kAttrKey);
    labels[v] = (int32_t)(((uint64_t)w.x * (uint32_t)classes) >> 32);
    float r = (float)(w.y >> 8) * 0x1p-24f;
    train[v] = r < t1;
    val[v] = r >= t1 && r < t2;
    test[v] = r >= t2;
  }
}

// out = float32 [n, ld], ld even >= dim, columns >= dim zero
void og_gen_features(int64_t n, int32_t dim, int32_t ld, int32_t classes, float noise, uint32_t seed,
                     const int32_t* labels, float* out, int threads) {
  const int pairs = ld / 2;
  std::vector<float> means((size_t)classes * ld, 0.f);
  for (int c = 0; c < classes; ++c)
    for (int q = 0; q < pairs; ++q) {
      U4 w = philox((uint32_t)q, (uint32_t)c, stream_word(42), 0u, seed, kAttrKey);
      means[(size_t)c * ld + 2 * q] = ih4_normal(w.x, w.y);
      means[(size_t)c * ld + 2 * q + 1] = ih4_normal(w.z, w.w);
    }
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int64_t v = 0; v < n; ++v) {
    const float* mu = means.data() + (size_t)labels[v] * ld;
    float* o = out + v * (int64_t)ld;
    for (int q = 0; q < pairs; ++q) {
      const int j = 2 * q;
      float a = 0.f, b = 0.f;
      if (j < dim) {
        U4 w = philox((uint32_t)q, (uint32_t)v, stream_word(43), (uint32_t)(v >> 32), seed, kAttrKey);
        a = mu[j] + noise * ih4_normal(w.x, w.y);
        if (j + 1 < dim) b = mu[j + 1] + noise * ih4_normal(w.z, w.w);
      }
      o[j] = a;
      o[j + 1] = b;
    }
  }
}

// Cached CSR (cache.py:185-197): row v = N(v) ∩ C in ascending order, i.e.
// the full CSR filtered by the cache mask (identical to the reference's
// gather_rows + lexsort construction, tests/test_oracle.py).  Writes
// out_indptr[n + 1]; fills out_indices when non-null; returns nnz.
int64_t og_cached_csr(int64_t n, const int64_t* indptr, const int32_t* indices, const uint8_t* mask,
                      int64_t* out_indptr, int32_t* out_indices, int threads) {
  std::vector<int64_t> cnt(n);
#pragma omp parallel for schedule(dynamic, 8192) num_threads(threads)
  for (int64_t r = 0; r < n; ++r) {
    int64_t c = 0;
    for (int64_t i = indptr[r]; i < indptr[r + 1]; ++i) c += mask[indices[i]] != 0;
    cnt[r] = c;
  }
  out_indptr[0] = 0;
  for (int64_t r = 0; r < n; ++r) out_indptr[r + 1] = out_indptr[r] + cnt[r];
  if (out_indices) {
#pragma omp parallel for schedule(dynamic, 8192) num_threads(threads)
    for (int64_t r = 0; r < n; ++r) {
      int64_t o = out_indptr[r];
      for (int64_t i = indptr[r]; i < indptr[r + 1]; ++i)
        if (mask[indices[i]]) out_indices[o++] = indices[i];
    }
  }
  return out_indptr[n];
}

}  // extern "C"
