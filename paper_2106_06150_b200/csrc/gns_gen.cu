// Device-side synthetic power-law graph generator (the graph.py:172-205 role
// for the papers100M/products/OAG-shaped benchmark graphs, which the
// reference's per-node Python loop cannot build at 111M nodes).
//
// Output contract = graph.py:142-169 build_csr: symmetric, no self loops, no
// duplicate edges, neighbour lists sorted ascending.
//
// Pair e draws two endpoint ranks from Philox with P(rank x) ~ (x+offset)^-alpha
// (closed-form inverse CDF of the continuous approximation), maps ranks to ids
// through a Feistel bijection (hubs scattered over the id space), and the
// pipeline is: count degrees -> scan -> scatter both directions -> per-row
// sort -> distinct count -> scan -> compact.  Pairs are regenerated from the
// counter instead of being stored.
#include <algorithm>

#include "gns_common.cuh"

namespace gns {

struct GenParams {
  int64_t n, m;
  double alpha, offset;
  double a0, span;  // offset^(1-alpha), (n+offset)^(1-alpha) - a0
  int h;            // Feistel half width
  uint32_t seed;
};

__device__ __forceinline__ int32_t gen_rank_to_id(uint64_t x, const GenParams& P) {
  uint64_t y = feistel_once(x, P.h, P.seed, 0x47454eu);
  while (y >= (uint64_t)P.n) y = feistel_once(y, P.h, P.seed, 0x47454eu);
  return (int32_t)y;
}

__device__ __forceinline__ int64_t gen_rank(double u, const GenParams& P) {
  // inverse CDF with the deterministic pow (gns_common.cuh det_pow): the same
  // IEEE op sequence as oracle/gen.c, so the host restatement rebuilds this
  // graph bit for bit (the CPU reference arm of bench.py uses it)
  const double oma = DSUB(1.0, P.alpha);
  double x = DSUB(det_pow(DADD(P.a0, DMUL(u, P.span)), DDIV(1.0, oma)), P.offset);
  int64_t r = (int64_t)x;
  if (r < 0) r = 0;
  if (r >= P.n) r = P.n - 1;
  return r;
}

__device__ __forceinline__ void gen_pair(int64_t e, const GenParams& P, int32_t& u, int32_t& v) {
  u32x4 w = philox4x32_10((uint32_t)e, (uint32_t)(e >> 32), stream_word(40, 0, 0), 0u, P.seed, 0x5041u);
  double u1 = (double)(((((uint64_t)w.x) << 32) | w.y) >> 11) * 0x1p-53;
  double u2 = (double)(((((uint64_t)w.z) << 32) | w.w) >> 11) * 0x1p-53;
  u = gen_rank_to_id(gen_rank(u1, P), P);
  v = gen_rank_to_id(gen_rank(u2, P), P);
}

// Pair sources: Philox power-law pairs, or caller-given (u, v) arrays
// (build_csr, graph.py:142-169).
struct GenSource {
  GenParams P;
  __device__ __forceinline__ void operator()(int64_t e, int32_t& u, int32_t& v) const { gen_pair(e, P, u, v); }
};
struct ArraySource {
  const int32_t* u;
  const int32_t* v;
  __device__ __forceinline__ void operator()(int64_t e, int32_t& a, int32_t& b) const {
    a = u[e];
    b = v[e];
  }
};

template <typename Src>
__global__ void gen_count_kernel(Src src, int64_t m, int32_t* __restrict__ deg) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t u, v;
    src(e, u, v);
    if (u == v) continue;
    atomicAdd(deg + u, 1);
    atomicAdd(deg + v, 1);
  }
}

template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) gen_scan_kernel(ScanStatus ss, int32_t* __restrict__ cnt, int64_t n,
                                                         int64_t* __restrict__ ptr, int64_t* __restrict__ total_dev,
                                                         int reset) {
  scan_tiles<BLOCK, ITEMS>(
      ss, n, [&](long long i) { return (unsigned long long)(uint32_t)cnt[i]; },
      [&](long long i, unsigned long long ex, unsigned long long) {
        ptr[i] = (int64_t)ex;
        if (reset) cnt[i] = 0;
      },
      [&](unsigned long long tot) {
        ptr[n] = (int64_t)tot;
        if (total_dev) total_dev[0] = (int64_t)tot;
      });
}

template <typename Src>
__global__ void gen_scatter_kernel(Src src, int64_t m, const int64_t* __restrict__ ptr0, int32_t* __restrict__ cursor,
                                   int32_t* __restrict__ raw) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t u, v;
    src(e, u, v);
    if (u == v) continue;
    raw[ptr0[u] + atomicAdd(cursor + u, 1)] = v;
    raw[ptr0[v] + atomicAdd(cursor + v, 1)] = u;
  }
}

// all-ascending bitonic network over a[0..L) (virtual +inf padding), by `nthreads`
template <typename SYNC>
__device__ __forceinline__ void bitonic_inplace(int32_t* a, int L, int tid, int nthreads, SYNC sync) {
  int P = 1;
  while (P < L) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    const int half = k >> 1;
    for (int t = tid; t < P / 2; t += nthreads) {
      int i = (t / half) * k + (t % half);
      int j = i ^ (k - 1);
      if (j < L && a[j] < a[i]) { int32_t x = a[i]; a[i] = a[j]; a[j] = x; }
    }
    sync();
    for (int st = k >> 2; st >= 1; st >>= 1) {
      for (int t = tid; t < P / 2; t += nthreads) {
        int i = (t / st) * 2 * st + (t % st);
        int j = i + st;
        if (j < L && a[j] < a[i]) { int32_t x = a[i]; a[i] = a[j]; a[j] = x; }
      }
      sync();
    }
  }
}

constexpr int kGenBigRow = 2048;

// warp per row: sort (<= kGenBigRow) and count distinct values
__global__ void gen_sort_small_kernel(const int64_t* __restrict__ ptr0, int64_t n, int32_t* __restrict__ raw,
                                      int32_t* __restrict__ ndeg, int32_t* __restrict__ big, int32_t* __restrict__ nbig) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw) {
    const int64_t b = ptr0[r];
    const int L = (int)(ptr0[r + 1] - b);
    int32_t* a = raw + b;
    if (L > kGenBigRow) {
      if (lane == 0) big[atomicAdd(nbig, 1)] = (int32_t)r;
      continue;
    }
    if (L <= 32) {
      int32_t x = lane < L ? a[lane] : INT32_MAX;
      int rank = 0;
      for (int j = 0; j < L; ++j) {
        int32_t y = __shfl_sync(GNS_FULL, x, j);
        rank += (y < x) || (y == x && j < lane);
      }
      __syncwarp();
      if (lane < L) a[rank] = x;
      __syncwarp();
    } else {
      bitonic_inplace(a, L, lane, 32, [] { __syncwarp(); });
    }
    int distinct = 0;
    for (int base = 0; base < L; base += 32) {
      int i = base + lane;
      bool nd = i < L && (i == 0 || a[i] != a[i - 1]);
      distinct += __popc(__ballot_sync(GNS_FULL, nd));
    }
    if (lane == 0) ndeg[r] = distinct;
  }
}

__global__ void gen_sort_big_kernel(const int64_t* __restrict__ ptr0, int32_t* __restrict__ raw,
                                    int32_t* __restrict__ ndeg, const int32_t* __restrict__ big,
                                    const int32_t* __restrict__ nbig) {
  __shared__ int s_cnt;
  for (int h = blockIdx.x; h < nbig[0]; h += gridDim.x) {
    const int64_t r = big[h];
    const int64_t b = ptr0[r];
    const int L = (int)(ptr0[r + 1] - b);
    int32_t* a = raw + b;
    bitonic_inplace(a, L, threadIdx.x, blockDim.x, [] { __syncthreads(); });
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int c = 0;
    for (int i = threadIdx.x; i < L; i += blockDim.x) c += (i == 0 || a[i] != a[i - 1]);
    atomicAdd(&s_cnt, c);
    __syncthreads();
    if (threadIdx.x == 0) ndeg[r] = s_cnt;
    __syncthreads();
  }
}

__global__ void gen_compact_kernel(const int64_t* __restrict__ ptr0, const int32_t* __restrict__ raw, int64_t n,
                                   const int64_t* __restrict__ ptr, int32_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw) {
    const int64_t b = ptr0[r], e = ptr0[r + 1];
    int64_t o = ptr[r];
    for (int64_t base = b; base < e; base += 32) {
      int64_t i = base + lane;
      int32_t x = i < e ? raw[i] : 0;
      bool nd = i < e && (i == b || raw[i - 1] != x);
      unsigned bal = __ballot_sync(GNS_FULL, nd);
      if (nd) out[o + __popc(bal & ((1u << lane) - 1u))] = x;
      o += __popc(bal);
    }
  }
}

// ---------------------------------------------------------------------------
// Node attributes: labels, train/val/test masks and class-mean + noise
// features (the graph.py:249-253 scheme), each a pure function of
// (seed, node[, column]) through Philox, so oracle/gen.c reproduces them bit
// for bit on the host.  The noise is an Irwin-Hall(4) normal: four 16-bit
// uniforms summed as an integer (exact), scaled by 2^-16, centred, times
// sqrt(3) -- float ops only, each explicitly rounded (no FMA contraction).
// ---------------------------------------------------------------------------
constexpr uint32_t kAttrKey = 0x4e4f4445u;  // "NODE"
constexpr float kSqrt3f = 0x1.bb67aep+0f;

__device__ __forceinline__ float ih4_normal(uint32_t a, uint32_t b) {
  uint32_t s = (a & 0xffffu) + (a >> 16) + (b & 0xffffu) + (b >> 16);
  return __fmul_rn(__fsub_rn(__fmul_rn((float)s, 0x1p-16f), 2.0f), kSqrt3f);
}

__global__ void gen_attrs_kernel(int64_t n, uint32_t classes, float t1, float t2, uint32_t seed,
                                 int32_t* __restrict__ labels, uint8_t* __restrict__ train,
                                 uint8_t* __restrict__ val, uint8_t* __restrict__ test) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    u32x4 w = philox4x32_10((uint32_t)v, (uint32_t)(v >> 32), stream_word(41, 0, 0), 0u, seed, kAttrKey);
    labels[v] = (int32_t)(((uint64_t)w.x * classes) >> 32);
    float r = __fmul_rn((float)(w.y >> 8), 0x1p-24f);
    train[v] = r < t1;
    val[v] = r >= t1 && r < t2;
    test[v] = r >= t2;
  }
}

// class means: one thread per (class, column pair)
__global__ void gen_means_kernel(int32_t classes, int32_t ld, uint32_t seed, float* __restrict__ means) {
  const int pairs = ld >> 1;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < classes * pairs; i += gridDim.x * blockDim.x) {
    const int c = i / pairs, q = i % pairs;
    u32x4 w = philox4x32_10((uint32_t)q, (uint32_t)c, stream_word(42, 0, 0), 0u, seed, kAttrKey);
    means[(int64_t)c * ld + 2 * q] = ih4_normal(w.x, w.y);
    means[(int64_t)c * ld + 2 * q + 1] = ih4_normal(w.z, w.w);
  }
}

__global__ void gen_feats_kernel(int64_t n, int32_t dim, int32_t ld, float noise, uint32_t seed,
                                 const int32_t* __restrict__ labels, const float* __restrict__ means,
                                 float* __restrict__ out) {
  const int pairs = ld >> 1;
  const int64_t total = n * pairs;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / pairs;
    const int q = (int)(i - v * pairs);
    const int j = 2 * q;
    float2 o = make_float2(0.f, 0.f);
    if (j < dim) {
      u32x4 w = philox4x32_10((uint32_t)q, (uint32_t)v, stream_word(43, 0, 0), (uint32_t)(v >> 32), seed, kAttrKey);
      const float* m = means + (int64_t)labels[v] * ld;
      o.x = __fadd_rn(m[j], __fmul_rn(noise, ih4_normal(w.x, w.y)));
      if (j + 1 < dim) o.y = __fadd_rn(m[j + 1], __fmul_rn(noise, ih4_normal(w.z, w.w)));
    }
    reinterpret_cast<float2*>(out)[i] = o;
  }
}

struct GenWs {
  int32_t* cnt;
  int64_t* ptr0;
  int32_t* raw;
  int32_t* big;
  int32_t* nbig;
  void* scan;
  long long tiles;
};

static size_t gen_ws(int64_t n, int64_t m, void* base, size_t cap, GenWs* w) {
  Workspace ws(base, cap);
  w->cnt = ws.take<int32_t>(n + 1);
  w->ptr0 = ws.take<int64_t>(n + 1);
  w->raw = ws.take<int32_t>(2 * m + 1);
  w->big = ws.take<int32_t>(n + 1);
  w->nbig = ws.take<int32_t>(64);
  w->tiles = (n + 256 * 16 - 1) / (256 * 16) + 1;
  w->scan = (void*)ws.take<char>(scan_status_bytes(w->tiles));
  return ws.off;
}

// host-side parameters: libm pow, the same call oracle/gen.c makes
static double gen_host_pow(double a, double b) { return pow(a, b); }

static GenParams make_params(int64_t n, int64_t m, double alpha, double offset, uint32_t seed) {
  GenParams P;
  P.n = n;
  P.m = m;
  P.alpha = alpha;
  P.offset = offset;
  P.a0 = gen_host_pow(offset, 1.0 - alpha);
  P.span = gen_host_pow((double)n + offset, 1.0 - alpha) - P.a0;
  int bits = 2;
  while ((1ll << bits) < n) ++bits;
  bits += bits & 1;
  P.h = bits / 2;
  P.seed = seed;
  return P;
}

}  // namespace gns

using namespace gns;

extern "C" {

size_t gns_gen_workspace_size(int64_t num_nodes, int64_t num_pairs) {
  GenWs w;
  return gen_ws(num_nodes, num_pairs, nullptr, 0, &w);
}

}  // extern "C"

template <typename Src>
static int csr_pipeline(Src src, int64_t n, int64_t m, int64_t* out_indptr, int64_t* out_nnz_dev, const GenWs& w,
                        cudaStream_t stream) {
  const int sms = num_sms();
  GNS_CUDA(cudaMemsetAsync(w.cnt, 0, (n + 1) * sizeof(int32_t), stream));
  GNS_CUDA(cudaMemsetAsync(w.nbig, 0, 64 * sizeof(int32_t), stream));
  gen_count_kernel<<<sms * 16, 256, 0, stream>>>(src, m, w.cnt);
  GNS_TRY(check_launch("csr_count"));
  GNS_CUDA(cudaMemsetAsync(w.scan, 0, scan_status_bytes(w.tiles), stream));
  gen_scan_kernel<256, 16><<<(unsigned)w.tiles, 256, 0, stream>>>(make_scan_status(w.scan, w.tiles), w.cnt, n, w.ptr0,
                                                                  nullptr, 1);
  gen_scatter_kernel<<<sms * 16, 256, 0, stream>>>(src, m, w.ptr0, w.cnt, w.raw);
  GNS_TRY(check_launch("csr_scatter"));
  gen_sort_small_kernel<<<sms * 16, 256, 0, stream>>>(w.ptr0, n, w.raw, w.cnt, w.big, w.nbig);
  gen_sort_big_kernel<<<sms * 2, 1024, 0, stream>>>(w.ptr0, w.raw, w.cnt, w.big, w.nbig);
  GNS_TRY(check_launch("csr_sort"));
  GNS_CUDA(cudaMemsetAsync(w.scan, 0, scan_status_bytes(w.tiles), stream));
  gen_scan_kernel<256, 16><<<(unsigned)w.tiles, 256, 0, stream>>>(make_scan_status(w.scan, w.tiles), w.cnt, n,
                                                                  out_indptr, out_nnz_dev, 0);
  return check_launch("csr_scan");
}

extern "C" {

int gns_gen_powerlaw_count(int64_t n, int64_t m, double alpha, double offset, uint32_t seed, int64_t* out_indptr,
                           int64_t* out_nnz_dev, void* ws, size_t ws_bytes, void* stream_) {
  if (n < 2 || m < 0 || !(alpha > 0.0 && alpha < 1.0) || !(offset > 0.0)) {
    set_error("gen_powerlaw: need n >= 2, m >= 0, 0 < alpha < 1, offset > 0");
    return GNS_EINVAL;
  }
  GenWs w;
  size_t need = gen_ws(n, m, ws, ws_bytes, &w);
  if (need > ws_bytes) {
    set_error("gen_powerlaw: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  GenSource src{make_params(n, m, alpha, offset, seed)};
  return csr_pipeline(src, n, m, out_indptr, out_nnz_dev, w, (cudaStream_t)stream_);
}

int gns_build_csr_count(int64_t n, const int32_t* u, const int32_t* v, int64_t m, int64_t* out_indptr,
                        int64_t* out_nnz_dev, void* ws, size_t ws_bytes, void* stream_) {
  if (n < 0 || m < 0) {
    set_error("build_csr: negative sizes");
    return GNS_EINVAL;
  }
  GenWs w;
  size_t need = gen_ws(n, m, ws, ws_bytes, &w);
  if (need > ws_bytes) {
    set_error("build_csr: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  ArraySource src{u, v};
  return csr_pipeline(src, n, m, out_indptr, out_nnz_dev, w, (cudaStream_t)stream_);
}

int gns_build_csr_fill(int64_t n, int64_t m, const int64_t* indptr, int32_t* out_indices, void* ws,
                       size_t ws_bytes, void* stream_) {
  return gns_gen_powerlaw_fill(n, m, indptr, out_indices, ws, ws_bytes, stream_);
}

int gns_gen_powerlaw_fill(int64_t n, int64_t m, const int64_t* indptr, int32_t* out_indices, void* ws,
                          size_t ws_bytes, void* stream_) {
  GenWs w;
  size_t need = gen_ws(n, m, ws, ws_bytes, &w);
  if (need > ws_bytes) {
    set_error("gen_powerlaw_fill: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  gen_compact_kernel<<<num_sms() * 16, 256, 0, (cudaStream_t)stream_>>>(w.ptr0, w.raw, n, indptr, out_indices);
  return check_launch("gen_compact");
}

}  // extern "C"

extern "C" int gns_gen_node_attrs(int64_t n, int32_t num_classes, double train_frac, uint32_t seed, int32_t* labels,
                                  uint8_t* train, uint8_t* val, uint8_t* test, void* stream_) {
  if (n < 0 || num_classes < 1 || !(train_frac >= 0.0 && train_frac <= 1.0)) {
    set_error("gen_node_attrs: need n >= 0, num_classes >= 1, 0 <= train_frac <= 1");
    return GNS_EINVAL;
  }
  if (n == 0) return GNS_OK;
  const float t1 = (float)train_frac;
  const float t2 = (float)(train_frac + (1.0 - train_frac) / 2);
  gen_attrs_kernel<<<num_sms() * 8, 256, 0, (cudaStream_t)stream_>>>(n, (uint32_t)num_classes, t1, t2, seed, labels,
                                                                     train, val, test);
  return check_launch("gen_attrs");
}

extern "C" int gns_gen_features(int64_t n, int32_t dim, int32_t ld, int32_t num_classes, float noise, uint32_t seed,
                                const int32_t* labels, float* class_means, float* out, void* stream_) {
  if (n < 0 || dim < 1 || ld < dim || (ld & 1) || num_classes < 1) {
    set_error("gen_features: need dim >= 1, even ld >= dim, num_classes >= 1");
    return GNS_EINVAL;
  }
  if (n == 0) return GNS_OK;
  cudaStream_t s = (cudaStream_t)stream_;
  gen_means_kernel<<<div_up((long long)num_classes * (ld / 2), 256), 256, 0, s>>>(num_classes, ld, seed, class_means);
  GNS_TRY(check_launch("gen_means"));
  gen_feats_kernel<<<num_sms() * 16, 256, 0, s>>>(n, dim, ld, noise, seed, labels, class_means, out);
  return check_launch("gen_feats");
}
