// Common device helpers for the GNS B200 library (sm_100a).
//
//  * Philox4x32-10 and the GNS key layout (bit-identical to oracle/philox.py)
//  * deterministic fp64 log/log1p/expm1 (bit-identical to oracle/detmath.py)
//  * decoupled-look-back device-wide scan used by every compaction/offset pass
//  * error/status plumbing for the C ABI (include/gns.h)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <unordered_map>

#include "../../include/gns.h"

#define GNS_WARP 32
#define GNS_FULL 0xffffffffu

namespace gns {

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define GNS_TRY(expr)                         \
  do {                                        \
    int _rc = (expr);                         \
    if (_rc != GNS_OK) return _rc;            \
  } while (0)

#define GNS_CUDA(expr)                                                   \
  do {                                                                   \
    cudaError_t _e = (expr);                                             \
    if (_e != cudaSuccess) {                                             \
      ::gns::set_error("%s: %s", #expr, cudaGetErrorString(_e));         \
      return GNS_ECUDA;                                                  \
    }                                                                    \
  } while (0)

int num_sms();

// Fork/join of independent kernels inside one entry point: work launched on
// `aux` runs concurrently with the calling stream (eagerly, and as parallel
// branches when the calling stream is being captured into a CUDA graph).
// Each calling stream gets its own auxiliary stream (same priority), so
// concurrent callers on different streams never share one.
struct Fork {
  cudaStream_t aux;
  cudaEvent_t ev_fork, ev_join;
};
int fork_begin(cudaStream_t s, Fork* f);  // aux waits for everything issued on s so far
}  // namespace gns
extern "C" int gns_sample_tune(const char* name, int32_t value);  // gns_tune's sampler knobs (internal)
namespace gns {
int fork_join(cudaStream_t s, const Fork& f);  // s waits for everything issued on aux

static inline unsigned div_up(long long a, long long b) { return (unsigned)((a + b - 1) / b); }
static inline int grid_for(long long want, long long cap) {
  long long g = want < cap ? want : cap;
  return (int)(g < 1 ? 1 : g);
}

// Grid for a grid-stride kernel: at most one wave of resident CTAs
// (cudaOccupancyMaxActiveBlocksPerMultiprocessor, cached per kernel), so no
// CTA waits for a second wave and no empty CTAs are launched past it.
template <typename Kernel>
static inline int resident_grid(Kernel kernel, int block, size_t smem, long long want) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> per_sm_cache;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_sm_cache.find((const void*)kernel);
    if (it != per_sm_cache.end()) {
      per_sm = it->second;
    } else {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem) != cudaSuccess) per_sm = 1;
      per_sm_cache[(const void*)kernel] = per_sm;
    }
  }
  return grid_for(want, (long long)num_sms() * (per_sm > 0 ? per_sm : 1));
}

// Bump allocator over a caller-given workspace (256-byte aligned slices).
struct Workspace {
  char* base;
  size_t cap;
  size_t off;
  __host__ Workspace(void* p, size_t n) : base((char*)p), cap(n), off(0) {}
  template <typename T>
  __host__ T* take(size_t count) {
    size_t bytes = (count * sizeof(T) + 255) & ~(size_t)255;
    if (base == nullptr) { off += bytes; return nullptr; }  // sizing pass
    if (off + bytes > cap) { off += bytes; return nullptr; }
    T* p = (T*)(base + off);
    off += bytes;
    return p;
  }
  __host__ bool ok() const { return base == nullptr || off <= cap; }
};

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al. SC'11); oracle/philox.py is the restatement.
// ---------------------------------------------------------------------------
struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                               uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

__host__ __device__ __forceinline__ uint32_t stream_word(uint32_t tag, uint32_t layer, uint32_t phase) {
  return ((tag & 0xffu) << 24) | ((layer & 0xffu) << 16) | ((phase & 0xffu) << 8);
}

// Two 53-bit keys for positions 2q and 2q+1 of one (node, stream) row.
__device__ __forceinline__ void key53_pair(uint32_t seed, uint32_t epoch, uint32_t node,
                                           uint32_t stream, uint32_t batch, uint32_t q,
                                           uint64_t& k_even, uint64_t& k_odd) {
  u32x4 w = philox4x32_10(q, node, stream, batch, seed, epoch);
  k_even = ((((uint64_t)w.x) << 32) | w.y) >> 11;
  k_odd = ((((uint64_t)w.z) << 32) | w.w) >> 11;
}

__device__ __forceinline__ uint64_t key53_at(uint32_t seed, uint32_t epoch, uint32_t node,
                                             uint32_t stream, uint32_t batch, uint64_t pos) {
  u32x4 w = philox4x32_10((uint32_t)(pos >> 1), node, stream, batch, seed, epoch);
  uint32_t hi = (pos & 1) ? w.z : w.x;
  uint32_t lo = (pos & 1) ? w.w : w.y;
  return ((((uint64_t)hi) << 32) | lo) >> 11;
}

// 4-round balanced Feistel over 2h bits + cycle walking (oracle/philox.py).
__device__ __forceinline__ uint64_t feistel_once(uint64_t x, int h, uint32_t seed, uint32_t epoch) {
  const uint64_t hmask = (h >= 64) ? ~0ull : ((1ull << h) - 1);
  uint64_t left = x >> h, right = x & hmask;
  const uint32_t stream = stream_word(31, 0, 0);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    u32x4 w = philox4x32_10((uint32_t)right, (uint32_t)r, stream, 0u, seed, epoch);
    uint64_t f = (uint64_t)w.x & hmask;
    uint64_t nl = right;
    right = left ^ f;
    left = nl;
  }
  return (left << h) | right;
}

// ---------------------------------------------------------------------------
// Deterministic fp64 transcendental pair (oracle/detmath.py).  Every step is an
// explicitly rounded IEEE op so ptxas cannot contract into FMA.
// ---------------------------------------------------------------------------
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))

__device__ __constant__ static const double kAtanhC[20] = {
    0x1p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3, 0x1.2492492492492p-3,
    0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4, 0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4,
    0x1.e1e1e1e1e1e1ep-5, 0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5,
    0x1.47ae147ae147bp-5, 0x1.2f684bda12f68p-5, 0x1.1a7b9611a7b96p-5, 0x1.0842108421084p-5,
    0x1.f07c1f07c1f08p-6, 0x1.d41d41d41d41dp-6, 0x1.bacf914c1bad0p-6, 0x1.a41a41a41a41ap-6};
__device__ __constant__ static const double kExpC[18] = {
    0x1p+0, 0x1p-1, 0x1.5555555555555p-3, 0x1.5555555555555p-5,
    0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-13, 0x1.a01a01a01a01ap-16,
    0x1.71de3a556c734p-19, 0x1.27e4fb7789f5cp-22, 0x1.ae64567f544e4p-26, 0x1.1eed8eff8d898p-29,
    0x1.6124613a86d09p-33, 0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-41, 0x1.ae7f3e733b81fp-45,
    0x1.952c77030ad4ap-49, 0x1.6827863b97d97p-53};

#define GNS_LN2_HI 0x1.62e42fee00000p-1
#define GNS_LN2_LO 0x1.a39ef35793c76p-33
#define GNS_INV_LN2 0x1.71547652b82fep+0
#define GNS_SQRT_HALF 0x1.6a09e667f3bcdp-1
#define GNS_ONE_MINUS_1EM15 0x1.ffffffffffff7p-1

__device__ __forceinline__ double atanh_series(double s, int nterms) {
  double z = DMUL(s, s);
  double p = kAtanhC[nterms - 1];
  for (int i = nterms - 2; i >= 0; --i) p = DADD(DMUL(p, z), kAtanhC[i]);
  return DMUL(DMUL(s, p), 2.0);
}

__device__ __forceinline__ double det_log(double x) {
  int e;
  double f = frexp(x, &e);
  if (f < GNS_SQRT_HALF) { f = DMUL(f, 2.0); e -= 1; }
  double s = DDIV(DSUB(f, 1.0), DADD(f, 1.0));
  double poly = atanh_series(s, 12);
  double ed = (double)e;
  return DADD(DMUL(ed, GNS_LN2_HI), DADD(DMUL(ed, GNS_LN2_LO), poly));
}

__device__ __forceinline__ double det_log1p(double x) {  // x in (-1, 0]
  if (x > -0.5) {
    double s = DDIV(x, DADD(x, 2.0));
    return atanh_series(s, 20);
  }
  return det_log(DADD(x, 1.0));
}

__device__ __forceinline__ double expm1_taylor(double y) {
  double p = kExpC[17];
  for (int i = 16; i >= 0; --i) p = DADD(DMUL(p, y), kExpC[i]);
  return DMUL(y, p);
}

__device__ __forceinline__ double det_expm1(double y) {  // y <= 0
  if (y > -0.5) return expm1_taylor(y);
  if (y < -40.0) return -1.0;
  double k = rint(DMUL(y, GNS_INV_LN2));
  double r = DSUB(DSUB(y, DMUL(k, GNS_LN2_HI)), DMUL(k, GNS_LN2_LO));
  double er = DADD(expm1_taylor(r), 1.0);
  return DSUB(ldexp(er, (int)k), 1.0);
}

// exp(y) for |y| < 700 and pow(a, b) = exp(b * log(a)) for a > 0, same IEEE
// op sequence as oracle/gen.c (the synthetic-graph generator's inverse CDF).
__device__ __forceinline__ double det_exp(double y) {
  double k = rint(DMUL(y, GNS_INV_LN2));
  double r = DSUB(DSUB(y, DMUL(k, GNS_LN2_HI)), DMUL(k, GNS_LN2_LO));
  return ldexp(DADD(expm1_taylor(r), 1.0), (int)k);
}

__device__ __forceinline__ double det_pow(double a, double b) { return det_exp(DMUL(b, det_log(a))); }

// ---------------------------------------------------------------------------
// warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(GNS_FULL, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(GNS_FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// ---------------------------------------------------------------------------
// Decoupled look-back scan over uint64 values (single pass, dynamic tile ids).
//
//   status layout (caller memsets to zero before each launch):
//     uint32 counter; uint32 pad; then per tile: flag[ntiles], agg[ntiles], incl[ntiles]
// ---------------------------------------------------------------------------
struct ScanStatus {
  unsigned int* counter;
  unsigned int* flag;
  unsigned long long* agg;
  unsigned long long* incl;
};

static inline size_t scan_status_bytes(long long max_tiles) {
  return 256 + (size_t)max_tiles * (4 + 8 + 8) + 256;
}

__host__ static inline ScanStatus make_scan_status(void* p, long long max_tiles) {
  char* b = (char*)p;
  ScanStatus s;
  s.counter = (unsigned int*)b;
  s.agg = (unsigned long long*)(b + 256);
  s.incl = s.agg + max_tiles;
  s.flag = (unsigned int*)(s.incl + max_tiles);
  return s;
}

enum : unsigned { kFlagNone = 0, kFlagAgg = 1, kFlagIncl = 2 };

// Block-wide exclusive scan of one uint64 per thread.  Returns exclusive
// prefix within the block, writes block total into *total (all threads).
template <int BLOCK>
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* smem_warp,
                                                              unsigned long long& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long inc = warp_incl_scan(v);
  if (lane == 31) smem_warp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = (lane < BLOCK / 32) ? smem_warp[lane] : 0ull;
    unsigned long long wi = warp_incl_scan(w);
    if (lane < BLOCK / 32) smem_warp[lane] = wi - w;  // exclusive
    if (lane == BLOCK / 32 - 1) smem_warp[BLOCK / 32] = wi;
  }
  __syncthreads();
  total = smem_warp[BLOCK / 32];
  unsigned long long r = smem_warp[warp] + inc - v;
  __syncthreads();
  return r;
}

// Look-back by warp 0: returns exclusive prefix of tile `tile` (valid in lane 0
// of warp 0 and broadcast through smem by the caller).
__device__ __forceinline__ unsigned long long tile_lookback(const ScanStatus& st, int tile) {
  const int lane = lane_id();
  unsigned long long excl = 0;
  long long pred = (long long)tile - 1;
  while (true) {
    long long idx = pred - lane;
    unsigned f = kFlagIncl;
    unsigned long long v = 0;
    if (idx >= 0) {
      volatile unsigned* fp = st.flag + idx;
      do { f = *fp; } while (f == kFlagNone);
      __threadfence();
      v = (f == kFlagIncl) ? ((volatile unsigned long long*)st.incl)[idx]
                           : ((volatile unsigned long long*)st.agg)[idx];
    }
    unsigned m = __ballot_sync(GNS_FULL, f == kFlagIncl);
    int stop = m ? (__ffs(m) - 1) : 31;
    unsigned long long c = (lane <= stop) ? v : 0ull;
    excl += warp_sum(c);
    if (m) break;
    pred -= 32;
  }
  return excl;
}

// Generic single-pass scan of n items (n read from device if n_dev != null).
// Loader:  unsigned long long operator()(long long i)          (value of item i, i < n)
// Storer:  void operator()(long long i, unsigned long long excl, unsigned long long val)
// Totaler: void operator()(unsigned long long total)             (called once)
template <int BLOCK, int ITEMS, typename Loader, typename Storer, typename Totaler>
__device__ __forceinline__ void scan_tiles(ScanStatus st, long long n, Loader load, Storer store,
                                           Totaler tot) {
  constexpr int TILE = BLOCK * ITEMS;
  __shared__ unsigned long long s_warp[BLOCK / 32 + 1];
  __shared__ unsigned long long s_items[TILE + TILE / 32];
  __shared__ int s_tile;
  __shared__ unsigned long long s_prefix;
  const long long ntiles = (n + TILE - 1) / TILE;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(st.counter, 1u);
  __syncthreads();
  const int tile = s_tile;
  if (tile >= ntiles) {
    if (n == 0 && tile == 0 && threadIdx.x == 0) tot(0ull);
    return;
  }
  // striped (coalesced) loads -> shared memory -> blocked per-thread items
  const long long tbase = (long long)tile * TILE;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int li = j * BLOCK + threadIdx.x;
    const long long i = tbase + li;
    s_items[li + (li >> 5)] = (i < n) ? load(i) : 0ull;
  }
  __syncthreads();
  const long long base = tbase + (long long)threadIdx.x * ITEMS;
  unsigned long long vals[ITEMS];
  unsigned long long tsum = 0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int li = threadIdx.x * ITEMS + j;
    vals[j] = s_items[li + (li >> 5)];
    tsum += vals[j];
  }
  unsigned long long block_total;
  unsigned long long texcl = block_excl_scan<BLOCK>(tsum, s_warp, block_total);
  if (threadIdx.x < 32) {
    unsigned long long prefix = 0;
    if (tile == 0) {
      if (threadIdx.x == 0) {
        st.incl[0] = block_total;
        __threadfence();
        atomicExch(st.flag + 0, kFlagIncl);
      }
    } else {
      if (threadIdx.x == 0) {
        st.agg[tile] = block_total;
        __threadfence();
        atomicExch(st.flag + tile, kFlagAgg);
      }
      prefix = tile_lookback(st, tile);
      if (threadIdx.x == 0) {
        st.incl[tile] = prefix + block_total;
        __threadfence();
        atomicExch(st.flag + tile, kFlagIncl);
      }
    }
    if (threadIdx.x == 0) {
      s_prefix = prefix;
      if (tile == ntiles - 1) tot(prefix + block_total);
    }
  }
  __syncthreads();
  unsigned long long run = s_prefix + texcl;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    long long i = base + j;
    if (i < n) store(i, run, vals[j]);
    run += vals[j];
  }
}

// ---------------------------------------------------------------------------
// Two-kernel scan for per-step sizes (<= a few thousand tiles): pass 1 writes
// one sum per tile; pass 2 forms each tile's exclusive prefix by summing the
// preceding tile sums directly (no look-back chain, no status memset) and
// scans the tile locally.  Grid = tiles for the capacity; n may live on the
// device and be smaller.
// ---------------------------------------------------------------------------
template <int BLOCK>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long* smem_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) smem_warp[warp] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x < 32) {
    t = (lane < BLOCK / 32) ? smem_warp[lane] : 0ull;
    t = warp_sum(t);
  }
  __syncthreads();
  if (threadIdx.x == 0) smem_warp[0] = t;
  __syncthreads();
  t = smem_warp[0];
  __syncthreads();
  return t;
}

template <int BLOCK, int ITEMS, typename Loader>
__device__ __forceinline__ void scan2_reduce(long long n, Loader load, unsigned long long* __restrict__ tile_sums) {
  constexpr int TILE = BLOCK * ITEMS;
  __shared__ unsigned long long s_warp[BLOCK / 32 + 1];
  const long long base = (long long)blockIdx.x * TILE;
  unsigned long long s = 0;
  if (base < n) {
#pragma unroll
    for (int j = 0; j < ITEMS; ++j) {
      const long long i = base + j * BLOCK + threadIdx.x;
      if (i < n) s += load(i);
    }
  }
  s = block_sum<BLOCK>(s, s_warp);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = s;
}

template <int BLOCK, int ITEMS, typename Loader, typename Storer, typename Totaler>
__device__ __forceinline__ void scan2_apply(long long n, Loader load, Storer store, Totaler tot,
                                            const unsigned long long* __restrict__ tile_sums) {
  constexpr int TILE = BLOCK * ITEMS;
  __shared__ unsigned long long s_warp[BLOCK / 32 + 1];
  __shared__ unsigned long long s_items[TILE + TILE / 32];
  const long long ntiles = (n + TILE - 1) / TILE;
  const long long tile = blockIdx.x;
  if (n == 0) {
    if (tile == 0 && threadIdx.x == 0) tot(0ull);
    return;
  }
  if (tile >= ntiles) return;
  unsigned long long pre = 0;
  for (long long j = threadIdx.x; j < tile; j += BLOCK) pre += tile_sums[j];
  pre = block_sum<BLOCK>(pre, s_warp);
  const long long tbase = tile * TILE;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int li = j * BLOCK + threadIdx.x;
    const long long i = tbase + li;
    s_items[li + (li >> 5)] = (i < n) ? load(i) : 0ull;
  }
  __syncthreads();
  unsigned long long vals[ITEMS];
  unsigned long long tsum = 0;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int li = threadIdx.x * ITEMS + j;
    vals[j] = s_items[li + (li >> 5)];
    tsum += vals[j];
  }
  unsigned long long block_total;
  unsigned long long run = pre + block_excl_scan<BLOCK>(tsum, s_warp, block_total);
  if (tile == ntiles - 1 && threadIdx.x == 0) tot(pre + block_total);
  const long long base = tbase + (long long)threadIdx.x * ITEMS;
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const long long i = base + j;
    if (i < n) store(i, run, vals[j]);
    run += vals[j];
  }
}

}  // namespace gns
