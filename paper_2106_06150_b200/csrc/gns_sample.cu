// Per-layer NS/GNS neighbour sampler and the frontier dedup/relabel on B200.
//
// Reference: sampling.py:155-170 (NS), :189-266 (GNS, gns-paper weights),
// :129-136 (_select_per_row), :139-152 (_assemble), graph.py:399-415
// (gather_rows).
//
// Selection per dst row and phase: the `take` smallest (key53, position)
// pairs among the row's valid candidates, keys from Philox at
// (node, layer, phase, position).  Keys are uniform, so a threshold T with
// E[#{key < T}] = take + 4 sqrt(take) + 8 keeps ~take+ candidates in one pass;
// T is bisected if the count falls outside [take, CAP] (rare).  The kept
// candidates are ranked exactly by (key, pos) — ties break by position like
// the reference's stable lexsort — so the result equals the full sort.  In the
// fill phase the cache-bitmap probe and the neighbour-id load happen only for
// positions whose key is under T, so a hub row costs Philox ALU, not HBM.
//
// Rows whose scan length exceeds kHubLen are taken by whole CTAs at the tail
// of the warp-tier launch.
//
// Dedup/relabel: one bit per node id (N/8 bytes) plus a summary bit per
// bitmap word, set by fire-and-forget atomicOr of the seeds and sampled
// neighbours; two passes over the summary (tile counts, then ranks) emit the
// sorted unique src set and per-word ranks and clear both levels as they go,
// and edge_src = word rank + popc(prefix bits).
#include <string.h>

#include <algorithm>

#include "gns_common.cuh"

namespace gns {

constexpr int kSampBlock = 256;
constexpr int kWarpCap = 256;
constexpr int kHubLen = 2048;   // <= 2^11: the warp tier packs positions in 11 bits
constexpr int kThreadLen = 16;    // rows scanning <= 16 positions: one thread per row, register sort
constexpr int kStreamK = 8;       // streaming top-k tier: take <= 8 and <= stream_len positions
static int g_stream_len = 32;     // (gns_tune "stream_len", <= 2047)
static int g_thread_len = 0;      // (gns_tune "thread_len", <= 16; 0 = no sorting-network tier: measured best)
static int g_stream_minb = 1;     // (gns_tune "stream_minb": 1, 3, 4) min resident CTAs/SM of the streaming tier
static int g_stream_k5 = 1;       // (gns_tune "stream_k5": 0/1) fanout <= 5: keep 5 keys in the streaming tier
static int g_warp_sort = 1;       // (gns_tune "warp_sort": 0/1) see LayerArgs::warp_sort
static int g_sampler_ctas = 0;    // (gns_tune "sampler_ctas") cap grid-stride sampler grids at this many CTAs
                                  // per SM (0 = no cap): leaves SM room to the concurrent training branch
constexpr int kHubCap = 512;
constexpr int kMaxFanout = 128;
constexpr uint64_t kTwo53 = 1ull << 53;

struct LayerArgs {
  const int64_t* indptr;
  const int32_t* indices;
  const int64_t* cindptr;
  const int32_t* cindices;
  const uint32_t* mask;
  const double* incl;
  const int32_t* cpos;     // cached CSR -> position in the full row (gns-exact)
  const double* exact_q;   // per-edge inclusion table (gns-exact) or NULL (gns-paper)
  const int32_t* seeds;
  const int32_t* n_dev;
  int k;
  int cache_only;
  int gns;
  int64_t max_dst;
  uint32_t seed, epoch, batch, layer;
  const gns_step_t* step_dev;
  uint32_t* dbits;  // dedup bitmap (bit v of word v>>5); NULL = no fused marking
  uint32_t* dsum;   // summary bitmap (bit w of word w>>5 set iff dbits[w] != 0)
  int stream_len;   // rows up to this many positions with take <= kStreamK: streaming tier
  int thread_len;   // other rows up to this many positions (<= kThreadLen): sorting-network tier
  int warp_sort;    // warp tier: rank <= 32 candidates by a shuffle bitonic sort (else the shared rank loop)
  struct RowDesc* desc;  // per-row descriptors (count pass -> selection kernels)
  gns_block_t b;
};

// mark node v in the two-level dedup bitmap: two fire-and-forget reductions
// (RED, no returned value to wait for).  The summary bit is set by every mark
// (idempotent), so every non-zero bitmap word has its summary bit.
__device__ __forceinline__ void mark_node(uint32_t* __restrict__ bits, uint32_t* __restrict__ sum, int32_t v) {
  const int32_t w = v >> 5;
  atomicOr(bits + w, 1u << (v & 31));
  atomicOr(sum + (w >> 5), 1u << (w & 31));
}

// Lists of (row, phase) work items per tier, packed in hub_rows[4*max_dst]:
// thread items from 0 up, warp items from 2*max_dst up, hub items from
// 4*max_dst-1 down; the counters are counts[GNS_CNT_THREADROWS/WARPROWS/HUBS].
// Tiers: 0 = thread + sorting network, 1 = warp, 2 = CTA (hub), 3 = thread +
// streaming top-k.
constexpr int kTiers = 4;
__device__ __forceinline__ int32_t* tier_counter(int32_t* counts, int tier) {
  return counts + (tier == 0 ? GNS_CNT_THREADROWS : tier == 1 ? GNS_CNT_WARPROWS
                   : tier == 2 ? GNS_CNT_HUBS : GNS_CNT_STREAMROWS);
}
__device__ __forceinline__ int64_t tier_slot(int64_t max_dst, int tier, int h) {
  return tier == 0 ? h : tier == 3 ? 2 * max_dst + h : tier == 1 ? 4 * max_dst + h : 6 * max_dst - 1 - h;
}

// Append each active lane's NI (row, phase) items (tier[i] = -1: none) to
// their tier lists; returns the list positions.  One atomic per tier and
// warp for all of them, the kTiers atomics issued together; item i of lane l
// lands after the items i' < i of every lane and item i of lanes l' < l.
template <int NI>
__device__ __forceinline__ void warp_append_tiers(int32_t* counts, const int (&tier)[NI], int (&h)[NI]) {
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int first = __ffs(act) - 1;
  int cnt[kTiers] = {0, 0, 0, 0};
  int pre[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    pre[i] = 0;
#pragma unroll
    for (int t = 0; t < kTiers; ++t) {
      const unsigned m = __ballot_sync(act, tier[i] == t);
      if (tier[i] == t) pre[i] = cnt[t] + __popc(m & lt);
      cnt[t] += __popc(m);
    }
  }
  int base[kTiers] = {0, 0, 0, 0};
#pragma unroll
  for (int t = 0; t < kTiers; ++t) {   // independent atomics: all in flight
    const int owner = ((act >> t) & 1u) ? t : first;
    if (lane == owner && cnt[t]) base[t] = atomicAdd(tier_counter(counts, t), cnt[t]);
  }
#pragma unroll
  for (int t = 0; t < kTiers; ++t) {
    const int owner = ((act >> t) & 1u) ? t : first;
    const int bt = __shfl_sync(act, base[t], owner);
#pragma unroll
    for (int i = 0; i < NI; ++i)
      if (tier[i] == t) h[i] = bt + pre[i];
  }
}

// Per-batch Philox key words: from the device gns_step_t when given (CUDA
// graph replay), else the launch arguments.  Kernels take LayerArgs as a
// __grid_constant__ parameter and keep only these three words per thread.
struct Rng3 {
  uint32_t seed, epoch, batch;
};
__device__ __forceinline__ Rng3 batch_rng(const LayerArgs& a) {
  if (a.step_dev) return {a.step_dev->seed, a.step_dev->epoch, a.step_dev->batch};
  return {a.seed, a.epoch, a.batch};
}

struct RowInfo {
  int64_t start, cstart;
  int32_t node, deg, nc, m, fill;
};

// Per-row descriptor written by the count pass (32 B, two 16-B loads): the
// selection kernels read one descriptor per item instead of the chain
// seeds[r] -> indptr/cindptr[node].
struct __align__(16) RowDesc {
  int64_t start, cstart;
  int32_t node, deg, nc, pad;
};

__device__ __forceinline__ RowInfo row_info(const LayerArgs& a, int64_t r) {
  const int4* d = reinterpret_cast<const int4*>(a.desc + r);
  const int4 lo = d[0], hi = d[1];
  RowInfo ri;
  ri.start = ((int64_t)(uint32_t)lo.y << 32) | (uint32_t)lo.x;
  ri.cstart = ((int64_t)(uint32_t)lo.w << 32) | (uint32_t)lo.z;
  ri.node = hi.x;
  ri.deg = hi.y;
  ri.nc = hi.z;
  if (a.gns) {
    ri.m = min(a.k, ri.nc);
    ri.fill = a.cache_only ? 0 : min(a.k - ri.m, ri.deg - ri.nc);
  } else {
    ri.m = 0;
    ri.fill = min(a.k, ri.deg);
  }
  return ri;
}

// Work item = (row, phase); tier by the positions the phase scans and the
// selections it makes: 3 = thread per item, streaming top-k (take <= 8,
// <= 64 positions), 0 = thread per item, sorting network (<= 16 positions),
// 1 = warp per item (<= kHubLen), 2 = CTA per item (hub)
__device__ __forceinline__ int phase_tier(int len, int take, int stream_len, int thread_len) {
  if (take <= kStreamK && len <= stream_len) return 3;
  if (len > kHubLen) return 2;
  if (len > thread_len) return 1;
  return 0;
}

__device__ __forceinline__ bool cached_bit(const uint32_t* __restrict__ mask, int32_t v) {
  return (__ldg(mask + (v >> 5)) >> (v & 31)) & 1u;
}

// ---- pass 1: per-row counts + exclusive scan (two kernels) ----------------------
// Reduce kernel: all per-row work — row bounds, dst degree, dedup mark of the
// seed, (row, phase) work items into the tier lists, the packed (m, fill)
// count in row_scan[r] and the tile sums.  A thread's kCntItems rows issue
// their loads together (seed ids, then the four CSR offsets) instead of one
// row's dependent chain after another.  Apply kernel: the exclusive scan of
// row_scan only.
constexpr int kCntBlock = 256;
static int g_count_items = 4;   // (gns_tune "count_items": 1, 2, 4) rows per thread of the count pass

template <int kCntItems>
__global__ void __launch_bounds__(kCntBlock) layer_count_reduce_kernel(const __grid_constant__ LayerArgs a,
                                                                       unsigned long long* tile_sums) {
  __shared__ unsigned long long s_warp[kCntBlock / 32 + 1];
  const long long n = a.n_dev[0];
  const long long base = (long long)blockIdx.x * (kCntBlock * kCntItems);
  unsigned long long tsum = 0;
  if (base < n) {
    int32_t node[kCntItems];
#pragma unroll
    for (int j = 0; j < kCntItems; ++j) {
      const long long r = base + j * kCntBlock + threadIdx.x;
      node[j] = r < n ? __ldg(a.seeds + r) : 0;
    }
    int64_t s0[kCntItems], s1[kCntItems], c0[kCntItems], c1[kCntItems];
#pragma unroll
    for (int j = 0; j < kCntItems; ++j) {
      const long long r = base + j * kCntBlock + threadIdx.x;
      s0[j] = s1[j] = c0[j] = c1[j] = 0;
      if (r < n) {
        s0[j] = __ldg(a.indptr + node[j]);
        s1[j] = __ldg(a.indptr + node[j] + 1);
        if (a.gns) {
          c0[j] = __ldg(a.cindptr + node[j]);
          c1[j] = __ldg(a.cindptr + node[j] + 1);
        }
      }
    }
    // per-row values and plain stores (no memory dependence between rows)
    int tier[2 * kCntItems];
#pragma unroll
    for (int j = 0; j < kCntItems; ++j) {
      const long long r = base + j * kCntBlock + threadIdx.x;
      const bool on = r < n;
      const int32_t deg = (int32_t)(s1[j] - s0[j]);
      int32_t m = 0, fill = 0, nc = 0;
      if (a.gns) {
        nc = (int32_t)(c1[j] - c0[j]);
        m = min(a.k, nc);
        fill = a.cache_only ? 0 : min(a.k - m, deg - nc);
      } else {
        fill = min(a.k, deg);
      }
      if (on) {
        const unsigned long long v = ((unsigned long long)m << 32) | (unsigned long long)fill;
        a.b.row_scan[r] = v;
        a.b.dst_degree[r] = deg;
        int4* d = reinterpret_cast<int4*>(a.desc + r);
        d[0] = make_int4((int32_t)(uint64_t)s0[j], (int32_t)((uint64_t)s0[j] >> 32), (int32_t)(uint64_t)c0[j],
                         (int32_t)((uint64_t)c0[j] >> 32));
        d[1] = make_int4(node[j], deg, nc, 0);
        tsum += v;
      }
      // (row, phase) work items into the tier lists (tier_slot); the two
      // phases of a row are independent (their output offsets come from
      // the scan), so they run concurrently
      tier[2 * j] = on && m > 0 ? phase_tier(nc, m, a.stream_len, a.thread_len) : -1;
      tier[2 * j + 1] = on && fill > 0 ? phase_tier(deg, fill, a.stream_len, a.thread_len) : -1;
    }
    // dedup marks of the seeds (fire-and-forget reductions)
    if (a.dbits) {
#pragma unroll
      for (int j = 0; j < kCntItems; ++j)
        if (base + j * kCntBlock + threadIdx.x < n) mark_node(a.dbits, a.dsum, node[j]);
    }
    // all 2*kCntItems (row, phase) items of the warp in one aggregated append
    int h[2 * kCntItems];
    warp_append_tiers<2 * kCntItems>(a.b.counts, tier, h);
#pragma unroll
    for (int j = 0; j < kCntItems; ++j) {
      const long long r = base + j * kCntBlock + threadIdx.x;
#pragma unroll
      for (int ph = 0; ph < 2; ++ph) {
        const int t = tier[2 * j + ph];
        if (t >= 0) a.b.hub_rows[tier_slot(a.max_dst, t, h[2 * j + ph])] = (int32_t)((r << 1) | ph);
      }
    }
  }
  tsum = block_sum<kCntBlock>(tsum, s_warp);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = tsum;
}

template <int kCntItems>
__global__ void __launch_bounds__(kCntBlock) layer_count_apply_kernel(const __grid_constant__ LayerArgs a,
                                                                      const unsigned long long* tile_sums) {
  const long long n = a.n_dev[0];
  scan2_apply<kCntBlock, kCntItems>(
      n, [&](long long r) { return (unsigned long long)a.b.row_scan[r]; },
      [&](long long r, unsigned long long ex, unsigned long long) { a.b.row_scan[r] = ex; },
      [&](unsigned long long tot) {
        a.b.row_scan[n] = tot;
        a.b.counts[GNS_CNT_DST] = (int32_t)n;
        a.b.counts[GNS_CNT_EDGES] = (int32_t)((tot >> 32) + (tot & 0xffffffffull));
        a.b.counts[GNS_CNT_CACHED] = (int32_t)(tot >> 32);
      },
      tile_sums);
}

// ---- selection helpers ------------------------------------------------------
struct PhaseDesc {
  int phase;          // 0 cached, 1 fill, 2 uniform
  int take, cnt, len; // selections, valid candidates, positions to scan
  const int32_t* ids; // neighbour ids of this row/phase (position-indexed)
  bool filter;        // fill phase: skip cached neighbours
  int64_t out_base;   // first output slot
};

// (float arithmetic: T only sets how many candidates pass the filter — the
// exact (key, position) ranking and the bisection retry make the selection
// independent of it — and fp64 sqrt/division cost ~40 instructions per item)
__device__ __forceinline__ uint64_t initial_threshold(int take, int cnt) {
  if (take >= cnt) return kTwo53;
  const float mu = (float)take + 4.f * sqrtf((float)take) + 8.f;
  if (mu >= (float)cnt) return kTwo53;
  const uint64_t t = (uint64_t)(__fdividef(mu, (float)cnt) * 9007199254740992.0f);
  return t < 1 ? 1 : (t > kTwo53 ? kTwo53 : t);
}

// gns-exact (sampling.py:238-250): w = 1 / q[global CSR position]
__device__ __forceinline__ double exact_weight(const LayerArgs& a, const RowInfo& ri, const PhaseDesc& ph,
                                               uint32_t pos) {
  const int64_t gpos = ri.start + (ph.phase == 0 ? (int64_t)__ldg(a.cpos + ri.cstart + pos) : (int64_t)pos);
  const double q = a.exact_q[gpos];
  if (!(q > 0.0)) atomicOr((unsigned*)(a.b.counts + GNS_CNT_ERR), GNS_ERRBIT_ZEROQ);
  return DDIV(1.0, q);
}

__device__ __forceinline__ void emit_edge(const LayerArgs& a, const RowInfo& ri, int64_t r,
                                          const PhaseDesc& ph, int rank, uint32_t pos) {
  const int64_t o = ph.out_base + rank;
  const int32_t u = __ldg(ph.ids + pos);
  double w;
  if (a.exact_q) {
    w = exact_weight(a, ri, ph, pos);
  } else if (ph.phase == 0) {
    double q = DDIV((double)a.k, (double)min(a.k, max(ri.nc, 1)));
    double coeff = DMUL(a.incl[u], q);
    if (!(coeff > 0.0)) atomicOr((unsigned*)(a.b.counts + GNS_CNT_ERR), GNS_ERRBIT_ZEROPROB);
    w = DDIV(1.0, coeff);
  } else if (ph.phase == 1) {
    w = DDIV((double)(ri.deg - ri.nc), (double)max(ri.fill, 1));
  } else {
    w = DDIV((double)ri.deg, (double)max(ri.fill, 1));
  }
  if (a.dbits) mark_node(a.dbits, a.dsum, u);
  a.b.edge_node[o] = u;
  a.b.edge_dst[o] = (int32_t)r;
  a.b.edge_weight[o] = w;
  a.b.edge_cached[o] = ph.phase == 0 ? 1 : 0;
}

// Weight of a selected edge (sampling.py:168,252-258).
__device__ __forceinline__ double edge_weight_of(const LayerArgs& a, const RowInfo& ri, const PhaseDesc& ph,
                                                 double incl_u) {
  if (ph.phase == 0) {
    double q = DDIV((double)a.k, (double)min(a.k, max(ri.nc, 1)));
    double coeff = DMUL(incl_u, q);
    if (!(coeff > 0.0)) atomicOr((unsigned*)(a.b.counts + GNS_CNT_ERR), GNS_ERRBIT_ZEROPROB);
    return DDIV(1.0, coeff);
  }
  if (ph.phase == 1) return DDIV((double)(ri.deg - ri.nc), (double)max(ri.fill, 1));
  return DDIV((double)ri.deg, (double)max(ri.fill, 1));
}

// warp-cooperative selection of one phase of one row
__device__ void warp_select(const LayerArgs& a, const Rng3& rk, const RowInfo& ri, int64_t r, const PhaseDesc& ph,
                            uint64_t* __restrict__ bkey, uint32_t* __restrict__ bpos) {
  const int lane = lane_id();
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t stream = stream_word(32, a.layer, ph.phase);
  uint64_t T = initial_threshold(ph.take, ph.cnt);
  uint64_t lo = 0, hi = kTwo53 + 1;
  const int64_t npairs = ((int64_t)ph.len + 1) >> 1;
  int found = 0;
  // Fill phase: collect every position under T first (Philox ALU only) and
  // probe the cache bitmap for the collected ones afterwards, all lanes'
  // loads in flight together, instead of a dependent id + bitmap load inside
  // every scan iteration that has a hit.  Falls back to the inline probe if
  // the unfiltered candidates overflow the buffer (densely cached rows).
  bool deferred = ph.filter;
  for (int iter = 0; iter < 64; ++iter) {
    found = 0;
    for (int64_t qb = 0; qb < npairs; qb += 32) {
      const int64_t q = qb + lane;
      uint64_t k0 = kTwo53, k1 = kTwo53;
      if (q < npairs) key53_pair(rk.seed, rk.epoch, (uint32_t)ri.node, stream, rk.batch, (uint32_t)q, k0, k1);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t p = 2 * q + j;
        const uint64_t key = j ? k1 : k0;
        bool pred = (q < npairs) && (p < ph.len) && (key < T);
        if (pred && ph.filter && !deferred) pred = !cached_bit(a.mask, __ldg(ph.ids + p));
        unsigned bal = __ballot_sync(GNS_FULL, pred);
        if (pred) {
          int o = found + __popc(bal & lt_mask);
          if (o < kWarpCap) {
            bkey[o] = key;
            bpos[o] = (uint32_t)p;
          }
        }
        found += __popc(bal);
      }
    }
    if (deferred) {
      if (found > kWarpCap) {   // too many cached candidates under T: probe inline
        deferred = false;
        --iter;
        continue;
      }
      __syncwarp();
      // probe the collected candidates: every lane's id loads, then bitmap loads
      constexpr int PER = kWarpCap / 32;
      int32_t idv[PER];
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        const int i = t * 32 + lane;
        idv[t] = i < found ? __ldg(ph.ids + bpos[i]) : 0;
      }
      bool keep[PER];
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        const int i = t * 32 + lane;
        keep[t] = i < found && !cached_bit(a.mask, idv[t]);
      }
      // in-place ordered compaction of the survivors
      int kept = 0;
#pragma unroll
      for (int t = 0; t < PER; ++t) {
        if (t * 32 >= found) break;
        const int i = t * 32 + lane;
        uint64_t kv = 0;
        uint32_t pv = 0;
        if (keep[t]) {
          kv = bkey[i];
          pv = bpos[i];
        }
        const unsigned bal = __ballot_sync(GNS_FULL, keep[t]);
        __syncwarp();
        if (keep[t]) {
          const int o = kept + __popc(bal & lt_mask);
          bkey[o] = kv;
          bpos[o] = pv;
        }
        kept += __popc(bal);
        __syncwarp();
      }
      found = kept;
    }
    if (found > kWarpCap) {
      hi = T;
      uint64_t nt = lo + (T - lo) / 2;
      if (nt <= lo) break;
      T = nt;
    } else if (found < ph.take) {
      lo = T;
      uint64_t nt = (hi > kTwo53) ? (T * 2 > kTwo53 ? kTwo53 : T * 2) : T + (hi - T) / 2;
      if (nt <= T) break;
      T = nt;
    } else {
      break;
    }
  }
  __syncwarp();
  if (found < ph.take || found > kWarpCap) {
    if (lane == 0) atomicOr((unsigned*)(a.b.counts + GNS_CNT_ERR), GNS_ERRBIT_CAPACITY);
    return;
  }
  if (found <= 32 && a.warp_sort) {
    // (the usual case: E[found] = take + 4 sqrt(take) + 8) one candidate per
    // lane, packed (key53 << 11 | pos) — pos < kHubLen = 2^11, so the packed
    // order is the (key, position) order — and a 32-lane bitonic sort by
    // shuffles; lane i then holds rank i
    uint64_t v = lane < found ? (bkey[lane] << 11) | (uint64_t)bpos[lane] : ~0ull;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const uint64_t o = __shfl_xor_sync(GNS_FULL, v, j);
        const bool keep_min = ((lane & j) == 0) == ((lane & k) == 0);
        v = keep_min ? (o < v ? o : v) : (o < v ? v : o);
      }
    }
    if (lane < ph.take) emit_edge(a, ri, r, ph, lane, (uint32_t)(v & 2047u));
    __syncwarp();
    return;
  }
  for (int i = lane; i < found; i += 32) {
    const uint64_t ki = bkey[i];
    const uint32_t pi = bpos[i];
    int rank = 0;
    for (int j = 0; j < found; ++j) {
      const uint64_t kj = bkey[j];
      rank += (kj < ki) || (kj == ki && bpos[j] < pi);
    }
    if (rank < ph.take) emit_edge(a, ri, r, ph, rank, pi);
  }
  __syncwarp();
}

// CTA-cooperative selection for hub rows (NT threads per CTA)
template <int NT>
__device__ void block_select(const LayerArgs& a, const Rng3& rk, const RowInfo& ri, int64_t r, const PhaseDesc& ph,
                             uint64_t* __restrict__ bkey, uint32_t* __restrict__ bpos, int* s_found) {
  const uint32_t stream = stream_word(32, a.layer, ph.phase);
  uint64_t T = initial_threshold(ph.take, ph.cnt);
  uint64_t lo = 0, hi = kTwo53 + 1;
  const int64_t npairs = ((int64_t)ph.len + 1) >> 1;
  int found = 0;
  for (int iter = 0; iter < 64; ++iter) {
    if (threadIdx.x == 0) *s_found = 0;
    __syncthreads();
    for (int64_t q = threadIdx.x; q < npairs; q += NT) {
      uint64_t k0, k1;
      key53_pair(rk.seed, rk.epoch, (uint32_t)ri.node, stream, rk.batch, (uint32_t)q, k0, k1);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int64_t p = 2 * q + j;
        const uint64_t key = j ? k1 : k0;
        bool pred = (p < ph.len) && (key < T);
        if (pred && ph.filter) pred = !cached_bit(a.mask, __ldg(ph.ids + p));
        if (pred) {
          int o = atomicAdd(s_found, 1);
          if (o < kHubCap) {
            bkey[o] = key;
            bpos[o] = (uint32_t)p;
          }
        }
      }
    }
    __syncthreads();
    found = *s_found;
    __syncthreads();
    if (found > kHubCap) {
      hi = T;
      uint64_t nt = lo + (T - lo) / 2;
      if (nt <= lo) break;
      T = nt;
    } else if (found < ph.take) {
      lo = T;
      uint64_t nt = (hi > kTwo53) ? (T * 2 > kTwo53 ? kTwo53 : T * 2) : T + (hi - T) / 2;
      if (nt <= T) break;
      T = nt;
    } else {
      break;
    }
  }
  if (found < ph.take || found > kHubCap) {
    if (threadIdx.x == 0) atomicOr((unsigned*)(a.b.counts + GNS_CNT_ERR), GNS_ERRBIT_CAPACITY);
    __syncthreads();
    return;
  }
  for (int i = threadIdx.x; i < found; i += NT) {
    const uint64_t ki = bkey[i];
    const uint32_t pi = bpos[i];
    int rank = 0;
    for (int j = 0; j < found; ++j) {
      const uint64_t kj = bkey[j];
      rank += (kj < ki) || (kj == ki && bpos[j] < pi);
    }
    if (rank < ph.take) emit_edge(a, ri, r, ph, rank, pi);
  }
  __syncthreads();
}

__device__ __forceinline__ void make_phases(const LayerArgs& a, const RowInfo& ri, int64_t r,
                                            PhaseDesc& pc, PhaseDesc& pf) {
  const uint64_t scan_r = a.b.row_scan[r];
  const uint64_t n = (uint64_t)a.n_dev[0];
  const uint64_t tm = a.b.row_scan[n] >> 32;
  pc.phase = 0;
  pc.take = ri.m;
  pc.cnt = ri.nc;
  pc.len = ri.nc;
  pc.ids = a.cindices + ri.cstart;
  pc.filter = false;
  pc.out_base = (int64_t)(scan_r >> 32);
  pf.phase = a.gns ? 1 : 2;
  pf.take = ri.fill;
  pf.cnt = a.gns ? ri.deg - ri.nc : ri.deg;
  pf.len = ri.deg;
  pf.ids = a.indices + ri.start;
  pf.filter = a.gns != 0;
  pf.out_base = (int64_t)(tm + (scan_r & 0xffffffffull));
}

// Ascending bitonic sorting network over 16 packed keys, compile-time
// indices only (stays in registers).
__device__ __forceinline__ void sort16(uint64_t (&a)[16]) {
#pragma unroll
  for (int k = 2; k <= 16; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const uint64_t x = a[i], y = a[l];
          const bool sw = up ? (y < x) : (x < y);
          a[i] = sw ? y : x;
          a[l] = sw ? x : y;
        }
      }
    }
  }
}

// One thread per row for rows scanning <= 16 positions (the bulk of the
// cache-only input layer): every valid candidate gets the packed key
// (key53 << 11 | position) — ordering = (key, position), exactly the
// reference's stable lexsort — a 16-wide sorting network orders them and the
// first `take` are emitted.  Keys are staged per thread in shared memory so
// the Philox and emit loops stay rolled (small code, no local memory).
__device__ __forceinline__ void thread_select16(const LayerArgs& a, const Rng3& rk, const RowInfo& ri, int64_t r,
                                                const PhaseDesc& ph) {
  const uint32_t stream = stream_word(32, a.layer, ph.phase);
  const int len = ph.len;
  // 1. all neighbour ids and cache-bitmap words of the fill phase in flight
  //    at once (independent loads: no dependent chain per candidate)
  int32_t idv[16];
  uint32_t mw[16];
  if (ph.filter) {
#pragma unroll
    for (int p = 0; p < 16; ++p) idv[p] = p < len ? __ldg(ph.ids + p) : 0;
#pragma unroll
    for (int p = 0; p < 16; ++p) mw[p] = p < len ? __ldg(a.mask + (idv[p] >> 5)) : 0u;
  }
  // 2. Philox keys (ALU) packed with the position: (key53 << 11) | pos
  uint64_t v[16];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint64_t k0 = ~0ull, k1 = ~0ull;
    if (2 * q < len) key53_pair(rk.seed, rk.epoch, (uint32_t)ri.node, stream, rk.batch, (uint32_t)q, k0, k1);
    bool ok0 = 2 * q < len, ok1 = 2 * q + 1 < len;
    if (ph.filter) {
      ok0 = ok0 && !((mw[2 * q] >> (idv[2 * q] & 31)) & 1u);
      ok1 = ok1 && !((mw[2 * q + 1] >> (idv[2 * q + 1] & 31)) & 1u);
    }
    v[2 * q] = ok0 ? ((k0 << 11) | (uint64_t)(2 * q)) : ~0ull;
    v[2 * q + 1] = ok1 ? ((k1 << 11) | (uint64_t)(2 * q + 1)) : ~0ull;
  }
  // 3. (key, position) order = the reference's stable lexsort
  sort16(v);
  // 4. emit the first `take`: every load (neighbour id, inclusion)
  //    of all selected edges is issued before any store, so the edges' memory
  //    latencies overlap instead of serialising behind possibly-aliasing stores
  const int take = ph.take;
  int32_t u[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) u[i] = i < take ? __ldg(ph.ids + (uint32_t)(v[i] & 2047u)) : 0;
  double inc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) inc[i] = (i < take && ph.phase == 0 && !a.exact_q) ? __ldg(a.incl + u[i]) : 0.0;
  const int64_t o0 = ph.out_base;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (i < take) {
      const double w = a.exact_q ? exact_weight(a, ri, ph, (uint32_t)(v[i] & 2047u))
                                 : edge_weight_of(a, ri, ph, inc[i]);
      mark_node(a.dbits, a.dsum, u[i]);
      a.b.edge_node[o0 + i] = u[i];
      a.b.edge_dst[o0 + i] = (int32_t)r;
      a.b.edge_weight[o0 + i] = w;
      a.b.edge_cached[o0 + i] = ph.phase == 0 ? 1 : 0;
    }
  }
}

// One thread per item, take <= kStreamK, <= kStreamLen positions: keys are
// generated 8 positions at a time and inserted into a sorted register array
// of the kStreamK smallest packed (key53 << 11 | position) values — the
// reference's (key, position) lexsort order — so only ~kStreamK live keys
// are held (the sorting-network tier holds 16 plus the candidates' ids).
template <int K>
__device__ __forceinline__ void insert_sorted(uint64_t (&best)[K], uint64_t v) {
#pragma unroll
  for (int i = K - 1; i >= 1; --i) {
    const uint64_t lo = best[i - 1];
    best[i] = v < lo ? lo : (v < best[i] ? v : best[i]);
  }
  best[0] = v < best[0] ? v : best[0];
}

// K = the kept-key count (>= take): kStreamK, or 5 for layers whose fanout
// is <= 5 (the cache-only input layer: each insertion is a K-1 step
// compare-select chain on 64-bit keys, as costly as the Philox pair itself)
template <int K>
__device__ __forceinline__ void thread_select_stream(const LayerArgs& a, const Rng3& rk, const RowInfo& ri,
                                                     int64_t r, const PhaseDesc& ph) {
  const uint32_t stream = stream_word(32, a.layer, ph.phase);
  const int len = ph.len;
  uint64_t best[K];
#pragma unroll
  for (int i = 0; i < K; ++i) best[i] = ~0ull;
  for (int p0 = 0; p0 < len; p0 += 8) {
    // fill phase: the 8 neighbour ids and cache-bitmap words in flight at once
    int32_t idv[8];
    uint32_t mw[8];
    if (ph.filter) {
#pragma unroll
      for (int j = 0; j < 8; ++j) idv[j] = p0 + j < len ? __ldg(ph.ids + p0 + j) : 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) mw[j] = p0 + j < len ? __ldg(a.mask + (idv[j] >> 5)) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int p = p0 + 2 * q;
      if (p >= len) break;
      uint64_t k0, k1;
      key53_pair(rk.seed, rk.epoch, (uint32_t)ri.node, stream, rk.batch, (uint32_t)(p >> 1), k0, k1);
      bool ok0 = true, ok1 = p + 1 < len;
      if (ph.filter) {
        ok0 = !((mw[2 * q] >> (idv[2 * q] & 31)) & 1u);
        ok1 = ok1 && !((mw[2 * q + 1] >> (idv[2 * q + 1] & 31)) & 1u);
      }
      if (ok0) insert_sorted<K>(best, (k0 << 11) | (uint64_t)p);
      if (ok1) insert_sorted<K>(best, (k1 << 11) | (uint64_t)(p + 1));
    }
  }
  // emit the first `take`, 4 at a time: every load of a chunk's edges
  // (neighbour id, inclusion, dedup word) before any of its stores
  const int take = ph.take;
  const int64_t o0 = ph.out_base;
#pragma unroll
  for (int c0 = 0; c0 < K; c0 += 4) {
    if (c0 >= take) break;
    int32_t u[4];
    double inc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
      u[i] = (c0 + i < K && c0 + i < take) ? __ldg(ph.ids + (uint32_t)(best[(c0 + i) % K] & 2047u)) : 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      inc[i] = (c0 + i < take && ph.phase == 0 && !a.exact_q) ? __ldg(a.incl + u[i]) : 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (c0 + i < take) {
        const double w = a.exact_q ? exact_weight(a, ri, ph, (uint32_t)(best[(c0 + i) % K] & 2047u))
                                   : edge_weight_of(a, ri, ph, inc[i]);
        mark_node(a.dbits, a.dsum, u[i]);
        a.b.edge_node[o0 + c0 + i] = u[i];
        a.b.edge_dst[o0 + c0 + i] = (int32_t)r;
        a.b.edge_weight[o0 + c0 + i] = w;
        a.b.edge_cached[o0 + c0 + i] = ph.phase == 0 ? 1 : 0;
      }
    }
  }
}

template <int MINB, int K = kStreamK>
__global__ void __launch_bounds__(256, MINB) sample_stream_kernel(const __grid_constant__ LayerArgs a) {
  const Rng3 rk = batch_rng(a);
  const int64_t nl = a.b.counts[GNS_CNT_STREAMROWS];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nl; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t item = a.b.hub_rows[2 * a.max_dst + j];
    const int64_t r = item >> 1;
    RowInfo ri = row_info(a, r);
    PhaseDesc pc, pf;
    make_phases(a, ri, r, pc, pf);
    thread_select_stream<K>(a, rk, ri, r, (item & 1) ? pf : pc);
  }
}

__global__ void __launch_bounds__(256) sample_thread_kernel(const __grid_constant__ LayerArgs a) {
  const Rng3 rk = batch_rng(a);
  const int64_t nl = a.b.counts[GNS_CNT_THREADROWS];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nl; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t item = a.b.hub_rows[j];
    const int64_t r = item >> 1;
    RowInfo ri = row_info(a, r);
    PhaseDesc pc, pf;
    make_phases(a, ri, r, pc, pf);
    thread_select16(a, rk, ri, r, (item & 1) ? pf : pc);
  }
}

// Warp tier, then the hub tier (rows scanning > kHubLen positions, rare) by
// whole CTAs at the tail of the same launch: one launch less per layer.
__global__ void __launch_bounds__(kSampBlock, 4) sample_warp_kernel(const __grid_constant__ LayerArgs a) {
  static_assert(kSampBlock / 32 * kWarpCap >= kHubCap, "hub stage must fit the warps' stages");
  const Rng3 rk = batch_rng(a);
  __shared__ uint64_t s_key[kSampBlock / 32][kWarpCap];
  __shared__ uint32_t s_pos[kSampBlock / 32][kWarpCap];
  __shared__ int s_found;
  const int w = threadIdx.x >> 5;
  const int64_t nl = a.b.counts[GNS_CNT_WARPROWS];
  const int64_t gw = (blockIdx.x * (int64_t)kSampBlock + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * kSampBlock) >> 5;
  for (int64_t j = gw; j < nl; j += nw) {
    const int32_t item = a.b.hub_rows[4 * a.max_dst + j];
    const int64_t r = item >> 1;
    RowInfo ri = row_info(a, r);
    PhaseDesc pc, pf;
    make_phases(a, ri, r, pc, pf);
    warp_select(a, rk, ri, r, (item & 1) ? pf : pc, s_key[w], s_pos[w]);
  }
  const int nh = a.b.counts[GNS_CNT_HUBS];
  if ((int)blockIdx.x >= nh) return;   // CTA-uniform
  __syncthreads();                      // the warps' stages become the CTA's
  for (int h = blockIdx.x; h < nh; h += gridDim.x) {
    const int32_t item = a.b.hub_rows[6 * a.max_dst - 1 - h];
    const int64_t r = item >> 1;
    RowInfo ri = row_info(a, r);
    PhaseDesc pc, pf;
    make_phases(a, ri, r, pc, pf);
    block_select<kSampBlock>(a, rk, ri, r, (item & 1) ? pf : pc, &s_key[0][0], &s_pos[0][0], &s_found);
  }
}

// ---- dedup / relabel ----------------------------------------------------------
// Two-level bitmap: bits (1 per node id, N/8 bytes) + summary (1 per bitmap
// word).  Enumeration scans only the summary (N/1024 words) and the non-zero
// bitmap words, emits the sorted unique ids, stores (rank << 32 | word) per
// non-zero word for the relabel lookups, and clears both levels as it goes —
// the bitmaps are left zero without a separate clearing pass.
__global__ void setbits_kernel(const int32_t* __restrict__ a, const int32_t* __restrict__ na_dev, int64_t na_host,
                               const int32_t* __restrict__ b, const int32_t* __restrict__ nb_dev,
                               uint32_t* __restrict__ bits, uint32_t* __restrict__ sum) {
  const int64_t na = na_dev ? na_dev[0] : na_host;
  const int64_t nb = (b && nb_dev) ? nb_dev[0] : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = i < na ? a[i] : b[i - na];
    mark_node(bits, sum, v);
  }
}

// A warp walks kEnumSeg segments of 8 summary words (256 bitmap words each);
// a segment's bitmap words are read as 8 consecutive words per lane (two
// 16-B loads, skipped when the lane's 8 summary bits are zero), so the output
// order — ascending word — is lane-major within a segment and one warp scan
// ranks a segment's words.  Tile = 8 warps x kEnumSeg segments (256 summary
// words, 262144 node ids per CTA): the per-CTA prefix / block sums are paid
// once per 4 segments (the work of a sparse layer is mostly that fixed cost).
constexpr int kEnumBlock = 256;
constexpr int kEnumWarps = kEnumBlock / 32;
constexpr int kEnumPerWarp = 8;   // summary words per segment
constexpr int kEnumSeg = 4;       // segments per warp
constexpr int kEnumTileSw = kEnumWarps * kEnumPerWarp * kEnumSeg;

// lane's 8 bitmap words of the segment at summary word sw0 (bitmap words
// sw0 * 32 + 8 * lane ...) and their popcount
__device__ __forceinline__ unsigned enum_lane_words(const uint32_t* __restrict__ bits,
                                                    const uint32_t* __restrict__ sum, int64_t nsw, long long sw0,
                                                    int lane, uint4& w0, uint4& w1) {
  const long long sw = sw0 + (lane >> 2);
  const uint32_t smw = sw < nsw ? sum[sw] : 0u;
  const uint32_t sb = (smw >> (8 * (lane & 3))) & 0xffu;
  w0 = make_uint4(0u, 0u, 0u, 0u);
  w1 = make_uint4(0u, 0u, 0u, 0u);
  const uint4* p = reinterpret_cast<const uint4*>(bits + sw0 * 32 + 8 * lane);
  if (sb & 0x0fu) w0 = p[0];
  if (sb & 0xf0u) w1 = p[1];
  return __popc(w0.x) + __popc(w0.y) + __popc(w0.z) + __popc(w0.w) + __popc(w1.x) + __popc(w1.y) + __popc(w1.z) +
         __popc(w1.w);
}

__device__ __forceinline__ long long enum_seg0(long long tile, int warp, int g) {
  return (tile * kEnumWarps + warp) * (long long)(kEnumPerWarp * kEnumSeg) + g * kEnumPerWarp;
}

__global__ void __launch_bounds__(kEnumBlock) enumerate_reduce_kernel(const uint32_t* __restrict__ bits,
                                                                      const uint32_t* __restrict__ sum, int64_t nsw,
                                                                      unsigned long long* tile_sums) {
  __shared__ unsigned long long s_w[kEnumWarps + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned c = 0;
#pragma unroll
  for (int g = 0; g < kEnumSeg; ++g) {
    uint4 w0, w1;
    c += enum_lane_words(bits, sum, nsw, enum_seg0(blockIdx.x, warp, g), lane, w0, w1);
  }
  unsigned long long t = block_sum<kEnumBlock>((unsigned long long)c, s_w);
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kEnumBlock) enumerate_apply_kernel(uint32_t* __restrict__ bits,
                                                                     uint32_t* __restrict__ sum, int64_t nsw,
                                                                     const unsigned long long* tile_sums,
                                                                     unsigned long long* __restrict__ rank2,
                                                                     int32_t* __restrict__ out,
                                                                     int32_t* __restrict__ out_n) {
  __shared__ unsigned long long s_w[kEnumWarps + 1];
  __shared__ unsigned long long s_wpre[kEnumWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long ntiles = (nsw + kEnumTileSw - 1) / kEnumTileSw;
  const long long tile = blockIdx.x;
  if (nsw == 0) {
    if (tile == 0 && threadIdx.x == 0) out_n[0] = 0;
    return;
  }
  if (tile >= ntiles) return;
  unsigned long long pre = 0;
  for (long long j = threadIdx.x; j < tile; j += kEnumBlock) pre += tile_sums[j];
  pre = block_sum<kEnumBlock>(pre, s_w);
  uint4 w[kEnumSeg][2];
  unsigned c[kEnumSeg], ct = 0;
#pragma unroll
  for (int g = 0; g < kEnumSeg; ++g) {
    c[g] = enum_lane_words(bits, sum, nsw, enum_seg0(tile, warp, g), lane, w[g][0], w[g][1]);
    ct += c[g];
  }
  const unsigned wtot = warp_sum(ct);
  if (lane == 0) s_wpre[warp] = wtot;
  __syncthreads();
  unsigned long long base = pre;
  for (int v = 0; v < warp; ++v) base += s_wpre[v];
  if (tile == ntiles - 1 && warp == kEnumWarps - 1 && lane == 0) out_n[0] = (int32_t)(base + wtot);
  if (wtot) {
#pragma unroll
    for (int g = 0; g < kEnumSeg; ++g) {
      const unsigned incl = warp_incl_scan(c[g]);
      unsigned long long o = base + incl - c[g];
      base += __shfl_sync(GNS_FULL, incl, 31);
      if (c[g]) {
        const uint32_t x8[8] = {w[g][0].x, w[g][0].y, w[g][0].z, w[g][0].w,
                                w[g][1].x, w[g][1].y, w[g][1].z, w[g][1].w};
        const long long wbase = enum_seg0(tile, warp, g) * 32 + 8 * lane;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t x = x8[i];
          if (x) {
            const long long wd = wbase + i;
            rank2[wd] = (o << 32) | (unsigned long long)x;
            bits[wd] = 0u;
            uint32_t y = x;
            while (y) {
              const int bb = __ffs(y) - 1;
              y &= y - 1;
              out[o++] = (int32_t)(wd * 32 + bb);
            }
          }
        }
      }
    }
  }
  if (lane < kEnumPerWarp * kEnumSeg) {
    const long long sw = enum_seg0(tile, warp, 0) + lane;
    if (sw < nsw) sum[sw] = 0u;
  }
}

__device__ __forceinline__ int32_t bit_rank(const unsigned long long* __restrict__ rank2, int32_t v) {
  const unsigned long long rw = rank2[v >> 5];
  return (int32_t)(rw >> 32) + __popc((uint32_t)rw & ((1u << (v & 31)) - 1u));
}

__global__ void relabel_kernel(const unsigned long long* __restrict__ rank2, const int32_t* __restrict__ seeds,
                               const int32_t* __restrict__ n_seeds_dev, const int32_t* __restrict__ edge_node,
                               const int32_t* __restrict__ counts, int32_t* __restrict__ self_pos,
                               int32_t* __restrict__ edge_src) {
  const int64_t ns = n_seeds_dev[0];
  const int64_t ne = counts[GNS_CNT_EDGES];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ns + ne;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < ns)
      self_pos[i] = bit_rank(rank2, seeds[i]);
    else
      edge_src[i - ns] = bit_rank(rank2, edge_node[i - ns]);
  }
}

// np.unique for small id lists (<= kSmallUnique, e.g. the 1000 targets of a
// batch): one CTA, bitonic sort in shared memory, then an ordered compaction
// of the first element of every run.  Replaces setbits + two enumerate passes
// over the N/1024-word summary bitmap.
constexpr int kSmallUnique = 4096;
constexpr int kSmallBlock = 1024;

__global__ void __launch_bounds__(kSmallBlock) unique_small_kernel(const int32_t* __restrict__ ids,
                                                                   const int32_t* __restrict__ n_dev, int64_t n_host,
                                                                   int32_t* __restrict__ out,
                                                                   int32_t* __restrict__ out_n) {
  __shared__ int32_t key[kSmallUnique];
  __shared__ unsigned long long s_warp[kSmallBlock / 32 + 1];
  const int n = (int)(n_dev ? min((int64_t)n_dev[0], n_host) : n_host);
  int P = 1;
  while (P < n) P <<= 1;
  for (int i = threadIdx.x; i < P; i += kSmallBlock) key[i] = i < n ? ids[i] : INT32_MAX;
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += kSmallBlock) {
        const int l = i ^ j;
        if (l > i) {
          const int32_t x = key[i], y = key[l];
          const bool up = (i & k) == 0;
          if (up ? (y < x) : (x < y)) {
            key[i] = y;
            key[l] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  // each thread owns a contiguous chunk of <= 4 sorted keys
  constexpr int IT = kSmallUnique / kSmallBlock;
  const int b0 = threadIdx.x * IT;
  unsigned c = 0;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const int i = b0 + q;
    if (i < n && (i == 0 || key[i] != key[i - 1])) ++c;
  }
  unsigned long long total;
  unsigned long long o = block_excl_scan<kSmallBlock>((unsigned long long)c, s_warp, total);
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const int i = b0 + q;
    if (i < n && (i == 0 || key[i] != key[i - 1])) out[o++] = key[i];
  }
  if (threadIdx.x == 0) out_n[0] = (int32_t)total;
}

struct DedupWs {
  uint32_t* bits;
  uint32_t* sum;
  unsigned long long* rank2;
  unsigned long long* tiles;
  int64_t nw, nsw;
};

static void dedup_ws(int64_t num_nodes, Workspace& w, DedupWs* d) {
  d->nw = (num_nodes + 31) / 32;
  d->nsw = (d->nw + 31) / 32;
  d->bits = w.take<uint32_t>(d->nw + 1);
  d->sum = w.take<uint32_t>(d->nsw + 1);
  d->rank2 = w.take<unsigned long long>(d->nw + 1);
  d->tiles = w.take<unsigned long long>(d->nsw / kEnumTileSw + 2);
}

static int run_enumerate(const DedupWs& d, int32_t* out, int32_t* out_n, cudaStream_t stream) {
  const unsigned tiles = (unsigned)((d.nsw + kEnumTileSw - 1) / kEnumTileSw);
  enumerate_reduce_kernel<<<tiles ? tiles : 1, kEnumBlock, 0, stream>>>(d.bits, d.sum, d.nsw, d.tiles);
  enumerate_apply_kernel<<<tiles ? tiles : 1, kEnumBlock, 0, stream>>>(d.bits, d.sum, d.nsw, d.tiles, d.rank2, out,
                                                                     out_n);
  return check_launch("enumerate");
}

static int run_relabel(const DedupWs& d, const int32_t* seeds, const int32_t* n_seeds_dev, int64_t max_dst,
                       gns_block_t* block, int64_t max_edges, cudaStream_t stream) {
  GNS_TRY(run_enumerate(d, block->src_nodes, block->counts + GNS_CNT_SRC, stream));
  const int grid = resident_grid(relabel_kernel, 256, 0,
                                 grid_for((max_dst + max_edges + 255) / 256 + 1,
                                          g_sampler_ctas ? (long long)num_sms() * g_sampler_ctas : (1LL << 30)));
  relabel_kernel<<<grid, 256, 0, stream>>>(d.rank2, seeds, n_seeds_dev, block->edge_node, block->counts,
                                           block->self_pos, block->edge_src);
  return check_launch("relabel");
}

}  // namespace gns

using namespace gns;

extern "C" {

// The dedup bitmaps come first so their offsets depend on num_nodes only:
// every layer of a batch (different max_dst) sees the same, zeroed bitmaps.
// (With the count tile sums first, a larger layer's tile sums were written
// over the bitmap words of the smaller layers' layout.)
static size_t sample_ws(int64_t num_nodes, int64_t max_dst, void* base, size_t cap, unsigned long long** tiles,
                        DedupWs* d, RowDesc** desc) {
  Workspace w(base, cap);
  dedup_ws(num_nodes, w, d);
  *tiles = w.take<unsigned long long>(max_dst / kCntBlock + 2);   // count tiles of >= kCntBlock rows
  *desc = w.take<RowDesc>(max_dst + 1);
  return w.off;
}

size_t gns_sample_workspace_size(int64_t num_nodes, int64_t max_dst) {
  unsigned long long* t;
  DedupWs d;
  RowDesc* desc;
  return sample_ws(num_nodes, max_dst, nullptr, 0, &t, &d, &desc);
}

int gns_sample_layer(const gns_graph_t* g, const gns_cache_t* cache, const int32_t* seeds,
                     const int32_t* n_seeds_dev, int64_t max_dst, int32_t k, int32_t cache_only,
                     const double* exact_q, const gns_rng_t* rng, const gns_step_t* step_dev, gns_block_t* block,
                     void* ws, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (k < 1) {
    set_error("fanout must be >= 1");
    return GNS_EINVAL;
  }
  if (k > kMaxFanout) {
    set_error("fanout %d exceeds the supported maximum %d", k, kMaxFanout);
    return GNS_EINVAL;
  }
  unsigned long long* ctiles;
  DedupWs dd;
  RowDesc* desc;
  size_t need = sample_ws(g->num_nodes, max_dst, ws, ws_bytes, &ctiles, &dd, &desc);
  if (ws_bytes < need) {
    set_error("sample_layer: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  LayerArgs a;
  a.indptr = g->indptr;
  a.indices = g->indices;
  a.gns = cache != nullptr;
  a.cindptr = cache ? cache->cached_indptr : nullptr;
  a.cindices = cache ? cache->cached_indices : nullptr;
  a.mask = cache ? cache->mask_bits : nullptr;
  a.incl = cache ? cache->inclusion : nullptr;
  a.cpos = cache ? cache->cached_pos : nullptr;
  a.exact_q = exact_q;
  if (exact_q && cache && !cache->cached_pos) {
    set_error("gns-exact needs the cache's cached_pos array");
    return GNS_EINVAL;
  }
  a.seeds = seeds;
  a.n_dev = n_seeds_dev;
  a.k = k;
  a.cache_only = cache_only;
  a.max_dst = max_dst;
  a.seed = rng->seed;
  a.epoch = rng->epoch;
  a.batch = rng->batch;
  a.layer = rng->layer;
  a.step_dev = step_dev;
  a.dbits = dd.bits;
  a.dsum = dd.sum;
  a.stream_len = g_stream_len;
  a.thread_len = g_thread_len;
  a.warp_sort = g_warp_sort;
  a.desc = desc;
  a.b = *block;
  GNS_CUDA(cudaMemsetAsync(block->counts, 0, GNS_CNT_N * sizeof(int32_t), stream));
#define GNS_COUNT(IT)                                                                                  \
  {                                                                                                    \
    const unsigned tiles = (unsigned)((max_dst + kCntBlock * IT - 1) / (kCntBlock * IT)) + 1;         \
    layer_count_reduce_kernel<IT><<<tiles, kCntBlock, 0, stream>>>(a, ctiles);                         \
    layer_count_apply_kernel<IT><<<tiles, kCntBlock, 0, stream>>>(a, ctiles);                          \
  }
  if (g_count_items == 1) GNS_COUNT(1)
  else if (g_count_items == 2) GNS_COUNT(2)
  else GNS_COUNT(4)
#undef GNS_COUNT
  GNS_TRY(check_launch("layer_count"));
  const int sms = num_sms();
  // the three tiers work on disjoint (row, phase) lists: thread tier on the
  // calling stream, warp and hub tiers on a forked branch, concurrently
  Fork fk;
  GNS_TRY(fork_begin(stream, &fk));
  // one wave of resident CTAs at most (grid-stride loops over the item lists)
  const long long cap = g_sampler_ctas ? (long long)sms * g_sampler_ctas : (1LL << 30);
  const long long titems = grid_for((2 * max_dst + 255) / 256, cap);
  if (k <= 5 && g_stream_k5)   // every take of this layer is <= k <= 5
    sample_stream_kernel<1, 5><<<resident_grid(sample_stream_kernel<1, 5>, 256, 0, titems), 256, 0, stream>>>(a);
  else if (g_stream_minb == 4)
    sample_stream_kernel<4><<<resident_grid(sample_stream_kernel<4>, 256, 0, titems), 256, 0, stream>>>(a);
  else if (g_stream_minb == 3)
    sample_stream_kernel<3><<<resident_grid(sample_stream_kernel<3>, 256, 0, titems), 256, 0, stream>>>(a);
  else
    sample_stream_kernel<1><<<resident_grid(sample_stream_kernel<1>, 256, 0, titems), 256, 0, stream>>>(a);
  GNS_TRY(check_launch("sample_stream"));
  if (g_thread_len > 0) {   // (thread_len 0: phase_tier never picks the sorting-network tier)
    sample_thread_kernel<<<resident_grid(sample_thread_kernel, 256, 0, titems), 256, 0, stream>>>(a);
    GNS_TRY(check_launch("sample_thread"));
  }
  // warp tier + the hub tier at its tail (at least one CTA per SM for hubs)
  const int grid = resident_grid(sample_warp_kernel, kSampBlock, 0,
                                 std::max<long long>(sms, grid_for((2 * max_dst * 32 + kSampBlock - 1) / kSampBlock,
                                                                   cap)));
  sample_warp_kernel<<<grid, kSampBlock, 0, fk.aux>>>(a);
  GNS_TRY(check_launch("sample_warp"));
  GNS_TRY(fork_join(stream, fk));
  // _assemble (sampling.py:139-152): seeds and sampled neighbours were marked
  // in the dedup bitmap by the count / sample kernels
  return run_relabel(dd, seeds, n_seeds_dev, max_dst, block, max_dst * (int64_t)k, stream);
}

int gns_sample_tune(const char* name, int32_t value) {
  if (!strcmp(name, "stream_len") && value >= 0 && value < 2048) {
    g_stream_len = value;
    return GNS_OK;
  }
  if (!strcmp(name, "thread_len") && value >= 0 && value <= kThreadLen) {
    g_thread_len = value;
    return GNS_OK;
  }
  if (!strcmp(name, "sampler_ctas") && value >= 0) {
    g_sampler_ctas = value;
    return GNS_OK;
  }
  if (!strcmp(name, "stream_k5") && (value == 0 || value == 1)) {
    g_stream_k5 = value;
    return GNS_OK;
  }
  if (!strcmp(name, "warp_sort") && (value == 0 || value == 1)) {
    g_warp_sort = value;
    return GNS_OK;
  }
  if (!strcmp(name, "count_items") && (value == 1 || value == 2 || value == 4)) {
    g_count_items = value;
    return GNS_OK;
  }
  if (!strcmp(name, "stream_minb") && (value == 1 || value == 3 || value == 4)) {
    g_stream_minb = value;
    return GNS_OK;
  }
  return GNS_EINVAL;
}

size_t gns_relabel_workspace_size(int64_t num_nodes) {
  Workspace w(nullptr, 0);
  DedupWs d;
  dedup_ws(num_nodes, w, &d);
  return w.off;
}

int gns_relabel(int64_t num_nodes, const int32_t* seeds, const int32_t* n_seeds_dev, int64_t max_dst,
                gns_block_t* block, int64_t max_edges, void* ws, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  Workspace w(ws, ws_bytes);
  DedupWs d;
  dedup_ws(num_nodes, w, &d);
  if (!w.ok()) {
    set_error("relabel: workspace %zu < %zu", ws_bytes, w.off);
    return GNS_EINVAL;
  }
  int grid = grid_for((max_dst + max_edges + 255) / 256 + 1, (long long)num_sms() * 16);
  setbits_kernel<<<grid, 256, 0, stream>>>(seeds, n_seeds_dev, 0, block->edge_node, block->counts + GNS_CNT_EDGES,
                                           d.bits, d.sum);
  GNS_TRY(check_launch("setbits"));
  return run_relabel(d, seeds, n_seeds_dev, max_dst, block, max_edges, stream);
}

int gns_unique_sorted(int64_t num_nodes, const int32_t* ids, const int32_t* n_dev, int64_t n_host, int32_t* out,
                      int32_t* out_n_dev, void* ws, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  Workspace w(ws, ws_bytes);
  DedupWs d;
  dedup_ws(num_nodes, w, &d);
  if (!w.ok()) {
    set_error("unique_sorted: workspace %zu < %zu", ws_bytes, w.off);
    return GNS_EINVAL;
  }
  if (n_host <= kSmallUnique) {
    unique_small_kernel<<<1, kSmallBlock, 0, stream>>>(ids, n_dev, n_host, out, out_n_dev);
    return check_launch("unique_small");
  }
  int grid = grid_for((n_host + 255) / 256 + 1, (long long)num_sms() * 16);
  setbits_kernel<<<grid, 256, 0, stream>>>(ids, n_dev, n_host, nullptr, nullptr, d.bits, d.sum);
  GNS_TRY(check_launch("setbits"));
  return run_enumerate(d, out, out_n_dev, stream);
}

}  // extern "C"
