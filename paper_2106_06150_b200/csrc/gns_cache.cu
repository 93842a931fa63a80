// Cache engine on B200: the degree-proportional cache draw (cache.py:87-103)
// and the induced cached-neighbour CSR (cache.py:185-197).
//
// Draw = exponential race.  key(i) = -log(1 - U_i) / p_i over p_i > 0, U_i from
// Philox at (tag 33, node 0, pos = i).  The |C| smallest (key, id) pairs are
// found with an 11-bit-digit radix select over the key bit patterns (positive
// doubles order like their uint64 bits), then one ordered stream compaction
// emits sorted ids and the membership bitmap.  Ties at the threshold key are
// broken by node id (oracle/gns.py:sample_cache).
#include "gns_common.cuh"

namespace gns {

static constexpr int kDigitBits[6] = {11, 11, 11, 11, 11, 9};
static constexpr int kDigitShift[6] = {53, 42, 31, 20, 9, 0};
static constexpr uint64_t kNoKey = ~0ull;  // non-support sentinel (> +inf bits)

struct SelectState {
  unsigned long long prefix;       // selected high bits so far
  unsigned long long prefix_mask;  // which bits are fixed
  long long remaining;             // rank (1-based) still to find inside the prefix
  long long k_eff;                 // min(cache_size, support)
  unsigned long long support;      // |{p > 0}|
  long long pad[3];
};

__global__ void cache_keys_kernel(const double* __restrict__ probs, int64_t n, uint32_t seed,
                                  uint32_t epoch, uint32_t tag, uint64_t* __restrict__ keys,
                                  SelectState* __restrict__ st) {
  const uint32_t stream = stream_word(tag, 0, 0);
  unsigned long long local = 0;
  // each thread handles pairs (2q, 2q+1) so one Philox block serves two nodes
  const int64_t npairs = (n + 1) >> 1;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < npairs;
       q += (int64_t)gridDim.x * blockDim.x) {
    uint64_t ke, ko;
    key53_pair(seed, epoch, 0u, stream, 0u, (uint32_t)q, ke, ko);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      int64_t i = 2 * q + j;
      if (i >= n) break;
      double p = probs[i];
      uint64_t out = kNoKey;
      if (p > 0.0) {
        uint64_t k53 = j ? ko : ke;
        double u = (double)k53 * 0x1p-53;   // exact
        double e = -det_log(DSUB(1.0, u));  // Exp(1); 1-u exact
        double key = DDIV(e, p);
        out = (uint64_t)__double_as_longlong(key);
        ++local;
      }
      keys[i] = out;
    }
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(&st->support, local);
}

__global__ void select_init_kernel(SelectState* st, int64_t cache_size) {
  long long sup = (long long)st->support;
  long long k = cache_size < sup ? cache_size : sup;
  if (k < 0) k = 0;
  st->k_eff = k;
  st->remaining = k;
  st->prefix = 0;
  st->prefix_mask = 0;
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) radix_hist_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                                           const SelectState* __restrict__ st, int shift,
                                                           int bits, unsigned int* __restrict__ hist) {
  __shared__ unsigned int sh[2048];
  const int nb = 1 << bits;
  for (int i = threadIdx.x; i < nb; i += BLOCK) sh[i] = 0;
  __syncthreads();
  const unsigned long long prefix = st->prefix, pmask = st->prefix_mask;
  if (st->remaining > 0) {
    for (int64_t i = blockIdx.x * (int64_t)BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
      uint64_t k = keys[i];
      if (k != kNoKey && (k & pmask) == prefix) atomicAdd(&sh[(k >> shift) & (nb - 1)], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += BLOCK)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
}

// one block of 1024 threads: find the digit that contains rank `remaining`.
__global__ void radix_pick_kernel(SelectState* st, int shift, int bits, unsigned int* hist) {
  __shared__ unsigned long long part[1024];
  __shared__ int s_bin;
  __shared__ unsigned long long s_below;
  const int nb = 1 << bits;
  const int per = (nb + 1023) / 1024;  // 2 for 2048 bins
  const long long rem = st->remaining;
  unsigned long long c[2] = {0, 0};
  unsigned long long tsum = 0;
  for (int j = 0; j < per; ++j) {
    int b = threadIdx.x * per + j;
    c[j] = (b < nb) ? hist[b] : 0;
    tsum += c[j];
  }
  part[threadIdx.x] = tsum;
  __syncthreads();
  // Hillis-Steele inclusive scan over 1024 partials
  for (int o = 1; o < 1024; o <<= 1) {
    unsigned long long t = (threadIdx.x >= o) ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += t;
    __syncthreads();
  }
  if (threadIdx.x == 0) { s_bin = -1; s_below = 0; }
  __syncthreads();
  if (rem > 0) {
    unsigned long long run = part[threadIdx.x] - tsum;  // exclusive
    for (int j = 0; j < per; ++j) {
      int b = threadIdx.x * per + j;
      if (b < nb && run < (unsigned long long)rem && run + c[j] >= (unsigned long long)rem) {
        s_bin = b;
        s_below = run;
      }
      run += c[j];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && rem > 0 && s_bin >= 0) {
    unsigned long long dmask = ((unsigned long long)(nb - 1)) << shift;
    st->prefix |= ((unsigned long long)s_bin) << shift;
    st->prefix_mask |= dmask;
    st->remaining = rem - (long long)s_below;
  }
  for (int b = threadIdx.x; b < nb; b += 1024) hist[b] = 0;  // ready for next pass
}

// classify: per 32-node word, bits of keys < T and keys == T.
__global__ void classify_kernel(const uint64_t* __restrict__ keys, int64_t n, const SelectState* __restrict__ st,
                                uint32_t* __restrict__ less_bits, uint32_t* __restrict__ eq_bits) {
  const bool any = st->k_eff > 0;
  const unsigned long long T = st->prefix;
  const int64_t nw = (n + 31) >> 5;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw * 32;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t k = (i < n) ? keys[i] : kNoKey;
    bool lt = any && k != kNoKey && k < T;
    bool eq = any && k != kNoKey && k == T;
    unsigned bl = __ballot_sync(GNS_FULL, lt);
    unsigned be = __ballot_sync(GNS_FULL, eq);
    if ((threadIdx.x & 31) == 0) {
      less_bits[i >> 5] = bl;
      eq_bits[i >> 5] = be;
    }
  }
}

// ordered compaction over words: value = (popc(less) << 32) | popc(eq)
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) cache_compact_kernel(ScanStatus ss, const uint32_t* __restrict__ less_bits,
                                                              const uint32_t* __restrict__ eq_bits, int64_t nw,
                                                              const SelectState* __restrict__ st,
                                                              int32_t* __restrict__ out_ids,
                                                              uint32_t* __restrict__ out_mask,
                                                              int64_t* __restrict__ out_counts) {
  const long long need_eq = st->remaining;  // equal keys still to take, in id order
  scan_tiles<BLOCK, ITEMS>(
      ss, nw,
      [&](long long w) {
        return ((unsigned long long)__popc(less_bits[w]) << 32) | (unsigned long long)__popc(eq_bits[w]);
      },
      [&](long long w, unsigned long long ex, unsigned long long) {
        long long a_ex = (long long)(ex >> 32), b_ex = (long long)(ex & 0xffffffffull);
        uint32_t lt = less_bits[w], eq = eq_bits[w];
        uint32_t sel = lt;
        long long taken_eq = b_ex < need_eq ? b_ex : need_eq;
        long long cnt_eq = b_ex;
        while (eq) {
          int b = __ffs(eq) - 1;
          eq &= eq - 1;
          if (cnt_eq < need_eq) sel |= 1u << b;
          ++cnt_eq;
        }
        out_mask[w] = sel;
        long long pos = a_ex + taken_eq;
        uint32_t s = sel;
        while (s) {
          int b = __ffs(s) - 1;
          s &= s - 1;
          out_ids[pos++] = (int32_t)(w * 32 + b);
        }
      },
      [&](unsigned long long tot) {
        long long a = (long long)(tot >> 32), b = (long long)(tot & 0xffffffffull);
        out_counts[0] = a + (b < need_eq ? b : need_eq);
        out_counts[1] = (long long)st->support;
      });
}

// ---- cached CSR --------------------------------------------------------------
// count: per node, number of neighbours in the cache (one warp per row)
template <int BLOCK, int ITEMS>
__global__ void __launch_bounds__(BLOCK) ccsr_count_scan_kernel(ScanStatus ss, const int64_t* __restrict__ rowcnt,
                                                                int64_t n, int64_t* __restrict__ c_indptr,
                                                                int64_t* __restrict__ nnz_dev) {
  scan_tiles<BLOCK, ITEMS>(
      ss, n, [&](long long i) { return (unsigned long long)rowcnt[i]; },
      [&](long long i, unsigned long long ex, unsigned long long) { c_indptr[i] = (int64_t)ex; },
      [&](unsigned long long tot) {
        c_indptr[n] = (int64_t)tot;
        nnz_dev[0] = (int64_t)tot;
      });
}

__device__ __forceinline__ bool in_mask(const uint32_t* __restrict__ mask, int32_t v) {
  return (__ldg(mask + (v >> 5)) >> (v & 31)) & 1u;
}

// ---- cached CSR, flat (entry-parallel) passes ----------------------------------
// A per-row count (warp per row) spends a dependent chain (row bounds -> entries ->
// bitmap probe) per row, ~1.5 us for 29 entries on average: 19 ms per pass at
// papers100M (111M rows, 3.23B entries), 0.7 TB/s.  The flat passes stream
// the index array instead: a warp owns tiles of kCsrTile consecutive entries
// (coalesced loads, 8 in flight per lane) and writes one keep bit per entry
// plus the tile's count; the tile counts are scanned; c_indptr[r] = the
// tile offset of indptr[r] + the popcount of the keep bits before it; the
// fill compacts each tile's kept entries at its offset.
constexpr int kCsrTile = 1024;   // entries per warp tile = 32 keep words

__global__ void ccsr_mark_kernel(const int32_t* __restrict__ indices, int64_t E, const uint32_t* __restrict__ mask,
                                 uint32_t* __restrict__ keep, int64_t* __restrict__ tile_cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t tiles = (E + kCsrTile - 1) / kCsrTile;
  for (int64_t t = gw; t < tiles; t += nw) {
    const int64_t base = t * kCsrTile;
    uint32_t my = 0;
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 8) {
      int32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t p = base + 32 * (i0 + j) + lane;
        v[j] = p < E ? __ldg(indices + p) : -1;
      }
      uint32_t mw[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) mw[j] = v[j] >= 0 ? __ldg(mask + (v[j] >> 5)) : 0u;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const unsigned b = __ballot_sync(GNS_FULL, v[j] >= 0 && ((mw[j] >> (v[j] & 31)) & 1u));
        if (lane == i0 + j) my = b;
      }
    }
    keep[t * 32 + lane] = my;
    const int c = warp_sum((int)__popc(my));
    if (lane == 0) tile_cnt[t] = c;
  }
}

// c_indptr[r] for r in [0, n]: flat rank of the first entry of row r among
// the kept entries
__global__ void ccsr_indptr_kernel(const int64_t* __restrict__ indptr, int64_t n, const uint32_t* __restrict__ keep,
                                   const int64_t* __restrict__ tile_off, int64_t* __restrict__ c_indptr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = indptr[r];
    const int64_t t = p / kCsrTile;
    const int w = (int)((p % kCsrTile) >> 5), b = (int)(p & 31);
    const uint4* kw = reinterpret_cast<const uint4*>(keep + t * 32);
    int64_t c = tile_off[t];
    for (int q = 0; q < (w >> 2); ++q) {
      const uint4 x = kw[q];
      c += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
    const uint4 x = kw[w >> 2];
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
    for (int j = 0; j < (w & 3); ++j) c += __popc(xs[j]);
    c += __popc(xs[w & 3] & ((1u << b) - 1u));
    c_indptr[r] = c;
  }
}

__global__ void ccsr_fill_flat_kernel(const int32_t* __restrict__ indices, int64_t E, const uint32_t* __restrict__ keep,
                                      const int64_t* __restrict__ tile_off, int32_t* __restrict__ c_indices) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t tiles = (E + kCsrTile - 1) / kCsrTile;
  for (int64_t t = gw; t < tiles; t += nw) {
    const int64_t base = t * kCsrTile;
    const uint32_t my = keep[t * 32 + lane];
    if (!__any_sync(GNS_FULL, my != 0u)) continue;
    int64_t off = tile_off[t];
#pragma unroll
    for (int i0 = 0; i0 < 32; i0 += 8) {
      uint32_t wd[8];
      int32_t v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        wd[j] = __shfl_sync(GNS_FULL, my, i0 + j);
        const int64_t p = base + 32 * (i0 + j) + lane;
        v[j] = ((wd[j] >> lane) & 1u) ? __ldg(indices + p) : 0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if ((wd[j] >> lane) & 1u) c_indices[off + __popc(wd[j] & lt)] = v[j];
        off += __popc(wd[j]);
      }
    }
  }
}

__global__ void ccsr_fill_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                 int64_t n, const uint32_t* __restrict__ mask,
                                 const int64_t* __restrict__ c_indptr, int32_t* __restrict__ c_indices,
                                 int32_t* __restrict__ c_pos) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {
    int64_t b = indptr[r], e = indptr[r + 1];
    int64_t out = c_indptr[r];
    if (c_indptr[r + 1] == out) continue;
    for (int64_t base = b; base < e; base += 32) {
      int64_t p = base + lane;
      int32_t v = (p < e) ? __ldg(indices + p) : 0;
      bool keep = (p < e) && in_mask(mask, v);
      unsigned bal = __ballot_sync(GNS_FULL, keep);
      if (keep) {
        const int64_t o = out + __popc(bal & ((1u << lane) - 1));
        c_indices[o] = v;
        if (c_pos) c_pos[o] = (int32_t)(p - b);  // position in the full row (gns-exact lookups)
      }
      out += __popc(bal);
    }
  }
}

}  // namespace gns

using namespace gns;

static size_t cache_draw_ws(int64_t n, char* base, size_t cap, uint64_t** keys, uint32_t** lt,
                            uint32_t** eq, unsigned** hist, SelectState** st, void** scan,
                            long long* tiles) {
  Workspace w(base, cap);
  int64_t nw = (n + 31) / 32;
  *keys = w.take<uint64_t>(n > 0 ? n : 1);
  *lt = w.take<uint32_t>(nw + 1);
  *eq = w.take<uint32_t>(nw + 1);
  *hist = w.take<unsigned>(2048);
  *st = w.take<SelectState>(1);
  *tiles = (nw + 256 * 8 - 1) / (256 * 8) + 1;
  *scan = (void*)w.take<char>(scan_status_bytes(*tiles));
  return w.off;
}

extern "C" {

size_t gns_cache_draw_workspace_size(int64_t num_nodes) {
  uint64_t* k; uint32_t *a, *b; unsigned* h; SelectState* s; void* sc; long long t;
  return cache_draw_ws(num_nodes, nullptr, 0, &k, &a, &b, &h, &s, &sc, &t);
}

int gns_cache_draw(const double* probs, int64_t n, int64_t cache_size, uint32_t seed, uint32_t epoch, uint32_t tag,
                   int32_t* out_ids, uint32_t* out_mask_bits, int64_t* out_counts, void* ws,
                   size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (n <= 0) {
    set_error("cache_draw: empty graph");
    return GNS_EINVAL;
  }
  uint64_t* keys; uint32_t *lt, *eq; unsigned* hist; SelectState* st; void* scan; long long tiles;
  size_t need = cache_draw_ws(n, (char*)ws, ws_bytes, &keys, &lt, &eq, &hist, &st, &scan, &tiles);
  if (need > ws_bytes) {
    set_error("cache_draw: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  if (cache_size < 0) cache_size = 0;
  const int sms = num_sms();
  GNS_CUDA(cudaMemsetAsync(hist, 0, 2048 * sizeof(unsigned), stream));
  GNS_CUDA(cudaMemsetAsync(st, 0, sizeof(SelectState), stream));
  cache_keys_kernel<<<sms * 8, 256, 0, stream>>>(probs, n, seed, epoch, tag, keys, st);
  GNS_TRY(check_launch("cache_keys"));
  select_init_kernel<<<1, 1, 0, stream>>>(st, cache_size);
  for (int pass = 0; pass < 6; ++pass) {
    radix_hist_kernel<256><<<sms * 4, 256, 0, stream>>>(keys, n, st, kDigitShift[pass], kDigitBits[pass], hist);
    radix_pick_kernel<<<1, 1024, 0, stream>>>(st, kDigitShift[pass], kDigitBits[pass], hist);
  }
  GNS_TRY(check_launch("radix_select"));
  int64_t nw = (n + 31) / 32;
  classify_kernel<<<sms * 8, 256, 0, stream>>>(keys, n, st, lt, eq);
  ScanStatus ss = make_scan_status(scan, tiles);
  GNS_CUDA(cudaMemsetAsync(scan, 0, scan_status_bytes(tiles), stream));
  cache_compact_kernel<256, 8><<<(unsigned)tiles, 256, 0, stream>>>(ss, lt, eq, nw, st, out_ids, out_mask_bits,
                                                                    out_counts);
  return check_launch("cache_compact");
}

// workspace: the keep bits (one per CSR entry), tile counts, tile offsets and
// the scan status; the same workspace must reach gns_cached_csr_fill
struct CcsrWs {
  uint32_t* keep;
  int64_t* tile_cnt;
  int64_t* tile_off;
  void* scan;
  long long tiles, scan_tiles;
};

static size_t ccsr_ws(int64_t num_edges, void* base, size_t cap, CcsrWs* w) {
  Workspace ws(base, cap);
  w->tiles = (num_edges + kCsrTile - 1) / kCsrTile;
  w->keep = ws.take<uint32_t>((size_t)w->tiles * 32 + 4);
  w->tile_cnt = ws.take<int64_t>(w->tiles + 1);
  w->tile_off = ws.take<int64_t>(w->tiles + 2);
  w->scan_tiles = (w->tiles + 256 * 16 - 1) / (256 * 16) + 1;
  w->scan = (void*)ws.take<char>(scan_status_bytes(w->scan_tiles));
  return ws.off;
}

size_t gns_cached_csr_workspace_size(int64_t num_nodes, int64_t num_edges) {
  (void)num_nodes;
  CcsrWs w;
  return ccsr_ws(num_edges, nullptr, 0, &w);
}

int gns_cached_csr_count(const gns_graph_t* g, const uint32_t* mask_bits, int64_t* out_c_indptr,
                         int64_t* out_nnz_dev, void* ws, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t n = g->num_nodes, E = g->num_edges;
  CcsrWs w;
  size_t need = ccsr_ws(E, ws, ws_bytes, &w);
  if (ws_bytes < need) {
    set_error("cached_csr: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  const int sms = num_sms();
  // the tile at index `tiles` (one past the end) must read as zero bits for
  // the row r = n (indptr[n] = E at a tile boundary)
  GNS_CUDA(cudaMemsetAsync(w.keep + (size_t)w.tiles * 32, 0, 4 * sizeof(uint32_t), stream));
  ccsr_mark_kernel<<<sms * 8, 256, 0, stream>>>(g->indices, E, mask_bits, w.keep, w.tile_cnt);
  GNS_TRY(check_launch("ccsr_mark"));
  GNS_CUDA(cudaMemsetAsync(w.scan, 0, scan_status_bytes(w.scan_tiles), stream));
  ccsr_count_scan_kernel<256, 16><<<(unsigned)w.scan_tiles, 256, 0, stream>>>(
      make_scan_status(w.scan, w.scan_tiles), w.tile_cnt, w.tiles, w.tile_off, out_nnz_dev);
  GNS_TRY(check_launch("ccsr_tile_scan"));
  ccsr_indptr_kernel<<<sms * 8, 256, 0, stream>>>(g->indptr, n, w.keep, w.tile_off, out_c_indptr);
  return check_launch("ccsr_indptr");
}

int gns_cached_csr_fill(const gns_graph_t* g, const uint32_t* mask_bits, const int64_t* c_indptr,
                        int32_t* out_c_indices, int32_t* out_c_pos, void* ws, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  CcsrWs w;
  size_t need = ccsr_ws(g->num_edges, ws, ws_bytes, &w);
  if (ws_bytes < need) {
    set_error("cached_csr_fill: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  if (out_c_pos) {
    // positions within the full row (gns-exact lookups): the per-row kernel
    ccsr_fill_kernel<<<num_sms() * 8, 256, 0, stream>>>(g->indptr, g->indices, g->num_nodes, mask_bits, c_indptr,
                                                        out_c_indices, out_c_pos);
    return check_launch("ccsr_fill");
  }
  ccsr_fill_flat_kernel<<<num_sms() * 8, 256, 0, stream>>>(g->indices, g->num_edges, w.keep, w.tile_off,
                                                           out_c_indices);
  return check_launch("ccsr_fill_flat");
}

}  // extern "C"

// ---- random-walk cache distribution (cache.py:61-84) -----------
// p0 = 1/|train| on the train set; L times p <- d * (A p) + p with
// d_i = min(fanout_l, deg_i) / max(deg_i, 1); then p / sum(p).
// A p is summed sequentially per row in CSR (ascending neighbour) order with
// explicitly rounded adds, exactly like scipy's csr_matvec, so the iterate is
// bit-identical to the reference.  The normalising sum is a fixed-order
// strided reduction (restated in oracle/gns.py:random_walk_probs).
namespace gns {

__global__ void rw_init_kernel(double* __restrict__ p, int64_t n, const int32_t* __restrict__ train, int64_t nt,
                               double val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

__global__ void rw_set_kernel(double* __restrict__ p, const int32_t* __restrict__ train, int64_t nt, double val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x)
    p[train[i]] = val;
}

__global__ void rw_step_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices, int64_t n,
                               double fanout, const double* __restrict__ p, double* __restrict__ q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = indptr[i], e = indptr[i + 1];
    double s = 0.0;
    int64_t j = b;
    for (; j + 4 <= e; j += 4) {  // loads in flight, adds in order
      const double x0 = p[__ldg(indices + j)], x1 = p[__ldg(indices + j + 1)];
      const double x2 = p[__ldg(indices + j + 2)], x3 = p[__ldg(indices + j + 3)];
      s = DADD(DADD(DADD(DADD(s, x0), x1), x2), x3);
    }
    for (; j < e; ++j) s = DADD(s, p[__ldg(indices + j)]);
    const double deg = (double)(e - b);
    const double d = DDIV(fmin(fanout, deg), fmax(deg, 1.0));
    q[i] = DADD(DMUL(d, s), p[i]);
  }
}

// Neumaier-compensated running sum (exact op sequence restated in the oracle)
__device__ __forceinline__ void neumaier_add(double& s, double& c, double x) {
  const double t = DADD(s, x);
  if (fabs(s) >= fabs(x))
    c = DADD(c, DADD(DSUB(s, t), x));
  else
    c = DADD(c, DADD(DSUB(x, t), s));
  s = t;
}

// partial[t] = compensated sum of x[t], x[t+T], x[t+2T], ... (T = gridDim*blockDim)
__global__ void strided_sum_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ partial) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  double s = 0.0, c = 0.0;
  for (int64_t i = t; i < n; i += T) neumaier_add(s, c, x[i]);
  partial[t] = DADD(s, c);
}

__global__ void seq_sum_kernel(const double* __restrict__ partial, int64_t T, double* __restrict__ total) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double s = 0.0, c = 0.0;
    for (int64_t t = 0; t < T; ++t) neumaier_add(s, c, partial[t]);
    total[0] = DADD(s, c);
  }
}

__global__ void scale_kernel(double* __restrict__ p, int64_t n, const double* __restrict__ total) {
  const double s = total[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = DDIV(p[i], s);
}

static constexpr int kSumGrid = 148, kSumBlock = 256;  // fixed T: part of the reduction order

}  // namespace gns

extern "C" {

size_t gns_random_walk_workspace_size(int64_t num_nodes) {
  return ((size_t)num_nodes * 8 + 255) / 256 * 256 + (size_t)kSumGrid * kSumBlock * 8 + 512;
}

int gns_random_walk_probs(const gns_graph_t* g, const int32_t* train_ids, int64_t n_train,
                          const int32_t* fanouts_host, int32_t num_layers, double* out_probs, void* ws,
                          size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t n = g->num_nodes;
  if (num_layers < 1) {
    set_error("num_layers must be >= 1");
    return GNS_EINVAL;
  }
  if (n_train <= 0) {
    set_error("training set is empty");
    return GNS_EINVAL;
  }
  if (ws_bytes < gns_random_walk_workspace_size(n)) {
    set_error("random_walk_probs: workspace too small");
    return GNS_EINVAL;
  }
  double* tmp = (double*)ws;
  double* partial = (double*)((char*)ws + ((size_t)n * 8 + 255) / 256 * 256);
  double* total = partial + kSumGrid * kSumBlock;
  const int grid = num_sms() * 8;
  rw_init_kernel<<<grid, 256, 0, stream>>>(out_probs, n, train_ids, n_train, 0.0);
  rw_set_kernel<<<grid, 256, 0, stream>>>(out_probs, train_ids, n_train, 1.0 / (double)n_train);
  double* p = out_probs;
  double* q = tmp;
  for (int l = 0; l < num_layers; ++l) {
    rw_step_kernel<<<grid, 256, 0, stream>>>(g->indptr, g->indices, n, (double)fanouts_host[l], p, q);
    double* t = p;
    p = q;
    q = t;
  }
  strided_sum_kernel<<<kSumGrid, kSumBlock, 0, stream>>>(p, n, partial);
  seq_sum_kernel<<<1, 32, 0, stream>>>(partial, (int64_t)kSumGrid * kSumBlock, total);
  scale_kernel<<<grid, 256, 0, stream>>>(p, n, total);
  if (p != out_probs) GNS_CUDA(cudaMemcpyAsync(out_probs, p, (size_t)n * 8, cudaMemcpyDeviceToDevice, stream));
  return check_launch("random_walk_probs");
}

}  // extern "C"

// ---- gns-exact per-edge inclusion table (sampling.py:269-296, §8(f)3) ------------
namespace gns {

// q[e] += cached(e) ? min(k,nc)/nc : fill/rest  (one resampled cache; rows in
// CSR order, one warp per row; adds in resample order -> deterministic)
__global__ void edge_incl_accum_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                       int64_t n, const uint32_t* __restrict__ mask, int k, int cache_only,
                                       double* __restrict__ q) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int64_t b = indptr[r], e = indptr[r + 1];
    unsigned c = 0;
    for (int64_t p = b + lane; p < e; p += 32) c += in_mask(mask, __ldg(indices + p));
    c = warp_sum(c);
    const double nc = (double)c, deg = (double)(e - b);
    const double m = fmin((double)k, nc);
    const double rest = DSUB(deg, nc);
    const double pc = nc > 0.0 ? DDIV(m, nc) : 0.0;
    double pf = 0.0;
    if (!cache_only && rest > 0.0) pf = DDIV(fmin(DSUB((double)k, m), rest), rest);
    for (int64_t p = b + lane; p < e; p += 32) q[p] = DADD(q[p], in_mask(mask, __ldg(indices + p)) ? pc : pf);
  }
}

__global__ void div_kernel(double* __restrict__ q, int64_t n, double d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    q[i] = DDIV(q[i], d);
}

}  // namespace gns

extern "C" {

size_t gns_edge_inclusion_workspace_size(int64_t num_nodes, int64_t cache_size) {
  return gns_cache_draw_workspace_size(num_nodes) + (((size_t)(num_nodes + 31) / 32 * 4 + 255) & ~(size_t)255) +
         (((size_t)(cache_size > 0 ? cache_size : 1) * 4 + 255) & ~(size_t)255) + 512;
}

int gns_estimate_edge_inclusion(const gns_graph_t* g, const double* probs, int64_t cache_size, int32_t k,
                                int32_t cache_only, int32_t resamples, uint32_t seed, double* out_q, void* ws,
                                size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int64_t n = g->num_nodes;
  if (k < 1 || resamples < 1) {
    set_error("estimate_edge_inclusion: need k >= 1 and resamples >= 1");
    return GNS_EINVAL;
  }
  if (ws_bytes < gns_edge_inclusion_workspace_size(n, cache_size)) {
    set_error("estimate_edge_inclusion: workspace too small");
    return GNS_EINVAL;
  }
  char* base = (char*)ws;
  const size_t dws = gns_cache_draw_workspace_size(n);
  uint32_t* mask = (uint32_t*)(base + dws);
  int32_t* ids = (int32_t*)(base + dws + (((size_t)(n + 31) / 32 * 4 + 255) & ~(size_t)255));
  int64_t* counts = (int64_t*)(base + gns_edge_inclusion_workspace_size(n, cache_size) - 256);
  GNS_CUDA(cudaMemsetAsync(out_q, 0, (size_t)g->num_edges * 8, stream));
  for (int r = 0; r < resamples; ++r) {
    // resample r: its own Philox stream (tag 21 = sampling.py:29 _FILL_STREAM)
    GNS_TRY(gns_cache_draw(probs, n, cache_size, seed, (uint32_t)r, 21u, ids, mask, counts, base, dws, stream_));
    edge_incl_accum_kernel<<<num_sms() * 8, 256, 0, stream>>>(g->indptr, g->indices, n, mask, k, cache_only, out_q);
    GNS_TRY(check_launch("edge_incl_accum"));
  }
  div_kernel<<<num_sms() * 8, 256, 0, stream>>>(out_q, g->num_edges, (double)resamples);
  return check_launch("edge_incl_div");
}

}  // extern "C"
