// Model-side hot ops on B200: input-feature gather (model.py:146), the weighted
// mean aggregation + self concat (model.py:131-138,153-154) and its backward
// (model.py:223-225), softmax cross-entropy (model.py:189-200) and Adam
// (model.py:229-242).  All HBM-bound; no tensor cores (the GraphSAGE linear
// layers are cuBLAS GEMMs issued by the Python side).
#include <string.h>

#include <algorithm>

#include <cuda.h>   // CUtensorMap (encoded through the runtime's driver entry point; no -lcuda)

#include "gns_common.cuh"

namespace gns {

// ---- gather ------------------------------------------------------------------
__device__ __forceinline__ float4 ld_stream_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// out[i, :] = table[rows[i], :] with 16-byte vectors.  A warp owns G
// consecutive rows per iteration (the ids are sorted, so they are near each
// other in the table); one coalesced load fetches the G row ids, lane l
// moves 16-byte chunks l, l+32, ... of each row, and all G*C loads of the
// iteration are issued before any store.  C column blocks of 32 chunks cover
// rows up to C*512 bytes (wider rows loop over column blocks).  Measured on
// B200 (scripts/gather_probe2.cu, 285K random 512-B rows, L2 full of dirty
// lines): G=2 at 8 resident CTAs/SM = 55 us, a grid-strided flat chunk loop
// = 60-68 us, cudaMemcpy of the same bytes = 56 us.
// (register cap: 8 resident CTAs/SM = full occupancy for <= 2 loads in
// flight per lane; the wider variants trade occupancy for loads in flight)
template <int G, int C>
__global__ void __launch_bounds__(256, (G == 2 && C == 1) ? 8 : 4) gather_f32x4_kernel(const float* __restrict__ table, int64_t ld_in,
                                                           const int32_t* __restrict__ rows,
                                                           const int32_t* __restrict__ n_dev, int64_t n_host,
                                                           int dim4, float* __restrict__ out, int64_t ld_out) {
  const int64_t n = n_dev ? n_dev[0] : n_host;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  if (G == 2 && C == 1 && dim4 == 32) {
    // 512-byte rows (D = 128, the papers100M shape): one chunk per lane
    for (int64_t r0 = warp * G; r0 < n; r0 += nw * G) {
      const int32_t myrow = (lane < G && r0 + lane < n) ? __ldg(rows + r0 + lane) : 0;
      float4 v[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int32_t src = __shfl_sync(GNS_FULL, myrow, g);
        if (r0 + g < n) v[g] = ld_stream_f4(reinterpret_cast<const float4*>(table + (int64_t)src * ld_in) + lane);
      }
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (r0 + g < n) reinterpret_cast<float4*>(out + (r0 + g) * ld_out)[lane] = v[g];
    }
    return;
  }
  for (int64_t r0 = warp * G; r0 < n; r0 += nw * G) {
    const int32_t myrow = (lane < G && r0 + lane < n) ? __ldg(rows + r0 + lane) : 0;
    for (int c0 = 0; c0 < dim4; c0 += 32 * C) {
      float4 v[G][C];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int32_t src = __shfl_sync(GNS_FULL, myrow, g);
        const float4* rp = reinterpret_cast<const float4*>(table + (int64_t)src * ld_in);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int ch = c0 + c * 32 + lane;
          if (r0 + g < n && ch < dim4) v[g][c] = ld_stream_f4(rp + ch);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float4* op = reinterpret_cast<float4*>(out + (r0 + g) * ld_out);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int ch = c0 + c * 32 + lane;
          if (r0 + g < n && ch < dim4) op[ch] = v[g][c];
        }
      }
    }
  }
}

template <typename TI, typename TO>
__global__ void gather_scalar_kernel(const TI* __restrict__ table, int64_t ld_in, const int32_t* __restrict__ rows,
                                     const int32_t* __restrict__ n_dev, int64_t n_host, int dim,
                                     TO* __restrict__ out, int64_t ld_out) {
  const int64_t n = n_dev ? n_dev[0] : n_host;
  const int64_t total = n * dim;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / dim;
    int c = (int)(i - r * dim);
    out[r * ld_out + c] = (TO)table[(int64_t)rows[r] * ld_in + c];
  }
}

__global__ void gather_mixed_kernel(const float* __restrict__ host_table, const float* __restrict__ cache_table,
                                    const uint32_t* __restrict__ mask, const int32_t* __restrict__ wrank, int64_t ld,
                                    const int32_t* __restrict__ rows, const int32_t* __restrict__ n_dev, int dim4,
                                    float* __restrict__ out, int64_t ld_out) {
  const int64_t n = n_dev[0];
  const int64_t total = n * dim4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / dim4;
    int c = (int)(i - r * dim4);
    int32_t v = __ldg(rows + r);
    uint32_t w = __ldg(mask + (v >> 5));
    const float4* src;
    if ((w >> (v & 31)) & 1u) {
      int32_t slot = __ldg(wrank + (v >> 5)) + __popc(w & ((1u << (v & 31)) - 1u));
      src = reinterpret_cast<const float4*>(cache_table + (int64_t)slot * ld) + c;
    } else {
      src = reinterpret_cast<const float4*>(host_table + (int64_t)v * ld) + c;
    }
    reinterpret_cast<float4*>(out + r * ld_out)[c] = *src;
  }
}

__global__ void refresh_rows_kernel(const float* __restrict__ host_table, int64_t ld, const int32_t* __restrict__ ids,
                                    const int64_t* __restrict__ n_dev, int dim4, float* __restrict__ cache_table) {
  const int64_t n = n_dev[0];
  const int64_t total = n * dim4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / dim4;
    int c = (int)(i - r * dim4);
    reinterpret_cast<float4*>(cache_table + r * ld)[c] =
        reinterpret_cast<const float4*>(host_table + (int64_t)ids[r] * ld)[c];
  }
}

// ---- SpMM forward --------------------------------------------------------------
template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int W = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int W = 2; };

template <typename V, typename T> __device__ __forceinline__ void vzero(V& v);
__device__ __forceinline__ void vzero(float4& v) { v = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void vzero(double2& v) { v = make_double2(0.0, 0.0); }

template <bool EXACT>
__device__ __forceinline__ void vfma(float4& acc, float w, const float4& x) {
  acc.x = fmaf(w, x.x, acc.x); acc.y = fmaf(w, x.y, acc.y);
  acc.z = fmaf(w, x.z, acc.z); acc.w = fmaf(w, x.w, acc.w);
}
template <bool EXACT>
__device__ __forceinline__ void vfma(double2& acc, double w, const double2& x) {
  acc.x = DADD(acc.x, DMUL(w, x.x));
  acc.y = DADD(acc.y, DMUL(w, x.y));
}
__device__ __forceinline__ float4 vdiv(const float4& a, float d) {
  return make_float4(__fdiv_rn(a.x, d), __fdiv_rn(a.y, d), __fdiv_rn(a.z, d), __fdiv_rn(a.w, d));
}
__device__ __forceinline__ double2 vdiv(const double2& a, double d) { return make_double2(DDIV(a.x, d), DDIV(a.y, d)); }

// Row r of a float32 row-major table: one IMAD.WIDE.U32 (32 x 32 -> 64 with
// the 64-bit base as addend) instead of a 64 x 64-bit multiply (3 IMADs + 3
// address ops per row).  Row ids are non-negative node / row indices and the
// row pitch in bytes fits 32 bits (checked on the host: ld * 4 < 2^32).
__device__ __forceinline__ const float4* row4(const float* __restrict__ base, int32_t r, uint32_t pitch_bytes) {
  return reinterpret_cast<const float4*>(reinterpret_cast<const char*>(base) + (uint64_t)(uint32_t)r * pitch_bytes);
}

constexpr int kRowCap = 128;  // max edges per dst row (fanout <= 128)
constexpr int kSpmmBlock = 256;

struct BlockView {
  const uint64_t* row_scan;
  const int32_t* dst_degree;
  const int32_t* self_pos;
  const int32_t* edge_src;
  const int32_t* edge_dst;
  const double* edge_weight;
  const int32_t* counts;
};

__host__ static inline BlockView view_of(const gns_block_t* b) {
  return {b->row_scan, b->dst_degree, b->self_pos, b->edge_src, b->edge_dst, b->edge_weight, b->counts};
}

// one warp per dst row: sort the row's (<= k) edges by src index (the scipy
// CSR order, model.py:133-135), then cat[r] = [h[self], sum w*h[src] / norm]
__device__ __forceinline__ float4 vrelu(float4 v) {
  return make_float4(fmaxf(v.x, 0.f), fmaxf(v.y, 0.f), fmaxf(v.z, 0.f), fmaxf(v.w, 0.f));
}
__device__ __forceinline__ double2 vrelu(double2 v) { return make_double2(fmax(v.x, 0.0), fmax(v.y, 0.0)); }

template <typename V, bool RELU>
__device__ __forceinline__ V ldv(const V* p) {
  V v = *p;
  if constexpr (RELU) v = vrelu(v);
  return v;
}

// relu' bits of a float32 row as the forward reads it (MASK variants): word
// blk*4+q, bit l <-> element 4*(blk*32+l)+q, so lane l of a backward warp
// finds its chunk's four bits at the same bit position of four words.
// Four ballots, then one 16-byte store by lane 0 (words blk*4 .. blk*4+3;
// rows are (dv+31)/32*4 words, so the store is aligned); every lane must
// call it.  (A per-lane select of the ballot for lanes 0..3 compiled to a
// jump table: ~2x the instructions per row read.)
__device__ __forceinline__ void put_relu_bits(uint32_t* __restrict__ mrow, int blk, const float4& v, bool valid) {
  const unsigned b0 = __ballot_sync(GNS_FULL, valid && v.x > 0.f), b1 = __ballot_sync(GNS_FULL, valid && v.y > 0.f);
  const unsigned b2 = __ballot_sync(GNS_FULL, valid && v.z > 0.f), b3 = __ballot_sync(GNS_FULL, valid && v.w > 0.f);
  if ((threadIdx.x & 31) == 0) reinterpret_cast<uint4*>(mrow)[blk] = make_uint4(b0, b1, b2, b3);
}
__device__ __forceinline__ void put_relu_bits(uint32_t*, int, const double2&, bool) {}

// RELU: the input rows are the previous layer's pre-activations z and
// relu(z) (model.py:156) is applied on load instead of being materialised.
// Rows [n, pad_rows) of cat are zero-filled (static-capacity GEMMs).
//
// GATHER (the input layer, fused feature gather, model.py:146+153): h is the
// node feature table and rows are addressed by global node id — edge_node for
// the neighbours, dst_ids[r] for the self row — so features[input_nodes] is
// never materialised.  src_nodes is sorted, so ordering a row's edges by node
// id is the same as ordering them by edge_src: the sums are bit-identical.
//
// MASK (float32 with RELU): also writes the relu' bits of every h row it
// reads (put_relu_bits, (dv+31)/32*4 words per row) for the backward, which
// then reads 32 bytes per row instead of the whole pre-activation row.  Every
// src row of a block is a dst (self) row or an edge source, so every row the
// backward needs gets its bits.
// A row longer than spmm_fwd_kernel's shared stage (full-neighbourhood
// blocks of hub rows, not sampled ones): the same ascending-source FMA
// sequence, each next source found by a warp arg-min over the row
// (O(L^2 / 32)).  Its own kernel (spmm_fwd_long_kernel, launched after
// spmm_fwd_kernel, which skips such rows): inlined into spmm_fwd_kernel this
// path took it from 79 to 128 registers and the OAG input layer from 225 to
// 275 us; a non-inlined call still cost spills.
template <typename T, int CH, bool RELU, bool GATHER, bool MASK>
__device__ __forceinline__ void spmm_fwd_row_long(const T* __restrict__ h, int64_t ld_h, int dv, BlockView bv,
                                               T* __restrict__ cat, int64_t ld_cat, const int32_t* __restrict__ eidx,
                                               const int32_t* __restrict__ dst_ids, uint32_t* __restrict__ relu_bits,
                                               int64_t r, int64_t cb, int nc, int64_t fb, int L, int lane) {
  using V = typename Vec<T>::type;
  const T norm = (T)max(bv.dst_degree[r], 1);
  const V* hs = reinterpret_cast<const V*>(h + (int64_t)(GATHER ? dst_ids[r] : bv.self_pos[r]) * ld_h);
  V* crow = reinterpret_cast<V*>(cat + r * ld_cat);
  const int mw = ((dv + 31) >> 5) * 4;
  for (int c0 = 0; c0 < dv; c0 += 32) {
    const int c = c0 + lane;
    V v;
    vzero(v);
    if (c < dv) {
      v = ldv<V, RELU>(hs + c);
      crow[c] = v;
    }
    if constexpr (MASK) put_relu_bits(relu_bits + (int64_t)bv.self_pos[r] * mw, c0 >> 5, v, c < dv);
  }
  for (int c0 = 0; c0 < dv; c0 += 32 * CH) {
    V acc[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) vzero(acc[j]);
    int64_t last = -1;
    for (int t = 0; t < L; ++t) {
      int32_t best = INT32_MAX;
      T bw = 0;
      for (int i = lane; i < L; i += 32) {
        const int64_t e = i < nc ? cb + i : fb + (i - nc);
        const int32_t v = eidx[e];
        if ((int64_t)v > last && v < best) {
          best = v;
          bw = (T)bv.edge_weight[e];
        }
      }
      int32_t mn = best;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(GNS_FULL, mn, o));
      const int win = __ffs(__ballot_sync(GNS_FULL, best == mn)) - 1;
      const T w0 = __shfl_sync(GNS_FULL, bw, win);
      last = mn;
      const V* r0 = reinterpret_cast<const V*>(h + (int64_t)mn * ld_h);
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = c0 + lane + 32 * j;
        V x;
        vzero(x);
        if (c < dv) {
          x = ldv<V, RELU>(r0 + c);
          vfma<true>(acc[j], w0, x);
        }
        if constexpr (MASK) put_relu_bits(relu_bits + (int64_t)mn * mw, (c0 >> 5) + j, x, c < dv);
      }
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = c0 + lane + 32 * j;
      if (c < dv) crow[dv + c] = vdiv(acc[j], norm);
    }
  }
}

template <typename T, int CH, bool RELU, bool GATHER = false, bool MASK = false>
__global__ void __launch_bounds__(kSpmmBlock) spmm_fwd_kernel(const T* __restrict__ h, int64_t ld_h, int dim,
                                                              BlockView bv, T* __restrict__ cat, int64_t ld_cat,
                                                              int64_t pad_rows,
                                                              const int32_t* __restrict__ edge_node = nullptr,
                                                              const int32_t* __restrict__ dst_ids = nullptr,
                                                              uint32_t* __restrict__ relu_bits = nullptr,
                                                              int64_t pad_chunk = 0) {
  const int32_t* __restrict__ eidx = GATHER ? edge_node : bv.edge_src;
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  __shared__ int32_t s_idx[kSpmmBlock / 32][kRowCap];
  __shared__ T s_w[kSpmmBlock / 32][kRowCap];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t n = bv.counts[GNS_CNT_DST];
  const uint64_t tot = bv.row_scan[n];
  const int64_t tm = (int64_t)(tot >> 32);
  const int dv = dim / VW;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw) {
    const uint64_t s0 = bv.row_scan[r], s1 = bv.row_scan[r + 1];
    const int64_t cb = (int64_t)(s0 >> 32), ce = (int64_t)(s1 >> 32);
    const int64_t fb = tm + (int64_t)(s0 & 0xffffffffull), fe = tm + (int64_t)(s1 & 0xffffffffull);
    const int nc = (int)(ce - cb), L = nc + (int)(fe - fb);
    if (L > kRowCap) {   // longer than the shared stage: spmm_fwd_long_kernel
      __syncwarp();
      continue;
    }
    // load + rank-sort by src index (distinct within a row)
    int32_t my_idx[kRowCap / 32];
    T my_w[kRowCap / 32];
#pragma unroll
    for (int j = 0; j < kRowCap / 32; ++j) {
      int i = lane + 32 * j;
      my_idx[j] = INT32_MAX;
      my_w[j] = 0;
      if (i < L) {
        int64_t e = i < nc ? cb + i : fb + (i - nc);
        my_idx[j] = eidx[e];
        my_w[j] = (T)bv.edge_weight[e];
      }
    }
#pragma unroll
    for (int j = 0; j < kRowCap / 32; ++j) {
      if (32 * j < L) {
        if (lane + 32 * j < L) s_idx[wib][lane + 32 * j] = my_idx[j];
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kRowCap / 32; ++j) {
      int i = lane + 32 * j;
      if (i < L) {
        int rank = 0;
        for (int t = 0; t < L; ++t) rank += s_idx[wib][t] < my_idx[j];
        my_idx[j] = rank;  // reuse as rank
      }
    }
    __syncwarp();
#pragma unroll
    for (int j = 0; j < kRowCap / 32; ++j) {
      int i = lane + 32 * j;
      if (i < L) {
        int64_t e = i < nc ? cb + i : fb + (i - nc);
        s_idx[wib][my_idx[j]] = eidx[e];
        s_w[wib][my_idx[j]] = my_w[j];
      }
    }
    __syncwarp();
    const T norm = (T)max(bv.dst_degree[r], 1);
    const V* hs = reinterpret_cast<const V*>(h + (int64_t)(GATHER ? dst_ids[r] : bv.self_pos[r]) * ld_h);
    V* crow = reinterpret_cast<V*>(cat + r * ld_cat);
    const int mw = ((dv + 31) >> 5) * 4;
    if constexpr (MASK) {
      uint32_t* mrow = relu_bits + (int64_t)bv.self_pos[r] * mw;
      for (int c0 = 0; c0 < dv; c0 += 32) {
        const int c = c0 + lane;
        V v;
        vzero(v);
        if (c < dv) {
          v = ldv<V, RELU>(hs + c);
          crow[c] = v;
        }
        put_relu_bits(mrow, c0 >> 5, v, c < dv);
      }
    } else {
      for (int c = lane; c < dv; c += 32) crow[c] = ldv<V, RELU>(hs + c);
    }
    for (int c0 = 0; c0 < dv; c0 += 32 * CH) {
      V acc[CH];
#pragma unroll
      for (int j = 0; j < CH; ++j) vzero(acc[j]);
      int t = 0;
      for (; t + 2 <= L; t += 2) {
        const V* r0 = reinterpret_cast<const V*>(h + (int64_t)s_idx[wib][t] * ld_h);
        const V* r1 = reinterpret_cast<const V*>(h + (int64_t)s_idx[wib][t + 1] * ld_h);
        const T w0 = s_w[wib][t], w1 = s_w[wib][t + 1];
        V x0[CH], x1[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int c = c0 + lane + 32 * j;
          if (c < dv) { x0[j] = ldv<V, RELU>(r0 + c); x1[j] = ldv<V, RELU>(r1 + c); }
        }
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          vfma<true>(acc[j], w0, x0[j]);
          vfma<true>(acc[j], w1, x1[j]);
        }
        if constexpr (MASK) {
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int c = c0 + lane + 32 * j;
            put_relu_bits(relu_bits + (int64_t)s_idx[wib][t] * mw, (c0 >> 5) + j, x0[j], c < dv);
            put_relu_bits(relu_bits + (int64_t)s_idx[wib][t + 1] * mw, (c0 >> 5) + j, x1[j], c < dv);
          }
        }
      }
      if (t < L) {
        const V* r0 = reinterpret_cast<const V*>(h + (int64_t)s_idx[wib][t] * ld_h);
        const T w0 = s_w[wib][t];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int c = c0 + lane + 32 * j;
          V x;
          vzero(x);
          if (c < dv) {
            x = ldv<V, RELU>(r0 + c);
            vfma<true>(acc[j], w0, x);
          }
          if constexpr (MASK) put_relu_bits(relu_bits + (int64_t)s_idx[wib][t] * mw, (c0 >> 5) + j, x, c < dv);
        }
      }
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = c0 + lane + 32 * j;
        if (c < dv) crow[dv + c] = vdiv(acc[j], norm);
      }
    }
    __syncwarp();
  }
  const int64_t pad_end = pad_chunk > 0 ? min(pad_rows, (n + pad_chunk - 1) / pad_chunk * pad_chunk) : pad_rows;
  for (int64_t r = n + gw; r < pad_end; r += nw) {
    V* crow = reinterpret_cast<V*>(cat + r * ld_cat);
    V zero;
    vzero(zero);
    for (int c = lane; c < 2 * dv; c += 32) crow[c] = zero;
  }
}

// rows of more than kRowCap edges (full-neighbourhood blocks), warp per row;
// every other row was written by spmm_fwd_kernel
template <typename T, int CH, bool RELU, bool GATHER = false, bool MASK = false>
__global__ void __launch_bounds__(kSpmmBlock) spmm_fwd_long_kernel(const T* __restrict__ h, int64_t ld_h, int dim,
                                                                   BlockView bv, T* __restrict__ cat, int64_t ld_cat,
                                                                   const int32_t* __restrict__ edge_node = nullptr,
                                                                   const int32_t* __restrict__ dst_ids = nullptr,
                                                                   uint32_t* __restrict__ relu_bits = nullptr) {
  const int32_t* __restrict__ eidx = GATHER ? edge_node : bv.edge_src;
  const int lane = threadIdx.x & 31;
  const int64_t n = bv.counts[GNS_CNT_DST];
  const int64_t tm = (int64_t)(bv.row_scan[n] >> 32);
  const int dv = dim / Vec<T>::W;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // lane-parallel length test over 32 rows at a time
  for (int64_t r0 = gw * 32; r0 < n; r0 += nw * 32) {
    int L = 0;
    if (r0 + lane < n) {
      const uint64_t s0 = bv.row_scan[r0 + lane], s1 = bv.row_scan[r0 + lane + 1];
      L = (int)((s1 >> 32) - (s0 >> 32)) + (int)((s1 & 0xffffffffull) - (s0 & 0xffffffffull));
    }
    for (unsigned m = __ballot_sync(GNS_FULL, L > kRowCap); m; m &= m - 1) {
      const int64_t r = r0 + __ffs(m) - 1;
      const uint64_t s0 = bv.row_scan[r], s1 = bv.row_scan[r + 1];
      const int64_t cb = (int64_t)(s0 >> 32), fb = tm + (int64_t)(s0 & 0xffffffffull);
      const int nc = (int)((s1 >> 32) - (s0 >> 32));
      const int Lr = nc + (int)((s1 & 0xffffffffull) - (s0 & 0xffffffffull));
      spmm_fwd_row_long<T, CH, RELU, GATHER, MASK>(h, ld_h, dv, bv, cat, ld_cat, eidx, dst_ids, relu_bits, r, cb, nc,
                                                   fb, Lr, lane);
    }
  }
}

// The next source index after `last` in a row (the row's edges in cached
// then fill segments; indices distinct within a row) and its weight: a warp
// arg-min over the row, O(L / 32) per lane — rows longer than the fast
// paths' 32-edge windows are walked in ascending-source order in O(L^2 / 32)
// (the rank-by-count loops these replace were O(L^3 / 32)).  Every lane calls
// it; all lanes get the result (INT32_MAX past the end).
__device__ __forceinline__ void next_src(const int32_t* __restrict__ eidx, const double* __restrict__ ew, int64_t cb,
                                         int nc, int64_t fb, int L, int lane, int64_t last, int32_t& v_out,
                                         float& w_out) {
  int32_t best = INT32_MAX;
  float bw = 0.f;
  for (int i = lane; i < L; i += 32) {
    const int64_t e = i < nc ? cb + i : fb + (i - nc);
    const int32_t v = eidx[e];
    if ((int64_t)v > last && v < best) {
      best = v;
      bw = (float)ew[e];
    }
  }
  int32_t mn = best;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(GNS_FULL, mn, o));
  const int win = __ffs(__ballot_sync(GNS_FULL, best == mn)) - 1;
  v_out = mn;
  w_out = __shfl_sync(GNS_FULL, bw, win);
}

// Narrow rows (float32, D <= 128: one 16-byte chunk per lane) with <= 32
// edges per dst row — the input layer.  Per warp and dst row: lane i loads
// edge i, the ranks by source index come from a shuffle count (no shared
// memory), the self row and up to kNarrowGroup neighbour rows are all in
// flight at once, then the weighted sum runs in ascending source order (the
// scipy CSR order, same FMA sequence as spmm_fwd_kernel: bit-identical).
// Rows with more than 32 edges take the generic per-row path.
template <bool RELU, bool GATHER, int kNarrowGroup = 3, int kMinBlocks = 4>
__global__ void __launch_bounds__(kSpmmBlock, kMinBlocks) spmm_fwd_narrow_kernel(const float* __restrict__ h, int64_t ld_h,
                                                                         int dim, BlockView bv,
                                                                         float* __restrict__ cat, int64_t ld_cat,
                                                                         int64_t pad_rows,
                                                                         const int32_t* __restrict__ edge_node,
                                                                         const int32_t* __restrict__ dst_ids,
                                                                         int64_t pad_chunk = 0) {
  const int32_t* __restrict__ eidx = GATHER ? edge_node : bv.edge_src;
  const int lane = threadIdx.x & 31;
  const int64_t n = bv.counts[GNS_CNT_DST];
  const int64_t tm = (int64_t)(bv.row_scan[n] >> 32);
  const int dv = dim >> 2;
  const bool on = lane < dv;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // the next row's scan bounds are requested while the current row's feature
  // rows are in flight, so its edge loads issue at once (one round trip less
  // per row; the self id and degree load alongside them)
  uint64_t n_s0 = 0, n_s1 = 0;
  if (gw < n) {
    n_s0 = bv.row_scan[gw];
    n_s1 = bv.row_scan[gw + 1];
  }
  for (int64_t r = gw; r < n; r += nw) {
    const uint64_t s0 = n_s0, s1 = n_s1;
    const int64_t self = GATHER ? (int64_t)dst_ids[r] : (int64_t)bv.self_pos[r];
    const float norm = (float)max(bv.dst_degree[r], 1);
    if (r + nw < n) {
      n_s0 = bv.row_scan[r + nw];
      n_s1 = bv.row_scan[r + nw + 1];
    }
    const int64_t cb = (int64_t)(s0 >> 32), ce = (int64_t)(s1 >> 32);
    const int64_t fb = tm + (int64_t)(s0 & 0xffffffffull), fe = tm + (int64_t)(s1 & 0xffffffffull);
    const int nc = (int)(ce - cb), L = nc + (int)(fe - fb);
    float4 xs = make_float4(0.f, 0.f, 0.f, 0.f);
    if (on) xs = ldv<float4, RELU>(reinterpret_cast<const float4*>(h + self * ld_h) + lane);
    float4* crow = reinterpret_cast<float4*>(cat + r * ld_cat);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (L <= 32) {
      int32_t idx = INT32_MAX;
      float w = 0.f;
      if (lane < L) {
        const int64_t e = lane < nc ? cb + lane : fb + (lane - nc);
        idx = eidx[e];
        w = (float)bv.edge_weight[e];
      }
      // rank among the row's edges by source index (distinct within a row)
      int rank = 0;
      for (int j = 0; j < L; ++j) rank += __shfl_sync(GNS_FULL, idx, j) < idx;
      // lane u fetches the edge of rank u
      int src = 0;
      for (int u = 0; u < L; ++u) {
        const unsigned m = __ballot_sync(GNS_FULL, lane < L && rank == u);
        if (lane == u) src = __ffs(m) - 1;
      }
      const int32_t sidx = __shfl_sync(GNS_FULL, idx, src);
      const float sw = __shfl_sync(GNS_FULL, w, src);
      for (int t = 0; t < L; t += kNarrowGroup) {
        float4 x[kNarrowGroup];
#pragma unroll
        for (int u = 0; u < kNarrowGroup; ++u) {
          const int32_t iu = __shfl_sync(GNS_FULL, sidx, (t + u) & 31);
          if (on && t + u < L) x[u] = ldv<float4, RELU>(reinterpret_cast<const float4*>(h + (int64_t)iu * ld_h) + lane);
        }
#pragma unroll
        for (int u = 0; u < kNarrowGroup; ++u) {
          const float wu = __shfl_sync(GNS_FULL, sw, (t + u) & 31);
          if (on && t + u < L) vfma<true>(acc, wu, x[u]);
        }
      }
    } else {
      // > 32 edges (full-neighbourhood hub rows): the ascending walk
      int64_t last = -1;
      for (int t = 0; t < L; ++t) {
        int32_t iu;
        float wu;
        next_src(eidx, bv.edge_weight, cb, nc, fb, L, lane, last, iu, wu);
        last = iu;
        if (on) vfma<true>(acc, wu, ldv<float4, RELU>(reinterpret_cast<const float4*>(h + (int64_t)iu * ld_h) + lane));
      }
    }
    if (on) {
      crow[lane] = xs;
      crow[dv + lane] = vdiv(acc, norm);
    }
  }
  // zero padding up to pad_rows, or (pad_chunk > 0) only up to the next
  // multiple of pad_chunk: the rows a size-switched GEMM body reads
  const int64_t pad_end = pad_chunk > 0 ? min(pad_rows, (n + pad_chunk - 1) / pad_chunk * pad_chunk) : pad_rows;
  for (int64_t r = n + gw; r < pad_end; r += nw) {
    float4* crow = reinterpret_cast<float4*>(cat + r * ld_cat);
    for (int c = lane; c < 2 * dv; c += 32) crow[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Narrow rows (float32, D <= 128), rows staged 32 at a time (the input
// layer: fused feature gather + mean aggregation).  A warp owns a chunk of 32
// consecutive dst rows; their metadata (row scan, self id, degree) and all of
// their edges (contiguous in the block's cached and fill regions) are read
// with coalesced loads into shared memory, each lane sorts ITS row's <= MAXL
// edges by source index in registers (a sorting network), and the warp then
// walks the rows with nothing but feature-row loads on the critical path:
// ROWS rows' self + neighbour rows are all issued before the first FMA.
// Sum order = ascending source index, the same FMA sequence as
// spmm_fwd_kernel / spmm_fwd_narrow_kernel: bit-identical.  Rows with more
// than MAXL edges (and chunks whose edges overflow the staging buffer) take
// the per-row path of spmm_fwd_narrow_kernel.
constexpr int kChunkRows = 32;

// x / d correctly rounded (== __fdiv_rn(x, d)) for an integer 1 <= d < 2^26,
// without the division subroutine: rd = RN64(1/d), RN32(RN64(x * rd)).  The
// exact quotient x/d is never a float rounding midpoint (a 25-bit odd
// significand cannot divide a 24-bit one) and stays >= 2^-25 / d relative
// away from one, while the two fp64 roundings add < 2^-51: the float
// rounding is the same as for the exact quotient.
__device__ __forceinline__ float div_by_count(float x, double rd) {
  return __double2float_rn(__dmul_rn((double)x, rd));
}
__device__ __forceinline__ float4 vdiv_count(const float4& a, double rd) {
  return make_float4(div_by_count(a.x, rd), div_by_count(a.y, rd), div_by_count(a.z, rd), div_by_count(a.w, rd));
}

template <int MAXL>
__device__ __forceinline__ void sort_pairs(int32_t (&k)[MAXL], float (&v)[MAXL]) {
  // odd-even transposition network: MAXL rounds, registers only
#pragma unroll
  for (int rnd = 0; rnd < MAXL; ++rnd) {
#pragma unroll
    for (int i = rnd & 1; i + 1 < MAXL; i += 2) {
      const bool sw = k[i + 1] < k[i];
      const int32_t a = sw ? k[i + 1] : k[i], b = sw ? k[i] : k[i + 1];
      const float x = sw ? v[i + 1] : v[i], y = sw ? v[i] : v[i + 1];
      k[i] = a; k[i + 1] = b; v[i] = x; v[i + 1] = y;
    }
  }
}

// one dst row through the per-row (ascending walk) path; every lane calls it
template <bool RELU>
__device__ __noinline__ void narrow_row_slow(const float* __restrict__ h, int64_t ld_h, const int32_t* __restrict__ eidx,
                                                const double* __restrict__ ew, int64_t cb, int nc, int64_t fb, int L,
                                                int lane, bool on, float4& acc) {
  int64_t last = -1;
  for (int t = 0; t < L; ++t) {
    int32_t iu;
    float wu;
    next_src(eidx, ew, cb, nc, fb, L, lane, last, iu, wu);
    last = iu;
    if (on) vfma<true>(acc, wu, ldv<float4, RELU>(reinterpret_cast<const float4*>(h + (int64_t)iu * ld_h) + lane));
  }
}

template <bool RELU, bool GATHER, int MAXL, int ROWS, int kMinBlocks>
__global__ void __launch_bounds__(kSpmmBlock, kMinBlocks) spmm_fwd_chunk_kernel(const float* __restrict__ h, int64_t ld_h,
                                                                        int dim, BlockView bv,
                                                                        float* __restrict__ cat, int64_t ld_cat,
                                                                        int64_t pad_rows,
                                                                        const int32_t* __restrict__ edge_node,
                                                                        const int32_t* __restrict__ dst_ids,
                                                                        int64_t pad_chunk = 0) {
  constexpr int CAP = kChunkRows * MAXL;  // staged edges per warp
  constexpr int W = kSpmmBlock / 32;
  __shared__ int32_t s_raw[W][CAP];       // chunk edges in position order (cached, then fill)
  __shared__ float s_rw[W][CAP];
  __shared__ int32_t s_idx[W][CAP];       // per row, sorted by source index
  __shared__ float s_w[W][CAP];
  __shared__ int32_t s_self[W][kChunkRows], s_base[W][kChunkRows], s_len[W][kChunkRows];
  __shared__ double s_rnorm[W][kChunkRows];   // 1 / max(deg, 1), fp64
  const int32_t* __restrict__ eidx = GATHER ? edge_node : bv.edge_src;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t n = bv.counts[GNS_CNT_DST];
  const int64_t tm = (int64_t)(bv.row_scan[n] >> 32);
  const int dv = dim >> 2;
  const bool on = lane < dv;
  const uint32_t pitch = (uint32_t)ld_h * 4u;   // row pitch in bytes (ld_h < 2^30: host check)
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  for (int64_t ch = gw; ch < nchunks; ch += nw) {
    const int64_t r0 = ch * kChunkRows;
    const int rows = (int)min((int64_t)kChunkRows, n - r0);
    unsigned fast;
    {
      // ---- stage the chunk: per-lane row metadata, then its edges
      uint64_t s0 = 0, s1 = 0;
      int32_t self = 0;
      int deg = 1;
      if (lane < rows) {
        s0 = bv.row_scan[r0 + lane];
        s1 = bv.row_scan[r0 + lane + 1];
        self = GATHER ? dst_ids[r0 + lane] : bv.self_pos[r0 + lane];
        deg = max(bv.dst_degree[r0 + lane], 1);
      }
      const uint64_t last0 = __shfl_sync(GNS_FULL, s0, 0), last1 = __shfl_sync(GNS_FULL, s1, rows - 1);
      const int64_t c_begin = (int64_t)(last0 >> 32), f_begin = tm + (int64_t)(last0 & 0xffffffffull);
      const int nC = (int)((int64_t)(last1 >> 32) - c_begin);
      const int nF = (int)(tm + (int64_t)(last1 & 0xffffffffull) - f_begin);
      // chunk-relative positions of my row's cached / fill edges
      const int cpos = (int)((int64_t)(s0 >> 32) - c_begin);
      const int fpos = nC + (int)(tm + (int64_t)(s0 & 0xffffffffull) - f_begin);
      const int nc = lane < rows ? (int)((s1 >> 32) - (s0 >> 32)) : 0;
      const int L = lane < rows ? nc + (int)((s1 & 0xffffffffull) - (s0 & 0xffffffffull)) : 0;
      const bool staged = nC + nF <= CAP;
      // exclusive prefix of the rows' edge counts = each row's slot base
      int base = L;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(GNS_FULL, base, o);
        if (lane >= o) base += y;
      }
      base -= L;
      s_self[wib][lane] = self;
      s_rnorm[wib][lane] = __drcp_rn((double)deg);
      s_base[wib][lane] = base;
      s_len[wib][lane] = L;
      if (staged) {
        for (int i = lane; i < nC; i += 32) {
          s_raw[wib][i] = eidx[c_begin + i];
          s_rw[wib][i] = (float)bv.edge_weight[c_begin + i];
        }
        for (int i = lane; i < nF; i += 32) {
          s_raw[wib][nC + i] = eidx[f_begin + i];
          s_rw[wib][nC + i] = (float)bv.edge_weight[f_begin + i];
        }
        __syncwarp();
        if (L <= MAXL) {
          int32_t k[MAXL];
          float v[MAXL];
#pragma unroll
          for (int t = 0; t < MAXL; ++t) {
            k[t] = INT32_MAX;
            v[t] = 0.f;
            if (t < L) {
              const int p = t < nc ? cpos + t : fpos + (t - nc);
              k[t] = s_raw[wib][p];
              v[t] = s_rw[wib][p];
            }
          }
          sort_pairs<MAXL>(k, v);
#pragma unroll
          for (int t = 0; t < MAXL; ++t)
            if (t < L) {
              s_idx[wib][base + t] = k[t];
              s_w[wib][base + t] = v[t];
            }
        }
      }
      fast = __ballot_sync(GNS_FULL, staged && lane < rows && L <= MAXL);
      __syncwarp();
    }
    // ---- the rows: ROWS at a time, every feature row in flight before any FMA
    for (int j0 = 0; j0 < rows; j0 += ROWS) {
      float4 xs[ROWS], x[ROWS][MAXL];
#pragma unroll
      for (int q = 0; q < ROWS; ++q) {
        const int j = j0 + q;
        const int Lj = (j < rows && ((fast >> j) & 1)) ? s_len[wib][j] : 0;
        const int bj = s_base[wib][j & 31];
        xs[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (on && j < rows && ((fast >> j) & 1))
          xs[q] = ldv<float4, RELU>(row4(h, s_self[wib][j], pitch) + lane);
#pragma unroll
        for (int t = 0; t < MAXL; ++t) {
          // defined on every path: a conditionally kept old value would pin
          // the array in local memory across iterations
          x[q][t] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (on && t < Lj)
            x[q][t] = ldv<float4, RELU>(row4(h, s_idx[wib][bj + t], pitch) + lane);
        }
      }
#pragma unroll
      for (int q = 0; q < ROWS; ++q) {
        const int j = j0 + q;
        if (j >= rows || !((fast >> j) & 1)) continue;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        const int Lj = s_len[wib][j], bj = s_base[wib][j];
#pragma unroll
        for (int t = 0; t < MAXL; ++t)
          if (on && t < Lj) vfma<true>(acc, s_w[wib][bj + t], x[q][t]);
        float4* crow = reinterpret_cast<float4*>(cat + (r0 + j) * ld_cat);
        if (on) {
          crow[lane] = xs[q];
          crow[dv + lane] = vdiv_count(acc, s_rnorm[wib][j]);
        }
      }
    }
    // wide rows / an overflowing chunk: the per-row path (rare; kept out of
    // the loop above so no feature registers are live across it)
    const unsigned slow = ~fast & (rows == 32 ? GNS_FULL : ((1u << rows) - 1u));
    for (unsigned m = slow; m; m &= m - 1) {
      const int j = __ffs(m) - 1;
      const uint64_t a0 = bv.row_scan[r0 + j], a1 = bv.row_scan[r0 + j + 1];
      const int64_t cbs = (int64_t)(a0 >> 32), fbs = tm + (int64_t)(a0 & 0xffffffffull);
      const int ncs = (int)((a1 >> 32) - (a0 >> 32));
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      narrow_row_slow<RELU>(h, ld_h, eidx, bv.edge_weight, cbs, ncs, fbs, s_len[wib][j], lane, on, acc);
      float4* crow = reinterpret_cast<float4*>(cat + (r0 + j) * ld_cat);
      if (on) {
        crow[lane] = ldv<float4, RELU>(row4(h, s_self[wib][j], pitch) + lane);
        crow[dv + lane] = vdiv_count(acc, s_rnorm[wib][j]);
      }
    }
    __syncwarp();
  }
  const int64_t pad_end = pad_chunk > 0 ? min(pad_rows, (n + pad_chunk - 1) / pad_chunk * pad_chunk) : pad_rows;
  for (int64_t r = n + gw; r < pad_end; r += nw) {
    float4* crow = reinterpret_cast<float4*>(cat + r * ld_cat);
    for (int c = lane; c < 2 * dv; c += 32) crow[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Rows of 32 < dim/4 <= 32*CH float4 chunks (the hidden layers, D = 256:
// CH = 2), float32, RELU on load: the narrow kernel's structure — lane-held
// edges, shuffle ranks, G neighbour rows in flight — with CH chunks per lane,
// and (MASK) the relu' bits of every row read (put_relu_bits) for the
// backward.  Same ascending-source FMA order as spmm_fwd_kernel.
template <int CH, int G, bool MASK>
__global__ void __launch_bounds__(kSpmmBlock, 3) spmm_fwd_wide_kernel(const float* __restrict__ h, int64_t ld_h,
                                                                       int dim, BlockView bv,
                                                                       float* __restrict__ cat, int64_t ld_cat,
                                                                       int64_t pad_rows,
                                                                       uint32_t* __restrict__ relu_bits) {
  const int lane = threadIdx.x & 31;
  const int64_t n = bv.counts[GNS_CNT_DST];
  const int64_t tm = (int64_t)(bv.row_scan[n] >> 32);
  const int dv = dim >> 2;
  const int mw = ((dv + 31) >> 5) * 4;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw) {
    const uint64_t s0 = bv.row_scan[r], s1 = bv.row_scan[r + 1];
    const int64_t self = (int64_t)bv.self_pos[r];
    const float norm = (float)max(bv.dst_degree[r], 1);
    const int64_t cb = (int64_t)(s0 >> 32), ce = (int64_t)(s1 >> 32);
    const int64_t fb = tm + (int64_t)(s0 & 0xffffffffull), fe = tm + (int64_t)(s1 & 0xffffffffull);
    const int nc = (int)(ce - cb), L = nc + (int)(fe - fb);
    float4 xs[CH], acc[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = lane + 32 * j;
      xs[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      acc[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (c < dv) xs[j] = vrelu(reinterpret_cast<const float4*>(h + self * ld_h)[c]);
    }
    if constexpr (MASK) {
#pragma unroll
      for (int j = 0; j < CH; ++j) put_relu_bits(relu_bits + self * mw, j, xs[j], lane + 32 * j < dv);
    }
    float4* crow = reinterpret_cast<float4*>(cat + r * ld_cat);
    int64_t last = -1;   // long rows: the walk's position
    for (int t0 = 0; t0 < L; t0 += 32) {
      // edges t0..t0+31 of the row in ascending source order: with L <= 32
      // one round; longer rows take each 32-edge window from the ascending walk
      const int m = min(32, L - t0);
      int32_t idx = INT32_MAX;
      float w = 0.f;
      if (L <= 32) {
        if (lane < L) {
          const int64_t e = lane < nc ? cb + lane : fb + (lane - nc);
          idx = bv.edge_src[e];
          w = (float)bv.edge_weight[e];
        }
        int rank = 0;
        for (int j = 0; j < L; ++j) rank += __shfl_sync(GNS_FULL, idx, j) < idx;
        int src = 0;
        for (int u = 0; u < L; ++u) {
          const unsigned mm = __ballot_sync(GNS_FULL, lane < L && rank == u);
          if (lane == u) src = __ffs(mm) - 1;
        }
        idx = __shfl_sync(GNS_FULL, idx, src);
        w = __shfl_sync(GNS_FULL, w, src);
      } else {
        // lane u < m takes the (t0 + u)-th source of the ascending walk
        for (int u = 0; u < m; ++u) {
          int32_t v;
          float wv;
          next_src(bv.edge_src, bv.edge_weight, cb, nc, fb, L, lane, last, v, wv);
          last = v;
          if (lane == u) {
            idx = v;
            w = wv;
          }
        }
      }
      for (int t = 0; t < m; t += G) {
        float4 x[G][CH];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const int32_t iu = __shfl_sync(GNS_FULL, idx, (t + u) & 31);
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const int c = lane + 32 * j;
            x[u][j] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t + u < m && c < dv) x[u][j] = vrelu(reinterpret_cast<const float4*>(h + (int64_t)iu * ld_h)[c]);
          }
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const float wu = __shfl_sync(GNS_FULL, w, (t + u) & 31);
          const int32_t iu = __shfl_sync(GNS_FULL, idx, (t + u) & 31);
          if (t + u < m) {
#pragma unroll
            for (int j = 0; j < CH; ++j) {
              if (lane + 32 * j < dv) vfma<true>(acc[j], wu, x[u][j]);
              if constexpr (MASK) put_relu_bits(relu_bits + (int64_t)iu * mw, j, x[u][j], lane + 32 * j < dv);
            }
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const int c = lane + 32 * j;
      if (c < dv) {
        crow[c] = xs[j];
        crow[dv + c] = vdiv(acc[j], norm);
      }
    }
  }
  for (int64_t r = n + gw; r < pad_rows; r += nw) {
    float4* crow = reinterpret_cast<float4*>(cat + r * ld_cat);
    for (int c = lane; c < 2 * dv; c += 32) crow[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// Column-split hidden-layer forward: warp task = (row, 128-float column
// chunk), so a row's chunks run on different warps (twice the independent
// chains of spmm_fwd_wide_kernel at D = 256, one float4 per lane per
// neighbour row, G rows in flight).  Each warp ranks the row's edges itself;
// per-element FMA order is unchanged (bit-identical).
template <int G, bool MASK, int MINB = 4>
__global__ void __launch_bounds__(kSpmmBlock, MINB) spmm_fwd_wide_split_kernel(const float* __restrict__ h,
                                                                             int64_t ld_h, int dim, BlockView bv,
                                                                             float* __restrict__ cat, int64_t ld_cat,
                                                                             int64_t pad_rows,
                                                                             uint32_t* __restrict__ relu_bits) {
  const int lane = threadIdx.x & 31;
  const int64_t n = bv.counts[GNS_CNT_DST];
  const int64_t tm = (int64_t)(bv.row_scan[n] >> 32);
  const int dv = dim >> 2;
  const uint32_t pitch = (uint32_t)ld_h * 4u;   // row pitch in bytes (ld_h < 2^30: host check)
  const int nch = (dv + 31) >> 5;
  const int mw = nch * 4;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t task = gw; task < n * nch; task += nw) {
    const int64_t r = task / nch;
    const int j = (int)(task - r * nch);
    const int c = lane + 32 * j;
    const bool on = c < dv;
    const uint64_t s0 = bv.row_scan[r], s1 = bv.row_scan[r + 1];
    const int64_t self = (int64_t)bv.self_pos[r];
    const float norm = (float)max(bv.dst_degree[r], 1);
    const int64_t cb = (int64_t)(s0 >> 32), ce = (int64_t)(s1 >> 32);
    const int64_t fb = tm + (int64_t)(s0 & 0xffffffffull), fe = tm + (int64_t)(s1 & 0xffffffffull);
    const int nc = (int)(ce - cb), L = nc + (int)(fe - fb);
    float4 xs = make_float4(0.f, 0.f, 0.f, 0.f), acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (on) xs = vrelu(reinterpret_cast<const float4*>(h + self * ld_h)[c]);
    if constexpr (MASK) put_relu_bits(relu_bits + self * mw, j, xs, on);
    int64_t last = -1;   // long rows: the walk's position
    for (int t0 = 0; t0 < L; t0 += 32) {
      const int m = min(32, L - t0);
      int32_t idx = INT32_MAX;
      float w = 0.f;
      if (L <= 32) {
        if (lane < L) {
          const int64_t e = lane < nc ? cb + lane : fb + (lane - nc);
          idx = bv.edge_src[e];
          w = (float)bv.edge_weight[e];
        }
        int rank = 0;
        for (int q = 0; q < L; ++q) rank += __shfl_sync(GNS_FULL, idx, q) < idx;
        int src = 0;
        for (int u = 0; u < L; ++u) {
          const unsigned mm = __ballot_sync(GNS_FULL, lane < L && rank == u);
          if (lane == u) src = __ffs(mm) - 1;
        }
        idx = __shfl_sync(GNS_FULL, idx, src);
        w = __shfl_sync(GNS_FULL, w, src);
      } else {
        // lane u < m takes the (t0 + u)-th source of the ascending walk
        for (int u = 0; u < m; ++u) {
          int32_t v;
          float wv;
          next_src(bv.edge_src, bv.edge_weight, cb, nc, fb, L, lane, last, v, wv);
          last = v;
          if (lane == u) {
            idx = v;
            w = wv;
          }
        }
      }
      for (int t = 0; t < m; t += G) {
        float4 x[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const int32_t iu = __shfl_sync(GNS_FULL, idx, (t + u) & 31);
          x[u] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (t + u < m && on) x[u] = vrelu(row4(h, iu, pitch)[c]);
        }
#pragma unroll
        for (int u = 0; u < G; ++u) {
          const float wu = __shfl_sync(GNS_FULL, w, (t + u) & 31);
          const int32_t iu = __shfl_sync(GNS_FULL, idx, (t + u) & 31);
          if (t + u < m) {
            if (on) vfma<true>(acc, wu, x[u]);
            if constexpr (MASK)
              put_relu_bits(reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(relu_bits) +
                                                        (uint64_t)(uint32_t)iu * (uint32_t)(mw * 4)),
                            j, x[u], on);
          }
        }
      }
    }
    if (on) {
      float4* crow = reinterpret_cast<float4*>(cat + r * ld_cat);
      crow[c] = xs;
      crow[dv + c] = vdiv(acc, norm);
    }
  }
  for (int64_t r = n + gw; r < pad_rows; r += nw) {
    float4* crow = reinterpret_cast<float4*>(cat + r * ld_cat);
    for (int cc = lane; cc < 2 * dv; cc += 32) crow[cc] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// experiment knobs (gns_tune)
static int g_tune_narrow = 2;  // narrow-row forward SpMM: 0 generic, 1 per-row narrow, 2+ chunk-staged
static int g_tune_wide = 2;    // hidden-layer forward: 2 = column-split, 1 = spmm_fwd_wide_kernel, 0 = generic
static int g_split_g = 4;      // column-split forward: neighbour rows in flight (2, 4, 8, 12, 16; 5 = 4 at 5 CTAs/SM)
static int g_tune_bwd = 4;     // transposed SpMM (bits): >= 1 lane-staged (rows in flight / occupancy, see the dispatch), 0 = per-row

// Forward SpMM grids: one wave of persistent CTAs (grid-stride rows).  Short
// CTAs (k rows per warp, many waves) were measured slower both alone and
// next to the sampling branch on B200.
template <typename Kernel>
static inline int spmm_grid(Kernel k, long long rows) {
  return resident_grid(k, kSpmmBlock, 0, (rows * 32 + kSpmmBlock - 1) / kSpmmBlock);
}

// ---- SpMM backward -------------------------------------------------------------
__global__ void tcount_kernel(BlockView bv, int32_t* __restrict__ tcount, int32_t* __restrict__ self_of) {
  const int64_t ne = bv.counts[GNS_CNT_EDGES], nd = bv.counts[GNS_CNT_DST];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne + nd; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < ne)
      atomicAdd(tcount + bv.edge_src[i], 1);
    else
      self_of[bv.self_pos[i - ne]] = (int32_t)(i - ne);
  }
}

constexpr int kTsBlock = 256, kTsItems = 8;

__global__ void __launch_bounds__(kTsBlock) tscan_reduce_kernel(BlockView bv, const int32_t* __restrict__ tcount,
                                                                unsigned long long* tile_sums) {
  const int64_t n = bv.counts[GNS_CNT_SRC];
  scan2_reduce<kTsBlock, kTsItems>(n, [&](long long i) { return (unsigned long long)tcount[i]; }, tile_sums);
}

__global__ void __launch_bounds__(kTsBlock) tscan_apply_kernel(BlockView bv, int32_t* __restrict__ tcount,
                                                               int32_t* __restrict__ tptr,
                                                               const unsigned long long* tile_sums) {
  const int64_t n = bv.counts[GNS_CNT_SRC];
  scan2_apply<kTsBlock, kTsItems>(
      n, [&](long long i) { return (unsigned long long)tcount[i]; },
      [&](long long i, unsigned long long ex, unsigned long long) {
        tptr[i] = (int32_t)ex;
        tcount[i] = 0;  // becomes the scatter cursor
      },
      [&](unsigned long long tot) { tptr[n] = (int32_t)tot; }, tile_sums);
}

__global__ void tscatter_kernel(BlockView bv, int32_t* __restrict__ cursor, const int32_t* __restrict__ tptr,
                                uint64_t* __restrict__ tkeys) {
  const int64_t ne = bv.counts[GNS_CNT_EDGES];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = bv.edge_src[e];
    int slot = atomicAdd(cursor + s, 1);
    tkeys[tptr[s] + slot] = ((uint64_t)(uint32_t)bv.edge_dst[e] << 32) | (uint64_t)(uint32_t)e;
  }
}

// Long transposed rows.  A sampled block's source rows have ~1 item, but a
// hub source can be the neighbour of thousands of dst rows (the reference's
// generate_powerlaw graph, real graphs): a warp per row then serialises the
// whole row.  Rows of more than kBwdLong items are split into kBwdSeg-item
// segments: tsort registers them (segment -> row map, per-row segment base),
// every warp of the float32 backward first computes unclaimed segments'
// partial sums (sequential FMAs in ascending dst order, from 0), and the
// warp that owns the row adds the partials in segment order — computing any
// segment nobody has claimed yet itself, so no warp waits on a CTA that is
// not running.  Claims and completion flags carry a generation number that
// the last CTA of each backward launch advances, so repeated launches over
// the same transpose need no reset.  Rows of more than kTsortWarpMax items
// are sorted by whole CTAs in shared memory (tsort_long_kernel).
#ifndef GNS_BWD_LONG
#define GNS_BWD_LONG 1   // (0: builds without the long-row path, for A/B)
#endif
constexpr int kBwdLong = 16, kBwdSeg = 32, kTsortWarpMax = 256;
enum { kCtrSegs = 0, kCtrSort = 1, kCtrGen = 2, kCtrTicket = 3, kCtrLong = 4, kCtrN = 8 };

struct LongRows {
  int32_t* ctr;             // kCtrN counters (zeroed with the transpose counts)
  int32_t* sbase;           // per source row: first segment (long rows only)
  int32_t* seg_row;         // per segment: its source row
  int32_t* claim;           // per segment: generation that claimed it
  int32_t* done;            // per segment: generation whose partial is stored
  float4* part;             // per segment: partial sum row (dim / 4 float4)
  int32_t* slist;           // rows sorted by tsort_long_kernel
  int32_t* llist;           // rows of more than kBwdLong items
};

__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ascending sort of a[0, L) in place: the all-ascending bitonic network
// (flip, then half-cleaners) with out-of-range partners skipped, so L need
// not be a power of two.  Threads tid = 0..nt-1 of the group call it; sync()
// is the group's barrier (warp or CTA; shared or global memory).
template <typename Sync>
__device__ __forceinline__ void bitonic_asc(uint64_t* a, int L, int tid, int nt, Sync sync) {
  int P = 1;
  while (P < L) P <<= 1;
  for (int k = 2; k <= P; k <<= 1) {
    const int half = k >> 1;
    for (int t = tid; t < P / 2; t += nt) {
      const int i = (t & (half - 1)) | ((t & ~(half - 1)) << 1), jj = i ^ (k - 1);
      if (jj < L && a[jj] < a[i]) { const uint64_t x = a[i]; a[i] = a[jj]; a[jj] = x; }
    }
    sync();
    for (int st = k >> 2; st >= 1; st >>= 1) {
      for (int t = tid; t < P / 2; t += nt) {
        const int i = (t & (st - 1)) | ((t & ~(st - 1)) << 1), jj = i + st;
        if (jj < L && a[jj] < a[i]) { const uint64_t x = a[i]; a[i] = a[jj]; a[jj] = x; }
      }
      sync();
    }
  }
}

struct WarpBar {
  __device__ void operator()() const { __syncwarp(); }
};
struct CtaBar {
  __device__ void operator()() const { __syncthreads(); }
};

__device__ __forceinline__ float twn_of(BlockView bv, uint64_t key) {
  const int32_t d = (int32_t)(key >> 32), e = (int32_t)(key & 0xffffffffu);
  return (float)bv.edge_weight[e] / (float)max(bv.dst_degree[d], 1);
}

// Per transposed row: sort its (dst << 32 | edge) keys ascending and write
// the coefficients twn[t] = w_e / max(deg(dst_e), 1) in float32 — the
// float32 backward's per-edge coefficient, computed exactly as that kernel
// would (IEEE division), so it reads one value instead of the dependent
// weight + dst-degree loads.  A warp takes 32 consecutive rows; rows of <= 8
// entries (nearly all: a sampled block's source rows have ~1 edge) are sorted
// by their own lane in registers (a 16-wide lane tier for 9..16 was measured
// no faster on cfg1 or papers100M), rows of <= 32 by the warp (shuffle ranks),
// rows of <= kTsortWarpMax by the warp in its shared-memory slice (bitonic),
// longer ones are listed for tsort_long_kernel.  Rows of more than kBwdLong
// entries are registered as segments for the backward.  Keys are unique, so
// every path gives the same order.
constexpr int kTsortLane = 8;

// one lane sorts its row of L <= N entries in registers (odd-even
// transposition network) and writes the keys and coefficients back
template <int N>
__device__ __forceinline__ void lane_sort(BlockView bv, uint64_t* __restrict__ tkeys, float* __restrict__ twn, int b,
                                          int L) {
  uint64_t x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = i < L ? tkeys[b + i] : ~0ull;
#pragma unroll
  for (int rnd = 0; rnd < N; ++rnd)
#pragma unroll
    for (int i = rnd & 1; i + 1 < N; i += 2) {
      const uint64_t lo = x[i] < x[i + 1] ? x[i] : x[i + 1], hi = x[i] < x[i + 1] ? x[i + 1] : x[i];
      x[i] = lo;
      x[i + 1] = hi;
    }
  float wv[N];
#pragma unroll
  for (int i = 0; i < N; ++i) wv[i] = i < L ? twn_of(bv, x[i]) : 0.f;
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (i < L) {
      tkeys[b + i] = x[i];
      twn[b + i] = wv[i];
    }
}

__global__ void __launch_bounds__(256) tsort_kernel(BlockView bv, const int32_t* __restrict__ tptr,
                                                    uint64_t* __restrict__ tkeys, float* __restrict__ twn,
                                                    LongRows lr) {
  __shared__ uint64_t slice[256 / 32][kTsortWarpMax];
  const int lane = threadIdx.x & 31;
  uint64_t* sa = slice[threadIdx.x >> 5];
  const int64_t n = bv.counts[GNS_CNT_SRC];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t s0 = gw * 32; s0 < n; s0 += nw * 32) {
    const int64_t s = s0 + lane;
    int b = 0, L = 0;
    if (s < n) {
      b = tptr[s];
      L = tptr[s + 1] - b;
    }
    if (L > kBwdLong) {   // register the row's backward segments
      const int nseg = (L + kBwdSeg - 1) / kBwdSeg;
      const int base = atomicAdd(lr.ctr + kCtrSegs, nseg);
      lr.sbase[s] = base;
      lr.llist[atomicAdd(lr.ctr + kCtrLong, 1)] = (int32_t)s;
      for (int j = 0; j < nseg; ++j) {
        lr.seg_row[base + j] = (int32_t)s;
        lr.claim[base + j] = 0;
        lr.done[base + j] = 0;
      }
    }
    if (L > kTsortWarpMax) lr.slist[atomicAdd(lr.ctr + kCtrSort, 1)] = (int32_t)s;
    if (L > 0 && L <= kTsortLane) lane_sort<kTsortLane>(bv, tkeys, twn, b, L);
    for (unsigned big = __ballot_sync(GNS_FULL, L > kTsortLane && L <= kTsortWarpMax); big; big &= big - 1) {
      const int j = __ffs(big) - 1;
      const int bj = __shfl_sync(GNS_FULL, b, j), Lj = __shfl_sync(GNS_FULL, L, j);
      uint64_t* a = tkeys + bj;
      if (Lj <= 32) {
        uint64_t x = lane < Lj ? a[lane] : ~0ull;
        int rank = 0;
        for (int i = 0; i < Lj; ++i) rank += __shfl_sync(GNS_FULL, x, i) < x;
        __syncwarp();
        if (lane < Lj) {
          a[rank] = x;
          twn[bj + rank] = twn_of(bv, x);
        }
        __syncwarp();
        continue;
      }
      for (int t = lane; t < Lj; t += 32) sa[t] = a[t];
      __syncwarp();
      bitonic_asc(sa, Lj, lane, 32, WarpBar());
      for (int t = lane; t < Lj; t += 32) {
        a[t] = sa[t];
        twn[bj + t] = twn_of(bv, sa[t]);
      }
      __syncwarp();
    }
  }
}

// Rows of more than kTsortWarpMax entries (listed by tsort_kernel): a CTA per
// row, bitonic in dynamic shared memory (kTsortLongKeys keys), in place in
// global memory beyond that.
constexpr int kTsortLongThreads = 512, kTsortLongKeys = 8192, kTsortLongGrid = 32;
__global__ void __launch_bounds__(kTsortLongThreads) tsort_long_kernel(BlockView bv, const int32_t* __restrict__ tptr,
                                                                       uint64_t* __restrict__ tkeys,
                                                                       float* __restrict__ twn, LongRows lr) {
  extern __shared__ uint64_t skeys[];
  // the segment count where the backward finds it with the block's sizes
  if (blockIdx.x == 0 && threadIdx.x == 0) const_cast<int32_t*>(bv.counts)[GNS_CNT_TSEGS] = lr.ctr[kCtrSegs];
  const int nlong = lr.ctr[kCtrSort];
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = blockIdx.x; k < nlong; k += gridDim.x) {
    const int32_t s = lr.slist[k];
    const int b = tptr[s], L = tptr[s + 1] - b;
    uint64_t* a = tkeys + b;
    if (L <= kTsortLongKeys) {
      for (int t = tid; t < L; t += nt) skeys[t] = a[t];
      __syncthreads();
      bitonic_asc(skeys, L, tid, nt, CtaBar());
      for (int t = tid; t < L; t += nt) {
        a[t] = skeys[t];
        twn[b + t] = twn_of(bv, skeys[t]);
      }
    } else {
      bitonic_asc(a, L, tid, nt, CtaBar());
      for (int t = tid; t < L; t += nt) twn[b + t] = twn_of(bv, a[t]);
    }
    __syncthreads();
  }
}

// Items [t0, t1) of a transposed row (ascending dst) accumulated into acc:
// acc = fma(w_t, dcat_nbr[d_t], acc) in item order — the per-row FMA order of
// every float32 backward path.  32 items' keys and coefficients are loaded
// at once (one per lane), then G neighbour rows are in flight per step.
template <int CH, int G>
__device__ __forceinline__ void bwd_chain(const float* __restrict__ dnb, uint32_t pitch, int dv,
                                          const uint64_t* __restrict__ tkeys, const float* __restrict__ twn, int t0,
                                          int t1, int lane, float4 (&acc)[CH]) {
  for (int tb = t0; tb < t1; tb += 32) {
    const int m = min(32, t1 - tb);
    int32_t d = 0;
    float w = 0.f;
    if (lane < m) {
      d = (int32_t)(tkeys[tb + lane] >> 32);
      w = twn[tb + lane];
    }
    for (int u0 = 0; u0 < m; u0 += G) {
      float4 x[G][CH];
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int32_t du = __shfl_sync(GNS_FULL, d, (u0 + u) & 31);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int c = lane + 32 * k;
          x[u][k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (u0 + u < m && c < dv) x[u][k] = row4(dnb, du, pitch)[c];
        }
      }
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const float wu = __shfl_sync(GNS_FULL, w, (u0 + u) & 31);
        if (u0 + u < m) {
#pragma unroll
          for (int k = 0; k < CH; ++k)
            if (lane + 32 * k < dv) vfma<true>(acc[k], wu, x[u][k]);
        }
      }
    }
  }
}

// the partial sum of segment `task` of row s (items b + j*kBwdSeg ...)
template <int CH, int G>
__device__ __forceinline__ void bwd_segment(const float* dnb, uint32_t pitch, int dv, const uint64_t* tkeys,
                                            const float* twn, int b, int e, int j, int lane, float4 (&p)[CH]) {
#pragma unroll
  for (int k = 0; k < CH; ++k) p[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  bwd_chain<CH, G>(dnb, pitch, dv, tkeys, twn, b + j * kBwdSeg, min(e, b + (j + 1) * kBwdSeg), lane, p);
}

// every warp, before its own rows: compute unclaimed segments
template <int CH, int G>
__device__ __noinline__ void bwd_long_produce(const LongRows lr, int nsegs, int gen, const int32_t* tptr,
                                                 const float* dnb, uint32_t pitch, int dv, const uint64_t* tkeys,
                                                 const float* twn, int64_t gw, int64_t nw, int lane) {
  for (int64_t task = gw; task < nsegs; task += nw) {
    int mine = 0;
    if (lane == 0) mine = atomicExch(lr.claim + task, gen) != gen;
    if (!__shfl_sync(GNS_FULL, mine, 0)) continue;
    const int s = lr.seg_row[task];
    const int b = tptr[s], e = tptr[s + 1];
    float4 p[CH];
    bwd_segment<CH, G>(dnb, pitch, dv, tkeys, twn, b, e, (int)task - lr.sbase[s], lane, p);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const int c = lane + 32 * k;
      if (c < dv) lr.part[task * dv + c] = p[k];
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(lr.done + task, gen);
  }
}

template <int CH> struct RowAcc { float4 v[CH]; };

// the owner of long row s: its segments' partials added in segment order.
// The warp claims 32 segments at once (one atomic per lane), computes the
// ones nobody had claimed (storing them like a producer), waits for the rest
// (each lane polls its segments' flags), then sums the partial rows with 8
// loads in flight.
template <int CH, int G>
__device__ __forceinline__ RowAcc<CH> bwd_long_row(const LongRows lr, int gen, const float* dnb, uint32_t pitch, int dv,
                                                const uint64_t* tkeys, const float* twn, int s, int b, int e,
                                                int lane) {
  const int base = lr.sbase[s];
  const int nseg = (e - b + kBwdSeg - 1) / kBwdSeg;
  for (int j0 = 0; j0 < nseg; j0 += 32) {
    const int j = j0 + lane;
    const bool mine = j < nseg && atomicExch(lr.claim + base + j, gen) != gen;
    for (unsigned mm = __ballot_sync(GNS_FULL, mine); mm; mm &= mm - 1) {
      const int jj = j0 + __ffs(mm) - 1;
      float4 p[CH];
      bwd_segment<CH, G>(dnb, pitch, dv, tkeys, twn, b, e, jj, lane, p);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int c = lane + 32 * k;
        if (c < dv) lr.part[(int64_t)(base + jj) * dv + c] = p[k];
      }
    }
    if (!mine && j < nseg)
      while (ld_acquire(lr.done + base + j) != gen) __nanosleep(32);
  }
  __threadfence();   // own partials (other lanes' stores) before the reads below
  __syncwarp();
  RowAcc<CH> out;
#pragma unroll
  for (int k = 0; k < CH; ++k) out.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  constexpr int B = 8;
  for (int j0 = 0; j0 < nseg; j0 += B) {
    float4 p[B][CH];
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int c = lane + 32 * k;
        p[u][k] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j0 + u < nseg && c < dv) p[u][k] = __ldcg(lr.part + (int64_t)(base + j0 + u) * dv + c);
      }
#pragma unroll
    for (int u = 0; u < B; ++u)
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        if (j0 + u >= nseg) continue;
        if (j0 + u == 0) {
          out.v[k] = p[u][k];
        } else {
          out.v[k].x += p[u][k].x; out.v[k].y += p[u][k].y; out.v[k].z += p[u][k].z; out.v[k].w += p[u][k].w;
        }
      }
  }
  return out;
}

// Long rows (more than kBwdLong items) run as empty rows in a backward
// kernel's row loop (dz = 0 written) and are finished here, after it, by the
// warp that owned them there ((r >> own_shift) % nw: program order makes the
// real row the last write; the bias-gradient partials group the same way
// every run),
// dz = mask(sum of segment partials + self row).  MASK: 0 none, 1 the
// pre-activation rows zmask, 2 the forward's relu' bits (mw words per row).
// (not inlined, like bwd_long_produce: the kernels' row loops keep their
// register allocation; the column-sum contribution comes back by value)
template <int CH, int G, int MASK>
__device__ __noinline__ RowAcc<CH> bwd_long_rows(const LongRows lr, int gen, const float* __restrict__ dcat,
                                                 int64_t ld_dcat, int dim, int dv, const int32_t* __restrict__ tptr,
                                                 const uint64_t* __restrict__ tkeys, const float* __restrict__ twn,
                                                 const int32_t* __restrict__ self_of, const float* __restrict__ zmask,
                                                 const uint32_t* __restrict__ relu_bits, int mw,
                                                 float* __restrict__ dh, int64_t ld_dh, int64_t gw, int64_t nw,
                                                 int lane, int own_shift) {
  RowAcc<CH> col;
#pragma unroll
  for (int k = 0; k < CH; ++k) col.v[k] = make_float4(0.f, 0.f, 0.f, 0.f);
  const int nl = lr.ctr[kCtrLong];
  const uint32_t pitch = (uint32_t)ld_dcat * 4u;
  for (int k0 = 0; k0 < nl; k0 += 32) {
    const int32_t r = k0 + lane < nl ? lr.llist[k0 + lane] : -1;
    for (unsigned m = __ballot_sync(GNS_FULL, r >= 0 && (int64_t)(r >> own_shift) % nw == gw); m; m &= m - 1) {
      const int s = __shfl_sync(GNS_FULL, r, __ffs(m) - 1);
      const int b = tptr[s], e = tptr[s + 1], sd = self_of[s];
      const RowAcc<CH> ra = bwd_long_row<CH, G>(lr, gen, dcat + dim, pitch, dv, tkeys, twn, s, b, e, lane);
#pragma unroll
      for (int k = 0; k < CH; ++k) {
        const int c = lane + 32 * k;
        if (c >= dv) continue;
        uint4 mk = make_uint4(~0u, ~0u, ~0u, ~0u);
        if constexpr (MASK == 2) mk = reinterpret_cast<const uint4*>(relu_bits + (int64_t)s * mw)[k];
        float4 a = ra.v[k];
        if (sd >= 0) {
          const float4 y = reinterpret_cast<const float4*>(dcat + (int64_t)sd * ld_dcat)[c];
          a.x += y.x; a.y += y.y; a.z += y.z; a.w += y.w;
        }
        if constexpr (MASK == 1) {
          const float4 z = reinterpret_cast<const float4*>(zmask + (int64_t)s * ld_dh)[c];
          a.x = z.x > 0.f ? a.x : 0.f; a.y = z.y > 0.f ? a.y : 0.f;
          a.z = z.z > 0.f ? a.z : 0.f; a.w = z.w > 0.f ? a.w : 0.f;
        } else if constexpr (MASK == 2) {
          a.x = ((mk.x >> lane) & 1u) ? a.x : 0.f; a.y = ((mk.y >> lane) & 1u) ? a.y : 0.f;
          a.z = ((mk.z >> lane) & 1u) ? a.z : 0.f; a.w = ((mk.w >> lane) & 1u) ? a.w : 0.f;
        }
        col.v[k].x += a.x; col.v[k].y += a.y; col.v[k].z += a.z; col.v[k].w += a.w;
        reinterpret_cast<float4*>(dh + (int64_t)s * ld_dh)[c] = a;
      }
    }
  }
  return col;
}

// after the last CTA of a backward launch: advance the generation
__device__ __forceinline__ void bwd_long_finish(const LongRows& lr, int nsegs) {
  if (nsegs <= 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(lr.ctr + kCtrTicket, 1) == (int)gridDim.x - 1) {
      lr.ctr[kCtrTicket] = 0;
      atomicAdd(lr.ctr + kCtrGen, 1);
    }
  }
}

template <typename T, bool EXACT>
__device__ __forceinline__ T div_norm(T x, T d);
template <> __device__ __forceinline__ float div_norm<float, false>(float x, float d) { return __fdiv_rn(x, d); }
template <> __device__ __forceinline__ double div_norm<double, true>(double x, double d) { return DDIV(x, d); }

// BITS: the relu' mask comes from the forward's put_relu_bits words
// (relu_bits, 32 B per row at D = 256) instead of the pre-activation rows.
template <typename T, int CH, bool BITS = false>
__global__ void __launch_bounds__(kSpmmBlock) spmm_bwd_kernel(const T* __restrict__ dcat, int64_t ld_dcat, int dim,
                                                              BlockView bv, const int32_t* __restrict__ tptr,
                                                              const uint64_t* __restrict__ tkeys,
                                                              const int32_t* __restrict__ self_of,
                                                              T* __restrict__ dh, int64_t ld_dh, int64_t pad_rows,
                                                              const T* __restrict__ zmask,
                                                              T* __restrict__ colpart,
                                                              const uint32_t* __restrict__ relu_bits = nullptr,
                                                              const float* __restrict__ twn = nullptr,
                                                              LongRows lr = LongRows{}) {
  // BITS (float32): the per-edge coefficient comes from the transpose's twn
  // and the self row of dcat is requested before the edge loop, so a row's
  // chain is bounds -> (keys, coefficients, self row) -> dcat rows
  using V = typename Vec<T>::type;
  constexpr int VW = Vec<T>::W;
  constexpr bool EXACT = sizeof(T) == 8;
  const int lane = threadIdx.x & 31;
  const int64_t n = bv.counts[GNS_CNT_SRC];
  const int dv = dim / VW;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // fused epilogue (model.py:218,220): dz = relu'(z) * dh and per-block
  // column partial sums of dz for the bias gradient (requires dv <= 32*CH)
  T colacc[CH][VW];
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int q = 0; q < VW; ++q) colacc[j][q] = (T)0;
  const int mw = ((dv + 31) >> 5) * 4;
  // float32, one column pass: long rows (> kBwdLong items) by segments, the
  // rows themselves after the row loop (bwd_long_rows)
  constexpr int GL = 8 / CH;   // segment chains: 8 float4 per lane in flight
  int nsegs = 0, gen = 0;
  if constexpr (!EXACT) {
    const int tsegs = bv.counts[GNS_CNT_TSEGS];   // loaded with n (one round trip)
    if (GNS_BWD_LONG && lr.ctr && dv <= 32 * CH) nsegs = tsegs;
    if (nsegs > 0) {
      gen = lr.ctr[kCtrGen] + 1;
      bwd_long_produce<CH, GL>(lr, nsegs, gen, tptr, reinterpret_cast<const float*>(dcat) + dim,
                               (uint32_t)ld_dcat * 4u, dv, tkeys, twn, gw, nw, lane);
    }
  }
  for (int64_t s = gw; s < n; s += nw) {
    const int b = tptr[s];
    int e_end = tptr[s + 1];
    int sd = self_of[s];
    if (nsegs > 0 && e_end - b > kBwdLong) {   // a long row: empty here, finished by this warp after the loop
      e_end = b;
      sd = -1;
    }
    uint32_t my_bits = 0;   // lane i < mw holds relu-bit word i of row s
    if constexpr (BITS) my_bits = lane < mw ? relu_bits[s * mw + lane] : 0u;
    for (int c0 = 0; c0 < dv; c0 += 32 * CH) {
      T acc[CH][VW];
#pragma unroll
      for (int j = 0; j < CH; ++j)
#pragma unroll
        for (int q = 0; q < VW; ++q) acc[j][q] = (T)0;
      V sv[CH];   // BITS: the self row, requested early
      if constexpr (BITS) {
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int c = c0 + lane + 32 * j;
          vzero(sv[j]);
          if (sd >= 0 && c < dv) sv[j] = reinterpret_cast<const V*>(dcat + (int64_t)sd * ld_dcat)[c];
        }
      }
      // transposed row in ascending dst order (csc_matvecs order, model.py:224)
      for (int t = b; t < e_end; ++t) {
        const uint64_t key = tkeys[t];
        const int32_t d = (int32_t)(key >> 32), e = (int32_t)(key & 0xffffffffu);
        T w = (T)0, nrm = (T)1;
        if constexpr (!BITS) {
          w = (T)bv.edge_weight[e];
          nrm = (T)max(bv.dst_degree[d], 1);
        }
        const V* grow = reinterpret_cast<const V*>(dcat + (int64_t)d * ld_dcat + dim);
        V g[CH];
#pragma unroll
        for (int j = 0; j < CH; ++j) {
          const int c = c0 + lane + 32 * j;
          if (c < dv) g[j] = grow[c];
        }
        if constexpr (EXACT) {
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const T* gp = reinterpret_cast<const T*>(&g[j]);
#pragma unroll
            for (int q = 0; q < VW; ++q) acc[j][q] = DADD(acc[j][q], DMUL(w, DDIV(gp[q], nrm)));
          }
        } else {
          T wn;
          if constexpr (BITS) wn = (T)twn[t];
          else wn = w / nrm;
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            const T* gp = reinterpret_cast<const T*>(&g[j]);
#pragma unroll
            for (int q = 0; q < VW; ++q) acc[j][q] = fmaf(wn, gp[q], acc[j][q]);
          }
        }
      }
      const V* srow = sd >= 0 ? reinterpret_cast<const V*>(dcat + (int64_t)sd * ld_dcat) : nullptr;
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        const int c = c0 + lane + 32 * j;
        uint32_t wq[VW];
        if constexpr (BITS) {   // every lane takes part in the shuffles
#pragma unroll
          for (int q = 0; q < VW; ++q) wq[q] = __shfl_sync(GNS_FULL, my_bits, ((c0 >> 5) + j) * 4 + q);
        }
        if (c >= dv) continue;
        if (srow) {
          V g;
          if constexpr (BITS) g = sv[j];
          else g = srow[c];
          const T* gp = reinterpret_cast<const T*>(&g);
#pragma unroll
          for (int q = 0; q < VW; ++q) {
            if constexpr (EXACT) acc[j][q] = DADD(acc[j][q], gp[q]);
            else acc[j][q] = acc[j][q] + gp[q];
          }
        }
        V out;
        T* op = reinterpret_cast<T*>(&out);
        if constexpr (BITS) {
#pragma unroll
          for (int q = 0; q < VW; ++q) op[q] = ((wq[q] >> lane) & 1u) ? acc[j][q] : (T)0;
        } else if (zmask) {
          V zv = reinterpret_cast<const V*>(zmask + s * ld_dh)[c];
          const T* zp = reinterpret_cast<const T*>(&zv);
#pragma unroll
          for (int q = 0; q < VW; ++q) op[q] = zp[q] > (T)0 ? acc[j][q] : (T)0;
        } else {
#pragma unroll
          for (int q = 0; q < VW; ++q) op[q] = acc[j][q];
        }
        if (c0 == 0) {
#pragma unroll
          for (int q = 0; q < VW; ++q) colacc[j][q] += op[q];
        }
        reinterpret_cast<V*>(dh + s * ld_dh)[c] = out;
      }
    }
  }
  if constexpr (!EXACT) {
    if (nsegs > 0) {
      RowAcc<CH> col;
      if constexpr (BITS)
        col = bwd_long_rows<CH, GL, 2>(lr, gen, (const float*)dcat, ld_dcat, dim, dv, tptr, tkeys, twn, self_of,
                                       nullptr, relu_bits, mw, (float*)dh, ld_dh, gw, nw, lane, 0);
      else if (zmask)
        col = bwd_long_rows<CH, GL, 1>(lr, gen, (const float*)dcat, ld_dcat, dim, dv, tptr, tkeys, twn, self_of,
                                       (const float*)zmask, nullptr, mw, (float*)dh, ld_dh, gw, nw, lane, 0);
      else
        col = bwd_long_rows<CH, GL, 0>(lr, gen, (const float*)dcat, ld_dcat, dim, dv, tptr, tkeys, twn, self_of,
                                       nullptr, nullptr, mw, (float*)dh, ld_dh, gw, nw, lane, 0);
#pragma unroll
      for (int j = 0; j < CH; ++j) {
        colacc[j][0] += col.v[j].x; colacc[j][1] += col.v[j].y; colacc[j][2] += col.v[j].z; colacc[j][3] += col.v[j].w;
      }
    }
  }
  for (int64_t s = n + gw; s < pad_rows; s += nw) {
    V zero;
    vzero(zero);
    for (int c = lane; c < dv; c += 32) reinterpret_cast<V*>(dh + s * ld_dh)[c] = zero;
  }
  if (colpart) {
    __shared__ T red[kSpmmBlock / 32][32 * CH * VW];
    const int wib = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int q = 0; q < VW; ++q) red[wib][(lane + 32 * j) * VW + q] = colacc[j][q];
    __syncthreads();
    for (int col = threadIdx.x; col < dim; col += blockDim.x) {
      T t = 0;
#pragma unroll
      for (int w = 0; w < kSpmmBlock / 32; ++w) t += red[w][col];
      colpart[(int64_t)blockIdx.x * dim + col] = t;
    }
  }
  bwd_long_finish(lr, nsegs);
}

// Column c of a [rows x ncols] row-major partial-sum matrix, summed in a
// fixed order by one thread: 8 interleaved accumulators (row b into b & 7,
// so 8 loads are in flight) combined in index order.  Deterministic.
template <typename T>
__device__ __forceinline__ T colsum_fixed(const T* __restrict__ part, int rows, int ncols, int c) {
  T a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = (T)0;
  int b = 0;
  for (; b + 8 <= rows; b += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += __ldcg(part + (int64_t)(b + j) * ncols + c);
  }
  for (int j = 0; b < rows; ++b, ++j) a[j] += __ldcg(part + (int64_t)b * ncols + c);
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

// Lane-staged transposed SpMM (float32, relu' from the forward's bits; the
// default for dim <= 256).  A warp owns kChunkRows consecutive source rows
// and lane j holds row j's metadata: transpose bounds, self position and
// relu-bit words (coalesced loads), then the dst and coefficient of the row's
// first edge (one more).  Nearly every source row of a sampled block has
// exactly one item (one edge, or only its self row), so the chunk's rows go
// R at a time with every row's first dcat row requested before the first
// FMA — about 2 + 32/R dependent round trips per 32 rows instead of ~3 per
// row.  A row's further items (more edges: hub sources; the self row of a
// row that also has edges) are read after its first: the per-row FMA order
// of spmm_bwd_kernel (ascending dst, then the self row, acc starting at 0),
// so dz is bit-identical.  No shared memory in the row loop (a shared-memory
// item stream was measured 10-30% slower: short-scoreboard bound).
template <int CH, int R, int MINB>
__global__ void __launch_bounds__(kSpmmBlock, MINB) spmm_bwd_rows_kernel(const float* __restrict__ dcat,
                                                                      int64_t ld_dcat, int dim, BlockView bv,
                                                                      const int32_t* __restrict__ tptr,
                                                                      const uint64_t* __restrict__ tkeys,
                                                                      const int32_t* __restrict__ self_of,
                                                                      float* __restrict__ dh, int64_t ld_dh,
                                                                      int64_t pad_rows, float* __restrict__ colpart,
                                                                      const uint32_t* __restrict__ relu_bits,
                                                                      const float* __restrict__ twn, LongRows lr) {
  constexpr int W = kSpmmBlock / 32;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t n = bv.counts[GNS_CNT_SRC];
  const int dv = dim >> 2;
  const int mw = CH * 4;   // relu-bit words per row: dv <= 32 -> 4, <= 64 -> 8
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nchunks = (n + kChunkRows - 1) / kChunkRows;
  // long rows (> kBwdLong items, hub sources): segments first, the rows
  // themselves after the row loop (bwd_long_rows)
  constexpr int GL = 8 / CH;   // segment chains: 8 float4 per lane in flight
  int nsegs = 0, gen = 0;
  const int tsegs = bv.counts[GNS_CNT_TSEGS];   // loaded with n (one round trip)
  if (GNS_BWD_LONG && lr.ctr) nsegs = tsegs;
  if (nsegs > 0) {
    gen = lr.ctr[kCtrGen] + 1;
    bwd_long_produce<CH, GL>(lr, nsegs, gen, tptr, dcat + dim, (uint32_t)ld_dcat * 4u, dv, tkeys, twn, gw, nw, lane);
  }
  float colacc[CH][4];
#pragma unroll
  for (int k = 0; k < CH; ++k)
#pragma unroll
    for (int q = 0; q < 4; ++q) colacc[k][q] = 0.f;
  for (int64_t ch = gw; ch < nchunks; ch += nw) {
    const int64_t s0 = ch * kChunkRows;
    const int rows = (int)min((int64_t)kChunkRows, n - s0);
    int b = 0, e = 0, sd = -1, d0 = 0;
    float w0 = 0.f;
    uint4 mb[CH];   // row `lane`'s relu-bit words
#pragma unroll
    for (int k = 0; k < CH; ++k) mb[k] = make_uint4(0u, 0u, 0u, 0u);
    if (lane < rows) {
      b = tptr[s0 + lane];
      e = tptr[s0 + lane + 1];
      sd = self_of[s0 + lane];
#pragma unroll
      for (int k = 0; k < CH; ++k) mb[k] = reinterpret_cast<const uint4*>(relu_bits + (s0 + lane) * mw)[k];
      // a long row runs as an empty one here (dz = 0 written) and is
      // finished by this warp after the loop (bwd_long_rows, owner = chunk's)
      if (nsegs > 0 && e - b > kBwdLong) {
        e = b;
        sd = -1;
      }
    }
    if (e > b) {
      d0 = (int32_t)(tkeys[b] >> 32);
      w0 = twn[b];
    }
    for (int j0 = 0; j0 < rows; j0 += R) {
      float4 x[R][CH];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        // (the row's scalars are shuffled again when it is consumed: fewer
        // live registers across the loads)
        const int j = (j0 + r) & 31;   // rows past `rows` have b == e, sd < 0
        const int bj = __shfl_sync(GNS_FULL, b, j), ej = __shfl_sync(GNS_FULL, e, j);
        const int sj = __shfl_sync(GNS_FULL, sd, j), dj = __shfl_sync(GNS_FULL, d0, j);
        // first item: the first edge's neighbour half, else the self half
        const bool edge = ej > bj;
        const float4* src = reinterpret_cast<const float4*>(
            edge ? dcat + dim + (uint64_t)(uint32_t)dj * ((uint32_t)ld_dcat)
                 : dcat + (uint64_t)(uint32_t)(sj < 0 ? 0 : sj) * ((uint32_t)ld_dcat));
        const bool any = edge || sj >= 0;
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int c = lane + 32 * k;
          x[r][k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (any && c < dv) x[r][k] = src[c];
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int j = j0 + r;
        if (j >= rows) break;
        const int bj = __shfl_sync(GNS_FULL, b, j), ej = __shfl_sync(GNS_FULL, e, j);
        const int sj = __shfl_sync(GNS_FULL, sd, j);
        const float wj = __shfl_sync(GNS_FULL, w0, j);
        float4 acc[CH];
        const bool edge = ej > bj;
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (edge) {
            vfma<true>(acc[k], wj, x[r][k]);
          } else if (sj >= 0) {
            acc[k].x += x[r][k].x; acc[k].y += x[r][k].y;
            acc[k].z += x[r][k].z; acc[k].w += x[r][k].w;
          }
        }
        if (edge) {
          for (int t = bj + 1; t < ej; ++t) {   // further edges, ascending dst
            const float4* src = reinterpret_cast<const float4*>(dcat + (int64_t)(int32_t)(tkeys[t] >> 32) * ld_dcat + dim);
            const float wn = twn[t];
#pragma unroll
            for (int k = 0; k < CH; ++k) {
              const int c = lane + 32 * k;
              if (c < dv) vfma<true>(acc[k], wn, src[c]);
            }
          }
          if (sj >= 0) {   // then the self row
            const float4* src = reinterpret_cast<const float4*>(dcat + (int64_t)sj * ld_dcat);
#pragma unroll
            for (int k = 0; k < CH; ++k) {
              const int c = lane + 32 * k;
              if (c < dv) {
                const float4 y = src[c];
                acc[k].x += y.x; acc[k].y += y.y; acc[k].z += y.z; acc[k].w += y.w;
              }
            }
          }
        }
        float4* drow = reinterpret_cast<float4*>(dh + (s0 + j) * ld_dh);
#pragma unroll
        for (int k = 0; k < CH; ++k) {
          const int c = lane + 32 * k;
          const uint32_t m0 = __shfl_sync(GNS_FULL, mb[k].x, j), m1 = __shfl_sync(GNS_FULL, mb[k].y, j);
          const uint32_t m2 = __shfl_sync(GNS_FULL, mb[k].z, j), m3 = __shfl_sync(GNS_FULL, mb[k].w, j);
          if (c >= dv) continue;
          float4 out;
          out.x = ((m0 >> lane) & 1u) ? acc[k].x : 0.f;
          out.y = ((m1 >> lane) & 1u) ? acc[k].y : 0.f;
          out.z = ((m2 >> lane) & 1u) ? acc[k].z : 0.f;
          out.w = ((m3 >> lane) & 1u) ? acc[k].w : 0.f;
          colacc[k][0] += out.x; colacc[k][1] += out.y; colacc[k][2] += out.z; colacc[k][3] += out.w;
          drow[c] = out;
        }
      }
    }
  }
  if (nsegs > 0) {
    const RowAcc<CH> col = bwd_long_rows<CH, GL, 2>(lr, gen, dcat, ld_dcat, dim, dv, tptr, tkeys, twn, self_of,
                                                    nullptr, relu_bits, mw, dh, ld_dh, gw, nw, lane, 5);
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      colacc[k][0] += col.v[k].x; colacc[k][1] += col.v[k].y; colacc[k][2] += col.v[k].z; colacc[k][3] += col.v[k].w;
    }
  }
  for (int64_t s = n + gw; s < pad_rows; s += nw)
    for (int c = lane; c < dv; c += 32) reinterpret_cast<float4*>(dh + s * ld_dh)[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (colpart) {
    __shared__ float red[W][32 * CH * 4];
#pragma unroll
    for (int k = 0; k < CH; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[wib][(lane + 32 * k) * 4 + q] = colacc[k][q];
    __syncthreads();
    for (int col = threadIdx.x; col < dim; col += blockDim.x) {
      float t = 0.f;
#pragma unroll
      for (int w = 0; w < W; ++w) t += red[w][col];
      colpart[(int64_t)blockIdx.x * dim + col] = t;
    }
  }
  bwd_long_finish(lr, nsegs);
}

// dz = relu'(z) * dh (model.py:218) fused with the bias gradient db = sum_r dz
// (model.py:220): per-block column partials, then a fixed-order reduction.
template <typename T>
__global__ void dense_bwd_partial_kernel(const T* __restrict__ dh, const T* __restrict__ z, int64_t ld,
                                         const int32_t* __restrict__ n_dev, int64_t n_host, int ncols,
                                         T* __restrict__ dz, T* __restrict__ partial, int rows_per_block) {
  __shared__ T red[4][64];
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int c = blockIdx.y * 64 + tx;
  const int64_t n = n_dev ? n_dev[0] : n_host;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(n, r0 + rows_per_block);
  T sum = 0;
  if (c < ncols) {
    for (int64_t r = r0 + ty; r < r1; r += 4) {
      T v = dh[r * ld + c];
      if (z) v = z[r * ld + c] > (T)0 ? v : (T)0;
      if (dz) dz[r * ld + c] = v;
      sum += v;
    }
  }
  red[ty][tx] = sum;
  __syncthreads();
  if (ty == 0 && c < ncols)
    partial[(int64_t)blockIdx.x * ncols + c] = (red[0][tx] + red[1][tx]) + (red[2][tx] + red[3][tx]);
}

// one warp per column: fixed lane-strided partial sums + shuffle tree (deterministic)
// db[c] = sum over blocks of partial[b][c] in a fixed order: CTA per 32
// columns, warp w sums rows w, w+8, ... (coalesced 128-byte row reads), then
// the 8 warp sums are added in warp order.  Launch with colsum_grid(ncols).
constexpr int kColsumWarps = 8;
template <typename T, int W = kColsumWarps>
__global__ void __launch_bounds__(W * 32) colsum_final_kernel(const T* __restrict__ partial, int nblocks, int ncols,
                                                              T* __restrict__ db) {
  __shared__ T red[W][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  T s = 0;
  if (c < ncols)
    for (int b = w; b < nblocks; b += W) s += partial[(int64_t)b * ncols + c];
  red[w][lane] = s;
  __syncthreads();
  if (w == 0 && c < ncols) {
    T t = red[0][lane];
#pragma unroll
    for (int i = 1; i < W; ++i) t += red[i][lane];
    db[c] = t;
  }
}
static inline unsigned colsum_grid(int ncols) { return (unsigned)((ncols + 31) / 32); }
// Few columns over many partial rows (a bias gradient: <= 1024 columns,
// hundreds of per-CTA partials) get 32 warps per column block, so each warp's
// dependent add chain is 4x shorter; wide reductions keep 8 warps.
template <typename T>
static inline void colsum_launch(const T* part, int nrows, int ncols, T* out, cudaStream_t stream) {
  if (ncols <= 1024 && nrows >= 128)
    colsum_final_kernel<T, 32><<<colsum_grid(ncols), 32 * 32, 0, stream>>>(part, nrows, ncols, out);
  else
    colsum_final_kernel<T><<<colsum_grid(ncols), kColsumWarps * 32, 0, stream>>>(part, nrows, ncols, out);
}

struct BwdWs {
  void* colpart;
  int32_t* tcount;
  int32_t* tptr;
  int32_t* self_of;
  uint64_t* tkeys;
  float* twn;
  void* scan;
  long long tiles;
  LongRows lr;
};

static size_t bwd_ws(int64_t max_src, int64_t max_edges, int32_t dim, void* base, size_t cap, BwdWs* w) {
  Workspace ws(base, cap);
  w->colpart = (void*)ws.take<double>((size_t)num_sms() * 8 * (size_t)(dim > 0 ? dim : 1));
  // tcount is followed by the long-row counters (one memset clears both)
  w->tcount = ws.take<int32_t>(max_src + 1 + kCtrN);
  w->tptr = ws.take<int32_t>(max_src + 1);
  w->self_of = ws.take<int32_t>(max_src + 1);
  w->tkeys = ws.take<uint64_t>(max_edges + 1);
  w->twn = ws.take<float>(max_edges + 1);
  w->tiles = (max_src + 256 * 8 - 1) / (256 * 8) + 1;
  w->scan = (void*)ws.take<char>(scan_status_bytes(w->tiles));
  // a long row (L > kBwdLong items) has ceil(L / kBwdSeg) < L / kBwdSeg + 1
  // segments, and there are fewer than E / kBwdLong long rows
  const int64_t max_segs = max_edges / kBwdSeg + max_edges / (kBwdLong + 1) + 1;
  LongRows& lr = w->lr;
  lr.ctr = w->tcount + max_src + 1;
  lr.sbase = ws.take<int32_t>(max_src + 1);
  lr.seg_row = ws.take<int32_t>(max_segs);
  lr.claim = ws.take<int32_t>(max_segs);
  lr.done = ws.take<int32_t>(max_segs);
  lr.slist = ws.take<int32_t>(max_edges / (kTsortWarpMax + 1) + 1);
  lr.llist = ws.take<int32_t>(max_edges / (kBwdLong + 1) + 1);
  lr.part = reinterpret_cast<float4*>(ws.take<float>((size_t)max_segs * (size_t)((dim + 3) / 4 * 4)));
  return ws.off;
}

// ---- softmax cross-entropy ------------------------------------------------------
template <typename T>
__global__ void xent_kernel(const T* __restrict__ logits, int64_t ld, const int32_t* __restrict__ n_dev, int C,
                            const int32_t* __restrict__ labels, const int32_t* __restrict__ targets,
                            T* __restrict__ grad, double* __restrict__ row_loss, int64_t pad_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t n = n_dev[0];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = gw; r < n; r += nw) {
    const T* z = logits + r * ld;
    T mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = max(mx, z[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(GNS_FULL, mx, o));
    T s = 0;
    for (int c = lane; c < C; c += 32) s += exp(z[c] - mx);
    s = warp_sum(s);
    const T lse = log(s);
    const int lab = labels[targets[r]];
    const T inv_n = (T)1 / (T)n;
    for (int c = lane; c < C; c += 32) {
      T lp = (z[c] - mx) - lse;
      T g = exp(lp);
      if (c == lab) g -= (T)1;
      grad[r * ld + c] = g * inv_n;
      if (c == lab) row_loss[r] = -(double)lp;
    }
  }
  for (int64_t r = n + gw; r < pad_rows; r += nw)
    for (int c = lane; c < C; c += 32) grad[r * ld + c] = (T)0;
}

// Output layer in one launch (the graphed engine's training step): softmax
// cross-entropy rows (xent_kernel's arithmetic, warp per row), the bias
// gradient db[c] = sum_r dlogits[r][c] (model.py:218-220: the output layer's
// dz is dlogits) as per-CTA column partials, and — in the last CTA to finish
// (ticket counter, reset for the next launch) — the mean loss and db, each
// summed in a fixed order (deterministic whichever CTA is last).  Replaces
// xent + mean + dense_bwd_partial + colsum: three launches fewer on the
// training branch.  Columns <= 32 * kXentCh.
constexpr int kXentCh = 8;
template <typename T>
__global__ void __launch_bounds__(256) xent_bias_kernel(const T* __restrict__ logits, int64_t ld,
                                                        const int32_t* __restrict__ n_dev, int C,
                                                        const int32_t* __restrict__ labels,
                                                        const int32_t* __restrict__ targets, T* __restrict__ grad,
                                                        double* __restrict__ loss_out, T* __restrict__ grad_bias,
                                                        double* __restrict__ row_loss, T* __restrict__ partial,
                                                        unsigned* __restrict__ ticket, int64_t pad_rows) {
  __shared__ T red[8][32 * kXentCh];
  __shared__ double s_red[8];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t n = n_dev[0];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  T col[kXentCh];
#pragma unroll
  for (int i = 0; i < kXentCh; ++i) col[i] = (T)0;
  for (int64_t r = gw; r < n; r += nw) {
    const T* z = logits + r * ld;
    T mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = max(mx, z[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(GNS_FULL, mx, o));
    T s = 0;
    for (int c = lane; c < C; c += 32) s += exp(z[c] - mx);
    s = warp_sum(s);
    const T lse = log(s);
    const int lab = labels[targets[r]];
    const T inv_n = (T)1 / (T)n;
#pragma unroll
    for (int i = 0; i < kXentCh; ++i) {
      const int c = lane + 32 * i;
      if (c < C) {
        T lp = (z[c] - mx) - lse;
        T g = exp(lp);
        if (c == lab) g -= (T)1;
        const T gv = g * inv_n;
        grad[r * ld + c] = gv;
        col[i] += gv;
        if (c == lab) row_loss[r] = -(double)lp;
      }
    }
  }
  for (int64_t r = n + gw; r < pad_rows; r += nw)
    for (int c = lane; c < C; c += 32) grad[r * ld + c] = (T)0;
  // per-CTA column partials (warp order)
#pragma unroll
  for (int i = 0; i < kXentCh; ++i) red[wib][lane + 32 * i] = col[i];
  __syncthreads();
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    T t = (T)0;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][c];
    partial[(int64_t)blockIdx.x * C + c] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) *ticket = 0u;   // ready for the next launch (graph replay)
  double acc = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += __ldcg(row_loss + i);
  acc = warp_sum(acc);
  if (lane == 0) s_red[wib] = acc;
  for (int c = threadIdx.x; c < C; c += blockDim.x) grad_bias[c] = colsum_fixed(partial, gridDim.x, C, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = 0;
    for (int w = 0; w < 8; ++w) v += s_red[w];
    loss_out[0] = n > 0 ? v / (double)n : 0.0;
  }
}

__global__ void mean_kernel(const double* __restrict__ x, const int32_t* __restrict__ n_dev, double* __restrict__ out) {
  __shared__ double sh[32];
  const int64_t n = n_dev[0];
  double s = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[0] = n > 0 ? v / (double)n : 0.0;
  }
}

// ---- Adam ---------------------------------------------------------------------------
template <typename T>
__global__ void adam_kernel(T* __restrict__ p, const T* __restrict__ g, T* __restrict__ m, T* __restrict__ v,
                            int64_t n, T lr, T b1, T b2, T eps, T bc1, T bc2, T gs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T gr = g[i] * gs;
    T mi = b1 * m[i] + ((T)1 - b1) * gr;
    T vi = b2 * v[i] + ((T)1 - b2) * gr * gr;
    m[i] = mi;
    v[i] = vi;
    T mh = mi / bc1, vh = vi / bc2;
    p[i] -= lr * mh / (sqrt(vh) + eps);
  }
}

// Adam with the step count read on the device (t = *step_dev + 1), so a step
// captured in a CUDA graph stays correct at every replay; the bias
// corrections are evaluated per thread in double exactly as gns_adam does on
// the host; the last CTA to finish advances the counter (step_dev[1] is its
// ticket, zero between launches).
template <typename T>
__global__ void adam_dev_kernel(T* __restrict__ p, const T* __restrict__ g, T* __restrict__ m, T* __restrict__ v,
                                int64_t n, double lr, double b1, double b2, double eps,
                                int64_t* __restrict__ step_dev, T gs) {
  const double t = (double)(step_dev[0] + 1);
  const T bc1 = (T)(1.0 - pow(b1, t)), bc2 = (T)(1.0 - pow(b2, t));
  const T lr_ = (T)lr, b1_ = (T)b1, b2_ = (T)b2, eps_ = (T)eps;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T gr = g[i] * gs;
    T mi = b1_ * m[i] + ((T)1 - b1_) * gr;
    T vi = b2_ * v[i] + ((T)1 - b2_) * gr * gr;
    m[i] = mi;
    v[i] = vi;
    T mh = mi / bc1, vh = vi / bc2;
    p[i] -= lr_ * mh / (sqrt(vh) + eps_);
  }
  // step_dev[1] is a ticket: the last CTA (every CTA has read step_dev[0] by
  // then) advances the step count and resets the ticket
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long* tk = reinterpret_cast<unsigned long long*>(step_dev + 1);
    if (atomicAdd(tk, 1ull) == (unsigned long long)gridDim.x - 1) {
      *tk = 0ull;
      step_dev[0] += 1;
    }
  }
}

}  // namespace gns

using namespace gns;

extern "C" {

// ---- TMA gather (features[input_nodes], float32, D <= 256) --------------------
// The Tensor Memory Accelerator fetches rows by index: one elected thread per
// warp issues cp.async.bulk.tensor.2d ... tile::gather4 (4 table rows of D
// floats into shared memory, completion on the slot's mbarrier), then a bulk
// shared->global store of the 4 rows to their contiguous place in `out`.
// kTmaSlots groups per warp are in flight; no feature bytes pass through
// registers.
constexpr int kTmaWarps = 8;
constexpr int kTmaSlots = 6;
constexpr int kTmaLag = 3;   // gathers in flight per warp; the other slots drain their stores
constexpr int kTmaBarBytes = 512;   // kTmaWarps * kTmaSlots mbarriers, padded

__device__ __forceinline__ uint32_t tma_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(kTmaWarps * 32) gather_tma_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                    const int32_t* __restrict__ rows,
                                                                    const int32_t* __restrict__ n_rows_dev,
                                                                    int64_t max_rows, int dim, float* __restrict__ out,
                                                                    int64_t ld_out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t row_bytes = (uint32_t)dim * 4u;
  // slots are 128-byte aligned (TMA shared-memory destinations)
  const uint32_t slot_bytes = (4u * row_bytes + 127u) & ~127u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + wib * kTmaSlots;
  unsigned char* slots = smem + kTmaBarBytes + (size_t)wib * kTmaSlots * slot_bytes;
  int64_t n = n_rows_dev ? (int64_t)n_rows_dev[0] : max_rows;
  if (n > max_rows) n = max_rows;
  const int64_t ngroups = (n + 3) >> 2;
  const int64_t gw = (int64_t)blockIdx.x * kTmaWarps + wib, nw = (int64_t)gridDim.x * kTmaWarps;
  const bool leader = lane == 0;   // one thread per warp drives the TMA unit
  if (leader) {
    for (int i = 0; i < kTmaSlots; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tma_smem_u32(&bars[i])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  auto store_group = [&](int64_t g, int slot, uint32_t parity) {
    // wait for the gather, then write the group's valid rows
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n\t"
        "DONE:\n\t}" ::"r"(tma_smem_u32(&bars[slot])),
        "r"(parity)
        : "memory");
    const int valid = (int)(n - 4 * g < 4 ? n - 4 * g : 4);
    unsigned char* src = slots + (size_t)slot * slot_bytes;
    if (ld_out == dim) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + 4 * g * ld_out),
                   "r"(tma_smem_u32(src)), "r"(row_bytes * (uint32_t)valid)
                   : "memory");
    } else {
      for (int i = 0; i < valid; ++i)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(out + (4 * g + i) * ld_out),
                     "r"(tma_smem_u32(src + i * row_bytes)), "r"(row_bytes)
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  // group k of this warp (global group gw + k*nw) lives in slot k % kTmaSlots;
  // at step k group k-lag is stored and the gather of group k is issued once
  // the store of group k-S (same slot, issued S-lag steps earlier) has
  // finished reading shared memory.  The warp's lanes load the row ids of
  // 32 groups at a time (one int4 each); the leader takes them by shuffle.
  const int64_t my_groups = gw < ngroups ? (ngroups - gw + nw - 1) / nw : 0;
  for (int64_t k0 = 0; k0 < my_groups; k0 += 32) {
    int4 ids = make_int4(0, 0, 0, 0);
    {
      const int64_t k = k0 + lane;
      if (k < my_groups) {
        const int64_t b = 4 * (gw + k * nw);
        if (b + 3 < n) {
          ids = *reinterpret_cast<const int4*>(rows + b);
        } else {
          ids.x = rows[b];
          ids.y = b + 1 < n ? rows[b + 1] : ids.x;
          ids.z = b + 2 < n ? rows[b + 2] : ids.x;
          ids.w = ids.x;
        }
      }
    }
    const int cnt = (int)(my_groups - k0 < 32 ? my_groups - k0 : 32);
    for (int u = 0; u < cnt; ++u) {
      const int r0 = __shfl_sync(GNS_FULL, ids.x, u), r1 = __shfl_sync(GNS_FULL, ids.y, u);
      const int r2 = __shfl_sync(GNS_FULL, ids.z, u), r3 = __shfl_sync(GNS_FULL, ids.w, u);
      if (leader) {
        const int64_t k = k0 + u;
        const int slot = (int)(k % kTmaSlots);
        if (k >= kTmaLag) {
          const int64_t q = k - kTmaLag;
          store_group(gw + q * nw, (int)(q % kTmaSlots), (uint32_t)((q / kTmaSlots) & 1));
        }
        // the store of group k-S (this slot's previous group) has read its
        // shared memory; the S-lag stores issued after it may still pend
        if (k >= kTmaSlots) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmaSlots - kTmaLag) : "memory");
        const uint32_t bar = tma_smem_u32(&bars[slot]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(4u * row_bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(tma_smem_u32(slots + (size_t)slot * slot_bytes)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(bar), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
            : "memory");
      }
    }
  }
  if (leader) {
    // drain: the groups not stored yet
    const int64_t first = my_groups > kTmaLag ? my_groups - kTmaLag : 0;
    for (int64_t k = first; k < my_groups; ++k)
      store_group(gw + k * nw, (int)(k % kTmaSlots), (uint32_t)((k / kTmaSlots) & 1));
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// (gns_tune "gather_tma") TMA gather4 path for float32 rows: 1 = for D <= 64
// (cfg1, D = 64: 0.33 vs 0.28 of HBM peak), 2 = for D <= 256 (papers100M,
// D = 128: 0.81 vs 0.84 for the register kernel, so not the default), 0 = off
static int g_gather_tma = 1;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

// 2-D float32 map over the table (rows x dim, row pitch ld floats), box = one
// full row: what tile::gather4 fetches per row index
static bool table_map(CUtensorMap* m, const float* table, int64_t ld, int dim) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)dim, (cuuint64_t)0x7fffffff};
  const cuuint64_t gstride[1] = {(cuuint64_t)ld * 4};
  const cuuint32_t box[2] = {(cuuint32_t)dim, 1};
  const cuuint32_t estride[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)table, gdim, gstride, box, estride,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool gather_tma(const float* table, int64_t ld_in, const int32_t* rows, const int32_t* n_rows_dev,
                       int64_t max_rows, int dim, float* out, int64_t ld_out, cudaStream_t stream, int* err) {
  *err = GNS_OK;
  if (!g_gather_tma || dim % 4 || dim > (g_gather_tma == 2 ? 256 : 64) || ld_in % 4 || ld_out % 4 ||
      (uintptr_t)table % 16 ||
      (uintptr_t)out % 16 || (uintptr_t)rows % 4)
    return false;
  CUtensorMap m;
  if (!table_map(&m, table, ld_in, dim)) return false;
  const size_t slot_bytes = ((size_t)16 * dim + 127) & ~(size_t)127;
  const size_t smem = kTmaBarBytes + (size_t)kTmaWarps * kTmaSlots * slot_bytes;
  const size_t smem_max = kTmaBarBytes + (size_t)kTmaWarps * kTmaSlots * 16 * 256;
  static std::once_flag attr;
  std::call_once(attr, [smem_max] {
    cudaFuncSetAttribute(gather_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
  });
  const long long want = ((max_rows + 3) / 4 + kTmaWarps - 1) / kTmaWarps;
  static std::mutex mu;
  static std::unordered_map<int, int> per_sm_by_dim;
  int per_sm = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = per_sm_by_dim.find(dim);
    if (it != per_sm_by_dim.end()) {
      per_sm = it->second;
    } else {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gather_tma_kernel, kTmaWarps * 32, smem) !=
          cudaSuccess)
        per_sm = 1;
      per_sm_by_dim[dim] = per_sm;
    }
  }
  const int grid = grid_for(want, (long long)num_sms() * (per_sm > 0 ? per_sm : 1));
  gather_tma_kernel<<<grid, kTmaWarps * 32, smem, stream>>>(m, rows, n_rows_dev, max_rows, dim, out, ld_out);
  *err = check_launch("gather_tma");
  return true;
}

int gns_gather_rows(const void* table, int64_t ld_in, int32_t dtype_in, const int32_t* rows,
                    const int32_t* n_rows_dev, int64_t max_rows, int32_t dim, void* out, int64_t ld_out,
                    int32_t dtype_out, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (max_rows <= 0 || dim <= 0) return GNS_OK;
  const int sms = num_sms();
  if (dtype_in == 0 && dtype_out == 0) {
    bool vec = (dim % 4 == 0) && (ld_in % 4 == 0) && (ld_out % 4 == 0) && ((uintptr_t)table % 16 == 0) &&
               ((uintptr_t)out % 16 == 0);
    int terr;
    if (vec && gather_tma((const float*)table, ld_in, rows, n_rows_dev, max_rows, dim, (float*)out, ld_out, stream,
                          &terr))
      return terr;
    if (vec) {
      // 8 resident 256-thread CTAs per SM; G rows x C column blocks per warp
      const int dim4 = dim / 4;
      const int G = dim4 <= 8 ? 8 : dim4 <= 16 ? 4 : dim4 <= 32 ? 2 : 1;
      const long long want = ((max_rows + G - 1) / G * 32 + 255) / 256;
      const int grid = grid_for(want, (long long)sms * 8);
#define GNS_GATHER(G_, C_)                                                                                     \
  gather_f32x4_kernel<G_, C_><<<grid, 256, 0, stream>>>((const float*)table, ld_in, rows, n_rows_dev, max_rows, \
                                                        dim4, (float*)out, ld_out)
      if (dim4 <= 8) GNS_GATHER(8, 1);
      else if (dim4 <= 16) GNS_GATHER(4, 1);
      else if (dim4 <= 32) GNS_GATHER(2, 1);
      else if (dim4 <= 64) GNS_GATHER(1, 2);
      else if (dim4 <= 128) GNS_GATHER(1, 4);
      else GNS_GATHER(1, 8);
#undef GNS_GATHER
      return check_launch("gather_f32x4");
    }
    gather_scalar_kernel<float, float><<<sms * 16, 256, 0, stream>>>((const float*)table, ld_in, rows, n_rows_dev,
                                                                     max_rows, dim, (float*)out, ld_out);
    return check_launch("gather_f32");
  }
  if (dtype_in == 0 && dtype_out == 1) {
    gather_scalar_kernel<float, double><<<sms * 16, 256, 0, stream>>>((const float*)table, ld_in, rows, n_rows_dev,
                                                                      max_rows, dim, (double*)out, ld_out);
    return check_launch("gather_f32_f64");
  }
  if (dtype_in == 1 && dtype_out == 1) {
    gather_scalar_kernel<double, double><<<sms * 16, 256, 0, stream>>>((const double*)table, ld_in, rows, n_rows_dev,
                                                                       max_rows, dim, (double*)out, ld_out);
    return check_launch("gather_f64");
  }
  set_error("gather_rows: unsupported dtype pair %d->%d", dtype_in, dtype_out);
  return GNS_EINVAL;
}

int gns_gather_rows_mixed(const float* host_table, const float* cache_table, const uint32_t* mask_bits,
                          const int32_t* mask_word_rank, int64_t ld, const int32_t* rows, const int32_t* n_rows_dev,
                          int64_t max_rows, int32_t dim, float* out, int64_t ld_out, void* stream_) {
  if (dim % 4 || ld % 4 || ld_out % 4) {
    set_error("gather_rows_mixed: dim and strides must be multiples of 4");
    return GNS_EINVAL;
  }
  if (max_rows <= 0) return GNS_OK;
  long long want = (max_rows * (dim / 4) + 255) / 256;
  int grid = grid_for(want, (long long)num_sms() * 16);
  gather_mixed_kernel<<<grid, 256, 0, (cudaStream_t)stream_>>>(host_table, cache_table, mask_bits, mask_word_rank, ld,
                                                               rows, n_rows_dev, dim / 4, out, ld_out);
  return check_launch("gather_mixed");
}

int gns_cache_refresh_rows(const float* host_table, int64_t ld, const int32_t* ids, const int64_t* n_dev,
                           int64_t max_rows, int32_t dim, float* cache_table, void* stream_) {
  if (dim % 4 || ld % 4) {
    set_error("cache_refresh_rows: dim and ld must be multiples of 4");
    return GNS_EINVAL;
  }
  if (max_rows <= 0) return GNS_OK;
  long long want = (max_rows * (dim / 4) + 255) / 256;
  int grid = grid_for(want, (long long)num_sms() * 16);
  refresh_rows_kernel<<<grid, 256, 0, (cudaStream_t)stream_>>>(host_table, ld, ids, n_dev, dim / 4, cache_table);
  return check_launch("cache_refresh_rows");
}

int gns_tune(const char* name, int32_t value) {
  if (!strcmp(name, "spmm_narrow")) {
    g_tune_narrow = value;
    return GNS_OK;
  }
  if (!strcmp(name, "gather_tma") && value >= 0 && value <= 2) {
    g_gather_tma = value;
    return GNS_OK;
  }
  if (!strcmp(name, "spmm_wide")) {
    g_tune_wide = value;
    return GNS_OK;
  }
  if (!strcmp(name, "split_g") && (value == 2 || value == 4 || value == 5 || value == 8 || value == 12 || value == 16)) {
    g_split_g = value;
    return GNS_OK;
  }
  if (!strcmp(name, "spmm_bwd") && value >= 0 && value <= 5) {
    g_tune_bwd = value;
    return GNS_OK;
  }
  if (gns_sample_tune(name, value) == GNS_OK) return GNS_OK;
  set_error("unknown tuning knob %s (or value %d out of range)", name, value);
  return GNS_EINVAL;
}

int gns_sum_rows(int32_t dtype, const void* part, int64_t nrows, int64_t ncols, void* out, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (ncols <= 0) return GNS_OK;
  if (dtype == 0)
    colsum_launch<float>((const float*)part, (int)nrows, (int)ncols, (float*)out, stream);
  else
    colsum_final_kernel<double><<<colsum_grid((int)ncols), kColsumWarps * 32, 0, stream>>>(
        (const double*)part, (int)nrows, (int)ncols, (double*)out);
  return check_launch("sum_rows");
}

int gns_spmm_fwd_gather(const float* table, int64_t ld_table, int32_t dim, const gns_block_t* block,
                        const int32_t* dst_ids, int64_t max_dst, int64_t pad_rows, int64_t pad_chunk,
                        int32_t max_row_edges, float* cat, int64_t ld_cat, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (max_dst <= 0 && pad_rows <= 0) return GNS_OK;
  if (dim % 4 || ld_table % 4 || ld_cat % 4 || (uintptr_t)table % 16 || (uintptr_t)cat % 16) {
    set_error("spmm_fwd_gather: dim/strides must be multiples of 4 floats, pointers 16-B aligned");
    return GNS_EINVAL;
  }
  if (ld_table >= (1LL << 30)) {   // the kernels address rows with a 32-bit byte pitch
    set_error("spmm_fwd_gather: row stride %lld floats >= 2^30", (long long)ld_table);
    return GNS_EINVAL;
  }
  const int sms = num_sms();
  long long rows = max_dst > pad_rows ? max_dst : pad_rows;
  BlockView bv = view_of(block);
  const int dv = dim / 4;
#define GNS_CHUNK(R, MB)                                                                                       \
  spmm_fwd_chunk_kernel<false, true, 6, R, MB><<<spmm_grid(spmm_fwd_chunk_kernel<false, true, 6, R, MB>, rows),      \
                                                 kSpmmBlock, 0, stream>>>(table, ld_table, dim, bv, cat, ld_cat,      \
                                                                          pad_rows, block->edge_node, dst_ids,        \
                                                                          pad_chunk)
  if (dv <= 32 && max_row_edges <= 6 && g_tune_narrow >= 2) {
    if (g_tune_narrow == 2) GNS_CHUNK(1, 4);
    else if (g_tune_narrow == 3) GNS_CHUNK(2, 4);
    else if (g_tune_narrow == 4) GNS_CHUNK(1, 5);
    else GNS_CHUNK(1, 6);
    return check_launch("spmm_fwd_gather");
  }
#undef GNS_CHUNK
  if (dv <= 32 && g_tune_narrow >= 1) {
    spmm_fwd_narrow_kernel<false, true><<<spmm_grid(spmm_fwd_narrow_kernel<false, true>, rows), kSpmmBlock, 0,
                                          stream>>>(table, ld_table, dim, bv, cat, ld_cat,
                                                                        pad_rows, block->edge_node, dst_ids,
                                                                        pad_chunk);
    return check_launch("spmm_fwd_gather");
  }
#define GNS_FWDG(CH)                                                                                          \
  do {                                                                                                         \
  spmm_fwd_kernel<float, CH, false, true><<<spmm_grid(spmm_fwd_kernel<float, CH, false, true>, rows), kSpmmBlock, \
                                            0, stream>>>(table, ld_table, dim, bv, cat, ld_cat,             \
                                                         pad_rows, block->edge_node, dst_ids, nullptr, pad_chunk); \
  if (max_row_edges <= 0 || max_row_edges > kRowCap)                                                          \
    spmm_fwd_long_kernel<float, CH, false, true><<<spmm_grid(spmm_fwd_long_kernel<float, CH, false, true>,       \
                                                             rows / 32 + 1), kSpmmBlock, 0, stream>>>(          \
        table, ld_table, dim, bv, cat, ld_cat, block->edge_node, dst_ids, nullptr);  \
  } while (0)
  if (dv <= 32) GNS_FWDG(1);
  else if (dv <= 64) GNS_FWDG(2);
  else GNS_FWDG(4);
#undef GNS_FWDG
  return check_launch("spmm_fwd_gather");
}

size_t gns_relu_bits_size(int64_t rows, int32_t dim) {
  return (size_t)(rows > 0 ? rows : 1) * (size_t)(((dim / 4 + 31) / 32) * 4) * sizeof(uint32_t);
}

int gns_spmm_fwd_bits(const float* h, int64_t ld_h, int32_t dim, const gns_block_t* block, int64_t max_dst,
                      int64_t pad_rows, float* cat, int64_t ld_cat, uint32_t* relu_bits, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (max_dst <= 0 && pad_rows <= 0) return GNS_OK;
  if (dim % 4 || ld_h % 4 || ld_cat % 4 || ld_h >= (1LL << 30)) {
    set_error("spmm_fwd_bits: dim/strides must be multiples of 4 (row stride < 2^30 floats)");
    return GNS_EINVAL;
  }
  long long rows = max_dst > pad_rows ? max_dst : pad_rows;
  BlockView bv = view_of(block);
  const int dv = dim / 4;
  if (g_tune_wide == 2 && dv > 32 && dv <= 128) {
    const long long tasks = rows * ((dv + 31) / 32);
#define GNS_SPLIT(G, B)                                                                                     \
  spmm_fwd_wide_split_kernel<G, true, B><<<spmm_grid(spmm_fwd_wide_split_kernel<G, true, B>, tasks), kSpmmBlock, \
                                           0, stream>>>(h, ld_h, dim, bv, cat, ld_cat, pad_rows, relu_bits)
    // (gns_tune "split_g": neighbour rows in flight per warp / resident CTAs per SM)
    if (g_split_g == 2) GNS_SPLIT(2, 6);
    else if (g_split_g == 5) GNS_SPLIT(4, 5);
    else if (g_split_g == 8) GNS_SPLIT(8, 3);
    else if (g_split_g == 12) GNS_SPLIT(12, 2);
    else if (g_split_g == 16) GNS_SPLIT(16, 2);
    else GNS_SPLIT(4, 4);
#undef GNS_SPLIT
    return check_launch("spmm_fwd_bits");
  }
  if (g_tune_wide && dv > 32 && dv <= 64) {
    spmm_fwd_wide_kernel<2, 4, true><<<spmm_grid(spmm_fwd_wide_kernel<2, 4, true>, rows), kSpmmBlock, 0,
                                       stream>>>(h, ld_h, dim, bv, cat, ld_cat, pad_rows,
                                                                     relu_bits);
    return check_launch("spmm_fwd_bits");
  }
  if (g_tune_wide && dv > 64 && dv <= 128) {
    spmm_fwd_wide_kernel<4, 2, true><<<spmm_grid(spmm_fwd_wide_kernel<4, 2, true>, rows), kSpmmBlock, 0,
                                       stream>>>(h, ld_h, dim, bv, cat, ld_cat, pad_rows,
                                                                     relu_bits);
    return check_launch("spmm_fwd_bits");
  }
#define GNS_FWDB(CH)                                                                                             \
  do {                                                                                                         \
  spmm_fwd_kernel<float, CH, true, false, true><<<spmm_grid(spmm_fwd_kernel<float, CH, true, false, true>, rows), \
                                                  kSpmmBlock, 0, stream>>>(h, ld_h, dim, bv, cat, ld_cat,       \
                                                                                pad_rows, nullptr, nullptr,   \
                                                                                relu_bits);                   \
  spmm_fwd_long_kernel<float, CH, true, false, true><<<spmm_grid(spmm_fwd_long_kernel<float, CH, true, false, true>, \
                                                                 rows / 32 + 1), kSpmmBlock, 0, stream>>>(      \
      h, ld_h, dim, bv, cat, ld_cat, nullptr, nullptr, relu_bits);  \
  } while (0)
  if (dv <= 32) GNS_FWDB(1);
  else if (dv <= 64) GNS_FWDB(2);
  else GNS_FWDB(4);
#undef GNS_FWDB
  return check_launch("spmm_fwd_bits");
}

int gns_spmm_bwd_transposed_bits(const float* dcat, int64_t ld_dcat, int32_t dim, const gns_block_t* block,
                                 int64_t max_dst, int64_t max_src, int64_t max_edges, int64_t pad_rows,
                                 const uint32_t* relu_bits, float* db, float* dh, int64_t ld_dh, void* ws,
                                 size_t ws_bytes, void* stream_) {
  (void)max_dst;
  cudaStream_t stream = (cudaStream_t)stream_;
  BwdWs w;
  size_t need = bwd_ws(max_src, max_edges, dim, ws, ws_bytes, &w);
  if (need > ws_bytes) {
    set_error("spmm_bwd_bits: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  if (dim % 4 || ld_dcat % 4 || ld_dh % 4 || dim > 512 || ld_dcat >= (1LL << 30)) {
    set_error("spmm_bwd_bits: dim/strides must be multiples of 4, dim <= 512, row stride < 2^30");
    return GNS_EINVAL;
  }
  BlockView bv = view_of(block);
  const long long want = ((max_src > pad_rows ? max_src : pad_rows) * 32 + 255) / 256;
  int g2 = 1;
  const int dv = dim / 4;
  // one wave of resident CTAs (<= 8 per SM: the colpart workspace bound)
#define GNS_BWDC(CH, R, B)                                                                                       \
  g2 = resident_grid(spmm_bwd_rows_kernel<CH, R, B>, kSpmmBlock, 0,                                             \
                     want < num_sms() * 8LL ? want : num_sms() * 8LL);                                          \
  spmm_bwd_rows_kernel<CH, R, B><<<g2, kSpmmBlock, 0, stream>>>(dcat, ld_dcat, dim, bv, w.tptr, w.tkeys,         \
                                                                w.self_of, dh, ld_dh, pad_rows,                 \
                                                                db ? (float*)w.colpart : nullptr, relu_bits,    \
                                                                w.twn, w.lr)
  // knob: 1 = R2/4 CTAs per SM, 2 = R2/3, 3 = R4/3, 4 = R4/2, 5 = R8/2
  if (g_tune_bwd > 0 && dv <= 64) {
    if (dv <= 32) {
      GNS_BWDC(1, 4, 4);
    } else if (g_tune_bwd == 1) {
      GNS_BWDC(2, 2, 4);
    } else if (g_tune_bwd == 2) {
      GNS_BWDC(2, 2, 3);
    } else if (g_tune_bwd == 3) {
      GNS_BWDC(2, 4, 3);
    } else if (g_tune_bwd == 4) {
      GNS_BWDC(2, 4, 2);
    } else {
      GNS_BWDC(2, 8, 2);
    }
    GNS_TRY(check_launch("spmm_bwd_bits"));
    // (a last-CTA reduction inside the kernel was measured slower: one SM
    // summing ~300 partial rows is latency-bound; colsum spreads it)
    if (db) colsum_launch<float>((const float*)w.colpart, g2, dim, db, stream);
    return check_launch("spmm_bwd_bits colsum");
  }
#undef GNS_BWDC
#define GNS_BWDB(CH)                                                                                             \
  g2 = resident_grid(spmm_bwd_kernel<float, CH, true>, kSpmmBlock, 0, want < num_sms() * 8LL ? want : num_sms() * 8LL); \
  spmm_bwd_kernel<float, CH, true><<<g2, kSpmmBlock, 0, stream>>>(dcat, ld_dcat, dim, bv, w.tptr, w.tkeys,       \
                                                                  w.self_of, dh, ld_dh, pad_rows, nullptr,       \
                                                                  db ? (float*)w.colpart : nullptr, relu_bits,   \
                                                                  w.twn, w.lr)
  if (dv <= 32) {
    GNS_BWDB(1);
  } else if (dv <= 64) {
    GNS_BWDB(2);
  } else {
    GNS_BWDB(4);
  }
#undef GNS_BWDB
  GNS_TRY(check_launch("spmm_bwd_bits"));
  if (db) colsum_launch<float>((const float*)w.colpart, g2, dim, db, stream);
  return check_launch("spmm_bwd_bits colsum");
}

int gns_spmm_fwd(int32_t dtype, const void* h, int64_t ld_h, int32_t dim, int32_t flags, const gns_block_t* block,
                 int64_t max_dst, int64_t pad_rows, void* cat, int64_t ld_cat, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (max_dst <= 0 && pad_rows <= 0) return GNS_OK;
  const int sms = num_sms();
  long long rows = max_dst > pad_rows ? max_dst : pad_rows;
  BlockView bv = view_of(block);
  const bool relu = flags & GNS_SPMM_RELU_INPUT;
#define GNS_FWD(T, CH, R)                                                                                      \
  do {                                                                                                         \
  spmm_fwd_kernel<T, CH, R><<<spmm_grid(spmm_fwd_kernel<T, CH, R>, rows), kSpmmBlock, 0, stream>>>(                \
      (const T*)h, ld_h, dim, bv, (T*)cat, ld_cat, pad_rows);                                                      \
  spmm_fwd_long_kernel<T, CH, R><<<spmm_grid(spmm_fwd_long_kernel<T, CH, R>, rows / 32 + 1), kSpmmBlock, 0,        \
                                   stream>>>((const T*)h, ld_h, dim, bv, (T*)cat, ld_cat);  \
  } while (0)
  if (dtype == 0) {
    if (dim % 4 || ld_h % 4 || ld_cat % 4) {
      set_error("spmm_fwd(f32): dim/strides must be multiples of 4");
      return GNS_EINVAL;
    }
    const int dv = dim / 4;
    if (dv <= 32 && g_tune_narrow) {
      if (relu)
        spmm_fwd_narrow_kernel<true, false><<<spmm_grid(spmm_fwd_narrow_kernel<true, false>, rows), kSpmmBlock, 0,
                                              stream>>>((const float*)h, ld_h, dim, bv,
                                                                            (float*)cat, ld_cat, pad_rows, nullptr,
                                                                            nullptr);
      else
        spmm_fwd_narrow_kernel<false, false><<<spmm_grid(spmm_fwd_narrow_kernel<false, false>, rows), kSpmmBlock, 0,
                                               stream>>>((const float*)h, ld_h, dim, bv,
                                                                             (float*)cat, ld_cat, pad_rows, nullptr,
                                                                             nullptr);
    } else if (dv <= 32) { if (relu) GNS_FWD(float, 1, true); else GNS_FWD(float, 1, false); }
    else if (dv <= 64) { if (relu) GNS_FWD(float, 2, true); else GNS_FWD(float, 2, false); }
    else { if (relu) GNS_FWD(float, 4, true); else GNS_FWD(float, 4, false); }
  } else {
    if (dim % 2 || ld_h % 2 || ld_cat % 2) {
      set_error("spmm_fwd(f64): dim/strides must be even");
      return GNS_EINVAL;
    }
    const int dv = dim / 2;
    if (dv <= 32) { if (relu) GNS_FWD(double, 1, true); else GNS_FWD(double, 1, false); }
    else { if (relu) GNS_FWD(double, 2, true); else GNS_FWD(double, 2, false); }
  }
#undef GNS_FWD
  return check_launch("spmm_fwd");
}

size_t gns_spmm_bwd_workspace_size(int64_t max_src, int64_t max_edges, int32_t dim) {
  BwdWs w;
  return bwd_ws(max_src, max_edges, dim, nullptr, 0, &w);
}

int gns_block_transpose(const gns_block_t* block, int64_t max_dst, int64_t max_src, int64_t max_edges, int32_t dim,
                        void* ws, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  BwdWs w;
  size_t need = bwd_ws(max_src, max_edges, dim, ws, ws_bytes, &w);
  if (need > ws_bytes) {
    set_error("block_transpose: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  const int sms = num_sms();
  BlockView bv = view_of(block);
  GNS_CUDA(cudaMemsetAsync(w.tcount, 0, (max_src + 1 + kCtrN) * sizeof(int32_t), stream));
  GNS_CUDA(cudaMemsetAsync(w.self_of, 0xff, (max_src + 1) * sizeof(int32_t), stream));
  int g1 = grid_for((max_edges + max_dst + 255) / 256, (long long)sms * 8);
  tcount_kernel<<<g1, 256, 0, stream>>>(bv, w.tcount, w.self_of);
  const unsigned ttiles = (unsigned)((max_src + kTsBlock * kTsItems - 1) / (kTsBlock * kTsItems)) + 1;
  tscan_reduce_kernel<<<ttiles, kTsBlock, 0, stream>>>(bv, w.tcount, (unsigned long long*)w.scan);
  tscan_apply_kernel<<<ttiles, kTsBlock, 0, stream>>>(bv, w.tcount, w.tptr, (unsigned long long*)w.scan);
  tscatter_kernel<<<g1, 256, 0, stream>>>(bv, w.tcount, w.tptr, w.tkeys);
  int g2 = grid_for((max_src + 255) / 256, (long long)sms * 8);   // a warp per 32 rows
  tsort_kernel<<<g2, 256, 0, stream>>>(bv, w.tptr, w.tkeys, w.twn, w.lr);
  // rows longer than a warp's shared slice: a CTA each (a small grid: with
  // no such rows its CTAs exit at once, and 64 KB CTAs must find room next
  // to the training branch's kernels)
  static bool attr = false;
  if (!attr) {
    GNS_CUDA(cudaFuncSetAttribute(tsort_long_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kTsortLongKeys * (int)sizeof(uint64_t)));
    attr = true;
  }
  tsort_long_kernel<<<kTsortLongGrid, kTsortLongThreads, kTsortLongKeys * sizeof(uint64_t), stream>>>(bv, w.tptr, w.tkeys,
                                                                                            w.twn, w.lr);
  return check_launch("block_transpose");
}

int gns_spmm_bwd(int32_t dtype, const void* dcat, int64_t ld_dcat, int32_t dim, const gns_block_t* block,
                 int64_t max_dst, int64_t max_src, int64_t max_edges, int64_t pad_rows, const void* z_mask,
                 void* db, void* dh, int64_t ld_dh, void* ws, size_t ws_bytes, void* stream_) {
  GNS_TRY(gns_block_transpose(block, max_dst, max_src, max_edges, dim, ws, ws_bytes, stream_));
  return gns_spmm_bwd_transposed(dtype, dcat, ld_dcat, dim, block, max_dst, max_src, max_edges, pad_rows, z_mask, db,
                                 dh, ld_dh, ws, ws_bytes, stream_);
}

int gns_spmm_bwd_transposed(int32_t dtype, const void* dcat, int64_t ld_dcat, int32_t dim, const gns_block_t* block,
                            int64_t max_dst, int64_t max_src, int64_t max_edges, int64_t pad_rows,
                            const void* z_mask, void* db, void* dh, int64_t ld_dh, void* ws, size_t ws_bytes,
                            void* stream_) {
  (void)max_dst;
  cudaStream_t stream = (cudaStream_t)stream_;
  BwdWs w;
  size_t need = bwd_ws(max_src, max_edges, dim, ws, ws_bytes, &w);
  if (need > ws_bytes) {
    set_error("spmm_bwd: workspace %zu < %zu", ws_bytes, need);
    return GNS_EINVAL;
  }
  const int VW = dtype == 0 ? 4 : 2;
  if (dim % VW || ld_dcat % VW || ld_dh % VW || ld_dcat >= (1LL << 29)) {
    set_error("spmm_bwd: dim/strides must be multiples of %d (row stride < 2^29)", VW);
    return GNS_EINVAL;
  }
  const int sms = num_sms();
  BlockView bv = view_of(block);
  int g2 = grid_for(((max_src > pad_rows ? max_src : pad_rows) * 32 + 255) / 256, (long long)sms * 8);
  const int dv = dim / VW;
  if (db && dv > 128) {
    set_error("spmm_bwd: fused bias gradient needs dim <= %d", 128 * VW);
    return GNS_EINVAL;
  }
#define GNS_BWD(T, CH)                                                                                       \
  spmm_bwd_kernel<T, CH><<<g2, kSpmmBlock, 0, stream>>>((const T*)dcat, ld_dcat, dim, bv, w.tptr, w.tkeys, \
                                                        w.self_of, (T*)dh, ld_dh, pad_rows, (const T*)z_mask,  \
                                                        db ? (T*)w.colpart : nullptr, nullptr, w.twn, w.lr)
  if (dtype == 0) {
    if (dv <= 32) GNS_BWD(float, 1);
    else if (dv <= 64) GNS_BWD(float, 2);
    else GNS_BWD(float, 4);
  } else {
    if (dv <= 32) GNS_BWD(double, 1);
    else if (dv <= 64) GNS_BWD(double, 2);
    else GNS_BWD(double, 4);
  }
#undef GNS_BWD
  GNS_TRY(check_launch("spmm_bwd"));
  if (db) {
    if (dtype == 0)
      colsum_launch<float>((const float*)w.colpart, g2, dim, (float*)db, stream);
    else
      colsum_final_kernel<double><<<colsum_grid(dim), kColsumWarps * 32, 0, stream>>>((const double*)w.colpart, g2, dim,
                                                                     (double*)db);
  }
  return check_launch("spmm_bwd colsum");
}

// rows per partial block: 64 for float32 (more CTAs, short per-thread add
// chains), 512 for the float64 parity mode
constexpr int kDenseRpbF32 = 64, kDenseRpbF64 = 512;

size_t gns_dense_bwd_workspace_size(int64_t max_rows, int32_t ncols) {
  return (size_t)((max_rows + kDenseRpbF32 - 1) / kDenseRpbF32 + 1) * (size_t)ncols * 8 + 256;
}

int gns_dense_bwd_bias(int32_t dtype, const void* dh, const void* z, int64_t ld, const int32_t* n_dev,
                       int64_t n_rows, int32_t ncols, void* dz, void* db, void* ws, size_t ws_bytes,
                       void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  const int rpb = dtype == 0 ? kDenseRpbF32 : kDenseRpbF64;
  const int nblocks = (int)((n_rows + rpb - 1) / rpb);
  if (ws_bytes < gns_dense_bwd_workspace_size(n_rows, ncols)) {
    set_error("dense_bwd_bias: workspace too small");
    return GNS_EINVAL;
  }
  if (nblocks == 0) {
    GNS_CUDA(cudaMemsetAsync(db, 0, (size_t)ncols * (dtype == 0 ? 4 : 8), stream));
    return GNS_OK;
  }
  dim3 grid(nblocks, (ncols + 63) / 64);
  if (dtype == 0) {
    dense_bwd_partial_kernel<float><<<grid, 256, 0, stream>>>((const float*)dh, (const float*)z, ld, n_dev, n_rows,
                                                              ncols, (float*)dz, (float*)ws, rpb);
    colsum_launch<float>((const float*)ws, nblocks, ncols, (float*)db, stream);
  } else {
    dense_bwd_partial_kernel<double><<<grid, 256, 0, stream>>>((const double*)dh, (const double*)z, ld, n_dev,
                                                               n_rows, ncols, (double*)dz, (double*)ws, rpb);
    colsum_final_kernel<double><<<colsum_grid(ncols), kColsumWarps * 32, 0, stream>>>((const double*)ws, nblocks, ncols,
                                                                     (double*)db);
  }
  return check_launch("dense_bwd_bias");
}

int gns_softmax_xent(int32_t dtype, const void* logits, int64_t ld, const int32_t* n_dev, int64_t max_rows,
                     int64_t pad_rows, int32_t num_classes, const int32_t* labels, const int32_t* targets,
                     void* grad_out, double* loss_out, void* ws, size_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if ((size_t)max_rows * sizeof(double) > ws_bytes) {
    set_error("softmax_xent: workspace %zu < %zu", ws_bytes, (size_t)max_rows * 8);
    return GNS_EINVAL;
  }
  double* row_loss = (double*)ws;
  const int sms = num_sms();
  int grid = grid_for(((max_rows > pad_rows ? max_rows : pad_rows) * 32 + 255) / 256, (long long)sms * 8);
  if (dtype == 0)
    xent_kernel<float><<<grid, 256, 0, stream>>>((const float*)logits, ld, n_dev, num_classes, labels, targets,
                                                 (float*)grad_out, row_loss, pad_rows);
  else
    xent_kernel<double><<<grid, 256, 0, stream>>>((const double*)logits, ld, n_dev, num_classes, labels, targets,
                                                  (double*)grad_out, row_loss, pad_rows);
  mean_kernel<<<1, 1024, 0, stream>>>(row_loss, n_dev, loss_out);
  return check_launch("softmax_xent");
}

// <= 64 CTAs: the last CTA's fixed-order column sums over the CTA partials
// stay a few round trips (each warp takes several rows instead)
static int xent_bias_grid(int64_t max_rows, int64_t pad_rows) {
  return grid_for(((max_rows > pad_rows ? max_rows : pad_rows) * 32 + 255) / 256, 64);
}

size_t gns_softmax_xent_bias_workspace_size(int64_t max_rows, int64_t pad_rows, int32_t num_classes) {
  Workspace w(nullptr, 0);
  w.take<double>(max_rows + 1);
  w.take<double>((size_t)xent_bias_grid(max_rows, pad_rows) * (num_classes > 0 ? num_classes : 1));
  w.take<unsigned>(1);
  return w.off;
}

int gns_softmax_xent_bias(int32_t dtype, const void* logits, int64_t ld, const int32_t* n_dev, int64_t max_rows,
                          int64_t pad_rows, int32_t num_classes, const int32_t* labels, const int32_t* targets,
                          void* grad_out, double* loss_out, void* grad_bias, void* ws, size_t ws_bytes,
                          void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (num_classes < 1 || num_classes > 32 * kXentCh) {
    set_error("softmax_xent_bias: num_classes %d outside [1, %d]", num_classes, 32 * kXentCh);
    return GNS_EINVAL;
  }
  if (ws_bytes < gns_softmax_xent_bias_workspace_size(max_rows, pad_rows, num_classes)) {
    set_error("softmax_xent_bias: workspace %zu < %zu", ws_bytes,
              gns_softmax_xent_bias_workspace_size(max_rows, pad_rows, num_classes));
    return GNS_EINVAL;
  }
  Workspace w(ws, ws_bytes);
  double* row_loss = w.take<double>(max_rows + 1);
  const int grid = xent_bias_grid(max_rows, pad_rows);
  void* partial = (void*)w.take<double>((size_t)grid * num_classes);
  unsigned* ticket = w.take<unsigned>(1);
  // the ticket must start at 0: the caller zeroes the workspace once (every
  // launch leaves it at 0)
  if (dtype == 0)
    xent_bias_kernel<float><<<grid, 256, 0, stream>>>((const float*)logits, ld, n_dev, num_classes, labels, targets,
                                                      (float*)grad_out, loss_out, (float*)grad_bias, row_loss,
                                                      (float*)partial, ticket, pad_rows);
  else
    xent_bias_kernel<double><<<grid, 256, 0, stream>>>((const double*)logits, ld, n_dev, num_classes, labels,
                                                       targets, (double*)grad_out, loss_out, (double*)grad_bias,
                                                       row_loss, (double*)partial, ticket, pad_rows);
  return check_launch("softmax_xent_bias");
}

int gns_adam(int32_t dtype, void* params, const void* grads, void* m, void* v, int64_t n, double lr, double beta1,
             double beta2, double eps, int64_t step, double grad_scale, void* stream_) {
  if (n <= 0) return GNS_OK;
  double bc1 = 1.0 - pow(beta1, (double)step), bc2 = 1.0 - pow(beta2, (double)step);
  int grid = grid_for((n + 255) / 256, (long long)num_sms() * 8);
  cudaStream_t stream = (cudaStream_t)stream_;
  if (dtype == 0)
    adam_kernel<float><<<grid, 256, 0, stream>>>((float*)params, (const float*)grads, (float*)m, (float*)v, n,
                                                 (float)lr, (float)beta1, (float)beta2, (float)eps, (float)bc1,
                                                 (float)bc2, (float)grad_scale);
  else
    adam_kernel<double><<<grid, 256, 0, stream>>>((double*)params, (const double*)grads, (double*)m, (double*)v, n,
                                                  lr, beta1, beta2, eps, bc1, bc2, grad_scale);
  return check_launch("adam");
}

int gns_adam_dev(int32_t dtype, void* params, const void* grads, void* m, void* v, int64_t n, double lr,
                 double beta1, double beta2, double eps, int64_t* step_dev, double grad_scale, void* stream_) {
  if (n <= 0) return GNS_OK;
  int grid = grid_for((n + 255) / 256, (long long)num_sms() * 8);
  cudaStream_t stream = (cudaStream_t)stream_;
  if (dtype == 0)
    adam_dev_kernel<float><<<grid, 256, 0, stream>>>((float*)params, (const float*)grads, (float*)m, (float*)v, n,
                                                     lr, beta1, beta2, eps, step_dev, (float)grad_scale);
  else
    adam_dev_kernel<double><<<grid, 256, 0, stream>>>((double*)params, (const double*)grads, (double*)m, (double*)v,
                                                      n, lr, beta1, beta2, eps, step_dev, grad_scale);
  return check_launch("adam_dev");
}

}  // extern "C"
