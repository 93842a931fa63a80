// Gather-kernel variants, round 2: load cache hints, unroll depth, grid size,
// and a warp-per-row-group layout, on a papers100M-sized table (111M x 128
// fp32), 285K sorted random rows (the bench's per-step input-node count).
// argv[2] = "dirty": flush L2 with a 256 MB memset (L2 full of dirty lines
// when the gather starts, as inside a training step); default: read-only flush.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gp2 scripts/gather_probe2.cu && /tmp/gp2 [n] [dirty]
// (add -DWITH_LIBGNS -Lpaper_2106_06150_b200 -lgns -Xlinker -rpath=$PWD/paper_2106_06150_b200 to also time
// the library's gns_gather_rows on the same buffers)
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#ifdef WITH_LIBGNS
#include "../include/gns.h"
#endif
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

// load modes: 0 = nc + L1::no_allocate; 1 = + L2::256B prefetch; 2 = + L2 evict_first policy
template <int LM>
__device__ __forceinline__ float4 ld(const float4* p, uint64_t pol) {
  float4 r;
  if (LM == 0)
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  else if (LM == 1)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p), "l"(pol));
  return r;
}
// store modes: 0 plain; 1 .cs; 2 evict_last policy
template <int SM_>
__device__ __forceinline__ void st(float4* p, float4 v, uint64_t pol) {
  if (SM_ == 0) *p = v;
  else if (SM_ == 1)
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
  else
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w), "l"(pol));
}

template <int U, int LM, int SMODE>
__global__ void g_flat(const float* __restrict__ t, const int* __restrict__ rows, int64_t n, int dim4,
                       float* __restrict__ out) {
  uint64_t pf = 0, pl = 0;
  if (LM == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  if (SMODE == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  const int64_t total = n * dim4, stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < total; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t ii = i + u * stride, r = ii / dim4;
      int c = (int)(ii - r * dim4);
      v[u] = ld<LM>(reinterpret_cast<const float4*>(t + (int64_t)__ldg(rows + r) * dim4 * 4) + c, pf);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) st<SMODE>(reinterpret_cast<float4*>(out) + i + u * stride, v[u], pl);
  }
  for (; i < total; i += stride) {
    int64_t r = i / dim4;
    int c = (int)(i - r * dim4);
    st<SMODE>(reinterpret_cast<float4*>(out) + i,
              ld<LM>(reinterpret_cast<const float4*>(t + (int64_t)rows[r] * dim4 * 4) + c, pf), pl);
  }
}

// warp-contiguous: each warp owns G consecutive rows per iteration (dim4 == 32:
// one lane per 16-B chunk), loads all G rows, then stores them.
template <int G, int LM, int SMODE = 0>
__global__ void g_warp(const float* __restrict__ t, const int* __restrict__ rows, int64_t n, float* __restrict__ out) {
  uint64_t pf = 0, pl = 0;
  if (LM == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  if (SMODE == 2) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = warp * G; r0 < n; r0 += nw * G) {
    int myrow = lane < G && r0 + lane < n ? __ldg(rows + r0 + lane) : 0;
    float4 v[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      int src = __shfl_sync(0xffffffffu, myrow, g);
      if (r0 + g < n) v[g] = ld<LM>(reinterpret_cast<const float4*>(t + (int64_t)src * 128) + lane, pf);
    }
#pragma unroll
    for (int g = 0; g < G; ++g)
      if (r0 + g < n) st<SMODE>(reinterpret_cast<float4*>(out + (r0 + g) * 128) + lane, v[g], pl);
  }
}

int main(int argc, char** argv) {
  const int64_t N = 111000000, D = 128, n = argc > 1 ? atol(argv[1]) : 285000;
  const bool dirty = argc > 2 && !strcmp(argv[2], "dirty");
  const int dim4 = D / 4;
  float* t;
  CK(cudaMalloc(&t, N * D * 4));
  CK(cudaMemset(t, 1, N * D * 4));
  std::mt19937_64 rng(1);
  std::vector<int> h(n);
  for (auto& x : h) x = (int)(rng() % N);
  std::sort(h.begin(), h.end());
  h.erase(std::unique(h.begin(), h.end()), h.end());
  const int64_t m = (int64_t)h.size();
  int* rows;
  float* out;
  CK(cudaMalloc(&rows, m * 4));
  CK(cudaMalloc(&out, m * D * 4));
  CK(cudaMemcpy(rows, h.data(), m * 4, cudaMemcpyHostToDevice));
  float* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  float* scratch;
  CK(cudaMalloc(&scratch, 512 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)m * (2.0 * D * 4 + 4);
  auto run = [&](const char* name, auto launch) {
    float best = 1e9, tot = 0;
    for (int it = 0; it < 22; ++it) {
      if (dirty) {
        CK(cudaMemsetAsync(flush, it, 256 << 20));
      } else {
        // evict the table/output from L2 without leaving dirty lines: read-only flush
        CK(cudaMemcpyAsync(scratch, flush, 256 << 20, cudaMemcpyDeviceToDevice));
        CK(cudaMemcpyAsync(flush, scratch, 8 << 20, cudaMemcpyDeviceToDevice));
      }
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it >= 2) { best = std::min(best, ms); tot += ms; }
    }
    CK(cudaGetLastError());
    printf("%-40s best %7.2f us  avg %7.2f us  %7.1f GB/s (avg)\n", name, best * 1e3, tot / 20 * 1e3,
           bytes / (tot / 20 / 1e3) / 1e9);
  };
  printf("rows %lld (unique of %lld)\n", (long long)m, (long long)n);
  char nm[96];
#define FLAT(U, LM, SMODE, GM, BS)                                                           \
  snprintf(nm, 96, "flat U%d ld%d st%d grid=%dxSM blk%d", U, LM, SMODE, GM, BS);            \
  run(nm, [&] { g_flat<U, LM, SMODE><<<sms * GM, BS>>>(t, rows, m, dim4, out); });
  FLAT(4, 0, 0, 16, 256)
  FLAT(2, 0, 0, 8, 256)
  FLAT(4, 0, 1, 16, 256)
  FLAT(4, 2, 1, 16, 256)
  FLAT(4, 0, 0, 6, 256)
  FLAT(2, 0, 0, 32, 128)
#define WARP(G, LM, GM, SMODE)                                                      \
  snprintf(nm, 96, "warp G%d ld%d st%d grid=%dxSM", G, LM, SMODE, GM);             \
  run(nm, [&] { g_warp<G, LM, SMODE><<<sms * GM, 256>>>(t, rows, m, out); });
  WARP(1, 0, 8, 0)
  WARP(2, 0, 8, 0)
  WARP(2, 0, 4, 0)
  WARP(2, 0, 16, 0)
  WARP(4, 0, 8, 0)
  WARP(2, 0, 8, 1)
  WARP(2, 2, 8, 1)
  WARP(2, 1, 8, 0)
  WARP(2, 2, 8, 0)
  WARP(2, 0, 8, 2)
  WARP(4, 0, 4, 1)
#ifdef WITH_LIBGNS
  run("libgns gns_gather_rows", [&] { gns_gather_rows(t, D, 0, rows, nullptr, m, (int)D, out, D, 0, nullptr); });
#endif
  run("cudaMemcpyAsync D2D (ref)", [&] { cudaMemcpyAsync(out, t, m * D * 4, cudaMemcpyDeviceToDevice); });
  return 0;
}
