// Gather-kernel variants on a papers100M-sized table (111M x 128 fp32):
// out[i,:] = table[rows[i],:] for 285K sorted random rows.  Standalone probe:
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/gp scripts/gather_probe.cu && /tmp/gp
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <random>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e = (x);                                                             \
    if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } \
  } while (0)

__device__ __forceinline__ float4 ldnc(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stcs(float4* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

template <int U, bool CS>
__global__ void g_flat(const float* __restrict__ t, const int* __restrict__ rows, int64_t n, int dim4,
                       float* __restrict__ out) {
  const int64_t total = n * dim4, stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < total; i += U * stride) {
    float4 v[U];
    int64_t o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t ii = i + u * stride, r = ii / dim4;
      int c = (int)(ii - r * dim4);
      v[u] = ldnc(reinterpret_cast<const float4*>(t + (int64_t)__ldg(rows + r) * dim4 * 4) + c);
      o[u] = ii;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (CS) stcs(reinterpret_cast<float4*>(out) + o[u], v[u]);
      else reinterpret_cast<float4*>(out)[o[u]] = v[u];
    }
  }
  for (; i < total; i += stride) {
    int64_t r = i / dim4;
    int c = (int)(i - r * dim4);
    reinterpret_cast<float4*>(out)[i] = ldnc(reinterpret_cast<const float4*>(t + (int64_t)rows[r] * dim4 * 4) + c);
  }
}

// bulk-copy (TMA engine, cp.async.bulk) staging: per CTA, S rows per stage are
// copied global->smem by one thread (one bulk copy per row), then the stage is
// written back as one contiguous bulk store smem->global.
template <int S, int STAGES>
__global__ void __launch_bounds__(32) g_bulk(const float* __restrict__ t, const int* __restrict__ rows, int64_t n,
                                             int row_bytes, float* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bar[STAGES];
  const int64_t nchunks = (n + S - 1) / S;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      uint32_t a = (uint32_t)__cvta_generic_to_shared(&bar[s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  uint32_t phase[STAGES] = {0};
  int k = 0;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x, ++k) {
    const int s = k % STAGES;
    unsigned char* buf = smem + (size_t)s * S * row_bytes;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(buf);
    const uint32_t ba = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    // the store that last read this stage must have drained
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(STAGES - 1));
    const int64_t r0 = ch * S;
    const int cnt = (int)((n - r0) < S ? (n - r0) : S);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(cnt * row_bytes));
    for (int j = 0; j < cnt; ++j) {
      const float* src = t + (int64_t)rows[r0 + j] * (row_bytes / 4);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sb + j * row_bytes),
                   "l"(src), "r"(row_bytes), "r"(ba)
                   : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"(ba), "r"(phase[s]));
    phase[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                     (unsigned char*)out + r0 * row_bytes),
                 "r"(sb), "r"(cnt * row_bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;");
  }
  asm volatile("cp.async.bulk.wait_group 0;");
}

int main() {
  const int64_t N = 111000000, D = 128, n = 285000;
  const int dim4 = D / 4;
  float* t;
  CK(cudaMalloc(&t, N * D * 4));
  CK(cudaMemset(t, 1, N * D * 4));
  std::mt19937_64 rng(1);
  std::vector<int> h(n);
  for (auto& x : h) x = (int)(rng() % N);
  std::sort(h.begin(), h.end());
  int* rows;
  float* out;
  CK(cudaMalloc(&rows, n * 4));
  CK(cudaMalloc(&out, n * D * 4));
  CK(cudaMemcpy(rows, h.data(), n * 4, cudaMemcpyHostToDevice));
  float* flush;
  CK(cudaMalloc(&flush, 512 << 20));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = (double)n * (2.0 * D * 4 + 4);
  auto run = [&](const char* name, auto launch) {
    float best = 1e9, tot = 0;
    for (int it = 0; it < 12; ++it) {
      CK(cudaMemset(flush, it, 512 << 20));
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (it >= 2) { best = std::min(best, ms); tot += ms; }
    }
    CK(cudaGetLastError());
    printf("%-34s best %7.2f us  avg %7.2f us  %7.1f GB/s (avg)\n", name, best * 1e3, tot / 10 * 1e3,
           bytes / (tot / 10 / 1e3) / 1e9);
  };
  for (int gm : {8, 16, 32}) {
    char nm[64];
    int grid = sms * gm;
    snprintf(nm, 64, "flat U4 grid=%dxSM", gm);
    run(nm, [&] { g_flat<4, false><<<grid, 256>>>(t, rows, n, dim4, out); });
    snprintf(nm, 64, "flat U8 grid=%dxSM", gm);
    run(nm, [&] { g_flat<8, false><<<grid, 256>>>(t, rows, n, dim4, out); });
    snprintf(nm, 64, "flat U8 .cs grid=%dxSM", gm);
    run(nm, [&] { g_flat<8, true><<<grid, 256>>>(t, rows, n, dim4, out); });
  }
  {
    constexpr int S = 32, ST = 4;
    size_t sm = (size_t)S * ST * D * 4;
    CK(cudaFuncSetAttribute(g_bulk<S, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (int cps : {2, 4, 6}) {
      char nm[64];
      snprintf(nm, 64, "bulk S=%d ST=%d %d CTA/SM", S, ST, cps);
      run(nm, [&] { g_bulk<S, ST><<<sms * cps, 32, sm>>>(t, rows, n, D * 4, out); });
    }
  }
  {
    constexpr int S = 16, ST = 4;
    size_t sm = (size_t)S * ST * D * 4;
    CK(cudaFuncSetAttribute(g_bulk<S, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (int cps : {4, 8, 12}) {
      char nm[64];
      snprintf(nm, 64, "bulk S=%d ST=%d %d CTA/SM", S, ST, cps);
      run(nm, [&] { g_bulk<S, ST><<<sms * cps, 32, sm>>>(t, rows, n, D * 4, out); });
    }
  }
  // plain copy reference (same bytes, sequential)
  run("cudaMemcpyAsync D2D (ref)", [&] { cudaMemcpyAsync(out, t, n * D * 4, cudaMemcpyDeviceToDevice); });
  return 0;
}
