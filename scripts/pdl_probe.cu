// Launch-gap probe: a CUDA graph of N dependent small kernels (each a
// 148-CTA grid doing a dependent global read + write), with plain stream
// ordering vs programmatic dependent launch (PDL: griddepcontrol.wait at the
// top of each kernel, launch_dependents right after).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/pdl scripts/pdl_probe.cu && /tmp/pdl
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void step_kernel(int* buf, int n, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = buf[(i * 7 + 1) % n] + 1;
}

int main() {
  const int N = 40, n = 148 * 256;
  int* buf;
  cudaMalloc(&buf, n * 4);
  cudaMemset(buf, 0, n * 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int k = 0; k < N; ++k) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, step_kernel, buf, n, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int r = 0; r < 50; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.2f us per kernel (%d-kernel chain)  err=%s\n", pdl ? "PDL  " : "plain", ms * 1e3 / 50 / N, N,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
