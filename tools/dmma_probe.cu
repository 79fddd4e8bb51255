// dmma_probe.cu -- how fast does one B200 SM run fp64 mma.sync (DMMA,
// m8n8k4, operands in registers) compared with DFMA? Decides whether the
// block NoTrans SBGEMV (K = 8 right-hand sides, FP64-issue bound with DFMA,
// DESIGN.md §9.1) can move its complex MACs onto the FP64 tensor path.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/dmma_probe tools/dmma_probe.cu
//   build/dmma_probe            -> DFMA/clk/SM equivalents for DMMA and DFMA
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(int iters, double* out) {
  double c[CH][2];
  double a = threadIdx.x * 1e-9, b = blockIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) dmma(c[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
__global__ void k_dfma(int iters, double* out) {
  double c[CH];
  double a = threadIdx.x * 1e-9, b = blockIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < CH; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) c[i] = fma(a, b, c[i]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);  // kHz
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    auto run = [&](auto kern, double fma_per_thread_iter, const char* name) {
      kern<<<sms, warps * 32>>>(100, out);
      cudaEventRecord(e0);
      kern<<<sms, warps * 32>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = (double)sms * warps * 32 * iters * fma_per_thread_iter;
      const double per_clk_sm = fmas / (ms * 1e-3) / sms / (clk * 1e3);
      printf("%-10s warps/SM %2d: %.3f ms, %.1f DFMA-equivalents/clk/SM (at the %d MHz attribute clock)\n", name,
             warps, ms, per_clk_sm, clk / 1000);
    };
    // one m8n8k4 = 256 FMAs per warp = 8 per thread
    run(k_dmma<4>, 4 * 8.0, "DMMA x4");
    run(k_dmma<8>, 8 * 8.0, "DMMA x8");
    run(k_dfma<8>, 8.0, "DFMA x8");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
