// fp64_probe.cu -- developer probe (not part of the product): the DFMA
// throughput this B200 sustains, to bound the block SBGEMV-N at K = 8 (32
// DFMAs per complex operator element). Three loops per CTA size:
//   reg  : 16 independent DFMA chains per thread, operands in registers
//   lds  : the block kernel's column step -- one LDS.128 of a (per thread), 8
//          LDS.128 broadcasts of x, 32 DFMAs into 32 accumulators
//   lds2 : the two-row step -- 2 LDS.128 of a, 4 of x, 32 DFMAs
// Prints DFMA per clock per SM (clock from clock64 on SM 0's CTA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_probe tools/fp64_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void k_reg(int iters, double* out, long long* clk) {
  double a[16];
  const double m = 1.0000001 + threadIdx.x * 1e-12, c = 1e-9;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = i;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], m, c);
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = t1 - t0;
}

// 16 accumulators, operands from 8 distinct registers (the outer-product step
// without the shared loads): two register-file operand reads per DFMA
__global__ void k_reg2(int iters, double* out, long long* clk) {
  double a[16], pv[4], qv[4];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = i;
#pragma unroll
  for (int i = 0; i < 4; ++i) pv[i] = 1.0 + (threadIdx.x + i) * 1e-9, qv[i] = 1.0 - i * 1e-9;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(pv[i & 3], qv[i >> 2], a[i]);
#pragma unroll
    for (int i = 0; i < 4; ++i) pv[i] = pv[i] * 0.999999999;  // keep p live-varying (4 DMULs per 16 DFMAs)
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = t1 - t0;
}

// float -> double conversions (F2F.F64.F32) feeding DFMAs: the 'm' SBGEMV's
// per-element cost (4 conversions + 4 DFMAs per complex MAC)
__global__ void k_f2f(int iters, double* out, long long* clk) {
  float f[8];
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = 1.0f + (threadIdx.x + i) * 1e-7f, a[i] = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma((double)f[i], (double)f[(i + 1) & 7], a[i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = __int_as_float(__float_as_int(f[i]) ^ 1);  // keep the inputs varying (ALU)
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = t1 - t0;
}

template <int ROWS2>
__global__ void k_lds(int iters, double* out, long long* clk) {
  __shared__ double2 xs[8 * 64];
  __shared__ double2 as[1024];
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) xs[i] = make_double2(i * 1e-3, 1.0 - i * 1e-3);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) as[i] = make_double2(i * 1e-4, 1.0 + i * 1e-4);
  __syncthreads();
  double rr[8], ii[8], ri[8], ir[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) rr[k] = ii[k] = ri[k] = ir[k] = 0;
  const int r = threadIdx.x % 100;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int j = it & 63;
    if (ROWS2) {
      const double2 a = as[(r + j) & 1023], b = as[(r + 50 + j) & 1023];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 x = xs[k * 64 + j];
        rr[k] = fma(a.x, x.x, rr[k]);
        ii[k] = fma(a.x, x.y, ii[k]);
        ri[k] = fma(b.x, x.x, ri[k]);
        ir[k] = fma(b.x, x.y, ir[k]);
        rr[k] = fma(-a.y, x.y, rr[k]);
        ii[k] = fma(a.y, x.x, ii[k]);
        ri[k] = fma(-b.y, x.y, ri[k]);
        ir[k] = fma(b.y, x.x, ir[k]);
      }
    } else {
      const double2 a = as[(r + j) & 1023];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double2 x = xs[k * 64 + j];
        rr[k] = fma(a.x, x.x, rr[k]);
        ii[k] = fma(a.y, x.y, ii[k]);
        ri[k] = fma(a.x, x.y, ri[k]);
        ir[k] = fma(a.y, x.x, ir[k]);
      }
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += rr[k] + ii[k] + ri[k] + ir[k];
  if (s == 1.2345) out[0] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) *clk = t1 - t0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* clk;
  cudaMalloc(&out, 8);
  cudaMalloc(&clk, 8);
  const int iters = 20000;
  const int threads[] = {128, 256, 416, 512, 704, 1024};
  for (int kind = 0; kind < 5; ++kind)
    for (int T : threads) {
      for (int w = 0; w < 2; ++w) {
        if (kind == 0) k_reg<<<nsm, T>>>(iters, out, clk);
        else if (kind == 1) k_lds<0><<<nsm, T>>>(iters, out, clk);
        else if (kind == 2) k_lds<1><<<nsm, T>>>(iters, out, clk);
        else if (kind == 3) k_reg2<<<nsm, T>>>(iters, out, clk);
        else k_f2f<<<nsm, T>>>(iters, out, clk);
      }
      cudaDeviceSynchronize();
      long long c = 0;
      cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
      const double dfma = (double)iters * (kind == 0 ? 16 : kind == 3 ? 20 : kind == 4 ? 8 : 32) * T;  // per CTA
      printf("%-4s %4d threads/SM: %6.2f DFMA/clk/SM (%s)\n",
             kind == 0 ? "reg" : kind == 1 ? "lds" : kind == 2 ? "lds2" : kind == 3 ? "reg2" : "f2f (DFMA with 2 F2F)", T,
             dfma / (double)c, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
