// jmajor_probe.cu -- developer probe (not part of the product): can the F*
// SBGEMV stream its operator column-group-major ("j-major": for a group of C
// columns, every bin's C x m block in turn, 8 MB apart) as fast as the flat
// bin-major stream? That order would let one CTA finish all bins of its series
// and run their c2r in the same kernel. Bare TMA ring, no math: GB/s of operator
// bytes, with and without the per-bin x_b (1.6 KB, L2-resident) copy per stage.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/jmajor_probe tools/jmajor_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                   sa(b)),
               "r"(ph));
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          sa(dst)),
      "l"(src), "r"(bytes), "r"(sa(b)), "l"(pol)
      : "memory");
}

// A: nb bins of (m x n) column-major complex128 (col = m*16 bytes). Group g =
// columns [g*C, (g+1)*C); stage = one bin's C columns (C*m*16 bytes) [+ x_b].
__global__ void __launch_bounds__(288) k_jmajor(const unsigned char* __restrict__ A, const unsigned char* __restrict__ X,
                                                int nb, int n, int m, int C, int NS, int with_x, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 32;
  unsigned char* ring = sm + 512;
  const int NC = blockDim.x - 32;
  const long col = (long)m * 16, SB = C * col + (with_x ? col : 0);
  const int groups = n / C;
  if (threadIdx.x == 0)
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC / 32);
    }
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  double acc = 0;
  long i = 0;
  if (threadIdx.x == NC) {
    uint64_t pf, pl;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
    for (int g = blockIdx.x; g < groups; g += gridDim.x)
      for (int b = 0; b < nb; ++b, ++i) {
        const int s = i % NS;
        if (i >= NS) mbar_wait(empty + s, ((i / NS) - 1) & 1);
        mbar_expect(full + s, (unsigned)SB);
        unsigned char* dst = ring + (long)s * SB;
        bulk(dst, A + ((long)b * n + (long)g * C) * col, (unsigned)(C * col), full + s, pf);
        if (with_x) bulk(dst + C * col, X + (long)b * col, (unsigned)col, full + s, pl);
      }
  } else if (threadIdx.x < NC) {
    for (int g = blockIdx.x; g < groups; g += gridDim.x)
      for (int b = 0; b < nb; ++b, ++i) {
        const int s = i % NS;
        mbar_wait(full + s, (i / NS) & 1);
        if (threadIdx.x % 32 == 0) acc += reinterpret_cast<const double*>(ring + (long)s * SB)[threadIdx.x];
        __syncwarp();
        if (threadIdx.x % 32 == 0)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(empty + s)));
      }
  }
  if (acc == 12345.678) *out = acc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int nb = 1001, n = 5000, m = 100;
  const long bytes = (long)nb * n * m * 16;
  unsigned char *A, *X;
  double* out;
  cudaMalloc(&A, bytes);
  cudaMalloc(&X, (long)nb * m * 16);
  cudaMalloc(&out, 8);
  cudaMemset(A, 0, bytes);
  cudaMemset(X, 0, (long)nb * m * 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int C, NS, per_sm, with_x; };
  const Cfg cfgs[] = {{4, 16, 2, 0}, {4, 16, 2, 1}, {8, 8, 2, 0}, {8, 8, 2, 1}, {8, 12, 1, 1}, {16, 6, 1, 1},
                      {4, 24, 1, 1}, {2, 32, 2, 1}};
  for (const Cfg& c : cfgs) {
    const long col = (long)m * 16, SB = c.C * col + (c.with_x ? col : 0);
    const size_t smem = 512 + (size_t)SB * c.NS;
    if (smem > 227 * 1024) continue;
    cudaFuncSetAttribute(k_jmajor, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = nsm * c.per_sm;
    for (int w = 0; w < 2; ++w) k_jmajor<<<grid, 288, smem>>>(A, X, nb, n, m, c.C, c.NS, c.with_x, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_jmajor<<<grid, 288, smem>>>(A, X, nb, n, m, c.C, c.NS, c.with_x, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("j-major C=%2d cols (%5ld B/stage) x %2d stages x %d CTA/SM, x_b %d: %7.0f GB/s of operator (%.3f ms)\n",
           c.C, SB, c.NS, c.per_sm, c.with_x, 5.0 * bytes / (ms * 1e6), ms / 5);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
