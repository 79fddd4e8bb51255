// Read-bandwidth ceiling probe (developer tool, not part of the product):
// how fast can a B200 stream N bytes from HBM with (a) 16-byte vector loads
// summed into a register and (b) a cp.async.bulk ring into shared memory
// (the SBGEMV's access pattern with no math)? Prints GB/s for 8 GB and 48 GB.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/read_ceiling tools/read_ceiling.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void __launch_bounds__(512) k_ldg(const double2* __restrict__ a, long n, double* out) {
  double s = 0;
  const long stride = (long)gridDim.x * blockDim.x;
  long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const double2 v0 = __ldcs(a + i), v1 = __ldcs(a + i + stride), v2 = __ldcs(a + i + 2 * stride),
                  v3 = __ldcs(a + i + 3 * stride);
    s += v0.x + v1.x + v2.x + v3.x + v0.y + v1.y + v2.y + v3.y;
  }
  for (; i < n; i += stride) s += a[i].x + a[i].y;
  if (s == 12345.678) *out = s;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
          (unsigned)__cvta_generic_to_shared(b)),
      "r"(ph));
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* b, int pol) {
  if (pol) {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            (unsigned)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b)), "l"(p)
        : "memory");
  } else {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (unsigned)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
                 : "memory");
  }
}

// One CTA streams a contiguous piece through an NS-deep ring of SB-byte stages;
// consumer warps 0-3 touch one word per stage; warp 4 produces (so the data is "used").
__global__ void __launch_bounds__(288) k_bulk(const unsigned char* __restrict__ a, long bytes, int SB, int NS,
                                              double* out, int pol, int consume) {
  const int NC = blockDim.x - 32;  // consumer threads
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  unsigned char* ring = sm + 256;
  const long per = (bytes / gridDim.x) & ~127L;
  const long b0 = per * blockIdx.x;
  const long nst = per / SB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, NC / 32);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;");
  __syncthreads();
  double acc = 0;
  if (threadIdx.x == NC) {  // producer warp
    for (long i = 0; i < nst; ++i) {
      const int s = i % NS;
      if (i >= NS) mbar_wait(empty + s, ((i / NS) - 1) & 1);
      mbar_expect(full + s, SB);
      bulk(ring + (long)s * SB, a + b0 + i * SB, SB, full + s, pol);
    }
  }
  if (threadIdx.x < NC) {
    for (long i = 0; i < nst; ++i) {
      const int s = i % NS;
      mbar_wait(full + s, (i / NS) & 1);
      const double2* st = reinterpret_cast<const double2*>(ring + (long)s * SB);
      if (consume == 1) {
        for (int k = threadIdx.x; k < SB / 16; k += NC) {
          const double2 v = st[k];
          acc = fma(v.x, v.y, acc);
        }
      } else if (consume == 2) {  // a complex MAC per element (4 DFMA), as the NoTrans SBGEMV
        double2 c = make_double2(acc, 0.0);
        const double2 xv = st[threadIdx.x & 7];
        for (int k = threadIdx.x; k < SB / 16; k += NC) {
          const double2 v = st[k];
          c.x = fma(v.x, xv.x, c.x);
          c.x = fma(-v.y, xv.y, c.x);
          c.y = fma(v.x, xv.y, c.y);
          c.y = fma(v.y, xv.x, c.y);
        }
        acc = c.x + c.y;
      } else if (consume == 3) {  // + a broadcast x load per element
        double2 c = make_double2(acc, 0.0);
        for (int k = threadIdx.x; k < SB / 16; k += NC) {
          const double2 v = st[k];
          const double2 xv = st[(k / 100) & 31];
          c.x = fma(v.x, xv.x, c.x);
          c.x = fma(-v.y, xv.y, c.x);
          c.y = fma(v.x, xv.y, c.y);
          c.y = fma(v.y, xv.x, c.y);
        }
        acc = c.x + c.y;
      } else if (threadIdx.x % 32 == 0) {
        acc += st[threadIdx.x].x;
      }
      __syncwarp();
      if (threadIdx.x % 32 == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(empty + s)));
    }
  }
  if (acc == 12345.678) *out = acc;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (long gb : {8L}) {
    const long bytes = gb * 1000L * 1000 * 1000;
    unsigned char* a;
    if (cudaMalloc(&a, bytes) != cudaSuccess) {
      printf("alloc %ld GB failed\n", gb);
      continue;
    }
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int blk : {512}) {
      for (int per_sm : {8}) {
        const int grid = nsm * per_sm;
        for (int w = 0; w < 2; ++w) k_ldg<<<grid, blk>>>((const double2*)a, bytes / 16, out);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) k_ldg<<<grid, blk>>>((const double2*)a, bytes / 16, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%2ld GB ldg.128  block %3d x %d/SM: %7.0f GB/s\n", gb, blk, per_sm, 5.0 * bytes / (ms * 1e6));
      }
    }
    struct Cfg { int SB, NS, per_sm, pol, consume; };
    const Cfg cfgs[] = {{32768, 3, 2, 0, 0}, {32768, 3, 2, 0, 1}, {32768, 3, 2, 0, 2}, {32768, 3, 2, 0, 3},
                        {32768, 3, 2, 1, 2}, {16384, 6, 2, 0, 2}, {24576, 4, 2, 0, 2}, {32768, 3, 1, 0, 2}};
    for (const Cfg& c : cfgs) {
      const size_t smem = 256 + (size_t)c.SB * c.NS;
      cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      const int grid = nsm * c.per_sm;
      for (int w = 0; w < 2; ++w) k_bulk<<<grid, 288, smem>>>(a, bytes, c.SB, c.NS, out, c.pol, c.consume);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_bulk<<<grid, 288, smem>>>(a, bytes, c.SB, c.NS, out, c.pol, c.consume);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const long per = (bytes / grid) & ~127L;
      const double moved = 5.0 * (double)(per / c.SB) * c.SB * grid;
      printf("%2ld GB bulk ring %5d B x %d x %d/SM evict_first=%d consume=%d: %7.0f GB/s (%.3f ms/pass)\n", gb, c.SB,
             c.NS, c.per_sm, c.pol, c.consume, moved / (ms * 1e6), ms / 5);
    }
    cudaFree(a);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
