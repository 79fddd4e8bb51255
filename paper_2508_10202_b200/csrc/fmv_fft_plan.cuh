// fmv_fft_plan.cuh -- plan types shared by the FFT kernels (fmv_fft.cuh,
// fmv_fft_rt.cuh) and the host runtime that builds them.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace fmv {

// Division by a runtime-invariant divisor with one multiply-high
// (Granlund-Montgomery round-up method; valid for n < 2^31).
struct FastDiv {
  uint32_t d = 1, m = 0, s = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (div > 1) {
      while ((1u << s) < div) ++s;
      m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << s) - div)) / div + 1);
    }
  }
  __device__ __forceinline__ int div(int n) const {
    return d == 1 ? n : (int)((__umulhi((uint32_t)n, m) + (uint32_t)n) >> s);
  }
};

constexpr int kRtMaxPasses = 8;
constexpr int kRtHold = 16;  // complex values a thread holds across a pass barrier (at most)
// Butterflies of radix Rn a thread may own in one pass: floor(16 / Rn), >= 1.
template <int Rn>
constexpr int rt_hold() {
  return kRtHold / Rn > 0 ? kRtHold / Rn : 1;
}

struct RtPlan {
  int N;   // complex length (= Nt of the pipeline; L = 2N)
  int np;  // passes
  int radix[kRtMaxPasses];
  int tw_off[kRtMaxPasses];  // offset of pass p's table [q*Ns + k] in the twiddle array (p >= 1)
  int Ns[kRtMaxPasses];      // product of the earlier radices
  FastDiv ns_div[kRtMaxPasses];
  int bpt[kRtMaxPasses];     // butterflies per thread of pass p
  int TS;                    // threads per series
  int S;                     // series per CTA
  int SS;                    // shared-memory series stride (complex elements)
  int sfast;                 // thread -> (series, j) mapping: 1 = series fastest (time-outer input)
};

}  // namespace fmv
