// fmv_sbgemv.cuh -- strided-batched GEMV for the per-frequency phase of the
// FFT matvec (phase 3, matvec.hpp:209-228), hand-written for sm_100a.
//
// Reference semantics: gemv.hpp:135-201 (y_b = op(A_b) x_b, column-major A_b,
// lda / stride_a / stride_x / stride_y, alpha=1 beta=0, accumulation in the
// operand precision -- except the fp16 'h' extension, which accumulates in
// fp32).
//
// Design:
//  * The whole batch is one FLAT COLUMN STREAM: column c = b*n + j of the
//    batch lives at A + b*stride_a + j*lda. The stream is cut into P equal
//    contiguous PIECES, one per persistent CTA (P = #SMs x CTAs/SM), so every
//    CTA streams the same number of bytes: no wave tail, no idle SMs, even
//    though nb = 1001 bins is not a multiple of 148.
//  * One producer lane per CTA issues cp.async.bulk (TMA bulk copy, SASS
//    UBLKCP) of each stage -- Jc contiguous columns of A plus the matching x
//    slice -- into a ring of shared-memory stages guarded by mbarrier
//    full/empty pairs, with an L2 evict_first policy (the operator is read
//    exactly once per matvec). Consumers never issue global loads for A.
//  * NoTrans (F): thread (r,g) owns row r (and r+RT, ...) and every G-th
//    column of a stage; partial rows are combined in a fixed order in shared
//    memory. A bin that spans several pieces is finished by the LAST CTA to
//    arrive (atomic ticket), which sums the per-piece partials in piece
//    order: bitwise deterministic for a given (P, shape), no second launch.
//  * ConjTrans/Trans (F*): each column is an independent dot product of
//    m contiguous elements with x_b: LPC lanes per column, conflict-free
//    shared-memory reads, xor-shuffle reduction, one store per column.
#pragma once

#include "fmv_common.cuh"

namespace fmv {

// ---------------------------------------------------------------- PTX ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// TMA bulk copy global -> shared (no tensor map: a contiguous byte range).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bar_consumers(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// -------------------------------------------------------- element traits --
template <class E>
struct ET;
template <>
struct ET<double2> {
  using A = double2;
  static constexpr bool cplx = true;
  static __device__ __forceinline__ A zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ A mac(A c, double2 a, double2 x) {  // c += a*x
    c.x = fma(a.x, x.x, c.x);
    c.x = fma(-a.y, x.y, c.x);
    c.y = fma(a.x, x.y, c.y);
    c.y = fma(a.y, x.x, c.y);
    return c;
  }
  static __device__ __forceinline__ A macc(A c, double2 a, double2 x) {  // c += conj(a)*x
    c.x = fma(a.x, x.x, c.x);
    c.x = fma(a.y, x.y, c.x);
    c.y = fma(a.x, x.y, c.y);
    c.y = fma(-a.y, x.x, c.y);
    return c;
  }
  static __device__ __forceinline__ A add(A a, A b) { return make_double2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ A shfl_xor(A a, int o) {
    return make_double2(__shfl_xor_sync(0xffffffffu, a.x, o), __shfl_xor_sync(0xffffffffu, a.y, o));
  }
};
template <>
struct ET<float2> {
  using A = float2;
  static constexpr bool cplx = true;
  static __device__ __forceinline__ A zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ A mac(A c, float2 a, float2 x) {
    c.x = fmaf(a.x, x.x, c.x);
    c.x = fmaf(-a.y, x.y, c.x);
    c.y = fmaf(a.x, x.y, c.y);
    c.y = fmaf(a.y, x.x, c.y);
    return c;
  }
  static __device__ __forceinline__ A macc(A c, float2 a, float2 x) {
    c.x = fmaf(a.x, x.x, c.x);
    c.x = fmaf(a.y, x.y, c.x);
    c.y = fmaf(a.x, x.y, c.y);
    c.y = fmaf(-a.y, x.x, c.y);
    return c;
  }
  static __device__ __forceinline__ A add(A a, A b) { return make_float2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ A shfl_xor(A a, int o) {
    return make_float2(__shfl_xor_sync(0xffffffffu, a.x, o), __shfl_xor_sync(0xffffffffu, a.y, o));
  }
};
// fp16 storage, fp32 accumulation (the 'h' extension).
template <>
struct ET<__half2> {
  using A = float2;
  static constexpr bool cplx = true;
  static __device__ __forceinline__ A zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ A mac(A c, __half2 a, __half2 x) {
    return ET<float2>::mac(c, __half22float2(a), __half22float2(x));
  }
  static __device__ __forceinline__ A macc(A c, __half2 a, __half2 x) {
    return ET<float2>::macc(c, __half22float2(a), __half22float2(x));
  }
  static __device__ __forceinline__ A add(A a, A b) { return ET<float2>::add(a, b); }
  static __device__ __forceinline__ A shfl_xor(A a, int o) { return ET<float2>::shfl_xor(a, o); }
};
template <>
struct ET<double> {
  using A = double;
  static constexpr bool cplx = false;
  static __device__ __forceinline__ A zero() { return 0.0; }
  static __device__ __forceinline__ A mac(A c, double a, double x) { return fma(a, x, c); }
  static __device__ __forceinline__ A macc(A c, double a, double x) { return fma(a, x, c); }
  static __device__ __forceinline__ A add(A a, A b) { return a + b; }
  static __device__ __forceinline__ A shfl_xor(A a, int o) { return __shfl_xor_sync(0xffffffffu, a, o); }
};
template <>
struct ET<float> {
  using A = float;
  static constexpr bool cplx = false;
  static __device__ __forceinline__ A zero() { return 0.f; }
  static __device__ __forceinline__ A mac(A c, float a, float x) { return fmaf(a, x, c); }
  static __device__ __forceinline__ A macc(A c, float a, float x) { return fmaf(a, x, c); }
  static __device__ __forceinline__ A add(A a, A b) { return a + b; }
  static __device__ __forceinline__ A shfl_xor(A a, int o) { return __shfl_xor_sync(0xffffffffu, a, o); }
};

// accumulator -> output element (single RNE rounding where narrowing)
template <class O, class A>
__device__ __forceinline__ O out_cast(A a);
template <>
__device__ __forceinline__ double2 out_cast<double2, double2>(double2 a) { return a; }
template <>
__device__ __forceinline__ float2 out_cast<float2, double2>(double2 a) { return cfrom_d<float2>(a); }
template <>
__device__ __forceinline__ double2 out_cast<double2, float2>(float2 a) { return make_double2(a.x, a.y); }
template <>
__device__ __forceinline__ float2 out_cast<float2, float2>(float2 a) { return a; }
template <>
__device__ __forceinline__ double out_cast<double, double>(double a) { return a; }
template <>
__device__ __forceinline__ float out_cast<float, float>(float a) { return a; }

template <class A>
__device__ __forceinline__ A ldcg(const A* p);
template <>
__device__ __forceinline__ double2 ldcg<double2>(const double2* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ float2 ldcg<float2>(const float2* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ double ldcg<double>(const double* p) { return __ldcg(p); }
template <>
__device__ __forceinline__ float ldcg<float>(const float* p) { return __ldcg(p); }

// ------------------------------------------------------------- params ----
enum GemvMode : int { GM_N = 0, GM_T = 1, GM_C = 2 };

struct GemvParams {
  const unsigned char* A;
  long lda, sa;  // elements
  const unsigned char* x;
  long sx;
  unsigned char* y;
  long sy;
  int m;
  long n, batch;
  long T;      // batch * n columns in the flat stream
  int P;       // pieces == gridDim.x
  int Jc;      // max columns per stage
  int a_slot;  // bytes per stage for A (multiple of 128)
  int x_slot;  // bytes per stage for x (multiple of 128)
  int nstage;
  int RT, G;   // NoTrans thread layout
  int LPC;     // (Conj)Trans lanes per column
  void* partials;
  unsigned* counters;
};

__device__ __forceinline__ long piece_of(long c, long T, int P) {
  // largest p with floor(p*T/P) <= c
  return ((c + 1) * (long)P - 1) / T;
}

struct Seg {
  long b, j, cnt;
};
__device__ __forceinline__ Seg next_seg(long c, long c1, const GemvParams& p) {
  Seg s;
  s.b = c / p.n;
  s.j = c - s.b * p.n;
  long cnt = p.Jc;
  cnt = min(cnt, c1 - c);
  cnt = min(cnt, p.n - s.j);
  s.cnt = cnt;
  return s;
}

template <int MODE, class E, class O, int RPT>
__global__ void __launch_bounds__(288, 2) k_sbgemv(const GemvParams p) {
  using Tr = ET<E>;
  using Acc = typename Tr::A;
  extern __shared__ __align__(128) unsigned char sm[];
  const int ncons = blockDim.x - 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  volatile int* s_flag = reinterpret_cast<volatile int*>(sm + 256);
  unsigned char* stages = sm + 512;
  const int slot = p.a_slot + p.x_slot;
  Acc* red = reinterpret_cast<Acc*>(stages + (long)p.nstage * slot);

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncons / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const long c0 = p.T * (long)blockIdx.x / p.P;
  const long c1 = p.T * (long)(blockIdx.x + 1) / p.P;
  constexpr int es = (int)sizeof(E);

  if (threadIdx.x >= ncons) {
    // ------------------------------------------------ producer lane ----
    if (threadIdx.x != ncons) return;
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    long it = 0;
    for (long c = c0; c < c1; ++it) {
      const Seg sg = next_seg(c, c1, p);
      const int s = (int)(it % p.nstage);
      const uint32_t par = (uint32_t)((it / p.nstage) & 1);
      mbar_wait(&empty[s], par ^ 1u);
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* a_lo = reinterpret_cast<const unsigned char*>(reinterpret_cast<uintptr_t>(a0) & ~uintptr_t(15));
      const uintptr_t a_end = reinterpret_cast<uintptr_t>(a0) + (uintptr_t)(((sg.cnt - 1) * p.lda + p.m) * es);
      const uint32_t a_bytes = (uint32_t)(((a_end + 15) & ~uintptr_t(15)) - reinterpret_cast<uintptr_t>(a_lo));
      const unsigned char* x0 = MODE == GM_N ? p.x + (sg.b * p.sx + sg.j) * es : p.x + sg.b * p.sx * es;
      const long xn = MODE == GM_N ? sg.cnt : p.m;
      const unsigned char* x_lo = reinterpret_cast<const unsigned char*>(reinterpret_cast<uintptr_t>(x0) & ~uintptr_t(15));
      const uintptr_t x_end = reinterpret_cast<uintptr_t>(x0) + (uintptr_t)(xn * es);
      const uint32_t x_bytes = (uint32_t)(((x_end + 15) & ~uintptr_t(15)) - reinterpret_cast<uintptr_t>(x_lo));
      unsigned char* dst = stages + (long)s * slot;
      mbar_expect_tx(&full[s], a_bytes + x_bytes);
      bulk_g2s(dst, a_lo, a_bytes, &full[s], pol_a);
      bulk_g2s(dst + p.a_slot, x_lo, x_bytes, &full[s], pol_x);
      c += sg.cnt;
    }
    return;
  }

  // ---------------------------------------------------- consumers ----
  const int t = threadIdx.x;
  const int lane = t & 31;
  if constexpr (MODE == GM_N) {
    const int r = t % p.RT;
    const int g = t / p.RT;
    const bool active = g < p.G;
    Acc acc[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) acc[q] = Tr::zero();
    long it = 0;
    for (long c = c0; c < c1; ++it) {
      const Seg sg = next_seg(c, c1, p);
      const int s = (int)(it % p.nstage);
      const uint32_t par = (uint32_t)((it / p.nstage) & 1);
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* x0 = p.x + (sg.b * p.sx + sg.j) * es;
      const unsigned char* base = stages + (long)s * slot;
      const E* As = reinterpret_cast<const E*>(base + (reinterpret_cast<uintptr_t>(a0) & 15));
      const E* Xs = reinterpret_cast<const E*>(base + p.a_slot + (reinterpret_cast<uintptr_t>(x0) & 15));
      mbar_wait(&full[s], par);
      if (active) {
        const int cnt = (int)sg.cnt;
        for (int jj = g; jj < cnt; jj += p.G) {
          const E xv = Xs[jj];
          const E* col = As + (long)jj * p.lda;
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int row = r + q * p.RT;
            if (row < p.m) acc[q] = Tr::mac(acc[q], col[row], xv);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      c += sg.cnt;
      if (sg.j + sg.cnt == p.n || c == c1) {
        // ---- flush bin sg.b: intra-CTA reduction over column groups ----
        if (active) {
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int row = r + q * p.RT;
            if (row < p.m) red[(long)g * p.m + row] = acc[q];
          }
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q) acc[q] = Tr::zero();
        bar_consumers(ncons);
        for (int i = t; i < p.m; i += ncons) {
          Acc v = red[i];
          for (int gg = 1; gg < p.G; ++gg) v = Tr::add(v, red[(long)gg * p.m + i]);
          red[i] = v;
        }
        bar_consumers(ncons);
        // ---- cross-CTA: the last piece to finish bin b sums in piece order ----
        const long b = sg.b;
        const long plo = piece_of(b * p.n, p.T, p.P);
        const long phi = piece_of(b * p.n + p.n - 1, p.T, p.P);
        O* yb = reinterpret_cast<O*>(p.y) + b * p.sy;
        if (plo == phi) {
          for (int i = t; i < p.m; i += ncons) yb[i] = out_cast<O>(red[i]);
        } else {
          Acc* part = reinterpret_cast<Acc*>(p.partials);
          const long slot_id = (long)blockIdx.x + b;
          for (int i = t; i < p.m; i += ncons) part[slot_id * p.m + i] = red[i];
          __threadfence();
          bar_consumers(ncons);
          if (t == 0) {
            const unsigned prev = atomicAdd(&p.counters[b], 1u);
            *s_flag = (prev == (unsigned)(phi - plo)) ? 1 : 0;
          }
          bar_consumers(ncons);
          if (*s_flag) {
            __threadfence();
            for (int i = t; i < p.m; i += ncons) {
              Acc v = ldcg(part + (plo + b) * p.m + i);
              for (long pp = plo + 1; pp <= phi; ++pp) v = Tr::add(v, ldcg(part + (pp + b) * p.m + i));
              yb[i] = out_cast<O>(v);
            }
            if (t == 0) p.counters[b] = 0u;
          }
        }
        bar_consumers(ncons);
      }
    }
  } else {
    // (Conj)Trans: LPC lanes per column, CPW columns per warp-iteration.
    const int W = ncons / 32;
    const int w = t >> 5;
    const int LPC = p.LPC;
    const int CPW = 32 / LPC;
    const int sub = lane / LPC;
    const int li = lane - sub * LPC;
    long it = 0;
    for (long c = c0; c < c1; ++it) {
      const Seg sg = next_seg(c, c1, p);
      const int s = (int)(it % p.nstage);
      const uint32_t par = (uint32_t)((it / p.nstage) & 1);
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* x0 = p.x + sg.b * p.sx * es;
      const unsigned char* base = stages + (long)s * slot;
      const E* As = reinterpret_cast<const E*>(base + (reinterpret_cast<uintptr_t>(a0) & 15));
      const E* Xs = reinterpret_cast<const E*>(base + p.a_slot + (reinterpret_cast<uintptr_t>(x0) & 15));
      O* yb = reinterpret_cast<O*>(p.y) + sg.b * p.sy + sg.j;
      mbar_wait(&full[s], par);
      const int cnt = (int)sg.cnt;
      for (int jb = w * CPW; jb < cnt; jb += W * CPW) {
        const int jj = jb + sub;
        const bool valid = jj < cnt;
        Acc a = Tr::zero();
        if (valid) {
          const E* col = As + (long)jj * p.lda;
          for (int i = li; i < p.m; i += LPC) {
            if constexpr (MODE == GM_C) a = Tr::macc(a, col[i], Xs[i]);
            else a = Tr::mac(a, col[i], Xs[i]);
          }
        }
        for (int o = LPC >> 1; o > 0; o >>= 1) a = Tr::add(a, Tr::shfl_xor(a, o));
        if (valid && li == 0) yb[jj] = out_cast<O>(a);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      c += sg.cnt;
    }
  }
}

// ------------------------------------------------ simple fallback GEMV ----
// Any shape/alignment (used when the staged kernel's limits are exceeded,
// and as a cross-check in tests). One thread per output element.
template <int MODE, class E, class O>
__global__ void k_sbgemv_simple(const GemvParams p) {
  using Tr = ET<E>;
  using Acc = typename Tr::A;
  const long b = blockIdx.y;
  const E* Ab = reinterpret_cast<const E*>(p.A) + b * p.sa;
  const E* xb = reinterpret_cast<const E*>(p.x) + b * p.sx;
  O* yb = reinterpret_cast<O*>(p.y) + b * p.sy;
  const long o = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (MODE == GM_N) {
    if (o >= p.m) return;
    Acc a = Tr::zero();
    for (long j = 0; j < p.n; ++j) a = Tr::mac(a, Ab[j * p.lda + o], xb[j]);
    yb[o] = out_cast<O>(a);
  } else {
    if (o >= p.n) return;
    Acc a = Tr::zero();
    for (long i = 0; i < p.m; ++i) {
      if constexpr (MODE == GM_C) a = Tr::macc(a, Ab[o * p.lda + i], xb[i]);
      else a = Tr::mac(a, Ab[o * p.lda + i], xb[i]);
    }
    yb[o] = out_cast<O>(a);
  }
}

}  // namespace fmv
