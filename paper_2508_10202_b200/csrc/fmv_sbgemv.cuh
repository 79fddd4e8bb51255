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

#include <type_traits>

#include "fmv_common.cuh"
#include "fmv_tma.cuh"

namespace fmv {

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
// fp16 storage, fp32 accumulation (the 'h' extension). Blackwell's
// mixed-precision FMA (fma.rn.f32.f16 -> SASS FHFMA, half-register selectors
// and negation folded) does f32 += f16*f16 in one instruction; the f16
// product is exact in f32, so this equals convert-then-FFMA bit for bit.
__device__ __forceinline__ float fhfma(__half a, __half b, float c) {
  float d;
  asm("fma.rn.f32.f16 %0, %1, %2, %3;" : "=f"(d) : "h"(__half_as_ushort(a)), "h"(__half_as_ushort(b)), "f"(c));
  return d;
}
__device__ __forceinline__ __half hlo(__half2 v) { return __low2half(v); }
__device__ __forceinline__ __half hhi(__half2 v) { return __high2half(v); }
__device__ __forceinline__ __half hneg(__half v) { return __hneg(v); }
template <>
struct ET<__half2> {
  using A = float2;
  static constexpr bool cplx = true;
  static __device__ __forceinline__ A zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ A mac(A c, __half2 a, __half2 x) {  // c += a*x
    c.x = fhfma(hlo(a), hlo(x), c.x);
    c.x = fhfma(hneg(hhi(a)), hhi(x), c.x);
    c.y = fhfma(hlo(a), hhi(x), c.y);
    c.y = fhfma(hhi(a), hlo(x), c.y);
    return c;
  }
  static __device__ __forceinline__ A macc(A c, __half2 a, __half2 x) {  // c += conj(a)*x
    c.x = fhfma(hlo(a), hlo(x), c.x);
    c.x = fhfma(hhi(a), hhi(x), c.x);
    c.y = fhfma(hlo(a), hhi(x), c.y);
    c.y = fhfma(hneg(hhi(a)), hlo(x), c.y);
    return c;
  }
  static __device__ __forceinline__ A add(A a, A b) { return ET<float2>::add(a, b); }
  static __device__ __forceinline__ A shfl_xor(A a, int o) { return ET<float2>::shfl_xor(a, o); }
};
// The 'm' SBGEMV variant: complex fp32 storage (operator
// and spectrum, layout-identical to float2) with fp64 accumulation. Each
// product of two fp32 values is exact in fp64, so the only roundings are the
// storage ones and the fp64 sums: ~3.6e-8 at C2 instead of ~1e-7 for 's',
// at the same 4 GB operator stream.
struct __align__(8) cf32d {
  float x, y;
};
using ::__ldg;
__device__ __forceinline__ cf32d __ldg(const cf32d* p) {
  const float2 v = ::__ldg(reinterpret_cast<const float2*>(p));
  return cf32d{v.x, v.y};
}
template <>
struct ET<cf32d> {
  using A = double2;
  static constexpr bool cplx = true;
  static __device__ __forceinline__ A zero() { return make_double2(0.0, 0.0); }
  static __device__ __forceinline__ A mac(A c, cf32d a, cf32d x) {  // c += a*x
    const double ax = a.x, ay = a.y, xx = x.x, xy = x.y;
    c.x = fma(ax, xx, c.x);
    c.x = fma(-ay, xy, c.x);
    c.y = fma(ax, xy, c.y);
    c.y = fma(ay, xx, c.y);
    return c;
  }
  static __device__ __forceinline__ A macc(A c, cf32d a, cf32d x) {  // c += conj(a)*x
    const double ax = a.x, ay = a.y, xx = x.x, xy = x.y;
    c.x = fma(ax, xx, c.x);
    c.x = fma(ay, xy, c.x);
    c.y = fma(ax, xy, c.y);
    c.y = fma(-ay, xx, c.y);
    return c;
  }
  static __device__ __forceinline__ A add(A a, A b) { return make_double2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ A shfl_xor(A a, int o) { return ET<double2>::shfl_xor(a, o); }
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
  // NoTrans column-chunk accumulation (the host splits the n columns into
  // chunks launched in order): 0 none (y = cast(sum)), 1 first (yacc = sum),
  // 2 middle (yacc += sum), 3 last (y = cast(yacc + sum)). yacc is [batch][m]
  // in the accumulator type; the fixed chunk order keeps results deterministic.
  void* yacc;
  int accum;
  // (Conj)Trans: x_b kept resident in two shared slots (by batch parity),
  // copied once per batch entry instead of with every stage. Requires every
  // batch entry to span >= nstage stages (then the slot being refilled is never
  // still in use).
  int xres;
  int xres_slot;
  int arrive_all;  // every consumer thread arrives on the empty barrier (else one lane per warp)
  // Block (multi-RHS) kernel k_sbgemm_block only: K right-hand sides per
  // batch entry, x_{b,r} at x + (b*sx + r*sxr)*es and y_{b,r} at
  // y + (b*sy + r*syr)*es; xr_slot = shared bytes per RHS x slice.
  int K;
  long sxr, syr;
  int xr_slot;
};

__device__ __forceinline__ long piece_of(long c, long T, int P) {
  // largest p with floor(p*T/P) <= c
  return ((c + 1) * (long)P - 1) / T;
}

// Walks the flat column stream of one piece, one stage-sized segment at a
// time, without per-stage 64-bit divisions: (b, j) = (batch entry, column),
// cnt = columns in this segment (never crosses a batch entry), ring slot s
// and its mbarrier phase parity advance incrementally.
struct SegIter {
  long b, j, c, c1, cnt;
  int s;
  uint32_t par;
  __device__ __forceinline__ SegIter(long c0, long c1_, const GemvParams& p) : c(c0), c1(c1_), s(0), par(0) {
    b = c0 / p.n;
    j = c0 - b * p.n;
    cnt = 0;
  }
  __device__ __forceinline__ bool more() const { return c < c1; }
  __device__ __forceinline__ void load(const GemvParams& p) {
    long k = p.Jc;
    k = min(k, c1 - c);
    k = min(k, p.n - j);
    cnt = k;
  }
  // true when this segment closed batch entry b (or the piece)
  __device__ __forceinline__ bool ends_bin(const GemvParams& p) const { return j + cnt == p.n || c + cnt == c1; }
  __device__ __forceinline__ void advance(const GemvParams& p) {
    c += cnt;
    j += cnt;
    if (j == p.n) {
      j = 0;
      ++b;
    }
    if (++s == p.nstage) {
      s = 0;
      par ^= 1u;
    }
  }
};

// V elements of E packed in one 16-byte shared-memory load.
template <class E, int V>
struct alignas(V == 1 ? alignof(E) : 16) VecT {
  E e[V];
};
template <class E, int V>
__device__ __forceinline__ VecT<E, V> ldv(const E* p) {
  if constexpr (V == 1) {
    return VecT<E, 1>{{*p}};
  } else {
    static_assert(sizeof(E) * V == 16, "vector must be 16 bytes");
    const int4 raw = *reinterpret_cast<const int4*>(p);
    VecT<E, V> r;
    memcpy(&r, &raw, 16);
    return r;
  }
}

// Neumaier compensated add s += x with compensation c (componentwise).
__device__ __forceinline__ void neumaier1(float& s, float& c, float x) {
  const float t = s + x;
  c += (fabsf(s) >= fabsf(x)) ? ((s - t) + x) : ((x - t) + s);
  s = t;
}
template <class A>
__device__ __forceinline__ void neumaier_add(A& s, A& c, A x) {
  if constexpr (std::is_same<A, float2>::value) {
    neumaier1(s.x, c.x, x.x);
    neumaier1(s.y, c.y, x.y);
  } else if constexpr (std::is_same<A, float>::value) {
    neumaier1(s, c, x);
  }
}

template <int MODE, class E, class O, int RPT, int V, int LPC>
// One CTA per SM with 16 consumer warps: measured at C2 (tools/ab_wide.sh) it
// streams 5-6% faster than two 8-warp CTAs per SM -- half as many concurrent
// DRAM streams with the same consumer width (the bare TMA ring shows the same
// 1-vs-2 CTA effect, tools/read_ceiling.cu).
#ifndef FMV_SBGEMV_MINB
#define FMV_SBGEMV_MINB 1  // resident CTAs per SM the register budget is sized for
#endif
#ifndef FMV_SBGEMV_CONS
#define FMV_SBGEMV_CONS 512  // consumer threads per CTA (+ one producer warp)
#endif
__global__ void __launch_bounds__(FMV_SBGEMV_CONS + 32, FMV_SBGEMV_MINB) k_sbgemv(const GemvParams p) {
  using Tr = ET<E>;
  using Acc = typename Tr::A;
  extern __shared__ __align__(128) unsigned char sm[];
  const int ncons = blockDim.x - 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  volatile int* s_flag = reinterpret_cast<volatile int*>(sm + 256);
  unsigned char* stages = sm + 512;
  const int slot = p.a_slot + (p.xres ? 0 : p.x_slot);
  unsigned char* xres_base = stages + (long)p.nstage * slot;
  Acc* red = reinterpret_cast<Acc*>(xres_base + (p.xres ? 2L * p.xres_slot : 0L));

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.arrive_all ? ncons : ncons / 32);
    }
    mbar_fence_init();
  }
  grid_dep_wait();  // (PDL) the previous kernel's x / y writes are visible from here on
  __syncthreads();

  const long c0 = p.T * (long)blockIdx.x / p.P;
  const long c1 = p.T * (long)(blockIdx.x + 1) / p.P;
  constexpr int es = (int)sizeof(E);

  if (threadIdx.x >= ncons) {
    // ------------------------------------------------ producer lane ----
    if (threadIdx.x != ncons) return;
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    long prev_b = -1;
    for (SegIter sg(c0, c1, p); sg.more(); sg.advance(p)) {
      sg.load(p);
      const int s = sg.s;
      mbar_wait(&empty[s], sg.par ^ 1u);
      const bool new_x = !p.xres || sg.b != prev_b;
      prev_b = sg.b;
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
      unsigned char* xdst = p.xres ? xres_base + (sg.b & 1) * (long)p.xres_slot : dst + p.a_slot;
      mbar_expect_tx(&full[s], a_bytes + (new_x ? x_bytes : 0u));
      bulk_g2s(dst, a_lo, a_bytes, &full[s], pol_a);
      if (new_x) bulk_g2s(xdst, x_lo, x_bytes, &full[s], pol_x);
    }
    return;
  }

  // ---------------------------------------------------- consumers ----
  const int t = threadIdx.x;
  const int lane = t & 31;
  const int MV = (p.m + V - 1) / V;  // 16-byte row vectors per column (V elements each)
  if constexpr (MODE == GM_N) {
    // thread (r, g): row vectors r, r+RT, ... (RPT of them), columns g, g+G, ...
    const int r = t % p.RT;
    const int g = t / p.RT;
    const bool active = g < p.G;
    // fp32 accumulators sum each stage into a fresh partial and fold it into
    // the running sum with a compensated (Neumaier) add: still fp32
    // arithmetic (SPEC.md "accumulation precision equals operand precision"),
    // but the error no longer grows with the ~300 columns a thread visits
    // per bin. fp64 accumulators use the plain running sum.
    constexpr bool kComp = !std::is_same<Acc, double2>::value && !std::is_same<Acc, double>::value;
    Acc acc[RPT][V], cmp[RPT][V];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[q][v] = cmp[q][v] = Tr::zero();
    for (SegIter sg(c0, c1, p); sg.more(); sg.advance(p)) {
      sg.load(p);
      const int s = sg.s;
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* x0 = p.x + (sg.b * p.sx + sg.j) * es;
      const unsigned char* base = stages + (long)s * slot;
      const E* As = reinterpret_cast<const E*>(base + (reinterpret_cast<uintptr_t>(a0) & 15));
      const E* Xs = reinterpret_cast<const E*>(base + p.a_slot + (reinterpret_cast<uintptr_t>(x0) & 15));
      mbar_wait_sleep(&full[s], sg.par);
      if (active) {
        const int cnt = (int)sg.cnt;
        // Two column chains (columns jj and jj + G) with their own partial
        // sums, both loads issued before either MAC, so a warp's LDS latency
        // and FMA dependency chain are paid once per two columns; the chains
        // are added once per stage (fixed order: deterministic).
        Acc part[RPT][V], part2[RPT][V];
#pragma unroll
        for (int q = 0; q < RPT; ++q)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            part[q][v] = kComp ? Tr::zero() : acc[q][v];
            part2[q][v] = Tr::zero();
          }
        // Pointers stepped per iteration (the thread's row offset folded in
        // once), so the loop body is loads + MACs + two pointer adds.
        const int G = p.G;
        const long cstep = (long)G * p.lda;  // elements between this thread's consecutive columns
        const E* colp = As + (long)g * p.lda + r * V;
        const E* xp = Xs + g;
        int jj = g;
        constexpr bool kTwo = RPT * V <= 4;  // register budget (wide RPT*V variants keep one chain)
        if constexpr (kTwo) for (; jj + G < cnt; jj += 2 * G, colp += 2 * cstep, xp += 2 * G) {
          const E xv0 = xp[0], xv1 = xp[G];
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int vi = r + q * p.RT;
            if (RPT == 1 || vi < MV) {  // RPT == 1: RT == MV, so every active row is in range
              const VecT<E, V> a0 = ldv<E, V>(colp + q * p.RT * V);
              const VecT<E, V> a1 = ldv<E, V>(colp + cstep + q * p.RT * V);
#pragma unroll
              for (int v = 0; v < V; ++v) {
                part[q][v] = Tr::mac(part[q][v], a0.e[v], xv0);
                part2[q][v] = Tr::mac(part2[q][v], a1.e[v], xv1);
              }
            }
          }
        }
        for (; jj < cnt; jj += G, colp += cstep, xp += G) {
          const E xv = xp[0];
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
            const int vi = r + q * p.RT;
            if (RPT == 1 || vi < MV) {
              const VecT<E, V> a = ldv<E, V>(colp + q * p.RT * V);
#pragma unroll
              for (int v = 0; v < V; ++v) part[q][v] = Tr::mac(part[q][v], a.e[v], xv);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < RPT; ++q)
#pragma unroll
          for (int v = 0; v < V; ++v) {
            const Acc sum = Tr::add(part[q][v], part2[q][v]);
            if constexpr (kComp) neumaier_add(acc[q][v], cmp[q][v], sum);
            else acc[q][v] = sum;
          }
      }
      __syncwarp();
      if (p.arrive_all || lane == 0) mbar_arrive(&empty[s]);
      if (sg.ends_bin(p)) {
        // ---- flush bin sg.b: intra-CTA reduction over column groups ----
        if (active) {
#pragma unroll
          for (int q = 0; q < RPT; ++q) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
              const int row = (r + q * p.RT) * V + v;
              if constexpr (kComp) {
                if (row < p.m) red[(long)g * p.m + row] = Tr::add(acc[q][v], cmp[q][v]);
                cmp[q][v] = Tr::zero();
              } else {
                if (row < p.m) red[(long)g * p.m + row] = acc[q][v];
              }
              acc[q][v] = Tr::zero();
            }
          }
        }
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
        Acc* ya = reinterpret_cast<Acc*>(p.yacc) + b * p.m;
        auto emit = [&](int i, Acc v) {
          if (p.accum == 0) yb[i] = out_cast<O>(v);
          else if (p.accum == 1) ya[i] = v;
          else if (p.accum == 2) ya[i] = Tr::add(ya[i], v);
          else yb[i] = out_cast<O>(Tr::add(ya[i], v));
        };
        if (plo == phi) {
          for (int i = t; i < p.m; i += ncons) emit(i, red[i]);
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
              emit(i, v);
            }
            if (t == 0) p.counters[b] = 0u;
          }
        }
        bar_consumers(ncons);
      }
    }
  } else {
    // (Conj)Trans: every consumer warp visits every stage (so every waiter
    // sees consecutive mbarrier phases); the stage's columns are dealt out
    // CPW at a time across the W warps, LPC lanes per column, 16-byte vector
    // loads, two accumulator chains and a fixed xor-shuffle tree per column.
    constexpr int CPW = LPC > 0 ? 32 / LPC : 1;
    const int W = ncons / 32;
    const int w = t >> 5;
    const int sub = LPC > 0 ? lane / LPC : 0;
    const int li = LPC > 0 ? lane - sub * LPC : lane;
    const bool ragged = (p.m % V) != 0;
    for (SegIter sg(c0, c1, p); sg.more(); sg.advance(p)) {
      sg.load(p);
      const int s = sg.s;
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* x0 = p.x + sg.b * p.sx * es;
      const unsigned char* base = stages + (long)s * slot;
      const E* As = reinterpret_cast<const E*>(base + (reinterpret_cast<uintptr_t>(a0) & 15));
      const unsigned char* xb = p.xres ? xres_base + (sg.b & 1) * (long)p.xres_slot : base + p.a_slot;
      const E* Xs = reinterpret_cast<const E*>(xb + (reinterpret_cast<uintptr_t>(x0) & 15));
      O* yb = reinterpret_cast<O*>(p.y) + sg.b * p.sy + sg.j;
      mbar_wait_sleep(&full[s], sg.par);
      const int cnt = (int)sg.cnt;
      auto dot = [&](const E* col, int vi, int vstep, Acc& a0c, Acc& a1c) {
        if constexpr (std::is_same<E, cf32d>::value) {
          // 'm': the four real products of each complex MAC go to separate
          // fp64 accumulators (8 independent DFMA chains per lane instead of
          // 2 x 2 chains four DFMAs deep per vector), folded at the end
          double q[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
          auto body4 = [&](double* c, int v0) {
            const VecT<E, V> a = ldv<E, V>(col + v0 * V);
            const VecT<E, V> x = ldv<E, V>(Xs + v0 * V);
#pragma unroll
            for (int v = 0; v < V; ++v) {
              if (V == 1 || !ragged || v0 * V + v < p.m) {
                const double ax = a.e[v].x, ay = a.e[v].y, xx = x.e[v].x, xy = x.e[v].y;
                c[0] = fma(ax, xx, c[0]);
                c[1] = fma(ay, xy, c[1]);
                c[2] = fma(ax, xy, c[2]);
                c[3] = fma(ay, xx, c[3]);
              }
            }
          };
          for (; vi + vstep < MV; vi += 2 * vstep) {
            body4(q[0], vi);
            body4(q[1], vi + vstep);
          }
          if (vi < MV) body4(q[0], vi);
          // ConjTrans: conj(a) x = (ax xx + ay xy, ax xy - ay xx); Trans: a x
          constexpr double sg = MODE == GM_C ? 1.0 : -1.0;
          a0c = make_double2(q[0][0] + sg * q[0][1], q[0][2] - sg * q[0][3]);
          a1c = make_double2(q[1][0] + sg * q[1][1], q[1][2] - sg * q[1][3]);
          return;
        }
        auto body = [&](Acc& acc, int v0) {
          const VecT<E, V> a = ldv<E, V>(col + v0 * V);
          const VecT<E, V> x = ldv<E, V>(Xs + v0 * V);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (V == 1 || !ragged || v0 * V + v < p.m) {
              if constexpr (MODE == GM_C) acc = Tr::macc(acc, a.e[v], x.e[v]);
              else acc = Tr::mac(acc, a.e[v], x.e[v]);
            }
          }
        };
        for (; vi + vstep < MV; vi += 2 * vstep) {
          body(a0c, vi);
          body(a1c, vi + vstep);
        }
        if (vi < MV) body(a0c, vi);
      };
      if constexpr (LPC > 0) {
        for (int jb = w * CPW; jb < cnt; jb += W * CPW) {
          const int jj = jb + sub;
          const bool valid = jj < cnt;
          Acc a0c = Tr::zero(), a1c = Tr::zero();
          if (valid) dot(As + (long)jj * p.lda, li, LPC, a0c, a1c);
          Acc a = Tr::add(a0c, a1c);
#pragma unroll
          for (int o = LPC >> 1; o > 0; o >>= 1) a = Tr::add(a, Tr::shfl_xor(a, o));
          if (valid && li == 0) yb[jj] = out_cast<O>(a);
        }
      } else {
        // tall columns: WPC warps per column, warp partials combined in
        // fixed warp order through shared memory
        const int WPC = p.LPC >> 5;
        const int CPI = W / WPC;  // columns per iteration
        const int cs = w / WPC, wi = w - cs * WPC;
        for (int jb = 0; jb < cnt; jb += CPI) {
          const int jj = jb + cs;
          Acc a0c = Tr::zero(), a1c = Tr::zero();
          if (jj < cnt) dot(As + (long)jj * p.lda, wi * 32 + lane, WPC * 32, a0c, a1c);
          Acc a = Tr::add(a0c, a1c);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) a = Tr::add(a, Tr::shfl_xor(a, o));
          if (lane == 0) red[w] = a;
          bar_consumers(ncons);
          if (t < CPI && jb + t < cnt) {
            Acc v = red[t * WPC];
            for (int k = 1; k < WPC; ++k) v = Tr::add(v, red[t * WPC + k]);
            yb[jb + t] = out_cast<O>(v);
          }
          bar_consumers(ncons);
        }
      }
      __syncwarp();
      if (p.arrive_all || lane == 0) mbar_arrive(&empty[s]);
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
    Acc* ya = reinterpret_cast<Acc*>(p.yacc) + b * p.m;
    if (p.accum == 0) yb[o] = out_cast<O>(a);
    else if (p.accum == 1) ya[o] = a;
    else if (p.accum == 2) ya[o] = Tr::add(ya[o], a);
    else yb[o] = out_cast<O>(Tr::add(ya[o], a));
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

// Latency-oriented (Conj)Trans SBGEMV for small problems with short columns
// (C4's m = 10 cells, a few MB in all): one thread per output y_b[j], flat
// over batch*n so a single wave covers the GPU, the column read with
// V-element 16-byte vector loads and x_b through the read-only cache. No TMA
// ring or mbarriers: the whole call is one DRAM round trip plus the launch,
// where the staged kernel's pipeline fill dominated (sbgemv_run_t picks it).
template <int MODE, class E, class O, int V>
__global__ void __launch_bounds__(128) k_sbgemv_small(const GemvParams p) {
  using Tr = ET<E>;
  using Acc = typename Tr::A;
  struct alignas(16) Vec {
    E v[V];
  };
  grid_dep_wait();
  const long o = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= p.T) return;
  const long b = o / p.n, j = o - b * p.n;
  const E* col = reinterpret_cast<const E*>(p.A) + b * p.sa + j * p.lda;
  const E* xb = reinterpret_cast<const E*>(p.x) + b * p.sx;
  Acc a = Tr::zero();
  // The column is read in groups of GR 16-byte loads that are all issued
  // before the first FMA: after an L2 flush each load is a DRAM round trip,
  // and a rolled (or load/FMA-interleaved) loop serialized them.
  constexpr int GR = V > 1 ? 8 : 16;
  for (int i0 = 0; i0 < p.m; i0 += GR * V) {
    Vec w[GR];
    E xv[GR * V];  // x_b too: after a flush it is a DRAM miss as well
#pragma unroll
    for (int g = 0; g < GR; ++g) {
      const int i = i0 + g * V;
      if (i < p.m) {
        if constexpr (V > 1) {
          const uint4 raw = __ldg(reinterpret_cast<const uint4*>(col + i));
          memcpy(&w[g], &raw, sizeof(Vec));
        } else {
          w[g].v[0] = __ldg(col + i);
        }
      }
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (i + v < p.m) xv[g * V + v] = __ldg(xb + i + v);
    }
#pragma unroll
    for (int g = 0; g < GR; ++g) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        if (i0 + g * V + v < p.m) {
          if constexpr (MODE == GM_C) a = Tr::macc(a, w[g].v[v], xv[g * V + v]);
          else a = Tr::mac(a, w[g].v[v], xv[g * V + v]);
        }
      }
    }
  }
  reinterpret_cast<O*>(p.y)[b * p.sy + j] = out_cast<O>(a);
}

}  // namespace fmv
