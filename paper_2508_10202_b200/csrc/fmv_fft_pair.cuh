// fmv_fft_pair.cuh -- paired-butterfly register FFTs for the big Nt = 1000
// transforms of the matvec (the Nm-series r2c of F and c2r of F*).
//
// Same math as k_r2c_reg / k_c2r_reg (fmv_fft.cuh): a real series of length
// L = 2N is packed as N complex points, a radix-10 Stockham FFT of length
// N = 10^3 runs in three passes, and a split post-pass (r2c) / pre-pass (c2r)
// converts between Z and the N + 1 real-signal bins (fft.hpp:32-148).
//
// What changes is who owns what. The post-pass pairs bin k with bin N - k,
// and the pre-pass pairs Z[n] with Z[N - n]. In the last Stockham pass the
// thread computing butterfly j produces Z[j + q*N/10], q = 0..9, and
// N - (j + q*N/10) = (N/10 - j) + (9 - q)*N/10: the partner values come out
// of butterfly N/10 - j. So each thread owns the two butterflies
// ja = t and jb = N/10 - t (t = 0 owns 0 and N/20, both self-paired), and
//   * the r2c post-pass runs on registers and writes the bins straight to
//     global memory (no shared-memory round trip for the post-pass);
//   * the c2r pre-pass reads the bins straight from global memory into
//     registers (no cp.async staging, no shared-memory reads for the
//     pre-pass), and its last pass writes the time samples to global.
// That leaves two shared round trips per transform instead of four, which
// is what bounded the one-butterfly-per-thread kernels (L1TEX at 77 %,
// profiles/ncu_fft_r02.md).
//
// Lanes are series-fastest (thread = t*S + s): a warp's TOSI stores / loads
// of one bin index touch S consecutive series (S = 4 fp64 / 8 fp32 = 64 B
// runs), and the series stride SS = 2 (mod 128 B) plus the q^1 store swizzle
// for odd t make every shared-memory phase conflict-free.
//
// The post-pass twiddle w^k (w = exp(-2 pi i / L)) for k = j + q*N/10 is
// w^j (table) * exp(-i pi q / 10) (constant); and the two bins of a pair
// share one complex product:
//   E = (Z_k + conj Z_{N-k}) / 2, D = (Z_k - conj Z_{N-k}) / 2, P = w^k D
//   X_k = E - i P,  X_{N-k} = conj(E + i P).
// Likewise in the c2r pre-pass (A = X_n, B = conj X_{N-n}, Q = conj(w^n)(A - B)):
//   Z_n = (A + B) + i Q,  Z_{N-n} = conj((A + B) - i Q).
#pragma once

#include "fmv_fft.cuh"

namespace fmv {

// Series stride (elements) of the paired kernels: N rounded up to 2 mod (128 B).
template <class C>
constexpr int pair_series_stride() {
  constexpr int per128 = 128 / (int)sizeof(C);
  int ss = 1000;
  while (ss % per128 != 2 % per128) ++ss;
  return ss;
}
template <class C, int S>
constexpr size_t pair_smem() {
  return (size_t)S * pair_series_stride<C>() * sizeof(C);
}

// o[q] = v[q] in swizzled order: lanes with d = 1 store the pair q^1 first
// (their base address is 2 elements off modulo a 128-byte phase).
template <class C>
__device__ __forceinline__ void store10_swz(C* o, const C* v, int d) {
#pragma unroll
  for (int q = 0; q < 10; ++q) o[q ^ d] = d ? v[q ^ 1] : v[q];
}

// v[q] *= w^(q*k), q = 1..9, all nine read from the pass table twp[q*Ns + k]
// (exact table values, no products). With series-fastest lanes the S lanes
// of one butterfly index share each read, so a warp's read of one q is one
// 128-byte wavefront; this trades ~8 complex products per butterfly for
// L1 hits, which the paired kernels have to spare.
template <class R, int D, int Ns>
__device__ __forceinline__ void apply_tw9(typename CT<R>::c* v, const typename CT<R>::c* __restrict__ twp, int k) {
#pragma unroll
  for (int q = 1; q < 10; ++q) v[q] = cmul(v[q], twiddle<D>(twp, q * Ns + k));
}

// Middle pass (Ns = 10) over both butterflies of the thread.
template <class R, int D>
__device__ __forceinline__ void pair_pass2(typename CT<R>::c* __restrict__ buf, int ja, int jb,
                                           typename CT<R>::c* a, typename CT<R>::c* b,
                                           const typename CT<R>::c* __restrict__ tw, bool act) {
  constexpr int RX = 10, N = 1000, NR = 100, Ns = 10;
  const typename CT<R>::c* __restrict__ twp = tw + reg_tw_offset<RX, N, Ns>();
  const int ka = ja % Ns, kb = jb % Ns;
  if (act) {
#pragma unroll
    for (int q = 0; q < RX; ++q) {
      a[q] = buf[ja + q * NR];
      b[q] = buf[jb + q * NR];
    }
    apply_tw9<R, D, Ns>(a, twp, ka);
    apply_tw9<R, D, Ns>(b, twp, kb);
    butterfly<R, D, RX>(a);
    butterfly<R, D, RX>(b);
  }
  __syncthreads();
  if (act) {
    const int oa = (ja - ka) * RX + ka, ob = (jb - kb) * RX + kb;
#pragma unroll
    for (int q = 0; q < RX; ++q) {
      buf[oa + q * Ns] = a[q];
      buf[ob + q * Ns] = b[q];
    }
  }
  __syncthreads();
}

// Last pass (Ns = 100): Z[j + q*NR] of both butterflies into registers.
template <class R, int D>
__device__ __forceinline__ void pair_pass3(const typename CT<R>::c* __restrict__ buf, int ja, int jb,
                                           typename CT<R>::c* a, typename CT<R>::c* b,
                                           const typename CT<R>::c* __restrict__ tw) {
  constexpr int RX = 10, N = 1000, NR = 100;
  const typename CT<R>::c* __restrict__ twp = tw + reg_tw_offset<RX, N, NR>();
#pragma unroll
  for (int q = 0; q < RX; ++q) {
    a[q] = buf[ja + q * NR];
    b[q] = buf[jb + q * NR];
  }
  apply_tw9<R, D, NR>(a, twp, ja);
  apply_tw9<R, D, NR>(b, twp, jb);
  butterfly<R, D, RX>(a);
  butterfly<R, D, RX>(b);
}

// Phases 1-2 + reorder for SOTI input in[s*in_ss + t], t < N (zero-padded to
// L = 2N: the matvec's pad stage), and TOSI output out[k*out_ks + s];
// N = 1000, S series per CTA, 50 threads per series.
template <int C0, int C1, int C2, class Tin, int S, int MINB>
__global__ void __launch_bounds__(S * 50, MINB)
    k_r2c_pair(const Tin* __restrict__ in, long in_ss, long nseries, bool vec,
               typename PT<C2>::cplx* __restrict__ out, long out_ks,
               const typename CT<typename PT<C1>::real>::c* __restrict__ tw) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  using OutC = typename PT<C2>::cplx;
  constexpr int RX = 10, N = 1000, NR = 100;
  constexpr int SS = pair_series_stride<C>();
  extern __shared__ __align__(16) unsigned char pair_smem_r2c[];
  C* sbuf = reinterpret_cast<C*>(pair_smem_r2c);
  const int s = threadIdx.x % S, t = threadIdx.x / S;
  const long s0 = (long)blockIdx.x * S;
  const int ns = (int)min((long)S, nseries - s0);
  const bool act = s < ns;
  const int ja = t, jb = t == 0 ? NR / 2 : NR - t;
  C* buf = sbuf + s * SS;
  C a[RX], b[RX];
  grid_dep_wait();  // (PDL)

  // Pass 1 (Ns = 1): z[n] = v[2n] + i v[2n+1], n = j + q*NR, from global.
  {
    const Tin* p = in + (s0 + (act ? s : 0)) * in_ss;
    // The matvec input is zero-padded to L = 2N (nvalid = N): z[n] = 0 for
    // n >= N/2, i.e. q >= 5 -- compile-time zeros the DFT folds away.
    auto load = [&](C* v, int j) {
#pragma unroll
      for (int q = 0; q < RX; ++q) {
        const int n = j + q * NR;
        v[q] = C{R(0), R(0)};
        if (q < RX / 2 && act) {
          if constexpr (sizeof(Tin) == 8) {
            if (vec) {
              const double2 pr = __ldg(reinterpret_cast<const double2*>(p) + n);
              v[q] = C{(R)rnd<C0>(pr.x), (R)rnd<C0>(pr.y)};
              continue;
            }
          } else if constexpr (sizeof(Tin) == 4) {
            if (vec) {
              const float2 pr = __ldg(reinterpret_cast<const float2*>(p) + n);
              v[q] = C{(R)rnd<C0>((double)pr.x), (R)rnd<C0>((double)pr.y)};
              continue;
            }
          }
          v[q] = C{(R)rnd<C0>(to_d(p[2 * n])), (R)rnd<C0>(to_d(p[2 * n + 1]))};
        }
      }
    };
    load(a, ja);
    load(b, jb);
    butterfly<R, -1, RX>(a);
    butterfly<R, -1, RX>(b);
    if (act) {
      const int d = t & 1;
      store10_swz(buf + ja * RX, a, d);
      store10_swz(buf + jb * RX, b, d);
    }
    __syncthreads();
  }
  pair_pass2<R, -1>(buf, ja, jb, a, b, tw, act);
  if (!act) return;  // (no barrier below)
  pair_pass3<R, -1>(buf, ja, jb, a, b, tw);

  // Post-pass on registers: bins k and N - k from Z_k = A, Z_{N-k} = B.
  OutC* o = out + s0 + s;
  const R half = R(0.5);
  auto emit = [&](C A, C B, C w, int k, bool both) {
    const C E = {(A.x + B.x) * half, (A.y - B.y) * half};  // (A + conj B) / 2
    const C Dm = {(A.x - B.x) * half, (A.y + B.y) * half};  // (A - conj B) / 2
    const C P = cmul(w, Dm);
    o[(long)k * out_ks] = cfrom_d<OutC>(to_cd(C{E.x + P.y, E.y - P.x}));  // E - iP
    if (both) o[(long)(N - k) * out_ks] = cfrom_d<OutC>(to_cd(C{E.x - P.y, -(E.y + P.x)}));  // conj(E + iP)
  };
  if (t != 0) {
    const C wa = __ldg(tw + ja);  // w^ja (base table, L = 2N)
#pragma unroll
    for (int q = 0; q < RX; ++q) emit(a[q], b[RX - 1 - q], q == 0 ? wa : cmul(wa, half_turn10<R>(q)), ja + q * NR, true);
  } else {
    emit(a[0], a[0], C{R(1), R(0)}, 0, true);  // X_0 and X_N
#pragma unroll
    for (int q = 1; q < RX / 2; ++q) emit(a[q], a[RX - q], half_turn10<R>(q), q * NR, true);
    emit(a[RX / 2], a[RX / 2], half_turn10<R>(RX / 2), N / 2, false);
    const C wb = __ldg(tw + NR / 2);
#pragma unroll
    for (int q = 0; q < RX / 2; ++q)
      emit(b[q], b[RX - 1 - q], q == 0 ? wb : cmul(wb, half_turn10<R>(q)), NR / 2 + q * NR, true);
  }
}

// Phases 4-5 + reorder for TOSI input in[k*in_ks + s] and SOTI output
// out[s*out_ss + t], t < N (the first half of the L = 2N samples: the
// matvec's unpad stage); N = 1000, S series per CTA.
template <int C3, int C4, class Tout, int S, int MINB>
__global__ void __launch_bounds__(S * 50, MINB)
    k_c2r_pair(const typename PT<C3>::cplx* __restrict__ in, long in_ks, long nseries, bool vec,
               Tout* __restrict__ out, long out_ss, const typename PT<C3>::cplx* __restrict__ tw) {
  using R = typename PT<C3>::real;
  using C = typename CT<R>::c;
  constexpr int RX = 10, N = 1000, NR = 100;
  constexpr int SS = pair_series_stride<C>();
  extern __shared__ __align__(16) unsigned char pair_smem_c2r[];
  C* sbuf = reinterpret_cast<C*>(pair_smem_c2r);
  const int s = threadIdx.x % S, t = threadIdx.x / S;
  const long s0 = (long)blockIdx.x * S;
  const int ns = (int)min((long)S, nseries - s0);
  const bool act = s < ns;
  const int ja = t, jb = t == 0 ? NR / 2 : NR - t;
  C* buf = sbuf + s * SS;
  C a[RX], b[RX];
  grid_dep_wait();  // (PDL)
  const R inv_len = R(1) / (R)(2 * N);

  // Pre-pass fused into pass 1, bins straight from global memory.
  {
    const C* p = in + s0 + (act ? s : 0);
    auto ld = [&](int k) {  // X_k * (1/L) in C3 arithmetic; Im X_0 = Im X_N = 0
      C x = act ? p[(long)k * in_ks] : C{R(0), R(0)};
      x.x = x.x * inv_len;
      x.y = (k == 0 || k == N) ? R(0) : x.y * inv_len;
      return x;
    };
#pragma unroll
    for (int q = 0; q < RX; ++q) {
      a[q] = ld(ja + q * NR);
      b[q] = ld(jb + q * NR);
    }
    // In place on a pair of slots: (X_n, X_{N-n}) -> (Z_n, Z_{N-n}), with
    // A = X_n, B = conj X_{N-n}, w = w^n.
    auto pre = [&](C& xn, C& xm, C w) {
      const C A = xn, B = cconj(xm);
      const C Sm = cadd(A, B);
      const C Q = cmul(C{w.x, -w.y}, csub(A, B));
      xn = C{Sm.x - Q.y, Sm.y + Q.x};     // S + iQ
      xm = C{Sm.x + Q.y, -(Sm.y - Q.x)};  // conj(S - iQ)
    };
    if (t != 0) {
      const C wa = __ldg(tw + ja);
#pragma unroll
      for (int q = 0; q < RX; ++q) pre(a[q], b[RX - 1 - q], q == 0 ? wa : cmul(wa, half_turn10<R>(q)));
    } else {
      C xN = ld(N);
      pre(a[0], xN, C{R(1), R(0)});
#pragma unroll
      for (int q = 1; q < RX / 2; ++q) pre(a[q], a[RX - q], half_turn10<R>(q));
      C a5 = a[RX / 2];
      pre(a[RX / 2], a5, half_turn10<R>(RX / 2));
      const C wb = __ldg(tw + NR / 2);
#pragma unroll
      for (int q = 0; q < RX / 2; ++q) pre(b[q], b[RX - 1 - q], q == 0 ? wb : cmul(wb, half_turn10<R>(q)));
    }
    butterfly<R, 1, RX>(a);
    butterfly<R, 1, RX>(b);
    if (act) {
      const int d = t & 1;
      store10_swz(buf + ja * RX, a, d);
      store10_swz(buf + jb * RX, b, d);
    }
    __syncthreads();
  }
  pair_pass2<R, 1>(buf, ja, jb, a, b, tw, act);
  if (!act) return;
  pair_pass3<R, 1>(buf, ja, jb, a, b, tw);
  Tout* po = out + (s0 + s) * out_ss;
  // (nout = N: only n < N/2, i.e. q < 5, is kept -- the unpad stage)
  auto put = [&](const C* v, int j) {
#pragma unroll
    for (int q = 0; q < RX / 2; ++q) {
      const int n = j + q * NR;
      const Tout x0 = (Tout)rnd<C4>((double)v[q].x);
      const Tout x1 = (Tout)rnd<C4>((double)v[q].y);
      if constexpr (sizeof(Tout) == 8) {
        if (vec) {
          reinterpret_cast<double2*>(po)[n] = make_double2(x0, x1);
          continue;
        }
      }
      po[2 * n] = x0;
      po[2 * n + 1] = x1;
    }
  };
  put(a, ja);
  put(b, jb);
}

}  // namespace fmv
