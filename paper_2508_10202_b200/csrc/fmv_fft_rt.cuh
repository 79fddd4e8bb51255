// fmv_fft_rt.cuh -- batched real FFTs of any even length L = 2N (fft.hpp:32-95
// plans every even L) on sm_100a, for the lengths the two Nt-specialised
// register kernels of fmv_fft.cuh (N = 1000, 100) do not cover.
//
// Two kernel families, both fusing the pipeline's pad / cast / reorder /
// unpad passes into their global loads and stores exactly as k_r2c_reg /
// k_c2r_reg do (matvec.hpp:83-205):
//
// * k_r2c_rt / k_c2r_rt -- register-resident in-place Stockham with a
//   RUNTIME plan (RtPlan): N = R_0 * RR^(np-1), R_0 (run time) and RR
//   (compile time, one kernel per RR) from {2, 3, 4, 5, 7, 8, 10, 16}.
//   Each thread owns at most floor(16 / R_p) butterflies of pass p (so it holds <= 16 complex values across the pass
//   barrier), one shared buffer of N (+1) complex per series, so a
//   series fits up to ~14 k fp64 points in the 227 KB of a CTA. The first r2c
//   pass reads global memory directly, the last c2r pass writes it directly.
// * k_fft_g* -- global-memory Stockham for everything else (series too long
//   for shared memory, prime factors > 7): a pack kernel, one kernel per
//   radix pass (any radix; primes through an O(r) per-output DFT), and an
//   unpack kernel, over a scratch buffer in HBM.
#pragma once

#include "fmv_fft.cuh"
#include "fmv_fft_plan.cuh"

namespace fmv {

// Runtime-precision rounding for the rt / global kernels (not the hot path):
// c in {PD, PS, PH}; same RNE roundings as rnd<P> (precision.hpp:44-61).
__device__ __forceinline__ double rnd_rt(int c, double v) {
  return c == PD ? v : c == PS ? rnd<PS>(v) : rnd<PH>(v);
}
// Store a complex value rounded to precision c into an output array of that precision.
__device__ __forceinline__ void store_c(void* out, long idx, int c, double2 v) {
  if (c == PD) static_cast<double2*>(out)[idx] = v;
  else if (c == PS) static_cast<float2*>(out)[idx] = cfrom_d<float2>(v);
  else static_cast<__half2*>(out)[idx] = cfrom_d<__half2>(v);
}

// 7-point DFT, direction D, by conjugate-pair symmetry (as the radix-5
// butterfly): t_j = v_j + v_{7-j}, u_j = v_j - v_{7-j}, j = 1..3;
// X_k = v_0 + sum_j cos(2 pi jk/7) t_j + D i sum_j sin(2 pi jk/7) u_j, k = 1..3,
// X_{7-k} the conjugate-sign twin.
template <class R, int D>
__device__ __forceinline__ void butterfly7(typename CT<R>::c* v) {
  using C = typename CT<R>::c;
  const R c1 = R(0.62348980185873353052500488400423981), c2 = R(-0.22252093395631440428890256449679476),
          c3 = R(-0.90096886790241912623610231950744505);
  const R s1 = R(0.78183148246802980870844452667405775), s2 = R(0.97492791218182360701813168299393122),
          s3 = R(0.43388373911755812047576833284835875);
  const C t1 = cadd(v[1], v[6]), t2 = cadd(v[2], v[5]), t3 = cadd(v[3], v[4]);
  const C u1 = csub(v[1], v[6]), u2 = csub(v[2], v[5]), u3 = csub(v[3], v[4]);
  const C x0 = v[0];
  v[0] = {x0.x + t1.x + t2.x + t3.x, x0.y + t1.y + t2.y + t3.y};
  // k = 1: cos (c1, c2, c3), sin (s1, s2, s3); k = 2: (c2, c3, c1), (s2, -s3, -s1); k = 3: (c3, c1, c2), (s3, -s1, s2)
  auto out = [&](R a1, R a2, R a3, R b1, R b2, R b3, int k) {
    const C a = {x0.x + a1 * t1.x + a2 * t2.x + a3 * t3.x, x0.y + a1 * t1.y + a2 * t2.y + a3 * t3.y};
    const C b = cmuli<D>(C{b1 * u1.x + b2 * u2.x + b3 * u3.x, b1 * u1.y + b2 * u2.y + b3 * u3.y});
    v[k] = cadd(a, b);
    v[7 - k] = csub(a, b);
  };
  out(c1, c2, c3, s1, s2, s3, 1);
  out(c2, c3, c1, s2, -s3, -s1, 2);
  out(c3, c1, c2, s3, -s1, s2, 3);
}

template <class R, int D, int Rn>
__device__ __forceinline__ void butterfly_any(typename CT<R>::c* v) {
  if constexpr (Rn == 7) butterfly7<R, D>(v);
  else butterfly<R, D, Rn>(v);
}

// v[q] *= w^(q*k) from pass table twp[q*Ns + k]. fp64 forms the powers of one
// table read (w1^q by repeated products, <= ~15 ulp at q = 15: far inside the
// 1e-12 contract); fp32 reads every power exactly from the table.
template <class R, int D, int Rn>
__device__ __forceinline__ void twiddle_rt(typename CT<R>::c* v, const typename CT<R>::c* __restrict__ twp, int k,
                                           int Ns) {
  using C = typename CT<R>::c;
  if constexpr (sizeof(R) == 8) {
    const C w1 = twiddle<D>(twp, Ns + k);
    C w = w1;
#pragma unroll
    for (int q = 1; q < Rn; ++q) {
      v[q] = cmul(v[q], w);
      if (q + 1 < Rn) w = cmul(w, w1);
    }
  } else {
#pragma unroll
    for (int q = 1; q < Rn; ++q) v[q] = cmul(v[q], twiddle<D>(twp, q * Ns + k));
  }
}

// One in-place pass (Ns > 1) of radix Rn over this thread's butterflies
// b = j + i*TS (b < N/Rn): read, twiddle, DFT, barrier, write, barrier.
template <class R, int D, int Rn>
__device__ __forceinline__ void rt_pass(typename CT<R>::c* __restrict__ buf, int j, bool act, const RtPlan& P, int p,
                                        const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  constexpr int MB = rt_hold<Rn>();
  const int NB = P.N / Rn, Ns = P.Ns[p], TS = P.TS, bpt = P.bpt[p];
  const C* __restrict__ twp = tw + P.tw_off[p];
  C v[MB][Rn];
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int b = j + i * TS;
    if (act && i < bpt && b < NB) {
      const int k = b - P.ns_div[p].div(b) * Ns;
#pragma unroll
      for (int q = 0; q < Rn; ++q) v[i][q] = buf[b + q * NB];
      twiddle_rt<R, D, Rn>(v[i], twp, k, Ns);
      butterfly_any<R, D, Rn>(v[i]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int b = j + i * TS;
    if (act && i < bpt && b < NB) {
      const int k = b - P.ns_div[p].div(b) * Ns;
      const int o = (b - k) * Rn + k;
#pragma unroll
      for (int q = 0; q < Rn; ++q) buf[o + q * Ns] = v[i][q];
    }
  }
  __syncthreads();
}

// r2c pass 0 (Ns = 1): z[n] = v[2n] + i v[2n+1] read from global (pad + casts
// fused), DFT, stored to shared at b*Rn + q.
template <class R, int Rn, class Tin>
__device__ __forceinline__ void rt_first_r2c(typename CT<R>::c* __restrict__ buf, int j, bool act, const RtPlan& P,
                                             const Tin* __restrict__ p, long in_ts, int nvalid, bool vec, int c0) {
  using C = typename CT<R>::c;
  constexpr int MB = rt_hold<Rn>();
  const int NB = P.N / Rn, TS = P.TS, bpt = P.bpt[0];
  C v[MB][Rn];
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int b = j + i * TS;
    if (act && i < bpt && b < NB) {
#pragma unroll
      for (int q = 0; q < Rn; ++q) {
        const int n = b + q * NB, t0 = 2 * n;
        C z = {R(0), R(0)};
        if (t0 < nvalid) {
          bool done = false;
          if constexpr (sizeof(Tin) == 8) {
            if (vec) {
              const double2 pr = __ldg(reinterpret_cast<const double2*>(p) + n);
              z = C{(R)rnd_rt(c0, pr.x), (R)rnd_rt(c0, pr.y)};
              done = true;
            }
          }
          if (!done) {
            z.x = (R)rnd_rt(c0, to_d(p[(long)t0 * in_ts]));
            z.y = t0 + 1 < nvalid ? (R)rnd_rt(c0, to_d(p[(long)(t0 + 1) * in_ts])) : R(0);
          }
        }
        v[i][q] = z;
      }
      butterfly_any<R, -1, Rn>(v[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int b = j + i * TS;
    if (act && i < bpt && b < NB) {
#pragma unroll
      for (int q = 0; q < Rn; ++q) buf[b * Rn + q] = v[i][q];
    }
  }
  __syncthreads();
}

template <class R, class Tin>
__device__ __forceinline__ void rt_first_r2c_any(typename CT<R>::c* buf, int j, bool act, const RtPlan& P,
                                                 const Tin* p, long in_ts, int nvalid, bool vec, int c0) {
  switch (P.radix[0]) {
    case 2: rt_first_r2c<R, 2>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
    case 3: rt_first_r2c<R, 3>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
    case 4: rt_first_r2c<R, 4>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
    case 5: rt_first_r2c<R, 5>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
    case 7: rt_first_r2c<R, 7>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
    case 8: rt_first_r2c<R, 8>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
    case 10: rt_first_r2c<R, 10>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
    default: rt_first_r2c<R, 16>(buf, j, act, P, p, in_ts, nvalid, vec, c0); break;
  }
}

// Real-signal post-pass X[k] = E[k] + w^k (-i) D[k] (k = 0..N) on shared Z,
// stored rounded to C2 at out[k*out_ks + s*out_ss]; bins k and N-k share the
// two loads. TOSI (out_ss == 1): consecutive threads take consecutive series.
template <class R>
__device__ __forceinline__ void rt_post_r2c(const typename CT<R>::c* __restrict__ sbuf, const RtPlan& P, int ns,
                                            long s0, void* __restrict__ out, int c2, long out_ks, long out_ss,
                                            const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  const int N = P.N, S = P.S, T = blockDim.x;
  const R half = R(0.5);
  auto post = [&](C A, C B, int k) {  // B = conj(Z[N-k])
    const C E = {(A.x + B.x) * half, (A.y + B.y) * half};
    const C Dm = {(A.x - B.x) * half, (A.y - B.y) * half};
    return cadd(E, cmul(__ldg(tw + k), cmuli<-1>(Dm)));
  };
  const int npair = N / 2 + 1;
  for (int e = threadIdx.x; e < S * npair; e += T) {
    int k, si;
    if (out_ss == 1) {
      k = e / S;
      si = e - k * S;
    } else {
      si = e / npair;
      k = e - si * npair;
    }
    if (si >= ns) continue;
    const C* Z = sbuf + si * P.SS;
    const int kp = k == 0 ? N : N - k;
    const C A1 = Z[k == N ? 0 : k];
    const C A2 = Z[k == 0 ? 0 : N - k];
    store_c(out, (long)k * out_ks + (s0 + si) * out_ss, c2, to_cd(post(A1, cconj(A2), k)));
    if (kp != k) store_c(out, (long)kp * out_ks + (s0 + si) * out_ss, c2, to_cd(post(A2, cconj(A1), kp)));
  }
}

// Phases 1-2 + reorder for N = R_0 * RR^(np-1) with a register plan: input
// element (s, t) at in[s*in_ss + t*in_ts] rounded to c0 then to R (pad +
// convert fused), bin k of series s stored rounded to c2 at
// out[k*out_ks + s*out_ss]. The first pass's radix R_0 is chosen at run time;
// the later passes are all radix RR (a compile-time radix keeps the pass loop
// free of register spills).
template <class R, class Tin, int RR>
__global__ void __launch_bounds__(512, 1) k_r2c_rt(const Tin* __restrict__ in, long in_ss, long in_ts, long nseries,
                                                   int nvalid, bool vec, int c0, void* __restrict__ out, int c2,
                                                   long out_ks, long out_ss, const RtPlan Pk,
                                                   const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  extern __shared__ __align__(16) unsigned char rt_smem[];
  // (the plan is read with runtime pass indices: keep it in shared memory --
  // dynamic indexing of a kernel parameter would copy it to local memory)
  __shared__ RtPlan P;
  if (threadIdx.x == 0) P = Pk;
  __syncthreads();
  C* sbuf = reinterpret_cast<C*>(rt_smem);
  const int s = P.sfast ? threadIdx.x % P.S : threadIdx.x / P.TS;
  const int j = P.sfast ? threadIdx.x / P.S : threadIdx.x - s * P.TS;
  const long s0 = (long)blockIdx.x * P.S;
  const int ns = (int)min((long)P.S, nseries - s0);
  const bool act = s < ns;
  C* buf = sbuf + s * P.SS;
  grid_dep_wait();
  rt_first_r2c_any<R>(buf, j, act, P, in + (s0 + (act ? s : 0)) * in_ss, in_ts, nvalid, vec, c0);
  for (int p = 1; p < P.np; ++p) rt_pass<R, -1, RR>(buf, j, act, P, p, tw);
  rt_post_r2c<R>(sbuf, P, ns, s0, out, c2, out_ks, out_ss, tw);
}

// c2r pass 0 with the pre-pass fused: Z[n] = (X[n] + conj X[N-n]) + i w^-n
// (X[n] - conj X[N-n]) from the shared bins (1/L already applied), DFT (D = +1).
// If it is also the last pass (np == 1) it writes global memory.
template <class R, int Rn, class Tout>
__device__ __forceinline__ void rt_first_c2r(typename CT<R>::c* __restrict__ buf, int j, bool act, const RtPlan& P,
                                             const typename CT<R>::c* __restrict__ tw, Tout* __restrict__ po,
                                             int nout, int c4) {
  using C = typename CT<R>::c;
  constexpr int MB = rt_hold<Rn>();
  const int N = P.N, NB = N / Rn, TS = P.TS, bpt = P.bpt[0];
  C v[MB][Rn];
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int b = j + i * TS;
    if (act && i < bpt && b < NB) {
#pragma unroll
      for (int q = 0; q < Rn; ++q) {
        const int n = b + q * NB;
        const C A = buf[n];
        const C B = cconj(buf[N - n]);
        const C w = __ldg(tw + n);
        v[i][q] = cadd(cadd(A, B), cmuli<1>(cmul(C{w.x, -w.y}, csub(A, B))));
      }
      butterfly_any<R, 1, Rn>(v[i]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int b = j + i * TS;
    if (act && i < bpt && b < NB) {
      if (P.np == 1) {  // b < NB = 1: output index b + q*NB = q
#pragma unroll
        for (int q = 0; q < Rn; ++q) {
          const int t0 = 2 * (b + q * NB);
          if (t0 < nout) po[t0] = (Tout)rnd_rt(c4, (double)v[i][q].x);
          if (t0 + 1 < nout) po[t0 + 1] = (Tout)rnd_rt(c4, (double)v[i][q].y);
        }
      } else {
#pragma unroll
        for (int q = 0; q < Rn; ++q) buf[b * Rn + q] = v[i][q];
      }
    }
  }
  __syncthreads();
}

template <class R, class Tout>
__device__ __forceinline__ void rt_first_c2r_any(typename CT<R>::c* buf, int j, bool act, const RtPlan& P,
                                                 const typename CT<R>::c* tw, Tout* po, int nout, int c4) {
  switch (P.radix[0]) {
    case 2: rt_first_c2r<R, 2>(buf, j, act, P, tw, po, nout, c4); break;
    case 3: rt_first_c2r<R, 3>(buf, j, act, P, tw, po, nout, c4); break;
    case 4: rt_first_c2r<R, 4>(buf, j, act, P, tw, po, nout, c4); break;
    case 5: rt_first_c2r<R, 5>(buf, j, act, P, tw, po, nout, c4); break;
    case 7: rt_first_c2r<R, 7>(buf, j, act, P, tw, po, nout, c4); break;
    case 8: rt_first_c2r<R, 8>(buf, j, act, P, tw, po, nout, c4); break;
    case 10: rt_first_c2r<R, 10>(buf, j, act, P, tw, po, nout, c4); break;
    default: rt_first_c2r<R, 16>(buf, j, act, P, tw, po, nout, c4); break;
  }
}

// Last c2r pass (Ns = N/Rn, so b = k): output index b + q*NB straight to
// global, keeping t < nout, rounded to C4 (unpad, matvec.hpp:184-192).
template <class R, int Rn, class Tout>
__device__ __forceinline__ void rt_last_c2r(const typename CT<R>::c* __restrict__ buf, int j, bool act,
                                            const RtPlan& P, int p, const typename CT<R>::c* __restrict__ tw,
                                            Tout* __restrict__ po, int nout, int c4) {
  using C = typename CT<R>::c;
  constexpr int MB = rt_hold<Rn>();
  const int NB = P.N / Rn, Ns = P.Ns[p], TS = P.TS, bpt = P.bpt[p];
  const C* __restrict__ twp = tw + P.tw_off[p];
#pragma unroll
  for (int i = 0; i < MB; ++i) {
    const int b = j + i * TS;
    if (act && i < bpt && b < NB) {
      C v[Rn];
#pragma unroll
      for (int q = 0; q < Rn; ++q) v[q] = buf[b + q * NB];
      twiddle_rt<R, 1, Rn>(v, twp, b, Ns);
      butterfly_any<R, 1, Rn>(v);
#pragma unroll
      for (int q = 0; q < Rn; ++q) {
        const int t0 = 2 * (b + q * NB);
        if (t0 < nout) po[t0] = (Tout)rnd_rt(c4, (double)v[q].x);
        if (t0 + 1 < nout) po[t0 + 1] = (Tout)rnd_rt(c4, (double)v[q].y);
      }
    }
  }
}

// Phases 4-5 + reorder for N = R_0 * RR^(np-1) with a register plan: bin k of
// series s at in[k*in_ks + s*in_ss], output sample t of series s at
// out[s*out_ss + t], t < nout, rounded to c4.
template <class R, class Tout, int RR>
__global__ void __launch_bounds__(512, 1) k_c2r_rt(const typename CT<R>::c* __restrict__ in, long in_ks, long in_ss,
                                                   long nseries, int nout, int c4, Tout* __restrict__ out,
                                                   long out_ss, const RtPlan Pk,
                                                   const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  extern __shared__ __align__(16) unsigned char rt_smem[];
  __shared__ RtPlan P;  // (see k_r2c_rt)
  if (threadIdx.x == 0) P = Pk;
  __syncthreads();
  C* sbuf = reinterpret_cast<C*>(rt_smem);
  const int N = P.N, S = P.S, T = blockDim.x;
  const int s = threadIdx.x / P.TS, j = threadIdx.x - s * P.TS;
  const long s0 = (long)blockIdx.x * S;
  const int ns = (int)min((long)S, nseries - s0);
  const bool act = s < ns;
  C* buf = sbuf + s * P.SS;
  grid_dep_wait();
  const R inv_len = R(1) / (R)(2 * N);
  // bins -> shared (series-major), 1/L in R arithmetic, Im(X0) = Im(XN) = 0
  // (fft.hpp:130-148); TOSI input: consecutive threads take consecutive series
  for (int e = threadIdx.x; e < S * (N + 1); e += T) {
    int k, si;
    if (in_ss == 1) {
      k = e / S;
      si = e - k * S;
    } else {
      si = e / (N + 1);
      k = e - si * (N + 1);
    }
    if (si >= ns) continue;
    C X = in[(long)k * in_ks + (s0 + si) * in_ss];
    X.x = X.x * inv_len;
    X.y = (k == 0 || k == N) ? R(0) : X.y * inv_len;
    sbuf[si * P.SS + k] = X;
  }
  __syncthreads();
  Tout* po = out + (s0 + (act ? s : 0)) * out_ss;
  rt_first_c2r_any<R>(buf, j, act, P, tw, po, nout, c4);
  for (int p = 1; p + 1 < P.np; ++p) rt_pass<R, 1, RR>(buf, j, act, P, p, tw);
  if (P.np >= 2) rt_last_c2r<R, RR>(buf, j, act, P, P.np - 1, tw, po, nout, c4);
}

// ======================================================================
// Global-memory Stockham (any N, any prime factor): pack -> passes -> unpack
// over a scratch buffer of nser x N complex values per side.
// ======================================================================
// z[s, n] = rnd_C1(rnd_C0(x[2n])) + i rnd_C1(rnd_C0(x[2n+1])), zero past nvalid.
template <class R, class Tin>
__global__ void k_fft_gpack(const Tin* __restrict__ in, long in_ss, long in_ts, long nser, int N, int nvalid, int c0,
                            typename CT<R>::c* __restrict__ z) {
  using C = typename CT<R>::c;
  const long total = nser * (long)N;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    long s, n;
    if (in_ts == 1) {
      s = e / N;
      n = e - s * N;
    } else {  // time-outer input: consecutive threads take consecutive series
      n = e / nser;
      s = e - n * nser;
    }
    const Tin* p = in + s * in_ss;
    const long t0 = 2 * n;
    C v = {R(0), R(0)};
    if (t0 < nvalid) v.x = (R)rnd_rt(c0, to_d(p[t0 * in_ts]));
    if (t0 + 1 < nvalid) v.y = (R)rnd_rt(c0, to_d(p[(t0 + 1) * in_ts]));
    z[s * N + n] = v;
  }
}

// One Stockham pass of radix r (Ns = product of the earlier radices) from
// src to dst: fixed radices one thread per butterfly, any other r one thread
// per output (O(r) DFT). Twiddles exp(-+2 pi i m / L) from the base table.
template <class R, int D, int Rn>
__global__ void k_fft_gpass(const typename CT<R>::c* __restrict__ src, typename CT<R>::c* __restrict__ dst, long nser,
                            int N, int Ns, const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  const int NB = N / Rn;
  const int L = 2 * N, tstep = L / (Ns * Rn);
  const long total = nser * (long)NB;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long s = e / NB;
    const int b = (int)(e - s * NB), k = b % Ns;
    const C* in = src + s * N;
    C v[Rn];
#pragma unroll
    for (int q = 0; q < Rn; ++q) v[q] = in[b + q * NB];
    if (Ns > 1) {
#pragma unroll
      for (int q = 1; q < Rn; ++q) v[q] = cmul(v[q], twiddle<D>(tw, (int)(((long)q * k * tstep) % L)));
    }
    butterfly_any<R, D, Rn>(v);
    C* out = dst + s * N + (b - k) * Rn + k;
#pragma unroll
    for (int q = 0; q < Rn; ++q) out[q * Ns] = v[q];
  }
}

// (fp64 accumulation and twiddles for any working precision, as stage_generic)
template <class R, int D>
__global__ void k_fft_gpass_generic(const typename CT<R>::c* __restrict__ src, typename CT<R>::c* __restrict__ dst,
                                    long nser, int N, int r, int Ns, const double2* __restrict__ twd) {
  using C = typename CT<R>::c;
  const int NB = N / r, span = Ns * r, L = 2 * N, tstep = L / span;
  const long total = nser * (long)N;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long s = e / N;
    const int o = (int)(e - s * N);
    const int blk = o / span, rem = o - blk * span, q = rem / Ns, k = rem - q * Ns;
    const int j = blk * Ns + k;
    const long estep = k + (long)q * Ns;
    const C* in = src + s * N;
    double2 acc = {0.0, 0.0};
    for (int m = 0; m < r; ++m)
      acc = cadd(acc, cmul(to_cd(in[j + m * NB]), twiddle<D>(twd, (int)(((long)m * estep % span) * tstep))));
    dst[s * N + o] = C{(R)acc.x, (R)acc.y};
  }
}

// r2c post-pass from the scratch Z to the bins (rounded to C2).
template <class R>
__global__ void k_fft_gpost(const typename CT<R>::c* __restrict__ z, long nser, int N, void* __restrict__ out, int c2,
                            long out_ks, long out_ss, const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  const R half = R(0.5);
  const long total = nser * (long)(N + 1);
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    long s, k;
    if (out_ss == 1) {
      k = e / nser;
      s = e - k * nser;
    } else {
      s = e / (N + 1);
      k = e - s * (N + 1);
    }
    const C A = z[s * N + (k == N ? 0 : k)];
    const C B = cconj(z[s * N + (k == 0 ? 0 : N - k)]);
    const C E = {(A.x + B.x) * half, (A.y + B.y) * half};
    const C Dm = {(A.x - B.x) * half, (A.y - B.y) * half};
    store_c(out, k * out_ks + s * out_ss, c2, to_cd(cadd(E, cmul(__ldg(tw + k), cmuli<-1>(Dm)))));
  }
}

// c2r pre-pass from the bins (1/L, Im(X0) = Im(XN) = 0) to the scratch Z.
template <class R>
__global__ void k_fft_gpre(const typename CT<R>::c* __restrict__ in, long in_ks, long in_ss, long nser, int N,
                           typename CT<R>::c* __restrict__ z, const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  const R inv_len = R(1) / (R)(2 * N);
  const long total = nser * (long)N;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long s = e / N;
    const int n = (int)(e - s * N);
    C A = in[(long)n * in_ks + s * in_ss], B = in[(long)(N - n) * in_ks + s * in_ss];
    A.x *= inv_len;
    A.y = n == 0 ? R(0) : A.y * inv_len;
    B.x *= inv_len;
    B.y = n == 0 ? -R(0) : -(B.y * inv_len);  // conj; Im(XN) = 0
    const C w = __ldg(tw + n);
    z[s * N + n] = cadd(cadd(A, B), cmuli<1>(cmul(C{w.x, -w.y}, csub(A, B))));
  }
}

// c2r unpack: out[s, t] = rnd_C4(x[t]), t < nout.
template <class R, class Tout>
__global__ void k_fft_gunpack(const typename CT<R>::c* __restrict__ z, long nser, int N, int nout, int c4,
                              Tout* __restrict__ out, long out_ss) {
  const long total = nser * (long)nout;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long s = e / nout;
    const int t = (int)(e - s * nout);
    const auto v = z[s * N + (t >> 1)];
    out[s * out_ss + t] = (Tout)rnd_rt(c4, (double)((t & 1) ? v.y : v.x));
  }
}

}  // namespace fmv

