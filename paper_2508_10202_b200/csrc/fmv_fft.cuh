// fmv_fft.cuh -- batched length-2Nt real<->complex FFTs as shared-memory
// Stockham kernels for sm_100a, with the pipeline's pad / cast / reorder /
// unpad passes fused into their load and store loops.
//
// Replaces the reference's FFTW facade (fft.hpp:32-148) on the matvec path
// (matvec.hpp:83-205) and in operator setup (operator.hpp:99-125):
//   * forward: unnormalized, sign -1, half spectrum (fft.hpp:5-8);
//   * inverse: bins pre-scaled by 1/L in the working precision, then an
//     unnormalized c2r that ignores Im of the DC and Nyquist bins
//     (fft.hpp:130-148; FFTW half-complex semantics).
//
// Algorithm: a real series of length L = 2N is packed as N complex points
// z[n] = x[2n] + i x[2n+1]; a mixed-radix Stockham autosort FFT of length N
// (radix 8/4/2/5/3 butterflies, a generic O(r) per-output DFT pass for any
// other prime) runs ping-pong between two shared-memory buffers, and a
// split post-pass (forward) / pre-pass (inverse) converts between Z and the
// L/2+1 real-signal bins. One CTA owns S whole series, so every global
// access is one coalesced pass: SOTI or time-outer input, TOSI (bin-major)
// output for the per-bin GEMV, and the reverse for the inverse.
#pragma once

#include "fmv_common.cuh"
#include "fmv_fft_plan.cuh"

namespace fmv {

constexpr int kMaxStages = 24;

struct FftGeom {
  int N;  // complex length = L/2 = Nt
  int L;  // real length 2*Nt
  int nst;
  int radix[kMaxStages];
  FastDiv nr_div[kMaxStages];    // N / radix (work items per series)
  FastDiv ns_div[kMaxStages];    // Ns (product of earlier radices)
  FastDiv span_div[kMaxStages];  // Ns * radix
  FastDiv n_div, nb_div, nout_div;  // N, N + 1, output samples per series
};

template <class R>
struct RadixK;
template <>
struct RadixK<double> {
  static constexpr double s3 = 0.86602540378443864676372317075293618;   // sin(2pi/3)
  static constexpr double c51 = 0.30901699437494742410229341718281906;  // cos(2pi/5)
  static constexpr double c52 = -0.80901699437494742410229341718281906; // cos(4pi/5)
  static constexpr double s51 = 0.95105651629515357211643933337938214;  // sin(2pi/5)
  static constexpr double s52 = 0.58778525229247312916870595463907277;  // sin(4pi/5)
  static constexpr double r2 = 0.70710678118654752440084436210484904;   // sqrt(1/2)
  static constexpr double c10 = 0.80901699437494742410229341718281906;  // cos(2pi/10)
  static constexpr double s10 = 0.58778525229247312916870595463907277;  // sin(2pi/10)
  static constexpr double c16 = 0.92387953251128675612818318939678829;  // cos(2pi/16)
  static constexpr double s16 = 0.38268343236508977172845998403039887;  // sin(2pi/16)
};
template <>
struct RadixK<float> {
  static constexpr float s3 = 0.86602540378443864676372317075293618f;
  static constexpr float c51 = 0.30901699437494742410229341718281906f;
  static constexpr float c52 = -0.80901699437494742410229341718281906f;
  static constexpr float s51 = 0.95105651629515357211643933337938214f;
  static constexpr float s52 = 0.58778525229247312916870595463907277f;
  static constexpr float r2 = 0.70710678118654752440084436210484904f;
  static constexpr float c10 = 0.80901699437494742410229341718281906f;
  static constexpr float s10 = 0.58778525229247312916870595463907277f;
  static constexpr float c16 = 0.92387953251128675612818318939678829f;
  static constexpr float s16 = 0.38268343236508977172845998403039887f;
};

// In-register DFT of size Rn, direction D (-1 forward, +1 inverse).
template <class R, int D, int Rn>
__device__ __forceinline__ void butterfly(typename CT<R>::c* v) {
  using C = typename CT<R>::c;
  using K = RadixK<R>;
  if constexpr (Rn == 2) {
    const C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (Rn == 4) {
    const C t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const C t2 = cadd(v[1], v[3]), t3 = cmuli<D>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else if constexpr (Rn == 8) {
    C e[4] = {v[0], v[2], v[4], v[6]};
    C o[4] = {v[1], v[3], v[5], v[7]};
    butterfly<R, D, 4>(e);
    butterfly<R, D, 4>(o);
    // twiddles W8^k, k = 0..3, W8 = exp(D*2*pi*i/8)
    const C o1 = {K::r2 * (o[1].x - D * o[1].y), K::r2 * (o[1].y + D * o[1].x)};
    const C o2 = cmuli<D>(o[2]);
    const C o3 = {K::r2 * (-o[3].x - D * o[3].y), K::r2 * (-o[3].y + D * o[3].x)};
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  } else if constexpr (Rn == 10) {
    // 10 = 2 x 5 (Cooley-Tukey): two 5-point DFTs, then X[k] = E[k] + W10^k O[k],
    // X[k+5] = E[k] - W10^k O[k], W10 = exp(D*2*pi*i/10).
    C e[5] = {v[0], v[2], v[4], v[6], v[8]};
    C o[5] = {v[1], v[3], v[5], v[7], v[9]};
    butterfly<R, D, 5>(e);
    butterfly<R, D, 5>(o);
    const R c1 = K::c10, s1 = D * K::s10;  // W10^1 = (cos 36, D sin 36)
    const R c2 = K::c51, s2 = D * K::s51;  // W10^2 = (cos 72, D sin 72)
    const C t1 = {c1 * o[1].x - s1 * o[1].y, c1 * o[1].y + s1 * o[1].x};
    const C t2 = {c2 * o[2].x - s2 * o[2].y, c2 * o[2].y + s2 * o[2].x};
    const C t3 = {-c2 * o[3].x - s2 * o[3].y, -c2 * o[3].y + s2 * o[3].x};  // W10^3 = (-cos 72, D sin 72)
    const C t4 = {-c1 * o[4].x - s1 * o[4].y, -c1 * o[4].y + s1 * o[4].x};  // W10^4 = (-cos 36, D sin 36)
    v[0] = cadd(e[0], o[0]);
    v[5] = csub(e[0], o[0]);
    v[1] = cadd(e[1], t1);
    v[6] = csub(e[1], t1);
    v[2] = cadd(e[2], t2);
    v[7] = csub(e[2], t2);
    v[3] = cadd(e[3], t3);
    v[8] = csub(e[3], t3);
    v[4] = cadd(e[4], t4);
    v[9] = csub(e[4], t4);
  } else if constexpr (Rn == 16) {
    // 16 = 4 x 4: four 4-point DFTs on the decimated inputs, twiddles W16^(a*b), four more.
    C a[4][4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int c = 0; c < 4; ++c) a[r][c] = v[c * 4 + r];
      butterfly<R, D, 4>(a[r]);
    }
    // a[r][k1] *= W16^(r*k1)
    const R cs8 = K::r2, c16 = K::c16, s16 = K::s16;
    auto rot = [&](C x, R c, R s) { return C{c * x.x - D * s * x.y, c * x.y + D * s * x.x}; };
    a[1][1] = rot(a[1][1], c16, s16);
    a[1][2] = rot(a[1][2], cs8, cs8);
    a[1][3] = rot(a[1][3], s16, c16);
    a[2][1] = rot(a[2][1], cs8, cs8);
    a[2][2] = cmuli<D>(a[2][2]);
    a[2][3] = rot(a[2][3], -cs8, cs8);
    a[3][1] = rot(a[3][1], s16, c16);
    a[3][2] = rot(a[3][2], -cs8, cs8);
    a[3][3] = rot(a[3][3], -c16, -s16);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      C b[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
      butterfly<R, D, 4>(b);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = b[k2];
    }
  } else if constexpr (Rn == 3) {
    const C t = cadd(v[1], v[2]);
    const C u = csub(v[1], v[2]);
    const C a = {v[0].x - R(0.5) * t.x, v[0].y - R(0.5) * t.y};
    const C su = cmuli<D>(C{K::s3 * u.x, K::s3 * u.y});
    v[0] = cadd(v[0], t);
    v[1] = cadd(a, su);
    v[2] = csub(a, su);
  } else if constexpr (Rn == 5) {
    const C t1 = cadd(v[1], v[4]), t2 = cadd(v[2], v[3]);
    const C t3 = csub(v[1], v[4]), t4 = csub(v[2], v[3]);
    const C b1 = {v[0].x + K::c51 * t1.x + K::c52 * t2.x, v[0].y + K::c51 * t1.y + K::c52 * t2.y};
    const C b2 = {v[0].x + K::c52 * t1.x + K::c51 * t2.x, v[0].y + K::c52 * t1.y + K::c51 * t2.y};
    const C d1 = cmuli<D>(C{K::s51 * t3.x + K::s52 * t4.x, K::s51 * t3.y + K::s52 * t4.y});
    const C d2 = cmuli<D>(C{K::s52 * t3.x - K::s51 * t4.x, K::s52 * t3.y - K::s51 * t4.y});
    v[0] = {v[0].x + t1.x + t2.x, v[0].y + t1.y + t2.y};
    v[1] = cadd(b1, d1);
    v[4] = csub(b1, d1);
    v[2] = cadd(b2, d2);
    v[3] = csub(b2, d2);
  }
}

// tw[e] = exp(-2*pi*i*e/L); the inverse uses its conjugate.
template <int D, class C>
__device__ __forceinline__ C twiddle(const C* __restrict__ tw, int e) {
  const C w = __ldg(tw + e);
  if constexpr (D < 0) return w;
  else return C{w.x, -w.y};
}

template <class R, int D, int Rn>
__device__ __forceinline__ void stage_fixed(const typename CT<R>::c* __restrict__ src, typename CT<R>::c* __restrict__ dst,
                                            int ss, int ns, int Ns, const FastDiv& nrd, const FastDiv& nsd,
                                            const typename CT<R>::c* __restrict__ tw, int N, int L) {
  using C = typename CT<R>::c;
  const int Nr = N / Rn;
  const int tstep = L / (Ns * Rn);
  for (int it = threadIdx.x; it < ns * Nr; it += blockDim.x) {
    const int s = nrd.div(it);
    const int j = it - s * Nr;
    const int k = j - nsd.div(j) * Ns;
    const C* in = src + s * ss;
    C v[Rn];
#pragma unroll
    for (int q = 0; q < Rn; ++q) v[q] = in[j + q * Nr];
    if (Ns > 1) {
      const int kt = k * tstep;
#pragma unroll
      for (int q = 1; q < Rn; ++q) v[q] = cmul(v[q], twiddle<D>(tw, q * kt));
    }
    butterfly<R, D, Rn>(v);
    C* out = dst + s * ss + (j - k) * Rn + k;
#pragma unroll
    for (int q = 0; q < Rn; ++q) out[q * Ns] = v[q];
  }
}

// Any radix r (used for primes other than 2,3,5): one thread per output,
// an O(r) DFT accumulated in fp64 with the fp64 twiddle table `twd` whatever
// the working precision R, then rounded to R once. (A long fp32 sum over a
// large prime -- n_t = 1009 -- would otherwise lose ~sqrt(r) ulps against the
// reference's FFTW-style single-precision transform.)
template <class R, int D>
__device__ __forceinline__ void stage_generic(const typename CT<R>::c* __restrict__ src,
                                              typename CT<R>::c* __restrict__ dst, int ss, int ns, int r, int Ns,
                                              const FastDiv& nd, const FastDiv& nsd, const FastDiv& spand,
                                              const double2* __restrict__ twd, int N, int L) {
  using C = typename CT<R>::c;
  const int Nr = N / r;
  const int span = Ns * r;
  const int tstep = L / span;
  for (int it = threadIdx.x; it < ns * N; it += blockDim.x) {
    const int s = nd.div(it);
    const int o = it - s * N;
    const int blk = spand.div(o);
    const int rem = o - blk * span;
    const int q = nsd.div(rem);
    const int k = rem - q * Ns;
    const int j = blk * Ns + k;
    const int estep = k + q * Ns;
    const C* in = src + s * ss;
    double2 acc = {0.0, 0.0};
    int e = 0;
    for (int m = 0; m < r; ++m) {
      const double2 x = to_cd(in[j + m * Nr]);
      acc = cadd(acc, cmul(x, twiddle<D>(twd, e * tstep)));
      e += estep;
      if (e >= span) e -= span * (e / span);
    }
    dst[s * ss + o] = C{(R)acc.x, (R)acc.y};
  }
}

// Runs all stages; returns the buffer holding the result.
template <class R, int D>
__device__ typename CT<R>::c* run_stages(typename CT<R>::c* a, typename CT<R>::c* b, int ss, int ns, const FftGeom& g,
                                         const typename CT<R>::c* __restrict__ tw, const double2* __restrict__ twd) {
  int Ns = 1;
  for (int st = 0; st < g.nst; ++st) {
    const int r = g.radix[st];
    switch (r) {
      case 2: stage_fixed<R, D, 2>(a, b, ss, ns, Ns, g.nr_div[st], g.ns_div[st], tw, g.N, g.L); break;
      case 3: stage_fixed<R, D, 3>(a, b, ss, ns, Ns, g.nr_div[st], g.ns_div[st], tw, g.N, g.L); break;
      case 4: stage_fixed<R, D, 4>(a, b, ss, ns, Ns, g.nr_div[st], g.ns_div[st], tw, g.N, g.L); break;
      case 5: stage_fixed<R, D, 5>(a, b, ss, ns, Ns, g.nr_div[st], g.ns_div[st], tw, g.N, g.L); break;
      case 8: stage_fixed<R, D, 8>(a, b, ss, ns, Ns, g.nr_div[st], g.ns_div[st], tw, g.N, g.L); break;
      default:
        stage_generic<R, D>(a, b, ss, ns, r, Ns, g.n_div, g.ns_div[st], g.span_div[st], twd, g.N, g.L);
        break;
    }
    __syncthreads();
    typename CT<R>::c* t = a;
    a = b;
    b = t;
    Ns *= r;
  }
  return a;
}

// Phases 1-2 (+ the SOTI->TOSI reorder of phase 3), fused:
//   v = rnd_C1(rnd_C0(in[s, t])) for t < nvalid (= Nt), 0 up to L  (matvec.hpp:84-90, :118-130)
//   X = r2c_L(v) in C1 arithmetic                                  (matvec.hpp:132-141)
//   out[k, s] = rnd_C2(X[k])                                       (matvec.hpp:155-165)
// Input element (s,t) at in[s*in_ss + t*in_ts]; output bin k of series s at
// out[k*out_ks + s*out_ss]. One CTA per S (a power of two) consecutive series.
template <int C0, int C1, int C2, class Tin>
__global__ void __launch_bounds__(256) k_r2c(const Tin* __restrict__ in, long in_ss, long in_ts, long nseries, int nvalid,
                                             typename PT<C2>::cplx* __restrict__ out, long out_ks, long out_ss,
                                             FftGeom g, const typename CT<typename PT<C1>::real>::c* __restrict__ tw,
                                             const double2* __restrict__ twd, int lgS) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  using OutC = typename PT<C2>::cplx;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = 1 << lgS;
  const int N = g.N;
  const int ss = N + 1;
  C* bufA = reinterpret_cast<C*>(smem_raw);
  C* bufB = bufA + S * ss;
  const long s0 = (long)blockIdx.x * S;
  const int ns = (int)min((long)S, nseries - s0);

  // Loads are batched U per thread (all issued before any shared store) so a
  // CTA pays the DRAM latency about once, not once per loop trip.
  constexpr int U = 4;
  const int T = blockDim.x;
  if (in_ts == 1) {
    bool vec = false;
    if constexpr (sizeof(Tin) == 8) {
      vec = (in_ss % 2 == 0) && (nvalid % 2 == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
    }
    const int total = ns * N;
    for (int base = threadIdx.x; base < total; base += U * T) {
      C v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * T;
        v[u] = C{R(0), R(0)};
        if (e < total) {
          const int s = g.n_div.div(e), n = e - s * N;
          const Tin* p = in + (s0 + s) * in_ss;
          const int t0 = 2 * n;
          if (vec) {
            if (t0 < nvalid) {
              const double2 pr = __ldg(reinterpret_cast<const double2*>(p) + n);
              v[u] = C{(R)rnd<C0>(pr.x), (R)rnd<C0>(pr.y)};
            }
          } else {
            const R a = t0 < nvalid ? (R)rnd<C0>(to_d(p[t0])) : R(0);
            const R b = t0 + 1 < nvalid ? (R)rnd<C0>(to_d(p[t0 + 1])) : R(0);
            v[u] = C{a, b};
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * T;
        if (e < total) {
          const int s = g.n_div.div(e), n = e - s * N;
          bufA[s * ss + n] = v[u];
        }
      }
    }
  } else {
    const int total = S * N;
    for (int base = threadIdx.x; base < total; base += U * T) {
      C v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * T;
        const int n = e >> lgS, s = e & (S - 1);
        v[u] = C{R(0), R(0)};
        if (e < total && s < ns) {
          const Tin* p = in + (s0 + s) * in_ss;
          const int t0 = 2 * n, t1 = 2 * n + 1;
          const R a = t0 < nvalid ? (R)rnd<C0>(to_d(p[(long)t0 * in_ts])) : R(0);
          const R b = t1 < nvalid ? (R)rnd<C0>(to_d(p[(long)t1 * in_ts])) : R(0);
          v[u] = C{a, b};
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = base + u * T;
        const int n = e >> lgS, s = e & (S - 1);
        if (e < total && s < ns) bufA[s * ss + n] = v[u];
      }
    }
  }
  __syncthreads();
  const C* Z = run_stages<R, -1>(bufA, bufB, ss, ns, g, tw, twd);

  // Real-signal post-pass: X[k] = E[k] + w^k * (-i) * D[k], k = 0..N.
  const R half = R(0.5);
  const int nbins = N + 1;
  auto post = [&](int s, int k) {
    const C A = Z[s * ss + (k == N ? 0 : k)];
    const C B = cconj(Z[s * ss + (k == 0 ? 0 : N - k)]);
    const C E = {(A.x + B.x) * half, (A.y + B.y) * half};
    const C Dm = {(A.x - B.x) * half, (A.y - B.y) * half};
    const C X = cadd(E, cmul(__ldg(tw + k), cmuli<-1>(Dm)));
    out[(long)k * out_ks + (s0 + s) * out_ss] = cfrom_d<OutC>(to_cd(X));
  };
  if (out_ss == 1) {  // bin-major (TOSI): consecutive threads -> consecutive series
    for (int e = threadIdx.x; e < S * nbins; e += blockDim.x) {
      const int k = e >> lgS, s = e & (S - 1);
      if (s < ns) post(s, k);
    }
  } else {
    for (int e = threadIdx.x; e < ns * nbins; e += blockDim.x) {
      const int s = g.nb_div.div(e), k = e - s * nbins;
      post(s, k);
    }
  }
}

// Phases 4-5 (+ the TOSI->SOTI reorder of phase 3), fused:
//   Xs = in[k, s] * (1/L) in C3 arithmetic, Im(X0)=Im(XN)=0        (fft.hpp:130-148)
//   x = c2r_L(Xs) in C3 arithmetic
//   out[s, t] = (double) rnd_C4(x[t]), t < nout (= Nt)             (matvec.hpp:184-192)
template <int C3, int C4, class Tout>
__global__ void __launch_bounds__(256) k_c2r(const typename PT<C3>::cplx* __restrict__ in, long in_ks, long in_ss,
                                             long nseries, int nout, Tout* __restrict__ out, long out_ss, FftGeom g,
                                             const typename PT<C3>::cplx* __restrict__ tw,
                                             const double2* __restrict__ twd, int lgS) {
  using R = typename PT<C3>::real;
  using C = typename CT<R>::c;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = 1 << lgS;
  const int N = g.N;
  const int ss = N + 1;
  C* bufA = reinterpret_cast<C*>(smem_raw);
  C* bufB = bufA + S * ss;
  const long s0 = (long)blockIdx.x * S;
  const int ns = (int)min((long)S, nseries - s0);
  const R inv_len = R(1) / (R)g.L;
  const int nbins = N + 1;
  auto fix = [&](C X, int k) {
    X.x = X.x * inv_len;
    X.y = (k == 0 || k == N) ? R(0) : X.y * inv_len;
    return X;
  };
  constexpr int U = 4;
  const int T = blockDim.x;
  const bool tosi = in_ss == 1;
  const int total = tosi ? S * nbins : ns * nbins;
  for (int base = threadIdx.x; base < total; base += U * T) {
    C v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * T;
      int s, k;
      if (tosi) {
        k = e >> lgS;
        s = e & (S - 1);
      } else {
        s = g.nb_div.div(e);
        k = e - s * nbins;
      }
      if (e < total && s < ns) v[u] = in[(long)k * in_ks + (s0 + s) * in_ss];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = base + u * T;
      int s, k;
      if (tosi) {
        k = e >> lgS;
        s = e & (S - 1);
      } else {
        s = g.nb_div.div(e);
        k = e - s * nbins;
      }
      if (e < total && s < ns) bufA[s * ss + k] = fix(v[u], k);
    }
  }
  __syncthreads();
  // Z[k] = (X[k] + conj X[N-k]) + i * w^-k * (X[k] - conj X[N-k])
  for (int e = threadIdx.x; e < ns * N; e += blockDim.x) {
    const int s = g.n_div.div(e), k = e - s * N;
    const C A = bufA[s * ss + k];
    const C B = cconj(bufA[s * ss + N - k]);
    const C w = __ldg(tw + k);
    const C Z = cadd(cadd(A, B), cmuli<1>(cmul(C{w.x, -w.y}, csub(A, B))));
    bufB[s * ss + k] = Z;
  }
  __syncthreads();
  const C* z = run_stages<R, 1>(bufB, bufA, ss, ns, g, tw, twd);
  for (int e = threadIdx.x; e < ns * nout; e += blockDim.x) {
    const int s = g.nout_div.div(e), t = e - s * nout;
    const C v = z[s * ss + (t >> 1)];
    out[(s0 + s) * out_ss + t] = (Tout)rnd<C4>((double)((t & 1) ? v.y : v.x));
  }
}

// ======================================================================
// Register-resident kernels for N = RX^NP (N = 1000 = 10^3, 100 = 10^2,
// 256 = 16^2, 4096 = 16^3, 512 = 8^3 ...): the matvec hot path.
//
// Each thread owns ONE radix-RX butterfly per pass (T = S * N/RX threads for
// S series), so a pass is: read RX values, twiddle, DFT-RX in registers,
// barrier, write in place, barrier -- one shared-memory round trip per pass
// instead of a ping-pong buffer per radix-2/4/8/5 stage. The r2c first pass
// reads straight from global memory (the pass-1 Stockham read pattern
// z[j + q*N/RX] is contiguous across j) and the c2r last pass writes straight
// to global memory (its write pattern z[j + q*N/RX] is contiguous too), so
// r2c costs NP smem round trips + the bin post-pass and c2r the bin pre-pass
// + NP - 1. Twiddles are index-exact table reads (the table of
// exp(-2*pi*i*m/L) the legacy kernel uses), so both kernels compute the same
// DFT; summation order differs (radix-10 vs 8/5 stages), rounding-level.
// ======================================================================
// cp.async (LDGSTS) helpers: global -> shared without register staging.
__device__ __forceinline__ void cp_async(void* dst, const void* src, int bytes_valid, int size) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  if (size == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(bytes_valid) : "memory");
  else if (size == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(bytes_valid) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(bytes_valid) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int I, int RX>
struct IPow {
  static constexpr int v = RX * IPow<I - 1, RX>::v;
};
template <int RX>
struct IPow<0, RX> {
  static constexpr int v = 1;
};

// N = R0 * RX^(NP-1): a first pass of radix R0 (R0 divides RX; each thread
// then does RX/R0 radix-R0 butterflies of it), the other NP-1 passes radix RX.
// R0 = RX is the uniform plan (1000 = 10^3, 100 = 10^2, 512 = 8^3, 4096 = 16^3);
// mixed ones cover 1024 = 4*16^2, 2048 = 8*16^2, 8192 = 2*16^3, 2000 = 2*10^3.
template <int RX, int NP, int R0 = RX>
struct RegPlan {
  static_assert(RX % R0 == 0, "the first-pass radix must divide RX");
  static constexpr int N = R0 * IPow<NP - 1, RX>::v;
  static constexpr int NR = N / RX;  // threads per series (radix-RX butterflies per pass)
};

// Shared series stride: N rounded up so consecutive series start 128/S bytes
// apart modulo 128 (at least one element): the S-interleaved post/pre-pass
// (thread e -> bin e/S, series e%S) then spreads over distinct banks.
template <class C, int N, int S>
constexpr int reg_series_stride() {
  constexpr int E = (int)sizeof(C);
  constexpr int per128 = 128 / E;                        // elements per 128 B
  constexpr int off = (128 / S > E ? 128 / S : E) / E;   // target offset in elements
  int ss = N;
  while (ss % per128 != off % per128) ++ss;
  return ss;
}

// One Stockham pass with Ns > 1 over the thread's butterfly: read, twiddle,
// DFT, barrier, write, barrier.
// Offset of pass Ns's twiddle table [q*Ns + k] behind the 2N-entry base table.
template <int RX, int N, int Ns, int R0 = RX>
constexpr int reg_tw_offset() {
  int off = 2 * N;
  for (int ns = R0; ns < Ns; ns *= RX) off += RX * ns;
  return off;
}

// v[q] *= w^(q*k), q = 1..RX-1, from the pass table twp[q*Ns + k]. For
// RX = 10 only q = 1, 2, 3, 6 are read and the rest formed as one product of
// two table values (w4 = w1 w3, w5 = w2 w3, w7 = w1 w6, w8 = w2 w6,
// w9 = w3 w6: ~1 ulp), cutting the L1 twiddle traffic that bounds the pass.
// fp64 (the all-double hot path) reads only w1 and forms w2 = w1^2,
// w3 = w1 w2, w6 = w3^2 (<= ~6 ulp on w9, ~1e-15: far inside the 1e-12
// contract); fp32 keeps four exact table reads, as its tolerance is tied to
// the reference's own fp32 error.
template <class R, int D, int RX, int Ns>
__device__ __forceinline__ void apply_twiddles(typename CT<R>::c* v, const typename CT<R>::c* __restrict__ twp, int k) {
  if constexpr (RX == 10) {
    using C = typename CT<R>::c;
    C w1, w2, w3, w6;
    if constexpr (sizeof(R) == 8) {
      w1 = twiddle<D>(twp, Ns + k);
      w2 = cmul(w1, w1);
      w3 = cmul(w1, w2);
      w6 = cmul(w3, w3);
    } else {
      w1 = twiddle<D>(twp, Ns + k), w2 = twiddle<D>(twp, 2 * Ns + k);
      w3 = twiddle<D>(twp, 3 * Ns + k), w6 = twiddle<D>(twp, 6 * Ns + k);
    }
    v[1] = cmul(v[1], w1);
    v[2] = cmul(v[2], w2);
    v[3] = cmul(v[3], w3);
    v[4] = cmul(v[4], cmul(w1, w3));
    v[5] = cmul(v[5], cmul(w2, w3));
    v[6] = cmul(v[6], w6);
    v[7] = cmul(v[7], cmul(w1, w6));
    v[8] = cmul(v[8], cmul(w2, w6));
    v[9] = cmul(v[9], cmul(w3, w6));
  } else {
#pragma unroll
    for (int q = 1; q < RX; ++q) v[q] = cmul(v[q], twiddle<D>(twp, q * Ns + k));
  }
}

// exp(-i*pi*q/10), q = 0..9 (the c2r pre-pass factor w^(q*N/10) for L = 2N).
template <class R>
__device__ __forceinline__ typename CT<R>::c half_turn10(int q) {
  using K = RadixK<R>;
  const R cs[10] = {R(1), K::s51, K::c10, K::s10, K::c51, R(0), -K::c51, -K::s10, -K::c10, -K::s51};
  const R sn[10] = {R(0), K::c51, K::s10, K::c10, K::s51, R(1), K::s51, K::c10, K::s10, K::c51};
  return {cs[q], -sn[q]};
}

// Pass-1 store o[q] = v[q], q < RX, for thread j at o = buf + j*RX. With
// 16-byte elements and even RX, lanes t and t+4 of a quarter-warp would hit
// the same bank group for every q; lanes with (t>>2)&1 store the pair q^1
// first, which spreads the quarter over all 8 groups.
template <int RX, class C>
__device__ __forceinline__ void store_stride_rx(C* o, const C* v) {
  if constexpr (RX % 2 == 0 && sizeof(C) == 16) {
    const int d = (threadIdx.x >> 2) & 1;
#pragma unroll
    for (int q = 0; q < RX; ++q) o[q ^ d] = d ? v[q ^ 1] : v[q];
  } else {
#pragma unroll
    for (int q = 0; q < RX; ++q) o[q] = v[q];
  }
}

template <class R, int D, int RX, int N, int Ns, int R0 = RX>
__device__ __forceinline__ void reg_pass(typename CT<R>::c* __restrict__ buf, int j, bool act,
                                         const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  constexpr int NR = N / RX;
  const C* __restrict__ twp = tw + reg_tw_offset<RX, N, Ns, R0>();
  C v[RX];
  const int k = j % Ns;
  if (act) {
#pragma unroll
    for (int q = 0; q < RX; ++q) v[q] = buf[j + q * NR];
    apply_twiddles<R, D, RX, Ns>(v, twp, k);
    butterfly<R, D, RX>(v);
  }
  __syncthreads();
  if (act) {
    const int o = (j - k) * RX + k;
#pragma unroll
    for (int q = 0; q < RX; ++q) buf[o + q * Ns] = v[q];
  }
  __syncthreads();
}

// Radix-RX passes with Ns = NS, NS*RX, ... up to NLAST (inclusive).
template <class R, int D, int RX, int N, int R0, int NS, int NLAST>
__device__ __forceinline__ void reg_passes(typename CT<R>::c* __restrict__ buf, int j, bool act,
                                           const typename CT<R>::c* __restrict__ tw) {
  if constexpr (NS <= NLAST) {
    reg_pass<R, D, RX, N, NS, R0>(buf, j, act, tw);
    reg_passes<R, D, RX, N, R0, NS * RX, NLAST>(buf, j, act, tw);
  }
}

// Dynamic shared-memory bytes of the register kernels (host launch sizes).
template <class C, int RX, int NP, int S, int R0 = RX>
constexpr size_t r2c_reg_smem() {
  return (size_t)S * reg_series_stride<C, RegPlan<RX, NP, R0>::N, S>() * sizeof(C);
}
template <class C, int RX, int NP, int S, int R0 = RX>
constexpr size_t c2r_reg_smem() {
  return (size_t)S * reg_series_stride<C, RegPlan<RX, NP, R0>::N + 1, S>() * sizeof(C);
}
// resident CTAs the register kernels ask for (register cap)
template <int RX, int NP, int S, int R0>
constexpr int reg_min_blocks() {
  constexpr int T = S * RegPlan<RX, NP, R0>::NR;
  if constexpr (R0 != RX && T >= 512) return 1;
  return RX >= 16 ? 2 : T <= 256 ? 5 : 2;
}

// Phases 1-2 + reorder (as k_r2c) for SOTI input in[s*in_ss + t] and TOSI
// output out[k*out_ks + s]; S series per CTA.
template <int C0, int C1, int C2, class Tin, int RX, int NP, int S, int R0 = RX>
__global__ void __launch_bounds__(S * RegPlan<RX, NP, R0>::NR, reg_min_blocks<RX, NP, S, R0>())
    k_r2c_reg(const Tin* __restrict__ in, long in_ss, long nseries, int nvalid, bool vec,
              typename PT<C2>::cplx* __restrict__ out, long out_ks,
              const typename CT<typename PT<C1>::real>::c* __restrict__ tw) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  using OutC = typename PT<C2>::cplx;
  constexpr int N = RegPlan<RX, NP, R0>::N, NR = RegPlan<RX, NP, R0>::NR, T = S * NR;
  constexpr int U = RX / R0, NB = N / R0;  // pass-1 butterflies per thread, radix-R0 butterflies per series
  constexpr int SS = reg_series_stride<C, N, S>();
  extern __shared__ __align__(16) unsigned char reg_smem[];  // S * SS complex (dynamic: S*SS may exceed 48 KB)
  C* sbuf = reinterpret_cast<C*>(reg_smem);
  const int s = threadIdx.x / NR, j = threadIdx.x - s * NR;
  const long s0 = (long)blockIdx.x * S;
  const int ns = (int)min((long)S, nseries - s0);
  const bool act = s < ns;
  C* buf = sbuf + s * SS;
  grid_dep_wait();  // (PDL)

  // Pass 1 (Ns = 1, no twiddles): z[n] = v[2n] + i v[2n+1]; butterfly
  // b = j + u*NR (u < U) reads n = b + r*NB (r < R0) into v[u*R0 + r]
  // (R0 = RX: n = j + q*NR).
  {
    C v[RX];
    const Tin* p = in + (s0 + s) * in_ss;
#pragma unroll
    for (int q = 0; q < RX; ++q) {
      const int n = j + (q / R0) * NR + (q % R0) * NB;
      const int t0 = 2 * n;
      v[q] = C{R(0), R(0)};
      if (act && t0 < nvalid) {
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
        const R a = (R)rnd<C0>(to_d(p[t0]));
        const R b = t0 + 1 < nvalid ? (R)rnd<C0>(to_d(p[t0 + 1])) : R(0);
        v[q] = C{a, b};
      }
    }
    if constexpr (R0 == RX) {
      butterfly<R, -1, RX>(v);
      if (act) store_stride_rx<RX>(buf + j * RX, v);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) butterfly<R, -1, R0>(v + u * R0);
      if (act) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < R0; ++r) buf[(j + u * NR) * R0 + r] = v[u * R0 + r];
      }
    }
    __syncthreads();
  }
  reg_passes<R, -1, RX, N, R0, R0, NR>(buf, j, act, tw);

  // Post-pass: X[k] = E[k] + w^k (-i) D[k] with E, D from Z[k] and
  // conj Z[N-k]. Bins k and N-k (k = 0 pairs with N) share the two loads.
  // Consecutive threads take consecutive series of one bin pair (S-element
  // contiguous TOSI runs).
  const R half = R(0.5);
  auto post = [&](C A, C B, int k) {  // B = conj(Z[N-k])
    const C E = {(A.x + B.x) * half, (A.y + B.y) * half};
    const C Dm = {(A.x - B.x) * half, (A.y - B.y) * half};
    return cadd(E, cmul(__ldg(tw + k), cmuli<-1>(Dm)));
  };
  for (int e = threadIdx.x; e < S * (N / 2 + 1); e += T) {
    const int k = e / S, si = e - k * S;
    if (si >= ns) continue;
    const C* Z = sbuf + si * SS;
    const int kp = k == 0 ? N : N - k;
    const C A1 = Z[k];
    const C A2 = Z[k == 0 ? 0 : N - k];
    out[(long)k * out_ks + s0 + si] = cfrom_d<OutC>(to_cd(post(A1, cconj(A2), k)));
    if (kp != k) out[(long)kp * out_ks + s0 + si] = cfrom_d<OutC>(to_cd(post(A2, cconj(A1), kp)));
  }
}

// Phases 4-5 + reorder (as k_c2r) for TOSI input in[k*in_ks + s] and SOTI
// output out[s*out_ss + t], t < nout; S series per CTA.
template <int C3, int C4, class Tout, int RX, int NP, int S, int R0 = RX>
__global__ void __launch_bounds__(S * RegPlan<RX, NP, R0>::NR, reg_min_blocks<RX, NP, S, R0>())
    k_c2r_reg(const typename PT<C3>::cplx* __restrict__ in, long in_ks, long nseries, int nout, bool vec,
              Tout* __restrict__ out, long out_ss, const typename PT<C3>::cplx* __restrict__ tw) {
  using R = typename PT<C3>::real;
  using C = typename CT<R>::c;
  constexpr int N = RegPlan<RX, NP, R0>::N, NR = RegPlan<RX, NP, R0>::NR, T = S * NR;
  constexpr int U = RX / R0, NB = N / R0;
  constexpr int SS = reg_series_stride<C, N + 1, S>();
  extern __shared__ __align__(16) unsigned char reg_smem[];  // S * SS complex (dynamic: S*SS may exceed 48 KB)
  C* sbuf = reinterpret_cast<C*>(reg_smem);
  const int s = threadIdx.x / NR, j = threadIdx.x - s * NR;
  const long s0 = (long)blockIdx.x * S;
  const int ns = (int)min((long)S, nseries - s0);
  const bool act = s < ns;
  C* buf = sbuf + s * SS;
  grid_dep_wait();  // (PDL)
  const R inv_len = R(1) / (R)(2 * N);

  // The N+1 bins of S series (bin-major runs of S in global memory) land in
  // the series-major shared buffer through cp.async -- no register staging,
  // which keeps the kernel at 4+ resident CTAs per SM; the 1/L scaling and
  // Im(X0) = Im(XN) = 0 (fft.hpp:130-148) are applied in the pre-pass read.
  for (int e = threadIdx.x; e < S * (N + 1); e += T) {
    const int k = e / S, si = e - k * S;
    const bool ok = si < ns;
    cp_async(sbuf + si * SS + k, in + (long)k * in_ks + s0 + (ok ? si : 0), ok ? (int)sizeof(C) : 0, (int)sizeof(C));
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  // Pre-pass fused into pass 1: Z[n] = (X[n] + conj X[N-n]) + i w^-n (X[n] - conj X[N-n]).
  {
    C v[RX];
    if (act) {
      const C wj = __ldg(tw + j);
#pragma unroll
      for (int q = 0; q < RX; ++q) {
        const int n = j + (q / R0) * NR + (q % R0) * NB;  // (R0 = RX: j + q*NR)
        C A = buf[n], B = buf[N - n];  // X[n], X[N-n]
        A.x = A.x * inv_len;
        A.y = n == 0 ? R(0) : A.y * inv_len;  // Im(X0) = 0
        B.x = B.x * inv_len;
        B.y = n == 0 ? -R(0) : -(B.y * inv_len);  // conj; Im(XN) = 0 (sign of zero as cconj(0))
        C w;  // w^n = w^j * w^(q*N/RX); for RX = 10 the second factor is a constant
        if constexpr (RX == 10 && R0 == RX) w = q == 0 ? wj : cmul(wj, half_turn10<R>(q));
        else w = __ldg(tw + n);
        v[q] = cadd(cadd(A, B), cmuli<1>(cmul(C{w.x, -w.y}, csub(A, B))));
      }
      if constexpr (R0 == RX) {
        butterfly<R, 1, RX>(v);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) butterfly<R, 1, R0>(v + u * R0);
      }
    }
    __syncthreads();
    if (act) {
      if constexpr (R0 == RX) {
        store_stride_rx<RX>(buf + j * RX, v);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int r = 0; r < R0; ++r) buf[(j + u * NR) * R0 + r] = v[u * R0 + r];
      }
    }
    __syncthreads();
  }
  reg_passes<R, 1, RX, N, R0, R0, NR / RX>(buf, j, act, tw);
  // Last pass (Ns = N/RX): out index j + q*NR, straight to global.
  {
    constexpr int Ns = NR;
    const C* __restrict__ twp = tw + reg_tw_offset<RX, N, Ns, R0>();
    C v[RX];
    if (act) {
#pragma unroll
      for (int q = 0; q < RX; ++q) v[q] = buf[j + q * NR];
      apply_twiddles<R, 1, RX, Ns>(v, twp, j);
      butterfly<R, 1, RX>(v);
      Tout* p = out + (s0 + s) * out_ss;
#pragma unroll
      for (int q = 0; q < RX; ++q) {
        const int n = j + q * NR;
        const int t0 = 2 * n;
        if (t0 >= nout) continue;
        const Tout a = (Tout)rnd<C4>((double)v[q].x);
        const Tout b = (Tout)rnd<C4>((double)v[q].y);
        if constexpr (sizeof(Tout) == 8) {
          if (vec) {
            reinterpret_cast<double2*>(p)[n] = make_double2(a, b);
            continue;
          }
        }
        p[t0] = a;
        if (t0 + 1 < nout) p[t0 + 1] = b;
      }
    }
  }
}

}  // namespace fmv
