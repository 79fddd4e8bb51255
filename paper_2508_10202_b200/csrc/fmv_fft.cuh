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

namespace fmv {

constexpr int kMaxStages = 24;

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
};
template <>
struct RadixK<float> {
  static constexpr float s3 = 0.86602540378443864676372317075293618f;
  static constexpr float c51 = 0.30901699437494742410229341718281906f;
  static constexpr float c52 = -0.80901699437494742410229341718281906f;
  static constexpr float s51 = 0.95105651629515357211643933337938214f;
  static constexpr float s52 = 0.58778525229247312916870595463907277f;
  static constexpr float r2 = 0.70710678118654752440084436210484904f;
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

// Any radix r (used for primes other than 2,3,5): one thread per output.
template <class R, int D>
__device__ __forceinline__ void stage_generic(const typename CT<R>::c* __restrict__ src,
                                              typename CT<R>::c* __restrict__ dst, int ss, int ns, int r, int Ns,
                                              const FastDiv& nd, const FastDiv& nsd, const FastDiv& spand,
                                              const typename CT<R>::c* __restrict__ tw, int N, int L) {
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
    C acc = {R(0), R(0)};
    int e = 0;
    for (int m = 0; m < r; ++m) {
      acc = cadd(acc, cmul(in[j + m * Nr], twiddle<D>(tw, e * tstep)));
      e += estep;
      if (e >= span) e -= span * (e / span);
    }
    dst[s * ss + o] = acc;
  }
}

// Runs all stages; returns the buffer holding the result.
template <class R, int D>
__device__ typename CT<R>::c* run_stages(typename CT<R>::c* a, typename CT<R>::c* b, int ss, int ns, const FftGeom& g,
                                         const typename CT<R>::c* __restrict__ tw) {
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
        stage_generic<R, D>(a, b, ss, ns, r, Ns, g.n_div, g.ns_div[st], g.span_div[st], tw, g.N, g.L);
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
                                             int lgS) {
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
  const C* Z = run_stages<R, -1>(bufA, bufB, ss, ns, g, tw);

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
                                             const typename PT<C3>::cplx* __restrict__ tw, int lgS) {
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
  const C* z = run_stages<R, 1>(bufB, bufA, ss, ns, g, tw);
  for (int e = threadIdx.x; e < ns * nout; e += blockDim.x) {
    const int s = g.nout_div.div(e), t = e - s * nout;
    const C v = z[s * ss + (t >> 1)];
    out[(s0 + s) * out_ss + t] = (Tout)rnd<C4>((double)((t & 1) ? v.y : v.x));
  }
}

}  // namespace fmv
