// fmv_fft_launch.cu -- dispatch of the batched real FFT kernels
// (fmv_fft.cuh) for the pipeline (phases 1-2 and 4-5, matvec.hpp:83-205),
// operator setup (operator.hpp:99-125) and the C ABI fmv_fft_r2c / c2r
// (fft.hpp:110-148).
#include "fmv_runtime.cuh"
#include "fmv_fft.cuh"
#include "fmv_fft_rt.cuh"
#include "fmv_fft_pair.cuh"
#include "fmv_fft_stream.cuh"

namespace fmv {
namespace rt {

// ======================================================================
// FFT geometry of the general mixed-radix kernels
// ======================================================================
inline FftGeom make_geom(int Nt, int nout) {
  FftGeom g{};
  g.N = Nt;
  g.L = 2 * Nt;
  g.n_div = FastDiv((uint32_t)Nt);
  g.nb_div = FastDiv((uint32_t)Nt + 1);
  g.nout_div = FastDiv((uint32_t)nout);
  int n = Nt;
  while (n > 1) {
    int r;
    if (n % 8 == 0 && n != 16) r = 8;  // 16 = 4*4 beats 8*2
    else if (n % 4 == 0) r = 4;
    else if (n % 2 == 0) r = 2;
    else if (n % 5 == 0) r = 5;
    else if (n % 3 == 0) r = 3;
    else {
      r = 7;
      while (n % r) r += 2;  // smallest remaining odd prime factor >= 7
    }
    if (g.nst >= kMaxStages) fail(FMV_EUNSUPPORTED, "FFT: too many stages");
    g.radix[g.nst++] = r;
    n /= r;
  }
  int Ns = 1;
  for (int st = 0; st < g.nst; ++st) {
    g.nr_div[st] = FastDiv((uint32_t)(Nt / g.radix[st]));
    g.ns_div[st] = FastDiv((uint32_t)Ns);
    g.span_div[st] = FastDiv((uint32_t)(Ns * g.radix[st]));
    Ns *= g.radix[st];
  }
  return g;
}

int fft_lg_series_per_cta(int N, size_t celem) {
  const size_t per = 2 * (size_t)(N + 1) * celem;
  if (per > 200 * 1024)
    fail(FMV_EUNSUPPORTED, "FFT: n_t = " + std::to_string(N) + " exceeds the shared-memory FFT capacity");
  const size_t budget = (size_t)env_int("FMV_FFT_SMEM_BUDGET", 64 * 1024);
  int lg = 0;
  while (lg < 4 && per * ((size_t)2 << lg) <= budget) ++lg;
  return lg;
}

// Kernel families, in dispatch order (FMV_FFT_PATH = auto | reg | rt | legacy
// | global forces one for tests; FMV_FFT_LEGACY=1 is the old switch for
// "legacy"):
//  * reg    -- k_r2c_reg / k_c2r_reg, compile-time radix-10 plans for the
//              pipeline's N = 1000 and N = 100 (SOTI <-> TOSI);
//  * rt     -- k_r2c_rt / k_c2r_rt, runtime register plans for every N whose
//              prime factors are <= 7, while a series fits shared memory;
//  * legacy -- k_r2c / k_c2r, ping-pong shared-memory mixed radix with a
//              generic prime stage (any N up to the two-buffer capacity;
//              also the time-outer input of operator setup);
//  * global -- k_fft_g*, HBM-scratch Stockham for any N (too long for shared
//              memory, or large prime factors).
enum FftPath { FP_AUTO, FP_REG, FP_RT, FP_LEGACY, FP_GLOBAL };
inline FftPath fft_path() {  // (read per call: tests switch paths within one process)
  if (env_int("FMV_FFT_LEGACY", 0)) return FP_LEGACY;
  const char* v = getenv("FMV_FFT_PATH");
  if (!v || !*v) return FP_AUTO;
  const std::string s = v;
  return s == "reg" ? FP_REG : s == "rt" ? FP_RT : s == "legacy" ? FP_LEGACY : s == "global" ? FP_GLOBAL : FP_AUTO;
}
#ifndef FMV_FFT_S64
#define FMV_FFT_S64 2  // fp64 Nt = 1000 series per CTA of the register FFT kernels
#endif
// Big N = 1000 transforms of the matvec (>= 1024 series, zero-padded input /
// first-half output) have three kernel sets: the one-shot one-butterfly-per-
// thread k_r2c_reg / k_c2r_reg ("reg"), the paired-butterfly kernels
// (fmv_fft_pair.cuh, "pair") and the persistent prefetching kernels
// (fmv_fft_stream.cuh, "stream"). Defaults are the measured best at C2
// (tools/tune_pair.py): fp64 r2c reg 47.9 / pair 50.2 /
// stream 50.7 us, fp64 c2r 44.2 / 63.3 / 57.7, fp32 r2c 39.0 / 46.3 / 35.2,
// fp32 c2r 39.4 / 35.5 / 41.4. (The fp32 stream r2c is faster by itself but
// its F matvec is not: 0.6329 vs 0.6279 ms for dssdd -- the SBGEMV after it
// runs slower.) FMV_FFT_BIG = reg | pair | stream forces one.
enum BigFft { BF_REG, BF_PAIR, BF_STREAM };
inline BigFft big_fft_kind(int N, long nseries, int nvalid, bool r2c, bool f64) {
  if (N != 1000 || nvalid != N || nseries < 1024) return BF_REG;
  const char* v = getenv("FMV_FFT_BIG");
  if (v && *v) {
    const std::string k = v;
    return k == "reg" ? BF_REG : k == "pair" ? BF_PAIR : BF_STREAM;
  }
  return f64 || r2c ? BF_REG : BF_PAIR;
}
#ifndef FMV_STREAM_S64
#define FMV_STREAM_S64 2
#endif
#ifndef FMV_STREAM_S32
#define FMV_STREAM_S32 4
#endif
// register caps (__maxnreg__) of the stream kernels: r2c / c2r, fp64 / fp32
#ifndef FMV_STREAM_R2C_R64
#define FMV_STREAM_R2C_R64 64
#endif
#ifndef FMV_STREAM_C2R_R64
#define FMV_STREAM_C2R_R64 80
#endif
#ifndef FMV_STREAM_R32
#define FMV_STREAM_R32 64
#endif
// Resident CTAs per SM of a kernel at a block size / dynamic smem (cached).
inline int occupancy(const void* fn, int block, size_t smem) {
  static std::mutex mu;
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(dev, fn, block, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int n = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fn, block, smem));
  return cache[key] = std::max(1, n);
}
#ifndef FMV_PAIR_S64
#define FMV_PAIR_S64 4
#endif
#ifndef FMV_PAIR_MINB64
#define FMV_PAIR_MINB64 2
#endif
#ifndef FMV_PAIR_S32
#define FMV_PAIR_S32 8
#endif
#ifndef FMV_PAIR_MINB32
#define FMV_PAIR_MINB32 2
#endif
// Compile-time register plans beyond the matvec's 1000 / 100 (matvec path only):
// 512 = 8^3, 4096 = 16^3, 1024 = 4*16^2, 2048 = 8*16^2, 8192 = 2*16^3, 2000 = 2*10^3.
inline bool fft_reg_extra(int N) {
  return N == 512 || N == 4096 || N == 1024 || N == 2048 || N == 8192 || N == 2000;
}
bool fft_reg_ok(int N) {
  return (N == 1000 || N == 100 || fft_reg_extra(N)) && (fft_path() == FP_AUTO || fft_path() == FP_REG);
}

// Legacy two-buffer capacity: S = 1 series of 2 (N + 1) complex in <= 200 KB.
bool fft_legacy_fits(int N, size_t celem) { return 2 * (size_t)(N + 1) * celem <= 200 * 1024; }

// Radices of the register / global plans: greedy largest-first from
// {16, 10, 8, 7, 5, 4, 3, 2}; false if a prime factor > 7 remains.
bool fft_factor(int N, std::vector<int>& radices) {
  static const int cand[] = {16, 10, 8, 7, 5, 4, 3, 2};
  radices.clear();
  int n = N;
  while (n > 1) {
    bool found = false;
    for (int r : cand)
      if (n % r == 0) {
        radices.push_back(r);
        n /= r;
        found = true;
        break;
      }
    if (!found) return false;
  }
  return true;
}

// Runtime register plan for complex length N (fmv_fft_rt.cuh): N = R_0 *
// RR^k with R_0, RR in {2, 3, 4, 5, 7, 8, 10, 16} (the fewest passes, then
// the largest RR); `extra` = 1 for the c2r (N + 1 bins per series in shared
// memory). False if N has no such form, needs more than 512 threads per
// series or a series does not fit a CTA's shared memory.
bool make_rt_plan(int N, size_t celem, int extra, RtPlan& P, std::vector<int>& radices, int& RR) {
  static const int cand[] = {16, 10, 8, 7, 5, 4, 3, 2};
  auto in_set = [](int r) { return r == 2 || r == 3 || r == 4 || r == 5 || r == 7 || r == 8 || r == 10 || r == 16; };
  if (N < 2) return false;
  int best_np = 1 << 30;
  radices.clear();
  for (int rr : cand) {
    // N = n * rr^k with the largest k for which n is 1 or a first-pass radix
    int n = N, k = 0, bn = -1, bk = 0;
    for (;;) {
      if (n == 1 && k >= 1) {
        bn = 1;
        bk = k;
      } else if (in_set(n)) {
        bn = n;
        bk = k;
      }
      if (n % rr) break;
      n /= rr;
      ++k;
    }
    if (bn < 0) continue;
    std::vector<int> rad;
    if (bn > 1) rad.push_back(bn);
    rad.insert(rad.end(), bk, rr);
    if ((int)rad.size() < best_np) {
      best_np = (int)rad.size();
      radices = rad;
      RR = rr;
    }
  }
  if (radices.empty() || (int)radices.size() > kRtMaxPasses) return false;
  P = RtPlan{};
  P.N = N;
  P.np = (int)radices.size();
  // threads per series: enough that no thread owns more than floor(16 / R_p)
  // butterflies of any pass (rt_hold in fmv_fft_plan.cuh)
  P.TS = 1;
  for (int r : radices) {
    const int hold = std::max(1, kRtHold / r);
    P.TS = std::max(P.TS, (N / r + hold - 1) / hold);
  }
  if (P.TS > 512) return false;
  int Ns = 1, off = 2 * N;
  for (int p = 0; p < P.np; ++p) {
    const int R = radices[p];
    P.radix[p] = R;
    P.Ns[p] = Ns;
    P.ns_div[p] = FastDiv((uint32_t)Ns);
    P.tw_off[p] = p == 0 ? 0 : off;
    if (p > 0) off += R * Ns;
    P.bpt[p] = (N / R + P.TS - 1) / P.TS;  // <= max(1, 16 / R) by the choice of TS
    Ns *= R;
  }
  P.SS = N + extra;
  if (P.SS % 2 == 0) ++P.SS;  // odd stride (in elements): consecutive series start on shifted banks
  const size_t per = (size_t)P.SS * celem;
  if (per > 220 * 1024) return false;
  const size_t budget = (size_t)env_int("FMV_FFT_SMEM_BUDGET", 64 * 1024);
  P.S = 1;
  while (P.S * 2 * P.TS <= 256 && (size_t)P.S * 2 * per <= budget) P.S *= 2;
  return true;
}

template <class... A>
void rt_r2c_any(int RR, A... a) {
  switch (RR) {
    case 16: rt_r2c_run<16>(a...); break;
    case 10: rt_r2c_run<10>(a...); break;
    case 8: rt_r2c_run<8>(a...); break;
    case 7: rt_r2c_run<7>(a...); break;
    case 5: rt_r2c_run<5>(a...); break;
    case 4: rt_r2c_run<4>(a...); break;
    case 3: rt_r2c_run<3>(a...); break;
    default: rt_r2c_run<2>(a...); break;
  }
}
template <class... A>
void rt_c2r_any(int RR, A... a) {
  switch (RR) {
    case 16: rt_c2r_run<16>(a...); break;
    case 10: rt_c2r_run<10>(a...); break;
    case 8: rt_c2r_run<8>(a...); break;
    case 7: rt_c2r_run<7>(a...); break;
    case 5: rt_c2r_run<5>(a...); break;
    case 4: rt_c2r_run<4>(a...); break;
    case 3: rt_c2r_run<3>(a...); break;
    default: rt_c2r_run<2>(a...); break;
  }
}

template <class T>
constexpr int prec_tag() {
  return sizeof(T) == 8 ? PD : sizeof(T) == 4 ? PS : PH;
}

// HBM-scratch Stockham passes over z (nser x N complex, ping-pong with the
// second half of the scratch); returns the buffer holding the result.
template <class R, int D>
typename CT<R>::c* global_passes(fmv_ctx* ctx, typename CT<R>::c* a, typename CT<R>::c* b, long nser, int N,
                                 const typename CT<R>::c* tw, int cls) {
  const double2* twd = static_cast<const double2*>(twiddles().get(ctx->device, 2 * N, PD));
  std::vector<int> rad;
  const bool smooth = fft_factor(N, rad);
  if (!smooth) {  // fixed radices for the smooth part, generic primes for the rest
    rad.clear();
    int n = N;
    for (int r : {16, 10, 8, 7, 5, 4, 3, 2})
      while (n % r == 0) {
        rad.push_back(r);
        n /= r;
      }
    for (int f = 11; n > 1; f += 2)
      while (n % f == 0) {
        rad.push_back(f);
        n /= f;
      }
  }
  int Ns = 1;
  const unsigned grid = grid_for(nser * (long)N, 256, ctx->device);
  for (int r : rad) {
    launch(ctx, cls, [&] {
      switch (r) {
#define GP(RR) \
  case RR: k_fft_gpass<R, D, RR><<<grid, 256, 0, ctx->stream>>>(a, b, nser, N, Ns, tw); break;
        GP(2) GP(3) GP(4) GP(5) GP(7) GP(8) GP(10) GP(16)
#undef GP
        default: k_fft_gpass_generic<R, D><<<grid, 256, 0, ctx->stream>>>(a, b, nser, N, r, Ns, twd); break;
      }
    });
    std::swap(a, b);
    Ns *= r;
  }
  return a;
}

// Series per scratch round of the global path: <= 2 x 256 MB of scratch.
inline long global_batch(long nseries, int N, size_t celem) {
  return std::max<long>(1, std::min<long>(nseries, (256L << 20) / ((long)N * (long)celem)));
}

template <int C0, int C1, int C2, class Tin>
void r2c_global(fmv_ctx* ctx, const Tin* in, long in_ss, long in_ts, long nseries, int N, int nvalid, void* out,
                long out_ks, long out_ss) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  using OutC = typename PT<C2>::cplx;
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, 2 * N, C1));
  const long B = global_batch(nseries, N, sizeof(C));
  ctx->fft_scratch.ensure(2 * (size_t)B * N * sizeof(C));
  C* za = static_cast<C*>(ctx->fft_scratch.p);
  C* zb = za + (size_t)B * N;
  for (long s0 = 0; s0 < nseries; s0 += B) {
    const long nb = std::min(B, nseries - s0);
    const unsigned grid = grid_for(nb * (long)N, 256, ctx->device);
    launch(ctx, 0, [&] {
      k_fft_gpack<R, Tin><<<grid, 256, 0, ctx->stream>>>(in + s0 * in_ss, in_ss, in_ts, nb, N, nvalid, (int)C0, za);
    });
    C* z = global_passes<R, -1>(ctx, za, zb, nb, N, tw, 0);
    const unsigned g2 = grid_for(nb * (long)(N + 1), 256, ctx->device);
    launch(ctx, 0, [&] {
      k_fft_gpost<R><<<g2, 256, 0, ctx->stream>>>(z, nb, N, static_cast<OutC*>(out) + s0 * out_ss, (int)C2, out_ks,
                                                  out_ss, tw);
    });
  }
}

// Twiddle table of a register plan (R0, RX, ..., RX): base + per-pass tables.
inline const void* reg_plan_twiddles(int dev, int N, int prec, int RX, int NP, int R0) {
  if (R0 == RX) return twiddles().get(dev, 2 * N, prec, RX);
  std::vector<int> radices(NP, RX);
  radices[0] = R0;
  return twiddles().get_plan(dev, 2 * N, prec, radices);
}

template <int C0, int C1, int C2, class Tin, int RX, int NP, int S, int R0 = RX>
void r2c_reg_launch(fmv_ctx* ctx, const Tin* in, long in_ss, long nseries, int nvalid, void* out, long out_ks) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  const int N = RegPlan<RX, NP, R0>::N;
  const C* tw = static_cast<const C*>(reg_plan_twiddles(ctx->device, N, C1, RX, NP, R0));
  bool vec = (in_ss % 2 == 0) && (nvalid % 2 == 0);
  if constexpr (sizeof(Tin) == 8) vec = vec && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  else if constexpr (sizeof(Tin) == 4) vec = vec && (reinterpret_cast<uintptr_t>(in) & 7) == 0;
  else vec = false;
  const long grid = (nseries + S - 1) / S;
  constexpr size_t smem = r2c_reg_smem<C, RX, NP, S, R0>();
  prep_smem((const void*)k_r2c_reg<C0, C1, C2, Tin, RX, NP, S, R0>, smem);
  prep_carveout((const void*)k_r2c_reg<C0, C1, C2, Tin, RX, NP, S, R0>);
  launch(ctx, 0, [&] {
    launch_pdl(k_r2c_reg<C0, C1, C2, Tin, RX, NP, S, R0>, dim3((unsigned)grid), dim3(S * RegPlan<RX, NP, R0>::NR), smem,
               ctx->stream, in, in_ss, nseries, nvalid, vec, static_cast<typename PT<C2>::cplx*>(out), out_ks, tw);
  });
}

template <int C0, int C1, int C2, class Tin, int S, int MINB>
void r2c_pair_launch(fmv_ctx* ctx, const Tin* in, long in_ss, long nseries, void* out, long out_ks) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, 2000, C1, 10));
  bool vec = in_ss % 2 == 0;
  if constexpr (sizeof(Tin) == 8) vec = vec && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  else if constexpr (sizeof(Tin) == 4) vec = vec && (reinterpret_cast<uintptr_t>(in) & 7) == 0;
  else vec = false;
  const long grid = (nseries + S - 1) / S;
  constexpr size_t smem = pair_smem<C, S>();
  auto kern = k_r2c_pair<C0, C1, C2, Tin, S, MINB>;
  prep_smem((const void*)kern, smem);
  prep_carveout((const void*)kern);
  launch(ctx, 0, [&] {
    launch_pdl(kern, dim3((unsigned)grid), dim3(S * 50), smem, ctx->stream, in, in_ss, nseries, vec,
               static_cast<typename PT<C2>::cplx*>(out), out_ks, tw);
  });
}

template <int C0, int C1, int C2, int S, int MAXR>
void r2c_stream_launch(fmv_ctx* ctx, const double* in, long nseries, void* out, long out_ks) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, 2000, C1, 10));
  constexpr size_t smem = r2c_stream_smem<C, S>();
  auto kern = k_r2c_stream<C0, C1, C2, S, MAXR>;
  prep_smem((const void*)kern, smem);
  prep_carveout((const void*)kern);
  const long ntiles = (nseries + S - 1) / S;
  const long grid = std::min(ntiles, (long)occupancy((const void*)kern, S * 100, smem) * sm_count(ctx->device));
  launch(ctx, 0, [&] {
    launch_pdl(kern, dim3((unsigned)grid), dim3(S * 100), smem, ctx->stream, in, nseries,
               static_cast<typename PT<C2>::cplx*>(out), out_ks, tw);
  });
}

template <int C0, int C1, int C2, class Tin>
void r2c_t(fmv_ctx* ctx, const Tin* in, long in_ss, long in_ts, long nseries, int N, int nvalid, void* out,
           long out_ks, long out_ss) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  constexpr bool tin_ok = sizeof(Tin) == 8 || (sizeof(Tin) == 4 && C0 == PS) || (sizeof(Tin) == 2 && C0 == PH);
  if constexpr (tin_ok) {
    if (in_ts == 1 && out_ss == 1 && fft_reg_ok(N) && (!fft_reg_extra(N) || sizeof(Tin) == 8)) {
      constexpr bool f64 = sizeof(R) == 8;
      if constexpr (sizeof(Tin) == 8) {
        if (big_fft_kind(N, nseries, nvalid, true, f64) == BF_STREAM && in_ss == N &&
            (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
          r2c_stream_launch<C0, C1, C2, f64 ? FMV_STREAM_S64 : FMV_STREAM_S32, f64 ? FMV_STREAM_R2C_R64 : FMV_STREAM_R32>(
              ctx, in, nseries, out, out_ks);
          return;
        }
      }
      if (big_fft_kind(N, nseries, nvalid, true, f64) == BF_PAIR) {
        if constexpr (f64)
          r2c_pair_launch<C0, C1, C2, Tin, FMV_PAIR_S64, FMV_PAIR_MINB64>(ctx, in, in_ss, nseries, out, out_ks);
        else
          r2c_pair_launch<C0, C1, C2, Tin, FMV_PAIR_S32, FMV_PAIR_MINB32>(ctx, in, in_ss, nseries, out, out_ks);
        return;
      }
      // the other compile-time plans (uniform radix-8 / 16, mixed R0 * RX^k)
      if (fft_reg_extra(N)) {
        if constexpr (sizeof(Tin) == 8) {
          if (N == 512) r2c_reg_launch<C0, C1, C2, Tin, 8, 3, 4>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
          else if (N == 4096) r2c_reg_launch<C0, C1, C2, Tin, 16, 3, 1>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
          else if (N == 1024) r2c_reg_launch<C0, C1, C2, Tin, 16, 3, 4, 4>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
          else if (N == 2048) r2c_reg_launch<C0, C1, C2, Tin, 16, 3, 2, 8>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
          else if (N == 8192) r2c_reg_launch<C0, C1, C2, Tin, 16, 4, 1, 2>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
          else r2c_reg_launch<C0, C1, C2, Tin, 10, 4, 1, 2>(ctx, in, in_ss, nseries, nvalid, out, out_ks);  // 2000
          return;
        }
      }
      // (fp64: one series per CTA for small batches -- more CTAs for the 100-series transforms)
      if (N == 1000 && f64 && nseries < 1024)
        r2c_reg_launch<C0, C1, C2, Tin, 10, 3, 1>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
      else if (N == 1000)
        r2c_reg_launch<C0, C1, C2, Tin, 10, 3, f64 ? FMV_FFT_S64 : 4>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
      else
        r2c_reg_launch<C0, C1, C2, Tin, 10, 2, f64 ? 16 : 32>(ctx, in, in_ss, nseries, nvalid, out, out_ks);
      return;
    }
  }
  const FftPath path = fft_path();
  if (path == FP_AUTO || path == FP_RT) {
    RtPlan P;
    std::vector<int> radices;
    int RR = 0;
    if (in_ts == 1 && make_rt_plan(N, sizeof(C), 0, P, radices, RR)) {
      const void* tw = twiddles().get_plan(ctx->device, 2 * N, C1, radices);
      rt_r2c_any(RR, ctx, (int)C1, prec_tag<Tin>(), (int)C0, (int)C2, (const void*)in, in_ss, nseries, nvalid, out,
                 out_ks, out_ss, (const RtPlan&)P, tw);
      return;
    }
  }
  if (path == FP_GLOBAL || !fft_legacy_fits(N, sizeof(C))) {
    r2c_global<C0, C1, C2, Tin>(ctx, in, in_ss, in_ts, nseries, N, nvalid, out, out_ks, out_ss);
    return;
  }
  const FftGeom g = make_geom(N, nvalid);
  const int lgS = fft_lg_series_per_cta(g.N, sizeof(C));
  const int S = 1 << lgS;
  const size_t smem = 2 * (size_t)S * (g.N + 1) * sizeof(C);
  auto kern = k_r2c<C0, C1, C2, Tin>;
  prep_smem((const void*)kern, smem);
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, g.L, C1));
  const double2* twd = static_cast<const double2*>(twiddles().get(ctx->device, g.L, PD));
  const long grid = (nseries + S - 1) / S;
  launch(ctx, 0, [&] {
    kern<<<(unsigned)grid, 256, smem, ctx->stream>>>(in, in_ss, in_ts, nseries, nvalid,
                                                     static_cast<typename PT<C2>::cplx*>(out), out_ks, out_ss, g, tw,
                                                     twd, lgS);
  });
}

// N = L/2 (complex FFT length); nvalid = input samples per series (Nt for
// the zero-padded matvec path, L for a plain transform).
template <class Tin>
void r2c_dispatch(fmv_ctx* ctx, int c0, int c1, int c2, const Tin* in, long in_ss, long in_ts, long nseries, int N,
                  int nvalid, void* out, long out_ks, long out_ss) {
#define R2C_CASE(A, B, C)                                                                      \
  if (c0 == A && c1 == B && c2 == C) {                                                         \
    r2c_t<A, B, C, Tin>(ctx, in, in_ss, in_ts, nseries, N, nvalid, out, out_ks, out_ss);       \
    return;                                                                                    \
  }
  R2C_CASE(PD, PD, PD) R2C_CASE(PD, PD, PS) R2C_CASE(PD, PD, PH)
  R2C_CASE(PD, PS, PD) R2C_CASE(PD, PS, PS) R2C_CASE(PD, PS, PH)
  R2C_CASE(PS, PD, PD) R2C_CASE(PS, PD, PS) R2C_CASE(PS, PD, PH)
  R2C_CASE(PS, PS, PD) R2C_CASE(PS, PS, PS) R2C_CASE(PS, PS, PH)
  R2C_CASE(PH, PD, PD) R2C_CASE(PH, PD, PS) R2C_CASE(PH, PD, PH)
  R2C_CASE(PH, PS, PD) R2C_CASE(PH, PS, PS) R2C_CASE(PH, PS, PH)
#undef R2C_CASE
  fail(FMV_EINVAL, "r2c: unsupported precision combination");
}

template <int C3, int C4, class Tout, int RX, int NP, int S, int R0 = RX>
void c2r_reg_launch(fmv_ctx* ctx, const void* in, long in_ks, long nseries, int nout, Tout* out, long out_ss) {
  using C = typename PT<C3>::cplx;
  const int N = RegPlan<RX, NP, R0>::N;
  const C* tw = static_cast<const C*>(reg_plan_twiddles(ctx->device, N, C3, RX, NP, R0));
  const bool vec = sizeof(Tout) == 8 && (out_ss % 2 == 0) && (nout % 2 == 0) &&
                   (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const long grid = (nseries + S - 1) / S;
  using Cr = typename CT<typename PT<C3>::real>::c;
  constexpr size_t smem = c2r_reg_smem<Cr, RX, NP, S, R0>();
  prep_smem((const void*)k_c2r_reg<C3, C4, Tout, RX, NP, S, R0>, smem);
  prep_carveout((const void*)k_c2r_reg<C3, C4, Tout, RX, NP, S, R0>);
  launch(ctx, 3, [&] {
    launch_pdl(k_c2r_reg<C3, C4, Tout, RX, NP, S, R0>, dim3((unsigned)grid), dim3(S * RegPlan<RX, NP, R0>::NR), smem,
               ctx->stream, static_cast<const C*>(in), in_ks, nseries, nout, vec, out, out_ss, tw);
  });
}

template <int C3, int C4, class Tout, int S, int MINB>
void c2r_pair_launch(fmv_ctx* ctx, const void* in, long in_ks, long nseries, Tout* out, long out_ss) {
  using C = typename PT<C3>::cplx;
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, 2000, C3, 10));
  const bool vec = sizeof(Tout) == 8 && (out_ss % 2 == 0) && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  const long grid = (nseries + S - 1) / S;
  constexpr size_t smem = pair_smem<C, S>();
  auto kern = k_c2r_pair<C3, C4, Tout, S, MINB>;
  prep_smem((const void*)kern, smem);
  prep_carveout((const void*)kern);
  launch(ctx, 3, [&] {
    launch_pdl(kern, dim3((unsigned)grid), dim3(S * 50), smem, ctx->stream, static_cast<const C*>(in), in_ks,
               nseries, vec, out, out_ss, tw);
  });
}

template <int C3, int C4, class Tout, int S, int MAXR>
void c2r_stream_launch(fmv_ctx* ctx, const void* in, long in_ks, long nseries, Tout* out, long out_ss) {
  using C = typename PT<C3>::cplx;
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, 2000, C3, 10));
  const bool vec = sizeof(Tout) == 8 && (out_ss % 2 == 0) && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  using Cr = typename CT<typename PT<C3>::real>::c;
  constexpr size_t smem = c2r_stream_smem<Cr, S>();
  auto kern = k_c2r_stream<C3, C4, Tout, S, MAXR>;
  prep_smem((const void*)kern, smem);
  prep_carveout((const void*)kern);
  const long ntiles = (nseries + S - 1) / S;
  const long grid = std::min(ntiles, (long)occupancy((const void*)kern, S * 100, smem) * sm_count(ctx->device));
  launch(ctx, 3, [&] {
    launch_pdl(kern, dim3((unsigned)grid), dim3(S * 100), smem, ctx->stream, static_cast<const C*>(in), in_ks,
               nseries, vec, out, out_ss, tw);
  });
}

template <int C3, int C4, class Tout>
void c2r_global(fmv_ctx* ctx, const void* in, long in_ks, long in_ss, long nseries, int N, int nout, Tout* out,
                long out_ss) {
  using R = typename PT<C3>::real;
  using C = typename CT<R>::c;
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, 2 * N, C3));
  const long B = global_batch(nseries, N, sizeof(C));
  ctx->fft_scratch.ensure(2 * (size_t)B * N * sizeof(C));
  C* za = static_cast<C*>(ctx->fft_scratch.p);
  C* zb = za + (size_t)B * N;
  for (long s0 = 0; s0 < nseries; s0 += B) {
    const long nb = std::min(B, nseries - s0);
    const unsigned grid = grid_for(nb * (long)N, 256, ctx->device);
    launch(ctx, 3, [&] {
      k_fft_gpre<R><<<grid, 256, 0, ctx->stream>>>(static_cast<const C*>(in) + s0 * in_ss, in_ks, in_ss, nb, N, za,
                                                   tw);
    });
    C* z = global_passes<R, 1>(ctx, za, zb, nb, N, tw, 3);
    const unsigned g2 = grid_for(nb * (long)nout, 256, ctx->device);
    launch(ctx, 3, [&] {
      k_fft_gunpack<R, Tout><<<g2, 256, 0, ctx->stream>>>(z, nb, N, nout, (int)C4, out + s0 * out_ss, out_ss);
    });
  }
}

template <int C3, int C4, class Tout>
void c2r_t(fmv_ctx* ctx, const void* in, long in_ks, long in_ss, long nseries, int N, int nout, Tout* out,
           long out_ss) {
  using C = typename PT<C3>::cplx;
  if (in_ss == 1 && fft_reg_ok(N)) {
    constexpr bool f64 = C3 == PD;
    if (big_fft_kind(N, nseries, nout, false, f64) == BF_STREAM) {
      c2r_stream_launch<C3, C4, Tout, f64 ? FMV_STREAM_S64 : FMV_STREAM_S32, f64 ? FMV_STREAM_C2R_R64 : FMV_STREAM_R32>(
          ctx, in, in_ks, nseries, out, out_ss);
      return;
    }
    if (big_fft_kind(N, nseries, nout, false, f64) == BF_PAIR) {
      if constexpr (f64) c2r_pair_launch<C3, C4, Tout, FMV_PAIR_S64, FMV_PAIR_MINB64>(ctx, in, in_ks, nseries, out, out_ss);
      else c2r_pair_launch<C3, C4, Tout, FMV_PAIR_S32, FMV_PAIR_MINB32>(ctx, in, in_ks, nseries, out, out_ss);
      return;
    }
    if (fft_reg_extra(N)) {
      if (N == 512) c2r_reg_launch<C3, C4, Tout, 8, 3, 4>(ctx, in, in_ks, nseries, nout, out, out_ss);
      else if (N == 4096) c2r_reg_launch<C3, C4, Tout, 16, 3, 1>(ctx, in, in_ks, nseries, nout, out, out_ss);
      else if (N == 1024) c2r_reg_launch<C3, C4, Tout, 16, 3, 4, 4>(ctx, in, in_ks, nseries, nout, out, out_ss);
      else if (N == 2048) c2r_reg_launch<C3, C4, Tout, 16, 3, 2, 8>(ctx, in, in_ks, nseries, nout, out, out_ss);
      else if (N == 8192) c2r_reg_launch<C3, C4, Tout, 16, 4, 1, 2>(ctx, in, in_ks, nseries, nout, out, out_ss);
      else c2r_reg_launch<C3, C4, Tout, 10, 4, 1, 2>(ctx, in, in_ks, nseries, nout, out, out_ss);  // 2000
      return;
    }
    if (N == 1000)
    {
      // fp32: 8 series per CTA for the big (Nm-series) transform, 2 for the small
      // one (tools/tune_fft.py at C2: 45.5 -> 39.3 us, and 10.5 us)
      if constexpr (f64) {
        if (nseries < 1024) c2r_reg_launch<C3, C4, Tout, 10, 3, 1>(ctx, in, in_ks, nseries, nout, out, out_ss);
        else c2r_reg_launch<C3, C4, Tout, 10, 3, FMV_FFT_S64>(ctx, in, in_ks, nseries, nout, out, out_ss);
      }
      else if (nseries >= 1024) c2r_reg_launch<C3, C4, Tout, 10, 3, 8>(ctx, in, in_ks, nseries, nout, out, out_ss);
      else c2r_reg_launch<C3, C4, Tout, 10, 3, 2>(ctx, in, in_ks, nseries, nout, out, out_ss);
    }
    else
      c2r_reg_launch<C3, C4, Tout, 10, 2, f64 ? 16 : 32>(ctx, in, in_ks, nseries, nout, out, out_ss);
    return;
  }
  const FftPath path = fft_path();
  if (path == FP_AUTO || path == FP_RT) {
    RtPlan P;
    std::vector<int> radices;
    int RR = 0;
    if (make_rt_plan(N, sizeof(C), 1, P, radices, RR)) {
      const void* tw = twiddles().get_plan(ctx->device, 2 * N, C3, radices);
      rt_c2r_any(RR, ctx, (int)C3, prec_tag<Tout>(), (int)C4, in, in_ks, in_ss, nseries, nout, (void*)out, out_ss,
                 (const RtPlan&)P, tw);
      return;
    }
  }
  if (path == FP_GLOBAL || !fft_legacy_fits(N, sizeof(C))) {
    c2r_global<C3, C4, Tout>(ctx, in, in_ks, in_ss, nseries, N, nout, out, out_ss);
    return;
  }
  const FftGeom g = make_geom(N, nout);
  const int lgS = fft_lg_series_per_cta(g.N, sizeof(C));
  const int S = 1 << lgS;
  const size_t smem = 2 * (size_t)S * (g.N + 1) * sizeof(C);
  auto kern = k_c2r<C3, C4, Tout>;
  prep_smem((const void*)kern, smem);
  const C* tw = static_cast<const C*>(twiddles().get(ctx->device, g.L, C3));
  const double2* twd = static_cast<const double2*>(twiddles().get(ctx->device, g.L, PD));
  const long grid = (nseries + S - 1) / S;
  launch(ctx, 3, [&] {
    kern<<<(unsigned)grid, 256, smem, ctx->stream>>>(static_cast<const C*>(in), in_ks, in_ss, nseries, nout, out,
                                                     out_ss, g, tw, twd, lgS);
  });
}

void c2r_dispatch(fmv_ctx* ctx, int c3, int c4, const void* in, long in_ks, long in_ss, long nseries, int N,
                  int nout, double* out, long out_ss) {
#define C2R_CASE(A, B)                                                              \
  if (c3 == A && c4 == B) {                                                         \
    c2r_t<A, B, double>(ctx, in, in_ks, in_ss, nseries, N, nout, out, out_ss);      \
    return;                                                                         \
  }
  C2R_CASE(PD, PD) C2R_CASE(PD, PS) C2R_CASE(PD, PH) C2R_CASE(PS, PD) C2R_CASE(PS, PS) C2R_CASE(PS, PH)
#undef C2R_CASE
  fail(FMV_EINVAL, "c2r: unsupported precision combination");
}

template void r2c_dispatch<double>(fmv_ctx*, int, int, int, const double*, long, long, long, int, int, void*, long, long);
template void r2c_dispatch<float>(fmv_ctx*, int, int, int, const float*, long, long, long, int, int, void*, long, long);
template void r2c_dispatch<__half>(fmv_ctx*, int, int, int, const __half*, long, long, long, int, int, void*, long, long);

}  // namespace rt
}  // namespace fmv

extern "C" {

int fmv_fft_r2c(fmv_ctx* ctx, size_t L, size_t batch, char prec, const void* d_in, void* d_out) {
  return guarded([&] {
    if (!ctx || !d_in || !d_out) fail(FMV_EINVAL, "fft: null argument");
    if (L < 2 || L % 2) fail(FMV_EINVAL, "FftPlan: length must be even and >= 2");
    if (batch < 1) fail(FMV_EINVAL, "FftPlan: batch must be >= 1");
    DeviceGuard dg(ctx->device);
    const long nb = (long)L / 2 + 1;
    if (prec == 'd')
      r2c_t<PD, PD, PD, double>(ctx, static_cast<const double*>(d_in), (long)L, 1, (long)batch, (int)L / 2, (int)L,
                                d_out, 1, nb);
    else if (prec == 's')
      r2c_t<PS, PS, PS, float>(ctx, static_cast<const float*>(d_in), (long)L, 1, (long)batch, (int)L / 2, (int)L,
                               d_out, 1, nb);
    else
      fail(FMV_EINVAL, "fft: prec must be 'd' or 's'");
  });
}

int fmv_fft_c2r(fmv_ctx* ctx, size_t L, size_t batch, char prec, const void* d_in, void* d_out) {
  return guarded([&] {
    if (!ctx || !d_in || !d_out) fail(FMV_EINVAL, "fft: null argument");
    if (L < 2 || L % 2) fail(FMV_EINVAL, "FftPlan: length must be even and >= 2");
    if (batch < 1) fail(FMV_EINVAL, "FftPlan: batch must be >= 1");
    DeviceGuard dg(ctx->device);
    const long nb = (long)L / 2 + 1;
    if (prec == 'd')
      c2r_t<PD, PD, double>(ctx, d_in, 1, nb, (long)batch, (int)L / 2, (int)L, static_cast<double*>(d_out), (long)L);
    else if (prec == 's')
      c2r_t<PS, PS, float>(ctx, d_in, 1, nb, (long)batch, (int)L / 2, (int)L, static_cast<float*>(d_out), (long)L);
    else
      fail(FMV_EINVAL, "fft: prec must be 'd' or 's'");
  });
}

}  // extern "C"
