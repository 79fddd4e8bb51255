// fmv_gemv_launch.cu -- planning and dispatch of the per-bin strided-batched
// GEMV (phase 3, gemv.hpp:74-240 / matvec.hpp:209-228: k_sbgemv, the TMA-ring
// kernel of fmv_sbgemv.cuh) and of the block multi-RHS SBGEMV
// (fmv_sbgemm_block.cuh), plus the C ABI fmv_sbgemv.
#include "fmv_runtime.cuh"
#include "fmv_sbgemv.cuh"
#include "fmv_sbgemm_block.cuh"

namespace fmv {
namespace rt {

// ------------------------------------------------------------- SBGEMV ----
struct GemvPlan {
  GemvParams p{};
  int block = 0;
  size_t smem = 0;
  int rpt = 1;
};


template <int MODE, class E, class O, int RPT, int V, int LPC>
void sbgemv_launch_t(fmv_ctx* ctx, GemvPlan& gp) {
  auto kern = k_sbgemv<MODE, E, O, RPT, V, LPC>;
  prep_smem((const void*)kern, gp.smem);
  static std::mutex mu;
  static std::map<std::tuple<int, int, size_t>, int> occ_cache;
  int occ = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(ctx->device, gp.block, gp.smem);
    auto it = occ_cache.find(key);
    if (it == occ_cache.end()) {
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, gp.block, gp.smem));
      occ_cache[key] = occ;
    } else {
      occ = it->second;
    }
  }
  if (occ < 1) fail(FMV_EUNSUPPORTED, "sbgemv: staged kernel does not fit on an SM");
  const int ctas_per_sm = std::min(occ, env_int("FMV_SBGEMV_CTAS_PER_SM", FMV_SBGEMV_MINB));
  long P = (long)sm_count(ctx->device) * ctas_per_sm;
  P = std::min(P, gp.p.T);
  gp.p.P = (int)P;
  if (MODE == GM_N) {
    const size_t part_bytes = (size_t)(P + gp.p.batch) * gp.p.m * sizeof(typename ET<E>::A);
    ctx->partials.ensure(part_bytes);
    gp.p.partials = ctx->partials.p;
    gp.p.counters = ctx->tickets((size_t)gp.p.batch);
  }
  launch(ctx, MODE == GM_N ? 1 : 2, [&] { launch_pdl(kern, dim3((unsigned)P), dim3(gp.block), gp.smem, ctx->stream, gp.p); });
}

template <int MODE, class E, class O>
void sbgemv_simple_t(fmv_ctx* ctx, GemvPlan& gp) {
  const long outs = MODE == GM_N ? gp.p.m : gp.p.n;
  dim3 grid((unsigned)((outs + 127) / 128), (unsigned)gp.p.batch);
  launch(ctx, MODE == GM_N ? 1 : 2, [&] { k_sbgemv_simple<MODE, E, O><<<grid, 128, 0, ctx->stream>>>(gp.p); });
}

constexpr int kConsumers = FMV_SBGEMV_CONS;  // k_sbgemv consumer threads per CTA (+1 producer warp)

// Fills the staged-kernel plan for V-element (16-byte) row vectors; returns
// false when the staged kernel's limits are exceeded (NoTrans: m > 4*256*V
// rows; a stage that does not fit shared memory).
bool plan_staged(GemvPlan& gp, int mode, size_t es, size_t accsz, int V) {
  GemvParams& p = gp.p;
  const long col_bytes = p.lda * (long)es;
  const int MV0 = (p.m + V - 1) / V;
  // short columns (one CTA per SM; tools/ab_wide.sh, tools/ab_half.sh): 3 x 48 KB,
  // except fp64 NoTrans 4 x 32 KB (fp16 NoTrans at 4 x 32 KB drops to 5.5 TB/s:
  // too few columns per thread per stage for its per-stage compensated fold)
  const bool n64 = mode == GM_N && es == 16;
  int a_target = n64 ? 32 * 1024 : 48 * 1024;
  int nst = n64 ? 4 : 3;
  if (mode != GM_N && MV0 > 128) {
    // tall (Conj)Trans columns: 64-96 KB stages (>= ~6 columns), one warp per
    // column, 3 stages when they fit the 227 KB per-CTA limit, else 2, shrunk
    // until they fit (tools/tune_conjtrans.py)
    const long xb = ((long)p.m * es + 32 + 127) / 128 * 128 + 128;
    const long budget = 220 * 1024;
    a_target = (int)std::min<long>(96 * 1024, std::max<long>(64 * 1024, 6 * col_bytes));
    nst = 3 * ((long)a_target + 256) + 2 * xb <= budget ? 3 : 2;
    while (a_target > col_bytes && (long)nst * (a_target + 256) + 2 * xb > budget) a_target -= (int)col_bytes;
  }
  a_target = env_int("FMV_SBGEMV_STAGE_BYTES", a_target);
  int Jc = (int)std::max<long>(1, a_target / std::max<long>(col_bytes, 1));
  const long max_a = ((long)(Jc - 1) * p.lda + p.m) * (long)es;
  if (max_a > 96 * 1024) return false;
  p.Jc = Jc;
  auto up128 = [](long v) { return (int)((v + 127) / 128 * 128); };
  p.a_slot = up128(max_a + 32);
  const long max_x = (mode == GM_N ? (long)Jc : (long)p.m) * (long)es;
  p.x_slot = up128(max_x + 32);
  p.nstage = std::max(2, std::min(16, env_int("FMV_SBGEMV_STAGES", nst)));
  size_t red = 0;
  const int MV = (p.m + V - 1) / V;
  if (mode == GM_N) {
    int rpt = 1;
    while ((MV + rpt - 1) / rpt > kConsumers) rpt *= 2;
    if (rpt > 4) return false;
    const int rpt_env = env_int("FMV_SBGEMV_RPT", 0);
    if ((rpt_env == 2 || rpt_env == 4) && rpt_env > rpt) rpt = rpt_env;
    p.RT = (MV + rpt - 1) / rpt;
    p.G = std::max(1, kConsumers / p.RT);
    const int ncons = (p.RT * p.G + 31) / 32 * 32;
    gp.block = ncons + 32;
    gp.rpt = rpt;
    red = (size_t)p.G * p.m * accsz;
  } else {
    // lanes per column: about <= 8 row vectors per lane for short columns,
    // whole warps (or several warps, combined in shared memory) for tall
    // ones; widen when a stage holds too few columns to keep 8 warps busy.
    // (fp16 C2 columns, 25 vectors: 4.9 TB/s with 8 lanes, 6.3 with 2, 6.5 with 4)
    int lpc = MV <= 16 ? 2 : MV <= 32 ? 4 : MV <= 128 ? 8 : MV <= 2048 ? 32 : 64;
    if (lpc > 32) {  // very tall columns: several warps per column
      while (lpc < kConsumers && lpc * 8 < MV) lpc *= 2;
      while ((long)Jc * lpc < kConsumers && lpc < kConsumers) lpc *= 2;
    }
    const int lpc_env = env_int("FMV_SBGEMV_LPC", 0);
    if (lpc_env == 2 || lpc_env == 4 || lpc_env == 8 || lpc_env == 32 || lpc_env == 64 || lpc_env == 128 ||
        lpc_env == 256)
      lpc = lpc_env;
    p.LPC = lpc;
    red = (size_t)(kConsumers / 32) * accsz;
    gp.block = kConsumers + 32;
  }
  // (Conj)Trans: keep x_b resident when every batch entry spans >= nstage stages
  p.xres = 0;
  p.xres_slot = 0;
  p.arrive_all = env_int("FMV_SBGEMV_ARRIVE_ALL", 0);
  if (mode != GM_N && (p.n + Jc - 1) / Jc >= p.nstage && env_int("FMV_SBGEMV_XRES", 1)) {
    p.xres = 1;
    p.xres_slot = p.x_slot;
  }
  gp.smem = 512 + (size_t)p.nstage * (p.a_slot + (p.xres ? 0 : p.x_slot)) + 2 * (size_t)p.xres_slot +
            (red + 127) / 128 * 128;
  if (gp.smem > 227 * 1024) return false;
  return true;
}

template <int MODE, class E, class O, int V>
void sbgemv_staged_v(fmv_ctx* ctx, GemvPlan& gp) {
  if constexpr (MODE == GM_N) {
    if (gp.rpt == 1) sbgemv_launch_t<MODE, E, O, 1, V, 0>(ctx, gp);
    else if (gp.rpt == 2) sbgemv_launch_t<MODE, E, O, 2, V, 0>(ctx, gp);
    else sbgemv_launch_t<MODE, E, O, 4, V, 0>(ctx, gp);
  } else {
    if (gp.p.LPC == 2) sbgemv_launch_t<MODE, E, O, 1, V, 2>(ctx, gp);
    else if (gp.p.LPC == 4) sbgemv_launch_t<MODE, E, O, 1, V, 4>(ctx, gp);
    else if (gp.p.LPC == 8) sbgemv_launch_t<MODE, E, O, 1, V, 8>(ctx, gp);
    else if (gp.p.LPC == 32) sbgemv_launch_t<MODE, E, O, 1, V, 32>(ctx, gp);
    else sbgemv_launch_t<MODE, E, O, 1, V, 0>(ctx, gp);  // multi-warp columns
  }
}

// Small (Conj)Trans problems (short columns, a few MB in all): the
// latency-oriented k_sbgemv_small (FMV_SBGEMV_SMALL=0 disables).
template <int MODE, class E, class O>
bool sbgemv_small_t(fmv_ctx* ctx, GemvPlan& gp) {
  if constexpr (MODE == GM_N) {
    return false;
  } else {
    constexpr int VMAX = (int)(16 / sizeof(E));
    const GemvParams& p = gp.p;
    const size_t bytes = (size_t)p.batch * p.n * p.m * sizeof(E);
    if (p.m > 64 || bytes > ((size_t)env_int("FMV_SBGEMV_SMALL_MB", 32) << 20) || !env_int("FMV_SBGEMV_SMALL", 1))
      return false;
    const auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    const bool vec = VMAX > 1 && p.m % VMAX == 0 && p.lda % VMAX == 0 && p.sa % VMAX == 0 && al16(p.A);
    const unsigned grid = (unsigned)((p.T + 127) / 128);
    launch(ctx, 2, [&] {
      if (vec) {
        if constexpr (VMAX > 1) launch_pdl(k_sbgemv_small<MODE, E, O, VMAX>, dim3(grid), dim3(128), 0, ctx->stream, gp.p);
      } else {
        launch_pdl(k_sbgemv_small<MODE, E, O, 1>, dim3(grid), dim3(128), 0, ctx->stream, gp.p);
      }
    });
    return true;
  }
}

template <int MODE, class E, class O>
void sbgemv_run_t(fmv_ctx* ctx, GemvPlan& gp, bool force_simple, int* used) {
  constexpr int VMAX = (int)(16 / sizeof(E));
  if (!force_simple && sbgemv_small_t<MODE, E, O>(ctx, gp)) {
    if (used) *used = 2;
    return;
  }
  // 16-byte row vectors need 16-byte aligned columns (and x for (Conj)Trans)
  const auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  bool vec = VMAX > 1 && gp.p.lda % VMAX == 0 && gp.p.sa % VMAX == 0 && al16(gp.p.A);
  if (MODE != GM_N) vec = vec && gp.p.sx % VMAX == 0 && al16(gp.p.x);
  const int V = vec ? VMAX : 1;
  const bool staged = !force_simple && plan_staged(gp, MODE, sizeof(E), sizeof(typename ET<E>::A), V);
  if (used) *used = staged ? 0 : 1;
  if (!staged) {
    sbgemv_simple_t<MODE, E, O>(ctx, gp);
    return;
  }
  if constexpr (VMAX > 1) {
    if (vec) {
      sbgemv_staged_v<MODE, E, O, VMAX>(ctx, gp);
      return;
    }
  }
  sbgemv_staged_v<MODE, E, O, 1>(ctx, gp);
}

template <class E, class O>
void sbgemv_mode(fmv_ctx* ctx, int mode, GemvPlan& gp, bool force_simple, int* used) {
  if (mode == GM_N) sbgemv_run_t<GM_N, E, O>(ctx, gp, force_simple, used);
  else if (mode == GM_T) sbgemv_run_t<GM_T, E, O>(ctx, gp, force_simple, used);
  else sbgemv_run_t<GM_C, E, O>(ctx, gp, force_simple, used);
}

GemvPlan make_gemv(const void* A, long m, long n, long batch, long lda, long sa, const void* x, long sx, void* y,
                   long sy) {
  GemvPlan gp;
  GemvParams& p = gp.p;
  p.A = static_cast<const unsigned char*>(A);
  p.lda = lda;
  p.sa = sa;
  p.x = static_cast<const unsigned char*>(x);
  p.sx = sx;
  p.y = static_cast<unsigned char*>(y);
  p.sy = sy;
  p.m = (int)m;
  p.n = n;
  p.batch = batch;
  p.T = batch * n;
  return gp;
}

template <class E>
void run_gemv_o(fmv_ctx* ctx, int p3, int mode, GemvPlan& gp) {
  if (p3 == PD) sbgemv_mode<E, double2>(ctx, mode, gp, false, nullptr);
  else sbgemv_mode<E, float2>(ctx, mode, gp, false, nullptr);
}
GemvPlan plan_of(const GemvArgs& a) {
  GemvPlan gp = make_gemv(a.A, a.m, a.n, a.batch, a.lda, a.sa, a.x, a.sx, a.y, a.sy);
  gp.p.yacc = a.yacc;
  gp.p.accum = a.accum;
  gp.p.K = a.K;
  gp.p.sxr = a.sxr;
  gp.p.syr = a.syr;
  return gp;
}

void gemv_run(fmv_ctx* ctx, int p2, int p3, int mode, const GemvArgs& a, bool acc64) {
  GemvPlan gp = plan_of(a);
  if (acc64 && p2 == PS) run_gemv_o<cf32d>(ctx, p3, mode, gp);  // the 'm' variant
  else if (p2 == PD) run_gemv_o<double2>(ctx, p3, mode, gp);
  else if (p2 == PS) run_gemv_o<float2>(ctx, p3, mode, gp);
  else run_gemv_o<__half2>(ctx, p3, mode, gp);
}

// ------------------------------------------------- block (multi-RHS) ----
// K right-hand sides through one pipeline, the per-bin
// SBGEMV replaced by the block kernel (fmv_sbgemm_block.cuh) that streams the
// operator once for up to kBlockMax RHS.
// Stage plan for k_sbgemm_block: ~32 KB of columns per stage, shrunk until
// two CTAs fit an SM; false if the shape is outside the kernel's limits.
bool plan_block(GemvPlan& gp, int mode, size_t es, size_t accsz, int KR) {
  GemvParams& p = gp.p;
  if (p.m < 1 || (mode == GM_N && p.m > kBlockConsumers)) return false;
  auto up128 = [](long v) { return (int)((v + 127) / 128 * 128); };
  const long col_bytes = std::max<long>(1, p.lda * (long)es);
  const long budget = FMV_BLOCK_MINB >= 2 ? 110 * 1024 : 220 * 1024;  // fit FMV_BLOCK_MINB CTAs per SM
  p.nstage = 3;
  int Jc = (int)std::max<long>(1, env_int("FMV_BLOCK_STAGE_BYTES", FMV_BLOCK_MINB >= 2 ? 32768 : 65536) / col_bytes);
  size_t red = 0;
  if (mode == GM_N) {
    p.RT = p.m;
    p.G = std::max(1, kBlockConsumers / p.RT);
    gp.block = (p.RT * p.G + 31) / 32 * 32 + 32;
  } else {
    gp.block = kBlockConsumers + 32;
  }
  for (;;) {
    const long max_a = ((long)(Jc - 1) * p.lda + p.m) * (long)es;
    p.Jc = Jc;
    p.a_slot = up128(max_a + 32);
    p.xr_slot = up128((mode == GM_N ? (long)Jc : (long)p.m) * (long)es + 32);
    p.xres = mode != GM_N && (p.n + Jc - 1) / Jc >= p.nstage;
    p.xres_slot = 0;
    red = mode == GM_N ? (size_t)p.G * KR * p.m * accsz : 0;
    const long xs = (long)KR * p.xr_slot;
    gp.smem = 512 + (size_t)p.nstage * (p.a_slot + (p.xres ? 0 : xs)) + (p.xres ? 2 * xs : 0) + (red + 127) / 128 * 128;
    if ((long)gp.smem <= budget || Jc == 1) break;
    Jc = std::max(1, Jc * 3 / 4);
  }
  p.arrive_all = env_int("FMV_SBGEMV_ARRIVE_ALL", 0);  // racecheck mode, as k_sbgemv
  return gp.smem <= 227 * 1024 && (long)(p.Jc - 1) * p.lda * (long)es + p.m * (long)es <= 96 * 1024;
}

template <int MODE, class E, class O, int KR, int LPC, int KX = 0, int XR = 0, int TC = 0>
void sbgemm_block_launch_t(fmv_ctx* ctx, GemvPlan& gp) {
  auto kern = k_sbgemm_block<MODE, E, O, KR, LPC, KX, XR, TC>;
  prep_smem((const void*)kern, gp.smem);
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, gp.block, gp.smem));
  if (occ < 1) fail(FMV_EUNSUPPORTED, "block sbgemv: kernel does not fit on an SM");
  long P = (long)sm_count(ctx->device) * std::min(occ, FMV_BLOCK_MINB);
  P = std::min(P, gp.p.T);
  gp.p.P = (int)P;
  if (MODE == GM_N) {
    ctx->partials.ensure((size_t)(P + gp.p.batch) * KR * gp.p.m * sizeof(typename ET<E>::A));
    gp.p.partials = ctx->partials.p;
    gp.p.counters = ctx->tickets((size_t)gp.p.batch);
  }
  launch(ctx, MODE == GM_N ? 1 : 2, [&] { kern<<<(unsigned)P, gp.block, gp.smem, ctx->stream>>>(gp.p); });
}

template <int MODE, class E, class O>
bool sbgemm_block_t(fmv_ctx* ctx, GemvPlan& gp) {
  const int K = gp.p.K;
  const int KR = K <= 2 ? 2 : K <= 4 ? 4 : 8;
  if (!plan_block(gp, MODE, sizeof(E), sizeof(typename ET<E>::A), KR)) return false;
  // ConjTrans lanes per column: 8 for columns up to 128 elements, else a warp
  constexpr int L1 = MODE == GM_N ? 0 : 8, L2 = MODE == GM_N ? 0 : 32;
  const bool wide = MODE != GM_N && gp.p.m > 128;
  if constexpr (MODE == GM_N && std::is_same<E, double2>::value) {
    // DMMA variant (K = 8, 88 < m <= 104: 13 row tiles of 8, 7 + 6 per warp
    // pair): nw consumer warps in nw/2 pairs, stages of exactly P column pairs
    // per warp pair, x slices 800 B apart (off the 128-byte bank period), one
    // K*m reduction buffer
    constexpr int kTC = 7, XRT = 800;  // tiles per warp: a warp pair covers 13 row tiles; x slot for <= 48 columns
    const int nw = env_int("FMV_BLOCK_TC_WARPS", 16);
    GemvParams& q = gp.p;
    if (K == 8 && q.m <= 8 * (2 * kTC - 1) && q.m > 8 * (2 * kTC - 3) && env_int("FMV_BLOCK_TC", 1) &&
        (nw == 8 || nw == 16)) {
      auto up128 = [](long v) { return (int)((v + 127) / 128 * 128); };
      // P = 2 column pairs per warp pair and stage (tools/bench_block.py, C2 K = 8
      // SBGEMV; the first design, one warp per column pair with all 13 tiles and
      // 8 warps: 1 pair 2.02 ms, 2 pairs 1.575 ms; CUDA-core kernel 1.754 ms)
      const int Jc = nw * std::max(1, env_int("FMV_BLOCK_TC_PAIRS", 2));
      const long a_bytes = ((long)(Jc - 1) * q.lda + q.m) * 16;
      const int a_slot = up128(a_bytes + 32);
      const size_t red = (size_t)(8 * q.m * 16 + 127) / 128 * 128;
      int ns = std::min(8, std::max(2, env_int("FMV_BLOCK_TC_STAGES", 8)));
      auto smem_of = [&](int n) { return (size_t)512 + (size_t)n * (a_slot + 8 * XRT) + red; };
      while (ns > 2 && smem_of(ns) > 227 * 1024) --ns;
      if (Jc * 16 + 32 <= XRT && smem_of(ns) <= 227 * 1024 && a_bytes <= 120 * 1024) {
        q.Jc = Jc;
        q.a_slot = a_slot;
        q.xr_slot = XRT;
        q.nstage = ns;
        q.G = 1;
        q.RT = q.m;
        gp.smem = smem_of(ns);
        gp.block = nw * 32 + 32;
        sbgemm_block_launch_t<MODE, E, O, 8, L1, 8, XRT, kTC>(ctx, gp);
        return true;
      }
    }
  }
  if constexpr (MODE == GM_N && std::is_same<E, double2>::value) {
    // exact-K variant with a fixed 1 KB x-slice stride (stages of <= 62 columns)
    constexpr int XR = 1024;
    GemvParams& q = gp.p;
    if ((K == 8 || K == 4) && K == KR && q.xr_slot <= XR && env_int("FMV_BLOCK_EXACT", 1)) {
      const size_t grow = (size_t)q.nstage * KR * (XR - q.xr_slot);
      if (gp.smem + grow <= 227 * 1024) {
        q.xr_slot = XR;
        gp.smem += grow;
        if (K == 8) sbgemm_block_launch_t<MODE, E, O, 8, L1, 8, XR>(ctx, gp);
        else sbgemm_block_launch_t<MODE, E, O, 4, L1, 4, XR>(ctx, gp);
        return true;
      }
    }
  }
  if constexpr (MODE != GM_N && std::is_same<E, double2>::value) {
    // two-columns-per-lane ConjTrans variant: W warps x 4 column groups x 2
    // columns per round, stages of exactly that many columns
    const int W = env_int("FMV_BLOCK_C2_WARPS", 8);  // tools/bench_block.py: W = 4..8 -> K=4 1.90 / 2.12 / 1.76 / 1.46 / 1.35 ms
    if (!wide && (K == 4 || K == 2) && K == KR && W >= 2 && W * 32 <= kBlockConsumers && env_int("FMV_BLOCK_C2", 1)) {
      GemvParams& q = gp.p;
      auto up128 = [](long v) { return (int)((v + 127) / 128 * 128); };
      const long es = (long)sizeof(E);
      const int Jc = W * 8;
      const long max_a = ((long)(Jc - 1) * q.lda + q.m) * es;
      const int a_slot = up128(max_a + 32), xr_slot = up128((long)q.m * es + 32);
      const long xs = (long)KR * xr_slot;
      int nst = 3;
      auto smem_of = [&](int ns, bool xres) {
        return (size_t)512 + (size_t)ns * (a_slot + (xres ? 0 : xs)) + (xres ? 2 * xs : 0);
      };
      if (smem_of(3, true) > 227 * 1024) nst = 2;
      const bool xres = (q.n + Jc - 1) / Jc >= nst;
      if (max_a <= 120 * 1024 && smem_of(nst, xres) <= 227 * 1024) {
        q.Jc = Jc;
        q.a_slot = a_slot;
        q.xr_slot = xr_slot;
        q.nstage = nst;
        q.xres = xres;
        q.xres_slot = 0;
        gp.smem = smem_of(nst, xres);
        gp.block = W * 32 + 32;
        if (K == 4) sbgemm_block_launch_t<MODE, E, O, 4, L1, 4>(ctx, gp);
        else sbgemm_block_launch_t<MODE, E, O, 2, L1, 2>(ctx, gp);
        return true;
      }
    }
  }
  if (KR == 2) wide ? sbgemm_block_launch_t<MODE, E, O, 2, L2>(ctx, gp) : sbgemm_block_launch_t<MODE, E, O, 2, L1>(ctx, gp);
  else if (KR == 4) wide ? sbgemm_block_launch_t<MODE, E, O, 4, L2>(ctx, gp) : sbgemm_block_launch_t<MODE, E, O, 4, L1>(ctx, gp);
  else wide ? sbgemm_block_launch_t<MODE, E, O, 8, L2>(ctx, gp) : sbgemm_block_launch_t<MODE, E, O, 8, L1>(ctx, gp);
  return true;
}

template <class E>
bool sbgemm_block_e(fmv_ctx* ctx, int p3, int mode, GemvPlan& gp) {
  if (mode == GM_N)
    return p3 == PD ? sbgemm_block_t<GM_N, E, double2>(ctx, gp) : sbgemm_block_t<GM_N, E, float2>(ctx, gp);
  return p3 == PD ? sbgemm_block_t<GM_C, E, double2>(ctx, gp) : sbgemm_block_t<GM_C, E, float2>(ctx, gp);
}

bool block_gemv_run(fmv_ctx* ctx, int p2, int p3, int mode, const GemvArgs& a) {
  GemvPlan gp = plan_of(a);
  return p2 == PD ? sbgemm_block_e<double2>(ctx, p3, mode, gp) : sbgemm_block_e<float2>(ctx, p3, mode, gp);
}

}  // namespace rt
}  // namespace fmv

extern "C" {

int fmv_sbgemv(fmv_ctx* ctx, int mode, char dtype, size_t m, size_t n, size_t batch, size_t lda, size_t stride_a,
               const void* A, size_t stride_x, const void* x, size_t stride_y, void* y, int force_simple,
               int* kernel_used) {
  return guarded([&] {
    if (!ctx || !A || !x || !y) fail(FMV_EINVAL, "gemv: null argument");
    if (m == 0 || n == 0 || batch == 0) fail(FMV_EINVAL, "gemv: empty matrix batch");
    if (lda < m) fail(FMV_EINVAL, "gemv: lda < rows");
    if (mode < 0 || mode > 2) fail(FMV_EINVAL, "gemv: bad mode");
    DeviceGuard dg(ctx->device);
    GemvPlan gp = make_gemv(A, (long)m, (long)n, (long)batch, (long)lda, (long)stride_a, x, (long)stride_x, y,
                            (long)stride_y);
    const bool fs = force_simple != 0;
    switch (dtype) {
      case 'z': sbgemv_mode<double2, double2>(ctx, mode, gp, fs, kernel_used); break;
      case 'c': sbgemv_mode<float2, float2>(ctx, mode, gp, fs, kernel_used); break;
      case 'h': sbgemv_mode<__half2, float2>(ctx, mode, gp, fs, kernel_used); break;
      case 'd':
        sbgemv_mode<double, double>(ctx, mode == GM_C ? GM_T : mode, gp, fs, kernel_used);
        break;
      case 's':
        sbgemv_mode<float, float>(ctx, mode == GM_C ? GM_T : mode, gp, fs, kernel_used);
        break;
      default: fail(FMV_EINVAL, "gemv: dtype must be s/d/c/z/h");
    }
  });
}

}  // extern "C"
