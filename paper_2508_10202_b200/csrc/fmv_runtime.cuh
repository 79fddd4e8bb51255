// fmv_runtime.cuh -- host runtime shared by the translation units of
// libfftmv_cuda (fmv_capi.cu: C ABI, pipeline, NCCL; fmv_fft_launch.cu: FFT
// kernel dispatch; fmv_gemv_launch.cu: SBGEMV / block SBGEMV dispatch):
// error mapping, contexts and operators, launch / timing helpers, caches of
// per-device kernel attributes and twiddle tables.
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/fftmv_cuda.h"
#include "fmv_common.cuh"
#include <nvtx3/nvToolsExt.h>
#include "fmv_fft_plan.cuh"

namespace fmv {
namespace rt {

// ======================================================================
// errors
// ======================================================================
extern thread_local std::string g_err;  // (fmv_capi.cu)

struct FmvError {
  int code;
  std::string msg;
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw FmvError{code, m}; }

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? FMV_ENOMEM : FMV_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define CK(x) ck((x), #x)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return FMV_OK;
  } catch (const FmvError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return FMV_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FMV_ECUDA;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    CK(cudaGetDevice(&prev));
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

extern std::atomic<uint64_t> g_casts;  // logical casts (precision.hpp:27-39; fmv_capi.cu)

inline int prec_of(char c) {
  switch (c) {
    case 'd': return PD;
    case 's': return PS;
    case 'h': return PH;
    default: fail(FMV_EINVAL, std::string("precision config: invalid character '") + c + "'");
  }
}

// A parsed config: p[0..4] the five phase precisions (PD / PS / PH), p[5] = 1
// for the 'm' SBGEMV variant (slot 3 only: fp32 operator and spectrum, fp64
// accumulation), whose storage precision p[2] is PS.
using Cfg = std::array<int, 6>;

// config.hpp:36-51 plus the extension rules: 'h' (fp16) at slots 1, 3, 5 and
// 'm' at slot 3.
inline Cfg parse_cfg(const char* cfg) {
  if (!cfg) fail(FMV_EINVAL, "precision config is null");
  const size_t len = strnlen(cfg, 16);
  if (len != 5)
    fail(FMV_EINVAL, "precision config must be exactly 5 characters, got " + std::to_string(len));
  Cfg p{};
  for (int i = 0; i < 5; ++i) {
    if (cfg[i] == 'm' && i == 2) {
      p[i] = PS;
      p[5] = 1;
      continue;
    }
    if (cfg[i] != 'd' && cfg[i] != 's' && cfg[i] != 'h')
      fail(FMV_EINVAL, std::string("precision config: invalid character '") + cfg[i] + "' at position " +
                           std::to_string(i + 1) + " (expected 'd', 's' or 'h'; 'm' at position 3)");
    p[i] = prec_of(cfg[i]);
  }
  if (p[1] == PH || p[3] == PH)
    fail(FMV_EINVAL, "precision config: fp16 ('h') is supported for phases 1, 3 and 5 only (pad, sbgemv, unpad)");
  return p;
}

// Logical cast passes of run_pipeline (matvec.hpp:88, :121-125, :163, :189-190);
// 'm' rounds exactly where 's' does.
inline uint64_t count_casts(const Cfg& p, bool payload) {
  uint64_t n = 0;
  if (!payload && p[0] != PD) ++n;
  if (p[0] != p[1]) ++n;
  if (p[1] != p[2]) ++n;
  if (p[2] != p[3]) ++n;
  if (p[3] != p[4]) ++n;
  if (p[4] != PD) ++n;
  return n;
}

inline size_t esize(int prec) { return prec == PD ? 16 : prec == PS ? 8 : 4; }

// ======================================================================
// twiddle tables (per device, per L, per precision) and kernel-attribute caches
// ======================================================================
struct TwiddleCache {
  std::mutex mu;
  // (device, L, prec, radices) -> device table: the base table
  // exp(-2*pi*i*m/L), m < L (exact at multiples of pi/2; fp32 tables hold the
  // float-rounded values), followed -- for a register FFT plan with radices
  // R_0..R_{np-1} -- by one table per pass p >= 1 laid out [q*Ns_p + k] =
  // base[q*k*L/(Ns_p*R_p)] (q < R_p, k < Ns_p = R_0*...*R_{p-1}), so a warp's
  // twiddle read for fixed q is contiguous in k (k_r2c_reg / k_c2r_reg,
  // k_r2c_rt / k_c2r_rt); the values are bitwise the base table's.
  std::map<std::tuple<int, int, int, std::vector<int>>, void*> tabs;
  ~TwiddleCache() {}  // tables live for the process (like the reference's plan cache, fft.hpp:152-164)

  // Base table only (RX = 0) or the uniform plan RX^NP of k_r2c_reg (RX > 1).
  const void* get(int dev, int L, int prec, int RX = 0) {
    std::vector<int> radices;
    if (RX > 1)
      for (int n = L / 2; n > 1; n /= RX) radices.push_back(RX);
    return get_plan(dev, L, prec, radices);
  }
  const void* get_plan(int dev, int L, int prec, const std::vector<int>& radices) {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, L, prec, radices);
    auto it = tabs.find(key);
    if (it != tabs.end()) return it->second;
    std::vector<double> re(L), im(L);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int m = 0; m < L; ++m) {
      long double c, s;
      if ((4L * m) % L == 0) {
        const int q = (int)((4L * m) / L);
        const int cs[4] = {1, 0, -1, 0}, sn[4] = {0, -1, 0, 1};
        c = cs[q];
        s = sn[q];
      } else {
        const long double a = -2.0L * pi * (long double)m / (long double)L;
        c = cosl(a);
        s = sinl(a);
      }
      re[m] = prec == PS ? (double)(float)c : (double)c;
      im[m] = prec == PS ? (double)(float)s : (double)s;
    }
    long Ns = radices.empty() ? 1 : radices[0];
    for (size_t p = 1; p < radices.size(); ++p) {
      const int R = radices[p];
      for (int q = 0; q < R; ++q)
        for (long k = 0; k < Ns; ++k) {
          const long m = (long)q * k * (L / (Ns * R));
          re.push_back(re[m]);
          im.push_back(im[m]);
        }
      Ns *= R;
    }
    const size_t n = re.size();
    void* d = nullptr;
    if (prec == PD) {
      std::vector<double2> h(n);
      for (size_t m = 0; m < n; ++m) h[m] = make_double2(re[m], im[m]);
      CK(cudaMalloc(&d, n * sizeof(double2)));
      CK(cudaMemcpy(d, h.data(), n * sizeof(double2), cudaMemcpyHostToDevice));
    } else {
      std::vector<float2> h(n);
      for (size_t m = 0; m < n; ++m) h[m] = make_float2((float)re[m], (float)im[m]);
      CK(cudaMalloc(&d, n * sizeof(float2)));
      CK(cudaMemcpy(d, h.data(), n * sizeof(float2), cudaMemcpyHostToDevice));
    }
    tabs[key] = d;
    return d;
  }
};
inline TwiddleCache& twiddles() {
  static TwiddleCache* c = new TwiddleCache;  // intentionally leaked: outlives static destructors
  return *c;
}

// Tunables (env overridable for on-GPU sweeps): SBGEMV stage bytes / ring
// depth / CTAs per SM, FFT shared-memory budget.
inline int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Kernel attributes are per device (cudaFuncSetAttribute applies to the
// current one), so both caches are keyed by (device, function).
inline int cur_device() {
  int d = 0;
  CK(cudaGetDevice(&d));
  return d;
}

// NVTX ranges (tracing): one per C-ABI matvec / setup call and one
// per pipeline phase group (r2c, SBGEMV, c2r, exchange), named "fftmv:...", so
// an nsys / ncu --nvtx timeline attributes every kernel to the reference's
// phases. Header-only NVTX3: a pointer test when no tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  explicit NvtxRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
inline std::string nvtx_matvec_name(const char* what, int kind, const char* cfg) {
  return std::string("fftmv:") + what + (kind == FMV_FORWARD ? " F " : " F* ") + (cfg ? cfg : "");
}

// Raise a kernel's dynamic shared-memory cap once per (device, function, size).
inline void prep_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> set;
  if (bytes <= 48 * 1024) return;
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = set[{dev, fn}];
  if (bytes > cur) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    cur = bytes;
  }
}

// Ask for the maximum shared-memory carveout once per (device, function), so
// more CTAs of the register FFT kernels fit per SM.
inline void prep_carveout(const void* fn) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, bool> set;
  const int dev = cur_device();
  std::lock_guard<std::mutex> lk(mu);
  bool& done = set[{dev, fn}];
  if (!done) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    done = true;
  }
}

inline int sm_count(int dev) {
  static std::mutex mu;
  static std::map<int, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  cache[dev] = n;
  return n;
}

}  // namespace rt
}  // namespace fmv

using namespace fmv;
using namespace fmv::rt;

// ======================================================================
// handles
// ======================================================================
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    CK(cudaMalloc(&p, bytes));
    n = bytes;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// Pinned (page-locked) host buffer, grow-only: staging for pageable caller I/O.
struct PinBuf {
  void* p = nullptr;
  size_t n = 0;
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
    CK(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
    n = bytes;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    n = 0;
  }
};

struct ProfRec {
  int cls;
  cudaEvent_t a, b;
};

struct fmv_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  DevBuf x, y, yacc, io_in, io_out, partials, counters, payload, red, fft_scratch;
  PinBuf pin_in, pin_out;  // staging for pageable host I/O (HostIO)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t cev[34] = {};
  // Queued host-I/O matvecs (fmv_matvec_host_async): two buffer slots used
  // alternately, so call i+1's input copy and r2c (copy_stream) run while
  // call i computes, and call i's output copy (out_stream) while call i+1
  // computes. q_done[s]: slot s's last compute finished (recorded on
  // `stream`); q_out[s]: its output copy finished (on out_stream).
  cudaStream_t out_stream = nullptr;
  DevBuf q_x[2], q_in[2], q_out_buf[2], q_scr[2];
  cudaEvent_t q_done[2] = {}, q_out[2] = {};
  int q_slot = 0;
  size_t counters_len = 0;
  uint64_t launches = 0;
  bool profiling = false;
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_pool;
  double prof_ms[5] = {0, 0, 0, 0, 0};
  uint64_t prof_n[5] = {0, 0, 0, 0, 0};
  void* comm = nullptr;
  int nranks = 1, rank = 0;
  // 2-D pr x pc grid (fmv_comm_init_2d): rank = ri * pc + cj; row_comm joins
  // the pc ranks of grid row ri, col_comm the pr ranks of grid column cj.
  void* row_comm = nullptr;
  void* col_comm = nullptr;
  int pr = 1, pc = 1, ri = 0, cj = 0;
  cudaEvent_t te[8] = {};
  // PhaseTimings of one blocking matvec (fmv_matvec with times != NULL):
  // every kernel launch, copy and collective records a CUDA-event pair on the
  // stream it runs on, tagged with the reference phase it belongs to.
  bool phase_timing = false;
  struct PhaseRec {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<PhaseRec> phase_recs;

  cudaEvent_t ev() {
    if (!ev_pool.empty()) {
      cudaEvent_t e = ev_pool.back();
      ev_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  // Zeroed ticket counters for the SBGEMV-N cross-CTA reduction.
  unsigned* tickets(size_t nbatch) {
    if (nbatch > counters_len) {
      counters.ensure(nbatch * sizeof(unsigned));
      CK(cudaMemsetAsync(counters.p, 0, nbatch * sizeof(unsigned), stream));
      counters_len = nbatch;
    }
    return static_cast<unsigned*>(counters.p);
  }
};

struct fmv_op {
  int device = 0;
  size_t nm = 0, nd = 0, nt = 0;
  void* bins_d = nullptr;  // double2, lda = nd
  // fp32 / fp16 copies, published (release) only after their cast kernel has
  // finished and lda_s / lda_h are set; readers load them with acquire.
  std::atomic<void*> bins_s{nullptr};  // float2, lda = lda_s
  std::atomic<void*> bins_h{nullptr};  // __half2, lda = lda_h
  size_t lda_s = 0, lda_h = 0;
  std::mutex mu;
  size_t nb() const { return nt + 1; }
};


namespace fmv {
namespace rt {


// ---------------------------------------------------------------- launch --
// Reference phase (matvec.hpp:42-51) a kernel class is charged to: r2c ->
// [1] fft (pad + convert + reorder fused in), SBGEMV -> [2], c2r -> [3] ifft
// (reorder + unpad fused in). Class 4 (cast kernels) is charged explicitly by
// the caller; a first fp32/fp16 operator materialization inside a matvec goes
// to [2] like the reference's ensure_single inside gemv_stage.
constexpr int kPhaseOfClass[5] = {1, 2, 2, 3, 2};

// Run fn (which enqueues work on `s`) inside a CUDA-event span of `phase`
// when the context is collecting PhaseTimings.
template <class Fn>
void phase_span(fmv_ctx* ctx, cudaStream_t s, int phase, Fn&& fn) {
  if (!ctx->phase_timing) {
    fn();
    return;
  }
  fmv_ctx::PhaseRec r{phase, ctx->ev(), ctx->ev()};
  CK(cudaEventRecord(r.a, s));
  fn();
  CK(cudaEventRecord(r.b, s));
  ctx->phase_recs.push_back(r);
}

template <class Fn>
void launch(fmv_ctx* ctx, int cls, Fn&& fn, int phase = -1) {
  ProfRec r{cls, nullptr, nullptr};
  if (ctx->profiling) {
    r.a = ctx->ev();
    r.b = ctx->ev();
    CK(cudaEventRecord(r.a, ctx->stream));
  }
  phase_span(ctx, ctx->stream, phase >= 0 ? phase : kPhaseOfClass[cls], [&] {
    fn();
    CK(cudaGetLastError());
  });
  ++ctx->launches;
  if (ctx->profiling) {
    CK(cudaEventRecord(r.b, ctx->stream));
    ctx->prof.push_back(r);
  }
}

// cudaMemcpyAsync charged to a phase ([0] for input copies, [4] for output).
inline void copy_async(fmv_ctx* ctx, int phase, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind,
                cudaStream_t s) {
  phase_span(ctx, s, phase, [&] { CK(cudaMemcpyAsync(dst, src, bytes, kind, s)); });
}

// Collects the phase spans of one matvec: sums the busy time per phase
// (spans of one phase never overlap each other; spans of different phases
// may, on the overlapped host-I/O path) and the wall time from `t0` to `t1`
// (events recorded on the matvec stream around everything). Call after the
// stream has been synchronized.
inline void collect_phase_times(fmv_ctx* ctx, cudaEvent_t t0, cudaEvent_t t1, fmv_phase_times* out) {
  double ms[5] = {0, 0, 0, 0, 0};
  for (auto& r : ctx->phase_recs) {
    float v = 0.f;
    CK(cudaEventElapsedTime(&v, r.a, r.b));
    ms[r.phase] += v;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->phase_recs.clear();
  float tot = 0.f;
  CK(cudaEventElapsedTime(&tot, t0, t1));
  for (int i = 0; i < 5; ++i) out->phase_s[i] = ms[i] * 1e-3;
  out->total_s = tot * 1e-3;
}

// Turns per-call phase timing on for a scope (and drops the records of a
// call that failed part-way).
struct PhaseTimingScope {
  fmv_ctx* ctx;
  PhaseTimingScope(fmv_ctx* c, bool on) : ctx(c) {
    for (auto& r : ctx->phase_recs) {
      ctx->ev_pool.push_back(r.a);
      ctx->ev_pool.push_back(r.b);
    }
    ctx->phase_recs.clear();
    ctx->phase_timing = on;
  }
  ~PhaseTimingScope() { ctx->phase_timing = false; }
};

// Launch with programmatic dependent launch allowed (FMV_PDL=0 disables).
template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  static const bool on = env_int("FMV_PDL", 1) != 0;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = on ? 1 : 0;
  CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

inline unsigned grid_for(long n, int block, int dev) {
  const long want = (n + block - 1) / block;
  const long cap = (long)sm_count(dev) * 16;
  return (unsigned)std::max<long>(1, std::min(want, cap));
}

// Host memcpy split across a small persistent thread pool (fmv_hostpool.cpp).
void parallel_memcpy(void* dst, const void* src, size_t bytes);

// Is p ordinary pageable host memory (not pinned / registered, not device)?
inline bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// ---- entry points shared across the translation units ----
// FFT dispatch (fmv_fft_launch.cu). N = L/2 (complex FFT length); nvalid =
// input samples per series (Nt for the zero-padded matvec path, L for a
// plain transform); input element (s, t) at in[s*in_ss + t*in_ts], bin k of
// series s at out[k*out_ks + s*out_ss].
template <class Tin>
void r2c_dispatch(fmv_ctx* ctx, int c0, int c1, int c2, const Tin* in, long in_ss, long in_ts, long nseries, int N,
                  int nvalid, void* out, long out_ks, long out_ss);
void c2r_dispatch(fmv_ctx* ctx, int c3, int c4, const void* in, long in_ks, long in_ss, long nseries, int N,
                  int nout, double* out, long out_ss);

// Runtime-plan register FFTs (fmv_fft_rt.cuh), one explicit instantiation per
// pass radix RR in fmv_fft_rt_{a,b,c}.cu: cr = arithmetic precision (PD/PS),
// tin / tout = precision of the real input / output array, c0 / c2 / c4 the
// pipeline roundings; tw = the plan's twiddle table (TwiddleCache::get_plan).
template <int RR>
void rt_r2c_run(fmv_ctx* ctx, int cr, int tin, int c0, int c2, const void* in, long in_ss, long nseries, int nvalid,
                void* out, long out_ks, long out_ss, const RtPlan& P, const void* tw);
template <int RR>
void rt_c2r_run(fmv_ctx* ctx, int cr, int tout, int c4, const void* in, long in_ks, long in_ss, long nseries,
                int nout, void* out, long out_ss, const RtPlan& P, const void* tw);

// SBGEMV dispatch (fmv_gemv_launch.cu): y_b = op(A_b) x_b for b < batch,
// strides in elements of the SBGEMV precision p2, output in p3.
struct GemvArgs {
  const void* A = nullptr;
  long m = 0, n = 0, batch = 0, lda = 0, sa = 0;
  const void* x = nullptr;
  long sx = 0;
  void* y = nullptr;
  long sy = 0;
  void* yacc = nullptr;  // NoTrans column-chunk fold buffer (GemvParams::yacc / accum)
  int accum = 0;
  int K = 1;             // block SBGEMV: right-hand sides, per-RHS strides of x / y within a bin
  long sxr = 0, syr = 0;
};
// acc64: the 'm' variant (p2 == PS storage, fp64 accumulators)
void gemv_run(fmv_ctx* ctx, int p2, int p3, int mode, const GemvArgs& a, bool acc64 = false);
// Block (multi-RHS) SBGEMV; false when the shape is outside the kernel's limits.
bool block_gemv_run(fmv_ctx* ctx, int p2, int p3, int mode, const GemvArgs& a);
constexpr int kBlockMax = 8;
inline int block_max(bool fwd) { return fwd ? kBlockMax : 4; }
#ifndef FMV_BLOCK_CONS
#define FMV_BLOCK_CONS 416  // k_sbgemm_block consumer threads per CTA (+ one producer warp)
#endif
constexpr int kBlockConsumers = FMV_BLOCK_CONS;

}  // namespace rt
}  // namespace fmv
