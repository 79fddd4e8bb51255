// fmv_capi.cu -- host runtime behind include/fftmv_cuda.h.
//
// Owns device memory for spectral operators, per-context workspaces and
// streams, runs the fused sm_100a kernels of the five-phase pipeline
// (matvec.hpp:233-289; FFT dispatch in fmv_fft_launch.cu, SBGEMV dispatch in
// fmv_gemv_launch.cu) and the 1 x p / 2-D NCCL partition
// (partition.hpp:141-217). No CPU fallback exists: every compute entry point
// launches CUDA kernels and fails loudly on any CUDA error.
#include <dlfcn.h>

#include "fmv_runtime.cuh"

namespace fmv {
namespace rt {
thread_local std::string g_err;
std::atomic<uint64_t> g_casts{0};
}  // namespace rt
}  // namespace fmv

namespace {
// ======================================================================
// NCCL (dlopen'ed on first use: only the partitioned path needs it)
// ======================================================================
struct Nccl {
  typedef int (*GetUniqueId)(void*);
  typedef int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t);
  typedef int (*Broadcast)(const void*, void*, size_t, int, int, void*, cudaStream_t);
  typedef int (*CommDestroy)(void*);
  typedef int (*CommAbort)(void*);
  typedef int (*CommSplit)(void*, int, int, void**, void*);
  typedef int (*GetAsyncError)(void*, int*);
  typedef const char* (*GetErrorString)(int);
  void* h = nullptr;
  std::string path;
  GetUniqueId get_unique_id = nullptr;
  void* comm_init_rank = nullptr;  // ncclUniqueId (128 bytes) is passed by value: cast at the call site
  AllReduce all_reduce = nullptr;
  AllGather all_gather = nullptr;
  Broadcast broadcast = nullptr;
  CommDestroy comm_destroy = nullptr;
  CommAbort comm_abort = nullptr;
  CommSplit comm_split = nullptr;
  GetAsyncError get_async_error = nullptr;
  GetErrorString err = nullptr;
};
// NCCL is dlopen'ed on first use (only the partitioned path needs it).
// FMV_NCCL_LIB names another library exporting the same symbols (e.g. the
// host-staged test transport, tests/stub/fmv_nccl_stub.cpp, which lets
// several processes share one GPU).
Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<std::string> names;
    if (const char* e = getenv("FMV_NCCL_LIB"); e && *e) names.push_back(e);
    else names = {"libnccl.so.2", "libnccl.so"};
    for (const auto& nm : names)
      if ((n.h = dlopen(nm.c_str(), RTLD_NOW | RTLD_GLOBAL))) {
        n.path = nm;
        break;
      }
    if (!n.h) return;
    n.get_unique_id = (Nccl::GetUniqueId)dlsym(n.h, "ncclGetUniqueId");
    n.comm_init_rank = dlsym(n.h, "ncclCommInitRank");
    n.all_reduce = (Nccl::AllReduce)dlsym(n.h, "ncclAllReduce");
    n.all_gather = (Nccl::AllGather)dlsym(n.h, "ncclAllGather");
    n.broadcast = (Nccl::Broadcast)dlsym(n.h, "ncclBroadcast");
    n.comm_destroy = (Nccl::CommDestroy)dlsym(n.h, "ncclCommDestroy");
    n.comm_abort = (Nccl::CommAbort)dlsym(n.h, "ncclCommAbort");
    n.comm_split = (Nccl::CommSplit)dlsym(n.h, "ncclCommSplit");
    n.get_async_error = (Nccl::GetAsyncError)dlsym(n.h, "ncclCommGetAsyncError");
    n.err = (Nccl::GetErrorString)dlsym(n.h, "ncclGetErrorString");
  });
  if (!n.h || !n.get_unique_id || !n.comm_init_rank || !n.all_gather || !n.broadcast)
    fail(FMV_ENCCL, std::string("NCCL (") + (getenv("FMV_NCCL_LIB") ? getenv("FMV_NCCL_LIB") : "libnccl.so.2") +
                        ") could not be loaded: " + (n.h ? "missing symbols" : dlerror() ? dlerror() : "dlopen failed"));
  return n;
}
void nck(int rc, const char* what) {
  if (rc != 0) fail(FMV_ENCCL, std::string(what) + ": " + (nccl().err ? nccl().err(rc) : "nccl error"));
}
// ncclDataType_t / ncclRedOp_t values (nccl.h)
constexpr int kNcclHalf = 6, kNcclFloat = 7, kNcclDouble = 8, kNcclSum = 0;

}  // namespace

// ======================================================================
// pipeline
// ======================================================================
namespace {

// ------------------------------------------------------------ pipeline ----
const void* op_bins(fmv_ctx* ctx, fmv_op* op, int prec, long* lda);

// Column chunking of the operator for the host-I/O pipeline (a function of
// shape, SBGEMV precision and direction only). Chunk sizes grow (F) or shrink
// (F*) geometrically by 1.6x: PCIe moves a column about 1.7x faster than the
// SBGEMV consumes one, so each chunk's copy hides behind its neighbour's
// SBGEMV and only the smallest chunk's copy is exposed. Edges on multiples of
// 4 columns.
std::vector<long> chunk_edges(const fmv_op* op, int prec2, bool grow, int force = 0) {
  const long nm = (long)op->nm;
  const size_t bytes = op->nb() * op->nm * op->nd * esize(prec2);
  long C = (bytes >= (size_t(1) << 30)) ? 6 : (bytes >= (size_t(1) << 27)) ? 3 : 1;
  const int env = env_int("FMV_CHUNKS", 0);
  if (env > 0) C = env;
  if (force > 0) C = force;
  C = std::max<long>(1, std::min<long>(C, nm / 4));
  std::vector<double> w(C);
  double tot = 0;
  for (long c = 0; c < C; ++c) tot += (w[c] = std::pow(1.6, (double)(grow ? c : C - 1 - c)));
  std::vector<long> e(C + 1, 0);
  double acc = 0;
  for (long c = 1; c < C; ++c) {
    acc += w[c - 1];
    e[c] = std::max(e[c - 1] + 4, ((long)(nm * acc / tot)) & ~3L);
  }
  e[C] = nm;
  for (long c = C - 1; c >= 1; --c) e[c] = std::min(e[c], e[c + 1] - 1);  // keep chunks non-empty
  return e;
}

// Run the launches of a scope on another stream (the ctx's launch helpers
// enqueue on ctx->stream).
struct StreamSwap {
  fmv_ctx* ctx;
  cudaStream_t saved;
  StreamSwap(fmv_ctx* c, cudaStream_t s) : ctx(c), saved(c->stream) { c->stream = s; }
  ~StreamSwap() { ctx->stream = saved; }
};

// Host side of a blocking matvec with host buffers. Pinned caller buffers are
// copied by DMA directly; pageable ones (the reference API's std::vectors)
// go through the context's pinned staging buffers, filled / drained by the
// host thread pool while the GPU works on neighbouring chunks.
struct HostIO {
  const void* h_in = nullptr;  // copy in (overlapped) to the device `in` buffer
  double* h_out = nullptr;     // copy out (overlapped) from the device `out` buffer
  size_t in_elem = 8;          // bytes per input element (a cfg[0] payload may be float / half)
  unsigned char* pin_in = nullptr;  // staging (set when h_in is pageable)
  double* pin_out = nullptr;        // staging (set when h_out is pageable)
  // Queued call (fmv_matvec_host_async): pinned buffers only; the copy stream
  // waits on `guard` (the slot's previous compute) instead of everything
  // enqueued before, output copies run on the ctx's out_stream and nothing
  // joins back into the matvec stream.
  bool queued = false;
  cudaEvent_t guard = nullptr;
  struct Pending {
    size_t off, count;
    cudaEvent_t ev;
  };
  std::vector<Pending> pending;  // staged output chunks not yet copied to h_out

  // host bytes [off, off + bytes) of the input -> device dst. A pageable
  // source is staged in ~2 MB pieces, each piece's DMA issued as soon as it
  // is staged, so the copy engine streams while the host copies the next
  // piece (one whole-chunk memcpy before the DMA serialized the two:
  // F 2.7 ms -> DESIGN.md §3.5).
  void h2d(fmv_ctx* ctx, void* dst, size_t off, size_t bytes, cudaStream_t s) const {
    const unsigned char* src = static_cast<const unsigned char*>(h_in) + off;
    if (!pin_in) {
      copy_async(ctx, 0, dst, src, bytes, cudaMemcpyHostToDevice, s);
      return;
    }
    const size_t piece = (size_t)env_int("FMV_STAGE_PIECE_KB", 2048) << 10;
    for (size_t o = 0; o < bytes; o += piece) {
      const size_t b = std::min(piece, bytes - o);
      parallel_memcpy(pin_in + off + o, src + o, b);
      copy_async(ctx, 0, static_cast<unsigned char*>(dst) + o, pin_in + off + o, b, cudaMemcpyHostToDevice, s);
    }
  }
  // device src -> output doubles [off, off + count); staged chunks complete in
  // drain(). A pageable destination is drained in ~2 MB pieces, each with its
  // own event, so the host copy of one piece overlaps the DMA of the next.
  fmv_ctx* ev_ctx = nullptr;
  size_t last_pieces = 0;  // pieces of the newest d2h call
  void d2h(fmv_ctx* ctx, size_t off, const double* src, size_t count, cudaStream_t s, cudaEvent_t ev) {
    if (!pin_out) {
      copy_async(ctx, 4, h_out + off, src, count * sizeof(double), cudaMemcpyDeviceToHost, s);
      return;
    }
    (void)ev;
    ev_ctx = ctx;
    const size_t piece = std::max<size_t>(1, ((size_t)env_int("FMV_STAGE_PIECE_KB", 2048) << 10) / sizeof(double));
    last_pieces = 0;
    for (size_t o = 0; o < count; o += piece) {
      const size_t c = std::min(piece, count - o);
      copy_async(ctx, 4, pin_out + off + o, src + o, c * sizeof(double), cudaMemcpyDeviceToHost, s);
      cudaEvent_t e = ctx->ev();
      CK(cudaEventRecord(e, s));
      pending.push_back({off + o, c, e});
      ++last_pieces;
    }
  }
  // Copy staged output pieces to h_out: all but those of the newest d2h call
  // (newest = true), or all of them.
  void drain(bool all_but_newest = false) {
    const size_t keep = all_but_newest ? last_pieces : 0;
    while (pending.size() > keep) {
      const Pending q = pending.front();
      pending.erase(pending.begin());
      CK(cudaEventSynchronize(q.ev));
      parallel_memcpy(h_out + q.off, pin_out + q.off, q.count * sizeof(double));
      ev_ctx->ev_pool.push_back(q.ev);
    }
  }
};

cudaStream_t copy_stream(fmv_ctx* ctx) {
  if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  return ctx->copy_stream;
}
cudaStream_t out_stream(fmv_ctx* ctx) {
  if (!ctx->out_stream) CK(cudaStreamCreateWithFlags(&ctx->out_stream, cudaStreamNonBlocking));
  return ctx->out_stream;
}
cudaEvent_t chunk_event(fmv_ctx* ctx, int i) {
  if (!ctx->cev[i]) CK(cudaEventCreateWithFlags(&ctx->cev[i], cudaEventDisableTiming));
  return ctx->cev[i];
}

// run_pipeline (matvec.hpp:233-289) on device buffers, enqueued on ctx->stream.
// payload_prec >= 0: `in` holds the broadcast payload already in that
// precision (partition.hpp:198-212); otherwise `in` is double. With `hio`, the
// host input is copied into `in` chunk by chunk (F) and the output leaves
// chunk by chunk (F*) on a copy stream, overlapped with the SBGEMV.
void pipeline(fmv_ctx* ctx, const fmv_op* cop, int kind, const Cfg& p, const void* in,
              int payload_prec, double* out, HostIO* hio = nullptr) {
  fmv_op* op = const_cast<fmv_op*>(cop);
  const bool fwd = kind == FMV_FORWARD;
  const long nt = (long)op->nt, nb = (long)op->nb();
  const long n_in = fwd ? (long)op->nm : (long)op->nd;
  const long n_out = fwd ? (long)op->nd : (long)op->nm;
  long lda = 0;
  const void* bins = op_bins(ctx, op, p[2], &lda);
  const size_t e2 = esize(p[2]), e3 = esize(p[3]);
  // TOSI stride of the spectrum padded to 4 elements so every bin's x_k starts
  // 16-byte aligned (vectorized SBGEMV-C loads).
  const long sx = (n_in + 3) / 4 * 4;
  ctx->x.ensure((size_t)nb * sx * e2 + 256);
  ctx->y.ensure((size_t)nb * n_out * e3 + 256);
  const long m = (long)op->nd, n = (long)op->nm;
  const bool h_in = hio && hio->h_in, h_out = hio && hio->h_out;
  // Device-resident I/O streams the SBGEMV in one launch; host I/O splits it
  // into column chunks so the copies hide behind it. (For F the chunk sums
  // are folded in chunk order, so the two entry points agree to rounding;
  // each is deterministic.)
  // (Device-resident F split the same way -- each chunk's r2c on the copy
  // stream beside the previous chunk's SBGEMV -- was measured slower: 1.206 ms
  // per F unchunked, 1.22 / 1.23 / 1.24 / 1.26 ms with 2 / 3 / 4 / 6 chunks.)
  // Queued calls overlap their copies with the neighbouring calls instead, so
  // they run unchunked by default (FMV_QCHUNKS: 1 -> 820, 2 -> 816, 3 -> 807,
  // 6 -> 784 e2e matvecs/s at C2; device-resident 817).
  const int qchunks = hio && hio->queued ? env_int("FMV_QCHUNKS", 1) : 0;
  const std::vector<long> edges =
      (h_in || h_out) ? chunk_edges(op, p[2], fwd, qchunks) : std::vector<long>{0, (long)op->nm};
  const int C = (int)edges.size() - 1;
  auto chunk_edge = [&](long, int c, int) { return edges[c]; };
  cudaStream_t cs = ctx->stream;
  if (C > 16) fail(FMV_EINVAL, "too many chunks");
  const bool queued = hio && hio->queued;
  if (queued) {  // only this slot's previous compute may still read its buffers
    CK(cudaStreamWaitEvent(copy_stream(ctx), hio->guard, 0));
  } else if (h_in || h_out) {  // the copy stream must not run ahead into a buffer still in use
    CK(cudaEventRecord(chunk_event(ctx, 32), cs));
    CK(cudaStreamWaitEvent(copy_stream(ctx), chunk_event(ctx, 32), 0));
  }

  // Phases 1-2 (+ reorder to TOSI, cast to cfg[2]) over series [s0, s1).
  auto r2c_series = [&](long s0, long s1) {
    NvtxRange nr("fftmv:r2c");
    void* xo = static_cast<unsigned char*>(ctx->x.p) + s0 * e2;
    const long cnt = s1 - s0;
    if (payload_prec < 0)
      r2c_dispatch<double>(ctx, p[0], p[1], p[2], static_cast<const double*>(in) + s0 * nt, nt, 1, cnt, (int)nt,
                           (int)nt, xo, sx, 1);
    else if (payload_prec == PD)
      r2c_dispatch<double>(ctx, PD, p[1], p[2], static_cast<const double*>(in) + s0 * nt, nt, 1, cnt, (int)nt,
                           (int)nt, xo, sx, 1);
    else if (payload_prec == PS)
      r2c_dispatch<float>(ctx, PS, p[1], p[2], static_cast<const float*>(in) + s0 * nt, nt, 1, cnt, (int)nt, (int)nt,
                          xo, sx, 1);
    else
      r2c_dispatch<__half>(ctx, PH, p[1], p[2], static_cast<const __half*>(in) + s0 * nt, nt, 1, cnt, (int)nt,
                           (int)nt, xo, sx, 1);
  };
  // Phase 3 SBGEMV in cfg[2] over columns [j0, j1), output cast to cfg[3], TOSI.
  auto gemv_chunk = [&](int c) {
    NvtxRange nr("fftmv:sbgemv");
    const long j0 = chunk_edge(n, c, C), j1 = chunk_edge(n, c + 1, C);
    const void* A = static_cast<const unsigned char*>(bins) + j0 * lda * (long)e2;
    GemvArgs g;
    g.A = A;
    g.m = m;
    g.n = j1 - j0;
    g.batch = nb;
    g.lda = lda;
    g.sa = n * lda;
    if (fwd) {
      g.x = static_cast<unsigned char*>(ctx->x.p) + j0 * e2;
      g.sx = sx;
      g.y = ctx->y.p;
      g.sy = m;
      ctx->yacc.ensure((size_t)nb * m * 16 + 256);
      g.yacc = ctx->yacc.p;
      g.accum = C == 1 ? 0 : c == 0 ? 1 : c == C - 1 ? 3 : 2;
    } else {
      g.x = ctx->x.p;
      g.sx = sx;
      g.y = static_cast<unsigned char*>(ctx->y.p) + j0 * e3;
      g.sy = n;
    }
    gemv_run(ctx, p[2], p[3], fwd ? FMV_GEMV_N : FMV_GEMV_C, g, p[5] != 0);
  };
  // Phases 4-5 (+ reorder back to SOTI, 1/L in cfg[3], unpad, cast cfg[4]) over series [s0, s1).
  auto c2r_series = [&](long s0, long s1) {
    NvtxRange nr("fftmv:c2r");
    c2r_dispatch(ctx, p[3], p[4], static_cast<unsigned char*>(ctx->y.p) + s0 * e3, n_out, 1, s1 - s0, (int)nt,
                 (int)nt, out + s0 * nt, nt);
  };

  if (fwd) {
    if (h_in) {
      cudaStream_t ks = copy_stream(ctx);
      // With overlap (default) the r2c of chunk c runs on the copy stream right
      // after its H2D, so it executes alongside the SBGEMV of chunk c-1 (one
      // 200-thread r2c CTA fits next to the one-CTA-per-SM SBGEMV) instead
      // of serializing with it on the matvec stream.
      const bool ovl = env_int("FMV_E2E_OVERLAP", 1) != 0;
      auto issue_in = [&](int c) {
        const long j0 = chunk_edge(n, c, C), j1 = chunk_edge(n, c + 1, C);
        const size_t ie = hio->in_elem;
        hio->h2d(ctx, const_cast<unsigned char*>(static_cast<const unsigned char*>(in)) + j0 * nt * ie, j0 * nt * ie,
                 (size_t)(j1 - j0) * nt * ie, ks);
        if (ovl) {
          StreamSwap sw(ctx, ks);
          r2c_series(j0, j1);
        }
        CK(cudaEventRecord(chunk_event(ctx, c), ks));
      };
      // Chunk c+1's copy is issued after chunk c's SBGEMV is enqueued: from a
      // pageable buffer cudaMemcpyAsync blocks the host until the data is
      // staged, and this order keeps the SBGEMV running meanwhile.
      issue_in(0);
      for (int c = 0; c < C; ++c) {
        CK(cudaStreamWaitEvent(cs, chunk_event(ctx, c), 0));
        if (!ovl) r2c_series(chunk_edge(n, c, C), chunk_edge(n, c + 1, C));
        gemv_chunk(c);
        if (c + 1 < C) issue_in(c + 1);
      }
    } else {
      r2c_series(0, n_in);
      for (int c = 0; c < C; ++c) gemv_chunk(c);
    }
    c2r_series(0, n_out);
    if (h_out && queued) {  // the next call's compute does not wait for this copy
      CK(cudaEventRecord(chunk_event(ctx, 30), cs));
      CK(cudaStreamWaitEvent(out_stream(ctx), chunk_event(ctx, 30), 0));
      hio->d2h(ctx, 0, out, (size_t)n_out * nt, out_stream(ctx), nullptr);
    } else if (h_out) {
      hio->d2h(ctx, 0, out, (size_t)n_out * nt, cs, chunk_event(ctx, 16));
    }
  } else {
    if (h_in && queued) {  // copied beside the previous call's compute
      hio->h2d(ctx, const_cast<void*>(in), 0, (size_t)n_in * nt * hio->in_elem, copy_stream(ctx));
      CK(cudaEventRecord(chunk_event(ctx, 31), copy_stream(ctx)));
      CK(cudaStreamWaitEvent(cs, chunk_event(ctx, 31), 0));
    } else if (h_in) {
      hio->h2d(ctx, const_cast<void*>(in), 0, (size_t)n_in * nt * hio->in_elem, cs);
    }
    r2c_series(0, n_in);
    if (h_out) {
      cudaStream_t ks = queued ? out_stream(ctx) : copy_stream(ctx);
      // (chunk c's c2r stays on the matvec stream: on the copy stream, running
      // alongside the SBGEMV of chunk c+1, it slowed F* from 1.37 to 1.62 ms
      // with a full grid and to 2.13 ms with one-CTA-per-SM sub-launches --
      // the c2r's shared-memory traffic competes with the ConjTrans consumers)
      // Chunk c's copy-out is issued after chunk c+1's SBGEMV is enqueued (a
      // pageable destination makes cudaMemcpyAsync block the host until the
      // copy is done).
      auto issue_out = [&](int c) {
        const long j0 = chunk_edge(n, c, C), j1 = chunk_edge(n, c + 1, C);
        CK(cudaStreamWaitEvent(ks, chunk_event(ctx, c), 0));
        hio->d2h(ctx, j0 * nt, out + j0 * nt, (size_t)(j1 - j0) * nt, ks, chunk_event(ctx, 16 + c));
        hio->drain(true);  // the previous staged chunk's host copy overlaps this chunk's SBGEMV
      };
      for (int c = 0; c < C; ++c) {
        const long j0 = chunk_edge(n, c, C), j1 = chunk_edge(n, c + 1, C);
        gemv_chunk(c);
        c2r_series(j0, j1);
        CK(cudaEventRecord(chunk_event(ctx, c), cs));
        if (c > 0) issue_out(c - 1);
      }
      issue_out(C - 1);
      if (!queued) {
        CK(cudaEventRecord(chunk_event(ctx, 33), ks));
        CK(cudaStreamWaitEvent(cs, chunk_event(ctx, 33), 0));
      }
    } else {
      for (int c = 0; c < C; ++c) gemv_chunk(c);
      c2r_series(0, n_out);
    }
  }
  g_casts.fetch_add(count_casts(p, payload_prec >= 0), std::memory_order_relaxed);
}

// Can the block kernel run this (op, cfg)? (fp16 'h' SBGEMV and NoTrans with
// nd > 256 rows run as K single-RHS pipelines instead.)
bool block_supported(const fmv_op* op, int kind, const Cfg& p) {
  if (p[2] == PH || p[5]) return false;
  return kind != FMV_FORWARD || op->nd <= (size_t)kBlockConsumers;
}

// run_pipeline over K right-hand sides: in = K SOTI vectors back to back
// (K*n_in*nt doubles), out likewise; device pointers, enqueued on ctx->stream.
void pipeline_block(fmv_ctx* ctx, const fmv_op* cop, int kind, const Cfg& p, long K, const double* in,
                    double* out) {
  fmv_op* op = const_cast<fmv_op*>(cop);
  const bool fwd = kind == FMV_FORWARD;
  const long nt = (long)op->nt, nb = (long)op->nb();
  const long n_in = fwd ? (long)op->nm : (long)op->nd;
  const long n_out = fwd ? (long)op->nd : (long)op->nm;
  if (K == 1 || !block_supported(op, kind, p)) {
    for (long r = 0; r < K; ++r) pipeline(ctx, op, kind, p, in + r * n_in * nt, -1, out + r * n_out * nt);
    return;
  }
  long lda = 0;
  const void* bins = op_bins(ctx, op, p[2], &lda);
  const size_t e2 = esize(p[2]), e3 = esize(p[3]);
  const long sx = (n_in + 3) / 4 * 4;  // per-RHS spectrum stride in a bin (16-byte aligned)
  ctx->x.ensure((size_t)nb * K * sx * e2 + 256);
  ctx->y.ensure((size_t)nb * K * n_out * e3 + 256);
  // phases 1-2: the K*n_in series in one launch when the RHS slices are contiguous
  if (sx == n_in) {
    r2c_dispatch<double>(ctx, p[0], p[1], p[2], in, nt, 1, K * n_in, (int)nt, (int)nt, ctx->x.p, K * sx, 1);
  } else {
    for (long r = 0; r < K; ++r)
      r2c_dispatch<double>(ctx, p[0], p[1], p[2], in + r * n_in * nt, nt, 1, n_in, (int)nt, (int)nt,
                           static_cast<unsigned char*>(ctx->x.p) + r * sx * e2, K * sx, 1);
  }
  // phase 3: block SBGEMV, <= kBlockMax RHS per launch
  const long m = (long)op->nd, n = (long)op->nm;
  const int kmax = block_max(fwd);
  for (long r0 = 0; r0 < K; r0 += kmax) {
    const int kc = (int)std::min<long>(kmax, K - r0);
    GemvArgs g;
    g.A = bins;
    g.m = m;
    g.n = n;
    g.batch = nb;
    g.lda = lda;
    g.sa = n * lda;
    g.x = static_cast<unsigned char*>(ctx->x.p) + r0 * sx * e2;
    g.sx = K * sx;
    g.y = static_cast<unsigned char*>(ctx->y.p) + r0 * n_out * e3;
    g.sy = K * n_out;
    g.K = kc;
    g.sxr = sx;
    g.syr = n_out;
    const bool ok = block_gemv_run(ctx, p[2], p[3], fwd ? FMV_GEMV_N : FMV_GEMV_C, g);
    if (!ok) fail(FMV_EUNSUPPORTED, "block sbgemv: shape outside the staged kernel's limits");
  }
  // phases 4-5 over the K*n_out series
  c2r_dispatch(ctx, p[3], p[4], ctx->y.p, K * n_out, 1, K * n_out, (int)nt, (int)nt, out, nt);
  g_casts.fetch_add((uint64_t)K * count_casts(p, false), std::memory_order_relaxed);
}

// --------------------------------------------------------- cast kernels --
template <class O>
__global__ void k_cast_bins(const double2* __restrict__ in, O* __restrict__ out, long ncols, long nd, long lda_out) {
  const long total = ncols * lda_out;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long c = e / lda_out, i = e - c * lda_out;
    out[e] = i < nd ? cfrom_d<O>(in[c * nd + i]) : cfrom_d<O>(make_double2(0.0, 0.0));
  }
}
template <class O>
__global__ void k_unpad_bins(const O* __restrict__ in, long lda_in, O* __restrict__ out, long ncols, long nd) {
  const long total = ncols * nd;
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (long)gridDim.x * blockDim.x) {
    const long c = e / nd, i = e - c * nd;
    out[e] = in[c * lda_in + i];
  }
}
__global__ void k_d2f(const double* __restrict__ in, float* __restrict__ out, long n) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
    out[e] = __double2float_rn(in[e]);
}
__global__ void k_f2d(const float* __restrict__ in, double* __restrict__ out, long n) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
    out[e] = (double)in[e];
}
__global__ void k_d2h(const double* __restrict__ in, __half* __restrict__ out, long n) {
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long)gridDim.x * blockDim.x)
    out[e] = __double2half(in[e]);
}


void materialize(fmv_ctx* ctx, fmv_op* op, int prec) {
  std::lock_guard<std::mutex> lk(op->mu);
  std::atomic<void*>& slot = prec == PS ? op->bins_s : op->bins_h;
  if (slot.load(std::memory_order_acquire)) return;
  const long ncols = (long)(op->nb() * op->nm);
  const long nd = (long)op->nd;
  // pad the leading dimension so every column starts 16-byte aligned (TMA)
  const long lda = prec == PS ? (nd + 1) / 2 * 2 : (nd + 3) / 4 * 4;
  const size_t bytes = (size_t)ncols * lda * (prec == PS ? 8 : 4) + 256;
  void* p = nullptr;
  CK(cudaMalloc(&p, bytes));
  try {
    if (prec == PS) {
      launch(ctx, 4, [&] {
        k_cast_bins<float2><<<grid_for(ncols * lda, 256, ctx->device), 256, 0, ctx->stream>>>(
            static_cast<const double2*>(op->bins_d), static_cast<float2*>(p), ncols, nd, lda);
      });
    } else {
      launch(ctx, 4, [&] {
        k_cast_bins<__half2><<<grid_for(ncols * lda, 256, ctx->device), 256, 0, ctx->stream>>>(
            static_cast<const double2*>(op->bins_d), static_cast<__half2*>(p), ncols, nd, lda);
      });
    }
    // the copy is complete before any other context can see it
    CK(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaFree(p);
    throw;
  }
  (prec == PS ? op->lda_s : op->lda_h) = (size_t)lda;
  slot.store(p, std::memory_order_release);
  g_casts.fetch_add(1, std::memory_order_relaxed);  // ensure_single's cast_buffer (operator.hpp:72)
}

const void* op_bins(fmv_ctx* ctx, fmv_op* op, int prec, long* lda) {
  if (prec == PD) {
    *lda = (long)op->nd;
    return op->bins_d;
  }
  std::atomic<void*>& slot = prec == PS ? op->bins_s : op->bins_h;
  void* p = slot.load(std::memory_order_acquire);
  if (!p) {
    materialize(ctx, op, prec);
    p = slot.load(std::memory_order_acquire);
  }
  *lda = (long)(prec == PS ? op->lda_s : op->lda_h);
  return p;
}

// Every entry point that pairs a context with an operator: the operator's
// memory lives on one device and is only valid there.
void check_same_device(const fmv_ctx* ctx, const fmv_op* op) {
  if (op->device != ctx->device)
    fail(FMV_EINVAL, "operator lives on device " + std::to_string(op->device) + " but the context is on device " +
                         std::to_string(ctx->device));
}

}  // namespace
// ======================================================================
// C ABI
// ======================================================================
namespace {
// ---- collectives of the partitioned matvecs (partition.hpp:157-217) ----

// Round `in` (n doubles, valid on the group root) to cfg[0] precision once and
// broadcast it over `comm`: the payload semantics of partition.hpp:196-206.
// Returns the payload pointer and its precision. Charged to phase [0]
// (partition.hpp:204-206).
std::pair<const void*, int> bcast_payload(fmv_ctx* ctx, void* comm, bool root, const double* in, long n, int p0) {
  NvtxRange nr("fftmv:broadcast");
  cudaStream_t s = ctx->stream;
  if (p0 == PD) {
    if (!comm) return {in, PD};
    ctx->payload.ensure(n * sizeof(double));
    phase_span(ctx, s, 0, [&] {
      if (root) CK(cudaMemcpyAsync(ctx->payload.p, in, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      nck(nccl().broadcast(ctx->payload.p, ctx->payload.p, n, kNcclDouble, 0, comm, s), "ncclBroadcast");
    });
    return {ctx->payload.p, PD};
  }
  ctx->payload.ensure(n * sizeof(float));
  if (root) {
    if (p0 == PS)
      launch(ctx, 4, [&] { k_d2f<<<grid_for(n, 256, ctx->device), 256, 0, s>>>(in, static_cast<float*>(ctx->payload.p), n); }, 0);
    else
      launch(ctx, 4, [&] { k_d2h<<<grid_for(n, 256, ctx->device), 256, 0, s>>>(in, static_cast<__half*>(ctx->payload.p), n); }, 0);
    g_casts.fetch_add(1, std::memory_order_relaxed);  // partition.hpp:203
  }
  if (comm)
    phase_span(ctx, s, 0, [&] {
      nck(nccl().broadcast(ctx->payload.p, ctx->payload.p, n, p0 == PS ? kNcclFloat : kNcclHalf, 0, comm, s),
          "ncclBroadcast");
    });
  return {ctx->payload.p, p0};
}

// Fixed left-balanced pairwise tree over the p gathered partials, in T
// (partition.hpp:84-107 / tree_reduce): round w pairs (k, k+w) for k a
// multiple of 2w -- p=4 gives ((b0+b1)+(b2+b3)), p=3 ((b0+b1)+b2) -- and the
// root is widened to double. One thread per element; G is p x n, rank-major.
template <class T>
__global__ void k_tree_reduce(T* __restrict__ G, long n, int p, double* __restrict__ out) {
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    for (int w = 1; w < p; w *= 2)
      for (int k = 0; k + w < p; k += 2 * w) G[(long)k * n + i] = G[(long)k * n + i] + G[(long)(k + w) * n + i];
    out[i] = (double)G[i];
  }
}

// Sum the n-double partial `buf` over `comm` (gsize ranks) in cfg[4]
// precision (partition.hpp:175-177): the partials are all-gathered in rank
// order and reduced on the device with the reference's fixed tree, so every
// rank gets the bits of the in-process tree_reduce (NCCL's own all-reduce
// order depends on the algorithm it picks). The message is nd*nt values
// (0.8 MB at C2), so gathering p of them costs little. Charged to phase [4]
// (partition.hpp:178-180). gsize == 1: nothing to do.
void reduce_partials(fmv_ctx* ctx, void* comm, int gsize, int grank, double* buf, long n, int p4) {
  NvtxRange nr("fftmv:reduce");
  if (!comm || gsize < 2) {
    // one worker: tree_reduce<float> still casts the lone partial to float and
    // back (2 casts); its value is already float-representable (the unpad
    // rounded it to cfg[4]), so only the counter moves
    if (p4 != PD) g_casts.fetch_add(2, std::memory_order_relaxed);
    return;
  }
  cudaStream_t s = ctx->stream;
  if (p4 == PD) {
    ctx->red.ensure((size_t)gsize * n * sizeof(double));
    double* G = static_cast<double*>(ctx->red.p);
    phase_span(ctx, s, 4, [&] { nck(nccl().all_gather(buf, G, n, kNcclDouble, comm, s), "ncclAllGather"); });
    launch(ctx, 4, [&] { k_tree_reduce<double><<<grid_for(n, 256, ctx->device), 256, 0, s>>>(G, n, gsize, buf); }, 4);
    return;
  }
  // cfg[4] single: every partial is cast to float (one cast per rank), the
  // tree runs in float and the root is cast back to double (counted once,
  // on group rank 0), as tree_reduce_impl<float> counts them in one process.
  ctx->red.ensure((size_t)(gsize + 1) * n * sizeof(float));
  float* G = static_cast<float*>(ctx->red.p);
  float* mine = G + (size_t)gsize * n;
  launch(ctx, 4, [&] { k_d2f<<<grid_for(n, 256, ctx->device), 256, 0, s>>>(buf, mine, n); }, 4);
  phase_span(ctx, s, 4, [&] { nck(nccl().all_gather(mine, G, n, kNcclFloat, comm, s), "ncclAllGather"); });
  launch(ctx, 4, [&] { k_tree_reduce<float><<<grid_for(n, 256, ctx->device), 256, 0, s>>>(G, n, gsize, buf); }, 4);
  g_casts.fetch_add(grank == 0 ? 2 : 1, std::memory_order_relaxed);
}

double env_seconds(const char* name, double dflt) {
  const char* v = getenv(name);
  return v && *v ? atof(v) : dflt;
}

// Wait for the matvec stream while watching the communicators: an
// asynchronous NCCL error (a peer died, a network failure) or no progress
// within FMV_NCCL_TIMEOUT_S seconds (default 600) aborts the communicators
// -- which also unblocks kernels stuck waiting for a dead peer -- and fails
// the call with FMV_ENCCL instead of hanging forever. The context then has
// no communicator; fmv_comm_init must be called again.
// Make the matvec stream wait for everything enqueued on the side streams
// (queued host-I/O output copies), without a host wait.
void join_side_streams(fmv_ctx* ctx) {
  int i = 28;
  for (cudaStream_t side : {ctx->copy_stream, ctx->out_stream}) {
    if (side) {
      CK(cudaEventRecord(chunk_event(ctx, i), side));
      CK(cudaStreamWaitEvent(ctx->stream, chunk_event(ctx, i), 0));
    }
    ++i;
  }
}

void comm_sync(fmv_ctx* ctx) {
  void* comms[3] = {ctx->comm, ctx->row_comm, ctx->col_comm};
  const bool any = comms[0] || comms[1] || comms[2];
  if (!any) {
    CK(cudaStreamSynchronize(ctx->stream));
    return;
  }
  const double limit = env_seconds("FMV_NCCL_TIMEOUT_S", 600.0);
  const auto t0 = std::chrono::steady_clock::now();
  auto abort_all = [&](const std::string& why) {
    for (void** c : {&ctx->row_comm, &ctx->col_comm, &ctx->comm}) {
      if (*c) {
        if (nccl().comm_abort) nccl().comm_abort(*c);
        else if (nccl().comm_destroy) nccl().comm_destroy(*c);
      }
      *c = nullptr;
    }
    ctx->nranks = 1;
    ctx->rank = 0;
    (void)cudaStreamSynchronize(ctx->stream);  // drains once the aborted kernels return
    (void)cudaGetLastError();
    fail(FMV_ENCCL, why);
  };
  for (long it = 0;; ++it) {
    const cudaError_t q = cudaStreamQuery(ctx->stream);
    if (q == cudaSuccess) return;
    if (q != cudaErrorNotReady) CK(q);
    if (nccl().get_async_error) {
      for (void* c : comms) {
        if (!c) continue;
        int e = 0;
        const int rc = nccl().get_async_error(c, &e);
        if (rc == 0 && e != 0 && e != 7 /* ncclInProgress */)
          abort_all(std::string("NCCL asynchronous error: ") + (nccl().err ? nccl().err(e) : "nccl error"));
      }
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > limit)
      abort_all("NCCL collective did not complete within " + std::to_string(limit) +
                " s (FMV_NCCL_TIMEOUT_S); communicator aborted");
    if (it < 2000) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}
}  // namespace

namespace {
// The blocking matvec behind fmv_matvec / fmv_matvec_payload. Host I/O
// always takes the overlapped path: the input copy and the output copy run
// chunk by chunk on a copy stream beside the SBGEMV. With
// `times`, each kernel / copy is bracketed by CUDA events and the
// PhaseTimings are the per-phase busy times (phases overlap on the host-I/O
// path, so their sum may exceed total_s, the wall time of the call).
void matvec_blocking(fmv_ctx* ctx, const fmv_op* op, int kind, const Cfg& p, int payload_prec,
                     const void* in, double* out, bool io_on_device, fmv_phase_times* times) {
  const bool fwd = kind == FMV_FORWARD;
  const size_t in_elem = payload_prec < 0 || payload_prec == PD ? 8 : payload_prec == PS ? 4 : 2;
  const size_t n_in = (fwd ? op->nm : op->nd) * op->nt, n_out = (fwd ? op->nd : op->nm) * op->nt;
  cudaStream_t s = ctx->stream;
  PhaseTimingScope pts(ctx, times != nullptr);
  if (times) CK(cudaEventRecord(ctx->te[0], s));
  if (io_on_device) {
    pipeline(ctx, op, kind, p, in, payload_prec, out);
  } else {
    ctx->io_in.ensure(n_in * in_elem);
    ctx->io_out.ensure(n_out * sizeof(double));
    HostIO hio;
    hio.h_in = in;
    hio.h_out = out;
    hio.in_elem = in_elem;
    if (is_pageable(in)) {
      ctx->pin_in.ensure(n_in * in_elem);
      hio.pin_in = static_cast<unsigned char*>(ctx->pin_in.p);
    }
    if (is_pageable(out)) {
      ctx->pin_out.ensure(n_out * sizeof(double));
      hio.pin_out = static_cast<double*>(ctx->pin_out.p);
    }
    pipeline(ctx, op, kind, p, ctx->io_in.p, payload_prec, static_cast<double*>(ctx->io_out.p), &hio);
    if (times) CK(cudaEventRecord(ctx->te[1], s));
    hio.drain();
    CK(cudaStreamSynchronize(s));
    if (times) collect_phase_times(ctx, ctx->te[0], ctx->te[1], times);
    return;
  }
  if (times) CK(cudaEventRecord(ctx->te[1], s));
  CK(cudaStreamSynchronize(s));
  if (times) collect_phase_times(ctx, ctx->te[0], ctx->te[1], times);
}
// partition.hpp:157-217 on this rank's shard, enqueued on ctx->stream:
// F: the shard pipeline on the local m slice, then the cfg[4] fixed-tree sum
// of the partial d over the communicator; F*: rank 0's d cast to cfg[0] and
// broadcast, then the shard pipeline from the payload.
void partitioned_enqueue(fmv_ctx* ctx, const fmv_op* op, int kind, const Cfg& p, const double* din, double* dout,
                         HostIO* hp) {
  const size_t nt = op->nt;
  if (kind == FMV_FORWARD) {
    pipeline(ctx, op, kind, p, din, -1, dout, hp);
    reduce_partials(ctx, ctx->comm, ctx->nranks, ctx->rank, dout, (long)(op->nd * nt), p[4]);
  } else {
    const auto pay = bcast_payload(ctx, ctx->comm, ctx->rank == 0, din, (long)(op->nd * nt), p[0]);
    pipeline(ctx, op, kind, p, pay.first, p[0] == PD && !ctx->comm ? -1 : pay.second, dout, hp);
  }
}
}  // namespace

extern "C" {

const char* fmv_last_error(void) { return g_err.c_str(); }
const char* fmv_version(void) { return "fftmv-b200 0.1 (sm_100a)"; }

int fmv_ctx_create(int device, void* stream, fmv_ctx** out) {
  return guarded([&] {
    if (!out) fail(FMV_EINVAL, "fmv_ctx_create: out is null");
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) fail(FMV_EINVAL, "fmv_ctx_create: bad device " + std::to_string(device));
    DeviceGuard dg(device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(FMV_EUNSUPPORTED, std::string("libfftmv_cuda is built for sm_100a (B200); device is ") + prop.name);
    auto* c = new fmv_ctx;
    c->device = device;
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    for (auto& e : c->te) CK(cudaEventCreate(&e));
    *out = c;
  });
}

int fmv_ctx_destroy(fmv_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    DeviceGuard dg(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->copy_stream) cudaStreamSynchronize(ctx->copy_stream);
    if (ctx->out_stream) cudaStreamSynchronize(ctx->out_stream);
    for (auto* b : {&ctx->x, &ctx->y, &ctx->yacc, &ctx->io_in, &ctx->io_out, &ctx->partials, &ctx->counters,
                    &ctx->payload, &ctx->red, &ctx->fft_scratch, &ctx->q_x[0], &ctx->q_x[1], &ctx->q_in[0],
                    &ctx->q_in[1], &ctx->q_out_buf[0], &ctx->q_out_buf[1], &ctx->q_scr[0], &ctx->q_scr[1]})
      b->release();
    ctx->pin_in.release();
    ctx->pin_out.release();
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    if (ctx->out_stream) cudaStreamDestroy(ctx->out_stream);
    for (auto e : {ctx->q_done[0], ctx->q_done[1], ctx->q_out[0], ctx->q_out[1]})
      if (e) cudaEventDestroy(e);
    for (auto e : ctx->cev)
      if (e) cudaEventDestroy(e);
    for (auto& r : ctx->prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : ctx->ev_pool) cudaEventDestroy(e);
    for (auto e : ctx->te) cudaEventDestroy(e);
    for (void* c : {ctx->row_comm, ctx->col_comm, ctx->comm})
      if (c && nccl().comm_destroy) nccl().comm_destroy(c);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

void* fmv_ctx_stream(fmv_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
uint64_t fmv_ctx_launches(fmv_ctx* ctx) { return ctx ? ctx->launches : 0; }

int fmv_ctx_set_profiling(fmv_ctx* ctx, int enable) {
  return guarded([&] {
    if (!ctx) fail(FMV_EINVAL, "null ctx");
    ctx->profiling = enable != 0;
  });
}

int fmv_ctx_profile_read(fmv_ctx* ctx, double* ms5, uint64_t* n5, int reset) {
  return guarded([&] {
    if (!ctx) fail(FMV_EINVAL, "null ctx");
    DeviceGuard dg(ctx->device);
    CK(cudaStreamSynchronize(ctx->stream));
    for (auto& r : ctx->prof) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, r.a, r.b));
      ctx->prof_ms[r.cls] += ms;
      ctx->prof_n[r.cls] += 1;
      ctx->ev_pool.push_back(r.a);
      ctx->ev_pool.push_back(r.b);
    }
    ctx->prof.clear();
    for (int i = 0; i < 5; ++i) {
      if (ms5) ms5[i] = ctx->prof_ms[i];
      if (n5) n5[i] = ctx->prof_n[i];
      if (reset) {
        ctx->prof_ms[i] = 0;
        ctx->prof_n[i] = 0;
      }
    }
  });
}

int fmv_synchronize(fmv_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(FMV_EINVAL, "null ctx");
    DeviceGuard dg(ctx->device);
    join_side_streams(ctx);
    comm_sync(ctx);  // a plain stream sync without communicators
  });
}

int fmv_join(fmv_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(FMV_EINVAL, "null ctx");
    DeviceGuard dg(ctx->device);
    join_side_streams(ctx);
  });
}

int fmv_op_create(fmv_ctx* ctx, size_t nm, size_t nd, size_t nt, const double* col, int col_on_device, fmv_op** out) {
  return guarded([&] {
    NvtxRange nr("fftmv:setup_operator");
    if (!ctx || !out) fail(FMV_EINVAL, "fmv_op_create: null argument");
    if (nm < 1 || nd < 1 || nt < 1) fail(FMV_EINVAL, "ProblemDims: all extents must be >= 1");
    if (!col) fail(FMV_EINVAL, "fmv_op_create: null block column");
    DeviceGuard dg(ctx->device);
    std::unique_ptr<fmv_op> op(new fmv_op);
    op->device = ctx->device;
    op->nm = nm;
    op->nd = nd;
    op->nt = nt;
    const size_t S = nd * nm, nb = nt + 1;
    // device allocations are released on every error path (an out-of-memory
    // operator returns FMV_ENOMEM and leaves the context usable)
    struct Guard {
      void* bins = nullptr;
      void* tmp = nullptr;
      ~Guard() {
        if (tmp) cudaFree(tmp);
        if (bins) cudaFree(bins);
      }
    } g;
    CK(cudaMalloc(&g.bins, nb * S * sizeof(double2) + 256));
    op->bins_d = g.bins;
    const double* dcol = col;
    if (!col_on_device) {
      CK(cudaMalloc(&g.tmp, nt * S * sizeof(double)));
      CK(cudaMemcpyAsync(g.tmp, col, nt * S * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      dcol = static_cast<const double*>(g.tmp);
    }
    // operator.hpp:99-125: every (i,j) series, time-outer in the column,
    // padded to 2nt and r2c'd in fp64, written bin-major.
    r2c_dispatch<double>(ctx, PD, PD, PD, dcol, 1, (long)S, (long)S, (int)nt, (int)nt, op->bins_d, (long)S, 1);
    CK(cudaStreamSynchronize(ctx->stream));
    g.bins = nullptr;  // owned by the operator from here on
    *out = op.release();
  });
}

int fmv_op_destroy(fmv_op* op) {
  return guarded([&] {
    if (!op) return;
    DeviceGuard dg(op->device);
    if (op->bins_d) cudaFree(op->bins_d);
    if (void* p = op->bins_s.load()) cudaFree(p);
    if (void* p = op->bins_h.load()) cudaFree(p);
    delete op;
  });
}

int fmv_op_dims(const fmv_op* op, size_t* nm, size_t* nd, size_t* nt) {
  return guarded([&] {
    if (!op) fail(FMV_EINVAL, "null op");
    if (nm) *nm = op->nm;
    if (nd) *nd = op->nd;
    if (nt) *nt = op->nt;
  });
}

int fmv_op_materialize(fmv_ctx* ctx, fmv_op* op, char prec) {
  return guarded([&] {
    if (!ctx || !op) fail(FMV_EINVAL, "null argument");
    check_same_device(ctx, op);
    if (prec != 's' && prec != 'h') fail(FMV_EINVAL, "fmv_op_materialize: prec must be 's' or 'h'");
    DeviceGuard dg(ctx->device);
    materialize(ctx, op, prec_of(prec));
  });
}

int fmv_op_has(const fmv_op* op, char prec) {
  if (!op) return 0;
  if (prec == 'd') return op->bins_d != nullptr;
  if (prec == 's') return op->bins_s.load(std::memory_order_acquire) != nullptr;
  if (prec == 'h') return op->bins_h.load(std::memory_order_acquire) != nullptr;
  return 0;
}

int fmv_op_download_bins(fmv_ctx* ctx, const fmv_op* cop, char prec, void* host_out) {
  return guarded([&] {
    if (!ctx || !cop || !host_out) fail(FMV_EINVAL, "null argument");
    fmv_op* op = const_cast<fmv_op*>(cop);
    check_same_device(ctx, op);
    DeviceGuard dg(ctx->device);
    const size_t ncols = op->nb() * op->nm;
    if (prec == 'd') {
      CK(cudaMemcpy(host_out, op->bins_d, ncols * op->nd * sizeof(double2), cudaMemcpyDeviceToHost));
    } else if (prec == 's') {
      long lda = 0;
      const void* bs = op_bins(ctx, op, PS, &lda);
      CK(cudaMemcpy2D(host_out, op->nd * sizeof(float2), bs, (size_t)lda * sizeof(float2),
                      op->nd * sizeof(float2), ncols, cudaMemcpyDeviceToHost));
    } else {
      fail(FMV_EINVAL, "fmv_op_download_bins: prec must be 'd' or 's'");
    }
  });
}

size_t fmv_op_device_bytes(const fmv_op* op) {
  if (!op) return 0;
  const size_t ncols = op->nb() * op->nm;
  size_t b = ncols * op->nd * sizeof(double2);
  if (op->bins_s.load()) b += ncols * op->lda_s * sizeof(float2);
  if (op->bins_h.load()) b += ncols * op->lda_h * sizeof(__half2);
  return b;
}

int fmv_matvec_block_async(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, size_t nrhs, const double* d_in,
                           double* d_out) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_block_async", kind, cfg));
    if (!ctx || !op || !d_in || !d_out) fail(FMV_EINVAL, "fmv_matvec_block_async: null argument");
    check_same_device(ctx, op);
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    if (nrhs == 0) return;
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    pipeline_block(ctx, op, kind, p, (long)nrhs, d_in, d_out);
  });
}
int fmv_matvec_block(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, size_t nrhs, const double* in,
                     double* out, int io_on_device) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_block", kind, cfg));
    if (!ctx || !op || !in || !out) fail(FMV_EINVAL, "fmv_matvec_block: null argument");
    check_same_device(ctx, op);
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    if (nrhs == 0) return;
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    const bool fwd = kind == FMV_FORWARD;
    const size_t n_in = nrhs * (fwd ? op->nm : op->nd) * op->nt, n_out = nrhs * (fwd ? op->nd : op->nm) * op->nt;
    const double* din = in;
    double* dout = out;
    cudaStream_t s = ctx->stream;
    if (!io_on_device) {
      ctx->io_in.ensure(n_in * sizeof(double));
      ctx->io_out.ensure(n_out * sizeof(double));
      din = static_cast<const double*>(ctx->io_in.p);
      dout = static_cast<double*>(ctx->io_out.p);
      CK(cudaMemcpyAsync(ctx->io_in.p, in, n_in * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    pipeline_block(ctx, op, kind, p, (long)nrhs, din, dout);
    if (!io_on_device) CK(cudaMemcpyAsync(out, dout, n_out * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}
int fmv_matvec_async(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* d_in, double* d_out) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_async", kind, cfg));
    if (!ctx || !op || !d_in || !d_out) fail(FMV_EINVAL, "fmv_matvec_async: null argument");
    check_same_device(ctx, op);
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    pipeline(ctx, op, kind, p, d_in, -1, d_out);
  });
}

int fmv_matvec(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* in, double* out,
               int io_on_device, fmv_phase_times* times) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec", kind, cfg));
    if (!ctx || !op || !in || !out) fail(FMV_EINVAL, "fmv_matvec: null argument");
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    check_same_device(ctx, op);
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    matvec_blocking(ctx, op, kind, p, -1, in, out, io_on_device != 0, times);
  });
}

int fmv_matvec_host_async(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* h_in,
                          double* h_out) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_host_async", kind, cfg));
    if (!ctx || !op || !h_in || !h_out) fail(FMV_EINVAL, "fmv_matvec_host_async: null argument");
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    check_same_device(ctx, op);
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    if (is_pageable(h_in) || is_pageable(h_out))
      fail(FMV_EINVAL, "fmv_matvec_host_async: host buffers must be pinned (cudaHostAlloc / cudaHostRegister)");
    const bool fwd = kind == FMV_FORWARD;
    const size_t n_in = (fwd ? op->nm : op->nd) * op->nt, n_out = (fwd ? op->nd : op->nm) * op->nt;
    const int s = ctx->q_slot;
    for (cudaEvent_t* e : {&ctx->q_done[s], &ctx->q_out[s]})
      if (!*e) CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    // slot s's output buffer was last read by the copy-out of the call two back
    CK(cudaStreamWaitEvent(ctx->stream, ctx->q_out[s], 0));
    // the pipeline works on ctx->x / io_in / io_out: lend it this slot's buffers
    struct Lend {
      fmv_ctx* c;
      int s;
      Lend(fmv_ctx* c_, int s_) : c(c_), s(s_) { swap(); }
      ~Lend() { swap(); }
      void swap() {
        std::swap(c->x, c->q_x[s]);
        std::swap(c->io_in, c->q_in[s]);
        std::swap(c->io_out, c->q_out_buf[s]);
        std::swap(c->fft_scratch, c->q_scr[s]);  // runtime-plan FFTs of the two slots may overlap
      }
    } lend(ctx, s);
    ctx->io_in.ensure(n_in * sizeof(double));
    ctx->io_out.ensure(n_out * sizeof(double));
    HostIO hio;
    hio.h_in = h_in;
    hio.h_out = h_out;
    hio.queued = true;
    hio.guard = ctx->q_done[s];
    pipeline(ctx, op, kind, p, ctx->io_in.p, -1, static_cast<double*>(ctx->io_out.p), &hio);
    CK(cudaEventRecord(ctx->q_done[s], ctx->stream));
    CK(cudaEventRecord(ctx->q_out[s], out_stream(ctx)));
    ctx->q_slot = s ^ 1;
  });
}

int fmv_matvec_payload(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, char payload_prec, const void* in,
                       double* out, int io_on_device, fmv_phase_times* times) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_payload", kind, cfg));
    if (!ctx || !op || !in || !out) fail(FMV_EINVAL, "fmv_matvec_payload: null argument");
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    check_same_device(ctx, op);
    const auto p = parse_cfg(cfg);
    const int pp = prec_of(payload_prec);
    DeviceGuard dg(ctx->device);
    matvec_blocking(ctx, op, kind, p, pp, in, out, io_on_device != 0, times);
  });
}

uint64_t fmv_casts_performed(void) { return g_casts.load(std::memory_order_relaxed); }
void fmv_reset_cast_counter(void) { g_casts.store(0, std::memory_order_relaxed); }

int fmv_comm_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) fail(FMV_EINVAL, "null out");
    nck(nccl().get_unique_id(out128), "ncclGetUniqueId");
  });
}

int fmv_comm_init(fmv_ctx* ctx, int nranks, int rank, const void* id128) {
  return guarded([&] {
    if (!ctx || nranks < 1 || rank < 0 || rank >= nranks) fail(FMV_EINVAL, "fmv_comm_init: bad arguments");
    DeviceGuard dg(ctx->device);
    ctx->nranks = nranks;
    ctx->rank = rank;
    // A single rank needs no communicator; given an id it still builds one
    // (NCCL supports 1-rank communicators), so the collectives run for real.
    if (!id128) {
      if (nranks == 1) return;
      fail(FMV_EINVAL, "fmv_comm_init: null unique id");
    }
    struct Id {
      char b[128];
    } id;
    std::memcpy(id.b, id128, 128);
    typedef int (*InitFn)(void**, int, Id, int);
    auto fn = reinterpret_cast<InitFn>(nccl().comm_init_rank);
    nck(fn(&ctx->comm, nranks, id, rank), "ncclCommInitRank");
  });
}

int fmv_comm_size(const fmv_ctx* ctx, int* nranks, int* rank) {
  return guarded([&] {
    if (!ctx) fail(FMV_EINVAL, "null ctx");
    if (nranks) *nranks = ctx->comm ? ctx->nranks : 1;
    if (rank) *rank = ctx->comm ? ctx->rank : 0;
  });
}

int fmv_comm_destroy(fmv_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(FMV_EINVAL, "null ctx");
    for (void** c : {&ctx->row_comm, &ctx->col_comm, &ctx->comm}) {
      if (*c && nccl().comm_destroy) nccl().comm_destroy(*c);
      *c = nullptr;
    }
    ctx->nranks = 1;
    ctx->rank = 0;
    ctx->pr = ctx->pc = 1;
    ctx->ri = ctx->cj = 0;
  });
}

int fmv_comm_init_2d(fmv_ctx* ctx, int pr, int pc, int rank, const void* id128) {
  return guarded([&] {
    if (!ctx || pr < 1 || pc < 1 || rank < 0 || rank >= pr * pc) fail(FMV_EINVAL, "fmv_comm_init_2d: bad arguments");
    const int rc = fmv_comm_init(ctx, pr * pc, rank, id128);
    if (rc != FMV_OK) fail(rc, fmv_last_error());
    DeviceGuard dg(ctx->device);
    ctx->pr = pr;
    ctx->pc = pc;
    ctx->ri = rank / pc;
    ctx->cj = rank % pc;
    if (!ctx->comm) return;  // single rank without a communicator
    if (!nccl().comm_split) fail(FMV_ENCCL, "ncclCommSplit is not available in the loaded NCCL");
    nck(nccl().comm_split(ctx->comm, ctx->ri, ctx->cj, &ctx->row_comm, nullptr), "ncclCommSplit(row)");
    nck(nccl().comm_split(ctx->comm, ctx->cj, ctx->ri, &ctx->col_comm, nullptr), "ncclCommSplit(col)");
  });
}

int fmv_matvec_partitioned(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* in, double* out,
                           int io_on_device, fmv_phase_times* times) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_partitioned", kind, cfg));
    if (!ctx || !op || !out) fail(FMV_EINVAL, "fmv_matvec_partitioned: null argument");
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    check_same_device(ctx, op);
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->stream;
    const bool fwd = kind == FMV_FORWARD;
    const size_t nt = op->nt;
    const size_t n_in = (fwd ? op->nm : op->nd) * nt, n_out = (fwd ? op->nd : op->nm) * nt;
    const bool have_in = fwd || ctx->rank == 0;
    if (have_in && !in) fail(FMV_EINVAL, "fmv_matvec_partitioned: null input");
    PhaseTimingScope pts(ctx, times != nullptr);
    if (times) CK(cudaEventRecord(ctx->te[0], s));
    const double* din = in;
    double* dout = out;
    // Host I/O: the shard pipeline overlaps the big copy with its SBGEMV
    // column chunks (F: the m slice in; F*: the m slice out), as fmv_matvec.
    HostIO hio{};
    if (!io_on_device) {
      ctx->io_in.ensure(std::max(n_in, op->nd * nt) * sizeof(double));
      ctx->io_out.ensure(n_out * sizeof(double));
      if (fwd) hio.h_in = in;
      else if (have_in) copy_async(ctx, 0, ctx->io_in.p, in, n_in * sizeof(double), cudaMemcpyHostToDevice, s);
      if (!fwd) hio.h_out = out;
      din = static_cast<const double*>(ctx->io_in.p);
      dout = static_cast<double*>(ctx->io_out.p);
    }
    HostIO* hp = io_on_device ? nullptr : &hio;
    partitioned_enqueue(ctx, op, kind, p, din, dout, hp);
    if (fwd && !io_on_device) copy_async(ctx, 4, out, dout, n_out * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (times) CK(cudaEventRecord(ctx->te[1], s));
    comm_sync(ctx);
    if (times) collect_phase_times(ctx, ctx->te[0], ctx->te[1], times);
  });
}

int fmv_matvec_partitioned_async(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* d_in,
                                 double* d_out) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_partitioned_async", kind, cfg));
    if (!ctx || !op || !d_out) fail(FMV_EINVAL, "fmv_matvec_partitioned_async: null argument");
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    check_same_device(ctx, op);
    if ((kind == FMV_FORWARD || ctx->rank == 0) && !d_in) fail(FMV_EINVAL, "fmv_matvec_partitioned_async: null input");
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    partitioned_enqueue(ctx, op, kind, p, d_in, d_out, nullptr);
  });
}

// 2-D pr x pc grid: grid row ri owns sensor
// rows [dlo, dhi), grid column cj owns parameter columns [mlo, mhi); this
// rank's shard is the (ri, cj) sub-block of every time block.
// FORWARD: in = m_cj (nm_cj*nt), read on grid row 0 only; it is rounded to
//   cfg[0] and broadcast down the column, each rank computes its partial
//   d_ri, and the row sums it in cfg[4] (fixed tree): out = d_ri (nd_ri*nt)
//   on every rank of grid row ri.
// ADJOINT: in = d_ri (nd_ri*nt), read on grid column 0 only; rounded to
//   cfg[0] and broadcast along the row, partial m_cj summed down the column
//   in cfg[4]: out = m_cj (nm_cj*nt) on every rank of grid column cj.
// With pr = 1 this is the 1 x p partition (the forward input is then local).
int fmv_matvec_partitioned_2d(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* in,
                              double* out, int io_on_device) {
  return guarded([&] {
    NvtxRange nr(nvtx_matvec_name("matvec_partitioned_2d", kind, cfg));
    if (!ctx || !op || !out) fail(FMV_EINVAL, "fmv_matvec_partitioned_2d: null argument");
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    check_same_device(ctx, op);
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    cudaStream_t s = ctx->stream;
    const bool fwd = kind == FMV_FORWARD;
    const size_t nt = op->nt;
    const size_t n_in = (fwd ? op->nm : op->nd) * nt, n_out = (fwd ? op->nd : op->nm) * nt;
    const bool root = fwd ? ctx->ri == 0 : ctx->cj == 0;
    void* bcomm = fwd ? ctx->col_comm : ctx->row_comm;
    void* rcomm = fwd ? ctx->row_comm : ctx->col_comm;
    const int rsize = fwd ? ctx->pc : ctx->pr, rrank = fwd ? ctx->cj : ctx->ri;
    if (root && !in) fail(FMV_EINVAL, "fmv_matvec_partitioned_2d: null input on a root rank");
    const double* din = in;
    double* dout = out;
    if (!io_on_device) {
      ctx->io_in.ensure(n_in * sizeof(double));
      ctx->io_out.ensure(n_out * sizeof(double));
      if (root) CK(cudaMemcpyAsync(ctx->io_in.p, in, n_in * sizeof(double), cudaMemcpyHostToDevice, s));
      din = static_cast<const double*>(ctx->io_in.p);
      dout = static_cast<double*>(ctx->io_out.p);
    }
    const auto pay = bcast_payload(ctx, bcomm, root, din, (long)n_in, p[0]);
    pipeline(ctx, op, kind, p, pay.first, p[0] == PD && !bcomm ? -1 : pay.second, dout);
    reduce_partials(ctx, rcomm, rsize, rrank, dout, (long)n_out, p[4]);
    if (!io_on_device) CK(cudaMemcpyAsync(out, dout, n_out * sizeof(double), cudaMemcpyDeviceToHost, s));
    comm_sync(ctx);
  });
}

// ---- CUDA-graph matvec: one device-resident matvec captured once, replayed
// with a single cudaGraphLaunch (iterative solvers applying F / F* many times
// to the same buffers; small problems are launch-bound). The graph owns a
// private workspace context, so later calls on the caller's context cannot
// move buffers the graph's kernels point at.
struct fmv_graph {
  fmv_ctx* wctx = nullptr;  // private workspace + capture stream
  cudaStream_t stream = nullptr;  // the caller's ctx stream (replays run there)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t casts = 0;  // logical casts per matvec (precision.hpp:27-39), ticked per replay
  int device = 0;
};

int fmv_graph_create(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* d_in, double* d_out,
                     fmv_graph** out) {
  fmv_graph* g = nullptr;
  const int rc = guarded([&] {
    if (!ctx || !op || !d_in || !d_out || !out) fail(FMV_EINVAL, "fmv_graph_create: null argument");
    check_same_device(ctx, op);
    if (kind != FMV_FORWARD && kind != FMV_ADJOINT) fail(FMV_EINVAL, "matvec: bad kind");
    const auto p = parse_cfg(cfg);
    DeviceGuard dg(ctx->device);
    g = new fmv_graph;
    g->device = ctx->device;
    g->stream = ctx->stream;
    const int rc2 = fmv_ctx_create(ctx->device, nullptr, &g->wctx);
    if (rc2 != FMV_OK) fail(rc2, fmv_last_error());
    fmv_ctx* w = g->wctx;
    // warm-up: sizes the workspace, builds twiddle tables, zeroes tickets and
    // caches kernel attributes, so the captured sequence is kernels only
    // (a first fp32 / fp16 materialization it triggers stays counted: it happened)
    g->casts = count_casts(p, false);
    pipeline(w, op, kind, p, d_in, -1, d_out);
    CK(cudaStreamSynchronize(w->stream));
    g_casts.fetch_sub(g->casts, std::memory_order_relaxed);  // the warm-up is not a user matvec
    CK(cudaStreamBeginCapture(w->stream, cudaStreamCaptureModeThreadLocal));
    try {
      pipeline(w, op, kind, p, d_in, -1, d_out);
    } catch (...) {
      cudaGraph_t dropped = nullptr;
      cudaStreamEndCapture(w->stream, &dropped);
      if (dropped) cudaGraphDestroy(dropped);
      throw;
    }
    CK(cudaStreamEndCapture(w->stream, &g->graph));
    g_casts.fetch_sub(g->casts, std::memory_order_relaxed);  // capture executes nothing
    CK(cudaGraphInstantiate(&g->exec, g->graph, 0));
    *out = g;
  });
  if (rc != FMV_OK && g) {
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->wctx) fmv_ctx_destroy(g->wctx);
    delete g;
  }
  return rc;
}

int fmv_graph_launch(fmv_graph* g) {
  NvtxRange nr("fftmv:graph_launch");
  return guarded([&] {
    if (!g) fail(FMV_EINVAL, "fmv_graph_launch: null graph");
    DeviceGuard dg(g->device);
    CK(cudaGraphLaunch(g->exec, g->stream));
    g_casts.fetch_add(g->casts, std::memory_order_relaxed);
  });
}

int fmv_graph_destroy(fmv_graph* g) {
  return guarded([&] {
    if (!g) return;
    DeviceGuard dg(g->device);
    cudaStreamSynchronize(g->stream);
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->wctx) fmv_ctx_destroy(g->wctx);
    delete g;
  });
}

}  // extern "C"

