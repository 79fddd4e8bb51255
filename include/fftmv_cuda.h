/* fftmv_cuda.h -- C ABI of libfftmv_cuda.so, the B200 (sm_100a) FFTMatvec.
 *
 * This is the drop-in boundary for the reference's FFTMatvec path
 * (/root/reference/proj/include/fftmv). Plain C types only: opaque handles,
 * pointers, sizes, 5-char precision configs. The C++ header set in
 * include/fftmv/ re-exposes the reference's C++ API (namespace fftmv) on top
 * of these functions; INTEGRATION.md shows the bindings.
 *
 * Conventions (same as the reference):
 *   - operator block column: col[t*nd*nm + i + j*nd]            (operator.hpp:28-29)
 *   - spectral bins: bins[(k*nd*nm + i + j*nd)] complex, interleaved  (operator.hpp:58)
 *   - vectors SOTI: m[c*nt + t], d[r*nt + t], always double at the I/O boundary
 *                                                                (matvec.hpp:291-299)
 *   - cfg: 5 chars, positions = phases {pad/broadcast, fft, sbgemv, ifft,
 *     unpad/reduce} (config.hpp:14-33), chars 'd' or 's', plus the 'h' (fp16)
 *     extension at positions 0, 2 and 4 and the 'm' extension at position 2
 *     (SBGEMV on the fp32 operator and spectrum with fp64 accumulation).
 * Return codes: FMV_OK, or an error code with a message in fmv_last_error()
 * (thread-local). The C++ wrapper maps FMV_EINVAL to std::invalid_argument
 * and everything else to std::runtime_error, like the reference.
 * Threading: an fmv_op is read-only after creation (materialization is
 * internally synchronized) and may be shared by any number of contexts; an
 * fmv_ctx (one CUDA stream + workspace) is used by one host thread at a time.
 */
#ifndef FFTMV_CUDA_H
#define FFTMV_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMV_OK 0
#define FMV_EINVAL 1
#define FMV_ECUDA 2
#define FMV_ENCCL 3
#define FMV_ENOMEM 4
#define FMV_EUNSUPPORTED 5

#define FMV_FORWARD 0 /* d = F m   (matvec.hpp:305-310) */
#define FMV_ADJOINT 1 /* m = F* d  (matvec.hpp:313-318) */

#define FMV_GEMV_N 0 /* GemvMode::NoTrans   (gemv.hpp:33) */
#define FMV_GEMV_T 1 /* GemvMode::Trans */
#define FMV_GEMV_C 2 /* GemvMode::ConjTrans */

typedef struct fmv_ctx fmv_ctx;
typedef struct fmv_op fmv_op;

/* PhaseTimings (matvec.hpp:42-51): seconds per phase + total. On B200 the
 * phases are fused, so: [0] host->device copy of the input (0 when the I/O is
 * device-resident; + payload cast and broadcast for the partitioned
 * adjoint, partition.hpp:204-206), [1] pad+cast+r2c kernels, [2] SBGEMV
 * kernels incl. both fused reorders, [3] c2r+unpad kernels, [4]
 * device->host copy (+ the reduce of the partitioned forward,
 * partition.hpp:178-180). Each phase is the summed CUDA-event time of its
 * kernels / copies. Host-I/O calls overlap the copies and the FFTs with the
 * SBGEMV (column chunks), so the phases may add up to more than total_s,
 * the wall time of the whole call; requesting times does not change the
 * schedule. */
typedef struct {
  double phase_s[5];
  double total_s;
} fmv_phase_times;

const char* fmv_last_error(void);
const char* fmv_version(void);

/* ---- contexts: one device, one stream, a grow-only workspace ---- */
/* stream: a cudaStream_t to run on, or NULL for a new non-blocking stream. */
int fmv_ctx_create(int device, void* stream, fmv_ctx** out);
int fmv_ctx_destroy(fmv_ctx* ctx);
void* fmv_ctx_stream(fmv_ctx* ctx);
/* Kernel-launch bookkeeping for benchmarks: total launches issued by this
 * context, and (when profiling is on) per-kernel-class CUDA-event time. */
uint64_t fmv_ctx_launches(fmv_ctx* ctx);
int fmv_ctx_set_profiling(fmv_ctx* ctx, int enable);
/* kernel classes: 0 r2c, 1 sbgemv-N, 2 sbgemv-C, 3 c2r, 4 other */
int fmv_ctx_profile_read(fmv_ctx* ctx, double* ms_per_class5, uint64_t* launches_per_class5, int reset);
/* Waits for the ctx stream; with communicators, under the NCCL error / timeout
 * watch of the partitioned entry points. */
int fmv_synchronize(fmv_ctx* ctx);

/* ---- operator: setup_operator (operator.hpp:99-125) ---- */
/* col: nt*nd*nm doubles (host, or device if col_on_device). */
int fmv_op_create(fmv_ctx* ctx, size_t nm, size_t nd, size_t nt, const double* col, int col_on_device,
                  fmv_op** out);
int fmv_op_destroy(fmv_op* op);
int fmv_op_dims(const fmv_op* op, size_t* nm, size_t* nd, size_t* nt);
/* materialize_single (operator.hpp:90-93); prec 's' (fp32) or 'h' (fp16 ext.). Idempotent. */
int fmv_op_materialize(fmv_ctx* ctx, fmv_op* op, char prec);
int fmv_op_has(const fmv_op* op, char prec);
/* Copy the bins to host in the reference layout: prec 'd' -> nb*nd*nm complex
 * doubles (bins_double, operator.hpp:59); 's' -> complex floats. */
int fmv_op_download_bins(fmv_ctx* ctx, const fmv_op* op, char prec, void* host_out);
size_t fmv_op_device_bytes(const fmv_op* op);

/* ---- matvecs: run_pipeline (matvec.hpp:233-289) ---- */
/* Blocking, like the reference. in/out: double SOTI vectors; host pointers
 * (pinned or pageable) unless io_on_device. times may be NULL. */
int fmv_matvec(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* in, double* out,
               int io_on_device, fmv_phase_times* times);
/* run_pipeline with a broadcast payload (matvec.hpp:233-289 `payload`,
 * partition.hpp:198-212): `in` holds the input already rounded to cfg[0] in
 * payload_prec ('d' double, 's' float, 'h' IEEE binary16 bits), so phase 1
 * pads it without another rounding and the cast counter does not count a pad
 * cast. Otherwise as fmv_matvec. */
int fmv_matvec_payload(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, char payload_prec, const void* in,
                       double* out, int io_on_device, fmv_phase_times* times);
/* Non-blocking variant: device pointers only, enqueued on the ctx stream. */
int fmv_matvec_async(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* d_in, double* d_out);
/* Queued host-I/O variant of fmv_matvec (an addition; the reference's
 * run_pipeline, matvec.hpp:233-289, is blocking): h_in / h_out must be PINNED
 * host buffers (cudaHostAlloc / cudaHostRegister, else FMV_EINVAL). The call
 * enqueues the input copy, the pipeline and the output copy and returns
 * without waiting; results are in h_out after fmv_synchronize(ctx). Two
 * workspace slots alternate, so consecutive queued calls overlap: call i+1's
 * input copy (and, for FORWARD, its chunked r2c) runs beside call i's SBGEMV,
 * and call i's output copy beside call i+1's. Results equal fmv_matvec's
 * with the same host buffers bit for bit. Do not modify h_in or read h_out
 * before fmv_synchronize. */
int fmv_matvec_host_async(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* h_in,
                          double* h_out);
/* Make the ctx stream wait (on the device, no host wait) for the output
 * copies queued by fmv_matvec_host_async; an event recorded on the ctx stream
 * afterwards marks the completion of every queued call. fmv_synchronize
 * includes it. */
int fmv_join(fmv_ctx* ctx);

/* ---- block (multi-RHS) matvec: SURVEY.md §8 f2 ----
 * nrhs independent inputs back to back (nrhs SOTI vectors of n_in*nt
 * doubles; n_in = nm for FORWARD, nd for ADJOINT), outputs likewise. Each
 * RHS goes through the same 5-phase pipeline and precision config as
 * fmv_matvec; the per-bin SBGEMV handles up to 8 (FORWARD) / 4 (ADJOINT) RHS
 * per operator pass (the operator is read from HBM once per pass instead of
 * once per RHS). Per-RHS results equal fmv_matvec's up to summation order
 * (fp64: ~1e-15 relative). 'h' and 'm' SBGEMV configs and FORWARD with nd > 416 run
 * as nrhs single-RHS pipelines. Blocking; host pointers unless io_on_device. */
int fmv_matvec_block(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, size_t nrhs, const double* in,
                     double* out, int io_on_device);
/* Non-blocking variant: device pointers only, enqueued on the ctx stream. */
int fmv_matvec_block_async(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, size_t nrhs, const double* d_in,
                           double* d_out);

/* ---- CUDA-graph matvec (device-resident I/O) ----
 * Captures one fmv_matvec_async(ctx, op, kind, cfg, d_in, d_out) into a CUDA
 * graph (after one warm-up run that sizes a private workspace); each
 * fmv_graph_launch replays it on ctx's stream with a single cudaGraphLaunch,
 * reading d_in and writing d_out as they are at replay time. For iterative
 * solvers that apply F / F* many times to the same buffers, and small,
 * launch-bound problems. The graph owns its workspace, so it stays valid
 * whatever else runs on ctx; destroy it before freeing d_in / d_out. */
typedef struct fmv_graph fmv_graph;
int fmv_graph_create(fmv_ctx* ctx, const fmv_op* op, int kind, const char* cfg, const double* d_in, double* d_out,
                     fmv_graph** out);
int fmv_graph_launch(fmv_graph* g);
int fmv_graph_destroy(fmv_graph* g);

/* ---- batched real FFTs (fft.hpp:110-148), device pointers ----
 * r2c: batch contiguous series of L reals -> batch x (L/2+1) complex bins,
 *      unnormalized, sign -1. c2r: the true inverse, 1/L folded in by
 *      pre-scaling in the working precision. prec 'd' (double/complex double)
 *      or 's' (float/complex float). L must be even and >= 2. */
int fmv_fft_r2c(fmv_ctx* ctx, size_t L, size_t batch, char prec, const void* d_in, void* d_out);
int fmv_fft_c2r(fmv_ctx* ctx, size_t L, size_t batch, char prec, const void* d_in, void* d_out);

/* ---- casts (precision.hpp:27-39): logical conversion passes performed ---- */
uint64_t fmv_casts_performed(void);
void fmv_reset_cast_counter(void);

/* ---- strided-batched GEMV (gemv.hpp:206-240), device pointers ----
 * dtype 's','d','c','z' (or 'h' = complex fp16 storage, fp32 accumulation,
 * output complex float). Strides/lda in elements. Returns the kernel used in
 * *kernel_used (0 staged/TMA, 1 simple, 2 small-problem (Conj)Trans) when non-NULL. A and x must be
 * readable up to the next 16-byte boundary past their last element. */
int fmv_sbgemv(fmv_ctx* ctx, int mode, char dtype, size_t m, size_t n, size_t batch, size_t lda, size_t stride_a,
               const void* A, size_t stride_x, const void* x, size_t stride_y, void* y, int force_simple,
               int* kernel_used);

/* ---- 1 x p partition over NCCL (partition.hpp:23-217) ---- */
int fmv_comm_unique_id(void* out128);
/* id128: the bytes from rank 0's fmv_comm_unique_id (exchange them out of band).
 * nranks == 1 with id128 == NULL needs no NCCL at all; with an id it builds a
 * real 1-rank communicator, so the collectives execute (useful for testing). */
int fmv_comm_init(fmv_ctx* ctx, int nranks, int rank, const void* id128);
int fmv_comm_destroy(fmv_ctx* ctx);
/* The live communicator's size and this rank (1 and 0 without one). */
int fmv_comm_size(const fmv_ctx* ctx, int* nranks, int* rank);
/* Each rank holds the operator shard of its Grid1xP column range.
 * FORWARD: in = this rank's m slice (shard_nm*nt), out = full d (nd*nt) on
 *   every rank, partial d summed in cfg[4] precision (partition.hpp:157-182)
 *   with the reference's fixed left-balanced tree over the all-gathered
 *   partials (tree_reduce, partition.hpp:84-107): bitwise the in-process
 *   result for every p.
 * Collectives are watched: an asynchronous NCCL error, or no completion
 *   within FMV_NCCL_TIMEOUT_S seconds (default 600), aborts the
 *   communicator and returns FMV_ENCCL (re-init before the next call).
 * FMV_NCCL_LIB (environment) loads another library with the NCCL API in
 *   place of libnccl.so.2.
 * ADJOINT: in = full d (nd*nt, read on rank 0 only), broadcast in cfg[0]
 *   precision; out = this rank's m slice (partition.hpp:187-217). */
int fmv_matvec_partitioned(fmv_ctx* ctx, const fmv_op* shard, int kind, const char* cfg, const double* in,
                           double* out, int io_on_device, fmv_phase_times* times);
/* Non-blocking fmv_matvec_partitioned: device pointers, the shard pipeline and
 * the collectives enqueued on the ctx stream, no host wait -- consecutive
 * partitioned matvecs pipeline like fmv_matvec_async. fmv_synchronize(ctx)
 * waits with the same NCCL error / timeout watch. */
int fmv_matvec_partitioned_async(fmv_ctx* ctx, const fmv_op* shard, int kind, const char* cfg, const double* d_in,
                                 double* d_out);

/* ---- 2-D pr x pc grid ----
 * rank = ri*pc + cj. Splits the world communicator into a row communicator
 * (the pc ranks of grid row ri) and a column communicator (the pr ranks of
 * grid column cj) with ncclCommSplit. */
int fmv_comm_init_2d(fmv_ctx* ctx, int pr, int pc, int rank, const void* id128);
/* Each rank holds the (ri, cj) operator block: sensor rows of grid row ri x
 * parameter columns of grid column cj (GridPxQ, partition.py).
 * FORWARD: in = m_cj (read on grid row 0 only), rounded to cfg[0] and
 *   broadcast down the column; partial d_ri summed along the row in cfg[4];
 *   out = d_ri (nd_ri*nt) on every rank of the row.
 * ADJOINT: in = d_ri (read on grid column 0 only), rounded to cfg[0] and
 *   broadcast along the row; partial m_cj summed down the column in cfg[4];
 *   out = m_cj (nm_cj*nt) on every rank of the column. */
int fmv_matvec_partitioned_2d(fmv_ctx* ctx, const fmv_op* shard, int kind, const char* cfg, const double* in,
                              double* out, int io_on_device);

/* ---- host helpers kept from the reference API ---- */
uint64_t fmv_seed_stream(uint64_t seed, uint64_t stream);                          /* random_fill.hpp:30-32 */
void fmv_uniform_fill(size_t count, uint64_t seed, double lo, double hi, double* out); /* random_fill.hpp:17-27 */
int fmv_non_representable_fill(size_t count, uint64_t seed, double* out);           /* sweep.hpp:32-46 */
int fmv_relative_error(size_t n, const double* x, const double* ref, double* out);  /* sweep.hpp:49-59 */
/* memcpy of host memory by the library's host thread pool (the one that
 * stages pageable matvec I/O): the drop-in's std::vector results are filled
 * with it from a pinned buffer. No reference counterpart. */
int fmv_host_copy(void* dst, const void* src, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif
