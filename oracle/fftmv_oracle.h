/* fftmv_oracle.h -- plain-C restatement of the reference FFTMatvec path.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load liboracle.so, and only as the checker
 * or the timed CPU baseline -- never as the product path.
 *
 * Each function restates the reference function cited beside it
 * (/root/reference/proj/include/fftmv/<file>:<line>). The restatement is
 * pinned against the reference itself (oracle/_ref, compiled verbatim) and
 * against committed golden vectors in tests/golden/ (tests/test_oracle.py).
 *
 * Conventions: complex buffers are interleaved (re, im) doubles; the
 * operator is bin-major, column-major within a bin (operator.hpp:58);
 * vectors are SOTI (block_vector.hpp:14-19). cfg strings are 5 chars over
 * {d,s,h}: 'h' is this project's fp16 extension.
 * Return codes: 0 ok, -1 invalid argument.
 */
#ifndef FFTMV_ORACLE_H
#define FFTMV_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);

/* random_fill.hpp:17-32, sweep.hpp:32-46 */
uint64_t orc_seed_stream(uint64_t seed, uint64_t stream);
void orc_uniform_fill(size_t count, uint64_t seed, double lo, double hi, double* out);
int orc_non_representable_fill(size_t count, uint64_t seed, double* out);
/* sweep.hpp:49-59 */
int orc_relative_error(size_t n, const double* x, const double* ref, double* out);
/* gemv.hpp:83-89 */
int orc_effective_bandwidth(size_t m, size_t n, size_t batch, size_t elem_bytes, double seconds, double* out);

/* fft.hpp:110-148: batch series of real length L <-> batch x (L/2+1) complex.
 * prec: 0 single, 1 double; inverse includes the 1/L pre-scale. */
int orc_fft_forward(size_t L, size_t batch, int prec, const void* in, void* out);
int orc_fft_inverse(size_t L, size_t batch, int prec, const void* in, void* out);

/* gemv.hpp:135-163: naive strided-batched GEMV (mode 0 N, 1 T, 2 C);
 * dtype 's','d','c','z'. Lengths are element counts. */
int orc_gemv(int mode, char dtype, size_t m, size_t n, size_t batch, size_t lda, size_t stride_a, const void* A,
             size_t stride_x, const void* x, size_t stride_y, void* y);

typedef struct orc_op orc_op;
/* operator.hpp:99-125 */
orc_op* orc_setup_operator(size_t nm, size_t nd, size_t nt, const double* col);
void orc_op_free(orc_op* op);
void orc_op_bins(const orc_op* op, double* out);

/* matvec.hpp:233-318: kind 0 forward (d = F m), 1 adjoint (m = F* d).
 * casts (optional) receives the number of conversion passes
 * (precision.hpp:27-39 counting rule). */
int orc_matvec(const orc_op* op, int kind, const char* cfg, const double* in, double* out, uint64_t* casts);

/* dense_ref.hpp:30-64 */
int orc_dense(int kind, size_t nm, size_t nd, size_t nt, const double* col, const double* in, double* out);

/* partition.hpp:27-40, :84-132, :141-217 */
int orc_grid_split(size_t p, size_t nm, size_t* ranges);
int orc_tree_reduce(size_t p, size_t n, const double* bufs, int prec, double* out);
int orc_matvec_partitioned(size_t nm, size_t nd, size_t nt, const double* col, size_t p, int kind, const char* cfg,
                           const double* in, double* out);

#ifdef __cplusplus
}
#endif
#endif
