/* FFTW3-API shim used ONLY to compile the reference headers verbatim for the
 * CPU oracle (oracle/_ref). Test infrastructure, never linked into the
 * product library.
 *
 * The reference includes <fftw3.h> at /root/reference/proj/include/fftmv/fft.hpp:24
 * and calls exactly these entry points (fft.hpp:51-61 plan, :68-69 destroy,
 * :114/:122/:136/:146 execute). FFTW itself is not installed in this image, so
 * the ten functions are implemented over Intel MKL DFTI as exported by
 * libtorch_cpu.so (see fftw_mkl_shim.cpp). Conventions kept: unnormalized
 * transforms, half-spectrum (CCE) storage, out-of-place, contiguous series at
 * distance idist/odist.
 */
#ifndef FFTMV_ORACLE_FFTW3_SHIM_H
#define FFTMV_ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef float fftwf_complex[2];
typedef struct fftmv_shim_plan* fftw_plan;
typedef struct fftmv_shim_plan* fftwf_plan;

#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_many_dft_r2c(int rank, const int* n, int howmany, double* in, const int* inembed, int istride,
                                 int idist, fftw_complex* out, const int* onembed, int ostride, int odist,
                                 unsigned flags);
fftw_plan fftw_plan_many_dft_c2r(int rank, const int* n, int howmany, fftw_complex* in, const int* inembed,
                                 int istride, int idist, double* out, const int* onembed, int ostride, int odist,
                                 unsigned flags);
fftwf_plan fftwf_plan_many_dft_r2c(int rank, const int* n, int howmany, float* in, const int* inembed, int istride,
                                   int idist, fftwf_complex* out, const int* onembed, int ostride, int odist,
                                   unsigned flags);
fftwf_plan fftwf_plan_many_dft_c2r(int rank, const int* n, int howmany, fftwf_complex* in, const int* inembed,
                                   int istride, int idist, float* out, const int* onembed, int ostride, int odist,
                                   unsigned flags);
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out);
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out);
void fftwf_execute_dft_r2c(const fftwf_plan p, float* in, fftwf_complex* out);
void fftwf_execute_dft_c2r(const fftwf_plan p, fftwf_complex* in, float* out);
void fftw_destroy_plan(fftw_plan p);
void fftwf_destroy_plan(fftwf_plan p);

#ifdef __cplusplus
}
#endif
#endif
