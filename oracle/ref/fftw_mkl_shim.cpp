// FFTW3-API shim over Intel MKL DFTI (exported by libtorch_cpu.so).
// TEST INFRASTRUCTURE ONLY: lets the reference headers under
// /root/reference/proj/include compile unmodified into oracle/_ref. The
// product library never links this.
//
// Mirrors the only FFTW usage in the reference (fft.hpp:45-61): rank-1,
// contiguous series (stride 1), distance idist/odist, FFTW_ESTIMATE. FFTW's
// r2c/c2r are unnormalized and use the n/2+1 half spectrum; DFTI with
// CONJUGATE_EVEN_STORAGE=COMPLEX_COMPLEX and default scales (1.0) matches.
#include "fftw3.h"

#include <cstdio>
#include <cstdlib>

extern "C" {
typedef void* DFTI_DESCRIPTOR_HANDLE;
long DftiCreateDescriptor_d_1d(DFTI_DESCRIPTOR_HANDLE*, int domain, long length);
long DftiCreateDescriptor_s_1d(DFTI_DESCRIPTOR_HANDLE*, int domain, long length);
long DftiSetValue(DFTI_DESCRIPTOR_HANDLE, int param, ...);
long DftiCommitDescriptor(DFTI_DESCRIPTOR_HANDLE);
long DftiComputeForward(DFTI_DESCRIPTOR_HANDLE, void*, ...);
long DftiComputeBackward(DFTI_DESCRIPTOR_HANDLE, void*, ...);
long DftiFreeDescriptor(DFTI_DESCRIPTOR_HANDLE*);
}

namespace {
// mkl_dfti.h enumerators (values fixed by the MKL ABI).
constexpr int DFTI_NUMBER_OF_TRANSFORMS = 7;
constexpr int DFTI_CONJUGATE_EVEN_STORAGE = 10;
constexpr int DFTI_PLACEMENT = 11;
constexpr int DFTI_INPUT_DISTANCE = 14;
constexpr int DFTI_OUTPUT_DISTANCE = 15;
constexpr int DFTI_REAL = 33;
constexpr int DFTI_COMPLEX_COMPLEX = 39;
constexpr int DFTI_NOT_INPLACE = 44;

void check(long status, const char* what) {
  if (status != 0) {
    std::fprintf(stderr, "fftw-mkl shim: %s failed with DFTI status %ld\n", what, status);
    std::abort();
  }
}
}  // namespace

struct fftmv_shim_plan {
  DFTI_DESCRIPTOR_HANDLE h = nullptr;
};

static fftmv_shim_plan* make_plan(bool dbl, int rank, const int* n, int howmany, int istride, int idist,
                                  int ostride, int odist) {
  if (rank != 1 || istride != 1 || ostride != 1) return nullptr;
  auto* p = new fftmv_shim_plan;
  check(dbl ? DftiCreateDescriptor_d_1d(&p->h, DFTI_REAL, n[0]) : DftiCreateDescriptor_s_1d(&p->h, DFTI_REAL, n[0]),
        "DftiCreateDescriptor");
  check(DftiSetValue(p->h, DFTI_NUMBER_OF_TRANSFORMS, (long)howmany), "NUMBER_OF_TRANSFORMS");
  check(DftiSetValue(p->h, DFTI_PLACEMENT, DFTI_NOT_INPLACE), "PLACEMENT");
  check(DftiSetValue(p->h, DFTI_CONJUGATE_EVEN_STORAGE, DFTI_COMPLEX_COMPLEX), "CONJUGATE_EVEN_STORAGE");
  check(DftiSetValue(p->h, DFTI_INPUT_DISTANCE, (long)idist), "INPUT_DISTANCE");
  check(DftiSetValue(p->h, DFTI_OUTPUT_DISTANCE, (long)odist), "OUTPUT_DISTANCE");
  check(DftiCommitDescriptor(p->h), "DftiCommitDescriptor");
  return p;
}

extern "C" {
fftw_plan fftw_plan_many_dft_r2c(int rank, const int* n, int howmany, double*, const int*, int istride, int idist,
                                 fftw_complex*, const int*, int ostride, int odist, unsigned) {
  return make_plan(true, rank, n, howmany, istride, idist, ostride, odist);
}
fftw_plan fftw_plan_many_dft_c2r(int rank, const int* n, int howmany, fftw_complex*, const int*, int istride,
                                 int idist, double*, const int*, int ostride, int odist, unsigned) {
  return make_plan(true, rank, n, howmany, istride, idist, ostride, odist);
}
fftwf_plan fftwf_plan_many_dft_r2c(int rank, const int* n, int howmany, float*, const int*, int istride, int idist,
                                   fftwf_complex*, const int*, int ostride, int odist, unsigned) {
  return make_plan(false, rank, n, howmany, istride, idist, ostride, odist);
}
fftwf_plan fftwf_plan_many_dft_c2r(int rank, const int* n, int howmany, fftwf_complex*, const int*, int istride,
                                   int idist, float*, const int*, int ostride, int odist, unsigned) {
  return make_plan(false, rank, n, howmany, istride, idist, ostride, odist);
}
void fftw_execute_dft_r2c(const fftw_plan p, double* in, fftw_complex* out) {
  check(DftiComputeForward(p->h, in, out), "DftiComputeForward");
}
void fftw_execute_dft_c2r(const fftw_plan p, fftw_complex* in, double* out) {
  check(DftiComputeBackward(p->h, in, out), "DftiComputeBackward");
}
void fftwf_execute_dft_r2c(const fftwf_plan p, float* in, fftwf_complex* out) {
  check(DftiComputeForward(p->h, in, out), "DftiComputeForward");
}
void fftwf_execute_dft_c2r(const fftwf_plan p, fftwf_complex* in, float* out) {
  check(DftiComputeBackward(p->h, in, out), "DftiComputeBackward");
}
void fftw_destroy_plan(fftw_plan p) {
  if (p) DftiFreeDescriptor(&p->h);
  delete p;
}
void fftwf_destroy_plan(fftwf_plan p) { fftw_destroy_plan(p); }
}
