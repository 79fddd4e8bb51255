/* fftmv_oracle.c -- plain-C restatement of the reference FFTMatvec algorithm.
 *
 * TEST INFRASTRUCTURE ONLY (see fftmv_oracle.h). This is the checker the
 * CUDA path is compared against; it is never the product. Every function
 * cites the reference file:line it restates (paths relative to
 * /root/reference/proj/include/fftmv/).
 *
 * The FFT is deliberately a different algorithm from the CUDA one (full-length
 * recursive mixed-radix DIT on the complex-embedded series here vs. a
 * half-length Stockham with a real post-pass on the GPU), so agreement is
 * evidence, not a tautology. FFTW (the reference's FFT backend, fft.hpp:24,
 * no version pinned) is restated by its contract: unnormalized forward DFT
 * with sign -1, half spectrum, c2r ignoring Im of DC/Nyquist (fft.hpp:5-8).
 */
#include "fftmv_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return -1;
}
const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ fills */
/* std::mt19937_64 (the engine random_fill.hpp:17 relies on), per the C++
 * standard's parameterisation [rand.predef]. */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}
static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* random_fill.hpp:30-32 */
uint64_t orc_seed_stream(uint64_t seed, uint64_t stream) { return seed ^ (0x9E3779B97F4A7C15ULL * (stream + 1)); }

/* random_fill.hpp:17-27 */
void orc_uniform_fill(size_t count, uint64_t seed, double lo, double hi, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  const double scale = hi - lo;
  for (size_t i = 0; i < count; ++i) {
    const double u01 = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
    out[i] = lo + scale * u01;
  }
}

/* sweep.hpp:32-46 */
int orc_non_representable_fill(size_t count, uint64_t seed, double* out) {
  if (count < 1) return fail("non_representable_fill: count must be >= 1");
  mt64 g;
  mt64_seed(&g, seed);
  for (size_t i = 0; i < count; ++i) {
    const uint64_t u = mt64_next(&g);
    double mag = 0.5 + (double)(u >> 12) * 0x1.0p-53;
    uint64_t bits;
    memcpy(&bits, &mag, 8);
    bits |= (1ULL << 29) - 1;
    memcpy(&mag, &bits, 8);
    out[i] = (u & 1u) ? -mag : mag;
  }
  return 0;
}

/* sweep.hpp:49-59 */
int orc_relative_error(size_t n, const double* x, const double* ref, double* out) {
  double num = 0.0, den = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double d = x[i] - ref[i];
    num += d * d;
    den += ref[i] * ref[i];
  }
  if (den == 0.0) return fail("relative_error: zero-norm reference");
  *out = sqrt(num) / sqrt(den);
  return 0;
}

/* gemv.hpp:83-89 */
int orc_effective_bandwidth(size_t m, size_t n, size_t batch, size_t es, double s, double* out) {
  if (!(s > 0.0)) return fail("effective_bandwidth: seconds must be > 0");
  const double elems = (double)m * (double)n + (double)m + (double)n;
  *out = (double)batch * elems * (double)es / s / 1e9;
  return 0;
}

/* ------------------------------------------------------- precision casts */
/* precision.hpp:44-61: RNE narrowing, exact widening. 'h' (fp16) is this
 * project's extension; double->half rounds once (no double rounding). */
static double rnd(char p, double v) {
  if (p == 's') return (double)(float)v;
  if (p == 'h') return (double)(_Float16)v;
  return v;
}

/* ------------------------------------------------------------------- FFT */
/* Recursive mixed-radix decimation-in-time complex DFT on interleaved data,
 * arithmetic in T. tw[m] = exp(-2*pi*i*m/Ltab), rounded once from long
 * double. sign -1 forward, +1 inverse (conjugated twiddles). */
#define DEFINE_FFT(T, SUF)                                                                                     \
  static void fft_rec_##SUF(const T* in, size_t stride, T* out, size_t n, const T* tw, size_t ltab, int sign) {   \
    if (n == 1) {                                                                                               \
      out[0] = in[0];                                                                                           \
      out[1] = in[1];                                                                                           \
      return;                                                                                                   \
    }                                                                                                           \
    size_t p = 2;                                                                                               \
    while (n % p) ++p;                                                                                          \
    const size_t m = n / p, step = ltab / n;                                                                    \
    for (size_t q = 0; q < p; ++q) fft_rec_##SUF(in + 2 * q * stride, stride * p, out + 2 * q * m, m, tw, ltab, sign); \
    T tloc[2 * 16];                                                                                             \
    T* t = p <= 16 ? tloc : (T*)malloc(2 * p * sizeof(T));                                                      \
    for (size_t k = 0; k < m; ++k) {                                                                            \
      for (size_t q = 0; q < p; ++q) {                                                                          \
        const size_t e = ((q * k) % n) * step;                                                                  \
        const T wr = tw[2 * e], wi = sign < 0 ? tw[2 * e + 1] : -tw[2 * e + 1];                                 \
        const T ar = out[2 * (q * m + k)], ai = out[2 * (q * m + k) + 1];                                       \
        t[2 * q] = ar * wr - ai * wi;                                                                           \
        t[2 * q + 1] = ar * wi + ai * wr;                                                                       \
      }                                                                                                         \
      for (size_t r = 0; r < p; ++r) {                                                                          \
        T sr = 0, si = 0;                                                                                       \
        for (size_t q = 0; q < p; ++q) {                                                                        \
          const size_t e = ((q * r * m) % n) * step;                                                            \
          const T wr = tw[2 * e], wi = sign < 0 ? tw[2 * e + 1] : -tw[2 * e + 1];                               \
          sr += t[2 * q] * wr - t[2 * q + 1] * wi;                                                              \
          si += t[2 * q] * wi + t[2 * q + 1] * wr;                                                              \
        }                                                                                                       \
        out[2 * (k + r * m)] = sr;                                                                              \
        out[2 * (k + r * m) + 1] = si;                                                                          \
      }                                                                                                         \
    }                                                                                                           \
    if (t != tloc) free(t);                                                                                     \
  }                                                                                                             \
  static T* twiddles_##SUF(size_t L) {                                                                          \
    T* tw = (T*)malloc(2 * L * sizeof(T));                                                                      \
    const long double pi = 3.141592653589793238462643383279502884L;                                            \
    for (size_t m = 0; m < L; ++m) {                                                                            \
      const long double a = -2.0L * pi * (long double)m / (long double)L;                                       \
      tw[2 * m] = (T)cosl(a);                                                                                   \
      tw[2 * m + 1] = (T)sinl(a);                                                                               \
    }                                                                                                           \
    return tw;                                                                                                  \
  }                                                                                                             \
  /* fft.hpp:110-125: real series -> L/2+1 bins, unnormalized, sign -1 */                                    \
  static void r2c_##SUF(size_t L, size_t batch, const T* in, T* out) {                                         \
    T* tw = twiddles_##SUF(L);                                                                                  \
    T* a = (T*)malloc(2 * L * sizeof(T));                                                                       \
    T* b = (T*)malloc(2 * L * sizeof(T));                                                                       \
    const size_t nb = L / 2 + 1;                                                                                \
    for (size_t s = 0; s < batch; ++s) {                                                                        \
      for (size_t t = 0; t < L; ++t) {                                                                          \
        a[2 * t] = in[s * L + t];                                                                               \
        a[2 * t + 1] = 0;                                                                                       \
      }                                                                                                         \
      fft_rec_##SUF(a, 1, b, L, tw, L, -1);                                                                     \
      memcpy(out + 2 * s * nb, b, 2 * nb * sizeof(T));                                                          \
    }                                                                                                           \
    free(a);                                                                                                    \
    free(b);                                                                                                    \
    free(tw);                                                                                                   \
  }                                                                                                             \
  /* fft.hpp:130-148: scratch = bins * (1/L in T), then unnormalized c2r that \
   * treats the spectrum as Hermitian (Im of DC and Nyquist ignored). */                                        \
  static void c2r_##SUF(size_t L, size_t batch, const T* in, T* out) {                                         \
    T* tw = twiddles_##SUF(L);                                                                                  \
    T* a = (T*)malloc(2 * L * sizeof(T));                                                                       \
    T* b = (T*)malloc(2 * L * sizeof(T));                                                                       \
    const size_t nb = L / 2 + 1;                                                                                \
    const T inv_len = (T)1 / (T)L;                                                                              \
    for (size_t s = 0; s < batch; ++s) {                                                                        \
      const T* x = in + 2 * s * nb;                                                                             \
      for (size_t k = 0; k < nb; ++k) {                                                                         \
        a[2 * k] = x[2 * k] * inv_len;                                                                          \
        a[2 * k + 1] = (k == 0 || k == L / 2) ? (T)0 : x[2 * k + 1] * inv_len;                                  \
      }                                                                                                         \
      for (size_t k = nb; k < L; ++k) {                                                                         \
        a[2 * k] = a[2 * (L - k)];                                                                              \
        a[2 * k + 1] = -a[2 * (L - k) + 1];                                                                     \
      }                                                                                                         \
      fft_rec_##SUF(a, 1, b, L, tw, L, +1);                                                                     \
      for (size_t t = 0; t < L; ++t) out[s * L + t] = b[2 * t];                                                 \
    }                                                                                                           \
    free(a);                                                                                                    \
    free(b);                                                                                                    \
    free(tw);                                                                                                   \
  }

DEFINE_FFT(double, d)
DEFINE_FFT(float, f)

int orc_fft_forward(size_t L, size_t batch, int prec, const void* in, void* out) {
  if (L < 2 || L % 2) return fail("FftPlan: length must be even and >= 2");
  if (batch < 1) return fail("FftPlan: batch must be >= 1");
  if (prec)
    r2c_d(L, batch, (const double*)in, (double*)out);
  else
    r2c_f(L, batch, (const float*)in, (float*)out);
  return 0;
}
int orc_fft_inverse(size_t L, size_t batch, int prec, const void* in, void* out) {
  if (L < 2 || L % 2) return fail("FftPlan: length must be even and >= 2");
  if (batch < 1) return fail("FftPlan: batch must be >= 1");
  if (prec)
    c2r_d(L, batch, (const double*)in, (double*)out);
  else
    c2r_f(L, batch, (const float*)in, (float*)out);
  return 0;
}

/* ------------------------------------------------------------------ GEMV */
/* gemv.hpp:100-108 madd; :135-148 naive_trans; :150-163 naive_notrans.
 * Arithmetic in the operand precision T. */
#define DEFINE_GEMV_REAL(T, SUF)                                                                                 \
  static void gemv_##SUF(int mode, size_t m, size_t n, size_t batch, size_t lda, size_t sa, const T* A, size_t sx, \
                         const T* x, size_t sy, T* y) {                                                           \
    for (size_t b = 0; b < batch; ++b) {                                                                          \
      const T* Ab = A + b * sa;                                                                                   \
      const T* xb = x + b * sx;                                                                                   \
      T* yb = y + b * sy;                                                                                         \
      if (mode == 0) {                                                                                            \
        for (size_t i = 0; i < m; ++i) yb[i] = 0;                                                                 \
        for (size_t j = 0; j < n; ++j)                                                                            \
          for (size_t i = 0; i < m; ++i) yb[i] = yb[i] + Ab[j * lda + i] * xb[j];                                 \
      } else {                                                                                                    \
        for (size_t j = 0; j < n; ++j) {                                                                          \
          T acc = 0;                                                                                              \
          for (size_t i = 0; i < m; ++i) acc = acc + Ab[j * lda + i] * xb[i];                                     \
          yb[j] = acc;                                                                                            \
        }                                                                                                         \
      }                                                                                                           \
    }                                                                                                             \
  }
#define DEFINE_GEMV_CPLX(T, SUF)                                                                                 \
  static void gemv_##SUF(int mode, size_t m, size_t n, size_t batch, size_t lda, size_t sa, const T* A, size_t sx, \
                         const T* x, size_t sy, T* y) {                                                           \
    for (size_t b = 0; b < batch; ++b) {                                                                          \
      const T* Ab = A + 2 * b * sa;                                                                               \
      const T* xb = x + 2 * b * sx;                                                                               \
      T* yb = y + 2 * b * sy;                                                                                     \
      if (mode == 0) {                                                                                            \
        for (size_t i = 0; i < 2 * m; ++i) yb[i] = 0;                                                             \
        for (size_t j = 0; j < n; ++j) {                                                                          \
          const T xr = xb[2 * j], xi = xb[2 * j + 1];                                                             \
          for (size_t i = 0; i < m; ++i) {                                                                        \
            const T ar = Ab[2 * (j * lda + i)], ai = Ab[2 * (j * lda + i) + 1];                                   \
            yb[2 * i] = yb[2 * i] + (ar * xr - ai * xi);                                                          \
            yb[2 * i + 1] = yb[2 * i + 1] + (ar * xi + ai * xr);                                                  \
          }                                                                                                       \
        }                                                                                                         \
      } else {                                                                                                    \
        const T cs = mode == 2 ? (T)-1 : (T)1;                                                                    \
        for (size_t j = 0; j < n; ++j) {                                                                          \
          T accr = 0, acci = 0;                                                                                   \
          for (size_t i = 0; i < m; ++i) {                                                                        \
            const T ar = Ab[2 * (j * lda + i)], ai = cs * Ab[2 * (j * lda + i) + 1];                              \
            const T xr = xb[2 * i], xi = xb[2 * i + 1];                                                           \
            accr = accr + (ar * xr - ai * xi);                                                                    \
            acci = acci + (ar * xi + ai * xr);                                                                    \
          }                                                                                                       \
          yb[2 * j] = accr;                                                                                       \
          yb[2 * j + 1] = acci;                                                                                   \
        }                                                                                                         \
      }                                                                                                           \
    }                                                                                                             \
  }
DEFINE_GEMV_REAL(float, s)
DEFINE_GEMV_REAL(double, d)
DEFINE_GEMV_CPLX(float, c)
DEFINE_GEMV_CPLX(double, z)

int orc_gemv(int mode, char dtype, size_t m, size_t n, size_t batch, size_t lda, size_t sa, const void* A, size_t sx,
             const void* x, size_t sy, void* y) {
  if (m == 0 || n == 0 || batch == 0) return fail("gemv: empty matrix batch");
  if (lda < m) return fail("gemv: lda < rows");
  switch (dtype) {
    case 's': gemv_s(mode, m, n, batch, lda, sa, A, sx, x, sy, y); break;
    case 'd': gemv_d(mode, m, n, batch, lda, sa, A, sx, x, sy, y); break;
    case 'c': gemv_c(mode, m, n, batch, lda, sa, A, sx, x, sy, y); break;
    case 'z': gemv_z(mode, m, n, batch, lda, sa, A, sx, x, sy, y); break;
    default: return fail("gemv: dtype must be s/d/c/z");
  }
  return 0;
}

/* ------------------------------------------------------------- operator */
struct orc_op {
  size_t nm, nd, nt;
  double* bins; /* nb * nd * nm complex, interleaved */
};

/* operator.hpp:99-125: pad every (i,j) series to L = 2nt, f64 r2c, scatter
 * to bins[k*nd*nm + s]. */
orc_op* orc_setup_operator(size_t nm, size_t nd, size_t nt, const double* col) {
  if (nm < 1 || nd < 1 || nt < 1) {
    fail("ProblemDims: all extents must be >= 1");
    return NULL;
  }
  const size_t S = nd * nm, L = 2 * nt, nb = nt + 1;
  orc_op* op = (orc_op*)calloc(1, sizeof(orc_op));
  op->nm = nm;
  op->nd = nd;
  op->nt = nt;
  op->bins = (double*)malloc(2 * nb * S * sizeof(double));
  double* pad = (double*)calloc(L, sizeof(double));
  double* spec = (double*)malloc(2 * nb * sizeof(double));
  for (size_t s = 0; s < S; ++s) {
    for (size_t t = 0; t < nt; ++t) pad[t] = col[t * S + s];
    r2c_d(L, 1, pad, spec);
    for (size_t k = 0; k < nb; ++k) {
      op->bins[2 * (k * S + s)] = spec[2 * k];
      op->bins[2 * (k * S + s) + 1] = spec[2 * k + 1];
    }
  }
  free(pad);
  free(spec);
  return op;
}
void orc_op_free(orc_op* op) {
  if (!op) return;
  free(op->bins);
  free(op);
}
void orc_op_bins(const orc_op* op, double* out) {
  memcpy(out, op->bins, 2 * (op->nt + 1) * op->nd * op->nm * sizeof(double));
}

/* ------------------------------------------------------------- pipeline */
static int check_cfg(const char* cfg) {
  if (!cfg || strlen(cfg) != 5) return fail("precision config must be exactly 5 characters");
  for (int i = 0; i < 5; ++i)
    if (cfg[i] != 'd' && cfg[i] != 's' && cfg[i] != 'h') return fail("precision config: invalid character");
  if (cfg[1] == 'h' || cfg[3] == 'h') return fail("precision config: fp16 FFT phases are not supported");
  return 0;
}

/* FFT in precision p over `batch` real series of length L (values held as
 * doubles already rounded to p). */
static void fft_fwd_p(char p, size_t L, size_t batch, const double* in, double* out) {
  const size_t nb = L / 2 + 1;
  if (p == 'd') {
    r2c_d(L, batch, in, out);
    return;
  }
  float* fi = (float*)malloc(L * batch * sizeof(float));
  float* fo = (float*)malloc(2 * nb * batch * sizeof(float));
  for (size_t i = 0; i < L * batch; ++i) fi[i] = (float)in[i];
  r2c_f(L, batch, fi, fo);
  for (size_t i = 0; i < 2 * nb * batch; ++i) out[i] = fo[i];
  free(fi);
  free(fo);
}
static void fft_inv_p(char p, size_t L, size_t batch, const double* in, double* out) {
  const size_t nb = L / 2 + 1;
  if (p == 'd') {
    c2r_d(L, batch, in, out);
    return;
  }
  float* fi = (float*)malloc(2 * nb * batch * sizeof(float));
  float* fo = (float*)malloc(L * batch * sizeof(float));
  for (size_t i = 0; i < 2 * nb * batch; ++i) fi[i] = (float)in[i];
  c2r_f(L, batch, fi, fo);
  for (size_t i = 0; i < L * batch; ++i) out[i] = fo[i];
  free(fi);
  free(fo);
}

/* matvec.hpp:209-228 + gemv.hpp: per-bin GEMV in precision p; x, y TOSI.
 * 'd': c128 arithmetic on bins_double; 's': c64 on rnd_f32(bins_double)
 * (operator.hpp:70-75); 'h': fp16-rounded operands, fp32 accumulation. */
static void gemv_stage_p(const orc_op* op, char p, int adjoint, const double* x, double* y) {
  const size_t nb = op->nt + 1, nd = op->nd, nm = op->nm, S = nd * nm;
  const size_t xl = adjoint ? nd : nm, yl = adjoint ? nm : nd;
  const int mode = adjoint ? 2 : 0;
  if (p == 'd') {
    gemv_z(mode, nd, nm, nb, nd, S, op->bins, xl, x, yl, y);
    return;
  }
  float* A = (float*)malloc(2 * nb * S * sizeof(float));
  float* xf = (float*)malloc(2 * nb * xl * sizeof(float));
  float* yf = (float*)malloc(2 * nb * yl * sizeof(float));
  for (size_t i = 0; i < 2 * nb * S; ++i) A[i] = (float)rnd(p, op->bins[i]);
  for (size_t i = 0; i < 2 * nb * xl; ++i) xf[i] = (float)x[i]; /* already rounded to p */
  gemv_c(mode, nd, nm, nb, nd, S, A, xl, xf, yl, yf);
  for (size_t i = 0; i < 2 * nb * yl; ++i) y[i] = yf[i];
  free(A);
  free(xf);
  free(yf);
}

/* matvec.hpp:233-289 run_pipeline. payload (partition adjoint) = input
 * already rounded to cfg[0], padded without further rounding (:106-114). */
static int pipeline(const orc_op* op, int kind, const char* cfg, const double* in, int payload, double* out,
                    uint64_t* casts) {
  if (check_cfg(cfg)) return -1;
  const size_t nt = op->nt, L = 2 * nt, nb = nt + 1;
  const int adj = kind != 0;
  const size_t n_in = adj ? op->nd : op->nm, n_out = adj ? op->nm : op->nd;
  uint64_t nc = 0;
  /* Phase 1 pad (+cast cfg0), Phase 2 convert to cfg1 + r2c in cfg1. */
  double* pad = (double*)calloc(n_in * L, sizeof(double));
  for (size_t s = 0; s < n_in; ++s)
    for (size_t t = 0; t < nt; ++t) pad[s * L + t] = rnd(cfg[1], payload ? in[s * nt + t] : rnd(cfg[0], in[s * nt + t]));
  if (!payload && cfg[0] != 'd') ++nc; /* matvec.hpp:88 */
  if (cfg[0] != cfg[1]) ++nc;          /* matvec.hpp:118-130 */
  double* spec = (double*)malloc(2 * n_in * nb * sizeof(double));
  fft_fwd_p(cfg[1], L, n_in, pad, spec);
  free(pad);
  /* Phase 3: SOTI->TOSI with cast to cfg2, GEMV in cfg2, TOSI->SOTI cast to cfg3. */
  double* x = (double*)malloc(2 * n_in * nb * sizeof(double));
  for (size_t s = 0; s < n_in; ++s)
    for (size_t k = 0; k < nb; ++k) {
      x[2 * (k * n_in + s)] = rnd(cfg[2], spec[2 * (s * nb + k)]);
      x[2 * (k * n_in + s) + 1] = rnd(cfg[2], spec[2 * (s * nb + k) + 1]);
    }
  if (cfg[1] != cfg[2]) ++nc;
  free(spec);
  double* y = (double*)malloc(2 * n_out * nb * sizeof(double));
  gemv_stage_p(op, cfg[2], adj, x, y);
  free(x);
  double* ys = (double*)malloc(2 * n_out * nb * sizeof(double));
  for (size_t k = 0; k < nb; ++k)
    for (size_t s = 0; s < n_out; ++s) {
      ys[2 * (s * nb + k)] = rnd(cfg[3], y[2 * (k * n_out + s)]);
      ys[2 * (s * nb + k) + 1] = rnd(cfg[3], y[2 * (k * n_out + s) + 1]);
    }
  if (cfg[2] != cfg[3]) ++nc;
  free(y);
  /* Phase 4: c2r in cfg3 (1/L pre-scale inside). Phase 5: unpad, cfg4, double. */
  double* ser = (double*)malloc(n_out * L * sizeof(double));
  fft_inv_p(cfg[3], L, n_out, ys, ser);
  free(ys);
  for (size_t s = 0; s < n_out; ++s)
    for (size_t t = 0; t < nt; ++t) out[s * nt + t] = rnd(cfg[4], ser[s * L + t]);
  if (cfg[3] != cfg[4]) ++nc; /* matvec.hpp:189-190 */
  if (cfg[4] != 'd') ++nc;
  free(ser);
  if (casts) *casts = nc;
  return 0;
}

int orc_matvec(const orc_op* op, int kind, const char* cfg, const double* in, double* out, uint64_t* casts) {
  if (!op) return fail("matvec: null operator");
  return pipeline(op, kind, cfg, in, 0, out, casts);
}

/* ---------------------------------------------------------------- dense */
/* dense_ref.hpp:22-64 */
int orc_dense(int kind, size_t nm, size_t nd, size_t nt, const double* col, const double* in, double* out) {
  if ((double)nd * (double)nm * (double)nt * (double)nt > 1e8)
    return fail("dense reference: instance too large (n_d*n_m*n_t^2 > 1e8)");
  const size_t S = nd * nm;
#define AT(t, r, c) col[(t) * S + (r) + (c) * nd]
  if (kind == 0) {
    memset(out, 0, nd * nt * sizeof(double));
    for (size_t i = 0; i < nt; ++i)
      for (size_t j = 0; j <= i; ++j)
        for (size_t c = 0; c < nm; ++c) {
          const double mv = in[c * nt + j];
          for (size_t r = 0; r < nd; ++r) out[r * nt + i] += AT(i - j, r, c) * mv;
        }
  } else {
    memset(out, 0, nm * nt * sizeof(double));
    for (size_t j = 0; j < nt; ++j)
      for (size_t i = j; i < nt; ++i)
        for (size_t c = 0; c < nm; ++c) {
          double acc = 0.0;
          for (size_t r = 0; r < nd; ++r) acc += AT(i - j, r, c) * in[r * nt + i];
          out[c * nt + j] += acc;
        }
  }
#undef AT
  return 0;
}

/* ------------------------------------------------------------ partition */
/* partition.hpp:27-40 */
int orc_grid_split(size_t p, size_t nm, size_t* ranges) {
  if (p < 1) return fail("Grid1xP: p must be >= 1");
  if (p > nm) return fail("Grid1xP: more workers than parameter columns");
  const size_t base = nm / p, rem = nm % p;
  size_t begin = 0;
  for (size_t w = 0; w < p; ++w) {
    const size_t sz = base + (w < rem ? 1 : 0);
    ranges[2 * w] = begin;
    ranges[2 * w + 1] = begin + sz;
    begin += sz;
  }
  return 0;
}

/* partition.hpp:84-132: inputs cast to prec, fixed left-balanced pairwise
 * tree ((b0+b1)+(b2+b3)), ((b0+b1)+b2) for odd levels, root cast to double. */
int orc_tree_reduce(size_t p, size_t n, const double* bufs, int prec, double* out) {
  if (p < 1) return fail("tree_reduce: no buffers");
  double* lv = (double*)malloc(p * n * sizeof(double));
  for (size_t i = 0; i < p * n; ++i) lv[i] = prec ? bufs[i] : (double)(float)bufs[i];
  size_t cnt = p;
  while (cnt > 1) {
    size_t nx = 0;
    for (size_t k = 0; k + 1 < cnt; k += 2, ++nx)
      for (size_t i = 0; i < n; ++i) {
        const double s = lv[k * n + i] + lv[(k + 1) * n + i];
        lv[nx * n + i] = prec ? s : (double)((float)lv[k * n + i] + (float)lv[(k + 1) * n + i]);
      }
    if (cnt % 2 == 1) {
      memmove(lv + nx * n, lv + (cnt - 1) * n, n * sizeof(double));
      ++nx;
    }
    cnt = nx;
  }
  memcpy(out, lv, n * sizeof(double));
  free(lv);
  return 0;
}

/* partition.hpp:63-80 shard_operator + :141-217 partitioned matvecs. */
int orc_matvec_partitioned(size_t nm, size_t nd, size_t nt, const double* col, size_t p, int kind, const char* cfg,
                           const double* in, double* out) {
  if (check_cfg(cfg)) return -1;
  size_t* rg = (size_t*)malloc(2 * p * sizeof(size_t));
  if (orc_grid_split(p, nm, rg)) {
    free(rg);
    return -1;
  }
  double* partials = kind == 0 ? (double*)malloc(p * nd * nt * sizeof(double)) : NULL;
  double* payload = NULL;
  if (kind != 0) { /* partition.hpp:196-206: cast d to cfg0 once */
    payload = (double*)malloc(nd * nt * sizeof(double));
    for (size_t i = 0; i < nd * nt; ++i) payload[i] = rnd(cfg[0], in[i]);
  }
  for (size_t w = 0; w < p; ++w) {
    const size_t lo = rg[2 * w], hi = rg[2 * w + 1], snm = hi - lo;
    double* sc = (double*)malloc(nt * nd * snm * sizeof(double));
    for (size_t t = 0; t < nt; ++t)
      for (size_t j = lo; j < hi; ++j)
        for (size_t i = 0; i < nd; ++i) sc[t * nd * snm + i + (j - lo) * nd] = col[t * nd * nm + i + j * nd];
    orc_op* op = orc_setup_operator(snm, nd, nt, sc);
    free(sc);
    if (kind == 0)
      pipeline(op, 0, cfg, in + lo * nt, 0, partials + w * nd * nt, NULL);
    else
      pipeline(op, 1, cfg, payload, 1, out + lo * nt, NULL);
    orc_op_free(op);
  }
  if (kind == 0) orc_tree_reduce(p, nd * nt, partials, cfg[4] == 'd', out);
  free(partials);
  free(payload);
  free(rg);
  return 0;
}
