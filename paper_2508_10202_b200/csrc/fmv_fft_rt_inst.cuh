// fmv_fft_rt_inst.cuh -- host launchers of the runtime-plan register FFT
// kernels (fmv_fft_rt.cuh) for one pass radix RR; included by
// fmv_fft_rt_{a,b,c}.cu, which instantiate them for disjoint RR sets so the
// kernels compile in parallel.
#pragma once

#include "fmv_runtime.cuh"
#include "fmv_fft_rt.cuh"

namespace fmv {
namespace rt {

template <class R, class Tin, int RR>
void r2c_rt_go(fmv_ctx* ctx, int c0, int c2, const void* vin, long in_ss, long nseries, int nvalid, void* out,
               long out_ks, long out_ss, const RtPlan& P, const void* vtw) {
  using C = typename CT<R>::c;
  const Tin* in = static_cast<const Tin*>(vin);
  const bool vec =
      sizeof(Tin) == 8 && (in_ss % 2 == 0) && (nvalid % 2 == 0) && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  const size_t smem = (size_t)P.S * P.SS * sizeof(C);
  auto kern = k_r2c_rt<R, Tin, RR>;
  prep_smem((const void*)kern, smem);
  const long grid = (nseries + P.S - 1) / P.S;
  launch(ctx, 0, [&] {
    launch_pdl(kern, dim3((unsigned)grid), dim3(P.S * P.TS), smem, ctx->stream, in, in_ss, 1L, nseries, nvalid, vec,
               c0, out, c2, out_ks, out_ss, P, static_cast<const C*>(vtw));
  });
}

template <class R, class Tout, int RR>
void c2r_rt_go(fmv_ctx* ctx, int c4, const void* in, long in_ks, long in_ss, long nseries, int nout, void* out,
               long out_ss, const RtPlan& P, const void* vtw) {
  using C = typename CT<R>::c;
  const size_t smem = (size_t)P.S * P.SS * sizeof(C);
  auto kern = k_c2r_rt<R, Tout, RR>;
  prep_smem((const void*)kern, smem);
  const long grid = (nseries + P.S - 1) / P.S;
  launch(ctx, 3, [&] {
    launch_pdl(kern, dim3((unsigned)grid), dim3(P.S * P.TS), smem, ctx->stream, static_cast<const C*>(in), in_ks,
               in_ss, nseries, nout, c4, static_cast<Tout*>(out), out_ss, P, static_cast<const C*>(vtw));
  });
}

template <int RR>
void rt_r2c_run(fmv_ctx* ctx, int cr, int tin, int c0, int c2, const void* in, long in_ss, long nseries, int nvalid,
                void* out, long out_ks, long out_ss, const RtPlan& P, const void* tw) {
#define GO(RT, TT) r2c_rt_go<RT, TT, RR>(ctx, c0, c2, in, in_ss, nseries, nvalid, out, out_ks, out_ss, P, tw)
  if (cr == PD) {
    if (tin == PD) GO(double, double);
    else if (tin == PS) GO(double, float);
    else GO(double, __half);
  } else {
    if (tin == PD) GO(float, double);
    else if (tin == PS) GO(float, float);
    else GO(float, __half);
  }
#undef GO
}

template <int RR>
void rt_c2r_run(fmv_ctx* ctx, int cr, int tout, int c4, const void* in, long in_ks, long in_ss, long nseries,
                int nout, void* out, long out_ss, const RtPlan& P, const void* tw) {
#define GO(RT, TT) c2r_rt_go<RT, TT, RR>(ctx, c4, in, in_ks, in_ss, nseries, nout, out, out_ss, P, tw)
  if (cr == PD) {
    if (tout == PD) GO(double, double);
    else GO(double, float);
  } else {
    if (tout == PD) GO(float, double);
    else GO(float, float);
  }
#undef GO
}

}  // namespace rt
}  // namespace fmv

#define FMV_RT_INSTANTIATE(RR)                                                                                       \
  template void fmv::rt::rt_r2c_run<RR>(fmv_ctx*, int, int, int, int, const void*, long, long, int, void*, long, long, \
                                        const fmv::RtPlan&, const void*);                                              \
  template void fmv::rt::rt_c2r_run<RR>(fmv_ctx*, int, int, int, const void*, long, long, long, int, void*, long,     \
                                        const fmv::RtPlan&, const void*);
