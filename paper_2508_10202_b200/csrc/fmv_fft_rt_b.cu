// fmv_fft_rt_b.cu -- runtime-plan register FFT kernels for pass radix 8, 5
// (fmv_fft_rt_inst.cuh).
#include "fmv_fft_rt_inst.cuh"

FMV_RT_INSTANTIATE(8)
FMV_RT_INSTANTIATE(5)
