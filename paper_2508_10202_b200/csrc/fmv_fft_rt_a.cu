// fmv_fft_rt_a.cu -- runtime-plan register FFT kernels for pass radix 16, 10
// (fmv_fft_rt_inst.cuh).
#include "fmv_fft_rt_inst.cuh"

FMV_RT_INSTANTIATE(16)
FMV_RT_INSTANTIATE(10)
