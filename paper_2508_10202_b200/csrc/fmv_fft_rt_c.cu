// fmv_fft_rt_c.cu -- runtime-plan register FFT kernels for pass radix 4, 3, 2, 7
// (fmv_fft_rt_inst.cuh).
#include "fmv_fft_rt_inst.cuh"

FMV_RT_INSTANTIATE(4)
FMV_RT_INSTANTIATE(3)
FMV_RT_INSTANTIATE(2)
FMV_RT_INSTANTIATE(7)
