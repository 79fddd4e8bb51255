// fmv_fft_stream.cuh -- persistent, prefetching register FFTs for the big
// Nt = 1000 transforms of the matvec (F's r2c over the Nm series of m, F*'s
// c2r over the Nm series of the SBGEMV output).
//
// The per-series math is k_r2c_reg / k_c2r_reg's (fmv_fft.cuh): radix-10
// Stockham passes with one butterfly per thread, the split post-/pre-pass
// to the N + 1 bins, all reorders and casts fused (fft.hpp:32-148,
// matvec.hpp:83-205). What changes is the schedule. ncu on the
// one-shot kernels (profiles/ncu_fft_r02.md) shows them latency-bound:
// each CTA loads its series, then computes with no memory traffic in
// flight, so DRAM runs at 18-26 % of peak and "long scoreboard" is the top
// stall. Here each CTA is persistent and owns a staging buffer next to its
// work buffer: as soon as pass 1 has consumed tile i's input from the stage,
// the fetch of tile i + gridDim.x's input is issued and lands while tile i
// runs its remaining passes and its output stores.
//   * r2c: the S series of a tile are S consecutive rows of the SOTI input,
//     one contiguous S*Nt*8-byte range -> ONE cp.async.bulk (TMA, UBLKCP)
//     issued by one thread, completion on an mbarrier.
//   * c2r: the tile is an (N+1) x S box of the TOSI input (S-element runs
//     with row stride in_ks) -> cp.async (LDGSTS) 16/8-byte copies spread
//     over the CTA, completion by cp.async.wait_group + barrier.
// Input reads are evict-first (read once); no register staging, so the
// prefetch costs no registers (a register-prefetching persistent variant
// spilled).
#pragma once

#include "fmv_fft.cuh"
#include "fmv_tma.cuh"

namespace fmv {

// An opaque copy of v: keeps per-thread index arithmetic inside the tile loop
// instead of letting the compiler hoist ~30 loop-invariant addresses into
// registers for the whole persistent loop (which spilled).
__device__ __forceinline__ int opaque(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// One Stockham pass (Ns > 1) as reg_pass, but for every thread: the series
// slots of a partial last tile are private scratch, so idle threads compute
// on them instead of branching -- no divergent region keeps the ten
// butterfly values alive across the barrier (which made ptxas spill).
template <class R, int D, int Ns>
__device__ __forceinline__ void stream_pass(typename CT<R>::c* __restrict__ buf, int j,
                                            const typename CT<R>::c* __restrict__ tw) {
  using C = typename CT<R>::c;
  constexpr int RX = 10, N = 1000, NR = 100;
  const C* __restrict__ twp = tw + reg_tw_offset<RX, N, Ns>();
  C v[RX];
  const int k = j % Ns;
#pragma unroll
  for (int q = 0; q < RX; ++q) v[q] = buf[j + q * NR];
  apply_twiddles<R, D, RX, Ns>(v, twp, k);
  butterfly<R, D, RX>(v);
  __syncthreads();
  const int o = (j - k) * RX + k;
#pragma unroll
  for (int q = 0; q < RX; ++q) buf[o + q * Ns] = v[q];
  __syncthreads();
}

template <class Tin, int S>
constexpr size_t r2c_stream_stage_bytes() {
  return (size_t)S * 1000 * sizeof(Tin);
}
template <class C, int S>
constexpr size_t r2c_stream_stage_off() {  // work buffer bytes, rounded to 128
  return ((size_t)S * reg_series_stride<C, 1000, S>() * sizeof(C) + 127) / 128 * 128;
}
template <class C, int S>
constexpr size_t r2c_stream_smem() {  // work | stage | mbarrier
  return r2c_stream_stage_off<C, S>() + r2c_stream_stage_bytes<double, S>() + 16;
}
template <class C, int S>
constexpr size_t c2r_stream_smem() {  // work | stage
  return 2 * (size_t)S * reg_series_stride<C, 1001, S>() * sizeof(C);
}

// Phases 1-2 + reorder: SOTI input in[s*1000 + t] (contiguous series,
// zero-padded to L = 2000 -- the matvec pad stage), TOSI output
// out[k*out_ks + s]. ntiles = ceil(nseries / S); CTA b runs tiles b, b + G, ...
template <int C0, int C1, int C2, int S, int MAXR>
__global__ void __launch_bounds__(S * 100) __maxnreg__(MAXR)
    k_r2c_stream(const double* __restrict__ in, long nseries, typename PT<C2>::cplx* __restrict__ out, long out_ks,
                 const typename CT<typename PT<C1>::real>::c* __restrict__ tw) {
  using R = typename PT<C1>::real;
  using C = typename CT<R>::c;
  using OutC = typename PT<C2>::cplx;
  constexpr int RX = 10, N = 1000, NR = 100, T = S * NR;
  constexpr int SS = reg_series_stride<C, N, S>();
  extern __shared__ __align__(128) unsigned char r2c_stream_smem_raw[];
  C* sbuf = reinterpret_cast<C*>(r2c_stream_smem_raw);
  double* stage = reinterpret_cast<double*>(r2c_stream_smem_raw + r2c_stream_stage_off<C, S>());
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(stage) + r2c_stream_stage_bytes<double, S>());
  const int s = threadIdx.x / NR;
  const long ntiles = (nseries + S - 1) / S;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  grid_dep_wait();  // (PDL)
  uint64_t pol = 0;
  auto fetch = [&](long tile) {  // thread 0 only
    const long s0 = tile * S;
    const uint32_t bytes = (uint32_t)(min((long)S, nseries - s0) * N * sizeof(double));
    mbar_expect_tx(bar, bytes);
    bulk_g2s(stage, in + s0 * N, bytes, bar, pol);
  };
  if (threadIdx.x == 0) {
    pol = policy_evict_first();
    if ((long)blockIdx.x < ntiles) fetch(blockIdx.x);
  }
  uint32_t phase = 0;
#pragma unroll 1
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long s0 = tile * S;
    const int ns = (int)min((long)S, nseries - s0);
    const int j = opaque(threadIdx.x - s * NR);
    C* buf = sbuf + s * SS;
    mbar_wait(bar, phase);
    phase ^= 1;
    // Pass 1 (Ns = 1): z[n] = v[2n] + i v[2n+1] from the stage; n >= N/2 is padding.
    // (a partial last tile leaves stale stage rows: idle threads transform
    // them into their own unused slots)
    {
      C v[RX];
      const double2* p = reinterpret_cast<const double2*>(stage + s * N);
#pragma unroll
      for (int q = 0; q < RX; ++q) {
        v[q] = C{R(0), R(0)};
        if (q < RX / 2) {
          const double2 pr = p[j + q * NR];
          v[q] = C{(R)rnd<C0>(pr.x), (R)rnd<C0>(pr.y)};
        }
      }
      butterfly<R, -1, RX>(v);
      store_stride_rx<RX>(buf + j * RX, v);
    }
    __syncthreads();  // the stage is consumed: prefetch the next tile into it
    if (threadIdx.x == 0 && tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
    stream_pass<R, -1, RX>(buf, j, tw);
    stream_pass<R, -1, RX * RX>(buf, j, tw);
    // Post-pass (as k_r2c_reg): bins k and N - k share Z[k], Z[N-k]; consecutive
    // threads take consecutive series of one bin (S-element TOSI runs).
    const R half = R(0.5);
    auto post = [&](C A, C B, int k) {  // B = conj(Z[N-k])
      const C E = {(A.x + B.x) * half, (A.y + B.y) * half};
      const C Dm = {(A.x - B.x) * half, (A.y - B.y) * half};
      return cadd(E, cmul(__ldg(tw + k), cmuli<-1>(Dm)));
    };
#pragma unroll 1
    for (int e = threadIdx.x; e < S * (N / 2 + 1); e += T) {
      const int k = e / S, si = e - k * S;
      if (si >= ns) continue;
      const C* Z = sbuf + si * SS;
      const int kp = k == 0 ? N : N - k;
      const C A1 = Z[k];
      const C A2 = Z[k == 0 ? 0 : N - k];
      out[(long)k * out_ks + s0 + si] = cfrom_d<OutC>(to_cd(post(A1, cconj(A2), k)));
      if (kp != k) out[(long)kp * out_ks + s0 + si] = cfrom_d<OutC>(to_cd(post(A2, cconj(A1), kp)));
    }
    __syncthreads();  // the work buffer is free for the next tile's pass 1
  }
}

// Phases 4-5 + reorder: TOSI input in[k*in_ks + s], SOTI output
// out[s*out_ss + t], t < N (the first half of the L = 2000 samples -- the
// matvec unpad stage).
template <int C3, int C4, class Tout, int S, int MAXR>
__global__ void __launch_bounds__(S * 100) __maxnreg__(MAXR)
    k_c2r_stream(const typename PT<C3>::cplx* __restrict__ in, long in_ks, long nseries, bool vec,
                 Tout* __restrict__ out, long out_ss, const typename PT<C3>::cplx* __restrict__ tw) {
  using R = typename PT<C3>::real;
  using C = typename CT<R>::c;
  constexpr int RX = 10, N = 1000, NR = 100, T = S * NR;
  constexpr int SS = reg_series_stride<C, N + 1, S>();
  extern __shared__ __align__(128) unsigned char c2r_stream_smem_raw[];
  C* sbuf = reinterpret_cast<C*>(c2r_stream_smem_raw);
  C* stage = sbuf + S * SS;
  const int s = threadIdx.x / NR;
  const long ntiles = (nseries + S - 1) / S;
  grid_dep_wait();  // (PDL)
  const R inv_len = R(1) / (R)(2 * N);
  auto fetch = [&](long tile) {  // all threads: the (N+1) x S box, bin-major runs of S
    const long s0 = tile * S;
    const int ns = (int)min((long)S, nseries - s0);
    for (int e = threadIdx.x; e < S * (N + 1); e += T) {
      const int k = e / S, si = e - k * S;
      const bool ok = si < ns;
      cp_async(stage + si * SS + k, in + (long)k * in_ks + s0 + (ok ? si : 0), ok ? (int)sizeof(C) : 0,
               (int)sizeof(C));
    }
    cp_async_commit();
  };
  if ((long)blockIdx.x < ntiles) fetch(blockIdx.x);
#pragma unroll 1
  for (long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const long s0 = tile * S;
    const int ns = (int)min((long)S, nseries - s0);
    const bool act = s < ns;
    const int j = opaque(threadIdx.x - s * NR);
    C* buf = sbuf + s * SS;
    cp_async_wait_all();
    __syncthreads();
    // Pre-pass fused into pass 1, from the stage: Z[n] = (X[n] + conj X[N-n])
    // + i w^-n (X[n] - conj X[N-n]) with X scaled by 1/L in C3 arithmetic and
    // Im X_0 = Im X_N = 0 (fft.hpp:130-148); result to the work buffer.
    {
      C v[RX];
      const C* xs = stage + s * SS;
      const C wj = __ldg(tw + j);
#pragma unroll
      for (int q = 0; q < RX; ++q) {
        const int n = j + q * NR;
        C A = xs[n], B = xs[N - n];  // X[n], X[N-n]
        A.x = A.x * inv_len;
        A.y = n == 0 ? R(0) : A.y * inv_len;
        B.x = B.x * inv_len;
        B.y = n == 0 ? -R(0) : -(B.y * inv_len);
        const C w = q == 0 ? wj : cmul(wj, half_turn10<R>(q));
        v[q] = cadd(cadd(A, B), cmuli<1>(cmul(C{w.x, -w.y}, csub(A, B))));
      }
      butterfly<R, 1, RX>(v);
      store_stride_rx<RX>(buf + j * RX, v);
    }
    __syncthreads();  // the stage is consumed: prefetch the next tile into it
    if (tile + gridDim.x < ntiles) fetch(tile + gridDim.x);
    stream_pass<R, 1, RX>(buf, j, tw);
    // Last pass (Ns = N/RX): Z -> the first N real samples, straight to global.
    {
      constexpr int Ns = NR;
      const C* __restrict__ twp = tw + reg_tw_offset<RX, N, Ns>();
      C v[RX];
      if (act) {
#pragma unroll
        for (int q = 0; q < RX; ++q) v[q] = buf[j + q * NR];
        apply_twiddles<R, 1, RX, Ns>(v, twp, j);
        butterfly<R, 1, RX>(v);
        Tout* p = out + (s0 + s) * out_ss;
#pragma unroll
        for (int q = 0; q < RX / 2; ++q) {  // n = j + q*NR < N/2: samples 2n, 2n+1 < N
          const int n = j + q * NR;
          const Tout a = (Tout)rnd<C4>((double)v[q].x);
          const Tout b = (Tout)rnd<C4>((double)v[q].y);
          if constexpr (sizeof(Tout) == 8) {
            if (vec) {
              reinterpret_cast<double2*>(p)[n] = make_double2(a, b);
              continue;
            }
          }
          p[2 * n] = a;
          p[2 * n + 1] = b;
        }
      }
    }
    // (the next iteration's wait + barrier orders this tile's work-buffer
    // reads before the next tile's pass-1 writes)
  }
  cp_async_wait_all();
}

}  // namespace fmv
