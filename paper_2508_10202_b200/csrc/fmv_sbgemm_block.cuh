// fmv_sbgemm_block.cuh -- multi-RHS (block) SBGEMV for the block matvec
// (Hessian assembly applies F / F* to many vectors,
// PAPER.md:431-434, :510). Per frequency bin b the K right-hand sides are
// handled together, so the operator -- the 8 GB that bounds a matvec -- is
// streamed from HBM ONCE for all K:
//   NoTrans (F):   Y_b[:, r] = A_b X_b[:, r]          (r < K)
//   ConjTrans (F*): Z_b[:, r] = A_b^H D_b[:, r]
// This is a complex GEMM with a skinny K (<= 8) and arithmetic intensity
// 4K flop/B of operator (fp64): memory-bound up to K ~ 8 on B200's FP64 pipe,
// so it stays on CUDA cores (tensor cores have no complex-fp64 advantage and
// lower precision would change the result).
//
// Same producer / ring / flat-column-stream design as k_sbgemv (one
// cp.async.bulk producer lane, nstage shared stages, equal pieces per
// persistent CTA); one element per thread row (V = 1):
//  * NoTrans: thread (r, g) owns row r, columns g, g+G, ... of each stage and
//    keeps K accumulators; the stage's K x slices arrive with it. Bin flush
//    and the cross-CTA (last-arriver, piece-ordered) reduction as k_sbgemv,
//    with K*m partials per piece. fp32: per-stage partials folded with a
//    Neumaier add, like the single-RHS kernel.
//  * ConjTrans: LPC lanes per column split its rows (as k_sbgemv), each lane
//    with K accumulators: A[i, c] is read once for all K right-hand sides,
//    x_r[i] comes from the K vectors x_{b, r} kept resident per batch entry
//    (two slots by batch parity); one xor-shuffle tree per RHS.
#pragma once

#include "fmv_sbgemv.cuh"

namespace fmv {

// One 16-warp CTA per SM with ~64 KB stages, as k_sbgemv: at C2 fp64 F K = 8
// goes 2949 -> 3190 RHS/s against two 8-warp CTAs per SM (tools/ab_block.sh).
#ifndef FMV_BLOCK_CONS
#define FMV_BLOCK_CONS 416  // consumer threads per CTA (+ one producer warp): 14 warps -> up to 128 registers (tools/bench_block.py)
#endif
#ifndef FMV_BLOCK_MINB
#define FMV_BLOCK_MINB 1  // resident CTAs per SM
#endif
// D += A B for one 8x8x4 fp64 tile held in PTX m8n8k4 fragments (DMMA).
__device__ __forceinline__ void dmma_884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// KX > 0, NoTrans fp64: exactly KX = KR right-hand sides and x slices XR
// bytes apart in shared memory, both compile-time -- the column loop then has
// no per-RHS predicates and every x read is one LDS.128 at an immediate offset
// from a single per-column base (the runtime-K loop spent ~30 integer /
// predicate instructions per 32 DFMAs on this).
// KX > 0, ConjTrans: exactly KX right-hand sides, two columns per lane.
// TC > 0, NoTrans fp64 with KX = 8: the complex MACs run on the FP64 tensor
// path (DMMA, mma.sync m8n8k4 f64) for up to TC row tiles of 8 (m <= 8 TC):
// see the TC branch below.
// (TC: up to 16 consumer warps + the producer; a warp holds TC tiles' 8 TC
// accumulator registers, so the 96 registers of 5 warps per SM sub-partition
// suffice.)
template <int MODE, class E, class O, int KR, int LPC, int KX = 0, int XR = 0, int TC = 0>
__global__ void __launch_bounds__(TC > 0 ? 16 * 32 + 32 : FMV_BLOCK_CONS + 32, FMV_BLOCK_MINB)
    k_sbgemm_block(const GemvParams p) {
  using Tr = ET<E>;
  using Acc = typename Tr::A;
  extern __shared__ __align__(128) unsigned char sm[];
  const int ncons = blockDim.x - 32;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  volatile int* s_flag = reinterpret_cast<volatile int*>(sm + 256);
  unsigned char* stages = sm + 512;
  const int xs_bytes = KR * p.xr_slot;  // all K x slices of one stage / batch entry
  const int slot = p.a_slot + (p.xres ? 0 : xs_bytes);
  unsigned char* xres_base = stages + (long)p.nstage * slot;
  Acc* red = reinterpret_cast<Acc*>(xres_base + (p.xres ? 2L * xs_bytes : 0L));
  const int K = p.K;

  if (threadIdx.x == 0) {
    for (int s = 0; s < p.nstage; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.arrive_all ? ncons : ncons / 32);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const long c0 = p.T * (long)blockIdx.x / p.P;
  const long c1 = p.T * (long)(blockIdx.x + 1) / p.P;
  constexpr int es = (int)sizeof(E);

  if (threadIdx.x >= ncons) {
    if (threadIdx.x != ncons) return;
    const uint64_t pol_a = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();
    long prev_b = -1;
    for (SegIter sg(c0, c1, p); sg.more(); sg.advance(p)) {
      sg.load(p);
      const int s = sg.s;
      mbar_wait(&empty[s], sg.par ^ 1u);
      const bool new_x = !p.xres || sg.b != prev_b;
      prev_b = sg.b;
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* a_lo = reinterpret_cast<const unsigned char*>(reinterpret_cast<uintptr_t>(a0) & ~uintptr_t(15));
      const uintptr_t a_end = reinterpret_cast<uintptr_t>(a0) + (uintptr_t)(((sg.cnt - 1) * p.lda + p.m) * es);
      const uint32_t a_bytes = (uint32_t)(((a_end + 15) & ~uintptr_t(15)) - reinterpret_cast<uintptr_t>(a_lo));
      const long xn = MODE == GM_N ? sg.cnt : p.m;
      uint32_t xb[KR];
      const unsigned char* xlo[KR];
      uint32_t x_total = 0;
#pragma unroll
      for (int r = 0; r < KR; ++r) {
        xb[r] = 0;
        xlo[r] = nullptr;
        if (r < K && new_x) {
          const unsigned char* x0 = p.x + (sg.b * p.sx + r * p.sxr + (MODE == GM_N ? sg.j : 0)) * es;
          xlo[r] = reinterpret_cast<const unsigned char*>(reinterpret_cast<uintptr_t>(x0) & ~uintptr_t(15));
          const uintptr_t x_end = reinterpret_cast<uintptr_t>(x0) + (uintptr_t)(xn * es);
          xb[r] = (uint32_t)(((x_end + 15) & ~uintptr_t(15)) - reinterpret_cast<uintptr_t>(xlo[r]));
          x_total += xb[r];
        }
      }
      unsigned char* dst = stages + (long)s * slot;
      unsigned char* xdst = p.xres ? xres_base + (sg.b & 1) * (long)xs_bytes : dst + p.a_slot;
      mbar_expect_tx(&full[s], a_bytes + x_total);
      bulk_g2s(dst, a_lo, a_bytes, &full[s], pol_a);
#pragma unroll
      for (int r = 0; r < KR; ++r)
        if (xb[r]) bulk_g2s(xdst + r * p.xr_slot, xlo[r], xb[r], &full[s], pol_x);
    }
    return;
  }

  const int t = threadIdx.x;
  const int lane = t & 31;
  if constexpr (MODE == GM_N) {
    const int r = t % p.RT;
    const int g = t / p.RT;
    const bool active = g < p.G && r < p.m;
    constexpr bool kComp = !std::is_same<Acc, double2>::value;
    // fp64: the four real products of each complex MAC go to four separate
    // accumulators (re = rr - ii, im = ri + ir at the bin flush), so the 4K
    // DFMAs of a column are independent: no DFMA -> DFMA dependency inside a
    // column, which left the FP64 pipe ~41 % busy behind `wait` stalls.
    constexpr bool kSplit = std::is_same<E, double2>::value;
    Acc acc[KR], cmp[KR];
    double rr[kSplit ? KR : 1], ii[kSplit ? KR : 1], ri[kSplit ? KR : 1], ir[kSplit ? KR : 1];
#pragma unroll
    for (int k = 0; k < KR; ++k) acc[k] = cmp[k] = Tr::zero();
#pragma unroll
    for (int k = 0; k < (kSplit ? KR : 1); ++k) rr[k] = ii[k] = ri[k] = ir[k] = 0.0;
    // TC: the consumer warps form nw/2 warp pairs; pair wp takes column pairs
    // wp, wp + nw/2, ... of each stage, its first warp row tiles 0..TC-1, its
    // second TC..2TC-2 (13 tiles of 8 rows for m <= 104). Per column pair and
    // row tile one 8-byte A load per lane feeds two DMMAs (real and imaginary
    // part of Y for all 8 right-hand sides). The real-ified product is
    //   Yr = [Ar Ai] [Xr; -Xi],  Yi = [Ar Ai] [Xi; Xr]
    // with the k index (column j, component c) matching the interleaved
    // complex layout of A, so A needs no reshuffle. Lane (g = lane/4, q =
    // lane%4) holds A[row 8T+g][k = q] = component q&1 of column 2jp + q/2,
    // B[k = q][rhs g], and D[row 8T+g][rhs 2q, 2q+1] (PTX m8n8k4 fragments).
    constexpr int TCT = TC > 0 ? TC : 1;
    double tR[TCT][2], tI[TCT][2];
#pragma unroll
    for (int T = 0; T < TCT; ++T) tR[T][0] = tR[T][1] = tI[T][0] = tI[T][1] = 0.0;
    for (SegIter sg(c0, c1, p); sg.more(); sg.advance(p)) {
      sg.load(p);
      const int s = sg.s;
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* base = stages + (long)s * slot;
      const E* As = reinterpret_cast<const E*>(base + (reinterpret_cast<uintptr_t>(a0) & 15));
      // x slice r starts at its slot + the source's offset within 16 bytes
      const unsigned char* xbase = base + p.a_slot;
      mbar_wait_sleep(&full[s], sg.par);
      if constexpr (TC > 0) {
        static_assert(KX == 8 && KR == 8 && kSplit, "DMMA variant: fp64, exactly 8 right-hand sides");
        const int w = t >> 5, nwp = ncons >> 6;
        const int half = (w >> 2) & 1, wp = (w & 3) + 4 * (w >> 3);
        const int q = lane & 3, g8 = lane >> 2;
        const int cnt = (int)sg.cnt;
        const int npair = (cnt + 1) >> 1;
        const unsigned char* x0 = p.x + (sg.b * p.sx + sg.j) * es;
        const unsigned char* xs = xbase + (reinterpret_cast<uintptr_t>(x0) & 15) + (long)g8 * XR;
#pragma unroll 2
        for (int jp = wp; jp < npair; jp += nwp) {
          const int jj = 2 * jp + (q >> 1);
          const bool vc = jj < cnt;
          const double2 xv = vc ? *reinterpret_cast<const double2*>(xs + jj * 16) : make_double2(0.0, 0.0);
          const double bR = (q & 1) ? -xv.y : xv.x;
          const double bI = (q & 1) ? xv.x : xv.y;
          const double* ac =
              reinterpret_cast<const double*>(As + (long)jj * p.lda + half * TCT * 8) + (q & 1);
          // all tiles' A fragments first, so the shared-load latency is paid
          // once per column pair; the second warp's last tile (rows 8(2TC-1)..)
          // is not live (warp-uniform skip)
          double a[TCT];
#pragma unroll
          for (int T = 0; T < TCT; ++T) {
            const int row = (half * TCT + T) * 8 + g8;
            a[T] = (vc && row < p.m) ? ac[2 * (T * 8 + g8)] : 0.0;
          }
#pragma unroll
          for (int T = 0; T < TCT; ++T) {
            if (T < TCT - 1 || half == 0) {
              dmma_884(tR[T], a[T], bR);
              dmma_884(tI[T], a[T], bI);
            }
          }
        }
      } else if (active && kSplit) {
        if constexpr (kSplit) {
          const int cnt = (int)sg.cnt;
          const E* Xs[KR];
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            const unsigned char* x0 = p.x + (sg.b * p.sx + k * p.sxr + sg.j) * es;
            Xs[k] = reinterpret_cast<const E*>(xbase + k * p.xr_slot + (reinterpret_cast<uintptr_t>(x0) & 15));
          }
          if constexpr (KX > 0 && XR > 0) {
            static_assert(KX == KR, "exact-K variant");
            // double2 slices are 16-byte aligned: Xs[k] = Xs[0] + k*XR
            const unsigned char* xp = reinterpret_cast<const unsigned char*>(Xs[0]) + (long)g * 16;
            const unsigned char* ap = reinterpret_cast<const unsigned char*>(As) + ((long)g * p.lda + r) * 16;
            const long astep = (long)p.G * p.lda * 16;
            const int xstep = p.G * 16;
#pragma unroll(KX >= 8 ? 1 : 2)
            for (int jj = g; jj < cnt; jj += p.G) {
              const double2 a = *reinterpret_cast<const double2*>(ap);
#pragma unroll
              for (int k = 0; k < KX; ++k) {
                const double2 x = *reinterpret_cast<const double2*>(xp + k * XR);
                rr[k] = fma(a.x, x.x, rr[k]);
                ii[k] = fma(a.y, x.y, ii[k]);
                ri[k] = fma(a.x, x.y, ri[k]);
                ir[k] = fma(a.y, x.x, ir[k]);
              }
              ap += astep;
              xp += xstep;
            }
          } else {
            for (int jj = g; jj < cnt; jj += p.G) {
              const double2 a = As[(long)jj * p.lda + r];
#pragma unroll
              for (int k = 0; k < KR; ++k)
                if (k < K) {
                  const double2 x = Xs[k][jj];
                  rr[k] = fma(a.x, x.x, rr[k]);
                  ii[k] = fma(a.y, x.y, ii[k]);
                  ri[k] = fma(a.x, x.y, ri[k]);
                  ir[k] = fma(a.y, x.x, ir[k]);
                }
            }
          }
        }
      } else if (active) {
        const int cnt = (int)sg.cnt;
        Acc part[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) part[k] = kComp ? Tr::zero() : acc[k];
        const E* Xs[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          const unsigned char* x0 = p.x + (sg.b * p.sx + k * p.sxr + sg.j) * es;
          Xs[k] = reinterpret_cast<const E*>(xbase + k * p.xr_slot + (reinterpret_cast<uintptr_t>(x0) & 15));
        }
        for (int jj = g; jj < cnt; jj += p.G) {
          const E a = As[(long)jj * p.lda + r];
#pragma unroll
          for (int k = 0; k < KR; ++k)
            if (k < K) part[k] = Tr::mac(part[k], a, Xs[k][jj]);
        }
#pragma unroll
        for (int k = 0; k < KR; ++k) {
          if constexpr (kComp) neumaier_add(acc[k], cmp[k], part[k]);
          else acc[k] = part[k];
        }
      }
      __syncwarp();
      if (p.arrive_all || lane == 0) mbar_arrive(&empty[s]);
      if (sg.ends_bin(p)) {
        const int KM = K * p.m;
        if constexpr (TC > 0) {
          // the warps' partial sums are added into red in warp order (fixed,
          // so the result is deterministic); p.G == 1 below
          // (warp pair 0 -- warps 0 and 4 -- stores its rows first)
          const int w = t >> 5, nw = ncons >> 5;
          const int half = (w >> 2) & 1, wp = (w & 3) + 4 * (w >> 3);
          const int q = lane & 3, g8 = lane >> 2;
          for (int ww = 0; ww < nw; ++ww) {
            if (w == ww) {
#pragma unroll
              for (int T = 0; T < TCT; ++T) {
                const int row = (half * TCT + T) * 8 + g8;
                if (row < p.m) {
#pragma unroll
                  for (int e = 0; e < 2; ++e) {
                    const int i = (2 * q + e) * p.m + row;
                    const double2 v = make_double2(tR[T][e], tI[T][e]);
                    red[i] = wp == 0 ? v : Tr::add(red[i], v);
                  }
                }
              }
            }
            bar_consumers(ncons);
          }
#pragma unroll
          for (int T = 0; T < TCT; ++T) tR[T][0] = tR[T][1] = tI[T][0] = tI[T][1] = 0.0;
        } else if (active) {
#pragma unroll
          for (int k = 0; k < KR; ++k) {
            if constexpr (kSplit) {
              acc[k] = make_double2(rr[k] - ii[k], ri[k] + ir[k]);
              rr[k] = ii[k] = ri[k] = ir[k] = 0.0;
            }
            if (k < K) red[((long)g * K + k) * p.m + r] = kComp ? Tr::add(acc[k], cmp[k]) : acc[k];
            acc[k] = cmp[k] = Tr::zero();
          }
        }
        bar_consumers(ncons);
        for (int i = t; i < KM; i += ncons) {
          Acc v = red[i];
          for (int gg = 1; gg < p.G; ++gg) v = Tr::add(v, red[(long)gg * KM + i]);
          red[i] = v;
        }
        bar_consumers(ncons);
        const long b = sg.b;
        const long plo = piece_of(b * p.n, p.T, p.P);
        const long phi = piece_of(b * p.n + p.n - 1, p.T, p.P);
        O* yb = reinterpret_cast<O*>(p.y) + b * p.sy;
        auto emit = [&](int i, Acc v) {
          const int k = i / p.m, row = i - k * p.m;
          yb[k * p.syr + row] = out_cast<O>(v);
        };
        if (plo == phi) {
          for (int i = t; i < KM; i += ncons) emit(i, red[i]);
        } else {
          Acc* part = reinterpret_cast<Acc*>(p.partials);
          const long slot_id = (long)blockIdx.x + b;
          for (int i = t; i < KM; i += ncons) part[slot_id * KM + i] = red[i];
          __threadfence();
          bar_consumers(ncons);
          if (t == 0) {
            const unsigned prev = atomicAdd(&p.counters[b], 1u);
            *s_flag = (prev == (unsigned)(phi - plo)) ? 1 : 0;
          }
          bar_consumers(ncons);
          if (*s_flag) {
            __threadfence();
            for (int i = t; i < KM; i += ncons) {
              Acc v = ldcg(part + (plo + b) * KM + i);
              for (long pp = plo + 1; pp <= phi; ++pp) v = Tr::add(v, ldcg(part + (pp + b) * KM + i));
              emit(i, v);
            }
            if (t == 0) p.counters[b] = 0u;
          }
        }
        bar_consumers(ncons);
      }
    }
  } else if constexpr (KX > 0) {
    // ConjTrans, exactly KX right-hand sides, TWO columns per lane: lane
    // (sub, li) takes rows li, li+LPC, ... of columns jb+sub and jb+CPW+sub,
    // so every D_b[i, k] read from shared memory serves two columns. A 128-bit
    // shared load costs four quarter-warp wavefronts whatever its broadcast,
    // and the K x reads were 80 % of the one-column kernel's LSU wavefronts
    // (DESIGN.md §9.1); the host gives this variant fewer consumer warps and
    // stages of 8 columns per warp so every warp has its two columns.
    static_assert(KX == KR, "exact-K variant");
    constexpr int CPW = 32 / LPC;
    const int W = ncons / 32;
    const int w = t >> 5;
    const int sub = lane / LPC;
    const int li = lane - sub * LPC;
    for (SegIter sg(c0, c1, p); sg.more(); sg.advance(p)) {
      sg.load(p);
      const int s = sg.s;
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* base = stages + (long)s * slot;
      const E* As = reinterpret_cast<const E*>(base + (reinterpret_cast<uintptr_t>(a0) & 15));
      const unsigned char* xb = p.xres ? xres_base + (sg.b & 1) * (long)xs_bytes : base + p.a_slot;
      const E* Xs[KX];
#pragma unroll
      for (int k = 0; k < KX; ++k) {
        const unsigned char* x0 = p.x + (sg.b * p.sx + (long)k * p.sxr) * es;
        Xs[k] = reinterpret_cast<const E*>(xb + k * p.xr_slot + (reinterpret_cast<uintptr_t>(x0) & 15));
      }
      O* yb = reinterpret_cast<O*>(p.y) + sg.b * p.sy + sg.j;
      mbar_wait_sleep(&full[s], sg.par);
      const int cnt = (int)sg.cnt;
      for (int jb = w * 2 * CPW; jb < cnt; jb += W * 2 * CPW) {
        const int ja = jb + sub, jc = jb + CPW + sub;
        const bool va = ja < cnt, vc = jc < cnt;
        Acc acca[KX], accc[KX];
#pragma unroll
        for (int k = 0; k < KX; ++k) acca[k] = accc[k] = Tr::zero();
        if (va) {
          const E* cola = As + (long)ja * p.lda;
          const E* colc = As + (long)(vc ? jc : ja) * p.lda;  // (a valid column when jc is past the stage)
          for (int i = li; i < p.m; i += LPC) {
            const E a = cola[i], c = colc[i];
#pragma unroll
            for (int k = 0; k < KX; ++k) {
              const E x = Xs[k][i];
              acca[k] = Tr::macc(acca[k], a, x);
              accc[k] = Tr::macc(accc[k], c, x);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < KX; ++k) {
#pragma unroll
          for (int o = LPC >> 1; o > 0; o >>= 1) {
            acca[k] = Tr::add(acca[k], Tr::shfl_xor(acca[k], o));
            accc[k] = Tr::add(accc[k], Tr::shfl_xor(accc[k], o));
          }
        }
#pragma unroll
        for (int k = 0; k < KX; ++k) {
          if (k % LPC == li) {
            if (va) yb[(long)k * p.syr + ja] = out_cast<O>(acca[k]);
            if (vc) yb[(long)k * p.syr + jc] = out_cast<O>(accc[k]);
          }
        }
      }
      __syncwarp();
      if (p.arrive_all || lane == 0) mbar_arrive(&empty[s]);
    }
  } else {
    // LPC lanes per column split its m rows (lane li: rows li, li+LPC, ...);
    // each lane keeps K accumulators, reads A[i, c] once for all K and
    // x_r[i] from the resident slice (a broadcast across the warp's columns);
    // then one xor-shuffle tree per RHS and lane li stores RHS li (and
    // li + LPC, ...).
    constexpr int CPW = 32 / LPC;
    const int W = ncons / 32;
    const int w = t >> 5;
    const int sub = lane / LPC;
    const int li = lane - sub * LPC;
    for (SegIter sg(c0, c1, p); sg.more(); sg.advance(p)) {
      sg.load(p);
      const int s = sg.s;
      const unsigned char* a0 = p.A + (sg.b * p.sa + sg.j * p.lda) * es;
      const unsigned char* base = stages + (long)s * slot;
      const E* As = reinterpret_cast<const E*>(base + (reinterpret_cast<uintptr_t>(a0) & 15));
      const unsigned char* xb = p.xres ? xres_base + (sg.b & 1) * (long)xs_bytes : base + p.a_slot;
      const E* Xs[KR];
#pragma unroll
      for (int k = 0; k < KR; ++k) {
        const int kk = min(k, K - 1);
        const unsigned char* x0 = p.x + (sg.b * p.sx + (long)kk * p.sxr) * es;
        Xs[k] = reinterpret_cast<const E*>(xb + kk * p.xr_slot + (reinterpret_cast<uintptr_t>(x0) & 15));
      }
      O* yb = reinterpret_cast<O*>(p.y) + sg.b * p.sy + sg.j;
      mbar_wait_sleep(&full[s], sg.par);
      const int cnt = (int)sg.cnt;
      for (int jb = w * CPW; jb < cnt; jb += W * CPW) {
        const int jj = jb + sub;
        const bool valid = jj < cnt;
        Acc acc[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) acc[k] = Tr::zero();
        if (valid) {
          const E* col = As + (long)jj * p.lda;
          for (int i = li; i < p.m; i += LPC) {
            const E a = col[i];
#pragma unroll
            for (int k = 0; k < KR; ++k) {
              if (k < K) {
                if constexpr (MODE == GM_C) acc[k] = Tr::macc(acc[k], a, Xs[k][i]);
                else acc[k] = Tr::mac(acc[k], a, Xs[k][i]);
              }
            }
          }
        }
#pragma unroll
        for (int k = 0; k < KR; ++k) {
#pragma unroll
          for (int o = LPC >> 1; o > 0; o >>= 1) acc[k] = Tr::add(acc[k], Tr::shfl_xor(acc[k], o));
        }
        if (valid) {
#pragma unroll
          for (int k = 0; k < KR; ++k)
            if (k < K && k % LPC == li) yb[(long)k * p.syr + jj] = out_cast<O>(acc[k]);
        }
      }
      __syncwarp();
      if (p.arrive_all || lane == 0) mbar_arrive(&empty[s]);
    }
  }
}

}  // namespace fmv
