// ax_helm element kernels for sm_100a (B200), FP64.
//
// Operator (reference: /root/reference/pkg/src/mdg/sem.py:300-337, tasklets
// axprogram.py:159-163 stage 1, :188-192 combine, :229 stage 2):
//
//   r[e,k,j,i] = sum_l dxd[l,i] u[e,k,j,l]     s = sum_l dyd[l,j] u[e,k,l,i]
//   t[e,k,j,i] = sum_l dzd[l,k] u[e,l,j,i]
//   ur = h1 ((g11 r + g12 s) + g13 t)  us = h1 ((g12 r + g22 s) + g23 t)
//   ut = h1 ((g13 r + g23 s) + g33 t)
//   w[e,k,j,i] = sum_l ((dxtd[l,i] ur[e,k,j,l] + dytd[l,j] us[e,k,l,i]) + dztd[l,k] ut[e,l,j,i])
//                (accumulated term by term, l ascending, from 0.0)
//
// Layout in HBM: every field is [nel][lx][lx][lx] row-major, i fastest
// (sem.py:68-100); the six matrices are [lx][lx] row-major.
//
// Two arithmetic modes, chosen at compile time:
//   Strict (FAST=false): every multiply and add is a separate IEEE-754
//     round-to-nearest operation (__dmul_rn / __dadd_rn) in exactly the
//     reference's association, so the output is bit-identical to
//     mdg.sem.ax_reference and to the reference's strict-fp compiled kernel.
//   Fast (FAST=true): the same sums with fused multiply-adds; differs from
//     the reference by FP64 reassociation only (<= 1e-12 normwise).
//
// Thread mapping ("k-walk"): one thread per (j,i) column of an element; the
// thread walks k.  Its u column and its ut column stay in registers, the
// element's u and the ur/us slices live in shared memory (row stride padded
// to an odd number of doubles so the row-broadcast reads hit distinct
// banks).  EPB elements share one CTA so the CTA has >= ~128 threads for
// every lx.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace axb {

struct AxPtrs {
  double* __restrict__ w;
  const double* __restrict__ u;
  const double* __restrict__ dx;
  const double* __restrict__ dy;
  const double* __restrict__ dz;
  const double* __restrict__ dxt;
  const double* __restrict__ dyt;
  const double* __restrict__ dzt;
  const double* __restrict__ h1;
  const double* __restrict__ g11;
  const double* __restrict__ g22;
  const double* __restrict__ g33;
  const double* __restrict__ g12;
  const double* __restrict__ g13;
  const double* __restrict__ g23;
};

// Per-call extensions honoured by the lx = 8 DMMA kernel only (kept out of
// AxPtrs: growing the vector kernels' parameter block shifted ptxas's
// register allocation and cost up to 35% at lx = 10).
struct AxExt {
  // 1: the caller reads w again soon (layer-blocked ax + DSSUM): inputs are
  // loaded L2 evict-first and w is stored evict-normal so it stays in L2;
  // 0 (default): w is streamed out evict-first.
  int keep_w = 0;
  // > 0 (DMMA kernel only): elements form x-runs of this length (box mesh,
  // e = (ez ny + ey) nx + ex) and each CTA takes one contiguous element
  // segment, summing the x-face nodes shared by consecutive elements of a
  // run (the DSSUM's class-2 nodes) in its epilogue — see ax_dmma8
  int xrun = 0;
  // optional completion counters for a concurrent consumer (the DSSUM
  // follower, mesh_gs.cu): after an element's w is stored, progress[e / lay]
  // is incremented with release semantics at gpu scope
  unsigned* progress = nullptr;
  int64_t lay = 0;
};

// Thread 0, after a __syncthreads that follows every thread's w stores of
// elements [e0, e0 + ne): publish them (the CUTLASS semaphore pattern: the
// barrier orders the CTA's stores before thread 0's release).
__device__ __forceinline__ void signal_done(const AxExt& X, int64_t e0, int64_t ne) {
  const int64_t end = e0 + ne;
  for (int64_t e = e0; e < end;) {
    const int64_t L = e / X.lay;
    const int64_t stop = (L + 1) * X.lay < end ? (L + 1) * X.lay : end;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(X.progress + L), "r"((unsigned)(stop - e))
                 : "memory");
    e = stop;
  }
}

template <int LX>
struct KCfg {
  static constexpr int L2 = LX * LX;
  static constexpr int L3 = LX * LX * LX;
  // elements per CTA: aim for ~128 threads, at least one element
  static constexpr int EPB = (L2 >= 128) ? 1 : (128 / L2);
  static constexpr int NT = EPB * L2;
  static constexpr int RS = LX | 1;        // padded row stride (doubles)
  static constexpr int SL = LX * RS;       // slice stride
  static constexpr int ES = LX * SL;       // element stride in smem
  static constexpr size_t SMEM = sizeof(double) * (6 * L2 + 3 * EPB * ES);
};

// acc + a*b with the requested rounding discipline
template <bool FAST>
__device__ __forceinline__ double madd(double acc, double a, double b) {
  if constexpr (FAST) {
    return fma(a, b, acc);
  } else {
    return __dadd_rn(acc, __dmul_rn(a, b));
  }
}

// h * ((ga*r + gb*s) + gc*t)
template <bool FAST>
__device__ __forceinline__ double combine(double h, double ga, double gb, double gc,
                                          double r, double s, double t) {
  if constexpr (FAST) {
    return h * fma(gc, t, fma(gb, s, ga * r));
  } else {
    return __dmul_rn(h, __dadd_rn(__dadd_rn(__dmul_rn(ga, r), __dmul_rn(gb, s)),
                                  __dmul_rn(gc, t)));
  }
}

__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void stg_stream(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// L2 cache policies (createpolicy): the TMA input stream and the w stores.
struct L2Pol {
  uint64_t in, w;
  bool keep;
};
__device__ __forceinline__ L2Pol make_l2pol(int keep_w) {
  L2Pol P;
  P.keep = keep_w != 0;
  if (P.keep) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(P.in));
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(P.w));
  } else {
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(P.in));
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(P.w));
  }
  return P;
}
// w store with the policy's L2 hint (evict-first = streamed, or evict-normal
// when w is read again soon); no branch, the policy is a register operand
__device__ __forceinline__ void stg_w(double* p, double v, const L2Pol& P) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(P.w) : "memory");
}
__device__ __forceinline__ void stg_w2(double* p, double v0, double v1, const L2Pol& P) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v0), "d"(v1), "l"(P.w)
               : "memory");
}

}  // namespace axb

namespace axb {

// ---------------------------------------------------------------------------
// v2: persistent k-walk with group-ahead TMA L2 prefetch.
//
// v1 is latency-bound (ncu: long-scoreboard stalls, 31% occupancy at 96
// regs, DRAM 51% busy): the geometric factors are loaded into registers,
// so bytes in flight are capped by registers x warps.  v2 keeps the same
// arithmetic but makes each CTA persistent over element groups and, while
// it computes group g, has 8 threads issue `cp.async.bulk.prefetch.L2` (the
// TMA engine: no registers, no shared memory) for all 8 input fields of
// the group it processes PF_DIST groups later.  The DRAM stream is then
// driven by the TMA unit ahead of the compute, whose LDGs hit L2.
//
// Shared-memory layout for LX = 8 / 16 is unpadded with an XOR swizzle of
// the column by the row (col ^ swz(j)), which makes the row-broadcast reads
// of stage 1 and 2 conflict-free without the store conflicts padding causes.
// ---------------------------------------------------------------------------

template <int LX>
struct SCfg {
  static constexpr bool SWZ = (LX == 8 || LX == 16);
  static constexpr int L2 = LX * LX;
  static constexpr int L3 = LX * LX * LX;
  static constexpr int EPB = KCfg<LX>::EPB;
  static constexpr int NT = EPB * L2;
  static constexpr int RS = SWZ ? LX : (LX | 1);
  static constexpr int SL = LX * RS;
  static constexpr int ES = LX * SL;
  static constexpr size_t SMEM = sizeof(double) * (6 * L2 + 3 * EPB * ES);
  // physical smem index of logical (k, j, i) inside one element
  __device__ static __forceinline__ int idx(int k, int j, int i) {
    if constexpr (LX == 8) {
      return k * SL + j * RS + (i ^ (((j >> 1) & 1) << 2));
    } else if constexpr (LX == 16) {
      return k * SL + j * RS + (i ^ ((j & 1) << 3));
    } else {
      return k * SL + j * RS + i;
    }
  }
};

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// L2 prefetch of input field f (0..7) of element group g.
template <int LX>
__device__ __forceinline__ void prefetch_group(const AxPtrs& A, int64_t g, int64_t nel, int f) {
  using C = SCfg<LX>;
  const double* base;
  switch (f) {
    case 0: base = A.u; break;
    case 1: base = A.h1; break;
    case 2: base = A.g11; break;
    case 3: base = A.g22; break;
    case 4: base = A.g33; break;
    case 5: base = A.g12; break;
    case 6: base = A.g13; break;
    default: base = A.g23; break;
  }
  const int64_t e0 = g * C::EPB;
  int64_t e1 = e0 + C::EPB;
  if (e1 > nel) e1 = nel;
  if (e0 >= e1) return;
  uintptr_t lo = (uintptr_t)(base + e0 * C::L3);
  uintptr_t hi = (uintptr_t)(base + e1 * C::L3);
  lo = (lo + 15) & ~(uintptr_t)15;  // stay inside the group, 16-B aligned
  hi = hi & ~(uintptr_t)15;
  while (hi > lo) {
    const uint32_t n = (uint32_t)((hi - lo) > 65536 ? 65536 : (hi - lo));
    prefetch_l2((const void*)lo, n);
    lo += n;
  }
}

template <int LX, bool FAST, int PF_DIST>
__global__ void __launch_bounds__(SCfg<LX>::NT)
ax_kwalk_pf(const AxPtrs A, const int64_t nel) {
  using C = SCfg<LX>;
  constexpr int L2 = C::L2, L3 = C::L3, ES = C::ES;
  extern __shared__ double smem[];
  double* sD = smem;
  double* sU = sD + 6 * L2;
  double* sR = sU + C::EPB * ES;
  double* sS = sR + C::EPB * ES;

  const int tid = threadIdx.x;
  const int64_t ngroups = (nel + C::EPB - 1) / C::EPB;
  const int64_t stride = gridDim.x;
  if (tid < 8) {
#pragma unroll
    for (int d = 0; d < PF_DIST; ++d) prefetch_group<LX>(A, blockIdx.x + d * stride, nel, tid);
  }
  for (int q = tid; q < L2; q += C::NT) {
    sD[0 * L2 + q] = A.dx[q];
    sD[1 * L2 + q] = A.dy[q];
    sD[2 * L2 + q] = A.dz[q];
    sD[3 * L2 + q] = A.dxt[q];
    sD[4 * L2 + q] = A.dyt[q];
    sD[5 * L2 + q] = A.dzt[q];
  }
  const int el = tid / L2;
  const int p = tid - el * L2;
  const int j = p / LX;
  const int i = p - j * LX;
  double* eU = sU + el * ES;
  double* eR = sR + el * ES;
  double* eS = sS + el * ES;
  __syncthreads();

  for (int64_t g = blockIdx.x; g < ngroups; g += stride) {
    if (tid < 8) prefetch_group<LX>(A, g + PF_DIST * stride, nel, tid);
    const int64_t e = g * C::EPB + el;
    const bool active = e < nel;
    const int64_t gbase = e * L3 + p;

    double ureg[LX];
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      ureg[k] = active ? ldg_stream(A.u + gbase + k * L2) : 0.0;
      eU[C::idx(k, j, i)] = ureg[k];
    }
    __syncthreads();

    double d1[LX], d2[LX];
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      d1[l] = sD[0 * L2 + l * LX + i];
      d2[l] = sD[1 * L2 + l * LX + j];
    }
    double utr[LX];
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      const int64_t gg = gbase + k * L2;
      double h = 0, a11 = 0, a22 = 0, a33 = 0, a12 = 0, a13 = 0, a23 = 0;
      if (active) {
        h = ldg_stream(A.h1 + gg);
        a11 = ldg_stream(A.g11 + gg);
        a22 = ldg_stream(A.g22 + gg);
        a33 = ldg_stream(A.g33 + gg);
        a12 = ldg_stream(A.g12 + gg);
        a13 = ldg_stream(A.g13 + gg);
        a23 = ldg_stream(A.g23 + gg);
      }
      double r = 0.0, s = 0.0, t = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        r = madd<FAST>(r, d1[l], eU[C::idx(k, j, l)]);
        s = madd<FAST>(s, d2[l], eU[C::idx(k, l, i)]);
        t = madd<FAST>(t, sD[2 * L2 + l * LX + k], ureg[l]);
      }
      eR[C::idx(k, j, i)] = combine<FAST>(h, a11, a12, a13, r, s, t);
      eS[C::idx(k, j, i)] = combine<FAST>(h, a12, a22, a23, r, s, t);
      utr[k] = combine<FAST>(h, a13, a23, a33, r, s, t);
    }
    __syncthreads();

#pragma unroll
    for (int l = 0; l < LX; ++l) {
      d1[l] = sD[3 * L2 + l * LX + i];
      d2[l] = sD[4 * L2 + l * LX + j];
    }
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      double w = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        w = madd<FAST>(w, d1[l], eR[C::idx(k, j, l)]);
        w = madd<FAST>(w, d2[l], eS[C::idx(k, l, i)]);
        w = madd<FAST>(w, sD[5 * L2 + l * LX + k], utr[l]);
      }
      if (active) stg_stream(A.w + gbase + k * L2, w);
    }
    __syncthreads();  // eU/eR/eS are rewritten by the next group
  }
}

}  // namespace axb
