// v11 ax_helm kernel for large lx (9..16): "line" contractions.
//
// Why a new formulation (profiles/r01_ncu_v4_d1_lx12_*): the
// v4 column walk (thread per (j,i) column, k walked) keeps four rows of the
// derivative matrices (dx[.][i], dy[.][j], dxt[.][i], dyt[.][j]) plus the u
// and ut columns in registers — 168 registers at lx = 12 — and stages all 8
// input fields of an element in shared memory (110 KiB at lx = 12).  Both
// cap the SM at ~2 elements / 10 warps, and each derivative value costs one
// shared-memory load per multiply-add (5,900 wavefronts per element at
// lx = 12, 72% of the SM's shared-memory cycles).
//
// Here every contraction is a 1-D "line" product done by one thread: the
// thread holds one line of its input (LX doubles) and produces the LX
// outputs of that line, out[o] = sum_l M[l][o] in[l], with BOTH matrix
// indices compile-time — so the matrix entry is a constant-bank operand of
// the DFMA / DMUL (the six matrices travel in the kernel parameter block,
// verified against the device arrays by every CTA, see ax_tma2.cuh), and a
// shared-memory load feeds LX multiply-adds instead of one.  Per element
// (LX^2 threads, thread (a, b) = (tid / LX, tid % LX)):
//   1a  r-line  (k=a, j=b): r[k][j][.]  = Dx-line of u row        -> X0
//   1b  s-line  (k=a, i=b): s[k][.][i]  = Dy-line of u (j-line)   -> X1
//   1c  t-line  (j=a, i=b): t[.][j][i]  = Dz-line of the u column (registers)
//   --- barrier
//   combine at (j=a, i=b) for every k: r, s from X0 / X1, t from registers,
//       h1 and G11..G23 straight from HBM (coalesced, L2-prefetched one
//       element ahead — they are read once, so they never touch shared
//       memory); ur -> X0, us -> X1 in place, ut stays in registers
//   --- barrier
//   fast:   2a  (k=a, j=b): X0 row    <- Dxt-line of the ur row (in place)
//           2b  (k=a, i=b): X1 j-line <- Dyt-line of the us j-line (in place)
//           wt = Dzt-line of the ut column (registers)
//           --- barrier;  w = (X0 + X1) + wt at (j=a, i=b), streamed out
//   strict: the reference adds the three stage-2 terms interleaved per l
//           (sem.py:332-335), so stage 2 stays a column walk: thread (j,i)
//           holds dxt[.][i], dyt[.][j] (from the shared copy) and its ut
//           column, reads ur rows / us j-lines from X0 / X1.
// Stage-1 sums (r, s, t each accumulated l-ascending from 0.0) and the
// combine keep the reference association, so strict output is bit-exact.
//
// Shared memory per CTA: u (TMA bulk copy of the element, linear layout, one
// buffer: the copy for the next element is issued right after stage 1, when
// u is dead, and has the combine + stage 2 to land), X0 and X1 (padded row
// stride RS / plane stride PS chosen by a bank-conflict model,
// tools/smem_conflicts.py) and the six matrices: 46 KiB at lx = 12 (v4: 110).
// Registers: two lines (2 LX doubles) + addressing.
#pragma once

#include "ax_tma.cuh"

namespace axb {

template <int LX>
struct LineCfg {
  static constexpr int L2 = LX * LX;
  static constexpr int L3 = LX * LX * LX;
  static constexpr int NT = L2;
  // X0 / X1 layout [k][j][i]: row stride RS, plane stride PS (doubles);
  // minimises the wavefronts of the row (r-line), j-line (s-line) and
  // column (combine) access patterns (LDS.64 / STS.64)
  static constexpr int RS = LX == 10 ? 10 : (LX == 12 || LX == 14 || LX == 16) ? LX + 1 : LX;
  static constexpr int PP = LX == 10 ? 1 : LX == 13 ? 4 : 0;
  static constexpr int PS = LX * RS + PP;
  static constexpr int XS = (LX * PS + 1) & ~1;      // doubles per X buffer (16-B multiple)
  static constexpr int US = (L3 + 2 + 1) & ~1;       // u buffer: a leading pad double + tail
  static constexpr size_t SMEM = 128 + sizeof(double) * (US + 2 * XS);
};

template <int LX>
struct LParams {
  AxPtrs A;
  int64_t nel;
  int* stale;                 // mapped host flag, set when the host matrix copy is stale
  int pf;                     // L2 prefetch point override (-1: LineGP<LX, FAST>::PF)
  double m[6][LX * LX];       // dx, dy, dz, dxt, dyt, dzt, row-major [l][o]
};

// Per-lx tuning (same-box A/B, tools/sweep.py): GP = planes of geometry (7
// doubles each) in flight in registers ahead of the combine, MINB = ptxas
// minimum-CTAs hint (register budget), PF = L2 prefetch point of the
// geometry (0 none, 1 after the combine for the CTA's next element, 2 at
// element start for the element itself, 3 after stage 1 for the next
// element).  AXL_* macros override every lx (variant builds for A/B).
template <int LX, bool FAST>
struct LineGP {
#ifdef AXL_GP_FAST
  static constexpr int GF = AXL_GP_FAST;
#else
  static constexpr int GF = LX == 11 ? 6 : LX <= 12 ? 4 : 2;
#endif
#ifdef AXL_GP_STRICT
  static constexpr int GS = AXL_GP_STRICT;
#else
  static constexpr int GS = LX <= 12 ? 4 : 2;
#endif
#ifdef AXL_MINB_FAST
  static constexpr int MF = AXL_MINB_FAST;
#else
  static constexpr int MF = LX <= 12 ? 3 : 0;
#endif
#ifdef AXL_MINB_STRICT
  static constexpr int MS = AXL_MINB_STRICT;
#else
  static constexpr int MS = 0;
#endif
  static constexpr int G0 = FAST ? GF : GS;
  static constexpr int GP = G0 < LX ? G0 : LX;
  static constexpr int MINB = FAST ? MF : MS;
  static constexpr int PF = FAST ? (LX <= 11 ? 0 : LX == 12 || LX == 16 ? 2 : 1)
                                 : (LX == 9 || LX == 12) ? 0 : (LX == 11 || LX == 15) ? 1 : 2;
};

__device__ __forceinline__ const double* mat_ptr(const AxPtrs& A, int mi) {
  return mi == 0 ? A.dx : mi == 1 ? A.dy : mi == 2 ? A.dz : mi == 3 ? A.dxt : mi == 4 ? A.dyt : A.dzt;
}

// matrix entry M_mi[l][o]: kernel parameter (constant bank) or, when the
// parameter copy failed verification, the device array (warp-uniform load)
template <int LX, bool UP>
__device__ __forceinline__ double mat(const LParams<LX>& P, int mi, int l, int o) {
  if constexpr (UP) return P.m[mi][l * LX + o];
  else return __ldg(mat_ptr(P.A, mi) + l * LX + o);
}

// out[o] = sum_l M_mi[l][o] in[l], l ascending from 0.0 (reference order)
template <int LX, bool FAST, bool UP>
__device__ __forceinline__ void line(const LParams<LX>& P, int mi,
                                     const double (&in)[LX], double (&out)[LX]) {
#pragma unroll
  for (int o = 0; o < LX; ++o) out[o] = 0.0;
#pragma unroll
  for (int l = 0; l < LX; ++l)
#pragma unroll
    for (int o = 0; o < LX; ++o) out[o] = madd<FAST>(out[o], mat<LX, UP>(P, mi, l, o), in[l]);
}

// Thread 0: start the bulk copy of element e's u into U (16-B aligned
// superset, data `pad` doubles in).  Returns false when the superset would
// read past the array (the consumers then load the element themselves).
template <int LX>
__device__ __forceinline__ void issue_u(const AxPtrs& A, int64_t nel, int64_t e, double* U, uint64_t* bar) {
  constexpr int64_t L3 = LX * LX * LX;
  const int64_t first = e * L3;
  const int64_t lo = first & ~(int64_t)1, hi = (first + L3 + 1) & ~(int64_t)1;
  if (hi > nel * L3) {
    mbar_arrive(bar);
    return;
  }
  const uint32_t bytes = (uint32_t)((hi - lo) * 8);
  mbar_arrive_expect_tx(bar, bytes);
  bulk_g2s(U, A.u + lo, bytes, bar);
}

template <int LX>
__device__ __forceinline__ void prefetch_geom(const AxPtrs& A, int64_t e, int f) {
  constexpr int64_t L3 = LX * LX * LX;
  // fields 1..7 of AxPtrs order (h1, g11, g22, g33, g12, g13, g23)
  uintptr_t lo = (uintptr_t)(field_ptr(A, f) + e * L3);
  uintptr_t hi = (uintptr_t)(field_ptr(A, f) + (e + 1) * L3);
  lo = (lo + 15) & ~(uintptr_t)15;
  hi = hi & ~(uintptr_t)15;
  while (hi > lo) {
    const uint32_t n = (uint32_t)((hi - lo) > 65536 ? 65536 : (hi - lo));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((const void*)lo), "r"(n) : "memory");
    lo += n;
  }
}

// One element.  The u buffer is re-armed for the CTA's next element right
// after stage 1 (inside, thread 0), the geometry of the element after that
// is L2-prefetched at the same point.
template <int LX, bool FAST, bool UP>
__device__ __forceinline__ void element_line(const LParams<LX>& P, const double* Uv,
                                             double* X0, double* X1, int64_t e, int a, int b,
                                             uint64_t* bar, double* Ubuf) {
  using C = LineCfg<LX>;
  constexpr int L2 = C::L2, L3 = C::L3, RS = C::RS, PS = C::PS;
  const AxPtrs& A = P.A;
  const int tid = threadIdx.x;
  const int64_t stride = gridDim.x;

  const int pf = P.pf >= 0 ? P.pf : LineGP<LX, FAST>::PF;
  if (pf == 2 && tid >= 1 && tid <= 7) prefetch_geom<LX>(A, e, tid);
  // ---- stage 1
  double t[LX];
  {
    double in[LX], out[LX];
    // 1a: r-line (k = a, j = b)
#pragma unroll
    for (int l = 0; l < LX; ++l) in[l] = Uv[a * L2 + b * LX + l];
    line<LX, FAST, UP>(P, 0, in, out);
#pragma unroll
    for (int i = 0; i < LX; ++i) X0[a * PS + b * RS + i] = out[i];
    // 1b: s-line (k = a, i = b)
#pragma unroll
    for (int l = 0; l < LX; ++l) in[l] = Uv[a * L2 + l * LX + b];
    line<LX, FAST, UP>(P, 1, in, out);
#pragma unroll
    for (int j = 0; j < LX; ++j) X1[a * PS + j * RS + b] = out[j];
    // 1c: t-line (j = a, i = b)
#pragma unroll
    for (int l = 0; l < LX; ++l) in[l] = Uv[l * L2 + a * LX + b];
    line<LX, FAST, UP>(P, 2, in, t);
  }
  // geometry of the first GP planes: loads in flight across the barrier
  constexpr int GP = LineGP<LX, FAST>::GP;
  const int64_t gbase = e * L3 + a * LX + b;
  double gv[GP][7];
#pragma unroll
  for (int p = 0; p < GP; ++p) {
#pragma unroll
    for (int f = 0; f < 7; ++f) gv[p][f] = ldg_stream(field_ptr(A, f + 1) + gbase + p * L2);
  }
  __syncthreads();  // X0 = r, X1 = s complete; u is dead
  if (tid == 0 && e + stride < P.nel) {
    fence_proxy_async();
    issue_u<LX>(A, P.nel, e + stride, Ubuf, bar);
  }
  if (pf == 3 && tid >= 1 && tid <= 7 && e + stride < P.nel) prefetch_geom<LX>(A, e + stride, tid);

  // ---- combine at (j = a, i = b); plane k + GP's geometry is loaded as
  // plane k's is consumed
  const int xb = a * RS + b;
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    double* g = gv[k % GP];
    const double h = g[0], a11 = g[1], a22 = g[2], a33 = g[3], a12 = g[4], a13 = g[5], a23 = g[6];
    if (k + GP < LX) {
#pragma unroll
      for (int f = 0; f < 7; ++f) g[f] = ldg_stream(field_ptr(A, f + 1) + gbase + (k + GP) * L2);
    }
    const double r = X0[k * PS + xb], s = X1[k * PS + xb];
    X0[k * PS + xb] = combine<FAST>(h, a11, a12, a13, r, s, t[k]);  // ur
    X1[k * PS + xb] = combine<FAST>(h, a12, a22, a23, r, s, t[k]);  // us
    t[k] = combine<FAST>(h, a13, a23, a33, r, s, t[k]);              // ut
  }
  if (pf == 1 && tid >= 1 && tid <= 7 && e + stride < P.nel) prefetch_geom<LX>(A, e + stride, tid);

  double* wout = A.w + gbase;
  if constexpr (FAST) {
    double wt[LX];
    line<LX, FAST, UP>(P, 5, t, wt);
    __syncthreads();  // ur / us complete
    {
      double in[LX], out[LX];
      // 2a: (k = a, j = b), ur row -> Dxt-line, in place
#pragma unroll
      for (int l = 0; l < LX; ++l) in[l] = X0[a * PS + b * RS + l];
      line<LX, FAST, UP>(P, 3, in, out);
#pragma unroll
      for (int i = 0; i < LX; ++i) X0[a * PS + b * RS + i] = out[i];
      // 2b: (k = a, i = b), us j-line -> Dyt-line, in place
#pragma unroll
      for (int l = 0; l < LX; ++l) in[l] = X1[a * PS + l * RS + b];
      line<LX, FAST, UP>(P, 4, in, out);
#pragma unroll
      for (int j = 0; j < LX; ++j) X1[a * PS + j * RS + b] = out[j];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < LX; ++k) stg_stream(wout + k * L2, (X0[k * PS + xb] + X1[k * PS + xb]) + wt[k]);
  } else {
    __syncthreads();  // ur / us complete
    double dxtr[LX], dytr[LX];
#pragma unroll
    for (int l = 0; l < LX; ++l) {
      dxtr[l] = __ldg(A.dxt + l * LX + b);
      dytr[l] = __ldg(A.dyt + l * LX + a);
    }
#pragma unroll
    for (int k = 0; k < LX; ++k) {
      double w = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        w = madd<false>(w, dxtr[l], X0[k * PS + a * RS + l]);
        w = madd<false>(w, dytr[l], X1[k * PS + l * RS + b]);
        w = madd<false>(w, mat<LX, UP>(P, 5, l, k), t[l]);
      }
      stg_stream(wout + k * L2, w);
    }
  }
}


template <int LX, bool FAST>
__global__ void __launch_bounds__(LineCfg<LX>::NT, LineGP<LX, FAST>::MINB)
ax_line(const __grid_constant__ LParams<LX> P) {
  using C = LineCfg<LX>;
  constexpr int L2 = C::L2, L3 = C::L3, RS = C::RS, PS = C::PS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
  double* U = reinterpret_cast<double*>(smem_raw + 128);
  double* X0 = U + C::US;
  double* X1 = X0 + C::XS;

  const AxPtrs& A = P.A;
  const int64_t nel = P.nel;
  const int tid = threadIdx.x;
  const int a = tid / LX, b = tid - (tid / LX) * LX;
  const int64_t stride = gridDim.x;

  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0 && (int64_t)blockIdx.x < nel) issue_u<LX>(A, nel, blockIdx.x, U, bar);
  const int pf = P.pf >= 0 ? P.pf : LineGP<LX, FAST>::PF;
  if ((pf == 1 || pf == 3) && tid >= 1 && tid <= 7 && (int64_t)blockIdx.x < nel)
    prefetch_geom<LX>(A, blockIdx.x, tid);
  // verification of the parameter copy against the device arrays
  int bad = 0;
  for (int q = tid; q < 6 * L2; q += C::NT) {
    const int mi = q / L2, r = q - mi * L2;
    bad |= __double_as_longlong(__ldg(mat_ptr(A, mi) + r)) != __double_as_longlong(P.m[mi][r]);
  }
  const bool use_param = !__syncthreads_or(bad);
  if (!use_param && tid == 0 && P.stale) *(volatile int*)P.stale = 1;

  uint32_t parity = 0;
  for (int64_t e = blockIdx.x; e < nel; e += stride, parity ^= 1u) {
    mbar_wait(bar, parity);
    const int64_t first = e * L3;
    int pad = (int)(first & 1);
    if ((((first + L3 + 1) & ~(int64_t)1)) > nel * L3) {  // fallback: load it ourselves
      pad = 0;
      for (int q = tid; q < L3; q += C::NT) U[q] = A.u[first + q];
      __syncthreads();
    }
    if (use_param) element_line<LX, FAST, true>(P, U + pad, X0, X1, e, a, b, bar, U);
    else element_line<LX, FAST, false>(P, U + pad, X0, X1, e, a, b, bar, U);
    __syncthreads();  // X0 / X1 free for the next element
  }
}

}  // namespace axb
