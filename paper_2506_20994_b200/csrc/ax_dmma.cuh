// v6 ax_helm kernel (FAST mode, lx = 8): the six tensor contractions on the
// FP64 tensor cores (DMMA m8n8k4), fed by v3's TMA ring.
//
// Why: at the sustained 1 kW power cap the FP64-vector kernels drop to
// ~1.65 GHz; their ~190 warp-instructions per 32 points (114 of them
// DMUL/DADD or DFMA) are what separates them from the 6.87 TB/s the same
// HBM stream reaches with trivial arithmetic (stream probe, profiles/).
// Every contraction here is a chain of 8x8x4 FP64 MMAs: 96 DMMAs (24,576
// FMAs) per element instead of ~960 DFMA warp-instructions, with the
// matrices' fragments held in registers for the whole persistent CTA.
// FMA-based, so this serves AXHELM_FAST only (<= 1e-12 normwise from the
// reference); strict mode keeps the bit-exact vector kernels.
//
// Per element (u, G, h1 staged by TMA; CTA = 2 warps, warp w owns k-tiles
// {4w..4w+3} and j-tiles {4w..4w+3}); lane (g = lane>>2, q = lane&3):
//   R_k = U_k(j x l) . Dx(l x i)        j-rows tile: lane has (k, g, 2q..2q+1)
//   S_k = Dy^T(j x l) . U_k(l x i)      j-rows tile
//   T_j = Dz^T(k x l) . U_j(l x i)      k-rows tile -> transposed through smem
//   combine (G loaded per own points) -> ur, us, ut
//   W_k  = UR_k . Dxt + Dyt^T . US_k    j-rows tile
//   Wz_j = Dzt^T . UT_j                 k-rows tile -> transposed through smem
// The contraction index l of an MMA step is assigned to lanes as l = 2q+s
// where the A operand is a row of a linear buffer (one 16-B load feeds
// both k-steps) and l = q+4s elsewhere; us / ut are written with XOR
// swizzles that make their fragment loads bank-conflict-free.
#pragma once

#include "ax_tma.cuh"

namespace axb {

struct DmCfg {
  static constexpr int LX = 8, L2 = 64, L3 = 512;
  static constexpr int NT = 64;  // 2 warps
  static constexpr int D = 2;
  static constexpr int FIELD = L3;
  static constexpr int BUF = 8 * FIELD;
  static constexpr size_t SMEM = 128 + sizeof(double) * (D * BUF + L3);
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void sts2(double* p, double x, double y) {
  *reinterpret_cast<double2*>(p) = make_double2(x, y);
}

// US layout: [k][row l][col i], col ^= 4 * ((l >> 1) & 1)
__device__ __forceinline__ int us_idx(int k, int l, int i) { return k * 64 + l * 8 + (i ^ (((l >> 1) & 1) << 2)); }
// UT layout: [l][j][i], row j ^= (l & 1), col ^= 4 * ((l >> 1) & 1)
__device__ __forceinline__ int ut_idx(int l, int j, int i) {
  return l * 64 + ((j ^ (l & 1)) << 3) + (i ^ (((l >> 1) & 1) << 2));
}

// DOT: also accumulate sum_p u_p w_p over the CTA's elements (in a fixed
// order) into dot_partial[blockIdx.x] — the PCG's <p, A p> without a pass.
//
// XF (X.xrun = nx > 0, box-mesh layers): the CTA walks one contiguous
// segment of elements instead of a grid stride, so consecutive elements of
// an x-run pass through it in order, and it sums the x-face nodes they share
// — the nodes that lie on no y or z element face (rows j, k in 1..lx-2),
// i.e. exactly the local DSSUM's class-2 nodes (mesh_gs.cu) — in the
// epilogue: the i = 7 column of element e-1 stays in a register of lane
// q = 3, is shuffled to lane q = 0 of element e, and both copies receive
// (0.0 + w[e-1]) + w[e], the DSSUM's ascending-copy sum, bit for bit.  The
// faces at segment seams are summed by xfold_seams afterwards.  The DSSUM
// pass then skips class 2, the half of its time that is sector-bound.
template <bool DOT, bool XF = false>
__global__ void __launch_bounds__(DmCfg::NT)
ax_dmma8(const AxPtrs A, const int64_t nel, double* __restrict__ dot_partial, const AxExt X) {
  using C = DmCfg;
  constexpr int FIELD = C::FIELD;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* bufs = reinterpret_cast<double*>(smem_raw + 128);
  double* ST = bufs + C::D * C::BUF;  // transpose scratch [k][j][i]

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;
  const int g = lane >> 2, q = lane & 3;
  const int64_t stride = gridDim.x;
  const L2Pol pol = make_l2pol(X.keep_w);
  // element walk: grid stride, or (XF) one contiguous segment per CTA
  int64_t e_begin = blockIdx.x, e_end = nel, e_step = stride;
  if constexpr (XF) {
    const int64_t seg = (nel + stride - 1) / stride;
    e_begin = (int64_t)blockIdx.x * seg;
    e_end = e_begin + seg < nel ? e_begin + seg : nel;
    e_step = 1;
  }

  if (tid == 0) {
    for (int d = 0; d < C::D; ++d) mbar_init(&bars[d], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int d = 0; d < C::D; ++d) {
      const int64_t e = e_begin + d * e_step;
      if (e < e_end) issue_group<8>(A, nel, e, bufs + d * C::BUF, &bars[d], pol.in);
    }

  // matrix fragments, fixed for the whole CTA
  //  R:  B[l][i]      = dx[l][i],     l = 2q+s, i = g
  //  S:  A[j][l]      = dy[l][j],     l = q+4s, j = g
  //  T:  A[k][l]      = dz[l][k],     l = q+4s, k = g
  //  x:  B[l][i]      = dxt[l][i],    l = 2q+s, i = g
  //  y:  A[j][l]      = dyt[l][j],    l = q+4s, j = g
  //  z:  A[k][l]      = dzt[l][k],    l = q+4s, k = g
  double fx[2], fy[2], fz[2], fxt[2], fyt[2], fzt[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    fx[s] = A.dx[(2 * q + s) * 8 + g];
    fy[s] = A.dy[(q + 4 * s) * 8 + g];
    fz[s] = A.dz[(q + 4 * s) * 8 + g];
    fxt[s] = A.dxt[(2 * q + s) * 8 + g];
    fyt[s] = A.dyt[(q + 4 * s) * 8 + g];
    fzt[s] = A.dzt[(q + 4 * s) * 8 + g];
  }

  double dot_acc = 0.0;
  double carry[4] = {0.0, 0.0, 0.0, 0.0};  // XF: deferred i = 7 values (lane q = 3)
  int64_t n = 0;
  for (int64_t e = e_begin; e < e_end; e += e_step, ++n) {
    const int b = (int)(n % C::D);
    double* buf = bufs + b * C::BUF;
    mbar_wait(&bars[b], (uint32_t)((n / C::D) & 1));
    double* U = buf;
    double* H = buf + 1 * FIELD;
    double* G11 = buf + 2 * FIELD;
    double* G22 = buf + 3 * FIELD;
    double* G33 = buf + 4 * FIELD;
    double* G12 = buf + 5 * FIELD;
    double* G13 = buf + 6 * FIELD;
    double* G23 = buf + 7 * FIELD;

    // ---- phase A: derivatives
    double r[4][2], sd[4][2], tt[4][2];
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const int k = warp * 4 + kt;
      r[kt][0] = r[kt][1] = 0.0;
      sd[kt][0] = sd[kt][1] = 0.0;
      const double2 a = lds2(U + k * 64 + g * 8 + 2 * q);  // U[k][g][2q], [2q+1]
      dmma(r[kt][0], r[kt][1], a.x, fx[0]);
      dmma(r[kt][0], r[kt][1], a.y, fx[1]);
#pragma unroll
      for (int s = 0; s < 2; ++s)
        dmma(sd[kt][0], sd[kt][1], fy[s], U[k * 64 + (q + 4 * s) * 8 + g]);
    }
#pragma unroll
    for (int jt = 0; jt < 4; ++jt) {
      const int j = warp * 4 + jt;
      tt[jt][0] = tt[jt][1] = 0.0;
#pragma unroll
      for (int s = 0; s < 2; ++s)
        dmma(tt[jt][0], tt[jt][1], fz[s], U[(q + 4 * s) * 64 + j * 8 + g]);
      sts2(ST + g * 64 + j * 8 + 2 * q, tt[jt][0], tt[jt][1]);  // T[k=g][j][2q..]
    }
    __syncthreads();  // T complete

    // ---- phase B: combine at the own points (k, g, 2q..2q+1)
    double ur[4][2], us[4][2], ut[4][2];
    double uown[4][2];  // DOT: u at the own points (U is overwritten below)
    if constexpr (DOT) {
#pragma unroll
      for (int kt = 0; kt < 4; ++kt) {
        const double2 uu = lds2(U + (warp * 4 + kt) * 64 + g * 8 + 2 * q);
        uown[kt][0] = uu.x;
        uown[kt][1] = uu.y;
      }
    }
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const int k = warp * 4 + kt;
      const int o = k * 64 + g * 8 + 2 * q;
      const double2 t2 = lds2(ST + o);
      const double2 h = lds2(H + o), a11 = lds2(G11 + o), a22 = lds2(G22 + o), a33 = lds2(G33 + o);
      const double2 a12 = lds2(G12 + o), a13 = lds2(G13 + o), a23 = lds2(G23 + o);
      const double tv[2] = {t2.x, t2.y};
      const double hv[2] = {h.x, h.y}, v11[2] = {a11.x, a11.y}, v22[2] = {a22.x, a22.y};
      const double v33[2] = {a33.x, a33.y}, v12[2] = {a12.x, a12.y}, v13[2] = {a13.x, a13.y};
      const double v23[2] = {a23.x, a23.y};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double rr = r[kt][c], ss = sd[kt][c], tv_ = tv[c];
        ur[kt][c] = hv[c] * fma(v13[c], tv_, fma(v12[c], ss, v11[c] * rr));
        us[kt][c] = hv[c] * fma(v23[c], tv_, fma(v22[c], ss, v12[c] * rr));
        ut[kt][c] = hv[c] * fma(v33[c], tv_, fma(v23[c], ss, v13[c] * rr));
      }
    }
    __syncthreads();  // every read of U, G and ST is done: regions are reused below
    double* UR = U;    // [k][j][l] linear
    double* US = G11;  // us_idx layout
    double* UT = G22;  // ut_idx layout
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const int k = warp * 4 + kt;
      sts2(UR + k * 64 + g * 8 + 2 * q, ur[kt][0], ur[kt][1]);
      sts2(US + us_idx(k, g, 2 * q), us[kt][0], us[kt][1]);
      sts2(UT + ut_idx(k, g, 2 * q), ut[kt][0], ut[kt][1]);
    }
    __syncthreads();

    // ---- phase C: stage 2
    double w[4][2];
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const int k = warp * 4 + kt;
      w[kt][0] = w[kt][1] = 0.0;
      const double2 a = lds2(UR + k * 64 + g * 8 + 2 * q);  // UR[k][g][2q], [2q+1]
      dmma(w[kt][0], w[kt][1], a.x, fxt[0]);
      dmma(w[kt][0], w[kt][1], a.y, fxt[1]);
#pragma unroll
      for (int s = 0; s < 2; ++s) dmma(w[kt][0], w[kt][1], fyt[s], US[us_idx(k, q + 4 * s, g)]);
    }
#pragma unroll
    for (int jt = 0; jt < 4; ++jt) {
      const int j = warp * 4 + jt;
      double z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int s = 0; s < 2; ++s) dmma(z0, z1, fzt[s], UT[ut_idx(q + 4 * s, j, g)]);
      sts2(ST + g * 64 + j * 8 + 2 * q, z0, z1);  // Wz[k=g][j][2q..]
    }
    __syncthreads();
    double* wout = A.w + e * C::L3;
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
      const int k = warp * 4 + kt;
      const int o = k * 64 + g * 8 + 2 * q;
      const double2 z = lds2(ST + o);
      double w0 = w[kt][0] + z.x;
      const double w1 = w[kt][1] + z.y;
      if constexpr (DOT) dot_acc = fma(uown[kt][0], w0, fma(uown[kt][1], w1, dot_acc));
      if constexpr (XF) {
        const int64_t ex = e % X.xrun;
        const bool row_in = k >= 1 && k <= 6 && g >= 1 && g <= 6;
        const double prev = __shfl_sync(0xffffffffu, carry[kt], lane | 3);
        if (q == 0 && row_in && ex > 0 && e > e_begin) {  // (k, g, 0) of e = (k, g, 7) of e-1
          w0 = __dadd_rn(__dadd_rn(0.0, prev), w0);
          stg_w(wout - C::L3 + o + 7, w0, pol);
        }
        if (q == 3 && row_in && ex < X.xrun - 1 && e + 1 < e_end) {  // deferred to element e+1
          carry[kt] = w1;
          stg_w(wout + o, w0, pol);
        } else {
          stg_w2(wout + o, w0, w1, pol);
        }
      } else {
        stg_w2(wout + o, w0, w1, pol);
      }
    }
    __syncthreads();  // buffer b and ST free
    if (tid == 0) {
      if (X.progress) signal_done(X, e, 1);
      const int64_t en = e + C::D * e_step;
      if (en < e_end) {
        fence_proxy_async();
        issue_group<8>(A, nel, en, buf, &bars[b], pol.in);
      }
    }
  }
  if constexpr (DOT) {
    // fixed-order CTA reduction of the per-thread sums
    double* red = ST;  // free after the loop
    __syncthreads();
    red[tid] = dot_acc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q2 = 0; q2 < C::NT; ++q2) t += red[q2];
      dot_partial[blockIdx.x] = t;
    }
  }
}

// XF seams: the x-face shared by the last element of one CTA's segment and
// the first of the next (same x-run), class-2 rows only; one CTA per seam.
__global__ void __launch_bounds__(64) xfold_seams(double* __restrict__ w, const int64_t nel,
                                                  const int64_t seg, const int xrun) {
  const int64_t a = ((int64_t)blockIdx.x + 1) * seg;
  if (a >= nel || a % xrun == 0) return;
  const int k = threadIdx.x >> 3, j = threadIdx.x & 7;
  if (k < 1 || k > 6 || j < 1 || j > 6) return;
  double* p = w + a * DmCfg::L3 + k * 64 + j * 8;
  const double s = __dadd_rn(__dadd_rn(0.0, p[7 - DmCfg::L3]), p[0]);
  p[7 - DmCfg::L3] = s;
  p[0] = s;
}

}  // namespace axb
