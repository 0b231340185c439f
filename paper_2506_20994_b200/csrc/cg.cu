// Jacobi-preconditioned CG building blocks for the assembled SEM Poisson
// operator (config C5).  No reference implementation:
// the solve is a reference non-goal; the weak form is
// PAPER.md:126-130.  Parity: oracle/oracle.py (NumPy PCG, same algorithm).
//
// Every kernel is a single fused pass over the local points; scalars (alpha,
// beta) are read from DEVICE memory, so an iteration needs no host round
// trip (graph-capturable; multi-GPU sums via NCCL all-reduce of the scalar
// slots).  Reductions are deterministic: grid-stride partials per block in
// a fixed order, then one block sums the partials in a fixed tree.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "../../include/axhelm.h"
#include "ax_launch.h"
#include "box_gs.cuh"

namespace {
// CG step ratios with exact convergence handled: when the solve has
// converged to an exactly zero residual (tiny problems), p.Ap or rz becomes
// 0 and the textbook a / b would turn x into NaN; the step is 0 instead, so
// further iterations leave x unchanged.
__device__ __forceinline__ double cg_ratio(double a, double b) { return b != 0.0 ? a / b : 0.0; }
}  // namespace

namespace axb {

constexpr int RT = 256;  // reduction block size

__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int s = RT / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// partial[NQ*blockIdx.x + q] for q < NQ
template <int NQ>
__device__ __forceinline__ void write_partials(const double (&v)[NQ], double* partial) {
  __shared__ double sh[RT];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double s = block_sum(v[q], sh);
    if (threadIdx.x == 0) partial[NQ * blockIdx.x + q] = s;
  }
}

// out[q] = sum_b partial[NQ*b + q]  (one block, fixed order)
__global__ void reduce_partials_kernel(const double* __restrict__ partial, int nblocks, int nq,
                                       double* __restrict__ out) {
  __shared__ double sh[RT];
  for (int q = 0; q < nq; ++q) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += RT) v += partial[nq * b + q];
    const double s = block_sum(v, sh);
    if (threadIdx.x == 0) out[q] = s;
  }
}

// sum a*b (weights w if non-null)
__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b,
                           const double* __restrict__ wt, int64_t n, double* __restrict__ partial) {
  double v[1] = {0.0};
  for (int64_t p = (int64_t)blockIdx.x * RT + threadIdx.x; p < n; p += (int64_t)gridDim.x * RT)
    v[0] += wt ? wt[p] * a[p] * b[p] : a[p] * b[p];
  write_partials<1>(v, partial);
}

// r = mask*f ; p = dinv*r ; partial: rz = sum cwt r dinv r, rr = sum cwt r r
__global__ void cg_init_kernel(const double* __restrict__ f, const double* __restrict__ mask,
                               const double* __restrict__ dinv, const double* __restrict__ cwt,
                               double* __restrict__ r, double* __restrict__ p,
                               double* __restrict__ x, int64_t n, double* __restrict__ partial) {
  double v[2] = {0.0, 0.0};
  for (int64_t q = (int64_t)blockIdx.x * RT + threadIdx.x; q < n; q += (int64_t)gridDim.x * RT) {
    const double rr = mask[q] * f[q];
    const double z = dinv[q] * rr;
    r[q] = rr;
    p[q] = z;
    x[q] = 0.0;
    v[0] += cwt[q] * rr * z;
    v[1] += cwt[q] * rr * rr;
  }
  write_partials<2>(v, partial);
}

// alpha = sc[0] / sc[1] (rz / pw); x += alpha p; r -= alpha w;
// partial: rz' = sum cwt r dinv r, rr = sum cwt r r, cwt = mask / multiplicity.
// r is not masked: its boundary values are never used (dinv and cwt vanish
// there, and p = dinv r + beta p stays zero on the boundary).
__global__ void cg_update_kernel(double* __restrict__ x, double* __restrict__ r,
                                 const double* __restrict__ p, const double* __restrict__ w,
                                 const double* __restrict__ dinv, const double* __restrict__ cwt,
                                 const double* __restrict__ sc, int64_t n,
                                 double* __restrict__ partial) {
  const double alpha = cg_ratio(sc[0], sc[1]);
  double v[2] = {0.0, 0.0};
  for (int64_t q = (int64_t)blockIdx.x * RT + threadIdx.x; q < n; q += (int64_t)gridDim.x * RT) {
    x[q] = fma(alpha, p[q], x[q]);
    const double rr = fma(-alpha, w[q], r[q]);
    r[q] = rr;
    const double c = cwt[q] * rr;
    v[0] += c * dinv[q] * rr;
    v[1] += c * rr;
  }
  write_partials<2>(v, partial);
}

// Structured-brick variant of cg_update with the local DSSUM folded in
// (no separate pass over w): w holds A_local p (after the interface-plane
// exchange, whose points already carry their final sums); every other point
// gathers its node's local copies in ascending local order — the DSSUM's own
// order, so the assembled value is bit-identical — and cwt = mask / mult is
// computed from the point's position (exact powers of two).
//   alpha = a[0] / a[1];  r -= alpha (QQ^T w);  partial: rz', rr as cg_update
// x is not touched here (cg_xpupdate advances it with the old p).
struct CgBox {
  BoxGS M;
  int64_t NZ;  // global node planes
  int has_below, has_above;
  int xfolded;  // w's class-2 (x-face-only) nodes are already summed (x-folding apply)
};

// One element per block iteration (grid-stride over elements): the
// element's brick coordinates are computed once; a point's copies follow
// from which of its faces are interior (the lowest copy is q minus the
// strides of its lower neighbours, the others the compile-time / per-mesh
// strides above it — the order of gs_box_copies); branch-free so the loads
// of a thread's points overlap.
// EPI elements per iteration, MINB resident blocks per SM (register cap):
// (1, 3) measured best at lx = 8 (0.94 ms at C2 vs 1.0-2.1 ms for (1, 1..8),
// (2, 1..4), (4, 2): profiles/r01_cg_update_box.txt)
template <int LX, int EPI, int MINB>
__global__ void __launch_bounds__(RT, MINB) cg_update_box_kernel(double* __restrict__ r, const double* __restrict__ w,
                                                           const double* __restrict__ dinv,
                                                           const double* __restrict__ a, const CgBox B,
                                                           int64_t nel, double* __restrict__ partial) {
  constexpr int n1 = LX - 1, L2 = LX * LX, L3 = L2 * LX;
  constexpr int PPT = (L3 + RT - 1) / RT;  // points per thread per element
  constexpr int NP = EPI * PPT;            // EPI elements per iteration: all loads issued first
  constexpr int64_t DX = L3 - n1;
  const BoxGS& M = B.M;
  const int64_t DY = (int64_t)M.nx * L3 - n1 * LX;
  const int64_t DZ = (int64_t)M.nx * M.ny * L3 - n1 * L2;
  const int nl = (int)(M.ez1 - M.ez0);
  const double alpha = cg_ratio(a[0], a[1]);
  double v[2] = {0.0, 0.0};
  for (int64_t e0 = (int64_t)blockIdx.x * EPI; e0 < nel; e0 += (int64_t)gridDim.x * EPI) {
    double c8[NP][8], rq[NP], dq[NP], cw[NP];
    int64_t qq[NP];
    bool act[NP], single[NP];
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const int64_t e = e0 + u / PPT;
      const int p = threadIdx.x + (u % PPT) * RT;
      act[u] = e < nel && (PPT * RT == L3 || p < L3);
      const int ei = act[u] ? (int)e : 0;
      const int pi = act[u] ? p : 0;
      const int t = ei / M.nx;
      const int ex = ei - t * M.nx;
      const int ezl = t / M.ny;
      const int ey = t - ezl * M.ny;
      const int k = pi / L2, j = (pi / LX) % LX, i = pi % LX;
      const int64_t q = (int64_t)ei * L3 + pi;
      qq[u] = q;
      const bool lox = i == 0 && ex > 0, hix = i == n1 && ex < M.nx - 1;
      const bool loy = j == 0 && ey > 0, hiy = j == n1 && ey < M.ny - 1;
      const bool iface = (k == 0 && ezl == 0 && B.has_below) || (k == n1 && ezl == nl - 1 && B.has_above);
      const bool loz = !iface && k == 0 && ezl > 0, hiz = !iface && k == n1 && ezl < nl - 1;
      // x copies to gather: none when the x-folding apply summed this node
      // already (class 2: on an x face, on no y / z element face)
      const bool xs = (lox || hix) && !iface && !(B.xfolded && j != 0 && j != n1 && k != 0 && k != n1);
      const int cx = xs ? 2 : 1, cy = (loy || hiy) && !iface ? 2 : 1;
      const int cz = loz || hiz ? 2 : 1;
      single[u] = cx * cy * cz == 1;
      const int64_t b0 = q - ((lox && xs) ? DX : 0) - ((loy && !iface) ? DY : 0) - (loz ? DZ : 0);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int dz = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
        c8[u][c] = (act[u] && dz < cz && dy < cy && dx < cx) ? w[b0 + dx * DX + dy * DY + dz * DZ] : 0.0;
      }
      rq[u] = act[u] ? r[q] : 0.0;
      dq[u] = act[u] ? dinv[q] : 0.0;
      const int gx = ex * n1 + i, gy = ey * n1 + j, gz = (int)(M.ez0 + ezl) * n1 + k;
      const bool bnd = gx == 0 || gx == M.NX - 1 || gy == 0 || gy == M.NY - 1 || gz == 0 || gz == B.NZ - 1;
      const int mult = (i % n1 == 0 ? 2 : 1) * (j % n1 == 0 ? 2 : 1) * (k % n1 == 0 ? 2 : 1);
      cw[u] = bnd ? 0.0 : 1.0 / (double)mult;
    }
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      // absent copies hold +0.0: adding them is exact (a running sum that
      // starts at +0.0 is never -0.0 under round-to-nearest), so the sum
      // equals the DSSUM's predicated one bit for bit
      double wa;
      if (single[u]) {
        wa = c8[u][0];  // unshared or interface point: w as is
      } else {
        wa = 0.0;
#pragma unroll
        for (int c = 0; c < 8; ++c) wa = __dadd_rn(wa, c8[u][c]);
      }
      if (!act[u]) continue;
      const double rr = fma(-alpha, wa, rq[u]);
      r[qq[u]] = rr;
      const double c = cw[u] * rr;
      v[0] += c * dq[u] * rr;
      v[1] += c * rr;
    }
  }
  write_partials<2>(v, partial);
}

// alpha = a[0] / a[1], beta = sc_new[0] / a[0] (a = (rz_old, p.Ap)):
// x += alpha p (the old p);  p = dinv r + beta p
__global__ void cg_xpupdate_kernel(double* __restrict__ x, double* __restrict__ p,
                                   const double* __restrict__ r, const double* __restrict__ dinv,
                                   const double* __restrict__ a, const double* __restrict__ sc_new,
                                   int64_t n) {
  const double alpha = cg_ratio(a[0], a[1]);
  const double beta = cg_ratio(sc_new[0], a[0]);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x) {
    const double pq = p[q];
    x[q] = fma(alpha, pq, x[q]);
    p[q] = fma(beta, pq, dinv[q] * r[q]);
  }
}

// beta = sc_new[0] / sc_old[0]; p = dinv r + beta p
__global__ void cg_pupdate_kernel(double* __restrict__ p, const double* __restrict__ r,
                                  const double* __restrict__ dinv, const double* __restrict__ sc_new,
                                  const double* __restrict__ sc_old, int64_t n) {
  const double beta = cg_ratio(sc_new[0], sc_old[0]);
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (int64_t)gridDim.x * blockDim.x)
    p[q] = fma(beta, p[q], dinv[q] * r[q]);
}

// Local diagonal of A_e (closed form of ax_helm applied to unit vectors):
//  sum_l dxt[l][i] dx[i][l] (h1 g11)(k,j,l) + sum_l dyt[l][j] dy[j][l] (h1 g22)(k,l,i)
//  + sum_l dzt[l][k] dz[k][l] (h1 g33)(l,j,i) + h1(p) [ dxt[i][i] (g12 dy[j][j] + g13 dz[k][k])
//  + dyt[j][j] (g12 dx[i][i] + g23 dz[k][k]) + dzt[k][k] (g13 dx[i][i] + g23 dy[j][j]) ](p)
__global__ void diag_kernel(double* __restrict__ dg, const AxPtrs A, int lx, int64_t npts) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= npts) return;
  const int L2 = lx * lx, L3 = L2 * lx;
  const int64_t e = q / L3;
  const int p = (int)(q - e * L3);
  const int k = p / L2, j = (p / lx) % lx, i = p % lx;
  const int64_t b = e * L3;
  double s = 0.0;
  for (int l = 0; l < lx; ++l) {
    const int64_t qx = b + (k * lx + j) * lx + l, qy = b + (k * lx + l) * lx + i, qz = b + (l * lx + j) * lx + i;
    s += A.dxt[l * lx + i] * A.dx[i * lx + l] * A.h1[qx] * A.g11[qx];
    s += A.dyt[l * lx + j] * A.dy[j * lx + l] * A.h1[qy] * A.g22[qy];
    s += A.dzt[l * lx + k] * A.dz[k * lx + l] * A.h1[qz] * A.g33[qz];
  }
  const double dxi = A.dx[i * lx + i], dyj = A.dy[j * lx + j], dzk = A.dz[k * lx + k];
  s += A.h1[q] * (A.dxt[i * lx + i] * (A.g12[q] * dyj + A.g13[q] * dzk) +
                  A.dyt[j * lx + j] * (A.g12[q] * dxi + A.g23[q] * dzk) +
                  A.dzt[k * lx + k] * (A.g13[q] * dxi + A.g23[q] * dyj));
  dg[q] = s;
}

static int red_blocks(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t b = (n + RT - 1) / RT;
  const int64_t cap = (int64_t)sms * 8;
  return (int)(b < cap ? (b > 0 ? b : 1) : cap);
}

}  // namespace axb

using namespace axb;

extern "C" {

int axhelm_reduce_blocks(int64_t n) { return red_blocks(n); }

int axhelm_dot(const double* a, const double* b, const double* wt, int64_t n, double* partial,
               double* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  dot_kernel<<<nb, RT, 0, st>>>(a, b, wt, n, partial);
  reduce_partials_kernel<<<1, RT, 0, st>>>(partial, nb, 1, out);
  return cuda_status(cudaGetLastError(), "axhelm_dot");
}

int axhelm_cg_init(const double* f, const double* mask, const double* dinv, const double* cwt,
                   double* r, double* p, double* x, int64_t n, double* partial, double* out,
                   void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  cg_init_kernel<<<nb, RT, 0, st>>>(f, mask, dinv, cwt, r, p, x, n, partial);
  reduce_partials_kernel<<<1, RT, 0, st>>>(partial, nb, 2, out);
  return cuda_status(cudaGetLastError(), "axhelm_cg_init");
}

int axhelm_cg_update(double* x, double* r, const double* p, const double* w, const double* dinv,
                     const double* cwt, const double* sc, int64_t n, double* partial, double* out,
                     void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(n);
  cg_update_kernel<<<nb, RT, 0, st>>>(x, r, p, w, dinv, cwt, sc, n, partial);
  reduce_partials_kernel<<<1, RT, 0, st>>>(partial, nb, 2, out);
  return cuda_status(cudaGetLastError(), "axhelm_cg_update");
}

int axhelm_cg_update_box(double* r, const double* w, const double* dinv, const double* a, int nx,
                         int ny, int64_t nz, int lx, int64_t ez0, int64_t ez1, int has_below,
                         int has_above, int xfolded, double* partial, double* out, void* stream) {
  if (lx < 2 || lx > 16 || nx < 1 || ny < 1 || ez0 < 0 || ez1 <= ez0 || ez1 > nz)
    return set_status(AXHELM_EINVAL, "axhelm_cg_update_box: bad sizes");
  const int n1 = lx - 1;
  CgBox B{BoxGS{nx, ny, lx, ez0, ez1, (int64_t)nx * n1 + 1, (int64_t)ny * n1 + 1}, nz * n1 + 1,
          has_below, has_above, xfolded ? 1 : 0};
  const int64_t nel = (ez1 - ez0) * nx * ny;
  if (nel >= ((int64_t)1 << 31)) return set_status(AXHELM_EINVAL, "axhelm_cg_update_box: too many elements");
  cudaStream_t st = (cudaStream_t)stream;
  const int nb = red_blocks(nel * lx * lx * lx);
  switch (lx) {
#define AXB_CGB(N) \
  case N:          \
    cg_update_box_kernel<N, 1, 3><<<nb, RT, 0, st>>>(r, w, dinv, a, B, nel, partial); \
    break;
    AXB_CGB(2) AXB_CGB(3) AXB_CGB(4) AXB_CGB(5) AXB_CGB(6) AXB_CGB(7) AXB_CGB(8) AXB_CGB(9)
    AXB_CGB(10) AXB_CGB(11) AXB_CGB(12) AXB_CGB(13) AXB_CGB(14) AXB_CGB(15) AXB_CGB(16)
#undef AXB_CGB
  }
  reduce_partials_kernel<<<1, RT, 0, st>>>(partial, nb, 2, out);
  return cuda_status(cudaGetLastError(), "axhelm_cg_update_box");
}

int axhelm_cg_xpupdate(double* x, double* p, const double* r, const double* dinv, const double* a,
                       const double* sc_new, int64_t n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  cg_xpupdate_kernel<<<red_blocks(n), RT, 0, st>>>(x, p, r, dinv, a, sc_new, n);
  return cuda_status(cudaGetLastError(), "axhelm_cg_xpupdate");
}

int axhelm_cg_pupdate(double* p, const double* r, const double* dinv, const double* sc_new,
                      const double* sc_old, int64_t n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  cg_pupdate_kernel<<<red_blocks(n), RT, 0, st>>>(p, r, dinv, sc_new, sc_old, n);
  return cuda_status(cudaGetLastError(), "axhelm_cg_pupdate");
}

}  // extern "C"

namespace axb {
// ax_helm + out[0] = sum u*w over the nel elements (fused for the lx = 8
// DMMA kernel, else a separate fixed-order dot pass); partial: block scratch
static cudaError_t ax_dot(const AxPtrs& A, int64_t nel, int lx, int mode, double* partial, double* out,
                          cudaStream_t st, const AxExt& X = AxExt{}) {
  const int64_t n = nel * lx * lx * lx;
  cudaError_t e;
  if (dmma8_selected(A, lx, mode)) {
    int nb = 0;
    e = launch_dmma8_dot(A, nel, partial, &nb, st, X);
    if (e == cudaSuccess) {
      reduce_partials_kernel<<<1, RT, 0, st>>>(partial, nb, 1, out);
      e = cudaGetLastError();
    }
    return e;
  }
  e = launch_ax(A, nel, lx, mode, st, nullptr, X);
  if (e == cudaSuccess) {
    const int nb = red_blocks(n);
    dot_kernel<<<nb, RT, 0, st>>>(A.u, A.w, nullptr, n, partial);
    reduce_partials_kernel<<<1, RT, 0, st>>>(partial, nb, 1, out);
    e = cudaGetLastError();
  }
  return e;
}

// the follower's stream and fork/join events, one set per device
struct FollowStreams {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static FollowStreams* follow_streams() {
  static std::mutex mu;
  static FollowStreams fs[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  FollowStreams& f = fs[dev];
  if (!f.side) {
    if (cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&f.join, cudaEventDisableTiming) != cudaSuccess) {
      f.side = nullptr;
      return nullptr;
    }
  }
  return &f;
}

static int max_partials() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * 8;  // >= red_blocks(n) and >= the DMMA grid
}
}  // namespace axb

extern "C" {

int axhelm_apply_dot(double* wd, const double* ud, const double* dxd, const double* dyd,
                     const double* dzd, const double* dxtd, const double* dytd, const double* dztd,
                     const double* h1d, const double* g11d, const double* g22d, const double* g33d,
                     const double* g12d, const double* g13d, const double* g23d, int64_t nel,
                     int lx, int mode, double* partial, double* out, void* stream) {
  if (lx < 2 || lx > 16 || nel < 0) return set_status(AXHELM_EINVAL, "axhelm_apply_dot: bad sizes");
  const int keep = (mode & AXHELM_KEEP_W_L2) != 0;
  mode &= ~AXHELM_KEEP_W_L2;
  if (mode != AXHELM_STRICT && mode != AXHELM_FAST)
    return set_status(AXHELM_EINVAL, "axhelm_apply_dot: unknown mode %d", mode);
  AxPtrs A{wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd, h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  AxExt X;
  X.keep_w = keep;
  if (nel == 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(double), (cudaStream_t)stream);
    return cuda_status(e, "axhelm_apply_dot");
  }
  return cuda_status(ax_dot(A, nel, lx, mode, partial, out, (cudaStream_t)stream, X), "axhelm_apply_dot");
}

int axhelm_apply_box(double* wd, const double* ud, const double* dxd, const double* dyd,
                     const double* dzd, const double* dxtd, const double* dytd, const double* dztd,
                     const double* h1d, const double* g11d, const double* g22d, const double* g33d,
                     const double* g12d, const double* g13d, const double* g23d, int nx, int64_t nel,
                     int lx, int mode, double* partial, double* dot_out, int* xfolded, void* stream) {
  // wd must start at an x-run start (ex = 0): the x-folding epilogue sums
  // the faces shared by consecutive elements of each run of nx
  if (xfolded) *xfolded = 0;
  if (lx < 2 || lx > 16 || nel < 0 || nx < 1 || nel % nx != 0)
    return set_status(AXHELM_EINVAL, "axhelm_apply_box: bad sizes (nel must be whole x-runs of nx)");
  const int keep = (mode & AXHELM_KEEP_W_L2) != 0;
  mode &= ~AXHELM_KEEP_W_L2;
  if (mode != AXHELM_STRICT && mode != AXHELM_FAST)
    return set_status(AXHELM_EINVAL, "axhelm_apply_box: unknown mode %d", mode);
  {
    const double* ptrs[15] = {wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd,
                              h1d, g11d, g22d, g33d, g12d, g13d, g23d};
    for (int q = 0; q < 15; ++q)
      if (!ptrs[q]) return set_status(AXHELM_EINVAL, "axhelm_apply_box: argument %d is NULL", q);
  }
  if (dot_out && !partial) return set_status(AXHELM_EINVAL, "axhelm_apply_box: dot needs partial scratch");
  cudaStream_t st = (cudaStream_t)stream;
  if (nel == 0) {
    cudaError_t e = dot_out ? cudaMemsetAsync(dot_out, 0, sizeof(double), st) : cudaSuccess;
    return cuda_status(e, "axhelm_apply_box");
  }
  AxPtrs A{wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd, h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  AxExt X;
  X.keep_w = keep;
  const char* xf_env = getenv("AXHELM_XFOLD");
  if (nx > 1 && lx > 2 && !(xf_env && xf_env[0] == '0') && dmma8_selected(A, lx, mode)) X.xrun = nx;
  cudaError_t e = dot_out ? ax_dot(A, nel, lx, mode, partial, dot_out, st, X)
                          : launch_ax(A, nel, lx, mode, st, nullptr, X);
  if (e == cudaSuccess && xfolded) *xfolded = X.xrun > 0;
  return cuda_status(e, "axhelm_apply_box");
}

int axhelm_ax_gs_scratch(int64_t nlayers) { return max_partials() + (int)(nlayers > 0 ? nlayers : 0); }

int axhelm_ax_gs_box(double* wd, const double* ud, const double* dxd, const double* dyd,
                     const double* dzd, const double* dxtd, const double* dytd, const double* dztd,
                     const double* h1d, const double* g11d, const double* g22d, const double* g33d,
                     const double* g12d, const double* g13d, const double* g23d, int nx, int ny,
                     int lx, int64_t ez0, int64_t ez1, int64_t l0, int64_t l1, int64_t zlo,
                     int64_t zhi, int mode, int schedule, unsigned* progress, double* partial,
                     double* dot_out, void* stream) {
  const int64_t nl = ez1 - ez0;
  if (const char* why = gs_box_range_check(nx, ny, lx, ez0, ez1, zlo, zhi))
    return set_status(AXHELM_EINVAL, "axhelm_ax_gs_box: %s", why);
  if (l0 < 0 || l1 > nl || l1 < l0) return set_status(AXHELM_EINVAL, "axhelm_ax_gs_box: bad layer range");
  if (mode != AXHELM_STRICT && mode != AXHELM_FAST)
    return set_status(AXHELM_EINVAL, "axhelm_ax_gs_box: unknown mode %d", mode);
  if (dot_out && !partial) return set_status(AXHELM_EINVAL, "axhelm_ax_gs_box: dot needs partial scratch");
  if (schedule == AXHELM_SCHED_FOLLOW && !progress)
    return set_status(AXHELM_EINVAL, "axhelm_ax_gs_box: the follow schedule needs progress scratch");
  cudaStream_t st = (cudaStream_t)stream;
  const int n1 = lx - 1;
  const int64_t L3 = (int64_t)lx * lx * lx, lay = (int64_t)nx * ny;
  const int pmax = max_partials();
  double* chunk_dot = partial ? partial + pmax : nullptr;
  auto ptrs_at = [&](int64_t layer) {
    const int64_t o = layer * lay * L3;
    return AxPtrs{wd + o, ud + o, dxd, dyd, dzd, dxtd, dytd, dztd, h1d + o, g11d + o, g22d + o, g33d + o,
                  g12d + o, g13d + o, g23d + o};
  };
  cudaError_t e = cudaSuccess;
  if (schedule == AXHELM_SCHED_FOLLOW) {
    AxPtrs A = ptrs_at(l0);
    AxExt X;
    X.keep_w = 1;
    X.progress = progress;
    X.lay = lay;
    // only the lx = 8 DMMA kernel publishes progress (its dot is fused, taken
    // before the follower assembles w); everything else runs sequentially
    // Co-residency assumption: the follower spins on counters the apply
    // publishes, so every apply CTA must be able to become resident while
    // follower CTAs occupy SMs.  The apply's persistent grid is sized by its
    // own occupancy and the follower takes only registers / threads it
    // leaves free; under an MPS SM limit (or another tenant) that no longer
    // holds, so the schedule falls back to sequential there.
    const char* mps = getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE");
    const bool sm_limited = mps && atoi(mps) > 0 && atoi(mps) < 100;
    if (l1 > l0 && !sm_limited && progress_capable(A, lx) && dmma8_selected(A, lx, mode)) {
      FollowStreams* fs = follow_streams();
      if (!fs) return set_status(AXHELM_ECUDA, "axhelm_ax_gs_box: cannot create the follower stream");
      // The apply is enqueued first and never waits on the follower, so it
      // always completes; the follower only waits on the apply's counters.
      // Its CTAs are small (128 threads, <= 64 registers, no shared memory)
      // and fit beside the apply's persistent CTAs on the same SMs.
      e = cudaMemsetAsync(progress, 0, sizeof(unsigned) * (size_t)(l1 - l0), st);
      if (e == cudaSuccess) e = cudaEventRecord(fs->fork, st);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(fs->side, fs->fork, 0);
      if (e == cudaSuccess)
        e = dot_out ? ax_dot(A, (l1 - l0) * lay, lx, mode, partial, dot_out, st, X)
                    : launch_ax(A, (l1 - l0) * lay, lx, mode, st, nullptr, X);
      if (e == cudaSuccess) e = gs_box_follow(wd, nx, ny, lx, ez0, ez1, zlo, zhi, progress, l0, l1, fs->side);
      if (e == cudaSuccess) e = cudaEventRecord(fs->join, fs->side);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, fs->join, 0);
      return cuda_status(e, "axhelm_ax_gs_box");
    }
    schedule = AXHELM_SCHED_SEQUENTIAL;
  }
  const int64_t B = schedule > 0 ? schedule : (l1 - l0 > 0 ? l1 - l0 : 1);
  // x-folding apply (ax_dmma.cuh, XF): the DMMA kernel sums the class-2
  // (x-face-only) nodes of its layers itself; the DSSUM pass skips those
  // planes' class 2.  Needs every class-2 plane of [l0, l1) in this call's
  // range [zlo, zhi], and nothing else in the call reading unassembled w.
  const int64_t s2lo = (ez0 + l0) * n1 + 1, s2hi = (ez0 + l1) * n1 - 1;
  const char* xf_env = getenv("AXHELM_XFOLD");
  const bool xfold = l1 > l0 && nx > 1 && n1 > 1 && !(xf_env && xf_env[0] == '0') && zlo <= s2lo &&
                     zhi >= s2hi && dmma8_selected(ptrs_at(l0), lx, mode);
  int64_t next = zlo;  // first plane not yet summed
  int nchunks = 0;
  for (int64_t a = l0; a < l1 && e == cudaSuccess; a += B, ++nchunks) {
    const int64_t b = (a + B < l1) ? a + B : l1;
    AxPtrs A = ptrs_at(a);
    AxExt X;
    X.keep_w = schedule > 0 ? 1 : 0;
    X.xrun = xfold ? nx : 0;
    const int64_t nel = (b - a) * lay;
    e = dot_out ? ax_dot(A, nel, lx, mode, partial, chunk_dot + nchunks, st, X)
                : launch_ax(A, nel, lx, mode, st, nullptr, X);
    if (e != cudaSuccess) break;
    // planes whose every copy is computed: below layer ez0 + b, or all when
    // the layers above l1 are done by the caller
    const int64_t top = (b == l1) ? zhi : ((ez0 + b) * n1 - 1 < zhi ? (ez0 + b) * n1 - 1 : zhi);
    if (top >= next) {
      e = xfold ? gs_box_range(wd, nx, ny, lx, ez0, ez1, next, top, st, s2lo, s2hi)
                : gs_box_range(wd, nx, ny, lx, ez0, ez1, next, top, st);
      next = top + 1;
    }
  }
  if (e == cudaSuccess && next <= zhi)
    e = xfold ? gs_box_range(wd, nx, ny, lx, ez0, ez1, next, zhi, st, s2lo, s2hi)
              : gs_box_range(wd, nx, ny, lx, ez0, ez1, next, zhi, st);
  if (e == cudaSuccess && dot_out) {
    if (nchunks == 0) {
      e = cudaMemsetAsync(dot_out, 0, sizeof(double), st);
    } else {
      reduce_partials_kernel<<<1, RT, 0, st>>>(chunk_dot, nchunks, 1, dot_out);
      e = cudaGetLastError();
    }
  }
  return cuda_status(e, "axhelm_ax_gs_box");
}

int axhelm_diag(double* diag, const double* dxd, const double* dyd, const double* dzd,
                const double* dxtd, const double* dytd, const double* dztd, const double* h1d,
                const double* g11d, const double* g22d, const double* g33d, const double* g12d,
                const double* g13d, const double* g23d, int64_t nel, int lx, void* stream) {
  if (lx < 2 || lx > 16 || nel < 0) return set_status(AXHELM_EINVAL, "axhelm_diag: bad sizes");
  const int64_t n = nel * lx * lx * lx;
  if (n == 0) return set_status(AXHELM_OK, "");
  AxPtrs A{diag, nullptr, dxd, dyd, dzd, dxtd, dytd, dztd, h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  diag_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(diag, A, lx, n);
  return cuda_status(cudaGetLastError(), "axhelm_diag");
}

}  // extern "C"
