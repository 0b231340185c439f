// Box mesh, device geometry store and gather-scatter (direct stiffness
// summation, DSSUM) for the B200 ax_helm path.
//
// No reference counterpart: SPEC.md:14 puts gather-scatter, meshes and the
// Poisson solve out of the reference's scope; PAPER.md:123 names
// gather-scatter as Neko's second ingredient.  Parity is against the
// restated CPU oracle (oracle/oracle.py: box_mesh_gid, dssum), bit-exact.
//
// DSSUM contract (the order that makes it bit-exact): every global node's
// value is the sum, from 0.0, of all its local copies in ascending local
// (flat [e][k][j][i]) index; the sum is written back to every copy.  The
// shared nodes are held in CSR form sorted by global id (host setup,
// gs.py); one thread per shared node walks its copies in order.
//
// Multi-GPU interface planes (slab partition along z, gs.py / dist.py):
// the lower rank sums its copies of a plane node (gs_plane_partial), the
// upper rank continues the same running sum with its own copies
// (gs_plane_finish: init = received partial) and both write the final
// value (gs_plane_write on the lower rank).  Because slabs are contiguous
// element ranges in z-major order, this is exactly the single-GPU order.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/axhelm.h"
#include "ax_launch.h"

namespace axb {

// ------------------------------------------------------------------ mesh

// global node id of local point (e_local, k, j, i) of a slab starting at
// element layer ez0 of an nx x ny x nz brick (element order e = (ez*ny+ey)*nx+ex)
__global__ void box_gid_kernel(int64_t* __restrict__ gid, int nx, int ny, int lx, int64_t ez0,
                               int64_t npts) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  const int64_t L3 = (int64_t)lx * lx * lx;
  const int64_t el = p / L3;
  const int r = (int)(p - el * L3);
  const int k = r / (lx * lx), j = (r / lx) % lx, i = r % lx;
  const int64_t exy = el % ((int64_t)nx * ny);
  const int64_t ez = ez0 + el / ((int64_t)nx * ny);
  const int64_t ey = exy / nx, ex = exy % nx;
  const int64_t n1 = lx - 1;
  const int64_t NX = nx * n1 + 1, NY = ny * n1 + 1;
  const int64_t gx = ex * n1 + i, gy = ey * n1 + j, gz = ez * n1 + k;
  gid[p] = (gz * NY + gy) * NX + gx;
}

// Geometric factors of a smoothly deformed brick [0,nx]x[0,ny]x[0,nz] of
// unit elements: X = X0 + d(X0) (1, 1, 1) with
//   d = (amp / c_min) sin(c_x X0) sin(c_y Y0) sin(c_z Z0),  c_a = 2 pi / n_a
// (boundary fixed, continuous across elements, |grad d| <= sqrt(3) amp, so
// det J = (1 + dd/dX + dd/dY + dd/dZ) / 8 > 0 for amp < 1/sqrt(3)).  J_ab = dX_a/dxi_b,
// G = w_i w_j w_k det(J) J^-1 J^-T (the Poisson metric with the quadrature
// weights folded in, as sem.py's GeomFactors expects), h1 = 1.
__global__ void box_geom_kernel(double* __restrict__ h1, double* __restrict__ g11,
                                double* __restrict__ g22, double* __restrict__ g33,
                                double* __restrict__ g12, double* __restrict__ g13,
                                double* __restrict__ g23, const double* __restrict__ pts,
                                const double* __restrict__ wts, int nx, int ny, int nz, int lx,
                                int64_t ez0, int64_t npts, double amp) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npts) return;
  const int64_t L3 = (int64_t)lx * lx * lx;
  const int64_t el = p / L3;
  const int r = (int)(p - el * L3);
  const int k = r / (lx * lx), j = (r / lx) % lx, i = r % lx;
  const int64_t exy = el % ((int64_t)nx * ny);
  const int64_t ez = ez0 + el / ((int64_t)nx * ny);
  const int64_t ey = exy / nx, ex = exy % nx;
  // unit-size elements: Lx = nx etc.
  const double X0 = (double)ex + 0.5 * (pts[i] + 1.0);
  const double Y0 = (double)ey + 0.5 * (pts[j] + 1.0);
  const double Z0 = (double)ez + 0.5 * (pts[k] + 1.0);
  const double cx = 2.0 * M_PI / nx, cy = 2.0 * M_PI / ny, cz = 2.0 * M_PI / nz;
  double sx, csx, sy, csy, sz, csz;
  sincos(cx * X0, &sx, &csx);
  sincos(cy * Y0, &sy, &csy);
  sincos(cz * Z0, &sz, &csz);
  const double cmin = fmin(cx, fmin(cy, cz));
  const double dX = amp * (cx / cmin) * csx * sy * sz;  // gradient of d
  const double dY = amp * (cy / cmin) * sx * csy * sz;
  const double dZ = amp * (cz / cmin) * sx * sy * csz;
  // dX0/dxi = 0.5 along each axis; X_a = X0_a + d  =>  J_ab = 0.5 (delta_ab + dd/dX0_b)
  double J[3][3];
  const double gd[3] = {dX, dY, dZ};
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) J[a][b] = 0.5 * ((a == b ? 1.0 : 0.0) + gd[b]);
  const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                     J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                     J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
  // inverse (rows b = dxi_b / dX_a over a)
  double I[3][3];
  I[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
  I[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
  I[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
  I[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
  I[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
  I[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
  I[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
  I[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
  I[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
  const double s = wts[i] * wts[j] * wts[k] * det;
  double G[3][3];
  for (int b = 0; b < 3; ++b)
    for (int c = 0; c < 3; ++c) G[b][c] = s * (I[b][0] * I[c][0] + I[b][1] * I[c][1] + I[b][2] * I[c][2]);
  h1[p] = 1.0;
  g11[p] = G[0][0];
  g22[p] = G[1][1];
  g33[p] = G[2][2];
  g12[p] = G[0][1];
  g13[p] = G[0][2];
  g23[p] = G[1][2];
}

// --------------------------------------------------------- gather-scatter

template <typename I>
__global__ void gs_sum_kernel(double* __restrict__ w, const int64_t* __restrict__ offs,
                              const I* __restrict__ idx, int64_t n) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const int64_t b = offs[q], e = offs[q + 1];
  double s = 0.0;
  for (int64_t c = b; c < e; ++c) s = __dadd_rn(s, w[idx[c]]);
  for (int64_t c = b; c < e; ++c) w[idx[c]] = s;
}

template <typename I>
__global__ void gs_plane_partial_kernel(const double* __restrict__ w, const int64_t* __restrict__ offs,
                                        const I* __restrict__ idx, const int64_t* __restrict__ slot,
                                        int64_t n, double* __restrict__ buf) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  double s = 0.0;
  for (int64_t c = offs[q]; c < offs[q + 1]; ++c) s = __dadd_rn(s, w[idx[c]]);
  buf[slot[q]] = s;
}

template <typename I>
__global__ void gs_plane_finish_kernel(double* __restrict__ w, const int64_t* __restrict__ offs,
                                       const I* __restrict__ idx, const int64_t* __restrict__ slot,
                                       int64_t n, double* __restrict__ buf) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  double s = buf[slot[q]];
  for (int64_t c = offs[q]; c < offs[q + 1]; ++c) s = __dadd_rn(s, w[idx[c]]);
  for (int64_t c = offs[q]; c < offs[q + 1]; ++c) w[idx[c]] = s;
  buf[slot[q]] = s;
}

template <typename I>
__global__ void gs_plane_write_kernel(double* __restrict__ w, const int64_t* __restrict__ offs,
                                      const I* __restrict__ idx, const int64_t* __restrict__ slot,
                                      int64_t n, const double* __restrict__ buf) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const double s = buf[slot[q]];
  for (int64_t c = offs[q]; c < offs[q + 1]; ++c) w[idx[c]] = s;
}

static unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace axb

using namespace axb;

extern "C" {

int axhelm_box_gid(int64_t* gid, int nx, int ny, int lx, int64_t ez0, int64_t nel, void* stream) {
  if (lx < 2 || lx > 16 || nx < 1 || ny < 1 || nel < 0 || ez0 < 0)
    return set_status(AXHELM_EINVAL, "axhelm_box_gid: bad sizes");
  const int64_t n = nel * lx * lx * lx;
  if (n == 0) return set_status(AXHELM_OK, "");
  box_gid_kernel<<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(gid, nx, ny, lx, ez0, n);
  return cuda_status(cudaGetLastError(), "axhelm_box_gid");
}

int axhelm_box_geometry(double* h1d, double* g11d, double* g22d, double* g33d, double* g12d,
                        double* g13d, double* g23d, const double* gll_points,
                        const double* gll_weights, int nx, int ny, int nz, int lx, int64_t ez0,
                        int64_t nel, double amp, void* stream) {
  if (lx < 2 || lx > 16 || nx < 1 || ny < 1 || nz < 1 || nel < 0 || ez0 < 0)
    return set_status(AXHELM_EINVAL, "axhelm_box_geometry: bad sizes");
  const int64_t n = nel * lx * lx * lx;
  if (n == 0) return set_status(AXHELM_OK, "");
  box_geom_kernel<<<blocks_for(n, 128), 128, 0, (cudaStream_t)stream>>>(
      h1d, g11d, g22d, g33d, g12d, g13d, g23d, gll_points, gll_weights, nx, ny, nz, lx, ez0, n, amp);
  return cuda_status(cudaGetLastError(), "axhelm_box_geometry");
}

int axhelm_gs_sum(double* w, const int64_t* offs, const void* idx, int idx_bytes, int64_t n,
                  void* stream) {
  if (n < 0) return set_status(AXHELM_EINVAL, "axhelm_gs_sum: n < 0");
  if (n == 0) return set_status(AXHELM_OK, "");
  if (idx_bytes == 4)
    gs_sum_kernel<int32_t><<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        w, offs, (const int32_t*)idx, n);
  else if (idx_bytes == 8)
    gs_sum_kernel<int64_t><<<blocks_for(n, 256), 256, 0, (cudaStream_t)stream>>>(
        w, offs, (const int64_t*)idx, n);
  else
    return set_status(AXHELM_EINVAL, "idx_bytes must be 4 or 8");
  return cuda_status(cudaGetLastError(), "axhelm_gs_sum");
}

int axhelm_gs_plane(int op, double* w, const int64_t* offs, const void* idx, int idx_bytes,
                    const int64_t* slot, int64_t n, double* buf, void* stream) {
  if (n < 0) return set_status(AXHELM_EINVAL, "axhelm_gs_plane: n < 0");
  if (n == 0) return set_status(AXHELM_OK, "");
  if (idx_bytes != 4 && idx_bytes != 8) return set_status(AXHELM_EINVAL, "idx_bytes must be 4 or 8");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned nb = blocks_for(n, 256);
  switch (op) {
    case AXHELM_GS_PARTIAL:
      if (idx_bytes == 4) gs_plane_partial_kernel<int32_t><<<nb, 256, 0, st>>>(w, offs, (const int32_t*)idx, slot, n, buf);
      else gs_plane_partial_kernel<int64_t><<<nb, 256, 0, st>>>(w, offs, (const int64_t*)idx, slot, n, buf);
      break;
    case AXHELM_GS_FINISH:
      if (idx_bytes == 4) gs_plane_finish_kernel<int32_t><<<nb, 256, 0, st>>>(w, offs, (const int32_t*)idx, slot, n, buf);
      else gs_plane_finish_kernel<int64_t><<<nb, 256, 0, st>>>(w, offs, (const int64_t*)idx, slot, n, buf);
      break;
    case AXHELM_GS_WRITE:
      if (idx_bytes == 4) gs_plane_write_kernel<int32_t><<<nb, 256, 0, st>>>(w, offs, (const int32_t*)idx, slot, n, buf);
      else gs_plane_write_kernel<int64_t><<<nb, 256, 0, st>>>(w, offs, (const int64_t*)idx, slot, n, buf);
      break;
    default:
      return set_status(AXHELM_EINVAL, "axhelm_gs_plane: unknown op %d", op);
  }
  return cuda_status(cudaGetLastError(), "axhelm_gs_plane");
}

}  // extern "C"
