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
#include <cstring>

#include "../../include/axhelm.h"
#include "ax_launch.h"
#include "box_gs.cuh"

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

// ===================================================================
// Structured DSSUM for BoxMesh slabs: the copies of a global node are found
// arithmetically (no index arrays: the CSR path's ~4.3 B/point of offsets
// and indices disappear; only the shared copies of w move).  One thread per
// global node of the slab's node planes [gz_lo, gz_hi] (x fastest); copies
// are visited in ascending (ez, ey, ex) = ascending local index, so the sum
// order equals the CSR path's and the oracle's.
// ===================================================================
namespace axb {

// Walks the copies of node (gx, gy, gz) in ascending local order: OP 0 sums
// and writes back (skipping unshared nodes), 1 = PARTIAL (sum -> buf),
// 2 = FINISH (continue from buf, write back, sum -> buf), 3 = WRITE (buf -> copies).
template <int LX, int OP>
__device__ __forceinline__ void gs_box_node(double* __restrict__ w, const BoxGS& M, int gx, int gy,
                                            int gz, const double* in, double* out) {
  constexpr int n1 = LX - 1;
  constexpr int L3 = LX * LX * LX;
  constexpr int64_t DX = L3 - n1;
  int64_t off0, DY, DZ;
  int cx, cy, cz;
  gs_box_copies<LX>(M, gx, gy, gz, off0, cx, cy, cz, DY, DZ);
  if (OP == 0 && cx * cy * cz < 2) return;
  const int64_t slot = (int64_t)gy * M.NX + gx;
  bool ok[8];
  int64_t off[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {  // c = (dz, dy, dx): ascending (ez, ey, ex)
    const int dz = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
    ok[c] = dz < cz && dy < cy && dx < cx;
    off[c] = off0 + dx * DX + dy * DY + dz * DZ;
  }
  double s = (OP == 2 || OP == 3) ? in[slot] : 0.0;
  if (OP != 3) {
    double v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = ok[c] ? w[off[c]] : 0.0;  // independent loads
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (ok[c]) s = __dadd_rn(s, v[c]);
  }
  if (OP == 1) {
    out[slot] = s;
    return;
  }
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (ok[c]) w[off[c]] = s;
  if (OP == 2) out[slot] = s;
}

// Interface-plane steps: one thread per node of plane gz (x fastest).
template <int LX, int OP>
__global__ void gs_box_plane_kernel(double* __restrict__ w, const BoxGS M, int gz,
                                    double* __restrict__ buf) {
  const int gx = blockIdx.x * blockDim.x + threadIdx.x;
  if (gx >= M.NX) return;
  gs_box_node<LX, OP>(w, M, gx, blockIdx.y, gz, buf, buf);
}

__device__ __forceinline__ unsigned long long peer_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// The same interface-plane steps with the neighbour's buffers in PEER memory
// (CUDA IPC over NVLink): the exchange is done by the kernels themselves, no
// NCCL and no host synchronisation.
//   PARTIAL (top plane)   : out = upper rank's receive buffer; signal its flag
//   FINISH  (bottom plane): wait own flag >= seq; in = own receive buffer
//                           (the lower rank's partials); out = lower rank's
//                           receive buffer; signal its flag
//   WRITE   (top plane)   : wait own flag >= seq; in = own receive buffer
// Signal: every CTA fences at system scope after its stores and counts
// itself in; the last one publishes seq with a system-scope release store.
// Wait: thread 0 of every CTA spins on an acquire load (10 s -> __trap()).
template <int LX, int OP>
__global__ void gs_box_plane_peer_kernel(double* __restrict__ w, const BoxGS M, int gz,
                                         const double* in, double* out,
                                         const unsigned long long* wait_flag,
                                         unsigned long long* signal_flag, unsigned long long seq,
                                         unsigned* counter, const unsigned long long* seq_dev) {
  if (seq_dev) seq = *seq_dev + 1;  // device-side sequence (graph replays advance it)
  if (OP >= 2) {
    if (threadIdx.x == 0) {
      unsigned long long v = 0, t0 = 0;
      for (;;) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(wait_flag) : "memory");
        if (v >= seq) break;
        __nanosleep(128);
        const unsigned long long t = peer_timer();
        if (t0 == 0) t0 = t;
        if (t - t0 > 10000000000ull) __trap();
      }
    }
    __syncthreads();
  }
  const int gx = blockIdx.x * blockDim.x + threadIdx.x;
  if (gx < M.NX) gs_box_node<LX, OP>(w, M, gx, blockIdx.y, gz, in, out);
  if (OP <= 2) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      const unsigned total = gridDim.x * gridDim.y;
      if (atomicAdd(counter, 1u) == total - 1) {
        *counter = 0;
        __threadfence_system();
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(signal_flag), "l"(seq) : "memory");
      }
    }
  }
}

// Local DSSUM, enumerating only (potentially) shared nodes, densely:
//  CLS 0: node planes on element faces (gz % n1 == 0): every (gx, gy)
//  CLS 1: the other planes, rows on y faces (gy % n1 == 0): every gx
//  CLS 2: the other planes and rows: x-face nodes only (gx = fx * n1)
// z-plane sets are [zlo, zhi] (inclusive) of node planes owned locally.
// A thread may take NB nodes (consecutive rows / planes) and issue all
// their loads before any sum; NB = 1 everywhere since the node-dense
// enumeration (2 and 4 measured neutral for classes 0 / 1 at 4.2 TB/s,
// profiles/r02_ab_gs_nb.txt).
template <int LX, int NB>
__device__ __forceinline__ void gs_box_local_nodes(double* __restrict__ w, const BoxGS& M,
                                                   const int (&gx)[NB], const int (&gy)[NB],
                                                   const int (&gz)[NB], const bool (&use)[NB]) {
  constexpr int n1 = LX - 1;
  constexpr int L3 = LX * LX * LX;
  constexpr int64_t DX = L3 - n1;
  int64_t off[NB][8];
  bool ok[NB][8];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    int64_t off0, DY, DZ;
    int cx, cy, cz;
    gs_box_copies<LX>(M, gx[b], gy[b], gz[b], off0, cx, cy, cz, DY, DZ);
    const bool shared = use[b] && cx * cy * cz >= 2;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int dz = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
      ok[b][c] = shared && dz < cz && dy < cy && dx < cx;
      off[b][c] = off0 + dx * DX + dy * DY + dz * DZ;
    }
  }
  double v[NB][8];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int c = 0; c < 8; ++c) v[b][c] = ok[b][c] ? w[off[b][c]] : 0.0;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (ok[b][c]) s = __dadd_rn(s, v[b][c]);
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (ok[b][c]) w[off[b][c]] = s;
  }
}

template <int CLS>
struct GsNB {
  static constexpr int NB = 1;
};

template <int LX, int CLS>
__global__ void gs_box_local_kernel(double* __restrict__ w, const BoxGS M, int zlo, int zhi, int qlo,
                                    int nrows) {
  constexpr int n1 = LX - 1;
  constexpr int NB = GsNB<CLS>::NB;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  int gx[NB], gy[NB], gz[NB];
  bool use[NB];
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int rb = (int)blockIdx.y * NB + b;  // batched index
    if (CLS == 0) {
      gz[b] = ((zlo + n1 - 1) / n1 + (int)blockIdx.z) * n1;
      gy[b] = rb;
      gx[b] = t;
      use[b] = gx[b] < M.NX && rb < nrows && gz[b] <= zhi;
    } else if (CLS == 1) {
      const int q = qlo + rb;  // the rb-th non-face plane of the range
      gz[b] = (q / (n1 - 1)) * n1 + 1 + q % (n1 - 1);
      gy[b] = (int)blockIdx.z * n1;
      gx[b] = t;
      use[b] = gx[b] < M.NX && rb < nrows && gz[b] <= zhi;
    } else {
      const int q = qlo + (int)blockIdx.z;
      gz[b] = (q / (n1 - 1)) * n1 + 1 + q % (n1 - 1);
      gy[b] = (rb / (n1 - 1)) * n1 + 1 + rb % (n1 - 1);
      gx[b] = (t + 1) * n1;
      use[b] = t < M.nx - 1 && rb < nrows && gz[b] <= zhi;
    }
    if (!use[b]) gx[b] = gy[b] = gz[b] = n1;  // any in-range node; not touched
  }
  gs_box_local_nodes<LX, NB>(w, M, gx, gy, gz, use);
}

// Local DSSUM of the owned node planes [lo, hi] (global z node-plane
// indices; every copy of those nodes lies in the slab): three launches, one
// per node class.
// class-2 nodes of non-face planes [a, b]
template <int LX>
static void gs_box_cls2(double* w, const BoxGS& M, int a, int b, cudaStream_t st) {
  constexpr int n1 = LX - 1;
  if (n1 < 2 || M.nx < 2 || b < a) return;
  const int fa = (a + n1 - 1) / n1, fb = b / n1;
  const int nnf = (b - a + 1) - (fb >= fa ? fb - fa + 1 : 0);
  if (nnf <= 0) return;
  const int a2 = (a % n1 == 0) ? a + 1 : a;
  const int qlo = (a2 / n1) * (n1 - 1) + (a2 % n1 - 1);
  gs_box_local_kernel<LX, 2><<<dim3((unsigned)((M.nx - 1 + 127) / 128),
                                    (unsigned)((int64_t)M.ny * (n1 - 1) + GsNB<2>::NB - 1) / GsNB<2>::NB,
                                    (unsigned)nnf),
                               128, 0, st>>>(w, M, a, b, qlo, M.ny * (n1 - 1));
}

// [s2lo, s2hi]: node planes whose class-2 nodes are already summed (the
// x-folding DMMA apply, ax_dmma.cuh); class 2 runs on [lo, hi] minus them
template <int LX>
static void gs_box_local_range(double* w, const BoxGS& M, int lo, int hi, cudaStream_t st,
                               int s2lo = 1, int s2hi = 0) {
  constexpr int n1 = LX - 1;
  if (hi < lo) return;
  const dim3 blk(128);
  const unsigned gxb = (unsigned)((M.NX + 127) / 128);
  // face planes in [lo, hi]
  const int f0 = (lo + n1 - 1) / n1, f1 = hi / n1;
  const auto nb = [](int64_t rows, int NB) { return (unsigned)((rows + NB - 1) / NB); };
  if (f1 >= f0)  // y: rows gy (batched), z: face planes
    gs_box_local_kernel<LX, 0><<<dim3(gxb, nb(M.NY, GsNB<0>::NB), (unsigned)(f1 - f0 + 1)), blk, 0,
                                 st>>>(w, M, lo, hi, 0, (int)M.NY);
  if (n1 > 1) {
    // non-face planes in [lo, hi]
    const int nnf = (hi - lo + 1) - (f1 >= f0 ? f1 - f0 + 1 : 0);
    const int lo2 = (lo % n1 == 0) ? lo + 1 : lo;
    const int qlo = (lo2 / n1) * (n1 - 1) + (lo2 % n1 - 1);
    if (nnf > 0) {
      // y: non-face planes (batched), z: y-face rows
      gs_box_local_kernel<LX, 1><<<dim3(gxb, nb(nnf, GsNB<1>::NB), (unsigned)(M.ny + 1)), blk, 0,
                                   st>>>(w, M, lo, hi, qlo, nnf);
      // y: non-face rows, z: non-face planes
      if (s2hi < s2lo || s2hi < lo || s2lo > hi) {
        gs_box_cls2<LX>(w, M, lo, hi, st);
      } else {
        gs_box_cls2<LX>(w, M, lo, s2lo - 1, st);
        gs_box_cls2<LX>(w, M, s2hi + 1, hi, st);
      }
    }
  }
}

template <int LX>
static cudaError_t gs_box_launch(int op, double* w, const BoxGS& M, int has_below, int has_above,
                                 double* buf, cudaStream_t st) {
  constexpr int n1 = LX - 1;
  const dim3 blk(128);
  const unsigned gxb = (unsigned)((M.NX + 127) / 128);
  switch (op) {
    case 0: {
      const int lo = (int)(M.ez0 * n1 + (has_below ? 1 : 0));
      const int hi = (int)(M.ez1 * n1 - (has_above ? 1 : 0));
      gs_box_local_range<LX>(w, M, lo, hi, st);
      break;
    }
    case 1 + AXHELM_GS_PARTIAL:
      gs_box_plane_kernel<LX, 1><<<dim3(gxb, (unsigned)M.NY, 1), blk, 0, st>>>(w, M, (int)(M.ez1 * n1), buf);
      break;
    case 1 + AXHELM_GS_FINISH:
      gs_box_plane_kernel<LX, 2><<<dim3(gxb, (unsigned)M.NY, 1), blk, 0, st>>>(w, M, (int)(M.ez0 * n1), buf);
      break;
    case 1 + AXHELM_GS_WRITE:
      gs_box_plane_kernel<LX, 3><<<dim3(gxb, (unsigned)M.NY, 1), blk, 0, st>>>(w, M, (int)(M.ez1 * n1), buf);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace axb

extern "C" int axhelm_gs_box(int op, double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1,
                             int has_below, int has_above, double* buf, void* stream) {
  if (lx < 2 || lx > 16 || nx < 1 || ny < 1 || ez1 <= ez0 || ez0 < 0)
    return set_status(AXHELM_EINVAL, "axhelm_gs_box: bad sizes");
  if (op < 0 || op > 3) return set_status(AXHELM_EINVAL, "axhelm_gs_box: unknown op %d", op);
  const int n1 = lx - 1;
  BoxGS M{nx, ny, lx, ez0, ez1, (int64_t)nx * n1 + 1, (int64_t)ny * n1 + 1};
  if (M.NY > 65535 || ez1 * n1 >= (int64_t)1 << 31 || (op == 0 && (ez1 - ez0) * n1 + 1 > 65535))
    return set_status(AXHELM_EINVAL, "axhelm_gs_box: mesh too large for the structured path");
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  switch (lx) {
#define AXB_GSB(N) \
  case N:          \
    e = gs_box_launch<N>(op, w, M, has_below, has_above, buf, st); \
    break;
    AXB_GSB(2) AXB_GSB(3) AXB_GSB(4) AXB_GSB(5) AXB_GSB(6) AXB_GSB(7) AXB_GSB(8) AXB_GSB(9)
    AXB_GSB(10) AXB_GSB(11) AXB_GSB(12) AXB_GSB(13) AXB_GSB(14) AXB_GSB(15) AXB_GSB(16)
#undef AXB_GSB
    default:
      e = cudaErrorInvalidValue;
  }
  return cuda_status(e, "axhelm_gs_box");
}

namespace axb {
// ------------------------------------------------------------------ follower
// The local DSSUM as a consumer running concurrently with the ax_helm
// kernel (on another stream): the apply publishes per-layer completion
// counters (signal_done, release); one persistent CTA per SM walks the
// slab's layers in order, waits (acquire) until layer L is complete, then
// sums the node planes of layer L — the face plane below it and its
// interior planes (the top plane too for the last layer) — while that w is
// still in L2 (the apply stores w evict-normal and streams its inputs
// evict-first).  Per node the copies are visited in the same ascending order
// as gs_box_node, so the result is bit-identical to the separate pass.
struct FollowArgs {
  double* w;
  BoxGS M;
  const unsigned* progress;
  int64_t l0, l1, lay;
  int zlo, zhi;
};

__device__ __forceinline__ bool layer_complete(const FollowArgs& F, int64_t L) {
  if (L < F.l0 || L >= F.l1) return true;
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(F.progress + (L - F.l0)) : "memory");
  return (int64_t)v >= F.lay;
}

// timing trace of the last follower launch (CTA 0): [0] start, [1 + L] the
// time layer L became available, [nl + 1] end — debug/profiling only
__device__ unsigned long long g_follow_trace[1024];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// One thread per node column (gx, gy) of the layer (grid-stride): the node
// on the face plane below layer L (copies in layers L-1 and L), then — for
// columns on a vertical element face (gx or gy a multiple of n1) — the nodes
// of layer L's interior planes, whose copies differ only by k within the
// same 2 or 4 elements (all their loads issued before any sum), and the top
// plane for the slab's last layer.
template <int LX, int PB>
__global__ void __launch_bounds__(128, 8) gs_follow_kernel(const FollowArgs F) {
  constexpr int n1 = LX - 1;
  constexpr int L2 = LX * LX;
  constexpr int L3 = LX * LX * LX;
  constexpr int64_t DX = L3 - n1;
  const BoxGS& M = F.M;
  const int NX = (int)M.NX, nx = M.nx, ny = M.ny;
  const int64_t ncol = M.NX * M.NY;
  const int64_t nl = M.ez1 - M.ez0;
  const int64_t DY = (int64_t)nx * L3 - n1 * LX;
  const int64_t DZ = (int64_t)nx * ny * L3 - n1 * L2;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t tg = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double* __restrict__ w = F.w;
  const bool trace = blockIdx.x == 0 && threadIdx.x == 0 && nl + 2 <= 1024;
  if (trace) g_follow_trace[0] = gtimer();
  for (int64_t L = 0; L < nl; ++L) {
    const int64_t gzf = (M.ez0 + L) * n1;  // face plane below layer L
    const bool face_ok = gzf >= F.zlo && gzf <= F.zhi;
    const bool top_ok = (L == nl - 1) && gzf + n1 <= F.zhi;
    if (threadIdx.x == 0) {  // the face plane below layer L also has copies in layer L - 1
      uint64_t t0 = 0;
      while (!layer_complete(F, L - 1) || !layer_complete(F, L)) {
        __nanosleep(256);
        const uint64_t t = gtimer();
        if (t0 == 0) t0 = t;
        if (t - t0 > 10000000000ull) __trap();  // 10 s without progress: fail loudly, never hang
      }
      if (trace) g_follow_trace[1 + L] = gtimer();
    }
    __syncthreads();
    for (int64_t col = tg; col < ncol; col += T) {
      const int gy = (int)(col / NX), gx = (int)(col - (int64_t)gy * NX);
      const int qx = gx / n1, rx = gx - qx * n1, qy = gy / n1, ry = gy - qy * n1;
      const int ex0 = (rx == 0 && qx > 0) ? qx - 1 : (qx < nx ? qx : nx - 1);
      const int ey0 = (ry == 0 && qy > 0) ? qy - 1 : (qy < ny ? qy : ny - 1);
      const int cx = (rx == 0 && qx > 0 && qx < nx) ? 2 : 1;
      const int cy = (ry == 0 && qy > 0 && qy < ny) ? 2 : 1;
      // copy (layer L, ey0, ex0) at k = 0
      const int64_t off = ((L * ny + ey0) * (int64_t)nx + ex0) * L3 + (int64_t)(gy - ey0 * n1) * LX +
                          (gx - ex0 * n1);
      if (face_ok) {
        const int cz = L > 0 ? 2 : 1;
        if (cx * cy * cz >= 2) {
          double v[8];
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // c = (dz, dy, dx): ascending (ez, ey, ex)
            const int dz = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
            const bool ok = dx < cx && dy < cy && (cz == 2 ? true : dz == 1);
            v[c] = ok ? __ldcg(w + off - (1 - dz) * DZ + dy * DY + dx * DX) : 0.0;
          }
          double sum = 0.0;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int dz = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
            if (dx < cx && dy < cy && (cz == 2 || dz == 1)) sum = __dadd_rn(sum, v[c]);
          }
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const int dz = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
            if (dx < cx && dy < cy && (cz == 2 || dz == 1)) __stcg(w + off - (1 - dz) * DZ + dy * DY + dx * DX, sum);
          }
        }
      }
      if (cx * cy < 2) continue;  // interior-plane nodes off the vertical faces are unshared
      const int rend = top_ok ? n1 : n1 - 1;
#pragma unroll
      for (int r0 = 1; r0 <= n1; r0 += PB) {
        if (r0 > rend) break;
        double v[PB][4];
#pragma unroll
        for (int b = 0; b < PB; ++b)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int dy = c >> 1, dx = c & 1;
            const bool ok = r0 + b <= rend && dx < cx && dy < cy;
            v[b][c] = ok ? __ldcg(w + off + (r0 + b) * L2 + dy * DY + dx * DX) : 0.0;
          }
#pragma unroll
        for (int b = 0; b < PB; ++b) {
          if (r0 + b > rend) break;
          double sum = 0.0;
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if ((c & 1) < cx && (c >> 1) < cy) sum = __dadd_rn(sum, v[b][c]);
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if ((c & 1) < cx && (c >> 1) < cy) __stcg(w + off + (r0 + b) * L2 + (c >> 1) * DY + (c & 1) * DX, sum);
        }
      }
    }
  }
  if (trace) g_follow_trace[nl + 1] = gtimer();
}

cudaError_t gs_box_follow(double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1, int64_t zlo,
                          int64_t zhi, const unsigned* progress, int64_t l0, int64_t l1, cudaStream_t st) {
  const int n1 = lx - 1;
  BoxGS M{nx, ny, lx, ez0, ez1, (int64_t)nx * n1 + 1, (int64_t)ny * n1 + 1};
  FollowArgs F{w, M, progress, l0, l1, (int64_t)nx * ny, (int)zlo, (int)zhi};
  if (zhi < zlo) return cudaSuccess;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // two 128-thread CTAs (<= 64 registers) per SM: they must fit beside the
  // apply's persistent CTAs; they spin only in thread 0, with nanosleep,
  // while the other threads wait at a barrier)
  // The follower never leaves an SM until the apply has finished, so it must
  // not pin an SM to an L1-heavy carveout the apply's CTAs cannot use: ask
  // for the maximum shared-memory carveout, like the apply kernels.
  switch (lx) {
#define AXB_FOL(N) \
  case N:          \
    cudaFuncSetAttribute(gs_follow_kernel<N, 4>, cudaFuncAttributePreferredSharedMemoryCarveout, \
                         (int)cudaSharedmemCarveoutMaxShared); \
    gs_follow_kernel<N, 4><<<2 * sms, 128, 0, st>>>(F); \
    break;
    AXB_FOL(2) AXB_FOL(3) AXB_FOL(4) AXB_FOL(5) AXB_FOL(6) AXB_FOL(7) AXB_FOL(8) AXB_FOL(9)
    AXB_FOL(10) AXB_FOL(11) AXB_FOL(12) AXB_FOL(13) AXB_FOL(14) AXB_FOL(15) AXB_FOL(16)
#undef AXB_FOL
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}
}  // namespace axb

namespace axb {
// enqueue the local DSSUM of node planes [zlo, zhi] (validated by the caller)
cudaError_t gs_box_range(double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1, int64_t zlo,
                         int64_t zhi, cudaStream_t st, int64_t s2lo, int64_t s2hi) {
  const int n1 = lx - 1;
  BoxGS M{nx, ny, lx, ez0, ez1, (int64_t)nx * n1 + 1, (int64_t)ny * n1 + 1};
  if (zhi < zlo) return cudaSuccess;
  switch (lx) {
#define AXB_GSR(N) \
  case N:          \
    gs_box_local_range<N>(w, M, (int)zlo, (int)zhi, st, (int)s2lo, (int)s2hi); \
    break;
    AXB_GSR(2) AXB_GSR(3) AXB_GSR(4) AXB_GSR(5) AXB_GSR(6) AXB_GSR(7) AXB_GSR(8) AXB_GSR(9)
    AXB_GSR(10) AXB_GSR(11) AXB_GSR(12) AXB_GSR(13) AXB_GSR(14) AXB_GSR(15) AXB_GSR(16)
#undef AXB_GSR
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

const char* gs_box_range_check(int nx, int ny, int lx, int64_t ez0, int64_t ez1, int64_t zlo,
                               int64_t zhi) {
  if (lx < 2 || lx > 16 || nx < 1 || ny < 1 || ez1 <= ez0 || ez0 < 0) return "bad sizes";
  const int n1 = lx - 1;
  if (zhi >= zlo && (zlo < ez0 * n1 || zhi > ez1 * n1)) return "node planes outside the slab";
  if ((int64_t)ny * n1 + 1 > 65535 || ez1 * n1 >= (int64_t)1 << 31 || zhi - zlo + 1 > 65535)
    return "mesh too large for the structured path";
  return nullptr;
}
}  // namespace axb

// Local DSSUM restricted to node planes [zlo, zhi] (global z node-plane
// indices inside the slab).  Lets a caller sum the planes whose copies are
// all computed while the w they touch is still in L2 (axhelm_ax_gs_box).
// Same per-node order as op 0.
// debug/profiling: the follower alone on a finished apply (every layer complete)
extern "C" int axhelm_debug_follow_only(double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1,
                                        int64_t zlo, int64_t zhi, void* stream) {
  return cuda_status(axb::gs_box_follow(w, nx, ny, lx, ez0, ez1, zlo, zhi, nullptr, 0, 0,
                                        (cudaStream_t)stream), "axhelm_debug_follow_only");
}

extern "C" int axhelm_debug_follow_trace(unsigned long long* out, int n) {
  if (n > 1024) n = 1024;
  return cuda_status(cudaMemcpyFromSymbol(out, axb::g_follow_trace, sizeof(unsigned long long) * n),
                     "axhelm_debug_follow_trace");
}

extern "C" int axhelm_gs_box_range(double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1,
                                   int64_t zlo, int64_t zhi, void* stream) {
  if (const char* why = axb::gs_box_range_check(nx, ny, lx, ez0, ez1, zlo, zhi))
    return set_status(AXHELM_EINVAL, "axhelm_gs_box_range: %s", why);
  return cuda_status(axb::gs_box_range(w, nx, ny, lx, ez0, ez1, zlo, zhi, (cudaStream_t)stream),
                     "axhelm_gs_box_range");
}

// ------------------------------------------------------------ peer memory
// IPC-shareable device allocations for the peer-memory interface exchange
// (dist.PeerExchange): allocated and zeroed here, exported as a 64-byte
// cudaIpcMemHandle, opened by the neighbouring ranks (NVLink peer mapping).
extern "C" int axhelm_peer_alloc(int64_t bytes, void** ptr, void* handle) {
  if (bytes <= 0 || !ptr || !handle) return set_status(AXHELM_EINVAL, "axhelm_peer_alloc: bad arguments");
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, (size_t)bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), *ptr);
  return cuda_status(e, "axhelm_peer_alloc");
}

extern "C" int axhelm_peer_open(const void* handle, void** ptr) {
  if (!handle || !ptr) return set_status(AXHELM_EINVAL, "axhelm_peer_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "axhelm_peer_open");
}

extern "C" int axhelm_peer_close(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr), "axhelm_peer_close"); }

extern "C" int axhelm_peer_free(void* ptr) { return cuda_status(cudaFree(ptr), "axhelm_peer_free"); }

// One interface-plane step of the structured DSSUM with peer buffers
// (op = AXHELM_GS_PARTIAL / _FINISH / _WRITE, see gs_box_plane_peer_kernel).
__global__ void peer_seq_bump_kernel(unsigned long long* ctr) { *ctr += 1; }

extern "C" int axhelm_peer_seq_bump(unsigned long long* ctr, void* stream) {
  if (!ctr) return set_status(AXHELM_EINVAL, "axhelm_peer_seq_bump: null counter");
  peer_seq_bump_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(ctr);
  return cuda_status(cudaGetLastError(), "axhelm_peer_seq_bump");
}

extern "C" int axhelm_gs_box_peer(int op, double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1,
                                  const double* in, double* out, const unsigned long long* wait_flag,
                                  unsigned long long* signal_flag, unsigned long long seq,
                                  unsigned* counter, const unsigned long long* seq_dev, void* stream) {
  if (lx < 2 || lx > 16 || nx < 1 || ny < 1 || ez1 <= ez0 || ez0 < 0)
    return set_status(AXHELM_EINVAL, "axhelm_gs_box_peer: bad sizes");
  if (op < 0 || op > 2) return set_status(AXHELM_EINVAL, "axhelm_gs_box_peer: unknown op %d", op);
  if ((op != AXHELM_GS_WRITE && (!out || !signal_flag || !counter)) ||
      (op != AXHELM_GS_PARTIAL && (!in || !wait_flag)))
    return set_status(AXHELM_EINVAL, "axhelm_gs_box_peer: missing buffer for op %d", op);
  const int n1 = lx - 1;
  BoxGS M{nx, ny, lx, ez0, ez1, (int64_t)nx * n1 + 1, (int64_t)ny * n1 + 1};
  if (M.NY > 65535) return set_status(AXHELM_EINVAL, "axhelm_gs_box_peer: mesh too large");
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 blk(128), grd((unsigned)((M.NX + 127) / 128), (unsigned)M.NY, 1);
  const int gz = (int)((op == AXHELM_GS_FINISH ? ez0 : ez1) * n1);
  switch (lx) {
#define AXB_PEER(N)                                                                                       \
  case N:                                                                                                 \
    /* waiting CTAs must not pin an SM to an L1-heavy carveout the apply's */                            \
    /* persistent CTAs (running concurrently on another stream) cannot use */                            \
    cudaFuncSetAttribute(axb::gs_box_plane_peer_kernel<N, 2>,                                             \
                         cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared); \
    cudaFuncSetAttribute(axb::gs_box_plane_peer_kernel<N, 3>,                                             \
                         cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared); \
    if (op == AXHELM_GS_PARTIAL)                                                                          \
      axb::gs_box_plane_peer_kernel<N, 1><<<grd, blk, 0, st>>>(w, M, gz, in, out, wait_flag, signal_flag, \
                                                               seq, counter, seq_dev);                    \
    else if (op == AXHELM_GS_FINISH)                                                                      \
      axb::gs_box_plane_peer_kernel<N, 2><<<grd, blk, 0, st>>>(w, M, gz, in, out, wait_flag, signal_flag, \
                                                               seq, counter, seq_dev);                    \
    else                                                                                                  \
      axb::gs_box_plane_peer_kernel<N, 3><<<grd, blk, 0, st>>>(w, M, gz, in, out, wait_flag, signal_flag, \
                                                               seq, counter, seq_dev);                    \
    break;
    AXB_PEER(2) AXB_PEER(3) AXB_PEER(4) AXB_PEER(5) AXB_PEER(6) AXB_PEER(7) AXB_PEER(8) AXB_PEER(9)
    AXB_PEER(10) AXB_PEER(11) AXB_PEER(12) AXB_PEER(13) AXB_PEER(14) AXB_PEER(15) AXB_PEER(16)
#undef AXB_PEER
  }
  return cuda_status(cudaGetLastError(), "axhelm_gs_box_peer");
}

// ------------------------------------------------------- peer all-reduce
// Sum of a few doubles over all ranks through peer memory (PCG's dot
// products): every rank writes its values into slot [parity][rank] of every
// rank's region (bases[q] + off) and raises flag [rank] there with a
// system-scope release store; then waits until all its flags reach seq and
// sums the slots in rank order — the same bits on every rank, no NCCL.
// Two parity buffers: a rank can run at most one call ahead of another
// rank's read (its next call needs that rank's next write).
namespace axb {
constexpr int PEER_MAXW = 64;
__global__ void peer_allreduce_kernel(const double* v, int n, double* out,
                                      const unsigned long long* __restrict__ bases, int64_t off,
                                      int world, int rank, unsigned long long seq,
                                      unsigned long long* seq_dev) {
  const int t = threadIdx.x;
  if (seq_dev) seq = *seq_dev + 1;  // device-side sequence (graph replays advance it)
  const int par = (int)(seq & 1);
  double val[4];
  for (int j = 0; j < 4; ++j) val[j] = j < n ? v[j] : 0.0;
  if (t < world) {  // write my values to rank t, then raise its flag [rank]
    unsigned char* b = reinterpret_cast<unsigned char*>(bases[t]) + off;
    unsigned long long* flags = reinterpret_cast<unsigned long long*>(b);
    double* data = reinterpret_cast<double*>(b + 8 * PEER_MAXW) + ((size_t)par * PEER_MAXW + rank) * 4;
    for (int j = 0; j < n; ++j) data[j] = val[j];
    __threadfence_system();
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flags + rank), "l"(seq) : "memory");
  }
  __syncthreads();
  unsigned char* mine = reinterpret_cast<unsigned char*>(bases[rank]) + off;
  if (t < world) {  // wait for rank t's values in my region
    const unsigned long long* f = reinterpret_cast<const unsigned long long*>(mine) + t;
    unsigned long long x = 0, t0 = 0;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(f) : "memory");
      if (x >= seq) break;
      __nanosleep(64);
      const unsigned long long now = peer_timer();
      if (t0 == 0) t0 = now;
      if (now - t0 > 10000000000ull) __trap();
    }
  }
  __syncthreads();
  if (t == 0) {
    const double* data = reinterpret_cast<const double*>(mine + 8 * PEER_MAXW) + (size_t)par * PEER_MAXW * 4;
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int q = 0; q < world; ++q) s += data[q * 4 + j];
      out[j] = s;
    }
    if (seq_dev) *seq_dev = seq;
  }
}
}  // namespace axb

// bytes of the all-reduce area a peer region must reserve at `off`
extern "C" int64_t axhelm_peer_allreduce_bytes(void) {
  return 8 * axb::PEER_MAXW + 2 * axb::PEER_MAXW * 4 * 8;
}

extern "C" int axhelm_peer_allreduce(const double* v, int n, double* out, const unsigned long long* bases,
                                     int64_t off, int world, int rank, unsigned long long seq,
                                     unsigned long long* seq_dev, void* stream) {
  if (n < 1 || n > 4 || world < 1 || world > axb::PEER_MAXW || rank < 0 || rank >= world || !v || !out ||
      !bases)
    return set_status(AXHELM_EINVAL, "axhelm_peer_allreduce: bad arguments");
  axb::peer_allreduce_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(v, n, out, bases, off, world, rank, seq,
                                                                  seq_dev);
  return cuda_status(cudaGetLastError(), "axhelm_peer_allreduce");
}
