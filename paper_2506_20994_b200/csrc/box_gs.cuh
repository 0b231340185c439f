// Structured-brick node geometry shared by the DSSUM kernels (mesh_gs.cu)
// and the PCG's gather-update (cg.cu): the local copies of a global node of
// an nx x ny x nz brick's z-slab, in ascending local (flat [e][k][j][i])
// index — the summation order of the DSSUM contract.
#pragma once

#include <cstdint>

namespace axb {

struct BoxGS {
  int nx, ny, lx;
  int64_t ez0, ez1;  // slab element layers
  int64_t NX, NY;
};

// element range of global node coordinate g along an axis with ne elements
__device__ __forceinline__ void node_elems(int64_t g, int n1, int64_t lo, int64_t hi, int64_t& e0,
                                           int64_t& e1) {
  // elements e with e*n1 <= g <= (e+1)*n1 (inclusive range), clipped to [lo, hi)
  e0 = (g % n1 == 0) ? g / n1 - 1 : g / n1;
  e1 = g / n1;
  if (e0 < lo) e0 = lo;
  if (e1 > hi - 1) e1 = hi - 1;
}

// Copies of node (gx, gy, gz): along each axis the node lies in one element,
// or in two when it sits on an interior element face.  The first copy's flat
// offset is computed once; the others differ by compile-time strides
// (next element in x: +L3 - n1, in y: +nx L3 - n1 LX, in z: +nx ny L3 - n1 LX^2).
template <int LX>
__device__ __forceinline__ void gs_box_copies(const BoxGS& M, int gx, int gy, int gz, int64_t& off0,
                                              int& cx, int& cy, int& cz, int64_t& DY, int64_t& DZ) {
  constexpr int n1 = LX - 1;
  constexpr int L3 = LX * LX * LX;
  const int qx = gx / n1, rx = gx - qx * n1;
  const int qy = gy / n1, ry = gy - qy * n1;
  const int qz = gz / n1, rz = gz - qz * n1;
  int ex0 = (rx == 0) ? qx - 1 : qx, ey0 = (ry == 0) ? qy - 1 : qy, ez0 = (rz == 0) ? qz - 1 : qz;
  int ex1 = min(qx, M.nx - 1), ey1 = min(qy, M.ny - 1), ez1 = min(qz, (int)M.ez1 - 1);
  ex0 = max(ex0, 0);
  ey0 = max(ey0, 0);
  ez0 = max(ez0, (int)M.ez0);
  cx = ex1 - ex0 + 1;
  cy = ey1 - ey0 + 1;
  cz = ez1 - ez0 + 1;
  const int64_t e = ((int64_t)(ez0 - M.ez0) * M.ny + ey0) * M.nx + ex0;
  off0 = e * L3 + ((gz - ez0 * n1) * LX + (gy - ey0 * n1)) * LX + (gx - ex0 * n1);
  DY = (int64_t)M.nx * L3 - n1 * LX;
  DZ = (int64_t)M.nx * M.ny * L3 - n1 * LX * LX;
}

}  // namespace axb
