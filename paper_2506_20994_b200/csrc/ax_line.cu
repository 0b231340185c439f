// Launch side of the v11 line kernel (ax_line.cuh), lx 9..16, both modes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "../../include/axhelm.h"
#include "ax_launch.h"
#include "ax_line.cuh"
#include "ax_ws.cuh"

namespace axb {

// AXL_PF overrides the per-lx L2 prefetch point of the geometry (LineGP::PF;
// 0 none, 1 after the combine for the next element, 2 at element start for
// the element, 3 after stage 1 for the next element)
static int g_line_pf = [] {
  const char* v = getenv("AXL_PF");
  return v ? atoi(v) : -1;
}();

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time libcuda dependency)
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// u viewed as [nel * lx^2 rows][lx columns]; box RSU x lx^2 (columns past
// lx are out of bounds and arrive as zeros: the padded row layout)
template <int LX>
static cudaError_t encode_u_map(CUtensorMap* map, const double* u, int64_t nel) {
  using C = LineCfg<LX>;
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {(cuuint64_t)LX, (cuuint64_t)(nel * LX * LX)};
  const cuuint64_t strides[1] = {(cuuint64_t)LX * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)C::RSU, (cuuint32_t)(LX * LX)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(u), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int LX, bool FAST>
static cudaError_t launch_line_t(const AxPtrs& A, int64_t nel, cudaStream_t st, const double* const* hm) {
  using C = LineCfg<LX>;
  static DevCache occ;
  int blocks_per_sm = 0;
  cudaError_t e = ctas_per_sm(occ, ax_line<LX, FAST>, C::NT, C::SMEM, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  LParams<LX> P;
  P.A = A;
  P.nel = nel;
  P.pf = g_line_pf;
  memset(&P.tmap, 0, sizeof P.tmap);
  if constexpr (LineCfg<LX>::UPAD) {
    if ((e = encode_u_map<LX>(&P.tmap, A.u, nel)) != cudaSuccess) return e;
  }
  double m6[6 * LX * LX];
  bool have = false;
  if ((e = host_matrices(A, LX, hm, st, m6, &P.stale, &have)) != cudaSuccess) return e;
  if (have) {
    memcpy(P.m, m6, sizeof P.m);
  } else {  // poison: every CTA's verification fails -> shared-memory path
    const long long bits = 0x7ff4deadbeef0001LL;
    double poison;
    memcpy(&poison, &bits, sizeof poison);
    for (int q = 0; q < 6 * LX * LX; ++q) (&P.m[0][0])[q] = poison;
  }
  const int64_t groups = (nel + C::EPC - 1) / C::EPC;
  int64_t grid = (int64_t)blocks_per_sm * num_sms();
  if (grid > groups) grid = groups;
  ax_line<LX, FAST><<<(unsigned)grid, C::NT, C::SMEM, st>>>(P);
  return cudaGetLastError();
}

// v12 warp-specialised variant (ax_ws.cuh), lx 9 / 10: one CTA per SM.
// WsPick: consumer groups NG and planes per ring chunk G; the default for
// fast mode, where it beats v11 on the same box (profiles/r02_ab_ws_kernel.txt:
// lx 9 1.07x, lx 10 1.06x); strict keeps v11 (AXHELM_KERNEL=ws forces v12
// for both modes, =line forces v11).
template <int LX, bool FAST>
struct WsPick {
  static constexpr bool ON = FAST;
  static constexpr int NG = LX == 9 ? 3 : 2;
  static constexpr int G = LX == 9 ? 9 : 4;
};

template <int LX, bool FAST>
static cudaError_t launch_ws_t(const AxPtrs& A, int64_t nel, cudaStream_t st, const double* const* hm) {
  constexpr int NG = WsPick<LX, FAST>::NG, G = WsPick<LX, FAST>::G;
  using W = WsCfg<LX, NG, G>;
  static DevCache occ;
  int blocks_per_sm = 0;
  cudaError_t e = ctas_per_sm(occ, ax_ws<LX, FAST, NG, G>, W::NT, W::SMEM, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  LParams<LX> P;
  P.A = A;
  P.nel = nel;
  P.pf = -1;
  memset(&P.tmap, 0, sizeof P.tmap);
  double m6[6 * LX * LX];
  bool have = false;
  if ((e = host_matrices(A, LX, hm, st, m6, &P.stale, &have)) != cudaSuccess) return e;
  if (have) {
    memcpy(P.m, m6, sizeof P.m);
  } else {
    const long long bits = 0x7ff4deadbeef0001LL;
    double poison;
    memcpy(&poison, &bits, sizeof poison);
    for (int q = 0; q < 6 * LX * LX; ++q) (&P.m[0][0])[q] = poison;
  }
  int64_t grid = (int64_t)num_sms();
  if (grid > nel) grid = nel;
  ax_ws<LX, FAST, NG, G><<<(unsigned)grid, W::NT, W::SMEM, st>>>(P);
  return cudaGetLastError();
}

// forced: v12 for lx 9 / 10 in both modes (AXHELM_KERNEL=ws); else WsPick
bool ws_selected(const AxPtrs& A, int64_t nel, int lx, int mode, bool forced) {
  if ((lx != 9 && lx != 10) || ((uintptr_t)A.u & 15u) != 0 || nel <= 0) return false;
  if (forced) return true;
  const bool fast = mode == AXHELM_FAST;
  return lx == 9 ? (fast ? WsPick<9, true>::ON : WsPick<9, false>::ON)
                 : (fast ? WsPick<10, true>::ON : WsPick<10, false>::ON);
}

cudaError_t launch_ws(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st,
                      const double* const* hm) {
  const bool fast = mode == AXHELM_FAST;
  switch (lx) {
#define AXB_WS(N) \
  case N:         \
    return fast ? launch_ws_t<N, true>(A, nel, st, hm) : launch_ws_t<N, false>(A, nel, st, hm);
    AXB_WS(9) AXB_WS(10)
#undef AXB_WS
    default:
      return cudaErrorInvalidValue;
  }
}

// Default for lx 9..16, both modes, and lx = 7 fast (same-box A/B against
// v4, profiles/r02_ab_line_*: at lx 5, 6, 8 and 7 strict v4 / v6 stay ahead).
bool line_selected(const AxPtrs& A, int64_t nel, int lx, int mode) {
  if (lx < 7 || lx == 8 || lx > 16 || ((uintptr_t)A.u & 15u) != 0) return false;
  if (nel * lx * lx >= (int64_t)1 << 31) return false;  // tensor-map row coordinate (int32)
  return lx >= 9 || mode == AXHELM_FAST;  // lx = 7: fast only
}

cudaError_t launch_line(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st,
                        const double* const* hm) {
  if (nel == 0) return cudaSuccess;
  const bool fast = mode == AXHELM_FAST;
  switch (lx) {
#define AXB_LINE(N) \
  case N:           \
    return fast ? launch_line_t<N, true>(A, nel, st, hm) : launch_line_t<N, false>(A, nel, st, hm);
    AXB_LINE(7) AXB_LINE(9) AXB_LINE(10) AXB_LINE(11) AXB_LINE(12) AXB_LINE(13) AXB_LINE(14) AXB_LINE(15) AXB_LINE(16)
#undef AXB_LINE
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace axb
