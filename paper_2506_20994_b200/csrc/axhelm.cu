// libaxhelm_sm100.so — C ABI entry points and launch dispatch for the B200
// ax_helm path.  See include/axhelm.h for the contract and the reference
// interfaces each entry replaces.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/axhelm.h"
#include "ax_kernels.cuh"
#include "ax_launch.h"

#ifndef AXHELM_VERSION
#define AXHELM_VERSION "0.1.0"
#endif

namespace axb {

// ------------------------------------------------------------ error state

static thread_local int t_status = AXHELM_OK;
static thread_local char t_msg[512] = "";

int set_status(int st, const char* fmt, ...) {
  t_status = st;
  if (st == AXHELM_OK) {
    t_msg[0] = 0;
    return st;
  }
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(t_msg, sizeof t_msg, fmt, ap);
  va_end(ap);
  return st;
}

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return set_status(AXHELM_OK, "");
  return set_status(AXHELM_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

// ---------------------------------------------------------------- launch

template <int LX, bool FAST>
static cudaError_t launch_kwalk(const AxPtrs& A, int64_t nel, cudaStream_t st) {
  using C = KCfg<LX>;
  static bool attr_done = false;  // benign race: idempotent attribute set
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ax_kwalk<LX, FAST>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  const int64_t blocks = (nel + C::EPB - 1) / C::EPB;
  if (blocks > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  ax_kwalk<LX, FAST><<<(unsigned)blocks, C::NT, C::SMEM, st>>>(A, nel);
  return cudaGetLastError();
}

template <int LX>
static cudaError_t launch_lx(const AxPtrs& A, int64_t nel, int mode, cudaStream_t st) {
  return mode == AXHELM_FAST ? launch_kwalk<LX, true>(A, nel, st)
                             : launch_kwalk<LX, false>(A, nel, st);
}

cudaError_t launch_ax(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st) {
  if (nel == 0) return cudaSuccess;
  switch (lx) {
#define AXB_CASE(N) \
  case N:           \
    return launch_lx<N>(A, nel, mode, st);
    AXB_CASE(2) AXB_CASE(3) AXB_CASE(4) AXB_CASE(5) AXB_CASE(6) AXB_CASE(7)
    AXB_CASE(8) AXB_CASE(9) AXB_CASE(10) AXB_CASE(11) AXB_CASE(12)
    AXB_CASE(13) AXB_CASE(14) AXB_CASE(15) AXB_CASE(16)
#undef AXB_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

static int g_mode = [] {
  const char* v = getenv("AXHELM_FP");
  return (v && (!strcmp(v, "fast") || !strcmp(v, "FAST"))) ? AXHELM_FAST : AXHELM_STRICT;
}();

int default_mode() { return g_mode; }

}  // namespace axb

using namespace axb;

// ===================================================================== ABI

extern "C" {

int axhelm_apply(double* wd, const double* ud, const double* dxd, const double* dyd,
                 const double* dzd, const double* dxtd, const double* dytd,
                 const double* dztd, const double* h1d, const double* g11d,
                 const double* g22d, const double* g33d, const double* g12d,
                 const double* g13d, const double* g23d, int64_t nel, int lx,
                 int mode, void* stream) {
  if (lx < 2 || lx > 16) return set_status(AXHELM_EINVAL, "lx=%d outside [2, 16]", lx);
  if (nel < 0) return set_status(AXHELM_EINVAL, "nel=%lld is negative", (long long)nel);
  if (mode != AXHELM_STRICT && mode != AXHELM_FAST)
    return set_status(AXHELM_EINVAL, "unknown mode %d", mode);
  if (nel == 0) return set_status(AXHELM_OK, "");
  const double* ptrs[15] = {wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd,
                            h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  for (int q = 0; q < 15; ++q)
    if (!ptrs[q]) return set_status(AXHELM_EINVAL, "argument %d is NULL", q);
  AxPtrs A{wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd, h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  return cuda_status(launch_ax(A, nel, lx, mode, (cudaStream_t)stream), "axhelm_apply");
}

void __dace_ax_helm(double* AXH_RESTRICT wd, const double* AXH_RESTRICT ud,
                    const double* AXH_RESTRICT dxd, const double* AXH_RESTRICT dyd,
                    const double* AXH_RESTRICT dzd, const double* AXH_RESTRICT dxtd,
                    const double* AXH_RESTRICT dytd, const double* AXH_RESTRICT dztd,
                    const double* AXH_RESTRICT h1d, const double* AXH_RESTRICT g11d,
                    const double* AXH_RESTRICT g22d, const double* AXH_RESTRICT g33d,
                    const double* AXH_RESTRICT g12d, const double* AXH_RESTRICT g13d,
                    const double* AXH_RESTRICT g23d, int nelv, int lx) {
  const double* ptrs[15] = {wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd,
                            h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  host_or_device_apply(ptrs, (int64_t)nelv, lx, g_mode);
}

int axhelm_apply_sync(double* wd, const double* ud, const double* dxd, const double* dyd,
                      const double* dzd, const double* dxtd, const double* dytd,
                      const double* dztd, const double* h1d, const double* g11d,
                      const double* g22d, const double* g33d, const double* g12d,
                      const double* g13d, const double* g23d, int64_t nel, int lx,
                      int mode) {
  if (mode != AXHELM_STRICT && mode != AXHELM_FAST)
    return set_status(AXHELM_EINVAL, "unknown mode %d", mode);
  const double* ptrs[15] = {wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd,
                            h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  return host_or_device_apply(ptrs, nel, lx, mode);
}

int axhelm_set_mode(int mode) {
  if (mode != AXHELM_STRICT && mode != AXHELM_FAST)
    return set_status(AXHELM_EINVAL, "unknown mode %d", mode);
  g_mode = mode;
  return set_status(AXHELM_OK, "");
}

int axhelm_get_mode(void) { return g_mode; }
int axhelm_last_status(void) { return t_status; }
const char* axhelm_last_error(void) { return t_msg; }
const char* axhelm_version(void) { return "libaxhelm_sm100 " AXHELM_VERSION " (sm_100a, FP64)"; }

int64_t axhelm_bytes_model(int64_t nel, int lx) {
  return 72LL * nel * (int64_t)lx * lx * lx;
}

int64_t axhelm_flops_model(int64_t nel, int lx) {
  return nel * (int64_t)lx * lx * lx * (12LL * lx + 18);
}

}  // extern "C"
