// libaxhelm_sm100.so — C ABI entry points and launch dispatch for the B200
// ax_helm path.  See include/axhelm.h for the contract and the reference
// interfaces each entry replaces.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <mutex>

#include "../../include/axhelm.h"
#include "ax_kernels.cuh"
#include "ax_tma.cuh"
#include "ax_tma2.cuh"
#include "ax_dmma.cuh"
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

// ------------------------------------------------------- per-device state
//
// Launch caches (max-dynamic-smem attribute done, resident CTAs per SM, SM
// count) are per device: cudaFuncSetAttribute applies to the current
// device's context only, so a process driving several GPUs needs one entry
// per device.  Entries are written once (idempotent, benign race).
// ---------------------------------------------------------------- launch

// Kernel variant (A/B switch for profiling): AXHELM_KERNEL = pf (v2,
// L2-prefetching k-walk), tma2 (v4, TMA ring + constant-bank dz/dzt
// + k-split), dmma (v6, FP64 tensor cores; fast mode, lx = 8), line (v11,
// lx 7 / 9..16) or ws (v12, lx 9 / 10).  Default ("auto"): v6 for fast lx
// = 8, v12 for fast lx 9 / 10, v11 for the other lx 9..16 and fast lx = 7
// (u 16-B aligned), v4 for every other lx <= 15 (16-B aligned fields), else
// v2.  (v1 = the k-walk without prefetch, v3 = v4
// without its refinements and v5 = row per thread were measured and
// retired.)
// AXHELM_PF (1..3, lx = 8 only) sets v2's prefetch distance in groups.
static int g_variant = [] {
  const char* v = getenv("AXHELM_KERNEL");
  if (v && !strcmp(v, "pf")) return 2;
  if (v && !strcmp(v, "tma2")) return 4;
  if (v && !strcmp(v, "dmma")) return 6;
  if (v && !strcmp(v, "line")) return 11;
  if (v && !strcmp(v, "ws")) return 12;
  return 0;  // auto
}();
static int g_pf = [] {
  const char* v = getenv("AXHELM_PF");
  int d = v ? atoi(v) : 1;
  return (d >= 1 && d <= 3) ? d : 1;
}();
static DevCache g_num_sms;
static bool aligned16(const AxPtrs& A);
// AXHELM_CTAS_PER_SM caps the persistent kernels' resident CTAs per SM
// (tuning knob; 0 = occupancy limit)
static int g_cta_cap = [] {
  const char* v = getenv("AXHELM_CTAS_PER_SM");
  return v ? atoi(v) : 0;
}();
int cap_ctas(int b) { return (g_cta_cap > 0 && g_cta_cap < b) ? g_cta_cap : b; }

int num_sms() {
  const int dev = cur_dev();
  if (dev < 0) return 1;
  int n = g_num_sms.v[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 1;
    g_num_sms.v[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}


// ---- host copies of the t-direction matrices for the parameter block (v4)
//
// The kernel verifies the copy against the device arrays and falls back to
// them (flagging *stale) if they differ, so a stale cache costs speed, never
// correctness.  The cache never blocks the caller: a miss enqueues an async
// D2H copy into the entry's pinned slot on the caller's stream (skipped while
// the stream is being captured into a CUDA graph) and that launch runs the
// kernel's shared-memory path; later launches use the copy once its event
// has completed.  axhelm_apply therefore stays purely stream-ordered.
struct MatEntry {
  const double* m[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int lx = 0;
  int dev = -1;
  bool ready = false;
  uint64_t used = 0;
  double* h = nullptr;  // pinned: matrix q at [q * 256, q * 256 + lx * lx)
  cudaEvent_t ev = nullptr;
};
static std::mutex g_mat_mu;
static MatEntry g_mat[16];
static uint64_t g_mat_clock = 0;
static int* g_stale = nullptr;  // mapped pinned host flag

static const double* mat_ptr(const AxPtrs& A, int q) {
  return q == 0 ? A.dx : q == 1 ? A.dy : q == 2 ? A.dz : q == 3 ? A.dxt : q == 4 ? A.dyt : A.dzt;
}

cudaError_t host_matrices(const AxPtrs& A, int lx, const double* const* hm, cudaStream_t st,
                          double* out, int** stale, bool* have) {
  const size_t n = (size_t)lx * lx;
  std::lock_guard<std::mutex> lock(g_mat_mu);
  *have = false;
  *stale = nullptr;
  if (!g_stale) {
    cudaError_t e = cudaHostAlloc(&g_stale, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return e;
    *g_stale = 0;
  }
  if (hm && hm[0] && hm[1] && hm[2] && hm[3] && hm[4] && hm[5]) {  // caller's host copies
    for (int q = 0; q < 6; ++q) memcpy(out + q * n, hm[q], n * sizeof(double));
    *stale = g_stale;
    *have = true;
    return cudaSuccess;
  }
  if (*(volatile int*)g_stale) {  // a kernel saw a changed matrix: drop every copy
    for (auto& m : g_mat) {
      for (auto& p : m.m) p = nullptr;
      m.ready = false;
    }
    *(volatile int*)g_stale = 0;
  }
  const int dev = cur_dev();
  MatEntry* hit = nullptr;
  MatEntry* lru = &g_mat[0];
  for (auto& m : g_mat) {
    bool same = m.lx == lx && m.dev == dev;
    for (int q = 0; q < 6 && same; ++q) same = m.m[q] == mat_ptr(A, q);
    if (same) hit = &m;
    if (m.used < lru->used) lru = &m;
  }
  if (hit && !hit->ready) {  // fetch in flight: ready once its event has completed
    const cudaError_t q = cudaEventQuery(hit->ev);
    if (q == cudaSuccess) hit->ready = true;
    else if (q == cudaErrorNotReady) (void)cudaGetLastError();
    else return q;
  }
  if (hit && hit->ready) {
    hit->used = ++g_mat_clock;
    for (int q = 0; q < 6; ++q) memcpy(out + q * n, hit->h + q * 256, n * sizeof(double));
    *stale = g_stale;
    *have = true;
    return cudaSuccess;
  }
  if (hit) return cudaSuccess;  // still in flight
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaError_t e = cudaStreamIsCapturing(st, &cs);
  if (e != cudaSuccess) return e;
  if (cs != cudaStreamCaptureStatusNone) return cudaSuccess;  // no side effects inside a capture
  MatEntry& m = *lru;
  if (!m.h && (e = cudaHostAlloc(&m.h, 6 * 256 * sizeof(double), cudaHostAllocPortable)) != cudaSuccess)
    return e;
  if (m.ev && m.dev != dev) {
    cudaEventDestroy(m.ev);  // events belong to the device they were created on
    m.ev = nullptr;
  }
  if (!m.ev && (e = cudaEventCreateWithFlags(&m.ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  for (auto& p : m.m) p = nullptr;
  m.ready = false;
  for (int q = 0; q < 6; ++q)
    if ((e = cudaMemcpyAsync(m.h + q * 256, mat_ptr(A, q), n * sizeof(double), cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
      return e;
  if ((e = cudaEventRecord(m.ev, st)) != cudaSuccess) return e;
  for (int q = 0; q < 6; ++q) m.m[q] = mat_ptr(A, q);
  m.lx = lx;
  m.dev = dev;
  m.used = ++g_mat_clock;
  return cudaSuccess;
}

// fill the kernel's transposed parameter copies (zT[k][l] = dz[l][k]) or
// poison them (shared-memory path, see host_matrices)
template <int LX>
static cudaError_t param_matrices(TParams<LX>& P, cudaStream_t st, const double* const* hm) {
  double m6[6 * LX * LX];
  bool have = false;
  cudaError_t e = host_matrices(P.A, LX, hm, st, m6, &P.stale, &have);
  if (e != cudaSuccess) return e;
  if (!have) {
    const long long bits = 0x7ff4deadbeef0001LL;
    double poison;
    memcpy(&poison, &bits, sizeof poison);
    for (int q = 0; q < LX * LX; ++q) P.zT[q] = P.ztT[q] = poison;
    return cudaSuccess;
  }
  const double* z = m6 + 2 * LX * LX;
  const double* zt = m6 + 5 * LX * LX;
  for (int l = 0; l < LX; ++l)
    for (int k = 0; k < LX; ++k) {
      P.zT[k * LX + l] = z[l * LX + k];
      P.ztT[k * LX + l] = zt[l * LX + k];
    }
  return cudaSuccess;
}

static int g_nks8 = [] {
  const char* v = getenv("AXHELM_NKS");
  int d = v ? atoi(v) : 2;
  return (d >= 1 && d <= 4) ? d : 2;
}();

template <int LX, bool FAST, int NKS, int D = 2>
static cudaError_t launch_tma2(const AxPtrs& A, int64_t nel, cudaStream_t st, const double* const* hm) {
  using C = T2Cfg<LX, NKS, D>;
  static DevCache occ;
  int blocks_per_sm = 0;
  cudaError_t e = ctas_per_sm(occ, ax_tma2<LX, FAST, NKS, D>, C::NT, C::SMEM, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  TParams<LX> P;
  P.A = A;
  P.nel = nel;
  if ((e = param_matrices<LX>(P, st, hm)) != cudaSuccess) return e;
  const int64_t groups = (nel + C::EPL - 1) / C::EPL;
  int64_t grid = (int64_t)blocks_per_sm * num_sms();
  if (grid > groups) grid = groups;
  ax_tma2<LX, FAST, NKS, D><<<(unsigned)grid, C::NT, C::SMEM, st>>>(P);
  return cudaGetLastError();
}

static int dmma8_grid(int64_t nel, cudaError_t* err) {
  using C = DmCfg;
  static DevCache occ;
  *err = cudaSuccess;
  const int dev = cur_dev();
  if (dev < 0) {
    *err = cudaErrorInvalidDevice;
    return 0;
  }
  int blocks_per_sm = occ.v[dev].load(std::memory_order_relaxed);
  if (blocks_per_sm == 0) {
    cudaError_t e = cudaFuncSetAttribute(ax_dmma8<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ax_dmma8<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ax_dmma8<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(ax_dmma8<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    int b = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, ax_dmma8<true>, C::NT, C::SMEM);
    if (e != cudaSuccess) {
      *err = e;
      return 0;
    }
    blocks_per_sm = cap_ctas(b > 0 ? b : 1);
    occ.v[dev].store(blocks_per_sm, std::memory_order_relaxed);
  }
  int64_t grid = (int64_t)blocks_per_sm * num_sms();
  return (int)(grid > nel ? nel : grid);
}

// X.xrun > 0: the x-folding variant (contiguous segments) + its seam pass
template <bool DOT>
static cudaError_t launch_dmma8_impl(const AxPtrs& A, int64_t nel, double* partial, int grid,
                                     cudaStream_t st, const AxExt& X) {
  // the x-folding epilogue writes element e's shared x-face after e + 1 is
  // done, so per-element progress counters would announce unassembled w
  if (X.xrun > 0 && X.progress) return cudaErrorInvalidValue;
  if (X.xrun <= 0) {
    ax_dmma8<DOT><<<grid, DmCfg::NT, DmCfg::SMEM, st>>>(A, nel, partial, X);
    return cudaGetLastError();
  }
  ax_dmma8<DOT, true><<<grid, DmCfg::NT, DmCfg::SMEM, st>>>(A, nel, partial, X);
  const int64_t seg = (nel + grid - 1) / grid;
  const int64_t nseams = (nel - 1) / seg;  // segment starts a = c * seg < nel, c >= 1
  if (nseams > 0) xfold_seams<<<(unsigned)nseams, 64, 0, st>>>(A.w, nel, seg, X.xrun);
  return cudaGetLastError();
}

static cudaError_t launch_dmma8(const AxPtrs& A, int64_t nel, cudaStream_t st, const AxExt& X) {
  cudaError_t e;
  const int grid = dmma8_grid(nel, &e);
  if (e != cudaSuccess) return e;
  return launch_dmma8_impl<false>(A, nel, nullptr, grid, st, X);
}

bool progress_capable(const AxPtrs& A, int lx) {
  return lx == 8 && (g_variant == 0 || g_variant == 6) && aligned16(A);
}

bool dmma8_selected(const AxPtrs& A, int lx, int mode) {
  return lx == 8 && mode == AXHELM_FAST && (g_variant == 0 || g_variant == 6) && aligned16(A);
}

// fused apply + sum u*w (lx = 8, fast): per-CTA partials, fixed-order reduce
cudaError_t launch_dmma8_dot(const AxPtrs& A, int64_t nel, double* partial, int* nparts,
                             cudaStream_t st, const AxExt& X) {
  cudaError_t e;
  const int grid = dmma8_grid(nel, &e);
  if (e != cudaSuccess) return e;
  *nparts = grid;
  return launch_dmma8_impl<true>(A, nel, partial, grid, st, X);
}

static bool aligned16(const AxPtrs& A) {
  const void* f[9] = {A.w, A.u, A.h1, A.g11, A.g22, A.g33, A.g12, A.g13, A.g23};
  for (const void* p : f)
    if (((uintptr_t)p & 15u) != 0) return false;
  return true;
}

template <int LX, bool FAST, int PF>
static cudaError_t launch_pf(const AxPtrs& A, int64_t nel, cudaStream_t st) {
  using C = SCfg<LX>;
  static DevCache occ;
  int blocks_per_sm = 0;
  cudaError_t e = ctas_per_sm(occ, ax_kwalk_pf<LX, FAST, PF>, C::NT, C::SMEM, &blocks_per_sm);
  if (e != cudaSuccess) return e;
  const int64_t groups = (nel + C::EPB - 1) / C::EPB;
  int64_t grid = (int64_t)blocks_per_sm * num_sms();
  if (grid > groups) grid = groups;
  ax_kwalk_pf<LX, FAST, PF><<<(unsigned)grid, C::NT, C::SMEM, st>>>(A, nel);
  return cudaGetLastError();
}

template <int LX, bool FAST>
static cudaError_t launch_variant(const AxPtrs& A, int64_t nel, cudaStream_t st, const double* const* hm,
                                  const AxExt& X) {
  if constexpr (LX == 9 || LX == 10) {
    constexpr int M = FAST ? AXHELM_FAST : AXHELM_STRICT;
    if ((g_variant == 12 || g_variant == 0) && ws_selected(A, nel, LX, M, g_variant == 12))
      return launch_ws(A, nel, LX, M, st, hm);
  }
  if constexpr (LX == 7 || LX >= 9) {
    constexpr int M = FAST ? AXHELM_FAST : AXHELM_STRICT;
    if ((g_variant == 11 && line_selected(A, nel, LX, AXHELM_FAST)) || (g_variant == 0 && line_selected(A, nel, LX, M)))
      return launch_line(A, nel, LX, M, st, hm);
  }
  if constexpr (LX <= 8) {
    if ((g_variant == 6 || g_variant == 0) && FAST && aligned16(A)) {
      if constexpr (LX == 8) return launch_dmma8(A, nel, st, X);
    }
  }
  if constexpr (LX <= 15) {
    if ((g_variant >= 4 || g_variant == 0) && aligned16(A)) {
      if constexpr (LX == 8) {
        if (g_nks8 == 1) return launch_tma2<LX, FAST, 1>(A, nel, st, hm);
        if (g_nks8 == 4) return launch_tma2<LX, FAST, 4>(A, nel, st, hm);
      }
      // lx = 7 strict: the one-deep ring (5 CTAs per SM instead of 2) is 1.08x
      // faster; for fast mode and lx 4..6 the two depths are within noise
      if constexpr (LX == 7 && !FAST) return launch_tma2<LX, FAST, 1, 1>(A, nel, st, hm);
      return launch_tma2<LX, FAST, T2Shape<LX>::NKS, T2Shape<LX>::D>(A, nel, st, hm);
    }
  }
  if constexpr (LX == 8) {
    if (g_pf == 2) return launch_pf<LX, FAST, 2>(A, nel, st);
    if (g_pf == 3) return launch_pf<LX, FAST, 3>(A, nel, st);
  }
  return launch_pf<LX, FAST, 1>(A, nel, st);
}

template <int LX>
static cudaError_t launch_lx(const AxPtrs& A, int64_t nel, int mode, cudaStream_t st,
                             const double* const* hm, const AxExt& X) {
  return mode == AXHELM_FAST ? launch_variant<LX, true>(A, nel, st, hm, X)
                             : launch_variant<LX, false>(A, nel, st, hm, X);
}

cudaError_t launch_ax(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st,
                      const double* const* hm, const AxExt& X) {
  if (nel == 0) return cudaSuccess;
  switch (lx) {
#define AXB_CASE(N) \
  case N:           \
    return launch_lx<N>(A, nel, mode, st, hm, X);
    AXB_CASE(2) AXB_CASE(3) AXB_CASE(4) AXB_CASE(5) AXB_CASE(6) AXB_CASE(7)
    AXB_CASE(8) AXB_CASE(9) AXB_CASE(10) AXB_CASE(11) AXB_CASE(12)
    AXB_CASE(13) AXB_CASE(14) AXB_CASE(15) AXB_CASE(16)
#undef AXB_CASE
    default:
      return cudaErrorInvalidValue;
  }
}

// __dace_ax_helm's mode: process-wide, set from any thread (atomic)
static std::atomic<int> g_mode{[] {
  const char* v = getenv("AXHELM_FP");
  return (v && (!strcmp(v, "fast") || !strcmp(v, "FAST"))) ? (int)AXHELM_FAST : (int)AXHELM_STRICT;
}()};

int default_mode() { return g_mode.load(std::memory_order_relaxed); }


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
  const int keep = (mode & AXHELM_KEEP_W_L2) != 0;
  mode &= ~AXHELM_KEEP_W_L2;
  if (mode != AXHELM_STRICT && mode != AXHELM_FAST)
    return set_status(AXHELM_EINVAL, "unknown mode %d", mode);
  if (nel == 0) return set_status(AXHELM_OK, "");
  const double* ptrs[15] = {wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd,
                            h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  for (int q = 0; q < 15; ++q)
    if (!ptrs[q]) return set_status(AXHELM_EINVAL, "argument %d is NULL", q);
  AxPtrs A{wd, ud, dxd, dyd, dzd, dxtd, dytd, dztd, h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  AxExt X;
  X.keep_w = keep;
  return cuda_status(launch_ax(A, nel, lx, mode, (cudaStream_t)stream, nullptr, X),
                     "axhelm_apply");
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
  host_or_device_apply(ptrs, (int64_t)nelv, lx, default_mode());
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
  g_mode.store(mode, std::memory_order_relaxed);
  return set_status(AXHELM_OK, "");
}

int axhelm_get_mode(void) { return default_mode(); }
int axhelm_last_status(void) { return t_status; }
const char* axhelm_last_error(void) { return t_msg; }
const char* axhelm_version(void) { return "libaxhelm_sm100 " AXHELM_VERSION " (sm_100a, FP64)"; }

int axhelm_probe_stream(double* wd, const double* ud, const double* h1d, const double* g11d,
                        const double* g22d, const double* g33d, const double* g12d,
                        const double* g13d, const double* g23d, int64_t nel, void* stream) {
  // lx = 8 only: the roofline probe for the headline configuration
  using C = TCfg<8>;
  static DevCache occ;
  int blocks_per_sm = 0;
  cudaError_t e = ctas_per_sm(occ, ax_stream_probe<8>, C::NT, C::SMEM, &blocks_per_sm);
  if (e != cudaSuccess) return cuda_status(e, "axhelm_probe_stream");
  AxPtrs A{wd, ud, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
           h1d, g11d, g22d, g33d, g12d, g13d, g23d};
  int64_t grid = (int64_t)blocks_per_sm * num_sms();
  if (grid > nel) grid = nel;
  if (grid < 1) return set_status(AXHELM_OK, "");
  ax_stream_probe<8><<<(unsigned)grid, C::NT, C::SMEM, (cudaStream_t)stream>>>(A, nel);
  return cuda_status(cudaGetLastError(), "axhelm_probe_stream");
}

int64_t axhelm_bytes_model(int64_t nel, int lx) {
  return 72LL * nel * (int64_t)lx * lx * lx;
}

int64_t axhelm_flops_model(int64_t nel, int lx) {
  return nel * (int64_t)lx * lx * lx * (12LL * lx + 18);
}

}  // extern "C"
