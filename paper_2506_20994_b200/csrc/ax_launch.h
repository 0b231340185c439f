// Internal (non-ABI) declarations shared by the translation units of
// libaxhelm_sm100.so.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "ax_kernels.cuh"

namespace axb {

// ------------------------------------------------------- per-device state
//
// Launch caches (max-dynamic-smem attribute done, resident CTAs per SM, SM
// count) are per device: cudaFuncSetAttribute applies to the current
// device's context only, so a process driving several GPUs needs one entry
// per device.  Entries are written once (idempotent, benign race).
constexpr int kMaxDev = 64;
inline int cur_dev() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDev) return -1;
  return d;
}
struct DevCache {
  std::atomic<int> v[kMaxDev];
  DevCache() {
    for (auto& x : v) x.store(0, std::memory_order_relaxed);
  }
};
int num_sms();           // SMs of the current device (cached)
int cap_ctas(int b);     // AXHELM_CTAS_PER_SM cap on resident CTAs per SM

// resident CTAs per SM of `kern` at `smem` bytes, per device; sets the
// max-dynamic-shared-memory attribute on first use on each device
template <typename K>
cudaError_t ctas_per_sm(DevCache& cache, K kern, int nt, size_t smem, int* out) {
  const int dev = cur_dev();
  if (dev < 0) return cudaErrorInvalidDevice;
  int b = cache.v[dev].load(std::memory_order_relaxed);
  if (b == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, nt, smem);
    if (e != cudaSuccess) return e;
    b = cap_ctas(b > 0 ? b : 1);
    cache.v[dev].store(b, std::memory_order_relaxed);
  }
  *out = b;
  return cudaSuccess;
}

// Host copies of the six matrices (dx, dy, dz, dxt, dyt, dzt; out[q*lx*lx
// ..]) for a kernel's parameter block.  hm: the caller's host arrays (all six
// or ignored); else a per-device, pointer-keyed cache that never blocks: a
// miss enqueues an async D2H fetch on st and returns *have = false (the
// kernel then reads the device arrays).  *stale: mapped flag the kernel sets
// when the device arrays differ from the copy.
cudaError_t host_matrices(const AxPtrs& A, int lx, const double* const* hm, cudaStream_t st,
                          double* out, int** stale, bool* have);

// v11 line kernel (ax_line.cu), lx 9..16; false = not handled (lx, alignment)
bool line_selected(const AxPtrs& A, int64_t nel, int lx, int mode);
cudaError_t launch_line(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st,
                        const double* const* hm);
// v12 warp-specialised line kernel (ax_ws.cuh), lx 9 / 10: the default for
// fast mode (forced: both modes)
bool ws_selected(const AxPtrs& A, int64_t nel, int lx, int mode, bool forced);
cudaError_t launch_ws(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st,
                      const double* const* hm);

int set_status(int st, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
int default_mode();

// enqueue one apply over device pointers (no validation).  hm: host copies
// of the six matrices when the caller has them (else looked up in / added to
// the pointer-keyed cache without blocking).
// X: keep-w-in-L2 / progress extensions (honoured by the lx = 8 DMMA kernel)
cudaError_t launch_ax(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st,
                      const double* const* hm = nullptr, const AxExt& X = AxExt{});

// fused lx = 8 fast apply + per-CTA partials of sum u*w (nparts written)
cudaError_t launch_dmma8_dot(const AxPtrs& A, int64_t nel, double* partial, int* nparts,
                             cudaStream_t st, const AxExt& X = AxExt{});
// true when launch_ax would run a kernel that honours AxExt (the lx = 8
// DMMA kernel; callers also check mode FAST via dmma8_selected)
bool progress_capable(const AxPtrs& A, int lx);
// true when launch_ax would run the fused-capable DMMA kernel
bool dmma8_selected(const AxPtrs& A, int lx, int mode);

// __dace_ax_helm body: classify the 15 pointers (device / pinned host /
// pageable host) and run the apply synchronously, staging host data through
// the GPU in copy/compute-overlapped chunks.
int host_or_device_apply(const double* const ptrs[15], int64_t nel, int lx, int mode);

// structured DSSUM of the slab's node planes [zlo, zhi] (mesh_gs.cu);
// gs_box_range_check returns nullptr or why the arguments are invalid
// [s2lo, s2hi]: planes whose class-2 (x-face-only) nodes the x-folding DMMA
// apply has summed already (skipped here)
cudaError_t gs_box_range(double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1, int64_t zlo,
                         int64_t zhi, cudaStream_t st, int64_t s2lo = 1, int64_t s2hi = 0);
const char* gs_box_range_check(int nx, int ny, int lx, int64_t ez0, int64_t ez1, int64_t zlo,
                               int64_t zhi);

// DSSUM follower: the local DSSUM of node planes [zlo, zhi] of local layers
// [0, nl), run CONCURRENTLY with an apply over layers [l0, l1) that signals
// per-layer completion in progress[L - l0] (layers outside [l0, l1) must be
// complete already).  Each layer's planes are summed once the layer is done.
cudaError_t gs_box_follow(double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1, int64_t zlo,
                          int64_t zhi, const unsigned* progress, int64_t l0, int64_t l1, cudaStream_t st);

}  // namespace axb
