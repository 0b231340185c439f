// Host-pointer path of __dace_ax_helm (reference: kernelrt.py:95-106 and
// cabi-harness/src/run.ts:64-74 both pass HOST buffers through the ABI).
//
// The apply is split into element chunks (<= 4 Mi points, 32 MiB per field)
// that cycle through NS = 4 device slots on NS streams: chunk c's host->device
// copies, its kernel and its device->host copy of w are enqueued on stream
// c % NS, so the H2D copy engine, the SMs and the D2H copy engine work on
// three different chunks at once.  Arrays that are already device (or
// managed) memory are used in place, so mixed host/device argument sets work.
// Pinned host buffers are DMA'd directly.  Pageable ones (what a NumPy
// caller of the reference ABI passes) are copied by a pool of host threads
// into pinned per-slot staging buffers — chunk c+1 while the copy engines
// move chunk c — and w comes back the same way (the driver's own pageable
// path serialises at ~10 GB/s: 0.16 GDOF/s at C2, slower than the CPU).
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <emmintrin.h>  // SSE2 streaming stores (x86-64 baseline)

#include "../../include/axhelm.h"
#include "ax_launch.h"

namespace axb {

namespace {

enum Kind { DEV = 0, PINNED = 1, PAGEABLE = 2 };

Kind classify(const void* p) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear the sticky-free error
    return PAGEABLE;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) return DEV;
  if (a.type == cudaMemoryTypeHost) return PINNED;
  return PAGEABLE;
}

constexpr int NS_MAX = 8;
constexpr int NF = 9;  // w + u + 7 geometry fields per slot

// pipeline depth (slots/streams) and points per chunk; AXHELM_STAGE_SLOTS /
// AXHELM_STAGE_CHUNK (points) override for tuning
int env_int(const char* name, int dflt, int lo, int hi) {
  const char* v = getenv(name);
  const long x = v ? atol(v) : dflt;
  return (int)(x < lo ? lo : (x > hi ? hi : x));
}
// (measured on B200 / PCIe Gen5 at C2: 3 x 1 Mi -> 51.5 GB/s H2D, 4 x 4 Mi
// -> 53.6 GB/s = 96% of the 55.6 GB/s raw pinned copy)
const int NS = env_int("AXHELM_STAGE_SLOTS", 4, 2, NS_MAX);
const int64_t CHUNK_PTS = env_int("AXHELM_STAGE_CHUNK", 1 << 22, 1 << 12, 1 << 26);
// chunk when some argument is pageable (host-thread staging copies)
const int64_t CHUNK_PTS_PAGEABLE = env_int("AXHELM_STAGE_CHUNK_PAGEABLE", 1 << 20, 1 << 12, 1 << 26);

// A small pool of host threads for parallel memcpy (pageable <-> pinned).
class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size(); }
  // run job(worker) on every worker and wait
  void run(const std::function<void(int)>& job) {
    std::unique_lock<std::mutex> lk(mu_);
    job_ = &job;
    pending_ = (int)th_.size();
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int i) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      (*job)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  int pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// one thread's part of a staging copy.  Non-temporal (streaming) stores: the
// destination is written once and read by the copy engine or the caller
// later, so skipping the read-for-ownership of every destination line cuts
// the host-memory traffic of the copy from three passes to two (the copy
// engines share that bandwidth).  sfence: the stores are visible before the
// pool reports the part done.
void stage_copy(double* dst, const double* src, int64_t n) {
#ifdef AX_NO_NT_COPY
  memcpy(dst, src, sizeof(double) * (size_t)n);
#else
  int64_t i = 0;
  if (((uintptr_t)dst & 15u) && n > 0) {
    dst[0] = src[0];
    i = 1;
  }
  for (; i + 8 <= n; i += 8) {
    const __m128d v0 = _mm_loadu_pd(src + i), v1 = _mm_loadu_pd(src + i + 2);
    const __m128d v2 = _mm_loadu_pd(src + i + 4), v3 = _mm_loadu_pd(src + i + 6);
    _mm_stream_pd(dst + i, v0);
    _mm_stream_pd(dst + i + 2, v1);
    _mm_stream_pd(dst + i + 4, v2);
    _mm_stream_pd(dst + i + 6, v3);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
#endif
}

// copy n doubles src -> dst with every pool thread taking a contiguous part
void par_copy(CopyPool& pool, double* dst, const double* src, int64_t n) {
  const int T = pool.size();
  pool.run([&](int i) {
    const int64_t a = n * i / T, b = n * (i + 1) / T;
    if (b > a) stage_copy(dst + a, src + a, b - a);
  });
}

struct Stager {
  std::mutex mu;
  bool ready = false;
  cudaStream_t st[NS_MAX] = {};
  cudaEvent_t mats_ready = nullptr;
  cudaEvent_t slot_done[NS_MAX] = {};
  double* slots = nullptr;  // NS * NF * slot_pts doubles (grow-only)
  int64_t slot_pts = 0;
  double* mats = nullptr;   // 6 * 16 * 16 doubles
  double* pinned = nullptr;  // NS * NF * pinned_pts doubles of pinned host staging (pageable callers)
  int64_t pinned_pts = 0;
  CopyPool* pool = nullptr;
};

Stager g_stager[64];

cudaError_t ensure(Stager& S, int64_t pts) {
  cudaError_t e;
  if (!S.ready) {
    for (int s = 0; s < NS; ++s)
      if ((e = cudaStreamCreateWithFlags(&S.st[s], cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&S.mats_ready, cudaEventDisableTiming)) != cudaSuccess) return e;
    for (int s = 0; s < NS; ++s)
      if ((e = cudaEventCreateWithFlags(&S.slot_done[s], cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&S.mats, sizeof(double) * 6 * 256)) != cudaSuccess) return e;
    S.ready = true;
  }
  if (S.slot_pts < pts) {  // grow the slots to this call's chunk size
    if (S.slots) {
      for (int s = 0; s < NS; ++s) cudaStreamSynchronize(S.st[s]);
      cudaFree(S.slots);
      S.slots = nullptr;
      S.slot_pts = 0;
    }
    if ((e = cudaMalloc(&S.slots, sizeof(double) * NS * NF * pts)) != cudaSuccess) return e;
    S.slot_pts = pts;
  }
  return cudaSuccess;
}

// pinned host staging + copy threads for pageable arguments (grow-only)
cudaError_t ensure_pinned(Stager& S, int64_t pts) {
  if (!S.pool) {
    const unsigned hc = std::thread::hardware_concurrency();
    S.pool = new CopyPool(env_int("AXHELM_COPY_THREADS", hc > 12 ? 12 : (hc > 0 ? (int)hc : 4), 1, 64));
  }
  if (S.pinned_pts < pts) {
    for (int s = 0; s < NS; ++s) cudaStreamSynchronize(S.st[s]);
    if (S.pinned) cudaFreeHost(S.pinned);
    S.pinned = nullptr;
    S.pinned_pts = 0;
    cudaError_t e = cudaHostAlloc(&S.pinned, sizeof(double) * NS * NF * pts, cudaHostAllocDefault);
    if (e != cudaSuccess) return e;
    S.pinned_pts = pts;
  }
  return cudaSuccess;
}

}  // namespace

int host_or_device_apply(const double* const ptrs[15], int64_t nel, int lx, int mode) {
  if (lx < 2 || lx > 16) return set_status(AXHELM_EINVAL, "lx=%d outside [2, 16]", lx);
  if (nel < 0) return set_status(AXHELM_EINVAL, "nelv=%lld is negative", (long long)nel);
  if (nel == 0) return set_status(AXHELM_OK, "");
  for (int q = 0; q < 15; ++q)
    if (!ptrs[q]) return set_status(AXHELM_EINVAL, "argument %d is NULL", q);

  Kind kind[15];
  bool all_dev = true;
  for (int q = 0; q < 15; ++q) {
    kind[q] = classify(ptrs[q]);
    all_dev &= kind[q] == DEV;
  }
  const int64_t L3 = (int64_t)lx * lx * lx;

  if (all_dev) {
    // plain device call, synchronous like the reference's CPU kernel: wait for
    // every stream of the device first (the caller may have produced the
    // buffers on any stream, blocking or not), then run on the legacy stream
    cudaError_t e0 = cudaDeviceSynchronize();
    if (e0 != cudaSuccess) return cuda_status(e0, "__dace_ax_helm (device)");
    AxPtrs A{const_cast<double*>(ptrs[0]), ptrs[1], ptrs[2], ptrs[3], ptrs[4], ptrs[5],
             ptrs[6], ptrs[7], ptrs[8], ptrs[9], ptrs[10], ptrs[11], ptrs[12], ptrs[13],
             ptrs[14]};
    cudaError_t e = launch_ax(A, nel, lx, mode, 0);
    if (e == cudaSuccess) e = cudaStreamSynchronize(0);
    return cuda_status(e, "__dace_ax_helm (device)");
  }

  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return set_status(AXHELM_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
  Stager& S = g_stager[dev & 63];
  std::lock_guard<std::mutex> lock(S.mu);
  // chunk: whole elements, at most CHUNK_PTS points (and no more than needed);
  // pageable arguments go through host-thread copies, which pipeline better
  // in 1 Mi-point chunks (C2: 235 -> 215 ms; pinned keeps 4 Mi: 51.5 -> 53.6 GB/s)
  bool pageable_args = false;
  for (int q = 0; q < 15; ++q) pageable_args |= kind[q] == PAGEABLE;
  const int64_t chunk_pts = pageable_args ? CHUNK_PTS_PAGEABLE : CHUNK_PTS;
  const int64_t chunk_el0 = chunk_pts / L3 > 0 ? chunk_pts / L3 : 1;
  const int64_t chunk_el = nel < chunk_el0 ? nel : chunk_el0;
  if ((e = ensure(S, chunk_el * L3)) != cudaSuccess) return cuda_status(e, "__dace_ax_helm (staging setup)");
  const int64_t SP = S.slot_pts;

  // the six [lx][lx] matrices: once per call
  const double* mat[6];
  const size_t mbytes = sizeof(double) * lx * lx;
  for (int q = 0; q < 6; ++q) {
    if (kind[2 + q] == DEV) {
      mat[q] = ptrs[2 + q];
    } else {
      double* d = S.mats + q * 256;
      if ((e = cudaMemcpyAsync(d, ptrs[2 + q], mbytes, cudaMemcpyHostToDevice, S.st[0])) != cudaSuccess)
        return cuda_status(e, "__dace_ax_helm (matrices)");
      mat[q] = d;
    }
  }
  cudaEventRecord(S.mats_ready, S.st[0]);
  for (int s = 1; s < NS; ++s) cudaStreamWaitEvent(S.st[s], S.mats_ready, 0);

  // field indices in ptrs[]: 0 = w, 1 = u, 8..14 = h1, g11, g22, g33, g12, g13, g23
  static const int fidx[NF] = {0, 1, 8, 9, 10, 11, 12, 13, 14};
  bool any_pageable = false;
  for (int q = 0; q < NF; ++q) any_pageable |= kind[fidx[q]] == PAGEABLE;
  if (any_pageable && (e = ensure_pinned(S, chunk_el * L3)) != cudaSuccess)
    return cuda_status(e, "__dace_ax_helm (pinned staging)");
  const int64_t PP = S.pinned_pts;  // pinned staging stride per field
  // pageable w: copy chunk cw's result out of its pinned slot (after its D2H)
  std::vector<int64_t> pending_out(NS, -1);  // element offset of the chunk awaiting copy-out, per slot
  std::vector<int64_t> pending_ne(NS, 0);
  auto copy_out = [&](int s) -> cudaError_t {
    if (pending_out[s] < 0) return cudaSuccess;
    cudaError_t ee = cudaEventSynchronize(S.slot_done[s]);
    if (ee != cudaSuccess) return ee;
    par_copy(*S.pool, const_cast<double*>(ptrs[0]) + pending_out[s] * L3, S.pinned + (size_t)s * NF * PP,
             pending_ne[s] * L3);
    pending_out[s] = -1;
    return cudaSuccess;
  };
  for (int64_t e0 = 0, c = 0; e0 < nel; e0 += chunk_el, ++c) {
    const int s = (int)(c % NS);
    const int64_t ne = (nel - e0 < chunk_el) ? nel - e0 : chunk_el;
    const int64_t off = e0 * L3;
    const size_t bytes = sizeof(double) * ne * L3;
    double* slot = S.slots + (size_t)s * NF * SP;
    double* hslot = any_pageable ? S.pinned + (size_t)s * NF * PP : nullptr;
    if (any_pageable) {  // slot s's previous chunk is done with its pinned staging
      if ((e = copy_out(s)) != cudaSuccess) return cuda_status(e, "__dace_ax_helm (D2H copy-out)");
      if ((e = cudaEventSynchronize(S.slot_done[s])) != cudaSuccess) return cuda_status(e, "__dace_ax_helm (slot)");
      // pageable inputs of this chunk -> pinned staging, all fields in one parallel pass
      int nq = 0;
      int qs[NF];
      for (int q = 1; q < NF; ++q)
        if (kind[fidx[q]] == PAGEABLE) qs[nq++] = q;
      if (nq > 0) {
        const int64_t n = ne * L3;
        const int T = S.pool->size();
        S.pool->run([&](int i) {
          const int64_t a = n * i / T, b = n * (i + 1) / T;
          if (b <= a) return;
          for (int k = 0; k < nq; ++k) stage_copy(hslot + (size_t)qs[k] * PP + a, ptrs[fidx[qs[k]]] + off + a, b - a);
        });
      }
    }
    const double* f[NF];
    for (int q = 0; q < NF; ++q) {
      const int a = fidx[q];
      if (kind[a] == DEV) {
        f[q] = ptrs[a] + off;
      } else {
        double* d = slot + (size_t)q * SP;
        const double* src = kind[a] == PAGEABLE ? hslot + (size_t)q * PP : ptrs[a] + off;
        if (q > 0 && (e = cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, S.st[s])) != cudaSuccess)
          return cuda_status(e, "__dace_ax_helm (H2D)");
        f[q] = d;
      }
    }
    AxPtrs A{const_cast<double*>(f[0]), f[1], mat[0], mat[1], mat[2], mat[3], mat[4], mat[5],
             f[2], f[3], f[4], f[5], f[6], f[7], f[8]};
    const double* hm[6];  // host copies of dxd .. dztd (when they are host arrays)
    for (int q = 0; q < 6; ++q) hm[q] = kind[2 + q] != DEV ? ptrs[2 + q] : nullptr;
    if ((e = launch_ax(A, ne, lx, mode, S.st[s], hm)) != cudaSuccess)
      return cuda_status(e, "__dace_ax_helm (kernel)");
    if (kind[0] == PINNED &&
        (e = cudaMemcpyAsync(const_cast<double*>(ptrs[0]) + off, f[0], bytes, cudaMemcpyDeviceToHost,
                             S.st[s])) != cudaSuccess)
      return cuda_status(e, "__dace_ax_helm (D2H)");
    if (kind[0] == PAGEABLE) {
      if ((e = cudaMemcpyAsync(hslot, f[0], bytes, cudaMemcpyDeviceToHost, S.st[s])) != cudaSuccess)
        return cuda_status(e, "__dace_ax_helm (D2H)");
      pending_out[s] = e0;
      pending_ne[s] = ne;
    }
    if (any_pageable && (e = cudaEventRecord(S.slot_done[s], S.st[s])) != cudaSuccess)
      return cuda_status(e, "__dace_ax_helm (event)");
  }
  for (int s = 0; s < NS; ++s)
    if (any_pageable && (e = copy_out(s)) != cudaSuccess) return cuda_status(e, "__dace_ax_helm (D2H copy-out)");
  for (int s = 0; s < NS; ++s)
    if ((e = cudaStreamSynchronize(S.st[s])) != cudaSuccess) return cuda_status(e, "__dace_ax_helm (sync)");
  return set_status(AXHELM_OK, "");
}

}  // namespace axb
