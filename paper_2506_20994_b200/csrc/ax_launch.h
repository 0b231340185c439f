// Internal (non-ABI) declarations shared by the translation units of
// libaxhelm_sm100.so.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ax_kernels.cuh"

namespace axb {

int set_status(int st, const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
int default_mode();

// enqueue one apply over device pointers (no validation).  hz / hzt / hx /
// hxt: host copies of dzd / dztd / dxd / dxtd when the caller has them
// (else looked up in / added to the pointer-keyed cache).
cudaError_t launch_ax(const AxPtrs& A, int64_t nel, int lx, int mode, cudaStream_t st,
                      const double* hz = nullptr, const double* hzt = nullptr,
                      const double* hx = nullptr, const double* hxt = nullptr);

// fused lx = 8 fast apply + per-CTA partials of sum u*w (nparts written)
cudaError_t launch_dmma8_dot(const AxPtrs& A, int64_t nel, double* partial, int* nparts,
                             cudaStream_t st);
// true when launch_ax would run the fused-capable DMMA kernel
bool dmma8_selected(const AxPtrs& A, int lx, int mode);

// __dace_ax_helm body: classify the 15 pointers (device / pinned host /
// pageable host) and run the apply synchronously, staging host data through
// the GPU in copy/compute-overlapped chunks.
int host_or_device_apply(const double* const ptrs[15], int64_t nel, int lx, int mode);

}  // namespace axb
