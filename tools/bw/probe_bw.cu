// Bandwidth experiments (not part of the product): TMA-ring streaming of 8
// fields of 4 KiB per element (+ optional 1 write), ring depth D, grid size
// chosen at launch.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared
//   -Xcompiler -fPIC probe_bw.cu -o libprobe_bw.so
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int D, bool WRITE>
__global__ void probe(const double* const* f, double* w, int64_t nel) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = (uint64_t*)sm;
  double* buf = (double*)(sm + 128);
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int d = 0; d < D; ++d) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[d])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int64_t e, int d) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[d])), "r"(8 * 4096));
    for (int q = 0; q < 8; ++q)
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(
                       sa(buf + d * 4096 + q * 512)),
                   "l"(f[q] + e * 512), "r"(sa(&bar[d]))
                   : "memory");
  };
  if (tid == 0)
    for (int d = 0; d < D; ++d)
      if (blockIdx.x + d * gridDim.x < nel) issue(blockIdx.x + d * gridDim.x, d);
  int64_t n = 0;
  for (int64_t e = blockIdx.x; e < nel; e += gridDim.x, ++n) {
    const int d = (int)(n % D);
    const uint32_t par = (uint32_t)((n / D) & 1);
    asm volatile("{.reg .pred P; W: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1; @!P bra W;}" ::"r"(
                     sa(&bar[d])),
                 "r"(par)
                 : "memory");
    const double* b = buf + d * 4096;
    for (int p = tid; p < 512; p += blockDim.x) {
      double s = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s += b[q * 512 + p];
      if (WRITE) asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(w + e * 512 + p), "d"(s) : "memory");
      else if (s == 12345.678) w[0] = s;
    }
    __syncthreads();
    if (tid == 0 && e + D * gridDim.x < nel) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(e + D * gridDim.x, d);
    }
  }
}

template <int D, bool W>
static int run(const double* const* f, double* w, int64_t nel, int grid, int threads, void* st) {
  const size_t smem = 128 + (size_t)D * 8 * 4096;
  cudaFuncSetAttribute(probe<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<D, W><<<grid, threads, smem, (cudaStream_t)st>>>(f, w, nel);
  return (int)cudaGetLastError();
}

extern "C" int probe_bw(const double* const* f, double* w, int64_t nel, int depth, int write, int grid,
                        int threads, void* st) {
  switch (depth * 2 + write) {
    case 2: return run<1, false>(f, w, nel, grid, threads, st);
    case 3: return run<1, true>(f, w, nel, grid, threads, st);
    case 4: return run<2, false>(f, w, nel, grid, threads, st);
    case 5: return run<2, true>(f, w, nel, grid, threads, st);
    case 6: return run<3, false>(f, w, nel, grid, threads, st);
    case 7: return run<3, true>(f, w, nel, grid, threads, st);
    case 8: return run<4, false>(f, w, nel, grid, threads, st);
    case 9: return run<4, true>(f, w, nel, grid, threads, st);
    case 12: return run<6, false>(f, w, nel, grid, threads, st);
    case 13: return run<6, true>(f, w, nel, grid, threads, st);
  }
  return -1;
}
