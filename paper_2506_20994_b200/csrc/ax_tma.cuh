// TMA bulk-copy ring building blocks (mbarrier, cp.async.bulk, group issue)
// shared by the v4 / v6 kernels, and the roofline stream probe.  The v3
// kernel that introduced them (retired, superseded by v4) is described here.
//
// Why: the k-walk kernels (v1/v2) load the six geometric factors and h1 into
// registers, so the bytes in flight per SM are capped by registers x warps;
// ncu shows them long-scoreboard bound at 51-56% DRAM busy.  Here the whole
// input stream goes through the TMA engine: each persistent CTA owns a ring
// of D buffers, each holding all 8 input fields (u, h1, g11, g22, g33, g12,
// g13, g23) of EPL elements, filled by `cp.async.bulk` (one 1-D bulk copy
// per field: every field of an element is contiguous in HBM) completing on
// an mbarrier.  While the CTA computes group n out of buffer n % D, the
// copies for groups n+1 .. n+D-1 are in flight — without registers.
//
// Compute per element (same arithmetic and association as the other
// kernels, see ax_kernels.cuh): one thread per (j,i) column walking k.
//   * u rows (r-derivative) are read as 16-B vectors, u columns (s) as
//     broadcast 8-B loads, the thread's own u column (t) once into registers;
//   * dx[l][i], dy[l][j], dxt[l][i], dyt[l][j] live in registers for the
//     whole persistent CTA; dz / dzt (warp-uniform [l][k] reads) are kept
//     transposed in shared memory so a slice reads them as broadcast 16-B
//     vectors;
//   * ur / us overwrite the g11 / g22 slots of the same point (each slot is
//     read and then written by the same thread: no race), ut stays in
//     registers; stage 2 reads ur rows / us columns after one barrier;
//   * w is streamed straight to HBM with coalesced st.global.cs.
#pragma once

#include "ax_kernels.cuh"

namespace axb {

template <int LX>
struct TCfg {
  static constexpr int L2 = LX * LX;
  static constexpr int L3 = LX * LX * LX;
  // elements per group: ~64 threads, and an even count when L3 is odd so
  // each field chunk (EPL*L3*8 B) is a multiple of 16 B (bulk-copy rule)
  static constexpr int EPL0 = (64 / L2) > 0 ? (64 / L2) : 1;
  static constexpr int EPL = ((L3 & 1) && (EPL0 & 1)) ? EPL0 + 1 : EPL0;
  static constexpr int NT = EPL * L2;                 // threads per CTA
  static constexpr int D = 2;                         // ring depth
  static constexpr int FIELD = EPL * L3;              // doubles per field chunk
  static constexpr int BUF = 8 * FIELD;               // doubles per buffer
  static constexpr uint32_t CHUNK_BYTES = FIELD * 8;  // bytes per bulk copy
  static constexpr size_t SMEM = 128 + sizeof(double) * (D * BUF + 2 * L2);
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ const double* field_ptr(const AxPtrs& A, int f) {
  switch (f) {
    case 0: return A.u;
    case 1: return A.h1;
    case 2: return A.g11;
    case 3: return A.g22;
    case 4: return A.g33;
    case 5: return A.g12;
    case 6: return A.g13;
    default: return A.g23;
  }
}

// Leader thread: start loading group g into buffer buf (or mark it for a
// cooperative fallback load when the bulk-copy size/alignment rules fail).
// Returns true when the bulk path was used.
template <int LX>
__device__ __forceinline__ bool issue_group(const AxPtrs& A, int64_t nel, int64_t g, double* buf,
                                            uint64_t* bar, uint64_t pol) {
  using C = TCfg<LX>;
  const int64_t e0 = g * C::EPL;
  const int64_t ne = (nel - e0 < C::EPL) ? nel - e0 : C::EPL;
  const uint32_t bytes = (uint32_t)(ne * C::L3 * 8);
  if ((bytes & 15u) != 0u) {  // tail chunk the bulk engine cannot move: plain arrive
    mbar_arrive(bar);
    return false;
  }
  mbar_arrive_expect_tx(bar, 8u * bytes);
#pragma unroll
  for (int f = 0; f < 8; ++f) bulk_g2s_hint(buf + f * C::FIELD, field_ptr(A, f) + e0 * C::L3, bytes, bar, pol);
  return true;
}

// LX consecutive doubles from shared memory (16-B vectors when LX is even)
template <int LX>
__device__ __forceinline__ void lds_row(const double* src, double (&dst)[LX]) {
  if constexpr ((LX & 1) == 0) {
    const double2* v = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int q = 0; q < LX / 2; ++q) {
      const double2 x = v[q];
      dst[2 * q] = x.x;
      dst[2 * q + 1] = x.y;
    }
  } else {
#pragma unroll
    for (int l = 0; l < LX; ++l) dst[l] = src[l];
  }
}

}  // namespace axb

namespace axb {

// Roofline probe: the same TMA ring and the same HBM traffic as the apply
// (8 fields in, w out) with trivial arithmetic (w = sum of the 8 fields).
// Its time is the memory-side ceiling of the ring design for this
// read:write mix; exported as axhelm_probe_stream for bench/profiling only.
template <int LX>
__global__ void __launch_bounds__(TCfg<LX>::NT)
ax_stream_probe(const AxPtrs A, const int64_t nel) {
  using C = TCfg<LX>;
  constexpr int L3 = C::L3, FIELD = C::FIELD;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  double* bufs = reinterpret_cast<double*>(smem_raw + 128);
  const int tid = threadIdx.x;
  const int64_t ngroups = (nel + C::EPL - 1) / C::EPL;
  const int64_t stride = gridDim.x;
  const L2Pol pol = make_l2pol(0);
  if (tid == 0) {
    for (int d = 0; d < C::D; ++d) mbar_init(&bars[d], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (int d = 0; d < C::D; ++d) {
      const int64_t g = blockIdx.x + d * stride;
      if (g < ngroups) issue_group<LX>(A, nel, g, bufs + d * C::BUF, &bars[d], pol.in);
    }
  int64_t n = 0;
  for (int64_t g = blockIdx.x; g < ngroups; g += stride, ++n) {
    const int b = (int)(n % C::D);
    double* buf = bufs + b * C::BUF;
    const int64_t e0 = g * C::EPL;
    const int64_t ne = (nel - e0 < C::EPL) ? nel - e0 : C::EPL;
    mbar_wait(&bars[b], (uint32_t)((n / C::D) & 1));
    for (int q = tid; q < ne * L3; q += C::NT) {
      double s = 0.0;
#pragma unroll
      for (int f = 0; f < 8; ++f) s += buf[f * FIELD + q];
      stg_stream(A.w + e0 * L3 + q, s);
    }
    __syncthreads();
    if (tid == 0) {
      const int64_t gn = g + C::D * stride;
      if (gn < ngroups) {
        fence_proxy_async();
        issue_group<LX>(A, nel, gn, buf, &bars[b], pol.in);
      }
    }
  }
}

}  // namespace axb
