// v12 ax_helm kernel for lx 9 / 10: the v11 line contractions (ax_line.cuh)
// fed by a warp-specialised geometry stream.
//
// Why (profiles/r02_s2lo_l12_strict.txt): v11 loads h1 and the
// six G straight into a register pipeline a few planes ahead of the combine,
// so HBM is busy only while a CTA is in its combine; stage 1 / stage 2 run
// with nothing in flight but the next element's u.  Three CTAs per SM overlap
// each other's phases only statistically (strict lx 12: FP64 pipe 55%,
// long-scoreboard 25%, barriers 16%).  Every cheaper decoupling (early
// register loads, L2 fills, a per-thread cp.async ring) measured slower.
//
// Here ONE CTA per SM holds NG consumer groups (LX^2 threads rounded to
// warps each, named barriers 1..NG) that work on the CTA's elements round
// robin, and one producer warp that streams, in element order, each
// element's u (one TMA bulk copy into the group's u buffer) and then its
// geometry in chunks of G planes (seven bulk copies per chunk, one per
// field) into a ring of NS chunks that fills the shared memory left.  The
// producer runs as far ahead as the ring allows in every phase, so the HBM
// stream no longer stops while the groups compute; the combine reads its
// geometry from shared memory.  (NG, G) per lx: WsPick in
// ax_line.cu, chosen by same-box A/B (profiles/r02_ab_ws_kernel.txt).
//
//   uFull[u] / uEmpty[u]: u buffer u = g * UB + (the group's element count
//                         mod UB) (arrive after stage 1)
//   full[s] / empty[s]:   ring slot s (one arrive per consumer thread)
//   chunk c of the CTA's j-th element (j-th in blockIdx + j*grid order):
//   q = j*NC + c  ->  slot q % NS, use q / NS (NS a multiple of NG*NC: a
//   slot is always refilled for the group that just released it)
//
// The arithmetic per point is v11's (line products with constant-bank
// matrices, the reference association in strict mode: bit-exact).
#pragma once

#include "ax_line.cuh"

namespace axb {

template <int LX, int NG_, int G_>
struct WsCfg {
  using C = LineCfg<LX>;
  static constexpr int L2 = LX * LX, L3 = L2 * LX;
  static constexpr int GT = (L2 + 31) / 32 * 32;  // threads per consumer group
  static constexpr int NG = NG_;                  // consumer groups
  static constexpr int NT = NG * GT + 32;         // the groups + the producer warp
  static constexpr int US = (L3 + 2 + 1) & ~1;    // u superset (odd lx^3: one pad double)
  static constexpr int XS = C::XS;
  // ring unit: G consecutive planes of all seven fields, one bulk copy per
  // field (single planes at lx 9 are 648-B copies: too small for the TMA
  // unit to stream, 0.3-0.5x)
  static constexpr int G = G_;
  static constexpr int NC = (LX + G - 1) / G;     // chunks per element
  static constexpr int SL = (G * L2 + 2 + 1) & ~1;  // ring field slot (16-B superset)
  static constexpr int PLANE = 7 * SL;            // doubles per ring slot
  static constexpr size_t HEAD = 1024;            // mbarriers
  // u buffers per group: two let the producer land the group's next u while
  // the group still works on the current one (1.01-1.02x,
  // profiles/r02_ab_ws_kernel.txt)
  static constexpr int UB = 2;
  static constexpr size_t FIXED = HEAD + 8 * (size_t)(UB * NG * US + 2 * NG * XS);
  static constexpr size_t BUDGET = 227 * 1024;
  static constexpr int NS0 = (int)((BUDGET - FIXED) / (8 * (size_t)PLANE));
  // Ring slots: a multiple of NG * NC, so chunk q and chunk q + NS (the next
  // use of the same slot) belong to elements NS / NC apart, a multiple of NG:
  // the same group.  Every slot then has ONE consumer that takes its phases
  // in order and waits one phase at a time.  (A ring whose slots pass between
  // groups lets a group that runs ahead wait on a parity two phases old and
  // read stale geometry: measured as a full-size fault; per-slot tickets
  // fixed that but left compute-sanitizer racecheck / synccheck findings.)
  static constexpr int NS = (((NS0 > 48 ? 48 : NS0) / (NG * NC)) * (NG * NC));
  static_assert(NS >= NG * NC, "ring too small for this lx / NG / G");
  static_assert(C::EPC == 1 && !C::UPAD, "one element per group, linear u");
  static constexpr size_t SMEM = FIXED + 8 * (size_t)NS * PLANE;
};

__device__ __forceinline__ void group_sync(int g, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "r"(n) : "memory");
}

// chunk c (planes [c G, min(c G + G, lx))) of element e, field f (1..7):
// 16-B aligned superset [lo, lo + n) clipped to the array; pad = doubles
// before the data
template <int LX, int G>
__device__ __forceinline__ void ws_plane_span(const AxPtrs& A, int64_t nel, int f, int64_t e, int c,
                                              const double** lo, int* pad, int* n) {
  constexpr int64_t L2 = LX * LX, L3 = L2 * LX;
  const int np = LX - c * G < G ? LX - c * G : G;
  const double* base = field_ptr(A, f);
  const uintptr_t p = (uintptr_t)(base + e * L3 + (int64_t)c * G * L2);
  const uintptr_t l = p & ~(uintptr_t)15;
  uintptr_t h = (p + 8 * L2 * np + 15) & ~(uintptr_t)15;
  const uintptr_t end = (uintptr_t)(base + nel * L3);
  if (h > end) h = end & ~(uintptr_t)15;  // last plane: the tail double is read from HBM
  *lo = reinterpret_cast<const double*>(l);
  *pad = (int)((p - l) >> 3);
  *n = (int)((h - l) >> 3);
}

template <int LX, bool FAST, bool UP, int NG, int G>
__device__ __forceinline__ void ws_element(const LParams<LX>& P, int g, int tg, bool act, int a, int b,
                                           int64_t e, int64_t j, const double* Uv, double* X0, double* X1,
                                           uint64_t* uEmpty, uint64_t* full, uint64_t* empty,
                                           const double* R) {
  using W = WsCfg<LX, NG, G>;
  using C = LineCfg<LX>;
  constexpr int L2 = W::L2, L3 = W::L3, RS = C::RS, PS = C::PS, NS = W::NS, NC = W::NC;
  const AxPtrs& A = P.A;
  // ---- stage 1 (v11): r-line (k=a, j=b) -> X0, s-line (k=a, i=b) -> X1,
  // t-line (j=a, i=b) in registers
  double t[LX];
  if (act) {
    double out[LX];
    line_s<LX, FAST, UP>(P, 0, Uv + a * L2 + b * LX, 1, out);
#pragma unroll
    for (int i = 0; i < LX; ++i) X0[a * PS + b * RS + i] = out[i];
    line_s<LX, FAST, UP>(P, 1, Uv + a * L2 + b, LX, out);
#pragma unroll
    for (int jj = 0; jj < LX; ++jj) X1[a * PS + jj * RS + b] = out[jj];
    line_s<LX, FAST, UP>(P, 2, Uv + a * LX + b, L2, t);
  } else {
#pragma unroll
    for (int k = 0; k < LX; ++k) t[k] = 0.0;
  }
  group_sync(g, W::GT);  // r, s complete; u dead
  if (tg == 0) mbar_arrive(uEmpty);
  // ---- combine: plane k is plane k - c G of chunk c = k / G, ring slot
  // (j NC + c) % NS; a field chunk's pad (0 / 1 double before its data in
  // the 16-B superset) is the parity of its start: per element (pbits) and
  // c G lx^2
  const int xb = a * RS + b;
  int pbits = 0;
#pragma unroll
  for (int f = 0; f < 7; ++f) pbits |= (int)(((uintptr_t)(field_ptr(A, f + 1) + e * L3) >> 3) & 1) << f;
  const int pt = a * LX + b;
  const int64_t pc = j * NC;  // the first chunk's number in production order
  int s = (int)(pc % NS);
  uint32_t ph = (uint32_t)((pc / NS) & 1);
#pragma unroll
  for (int k = 0; k < LX; ++k) {
    const int c = k / G, kk = k - c * G;
    if (kk == 0) {
      mbar_wait(&full[s], ph);
    }
    if (act) {
      double gq[7];
      const double* Rs = R + (size_t)s * 7 * W::SL;
      if (e != P.nel - 1 || c != NC - 1) {
#pragma unroll
        for (int f = 0; f < 7; ++f) gq[f] = Rs[f * W::SL + (((pbits >> f) ^ (c * G * L2)) & 1) + kk * L2 + pt];
      } else {  // the array's last chunk: its superset may be clipped
#pragma unroll
        for (int f = 0; f < 7; ++f) {
          const double* lo;
          int pad, n;
          ws_plane_span<LX, G>(A, P.nel, f + 1, e, c, &lo, &pad, &n);
          const int q = pad + kk * L2 + pt;
          gq[f] = q < n ? Rs[f * W::SL + q] : lo[q];
        }
      }
      const double r = X0[k * PS + xb], sv = X1[k * PS + xb];
      X0[k * PS + xb] = combine<FAST>(gq[0], gq[1], gq[4], gq[5], r, sv, t[k]);  // ur
      X1[k * PS + xb] = combine<FAST>(gq[0], gq[4], gq[2], gq[6], r, sv, t[k]);  // us
      t[k] = combine<FAST>(gq[0], gq[5], gq[6], gq[3], r, sv, t[k]);             // ut
    }
    if (kk == G - 1 || k == LX - 1) {  // chunk consumed
      mbar_arrive(&empty[s]);  // every thread of the group: its own reads are done
      if (++s == NS) {
        s = 0;
        ph ^= 1u;
      }
    }
  }
  double* wout = A.w + e * L3 + a * LX + b;
  if constexpr (FAST) {
    double wt[LX];
    line<LX, FAST, UP>(P, 5, t, wt);
    group_sync(g, W::GT);  // ur / us complete
    if (act) {
      double out[LX];
      line_s<LX, FAST, UP>(P, 3, X0 + a * PS + b * RS, 1, out);
#pragma unroll
      for (int i = 0; i < LX; ++i) X0[a * PS + b * RS + i] = out[i];
      line_s<LX, FAST, UP>(P, 4, X1 + a * PS + b, RS, out);
#pragma unroll
      for (int jj = 0; jj < LX; ++jj) X1[a * PS + jj * RS + b] = out[jj];
    }
    group_sync(g, W::GT);
    if (act) {
#pragma unroll
      for (int k = 0; k < LX; ++k) stg_stream(wout + k * L2, (X0[k * PS + xb] + X1[k * PS + xb]) + wt[k]);
    }
  } else {
    group_sync(g, W::GT);  // ur / us complete
    if (act) {
      double w[LX];
#pragma unroll
      for (int k = 0; k < LX; ++k) w[k] = 0.0;
#pragma unroll
      for (int l = 0; l < LX; ++l) {
        const double dxl = __ldg(A.dxt + l * LX + b), dyl = __ldg(A.dyt + l * LX + a);
#pragma unroll
        for (int k = 0; k < LX; ++k) {
          w[k] = madd<false>(w[k], dxl, X0[k * PS + a * RS + l]);
          w[k] = madd<false>(w[k], dyl, X1[k * PS + l * RS + b]);
          w[k] = madd<false>(w[k], mat<LX, UP>(P, 5, l, k), t[l]);
        }
      }
#pragma unroll
      for (int k = 0; k < LX; ++k) stg_stream(wout + k * L2, w[k]);
    }
  }
  group_sync(g, W::GT);  // X0 / X1 free for the group's next element
}

template <int LX, bool FAST, int NG, int G>
__global__ void __launch_bounds__(WsCfg<LX, NG, G>::NT, 1) ax_ws(const __grid_constant__ LParams<LX> P) {
  using W = WsCfg<LX, NG, G>;
  constexpr int L2 = W::L2, L3 = W::L3, NS = W::NS;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NU = W::UB * NG;  // u buffers: group g, buffer b -> g * UB + b
  uint64_t* uFull = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* uEmpty = uFull + NU;
  uint64_t* full = uFull + 2 * NU;
  uint64_t* empty = full + NS;
  double* U = reinterpret_cast<double*>(smem_raw + W::HEAD);
  double* X = U + NU * W::US;
  double* R = X + 2 * NG * W::XS;

  const AxPtrs& A = P.A;
  const int64_t nel = P.nel, grid = gridDim.x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int g = 0; g < NU; ++g) {
      mbar_init(&uFull[g], 1);
      mbar_init(&uEmpty[g], 1);
    }
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W::GT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  int bad = 0;
  for (int q = tid; q < 6 * L2; q += W::NT) {
    const int mi = q / L2, rr = q - mi * L2;
    bad |= __double_as_longlong(__ldg(mat_ptr(A, mi) + rr)) != __double_as_longlong(P.m[mi][rr]);
  }
  const bool use_param = !__syncthreads_or(bad);  // also publishes the barrier inits
  if (!use_param && tid == 0 && P.stale) *(volatile int*)P.stale = 1;
  const int64_t nmine = (int64_t)blockIdx.x < nel ? (nel - 1 - blockIdx.x) / grid + 1 : 0;

  if (tid >= NG * W::GT) {  // ---- producer warp (one lane)
    if (tid == NG * W::GT) {
      for (int64_t j = 0; j < nmine; ++j) {
        const int64_t e = blockIdx.x + j * grid;
        const int g = (int)(j % NG);
        const int64_t gu = j / NG;                        // the group's element count
        const int ub = g * W::UB + (int)(gu % W::UB);     // its u buffer
        const int64_t use = gu / W::UB;                   // that buffer's use count
        if (use > 0) mbar_wait(&uEmpty[ub], (uint32_t)((use - 1) & 1));
        fence_proxy_async();
        const int64_t first = e * L3;
        const int64_t lo = first & ~(int64_t)1, hi = (first + L3 + 1) & ~(int64_t)1;
        if (hi > nel * L3) {
          mbar_arrive(&uFull[ub]);  // past the end: the group loads u itself
        } else {
          const uint32_t bytes = (uint32_t)((hi - lo) * 8);
          mbar_arrive_expect_tx(&uFull[ub], bytes);
          bulk_g2s(U + ub * W::US, A.u + lo, bytes, &uFull[ub]);
        }
        for (int c = 0; c < W::NC; ++c) {
          const int64_t q = j * W::NC + c;  // chunk number in production order
          const int s = (int)(q % NS);
          const int64_t n = q / NS;
          if (n > 0) mbar_wait(&empty[s], (uint32_t)((n - 1) & 1));
          fence_proxy_async();
          const double* src[7];
          int cnt[7], tot = 0;
#pragma unroll
          for (int f = 0; f < 7; ++f) {
            int pad;
            ws_plane_span<LX, G>(A, nel, f + 1, e, c, &src[f], &pad, &cnt[f]);
            tot += cnt[f];
          }
          mbar_arrive_expect_tx(&full[s], (uint32_t)(8 * tot));
#pragma unroll
          for (int f = 0; f < 7; ++f)
            bulk_g2s(R + ((size_t)s * 7 + f) * W::SL, src[f], (uint32_t)(8 * cnt[f]), &full[s]);
        }
      }
    }
    return;
  }
  // ---- consumer groups
  const int g = tid / W::GT, tg = tid - g * W::GT;
  const bool act = tg < L2;
  const int a = act ? tg / LX : 0, b = act ? tg - (tg / LX) * LX : 0;

  double* X0 = X + (2 * g) * W::XS;
  double* X1 = X0 + W::XS;
  for (int64_t j = g; j < nmine; j += NG) {
    const int64_t e = blockIdx.x + j * grid;
    const int64_t gu = j / NG;
    const int ub = g * W::UB + (int)(gu % W::UB);
    double* Ug = U + ub * W::US;
    mbar_wait(&uFull[ub], (uint32_t)((gu / W::UB) & 1));
    const int64_t first = e * L3;
    int pad = (int)(first & 1);
    if (((first + L3 + 1) & ~(int64_t)1) > nel * L3) {  // fallback: load u ourselves
      pad = 0;
      for (int q = tg; q < L3; q += W::GT) Ug[q] = A.u[first + q];
      group_sync(g, W::GT);
    }
    if (use_param)
      ws_element<LX, FAST, true, NG, G>(P, g, tg, act, a, b, e, j, Ug + pad, X0, X1, &uEmpty[ub], full, empty, R);
    else
      ws_element<LX, FAST, false, NG, G>(P, g, tg, act, a, b, e, j, Ug + pad, X0, X1, &uEmpty[ub], full, empty, R);
  }
}

}  // namespace axb
