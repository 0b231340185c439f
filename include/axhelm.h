/*
 * axhelm.h — C ABI of libaxhelm_sm100.so, the B200 (sm_100a) drop-in for the
 * reference's ax_helm kernel.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg):
 *   __dace_ax_helm        src/mdg/codegen.py:183-194 (_signature), pinned by
 *                         tests/test_codegen.py:27-36; ABI order
 *                         src/mdg/axprogram.py:32-48.
 *                         Bound by src/mdg/kernelrt.py:77-108 (ctypes) and
 *                         cabi-harness/src/run.ts:64-74 (koffi).
 *   axhelm_*              extensions the reference's void ABI lacks
 *                         (SURVEY §8b): a stream-ordered device entry with an
 *                         error return and 64-bit element count, and an
 *                         error/version query.  Gather-scatter and the mesh
 *                         store have no reference counterpart.
 *
 * Data layout: fields are [nel][lx][lx][lx] row-major FP64 (i fastest), the
 * six matrices [lx][lx] row-major.  lx must lie in [2, 16] (sem.py:36-37).
 *
 * Arithmetic modes: AXHELM_STRICT reproduces the reference's strict-fp
 * operation order bit for bit; AXHELM_FAST fuses multiply-adds (<= 1e-12
 * normwise from the reference, the tolerance of tests/test_codegen.py:180-187).
 */
#ifndef AXHELM_SM100_H
#define AXHELM_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
#define AXH_RESTRICT __restrict__
extern "C" {
#else
#define AXH_RESTRICT restrict
#endif

enum axhelm_mode { AXHELM_STRICT = 0, AXHELM_FAST = 1 };
/* Flag OR-ed into the mode of axhelm_apply / axhelm_apply_dot: the caller
 * reads w again right after the apply (layer-blocked ax + DSSUM), so the
 * kernel loads its inputs L2 evict-first and keeps w in L2 instead of
 * streaming it out.  Results are identical with or without it. */
enum { AXHELM_KEEP_W_L2 = 0x100 };

enum axhelm_status {
  AXHELM_OK = 0,
  AXHELM_EINVAL = 1,   /* bad lx, negative nel, null pointer */
  AXHELM_ECUDA = 2,    /* CUDA runtime error (message in last_error) */
  AXHELM_ENODEV = 3,   /* no usable sm_100 device */
};

/* The reference ABI, exactly (codegen.py:183-194).  Synchronous: returns
 * with wd written.  Accepts device pointers (kernel on the calling thread's
 * default stream) or host pointers, pinned or pageable (chunked,
 * copy/compute-overlapped staging through the GPU).  The void return has no
 * error channel: failures are reported by axhelm_last_status(). */
void __dace_ax_helm(double* AXH_RESTRICT wd, const double* AXH_RESTRICT ud,
                    const double* AXH_RESTRICT dxd, const double* AXH_RESTRICT dyd,
                    const double* AXH_RESTRICT dzd, const double* AXH_RESTRICT dxtd,
                    const double* AXH_RESTRICT dytd, const double* AXH_RESTRICT dztd,
                    const double* AXH_RESTRICT h1d, const double* AXH_RESTRICT g11d,
                    const double* AXH_RESTRICT g22d, const double* AXH_RESTRICT g33d,
                    const double* AXH_RESTRICT g12d, const double* AXH_RESTRICT g13d,
                    const double* AXH_RESTRICT g23d, int nelv, int lx);

/* Stream-ordered device entry: every pointer is a device pointer; enqueues
 * the apply on `stream` (a cudaStream_t, NULL = legacy default stream) and
 * returns without synchronising. */
int axhelm_apply(double* wd, const double* ud, const double* dxd,
                 const double* dyd, const double* dzd, const double* dxtd,
                 const double* dytd, const double* dztd, const double* h1d,
                 const double* g11d, const double* g22d, const double* g33d,
                 const double* g12d, const double* g13d, const double* g23d,
                 int64_t nel, int lx, int mode, void* stream);

/* __dace_ax_helm with an explicit mode and a status return: synchronous,
 * host or device pointers (per-array), 64-bit element count. */
int axhelm_apply_sync(double* wd, const double* ud, const double* dxd,
                      const double* dyd, const double* dzd, const double* dxtd,
                      const double* dytd, const double* dztd, const double* h1d,
                      const double* g11d, const double* g22d, const double* g33d,
                      const double* g12d, const double* g13d, const double* g23d,
                      int64_t nel, int lx, int mode);

/* Mode used by __dace_ax_helm (default AXHELM_STRICT, or AXHELM_FAST when
 * the environment variable AXHELM_FP=fast is set at load time). */
int axhelm_set_mode(int mode);
int axhelm_get_mode(void);

/* Status of the last call on this thread, and its message. */
int axhelm_last_status(void);
const char* axhelm_last_error(void);
const char* axhelm_version(void);

/* Roofline probe (diagnostics): lx = 8 only, same TMA ring and the same HBM
 * traffic as the apply (8 fields read, wd written, wd = sum of the fields).
 * Its time is the memory-side ceiling of the kernel design. */
int axhelm_probe_stream(double* wd, const double* ud, const double* h1d,
                        const double* g11d, const double* g22d, const double* g33d,
                        const double* g12d, const double* g13d, const double* g23d,
                        int64_t nel, void* stream);

/* ---- box mesh, device geometry store, gather-scatter (DSSUM) -----------
 * No reference counterpart (SPEC.md:14 scopes them out of the reference;
 * PAPER.md:123 names gather-scatter as Neko's second ingredient).  All
 * pointers are device pointers; every call is stream-ordered. */

/* Global node ids of a z-slab [ez0, ez0 + nel/(nx*ny)) of an nx*ny*nz brick
 * of lx^3 elements (element order e = (ez*ny + ey)*nx + ex); gid of point
 * (gx, gy, gz) = (gz*NY + gy)*NX + gx with NX = nx*(lx-1)+1. */
int axhelm_box_gid(int64_t* gid, int nx, int ny, int lx, int64_t ez0, int64_t nel, void* stream);

/* Geometric factors (h1 = 1, G = w_i w_j w_k det J J^-1 J^-T) of the same
 * slab of a smoothly deformed brick, X = X0 + amp*sin sin sin. */
int axhelm_box_geometry(double* h1d, double* g11d, double* g22d, double* g33d, double* g12d,
                        double* g13d, double* g23d, const double* gll_points,
                        const double* gll_weights, int nx, int ny, int nz, int lx, int64_t ez0,
                        int64_t nel, double amp, void* stream);

/* DSSUM over n shared global nodes in CSR form: copies of node q are
 * w[idx[offs[q]] .. idx[offs[q+1]-1]] in ascending order; each gets the sum
 * (from 0.0, in that order).  idx_bytes = 4 (int32) or 8 (int64). */
int axhelm_gs_sum(double* w, const int64_t* offs, const void* idx, int idx_bytes, int64_t n,
                  void* stream);

/* Interface-plane steps of the multi-GPU DSSUM: PARTIAL buf[slot[q]] = sum
 * of own copies; FINISH continues from buf[slot[q]] with own copies, writes
 * the sum to the copies and to buf; WRITE copies buf[slot[q]] to own copies. */
enum axhelm_gs_op { AXHELM_GS_PARTIAL = 0, AXHELM_GS_FINISH = 1, AXHELM_GS_WRITE = 2 };
int axhelm_gs_plane(int op, double* w, const int64_t* offs, const void* idx, int idx_bytes,
                    const int64_t* slot, int64_t n, double* buf, void* stream);

/* Structured DSSUM on a BoxMesh slab (element layers [ez0, ez1) of an
 * nx*ny*nz brick; no index arrays).  op 0: every shared node of the slab
 * except those on an exchanged interface plane (has_below: bottom plane
 * shared with the rank below; has_above: top plane shared with the rank
 * above); op 1 + AXHELM_GS_PARTIAL / _FINISH / _WRITE: the interface-plane
 * steps on buf[NX*NY] (PARTIAL, WRITE: top plane; FINISH: bottom plane).
 * Same summation order as axhelm_gs_sum. */
int axhelm_gs_box(int op, double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1,
                  int has_below, int has_above, double* buf, void* stream);

/* Local DSSUM (op 0 of axhelm_gs_box) restricted to the global z node planes
 * [zlo, zhi] of the slab, which must not include an exchanged interface
 * plane.  Summing the planes in ascending blocks gives the same result as
 * one op-0 call; a caller interleaves it with ax_helm on element layers so
 * the w it touches is still in L2. */
int axhelm_gs_box_range(double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1,
                        int64_t zlo, int64_t zhi, void* stream);

/* Peer-memory interface exchange (multi-GPU DSSUM without NCCL): device
 * allocations shared between the ranks' processes with CUDA IPC (64-byte
 * cudaIpcMemHandle), and the interface-plane steps writing the neighbour's
 * receive buffer / flag directly over NVLink.  op AXHELM_GS_PARTIAL: top
 * plane partial sums -> out (upper rank's buffer), then signal_flag = seq;
 * AXHELM_GS_FINISH: wait *wait_flag >= seq, continue from in (own buffer),
 * write the bottom-plane copies, final sums -> out (lower rank's buffer),
 * signal; AXHELM_GS_WRITE: wait, write the top-plane copies from in.
 * counter: a zeroed unsigned in local device memory per op.  Same
 * summation order as axhelm_gs_box ops 1..3 (bit-identical). */
int axhelm_peer_alloc(int64_t bytes, void** ptr, void* handle);
int axhelm_peer_open(const void* handle, void** ptr);
int axhelm_peer_close(void* ptr);
int axhelm_peer_free(void* ptr);
int axhelm_gs_box_peer(int op, double* w, int nx, int ny, int lx, int64_t ez0, int64_t ez1,
                       const double* in, double* out, const unsigned long long* wait_flag,
                       unsigned long long* signal_flag, unsigned long long seq, unsigned* counter,
                       const unsigned long long* seq_dev, void* stream);
/* seq_dev (nullable): take the sequence number as *seq_dev + 1 on the device
 * instead of `seq` (so a captured CUDA graph advances it on every replay);
 * axhelm_peer_seq_bump increments it after one exchange's steps. */
int axhelm_peer_seq_bump(unsigned long long* seq_dev, void* stream);
/* All-reduce (sum) of n <= 4 doubles over `world` ranks through peer
 * memory: bases = device array of every rank's peer region (own included),
 * each reserving axhelm_peer_allreduce_bytes() at byte offset `off`; seq
 * increases by one per call on every rank.  The sum is taken in rank order,
 * so every rank gets the same bits.  v may alias out. */
int64_t axhelm_peer_allreduce_bytes(void);
int axhelm_peer_allreduce(const double* v, int n, double* out, const unsigned long long* bases,
                          int64_t off, int world, int rank, unsigned long long seq,
                          unsigned long long* seq_dev, void* stream);  /* seq_dev: as above, bumped here */

/* Assembled local operator on a BoxMesh slab: ax_helm on the slab's local
 * element layers [l0, l1) and the local DSSUM of the owned node planes
 * [zlo, zhi] (layers outside [l0, l1) must already be applied, stream-
 * ordered before this call).  The 15 pointers are the slab's arrays
 * (element 0 = first element of layer ez0).  schedule:
 *   AXHELM_SCHED_SEQUENTIAL (0): one apply streaming w to HBM, then one
 *       DSSUM pass (reads and writes w again);
 *   AXHELM_SCHED_FOLLOW (-1): the apply keeps w in L2 and publishes per-layer
 *       completion counters in progress[l1 - l0] (zeroed here); a DSSUM
 *       follower kernel runs concurrently on an internal stream (joined back
 *       into `stream`) and sums each layer's planes as soon as it is
 *       complete (the lx = 8 FAST DMMA kernel; else sequential);
 *   n > 0: blocks of n layers, each apply followed by the DSSUM of the planes
 *       it completes (kernel-boundary version of FOLLOW).
 * dot_out (nullable): sum_p u_p (A u)_p over the applied elements before
 * assembly (fixed order); partial then needs axhelm_ax_gs_scratch(l1 - l0)
 * doubles.  Every schedule gives bit-identical w. */
enum { AXHELM_SCHED_SEQUENTIAL = 0, AXHELM_SCHED_FOLLOW = -1 };
int axhelm_ax_gs_box(double* wd, const double* ud, const double* dxd, const double* dyd,
                     const double* dzd, const double* dxtd, const double* dytd, const double* dztd,
                     const double* h1d, const double* g11d, const double* g22d, const double* g33d,
                     const double* g12d, const double* g13d, const double* g23d, int nx, int ny,
                     int lx, int64_t ez0, int64_t ez1, int64_t l0, int64_t l1, int64_t zlo,
                     int64_t zhi, int mode, int schedule, unsigned* progress, double* partial,
                     double* dot_out, void* stream);
int axhelm_ax_gs_scratch(int64_t nlayers);

/* ---- Jacobi-PCG building blocks (no reference) --------
 * Deterministic reductions: `partial` holds axhelm_reduce_blocks(n) * 2
 * doubles of scratch; results land in DEVICE memory (`out`), and alpha /
 * beta are read from device memory, so an iteration needs no host sync. */
int axhelm_reduce_blocks(int64_t n);
/* out[0] = sum a*b (times wt if non-NULL) */
int axhelm_dot(const double* a, const double* b, const double* wt, int64_t n, double* partial,
               double* out, void* stream);
/* r = mask*f, p = dinv*r, x = 0; out = {sum cwt r dinv r, sum cwt r r}
 * with cwt = mask / multiplicity (each interior node counted once) */
int axhelm_cg_init(const double* f, const double* mask, const double* dinv, const double* cwt,
                   double* r, double* p, double* x, int64_t n, double* partial, double* out,
                   void* stream);
/* alpha = sc[0]/sc[1]; x += alpha p; r -= alpha w; out = {rz, rr} (weights cwt) */
int axhelm_cg_update(double* x, double* r, const double* p, const double* w, const double* dinv,
                     const double* cwt, const double* sc, int64_t n, double* partial, double* out,
                     void* stream);
/* w = A_local u (element-local ax_helm, no DSSUM) and out[0] = sum u*w over
 * the local points, fused into the FP64-DMMA kernel for lx = 8 fast mode.
 * For a continuous u vanishing where the mask does, this equals the
 * assembled <u, mask QQ^T A u> (each node once) — the PCG's p.Ap. */
int axhelm_apply_dot(double* wd, const double* ud, const double* dxd, const double* dyd,
                     const double* dzd, const double* dxtd, const double* dytd, const double* dztd,
                     const double* h1d, const double* g11d, const double* g22d, const double* g33d,
                     const double* g12d, const double* g13d, const double* g23d, int64_t nel,
                     int lx, int mode, double* partial, double* out, void* stream);
/* axhelm_apply / axhelm_apply_dot (dot_out may be NULL) for nel elements that
 * form whole x-runs of a brick (e = (ez ny + ey) nx + ex, nel % nx == 0).
 * When the lx = 8 fast DMMA kernel runs, it also sums the class-2 DSSUM
 * nodes — x-face nodes on no y / z element face, shared by consecutive
 * elements of a run — in its epilogue, bit for bit as the DSSUM would
 * ((0.0 + w[e-1]) + w[e]), and sets *xfolded = 1; else *xfolded = 0 and w
 * is the plain element-local apply.  Pass *xfolded on to
 * axhelm_cg_update_box.  AXHELM_XFOLD=0 in the environment disables it. */
int axhelm_apply_box(double* wd, const double* ud, const double* dxd, const double* dyd,
                     const double* dzd, const double* dxtd, const double* dytd, const double* dztd,
                     const double* h1d, const double* g11d, const double* g22d, const double* g33d,
                     const double* g12d, const double* g13d, const double* g23d, int nx, int64_t nel,
                     int lx, int mode, double* partial, double* dot_out, int* xfolded, void* stream);
/* Structured-brick PCG update with the local DSSUM folded in: w = A_local p
 * after the interface-plane exchange (axhelm_gs_box ops 1..3) but WITHOUT the
 * local DSSUM; each point gathers its node's local copies in the DSSUM's
 * order (bit-identical assembled value), r -= (a[0]/a[1]) QQ^T w, and
 * out = (sum cwt r dinv r, sum cwt r r) with cwt = mask/multiplicity computed
 * from the point's position (mask: the brick's outer boundary).  The slab is
 * element layers [ez0, ez1) of an nx*ny*nz brick.  xfolded: w came from
 * axhelm_apply_box with *xfolded = 1 (class-2 nodes already summed: read
 * once, not gathered). */
int axhelm_cg_update_box(double* r, const double* w, const double* dinv, const double* a, int nx,
                         int ny, int64_t nz, int lx, int64_t ez0, int64_t ez1, int has_below,
                         int has_above, int xfolded, double* partial, double* out, void* stream);
/* x += (a[0]/a[1]) p; p = dinv r + (sc_new[0]/a[0]) p  (a = (rz_old, p.Ap)) */
int axhelm_cg_xpupdate(double* x, double* p, const double* r, const double* dinv, const double* a,
                       const double* sc_new, int64_t n, void* stream);
/* p = dinv r + (sc_new[0]/sc_old[0]) p */
int axhelm_cg_pupdate(double* p, const double* r, const double* dinv, const double* sc_new,
                      const double* sc_old, int64_t n, void* stream);
/* element-local diagonal of A (the Jacobi preconditioner before DSSUM) */
int axhelm_diag(double* diag, const double* dxd, const double* dyd, const double* dzd,
                const double* dxtd, const double* dytd, const double* dztd, const double* h1d,
                const double* g11d, const double* g22d, const double* g33d, const double* g12d,
                const double* g13d, const double* g23d, int64_t nel, int lx, void* stream);

/* Algorithmic model: bytes = 72*nel*lx^3, flops =
 * nel*lx^3*(12*lx+18) (sem.py:367-375). */
int64_t axhelm_bytes_model(int64_t nel, int lx);
int64_t axhelm_flops_model(int64_t nel, int lx);

#ifdef __cplusplus
}
#endif

#endif /* AXHELM_SM100_H */
