/*
 * CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).
 *
 * C restatement of the reference apply mdg.sem.ax_reference
 * (/root/reference/pkg/src/mdg/sem.py:300-337) with the per-point operation
 * order of the IR tasklets (axprogram.py:159-163, :188-192, :229).  Compiled
 * with -ffp-contract=off so no multiply-add is fused: every result is
 * bit-identical to the NumPy oracle and to the reference.
 *
 * Used by tests/ (parity at sizes NumPy is too slow for) and by bench.py's
 * cpu_baseline leg when the reference's own generated kernel (oracle/_ref)
 * is absent.  Never linked by the product library.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#pragma STDC FP_CONTRACT OFF

#define LXMAX 16

int oracle_ax_helm(double *restrict wd, const double *restrict ud,
                   const double *restrict dxd, const double *restrict dyd,
                   const double *restrict dzd, const double *restrict dxtd,
                   const double *restrict dytd, const double *restrict dztd,
                   const double *restrict h1d, const double *restrict g11d,
                   const double *restrict g22d, const double *restrict g33d,
                   const double *restrict g12d, const double *restrict g13d,
                   const double *restrict g23d, int64_t nel, int lx,
                   int nthreads)
{
    if (lx < 2 || lx > LXMAX || nel < 0)
        return -1;
#ifdef _OPENMP
    if (nthreads > 0)
        omp_set_num_threads(nthreads);
#else
    (void)nthreads;
#endif
    const int64_t n3 = (int64_t)lx * lx * lx;
#pragma omp parallel
    {
        double ur[LXMAX * LXMAX * LXMAX], us[LXMAX * LXMAX * LXMAX],
            ut[LXMAX * LXMAX * LXMAX];
#pragma omp for schedule(static)
        for (int64_t e = 0; e < nel; ++e) {
            const double *u = ud + e * n3;
            const int64_t b = e * n3;
            /* stage 1 + combine, point by point */
            for (int k = 0; k < lx; ++k)
                for (int j = 0; j < lx; ++j)
                    for (int i = 0; i < lx; ++i) {
                        double r = 0.0, s = 0.0, t = 0.0;
                        for (int l = 0; l < lx; ++l) {
                            r = r + dxd[l * lx + i] * u[(k * lx + j) * lx + l];
                            s = s + dyd[l * lx + j] * u[(k * lx + l) * lx + i];
                            t = t + dzd[l * lx + k] * u[(l * lx + j) * lx + i];
                        }
                        const int p = (k * lx + j) * lx + i;
                        const double h = h1d[b + p];
                        const double a11 = g11d[b + p], a22 = g22d[b + p],
                                     a33 = g33d[b + p], a12 = g12d[b + p],
                                     a13 = g13d[b + p], a23 = g23d[b + p];
                        ur[p] = h * ((a11 * r + a12 * s) + a13 * t);
                        us[p] = h * ((a12 * r + a22 * s) + a23 * t);
                        ut[p] = h * ((a13 * r + a23 * s) + a33 * t);
                    }
            /* stage 2 */
            for (int k = 0; k < lx; ++k)
                for (int j = 0; j < lx; ++j)
                    for (int i = 0; i < lx; ++i) {
                        double w = 0.0;
                        for (int l = 0; l < lx; ++l) {
                            w = w + dxtd[l * lx + i] * ur[(k * lx + j) * lx + l];
                            w = w + dytd[l * lx + j] * us[(k * lx + l) * lx + i];
                            w = w + dztd[l * lx + k] * ut[(l * lx + j) * lx + i];
                        }
                        wd[b + (k * lx + j) * lx + i] = w;
                    }
        }
    }
    return 0;
}

/* Direct stiffness summation restated for the checker (no reference
 * implementation exists: SPEC.md:14).  acc (nglob doubles) must be zeroed by
 * the caller.  Accumulates every local copy into its global node in ascending
 * local index, then writes the sums back to every copy. */
void oracle_dssum(double *w, const int64_t *gid, double *acc, int64_t n)
{
    for (int64_t p = 0; p < n; ++p)
        acc[gid[p]] = acc[gid[p]] + w[p];
    for (int64_t p = 0; p < n; ++p)
        w[p] = acc[gid[p]];
}
