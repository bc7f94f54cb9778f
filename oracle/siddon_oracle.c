/*
 * oracle/siddon_oracle.c -- CPU restatement of the reference cone-beam operator.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2110_13526_b200/csrc).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  It is never
 * called by the product path.
 *
 * It restates, in plain C99 + OpenMP, the fp64 Numba kernels of the reference
 * package cbctkit 0.1.0:
 *
 *   oracle_traverse        <- /root/reference/pkg/src/cbctkit/operator.py:53-187  (_traverse)
 *   oracle_project         <- operator.py:190-206  (_project_kernel, prange over rays)
 *   oracle_backproject     <- operator.py:209-233  (_backproject_kernel: views dealt
 *                             round-robin to n_workers private accumulators, merged
 *                             serially in worker order -> bit-deterministic per W)
 *   oracle_ray_segments    <- operator.py:236-259  (_segments_kernel)
 *
 * The per-view tables (srcs, det00, ustep, vstep: [V][3] fp64) are built by the
 * caller with numpy exactly as operator.py:262-281 does, so both sides share
 * bit-identical geometry.  Arithmetic order follows the reference line by line
 * (no FMA contraction: build with -ffp-contract=off).
 *
 * Pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py writes tests/golden/ fixtures).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SEG_EPS 1e-12 /* operator.py:23 */

/* operator.py:53-187.  mode 0: return sum(w*vol); 1: acc += w*pixval; 2: acc += w*w */
static double oracle_traverse(double sx, double sy, double sz, double rx, double ry, double rz,
                              double lo0, double lo1, double lo2, double p0, double p1, double p2,
                              int64_t n0, int64_t n1, int64_t n2, int mode, const double* vol,
                              double* acc, double pixval) {
    double tmin = 0.0, tmax = 1.0, t1, t2, tt;
    /* box clip, axis-parallel below 1e-12*pitch (operator.py:62-100) */
    if (fabs(rx) < 1e-12 * p0) {
        if (sx < lo0 || sx >= lo0 + (double)n0 * p0) return 0.0;
    } else {
        t1 = (lo0 - sx) / rx;
        t2 = (lo0 + (double)n0 * p0 - sx) / rx;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(ry) < 1e-12 * p1) {
        if (sy < lo1 || sy >= lo1 + (double)n1 * p1) return 0.0;
    } else {
        t1 = (lo1 - sy) / ry;
        t2 = (lo1 + (double)n1 * p1 - sy) / ry;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(rz) < 1e-12 * p2) {
        if (sz < lo2 || sz >= lo2 + (double)n2 * p2) return 0.0;
    } else {
        t1 = (lo2 - sz) / rz;
        t2 = (lo2 + (double)n2 * p2 - sz) / rz;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (tmax <= tmin) return 0.0;

    const double raylen = sqrt(rx * rx + ry * ry + rz * rz); /* operator.py:102 */

    /* entry voxel, clamped (operator.py:104-119) */
    int64_t ix = (int64_t)floor((sx + tmin * rx - lo0) / p0);
    int64_t iy = (int64_t)floor((sy + tmin * ry - lo1) / p1);
    int64_t iz = (int64_t)floor((sz + tmin * rz - lo2) / p2);
    if (ix < 0) ix = 0; else if (ix >= n0) ix = n0 - 1;
    if (iy < 0) iy = 0; else if (iy >= n1) iy = n1 - 1;
    if (iz < 0) iz = 0; else if (iz >= n2) iz = n2 - 1;

    /* per-axis next-plane parameter and increment (operator.py:121-148) */
    const double big = 1e300;
    double tx, ty, tz, dtx, dty, dtz, plane;
    int stx, sty, stz;
    if (fabs(rx) < 1e-12 * p0) { tx = big; dtx = big; stx = 0; }
    else {
        stx = rx > 0 ? 1 : -1;
        plane = lo0 + (double)(ix + (stx > 0 ? 1 : 0)) * p0;
        tx = (plane - sx) / rx;
        dtx = p0 / fabs(rx);
    }
    if (fabs(ry) < 1e-12 * p1) { ty = big; dty = big; sty = 0; }
    else {
        sty = ry > 0 ? 1 : -1;
        plane = lo1 + (double)(iy + (sty > 0 ? 1 : 0)) * p1;
        ty = (plane - sy) / ry;
        dty = p1 / fabs(ry);
    }
    if (fabs(rz) < 1e-12 * p2) { tz = big; dtz = big; stz = 0; }
    else {
        stz = rz > 0 ? 1 : -1;
        plane = lo2 + (double)(iz + (stz > 0 ? 1 : 0)) * p2;
        tz = (plane - sz) / rz;
        dtz = p2 / fabs(rz);
    }

    /* incremental walk, ties x then y then z (operator.py:150-187) */
    double t = tmin, total = 0.0;
    for (;;) {
        double tn = tx;
        if (ty < tn) tn = ty;
        if (tz < tn) tn = tz;
        const double t_end = tn < tmax ? tn : tmax;
        const double seg = (t_end - t) * raylen;
        if (seg > SEG_EPS) {
            const int64_t lin = ix + n0 * (iy + n1 * iz);
            if (mode == 0) total += seg * vol[lin];
            else if (mode == 1) acc[lin] += seg * pixval;
            else acc[lin] += seg * seg;
        }
        if (tn >= tmax) break;
        t = tn;
        if (tx <= ty && tx <= tz) {
            ix += stx;
            if (ix < 0 || ix >= n0) break;
            tx += dtx;
        } else if (ty <= tz) {
            iy += sty;
            if (iy < 0 || iy >= n1) break;
            ty += dty;
        } else {
            iz += stz;
            if (iz < 0 || iz >= n2) break;
            tz += dtz;
        }
    }
    return total;
}

static inline void pixel(const double* det00, const double* ustep, const double* vstep, int64_t view,
                         int64_t u, int64_t v, double* px, double* py, double* pz) {
    /* operator.py:201-203 (same association order) */
    *px = det00[view * 3 + 0] + (double)u * ustep[view * 3 + 0] + (double)v * vstep[view * 3 + 0];
    *py = det00[view * 3 + 1] + (double)u * ustep[view * 3 + 1] + (double)v * vstep[view * 3 + 1];
    *pz = det00[view * 3 + 2] + (double)u * ustep[view * 3 + 2] + (double)v * vstep[view * 3 + 2];
}

/* operator.py:190-206: y = A x, one ray per detector pixel, u fastest then v then view. */
void oracle_project(const double* vol, double* out, const double* srcs, const double* det00,
                    const double* ustep, const double* vstep, int64_t n_views, int64_t nu, int64_t nv,
                    double lo0, double lo1, double lo2, double p0, double p1, double p2, int64_t n0,
                    int64_t n1, int64_t n2, int threads) {
    const int64_t nrays = n_views * nv * nu;
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 256) num_threads(threads)
#endif
    for (int64_t ray = 0; ray < nrays; ++ray) {
        const int64_t view = ray / (nv * nu);
        const int64_t rem = ray - view * nv * nu;
        const int64_t v = rem / nu;
        const int64_t u = rem - v * nu;
        const double sx = srcs[view * 3 + 0], sy = srcs[view * 3 + 1], sz = srcs[view * 3 + 2];
        double px, py, pz;
        pixel(det00, ustep, vstep, view, u, v, &px, &py, &pz);
        out[ray] = oracle_traverse(sx, sy, sz, px - sx, py - sy, pz - sz, lo0, lo1, lo2, p0, p1, p2, n0,
                                   n1, n2, 0, vol, NULL, 0.0);
    }
}

/* operator.py:209-233: out += A^T proj (mode 1) or diag(A^T A) (mode 2).
 * Worker w owns views w, w+W, ...; private accumulators merged in worker order. */
int oracle_backproject(const double* proj, double* out, const double* srcs, const double* det00,
                       const double* ustep, const double* vstep, int64_t n_views, int64_t nu, int64_t nv,
                       double lo0, double lo1, double lo2, double p0, double p1, double p2, int64_t n0,
                       int64_t n1, int64_t n2, int64_t n_workers, int mode, int threads) {
    const int64_t nvox = n0 * n1 * n2;
    if (n_workers < 1) return -1;
    double* acc = (double*)calloc((size_t)(n_workers * nvox), sizeof(double));
    if (!acc) return -2;
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
#endif
    for (int64_t w = 0; w < n_workers; ++w) {
        double* accw = acc + w * nvox;
        for (int64_t view = w; view < n_views; view += n_workers) {
            const double sx = srcs[view * 3 + 0], sy = srcs[view * 3 + 1], sz = srcs[view * 3 + 2];
            const int64_t base = view * nv * nu;
            for (int64_t v = 0; v < nv; ++v)
                for (int64_t u = 0; u < nu; ++u) {
                    double px, py, pz;
                    pixel(det00, ustep, vstep, view, u, v, &px, &py, &pz);
                    oracle_traverse(sx, sy, sz, px - sx, py - sy, pz - sz, lo0, lo1, lo2, p0, p1, p2, n0, n1,
                                    n2, mode, NULL, accw, proj ? proj[base + v * nu + u] : 1.0);
                }
        }
    }
    for (int64_t w = 0; w < n_workers; ++w) {
        const double* accw = acc + w * nvox;
        for (int64_t j = 0; j < nvox; ++j) out[j] += accw[j];
    }
    free(acc);
    return 0;
}

/* operator.py:236-259 + 364-374: (voxel index, length) pairs of one ray, count returned. */
int64_t oracle_ray_segments(double sx, double sy, double sz, double px, double py, double pz, double lo0,
                            double lo1, double lo2, double p0, double p1, double p2, int64_t n0, int64_t n1,
                            int64_t n2, int64_t* idx_out, double* len_out) {
    const int64_t nvox = n0 * n1 * n2;
    double* acc = (double*)calloc((size_t)nvox, sizeof(double));
    if (!acc) return -1;
    oracle_traverse(sx, sy, sz, px - sx, py - sy, pz - sz, lo0, lo1, lo2, p0, p1, p2, n0, n1, n2, 1, NULL, acc,
                    1.0);
    int64_t count = 0;
    for (int64_t j = 0; j < nvox; ++j)
        if (acc[j] != 0.0) { idx_out[count] = j; len_out[count] = acc[j]; ++count; }
    free(acc);
    return count;
}

/* Number of nonzeros of A over a view range (nnz = segments with seg > SEG_EPS). Used to
 * derive the algorithmic work of the roofline. */
static int64_t traverse_count(double sx, double sy, double sz, double rx, double ry, double rz, double lo0,
                              double lo1, double lo2, double p0, double p1, double p2, int64_t n0, int64_t n1,
                              int64_t n2) {
    /* Same walk as oracle_traverse; counts emitted segments instead of accumulating. */
    double tmin = 0.0, tmax = 1.0, t1, t2, tt;
    const double r[3] = {rx, ry, rz}, s[3] = {sx, sy, sz}, lo[3] = {lo0, lo1, lo2}, p[3] = {p0, p1, p2};
    const int64_t n[3] = {n0, n1, n2};
    for (int a = 0; a < 3; ++a) {
        if (fabs(r[a]) < 1e-12 * p[a]) {
            if (s[a] < lo[a] || s[a] >= lo[a] + (double)n[a] * p[a]) return 0;
        } else {
            t1 = (lo[a] - s[a]) / r[a];
            t2 = (lo[a] + (double)n[a] * p[a] - s[a]) / r[a];
            if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
            if (t1 > tmin) tmin = t1;
            if (t2 < tmax) tmax = t2;
        }
    }
    if (tmax <= tmin) return 0;
    const double raylen = sqrt(rx * rx + ry * ry + rz * rz);
    int64_t i[3];
    double tn3[3], dt[3];
    int st[3];
    for (int a = 0; a < 3; ++a) {
        i[a] = (int64_t)floor((s[a] + tmin * r[a] - lo[a]) / p[a]);
        if (i[a] < 0) i[a] = 0; else if (i[a] >= n[a]) i[a] = n[a] - 1;
        if (fabs(r[a]) < 1e-12 * p[a]) { tn3[a] = 1e300; dt[a] = 1e300; st[a] = 0; }
        else {
            st[a] = r[a] > 0 ? 1 : -1;
            tn3[a] = (lo[a] + (double)(i[a] + (st[a] > 0 ? 1 : 0)) * p[a] - s[a]) / r[a];
            dt[a] = p[a] / fabs(r[a]);
        }
    }
    double t = tmin;
    int64_t count = 0;
    for (;;) {
        double tn = tn3[0];
        if (tn3[1] < tn) tn = tn3[1];
        if (tn3[2] < tn) tn = tn3[2];
        const double te = tn < tmax ? tn : tmax;
        if ((te - t) * raylen > SEG_EPS) ++count;
        if (tn >= tmax) break;
        t = tn;
        int a = (tn3[0] <= tn3[1] && tn3[0] <= tn3[2]) ? 0 : (tn3[1] <= tn3[2] ? 1 : 2);
        i[a] += st[a];
        if (i[a] < 0 || i[a] >= n[a]) break;
        tn3[a] += dt[a];
    }
    return count;
}

int64_t oracle_count_nnz(const double* srcs, const double* det00, const double* ustep, const double* vstep,
                         int64_t view0, int64_t view1, int64_t nu, int64_t nv, double lo0, double lo1,
                         double lo2, double p0, double p1, double p2, int64_t n0, int64_t n1, int64_t n2,
                         int threads) {
    int64_t total = 0;
    const int64_t nrays = (view1 - view0) * nv * nu;
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total) num_threads(threads)
#endif
    for (int64_t k = 0; k < nrays; ++k) {
        const int64_t view = view0 + k / (nv * nu);
        const int64_t rem = k % (nv * nu);
        const int64_t v = rem / nu, u = rem % nu;
        const double sx = srcs[view * 3 + 0], sy = srcs[view * 3 + 1], sz = srcs[view * 3 + 2];
        double px, py, pz;
        pixel(det00, ustep, vstep, view, u, v, &px, &py, &pz);
        total += traverse_count(sx, sy, sz, px - sx, py - sy, pz - sz, lo0, lo1, lo2, p0, p1, p2, n0, n1, n2);
    }
    return total;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
