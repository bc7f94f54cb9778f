// f64.cu -- the fp64 "reference precision" path of libcbct: A, A^T, diag(A^T A), the solver
// vector kernels and the layout conversions, all in fp64 on the device layouts.
//
// Why it exists.  CGLS and LSQR in floating point lose orthogonality once the first Ritz
// values converge; from then on any rounding difference between two runs grows roughly
// geometrically until it saturates (measured: tests/golden/make_golden_trajectory.py --
// the reference itself, with only its worker count changed, i.e. another summation order in
// the backprojector merge, moves its own CGLS-40 iterate).  An fp32 operator (~1e-6 relative
// per application) therefore cannot track the reference's fp64 iterate to 1e-3 after 40
// iterations, whatever its vector precision.  This path computes every operator application
// and vector update in fp64, in the reference's arithmetic, so that it sits at the
// reference's own reproducibility floor.  The fp32 kernels (project.cu, backproject.cu,
// vec.cu) remain the fast path.
//
// Compiled with -fmad=false: no FMA contraction, so every expression rounds like the
// reference's NumPy / Numba code (operator.py, solvers.py), operation by operation.
//
//   k_project_f64   A x: one thread per ray, the reference's incremental Siddon walk
//                   (operator.py:53-187, mode 0) statement by statement; the column-major
//                   ray order (v fastest) keeps a warp's rays in one detector column.
//                   For a ray that enters through the side faces of the box this is
//                   bitwise the reference's _project_kernel value.
//   k_bp_f64        A^T y (mode 1) and diag(A^T A) (mode 2): voxel-driven deterministic (TwoSum-compensated)
//                   gather (no atomics), one CTA per cell, one thread per voxel, over the
//                   cell's list of crossing columns (plan.cu); per crossing the fp64 xy
//                   interval [t_a, t_b] is recomputed from the column's ray and the cell's
//                   planes, and each candidate ray's segment is the fp64 clip of that
//                   interval by the voxel's z planes, seg = dt * |r| (operator.py:158-167).
//   vector kernels  the NumPy updates of solvers.py:317-357, 429-452, 550-557 in fp64.
#include <cmath>

#include "cbct_internal.cuh"
#include "reduce.cuh"

namespace {

constexpr double kSegEps = 1e-12;  // operator.py:23
constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 8;

inline int vblocks(int64_t n) {
    const int64_t b = (n + kThreads - 1) / kThreads;
    return (int)(b < 1 ? 1 : (b > kMaxBlocks ? kMaxBlocks : b));
}

__device__ __forceinline__ void finish(double s, double* partials) {
    if (partials) {
        const double t = block_sum(s);
        if (threadIdx.x == 0) partials[blockIdx.x] = t;
    }
}

struct Grid3 {
    double lo0, lo1, lo2, p0, p1, p2;
    int64_t n0, n1, n2, zs;
};

// ---------------------------------------------------------------------------------- A --
// operator.py:53-187 with mode 0, reading the internal volume layout.
__device__ double walk_ray(const Grid3& g, double sx, double sy, double sz, double rx, double ry, double rz,
                           const double* __restrict__ vol) {
    double tmin = 0.0, tmax = 1.0, t1, t2, tt;
    if (fabs(rx) < 1e-12 * g.p0) {
        if (sx < g.lo0 || sx >= g.lo0 + (double)g.n0 * g.p0) return 0.0;
    } else {
        t1 = (g.lo0 - sx) / rx;
        t2 = (g.lo0 + (double)g.n0 * g.p0 - sx) / rx;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(ry) < 1e-12 * g.p1) {
        if (sy < g.lo1 || sy >= g.lo1 + (double)g.n1 * g.p1) return 0.0;
    } else {
        t1 = (g.lo1 - sy) / ry;
        t2 = (g.lo1 + (double)g.n1 * g.p1 - sy) / ry;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(rz) < 1e-12 * g.p2) {
        if (sz < g.lo2 || sz >= g.lo2 + (double)g.n2 * g.p2) return 0.0;
    } else {
        t1 = (g.lo2 - sz) / rz;
        t2 = (g.lo2 + (double)g.n2 * g.p2 - sz) / rz;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (tmax <= tmin) return 0.0;
    const double raylen = sqrt(rx * rx + ry * ry + rz * rz);
    int64_t ix = (int64_t)floor((sx + tmin * rx - g.lo0) / g.p0);
    int64_t iy = (int64_t)floor((sy + tmin * ry - g.lo1) / g.p1);
    int64_t iz = (int64_t)floor((sz + tmin * rz - g.lo2) / g.p2);
    ix = ix < 0 ? 0 : (ix >= g.n0 ? g.n0 - 1 : ix);
    iy = iy < 0 ? 0 : (iy >= g.n1 ? g.n1 - 1 : iy);
    iz = iz < 0 ? 0 : (iz >= g.n2 ? g.n2 - 1 : iz);
    const double big = 1e300;
    double tx, ty, tz, dtx, dty, dtz;
    int stx, sty, stz;
    if (fabs(rx) < 1e-12 * g.p0) { tx = big; dtx = big; stx = 0; }
    else { stx = rx > 0 ? 1 : -1; tx = (g.lo0 + (double)(ix + (stx > 0 ? 1 : 0)) * g.p0 - sx) / rx; dtx = g.p0 / fabs(rx); }
    if (fabs(ry) < 1e-12 * g.p1) { ty = big; dty = big; sty = 0; }
    else { sty = ry > 0 ? 1 : -1; ty = (g.lo1 + (double)(iy + (sty > 0 ? 1 : 0)) * g.p1 - sy) / ry; dty = g.p1 / fabs(ry); }
    if (fabs(rz) < 1e-12 * g.p2) { tz = big; dtz = big; stz = 0; }
    else { stz = rz > 0 ? 1 : -1; tz = (g.lo2 + (double)(iz + (stz > 0 ? 1 : 0)) * g.p2 - sz) / rz; dtz = g.p2 / fabs(rz); }
    double t = tmin, total = 0.0;
    // the cell column base moves only on x / y steps; z indexes inside it
    int64_t base = (iy * g.n0 + ix) * g.zs + CBCT_ZPAD;
    for (;;) {
        double tn = tx;
        if (ty < tn) tn = ty;
        if (tz < tn) tn = tz;
        const double t_end = tn < tmax ? tn : tmax;
        const double seg = (t_end - t) * raylen;
        if (seg > kSegEps) total += seg * __ldg(vol + base + iz);
        if (tn >= tmax) break;
        t = tn;
        if (tx <= ty && tx <= tz) {
            ix += stx;
            if (ix < 0 || ix >= g.n0) break;
            tx += dtx;
            base += stx * g.zs;
        } else if (ty <= tz) {
            iy += sty;
            if (iy < 0 || iy >= g.n1) break;
            ty += dty;
            base += sty * g.n0 * g.zs;
        } else {
            iz += stz;
            if (iz < 0 || iz >= g.n2) break;
            tz += dtz;
        }
    }
    return total;
}

// y[c*nv + v] = walk of ray (view, u, v), c = view*nu + u; grid-stride over rays, so each
// thread's rays and its partial of ||y||^2 are fixed by the launch shape (deterministic).
// Four CTAs per SM (64 registers): the walk is latency-bound on its volume loads and its fp64
// dependency chain, so occupancy pays (config 3: 810 -> 624 ms at 78 registers / 37% occupancy).
__global__ void __launch_bounds__(256, 4) k_project_f64(Grid3 g, const double* __restrict__ srcs,
                                                   const double* __restrict__ det00,
                                                   const double* __restrict__ ustep,
                                                   const double* __restrict__ vstep, int64_t nu, int64_t nv,
                                                   int64_t n_rays, const double* __restrict__ vol,
                                                   double* __restrict__ out, double* __restrict__ partials) {
    double sq = 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_rays; i += stride) {
        const int64_t c = i / nv, v = i - c * nv;
        const int64_t view = c / nu, u = c - view * nu;
        const double* s = srcs + view * 3;
        const double* d0 = det00 + view * 3;
        const double* us = ustep + view * 3;
        const double* vs = vstep + view * 3;
        // operator.py:200-204: pixel = det00 + u*ustep + v*vstep, r = pixel - src
        const double px = d0[0] + (double)u * us[0] + (double)v * vs[0];
        const double py = d0[1] + (double)u * us[1] + (double)v * vs[1];
        const double pz = d0[2] + (double)u * us[2] + (double)v * vs[2];
        const double val = walk_ray(g, s[0], s[1], s[2], px - s[0], py - s[1], pz - s[2], vol);
        out[i] = val;
        sq += val * val;
    }
    finish(sq, partials);
}

// ------------------------------------------------------------------------------- A^T --
// To reproduce the reference's segment values bit for bit, the gather uses the reference's
// own crossing parameters: the x/y plane parameters of a column's walk (tx += dtx,
// ty += dty, operator.py:171-180 -- identical for every ray of the column that enters
// through the side faces) and, per ray, the accumulated z plane parameters (tz += dtz,
// operator.py:181-186) from the ray's own entry slab.  A visit of ray v to voxel (cell, iz)
// then spans [max(t_a, t_in), min(t_b, t_out, tmax)] with t_a/t_b the column's crossing of
// the cell and t_in/t_out the ray's z crossings -- the walk's own t and t_end, so
// seg = (t_end - t) * |r| is the reference's value and only the summation order differs
// (the reference's own worker count changes that too).

struct RayZ {  // per ray, internal order: the prologue of _traverse (operator.py:60-148), |r|, entry slab
    double tmin, tmax, tz0, dtz, len;
    int iz0, step;  // entry slab and z step (0 for a flat ray)
};

// |r|, the box clip and the z walk start of every ray (operator.py:60-148).
__global__ void k_ray_table_f64(Grid3 g, const double* __restrict__ srcs, const double* __restrict__ det00,
                                const double* __restrict__ ustep, const double* __restrict__ vstep, int64_t nu,
                                int64_t nv, int64_t n_rays, double* __restrict__ len, RayZ* __restrict__ rz_tab,
                                int2* __restrict__ iz_tab) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_rays) return;
    const int64_t c = i / nv, v = i - c * nv;
    const int64_t view = c / nu, u = c - view * nu;
    const double sx = srcs[view * 3 + 0], sy = srcs[view * 3 + 1], sz = srcs[view * 3 + 2];
    const double px = det00[view * 3 + 0] + (double)u * ustep[view * 3 + 0] + (double)v * vstep[view * 3 + 0];
    const double py = det00[view * 3 + 1] + (double)u * ustep[view * 3 + 1] + (double)v * vstep[view * 3 + 1];
    const double pz = det00[view * 3 + 2] + (double)u * ustep[view * 3 + 2] + (double)v * vstep[view * 3 + 2];
    const double rx = px - sx, ry = py - sy, rz = pz - sz;
    len[i] = sqrt(rx * rx + ry * ry + rz * rz);
    RayZ out{0.0, 0.0, 1e300, 1e300, 0.0, 0, 0};
    int2 iz_st = make_int2(0, 0);
    double tmin = 0.0, tmax = 1.0, t1, t2, tt;
    bool hit = true;
    if (fabs(rx) < 1e-12 * g.p0) {
        if (sx < g.lo0 || sx >= g.lo0 + (double)g.n0 * g.p0) hit = false;
    } else {
        t1 = (g.lo0 - sx) / rx;
        t2 = (g.lo0 + (double)g.n0 * g.p0 - sx) / rx;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(ry) < 1e-12 * g.p1) {
        if (sy < g.lo1 || sy >= g.lo1 + (double)g.n1 * g.p1) hit = false;
    } else {
        t1 = (g.lo1 - sy) / ry;
        t2 = (g.lo1 + (double)g.n1 * g.p1 - sy) / ry;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(rz) < 1e-12 * g.p2) {
        if (sz < g.lo2 || sz >= g.lo2 + (double)g.n2 * g.p2) hit = false;
    } else {
        t1 = (g.lo2 - sz) / rz;
        t2 = (g.lo2 + (double)g.n2 * g.p2 - sz) / rz;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (hit && tmax > tmin) {
        out.tmin = tmin;
        out.tmax = tmax;
        int64_t iz = (int64_t)floor((sz + tmin * rz - g.lo2) / g.p2);
        iz = iz < 0 ? 0 : (iz >= g.n2 ? g.n2 - 1 : iz);
        iz_st.x = (int)iz;
        if (!(fabs(rz) < 1e-12 * g.p2)) {
            const int stz = rz > 0 ? 1 : -1;
            out.tz0 = (g.lo2 + (double)(iz + (stz > 0 ? 1 : 0)) * g.p2 - sz) / rz;
            out.dtz = g.p2 / fabs(rz);
            iz_st.y = stz;
        }
    }
    out.len = len[i];
    out.iz0 = iz_st.x;
    out.step = iz_st.y;
    rz_tab[i] = out;
    iz_tab[i] = iz_st;
}

// The xy walk of every column (operator.py:60-180, x and y only, -fmad=false): te64[k] for
// the column's k-th interval, in the order plan.cu's k_column_fill wrote them.  A column
// whose interval count differs from the plan's (a rounding tie the fp32 tables resolved
// differently) is flagged and its crossings fall back to direct plane parameters.
__global__ void k_col_walk64(Grid3 g, const double* __restrict__ srcs, const double* __restrict__ det00,
                             const double* __restrict__ ustep, int64_t nu, int64_t n_cols,
                             const int64_t* __restrict__ col_off, double* __restrict__ te64,
                             double2* __restrict__ col_clip, int* __restrict__ bad) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cols) return;
    const int64_t view = c / nu, u = c - view * nu;
    const double sx = srcs[view * 3 + 0], sy = srcs[view * 3 + 1];
    const double rx = (det00[view * 3 + 0] + (double)u * ustep[view * 3 + 0]) - sx;
    const double ry = (det00[view * 3 + 1] + (double)u * ustep[view * 3 + 1]) - sy;
    double tmin = 0.0, tmax = 1.0, t1, t2, tt;
    bool hit = true;
    if (fabs(rx) < 1e-12 * g.p0) {
        if (sx < g.lo0 || sx >= g.lo0 + (double)g.n0 * g.p0) hit = false;
    } else {
        t1 = (g.lo0 - sx) / rx;
        t2 = (g.lo0 + (double)g.n0 * g.p0 - sx) / rx;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(ry) < 1e-12 * g.p1) {
        if (sy < g.lo1 || sy >= g.lo1 + (double)g.n1 * g.p1) hit = false;
    } else {
        t1 = (g.lo1 - sy) / ry;
        t2 = (g.lo1 + (double)g.n1 * g.p1 - sy) / ry;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    col_clip[c] = make_double2(tmin, tmax);
    const int64_t k0 = col_off[c], n = col_off[c + 1] - k0;
    if (!hit || !(tmax > tmin)) {
        bad[c] = n != 0;
        return;
    }
    int64_t ix = (int64_t)floor((sx + tmin * rx - g.lo0) / g.p0);
    int64_t iy = (int64_t)floor((sy + tmin * ry - g.lo1) / g.p1);
    ix = ix < 0 ? 0 : (ix >= g.n0 ? g.n0 - 1 : ix);
    iy = iy < 0 ? 0 : (iy >= g.n1 ? g.n1 - 1 : iy);
    const double big = 1e300;
    double tx, ty, dtx, dty;
    int stx, sty;
    if (fabs(rx) < 1e-12 * g.p0) { tx = big; dtx = big; stx = 0; }
    else { stx = rx > 0 ? 1 : -1; tx = (g.lo0 + (double)(ix + (stx > 0 ? 1 : 0)) * g.p0 - sx) / rx; dtx = g.p0 / fabs(rx); }
    if (fabs(ry) < 1e-12 * g.p1) { ty = big; dty = big; sty = 0; }
    else { sty = ry > 0 ? 1 : -1; ty = (g.lo1 + (double)(iy + (sty > 0 ? 1 : 0)) * g.p1 - sy) / ry; dty = g.p1 / fabs(ry); }
    double t = tmin;
    int64_t k = 0;
    for (;;) {
        const double tn = ty < tx ? ty : tx;
        const double te = tn < tmax ? tn : tmax;
        if (te > t) {
            if (k < n) te64[k0 + k] = te;
            ++k;
        }
        if (tn >= tmax) break;
        t = tn;
        if (tx <= ty) {
            ix += stx;
            if (ix < 0 || ix >= g.n0) break;
            tx += dtx;
        } else {
            iy += sty;
            if (iy < 0 || iy >= g.n1) break;
            ty += dty;
        }
    }
    bad[c] = k != n;
}

// Per cell entry: the column's walk parameters bounding its crossing of the cell.  The
// entry's interval is found in the column's fp32 list by its tau_end (exact copy) and cell.
__global__ void k_cell_t64(Grid3 g, const int64_t* __restrict__ cell_off, const CellEntry* __restrict__ cell_ent,
                           const int64_t* __restrict__ col_off, const float2* __restrict__ col_ent,
                           const double* __restrict__ te64, const double2* __restrict__ col_clip,
                           const int* __restrict__ bad, const double* __restrict__ srcs,
                           const double* __restrict__ det00, const double* __restrict__ ustep, int64_t nu,
                           double2* __restrict__ out) {
    const int64_t cell = blockIdx.x;
    const int ix = (int)(cell % g.n0), iy = (int)(cell / g.n0);
    const int cbase = (int)(cell * g.zs);
    for (int64_t k = cell_off[cell] + threadIdx.x; k < cell_off[cell + 1]; k += blockDim.x) {
        const CellEntry ce = cell_ent[k];
        const int64_t c = ce.vu, a = col_off[c], b = col_off[c + 1];
        int64_t e = -1;
        if (!bad[c]) {
            int64_t lo = a, hi = b;  // first entry with tau_end >= tau_b
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (col_ent[mid].x < ce.tau_b) lo = mid + 1; else hi = mid;
            }
            for (; lo < b && col_ent[lo].x == ce.tau_b; ++lo)
                if (__float_as_int(col_ent[lo].y) == cbase) { e = lo; break; }
        }
        if (e >= 0) {
            out[k] = make_double2(e == a ? col_clip[c].x : te64[e - 1], te64[e]);
        } else {  // fallback: direct plane parameters of the cell (rounding-level differences)
            const int64_t view = c / nu, u = c - view * nu;
            const double sx = srcs[view * 3 + 0], sy = srcs[view * 3 + 1];
            const double rx = (det00[view * 3 + 0] + (double)u * ustep[view * 3 + 0]) - sx;
            const double ry = (det00[view * 3 + 1] + (double)u * ustep[view * 3 + 1]) - sy;
            double ta = col_clip[c].x, tb = col_clip[c].y;
            if (!(fabs(rx) < 1e-12 * g.p0)) {
                double t1 = (g.lo0 + (double)ix * g.p0 - sx) / rx, t2 = (g.lo0 + (double)(ix + 1) * g.p0 - sx) / rx;
                if (t1 > t2) { const double tt = t1; t1 = t2; t2 = tt; }
                ta = fmax(ta, t1);
                tb = fmin(tb, t2);
            }
            if (!(fabs(ry) < 1e-12 * g.p1)) {
                double t1 = (g.lo1 + (double)iy * g.p1 - sy) / ry, t2 = (g.lo1 + (double)(iy + 1) * g.p1 - sy) / ry;
                if (t1 > t2) { const double tt = t1; t1 = t2; t2 = tt; }
                ta = fmax(ta, t1);
                tb = fmin(tb, t2);
            }
            out[k] = make_double2(ta, tb);
        }
    }
}

struct Cross {  // one staged crossing (column c, the walk's parameters bounding it)
    double ta, tb;
    float ia, ib;  // 1 / (t pv) at both ends, fp32: only bound the candidate rows
    int c, pad;
};

constexpr int kChunk = 128;

__device__ __forceinline__ int64_t tiled_cell(int64_t b, int nx, int row0, int row1) {
    const int T = 16;
    const int tx = (nx + T - 1) / T;
    const int64_t per_tile = (int64_t)T * T;
    const int64_t tile = b / per_tile;
    const int k = (int)(b - tile * per_tile);
    const int ty0 = row0 + (int)(tile / tx) * T, tx0 = (int)(tile % tx) * T;
    const int iy = ty0 + k / T, ix = tx0 + k % T;
    if (ix >= nx || iy >= row1) return -1;
    return (int64_t)iy * nx + ix;
}

// Voxel-driven fp64 gather: one CTA per cell, one thread per voxel (ZPT per thread).
template <int ZPT>
__global__ void __launch_bounds__(512) k_bp_f64(const int64_t* __restrict__ cell_off,
                                              const CellEntry* __restrict__ cell_ent,
                                              const double2* __restrict__ cell_t,
                                              const double* __restrict__ wtab, const double* __restrict__ len,
                                              const RayZ* __restrict__ rz_tab, const int2* __restrict__ iz_tab,
                                              const double* __restrict__ y, double* __restrict__ vol,
                                              const double* __restrict__ col_scale, double* __restrict__ partials,
                                              Grid3 g, int nv, double det00z, double pv, int mode, int row0,
                                              int row1) {
    __shared__ Cross s_x[kChunk];
    const int nx = (int)g.n0, nz = (int)g.n2;
    const int64_t cell = tiled_cell(blockIdx.x, nx, row0, row1);
    if (cell < 0) {
        if (partials && threadIdx.x == 0) partials[blockIdx.x] = 0.0;
        return;
    }
    const int64_t off = cell_off[cell];
    const int ne = (int)(cell_off[cell + 1] - off);
    double z0[ZPT], z1[ZPT], acc[ZPT], cmp[ZPT];
    float zf0[ZPT], zf1[ZPT];
    const float c0p = (float)(det00z / pv);
    int iz[ZPT];
#pragma unroll
    for (int r = 0; r < ZPT; ++r) {
        iz[r] = threadIdx.x + r * blockDim.x;
        z0[r] = g.lo2 + (double)iz[r] * g.p2;
        zf0[r] = (float)z0[r];
        z1[r] = g.lo2 + (double)(iz[r] + 1) * g.p2;
        zf1[r] = (float)z1[r];
        acc[r] = 0.0;
        cmp[r] = 0.0;
    }
    for (int base = 0; base < ne; base += kChunk) {
        const int nch = min(kChunk, ne - base);
        __syncthreads();
        for (int k = threadIdx.x; k < nch; k += blockDim.x) {
            const double2 t = cell_t[off + base + k];
            s_x[k] = Cross{t.x, t.y, (float)(1.0 / (t.x * pv)), (float)(1.0 / (t.y * pv)), cell_ent[off + base + k].vu, 0};
        }
        __syncthreads();
        for (int k = 0; k < nch; ++k) {
            const Cross x = s_x[k];
            if (!(x.tb > x.ta)) continue;
            const int64_t rb = (int64_t)x.c * nv;

#pragma unroll
            for (int r = 0; r < ZPT; ++r) {
                if (iz[r] >= nz) continue;
                // candidate rows from the direct plane parameters: a ray can meet the voxel inside the
                // crossing only if its row lies in [vmin, vmax]; 1e-6 rows of margin cover the
                // rounding of these bounds (the exact clip below decides)
                // (fp32 bounds: ~1e-4 rows of rounding at |v| ~ 1000, covered by 2e-3 rows of margin)
                const float qa0 = zf0[r] * x.ia, qb0 = zf0[r] * x.ib, qa1 = zf1[r] * x.ia, qb1 = zf1[r] * x.ib;
                const float vmin = fminf(fminf(qa0, qb0), fminf(qa1, qb1)) - c0p;
                const float vmax = fmaxf(fmaxf(qa0, qb0), fmaxf(qa1, qb1)) - c0p;
                const int va = max(0, (int)ceilf(vmin - 2e-3f));
                const int vb = min(nv - 1, (int)floorf(vmax + 2e-3f));
                for (int v = va; v <= vb; ++v) {
                    const int64_t ray = rb + v;
                    const RayZ q = rz_tab[ray];  // one 48-byte record per candidate
                    const int d = (iz[r] - q.iz0) * q.step;  // z steps from the entry slab to this slab
                    if (q.step == 0 ? iz[r] != q.iz0 : d < 0) continue;
                    double t_in = -1e300, t_out = q.tz0;  // accumulated z planes (tz += dtz)
                    for (int j = 0; j < d; ++j) {
                        t_in = t_out;
                        t_out = t_out + q.dtz;
                    }
                    const double t0 = fmax(fmax(x.ta, q.tmin), t_in);
                    double t1 = x.tb < t_out ? x.tb : t_out;
                    t1 = t1 < q.tmax ? t1 : q.tmax;
                    const double seg = (t1 - t0) * q.len;  // operator.py:158-159
                    if (seg > kSegEps) {  // operator.py:162-167
                        // compensated (TwoSum) accumulation: the voxel's sum of the same rounded
                        // products as the reference's, rounded once at the end, so our summation
                        // order adds no error of its own (the reference's merge order differs by W)
                        const double v = mode == 1 ? seg * y[ray] : seg * seg;
                        const double sm = acc[r] + v;
                        const double bv = sm - acc[r];
                        cmp[r] += (acc[r] - (sm - bv)) + (v - bv);
                        acc[r] = sm;
                    }
                }
            }
        }
    }
    const int64_t lcell = cell - (int64_t)row0 * nx;
    double* out = vol + lcell * g.zs;
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < ZPT; ++r) {
        if (iz[r] < nz) {
            double val = acc[r] + cmp[r];
            if (col_scale) val = col_scale[lcell * g.zs + CBCT_ZPAD + iz[r]] * val;
            out[CBCT_ZPAD + iz[r]] = val;
            sq += val * val;
        }
    }
    for (int k = threadIdx.x; k < g.zs - nz; k += blockDim.x) out[k < CBCT_ZPAD ? k : nz + k] = 0.0;
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}

// --------------------------------------------------------------------------- vectors --
// The NumPy updates in the reference's rounding: every product and sum rounded separately.
__global__ void k_axpby64(int64_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y,
                          double* __restrict__ partials) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = x ? a * x[i] + b * y[i] : b * y[i];
        y[i] = v;
        sq += v * v;
    }
    finish(sq, partials);
}

__global__ void k_scale_div64(int64_t n, double* __restrict__ y, double d, double* __restrict__ partials) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = y[i] / d;  // u /= beta (solvers.py:407, 434, 441)
        y[i] = v;
        sq += v * v;
    }
    finish(sq, partials);
}

__global__ void k_sub64(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                        double* __restrict__ out, double* __restrict__ partials) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const double v = a[i] - b[i];
        out[i] = v;
        sq += v * v;
    }
    finish(sq, partials);
}

__global__ void k_dot64(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                        double* __restrict__ partials) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) s += x[i] * y[i];
    finish(s, partials);
}

__global__ void k_mul64(int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                        double* __restrict__ o) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) o[i] = a[i] * b[i];
}

// x += alpha_prev * d (if do_x) ; d = beta * d + r   (solvers.py:340-341, 354: d_x *= beta; d_x += r_x)
__global__ void k_cgls_volume64(int64_t n, double* __restrict__ x, double* __restrict__ d,
                                const double* __restrict__ r, double alpha_prev, int do_x, double beta) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const double dv = d[i];
        if (do_x) x[i] = x[i] + alpha_prev * dv;
        d[i] = dv * beta + r[i];
    }
}

__global__ void k_fill_volume64(int64_t n, int64_t zs, int64_t nz, double* __restrict__ x, double v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t k = i % zs;
        x[i] = (k >= CBCT_ZPAD && k < CBCT_ZPAD + nz) ? v : 0.0;
    }
}

__global__ void k_clip64(int64_t n, int64_t zs, int64_t nz, double* __restrict__ x, double lo, double hi) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t k = i % zs;
        if (k >= CBCT_ZPAD && k < CBCT_ZPAD + nz) x[i] = fmin(fmax(x[i], lo), hi);  // np.clip
    }
}

// --------------------------------------------------------------------------- layouts --
constexpr int T = 32;

// out[b][c*ostride + ooff + r] = in[b][r*C + c]
__global__ void k_transpose64(const double* __restrict__ in, double* __restrict__ out, int64_t R, int64_t C,
                              int64_t ostride, int64_t ooff, int64_t in_batch, int64_t out_batch) {
    __shared__ double tile[T][T + 1];
    const int64_t b = blockIdx.z;
    const int64_t r0 = (int64_t)blockIdx.y * T, c0 = (int64_t)blockIdx.x * T;
    const double* ib = in + b * in_batch;
    double* ob = out + b * out_batch;
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < R && c < C) tile[i][threadIdx.x] = ib[r * C + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < R && c < C) ob[c * ostride + ooff + r] = tile[threadIdx.x][i];
    }
}

// out[b][r*C + c] = in[b][c*istride + ioff + r]
__global__ void k_transpose_back64(const double* __restrict__ in, double* __restrict__ out, int64_t R, int64_t C,
                                   int64_t istride, int64_t ioff, int64_t in_batch, int64_t out_batch) {
    __shared__ double tile[T][T + 1];
    const int64_t b = blockIdx.z;
    const int64_t r0 = (int64_t)blockIdx.y * T, c0 = (int64_t)blockIdx.x * T;
    const double* ib = in + b * in_batch;
    double* ob = out + b * out_batch;
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < R && c < C) tile[threadIdx.x][i] = ib[c * istride + ioff + r];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < R && c < C) ob[r * C + c] = tile[i][threadIdx.x];
    }
}

__global__ void k_zero_guards64(double* vol, int64_t n_cells, int64_t zs, int64_t nz) {
    const int64_t ng = zs - nz;
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_cells * ng) return;
    const int64_t cell = i / ng;
    const int64_t k = i - cell * ng;
    vol[cell * zs + (k < CBCT_ZPAD ? k : nz + k)] = 0.0;
}

int tr(const double* in, double* out, int64_t R, int64_t C, int64_t ostride, int64_t ooff, int64_t nb,
       int64_t ib, int64_t ob, cudaStream_t s, bool back) {
    dim3 grid((unsigned)((C + T - 1) / T), (unsigned)((R + T - 1) / T), (unsigned)nb);
    if (back) k_transpose_back64<<<grid, dim3(T, 8), 0, s>>>(in, out, R, C, ostride, ooff, ib, ob);
    else k_transpose64<<<grid, dim3(T, 8), 0, s>>>(in, out, R, C, ostride, ooff, ib, ob);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

Grid3 grid3(const cbct_plan* p) {
    return Grid3{p->lo[0], p->lo[1], p->lo[2], p->pitch[0], p->pitch[1], p->pitch[2], p->nx, p->ny, p->nz, p->zs};
}

}  // namespace

// ------------------------------------------------------------------------------ C ABI --
extern "C" int cbct_plan_enable_f64(cbct_plan* p, void* stream) {
    if (!p) return cbct_fail(CBCT_E_ARG, "cbct_plan_enable_f64: null plan");
    if (p->sharded) return cbct_fail(CBCT_E_ARG, "cbct_plan_enable_f64: the fp64 path needs an unsharded plan");
    if (p->d_len64) return 0;
    cudaStream_t s = (cudaStream_t)stream;
    const Grid3 g = grid3(p);
    const int64_t nr = p->n_rays, ni = p->n_intervals, nc = p->n_cols;
    double* te64 = nullptr;
    double2* clip = nullptr;
    int* bad = nullptr;
    CBCT_CHECK(cudaMalloc((void**)&p->d_len64, (size_t)nr * sizeof(double)));
    CBCT_CHECK(cudaMalloc((void**)&p->d_rayz64, (size_t)nr * sizeof(RayZ)));
    CBCT_CHECK(cudaMalloc((void**)&p->d_rayiz64, (size_t)nr * sizeof(int2)));
    CBCT_CHECK(cudaMalloc((void**)&p->d_cell_t64, (size_t)(ni ? ni : 1) * sizeof(double2)));
    p->table_bytes += (size_t)nr * (sizeof(double) + sizeof(RayZ) + sizeof(int2)) + (size_t)ni * sizeof(double2);
    k_ray_table_f64<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(g, p->d_srcs, p->d_det00, p->d_ustep, p->d_vstep,
                                                                 p->nu, p->nv, nr, p->d_len64,
                                                                 (RayZ*)p->d_rayz64, (int2*)p->d_rayiz64);
    CBCT_CHECK(cudaGetLastError());
    CBCT_CHECK(cudaMalloc((void**)&te64, (size_t)(ni ? ni : 1) * sizeof(double)));
    CBCT_CHECK(cudaMalloc((void**)&clip, (size_t)nc * sizeof(double2)));
    CBCT_CHECK(cudaMalloc((void**)&bad, (size_t)nc * sizeof(int)));
    k_col_walk64<<<(unsigned)((nc + 127) / 128), 128, 0, s>>>(g, p->d_srcs, p->d_det00, p->d_ustep, p->nu, nc,
                                                              p->d_col_off, te64, clip, bad);
    CBCT_CHECK(cudaGetLastError());
    k_cell_t64<<<(unsigned)p->n_cells, 128, 0, s>>>(g, p->d_cell_off, p->d_cell_ent, p->d_col_off, p->d_col_ent,
                                                     te64, clip, bad, p->d_srcs, p->d_det00, p->d_ustep, p->nu,
                                                     (double2*)p->d_cell_t64);
    CBCT_CHECK(cudaGetLastError());
    CBCT_CHECK(cudaStreamSynchronize(s));
    cudaFree(te64);
    cudaFree(clip);
    cudaFree(bad);
    cbct_count_launch(3);
    return 0;
}

extern "C" int cbct_f64_vec_blocks(int64_t n) { return vblocks(n); }

extern "C" int cbct_project_f64(const cbct_plan* p, const double* vol, double* proj, double* partials,
                                void* stream) {
    CbctRange range("cbct_project_f64");
    if (!p || !vol || !proj) return cbct_fail(CBCT_E_ARG, "cbct_project_f64: null argument");
    const int blocks = cbct_f64_proj_blocks(p);
    k_project_f64<<<blocks, 256, 0, (cudaStream_t)stream>>>(grid3(p), p->d_srcs, p->d_det00, p->d_ustep, p->d_vstep,
                                                           p->nu, p->nv, p->n_rays, vol, proj, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_f64_proj_blocks(const cbct_plan* p) {
    const int64_t b = (p->n_rays + 255) / 256;
    return (int)(b < 148 * 16 ? b : 148 * 16);
}

extern "C" int cbct_backproject_f64(const cbct_plan* p, const double* proj, double* vol, int mode,
                                    const double* col_scale, double* partials, void* stream) {
    CbctRange range(mode == 2 ? "cbct_normal_diagonal_f64" : "cbct_backproject_f64");
    if (!p || !vol) return cbct_fail(CBCT_E_ARG, "cbct_backproject_f64: null argument");
    if (mode != 1 && mode != 2) return cbct_fail(CBCT_E_ARG, "cbct_backproject_f64: mode must be 1 or 2");
    if (mode == 1 && !proj) return cbct_fail(CBCT_E_ARG, "cbct_backproject_f64: mode 1 needs projections");
    if (!p->d_len64) return cbct_fail(CBCT_E_ARG, "cbct_backproject_f64: call cbct_plan_enable_f64 first");
    cudaStream_t s = (cudaStream_t)stream;
    const dim3 grid((unsigned)(((p->nx + 15) / 16) * ((p->ny + 15) / 16) * 256));
#define LAUNCH64(Z)                                                                                          \
    do {                                                                                                     \
        k_bp_f64<Z><<<grid, p->bp_threads, 0, s>>>(p->d_cell_off, p->d_cell_ent, (const double2*)p->d_cell_t64, \
                                                      p->d_w, p->d_len64, (const RayZ*)p->d_rayz64,             \
                                                      (const int2*)p->d_rayiz64, proj, vol, col_scale, partials, \
                                                      grid3(p), (int)p->nv, p->det00z, p->pv, mode, 0,          \
                                                      (int)p->ny);                                              \
    } while (0)
    switch (p->bp_zpt) {
        case 1: LAUNCH64(1); break;
        case 2: LAUNCH64(2); break;
        default: LAUNCH64(4); break;
    }
#undef LAUNCH64
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_axpby_f64(int64_t n, double a, const double* x, double b, double* y, double* partials,
                              void* stream) {
    if (!y) return cbct_fail(CBCT_E_ARG, "cbct_axpby_f64: null y");
    k_axpby64<<<vblocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, a, x, b, y, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_scale_div_f64(int64_t n, double* y, double d, double* partials, void* stream) {
    if (!y) return cbct_fail(CBCT_E_ARG, "cbct_scale_div_f64: null y");
    k_scale_div64<<<vblocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, y, d, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_sub_f64(int64_t n, const double* a, const double* b, double* out, double* partials,
                            void* stream) {
    if (!a || !b || !out) return cbct_fail(CBCT_E_ARG, "cbct_sub_f64: null argument");
    k_sub64<<<vblocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, a, b, out, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_dot_f64(int64_t n, const double* x, const double* y, double* partials, void* stream) {
    if (!x || !y || !partials) return cbct_fail(CBCT_E_ARG, "cbct_dot_f64: null argument");
    k_dot64<<<vblocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, y, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_mul_f64(int64_t n, const double* a, const double* b, double* out, void* stream) {
    if (!a || !b || !out) return cbct_fail(CBCT_E_ARG, "cbct_mul_f64: null argument");
    k_mul64<<<vblocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, a, b, out);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_cgls_volume_update_f64(int64_t n, double* x, double* d, const double* r, double alpha_prev,
                                           int do_x, double beta, void* stream) {
    if (!d || !r || (do_x && !x)) return cbct_fail(CBCT_E_ARG, "cbct_cgls_volume_update_f64: null argument");
    k_cgls_volume64<<<vblocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, d, r, alpha_prev, do_x, beta);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_fill_volume_f64(const cbct_plan* p, double* vol, double value, void* stream) {
    if (!p || !vol) return cbct_fail(CBCT_E_ARG, "cbct_fill_volume_f64: null argument");
    k_fill_volume64<<<vblocks(p->vol_elems), kThreads, 0, (cudaStream_t)stream>>>(p->vol_elems, p->zs, p->nz, vol,
                                                                                   value);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_clip_f64(const cbct_plan* p, double* vol, double lo, double hi, void* stream) {
    if (!p || !vol) return cbct_fail(CBCT_E_ARG, "cbct_clip_f64: null argument");
    k_clip64<<<vblocks(p->vol_elems), kThreads, 0, (cudaStream_t)stream>>>(p->vol_elems, p->zs, p->nz, vol, lo, hi);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_volume_to_internal_f64(const cbct_plan* p, const double* src, double* dst, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_volume_to_internal_f64: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    int rc = tr(src, dst, p->nz, p->n_cells, p->zs, CBCT_ZPAD, 1, 0, 0, s, false);
    if (rc) return rc;
    const int64_t ng = p->n_cells * (p->zs - p->nz);
    k_zero_guards64<<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(dst, p->n_cells, p->zs, p->nz);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_volume_from_internal_f64(const cbct_plan* p, const double* src, double* dst, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_volume_from_internal_f64: null argument");
    return tr(src, dst, p->nz, p->n_cells, p->zs, CBCT_ZPAD, 1, 0, 0, (cudaStream_t)stream, true);
}

extern "C" int cbct_proj_to_internal_f64(const cbct_plan* p, const double* src, double* dst, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_proj_to_internal_f64: null argument");
    const int64_t per = p->nu * p->nv;
    return tr(src, dst, p->nv, p->nu, p->nv, 0, p->V, per, per, (cudaStream_t)stream, false);
}

extern "C" int cbct_proj_from_internal_f64(const cbct_plan* p, const double* src, double* dst, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_proj_from_internal_f64: null argument");
    const int64_t per = p->nu * p->nv;
    return tr(src, dst, p->nv, p->nu, p->nv, 0, p->V, per, per, (cudaStream_t)stream, true);
}
