// plan.cu -- builds the device-resident 2-D fan-beam tables of one operator.
//
// Geometry facts used (all hold for every trajectory the reference can build,
// geometry.py:144-164): the source is at z = 0, the detector v axis is +z and
// the u axis is horizontal.  Hence every ray of a detector column (view, u)
// shares (rx, ry): the column's rays all lie in one vertical plane and cross
// the same sequence of (ix, iy) cells at the same ray parameters t.  Only the
// z walk differs from ray to ray (rz = det00z + v*pv).
//
// The xy walk below restates the x/y part of _traverse (operator.py:60-186)
// in fp64: same box clip, same axis-parallel rule (|r| < 1e-12 * pitch), same
// clamped entry cell, same incremental plane parameters and tie order.  It
// runs once per operator; the projector and backprojector then stream the
// resulting fp32 tables.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "cbct_internal.cuh"

namespace {

struct GeomDev {
    double lo0, lo1, p0, p1;
    int64_t nx, ny, nu, zs;
};

// Walk the xy part of one column.  Calls emit(tau_end_double, ix, iy) for every
// interval of non-zero length; returns the number of intervals.
template <typename Emit>
__device__ int64_t walk_column(const GeomDev& g, double sx, double sy, double rx, double ry, double tmin,
                               double tmax, Emit emit) {
    int64_t ix = (int64_t)floor((sx + tmin * rx - g.lo0) / g.p0);  // operator.py:105-111
    int64_t iy = (int64_t)floor((sy + tmin * ry - g.lo1) / g.p1);
    if (ix < 0) ix = 0; else if (ix >= g.nx) ix = g.nx - 1;
    if (iy < 0) iy = 0; else if (iy >= g.ny) iy = g.ny - 1;
    const double big = 1e300;
    double tx, ty, dtx, dty;
    int stx, sty;
    if (fabs(rx) < 1e-12 * g.p0) { tx = big; dtx = big; stx = 0; }  // operator.py:122-130
    else {
        stx = rx > 0 ? 1 : -1;
        const double plane = g.lo0 + (double)(ix + (stx > 0 ? 1 : 0)) * g.p0;
        tx = (plane - sx) / rx;
        dtx = g.p0 / fabs(rx);
    }
    if (fabs(ry) < 1e-12 * g.p1) { ty = big; dty = big; sty = 0; }
    else {
        sty = ry > 0 ? 1 : -1;
        const double plane = g.lo1 + (double)(iy + (sty > 0 ? 1 : 0)) * g.p1;
        ty = (plane - sy) / ry;
        dty = g.p1 / fabs(ry);
    }
    double t = tmin;
    int64_t count = 0;
    for (;;) {  // operator.py:152-186, x before y on ties
        const double tn = ty < tx ? ty : tx;
        const double te = tn < tmax ? tn : tmax;
        if (te > t) { emit(te, ix, iy); ++count; }
        if (tn >= tmax) break;
        t = tn;
        if (tx <= ty) {
            ix += stx;
            if (ix < 0 || ix >= g.nx) break;
            tx += dtx;
        } else {
            iy += sty;
            if (iy < 0 || iy >= g.ny) break;
            ty += dty;
        }
    }
    return count;
}

// Column geometry: (sx, sy, rx, ry) exactly as operator.py:200-204 forms them
// (no FMA contraction: the pixel position is det00 + u*ustep + v*vstep with
// vstep_xy = 0).
__device__ void column_ray(const double* srcs, const double* det00, const double* ustep, int64_t view, int64_t u,
                           double& sx, double& sy, double& rx, double& ry) {
    sx = srcs[view * 3 + 0];
    sy = srcs[view * 3 + 1];
    const double px = __dadd_rn(det00[view * 3 + 0], __dmul_rn((double)u, ustep[view * 3 + 0]));
    const double py = __dadd_rn(det00[view * 3 + 1], __dmul_rn((double)u, ustep[view * 3 + 1]));
    rx = __dsub_rn(px, sx);
    ry = __dsub_rn(py, sy);
}

// operator.py:62-86 (x and y clips only; z is per ray).
__device__ bool clip_xy(const GeomDev& g, double sx, double sy, double rx, double ry, double& tmin, double& tmax) {
    tmin = 0.0;
    tmax = 1.0;
    double t1, t2, tt;
    if (fabs(rx) < 1e-12 * g.p0) {
        if (sx < g.lo0 || sx >= g.lo0 + (double)g.nx * g.p0) return false;
    } else {
        t1 = (g.lo0 - sx) / rx;
        t2 = (g.lo0 + (double)g.nx * g.p0 - sx) / rx;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    if (fabs(ry) < 1e-12 * g.p1) {
        if (sy < g.lo1 || sy >= g.lo1 + (double)g.ny * g.p1) return false;
    } else {
        t1 = (g.lo1 - sy) / ry;
        t2 = (g.lo1 + (double)g.ny * g.p1 - sy) / ry;
        if (t1 > t2) { tt = t1; t1 = t2; t2 = tt; }
        if (t1 > tmin) tmin = t1;
        if (t2 < tmax) tmax = t2;
    }
    return tmax > tmin;
}

__global__ void k_column_headers(GeomDev g, const double* srcs, const double* det00, const double* ustep,
                                 int64_t n_cols, double flat_w, int flat_v, double lo2, double p2, int64_t nz,
                                 ColumnHeader* cols, int64_t* counts) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cols) return;
    const int64_t view = c / g.nu, u = c - view * g.nu;
    double sx, sy, rx, ry, tmin, tmax;
    column_ray(srcs, det00, ustep, view, u, sx, sy, rx, ry);
    ColumnHeader h;
    h.rxy2 = rx * rx + ry * ry;
    h.flat_slab = INT_MIN;
    h.pad = 0;
    int64_t n = 0;
    if (clip_xy(g, sx, sy, rx, ry, tmin, tmax)) {
        h.tmin = tmin;
        h.tmax = tmax;
        h.t_ref = (float)(0.5 * (tmin + tmax));
        h.tau_start = (float)(tmin - (double)h.t_ref);
        n = walk_column(g, sx, sy, rx, ry, tmin, tmax, [](double, int64_t, int64_t) {});
        if (flat_v >= 0) {
            // flat ray: z never changes; operator.py:87-89 inside test, 107 entry slab, 116-119 clamp
            const double sz = 0.0;
            if (!(sz < lo2 || sz >= lo2 + (double)nz * p2)) {
                int64_t iz = (int64_t)floor((sz + tmin * flat_w - lo2) / p2);
                if (iz < 0) iz = 0; else if (iz >= nz) iz = nz - 1;
                h.flat_slab = (int32_t)iz;
            }
        }
    } else {
        h.tmin = 0.0;
        h.tmax = 0.0;
        h.t_ref = 0.0f;
        h.tau_start = 0.0f;
    }
    cols[c] = h;
    counts[c] = n;
}

__global__ void k_column_fill(GeomDev g, const double* srcs, const double* det00, const double* ustep,
                              int64_t n_cols, const ColumnHeader* cols, const int64_t* off, float2* ent,
                              int32_t* cellkey, int32_t* colid) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cols) return;
    const ColumnHeader h = cols[c];
    if (off[c + 1] == off[c]) return;
    const int64_t view = c / g.nu, u = c - view * g.nu;
    double sx, sy, rx, ry;
    column_ray(srcs, det00, ustep, view, u, sx, sy, rx, ry);
    int64_t k = off[c];
    const double tref = (double)h.t_ref;
    walk_column(g, sx, sy, rx, ry, h.tmin, h.tmax, [&](double te, int64_t ix, int64_t iy) {
        const int64_t cell = iy * g.nx + ix;
        ent[k] = make_float2((float)(te - tref), __int_as_float((int32_t)(cell * g.zs)));
        if (cellkey) {  // full plan: the cell table is sorted out of the column table
            cellkey[k] = (int32_t)cell;
            colid[k] = (int32_t)c;
        }
        ++k;
    });
}

// Shard plans (cbct_plan_create_shard): the cell table of cell rows [r0, r1) straight from the
// column walks of ALL columns, without a full column table.  Same fp32 interval ends as
// k_column_fill + k_cell_entries (tau_a = the previous interval end of the column, or its
// tau_start), so the shard's cell entries equal the full plan's for those rows bit for bit.
// FILL = false: count the entries per column and take the straddle statistics of k_max_dtau over
// every column; FILL = true: write them at off[c] with their cell as the sort key.
template <bool FILL>
__global__ void k_cell_walk(GeomDev g, const double* srcs, const double* det00, const double* ustep, int64_t n_cols,
                            const ColumnHeader* cols, int64_t r0, int64_t r1, int64_t* counts, const int64_t* off,
                            CellEntry* tmp, int32_t* keys, unsigned int* out_bits, unsigned int* out_tmin) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cols) return;
    const ColumnHeader h = cols[c];
    int64_t n = 0;
    if (h.tmax > h.tmin) {  // clip_xy succeeded (k_column_headers)
        const int64_t view = c / g.nu, u = c - view * g.nu;
        double sx, sy, rx, ry;
        column_ray(srcs, det00, ustep, view, u, sx, sy, rx, ry);
        const double tref = (double)h.t_ref;
        float prev = h.tau_start, mx = 0.0f;
        int64_t k = FILL ? off[c] : 0;
        const int64_t any = walk_column(g, sx, sy, rx, ry, h.tmin, h.tmax, [&](double te, int64_t ix, int64_t iy) {
            const float x = (float)(te - tref);
            if (!FILL) mx = fmaxf(mx, x - prev);
            if (iy >= r0 && iy < r1) {
                if (FILL) {
                    CellEntry ce;
                    ce.vu = (int32_t)c;
                    ce.tau_a = prev;
                    ce.tau_b = x;
                    tmp[k] = ce;
                    keys[k] = (int32_t)(iy * g.nx + ix);
                    ++k;
                } else {
                    ++n;
                }
            }
            prev = x;
        });
        if (!FILL && any) {
            atomicMax(out_bits, __float_as_uint(mx));
            atomicMin(out_tmin, __float_as_uint((float)h.tmin));
        }
    }
    if (!FILL) counts[c] = n;
}

__global__ void k_flag_positive(const int64_t* counts, int64_t n, char* flags) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) flags[k] = counts[k] > 0;
}

__global__ void k_cell_gather(const int32_t* sorted_idx, int64_t n, const CellEntry* tmp, CellEntry* out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) out[k] = tmp[(int64_t)(uint32_t)sorted_idx[k]];
}

// Shard plans keep the column table of views [c0, c1) / nu only; the launch shapes still follow
// the longest column of the whole geometry (same kernels as the unsharded plan).
__global__ void k_keep_columns(int64_t* counts, int64_t n_cols, int64_t c0, int64_t c1, unsigned long long* mx) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cols) return;
    atomicMax(mx, (unsigned long long)counts[c]);
    if (c < c0 || c >= c1) counts[c] = 0;
}

__global__ void k_cell_entries(const int32_t* sorted_idx, int64_t n, const float2* ent, const int32_t* colid,
                               const int64_t* col_off, const ColumnHeader* cols, CellEntry* out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t e = (int64_t)(uint32_t)sorted_idx[k];
    const int32_t c = colid[e];
    CellEntry ce;
    ce.vu = c;
    ce.tau_b = ent[e].x;
    ce.tau_a = (e == col_off[c]) ? cols[c].tau_start : ent[e - 1].x;
    out[k] = ce;
}

__global__ void k_cell_offsets(const int32_t* sorted_keys, int64_t n, int64_t n_cells, int64_t* cell_off) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k > n_cells) return;
    // lower_bound(sorted_keys, k)
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted_keys[mid] < k) lo = mid + 1; else hi = mid;
    }
    cell_off[k] = lo;
}

// Per cell, the entry offsets (relative to the cell's first entry) where view batch b starts:
// the entries of a cell ascend in column index vu = view * nu + u (stable sort by cell).
__global__ void k_cell_batch_offsets(const int64_t* cell_off, const CellEntry* ent, int64_t n_cells, int nb,
                                     int64_t V, int64_t nu, int32_t* boff) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n_cells * (nb + 1)) return;
    const int64_t cell = k / (nb + 1);
    const int b = (int)(k - cell * (nb + 1));
    const int64_t first = cell_off[cell], n = cell_off[cell + 1] - first;
    const int64_t bound = (V * b / nb) * nu;  // first column of batch b
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)ent[first + mid].vu < bound) lo = mid + 1; else hi = mid;
    }
    boff[k] = (int32_t)lo;
}

__global__ void k_max_span(const int64_t* off, int64_t n, unsigned long long* out) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= n) return;
    atomicMax(out, (unsigned long long)(off[k + 1] - off[k]));
}

__global__ void k_max_dtau(const float2* ent, const int64_t* col_off, const ColumnHeader* cols, int64_t n_cols,
                           unsigned int* out_bits, unsigned int* out_tmin) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cols) return;
    const int64_t a = col_off[c], b = col_off[c + 1];
    if (a == b) return;
    float prev = cols[c].tau_start, mx = 0.0f;
    for (int64_t k = a; k < b; ++k) {
        mx = fmaxf(mx, ent[k].x - prev);
        prev = ent[k].x;
    }
    atomicMax(out_bits, __float_as_uint(mx));  // non-negative floats order like their bit patterns
    atomicMin(out_tmin, __float_as_uint((float)cols[c].tmin));  // tmin >= 0: bit order == value order
}

__global__ void k_row_tables(int64_t nv, double det00z, double pv, double p2, double* w, float* invw) {
    const int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= nv) return;
    // operator.py:203 with ustep_z = 0, sz = 0: rz = (det00z + u*0.0) + v*pv
    const double wv = __dadd_rn(det00z, __dmul_rn((double)v, pv));
    w[v] = wv;
    invw[v] = fabs(wv) < 1e-12 * p2 ? 1e30f : (float)(1.0 / wv);
}

__global__ void k_iota(int32_t* q, int64_t n) {
    const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k < n) q[k] = (int32_t)(uint32_t)k;
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

template <typename T>
static int dev_alloc(T** p, size_t count, size_t* total) {
    const size_t bytes = (count ? count : 1) * sizeof(T);
    cudaError_t e = cudaMalloc((void**)p, bytes);
    if (e != cudaSuccess) return cbct_fail(CBCT_E_NOMEM, "cudaMalloc failed while building the plan");
    if (total) *total += bytes;
    return 0;
}

extern "C" int cbct_plan_destroy(cbct_plan* p) {
    if (!p) return 0;
    cudaFree(p->d_cols);
    cudaFree(p->d_col_off);
    cudaFree(p->d_col_ent);
    cudaFree(p->d_cell_off);
    cudaFree(p->d_cell_boff);
    cudaFree(p->d_cell_ent);
    cudaFree(p->d_pref_cols);
    cudaFree(p->d_w);
    cudaFree(p->d_invw);
    cudaFree(p->d_srcs);
    cudaFree(p->d_det00);
    cudaFree(p->d_ustep);
    cudaFree(p->d_vstep);
    cudaFree(p->d_len64);
    cudaFree(p->d_rayz64);
    cudaFree(p->d_rayiz64);
    cudaFree(p->d_cell_t64);
    delete p;
    return 0;
}

// v0..v1: views whose column table (A) the plan keeps; r0..r1: cell rows whose cell table (A^T)
// it keeps.  The unsharded plan keeps all of both.
static int plan_create(cbct_plan** out, const cbct_geometry* g, int64_t v0, int64_t v1, int64_t r0, int64_t r1,
                       void* stream_) {
    if (!out || !g || !g->srcs || !g->det00 || !g->ustep || !g->vstep)
        return cbct_fail(CBCT_E_ARG, "cbct_plan_create: null argument");
    *out = nullptr;
    if (g->nx < 1 || g->ny < 1 || g->nz < 1 || g->nu < 1 || g->nv < 1 || g->n_views < 1)
        return cbct_fail(CBCT_E_ARG, "cbct_plan_create: counts must be >= 1");
    if (v0 < 0 || v1 > g->n_views || v0 >= v1 || r0 < 0 || r1 > g->ny || r0 >= r1)
        return cbct_fail(CBCT_E_ARG, "cbct_plan_create_shard: empty or out-of-range view / row block");
    const bool shard = v0 > 0 || v1 < g->n_views || r0 > 0 || r1 < g->ny;
    if (!(g->pitch[0] > 0 && g->pitch[1] > 0 && g->pitch[2] > 0))
        return cbct_fail(CBCT_E_ARG, "cbct_plan_create: voxel pitch must be > 0");
    const int64_t zs = (g->nz + 2 * CBCT_ZPAD + 3) / 4 * 4;  // 16-B aligned cell columns (TMA)
    if (g->nx * g->ny * zs >= (int64_t)INT32_MAX)
        return cbct_fail(CBCT_E_GEOMETRY, "volume too large for 32-bit cell offsets on one device");
    // Launch-shape limits, checked here so an unsupported size fails at construction with a
    // clear message instead of a generic launch error at the first A / A^T call:
    //  * projector: <= 4 rays per thread and <= 512 ray threads + 1 producer warp
    //    (__launch_bounds__(544), project.cu)  ->  nv <= 2048;
    //  * direct backprojector (mode 2 / normal_diagonal): <= 4 voxels per thread and
    //    <= 512 threads (__launch_bounds__(512), backproject.cu)  ->  nz <= 2048;
    //  * layout transposes put the view index in gridDim.z (layout.cu)  ->  n_views <= 65535.
    if (g->nv > 2048)
        return cbct_fail(CBCT_E_GEOMETRY, "cbct_plan_create: detector rows nv > 2048 are not supported");
    if (g->nz > 2048)
        return cbct_fail(CBCT_E_GEOMETRY, "cbct_plan_create: volume slices nz > 2048 are not supported");
    if (g->n_views > 65535)
        return cbct_fail(CBCT_E_GEOMETRY, "cbct_plan_create: more than 65535 views are not supported");
    const int64_t V = g->n_views;
    // The circular-trajectory family (geometry.py:144-164): source z = 0, u axis
    // horizontal, v axis = +z with one common pitch and one common det00 z.
    const double det00z = g->det00[2], pv = g->vstep[2];
    for (int64_t k = 0; k < V; ++k) {
        if (g->srcs[k * 3 + 2] != 0.0 || g->ustep[k * 3 + 2] != 0.0 || g->vstep[k * 3 + 0] != 0.0 ||
            g->vstep[k * 3 + 1] != 0.0 || g->vstep[k * 3 + 2] != pv || g->det00[k * 3 + 2] != det00z)
            return cbct_fail(CBCT_E_GEOMETRY,
                             "trajectory is not a circular orbit with a +z detector v axis (geometry.py:144-164)");
    }
    if (!(pv > 0)) return cbct_fail(CBCT_E_GEOMETRY, "detector v pitch must be > 0");
    cudaStream_t stream = (cudaStream_t)stream_;

    cbct_plan* p = new cbct_plan();
    p->nx = g->nx; p->ny = g->ny; p->nz = g->nz; p->zs = zs;
    for (int a = 0; a < 3; ++a) { p->lo[a] = g->lo[a]; p->pitch[a] = g->pitch[a]; }
    p->nu = g->nu; p->nv = g->nv; p->V = V;
    p->det00z = det00z; p->pv = pv;
    p->flat_v = -1;
    for (int64_t v = 0; v < g->nv; ++v) {
        const double wv = det00z + (double)v * pv;  // k_row_tables' association
        if (fabs(wv) < 1e-12 * g->pitch[2]) { p->flat_v = (int32_t)v; break; }
    }
    p->n_cols = V * g->nu;
    p->n_cells = g->nx * g->ny;
    p->own_v0 = v0; p->own_v1 = v1; p->own_r0 = r0; p->own_r1 = r1;
    p->sharded = shard;
    p->vol_elems = p->n_cells * zs;
    p->n_rays = p->n_cols * g->nv;
    size_t total = 0;
    int rc = 0;

    double *d_srcs = nullptr, *d_det00 = nullptr, *d_ustep = nullptr;
    int64_t* d_counts = nullptr;
    int32_t *d_cellkey = nullptr, *d_colid = nullptr, *d_keys_sorted = nullptr, *d_idx = nullptr,
            *d_idx_sorted = nullptr;
    void* d_tmp = nullptr;
    unsigned long long* d_max = nullptr;
    unsigned int* d_bits = nullptr;
    int64_t *d_ccount = nullptr, *d_coff = nullptr;
    CellEntry* d_ctmp = nullptr;

#define TRY(x) do { rc = (x); if (rc) goto fail; } while (0)
#define TRYC(x) do { cudaError_t _e = (x); if (_e != cudaSuccess) { rc = cbct_fail_cuda(_e, #x); goto fail; } } while (0)
    {
        const size_t tb = (size_t)V * 3 * sizeof(double);
        // the plan keeps the per-view tables (the fp64 path, f64.cu, walks rays from them)
        TRY(dev_alloc(&p->d_srcs, V * 3, nullptr));
        TRY(dev_alloc(&p->d_det00, V * 3, nullptr));
        TRY(dev_alloc(&p->d_ustep, V * 3, nullptr));
        d_srcs = p->d_srcs;
        d_det00 = p->d_det00;
        d_ustep = p->d_ustep;
        TRYC(cudaMemcpyAsync(d_srcs, g->srcs, tb, cudaMemcpyHostToDevice, stream));
        TRYC(cudaMemcpyAsync(d_det00, g->det00, tb, cudaMemcpyHostToDevice, stream));
        TRYC(cudaMemcpyAsync(d_ustep, g->ustep, tb, cudaMemcpyHostToDevice, stream));
        TRY(dev_alloc(&p->d_vstep, V * 3, nullptr));
        TRYC(cudaMemcpyAsync(p->d_vstep, g->vstep, tb, cudaMemcpyHostToDevice, stream));

        GeomDev gd{g->lo[0], g->lo[1], g->pitch[0], g->pitch[1], g->nx, g->ny, g->nu, zs};
        TRY(dev_alloc(&p->d_cols, p->n_cols, &total));
        TRY(dev_alloc(&p->d_col_off, p->n_cols + 1, &total));
        TRY(dev_alloc(&d_counts, p->n_cols + 1, nullptr));
        TRYC(cudaMemsetAsync(d_counts, 0, (p->n_cols + 1) * sizeof(int64_t), stream));
        const double flat_w = p->flat_v >= 0 ? det00z + (double)p->flat_v * pv : 0.0;
        k_column_headers<<<blocks_for(p->n_cols, 128), 128, 0, stream>>>(gd, d_srcs, d_det00, d_ustep, p->n_cols,
                                                                         flat_w, p->flat_v, g->lo[2], g->pitch[2],
                                                                         g->nz, p->d_cols, d_counts);
        TRYC(cudaGetLastError());
        // d_max: longest column list, longest cell list, (shard) longest column list of all views;
        // d_bits: straddle statistics (max interval, min t) over every column
        TRY(dev_alloc(&d_max, 3, nullptr));
        TRYC(cudaMemsetAsync(d_max, 0, 3 * sizeof(unsigned long long), stream));
        TRY(dev_alloc(&d_bits, 2, nullptr));
        {
            const unsigned int init[2] = {0u, 0x7f7fffffu};
            TRYC(cudaMemcpyAsync(d_bits, init, sizeof(init), cudaMemcpyHostToDevice, stream));
            TRYC(cudaStreamSynchronize(stream));
        }
        if (shard) {
            k_keep_columns<<<blocks_for(p->n_cols, 256), 256, 0, stream>>>(d_counts, p->n_cols, v0 * g->nu,
                                                                           v1 * g->nu, d_max + 2);
            TRYC(cudaGetLastError());
        }
        size_t tmp_bytes = 0;
        TRYC(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_counts, p->d_col_off, p->n_cols + 1, stream));
        TRYC(cudaMalloc(&d_tmp, tmp_bytes));
        TRYC(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_counts, p->d_col_off, p->n_cols + 1, stream));
        cudaFree(d_tmp); d_tmp = nullptr;
        TRYC(cudaMemcpyAsync(&p->n_intervals, p->d_col_off + p->n_cols, sizeof(int64_t), cudaMemcpyDeviceToHost,
                             stream));
        TRYC(cudaStreamSynchronize(stream));
        const int64_t n = p->n_intervals;
        if (n >= (int64_t)UINT32_MAX) { rc = cbct_fail(CBCT_E_GEOMETRY, "too many fan-beam intervals"); goto fail; }

        TRY(dev_alloc(&p->d_col_ent, n, &total));
        int end_bit = 1;
        while ((int64_t(1) << end_bit) <= p->n_cells) ++end_bit;
        if (!shard) {
            TRY(dev_alloc(&d_cellkey, n, nullptr));
            TRY(dev_alloc(&d_colid, n, nullptr));
            k_column_fill<<<blocks_for(p->n_cols, 128), 128, 0, stream>>>(gd, d_srcs, d_det00, d_ustep, p->n_cols,
                                                                          p->d_cols, p->d_col_off, p->d_col_ent,
                                                                          d_cellkey, d_colid);
            TRYC(cudaGetLastError());

            // cell-major order: stable radix sort of entry indices by cell (keeps column order per cell)
            TRY(dev_alloc(&d_idx, n, nullptr));
            TRY(dev_alloc(&d_idx_sorted, n, nullptr));
            TRY(dev_alloc(&d_keys_sorted, n, nullptr));
            k_iota<<<blocks_for(n, 256), 256, 0, stream>>>(d_idx, n);
            TRYC(cudaGetLastError());
            tmp_bytes = 0;
            TRYC(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_cellkey, d_keys_sorted, d_idx, d_idx_sorted,
                                                 (int64_t)n, 0, end_bit, stream));
            TRYC(cudaMalloc(&d_tmp, tmp_bytes));
            TRYC(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_cellkey, d_keys_sorted, d_idx, d_idx_sorted,
                                                 (int64_t)n, 0, end_bit, stream));
            cudaFree(d_tmp); d_tmp = nullptr;

            TRY(dev_alloc(&p->d_cell_ent, n, &total));
            TRY(dev_alloc(&p->d_cell_off, p->n_cells + 1, &total));
            k_cell_entries<<<blocks_for(n, 256), 256, 0, stream>>>(d_idx_sorted, n, p->d_col_ent, d_colid,
                                                                   p->d_col_off, p->d_cols, p->d_cell_ent);
            TRYC(cudaGetLastError());
            k_cell_offsets<<<blocks_for(p->n_cells + 1, 256), 256, 0, stream>>>(d_keys_sorted, n, p->n_cells,
                                                                                p->d_cell_off);
            TRYC(cudaGetLastError());
            k_max_dtau<<<blocks_for(p->n_cols, 128), 128, 0, stream>>>(p->d_col_ent, p->d_col_off, p->d_cols,
                                                                       p->n_cols, d_bits, d_bits + 1);
            TRYC(cudaGetLastError());
        } else {
            k_column_fill<<<blocks_for(p->n_cols, 128), 128, 0, stream>>>(gd, d_srcs, d_det00, d_ustep, p->n_cols,
                                                                          p->d_cols, p->d_col_off, p->d_col_ent,
                                                                          nullptr, nullptr);
            TRYC(cudaGetLastError());
            // cell rows [r0, r1): count per column (and the straddle statistics of all columns),
            // scan, fill in column order, stable sort by cell -- the full plan's cell order
            TRY(dev_alloc(&d_ccount, p->n_cols + 1, nullptr));
            TRY(dev_alloc(&d_coff, p->n_cols + 1, nullptr));
            TRYC(cudaMemsetAsync(d_ccount, 0, (p->n_cols + 1) * sizeof(int64_t), stream));
            k_cell_walk<false><<<blocks_for(p->n_cols, 128), 128, 0, stream>>>(
                gd, d_srcs, d_det00, d_ustep, p->n_cols, p->d_cols, r0, r1, d_ccount, nullptr, nullptr, nullptr, d_bits,
                d_bits + 1);
            TRYC(cudaGetLastError());
            tmp_bytes = 0;
            TRYC(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_ccount, d_coff, p->n_cols + 1, stream));
            TRYC(cudaMalloc(&d_tmp, tmp_bytes));
            TRYC(cub::DeviceScan::ExclusiveSum(d_tmp, tmp_bytes, d_ccount, d_coff, p->n_cols + 1, stream));
            cudaFree(d_tmp); d_tmp = nullptr;
            {
                // the columns with entries in rows [r0, r1): the only prefix rows this plan's A^T reads
                TRY(dev_alloc(&p->d_pref_cols, p->n_cols, &total));
                char* d_flags = nullptr;
                int64_t* d_nsel = nullptr;
                TRYC(cudaMalloc(&d_flags, p->n_cols));
                TRYC(cudaMalloc(&d_nsel, sizeof(int64_t)));
                k_flag_positive<<<blocks_for(p->n_cols, 256), 256, 0, stream>>>(d_ccount, p->n_cols, d_flags);
                cub::CountingInputIterator<int32_t> ids(0);
                tmp_bytes = 0;
                cudaError_t e1 = cub::DeviceSelect::Flagged(nullptr, tmp_bytes, ids, d_flags, p->d_pref_cols, d_nsel,
                                                            p->n_cols, stream);
                if (e1 == cudaSuccess) e1 = cudaMalloc(&d_tmp, tmp_bytes);
                if (e1 == cudaSuccess)
                    e1 = cub::DeviceSelect::Flagged(d_tmp, tmp_bytes, ids, d_flags, p->d_pref_cols, d_nsel, p->n_cols,
                                                    stream);
                if (e1 == cudaSuccess)
                    e1 = cudaMemcpyAsync(&p->n_pref_cols, d_nsel, sizeof(int64_t), cudaMemcpyDeviceToHost, stream);
                if (e1 == cudaSuccess) e1 = cudaStreamSynchronize(stream);
                cudaFree(d_flags);
                cudaFree(d_nsel);
                cudaFree(d_tmp); d_tmp = nullptr;
                if (e1 != cudaSuccess) { rc = cbct_fail_cuda(e1, "shard plan column list"); goto fail; }
            }
            int64_t nr = 0;
            TRYC(cudaMemcpyAsync(&nr, d_coff + p->n_cols, sizeof(int64_t), cudaMemcpyDeviceToHost, stream));
            TRYC(cudaStreamSynchronize(stream));
            if (nr >= (int64_t)UINT32_MAX) { rc = cbct_fail(CBCT_E_GEOMETRY, "too many fan-beam intervals"); goto fail; }
            TRY(dev_alloc(&d_ctmp, nr, nullptr));
            TRY(dev_alloc(&d_cellkey, nr, nullptr));
            k_cell_walk<true><<<blocks_for(p->n_cols, 128), 128, 0, stream>>>(
                gd, d_srcs, d_det00, d_ustep, p->n_cols, p->d_cols, r0, r1, nullptr, d_coff, d_ctmp, d_cellkey, nullptr,
                nullptr);
            TRYC(cudaGetLastError());
            TRY(dev_alloc(&d_idx, nr, nullptr));
            TRY(dev_alloc(&d_idx_sorted, nr, nullptr));
            TRY(dev_alloc(&d_keys_sorted, nr, nullptr));
            k_iota<<<blocks_for(nr, 256), 256, 0, stream>>>(d_idx, nr);
            TRYC(cudaGetLastError());
            tmp_bytes = 0;
            TRYC(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_cellkey, d_keys_sorted, d_idx, d_idx_sorted,
                                                 nr, 0, end_bit, stream));
            TRYC(cudaMalloc(&d_tmp, tmp_bytes));
            TRYC(cub::DeviceRadixSort::SortPairs(d_tmp, tmp_bytes, d_cellkey, d_keys_sorted, d_idx, d_idx_sorted,
                                                 nr, 0, end_bit, stream));
            cudaFree(d_tmp); d_tmp = nullptr;
            TRY(dev_alloc(&p->d_cell_ent, nr, &total));
            TRY(dev_alloc(&p->d_cell_off, p->n_cells + 1, &total));
            k_cell_gather<<<blocks_for(nr, 256), 256, 0, stream>>>(d_idx_sorted, nr, d_ctmp, p->d_cell_ent);
            TRYC(cudaGetLastError());
            k_cell_offsets<<<blocks_for(p->n_cells + 1, 256), 256, 0, stream>>>(d_keys_sorted, nr, p->n_cells,
                                                                                p->d_cell_off);
            TRYC(cudaGetLastError());
        }
        // A^T in view batches once the ray-prefix table outgrows half of L2: 2 up to 4 GiB, then one
        // per 2 GiB up to 4 (measured: config 2 14.75 -> 14.46 ms with 2, 3-8 batches slower; config
        // 3 131.9 -> 127.6 ms with 2, 128.9 with 4; config 5 (9 GB) G=6 1965 ms -> 1679 with 4-6, 1684
        // with 8, 1703 with 12)
        {
            const double tb = (double)p->n_cols * (double)(p->nv + 2) * 8.0;
            p->bp_vbatch = tb <= 64.0 * 1024 * 1024 ? 1 : (int)std::min(4.0, std::max(2.0, std::floor(tb / 2147483648.0)));
            p->bp_vbatch = (int)std::min<int64_t>(p->bp_vbatch, p->V);
        }
        if (const char* e = getenv("CBCT_BP_VBATCH")) p->bp_vbatch = std::max(1, std::min(atoi(e), (int)p->V));
        if (p->bp_vbatch > 1) {
            const int64_t nbo = p->n_cells * (p->bp_vbatch + 1);
            TRY(dev_alloc(&p->d_cell_boff, nbo, &total));
            k_cell_batch_offsets<<<blocks_for(nbo, 256), 256, 0, stream>>>(p->d_cell_off, p->d_cell_ent, p->n_cells,
                                                                           p->bp_vbatch, p->V, p->nu, p->d_cell_boff);
            TRYC(cudaGetLastError());
        }

        k_max_span<<<blocks_for(p->n_cols, 256), 256, 0, stream>>>(p->d_col_off, p->n_cols, d_max);
        k_max_span<<<blocks_for(p->n_cells, 256), 256, 0, stream>>>(p->d_cell_off, p->n_cells, d_max + 1);
        unsigned long long mx[3];
        TRYC(cudaMemcpyAsync(mx, d_max, sizeof(mx), cudaMemcpyDeviceToHost, stream));

        {
            // straddle bound for the boundary-form backprojector (backproject.cu)
            unsigned int hb[2];
            TRYC(cudaMemcpyAsync(hb, d_bits, sizeof(hb), cudaMemcpyDeviceToHost, stream));
            TRYC(cudaStreamSynchronize(stream));
            float mx, tmin_f;
            memcpy(&mx, &hb[0], 4);
            memcpy(&tmin_f, &hb[1], 4);
            p->max_dtau = mx;
            const double wmax = fmax(fabs(det00z), fabs(det00z + (double)(g->nv - 1) * pv));
            // two rays can straddle one boundary only if |w| dt > pv t_a somewhere
            p->bp_boundary_ok = wmax * (double)mx < 0.9 * pv * (double)tmin_f;
            // row range of W = z / (t pv) + c0 over the volume's boundaries (|z| <= zmax, t >= tmin):
            // the prefix table is padded to cover it so the backprojector never clamps a row index
            const double zmax = fmax(fabs(g->lo[2]), fabs(g->lo[2] + (double)g->nz * g->pitch[2]));
            const double rr = tmin_f > 0.0f ? ceil(zmax / ((double)tmin_f * pv)) + 2.0 : 1e9;
            const double c0i = floor(-det00z / pv + 0.5);
            const double lo_need = rr + 2.0 - c0i, hi_need = c0i + rr + 3.0 - (double)g->nv;
            if (rr > 1e6 || lo_need > 1e6 || hi_need > 1e6) p->bp_boundary_ok = false;
            p->bp_pad_lo = p->bp_boundary_ok ? (int32_t)fmax(0.0, lo_need) + 1 : 0;
            p->bp_pad_hi = p->bp_boundary_ok ? (int32_t)fmax(0.0, hi_need) + 1 : 0;
            // first-order closed form error <= eps^2 / 4 (backproject.cu)
            p->bp_closed_ok = tmin_f > 0.0f && (double)mx <= 3e-3 * (double)tmin_f;
            // diag(A^T A) in boundary form (k_bp_sided MODE2): no ray's z extent inside one crossing
            // (|w| dt) may reach a voxel height, so a voxel never has the same straddler at both ends
            p->bps_mode2_ok = p->bp_boundary_ok && wmax * (double)mx < 0.9 * g->pitch[2];
        }
        TRY(dev_alloc(&p->d_w, g->nv, &total));
        TRY(dev_alloc(&p->d_invw, g->nv, &total));
        k_row_tables<<<blocks_for(g->nv, 128), 128, 0, stream>>>(g->nv, det00z, pv, g->pitch[2], p->d_w, p->d_invw);
        TRYC(cudaGetLastError());
        TRYC(cudaStreamSynchronize(stream));
        // a shard plan sizes the projector for the longest column of ALL views (the same launch
        // shapes, hence the same results, as the unsharded plan)
        p->max_intervals = (int64_t)(shard ? mx[2] : mx[0]);
        p->max_cell_entries = (int64_t)mx[1];
    }
    cbct_count_launch(9);
    // launch shapes (DESIGN.md 4.1 / 4.2)
    // two rays per thread: more loads in flight, per-interval overhead shared (measured 10% faster at config 2)
    p->proj_rpt = g->nv <= 64 ? 1 : (g->nv <= 1024 ? 2 : 4);
    if (const char* e = getenv("CBCT_PROJ_RPT")) p->proj_rpt = atoi(e);
    // the projector kernels run <= 512 ray threads + one producer warp (__launch_bounds__(544))
    while (p->proj_rpt < 4 && ((g->nv + p->proj_rpt - 1) / p->proj_rpt + 31) / 32 * 32 > 512) p->proj_rpt *= 2;
    p->proj_threads = (int)(((g->nv + p->proj_rpt - 1) / p->proj_rpt + 31) / 32 * 32);
    p->proj_blocks = (int32_t)p->n_cols;
    {
        // ring of ~32 KB of cell columns, stages of K intervals (project.cu k_project_tma)
        const int64_t col_bytes = zs * 4;
        const int64_t ring_cols = std::max<int64_t>(8, 49152 / col_bytes);
        p->proj_tma_k = ring_cols >= 32 ? 8 : (ring_cols >= 16 ? 4 : 2);
        p->proj_tma_stages = (int)std::min<int64_t>(16, std::max<int64_t>(3, ring_cols / p->proj_tma_k));
        if (const char* e = getenv("CBCT_PROJ_TMA_K")) p->proj_tma_k = atoi(e);
        if (const char* e = getenv("CBCT_PROJ_TMA_STAGES")) p->proj_tma_stages = atoi(e);
        const int64_t smem = 16 * ((2 * p->proj_tma_stages * 8 + 15) / 16) + (p->max_intervals + 4) * 8 +
                             (int64_t)p->proj_tma_stages * p->proj_tma_k * col_bytes;
        p->proj_tma = smem <= 200 * 1024 ? 1 : 0;
        // prefix-sum projector: 2 ring stages + Qc of C cells, ~<= 64 KB
        const int64_t per_c = 2 * col_bytes;  // two ring slots; the prefix is built in place
        // chunk of 16 cells; per-slot zero row (Qc[0]) only if the CTA still fits ~76 KB, i.e.
        // 3 CTAs per SM (measured: config 2 16+zr 10.3 ms, 16 11.1 ms, 8 14.6 ms; config 3
        // 16 85 ms, 16+zr 103 ms, 12+zr 92 ms)
        auto qsm = [&](int cc, int zr) {
            return 48 + (p->max_intervals + 3) * 8 + per_c * (cc + zr) + 3 * (2 * cc + 33) * 4;
        };
        // C = 16 unless two CTAs of it no longer fit an SM's shared memory (zs >~ 800 slabs, i.e.
        // config 5's 1024 slabs: C=16 1514 ms with one CTA per SM, C=8 1279 ms with two; config
        // 3, two CTAs either way: C=16 79.4 ms, C=8 94.5)
        int cq = qsm(16, 0) <= 113 * 1024 ? 16 : 8;
        if (const char* e = getenv("CBCT_PROJ_Q_C")) cq = atoi(e);
        p->proj_q_c = cq;
        p->proj_q_zr = qsm(cq, 1) <= 76 * 1024 ? 1 : 0;
        if (const char* e = getenv("CBCT_PROJ_Q_ZR")) p->proj_q_zr = atoi(e) ? 1 : 0;
        const int64_t qsmem = qsm(cq, p->proj_q_zr);
        // the slab-parallel prefix pays off unless z slabs far outnumber rays (measured: config 1
        // 0.11 vs 0.22 ms, config 2 11.0 vs 15.0 ms, config 3 86 vs 115 ms against the TMA walk)
        p->proj_q = (qsmem <= 220 * 1024 && (double)g->nv >= 0.5 * (double)zs) ? 1 : 0;
        if (const char* e = getenv("CBCT_PROJ_Q")) p->proj_q = atoi(e);
    }
    p->bp_zpt = g->nz <= 512 ? 1 : (g->nz <= 1024 ? 2 : 4);
    p->bp_threads = (int)(((g->nz + p->bp_zpt - 1) / p->bp_zpt + 31) / 32 * 32);
    p->bp_blocks = (int32_t)(((g->nx + 15) / 16) * ((g->ny + 15) / 16) * 256);  // tiled grid (backproject.cu)
    {
        // 31 voxels per boundary group (32 boundaries = one warp's lanes); a warp runs G
        // groups so the per-crossing shared loads are amortised (backproject.cu).  Pick G
        // covering the groups with the least waste, at most 32 warps, ties to the larger G.
        // G = 5 is skipped: at the 64-register cap its closed-form instance spills (config 5:
        // G=5 2169 ms, G=4 1984, G=6 1965 with one view batch).
        const int64_t groups = (g->nz + 30) / 31;
        int best_g = 1;
        int64_t best_waste = INT64_MAX;
        for (int G : {3, 4, 6}) {
            const int64_t warps = (groups + G - 1) / G;
            if (warps > 32) continue;
            const int64_t waste = warps * G - groups;
            if (waste <= best_waste) { best_waste = waste; best_g = G; }
        }
        if (best_waste == INT64_MAX) best_g = 6;
        if (groups == 1) best_g = 1;
        if (const char* e = getenv("CBCT_BP_G")) best_g = atoi(e);
        p->bpg_groups = best_g;
        p->bpg_threads = (int)(((groups + best_g - 1) / best_g) * 32);
    }
    {
        // sided groups (backproject.cu k_bp_sided): below groups end at k0, above groups start there
        int64_t k0 = g->nz + 1;
        for (int64_t k = 0; k <= g->nz; ++k)
            if (g->lo[2] + (double)k * g->pitch[2] >= 0.0) { k0 = k; break; }
        const bool both = k0 > 0 && k0 <= g->nz;
        const bool zero = both && g->lo[2] + (double)k0 * g->pitch[2] == 0.0;
        const int64_t nb = (std::min<int64_t>(k0, g->nz) + 30) / 31;
        const int64_t na = (std::max<int64_t>(g->nz - k0, 0) + 30) / 31;
        // GS = 3 (four crossings per shuffle, backproject.cu) when at most 10% of its group slots are
        // wasted, else GS = 2 under the same rule, else k_bp_boundary.  Measured A^T: config 3 GS=3
        // 94.9 ms vs 128 for k_bp_boundary; config 5 GS=3 1231 ms vs GS=2 1414-1422 and 1684 for
        // k_bp_boundary; config 2 (5 + 5 groups, 2 of 12 slots wasted) GS=3 14.6 vs 14.0 ms, so it
        // keeps k_bp_boundary.
        int best = 0;
        int64_t best_waste = 0, best_slots = 1;
        for (int gs : {3, 2}) {
            const int64_t warps = (std::max(nb, na) + gs - 1) / gs;
            if (warps > 32) continue;
            const int64_t waste = warps * gs * 2 - nb - na;
            if (best == 0 || (10 * waste <= warps * gs * 2 && 10 * best_waste > best_slots)) {
                best = gs;
                best_waste = waste;
                best_slots = warps * gs * 2;
            }
        }
        bool use = best > 0 && 10 * best_waste <= best_slots;
        if (const char* e = getenv("CBCT_BP_GS")) { best = atoi(e); use = best > 0; }
        p->bps_eligible = (!both || zero) && best > 0;
        p->bps_ok = p->bps_eligible && use && getenv("CBCT_BP_SIDED_OFF") == nullptr;
        p->bps_gs = best;
        p->bps_threads = best > 0 ? (int)((std::max(nb, na) + best - 1) / best * 32) : 0;
        p->bps_k0 = (int)k0;
        p->bps_zero = zero ? 1 : 0;
    }
    p->table_bytes = total;
    cudaFree(d_counts); cudaFree(d_cellkey);  // d_srcs/d_det00/d_ustep belong to the plan
    cudaFree(d_colid); cudaFree(d_keys_sorted); cudaFree(d_idx); cudaFree(d_idx_sorted); cudaFree(d_max);
    cudaFree(d_bits); cudaFree(d_ccount); cudaFree(d_coff); cudaFree(d_ctmp);
    *out = p;
    return 0;
fail:
    cudaFree(d_counts); cudaFree(d_cellkey);  // d_srcs/d_det00/d_ustep belong to the plan
    cudaFree(d_colid); cudaFree(d_keys_sorted); cudaFree(d_idx); cudaFree(d_idx_sorted); cudaFree(d_max);
    cudaFree(d_bits); cudaFree(d_ccount); cudaFree(d_coff); cudaFree(d_ctmp);
    cudaFree(d_tmp);
    cbct_plan_destroy(p);
    return rc;
#undef TRY
#undef TRYC
}

extern "C" int cbct_plan_create(cbct_plan** out, const cbct_geometry* g, void* stream) {
    CbctRange range("cbct_plan_create");
    if (!g) return cbct_fail(CBCT_E_ARG, "cbct_plan_create: null argument");
    return plan_create(out, g, 0, g->n_views, 0, g->ny, stream);
}

extern "C" int cbct_plan_create_shard(cbct_plan** out, const cbct_geometry* g, int64_t view0, int64_t view1,
                                      int64_t row0, int64_t row1, void* stream) {
    CbctRange range("cbct_plan_create_shard");
    if (!g) return cbct_fail(CBCT_E_ARG, "cbct_plan_create_shard: null argument");
    return plan_create(out, g, view0, view1, row0, row1, stream);
}

extern "C" int cbct_plan_get_info(const cbct_plan* p, cbct_plan_info* info) {
    if (!p || !info) return cbct_fail(CBCT_E_ARG, "cbct_plan_get_info: null argument");
    info->n_voxels = p->nx * p->ny * p->nz;
    info->n_rays = p->n_rays;
    info->vol_elems = p->vol_elems;
    info->zstride = p->zs;
    info->n_columns = p->n_cols;
    info->n_intervals = p->n_intervals;
    info->max_intervals = p->max_intervals;
    info->max_cell_entries = p->max_cell_entries;
    info->table_bytes = (int64_t)p->table_bytes;
    info->proj_blocks = p->proj_blocks;
    info->bp_scratch_floats =
        std::max<int64_t>(p->n_cols * 2 * (p->nv + 2 + p->bp_pad_lo + p->bp_pad_hi) + p->n_cols, p->n_rays);
    info->bp_fast_path = p->bp_boundary_ok ? 1 : 0;
    info->bp_closed_form = (p->bp_boundary_ok && p->bp_closed_ok && !getenv("CBCT_BP_TABLE")) ? 1 : 0;
    info->bp_blocks = p->bp_blocks;
    info->proj_chunk = p->proj_q ? p->proj_q_c : 0;
    info->bp_groups = p->bpg_groups;
    info->bp_view_batches = p->bp_vbatch;
    const bool closed = p->bp_boundary_ok && p->bp_closed_ok && !getenv("CBCT_BP_TABLE");
    info->bp_sided_gs = (closed && p->bps_ok) ? p->bps_gs : 0;
    return 0;
}
