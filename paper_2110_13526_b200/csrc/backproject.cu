// backproject.cu -- adjoint x = A^T y and diag(A^T A)
// (replaces _backproject_kernel modes 1 and 2, operator.py:209-233, 353-362).
//
// Voxel-driven gather: one CTA per cell (ix, iy), one thread per voxel of the
// cell's z column (ZPT voxels per thread when nz > 512).  The CTA walks the
// cell's list of crossing columns (view, u) with their ray-parameter interval
// [tau_a, tau_b] (plan.cu, the same intervals the projector uses).  For each
// crossing a thread finds the detector rows v whose ray passes through its
// voxel's z slab inside that interval and adds
//
//     |r| * |[tau_a, tau_b] ∩ [z0/rz_v, z1/rz_v]| * y[view, u, v]
//
// i.e. exactly the reference's segment weight seg = dt * raylen (operator.py:
// 159, 165-167).  Every output element is owned by one thread and summed in a
// fixed order, so results are bitwise reproducible without atomics.
// |r| is folded into y by a prepass (k_weight_rays) so the inner loop is pure
// fp32 min/max/fma.
#include <climits>
#include <cmath>
#include <cstdlib>

#include "cbct_internal.cuh"
#include "reduce.cuh"

namespace {

struct Tri {  // staged per-crossing data
    float ta, tb, tref, ia, ib;
    int vu, flat_slab, pad;
};

constexpr int kChunk = 256;

// yw[c, v] = |r(c, v)| * y[c, v]  (y == NULL -> |r|)   operator.py:102
__global__ void k_weight_rays(const ColumnHeader* __restrict__ cols, const double* __restrict__ wtab,
                              const float* __restrict__ y, float* __restrict__ yw, int64_t n_cols, int nv) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_cols * nv) return;
    const int64_t c = i / nv;
    const int v = (int)(i - c * nv);
    const double w = wtab[v];
    const float len = (float)sqrt(cols[c].rxy2 + w * w);
    yw[i] = y ? len * y[i] : len;
}

template <int ZPT, bool PRECISE>
__global__ void __launch_bounds__(512) k_backproject(const int64_t* __restrict__ cell_off,
                                                     const CellEntry* __restrict__ cell_ent,
                                                     const ColumnHeader* __restrict__ cols,
                                                     const float* __restrict__ invw, const double* __restrict__ wtab,
                                                     const float* __restrict__ yw,
                                                     float* __restrict__ vol, const float* __restrict__ col_scale,
                                                     double* __restrict__ partials, int nv, int nz, int zs,
                                                     double lo2, double p2, double det00z, double pv, int flat_v,
                                                     int mode) {
    extern __shared__ float s_invw[];
    __shared__ Tri s_tri[kChunk];
    const int64_t cell = blockIdx.x;
    const int64_t off = cell_off[cell];
    const int ne = (int)(cell_off[cell + 1] - off);
    for (int k = threadIdx.x; k < nv; k += blockDim.x) s_invw[k] = invw[k];

    float z0[ZPT], z1[ZPT], acc[ZPT];
    int iz[ZPT];
#pragma unroll
    for (int r = 0; r < ZPT; ++r) {
        iz[r] = threadIdx.x + r * blockDim.x;
        z0[r] = (float)(lo2 + (double)iz[r] * p2);
        z1[r] = (float)(lo2 + (double)(iz[r] + 1) * p2);
        acc[r] = 0.0f;
    }
    const float c0 = (float)(-det00z / pv);
    const float fpv = (float)pv;

    for (int base = 0; base < ne; base += kChunk) {
        const int nch = min(kChunk, ne - base);
        __syncthreads();
        for (int k = threadIdx.x; k < nch; k += blockDim.x) {
            const CellEntry ce = cell_ent[off + base + k];
            const ColumnHeader& h = cols[ce.vu];
            Tri t;
            t.ta = ce.tau_a;
            t.tb = ce.tau_b;
            t.tref = h.t_ref;
            t.ia = 1.0f / ((ce.tau_a + h.t_ref) * fpv);
            t.ib = 1.0f / ((ce.tau_b + h.t_ref) * fpv);
            t.vu = ce.vu;
            t.flat_slab = h.flat_slab;
            t.pad = 0;
            s_tri[k] = t;
        }
        __syncthreads();
        for (int k = 0; k < nch; ++k) {
            const Tri t = s_tri[k];
            const float* __restrict__ ycol = yw + (int64_t)t.vu * nv;
#pragma unroll
            for (int r = 0; r < ZPT; ++r) {
                if (iz[r] >= nz) continue;
                const float vlo = fminf(fmaf(z0[r], t.ia, c0), fmaf(z0[r], t.ib, c0));
                const float vhi = fmaxf(fmaf(z1[r], t.ia, c0), fmaf(z1[r], t.ib, c0));
                const int va = max(0, (int)ceilf(vlo - 1e-3f));
                const int vb = min(nv - 1, (int)floorf(vhi + 1e-3f));
                for (int v = va; v <= vb; ++v) {
                    float d;
                    if (v == flat_v) {
                        d = (iz[r] == t.flat_slab) ? t.tb - t.ta : 0.0f;
                    } else if (PRECISE) {  // fp64 z clip (diagnostic / reference-precision path)
                        const double w = wtab[v];
                        const double u1 = (lo2 + (double)iz[r] * p2) / w - (double)t.tref;
                        const double u2 = (lo2 + (double)(iz[r] + 1) * p2) / w - (double)t.tref;
                        d = (float)(fmin((double)t.tb, fmax(u1, u2)) - fmax((double)t.ta, fmin(u1, u2)));
                    } else {
                        const float iw = s_invw[v];
                        const float u1 = fmaf(z0[r], iw, -t.tref);
                        const float u2 = fmaf(z1[r], iw, -t.tref);
                        d = fminf(t.tb, fmaxf(u1, u2)) - fmaxf(t.ta, fminf(u1, u2));
                    }
                    if (d > 0.0f) {
                        const float q = d * __ldg(ycol + v);
                        acc[r] = mode == 1 ? acc[r] + q : fmaf(q, q, acc[r]);
                    }
                }
            }
        }
    }

    float* out = vol + cell * zs;
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < ZPT; ++r) {
        if (iz[r] < nz) {
            float val = acc[r];
            if (col_scale) val *= col_scale[cell * zs + CBCT_ZPAD + iz[r]];
            out[CBCT_ZPAD + iz[r]] = val;
            sq += (double)val * (double)val;
        }
    }
    for (int k = threadIdx.x; k < CBCT_ZPAD; k += blockDim.x) {
        out[k] = 0.0f;
        out[CBCT_ZPAD + nz + k] = 0.0f;
    }
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}

}  // namespace

extern "C" int cbct_backproject(const cbct_plan* p, const float* proj, float* vol, int mode, float* scratch,
                                const float* col_scale, double* partials, void* stream) {
    if (!p || !vol || !scratch) return cbct_fail(CBCT_E_ARG, "cbct_backproject: null argument");
    if (mode != 1 && mode != 2) return cbct_fail(CBCT_E_ARG, "cbct_backproject: mode must be 1 or 2");
    if (mode == 1 && !proj) return cbct_fail(CBCT_E_ARG, "cbct_backproject: mode 1 needs projections");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t nr = p->n_rays;
    k_weight_rays<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(p->d_cols, p->d_w, mode == 1 ? proj : nullptr,
                                                                 scratch, p->n_cols, (int)p->nv);
    CBCT_CHECK(cudaGetLastError());
    const size_t smem = (size_t)p->nv * sizeof(float);
    const dim3 grid((unsigned)p->n_cells);
#define LAUNCH(Z, PR)                                                                                         \
    do {                                                                                                      \
        if (smem > 40 * 1024)                                                                                 \
            CBCT_CHECK(cudaFuncSetAttribute(k_backproject<Z, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                            (int)smem));                                                      \
        k_backproject<Z, PR><<<grid, p->bp_threads, smem, s>>>(p->d_cell_off, p->d_cell_ent, p->d_cols,       \
                                                               p->d_invw, p->d_w, scratch, vol, col_scale,    \
                                                               partials, (int)p->nv, (int)p->nz, (int)p->zs,  \
                                                               p->lo[2], p->pitch[2], p->det00z, p->pv,       \
                                                               p->flat_v, mode);                              \
    } while (0)
    const bool precise = getenv("CBCT_BP_PRECISE") != nullptr;
    switch (p->bp_zpt * 2 + (precise ? 1 : 0)) {
        case 2: LAUNCH(1, false); break;
        case 3: LAUNCH(1, true); break;
        case 4: LAUNCH(2, false); break;
        case 5: LAUNCH(2, true); break;
        case 8: LAUNCH(4, false); break;
        default: LAUNCH(4, true); break;
    }
#undef LAUNCH
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch(2);
    return 0;
}
