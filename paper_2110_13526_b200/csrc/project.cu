// project.cu -- forward projector p = A x (replaces _project_kernel, operator.py:190-206).
//
// One CTA per detector column (view, u); one thread per detector row v (RPT rows
// per thread when nv > 512).  All rays of a column share the column's xy cell
// sequence (plan.cu), which is staged once in shared memory and read as a
// warp-uniform broadcast.  Each thread walks that sequence for its ray and
// tracks the ray's z slab incrementally:
//
//   acc += (tau_end - tau_prev) * vol[cell, iz]                   every interval
//   acc += (tau_end - tau_z) * (vol[cell, iz+dz] - vol[cell, iz])  at a z crossing
//
// which is the reference's segment sum  sum_k seg_k * vol[lin_k]  (operator.py:
// 152-167) regrouped per xy interval.  Rays leaving the volume through its top or
// bottom walk into the zero guard slices, so no per-ray clipping is needed in the
// loop.  Lanes of a warp are consecutive rows v, so vol[cell, iz] loads are
// coalesced along z (the internal volume layout is z-fastest).
#include <cmath>

#include "cbct_internal.cuh"
#include "reduce.cuh"

namespace {

struct RayState {
    float acc;
    float tz;    // tau of the next z-plane crossing (INF when none left)
    float tz0;   // tau of the first crossing
    float dtz;   // tau spacing of z planes
    float jf;    // crossings taken so far
    float kf;    // crossings available
    int iz;      // current slab + CBCT_ZPAD (guard-padded index)
    int dz;      // +1 / -1
};

__device__ __forceinline__ void ray_setup(RayState& s, const ColumnHeader& h, int v, int nv, const double* wtab,
                                          double lo2, double p2, int nz, int flat_v) {
    s.acc = 0.0f;
    s.tz = INFINITY;
    s.tz0 = 0.0f;
    s.dtz = 0.0f;
    s.jf = 0.0f;
    s.kf = 0.0f;
    s.dz = 1;
    s.iz = CBCT_ZPAD - 1;  // guard (reads 0)
    if (v >= nv) return;
    if (v == flat_v) {  // |rz| < 1e-12 p2: z stays at the source height (operator.py:87-89)
        if (h.flat_slab != INT_MIN) s.iz = h.flat_slab + CBCT_ZPAD;
        return;
    }
    const double w = wtab[v];
    const double zs0 = 0.0 + h.tmin * w;  // z at the column entry (operator.py:107)
    const double ze = 0.0 + h.tmax * w;
    int s0 = (int)floor((zs0 - lo2) / p2);
    int s1 = (int)floor((ze - lo2) / p2);
    s0 = s0 < -1 ? -1 : (s0 > nz ? nz : s0);
    s1 = s1 < -1 ? -1 : (s1 > nz ? nz : s1);
    const int stz = w > 0 ? 1 : -1;
    const int kp = s0 + (stz > 0 ? 1 : 0);                 // first plane crossed (operator.py:146)
    const double t0 = (lo2 + (double)kp * p2 - 0.0) / w;  // operator.py:147
    s.iz = s0 + CBCT_ZPAD;
    s.dz = stz;
    s.kf = (float)abs(s1 - s0);
    s.tz0 = (float)(t0 - (double)h.t_ref);
    s.dtz = (float)(p2 / fabs(w));  // operator.py:148
    s.tz = s.kf > 0.0f ? s.tz0 : INFINITY;
}

template <int RPT>
__global__ void __launch_bounds__(512) k_project(const ColumnHeader* __restrict__ cols,
                                                 const int64_t* __restrict__ col_off,
                                                 const float2* __restrict__ col_ent, const double* __restrict__ wtab,
                                                 const float* __restrict__ vol, float* __restrict__ proj,
                                                 double* __restrict__ partials, int nv, int nz, double lo2,
                                                 double p2, int flat_v) {
    extern __shared__ float2 s_ent[];
    const int64_t c = blockIdx.x;
    const ColumnHeader h = cols[c];
    const int64_t off = col_off[c];
    const int M = (int)(col_off[c + 1] - off);
    for (int k = threadIdx.x; k < M; k += blockDim.x) s_ent[k] = col_ent[off + k];

    RayState st[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) ray_setup(st[r], h, threadIdx.x + r * blockDim.x, nv, wtab, lo2, p2, nz, flat_v);
    __syncthreads();

    float a = h.tau_start;
    for (int m = 0; m < M; ++m) {
        const float2 e = s_ent[m];
        const float bn = e.x;
        const float* __restrict__ colp = vol + __float_as_int(e.y);
        const float dl = bn - a;
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            RayState& s = st[r];
            float val = __ldg(colp + s.iz);
            s.acc = fmaf(dl, val, s.acc);
            while (s.tz < bn) {  // z-plane crossing inside this interval
                const float v2 = __ldg(colp + s.iz + s.dz);
                s.acc = fmaf(bn - s.tz, v2 - val, s.acc);
                val = v2;
                s.iz += s.dz;
                s.jf += 1.0f;
                s.tz = s.jf < s.kf ? fmaf(s.jf, s.dtz, s.tz0) : INFINITY;
            }
        }
        a = bn;
    }

    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int v = threadIdx.x + r * blockDim.x;
        if (v < nv) {
            const double w = wtab[v];
            const float raylen = (float)sqrt(h.rxy2 + w * w);  // operator.py:102
            const float out = st[r].acc * raylen;
            proj[c * nv + v] = out;
            sq += (double)out * (double)out;
        }
    }
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}

}  // namespace

extern "C" int cbct_project(const cbct_plan* p, const float* vol, float* proj, double* partials, void* stream) {
    if (!p || !vol || !proj) return cbct_fail(CBCT_E_ARG, "cbct_project: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const size_t smem = (size_t)(p->max_intervals > 0 ? p->max_intervals : 1) * sizeof(float2);
    const dim3 grid((unsigned)p->n_cols);
    const int nt = p->proj_threads;
#define LAUNCH(R)                                                                                            \
    do {                                                                                                     \
        if (smem > 48 * 1024)                                                                                \
            CBCT_CHECK(cudaFuncSetAttribute(k_project<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                            (int)smem));                                                     \
        k_project<R><<<grid, nt, smem, s>>>(p->d_cols, p->d_col_off, p->d_col_ent, p->d_w, vol, proj,        \
                                            partials, (int)p->nv, (int)p->nz, p->lo[2], p->pitch[2], p->flat_v); \
    } while (0)
    switch (p->proj_rpt) {
        case 1: LAUNCH(1); break;
        case 2: LAUNCH(2); break;
        default: LAUNCH(4); break;
    }
#undef LAUNCH
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}
