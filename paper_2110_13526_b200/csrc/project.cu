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
#include <cstdlib>

#include "cbct_internal.cuh"
#include "reduce.cuh"
#include "tma.cuh"

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

// One interval of the column walk for one ray.  `idx` is the guard-padded
// element index cell_base + iz, kept in 32 bits so the address is a single
// IMAD.WIDE.U32 off the uniform volume pointer.
__device__ __forceinline__ void interval_step(RayState& s, const float* __restrict__ vol, float bn, int cell,
                                              float dl) {
    const uint32_t idx = (uint32_t)(cell + s.iz);
    float val = __ldg(vol + idx);
    s.acc = fmaf(dl, val, s.acc);
    while (s.tz < bn) {  // z-plane crossing inside this interval (rare per lane)
        const float v2 = __ldg(vol + (uint32_t)(cell + s.iz + s.dz));
        s.acc = fmaf(bn - s.tz, v2 - val, s.acc);
        val = v2;
        s.iz += s.dz;
        s.jf += 1.0f;
        s.tz = s.jf < s.kf ? fmaf(s.jf, s.dtz, s.tz0) : INFINITY;
    }
}

template <int RPT>
__global__ void __launch_bounds__(512) k_project(const ColumnHeader* __restrict__ cols,
                                                 const int64_t* __restrict__ col_off,
                                                 const float2* __restrict__ col_ent, const double* __restrict__ wtab,
                                                 const float* __restrict__ vol, float* __restrict__ proj,
                                                 double* __restrict__ partials, int nv, int nz, double lo2,
                                                 double p2, int flat_v, int64_t c0) {
    extern __shared__ float4 s_ent4[];  // column entries, two per float4, padded to an even count
    float2* s_ent = reinterpret_cast<float2*>(s_ent4);
    const int64_t c = c0 + blockIdx.x;  // detector column (view * nu + u)
    const ColumnHeader h = cols[c];
    const int64_t off = col_off[c];
    const int M = (int)(col_off[c + 1] - off);
    for (int k = threadIdx.x; k < M; k += blockDim.x) s_ent[k] = col_ent[off + k];
    // odd count: pad with a zero-length interval (cell 0, reads a valid zero-weight element)
    if (threadIdx.x == 0 && (M & 1)) s_ent[M] = make_float2(col_ent[off + M - 1].x, __int_as_float(0));

    RayState st[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) ray_setup(st[r], h, threadIdx.x + r * blockDim.x, nv, wtab, lo2, p2, nz, flat_v);
    __syncthreads();

    float a = h.tau_start;
    const int M2 = (M + 1) >> 1;
    for (int m2 = 0; m2 < M2; ++m2) {
        const float4 e = s_ent4[m2];  // {tau_end0, cell0, tau_end1, cell1}
        const float dl0 = e.x - a;
        const float dl1 = e.z - e.x;  // 0 for the pad entry (tau_end1 == tau_end0)
        const int c0 = __float_as_int(e.y), c1 = __float_as_int(e.w);
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            interval_step(st[r], vol, e.x, c0, dl0);
            interval_step(st[r], vol, e.z, c1, dl1);
        }
        a = e.z;
    }

    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < RPT; ++r) {
        const int v = threadIdx.x + r * blockDim.x;
        if (v < nv) {
            const double w = wtab[v];
            const float raylen = (float)sqrt(h.rxy2 + w * w);  // operator.py:102
            const float out = st[r].acc * raylen;
            proj[(c - c0) * nv + v] = out;
            sq += (double)out * (double)out;
        }
    }
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}


// ---------------------------------------------------------------------------
// TMA-staged variant.  A producer warp streams the z column of every upcoming
// cell of this detector column (zs contiguous floats, 16-B aligned) into a
// shared-memory ring with cp.async.bulk; full/empty mbarriers hand stages of K
// intervals to the ray warps, which then read the volume with LDS instead of
// waiting ~L2 latency on each LDG.
__device__ __forceinline__ void interval_step_smem(RayState& s, const float* __restrict__ colp, float bn, float dl) {
    float val = colp[s.iz];
    s.acc = fmaf(dl, val, s.acc);
    while (s.tz < bn) {
        const float v2 = colp[s.iz + s.dz];
        s.acc = fmaf(bn - s.tz, v2 - val, s.acc);
        val = v2;
        s.iz += s.dz;
        s.jf += 1.0f;
        s.tz = s.jf < s.kf ? fmaf(s.jf, s.dtz, s.tz0) : INFINITY;
    }
}

template <int RPT, int K>
__global__ void __launch_bounds__(544) k_project_tma(const ColumnHeader* __restrict__ cols,
                                                     const int64_t* __restrict__ col_off,
                                                     const float2* __restrict__ col_ent,
                                                     const double* __restrict__ wtab, const float* __restrict__ vol,
                                                     float* __restrict__ proj, double* __restrict__ partials, int nv,
                                                     int nz, int zs, double lo2, double p2, int flat_v, int nstages,
                                                     int ent_cap, int64_t c0) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
    uint64_t* empty = full + nstages;
    float4* s_ent4 = reinterpret_cast<float4*>(smem_raw + 16 * ((2 * nstages * 8 + 15) / 16));
    float2* s_ent = reinterpret_cast<float2*>(s_ent4);
    float* ring = reinterpret_cast<float*>(s_ent4 + ent_cap / 2);
    const int nwc = (blockDim.x >> 5) - 1;  // consumer warps; the last warp produces
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp == nwc;

    const int64_t c = c0 + blockIdx.x;  // detector column (view * nu + u)
    const ColumnHeader h = cols[c];
    const int64_t off = col_off[c];
    const int M = (int)(col_off[c + 1] - off);
    for (int k = threadIdx.x; k < M; k += blockDim.x) s_ent[k] = col_ent[off + k];
    if (threadIdx.x == 0) {
        if (M & 1) s_ent[M] = make_float2(col_ent[off + M - 1].x, __int_as_float(0));
        for (int i = 0; i < nstages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], nwc);
        }
        mbar_fence_init();
    }
    RayState st[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r)
        ray_setup(st[r], h, producer ? nv : threadIdx.x + r * nwc * 32, nv, wtab, lo2, p2, nz, flat_v);
    __syncthreads();

    const int nst = (M + K - 1) / K;  // stages of K intervals
    const uint32_t col_bytes = (uint32_t)zs * 4u;
    if (producer) {
        // one lane arms the stage's barrier, then lanes j < cnt each issue one bulk copy
        for (int i = 0; i < nst; ++i) {
            const int slot = i % nstages, round = i / nstages;
            if (round > 0) mbar_wait(&empty[slot], (round - 1) & 1);
            const int m0 = i * K, cnt = min(K, M - m0);
            if (lane == 0) mbar_arrive_expect_tx(&full[slot], cnt * col_bytes);
            __syncwarp();
            if (lane < cnt)
                bulk_g2s(ring + ((size_t)slot * K + lane) * zs,
                         vol + (uint32_t)__float_as_int(s_ent[m0 + lane].y), col_bytes, &full[slot]);
        }
    } else {
        float a = h.tau_start;
        for (int i = 0; i < nst; ++i) {
            const int slot = i % nstages, round = i / nstages;
            mbar_wait(&full[slot], round & 1);
            const float* stage = ring + (size_t)slot * K * zs;
            const int m0 = i * K;
#pragma unroll
            for (int j = 0; j < K; j += 2) {
                if (m0 + j >= M) break;
                const float4 e = s_ent4[(m0 + j) >> 1];
                const float dl0 = e.x - a, dl1 = e.z - e.x;
                const float* c0p = stage + j * zs;
                const float* c1p = (m0 + j + 1 < M) ? c0p + zs : c0p;  // pad entry: zero-length, any column
#pragma unroll
                for (int r = 0; r < RPT; ++r) {
                    interval_step_smem(st[r], c0p, e.x, dl0);
                    interval_step_smem(st[r], c1p, e.z, dl1);
                }
                a = e.z;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);
        }
    }

    double sq = 0.0;
    if (!producer) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int v = threadIdx.x + r * nwc * 32;
            if (v < nv) {
                const double w = wtab[v];
                const float raylen = (float)sqrt(h.rxy2 + w * w);
                const float out = st[r].acc * raylen;
                proj[(c - c0) * nv + v] = out;
                sq += (double)out * (double)out;
            }
        }
    }
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}


// ---------------------------------------------------------------------------
// Column prefix-sum variant.  All rays of a detector column share the interval
// sequence, so per chunk of C cells the CTA first builds, for every z slab,
//     Qc[j][iz] = sum_{j' < j} dtau_j' * vol[cell_j', iz]          (phase 1, slab-parallel)
// and each ray then adds  Qc[C][iz]  for the slab it leaves the chunk in, plus,
// for every z-plane crossing inside the chunk, R_old(tz) - R_new(tz), where
// R_iz(tau) interpolates Qc linearly inside the interval holding tau (phase 2).
// This is the same segment sum as the interval walk, but the per-interval work is
// done once per slab instead of once per ray, and the divergent per-ray work
// only happens at z crossings.
__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Block -> detector column, in tiles of kTileV views x kTileU columns (a bijection onto the
// (view1 - view0) * nu columns of the launch).  The columns of a tile cross one ~40 mm strip of
// the volume, so the CTAs in flight re-read the same cell columns from L2 instead of streaming
// the whole volume once per view from DRAM (config 3: 537 MB volume > 126 MB L2).
constexpr int kTileV = 8, kTileU = 64;
__device__ __forceinline__ int64_t tiled_column(int b, int view0, int nviews, int nu) {
    const int band = b / (kTileV * nu);               // band of kTileV views
    const int vb = min(kTileV, nviews - band * kTileV);
    const int r = b - band * kTileV * nu;             // index inside the band: [0, vb * nu)
    const int ut = r / (vb * kTileU);                 // column tile
    const int ub = min(kTileU, nu - ut * kTileU);
    const int rem = r - ut * vb * kTileU;             // [0, vb * ub)
    const int dv = rem / ub, du = rem - dv * ub;      // adjacent columns of one view run together
    return (int64_t)(view0 + band * kTileV + dv) * nu + ut * kTileU + du;
}

// Guard-padded slab range [x, y] that some ray of a column can occupy while tau is in
// [tau_a, tau_b]: z = w t is extremal at the corners of [w_lo, w_hi] x [t_a, t_b]; one slab of
// margin on each side absorbs rounding.  Producer and consumers evaluate it identically.
__device__ __forceinline__ int2 chunk_slabs(float tau_a, float tau_b, float tref, float wlo, float whi, float lo2f,
                                            float ip2, int nz) {
    const float ta = tau_a + tref, tb = tau_b + tref;
    const float zlo = fminf(wlo * ta, wlo * tb), zhi = fmaxf(whi * ta, whi * tb);
    const int ilo = (int)floorf((zlo - lo2f) * ip2) - 1 + CBCT_ZPAD;
    const int ihi = (int)floorf((zhi - lo2f) * ip2) + 1 + CBCT_ZPAD;
    // both ends clamped into [guard below, guard above]: the window is never empty and always
    // holds the guard slab a ray outside the volume sits in (reads a prefix of zeros)
    return make_int2(min(max(ilo, CBCT_ZPAD - 1), CBCT_ZPAD + nz), min(max(ihi, CBCT_ZPAD - 1), CBCT_ZPAD + nz));
}

// ZS > 0: the slab stride zs as a compile-time constant (the BASELINE sizes and the parity
// subsets), so phase 1 runs fully unrolled over a full chunk with immediate row offsets and the
// chunk's dtau in registers; ZS = 0 keeps the runtime stride.  prod_hint > 0: the producer waits
// on a drained slot with a hardware suspend hint instead of nanosleep polling.
template <int RPT, int C, bool ZR, int ZS>
__global__ void __launch_bounds__(544) k_project_q(const ColumnHeader* __restrict__ cols,
                                                   const int64_t* __restrict__ col_off,
                                                   const float2* __restrict__ col_ent, const double* __restrict__ wtab,
                                                   const float* __restrict__ vol, float* __restrict__ proj,
                                                   double* __restrict__ partials, int nv, int nz, int zs_rt, double lo2,
                                                   double p2, int flat_v, int ent_cap, int64_t c0, int nu,
                                                   int nviews, uint32_t prod_hint) {
    const int zs = ZS > 0 ? ZS : zs_rt;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);  // [2]
    uint64_t* empty = full + 2;                               // [2]
    int2* s_win = reinterpret_cast<int2*>(smem_raw + 32);     // [2] staged slab window of each slot's chunk
    float2* s_ent = reinterpret_cast<float2*>(smem_raw + 48);
    // ZR: [2][C+1][zs], row 0 of a slot is Qc[0] = 0 (never written after init) and rows
    // 1..cnt receive the staged cell columns; !ZR: [2][C][zs] (one row less per slot, when the
    // extra rows would cost a resident CTA) and Qc[0] = 0 is a predicated load.  Phase 1 turns
    // the staged rows into Qc[1..cnt] in place.
    constexpr int RZ = ZR ? 1 : 0;
    float* ring = reinterpret_cast<float*>(s_ent + ent_cap);
    constexpr int PC = C <= 8 ? 8 : (C <= 16 ? 16 : 32);  // power-of-two search span
    // three chunk tables of {sB [PC+1]: interval starts, chunk end, then +inf padding; sInv [C]:
    // 1/dtau; sDl [C]: dtau}
    constexpr int SBW = PC + 1 + 2 * C;
    float* sTab = ring + 2 * (C + RZ) * zs;
    const int nwc = (blockDim.x >> 5) - 1;
    const int nct = nwc * 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool producer = warp == nwc;
    const int slot_elems = (C + RZ) * zs;

    const int64_t c = tiled_column((int)blockIdx.x, (int)(c0 / nu), nviews, nu);  // detector column (view * nu + u)
    const ColumnHeader h = cols[c];
    const int64_t off = col_off[c];
    const int M = (int)(col_off[c + 1] - off);
    for (int k = threadIdx.x; k < M; k += blockDim.x) s_ent[k] = col_ent[off + k];
    for (int k = threadIdx.x; ZR && k < zs; k += blockDim.x) ring[k] = ring[slot_elems + k] = 0.0f;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], nwc);
        }
        mbar_fence_init();
    }
    RayState st[RPT];
#pragma unroll
    for (int r = 0; r < RPT; ++r) ray_setup(st[r], h, producer ? nv : threadIdx.x + r * nct, nv, wtab, lo2, p2, nz, flat_v);
    const float wlo = (float)fmin(wtab[0], wtab[nv - 1]), whi = (float)fmax(wtab[0], wtab[nv - 1]);
    const float tref = h.t_ref, lo2f = (float)lo2, ip2 = (float)(1.0 / p2);
    __syncthreads();

    const int nch = (M + C - 1) / C;
    if (producer) {
        // stage only the 16-B-aligned slab window the chunk's rays can reach (the cone bound)
        for (int i = 0; i < nch; ++i) {
            const int slot = i & 1, round = i >> 1;
            if (round > 0) {
                if (prod_hint) mbar_wait_hint(&empty[slot], (round - 1) & 1, prod_hint);
                else mbar_wait_backoff(&empty[slot], (round - 1) & 1);
            }
            const int m0 = i * C, cnt = min(C, M - m0);
            const int2 sl = chunk_slabs(i == 0 ? h.tau_start : s_ent[m0 - 1].x, s_ent[m0 + cnt - 1].x, tref, wlo,
                                        whi, lo2f, ip2, nz);
            const int lo4 = sl.x & ~3, hi4 = (sl.y + 4) & ~3;
            CBCT_DCHECK(m0 + cnt <= M && M <= ent_cap && lo4 >= 0 && hi4 <= zs && lo4 < hi4);
            const uint32_t bytes = (uint32_t)(hi4 - lo4) * 4u;
            float* dst = ring + (size_t)slot * slot_elems + RZ * zs + lo4;
            if (lane == 0) {
                s_win[slot] = sl;  // released to the consumers by the arrive below
                mbar_arrive_expect_tx(&full[slot], cnt * bytes);
            }
            __syncwarp();
            for (int j = lane; j < cnt; j += 32)
                bulk_g2s(dst + (size_t)j * zs, vol + (uint32_t)(__float_as_int(s_ent[m0 + j].y) + lo4), bytes,
                         &full[slot]);
        }
    } else {
        // The chunk tables are triple-buffered: chunk i+1's is written during chunk i's phase 1,
        // so a single CTA barrier per chunk (after phase 1) orders everything.  A thread writing
        // table (i+1)%3 has passed barrier i-1, so no thread still reads it (phase 2 of chunk i-2
        // precedes barrier i-1); the ring slots are ordered by the full/empty mbarriers.
        auto fill = [&](float* t, int i, float start) {
            const int m0 = i * C, cnt = min(C, M - m0);
            for (int k = threadIdx.x; k <= PC; k += nct) {
                const float bb = k == 0 ? start : (k <= cnt ? s_ent[m0 + k - 1].x : INFINITY);
                t[k] = bb;
                if (k < cnt) {
                    const float e = s_ent[m0 + k].x;
                    t[PC + 1 + k] = e > bb ? 1.0f / (e - bb) : 0.0f;  // fp32-degenerate interval
                    t[PC + 1 + C + k] = e - bb;
                }
            }
        };
        float chunk_start = h.tau_start;
        fill(sTab, 0, chunk_start);
        named_bar(1, nct);
        int tb = 0;
        for (int i = 0; i < nch; ++i) {
            const int slot = i & 1, round = i >> 1;
            const int cnt = min(C, M - i * C);
            const float* sB = sTab + tb * SBW;
            const float* sInv = sB + (PC + 1);
            const float* sDl = sInv + C;
            const int tn = tb == 2 ? 0 : tb + 1;
            const float cend = sB[cnt];
            mbar_wait(&full[slot], round & 1);
            // phase 1, in place: row j+1 of the slot becomes Qc[j+1] = sum_{j'<=j} dtau_j' vol_j'
            // (row 0 = Qc[0] = 0), two slabs per thread (float2), only over the slabs some ray of
            // the column can occupy while tau is in this chunk (chunk_slabs; the producer staged
            // exactly that window).
            float* stage = ring + (size_t)slot * slot_elems;
            {
                const int2 sl = ZS > 0 ? s_win[slot] : chunk_slabs(chunk_start, cend, tref, wlo, whi, lo2f, ip2, nz);
                const int zs2 = zs >> 1;
                CBCT_DCHECK(sl.x >= 0 && sl.y < zs && sl.x <= sl.y);
                float2* col2 = reinterpret_cast<float2*>(stage + RZ * zs);
                if (ZS > 0 && cnt == C) {
                    // full chunk: C rows at compile-time offsets, dtau in registers
                    float dl[C];
#pragma unroll
                    for (int j = 0; j < C; ++j) dl[j] = sDl[j];
                    for (int pi = (sl.x >> 1) + threadIdx.x; pi <= (sl.y >> 1); pi += nct) {
                        float2 q = make_float2(0.0f, 0.0f);
                        float2* cp = col2 + pi;
#pragma unroll
                        for (int j = 0; j < C; ++j) {
                            const float2 x = cp[j * (ZS / 2)];
                            q.x = fmaf(dl[j], x.x, q.x);
                            q.y = fmaf(dl[j], x.y, q.y);
                            cp[j * (ZS / 2)] = q;
                        }
                    }
                } else {
                    for (int pi = (sl.x >> 1) + threadIdx.x; pi <= (sl.y >> 1); pi += nct) {
                        float2 q = make_float2(0.0f, 0.0f);
                        float2* cp = col2 + pi;
#pragma unroll 4
                        for (int j = 0; j < cnt; ++j) {
                            const float dl = sDl[j];
                            const float2 x = cp[j * zs2];
                            q.x = fmaf(dl, x.x, q.x);
                            q.y = fmaf(dl, x.y, q.y);
                            cp[j * zs2] = q;
                        }
                    }
                }
            }
            if (i + 1 < nch) fill(sTab + tn * SBW, i + 1, cend);
            named_bar(1, nct);  // Qc and the next chunk's table visible
            // phase 2: per ray, the slab it ends in plus one correction per z crossing.  The
            // interval search needs no bounds checks (sB is +inf-padded past the chunk end, which
            // the crossing is before).
            const float* last = stage + (cnt - 1 + RZ) * zs;  // Qc[cnt]
#pragma unroll
            for (int r = 0; r < RPT; ++r) {
                RayState& s = st[r];
                while (s.tz < cend) {
                    int m = 0;
#pragma unroll
                    for (int step = PC / 2; step > 0; step >>= 1)
                        if (sB[m + step] <= s.tz) m += step;
                    const float f = (s.tz - sB[m]) * sInv[m];
                    const float* q1 = stage + (m + RZ) * zs;  // Qc[m+1]
                    const int izn = s.iz + s.dz;
                    CBCT_DCHECK(m >= 0 && m < cnt && s.iz >= 0 && s.iz < zs && izn >= 0 && izn < zs);
                    float a0, b0;
                    if (ZR) {
                        a0 = q1[s.iz - zs];
                        b0 = q1[izn - zs];
                    } else {
                        a0 = m > 0 ? q1[s.iz - zs] : 0.0f;
                        b0 = m > 0 ? q1[izn - zs] : 0.0f;
                    }
                    const float a1 = q1[s.iz], b1 = q1[izn];
                    s.acc += fmaf(f, a1 - a0, a0) - fmaf(f, b1 - b0, b0);
                    s.iz = izn;
                    s.jf += 1.0f;
                    s.tz = s.jf < s.kf ? fmaf(s.jf, s.dtz, s.tz0) : INFINITY;
                }
                CBCT_DCHECK(s.iz >= 0 && s.iz < zs);
                s.acc += last[s.iz];
            }
            chunk_start = cend;
            tb = tn;
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[slot]);  // this warp is done with the slot
        }
    }

    double sq = 0.0;
    if (!producer) {
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            const int v = threadIdx.x + r * nct;
            if (v < nv) {
                const double w = wtab[v];
                const float raylen = (float)sqrt(h.rxy2 + w * w);
                const float out = st[r].acc * raylen;
                proj[(c - c0) * nv + v] = out;
                sq += (double)out * (double)out;
            }
        }
    }
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}

}  // namespace

extern "C" int cbct_project_views(const cbct_plan* p, const float* vol, float* proj, int64_t view0, int64_t view1,
                                  double* partials, void* stream) {
    CbctRange range("cbct_project");
    if (!p || !vol || !proj) return cbct_fail(CBCT_E_ARG, "cbct_project: null argument");
    if (view0 < 0 || view1 > p->V || view0 >= view1) return cbct_fail(CBCT_E_ARG, "cbct_project: bad view range");
    if (view0 < p->own_v0 || view1 > p->own_v1)
        return cbct_fail(CBCT_E_ARG, "cbct_project: views outside this shard plan's view block");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t c0 = view0 * p->nu;
    const dim3 grid((unsigned)((view1 - view0) * p->nu));
    if (p->proj_q && getenv("CBCT_PROJ_LDG") == nullptr && getenv("CBCT_PROJ_TMA") == nullptr) {
        const int Cq = p->proj_q_c;
        const int ent_cap = (int)((p->max_intervals + 3) / 2 * 2);  // even: keeps the TMA ring 16-B aligned
        const int zr = p->proj_q_zr;
        const size_t smem = 48 + (size_t)ent_cap * sizeof(float2) + (size_t)2 * (Cq + zr) * p->zs * 4 +
                            (size_t)3 * (2 * Cq + 33) * 4;
        const int nt = p->proj_threads + 32;
        // compile-time slab strides: BASELINE configs 1/2/3/5 (zs = 72/264/520/1032) and 32-slice subsets (40)
        static const int zs_ct_off = getenv("CBCT_PROJ_ZS_RT") != nullptr;
        const int zsc = zs_ct_off ? 0 : (int)p->zs;
        static const uint32_t hint = getenv("CBCT_PROJ_HINT") ? (uint32_t)atoi(getenv("CBCT_PROJ_HINT")) : 0u;
#define LAUNCH_Q3(R, CC, Z, ZSV)                                                                               \
        do {                                                                                                   \
            CBCT_CHECK(cudaFuncSetAttribute(k_project_q<R, CC, Z, ZSV>,                                        \
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));          \
            k_project_q<R, CC, Z, ZSV><<<grid, nt, smem, s>>>(p->d_cols, p->d_col_off, p->d_col_ent, p->d_w,   \
                                                              vol, proj, partials, (int)p->nv, (int)p->nz,     \
                                                              (int)p->zs, p->lo[2], p->pitch[2], p->flat_v,    \
                                                              ent_cap, c0, (int)p->nu, (int)(view1 - view0),   \
                                                              hint);                                           \
        } while (0)
#define LAUNCH_Q2(R, CC, Z) LAUNCH_Q3(R, CC, Z, 0)
#define LAUNCH_Q2Z(R, CC, Z)                                                                                   \
        do {                                                                                                   \
            switch (zsc) {                                                                                     \
                case 40: LAUNCH_Q3(R, CC, Z, 40); break;                                                       \
                case 72: LAUNCH_Q3(R, CC, Z, 72); break;                                                       \
                case 264: LAUNCH_Q3(R, CC, Z, 264); break;                                                     \
                case 520: LAUNCH_Q3(R, CC, Z, 520); break;                                                     \
                case 1032: LAUNCH_Q3(R, CC, Z, 1032); break;                                                   \
                default: LAUNCH_Q3(R, CC, Z, 0); break;                                                        \
            }                                                                                                  \
        } while (0)
#define LAUNCH_Q(R, CC)                                                                                        \
        do {                                                                                                   \
            if (zr) LAUNCH_Q2(R, CC, true); else LAUNCH_Q2(R, CC, false);                                      \
        } while (0)
#define LAUNCH_QZ(R, CC)                                                                                       \
        do {                                                                                                   \
            if (zr) LAUNCH_Q2Z(R, CC, true); else LAUNCH_Q2Z(R, CC, false);                                    \
        } while (0)
        switch (p->proj_rpt * 100 + Cq) {
            case 108: LAUNCH_Q(1, 8); break;
            case 112: LAUNCH_Q(1, 12); break;
            case 116: LAUNCH_Q(1, 16); break;
            case 132: LAUNCH_Q(1, 32); break;
            case 208: LAUNCH_QZ(2, 8); break;
            case 212: LAUNCH_Q(2, 12); break;
            case 216: LAUNCH_QZ(2, 16); break;
            case 232: LAUNCH_Q(2, 32); break;
            case 408: LAUNCH_Q(4, 8); break;
            case 412: LAUNCH_Q(4, 12); break;
            case 416: LAUNCH_Q(4, 16); break;
            default: LAUNCH_Q(4, 32); break;
        }
#undef LAUNCH_Q
#undef LAUNCH_QZ
#undef LAUNCH_Q2
#undef LAUNCH_Q2Z
#undef LAUNCH_Q3
        CBCT_CHECK(cudaGetLastError());
        cbct_count_launch();
        return 0;
    }
    if (p->proj_tma && getenv("CBCT_PROJ_LDG") == nullptr) {
        const int K = p->proj_tma_k, ns = p->proj_tma_stages;
        const int ent_cap = (int)((p->max_intervals + 2 + 1) / 2 * 2);
        const size_t smem = 16 * ((2 * ns * 8 + 15) / 16) + (size_t)ent_cap * sizeof(float2) +
                            (size_t)ns * K * p->zs * sizeof(float);
        const int nt = p->proj_threads + 32;
#define LAUNCH_T(R, KK)                                                                                        \
        do {                                                                                                   \
            CBCT_CHECK(cudaFuncSetAttribute(k_project_tma<R, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                                            (int)smem));                                                       \
            k_project_tma<R, KK><<<grid, nt, smem, s>>>(p->d_cols, p->d_col_off, p->d_col_ent, p->d_w, vol,      \
                                                        proj, partials, (int)p->nv, (int)p->nz, (int)p->zs,      \
                                                        p->lo[2], p->pitch[2], p->flat_v, ns, ent_cap, c0);      \
        } while (0)
        switch (p->proj_rpt * 10 + K) {
            case 12: LAUNCH_T(1, 2); break;
            case 14: LAUNCH_T(1, 4); break;
            case 18: LAUNCH_T(1, 8); break;
            case 22: LAUNCH_T(2, 2); break;
            case 24: LAUNCH_T(2, 4); break;
            case 28: LAUNCH_T(2, 8); break;
            case 42: LAUNCH_T(4, 2); break;
            case 44: LAUNCH_T(4, 4); break;
            default: LAUNCH_T(4, 8); break;
        }
#undef LAUNCH_T
        CBCT_CHECK(cudaGetLastError());
        cbct_count_launch();
        return 0;
    }
    const size_t smem = (size_t)(p->max_intervals + 2) * sizeof(float2);
    const int nt = p->proj_threads;
#define LAUNCH(R)                                                                                            \
    do {                                                                                                     \
        if (smem > 48 * 1024)                                                                                \
            CBCT_CHECK(cudaFuncSetAttribute(k_project<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                            (int)smem));                                                     \
        k_project<R><<<grid, nt, smem, s>>>(p->d_cols, p->d_col_off, p->d_col_ent, p->d_w, vol, proj,        \
                                            partials, (int)p->nv, (int)p->nz, p->lo[2], p->pitch[2], p->flat_v, c0); \
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

extern "C" int cbct_project(const cbct_plan* p, const float* vol, float* proj, double* partials, void* stream) {
    if (!p) return cbct_fail(CBCT_E_ARG, "cbct_project: null plan");
    return cbct_project_views(p, vol, proj, 0, p->V, partials, stream);
}
