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
#ifdef CBCT_BP_SINGLE
constexpr int kPrefWords = 1;  // ray-prefix table: P[v]
#else
constexpr int kPrefWords = 2;  // ray-prefix table: {P[v], yw[v]} pairs
#endif

// Cells are visited in 16x16 tiles so concurrently resident CTAs share the
// detector columns they read (L2 locality of the prefix arrays).
// Rows [row0, row1) of cells only (a rank's slab in the sharded path).
__device__ __forceinline__ int64_t tiled_cell(int64_t b, int nx, int row0, int row1) {
    const int T = 16;
    const int tx = (nx + T - 1) / T;
    const int64_t per_tile = (int64_t)T * T;
    const int64_t tile = b / per_tile;
    const int k = (int)(b - tile * per_tile);
    const int ty0 = row0 + (int)(tile / tx) * T, tx0 = (int)(tile % tx) * T;
    const int iy = ty0 + k / T, ix = tx0 + k % T;  // padding slots of partial edge tiles return -1
    if (ix >= nx || iy >= row1) return -1;
    return (int64_t)iy * nx + ix;
}


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
__global__ void __launch_bounds__(512) k_bp_direct(const int64_t* __restrict__ cell_off,
                                                     const CellEntry* __restrict__ cell_ent,
                                                     const ColumnHeader* __restrict__ cols,
                                                     const float* __restrict__ invw, const double* __restrict__ wtab,
                                                     const float* __restrict__ yw,
                                                     float* __restrict__ vol, const float* __restrict__ col_scale,
                                                     double* __restrict__ partials, int nv, int nz, int zs,
                                                     double lo2, double p2, double det00z, double pv, int flat_v,
                                                     int mode, int nx, int row0, int row1) {
    extern __shared__ float s_invw[];
    __shared__ Tri s_tri[kChunk];
    const int64_t cell = tiled_cell(blockIdx.x, nx, row0, row1);
    if (cell < 0) {  // padding slot of an edge tile
        if (partials && threadIdx.x == 0) partials[blockIdx.x] = 0.0;
        return;
    }
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

    const int64_t lcell = cell - (int64_t)row0 * nx;  // local cell in the output slab
    float* out = vol + lcell * zs;
    double sq = 0.0;
#pragma unroll
    for (int r = 0; r < ZPT; ++r) {
        if (iz[r] < nz) {
            float val = acc[r];
            if (col_scale) val *= col_scale[lcell * zs + CBCT_ZPAD + iz[r]];
            out[CBCT_ZPAD + iz[r]] = val;
            sq += (double)val * (double)val;
        }
    }
    for (int k = threadIdx.x; k < zs - nz; k += blockDim.x) out[k < CBCT_ZPAD ? k : nz + k] = 0.0f;  // guards
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}


// ---------------------------------------------------------------------------
// Mode-1 fast path: boundary form.  For one crossing (column c, [t_a, t_b]) let
// F_v(z) = |{t in [t_a,t_b] : z_v(t) < z}| be the part of ray v below height z.
// The voxel [z_k, z_k+1) receives  G(z_k+1) - G(z_k)  with
//   G(z) = sum_v yw_v F_v(z) = dt * P_c[V(z)] + yw_s F_s(z)
// where V(z) counts the rays lying entirely below z (a prefix of v because rz_v
// increases with v), P_c is the prefix sum of yw along v, and s = V(z) is the one
// ray that can straddle z (segments are shorter than the ray spacing; the plan
// checks this and otherwise uses k_bp_direct).  One lane per boundary; a warp
// covers 32 boundaries = 31 voxels and exchanges G with its neighbour lane.

// P[c][v] = sum_{v' < v} yw[c][v'], v = 0..nv (yw = |r| * y), padded past both detector
// edges (P = 0 below, P[nv] above; v = -pad_lo .. nv + pad_hi + 1) so the backprojector
// never clamps a row index.
// The straddling ray's own weight is recovered as P[v+1] - P[v] (it only scales
// the straddle fraction F, so the fp32 cancellation there is harmless), which
// halves the bytes per boundary lookup.  The flat row (if any) is kept out of P
// and stored in flatw[c].
// squared (mode 2): yw = |r|^2 (y ignored), the weights of diag(A^T A)'s boundary form (k_bp_sided).
// colidx (shard plans): only the listed columns, the ones crossing the plan's cell rows.
__global__ void k_prefix_rays(const ColumnHeader* __restrict__ cols, const double* __restrict__ wtab,
                              const float* __restrict__ y, float* __restrict__ pref, float* __restrict__ flatw,
                              int64_t n_cols, int nv, int flat_v, int pad_lo, int pad_hi, int squared = 0,
                              const int32_t* __restrict__ colidx = nullptr) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n_cols) return;
    const int64_t c = colidx ? (int64_t)colidx[i] : i;
    const float rxy2 = (float)cols[c].rxy2;
    const float* yc = y + c * nv;
    const int nvq = nv + 2 + pad_lo + pad_hi;
#ifdef CBCT_BP_SINGLE
    float* pc = pref + c * (int64_t)nvq;  // P[v] at row pad_lo + v
    for (int k = lane; k < pad_lo; k += 32) pc[k] = 0.0f;
#else
    float2* pc = reinterpret_cast<float2*>(pref) + c * (int64_t)nvq;  // {P[v], yw[v]} at row pad_lo + v
    for (int k = lane; k < pad_lo; k += 32) pc[k] = make_float2(0.0f, 0.0f);
#endif
    pc += pad_lo;
    double carry = 0.0;
    for (int base = 0; base < nv; base += 32) {
        const int v = base + lane;
        float yw = 0.0f;
        if (v < nv) {
            const float w = (float)wtab[v];
            yw = squared ? fmaf(w, w, rxy2) : sqrtf(fmaf(w, w, rxy2)) * yc[v];  // operator.py:102, 165-167
            if (v == flat_v) {
                flatw[c] = yw;
                yw = 0.0f;
            }
        }
        double incl = (double)yw;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
#ifdef CBCT_BP_SINGLE
        if (v < nv) pc[v] = (float)(carry + incl - (double)yw);
#else
        if (v < nv) pc[v] = make_float2((float)(carry + incl - (double)yw), yw);
#endif
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
#ifdef CBCT_BP_SINGLE
    for (int k = nv + lane; k <= nv + pad_hi + 1; k += 32) pc[k] = (float)carry;
#else
    for (int k = nv + lane; k <= nv + pad_hi + 1; k += 32) pc[k] = make_float2((float)carry, 0.0f);
#endif
}

template <int G, bool FLAT, bool TABLE>
__global__ void __launch_bounds__(1024, 1) k_bp_boundary(const int64_t* __restrict__ cell_off,
                                                      const CellEntry* __restrict__ cell_ent,
                                                      const ColumnHeader* __restrict__ cols,
                                                      const float* __restrict__ invw, const float* __restrict__ pref,
                                                      const float* __restrict__ flatw, float* __restrict__ vol,
                                                      const float* __restrict__ col_scale,
                                                      double* __restrict__ partials, int nv, int nz, int zs,
                                                      double lo2, double p2, double det00z, double pv, int nx,
                                                      int row0, int row1, int pad_lo, int pad_hi,
                                                      const int32_t* __restrict__ boff, int nb, int vb, int accum) {
    extern __shared__ float s_iw[];  // 2 x nvq rows: 1/rz (pad 0); 1/rz for rz < 0, else -inf
    __shared__ float4 s_t0[kChunk], s_t1[kChunk];
    __shared__ int s_vu[kChunk], s_fs[kChunk];
    const int64_t cell = tiled_cell(blockIdx.x, nx, row0, row1);
    if (cell < 0) {  // padding slot of an edge tile
        if (partials && threadIdx.x == 0) partials[blockIdx.x] = 0.0;
        return;
    }
    int64_t off = cell_off[cell];
    int ne = (int)(cell_off[cell + 1] - off);
    if (boff) {  // view batch vb of nb: a contiguous run of the cell's (column-ordered) entries
        const int32_t* bo = boff + cell * (nb + 1) + vb;
        off += bo[0];
        ne = bo[1] - bo[0];
    }
    const int nvq = nv + 2 + pad_lo + pad_hi;
    float* s_iwn = s_iw + nvq;
    for (int k = threadIdx.x; TABLE && k < nvq; k += blockDim.x) {
        const int v = k - pad_lo;
        const float iw = (v >= 0 && v < nv) ? invw[v] : 0.0f;
        s_iw[k] = iw;
        s_iwn[k] = (v >= 0 && v < nv && iw < 0.0f) ? iw : -INFINITY;
    }

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    float z[G], zlo[G], acc[G], sgn[G], sgn2[G], iz[G], sdn[G];
    int kb[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        kb[g] = (warp + g * nwarps) * 31 + lane;  // boundary index (voxel below it is kb-1)
        const double zd = lo2 + (double)min(kb[g], nz) * p2;  // lanes past the top reuse it (unused)
        z[g] = (float)zd;
        zlo[g] = (float)(zd - (double)z[g]);  // the closed form carries z to ~1e-15 (two words)
        acc[g] = 0.0f;
        sgn[g] = z[g] >= 0.0f ? 1.0f : 0.0f;
        sgn2[g] = z[g] >= 0.0f ? 1.0f : -1.0f;
        iz[g] = (float)(1.0 / (lo2 + (double)min(kb[g], nz) * p2));  // 1/z (z = 0: s saturates to 0)
        sdn[g] = 1.0f - sgn[g];  // f = f_t above the mid-plane, 1 - f_t below
    }
    uint32_t tbase[G];
    // Row coordinate of a ray through height z at parameter t: v = z/(t pv) + c0,
    // c0 = -det00z/pv (= nv/2 - 1/2 without a principal-point offset).  c0 is split
    // into an integer and a fraction so the fp32 FFMA only carries z/(t pv) + frac:
    // its rounding then scales with |rz| of the rays near the boundary instead of
    // with |c0| (which would misclassify near-mid-plane rays by ~1e-5 pixel).
    const double c0d = -det00z / pv;
    const double c0i = floor(c0d + 0.5);
    const float c0f = (float)(c0d - c0i);
    const int magic = 0x4B400000 - (int)c0i - 1;  // floor(W) + c0i + 1 via the 1.5*2^23 trick
    const float fpv = (float)pv;
#pragma unroll
    for (int g = 0; g < G; ++g)  // shared address of row 0 of the lane's table minus 4 * magic (mod 2^32)
        tbase[g] = (uint32_t)__cvta_generic_to_shared(sgn[g] != 0.0f ? s_iw : s_iwn) +
                   4u * (uint32_t)(pad_lo - magic);

    for (int base = 0; base < ne; base += kChunk) {
        const int nch = min(kChunk, ne - base);
        __syncthreads();
        for (int k = threadIdx.x; k < nch; k += blockDim.x) {
            const CellEntry ce = cell_ent[off + base + k];
            const ColumnHeader& h = cols[ce.vu];
            const float ta = ce.tau_a, tb = ce.tau_b, tr = h.t_ref;
            const float dt = tb - ta;
            const float idt = dt > 0.0f ? 1.0f / dt : 0.0f;
            const float taa = ta + tr, tba = tb + tr;  // absolute ray parameters
            // 1/(t_a pv) as a two-word fp32 (hi + lo) from fp64: the closed-form straddle
            // fraction needs z / (t_a pv) to ~1e-9 relative (see the inner loop)
            const double iad = 1.0 / (((double)ta + (double)tr) * pv);
            const float ia = (float)iad, ia_lo = (float)(iad - (double)ia);
            const float ib = (float)(1.0 / (((double)tb + (double)tr) * pv));
            // side-blended forms: value = below + up01 * (above - below), up01 in {0, 1} per lane
            if (TABLE) {
                // {1/(t_a pv), 1/(t_b pv) - 1/(t_a pv), t_ref, dt}, {1/dt, -t_a/dt, t_b/dt, flat weight}
                s_t0[k] = make_float4(ia, ib - ia, tr, dt);
                s_t1[k] = make_float4(idt, tb * idt, -(ta + tb) * idt, FLAT ? flatw[ce.vu] : 0.0f);
            } else {
                // {ia (hi), ib - ia, kI = 1/(ia - ib) = pv t_a t_b / dt (from dt: no cancellation), dt},
                // {eps = dt / t_a, ia (lo), 1 - eps, flat weight}
                s_t0[k] = make_float4(ia, ib - ia, dt > 0.0f ? fpv * taa * tba / dt : 0.0f, dt);
                s_t1[k] = make_float4(dt / taa, ia_lo, 1.0f - dt / taa, FLAT ? flatw[ce.vu] : 0.0f);
            }
            s_vu[k] = ce.vu;
            s_fs[k] = FLAT ? h.flat_slab : 0;
        }
        __syncthreads();
#pragma unroll 2  // two entries per trip: the next entry's loads overlap this entry's arithmetic
        for (int k = 0; k < nch; ++k) {
            const float4 t0 = s_t0[k], t1 = s_t1[k];
            // the float->int magic offset is folded into the base: element address = base + bits
#ifdef CBCT_BP_SINGLE
            const float* pyc = pref + (size_t)(uint32_t)s_vu[k] * (uint32_t)nvq + pad_lo - (uint32_t)magic;
#else
            const float2* pyc = reinterpret_cast<const float2*>(pref) + (size_t)(uint32_t)s_vu[k] * (uint32_t)nvq +
                                pad_lo - (uint32_t)magic;
#endif
            asm("mov.b64 %0, %0;" : "+l"(pyc));  // keep the column base in a register (1 IMAD.WIDE per lookup)
            // all lookups first, so the loads of every group are in flight before any use
            float Wg[G], P0[G], P1[G];
            uint32_t bg[G];
#pragma unroll
            for (int g = 0; g < G; ++g) {
                // V(z): rays entirely below z, with t* = t_b above the mid-plane and t_a below
                // (blended with the lane's up01 so no select sits on the ALU pipe).  No row
                // clamping: the prefix table is padded past both detector edges.
                Wg[g] = fmaf(z[g], fmaf(sgn[g], t0.y, t0.x), c0f);
                bg[g] = (uint32_t)__float_as_int(__fadd_rd(Wg[g], 12582912.0f));  // vh + magic
                CBCT_DCHECK(pad_lo - magic + (int)bg[g] >= 0 && pad_lo - magic + (int)bg[g] < nvq);
#ifdef CBCT_BP_SINGLE
                // P[vh] and P[vh+1] (the second load hits the line the first brought to L1)
                P0[g] = __ldg(pyc + bg[g]);
                P1[g] = __ldg(pyc + bg[g] + 1) - P0[g];  // yw[vh]
#else
                const float2 py = __ldg(pyc + bg[g]);  // {P[vh], yw[vh]}: one 8-byte load
                P0[g] = py.x;
                P1[g] = py.y;
#endif
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const uint32_t bits = bg[g];
                float f;
                if (TABLE) {
                    // Straddler (ray vh): fraction of [t_a, t_b] below z as one saturated FFMA
                    // (FMA pipe); below the mid-plane the table holds -inf for rz >= 0 rays, which
                    // saturates to 0 (such a ray cannot straddle a negative z).
                    float iw;
                    asm("ld.shared.f32 %0, [%1];" : "=f"(iw) : "r"(tbase[g] + bits * 4u));
                    const float u = fmaf(z[g], iw, -t0.z);
                    // above: (u - t_a)/dt = u/dt - t_a/dt ; below: (t_b - u)/dt   (t_a/dt = t_b/dt - 1)
                    const float kap = fmaf(sgn[g], t1.z, t1.y);  // up: -t_a/dt, down: t_b/dt
                    f = __saturatef(fmaf(u, sgn2[g] * t1.x, kap));
                } else {
                    // Straddler without a table.  W(t) = z/(t pv) + c0 is linear in 1/t, so the
                    // straddler (row coordinate R = floor(W) + 1) meets height z at the 1/t-fraction
                    //   s = (W_a - R) / (W_a - W_b) = (z ia + c0f - R) kI / z      (both sides)
                    // of [t_a, t_b], and at the t-fraction  f_t = s / (1 + eps (1 - s)),
                    // eps = dt / t_a, taken to first order (error <= eps^2/4; the plan selects this
                    // form for eps <= 3e-3).  f = f_t above the mid-plane (a rising ray is below z
                    // before t*), 1 - f_t below; rays that cannot straddle saturate to 0.
                    // W_a - R is formed as fma(z, ia_lo, fma(z, ia_hi, -R) + c0f): every rounding
                    // happens on an O(1) quantity, so f carries ~1e-7 absolute error instead of
                    // the ~1e-4 an fp32 z/(t pv) near |W| ~ 300 rows would give.
                    const float R = __int_as_float((int)bits) - 12582911.0f;  // floor(W) + 1, exact
                    // s is saturated to [0, 1] first (the first-order f_t is only valid there; rays
                    // that cannot straddle have s < 0 or > 1), then f_t = s (1 - eps + eps s).
                    // z ia_lo + z_lo ia + c0f, independent of R: with z and 1/(t_a pv) both carried as
                    // two fp32 words, W_a - R keeps ~1e-7 rows of absolute error even where the
                    // straddle window W_a - W_b is only ~|W| eps wide (config 5: 0.04 rows)
                    const float tail = fmaf(zlo[g], t0.x, fmaf(z[g], t1.y, c0f));
                    const float sv = __saturatef((fmaf(z[g], t0.x, -R) + tail) * (iz[g] * t0.z));
                    const float h = fmaf(t1.x, sv, t1.z);            // 1 - eps + eps s
                    f = fmaf(sgn2[g] * sv, h, sdn[g]);               // f_t above, 1 - f_t below
                }
                const float Gv = fmaf(f, P1[g], P0[g]);  // P[vh] + f yw[vh]; dt applied once below
                const float Gn = __shfl_down_sync(0xffffffffu, Gv, 1);
                acc[g] = fmaf(t0.w, Gn - Gv, acc[g]);
                if (FLAT) acc[g] += (kb[g] == s_fs[k]) ? t0.w * t1.w : 0.0f;
            }
        }
    }

    const int64_t lcell = cell - (int64_t)row0 * nx;  // local cell in the output slab
    float* out = vol + lcell * zs;
    double sq = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int iz = kb[g];  // voxel [z_kb, z_kb+1)
        if (lane < 31 && iz < nz) {
            float val = acc[g];
            if (col_scale) val *= col_scale[lcell * zs + CBCT_ZPAD + iz];
            if (accum) val += out[CBCT_ZPAD + iz];  // later view batches add to the earlier ones
            out[CBCT_ZPAD + iz] = val;
            sq += (double)val * (double)val;
        }
    }
    for (int k = threadIdx.x; k < zs - nz; k += blockDim.x) out[k < CBCT_ZPAD ? k : nz + k] = 0.0f;  // guards
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}

// ---------------------------------------------------------------------------
// Sided variant of the closed-form boundary kernel.  The boundary form needs, per
// boundary, which end of the crossing bounds a ray's height (t_b above the mid-plane,
// t_a below) and whether the straddle fraction is f_t or 1 - f_t.  k_bp_boundary blends
// both per lane with sign registers; at 64 registers and six groups the compiler
// rematerialises them every entry (~5 of ~23 instructions per boundary).  Here the
// boundaries are grouped so that every group lies on one side: above groups start at k0
// (the first boundary with z >= 0) and run up, below groups end at k0 and run down, and
// each warp runs GS below groups and GS above groups with the side known at compile time.
// The top below group's last lane sits on z_k0; the plan only selects this kernel when
// that boundary is exactly z = 0 (or one side is empty), where the below formula with
// z = -0 (1/z = -inf) yields the above formula's value: no ray straddles the plane z = 0
// (rays through the source height are the separate flat row).
// MODE2: diag(A^T A) = sum seg^2 (operator.py:166-167) in the same boundary form.  With the table
// holding the prefix P2 of |r|^2 and H(z) = P2[V] + f^2 |r_V|^2, voxel k receives
//   dt^2 (H(z_k+1) - H(z_k) - 2 f_k (1 - f_k) |r_V_k|^2)
// (the straddler of the lower boundary contributes (1 - f_k)^2, not 1 - f_k^2); exact while no ray
// spans a whole voxel height inside one crossing, which the plan checks (bps_mode2_ok).
template <int GS, bool FLAT, int MAXR, bool MODE2 = false, bool PAIR = false>
__global__ void __maxnreg__(MAXR) k_bp_sided(const int64_t* __restrict__ cell_off,
                                                    const CellEntry* __restrict__ cell_ent,
                                                    const ColumnHeader* __restrict__ cols,
                                                    const float* __restrict__ pref, const float* __restrict__ flatw,
                                                    float* __restrict__ vol, const float* __restrict__ col_scale,
                                                    double* __restrict__ partials, int nv, int nz, int zs,
                                                    double lo2, double p2, double det00z, double pv, int nx,
                                                    int row0, int row1, int pad_lo, int pad_hi,
                                                    const int32_t* __restrict__ boff, int nb, int vb, int accum,
                                                    int k0, int zero_at_k0) {
    constexpr int G = 2 * GS;  // groups [0, GS): below, [GS, 2 GS): above
    __shared__ float4 s_t0[kChunk], s_t1[kChunk];
    __shared__ float2 s_t2[kChunk];
    __shared__ long long s_base[kChunk];
    __shared__ int s_fs[FLAT ? kChunk : 1];
#ifdef CBCT_CHECKED
    __shared__ int s_vuc[kChunk];
#endif
    const int64_t cell = tiled_cell(blockIdx.x, nx, row0, row1);
    if (cell < 0) {
        if (partials && threadIdx.x == 0) partials[blockIdx.x] = 0.0;
        return;
    }
    int64_t off = cell_off[cell];
    int ne = (int)(cell_off[cell + 1] - off);
    if (boff) {
        const int32_t* bo = boff + cell * (nb + 1) + vb;
        off += bo[0];
        ne = bo[1] - bo[0];
    }
    const int nvq = nv + 2 + pad_lo + pad_hi;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // Boundary heights are z = z_off + zp p2 with zp = k - k0 an exact small integer in fp32, so
    // z / (t pv) = zp (p2 / (t pv)) + z_off / (t pv): the per-crossing slopes p2/(t pv) carry the
    // precision (two fp32 words for the t_a slope) and z needs no second word.
    const int kk0 = min(k0, nz);
    const double zoff = lo2 + (double)kk0 * p2;  // z at k0 (0 when both sides are present)
    float zp[G], acc[G], iz[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int gi = warp * GS + (g < GS ? g : g - GS);
        const int kb = g < GS ? k0 - 31 * (gi + 1) + lane : k0 + 31 * gi + lane;  // boundary index
        const int kc = min(max(kb, 0), nz);  // lanes outside the volume reuse an end (results unused)
        zp[g] = (float)(kc - kk0);
        iz[g] = (float)(1.0 / (zoff + (double)(kc - kk0) * p2));
        if (g < GS && kc == k0 && zero_at_k0) {  // z_k0 = 0 seen from below: -0 and 1/z = -inf
            zp[g] = -0.0f;
            iz[g] = -INFINITY;
        }
        acc[g] = 0.0f;
    }
    const double c0d = -det00z / pv;
    // side of the row lookup when only one side exists (with both, z_off = 0 and both agree)
    const bool look_b = k0 == 0;

    for (int base = 0; base < ne; base += kChunk) {
        const int nch = min(kChunk, ne - base);
        __syncthreads();
        for (int k = threadIdx.x; k < nch; k += blockDim.x) {
            const CellEntry ce = cell_ent[off + base + k];
            const ColumnHeader& h = cols[ce.vu];
            const float ta = ce.tau_a, tb = ce.tau_b, tr = h.t_ref;
            const float dt = tb - ta;
            const float taa = ta + tr, tba = tb + tr;
            const double iad = 1.0 / (((double)ta + (double)tr) * pv);
            const double ibd = 1.0 / (((double)tb + (double)tr) * pv);
            const double sad = p2 * iad;
            const float sa = (float)sad, sa_lo = (float)(sad - (double)sa);
            // row coordinates at z_off: W = zp * slope + B; B's integer part goes into the table base
            const double Ba = zoff * iad + c0d;
            const double Bl = look_b ? zoff * ibd + c0d : Ba;
            const double Bi = floor(Bl + 0.5);
            const int magic = 0x4B400000 - (int)Bi - 1;  // floor(W) + Bi + 1 via the 1.5*2^23 trick
            // {p2/(t_a pv), p2/(t_b pv), kI = pv t_a t_b / dt, dt}, {eps = dt / t_a, p2/(t_a pv) lo, 1 - eps, flat},
            // {lookup B fraction, W_a offset relative to the lookup's integer}
            s_t0[k] = make_float4(sa, (float)(p2 * ibd), dt > 0.0f ? (float)pv * taa * tba / dt : 0.0f,
                                  MODE2 ? dt * dt : dt);
            s_t1[k] = make_float4(dt / taa, sa_lo, 1.0f - dt / taa, FLAT ? flatw[ce.vu] : 0.0f);
            s_t2[k] = make_float2((float)(Bl - Bi), (float)(Ba - Bi));
            s_base[k] = (long long)ce.vu * nvq + pad_lo - (long long)magic;
            if (FLAT) s_fs[k] = cols[ce.vu].flat_slab;
#ifdef CBCT_CHECKED
            s_vuc[k] = ce.vu;
#endif
        }
        __syncthreads();
        // PAIR: entries in groups of EPT = 4, the crossings' dt-weighted boundary values summed before
        // the neighbour shuffle, H = sum_e dt_e G_e and voxel += H(k+1) - H(k), so one shuffle serves
        // four crossings (the shuffle was a third of the L1 data-pipe work; config 3 at GS = 3: one
        // entry per shuffle 104.9-107.1 ms, two 101.0-102.1, four 96.6-96.8, eight 96.0).  G carries
        // ~1e-7 relative rounding either way; the difference keeps the same absolute error per
        // crossing.  Without PAIR one entry per shuffle, two entries unrolled.
#ifndef CBCT_BP_EPT
#define CBCT_BP_EPT 4
#endif
        constexpr int EPT = PAIR ? CBCT_BP_EPT : 1;
#pragma unroll(PAIR ? 1 : 2)
        for (int k = 0; k < nch; k += EPT) {
            float H[G], Cm[MODE2 ? G : 1];
#pragma unroll
            for (int e = 0; e < EPT; ++e) {
                const int ke = k + e;
                if (e > 0 && ke >= nch) break;
                const float4 t0 = s_t0[ke], t1 = s_t1[ke];
                const float2 t2 = s_t2[ke];
                const float2* pyc = reinterpret_cast<const float2*>(pref) + s_base[ke];
                asm("mov.b64 %0, %0;" : "+l"(pyc));
                float P0[G], P1[G];
                uint32_t bg[G];
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    // rays entirely below z: rows under W(t_b) above the mid-plane, W(t_a) below
                    const float W = fmaf(zp[g], g < GS ? t0.x : t0.y, t2.x);
                    bg[g] = (uint32_t)__float_as_int(__fadd_rd(W, 12582912.0f));
                    CBCT_DCHECK(s_base[ke] + (long long)bg[g] - (long long)s_vuc[ke] * nvq >= 0 &&
                                s_base[ke] + (long long)bg[g] - (long long)s_vuc[ke] * nvq < nvq);
                    const float2 py = __ldg(pyc + bg[g]);
                    P0[g] = py.x;
                    P1[g] = py.y;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    // straddle fraction (closed form, k_bp_boundary): s = (W_a - R) kI / z in 1/t,
                    // f_t = s (1 - eps + eps s); W_a - R = zp sa + (B_a - Bi) - R with every rounding on O(1)
                    const float R = __int_as_float((int)bg[g]) - 12582911.0f;
                    const float u = fmaf(zp[g], t1.y, fmaf(zp[g], t0.x, t2.y - R));
                    const float sv = __saturatef(u * (iz[g] * t0.z));
                    const float h = fmaf(t1.x, sv, t1.z);
                    const float f = g < GS ? fmaf(-sv, h, 1.0f) : sv * h;  // below: 1 - f_t ; above: f_t
                    if (MODE2) {
                        const float fw = f * P1[g];
                        const float Gv = fmaf(f, fw, P0[g]);   // P2[V] + f^2 w2
                        const float c = 2.0f * (fw - f * fw);  // 2 f (1 - f) w2
                        H[g] = e == 0 ? t0.w * Gv : fmaf(t0.w, Gv, H[g]);
                        Cm[g] = e == 0 ? t0.w * c : fmaf(t0.w, c, Cm[g]);
                    } else {
                        const float Gv = fmaf(f, P1[g], P0[g]);
                        H[g] = e == 0 ? t0.w * Gv : fmaf(t0.w, Gv, H[g]);
                    }
                    if (FLAT) {
                        const int gi = warp * GS + (g < GS ? g : g - GS);
                        const int kb = g < GS ? k0 - 31 * (gi + 1) + lane : k0 + 31 * gi + lane;
                        acc[g] += (kb == s_fs[ke]) ? t0.w * t1.w : 0.0f;
                    }
                }
            }
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float Hn = __shfl_down_sync(0xffffffffu, H[g], 1);
                acc[g] += MODE2 ? (Hn - H[g]) - Cm[MODE2 ? g : 0] : Hn - H[g];
            }
        }
    }

    const int64_t lcell = cell - (int64_t)row0 * nx;
    float* out = vol + lcell * zs;
    double sq = 0.0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int gi = warp * GS + (g < GS ? g : g - GS);
        const int kv = g < GS ? k0 - 31 * (gi + 1) + lane : k0 + 31 * gi + lane;  // voxel [z_kv, z_kv+1)
        const bool mine = lane < 31 && kv >= 0 && kv < nz && (g < GS ? kv < k0 : kv >= k0);
        if (mine) {
            float val = acc[g];
            if (col_scale) val *= col_scale[lcell * zs + CBCT_ZPAD + kv];
            if (accum) val += out[CBCT_ZPAD + kv];
            out[CBCT_ZPAD + kv] = val;
            sq += (double)val * (double)val;
        }
    }
    for (int k = threadIdx.x; k < zs - nz; k += blockDim.x) out[k < CBCT_ZPAD ? k : nz + k] = 0.0f;
    if (partials) {
        const double tot = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = tot;
    }
}

}  // namespace

extern "C" int cbct_backproject_rows(const cbct_plan* p, const float* proj, float* vol, int64_t row0, int64_t row1,
                                     int mode, float* scratch, const float* col_scale, double* partials,
                                     void* stream) {
    CbctRange range(mode == 2 ? "cbct_normal_diagonal" : "cbct_backproject");
    if (p && (row0 < 0 || row1 > p->ny || row0 >= row1))
        return cbct_fail(CBCT_E_ARG, "cbct_backproject: bad row range");
    if (!p || !vol || !scratch) return cbct_fail(CBCT_E_ARG, "cbct_backproject: null argument");
    if (row0 < p->own_r0 || row1 > p->own_r1)
        return cbct_fail(CBCT_E_ARG, "cbct_backproject: cell rows outside this shard plan's row block");
    if (mode != 1 && mode != 2) return cbct_fail(CBCT_E_ARG, "cbct_backproject: mode must be 1 or 2");
    if (mode == 1 && !proj) return cbct_fail(CBCT_E_ARG, "cbct_backproject: mode 1 needs projections");
    cudaStream_t s = (cudaStream_t)stream;
    // Mode 2 (diag(A^T A), once per Jacobi solve) always clips in fp64: its squared weights
    // double the fp32 clip's relative error, which reaches ~1e-4 at 0.43 mm voxels.
    // Where the sided boundary kernel runs (closed form, z = 0 on a boundary or one-sided), mode 2
    // uses its squared-weight boundary form instead (bps_mode2_ok: no ray spans a voxel height in a
    // crossing); CBCT_BP_DIAG_DIRECT=1 keeps the fp64-clip direct kernel.
    static const bool diag_direct = getenv("CBCT_BP_DIAG_DIRECT") != nullptr;
    const bool closed_rt = p->bp_closed_ok && getenv("CBCT_BP_TABLE") == nullptr;
    const bool mode2_sided = mode == 2 && p->bp_boundary_ok && closed_rt && p->bps_eligible && p->bps_mode2_ok &&
                             !diag_direct;
    const bool precise = (mode == 2 && !mode2_sided) || getenv("CBCT_BP_PRECISE") != nullptr;
    static const bool force_direct = getenv("CBCT_BP_DIRECT") != nullptr;  // diagnosis: fp32 direct kernel
    if ((mode == 1 || mode2_sided) && p->bp_boundary_ok && !precise && !force_direct) {
        float* pyb = scratch;
        const int nvq = (int)p->nv + 2 + p->bp_pad_lo + p->bp_pad_hi;
        float* flatw = scratch + p->n_cols * nvq * kPrefWords;
        // shard plans: the prefix of the columns crossing the plan's rows only (the others are never read)
        static const bool pref_all = getenv("CBCT_BP_PREF_ALL") != nullptr;
        const bool listed = p->d_pref_cols && !pref_all;
        const int64_t ncp = listed ? p->n_pref_cols : p->n_cols;
        const int64_t nthreads = ncp * 32;
        if (ncp > 0)
            k_prefix_rays<<<(unsigned)((nthreads + 255) / 256), 256, 0, s>>>(
                p->d_cols, p->d_w, proj, pyb, flatw, ncp, (int)p->nv, p->flat_v, p->bp_pad_lo, p->bp_pad_hi,
                mode == 2 ? 1 : 0, listed ? p->d_pref_cols : nullptr);
        CBCT_CHECK(cudaGetLastError());
        // closed-form straddle fraction unless the cells are long relative to the source distance
        static const bool force_table = getenv("CBCT_BP_TABLE") != nullptr;
        const bool table = force_table || !p->bp_closed_ok;
        const size_t smem = table ? 2 * (size_t)nvq * sizeof(float) : 0;
        const int64_t tiles = ((p->nx + 15) / 16) * ((row1 - row0 + 15) / 16);
        const dim3 grid((unsigned)(tiles * 256));
#define LAUNCH_G(G, FL)                                                                                        \
        do {                                                                                                   \
            if (table) {                                                                                       \
                CBCT_CHECK(cudaFuncSetAttribute(k_bp_boundary<G, FL, true>,                                    \
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));      \
                k_bp_boundary<G, FL, true><<<grid, p->bpg_threads, smem, s>>>(                                 \
                    p->d_cell_off, p->d_cell_ent, p->d_cols, p->d_invw, pyb, flatw, vol, col_scale, part,  \
                    (int)p->nv, (int)p->nz, (int)p->zs, p->lo[2], p->pitch[2], p->det00z, p->pv, (int)p->nx,  \
                    (int)row0, (int)row1, p->bp_pad_lo, p->bp_pad_hi, boff, nb, vb, vb > 0);                                                                               \
                break;                                                                                         \
            }                                                                                                  \
            k_bp_boundary<G, FL, false><<<grid, p->bpg_threads, smem, s>>>(                                    \
                p->d_cell_off, p->d_cell_ent, p->d_cols, p->d_invw, pyb, flatw, vol, col_scale, part,      \
                (int)p->nv, (int)p->nz, (int)p->zs, p->lo[2], p->pitch[2], p->det00z, p->pv, (int)p->nx,      \
                (int)row0, (int)row1, p->bp_pad_lo, p->bp_pad_hi, boff, nb, vb, vb > 0);                                                                                   \
        } while (0)
        const bool fl = p->flat_v >= 0;
        // view batches (plan.bp_vbatch): one launch per batch of views keeps the ray-prefix
        // columns the resident CTAs gather from closer to L2's size; the last launch writes the
        // norm partials
        const int nb = p->bp_vbatch;
        const int32_t* boff = nb > 1 ? p->d_cell_boff : nullptr;
        const bool sided = !table && (p->bps_ok || mode2_sided);
        // register cap of the sided kernel: 56 for GS = 3 (11 CTAs of 96 threads instead of 10; config 3
        // A^T 107.8 -> 105.7 ms), 64 for GS = 2 (config 5: 56 regs spill, 1379 vs 1418 ms)
        // entry pairs per shuffle for GS = 3 at 64 registers (config 3: 101.0 ms; 56 registers spill), single
        // entries at GS = 2 (config 5: pairs 1455 vs 1375 ms)
        static const int regs_env = getenv("CBCT_BP_REGS") ? atoi(getenv("CBCT_BP_REGS")) : 0;
        static const int pair_env = getenv("CBCT_BP_PAIR") ? atoi(getenv("CBCT_BP_PAIR")) : -1;
        const bool pair = pair_env >= 0 ? pair_env != 0 : p->bps_gs == 3;
        const int sided_regs = regs_env ? regs_env : (p->bps_gs == 3 && !pair ? 56 : 64);
#define LAUNCH_S1(GS, FL, MR)                                                                                  \
        do {                                                                                                   \
            if (pair) {                                                                                        \
                if (mode == 2) LAUNCH_S2(GS, FL, MR, true, true); else LAUNCH_S2(GS, FL, MR, false, true);     \
            } else {                                                                                           \
                if (mode == 2) LAUNCH_S2(GS, FL, MR, true, false); else LAUNCH_S2(GS, FL, MR, false, false);   \
            }                                                                                                  \
        } while (0)
#define LAUNCH_S2(GS, FL, MR, M2, PR)                                                                          \
        k_bp_sided<GS, FL, MR, M2, PR><<<grid, p->bps_threads, 0, s>>>(                                       \
            p->d_cell_off, p->d_cell_ent, p->d_cols, pyb, flatw, vol, col_scale, part, (int)p->nv, (int)p->nz, \
            (int)p->zs, p->lo[2], p->pitch[2], p->det00z, p->pv, (int)p->nx, (int)row0, (int)row1,             \
            p->bp_pad_lo, p->bp_pad_hi, boff, nb, vb, vb > 0, p->bps_k0, p->bps_zero)
#define LAUNCH_S(GS, FL)                                                                                       \
        do {                                                                                                   \
            if (sided_regs == 48) LAUNCH_S1(GS, FL, 48);                                                       \
            else if (sided_regs == 56) LAUNCH_S1(GS, FL, 56);                                                  \
            else LAUNCH_S1(GS, FL, 64);                                                                        \
        } while (0)
        for (int vb = 0; vb < nb; ++vb) {
            double* part = vb == nb - 1 ? partials : nullptr;
            if (sided) {
                switch (p->bps_gs * 2 + (fl ? 1 : 0)) {
                    case 2: LAUNCH_S(1, false); break;
                    case 3: LAUNCH_S(1, true); break;
                    case 4: LAUNCH_S(2, false); break;
                    case 5: LAUNCH_S(2, true); break;
                    case 6: LAUNCH_S(3, false); break;
                    default: LAUNCH_S(3, true); break;
                }
                continue;
            }
            switch (p->bpg_groups * 2 + (fl ? 1 : 0)) {
                case 2: LAUNCH_G(1, false); break;
                case 3: LAUNCH_G(1, true); break;
                case 4: LAUNCH_G(2, false); break;
                case 5: LAUNCH_G(2, true); break;
                case 6: LAUNCH_G(3, false); break;
                case 7: LAUNCH_G(3, true); break;
                case 8: LAUNCH_G(4, false); break;
                case 9: LAUNCH_G(4, true); break;
                case 10: LAUNCH_G(5, false); break;
                case 11: LAUNCH_G(5, true); break;
                case 12: LAUNCH_G(6, false); break;
                default: LAUNCH_G(6, true); break;
            }
        }
#undef LAUNCH_G
#undef LAUNCH_S
#undef LAUNCH_S1
#undef LAUNCH_S2
        CBCT_CHECK(cudaGetLastError());
        cbct_count_launch(1 + nb);
        return 0;
    }
    const int64_t nr = p->n_rays;
    k_weight_rays<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(p->d_cols, p->d_w, mode == 1 ? proj : nullptr,
                                                                 scratch, p->n_cols, (int)p->nv);
    CBCT_CHECK(cudaGetLastError());
    const size_t smem = (size_t)p->nv * sizeof(float);
    const dim3 grid((unsigned)(((p->nx + 15) / 16) * ((row1 - row0 + 15) / 16) * 256));
#define LAUNCH(Z, PR)                                                                                         \
    do {                                                                                                      \
        if (smem > 40 * 1024)                                                                                 \
            CBCT_CHECK(cudaFuncSetAttribute(k_bp_direct<Z, PR>, cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                            (int)smem));                                                      \
        k_bp_direct<Z, PR><<<grid, p->bp_threads, smem, s>>>(p->d_cell_off, p->d_cell_ent, p->d_cols,         \
                                                             p->d_invw, p->d_w, scratch, vol, col_scale,      \
                                                             partials, (int)p->nv, (int)p->nz, (int)p->zs,    \
                                                             p->lo[2], p->pitch[2], p->det00z, p->pv,         \
                                                             p->flat_v, mode, (int)p->nx, (int)row0, (int)row1);        \
    } while (0)
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

extern "C" int cbct_backproject(const cbct_plan* p, const float* proj, float* vol, int mode, float* scratch,
                                const float* col_scale, double* partials, void* stream) {
    if (!p) return cbct_fail(CBCT_E_ARG, "cbct_backproject: null plan");
    return cbct_backproject_rows(p, proj, vol, 0, p->ny, mode, scratch, col_scale, partials, stream);
}
