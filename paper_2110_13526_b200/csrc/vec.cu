// vec.cu -- fused solver vector kernels (HBM-bound), deterministic fp64 partials.
//
// A CGLS iteration (solvers.py:339-357) is, besides A and A^T:
//   volume:      x += alpha_prev*d ; d = r + beta*d        (x-update deferred one
//                iteration so both fuse into one pass: 20 B/voxel)
//   projection:  e -= alpha*p ; ||e||^2                    (12 B/ray)
// ||r||^2 and ||p||^2 come from the A^T / A epilogues.  Every reduction writes one
// fp64 partial per CTA with a fixed element->thread map, then cbct_reduce_partials
// sums them in a fixed order, so results are bitwise reproducible.
#include <cmath>

#include "cbct_internal.cuh"
#include "reduce.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 8;

inline int vec_blocks(int64_t n) {
    const int64_t b = (n + kThreads * 4 - 1) / (kThreads * 4);
    return (int)(b < 1 ? 1 : (b > kMaxBlocks ? kMaxBlocks : b));
}

__device__ __forceinline__ void finish(double sq, double* partials) {
    if (partials) {
        const double t = block_sum(sq);
        if (threadIdx.x == 0) partials[blockIdx.x] = t;
    }
}

__global__ void k_cgls_volume(int64_t n, float* __restrict__ x, float* __restrict__ d, const float* __restrict__ r,
                              float alpha_prev, int do_x, float beta, int use4) {
    const int64_t n4 = use4 ? n >> 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float4* x4 = reinterpret_cast<float4*>(x);
    float4* d4 = reinterpret_cast<float4*>(d);
    const float4* r4 = reinterpret_cast<const float4*>(r);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 dv = d4[i];
        const float4 rv = r4[i];
        if (do_x) {
            float4 xv = x4[i];
            xv.x = fmaf(alpha_prev, dv.x, xv.x); xv.y = fmaf(alpha_prev, dv.y, xv.y);
            xv.z = fmaf(alpha_prev, dv.z, xv.z); xv.w = fmaf(alpha_prev, dv.w, xv.w);
            x4[i] = xv;
        }
        dv.x = fmaf(beta, dv.x, rv.x); dv.y = fmaf(beta, dv.y, rv.y);
        dv.z = fmaf(beta, dv.z, rv.z); dv.w = fmaf(beta, dv.w, rv.w);
        d4[i] = dv;
    }
    for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        if (do_x) x[i] = fmaf(alpha_prev, d[i], x[i]);
        d[i] = fmaf(beta, d[i], r[i]);
    }
}

// y = a*x + b*y (x may be NULL: y = b*y); partials of y^2
__global__ void k_axpby(int64_t n, float a, const float* __restrict__ x, float b, float* __restrict__ y,
                        double* __restrict__ partials, int use4) {
    const int64_t n4 = use4 ? n >> 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 yv = y4[i];
        if (x) {
            const float4 xv = x4[i];
            yv.x = fmaf(a, xv.x, b * yv.x); yv.y = fmaf(a, xv.y, b * yv.y);
            yv.z = fmaf(a, xv.z, b * yv.z); yv.w = fmaf(a, xv.w, b * yv.w);
        } else {
            yv.x *= b; yv.y *= b; yv.z *= b; yv.w *= b;
        }
        y4[i] = yv;
        sq += (double)yv.x * yv.x + (double)yv.y * yv.y + (double)yv.z * yv.z + (double)yv.w * yv.w;
    }
    for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float yv = x ? fmaf(a, x[i], b * y[i]) : b * y[i];
        y[i] = yv;
        sq += (double)yv * yv;
    }
    finish(sq, partials);
}

// out = a - b ; partials of out^2
__global__ void k_sub(int64_t n, const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ out,
                      double* __restrict__ partials) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float v = a[i] - b[i];
        out[i] = v;
        sq += (double)v * v;
    }
    finish(sq, partials);
}

// partials of x.y
__global__ void k_dot(int64_t n, const float* __restrict__ x, const float* __restrict__ y,
                      double* __restrict__ partials) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        s += (double)x[i] * (double)y[i];
    finish(s, partials);
}

__global__ void k_mul(int64_t n, const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ o) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) o[i] = a[i] * b[i];
}

__global__ void k_fill(int64_t n, float* __restrict__ x, float v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) x[i] = v;
}

__global__ void k_fill_volume(int64_t n, int64_t zs, int64_t nz, float* __restrict__ x, float v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t k = i % zs;
        x[i] = (k >= CBCT_ZPAD && k < CBCT_ZPAD + nz) ? v : 0.0f;
    }
}

__global__ void k_clip(int64_t n, int64_t zs, int64_t nz, float* __restrict__ x, float lo, float hi) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const int64_t k = i % zs;
        if (k >= CBCT_ZPAD && k < CBCT_ZPAD + nz) x[i] = fminf(fmaxf(x[i], lo), hi);
    }
}

__global__ void k_reduce(const double* __restrict__ partials, int n, double* __restrict__ out) {
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += partials[i];
    const double t = block_sum(s);
    if (threadIdx.x == 0) *out = t;
}

bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// ---------------------------------------------------------------------------
// Device-resident CGLS scalars (the host loop's recurrences, solvers.py:339-357, in the same
// fp64 operations, so results are bitwise identical to it).  Layout of S (include/cbct.h):
enum : int {
    kSNr2Old = 0, kSNr2 = 1, kSNp2 = 2, kSAlpha = 3, kSBeta = 4, kSNb2 = 5, kSState = 6, kSIter = 7, kSNb0 = 8,
    kSTol = 9, kSDoX = 10, kSHist = 16
};

__global__ void k_cgls_scalars(double* __restrict__ S, int stage) {
    if (S[kSState] != 0.0) return;  // stopped: every later stage and vector update is a no-op
    if (stage == 1) {               // after A^T: ||r||^2 in S[kSNr2]
        const double nr2 = S[kSNr2];
        if (nr2 == 0.0) {
            S[kSState] = 1.0;  // breakdown (the deferred x update stays pending)
            return;
        }
        S[kSBeta] = nr2 / S[kSNr2Old];
        S[kSDoX] = S[kSAlpha] != 0.0 ? 1.0 : 0.0;
        S[kSNr2Old] = nr2;
    } else if (stage == 2) {  // after A: ||p||^2 in S[kSNp2]
        const double np2 = S[kSNp2];
        if (np2 == 0.0) {
            S[kSState] = 1.0;
            S[kSAlpha] = 0.0;  // the update already consumed the pending alpha
            return;
        }
        S[kSAlpha] = S[kSNr2Old] / np2;
    } else {  // after e -= alpha p: ||e||^2 in S[kSNb2]
        const double it = S[kSIter] + 1.0;
        S[kSIter] = it;
        S[kSHist + (int)it] = S[kSNb2];
        const double nb0 = S[kSNb0];
        const double rel = nb0 > 0.0 ? sqrt(S[kSNb2]) / nb0 : 0.0;
        if (!(rel > S[kSTol])) S[kSState] = 2.0;  // converged to the tolerance
    }
}

// ---------------------------------------------------------------------------
// Fused update + all-gather over NVLink peer memory (multi-GPU CGLS).
// The rank's slab of the new d (or e) is stored into every rank's full-size buffer (peer
// pointers from the symmetric-memory rendezvous, self included) at the same offset, so the
// next operator finds the full vector in place after one device barrier: the all_gather's
// transfer is issued by the update kernel itself, store by store, instead of by a separate
// collective.  The rank's own slab of its full buffer is its local vector.
// Same element -> thread map as k_cgls_volume_dev / k_cgls_proj_dev (float4 body + scalar tail),
// so values and fp64 partial sums are bitwise those of the gathered path.
__global__ void k_cgls_volume_dev_p2p(int64_t n, float* __restrict__ x, const float* __restrict__ d_own,
                                      const float* __restrict__ r, const double* __restrict__ S,
                                      float* const* __restrict__ peers, int npeers, int64_t offset, int use4) {
    if (S[kSState] != 0.0) return;
    const float alpha_prev = (float)S[kSAlpha], beta = (float)S[kSBeta];
    const int do_x = S[kSDoX] != 0.0;
    const int64_t n4 = use4 ? n >> 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float4* x4 = reinterpret_cast<float4*>(x);
    const float4* d4 = reinterpret_cast<const float4*>(d_own);
    const float4* r4 = reinterpret_cast<const float4*>(r);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 dv = d4[i];
        const float4 rv = r4[i];
        if (do_x) {
            float4 xv = x4[i];
            xv.x = fmaf(alpha_prev, dv.x, xv.x); xv.y = fmaf(alpha_prev, dv.y, xv.y);
            xv.z = fmaf(alpha_prev, dv.z, xv.z); xv.w = fmaf(alpha_prev, dv.w, xv.w);
            x4[i] = xv;
        }
        dv.x = fmaf(beta, dv.x, rv.x); dv.y = fmaf(beta, dv.y, rv.y);
        dv.z = fmaf(beta, dv.z, rv.z); dv.w = fmaf(beta, dv.w, rv.w);
        for (int q = 0; q < npeers; ++q) reinterpret_cast<float4*>(peers[q] + offset)[i] = dv;  // NVLink stores
    }
    for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float dv = d_own[i];
        if (do_x) x[i] = fmaf(alpha_prev, dv, x[i]);
        const float dn = fmaf(beta, dv, r[i]);
        for (int q = 0; q < npeers; ++q) peers[q][offset + i] = dn;
    }
    __threadfence_system();  // the stores are visible to the peers before the barrier that follows
}

__global__ void k_cgls_proj_dev_p2p(int64_t n, const float* __restrict__ e_own, const float* __restrict__ p,
                                    const double* __restrict__ S, double* __restrict__ partials,
                                    float* const* __restrict__ peers, int npeers, int64_t offset, int use4) {
    if (S[kSState] != 0.0) return;
    const float a = (float)(-S[kSAlpha]), b = 1.0f;
    const int64_t n4 = use4 ? n >> 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const float4* p4 = reinterpret_cast<const float4*>(p);
    const float4* e4 = reinterpret_cast<const float4*>(e_own);
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 yv = e4[i];
        const float4 xv = p4[i];
        yv.x = fmaf(a, xv.x, b * yv.x); yv.y = fmaf(a, xv.y, b * yv.y);
        yv.z = fmaf(a, xv.z, b * yv.z); yv.w = fmaf(a, xv.w, b * yv.w);
        for (int q = 0; q < npeers; ++q) reinterpret_cast<float4*>(peers[q] + offset)[i] = yv;
        sq += (double)yv.x * yv.x + (double)yv.y * yv.y + (double)yv.z * yv.z + (double)yv.w * yv.w;
    }
    for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float yv = fmaf(a, p[i], b * e_own[i]);
        for (int q = 0; q < npeers; ++q) peers[q][offset + i] = yv;
        sq += (double)yv * yv;
    }
    finish(sq, partials);
    __threadfence_system();
}

// sum of n per-rank values in index (rank) order: the host loop's `acc += v` sequence, on device
__global__ void k_sum_ranks(const double* __restrict__ vals, int n, double* __restrict__ out) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += vals[i];
    *out = acc;
}

__global__ void k_cgls_volume_dev(int64_t n, float* __restrict__ x, float* __restrict__ d,
                                  const float* __restrict__ r, const double* __restrict__ S, int use4) {
    if (S[kSState] != 0.0) return;
    const float alpha_prev = (float)S[kSAlpha], beta = (float)S[kSBeta];
    const int do_x = S[kSDoX] != 0.0;
    const int64_t n4 = use4 ? n >> 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float4* x4 = reinterpret_cast<float4*>(x);
    float4* d4 = reinterpret_cast<float4*>(d);
    const float4* r4 = reinterpret_cast<const float4*>(r);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 dv = d4[i];
        const float4 rv = r4[i];
        if (do_x) {
            float4 xv = x4[i];
            xv.x = fmaf(alpha_prev, dv.x, xv.x); xv.y = fmaf(alpha_prev, dv.y, xv.y);
            xv.z = fmaf(alpha_prev, dv.z, xv.z); xv.w = fmaf(alpha_prev, dv.w, xv.w);
            x4[i] = xv;
        }
        dv.x = fmaf(beta, dv.x, rv.x); dv.y = fmaf(beta, dv.y, rv.y);
        dv.z = fmaf(beta, dv.z, rv.z); dv.w = fmaf(beta, dv.w, rv.w);
        d4[i] = dv;
    }
    for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        if (do_x) x[i] = fmaf(alpha_prev, d[i], x[i]);
        d[i] = fmaf(beta, d[i], r[i]);
    }
}

// e -= alpha p with alpha = S[kSAlpha]; partials of e^2 (same arithmetic as k_axpby(-alpha, p, 1, e))
__global__ void k_cgls_proj_dev(int64_t n, float* __restrict__ e, const float* __restrict__ p,
                                const double* __restrict__ S, double* __restrict__ partials, int use4) {
    if (S[kSState] != 0.0) return;
    const float a = (float)(-S[kSAlpha]), b = 1.0f;
    const int64_t n4 = use4 ? n >> 2 : 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const float4* p4 = reinterpret_cast<const float4*>(p);
    float4* e4 = reinterpret_cast<float4*>(e);
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 yv = e4[i];
        const float4 xv = p4[i];
        yv.x = fmaf(a, xv.x, b * yv.x); yv.y = fmaf(a, xv.y, b * yv.y);
        yv.z = fmaf(a, xv.z, b * yv.z); yv.w = fmaf(a, xv.w, b * yv.w);
        e4[i] = yv;
        sq += (double)yv.x * yv.x + (double)yv.y * yv.y + (double)yv.z * yv.z + (double)yv.w * yv.w;
    }
    for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float yv = fmaf(a, p[i], b * e[i]);
        e[i] = yv;
        sq += (double)yv * yv;
    }
    finish(sq, partials);
}


// ---------------------------------------------------------------------------
// Device-resident LSQR (solvers.py:361-459, Golub-Kahan + Givens) with two fused vector passes
// per iteration.  u and v are kept unnormalised, u = uh / nu and v = vh / nv, so each
// normalisation folds into the next pass, and the Givens update of x and w (which needs the
// new v) is deferred into the next v pass:
//   U pass:  uh <- tmp_m / nv - (alpha / nu) uh            (= A v - alpha u), ||uh||^2
//   V pass:  x += a_x w ; w = vh / nv + a_w w               (previous iteration's update)
//            vh <- tmp_n / nu' - (beta / nv) vh             (= A^T u - beta v), sv = scale vh, ||vh||^2
// with tmp_m = A (scale vh) and tmp_n = scale A^T uh.  Scalars (fp64, one thread) between them.
enum : int {
    kLAlpha = 0, kLBeta = 1, kLRhobar = 2, kLPhibar = 3, kLNu = 4, kLNv = 5, kLAx = 6, kLAw = 7,
    kLPending = 8, kLU2 = 9, kLV2 = 10, kLState = 11, kLIter = 12, kLNb0 = 13, kLTol = 14, kLMax = 15,
    kLFinal = 16, kLHist = 24
};

__global__ void k_lsqr_u(int64_t n, float* __restrict__ uh, const float* __restrict__ tmp_m,
                         const double* __restrict__ S, double* __restrict__ partials) {
    if (S[kLState] != 0.0) return;
    const float c1 = (float)(1.0 / S[kLNv]), c2 = (float)(S[kLAlpha] / S[kLNu]);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float v = fmaf(tmp_m[i], c1, -c2 * uh[i]);
        uh[i] = v;
        sq += (double)v * v;
    }
    finish(sq, partials);
}

__global__ void k_lsqr_v(int64_t n, float* __restrict__ x, float* __restrict__ w, float* __restrict__ vh,
                         const float* __restrict__ tmp_n, float* __restrict__ sv, const float* __restrict__ scale,
                         const double* __restrict__ S, double* __restrict__ partials) {
    if (S[kLState] != 0.0) return;
    const bool pend = S[kLPending] != 0.0;
    const float ax = (float)S[kLAx], aw = (float)S[kLAw], inv_nv = (float)(1.0 / S[kLNv]);
    const float c1 = (float)(1.0 / S[kLNu]), c2 = (float)(S[kLBeta] / S[kLNv]);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float vo = vh[i];
        if (pend) {
            const float wv = w[i];
            x[i] = fmaf(ax, wv, x[i]);
            w[i] = fmaf(aw, wv, vo * inv_nv);
        }
        const float v = fmaf(tmp_n[i], c1, -c2 * vo);
        vh[i] = v;
        if (sv) sv[i] = scale[i] * v;
        sq += (double)v * v;
    }
    finish(sq, partials);
}

// x += a_x w (the deferred update of the last iteration); after a zero-beta breakdown also the
// final Givens step with the updated w, x += a_final (v + a_w w)
__global__ void k_lsqr_flush(int64_t n, float* __restrict__ x, const float* __restrict__ w,
                             const float* __restrict__ vh, const double* __restrict__ S) {
    if (S[kLPending] == 0.0) return;
    const float ax = (float)S[kLAx], aw = (float)S[kLAw], af = (float)S[kLFinal], inv_nv = (float)(1.0 / S[kLNv]);
    const bool fin = S[kLFinal] != 0.0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float wv = w[i];
        float xv = fmaf(ax, wv, x[i]);
        if (fin) xv = fmaf(af, fmaf(aw, wv, vh[i] * inv_nv), xv);
        x[i] = xv;
    }
}

// stage 1, after the U pass: beta, nu.  stage 2, after the V pass: alpha, nv, the Givens
// rotation (solvers.py:443-452), the deferred update's coefficients, the history record and the
// stop tests.  A zero beta or alpha (breakdown) stops the loop with the state the reference
// leaves: the final x update is pending (a_x) and applied by k_lsqr_flush.
__global__ void k_lsqr_scalars(double* __restrict__ S, int stage) {
    if (S[kLState] != 0.0) return;
    if (stage == 1) {
        const double beta = sqrt(S[kLU2]);
        S[kLBeta] = beta;
        S[kLNu] = beta;  // u = uh / beta from here on (the V pass divides A^T uh by it)
        if (beta == 0.0) {  // solvers.py:432-452 with beta = 0: alpha kept, Givens, then break
            const double rhobar = S[kLRhobar];
            const double rho = hypot(rhobar, 0.0);
            const double c = rhobar / rho;
            const double phi = c * S[kLPhibar];
            S[kLPhibar] = 0.0;
            S[kLFinal] = phi / rho;  // applied by k_lsqr_flush after the pending update (pending if it > 0)
            if (S[kLIter] == 0.0) {  // no earlier update pending: the final step alone
                S[kLAx] = 0.0;
                S[kLAw] = 0.0;
                S[kLPending] = 1.0;
            }
            const double it = S[kLIter];
            S[kLHist + (int)it] = 0.0;
            S[kLIter] = it + 1.0;
            S[kLState] = 1.0;
            return;
        }
        return;
    }
    const double alpha = sqrt(S[kLV2]), beta = S[kLBeta];
    const double rho = hypot(S[kLRhobar], beta);
    const double c = S[kLRhobar] / rho, s = beta / rho;
    const double theta = s * alpha;
    S[kLRhobar] = -c * alpha;
    const double phi = c * S[kLPhibar];
    S[kLPhibar] = s * S[kLPhibar];
    S[kLAx] = phi / rho;
    S[kLAw] = -(theta / rho);
    S[kLPending] = 1.0;
    S[kLAlpha] = alpha;
    S[kLNv] = alpha;
    const double it = S[kLIter];
    S[kLHist + (int)it] = S[kLPhibar];
    S[kLIter] = it + 1.0;
    const double nb0 = S[kLNb0];
    const double rel = nb0 > 0.0 ? S[kLPhibar] / nb0 : 0.0;
    if (alpha == 0.0) S[kLState] = 1.0;                          // breakdown (v stays 0)
    else if (S[kLTol] > 0.0 && rel <= S[kLTol]) S[kLState] = 2.0;  // converged
    else if (it + 1.0 >= S[kLMax]) S[kLState] = 3.0;               // budget (max_iterations + 1 updates)
}


// ---------------------------------------------------------------------------
// Device-resident SIRT / PSIRT (solvers.py:505-569): per iteration A^T w, one fused volume pass
// (x += step upd, or step_vec * upd for SIRT, then the box clip on the voxels), A x, one fused
// projection pass (r = b - A x, w = r / row sums for the next A^T, ||r||^2) and a one-thread
// scalar stage (history, tolerance and budget stops).  Same values as the host loop's
// mul / axpby / clip / sub kernels.
enum : int { kPR2 = 0, kPState = 1, kPIter = 2, kPNb0 = 3, kPTol = 4, kPMax = 5, kPHist = 8 };

__global__ void k_psirt_volume(int64_t n, int64_t zs, int64_t nz, float* __restrict__ x,
                               const float* __restrict__ upd, const float* __restrict__ step_vec, float step,
                               int clip, float lo, float hi, const double* __restrict__ S) {
    if (S[kPState] != 0.0) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        // SIRT: the product rounded on its own (__fmul_rn: no contraction), as the host loop's mul + axpby
        float xv = step_vec ? __fadd_rn(__fmul_rn(upd[i], step_vec[i]), x[i]) : fmaf(step, upd[i], 1.0f * x[i]);
        if (clip) {
            const int64_t k = i % zs;
            if (k >= CBCT_ZPAD && k < CBCT_ZPAD + nz) xv = fminf(fmaxf(xv, lo), hi);
        }
        x[i] = xv;
    }
}

__global__ void k_psirt_proj(int64_t m, float* __restrict__ r, float* __restrict__ w, const float* __restrict__ b,
                             const float* __restrict__ p, const float* __restrict__ inv_row,
                             const double* __restrict__ S, double* __restrict__ partials) {
    if (S[kPState] != 0.0) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    double sq = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += stride) {
        const float rv = b[i] - p[i];
        r[i] = rv;
        w[i] = rv * inv_row[i];
        sq += (double)rv * rv;
    }
    finish(sq, partials);
}

__global__ void k_psirt_scalars(double* __restrict__ S) {
    if (S[kPState] != 0.0) return;
    const double nb0 = S[kPNb0];
    const double e = nb0 > 0.0 ? sqrt(S[kPR2]) / nb0 : 0.0;
    const double it = S[kPIter] + 1.0;
    S[kPIter] = it;
    S[kPHist + (int)it] = e;
    if (S[kPTol] > 0.0 && e <= S[kPTol]) S[kPState] = 2.0;
    else if (it >= S[kPMax]) S[kPState] = 3.0;
}

}  // namespace

extern "C" int cbct_vec_blocks(int64_t n) { return vec_blocks(n); }

extern "C" int cbct_cgls_volume_update(int64_t n, float* x, float* d, const float* r, double alpha_prev, int do_x,
                                       double beta, void* stream) {
    if (!d || !r || (do_x && !x)) return cbct_fail(CBCT_E_ARG, "cbct_cgls_volume_update: null argument");
    const int use4 = aligned16(x) && aligned16(d) && aligned16(r);
    k_cgls_volume<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, d, r, (float)alpha_prev, do_x,
                                                                       (float)beta, use4);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_axpby(int64_t n, double a, const float* x, double b, float* y, double* partials,
                          void* stream) {
    if (!y) return cbct_fail(CBCT_E_ARG, "cbct_axpby: null y");
    const int use4 = aligned16(x) && aligned16(y);
    k_axpby<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, (float)a, x, (float)b, y, partials, use4);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_cgls_proj_update(int64_t n, float* e, const float* p, double alpha, double* partials,
                                     void* stream) {
    // e -= alpha*p  ==  axpby(-alpha, p, 1, e)
    return cbct_axpby(n, -alpha, p, 1.0, e, partials, stream);
}

extern "C" int cbct_sub(int64_t n, const float* a, const float* b, float* out, double* partials, void* stream) {
    if (!a || !b || !out) return cbct_fail(CBCT_E_ARG, "cbct_sub: null argument");
    k_sub<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, a, b, out, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_dot(int64_t n, const float* x, const float* y, double* partials, void* stream) {
    if (!x || !y || !partials) return cbct_fail(CBCT_E_ARG, "cbct_dot: null argument");
    k_dot<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, y, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_mul(int64_t n, const float* a, const float* b, float* out, void* stream) {
    if (!a || !b || !out) return cbct_fail(CBCT_E_ARG, "cbct_mul: null argument");
    k_mul<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, a, b, out);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_fill(int64_t n, float* x, float value, void* stream) {
    if (!x) return cbct_fail(CBCT_E_ARG, "cbct_fill: null argument");
    k_fill<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, value);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_fill_volume(const cbct_plan* p, float* vol, float value, void* stream) {
    if (!p || !vol) return cbct_fail(CBCT_E_ARG, "cbct_fill_volume: null argument");
    k_fill_volume<<<vec_blocks(p->vol_elems), kThreads, 0, (cudaStream_t)stream>>>(p->vol_elems, p->zs, p->nz, vol,
                                                                                   value);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_clip(const cbct_plan* p, float* vol, float lo, float hi, void* stream) {
    if (!p || !vol) return cbct_fail(CBCT_E_ARG, "cbct_clip: null argument");
    k_clip<<<vec_blocks(p->vol_elems), kThreads, 0, (cudaStream_t)stream>>>(p->vol_elems, p->zs, p->nz, vol, lo, hi);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_reduce_partials(const double* partials, int32_t n, double* dev_out, double* host_out,
                                    void* stream) {
    if (!partials || !dev_out || n < 1) return cbct_fail(CBCT_E_ARG, "cbct_reduce_partials: bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    k_reduce<<<1, 1024, 0, s>>>(partials, n, dev_out);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    if (host_out) {
        CBCT_CHECK(cudaMemcpyAsync(host_out, dev_out, sizeof(double), cudaMemcpyDeviceToHost, s));
        CBCT_CHECK(cudaStreamSynchronize(s));
    }
    return 0;
}

extern "C" int cbct_cgls_scalars(double* scalars, int stage, void* stream) {
    if (!scalars || stage < 1 || stage > 3) return cbct_fail(CBCT_E_ARG, "cbct_cgls_scalars: bad argument");
    k_cgls_scalars<<<1, 1, 0, (cudaStream_t)stream>>>(scalars, stage);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_cgls_volume_update_dev(int64_t n, float* x, float* d, const float* r, const double* scalars,
                                           void* stream) {
    if (!x || !d || !r || !scalars) return cbct_fail(CBCT_E_ARG, "cbct_cgls_volume_update_dev: null argument");
    const int use4 = aligned16(x) && aligned16(d) && aligned16(r);
    k_cgls_volume_dev<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, d, r, scalars, use4);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_cgls_proj_update_dev(int64_t n, float* e, const float* p, const double* scalars,
                                         double* partials, void* stream) {
    if (!e || !p || !scalars) return cbct_fail(CBCT_E_ARG, "cbct_cgls_proj_update_dev: null argument");
    const int use4 = aligned16(e) && aligned16(p);
    k_cgls_proj_dev<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, e, p, scalars, partials, use4);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_sum_ranks(const double* vals, int n, double* out, void* stream) {
    if (!vals || !out || n < 1) return cbct_fail(CBCT_E_ARG, "cbct_sum_ranks: bad argument");
    k_sum_ranks<<<1, 1, 0, (cudaStream_t)stream>>>(vals, n, out);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_cgls_volume_update_p2p(int64_t n, float* x, const float* d_own, const float* r,
                                           const double* scalars, float* const* peers, int npeers, int64_t offset,
                                           void* stream) {
    if (!x || !d_own || !r || !scalars || !peers || npeers < 1)
        return cbct_fail(CBCT_E_ARG, "cbct_cgls_volume_update_p2p: bad argument");
    // float4 body only when every rank's slab is 16-B aligned (peer bases are allocation-aligned)
    const int use4 = aligned16(x) && aligned16(d_own) && aligned16(r) && (offset & 3) == 0;
    k_cgls_volume_dev_p2p<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, d_own, r, scalars, peers,
                                                                                npeers, offset, use4);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_cgls_proj_update_p2p(int64_t n, const float* e_own, const float* p, const double* scalars,
                                         double* partials, float* const* peers, int npeers, int64_t offset,
                                         void* stream) {
    if (!e_own || !p || !scalars || !peers || npeers < 1)
        return cbct_fail(CBCT_E_ARG, "cbct_cgls_proj_update_p2p: bad argument");
    const int use4 = aligned16(e_own) && aligned16(p) && (offset & 3) == 0;
    k_cgls_proj_dev_p2p<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, e_own, p, scalars, partials, peers,
                                                                              npeers, offset, use4);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_lsqr_u_update(int64_t n, float* uh, const float* tmp_m, const double* scalars,
                                  double* partials, void* stream) {
    if (!uh || !tmp_m || !scalars) return cbct_fail(CBCT_E_ARG, "cbct_lsqr_u_update: null argument");
    k_lsqr_u<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, uh, tmp_m, scalars, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_lsqr_v_update(int64_t n, float* x, float* w, float* vh, const float* tmp_n, float* sv,
                                  const float* scale, const double* scalars, double* partials, void* stream) {
    if (!x || !w || !vh || !tmp_n || !scalars || (sv && !scale))
        return cbct_fail(CBCT_E_ARG, "cbct_lsqr_v_update: bad argument");
    k_lsqr_v<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, w, vh, tmp_n, sv, scale, scalars, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_lsqr_flush(int64_t n, float* x, const float* w, const float* vh, const double* scalars,
                               void* stream) {
    if (!x || !w || !vh || !scalars) return cbct_fail(CBCT_E_ARG, "cbct_lsqr_flush: null argument");
    k_lsqr_flush<<<vec_blocks(n), kThreads, 0, (cudaStream_t)stream>>>(n, x, w, vh, scalars);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_lsqr_scalars(double* scalars, int stage, void* stream) {
    if (!scalars || stage < 1 || stage > 2) return cbct_fail(CBCT_E_ARG, "cbct_lsqr_scalars: bad argument");
    k_lsqr_scalars<<<1, 1, 0, (cudaStream_t)stream>>>(scalars, stage);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_psirt_volume_update(const cbct_plan* p, float* x, const float* upd, const float* step_vec,
                                        float step, int clip, float lo, float hi, const double* scalars,
                                        void* stream) {
    if (!p || !x || !upd || !scalars) return cbct_fail(CBCT_E_ARG, "cbct_psirt_volume_update: null argument");
    k_psirt_volume<<<vec_blocks(p->vol_elems), kThreads, 0, (cudaStream_t)stream>>>(
        p->vol_elems, p->zs, p->nz, x, upd, step_vec, step, clip, lo, hi, scalars);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_psirt_proj_update(int64_t m, float* r, float* w, const float* b, const float* p,
                                      const float* inv_row, const double* scalars, double* partials, void* stream) {
    if (!r || !w || !b || !p || !inv_row || !scalars) return cbct_fail(CBCT_E_ARG, "cbct_psirt_proj_update: null argument");
    k_psirt_proj<<<vec_blocks(m), kThreads, 0, (cudaStream_t)stream>>>(m, r, w, b, p, inv_row, scalars, partials);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_psirt_scalars(double* scalars, void* stream) {
    if (!scalars) return cbct_fail(CBCT_E_ARG, "cbct_psirt_scalars: null argument");
    k_psirt_scalars<<<1, 1, 0, (cudaStream_t)stream>>>(scalars);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}
