// layout.cu -- reference layouts <-> internal layouts (HBM-bound tiled transposes).
//
// volume:      reference (nz, ny, nx) x-fastest (phantom.py:55-75)  <->  internal [ny*nx][zs] z-fastest
// projections: reference (V, nv, nu) u-fastest (operator.py:30-50)   <->  internal [V][nu][nv] v-fastest
// Both are batched 2-D transposes of a (R x C) row-major matrix into (C x R)
// with an output row stride, done through a 32x33 shared-memory tile so that
// reads and writes are both coalesced.
#include "cbct_internal.cuh"

namespace {

constexpr int T = 32;

// out[b][c*ostride + ooff + r] = in[b][r*C + c]
template <typename Tin, typename Tout>
__global__ void k_transpose(const Tin* __restrict__ in, Tout* __restrict__ out, int64_t R, int64_t C,
                            int64_t ostride, int64_t ooff, int64_t in_batch, int64_t out_batch) {
    __shared__ float tile[T][T + 1];
    const int64_t b = blockIdx.z;
    const int64_t r0 = (int64_t)blockIdx.y * T, c0 = (int64_t)blockIdx.x * T;
    const Tin* ib = in + b * in_batch;
    Tout* ob = out + b * out_batch;
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < R && c < C) tile[i][threadIdx.x] = (float)ib[r * C + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < R && c < C) ob[c * ostride + ooff + r] = (Tout)tile[threadIdx.x][i];
    }
}

// out[b][r*C + c] = in[b][c*istride + ioff + r]   (inverse of the above)
template <typename Tin, typename Tout>
__global__ void k_transpose_back(const Tin* __restrict__ in, Tout* __restrict__ out, int64_t R, int64_t C,
                                 int64_t istride, int64_t ioff, int64_t in_batch, int64_t out_batch) {
    __shared__ float tile[T][T + 1];
    const int64_t b = blockIdx.z;
    const int64_t r0 = (int64_t)blockIdx.y * T, c0 = (int64_t)blockIdx.x * T;
    const Tin* ib = in + b * in_batch;
    Tout* ob = out + b * out_batch;
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < R && c < C) tile[threadIdx.x][i] = (float)ib[c * istride + ioff + r];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < T; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < R && c < C) ob[r * C + c] = (Tout)tile[i][threadIdx.x];
    }
}

__global__ void k_zero_guards(float* vol, int64_t n_cells, int64_t zs, int64_t nz) {
    const int64_t ng = zs - nz;  // guard slots per cell column
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n_cells * ng) return;
    const int64_t cell = i / ng;
    const int64_t k = i - cell * ng;
    vol[cell * zs + (k < CBCT_ZPAD ? k : nz + k)] = 0.0f;
}

template <typename Tin, typename Tout>
int launch_t(const Tin* in, Tout* out, int64_t R, int64_t C, int64_t ostride, int64_t ooff, int64_t nb,
             int64_t in_batch, int64_t out_batch, cudaStream_t s) {
    dim3 grid((unsigned)((C + T - 1) / T), (unsigned)((R + T - 1) / T), (unsigned)nb);
    k_transpose<Tin, Tout><<<grid, dim3(T, 8), 0, s>>>(in, out, R, C, ostride, ooff, in_batch, out_batch);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

template <typename Tin, typename Tout>
int launch_tb(const Tin* in, Tout* out, int64_t R, int64_t C, int64_t istride, int64_t ioff, int64_t nb,
              int64_t in_batch, int64_t out_batch, cudaStream_t s) {
    dim3 grid((unsigned)((C + T - 1) / T), (unsigned)((R + T - 1) / T), (unsigned)nb);
    k_transpose_back<Tin, Tout><<<grid, dim3(T, 8), 0, s>>>(in, out, R, C, istride, ioff, in_batch, out_batch);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

}  // namespace

extern "C" int cbct_volume_to_internal(const cbct_plan* p, const void* src, int f64, float* dst, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_volume_to_internal: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t cells = p->n_cells;
    int rc = f64 ? launch_t((const double*)src, dst, p->nz, cells, p->zs, CBCT_ZPAD, 1, 0, 0, s)
                 : launch_t((const float*)src, dst, p->nz, cells, p->zs, CBCT_ZPAD, 1, 0, 0, s);
    if (rc) return rc;
    const int64_t ng = cells * (p->zs - p->nz);
    k_zero_guards<<<(unsigned)((ng + 255) / 256), 256, 0, s>>>(dst, cells, p->zs, p->nz);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch();
    return 0;
}

extern "C" int cbct_volume_from_internal(const cbct_plan* p, const float* src, void* dst, int f64, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_volume_from_internal: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    return f64 ? launch_tb(src, (double*)dst, p->nz, p->n_cells, p->zs, CBCT_ZPAD, 1, 0, 0, s)
               : launch_tb(src, (float*)dst, p->nz, p->n_cells, p->zs, CBCT_ZPAD, 1, 0, 0, s);
}

extern "C" int cbct_proj_to_internal(const cbct_plan* p, const void* src, int f64, float* dst, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_proj_to_internal: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t per = p->nu * p->nv;
    return f64 ? launch_t((const double*)src, dst, p->nv, p->nu, p->nv, 0, p->V, per, per, s)
               : launch_t((const float*)src, dst, p->nv, p->nu, p->nv, 0, p->V, per, per, s);
}

extern "C" int cbct_proj_from_internal(const cbct_plan* p, const float* src, void* dst, int f64, void* stream) {
    if (!p || !src || !dst) return cbct_fail(CBCT_E_ARG, "cbct_proj_from_internal: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t per = p->nu * p->nv;
    return f64 ? launch_tb(src, (double*)dst, p->nv, p->nu, p->nv, 0, p->V, per, per, s)
               : launch_tb(src, (float*)dst, p->nv, p->nu, p->nv, 0, p->V, per, per, s);
}
