// phantom.cu -- GPU voxelizer for the ellipsoid phantom.
//
// Restates generate_phantom (phantom.py:87-106): each voxel is the sum of the
// intensities of the ellipsoids that contain its centre, point-sampled on the
// normalised cube (phantom.py:78-84: c = (2 k + 1 - n) / n per axis).  The
// membership test is evaluated in fp64 in numpy's operation order with explicit
// round-to-nearest intrinsics (no FMA contraction), using the rotation matrices the
// host computes with the reference's own expressions, so every inside/outside
// decision -- and therefore every voxel -- is bit-identical to the host generator.
// The fp64 sum is rounded once to fp32 (exact for the dyadic Shepp-Logan table).
//
// The host generator materialises several full-size fp64 temporaries per
// ellipsoid (8.6 GB each at 1024^3); this writes the solver's device layout
// directly, guard slices included, at one pass over the volume.
#include "cbct_internal.cuh"

namespace {

constexpr int kEllWords = 16;  // cx cy cz  a b c  R00 R01 R02 R10 R11 R12 R20 R21 R22  intensity

__device__ __forceinline__ double axis_centre(int k, int n) {  // phantom.py:81-83
    return __ddiv_rn((double)(2 * k + 1 - n), (double)n);
}

__device__ __forceinline__ double ellipsoid_sum(const double* __restrict__ e, int n_ell, double X, double Y,
                                                double Z) {
    double out = 0.0;
    for (int k = 0; k < n_ell; ++k, e += kEllWords) {
        const double dx = __dsub_rn(X, e[0]), dy = __dsub_rn(Y, e[1]), dz = __dsub_rn(Z, e[2]);
        // (R[i,0] dx + R[i,1] dy + R[i,2] dz) / semi_axes[i], left to right (phantom.py:100-102)
        const double px = __ddiv_rn(__dadd_rn(__dadd_rn(__dmul_rn(e[6], dx), __dmul_rn(e[7], dy)), __dmul_rn(e[8], dz)),
                                    e[3]);
        const double py = __ddiv_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(e[9], dx), __dmul_rn(e[10], dy)), __dmul_rn(e[11], dz)), e[4]);
        const double pz = __ddiv_rn(
            __dadd_rn(__dadd_rn(__dmul_rn(e[12], dx), __dmul_rn(e[13], dy)), __dmul_rn(e[14], dz)), e[5]);
        const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(pz, pz));
        out = __dadd_rn(out, r2 <= 1.0 ? e[15] : 0.0);  // phantom.py:103-105
    }
    return out;
}

// device layout [ny][nx][zs], z fastest, zero guard slices
__global__ void k_phantom_internal(const double* __restrict__ ell, int n_ell, int nx, int ny, int nz, int zs,
                                   float* __restrict__ vol) {
    const int64_t total = (int64_t)ny * nx * zs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int zi = (int)(i % zs);
        const int64_t cell = i / zs;
        const int ix = (int)(cell % nx), iy = (int)(cell / nx);
        const int iz = zi - CBCT_ZPAD;
        float v = 0.0f;
        if (iz >= 0 && iz < nz)
            v = (float)ellipsoid_sum(ell, n_ell, axis_centre(ix, nx), axis_centre(iy, ny), axis_centre(iz, nz));
        vol[i] = v;
    }
}

// reference layout (nz, ny, nx), x fastest (phantom.py:72-75); T = float or double
template <typename T>
__global__ void k_phantom_ref(const double* __restrict__ ell, int n_ell, int nx, int ny, int nz,
                              T* __restrict__ out) {
    const int64_t total = (int64_t)nz * ny * nx;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int ix = (int)(i % nx);
        const int64_t r = i / nx;
        const int iy = (int)(r % ny), iz = (int)(r / ny);
        out[i] = (T)ellipsoid_sum(ell, n_ell, axis_centre(ix, nx), axis_centre(iy, ny), axis_centre(iz, nz));
    }
}

unsigned grid_for(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (unsigned)(b < 148 * 64 ? (b > 0 ? b : 1) : 148 * 64);  // grid-stride beyond 64 CTAs per SM
}

}  // namespace

extern "C" int cbct_phantom(const cbct_plan* p, const double* ellipsoids, int n_ell, float* vol, void* stream) {
    if (!p || !vol || (n_ell > 0 && !ellipsoids) || n_ell < 0)
        return cbct_fail(CBCT_E_ARG, "cbct_phantom: null argument or negative count");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    k_phantom_internal<<<grid_for(p->ny * p->nx * p->zs), 256, 0, s>>>(ellipsoids, n_ell, (int)p->nx, (int)p->ny,
                                                                       (int)p->nz, (int)p->zs, vol);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch(1);
    return 0;
}

template <typename T>
int phantom_ref(int64_t nx, int64_t ny, int64_t nz, const double* ellipsoids, int n_ell, T* out, void* stream) {
    if (nx <= 0 || ny <= 0 || nz <= 0 || nx > INT32_MAX || ny > INT32_MAX || nz > INT32_MAX)
        return cbct_fail(CBCT_E_ARG, "cbct_phantom_ref: bad dimensions");
    if (!out || (n_ell > 0 && !ellipsoids) || n_ell < 0)
        return cbct_fail(CBCT_E_ARG, "cbct_phantom_ref: null argument or negative count");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    k_phantom_ref<T><<<grid_for(nx * ny * nz), 256, 0, s>>>(ellipsoids, n_ell, (int)nx, (int)ny, (int)nz, out);
    CBCT_CHECK(cudaGetLastError());
    cbct_count_launch(1);
    return 0;
}

extern "C" int cbct_phantom_ref(int64_t nx, int64_t ny, int64_t nz, const double* ellipsoids, int n_ell, float* out,
                                void* stream) {
    return phantom_ref<float>(nx, ny, nz, ellipsoids, n_ell, out, stream);
}

extern "C" int cbct_phantom_ref_f64(int64_t nx, int64_t ny, int64_t nz, const double* ellipsoids, int n_ell,
                                    double* out, void* stream) {
    return phantom_ref<double>(nx, ny, nz, ellipsoids, n_ell, out, stream);
}
