// reduce.cuh -- deterministic block reductions (fixed shuffle tree, fixed warp order).
#pragma once
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Sum over the whole block; valid in thread 0.  All threads must call it.
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double s_warp[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();  // protect s_warp reuse across consecutive calls
    if (lane == 0) s_warp[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    double t = 0.0;
    if (wid == 0) {
        t = lane < nw ? s_warp[lane] : 0.0;
        t = warp_sum(t);
    }
    return t;
}
