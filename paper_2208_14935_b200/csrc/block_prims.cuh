// block_prims.cuh -- warp/block reductions and scans used by the plan and relax kernels.
#pragma once
#include <cstdint>

namespace hyt {

#define FULL_MASK 0xFFFFFFFFu

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL_MASK, x, o);
    return x;
}
__device__ __forceinline__ double warp_sum_f64(double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL_MASK, x, o);
    return x;
}
// inclusive warp scan
__device__ __forceinline__ uint64_t warp_incl_u64(uint64_t x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(FULL_MASK, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

// Block-wide sum; every thread gets the result.  `sh` needs 32 slots.
__device__ __forceinline__ uint64_t block_sum_u64(uint64_t x, uint64_t *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    x = warp_sum_u64(x);
    __syncthreads();
    if (lane == 0) sh[wid] = x;
    __syncthreads();
    uint64_t y = lane < nw ? sh[lane] : 0;
    return warp_sum_u64(y);
}
__device__ __forceinline__ double block_sum_f64(double x, double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    x = warp_sum_f64(x);
    __syncthreads();
    if (lane == 0) sh[wid] = x;
    __syncthreads();
    double y = lane < nw ? sh[lane] : 0.0;
    return warp_sum_f64(y);
}

// Block-wide exclusive scan of u64; returns the exclusive prefix, *total = sum.
// `sh` needs 33 slots.
__device__ __forceinline__ uint64_t block_exscan_u64(uint64_t x, uint64_t *sh, uint64_t *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint64_t inc = warp_incl_u64(x);
    __syncthreads();
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const uint64_t s = lane < nw ? sh[lane] : 0;
        const uint64_t si = warp_incl_u64(s);
        if (lane < nw) sh[lane] = si - s;
        if (lane == 31) sh[32] = si;
    }
    __syncthreads();
    const uint64_t r = sh[wid] + inc - x;
    *total = sh[32];
    return r;
}

// Bits of bitmap word w that lie in [vlo, vhi).
__device__ __forceinline__ uint32_t range_mask(uint64_t w, uint64_t vlo, uint64_t vhi) {
    const uint64_t base = w << 5;
    uint32_t m = FULL_MASK;
    if (base < vlo) m &= (vlo - base >= 32) ? 0u : (FULL_MASK << (uint32_t)(vlo - base));
    if (base + 32 > vhi) {
        const uint64_t n = vhi > base ? vhi - base : 0;
        m &= n >= 32 ? FULL_MASK : ((1u << (uint32_t)n) - 1u);
    }
    return m;
}

// Zero-copy requests of one vertex (Eq. 3 per-vertex term): ceil(len/m) + am(v)
// equals the number of m-byte lines its span touches (P:368 footnote).
__device__ __forceinline__ uint64_t zc_lines(uint64_t start, uint64_t len, uint64_t m) {
    if (len == 0) return 0;
    return (start + len - 1) / m - start / m + 1;
}

}  // namespace hyt
