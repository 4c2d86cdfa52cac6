// scan.cu -- the library's own device scan and stable key sort (load time, A0).
//
// Replaces the cub::DeviceScan / cub::DeviceRadixSort calls round 1 used in the
// hub sort: everything on the load path is now this library's code.
//
//   exclusive_scan   out[i] = sum_{j<i} in[j]   (u32 -> u32, u32 -> u64, u64 -> u64)
//                    three launches: per-CTA sums, one CTA scans the sums, per-CTA
//                    scan with its carry.  2048 items per CTA (256 threads x 8).
//   sort_desc_stable (key u64, val u32) pairs by key DESCENDING, equal keys keeping
//                    their input order: one stable split per key bit from the
//                    least significant up (LSD radix sort with 1-bit digits), each
//                    split = a scan of the "bit is 0" flags + a scatter.  Only the
//                    bits below the highest set bit of the largest key are split.
//                    Used on the h = ceil(0.08 V) hubs only (3.3 M on TW).
#include "graph.h"
#include "block_prims.cuh"
#include "scan.h"

namespace hyt {

constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

template <class In>
__global__ void __launch_bounds__(kScanThreads) k_scan_sums(const In *__restrict__ in, uint64_t n,
                                                             uint64_t *__restrict__ sums) {
    __shared__ uint64_t sh[33];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + (uint64_t)k * kScanThreads + threadIdx.x;
        if (i < n) s += (uint64_t)in[i];
    }
    s = block_sum_u64(s, sh);
    if (threadIdx.x == 0) sums[blockIdx.x] = s;
}

// one CTA: exclusive scan of the nb per-CTA sums in place
__global__ void __launch_bounds__(kScanThreads) k_scan_carry(uint64_t *__restrict__ sums, uint64_t nb) {
    __shared__ uint64_t sh[33];
    uint64_t carry = 0;
    for (uint64_t b0 = 0; b0 < nb; b0 += kScanThreads) {
        const uint64_t i = b0 + threadIdx.x;
        const uint64_t x = i < nb ? sums[i] : 0;
        uint64_t tot;
        const uint64_t ex = block_exscan_u64(x, sh, &tot);
        if (i < nb) sums[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
}

// per CTA: thread t owns items [t*8, t*8+8) of the tile (blocked), scans them
// serially, then one block scan of the per-thread totals
template <class In, class Out>
__global__ void __launch_bounds__(kScanThreads) k_scan_tiles(const In *__restrict__ in, Out *__restrict__ out,
                                                              uint64_t n, const uint64_t *__restrict__ carry) {
    __shared__ uint64_t sh[33];
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
    uint64_t v[kScanItems];
    uint64_t s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + k;
        v[k] = i < n ? (uint64_t)in[i] : 0;
        s += v[k];
    }
    uint64_t tot;
    uint64_t run = carry[blockIdx.x] + block_exscan_u64(s, sh, &tot);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const uint64_t i = base + k;
        if (i < n) out[i] = (Out)run;
        run += v[k];
    }
}

uint64_t scan_temp_bytes(uint64_t n) { return ((n + kScanTile - 1) / kScanTile + 1) * 8; }

template <class In, class Out>
void exclusive_scan(const In *in, Out *out, uint64_t n, void *temp, cudaStream_t st) {
    if (n == 0) return;
    const uint64_t nb = (n + kScanTile - 1) / kScanTile;
    uint64_t *sums = (uint64_t *)temp;
    k_scan_sums<In><<<(unsigned)nb, kScanThreads, 0, st>>>(in, n, sums);
    k_scan_carry<<<1, kScanThreads, 0, st>>>(sums, nb);
    k_scan_tiles<In, Out><<<(unsigned)nb, kScanThreads, 0, st>>>(in, out, n, sums);
}
template void exclusive_scan<uint32_t, uint32_t>(const uint32_t *, uint32_t *, uint64_t, void *, cudaStream_t);
template void exclusive_scan<uint32_t, uint64_t>(const uint32_t *, uint64_t *, uint64_t, void *, cudaStream_t);
template void exclusive_scan<uint64_t, uint64_t>(const uint64_t *, uint64_t *, uint64_t, void *, cudaStream_t);

// ---------------------------------------------------------------------------
// stable descending sort by 1-bit splits
// ---------------------------------------------------------------------------
__global__ void k_key_max(const uint64_t *__restrict__ key, uint64_t n, unsigned long long *__restrict__ mx) {
    __shared__ unsigned long long sm;
    if (threadIdx.x == 0) sm = 0;
    __syncthreads();
    unsigned long long m = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) m = max(m, (unsigned long long)key[i]);
    atomicMax(&sm, m);
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(mx, sm);
}

// flag = 1 for keys whose bit is 0 (they go AFTER the ones: descending order)
__global__ void k_bit_flags(const uint64_t *__restrict__ key, uint64_t n, int bit, uint32_t *__restrict__ zero) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        zero[i] = ((key[i] >> bit) & 1ull) ? 0u : 1u;
}

// stable split: ones first in input order, then zeros in input order.
// zpos = exclusive scan of the zero flags; nzero = their total.
__global__ void k_bit_scatter(const uint64_t *__restrict__ key, const uint32_t *__restrict__ val, uint64_t n,
                              const uint32_t *__restrict__ zero, const uint32_t *__restrict__ zpos,
                              uint64_t *__restrict__ key2, uint32_t *__restrict__ val2) {
    const uint64_t nzero = (uint64_t)zpos[n - 1] + zero[n - 1], nones = n - nzero;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t p = zero[i] ? nones + zpos[i] : i - zpos[i];
        key2[p] = key[i];
        val2[p] = val[i];
    }
}

void sort_desc_stable(uint64_t *key, uint32_t *val, uint64_t *key2, uint32_t *val2, uint64_t n, uint32_t *flags,
                      uint32_t *pos, void *scan_temp, unsigned long long *mx_dev, cudaStream_t st) {
    if (n < 2) return;
    unsigned grid = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms() * 16);
    HYT_CUDA(cudaMemsetAsync(mx_dev, 0, 8, st));
    k_key_max<<<grid, 256, 0, st>>>(key, n, mx_dev);
    unsigned long long mx = 0;
    HYT_CUDA(copy_sync(&mx, mx_dev, 8, st));
    int bits = 0;
    while (bits < 64 && (mx >> bits)) ++bits;
    uint64_t *ka = key, *kb = key2;
    uint32_t *va = val, *vb = val2;
    for (int b = 0; b < bits; ++b) {
        k_bit_flags<<<grid, 256, 0, st>>>(ka, n, b, flags);
        exclusive_scan<uint32_t, uint32_t>(flags, pos, n, scan_temp, st);
        k_bit_scatter<<<grid, 256, 0, st>>>(ka, va, n, flags, pos, kb, vb);
        std::swap(ka, kb);
        std::swap(va, vb);
    }
    if (ka != key) {   // odd number of passes: the result is in the second buffers
        HYT_CUDA(cudaMemcpyAsync(key, ka, n * 8, cudaMemcpyDeviceToDevice, st));
        HYT_CUDA(cudaMemcpyAsync(val, va, n * 4, cudaMemcpyDeviceToDevice, st));
    }
    HYT_CUDA(cudaGetLastError());
}

}  // namespace hyt
