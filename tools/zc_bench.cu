// zc_bench.cu -- zero-copy read throughput vs request size on this box (the Fig. 3e
// analog of the paper): the host-link denominator for the
// zero-copy engine and a sanity check of the cost model's gamma.
//
// A warp issues requests of S bytes (S = 32, 64, 96, 128) at random 128-byte-aligned
// positions of a 4 GiB pinned, mapped host buffer; lanes read 16 B each (S/16 lanes
// per request).  Throughput = requested bytes / kernel time.  Also reports the
// pinned cudaMemcpy H2D rate and the contiguous 512-B-per-warp zero-copy stream rate.
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdint>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

template <int S>
__global__ void k_zc(const uint4 *__restrict__ host, uint64_t nlines, uint64_t reqs_per_warp, uint32_t *sink) {
    constexpr int LPR = S / 16;                 // lanes per request
    constexpr int RPW = 32 / LPR;               // requests per warp instruction
    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    uint32_t acc = 0;
    for (uint64_t i = 0; i < reqs_per_warp; i += RPW * 4) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t req = i + u * RPW + lane / LPR;
            const uint64_t line = mix(warp * 1000003ull + req) % nlines;
            v[u] = lane < RPW * LPR ? host[line * 8 + (lane % LPR)] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_stream(const uint4 *__restrict__ host, uint64_t n16, uint32_t *sink) {
    uint32_t acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) acc ^= host[i].x;
    if (acc == 0x12345678u) *sink = acc;
}

template <int S>
static double run(const uint4 *dev, uint64_t nlines, uint32_t *sink, int blocks) {
    const uint64_t reqs = 1 << 14;              // per warp
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_zc<S><<<blocks, 256>>>(dev, nlines, reqs / 8, sink);
    cudaEventRecord(a);
    k_zc<S><<<blocks, 256>>>(dev, nlines, reqs, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)blocks * 8 * reqs * S;
    return bytes / (ms / 1e3) / 1e9;
}

int main() {
    const uint64_t bytes = 4ull << 30;
    void *h = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    madvise(h, bytes, MADV_HUGEPAGE);
    memset(h, 1, bytes);
    cudaHostRegister(h, bytes, cudaHostRegisterMapped);
    uint4 *dev = nullptr;
    cudaHostGetDevicePointer((void **)&dev, h, 0);
    uint32_t *sink;
    cudaMalloc(&sink, 4);
    void *d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(a);
    cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double memcpy_gbs = bytes / (ms / 1e3) / 1e9;
    cudaEventRecord(a);
    k_stream<<<148 * 4, 256>>>(dev, bytes / 16, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    const double stream_gbs = bytes / (ms / 1e3) / 1e9;
    const uint64_t nlines = bytes / 128;
    printf("{\"memcpy_h2d_gbs\": %.2f, \"zc_stream_gbs\": %.2f, \"zc_random_request_gbs\": {", memcpy_gbs, stream_gbs);
    for (int blocks : {148 * 2, 148 * 8}) {
        printf("\"blocks_%d\": {\"32\": %.2f, \"64\": %.2f, \"96\": %.2f, \"128\": %.2f}%s", blocks,
               run<32>(dev, nlines, sink, blocks), run<64>(dev, nlines, sink, blocks),
               run<96>(dev, nlines, sink, blocks), run<128>(dev, nlines, sink, blocks),
               blocks == 148 * 2 ? ", " : "");
    }
    printf("}, \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
