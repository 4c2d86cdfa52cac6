// dsmem_bench.cu -- could a hub block spread over a thread-block cluster's distributed
// shared memory carry PR reductions beside the L2 (whose reduction rate is 188-194
// G/s, tools/red_ceiling.cu)?  Measures random f32 / u32 reductions into the
// cluster's shared memory (red.shared::cluster), local-only shared memory, and a
// mix of one DSMEM and one L2 reduction per element, for cluster sizes 1-16.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint32_t cluster_rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t cluster_n() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) {
    uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}

constexpr int S = 40960;   // floats per CTA (160 KB)

// MODE 0: f32 red into the cluster (random rank, random slot)
// MODE 1: u32 red into the cluster
// MODE 2: f32 atomicAdd into the CTA's own shared memory (CAS loop on sm_100a)
// MODE 3: u32 atomicAdd into the CTA's own shared memory
// MODE 4: one f32 cluster red + one L2 red per element
// MODE 5: one L2 red per element only (same grid; the reference)
template <int MODE>
__global__ void k(float *g, uint32_t Vg, uint64_t n, uint32_t seed) {
    extern __shared__ float sm[];
    for (int i = threadIdx.x; i < S; i += blockDim.x) sm[i] = 0.f;
    cluster_sync();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t nc = cluster_n();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t h = hash32((uint32_t)i ^ seed);
        const uint32_t slot = h % S, r = (h >> 20) % nc;
        if (MODE == 0 || MODE == 4)
            asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(mapa(base + 4 * slot, r)), "f"(1e-3f) : "memory");
        if (MODE == 1)
            asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(mapa(base + 4 * slot, r)), "r"((h >> 8) & 7u) : "memory");
        if (MODE == 2) atomicAdd(&sm[slot], 1e-3f);
        if (MODE == 3) atomicAdd(reinterpret_cast<uint32_t *>(sm) + slot, (h >> 8) & 7u);
        if (MODE == 4 || MODE == 5) {
            const uint32_t d = hash32(h + 0x9e3779b9u) % Vg;
            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(g + d), "f"(1e-3f) : "memory");
        }
    }
    cluster_sync();
    if (threadIdx.x == 0 && sm[seed % S] == -1.f) g[0] = 1.f;   // keep the block alive
}

template <int MODE>
static float run(int cs, int threads, float *g, uint32_t Vg, uint64_t n, int *clusters) {
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * 4);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = S * 4;
    cfg.attrs = at; cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int nclu = 0;
    if (cudaOccupancyMaxActiveClusters(&nclu, k<MODE>, &cfg) != cudaSuccess || nclu < 1) { cudaGetLastError(); return -1; }
    *clusters = nclu;
    cfg.gridDim = dim3(nclu * cs);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    if (cudaLaunchKernelEx(&cfg, k<MODE>, g, Vg, n, 1u) != cudaSuccess) { cudaGetLastError(); return -2; }
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, k<MODE>, g, Vg, n, 2u);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    return ms;
}

int main() {
    const uint32_t Vg = 16u << 20;   // 64 MB: L2-resident
    const uint64_t n = 1ull << 29;
    float *g;
    cudaMalloc(&g, Vg * 4ull);
    cudaMemset(g, 0, Vg * 4ull);
    printf("{\"n\": %llu, \"rows\": [\n", (unsigned long long)n);
    bool first = true;
    const char *names[6] = {"cluster_red_f32", "cluster_red_u32", "local_atomic_f32", "local_atomic_u32",
                            "cluster_f32_plus_l2", "l2_only"};
    for (int cs : {1, 2, 4, 8, 16})
        for (int mode = 0; mode < 6; ++mode) {
            int clu = 0;
            float ms = -3;
            switch (mode) {
                case 0: ms = run<0>(cs, 1024, g, Vg, n, &clu); break;
                case 1: ms = run<1>(cs, 1024, g, Vg, n, &clu); break;
                case 2: ms = run<2>(cs, 1024, g, Vg, n, &clu); break;
                case 3: ms = run<3>(cs, 1024, g, Vg, n, &clu); break;
                case 4: ms = run<4>(cs, 1024, g, Vg, n, &clu); break;
                default: ms = run<5>(cs, 1024, g, Vg, n, &clu); break;
            }
            const double ops = (mode == 4 ? 2.0 : 1.0) * n;
            printf("%s{\"cluster\": %d, \"clusters\": %d, \"ctas\": %d, \"mode\": \"%s\", \"ms\": %.3f, \"g_ops_per_s\": %.1f}",
                   first ? "" : ",\n", cs, clu, clu * cs, names[mode], ms, ms > 0 ? ops / (ms / 1e3) / 1e9 : 0.0);
            first = false;
        }
    printf("\n], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
