// red_ceiling.cu -- is the 174 G/s L2-resident red.add rate of tools/scatter_bench
// the hardware's?  Uniform random f32 reductions into a 64 MB (L2-resident) array,
// swept over threads per SM, reductions in flight per thread and the PTX form
// (atomicAdd / red.global.add.f32 / red with an evict_last policy / red.add.u32).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int FORM, int K>
__global__ void k_red(float *fv, uint32_t *uv, uint32_t V, uint64_t n, uint32_t seed) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * K;
    for (uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * K; i < n; i += stride) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t d = hash32((uint32_t)(i + k) ^ seed) % V;
            if (FORM == 0) atomicAdd(fv + d, 1e-3f);
            else if (FORM == 1) asm volatile("red.global.add.f32 [%0], %1;" ::"l"(fv + d), "f"(1e-3f) : "memory");
            else if (FORM == 2) asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(fv + d), "f"(1e-3f), "l"(pol) : "memory");
            else asm volatile("red.global.add.u32 [%0], %1;" ::"l"(uv + d), "r"(1u) : "memory");
        }
    }
}

template <int FORM, int K>
float run(int threads, int per_sm, int sms, float *fv, uint32_t *uv, uint32_t V, uint64_t n) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    k_red<FORM, K><<<sms * per_sm, threads>>>(fv, uv, V, n, 1);
    cudaEventRecord(a);
    k_red<FORM, K><<<sms * per_sm, threads>>>(fv, uv, V, n, 2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a); cudaEventDestroy(b);
    return ms;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t Vs[2] = {16u << 20, 4u << 20};     // 64 MB and 16 MB of f32
    const uint64_t n = 1ull << 30;
    float *fv; uint32_t *uv;
    cudaMalloc(&fv, 64ull << 20); cudaMalloc(&uv, 64ull << 20);
    cudaMemset(fv, 0, 64ull << 20); cudaMemset(uv, 0, 64ull << 20);
    printf("{\"sms\": %d, \"n\": %llu, \"rows\": [\n", sms, (unsigned long long)n);
    bool first = true;
    for (uint32_t V : Vs)
        for (int cfg = 0; cfg < 3; ++cfg) {
            const int threads = cfg == 0 ? 256 : 1024, per_sm = cfg == 0 ? 4 : (cfg == 1 ? 1 : 2);
            struct { const char *name; float ms; } r[6] = {
                {"atomicAdd_k4", run<0, 4>(threads, per_sm, sms, fv, uv, V, n)},
                {"red_k4", run<1, 4>(threads, per_sm, sms, fv, uv, V, n)},
                {"red_k16", run<1, 16>(threads, per_sm, sms, fv, uv, V, n)},
                {"red_evict_last_k16", run<2, 16>(threads, per_sm, sms, fv, uv, V, n)},
                {"red_u32_k16", run<3, 16>(threads, per_sm, sms, fv, uv, V, n)},
                {"red_k1", run<1, 1>(threads, per_sm, sms, fv, uv, V, n)}};
            for (auto &x : r) {
                printf("%s{\"V_mb\": %u, \"threads\": %d, \"ctas_per_sm\": %d, \"form\": \"%s\", \"ms\": %.3f, \"g_per_s\": %.1f}",
                       first ? "" : ",\n", V * 4 >> 20, threads, per_sm, x.name, x.ms, n / (x.ms / 1e3) / 1e9);
                first = false;
            }
        }
    printf("\n], \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
