// scatter_bench.cu -- the achievable rate of the relax kernels' access pattern on this
// GPU, as a second denominator next to the HBM copy peak.
//
// A resident push relaxation streams E edge records and, per edge, touches one
// 4-byte destination slot at a data-dependent address: an
// L2 reduction (Δ-PR, red.add.f32), or a load followed by an atomicMin when the
// candidate improves (BFS/SSSP/CC).  This tool times exactly that pattern without
// any of the engine's bookkeeping:
//
//   stream   read the E x 4-byte index array only (HBM streaming roofline check)
//   red_add  stream + red.global.add.f32 at the index           (Δ-PR push)
//   ld       stream + 4-byte load at the index                  (min-algo, no improvement)
//   ld_min   stream + load + atomicMin when the candidate wins  (min-algo, nearly every edge improving)
//
// over V = 41.7M slots (the TW-shaped config, 167 MB: larger than the 126 MB L2)
// and E = 1.47B edges, with destinations drawn uniformly or RMAT-skewed
// (a, b, c = 0.57, 0.19, 0.19: column bit 1 with probability b + d = 0.24 at each
// of 26 levels, rejected to < V), so low ids are the hot ones, as after the hub
// sort.  One JSON line: per pattern, ms per pass, G edges/s and algorithmic GB/s
// (4-byte index + 4-byte destination access per edge).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void k_gen(uint32_t *idx, uint64_t E, uint64_t V, int skew) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += stride) {
        uint64_t d = 0;
        for (uint64_t t = 0;; ++t) {
            if (!skew) {
                d = mix(i * 0x100000001B3ull + t) % V;
                break;
            }
            d = 0;
            uint64_t r = mix(i * 977ull + t * 0x5851F42D4C957F2Dull);
            for (int l = 0; l < 26; ++l) {
                if ((l & 1) == 0 && l) r = mix(r);
                const uint32_t u = (uint32_t)(r >> (32 * (l & 1))) ;
                d = (d << 1) | (u < 1030792151u ? 1u : 0u);   // 0.24 * 2^32
            }
            if (d < V) break;
        }
        idx[i] = (uint32_t)d;
    }
}

template <int OP>
__global__ void __launch_bounds__(256, 4) k_scatter(const uint4 *__restrict__ idx, uint64_t n4, float *fv,
                                                   uint32_t *uv, uint32_t *sink) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        const uint4 q = __ldcs(idx + i);
        const uint32_t d[4] = {q.x, q.y, q.z, q.w};
        if (OP == 0) {
            acc ^= q.x ^ q.y ^ q.z ^ q.w;
        } else if (OP == 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) atomicAdd(fv + d[k], 1e-3f);
        } else {
            uint32_t cur[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) cur[k] = __ldcg(uv + d[k]);
            if (OP == 2) {
#pragma unroll
                for (int k = 0; k < 4; ++k) acc ^= cur[k];
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t cand = 0xFFFFFFF0u - (uint32_t)i;   // decreases over the pass: mostly improving
                    if (cand < cur[k]) acc ^= atomicMin(uv + d[k], cand);
                }
            }
        }
    }
    if (acc == 0x9E3779B9u) *sink = acc;
}

int main() {
    const uint64_t V = 41700000ull, E = 1470000000ull;
    uint32_t *idx, *uv, *sink;
    float *fv;
    cudaMalloc(&idx, E * 4);
    cudaMalloc(&uv, V * 4);
    cudaMalloc(&fv, V * 4);
    cudaMalloc(&sink, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("{\"V\": %llu, \"E\": %llu, \"sms\": %d", (unsigned long long)V, (unsigned long long)E, sms);
    const char *names[4] = {"stream", "red_add", "ld", "ld_min"};
    // third case: uniform over 16M slots (64 MB, L2-resident): the L2 rate of the
    // pattern without DRAM misses
    const uint64_t V_l2 = 16u << 20;
    for (int skew = 0; skew < 3; ++skew) {
        k_gen<<<sms * 8, 256>>>(idx, E, skew == 2 ? V_l2 : V, skew == 1);
        printf(", \"%s\": {", skew == 1 ? "rmat" : skew == 2 ? "uniform_l2_resident" : "uniform");
        for (int op = 0; op < 4; ++op) {
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(fv, 0, V * 4);
                cudaMemset(uv, 0xFF, V * 4);
                cudaEventRecord(a);
                switch (op) {
                    case 0: k_scatter<0><<<sms * 4, 256>>>((const uint4 *)idx, E / 4, fv, uv, sink); break;
                    case 1: k_scatter<1><<<sms * 4, 256>>>((const uint4 *)idx, E / 4, fv, uv, sink); break;
                    case 2: k_scatter<2><<<sms * 4, 256>>>((const uint4 *)idx, E / 4, fv, uv, sink); break;
                    default: k_scatter<3><<<sms * 4, 256>>>((const uint4 *)idx, E / 4, fv, uv, sink); break;
                }
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            const double bytes = op == 0 ? E * 4.0 : E * 8.0;
            printf("%s\"%s\": {\"ms\": %.3f, \"gedges_s\": %.2f, \"alg_gbs\": %.1f}", op ? ", " : "", names[op], best,
                   E / (best / 1e3) / 1e9, bytes / (best / 1e3) / 1e9);
        }
        printf("}");
    }
    printf(", \"error\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
