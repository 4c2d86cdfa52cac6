// kernels.cu -- sm_100a kernels of the per-iteration hot path.
//
//   k_pr_frontier   PR frontier = {v : delta[v] > eps} as a bitmap
//   k_relax         the push over a chunk window of a queue segment,
//                   reading edges from device memory, a staged filter unit, the
//                   compacted buffer, or mapped host memory (zero-copy).
//   (the plan / fill / recompute-queue kernels are in plan.cu)
#include "hyt_internal.h"
#include "block_prims.cuh"
#include <algorithm>
#include <cstdio>

namespace hyt {

// ---------------------------------------------------------------------------
// PR frontier
// ---------------------------------------------------------------------------
__global__ void k_pr_frontier(const float *__restrict__ delta, uint32_t *__restrict__ bm, uint64_t V,
                              float eps) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t Vr = (V + 31) & ~31ull;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < Vr; v += stride) {
        const bool act = v < V && delta[v] > eps;
        const uint32_t w = __ballot_sync(FULL_MASK, act);
        if ((threadIdx.x & 31) == 0) bm[v >> 5] = w;
    }
}

void launch_pr_frontier(const DevState &s, cudaStream_t st) {
    const uint64_t Vr = (s.V + 31) & ~31ull;
    uint64_t blocks = (Vr + 255) / 256;
    if (blocks > num_sms() * 16) blocks = num_sms() * 16;
    if (blocks == 0) blocks = 1;
    k_pr_frontier<<<(unsigned)blocks, 256, 0, st>>>(s.delta, s.bm_cur, s.V, s.epsilon);
}

// ---------------------------------------------------------------------------
// Relax: the push over a chunk window [c_lo, c_hi) of one queue segment.
//
// Work unit = a WARP tile of kTile = 128 consecutive chunks of the segment's chunk
// space (warps are independent: no CTA barriers on the hot loop).  Per tile the
// lanes stage the <= kTile+1 overlapping queue entries (prefix, first edge,
// degree, source value) in the warp's shared-memory slice, then each lane finds
// the entry of each of its 4 chunks from a 128-bit map of entry start positions
// (one popc) and issues 4 independent
// 16-byte loads; 8 consecutive lanes cover one aligned 128-byte line.
// Hub block (ids < kHotV, the highest-H vertices after hub sorting):
// PR pushes into it are accumulated in shared memory and flushed once per CTA, so
// the hottest destinations do not serialise L2 atomics.  Min-algorithms keep a
// per-CTA copy of the hub values: values only decrease, so the copy is never below
// the global value and a candidate that does not beat it cannot beat the global
// one either.  A candidate that lowers the copy (smem atomicMin) goes on to the
// global atomicMin, so at most a few global atomics per hub per CTA remain.
// ---------------------------------------------------------------------------
struct RelaxArgs {
    DevState s;
    const uint32_t *qv;
    const uint64_t *qpre, *qbeg;
    const uint32_t *qdeg;
    const float *qaux;
    const uint32_t *tile;      // segment's tile map (already offset by tile_base)
    uint64_t c_lo, c_hi;       // window (host values)
    uint64_t seg_chunks;       // total chunks of the segment
    uint64_t seg_first, seg_end;   // global entry index range of the segment
    const uint64_t *dev_tot;   // optional: [0] = entry count, [1] = chunk total (range queues)
    const uint4 *base;
    int64_t shift;
    uint32_t n_hot;            // hub-block size cached in shared memory (0 = off)
    uint32_t hot_force;        // keep the hub block however small the launch (relax_hot = 2)
    uint32_t bands;            // destination bands (1 = one pass)
    PeerPush pp;               // fused multi-rank push (PEER instantiations only)
};


// L2 eviction-priority hints: the edge stream is read once per task (evict first),
// the vertex values / deltas are re-read by every task (evict last), so the
// streaming edges do not push the value array out of the 126 MB L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_stream(const uint4 *p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint32_t ld_keep(const uint32_t *p, uint64_t pol) {
    uint32_t r;
    asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ void red_min_keep(uint32_t *p, uint32_t x, uint64_t pol) {
    asm volatile("red.global.min.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(x), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add_keep(float *p, float x, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(p), "f"(x), "l"(pol) : "memory");
}

// owner rank of a remote destination (ranks own contiguous ranges)
__device__ __forceinline__ int peer_owner(const PeerPush &pp, uint32_t d) {
    int o = 0;
#pragma unroll
    for (int k = 1; k < kMaxPeers; ++k) o += (k < (int)pp.n && (uint64_t)d >= pp.rb[k]);
    return o;
}
__device__ __forceinline__ bool peer_remote(const PeerPush &pp, uint32_t d) {
    return (uint64_t)d < pp.lo || (uint64_t)d >= pp.hi;
}

// Per-warp staging of the <= kTile+1 queue entries overlapping one tile, 16 B per
// entry (the round-1 layout held prefix / first edge as u64 and spent 24 B):
//   a[e]  = absolute chunk address of TILE POSITION 0 for entry e, so tile position
//           p of the entry is chunk a[e] + p (one 64-bit add per chunk);
//   lh[e] = the entry's first / end edge SLOT relative to tile position 0, as two
//           int16 (clamped to [-EPC, (kTile+1)*EPC]: only [0, EPC) matters for any p);
//           at position p the valid slots of the chunk are
//           [max(0, lo - p*EPC), min(EPC, hi - p*EPC));
//   src[e] = the pushed value (PR: f32 contribution d*delta/D_o; else u32 value).
struct WarpStage {
    uint64_t a[kTile + 1];
    uint32_t lh[kTile + 1];
    uint32_t src[kTile + 1];
    uint32_t mask[kChunksPerThread];
};

// PR hub block in fixed point: x in units of 2^-32 as a 64-bit (hi, lo) pair of u32
// words, so every add is a native shared-memory ATOMS.ADD (an f32 or u64 atomicAdd
// on shared memory compiles to a CAS spin loop on sm_100a, which serialises the
// lanes of a warp that hit the same hub).  The carry out of lo is detected from
// the returned old value and added to hi.  Range: 2^32 per hub per CTA, above any
// mass one launch can push (sum of pushes <= sum of delta <= V < 2^32).  Rounding:
// <= 2^-33 absolute per add, i.e. at or below f32 rounding for any partial sum
// >= 2^-9; the flush converts the pair back to f32 once per CTA.
__device__ __forceinline__ void hub_add_fx(uint32_t *lo, uint32_t *hi, uint32_t d, uint32_t xlo, uint32_t xhi) {
    if (xhi) atomicAdd(&hi[d], xhi);
    const uint32_t old = atomicAdd(&lo[d], xlo);
    if (old + xlo < old) atomicAdd(&hi[d], 1u);
}

template <int ALGO, bool COMPACT, bool PEER, int NT>
__global__ void __launch_bounds__(NT, NT >= 1024 ? 1 : 2)
k_relax(RelaxArgs A) {
    constexpr uint32_t D1 = (ALGO == ALGO_SSSP) ? 8u : 4u;   // ALGO_SSSP_PACKED: 4-byte records
    constexpr int EPC = 16 / D1;                  // edge records per chunk
    constexpr bool PR = (ALGO == ALGO_PR);
    constexpr int kWarps = NT / 32;
    // dynamic shared memory: the warps' staging, then the hub block (PR = n_hot lo
    // words then n_hot hi words, fixed point; min-algorithms = n_hot hub values)
    extern __shared__ __align__(16) uint8_t s_dyn[];
    WarpStage *s_st = reinterpret_cast<WarpStage *>(s_dyn);
    uint32_t *s_hotw = reinterpret_cast<uint32_t *>(s_dyn + kWarps * sizeof(WarpStage));
    const DevState &S = A.s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    WarpStage &W = s_st[w];
    const uint64_t pol_stream = policy_evict_first(), pol_keep = policy_evict_last();

    uint64_t c_lo = A.c_lo, c_hi = A.c_hi, seg_chunks = A.seg_chunks, seg_end = A.seg_end;
    if (A.dev_tot) {
        seg_end = A.seg_first + A.dev_tot[0];
        seg_chunks = A.dev_tot[1];
        c_hi = seg_chunks;
    }
    // The hub block costs a per-CTA init (and for PR a flush) proportional to its size:
    // a CTA whose share of the window is small does without it (decided from the
    // device-side totals, so recompute passes of unknown size are covered too).
    // hot_force (relax_hot = 2, tests) keeps it whatever the size.
    uint32_t n_hot = A.n_hot;
    if (n_hot && !A.hot_force) {
        const uint64_t chunks = c_hi > c_lo ? c_hi - c_lo : 0;
        const uint64_t edges_per_cta = chunks * EPC / gridDim.x;
        if (edges_per_cta < 2ull * n_hot) n_hot = 0;
    }
    uint32_t *const s_lo = s_hotw, *const s_hi = s_hotw + n_hot;
    if (n_hot) {
        if (PR) {
            for (uint32_t i = threadIdx.x; i < 2 * n_hot; i += blockDim.x) s_hotw[i] = 0u;
        } else {
            for (uint32_t i = threadIdx.x; i < n_hot; i += blockDim.x) s_hotw[i] = ld_keep(&S.val[i], pol_keep);
        }
        __syncthreads();
    }
    // Destination bands (relax_bands): with device-resident edges and a value / delta
    // array larger than the L2, the window is swept once per band of destinations,
    // each pass pushing only into its band (hubs in the shared-memory block are
    // pushed in band 0), so the random destination accesses of a pass stay in an
    // L2-sized slice.  The edges are re-read from HBM once per band (streamed,
    // evict-first) instead of missing L2 on a random 4-byte access.
    const uint32_t nb = A.bands ? A.bands : 1;
    if (c_hi > c_lo)
    for (uint32_t band = 0; band < nb; ++band) {
        const uint32_t b_lo = (uint32_t)(S.V * band / nb), b_hi = (uint32_t)(S.V * (band + 1) / nb);
        const uint32_t hub_cut = band == 0 ? n_hot : 0u;   // hub pushes go to smem in band 0 only
        const uint64_t ntiles_seg = (seg_chunks + kTile - 1) / kTile;
        const uint64_t t_first = c_lo / kTile, t_last = (c_hi - 1) / kTile;
        const uint64_t gw = (uint64_t)blockIdx.x * kWarps + w, nw = (uint64_t)gridDim.x * kWarps;
        for (uint64_t t = t_first + gw; t <= t_last; t += nw) {
            const uint64_t tb = t * kTile;
            const uint64_t cb = tb > c_lo ? tb : c_lo;
            const uint64_t ce = (tb + kTile) < c_hi ? (tb + kTile) : c_hi;
            const uint64_t k0 = A.tile[t];
            const uint64_t k1 = (t + 1 < ntiles_seg) ? (uint64_t)A.tile[t + 1] : seg_end - 1;
            const int ne = (int)(k1 - k0 + 1);
            if (lane < kChunksPerThread) W.mask[lane] = 0u;
            __syncwarp();
            for (int e = lane; e < ne; e += 32) {
                const uint64_t k = k0 + e;
                const uint64_t pre = A.qpre[k], beg = A.qbeg[k];
                const uint32_t deg = A.qdeg[k];
                const int64_t rel = (int64_t)pre - (int64_t)tb;       // entry start - tile start (chunks)
                W.a[e] = chunk_lo(beg, D1) - (uint64_t)rel;
                const int64_t lo = (int64_t)(beg % EPC) + rel * EPC, hi = lo + deg;
                const int64_t cap = (int64_t)(kTile + 1) * EPC;
                const int32_t l16 = (int32_t)(lo < -EPC ? -EPC : lo);
                const int32_t h16 = (int32_t)(hi > cap ? cap : hi);
                W.lh[e] = ((uint32_t)l16 & 0xFFFFu) | ((uint32_t)h16 << 16);
                W.src[e] = PR ? __float_as_uint(A.qaux[k]) : ld_keep(&S.val[A.qv[k]], pol_keep);
                // 128-bit map of the tile positions where an entry starts (the entry
                // covering the tile's first chunk starts at position 0)
                const uint64_t pos = rel > 0 ? (uint64_t)rel : 0;
                if (pos < (uint64_t)kTile) atomicOr(&W.mask[pos >> 5], 1u << (pos & 31));
            }
            __syncwarp();
            uint4 data[kChunksPerThread];
            int ent[kChunksPerThread];
            // lane L's r-th chunk is tile position 32 r + L: its entry index is the
            // number of starts at positions <= 32 r + L, minus one
            const uint32_t le = 0xFFFFFFFFu >> (31 - lane);
            int before = 0;
#pragma unroll
            for (int r = 0; r < kChunksPerThread; ++r) {
                const uint32_t m = W.mask[r];
                const int p = r * 32 + lane;
                const uint64_t c = tb + p;
                const int e = before + __popc(m & le) - 1;
                before += __popc(m);
                ent[r] = -1;
                if (c >= cb && c < ce) {
                    const uint4 *ptr = COMPACT ? (A.base + (c - c_lo)) : (A.base + ((int64_t)(W.a[e] + p) - A.shift));
                    data[r] = ld_stream(ptr, pol_stream);
                    ent[r] = e;
                }
            }
            if constexpr (PR) {
#pragma unroll
                for (int r = 0; r < kChunksPerThread; ++r) {
                    if (ent[r] < 0) continue;
                    const int e = ent[r];
                    const int p = r * 32 + lane;
                    const uint32_t lh = W.lh[e];
                    const int lo = (int)(int16_t)(lh & 0xFFFFu) - p * EPC;
                    const int hi = (int)(int16_t)(lh >> 16) - p * EPC;
                    const float x = __uint_as_float(W.src[e]);
                    const unsigned long long X = __float2ull_rn(x * 4294967296.0f);
                    const uint32_t xlo = (uint32_t)X, xhi = (uint32_t)(X >> 32);
                    const uint32_t words[4] = {data[r].x, data[r].y, data[r].z, data[r].w};
#pragma unroll
                    for (int qd = 0; qd < EPC; ++qd) {
                        if (qd < lo || qd >= hi) continue;
                        const uint32_t dst = words[qd];
                        if (dst < n_hot) {
                            if (dst < hub_cut) hub_add_fx(s_lo, s_hi, dst, xlo, xhi);
                        } else if (dst < b_lo || dst >= b_hi) {
                            // another band's destination
                        } else if (PEER && peer_remote(A.pp, dst)) {
                            atomicAdd(&A.pp.delta[peer_owner(A.pp, dst)][dst], x);
                        } else {
                            red_add_keep(&S.delta[dst], x, pol_keep);
                        }
                    }
                }
            } else {
                // two halves of two chunks: gather every destination value first (up
                // to 8 loads in flight per lane), then compare and update
#pragma unroll
                for (int h = 0; h < kChunksPerThread; h += 2) {
                    uint32_t dst[2][EPC], cand[2][EPC], cur[2][EPC];
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr) {
                        const int r = h + rr;
                        int lo = EPC, hi = 0;
                        uint32_t src = 0;
                        if (ent[r] >= 0) {
                            const int e = ent[r];
                            const int p = r * 32 + lane;
                            const uint32_t lh = W.lh[e];
                            lo = (int)(int16_t)(lh & 0xFFFFu) - p * EPC;
                            hi = (int)(int16_t)(lh >> 16) - p * EPC;
                            src = W.src[e];
                        }
                        const uint32_t words[4] = {data[r].x, data[r].y, data[r].z, data[r].w};
#pragma unroll
                        for (int qd = 0; qd < EPC; ++qd) {
                            uint32_t d, wgt = 0;
                            if (D1 == 8) { d = words[2 * qd]; wgt = words[2 * qd + 1]; }
                            else if (ALGO == ALGO_SSSP_PACKED) {
                                d = words[qd] & ((1u << S.wshift) - 1u);
                                wgt = words[qd] >> S.wshift;
                            } else d = words[qd];
                            // this band's destinations only (hubs: band 0)
                            const bool ok = qd >= lo && qd < hi &&
                                            (d < n_hot ? band == 0 : (d >= b_lo && d < b_hi));
                            uint32_t cnd;
                            if (ALGO == ALGO_BFS) cnd = src + 1u;
                            else if (ALGO == ALGO_SSSP || ALGO == ALGO_SSSP_PACKED) {
                                const uint64_t c64 = (uint64_t)src + wgt;
                                cnd = c64 >= kInf ? kInf - 1u : (uint32_t)c64;
                            } else cnd = src;
                            dst[rr][qd] = d;
                            cand[rr][qd] = ok ? cnd : kInf;
                            cur[rr][qd] = !ok ? 0u : d < n_hot ? s_hotw[d] : ld_keep(&S.val[d], pol_keep);
                        }
                    }
                    // issue every improving atomicMin first (their round trips overlap),
                    // then mark the vertices whose value this lane actually lowered.  The
                    // mark depends on the returned value, so it is ordered after the
                    // min: the recompute pass's clear-then-read protocol stays sound.
                    uint32_t old[2][EPC];
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                        for (int qd = 0; qd < EPC; ++qd) {
                            old[rr][qd] = 0u;          // "not issued": never marks
                            const uint32_t d = dst[rr][qd], cn = cand[rr][qd];
                            if (cn < cur[rr][qd]) {
                                if (d < n_hot && cn >= atomicMin(&s_hotw[d], cn)) continue;
                                if (PEER && peer_remote(A.pp, d)) {
                                    // the owner's copy decides; the local copy only filters
                                    old[rr][qd] = atomicMin(&A.pp.val[peer_owner(A.pp, d)][d], cn);
                                    red_min_keep(&S.val[d], cn, pol_keep);
                                } else {
                                    old[rr][qd] = atomicMin(&S.val[d], cn);
                                }
                            }
                        }
#pragma unroll
                    for (int rr = 0; rr < 2; ++rr)
#pragma unroll
                        for (int qd = 0; qd < EPC; ++qd) {
                            const uint32_t d = dst[rr][qd];
                            if (cand[rr][qd] < old[rr][qd]) {
                                uint32_t *bm = S.bm_next;
                                if (PEER && peer_remote(A.pp, d)) bm = A.pp.bm[peer_owner(A.pp, d)];
                                atomicOr(&bm[d >> 5], 1u << (d & 31));
                            }
                        }
                }
            }
            __syncwarp();
        }
    }
    if (PR && n_hot) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < n_hot; i += blockDim.x) {
            const uint64_t X = ((uint64_t)s_hi[i] << 32) | s_lo[i];
            if (X == 0) continue;
            const float x = (float)((double)X * (1.0 / 4294967296.0));
            if (PEER && peer_remote(A.pp, i)) atomicAdd(&A.pp.delta[peer_owner(A.pp, i)][i], x);
            else atomicAdd(&S.delta[i], x);
        }
    }
}

// Launch with a dynamic hub block of `smem` bytes: raise the kernel's dynamic shared
// memory limit once, and cap the persistent grid at what stays resident (a second
// wave of a grid-stride kernel would double the tail).
static void relax_go(void (*k)(RelaxArgs), int nt, const RelaxArgs &A, uint64_t grid, size_t smem, cudaStream_t st) {
    // cached per (device, kernel, smem): the attribute and the occupancy belong to a
    // device context, and one thread may drive handles on several GPUs
    struct Occ { int dev; void (*k)(RelaxArgs); size_t smem; int per_sm; };
    static thread_local Occ cache[128];
    static thread_local int ncache = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    int per_sm = -1;
    for (int i = 0; i < ncache; ++i)
        if (cache[i].dev == dev && cache[i].k == k && cache[i].smem == smem) { per_sm = cache[i].per_sm; break; }
    if (per_sm < 0) {
        // past the 48 KB default, allow the kernel the device's opt-in maximum (one
        // setting serves every hub-block size of this kernel on this device)
        cudaFuncAttributes fa{};
        cudaFuncGetAttributes(&fa, k);
        if (fa.sharedSizeBytes + smem > 48 * 1024) {
            int optin = 0;
            if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess ||
                optin < 1)
                optin = 227 * 1024;
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
        }
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, nt, smem) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        if (ncache < 128) cache[ncache++] = Occ{dev, k, smem, per_sm};
    }
    if (grid > (uint64_t)num_sms() * per_sm) grid = (uint64_t)num_sms() * per_sm;
    k<<<(unsigned)grid, nt, smem, st>>>(A);
}

void launch_relax(const DevState &s, const QueueBufs &q, uint64_t tile_base, uint64_t seg_first,
                  uint64_t seg_end, uint64_t seg_chunks, uint64_t c_lo, uint64_t c_hi,
                  const uint64_t *dev_tot, EdgeSrc src, int max_ctas, cudaStream_t st, int hot,
                  const PeerPush *peer) {
    RelaxArgs A;
    A.s = s; A.qv = q.qv; A.qpre = q.qpre; A.qbeg = q.qbeg; A.qdeg = q.qdeg; A.qaux = q.qaux;
    A.tile = q.tile + tile_base;
    A.c_lo = c_lo; A.c_hi = c_hi; A.seg_chunks = seg_chunks; A.seg_first = seg_first; A.seg_end = seg_end;
    A.dev_tot = dev_tot; A.base = src.base; A.shift = src.shift;
    if (peer) A.pp = *peer;
    // threads per CTA (relax_threads; 0 = auto: PR 1024 so one CTA per SM shares a
    // 16384-hub block, min-algorithms 512 with two CTAs per SM)
    const int nt = s.relax_nt == 0 ? (s.algo == ALGO_PR ? 1024 : 512) : (s.relax_nt >= 1024 ? 1024 : 512);
    const uint64_t nwarps = (uint64_t)nt / 32;
    if (nt == 1024) max_ctas = (max_ctas + 1) / 2;           // same threads per SM
    uint64_t grid;
    if (dev_tot) grid = (uint64_t)max_ctas;
    else {
        if (c_hi <= c_lo) return;
        const uint64_t tiles = (c_hi - 1) / kTile - c_lo / kTile + 1;
        grid = (tiles + nwarps - 1) / nwarps;
        if (grid > (uint64_t)max_ctas) grid = (uint64_t)max_ctas;
    }
    if (grid == 0) grid = 1;
    // PR: always (the flush touches only non-zero accumulators).  Min-algorithms:
    // only when every warp has >= 4 tiles (64 KiB of edges per CTA against the 16 KiB
    // hub-value load); range queues (device-side size) do not qualify.  hot = 2
    // forces it on (tests), 0 turns both off.
    // PR accumulates into up to hot_v hubs; min-algorithms copy at most kHotV hub values
    // (the copy is a per-CTA load, a larger one does not pay: profiles/r01_hot_v.md)
    const uint64_t hv_cap = s.algo == ALGO_PR ? (uint64_t)s.hot_v : std::min<uint64_t>(s.hot_v, kHotV);
    const uint64_t hv = s.V < hv_cap ? s.V : hv_cap;
    // destination bands: only for edges in device memory, and only when the array
    // the pushes land in (4 B per vertex) exceeds three quarters of the L2
    A.bands = 1;
    if (!src.host) {
        if (s.bands) A.bands = s.bands;
        else {
            static thread_local int l2[64] = {};
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev >= 0 && dev < 64 && !l2[dev] &&
                (cudaDeviceGetAttribute(&l2[dev], cudaDevAttrL2CacheSize, dev) != cudaSuccess || l2[dev] <= 0))
                l2[dev] = 126 << 20;
            const uint64_t slice = (uint64_t)(dev >= 0 && dev < 64 ? l2[dev] : (126 << 20)) * 3 / 4;
            A.bands = (uint32_t)std::max<uint64_t>(1, (s.V * 4 + slice - 1) / slice);
            if (A.bands > 16) A.bands = 16;
        }
    }
    A.n_hot = 0;
    A.hot_force = hot == 2;
    if (hot && s.algo == ALGO_PR) A.n_hot = (uint32_t)hv;
    else if (hot == 2 || (hot == 1 && !dev_tot && (c_hi - c_lo) >= grid * nwarps * 4 * kTile)) A.n_hot = (uint32_t)hv;
    // staging of every warp + the hub block (PR: fixed-point (lo, hi) pairs)
    const size_t smem = nwarps * sizeof(WarpStage) + (size_t)A.n_hot * (s.algo == ALGO_PR ? 8 : 4);
#define HYT_RELAX_N(ALG, CO, PE)                                                                 \
    if (nt == 1024) relax_go(k_relax<ALG, CO, PE, 1024>, nt, A, grid, smem, st);              \
    else relax_go(k_relax<ALG, CO, PE, 512>, nt, A, grid, smem, st);
#define HYT_RELAX_B(ALG, PE)                                                                     \
    if (src.compact) { HYT_RELAX_N(ALG, true, PE) }                                              \
    else { HYT_RELAX_N(ALG, false, PE) }
#define HYT_RELAX(ALG)                                                                           \
    if (peer && peer->n) { HYT_RELAX_B(ALG, true) }                                              \
    else { HYT_RELAX_B(ALG, false) }
    switch (s.algo) {
        case ALGO_BFS: HYT_RELAX(ALGO_BFS); break;
        case ALGO_SSSP:
            if (s.d1 == 4) { HYT_RELAX(ALGO_SSSP_PACKED); }
            else { HYT_RELAX(ALGO_SSSP); }
            break;
        case ALGO_CC: HYT_RELAX(ALGO_CC); break;
        default: HYT_RELAX(ALGO_PR); break;
    }
#undef HYT_RELAX_N
#undef HYT_RELAX_B
#undef HYT_RELAX
}

// ---------------------------------------------------------------------------
// Initial values and frontier
// ---------------------------------------------------------------------------
__global__ void k_init(DevState s, uint64_t src, const uint32_t *__restrict__ old_of) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < s.V; v += stride) {
        switch (s.algo) {
            case ALGO_BFS:
            case ALGO_SSSP: s.val[v] = (v == src) ? 0u : kInf; break;
            case ALGO_CC: s.val[v] = old_of[v]; break;      // label = caller id -> min caller id
            default: s.rank[v] = 0.0f; s.delta[v] = 1.0f - s.damping; break;
        }
    }
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < s.W; w += stride) {
        uint32_t bits = 0;
        if (s.algo == ALGO_CC) bits = range_mask(w, 0, s.V);
        else if (s.algo != ALGO_PR && (src >> 5) == w) bits = 1u << (src & 31);
        s.bm_cur[w] = bits;
        s.bm_next[w] = 0;
    }
}

void launch_init_values(const DevState &s, uint64_t src_internal, const uint32_t *old_of, cudaStream_t st) {
    uint64_t blocks = (s.V + 255) / 256;
    if (blocks > num_sms() * 16) blocks = num_sms() * 16;
    if (blocks == 0) blocks = 1;
    k_init<<<(unsigned)blocks, 256, 0, st>>>(s, src_internal, old_of);
}

// Zero-copy probe for the calibrated cost model: random 128-byte lines (mode 0) or
// a contiguous stream (mode 1) of the mapped edge store.
__global__ void k_zc_probe(const uint4 *__restrict__ host, uint64_t nlines, uint64_t per_warp, int mode,
                           uint32_t *__restrict__ sink) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t acc = 0;
    for (uint64_t i = 0; i < per_warp; i += 16) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            uint64_t line;
            if (mode == 0) {
                uint64_t x = (warp * 0x9E3779B97F4A7C15ull) ^ ((i + u * 4 + lane / 8) * 0xBF58476D1CE4E5B9ull);
                x ^= x >> 31; x *= 0x94D049BB133111EBull; x ^= x >> 29;
                line = x % nlines;
            } else {
                line = ((i + u * 4) * nwarps + warp) * 4 + lane / 8;
                line %= nlines;
            }
            v[u] = host[line * 8 + (lane & 7)];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= v[u].x;
    }
    if (acc == 0x9E3779B9u) *sink = acc;
}

float time_zc_probe(const uint4 *mapped, uint64_t nlines, int mode, uint32_t *sink, uint64_t *lines_read,
                    cudaStream_t st) {
    const int blocks = num_sms() * 2, threads = 256;
    const uint64_t per_warp = 2048;    // 4 lines per warp instruction, 16 per step
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_zc_probe<<<blocks, threads, 0, st>>>(mapped, nlines, per_warp / 8, mode, sink);   // warm
    cudaEventRecord(a, st);
    k_zc_probe<<<blocks, threads, 0, st>>>(mapped, nlines, per_warp, mode, sink);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *lines_read = (uint64_t)blocks * (threads / 32) * per_warp;
    return ms;
}

// Multi-GPU: after the min-reduction, own vertices improved by another rank join
// the next frontier (owner-side frontier merge).
__global__ void k_mark_improved(const uint32_t *__restrict__ val, const uint32_t *__restrict__ snap, uint64_t lo,
                                uint64_t hi, uint32_t *__restrict__ bm) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < hi; v += stride)
        if (val[v] < snap[v - lo]) atomicOr(&bm[v >> 5], 1u << (v & 31));
}

void launch_mark_improved(const uint32_t *val, const uint32_t *snap, uint64_t lo, uint64_t hi, uint32_t *bm,
                          cudaStream_t st) {
    if (hi <= lo) return;
    uint64_t blocks = (hi - lo + 255) / 256;
    if (blocks > num_sms() * 16) blocks = num_sms() * 16;
    k_mark_improved<<<(unsigned)blocks, 256, 0, st>>>(val, snap, lo, hi, bm);
}

// ---------------------------------------------------------------------------
// Sparse inter-GPU exchange: (id, payload) pairs of the entries a
// rank changed this iteration, all-gathered instead of a dense V-entry reduction.
//   min-algorithms: every v with val[v] < its value at iteration start
//   PR: every non-owned v with a non-zero delta (the outbox)
// Each CTA appends its pairs through one atomicAdd; entries past `cap` are
// counted but not written (the host then takes the dense path).
// ---------------------------------------------------------------------------
__global__ void k_collect_changed(int pr, uint64_t V, uint64_t lo, uint64_t hi, const uint32_t *__restrict__ val,
                                  const uint32_t *__restrict__ snap, const float *__restrict__ delta,
                                  uint2 *__restrict__ pairs, uint64_t cap, unsigned long long *cnt) {
    __shared__ unsigned long long s_base;
    __shared__ uint32_t s_n;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v0 = (uint64_t)blockIdx.x * blockDim.x; v0 < V; v0 += stride) {
        const uint64_t v = v0 + threadIdx.x;
        bool take = false;
        uint32_t x = 0;
        if (v < V) {
            if (pr) {
                const float d = delta[v];
                take = (v < lo || v >= hi) && d != 0.0f;
                x = __float_as_uint(d);
            } else {
                x = val[v];
                take = x < snap[v];
            }
        }
        if (threadIdx.x == 0) s_n = 0;
        __syncthreads();
        const uint32_t b = __ballot_sync(FULL_MASK, take);
        uint32_t wbase = 0;
        if ((threadIdx.x & 31) == 0 && b) wbase = atomicAdd(&s_n, (uint32_t)__popc(b));
        wbase = __shfl_sync(FULL_MASK, wbase, 0);
        __syncthreads();
        if (threadIdx.x == 0) s_base = s_n ? atomicAdd(cnt, (unsigned long long)s_n) : 0ull;
        __syncthreads();
        if (take) {
            const uint64_t k = s_base + wbase + __popc(b & ((1u << (threadIdx.x & 31)) - 1u));
            if (k < cap) pairs[k] = make_uint2((uint32_t)v, x);
        }
        __syncthreads();
    }
}

// fill [count, n) with the empty pair (id 0xFFFFFFFF) before the all-gather
__global__ void k_pad_pairs(uint2 *pairs, const unsigned long long *cnt, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = *cnt + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride)
        pairs[k] = make_uint2(0xFFFFFFFFu, 0u);
}

// apply every rank's pairs: min into val (and mark owned vertices another rank
// lowered), or add the deltas addressed to this rank's vertices
__global__ void k_apply_pairs(int pr, const uint2 *__restrict__ pairs, uint64_t n, uint64_t lo, uint64_t hi,
                              uint32_t *val, float *delta, uint32_t *bm_next) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const uint2 p = pairs[k];
        if (p.x == 0xFFFFFFFFu) continue;
        const bool own = p.x >= lo && p.x < hi;
        if (pr) {
            if (own) atomicAdd(&delta[p.x], __uint_as_float(p.y));
        } else {
            const uint32_t old = atomicMin(&val[p.x], p.y);
            if (own && p.y < old) atomicOr(&bm_next[p.x >> 5], 1u << (p.x & 31));
        }
    }
}

void launch_collect_changed(int pr, uint64_t V, uint64_t lo, uint64_t hi, const uint32_t *val, const uint32_t *snap,
                            const float *delta, uint2 *pairs, uint64_t cap, unsigned long long *cnt,
                            cudaStream_t st) {
    uint64_t blocks = (V + 255) / 256;
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    if (blocks == 0) blocks = 1;
    k_collect_changed<<<(unsigned)blocks, 256, 0, st>>>(pr, V, lo, hi, val, snap, delta, pairs, cap, cnt);
}

void launch_pad_pairs(uint2 *pairs, const unsigned long long *cnt, uint64_t n, cudaStream_t st) {
    k_pad_pairs<<<num_sms(), 256, 0, st>>>(pairs, cnt, n);
}

void launch_apply_pairs(int pr, const uint2 *pairs, uint64_t n, uint64_t lo, uint64_t hi, uint32_t *val,
                        float *delta, uint32_t *bm_next, cudaStream_t st) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    if (blocks == 0) return;
    k_apply_pairs<<<(unsigned)blocks, 256, 0, st>>>(pr, pairs, n, lo, hi, val, delta, bm_next);
}

// out[caller id] = value[new_id[caller id]]
__global__ void k_gather_out(const uint32_t *__restrict__ vals, const uint32_t *__restrict__ new_id,
                             uint32_t *__restrict__ out, uint64_t V) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride)
        out[v] = vals[new_id[v]];
}

void launch_gather_out(const DevState &s, const uint32_t *new_id, void *out_dev, cudaStream_t st) {
    uint64_t blocks = (s.V + 255) / 256;
    if (blocks > num_sms() * 16) blocks = num_sms() * 16;
    if (blocks == 0) blocks = 1;
    const uint32_t *vals = s.algo == ALGO_PR ? (const uint32_t *)s.rank : s.val;
    k_gather_out<<<(unsigned)blocks, 256, 0, st>>>(vals, new_id, (uint32_t *)out_dev, s.V);
}

}  // namespace hyt
