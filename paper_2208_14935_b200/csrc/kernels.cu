// kernels.cu -- sm_100a kernels of the per-iteration hot path.
//
//   k_pr_frontier   PR frontier = {v : delta[v] > eps} as a bitmap
//   k_plan          Algorithm 1 lines 2-12: per-partition activity
//                   (a_i, e_i, z_i of Eq. 1-3) + engine selection,
//                   one CTA per partition; the last CTA scans the per-engine
//                   queue offsets ("pre-combine on GPU").
//   k_fill          writes the active vertices of every partition into its
//                   engine's queue segment (ballot/prefix-sum compaction) with the
//                   exclusive 16-B-chunk prefix (the "new compressed neighbour
//                   index array" of P:490) and the tile map; PR takes delta here.
//   k_relax         the push over a chunk window of a queue segment,
//                   reading edges from device memory, a staged filter unit, the
//                   compacted buffer, or mapped host memory (zero-copy).
//   k_range_count / k_range_fill   queue of a vertex range (filter recompute pass,
//                   P:460/P:465) built from the next frontier.
#include "hyt_internal.h"
#include <cstdio>

namespace hyt {

#define FULL_MASK 0xFFFFFFFFu

// ---------------------------------------------------------------------------
// small block primitives (blockDim multiple of 32, <= 1024)
// ---------------------------------------------------------------------------
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

// Block-wide sum; every thread gets the result.  `sh` needs 32 slots.
__device__ uint64_t block_sum_u64(uint64_t x, uint64_t *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    x = warp_sum_u64(x);
    __syncthreads();
    if (lane == 0) sh[wid] = x;
    __syncthreads();
    uint64_t y = lane < nw ? sh[lane] : 0;
    y = warp_sum_u64(y);
    return y;
}
__device__ double block_sum_f64(double x, double *sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    x = warp_sum_f64(x);
    __syncthreads();
    if (lane == 0) sh[wid] = x;
    __syncthreads();
    double y = lane < nw ? sh[lane] : 0.0;
    y = warp_sum_f64(y);
    return y;
}

// Block-wide exclusive scan of u64; returns the exclusive prefix, *total = sum.
__device__ uint64_t block_exscan_u64(uint64_t x, uint64_t *sh, uint64_t *total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint64_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(FULL_MASK, inc, o);
        if (lane >= o) inc += y;
    }
    __syncthreads();
    if (lane == 31) sh[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        uint64_t s = lane < nw ? sh[lane] : 0;
        uint64_t si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(FULL_MASK, si, o);
            if (lane >= o) si += y;
        }
        if (lane < nw) sh[lane] = si - s;     // exclusive warp offsets
        if (lane == 31) sh[32] = si;          // total
    }
    __syncthreads();
    uint64_t r = sh[wid] + inc - x;
    *total = sh[32];
    return r;
}

// Bits of bitmap word w that lie in [vlo, vhi).
__device__ __forceinline__ uint32_t range_mask(uint64_t w, uint64_t vlo, uint64_t vhi) {
    const uint64_t base = w << 5;
    uint32_t m = FULL_MASK;
    if (base < vlo) m &= FULL_MASK << (uint32_t)(vlo - base);
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
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    k_pr_frontier<<<(unsigned)blocks, 256, 0, st>>>(s.delta, s.bm_cur, s.V, s.epsilon);
}

// ---------------------------------------------------------------------------
// Plan: activity + selection (+ last-CTA segment scan)
// ---------------------------------------------------------------------------
template <bool PR>
__global__ void __launch_bounds__(kPlanThreads)
k_plan(DevState s, const uint64_t *__restrict__ bounds, const uint64_t *__restrict__ t_static,
       uint64_t p_lo, uint64_t np, int mode, CostParams cp, PartIter *__restrict__ parts,
       SegHdr *__restrict__ hdr) {
    __shared__ uint64_t sh[33];
    __shared__ double shd[32];
    __shared__ bool is_last;
    const uint64_t i = p_lo + blockIdx.x;
    const uint64_t vlo = bounds[i], vhi = bounds[i + 1];
    const uint64_t wlo = vlo >> 5, whi = (vhi + 31) >> 5;
    const uint32_t d1 = s.d1;
    uint64_t e = 0, a = 0, z = 0, ent = 0, chunks = 0, hub = 0;
    double dsum = 0.0;
    for (uint64_t w = wlo + threadIdx.x; w < whi; w += blockDim.x) {
        uint32_t bits = s.bm_cur[w] & range_mask(w, vlo, vhi);
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            const uint64_t v = (w << 5) + b;
            const uint64_t o0 = s.off[v], o1 = s.off[v + 1], deg = o1 - o0;
            a += 1;
            e += deg;
            if (deg) {
                ent += 1;
                chunks += chunk_hi(o1, d1) - chunk_lo(o0, d1);
                z += zc_lines(o0 * d1, deg * d1, cp.m);
                hub += deg * (uint64_t)s.din[v];
            }
            if (PR) dsum += (double)s.delta[v];
        }
    }
    e = block_sum_u64(e, sh);
    a = block_sum_u64(a, sh);
    z = block_sum_u64(z, sh);
    ent = block_sum_u64(ent, sh);
    chunks = block_sum_u64(chunks, sh);
    hub = block_sum_u64(hub, sh);
    if (PR) dsum = block_sum_f64(dsum, shd);
    if (threadIdx.x == 0) {
        int p = ENG_NONE;
        if (e > 0) {
            switch (mode) {
                case MODE_HYBRID: p = select_engine(t_static[i], e, a, z, cp); break;
                case MODE_FILTER: p = ENG_F; break;
                case MODE_COMPACTION: p = ENG_C; break;
                case MODE_ZEROCOPY: p = ENG_Z; break;
                default: p = ENG_R; break;
            }
        }
        PartIter r;
        r.e = e; r.a = a; r.z = z; r.ent = ent; r.chunks = chunks; r.hub = hub;
        r.ent_base = 0; r.chunk_base = 0; r.dsum = dsum; r.p = (uint32_t)p; r.pad = 0;
        parts[i] = r;
        atomicAdd((unsigned long long *)&hdr->active_vertices, (unsigned long long)a);
        atomicAdd((unsigned long long *)&hdr->active_edges, (unsigned long long)e);
        atomicAdd((unsigned long long *)&hdr->zc_requests, (unsigned long long)z);
        __threadfence();
        const uint32_t ticket = atomicAdd(&hdr->done, 1u);
        is_last = (ticket == np - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // ---- last CTA: per-engine exclusive scans over partitions in index order ----
    uint64_t carry_e[ENG_COUNT] = {0, 0, 0, 0, 0}, carry_c[ENG_COUNT] = {0, 0, 0, 0, 0};
    uint64_t cnt[ENG_COUNT] = {0, 0, 0, 0, 0};
    for (uint64_t base = 0; base < np; base += blockDim.x) {
        const uint64_t j = p_lo + base + threadIdx.x;
        const bool in = base + threadIdx.x < np;
        int pj = ENG_NONE;
        uint64_t ej = 0, cj = 0;
        if (in) {
            const PartIter *pp = (const PartIter *)&parts[j];
            pj = (int)((volatile const uint32_t *)&pp->p)[0];
            ej = ((volatile const uint64_t *)&pp->ent)[0];
            cj = ((volatile const uint64_t *)&pp->chunks)[0];
        }
        uint64_t my_eb = 0, my_cb = 0;
        for (int en = ENG_F; en < ENG_COUNT; ++en) {
            uint64_t tot;
            const bool mine = in && pj == en;
            const uint64_t xe = block_exscan_u64(mine ? ej : 0, sh, &tot);
            const uint64_t te = tot;
            const uint64_t xc = block_exscan_u64(mine ? cj : 0, sh, &tot);
            const uint64_t tc = tot;
            const uint64_t np_en = block_sum_u64(mine ? 1 : 0, sh);
            if (mine) { my_eb = carry_e[en] + xe; my_cb = carry_c[en] + xc; }
            carry_e[en] += te; carry_c[en] += tc; cnt[en] += np_en;
        }
        if (in && pj != ENG_NONE) { parts[j].ent_base = my_eb; parts[j].chunk_base = my_cb; }
    }
    if (threadIdx.x == 0) {
        uint64_t eb = 0, tb = 0;
        const int order[4] = {ENG_F, ENG_C, ENG_Z, ENG_R};
        for (int k = 0; k < 4; ++k) {
            const int en = order[k];
            hdr->ent_base[en] = eb;
            hdr->ent_count[en] = carry_e[en];
            hdr->chunk_total[en] = carry_c[en];
            hdr->tile_base[en] = tb;
            hdr->parts[en] = cnt[en];
            eb += carry_e[en];
            tb += (carry_c[en] + kTile - 1) / kTile;
        }
        hdr->done = 0;
    }
}

void launch_plan(const DevState &s, const uint64_t *bounds, const uint64_t *t_static, uint64_t p_lo,
                 uint64_t p_hi, int mode, const CostParams &cp, PartIter *parts, SegHdr *hdr,
                 cudaStream_t st) {
    const uint64_t np = p_hi - p_lo;
    if (np == 0) return;
    if (s.algo == ALGO_PR)
        k_plan<true><<<(unsigned)np, kPlanThreads, 0, st>>>(s, bounds, t_static, p_lo, np, mode, cp, parts, hdr);
    else
        k_plan<false><<<(unsigned)np, kPlanThreads, 0, st>>>(s, bounds, t_static, p_lo, np, mode, cp, parts, hdr);
}

// ---------------------------------------------------------------------------
// Fill: queue segments (+ PR delta take-over) -- one CTA per partition
// ---------------------------------------------------------------------------
__device__ __forceinline__ void write_tiles(uint32_t *tile, uint64_t pre, uint64_t nch, uint32_t idx) {
    // every tile whose first chunk lies in [pre, pre+nch) starts inside this entry
    const uint64_t t0 = (pre + kTile - 1) / kTile, t1 = (pre + nch - 1) / kTile;
    for (uint64_t t = t0; t <= t1; ++t) tile[t] = idx;
}

template <bool PR>
__global__ void __launch_bounds__(kPlanThreads)
k_fill(DevState s, const uint64_t *__restrict__ bounds, uint64_t p_lo, const PartIter *__restrict__ parts,
       const SegHdr *__restrict__ hdr, QueueBufs q) {
    __shared__ uint64_t sh[33];
    const uint64_t i = p_lo + blockIdx.x;
    const PartIter P = parts[i];
    const int eng = (int)P.p;
    if (eng == ENG_NONE && !(PR && P.a > 0)) return;
    const uint64_t vlo = bounds[i], vhi = bounds[i + 1];
    const uint64_t wlo = vlo >> 5, whi = (vhi + 31) >> 5;
    const uint32_t d1 = s.d1;
    uint64_t seg_ent = 0, tile_base = 0;
    if (eng != ENG_NONE) { seg_ent = hdr->ent_base[eng] + P.ent_base; tile_base = hdr->tile_base[eng]; }
    uint64_t carry_e = 0, carry_c = P.chunk_base;
    for (uint64_t wb = wlo; wb < whi; wb += blockDim.x) {
        const uint64_t w = wb + threadIdx.x;
        uint32_t bits = w < whi ? (s.bm_cur[w] & range_mask(w, vlo, vhi)) : 0u;
        uint64_t ne = 0, nc = 0;
        for (uint32_t b2 = bits; b2; b2 &= b2 - 1) {
            const uint64_t v = (w << 5) + (__ffs(b2) - 1);
            const uint64_t o0 = s.off[v], o1 = s.off[v + 1];
            if (o1 > o0) { ne += 1; nc += chunk_hi(o1, d1) - chunk_lo(o0, d1); }
        }
        uint64_t te, tc;
        uint64_t xe = block_exscan_u64(ne, sh, &te);
        uint64_t xc = block_exscan_u64(nc, sh, &tc);
        while (bits) {
            const uint64_t v = (w << 5) + (__ffs(bits) - 1);
            bits &= bits - 1;
            const uint64_t o0 = s.off[v], o1 = s.off[v + 1], deg = o1 - o0;
            if (PR) {
                const float dl = atomicExch(&s.delta[v], 0.0f);
                s.rank[v] += dl;
                if (deg) {
                    const uint64_t idx = seg_ent + carry_e + xe;
                    q.qaux[idx] = s.damping * dl / (float)deg;
                }
            }
            if (!deg || eng == ENG_NONE) continue;
            const uint64_t idx = seg_ent + carry_e + xe;
            const uint64_t pre = carry_c + xc;
            const uint64_t nch = chunk_hi(o1, d1) - chunk_lo(o0, d1);
            q.qv[idx] = (uint32_t)v;
            q.qpre[idx] = pre;
            write_tiles(q.tile + tile_base, pre, nch, (uint32_t)idx);
            xe += 1;
            xc += nch;
        }
        carry_e += te;
        carry_c += tc;
    }
}

void launch_fill(const DevState &s, const uint64_t *bounds, uint64_t p_lo, uint64_t p_hi,
                 const PartIter *parts, const SegHdr *hdr, QueueBufs q, cudaStream_t st) {
    const uint64_t np = p_hi - p_lo;
    if (np == 0) return;
    if (s.algo == ALGO_PR)
        k_fill<true><<<(unsigned)np, kPlanThreads, 0, st>>>(s, bounds, p_lo, parts, hdr, q);
    else
        k_fill<false><<<(unsigned)np, kPlanThreads, 0, st>>>(s, bounds, p_lo, parts, hdr, q);
}

// ---------------------------------------------------------------------------
// Relax: the push over a chunk window [c_lo, c_hi) of one queue segment.
// ---------------------------------------------------------------------------
struct RelaxArgs {
    DevState s;
    const uint32_t *qv;
    const uint64_t *qpre;
    const float *qaux;
    const uint32_t *tile;      // segment's tile map (already offset by tile_base)
    uint64_t c_lo, c_hi;       // window (host values)
    uint64_t seg_chunks;       // total chunks of the segment
    uint64_t seg_first, seg_end;   // global entry index range of the segment
    const uint64_t *dev_tot;   // optional: [0] = entry count, [1] = chunk total (range queues)
    const uint4 *base;
    int64_t shift;
};

template <int ALGO, bool COMPACT>
__global__ void __launch_bounds__(kRelaxThreads)
k_relax(RelaxArgs A) {
    constexpr uint32_t D1 = (ALGO == ALGO_SSSP) ? 8u : 4u;
    constexpr int EPC = 16 / D1;                  // edge records per chunk
    __shared__ uint64_t s_pre[kTile + 1];
    __shared__ uint64_t s_beg[kTile + 1];
    __shared__ uint64_t s_end[kTile + 1];
    __shared__ uint32_t s_src[kTile + 1];
    const DevState &S = A.s;

    uint64_t c_lo = A.c_lo, c_hi = A.c_hi, seg_chunks = A.seg_chunks, seg_end = A.seg_end;
    if (A.dev_tot) {
        seg_end = A.seg_first + A.dev_tot[0];
        seg_chunks = A.dev_tot[1];
        c_hi = seg_chunks;
    }
    if (c_hi <= c_lo) return;
    const uint64_t ntiles_seg = (seg_chunks + kTile - 1) / kTile;
    const uint64_t t_first = c_lo / kTile, t_last = (c_hi - 1) / kTile;

    for (uint64_t t = t_first + blockIdx.x; t <= t_last; t += gridDim.x) {
        const uint64_t tb = t * kTile;
        const uint64_t cb = tb > c_lo ? tb : c_lo;
        const uint64_t ce = (tb + kTile) < c_hi ? (tb + kTile) : c_hi;
        const uint64_t k0 = A.tile[t];
        const uint64_t k1 = (t + 1 < ntiles_seg) ? (uint64_t)A.tile[t + 1] : seg_end - 1;
        const int ne = (int)(k1 - k0 + 1);
        __syncthreads();   // previous tile finished with smem
        for (int e = threadIdx.x; e < ne; e += blockDim.x) {
            const uint64_t k = k0 + e;
            const uint32_t v = A.qv[k];
            s_pre[e] = A.qpre[k];
            s_beg[e] = S.off[v];
            s_end[e] = S.off[(uint64_t)v + 1];
            if (ALGO == ALGO_PR) s_src[e] = __float_as_uint(A.qaux[k]);
            else s_src[e] = __ldcg(&S.val[v]);
        }
        __syncthreads();

        uint4 data[kChunksPerThread];
        int ent[kChunksPerThread];
        uint64_t absc[kChunksPerThread];
#pragma unroll
        for (int r = 0; r < kChunksPerThread; ++r) {
            const uint64_t c = tb + (uint64_t)r * kRelaxThreads + threadIdx.x;
            ent[r] = -1;
            if (c >= cb && c < ce) {
                int lo = 0, hi = ne - 1;          // largest e with s_pre[e] <= c
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_pre[mid] <= c) lo = mid; else hi = mid - 1;
                }
                const uint64_t j = c - s_pre[lo];
                const uint64_t ac = chunk_lo(s_beg[lo], D1) + j;
                const uint4 *p = COMPACT ? (A.base + (c - c_lo)) : (A.base + ((int64_t)ac - A.shift));
                data[r] = *p;
                ent[r] = lo;
                absc[r] = ac;
            }
        }
#pragma unroll
        for (int r = 0; r < kChunksPerThread; ++r) {
            if (ent[r] < 0) continue;
            const int e = ent[r];
            const uint64_t beg = s_beg[e], end = s_end[e];
            const uint32_t src = s_src[e];
            const uint32_t words[4] = {data[r].x, data[r].y, data[r].z, data[r].w};
#pragma unroll
            for (int qd = 0; qd < EPC; ++qd) {
                const uint64_t idx = absc[r] * EPC + qd;
                if (idx < beg || idx >= end) continue;
                uint32_t dst, wgt = 0;
                if (D1 == 8) { dst = words[2 * qd]; wgt = words[2 * qd + 1]; }
                else dst = words[qd];
                if (ALGO == ALGO_PR) {
                    atomicAdd(&S.delta[dst], __uint_as_float(src));
                } else {
                    uint32_t cand;
                    if (ALGO == ALGO_BFS) cand = src + 1u;
                    else if (ALGO == ALGO_SSSP) {
                        const uint64_t c64 = (uint64_t)src + wgt;
                        cand = c64 >= kInf ? kInf - 1u : (uint32_t)c64;
                    } else cand = src;
                    if (cand < __ldcg(&S.val[dst])) {
                        const uint32_t old = atomicMin(&S.val[dst], cand);
                        if (cand < old) atomicOr(&S.bm_next[dst >> 5], 1u << (dst & 31));
                    }
                }
            }
        }
    }
}

void launch_relax(const DevState &s, const QueueBufs &q, uint64_t tile_base, uint64_t seg_first,
                  uint64_t seg_end, uint64_t seg_chunks, uint64_t c_lo, uint64_t c_hi,
                  const uint64_t *dev_tot, EdgeSrc src, int max_ctas, cudaStream_t st) {
    RelaxArgs A;
    A.s = s; A.qv = q.qv; A.qpre = q.qpre; A.qaux = q.qaux; A.tile = q.tile + tile_base;
    A.c_lo = c_lo; A.c_hi = c_hi; A.seg_chunks = seg_chunks; A.seg_first = seg_first; A.seg_end = seg_end;
    A.dev_tot = dev_tot; A.base = src.base; A.shift = src.shift;
    uint64_t grid;
    if (dev_tot) grid = (uint64_t)max_ctas;
    else {
        if (c_hi <= c_lo) return;
        grid = (c_hi - 1) / kTile - c_lo / kTile + 1;
        if (grid > (uint64_t)max_ctas) grid = (uint64_t)max_ctas;
    }
    if (grid == 0) grid = 1;
#define HYT_RELAX(ALG)                                                                       \
    if (src.compact) k_relax<ALG, true><<<(unsigned)grid, kRelaxThreads, 0, st>>>(A);      \
    else k_relax<ALG, false><<<(unsigned)grid, kRelaxThreads, 0, st>>>(A);
    switch (s.algo) {
        case ALGO_BFS: HYT_RELAX(ALGO_BFS); break;
        case ALGO_SSSP: HYT_RELAX(ALGO_SSSP); break;
        case ALGO_CC: HYT_RELAX(ALGO_CC); break;
        default: HYT_RELAX(ALGO_PR); break;
    }
#undef HYT_RELAX
}

// ---------------------------------------------------------------------------
// Range queue (recompute pass of a filter unit): the vertices of
// [v_lo, v_hi) that are active NOW (min-algorithms: bit set in the next
// frontier, taken with atomicAnd before their value is read -- a racing
// improver sets the bit again after its atomicMin, so nothing is lost; PR:
// delta > eps, taken with atomicExch).
// k_range_count: take + per-CTA aggregates.  k_range_fill: prefix + write.
// ---------------------------------------------------------------------------
template <bool PR>
__global__ void __launch_bounds__(kRangeWords)
k_range_count(DevState s, uint64_t v_lo, uint64_t v_hi, RangeBufs r) {
    __shared__ uint64_t sh[33];
    const uint64_t wlo = v_lo >> 5, whi = (v_hi + 31) >> 5;
    const uint64_t w = wlo + (uint64_t)blockIdx.x * kRangeWords + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint32_t bits = 0;
    if (PR) {
        // warp-cooperative coalesced delta reads: word (warp_base + i) built by ballot
        const uint64_t wbase = wlo + (uint64_t)blockIdx.x * kRangeWords + (threadIdx.x & ~31u);
        for (int i = 0; i < 32; ++i) {
            const uint64_t ww = wbase + i;
            const uint64_t v = (ww << 5) + lane;
            bool act = false;
            if (ww < whi && v >= v_lo && v < v_hi) act = s.delta[v] > s.epsilon;
            const uint32_t word = __ballot_sync(FULL_MASK, act);
            if (lane == i) bits = word;
        }
        for (uint32_t b2 = bits; b2; b2 &= b2 - 1) {
            const uint64_t v = (w << 5) + (__ffs(b2) - 1);
            const float dl = atomicExch(&s.delta[v], 0.0f);
            s.rank[v] += dl;
            r.scratch[v - v_lo] = dl;
        }
    } else if (w < whi) {
        const uint32_t m = range_mask(w, v_lo, v_hi);
        if (s.bm_next[w] & m) bits = atomicAnd(&s.bm_next[w], ~m) & m;
    }
    uint64_t ne = 0, nc = 0;
    for (uint32_t b2 = bits; b2; b2 &= b2 - 1) {
        const uint64_t v = (w << 5) + (__ffs(b2) - 1);
        const uint64_t o0 = s.off[v], o1 = s.off[v + 1];
        if (o1 > o0) { ne += 1; nc += chunk_hi(o1, s.d1) - chunk_lo(o0, s.d1); }
    }
    if (w < whi) r.taken[w - wlo] = bits;
    ne = block_sum_u64(ne, sh);
    nc = block_sum_u64(nc, sh);
    if (threadIdx.x == 0) { r.cta_agg[2 * blockIdx.x] = ne; r.cta_agg[2 * blockIdx.x + 1] = nc; }
}

template <bool PR>
__global__ void __launch_bounds__(kRangeWords)
k_range_fill(DevState s, uint64_t v_lo, uint64_t v_hi, RangeBufs r) {
    __shared__ uint64_t sh[33];
    const uint64_t wlo = v_lo >> 5, whi = (v_hi + 31) >> 5;
    const uint64_t w = wlo + (uint64_t)blockIdx.x * kRangeWords + threadIdx.x;
    // exclusive prefix of this CTA = sum of the aggregates of the CTAs before it
    uint64_t pe = 0, pc = 0;
    for (uint64_t j = threadIdx.x; j < blockIdx.x; j += blockDim.x) { pe += r.cta_agg[2 * j]; pc += r.cta_agg[2 * j + 1]; }
    pe = block_sum_u64(pe, sh);
    pc = block_sum_u64(pc, sh);
    const uint32_t bits0 = w < whi ? r.taken[w - wlo] : 0u;
    uint64_t ne = 0, nc = 0;
    for (uint32_t b2 = bits0; b2; b2 &= b2 - 1) {
        const uint64_t v = (w << 5) + (__ffs(b2) - 1);
        const uint64_t o0 = s.off[v], o1 = s.off[v + 1];
        if (o1 > o0) { ne += 1; nc += chunk_hi(o1, s.d1) - chunk_lo(o0, s.d1); }
    }
    uint64_t te, tc;
    uint64_t xe = block_exscan_u64(ne, sh, &te);
    uint64_t xc = block_exscan_u64(nc, sh, &tc);
    for (uint32_t bits = bits0; bits; bits &= bits - 1) {
        const uint64_t v = (w << 5) + (__ffs(bits) - 1);
        const uint64_t o0 = s.off[v], o1 = s.off[v + 1], deg = o1 - o0;
        if (!deg) continue;
        const uint64_t idx = pe + xe, pre = pc + xc;
        const uint64_t nch = chunk_hi(o1, s.d1) - chunk_lo(o0, s.d1);
        r.q.qv[idx] = (uint32_t)v;
        r.q.qpre[idx] = pre;
        if (PR) r.q.qaux[idx] = s.damping * r.scratch[v - v_lo] / (float)deg;
        write_tiles(r.q.tile, pre, nch, (uint32_t)idx);
        xe += 1;
        xc += nch;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) { r.total[0] = pe + te; r.total[1] = pc + tc; }
}

void launch_range_queue(const DevState &s, uint64_t v_lo, uint64_t v_hi, RangeBufs r, cudaStream_t st) {
    const uint64_t wlo = v_lo >> 5, whi = (v_hi + 31) >> 5;
    const uint64_t nctas = (whi - wlo + kRangeWords - 1) / kRangeWords;
    if (nctas == 0) { cudaMemsetAsync(r.total, 0, 2 * sizeof(uint64_t), st); return; }
    if (s.algo == ALGO_PR) {
        k_range_count<true><<<(unsigned)nctas, kRangeWords, 0, st>>>(s, v_lo, v_hi, r);
        k_range_fill<true><<<(unsigned)nctas, kRangeWords, 0, st>>>(s, v_lo, v_hi, r);
    } else {
        k_range_count<false><<<(unsigned)nctas, kRangeWords, 0, st>>>(s, v_lo, v_hi, r);
        k_range_fill<false><<<(unsigned)nctas, kRangeWords, 0, st>>>(s, v_lo, v_hi, r);
    }
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
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    k_init<<<(unsigned)blocks, 256, 0, st>>>(s, src_internal, old_of);
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
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_mark_improved<<<(unsigned)blocks, 256, 0, st>>>(val, snap, lo, hi, bm);
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
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    const uint32_t *vals = s.algo == ALGO_PR ? (const uint32_t *)s.rank : s.val;
    k_gather_out<<<(unsigned)blocks, 256, 0, st>>>(vals, new_id, (uint32_t *)out_dev, s.V);
}

}  // namespace hyt
