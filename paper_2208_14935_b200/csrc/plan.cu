// plan.cu -- the per-iteration plan (Algorithm 1) and queue building.
//
// Work is split into ITEMS of 256 bitmap words (8192 vertices) that never cross a
// partition boundary, so every CTA does the same amount of work whatever the
// partitions' vertex counts (hub-sorted graphs put a few huge vertices in the
// first partition and millions of low-degree ones in the last).  Inside an item a
// warp owns 32 words; for each non-empty word the 32 lanes handle its 32 vertices,
// so offsets / degrees / deltas are read with coalesced loads.
//
//   k_plan_items   Alg. 1 L2-12: per-item activity (a, e, z of Eq. 1-3),
//                  accumulated per partition; the last CTA selects the engine of
//                  every partition (exact integer §5.1 rule) and scans the
//                  per-engine queue offsets ("pre-combine on GPU").
//   k_fill_items   writes each active vertex of a partition with a task into its
//                  engine's queue segment with its exclusive 16-byte-chunk prefix
//                  (the compacted index of P:490) and the tile map; PR takes delta.
//   k_range_count / k_range_fill   the queue of a filter unit's vertex range for the
//                  recompute pass, built from the next frontier.
#include "hyt_internal.h"
#include "block_prims.cuh"

namespace hyt {

static_assert(kItemThreads == kItemWords, "one thread per word of an item");

struct PlanArgs {
    DevState s;
    const uint64_t *bounds, *t_static;
    Items it;
    uint64_t item_lo, item_hi, p_lo, p_hi, cache_hi;
    int mode;
    CostParams cp;
    PlanBufs pb;
};

__device__ __forceinline__ void write_tiles(uint32_t *tile, uint64_t pre, uint64_t nch, uint32_t idx) {
    // every tile whose first chunk lies in [pre, pre+nch) starts inside this entry
    const uint64_t t0 = (pre + kTile - 1) / kTile, t1 = (pre + nch - 1) / kTile;
    for (uint64_t t = t0; t <= t1; ++t) tile[t] = idx;
}

// ---------------------------------------------------------------------------
// k_plan_items
// ---------------------------------------------------------------------------
template <bool PR>
__global__ void __launch_bounds__(kItemThreads) k_plan_items(PlanArgs A) {
    __shared__ uint64_t sh[33];
    __shared__ bool is_last;
    const DevState &s = A.s;
    const uint64_t item = A.item_lo + blockIdx.x;
    const uint32_t i = A.it.part[item];
    const uint64_t w0 = A.it.w0[item], w1 = A.it.w1[item];
    const uint64_t vlo = A.bounds[i], vhi = A.bounds[i + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t ws = w0 + (uint64_t)warp * 32;
    const uint32_t d1 = s.d1;
    uint32_t myword = 0;
    if (ws + lane < w1) myword = s.bm_cur[ws + lane] & range_mask(ws + lane, vlo, vhi);
    uint64_t e = 0, a = 0, z = 0, ent = 0, ch = 0, hub = 0;
    double ds = 0.0;
    const int ms = A.cp.m_shift;     // m = 2^ms (the default 128) -> no 64-bit division
    for (uint32_t m = __ballot_sync(FULL_MASK, myword != 0); m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const uint32_t bits = __shfl_sync(FULL_MASK, myword, j);
        if ((bits >> lane) & 1u) {
            const uint64_t v = ((ws + j) << 5) + lane;
            const uint64_t o0 = s.off[v], o1 = s.off[v + 1], deg = o1 - o0;
            a += 1;
            e += deg;
            if (deg) {
                ent += 1;
                ch += chunk_hi(o1, d1) - chunk_lo(o0, d1);
                const uint64_t st = o0 * d1, en = o1 * d1 - 1;
                z += ms >= 0 ? (en >> ms) - (st >> ms) + 1 : zc_lines(st, deg * d1, A.cp.m);
                hub += deg * (uint64_t)s.din[v];
            }
            if (PR) ds += (double)s.delta[v];
        }
    }
    // one reduction pass for all seven aggregates
    {
        __shared__ uint64_t sred[6][kItemThreads / 32];
        __shared__ double sdred[kItemThreads / 32];
        uint64_t vals[6] = {e, a, z, ent, ch, hub};
#pragma unroll
        for (int f = 0; f < 6; ++f) vals[f] = warp_sum_u64(vals[f]);
        if (PR) ds = warp_sum_f64(ds);
        if (lane == 0) {
#pragma unroll
            for (int f = 0; f < 6; ++f) sred[f][warp] = vals[f];
            sdred[warp] = ds;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint64_t t[6] = {0, 0, 0, 0, 0, 0};
            double td = 0.0;
            for (int k = 0; k < kItemThreads / 32; ++k) {
#pragma unroll
                for (int f = 0; f < 6; ++f) t[f] += sred[f][k];
                td += sdred[k];
            }
            e = t[0]; a = t[1]; z = t[2]; ent = t[3]; ch = t[4]; hub = t[5]; ds = td;
        }
    }
    if (threadIdx.x == 0) {
        ItemAgg g;
        g.e = e; g.a = a; g.z = z; g.ent = ent; g.chunks = ch; g.hub = hub; g.dsum = ds;
        A.pb.iagg[item] = g;
        PartIter *P = &A.pb.parts[i];
        if (a) {
            atomicAdd((unsigned long long *)&P->e, (unsigned long long)e);
            atomicAdd((unsigned long long *)&P->a, (unsigned long long)a);
            atomicAdd((unsigned long long *)&P->z, (unsigned long long)z);
            atomicAdd((unsigned long long *)&P->ent, (unsigned long long)ent);
            atomicAdd((unsigned long long *)&P->chunks, (unsigned long long)ch);
            atomicAdd((unsigned long long *)&P->hub, (unsigned long long)hub);
            if (PR) atomicAdd(&P->dsum, ds);
        }
        __threadfence();
        const uint32_t ticket = atomicAdd(&A.pb.hdr->done, 1u);
        is_last = (ticket == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();

    // ---- last CTA (a): engine selection per partition (§5.1) ----
    uint64_t np_en[ENG_COUNT] = {0, 0, 0, 0, 0};
    uint64_t ta = 0, te = 0, tz = 0;
    for (uint64_t pi = A.p_lo + threadIdx.x; pi < A.p_hi; pi += blockDim.x) {
        PartIter *P = &A.pb.parts[pi];
        const uint64_t pe = __ldcg(&P->e), pa = __ldcg(&P->a), pz = __ldcg(&P->z), pr = __ldcg(&P->ent);
        int p = ENG_NONE;
        if (pe > 0 && pi < A.cache_hi) {
            p = ENG_R;                   // edges resident in device memory: no transfer
        } else if (pe > 0) {
            switch (A.mode) {
                case MODE_HYBRID: p = select_engine(A.t_static[pi], pe, pa, pz, pr, A.cp); break;
                case MODE_FILTER: p = ENG_F; break;
                case MODE_COMPACTION: p = ENG_C; break;
                case MODE_ZEROCOPY: p = ENG_Z; break;
                default: p = ENG_R; break;
            }
        }
        P->p = (uint32_t)p;
        np_en[p] += 1;
        ta += pa; te += pe; tz += pz;
    }
    for (int en = ENG_F; en < ENG_COUNT; ++en) np_en[en] = block_sum_u64(np_en[en], sh);
    ta = block_sum_u64(ta, sh);
    te = block_sum_u64(te, sh);
    tz = block_sum_u64(tz, sh);
    __syncthreads();
    // ---- (b) per-engine exclusive scans over the items in order ----
    uint64_t carry_e[ENG_COUNT] = {0, 0, 0, 0, 0}, carry_c[ENG_COUNT] = {0, 0, 0, 0, 0};
    for (uint64_t base = A.item_lo; base < A.item_hi; base += blockDim.x) {
        const uint64_t j = base + threadIdx.x;
        const bool in = j < A.item_hi;
        int pj = ENG_NONE;
        uint64_t ej = 0, cj = 0;
        if (in) {
            pj = (int)A.pb.parts[A.it.part[j]].p;
            ej = __ldcg(&A.pb.iagg[j].ent);
            cj = __ldcg(&A.pb.iagg[j].chunks);
        }
        for (int en = ENG_F; en < ENG_COUNT; ++en) {
            const bool mine = in && pj == en;
            uint64_t tot_e, tot_c;
            const uint64_t xe = block_exscan_u64(mine ? ej : 0, sh, &tot_e);
            const uint64_t xc = block_exscan_u64(mine ? cj : 0, sh, &tot_c);
            if (mine) { A.pb.ibase[2 * j] = carry_e[en] + xe; A.pb.ibase[2 * j + 1] = carry_c[en] + xc; }
            carry_e[en] += tot_e;
            carry_c[en] += tot_c;
        }
    }
    __syncthreads();
    // ---- (c) partition bases = bases of their first item ----
    for (uint64_t pi = A.p_lo + threadIdx.x; pi < A.p_hi; pi += blockDim.x) {
        PartIter *P = &A.pb.parts[pi];
        if (P->p == ENG_NONE) continue;
        const uint64_t fi = A.it.first[pi];
        P->ent_base = A.pb.ibase[2 * fi];
        P->chunk_base = A.pb.ibase[2 * fi + 1];
    }
    // ---- (d) segment header: F | C | Z | R ----
    if (threadIdx.x == 0) {
        SegHdr *H = A.pb.hdr;
        uint64_t eb = 0, tb = 0;
        const int order[4] = {ENG_F, ENG_C, ENG_Z, ENG_R};
        for (int k = 0; k < 4; ++k) {
            const int en = order[k];
            H->ent_base[en] = eb;
            H->ent_count[en] = carry_e[en];
            H->chunk_total[en] = carry_c[en];
            H->tile_base[en] = tb;
            H->parts[en] = np_en[en];
            eb += carry_e[en];
            tb += (carry_c[en] + kTile - 1) / kTile;
        }
        H->active_vertices = ta;
        H->active_edges = te;
        H->zc_requests = tz;
        H->done = 0;
    }
}

// ---------------------------------------------------------------------------
// word-slice helpers shared by the fill kernels.  A warp owns 32 words; lane j
// holds word j (already masked).  Pass 1 counts the warp's entries / chunks,
// pass 2 writes them at base + exclusive position.
// ---------------------------------------------------------------------------
struct WarpCount { uint64_t e, c, d; };   // entries, chunks, edges

// The set words of a warp's slice are visited in batches of kBatch: the offsets of
// every lane's vertex in all words of a batch are loaded first (independent loads
// in flight), then consumed -- one word at a time, the loads formed a chain of
// dependent round trips that dominated the range / fill kernels.
constexpr int kBatch = 4;

__device__ __forceinline__ int next_words(uint32_t &m, int (&js)[kBatch]) {
    int n = 0;
#pragma unroll
    for (int k = 0; k < kBatch; ++k) {
        js[k] = -1;
        if (m) { js[k] = __ffs(m) - 1; m &= m - 1; ++n; }
    }
    return n;
}

__device__ __forceinline__ WarpCount warp_count(const DevState &s, uint64_t ws, uint32_t myword) {
    const int lane = threadIdx.x & 31;
    WarpCount r{0, 0, 0};
    uint64_t c = 0, d = 0;
    uint32_t m = __ballot_sync(FULL_MASK, myword != 0);
    while (m) {
        int js[kBatch];
        next_words(m, js);
        uint64_t o0[kBatch], o1[kBatch];
        bool act[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            const uint32_t bits = __shfl_sync(FULL_MASK, myword, js[k] < 0 ? 0 : js[k]);
            act[k] = js[k] >= 0 && ((bits >> lane) & 1u);
            o0[k] = o1[k] = 0;
            if (act[k]) {
                const uint64_t v = ((ws + js[k]) << 5) + lane;
                o0[k] = s.off[v];
                o1[k] = s.off[v + 1];
            }
        }
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            const bool ent = act[k] && o1[k] > o0[k];
            if (ent) { c += chunk_hi(o1[k], s.d1) - chunk_lo(o0[k], s.d1); d += o1[k] - o0[k]; }
            r.e += __popc(__ballot_sync(FULL_MASK, ent));
        }
    }
    r.c = warp_sum_u64(c);
    r.d = warp_sum_u64(d);
    return r;
}

// Exclusive warp base inside the CTA from per-warp totals in shared memory.
__device__ __forceinline__ void cta_warp_bases(WarpCount wc, uint64_t *s_e, uint64_t *s_c, uint64_t *be,
                                               uint64_t *bc, uint64_t *tot_e, uint64_t *tot_c) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) { s_e[warp] = wc.e; s_c[warp] = wc.c; }
    __syncthreads();
    uint64_t xe = 0, xc = 0, te = 0, tc = 0;
    for (int k = 0; k < nw; ++k) {
        if (k < warp) { xe += s_e[k]; xc += s_c[k]; }
        te += s_e[k]; tc += s_c[k];
    }
    *be = xe; *bc = xc; *tot_e = te; *tot_c = tc;
}

// Pass 2: write the warp's entries.  PR in the plan fill (TAKE_DELTA): active
// vertices without out-edges are absorbed here (rank += delta, nothing pushed,
// S:457); the others take their delta right before their task runs
// (launch_take_delta), so a task pushes the mass that arrived earlier in the same
// iteration (asynchronous processing).  PR in a recompute range queue: the
// delta taken by k_range_count is in `scratch`.
template <bool PR, bool TAKE_DELTA>
__device__ __forceinline__ void warp_write(const DevState &s, uint64_t ws, uint32_t myword, uint64_t base_e,
                                           uint64_t base_c, QueueBufs q, uint64_t tile_base, const float *scratch,
                                           uint64_t v_lo) {
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    uint64_t run_e = base_e, run_c = base_c;
    uint32_t m = __ballot_sync(FULL_MASK, myword != 0);
    while (m) {
        int js[kBatch];
        next_words(m, js);
        uint64_t o0[kBatch], o1[kBatch];
        bool act[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            const uint32_t bits = __shfl_sync(FULL_MASK, myword, js[k] < 0 ? 0 : js[k]);
            act[k] = js[k] >= 0 && ((bits >> lane) & 1u);
            o0[k] = o1[k] = 0;
            if (act[k]) {
                const uint64_t v = ((ws + js[k]) << 5) + lane;
                o0[k] = s.off[v];
                o1[k] = s.off[v + 1];
            }
        }
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
            if (js[k] < 0) break;                          // warp-uniform
            const uint64_t v = ((ws + js[k]) << 5) + lane;
            const uint64_t deg = o1[k] - o0[k];
            const bool ent = act[k] && deg > 0;
            const uint64_t nch = ent ? chunk_hi(o1[k], s.d1) - chunk_lo(o0[k], s.d1) : 0;
            const uint32_t b = __ballot_sync(FULL_MASK, ent);
            const uint64_t inc = warp_incl_u64(nch);
            const uint64_t tot = __shfl_sync(FULL_MASK, inc, 31);
            if (PR && TAKE_DELTA && act[k] && deg == 0) s.rank[v] += atomicExch(&s.delta[v], 0.0f);
            if (ent) {
                const uint64_t idx = run_e + __popc(b & lt);
                const uint64_t pre = run_c + inc - nch;
                q.qv[idx] = (uint32_t)v;
                q.qpre[idx] = pre;
                q.qbeg[idx] = o0[k];
                q.qdeg[idx] = (uint32_t)deg;
                if (PR && !TAKE_DELTA) q.qaux[idx] = s.damping * scratch[v - v_lo] / (float)deg;
                write_tiles(q.tile + tile_base, pre, nch, (uint32_t)idx);
            }
            run_e += __popc(b);
            run_c += tot;
        }
    }
}

// ---------------------------------------------------------------------------
// k_fill_items
// ---------------------------------------------------------------------------
struct FillArgs {
    DevState s;
    const uint64_t *bounds;
    Items it;
    uint64_t item_lo;
    PlanBufs pb;
    QueueBufs q;
};

template <bool PR>
__global__ void __launch_bounds__(kItemThreads) k_fill_items(FillArgs A) {
    __shared__ uint64_t s_e[32], s_c[32];
    const DevState &s = A.s;
    const uint64_t item = A.item_lo + blockIdx.x;
    const uint32_t i = A.it.part[item];
    const int eng = (int)A.pb.parts[i].p;
    if (eng == ENG_NONE && !(PR && A.pb.parts[i].a > 0)) return;
    const uint64_t w0 = A.it.w0[item], w1 = A.it.w1[item];
    const uint64_t vlo = A.bounds[i], vhi = A.bounds[i + 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t ws = w0 + (uint64_t)warp * 32;
    uint32_t myword = 0;
    if (ws + lane < w1) myword = s.bm_cur[ws + lane] & range_mask(ws + lane, vlo, vhi);
    const WarpCount wc = warp_count(s, ws, myword);
    uint64_t be, bc, te, tc;
    cta_warp_bases(wc, s_e, s_c, &be, &bc, &te, &tc);
    uint64_t base_e = 0, base_c = 0, tile_base = 0;
    if (eng != ENG_NONE) {
        const SegHdr *H = A.pb.hdr;
        base_e = H->ent_base[eng] + A.pb.ibase[2 * item];
        base_c = A.pb.ibase[2 * item + 1];
        tile_base = H->tile_base[eng];
    }
    warp_write<PR, true>(s, ws, myword, base_e + be, base_c + bc, A.q, tile_base, nullptr, 0);
}

void launch_plan(const DevState &s, const uint64_t *bounds, const uint64_t *t_static, Items it,
                 uint64_t item_lo, uint64_t item_hi, uint64_t p_lo, uint64_t p_hi, uint64_t cache_hi, int mode,
                 const CostParams &cp, PlanBufs pb, cudaStream_t st) {
    if (item_hi <= item_lo) return;
    PlanArgs A;
    A.s = s; A.bounds = bounds; A.t_static = t_static; A.it = it;
    A.item_lo = item_lo; A.item_hi = item_hi; A.p_lo = p_lo; A.p_hi = p_hi; A.cache_hi = cache_hi;
    A.mode = mode; A.cp = cp; A.pb = pb;
    const unsigned grid = (unsigned)(item_hi - item_lo);
    if (s.algo == ALGO_PR) k_plan_items<true><<<grid, kItemThreads, 0, st>>>(A);
    else k_plan_items<false><<<grid, kItemThreads, 0, st>>>(A);
}

void launch_fill(const DevState &s, const uint64_t *bounds, Items it, uint64_t item_lo, uint64_t item_hi,
                 PlanBufs pb, QueueBufs q, cudaStream_t st) {
    if (item_hi <= item_lo) return;
    FillArgs A;
    A.s = s; A.bounds = bounds; A.it = it; A.item_lo = item_lo; A.pb = pb; A.q = q;
    const unsigned grid = (unsigned)(item_hi - item_lo);
    if (s.algo == ALGO_PR) k_fill_items<true><<<grid, kItemThreads, 0, st>>>(A);
    else k_fill_items<false><<<grid, kItemThreads, 0, st>>>(A);
}

// ---------------------------------------------------------------------------
// Range queue (recompute pass of a filter unit): the vertices of
// [v_lo, v_hi) active NOW.  Min-algorithms: bit set in the next frontier, taken
// with atomicAnd BEFORE the relax reads its value -- a racing improver sets the
// bit again after its atomicMin, so nothing is lost.  PR: delta > eps, taken
// with atomicExch.  One CTA per 256 words; count pass then fill pass.
// ---------------------------------------------------------------------------
template <bool PR>
__global__ void __launch_bounds__(kItemThreads) k_range_count(DevState s, uint64_t v_lo, uint64_t v_hi, RangeBufs r) {
    __shared__ uint64_t sh[33];
    const uint64_t wlo = v_lo >> 5, whi = (v_hi + 31) >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t ws = wlo + (uint64_t)blockIdx.x * kItemWords + (uint64_t)warp * 32;
    const uint64_t w = ws + lane;
    uint32_t taken = 0;
    if (!PR) {
        if (w < whi) {
            const uint32_t m = range_mask(w, v_lo, v_hi);
            if (s.bm_next[w] & m) taken = atomicAnd(&s.bm_next[w], ~m) & m;
        }
    } else {
        for (int j0 = 0; j0 < 32; j0 += 8) {   // 8 words' deltas in flight per lane
            float dl[8];
            bool inr[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t ww = ws + j0 + u;
                const uint64_t v = (ww << 5) + lane;
                inr[u] = ww < whi && v >= v_lo && v < v_hi;
                dl[u] = inr[u] ? s.delta[v] : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t v = ((ws + j0 + u) << 5) + lane;
                const bool act = inr[u] && dl[u] > s.epsilon;
                const uint32_t b = __ballot_sync(FULL_MASK, act);
                if (lane == j0 + u) taken = b;
                if (act) {
                    const float x = atomicExch(&s.delta[v], 0.0f);
                    s.rank[v] += x;
                    r.scratch[v - v_lo] = x;
                }
            }
        }
    }
    if (w < whi) r.taken[w - wlo] = taken;
    const WarpCount wc = warp_count(s, ws, taken);
    const uint64_t e = block_sum_u64(lane == 0 ? wc.e : 0, sh);
    const uint64_t c = block_sum_u64(lane == 0 ? wc.c : 0, sh);
    if (threadIdx.x == 0) { r.cta_agg[2 * blockIdx.x] = e; r.cta_agg[2 * blockIdx.x + 1] = c; }
}

template <bool PR>
__global__ void __launch_bounds__(kItemThreads) k_range_fill(DevState s, uint64_t v_lo, uint64_t v_hi, RangeBufs r) {
    __shared__ uint64_t sh[33], s_e[32], s_c[32];
    const uint64_t wlo = v_lo >> 5, whi = (v_hi + 31) >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t ws = wlo + (uint64_t)blockIdx.x * kItemWords + (uint64_t)warp * 32;
    const uint64_t w = ws + lane;
    uint64_t pe = 0, pc = 0;    // exclusive prefix of this CTA
    for (uint64_t j = threadIdx.x; j < blockIdx.x; j += blockDim.x) { pe += r.cta_agg[2 * j]; pc += r.cta_agg[2 * j + 1]; }
    pe = block_sum_u64(pe, sh);
    pc = block_sum_u64(pc, sh);
    const uint32_t myword = w < whi ? r.taken[w - wlo] : 0u;
    const WarpCount wc = warp_count(s, ws, myword);
    uint64_t be, bc, te, tc;
    cta_warp_bases(wc, s_e, s_c, &be, &bc, &te, &tc);
    warp_write<PR, false>(s, ws, myword, pe + be, pc + bc, r.q, 0, r.scratch, v_lo);
    const uint64_t dsum = block_sum_u64(lane == 0 ? wc.d : 0, sh);
    if (threadIdx.x == 0 && (tc || dsum)) {   // run statistics of the recompute pass
        atomicAdd((unsigned long long *)&r.acc[1], (unsigned long long)tc);
        atomicAdd((unsigned long long *)&r.acc[2], (unsigned long long)dsum);
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) { r.total[0] = pe + te; r.total[1] = pc + tc; }
}

// PR: take the delta of queue entries [e_lo, e_hi) right before their task runs.
__global__ void k_take_delta(DevState s, const uint32_t *__restrict__ qv, const uint32_t *__restrict__ qdeg,
                             float *__restrict__ qaux, uint64_t e_lo, uint64_t e_hi) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = e_lo + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < e_hi; k += stride) {
        const uint32_t v = qv[k];
        const float dl = atomicExch(&s.delta[v], 0.0f);
        s.rank[v] += dl;
        qaux[k] = s.damping * dl / (float)qdeg[k];
    }
}

void launch_take_delta(const DevState &s, const QueueBufs &q, uint64_t e_lo, uint64_t e_hi, cudaStream_t st) {
    if (e_hi <= e_lo) return;
    uint64_t blocks = (e_hi - e_lo + 255) / 256;
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    k_take_delta<<<(unsigned)blocks, 256, 0, st>>>(s, q.qv, q.qdeg, q.qaux, e_lo, e_hi);
}

void launch_range_queue(const DevState &s, uint64_t v_lo, uint64_t v_hi, RangeBufs r, cudaStream_t st) {
    const uint64_t wlo = v_lo >> 5, whi = (v_hi + 31) >> 5;
    const uint64_t nctas = (whi - wlo + kItemWords - 1) / kItemWords;
    if (nctas == 0) { cudaMemsetAsync(r.total, 0, 2 * sizeof(uint64_t), st); return; }
    if (s.algo == ALGO_PR) {
        k_range_count<true><<<(unsigned)nctas, kItemThreads, 0, st>>>(s, v_lo, v_hi, r);
        k_range_fill<true><<<(unsigned)nctas, kItemThreads, 0, st>>>(s, v_lo, v_hi, r);
    } else {
        k_range_count<false><<<(unsigned)nctas, kItemThreads, 0, st>>>(s, v_lo, v_hi, r);
        k_range_fill<false><<<(unsigned)nctas, kItemThreads, 0, st>>>(s, v_lo, v_hi, r);
    }
}

}  // namespace hyt
