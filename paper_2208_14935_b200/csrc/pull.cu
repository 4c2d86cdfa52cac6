// pull.cu -- sm_100a pull (bottom-up) iterations for BFS and CC on symmetric graphs
// whose edges are all resident in device memory (the SEP-Graph
// push/pull and data-/topology-driven switching HyTGraph inherits).
//
// A pull iteration is TOPOLOGY-driven: every vertex of the own range is visited
// (no queue), and a vertex reads the frontier bits of its neighbours instead of
// frontier vertices writing into their neighbours.  On a symmetric graph the out-list
// of v is also its in-list, so no transposed CSR is needed.
//   BFS: an unvisited v takes the iteration's level (frontier level + 1) once it finds
//        ANY neighbour in the frontier and stops scanning (Beamer's bottom-up step).
//        Exact only when iterations are level-synchronous, which holds when every
//        own partition of every rank is resident (no recompute pass): the engine
//        enables pull only then.  With several ranks the frontier read is the OR of
//        every rank's own frontier words (one all-reduce per pull iteration).
//   CC:  every v takes min(label(v), min over frontier neighbours label(u)).  Correct
//        under any schedule: the push invariant "label(v) <= label(u) on every edge
//        unless u is in the frontier" is kept because v pulls from every frontier u.
// The vertex owns its slot: light vertices are written with plain stores, heavy ones
// (split into slices scanned by several warps) with atomicMin.  A lowered vertex is
// set in the next frontier, exactly as the push kernel does.
// Load balance: a lane scans a list of <= 32 edges, a warp a list of <= heavy edges,
// and longer lists are cut into kSlice-edge slices, one warp each.
#include "hyt_internal.h"
#include "block_prims.cuh"

namespace hyt {

struct PullArgs {
    const uint64_t *off;
    const uint32_t *nbr;       // nbr[e] valid for the own range's edges
    uint32_t *val;
    const uint32_t *bm_cur;
    uint32_t *bm_next;
    uint64_t v_lo, v_hi;
    uint32_t heavy;            // lists longer than this go to the slice kernel
    uint32_t lvl;              // BFS: level assigned by this (level-synchronous) iteration
};

__device__ __forceinline__ bool in_frontier(const uint32_t *bm, uint32_t u) {
    return (__ldg(&bm[u >> 5]) >> (u & 31)) & 1u;
}
__device__ __forceinline__ void mark(uint32_t *bm, uint64_t v) {
    atomicOr(&bm[v >> 5], 1u << (v & 31));
}

template <int ALGO>
__global__ void __launch_bounds__(256) k_pull(PullArgs A) {
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t n = A.v_hi - A.v_lo;
    for (uint64_t wb = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; wb < n;
         wb += nwarps * 32) {
        const uint64_t v = A.v_lo + wb + lane;
        const bool in = wb + lane < n;
        uint64_t beg = 0, deg = 0;
        uint32_t cur = 0;
        bool want = false;
        if (in) {
            beg = A.off[v];
            deg = A.off[v + 1] - beg;
            cur = A.val[v];
            want = deg > 0 && (ALGO == ALGO_CC || cur == kInf);
        }
        // (1) short lists: one lane, sequential, early exit for BFS
        if (want && deg <= 32) {
            uint32_t best = cur;
            for (uint64_t j = 0; j < deg; ++j) {
                const uint32_t u = __ldg(&A.nbr[beg + j]);
                if (!in_frontier(A.bm_cur, u)) continue;
                if (ALGO == ALGO_BFS) { best = A.lvl; break; }
                const uint32_t x = __ldcg(&A.val[u]);
                best = x < best ? x : best;
            }
            if (best < cur) { A.val[v] = best; mark(A.bm_next, v); }
        }
        // (2) medium lists: the whole warp, 32 neighbours per step
        uint32_t todo = __ballot_sync(FULL_MASK, want && deg > 32 && deg <= A.heavy);
        while (todo) {
            const int l = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint64_t b = __shfl_sync(FULL_MASK, beg, l);
            const uint64_t d = __shfl_sync(FULL_MASK, deg, l);
            const uint32_t c0 = __shfl_sync(FULL_MASK, cur, l);
            uint32_t best = c0;
            for (uint64_t j = 0; j < d; j += 32) {
                uint32_t x = kInf;
                bool f = false;
                if (j + lane < d) {
                    const uint32_t u = __ldg(&A.nbr[b + j + lane]);
                    if (in_frontier(A.bm_cur, u)) { x = ALGO == ALGO_BFS ? 0u : __ldcg(&A.val[u]); f = true; }
                }
                if (ALGO == ALGO_BFS) {
                    if (__ballot_sync(FULL_MASK, f)) { best = A.lvl; break; }
                } else {
                    best = x < best ? x : best;
                }
            }
            if (ALGO == ALGO_CC)
                for (int o = 16; o; o >>= 1) {
                    const uint32_t y = __shfl_xor_sync(FULL_MASK, best, o);
                    best = y < best ? y : best;
                }
            if (lane == l && best < c0) { A.val[v] = best; mark(A.bm_next, v); }
        }
    }
}

// Heavy lists: slice s covers edges [e0[s], e1[s]) of vertex sv[s]; one warp per slice.
template <int ALGO>
__global__ void __launch_bounds__(256) k_pull_heavy(PullArgs A, const uint32_t *__restrict__ sv,
                                                  const uint64_t *__restrict__ e0, const uint64_t *__restrict__ e1,
                                                  uint64_t ns) {
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t s = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); s < ns; s += nwarps) {
        const uint32_t v = sv[s];
        const uint64_t a = e0[s], z = e1[s];
        const uint32_t c0 = __ldcg(&A.val[v]);
        if (ALGO == ALGO_BFS && c0 != kInf) continue;
        uint32_t best = c0;
        for (uint64_t j = a; j < z; j += 32) {
            uint32_t x = kInf;
            bool f = false;
            if (j + lane < z) {
                const uint32_t u = __ldg(&A.nbr[j + lane]);
                if (in_frontier(A.bm_cur, u)) { x = ALGO == ALGO_BFS ? 0u : __ldcg(&A.val[u]); f = true; }
            }
            if (ALGO == ALGO_BFS) {
                if (__ballot_sync(FULL_MASK, f)) { best = A.lvl; break; }
            } else {
                best = x < best ? x : best;
            }
        }
        if (ALGO == ALGO_CC)
            for (int o = 16; o; o >>= 1) {
                const uint32_t y = __shfl_xor_sync(FULL_MASK, best, o);
                best = y < best ? y : best;
            }
        if (lane == 0 && best < c0) {
            const uint32_t old = atomicMin(&A.val[v], best);
            if (best < old) mark(A.bm_next, v);
        }
    }
}

// out = the words of bm restricted to [lo, hi), zero elsewhere (nw words)
__global__ void k_own_words(const uint32_t *__restrict__ bm, uint32_t *__restrict__ out, uint64_t nw, uint64_t lo,
                            uint64_t hi) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t w = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nw; w += stride)
        out[w] = bm[w] & range_mask(w, lo, hi);
}

void launch_own_words(const uint32_t *bm, uint32_t *out, uint64_t nw, uint64_t lo, uint64_t hi, cudaStream_t st) {
    uint64_t grid = (nw + 255) / 256;
    if (grid > (uint64_t)num_sms() * 8) grid = (uint64_t)num_sms() * 8;
    if (grid == 0) return;
    k_own_words<<<(unsigned)grid, 256, 0, st>>>(bm, out, nw, lo, hi);
}

void launch_pull(int algo, const uint64_t *off, const uint32_t *nbr, uint32_t *val, const uint32_t *bm_cur,
                 uint32_t *bm_next, uint64_t v_lo, uint64_t v_hi, uint32_t heavy, const uint32_t *sv,
                 const uint64_t *e0, const uint64_t *e1, uint64_t ns, uint32_t lvl, cudaStream_t st) {
    PullArgs A{off, nbr, val, bm_cur, bm_next, v_lo, v_hi, heavy, lvl};
    const uint64_t n = v_hi > v_lo ? v_hi - v_lo : 0;
    uint64_t grid = (n + 255) / 256;
    if (grid > (uint64_t)num_sms() * 8) grid = (uint64_t)num_sms() * 8;
    if (grid == 0) grid = 1;
    uint64_t hg = (ns + 7) / 8;
    if (hg > (uint64_t)num_sms() * 8) hg = (uint64_t)num_sms() * 8;
    if (algo == ALGO_BFS) {
        if (n) k_pull<ALGO_BFS><<<(unsigned)grid, 256, 0, st>>>(A);
        if (ns) k_pull_heavy<ALGO_BFS><<<(unsigned)hg, 256, 0, st>>>(A, sv, e0, e1, ns);
    } else {
        if (n) k_pull<ALGO_CC><<<(unsigned)grid, 256, 0, st>>>(A);
        if (ns) k_pull_heavy<ALGO_CC><<<(unsigned)hg, 256, 0, st>>>(A, sv, e0, e1, ns);
    }
}

}  // namespace hyt
