// load.cu -- hyt_load_csr: CSR validation, hub sorting and the
// relabelled copy of the edges into library-owned pinned, mapped host memory
// (the paper's storage split: vertex data on the GPU, edges in host memory,
// P:75).  All per-vertex and per-edge work runs on the GPU; the
// caller's edge arrays are read in place through a temporary host mapping.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <exception>
#include <mutex>
#include <sys/mman.h>
#include <thread>
#include <unordered_map>
#include "graph.h"
#include "scan.h"
#include "block_prims.cuh"

namespace hyt {

// ---------------------------------------------------------------------------
// pinned mapped host memory
// ---------------------------------------------------------------------------
static std::mutex g_pin_mu;
static std::unordered_map<void *, uint64_t> g_pinned;

// Pinning is expensive (first touch of every page + cudaHostRegister: about 1.3 s for
// TW's 17.6 GB store on the pool's 16-core hosts, and the registration holds the
// driver while it runs), so freed blocks are kept, still registered, and handed to
// the next allocation that fits (a new handle's edge store, a run context's staging):
// a caching host allocator like the device-side ones.  Bounded by HYT_PIN_CACHE_GB
// (default 32 GiB; 0 disables it); hyt_trim_pinned_cache() returns everything.
struct PinBlock { void *p; uint64_t len; };
static std::vector<PinBlock> g_pin_cache;
static uint64_t g_pin_cached = 0;

static uint64_t pin_cache_cap() {
    static uint64_t cap = [] {
        const char *e = getenv("HYT_PIN_CACHE_GB");
        const double gb = e ? atof(e) : 32.0;
        return (uint64_t)(gb > 0 ? gb * (double)(1ull << 30) : 0.0);
    }();
    return cap;
}

static bool pin_verbose() {
    static const bool v = getenv("HYT_VERBOSE") != nullptr;
    return v;
}
static double pin_now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void *pinned_alloc(uint64_t bytes) {
    const uint64_t huge = 2ull << 20;
    const double t0 = pin_now_ms();
    const uint64_t len = (bytes + huge - 1) / huge * huge;
    {   // a cached block of at least len and at most 5/4 of it (contents are not zeroed:
        // every user writes what it reads; the edge store's padding is never interpreted)
        std::lock_guard<std::mutex> l(g_pin_mu);
        int best = -1;
        for (int i = 0; i < (int)g_pin_cache.size(); ++i) {
            const uint64_t L = g_pin_cache[i].len;
            if (L >= len && L <= len + len / 4 && (best < 0 || L < g_pin_cache[best].len)) best = i;
        }
        if (best >= 0) {
            PinBlock b = g_pin_cache[best];
            g_pin_cache.erase(g_pin_cache.begin() + best);
            g_pin_cached -= b.len;
            g_pinned[b.p] = b.len;
            return b.p;
        }
    }
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) throw Err{HYT_ENOMEM, "mmap of " + std::to_string(len) + " B failed"};
    madvise(p, len, MADV_HUGEPAGE);
    // parallel first touch (the registration pins resident pages); two cores stay free
    // for the thread that drives the GPU meanwhile (the load pins its store while the
    // GPU hub-sorts)
    const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
    unsigned nt = std::max(1u, std::min(16u, hc > 4 ? hc - 2 : hc));
    if (len < (256ull << 20)) nt = 1;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        const uint64_t a = len / huge * t / nt * huge, b = len / huge * (t + 1) / nt * huge;
        th.emplace_back([=] { std::memset((char *)p + a, 0, b - a); });
    }
    for (auto &x : th) x.join();
    cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterMapped | cudaHostRegisterPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        munmap(p, len);
        throw Err{HYT_ENOMEM, std::string("cudaHostRegister failed: ") + cudaGetErrorString(e)};
    }
    if (pin_verbose() && len >= (64ull << 20))
        fprintf(stderr, "[hyt pin] new block %8.3f GB  %7.1f ms (cache holds %.3f GB)\n", len / 1e9,
                pin_now_ms() - t0, g_pin_cached / 1e9);
    std::lock_guard<std::mutex> l(g_pin_mu);
    g_pinned[p] = len;
    return p;
}

static void pin_release(void *p, uint64_t len) {
    const double t0 = pin_now_ms();
    cudaHostUnregister(p);
    munmap(p, len);
    if (pin_verbose() && len >= (64ull << 20))
        fprintf(stderr, "[hyt pin] released %8.3f GB  %7.1f ms\n", len / 1e9, pin_now_ms() - t0);
}

void pinned_free(void *p) {
    if (!p) return;
    uint64_t len = 0;
    std::vector<PinBlock> evict;
    {
        std::lock_guard<std::mutex> l(g_pin_mu);
        auto it = g_pinned.find(p);
        if (it == g_pinned.end()) return;
        len = it->second;
        g_pinned.erase(it);
        const uint64_t cap = pin_cache_cap();
        if (len <= cap) {   // keep it; evict the oldest blocks beyond the cap
            g_pin_cache.push_back({p, len});
            g_pin_cached += len;
            while (g_pin_cached > cap) {
                evict.push_back(g_pin_cache.front());
                g_pin_cached -= g_pin_cache.front().len;
                g_pin_cache.erase(g_pin_cache.begin());
            }
            p = nullptr;
        }
    }
    for (auto &b : evict) pin_release(b.p, b.len);
    if (p) pin_release(p, len);
}

void pinned_trim() {
    std::vector<PinBlock> all;
    {
        std::lock_guard<std::mutex> l(g_pin_mu);
        all.swap(g_pin_cache);
        g_pin_cached = 0;
    }
    for (auto &b : all) pin_release(b.p, b.len);
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// In-degrees from the caller's ids read in place over the link (zero-copy): 16-byte
// loads (4 ids per lane, 512 B per warp instruction) from the first 16-byte aligned
// id on, the unaligned head and the tail one id per thread.
__global__ void k_indeg(const uint32_t *__restrict__ nbr, uint64_t E, uint64_t V, uint32_t *__restrict__ din,
                        uint32_t *__restrict__ bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint64_t head = std::min<uint64_t>(E, ((16 - ((uintptr_t)nbr & 15)) & 15) / 4);
    const uint64_t nvec = (E - head) / 4;
    auto one = [&](uint32_t x) {
        if (x >= V) { *bad = 1; return; }
        atomicAdd(&din[x], 1u);
    };
    if (tid < head) one(nbr[tid]);
    const uint4 *v4 = reinterpret_cast<const uint4 *>(nbr + head);
    // 4 coalesced 16-byte loads in flight per thread before the atomics (the ids
    // are read over the host link)
    uint64_t i = tid;
    for (; i + 3 * stride < nvec; i += 4 * stride) {
        uint4 q[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) q[u] = v4[i + u * stride];
#pragma unroll
        for (int u = 0; u < 4; ++u) { one(q[u].x); one(q[u].y); one(q[u].z); one(q[u].w); }
    }
    for (; i < nvec; i += stride) {
        const uint4 q = v4[i];
        one(q.x); one(q.y); one(q.z); one(q.w);
    }
    for (uint64_t i = head + nvec * 4 + tid; i < E; i += stride) one(nbr[i]);
}

// HYT_SYMMETRIC sanity check: a symmetric edge multiset has D_i(v) = D_o(v) for
// every v (necessary, not sufficient; it catches a directed graph declared symmetric).
__global__ void k_sym_degrees(const uint64_t *__restrict__ off, const uint32_t *__restrict__ din, uint64_t V,
                              uint32_t *__restrict__ bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride)
        if ((uint64_t)din[v] != off[v + 1] - off[v]) *bad = 2;
}

// H(v) = D_o D_i / (D_omax D_imax): the denominator is common, so the exact
// integer key D_o*D_i orders the vertices as H does.
__device__ __forceinline__ uint64_t hub_key(const uint64_t *off, const uint32_t *din, uint64_t v) {
    return (off[v + 1] - off[v]) * (uint64_t)din[v];
}

// radix select, one 8-bit digit per pass: histogram of the digit at `shift` among
// keys whose higher bits equal `prefix` (under `mask`)
// One digit's histogram.  Most keys share a few digits (every vertex without in- or
// out-edges has key 0), so lanes with equal digits are aggregated first
// (__match_any_sync) and one lane adds the group's count: a per-key shared-memory
// atomic on one hot bin serialised the early passes.
__global__ void k_key_hist(const uint64_t *__restrict__ off, const uint32_t *__restrict__ din, uint64_t V,
                           uint64_t prefix, uint64_t mask, int shift, unsigned long long *__restrict__ hist) {
    __shared__ unsigned int sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const uint64_t Vr = (V + 31) & ~31ull;                   // whole warps take part in the match
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < Vr; v += stride) {
        uint32_t digit = 256u;                               // 256: not counted
        if (v < V) {
            const uint64_t k = hub_key(off, din, v);
            if ((k & mask) == prefix) digit = (uint32_t)((k >> shift) & 0xFF);
        }
        const uint32_t grp = __match_any_sync(FULL_MASK, digit);
        if (digit != 256u && lane == __ffs(grp) - 1) atomicAdd(&sh[digit], (unsigned)__popc(grp));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (sh[i]) atomicAdd(&hist[i], (unsigned long long)sh[i]);
}

__global__ void k_tie_flags(const uint64_t *__restrict__ off, const uint32_t *__restrict__ din, uint64_t V,
                            uint64_t T, uint32_t *__restrict__ flag) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride)
        flag[v] = hub_key(off, din, v) == T;
}

// hub iff key > T, or key == T and among the first `ties` such vertices by id
__global__ void k_hub_flags(const uint64_t *__restrict__ off, const uint32_t *__restrict__ din, uint64_t V,
                            uint64_t T, uint64_t ties, const uint32_t *__restrict__ tie_rank,
                            uint32_t *__restrict__ flag) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride) {
        const uint64_t k = hub_key(off, din, v);
        flag[v] = k > T || (k == T && tie_rank[v] < ties);
    }
}

__global__ void k_scatter_hubs(const uint64_t *__restrict__ off, const uint32_t *__restrict__ din, uint64_t V,
                               const uint32_t *__restrict__ flag, const uint32_t *__restrict__ pos,
                               uint32_t *__restrict__ hub_ids, uint64_t *__restrict__ hub_keys) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride)
        if (flag[v]) { hub_ids[pos[v]] = (uint32_t)v; hub_keys[pos[v]] = hub_key(off, din, v); }
}

__global__ void k_mark_hubs(const uint32_t *__restrict__ sorted_ids, uint64_t h, uint32_t *__restrict__ new_id,
                            uint32_t *__restrict__ nonhub) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < h; i += stride) {
        const uint32_t v = sorted_ids[i];
        new_id[v] = (uint32_t)i;      // hubs: 0..h-1 in descending H, ties by id
        nonhub[v] = 0;
    }
}

__global__ void k_fill_u32(uint32_t *p, uint64_t n, uint32_t x) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = x;
}

// non-hubs keep their natural order after the hubs; build the inverse map and
// the degree / in-degree arrays in the new order.
__global__ void k_finish_perm(uint64_t V, uint64_t h, const uint32_t *__restrict__ nonhub,
                              const uint32_t *__restrict__ nonhub_scan, const uint64_t *__restrict__ off,
                              const uint32_t *__restrict__ din, uint32_t *__restrict__ new_id,
                              uint32_t *__restrict__ old_of, uint64_t *__restrict__ deg2,
                              uint32_t *__restrict__ din2) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride) {
        uint32_t n;
        if (nonhub[v]) { n = (uint32_t)(h + nonhub_scan[v]); new_id[v] = n; }
        else n = new_id[v];
        old_of[n] = (uint32_t)v;
        deg2[n] = off[v + 1] - off[v];
        din2[n] = din[v];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) deg2[V] = 0;
}

// Relabelled copy of the edges, edge-parallel: a CTA takes a tile of 8192 new edge
// slots; the rows overlapping it are staged in shared memory (new start, old start)
// and each thread finds its row by binary search, then copies id (mapped through
// new_id) and weight.  Reads of the caller's arrays and writes of the pinned store
// are both coalesced (consecutive slots of a row are consecutive on both sides).
constexpr int kRelabelTile = 8192, kRelabelRows = 2048;

// 16-byte warp helpers of the relabel kernel: the next lane's vector, the r <= 3
// values past a warp block (scalar loads of exactly those: nothing past the array),
// and lane values r..r+3 of the concatenation (a, b).
__device__ __forceinline__ uint4 shfl_down_u4(uint4 v) {
    return make_uint4(__shfl_down_sync(FULL_MASK, v.x, 1), __shfl_down_sync(FULL_MASK, v.y, 1),
                      __shfl_down_sync(FULL_MASK, v.z, 1), __shfl_down_sync(FULL_MASK, v.w, 1));
}
__device__ __forceinline__ uint4 tail_u4(const uint32_t *p, int r) {
    return make_uint4(r > 0 ? p[0] : 0u, r > 1 ? p[1] : 0u, r > 2 ? p[2] : 0u, 0u);
}
__device__ __forceinline__ void pick4(const uint4 &a, const uint4 &b, int r, uint32_t *o) {
    const uint32_t c[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t x = c[k];
#pragma unroll
        for (int q = 1; q < 4; ++q)
            if (r == q) x = c[k + q];
        o[k] = x;
    }
}

// row_start (shard loads): the first edge of internal row r in the caller's local
// arrays is row_start[r - r_base] (rows r_base..r_end-1 only); otherwise it is
// off_old[old_of[r]] in the caller's full arrays.  A neighbour id >= V sets *bad.
// nbr_out may be null (HYT_ADOPT_HOST: the caller's ids are the store).
__global__ void __launch_bounds__(512)
k_relabel_tiles(uint64_t V, uint64_t e_lo, uint64_t e_hi, const uint64_t *__restrict__ off_old,
                const uint64_t *__restrict__ off_new,
                const uint32_t *__restrict__ old_of, const uint32_t *__restrict__ new_id,
                const uint64_t *__restrict__ row_start, uint64_t r_base, uint64_t r_end,
                const uint32_t *__restrict__ nbr_in, const uint32_t *__restrict__ w_in,
                uint32_t *__restrict__ nbr_out, uint64_t *__restrict__ ew_out,
                uint32_t *__restrict__ pw_out, uint32_t wshift, uint32_t *__restrict__ wbig,
                uint32_t *__restrict__ bad) {
    __shared__ uint64_t s_new[kRelabelRows + 1];
    __shared__ uint64_t s_old[kRelabelRows];
    __shared__ uint64_t s_r0;
    // edges [e_lo, e_hi) of the new order; nbr_out / ew_out are indexed by the
    // global edge index (the caller offsets them to its store's first record)
    const uint64_t ntiles = (e_hi - e_lo + kRelabelTile - 1) / kRelabelTile;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        uint64_t e = e_lo + t * kRelabelTile;
        const uint64_t e_end = min(e_hi, e + kRelabelTile);
        while (e < e_end) {
            __syncthreads();
            if (threadIdx.x == 0) {        // last row whose start <= e (skips empty rows)
                uint64_t lo = 0, hi = V - 1;
                while (lo < hi) {
                    const uint64_t mid = (lo + hi + 1) / 2;
                    if (off_new[mid] <= e) lo = mid; else hi = mid - 1;
                }
                s_r0 = lo;
            }
            __syncthreads();
            const uint64_t r0 = s_r0;
            const uint64_t nr = min((uint64_t)kRelabelRows, V - r0);
            for (uint64_t i = threadIdx.x; i <= nr; i += blockDim.x) {
                s_new[i] = off_new[r0 + i];
                if (i < nr) {
                    const uint64_t r = r0 + i;
                    s_old[i] = row_start ? ((r >= r_base && r < r_end) ? row_start[r - r_base] : 0)
                                         : off_old[old_of[r]];
                }
            }
            __syncthreads();
            const uint64_t stop = min(e_end, s_new[nr]);   // edges the staged rows cover
            // Warp blocks of 128 consecutive slots, 4 per lane.  Stores: one 16-byte
            // store per lane whenever its 4 slots are all in range (x % 4 == 0, and the
            // stores are chunk-aligned).  Loads: when the block's 128 slots come from
            // 128 consecutive source edges (one shift; the common case, since non-hub
            // rows keep their order), each lane reads 16 aligned bytes and takes its 4
            // values across its own and the next lane's vector; otherwise 4 scalar
            // loads per lane.  The caller's arrays are read over the host link.
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
            const bool vec_in = ((((uintptr_t)nbr_in) | (w_in ? (uintptr_t)w_in : 0)) & 15) == 0;
            const bool need_w = ew_out || pw_out;
            for (uint64_t xb = (e & ~127ull) + (uint64_t)warp * 128; xb < stop; xb += (uint64_t)nwarps * 128) {
                const uint64_t xl = xb + 4ull * lane;
                uint64_t src[4];
                bool val[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint64_t x = xl + k;
                    val[k] = x >= e && x < stop;
                    src[k] = 0;
                    if (val[k]) {
                        int lo = 0, hi = (int)nr - 1;      // last staged row starting <= x
                        while (lo < hi) {
                            const int mid = (lo + hi + 1) >> 1;
                            if (s_new[mid] <= x) lo = mid; else hi = mid - 1;
                        }
                        src[k] = s_old[lo] + (x - s_new[lo]);
                    }
                }
                const bool full = val[0] && val[1] && val[2] && val[3];
                const uint64_t shift = src[0] - xl;       // source - slot (mod 2^64)
                const bool mine = full && src[1] == src[0] + 1 && src[2] == src[0] + 2 && src[3] == src[0] + 3;
                const uint64_t shift0 = __shfl_sync(FULL_MASK, shift, 0);
                const bool uni = vec_in && __all_sync(FULL_MASK, mine && shift == shift0);
                uint32_t id[4], wt[4] = {0u, 0u, 0u, 0u};
                if (uni) {
                    const uint64_t s0 = xb + shift0, a = s0 & ~3ull;
                    const int r = (int)(s0 - a);
                    uint4 v = reinterpret_cast<const uint4 *>(nbr_in + a)[lane];
                    uint4 vn = shfl_down_u4(v);
                    if (lane == 31) vn = tail_u4(nbr_in + a + 128, r);
                    pick4(v, vn, r, id);
                    if (need_w) {
                        uint4 w4 = reinterpret_cast<const uint4 *>(w_in + a)[lane];
                        uint4 wn = shfl_down_u4(w4);
                        if (lane == 31) wn = tail_u4(w_in + a + 128, r);
                        pick4(w4, wn, r, wt);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        id[k] = val[k] ? nbr_in[src[k]] : 0u;
                        if (need_w && val[k]) wt[k] = w_in[src[k]];
                    }
                }
                uint32_t y[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    y[k] = 0u;
                    if (!val[k]) continue;
                    if (id[k] >= V) { *bad = 1; continue; }
                    y[k] = new_id[id[k]];
                    if (pw_out && ((uint64_t)wt[k] >> (32 - wshift))) *wbig = 1;
                }
                if (full) {
                    if (nbr_out) *reinterpret_cast<uint4 *>(nbr_out + xl) = make_uint4(y[0], y[1], y[2], y[3]);
                    if (pw_out)
                        *reinterpret_cast<uint4 *>(pw_out + xl) =
                            make_uint4(y[0] | (wt[0] << wshift), y[1] | (wt[1] << wshift), y[2] | (wt[2] << wshift),
                                       y[3] | (wt[3] << wshift));
                    if (ew_out) {
                        uint4 *o = reinterpret_cast<uint4 *>(ew_out + xl);
                        o[0] = make_uint4(y[0], wt[0], y[1], wt[1]);
                        o[1] = make_uint4(y[2], wt[2], y[3], wt[3]);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if (!val[k] || id[k] >= V) continue;
                        const uint64_t x = xl + k;
                        if (nbr_out) nbr_out[x] = y[k];
                        if (ew_out) ew_out[x] = (uint64_t)y[k] | ((uint64_t)wt[k] << 32);
                        if (pw_out) pw_out[x] = y[k] | (wt[k] << wshift);
                    }
                }
            }
            e = stop;
        }
    }
}

// Offsets must be non-decreasing (the O(1) end checks run on the host).
__global__ void k_check_offsets(const uint64_t *__restrict__ off, uint64_t V, uint32_t *__restrict__ bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride)
        if (off[v] > off[v + 1]) *bad = 3;
}

__global__ void k_u32_to_u64(const uint32_t *__restrict__ in, uint64_t n, uint64_t *__restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = in[i];
}

__global__ void k_sum_u32(const uint32_t *__restrict__ in, uint64_t n, unsigned long long *__restrict__ sum) {
    __shared__ uint64_t sh[33];
    uint64_t s = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) s += in[i];
    s = block_sum_u64(s, sh);
    if (threadIdx.x == 0 && s) atomicAdd(sum, (unsigned long long)s);
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
static unsigned grid_for(uint64_t n, int threads = 256, uint64_t cap = num_sms() * 32) {
    uint64_t b = (n + threads - 1) / threads;
    if (b > cap) b = cap;
    if (b == 0) b = 1;
    return (unsigned)b;
}

static void parallel_memcpy(void *dst, const void *src, uint64_t bytes) {
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (bytes < (64ull << 20)) nt = 1;
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t) {
        uint64_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
        th.emplace_back([=] { std::memcpy((char *)dst + a, (const char *)src + a, b - a); });
    }
    for (auto &x : th) x.join();
}

// Maps a caller host array for device reads: cudaHostRegister in place, or a
// temporary pinned copy if registration is refused.
// Registrations of caller arrays are reference-counted process-wide: several
// handles (e.g. the ranks of an in-process group) may load from the same arrays
// at once, and the first to finish must not unregister memory another is reading.
static std::mutex g_reg_mu;
struct RegEntry { uint64_t bytes; int refs; const void *dev; };
static std::unordered_map<const void *, RegEntry> g_reg;

struct HostView {
    const void *dev = nullptr;
    const void *reg = nullptr;  // registry key (registered by us, refcounted)
    void *tmp = nullptr;        // pinned copy (to free)
    void open(const void *p, uint64_t bytes) {
        if (!p || bytes == 0) return;
        std::lock_guard<std::mutex> l(g_reg_mu);
        auto it = g_reg.find(p);
        if (it != g_reg.end() && it->second.bytes >= bytes) {
            ++it->second.refs;
            reg = p;
            dev = it->second.dev;
            return;
        }
        cudaError_t e = cudaHostRegister((void *)p, bytes, cudaHostRegisterMapped | cudaHostRegisterReadOnly);
        if (e != cudaSuccess) {
            cudaGetLastError();
            e = cudaHostRegister((void *)p, bytes, cudaHostRegisterMapped);
        }
        if (e == cudaSuccess) {
            void *d = nullptr;
            HYT_CUDA(cudaHostGetDevicePointer(&d, (void *)p, 0));
            g_reg[p] = RegEntry{bytes, 1, d};
            reg = p;
            dev = d;
            return;
        }
        cudaGetLastError();
        cudaPointerAttributes at{};
        if (e == cudaErrorHostMemoryAlreadyRegistered && cudaPointerGetAttributes(&at, p) == cudaSuccess &&
            at.devicePointer) {
            dev = at.devicePointer;         // registered by the caller: theirs to release
            return;
        }
        cudaGetLastError();
        HYT_CUDA(cudaHostAlloc(&tmp, bytes, cudaHostAllocMapped));
        parallel_memcpy(tmp, p, bytes);
        void *d = nullptr;
        HYT_CUDA(cudaHostGetDevicePointer(&d, tmp, 0));
        dev = d;
    }
    void close() {
        if (reg) {
            std::lock_guard<std::mutex> l(g_reg_mu);
            auto it = g_reg.find(reg);
            if (it != g_reg.end() && --it->second.refs == 0) {
                cudaHostUnregister((void *)reg);
                g_reg.erase(it);
            }
        }
        if (tmp) cudaFreeHost(tmp);
        reg = nullptr;
        tmp = nullptr;
        dev = nullptr;
    }
};

// ---------------------------------------------------------------------------
// load, in two phases.
//   plan: validate the degrees, hub-sort on the GPU, build the new
//         offsets and this rank's vertex range.  Needs only O(V) data: the
//         caller's offsets (or out-degrees) and in-degrees (computed from the
//         caller's edges when not given).
//   rows: pin this rank's edge store and write the relabelled rows into it,
//         reading the caller's rows in place through a host mapping: either the
//         whole CSR (hyt_load_csr) or only the rows of this rank's range in
//         internal order (hyt_load_shard_rows: no process holds the whole graph).
// ---------------------------------------------------------------------------
static double wall_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Phase {
    hyt_graph *g;
    bool verbose = getenv("HYT_VERBOSE") != nullptr;
    double t = wall_ms();
    void operator()(const char *name) {
        if (!verbose) return;
        cudaStreamSynchronize(g->main);
        const double n = wall_ms();
        fprintf(stderr, "[hyt load] %-28s %8.1f ms\n", name, n - t);
        t = n;
    }
};

// Pinning the store on a host thread while the GPU computes the hub sort (one
// rank owns every edge, so the store's size is known before the plan).
struct EarlyStore {
    std::thread th;
    void *n = nullptr, *w = nullptr;
    uint64_t nbytes = 0, wbytes = 0;
    std::exception_ptr err;
    ~EarlyStore() {
        if (th.joinable()) th.join();
        pinned_free(n);
        pinned_free(w);
    }
};

struct Temps {   // arena temporaries, released in reverse order
    Arena &A;
    std::vector<void *> v;
    explicit Temps(Arena &a) : A(a) {}
    void *get(uint64_t bytes, const char *what) { void *p = A.alloc(bytes, what); v.push_back(p); return p; }
    void drop(void *p) {
        A.release(p);
        v.erase(std::find(v.begin(), v.end(), p));
    }
    ~Temps() { for (auto it = v.rbegin(); it != v.rend(); ++it) A.release(*it); }
};

static uint32_t read_flag(uint32_t *bad, cudaStream_t st) {
    uint32_t h = 0;
    HYT_CUDA(copy_sync(&h, bad, 4, st));
    return h;
}

// Host copy of the internal offsets (partitioning, filter spans, host gathers).
static void fetch_host_offsets(hyt_graph *g, cudaStream_t st) {
    g->off_h.resize(g->V + 1);
    HYT_CUDA(copy_sync(g->off_h.data(), g->off_d, (g->V + 1) * 8, st));
    HYT_REQUIRE(g->off_h[g->V] == g->E, HYT_ESTATE, "internal: permuted offsets do not sum to E");
    g->off_h_pending = false;
}

// off_host: caller offsets u64[V+1] (full CSR), or out_deg u32[V] (shard);
// in_deg u32[V] or null (then nbr_dev, the caller's full ids mapped, is counted).
static void plan_phase(hyt_graph *g, uint64_t V, uint64_t E, const uint64_t *off_host, const uint32_t *out_deg,
                       const uint32_t *in_deg, const uint32_t *nbr_dev, uint32_t flags, Phase &phase) {
    Arena &A = g->arena;
    cudaStream_t st = g->main;
    g->V = V; g->E = E; g->symmetric = (flags & HYT_SYMMETRIC) != 0;
    g->off_d = arena_new<uint64_t>(A, V + 1, "offsets");
    g->new_id_d = arena_new<uint32_t>(A, V, "new_id");
    g->old_of_d = arena_new<uint32_t>(A, V, "old_of");
    g->din_d = arena_new<uint32_t>(A, V, "in_degree");
    // caller offsets: kept until the rows are loaded (the full-CSR relabel reads them)
    g->ld_off_old = arena_new<uint64_t>(A, V + 1, "load: caller offsets");
    uint64_t *off_old = g->ld_off_old;
    Temps T(A);
    uint32_t *din = (uint32_t *)T.get(V * 4 + 16, "load: in-degree");
    uint32_t *bad = (uint32_t *)T.get(16, "load: flag");
    uint32_t *nonhub = (uint32_t *)T.get(V * 4 + 16, "load: non-hub flags");
    uint32_t *nonhub_scan = (uint32_t *)T.get(V * 4 + 16, "load: non-hub scan");
    void *stemp = T.get(scan_temp_bytes(V + 1) + 16, "load: scan temp");
    HYT_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    if (off_host) {
        HYT_CUDA(cudaMemcpyAsync(off_old, off_host, (V + 1) * 8, cudaMemcpyHostToDevice, st));
        k_check_offsets<<<grid_for(V), 256, 0, st>>>(off_old, V, bad);
        HYT_REQUIRE(read_flag(bad, st) == 0, HYT_EINVAL, "offsets not non-decreasing");
    } else {   // offsets = exclusive scan of the out-degrees (V+1 items, the last 0)
        uint32_t *od = (uint32_t *)T.get((V + 1) * 4 + 16, "load: out-degrees");
        HYT_CUDA(cudaMemcpyAsync(od, out_deg, V * 4, cudaMemcpyHostToDevice, st));
        HYT_CUDA(cudaMemsetAsync(od + V, 0, 4, st));
        exclusive_scan<uint32_t, uint64_t>(od, off_old, V + 1, stemp, st);
        HYT_CUDA(copy_sync(&E, off_old + V, 8, st));
        g->E = E;
        T.drop(od);
    }
    if (in_deg) {
        HYT_CUDA(cudaMemcpyAsync(din, in_deg, V * 4, cudaMemcpyHostToDevice, st));
        unsigned long long *sum = (unsigned long long *)T.get(16, "load: in-degree sum");
        HYT_CUDA(cudaMemsetAsync(sum, 0, 8, st));
        k_sum_u32<<<grid_for(V, 256, num_sms() * 8), 256, 0, st>>>(din, V, sum);
        unsigned long long se = 0;
        HYT_CUDA(copy_sync(&se, sum, 8, st));
        HYT_REQUIRE(se == E, HYT_EINVAL, "sum of in-degrees != sum of out-degrees");
        T.drop(sum);
    } else {
        HYT_CUDA(cudaMemsetAsync(din, 0, V * 4, st));
        if (E) k_indeg<<<grid_for(E), 256, 0, st>>>(nbr_dev, E, V, din, bad);
        HYT_REQUIRE(read_flag(bad, st) == 0, HYT_EINVAL, "neighbour id >= V");
    }
    if (flags & HYT_SYMMETRIC) {
        k_sym_degrees<<<grid_for(V), 256, 0, st>>>(off_old, din, V, bad);
        HYT_REQUIRE(read_flag(bad, st) == 0, HYT_EINVAL,
                    "HYT_SYMMETRIC: some vertex's in-degree differs from its out-degree");
    }
    phase("degrees");

    // ---- hub sort: top h = ceil(frac*V) by D_o*D_i ----
    const uint64_t fden = 1000000;
    const uint64_t fnum = (uint64_t)(g->prm.hub_fraction * (double)fden + 0.5);
    uint64_t h = (flags & HYT_NO_HUBSORT) ? 0 : (fnum * V + fden - 1) / fden;
    if (h > V) h = V;
    k_fill_u32<<<grid_for(V), 256, 0, st>>>(nonhub, V, 1u);
    if (h > 0) {
        // exact radix select of the h-th largest key T (8 passes of 8 bits), then
        // only the h hubs are sorted: O(V) memory instead of a full-V key sort
        unsigned long long *hist = (unsigned long long *)T.get(256 * 8, "load: select histogram");
        std::vector<unsigned long long> hh(256);
        uint64_t prefix = 0, mask = 0, kk = h;
        for (int pass = 0; pass < 8; ++pass) {
            const int shift = 56 - 8 * pass;
            HYT_CUDA(cudaMemsetAsync(hist, 0, 256 * 8, st));
            k_key_hist<<<grid_for(V, 256, num_sms() * 8), 256, 0, st>>>(off_old, din, V, prefix, mask, shift, hist);
            HYT_CUDA(copy_sync(hh.data(), hist, 256 * 8, st));
            unsigned long long acc = 0;
            int d = 255;
            for (; d > 0; --d) {
                if (acc + hh[d] >= kk) break;
                acc += hh[d];
            }
            kk -= acc;
            prefix |= (uint64_t)d << shift;
            mask |= 0xFFull << shift;
        }
        phase("  radix select (8 passes)");
        const uint64_t Tkey = prefix, ties = kk;      // hubs: key > T, plus `ties` of key == T by id
        k_tie_flags<<<grid_for(V), 256, 0, st>>>(off_old, din, V, Tkey, nonhub);
        exclusive_scan<uint32_t, uint32_t>(nonhub, nonhub_scan, V, stemp, st);
        k_hub_flags<<<grid_for(V), 256, 0, st>>>(off_old, din, V, Tkey, ties, nonhub_scan, nonhub);
        exclusive_scan<uint32_t, uint32_t>(nonhub, nonhub_scan, V, stemp, st);
        uint32_t *hid = (uint32_t *)T.get(h * 4 + 16, "load: hub ids");
        uint32_t *hid2 = (uint32_t *)T.get(h * 4 + 16, "load: hub ids (scratch)");
        uint64_t *hkey = (uint64_t *)T.get(h * 8 + 16, "load: hub keys");
        uint64_t *hkey2 = (uint64_t *)T.get(h * 8 + 16, "load: hub keys (scratch)");
        uint32_t *sflag = (uint32_t *)T.get(h * 4 + 16, "load: sort flags");
        uint32_t *spos = (uint32_t *)T.get(h * 4 + 16, "load: sort positions");
        unsigned long long *smax = (unsigned long long *)T.get(16, "load: sort max");
        // hub ids in ascending id order, so the stable sort keeps ties by id (C11)
        k_scatter_hubs<<<grid_for(V), 256, 0, st>>>(off_old, din, V, nonhub, nonhub_scan, hid, hkey);
        phase("  hub flags + scatter");
        sort_desc_stable(hkey, hid, hkey2, hid2, h, sflag, spos, stemp, smax, st);
        phase("  sort the hubs");
        k_fill_u32<<<grid_for(V), 256, 0, st>>>(nonhub, V, 1u);
        k_mark_hubs<<<grid_for(h), 256, 0, st>>>(hid, h, g->new_id_d, nonhub);
        HYT_CUDA(cudaStreamSynchronize(st));
        for (void *q : {(void *)smax, (void *)spos, (void *)sflag, (void *)hkey2, (void *)hkey, (void *)hid2,
                        (void *)hid, (void *)hist})
            T.drop(q);
    }
    uint64_t *deg2 = (uint64_t *)T.get((V + 1) * 8, "load: degrees");
    exclusive_scan<uint32_t, uint32_t>(nonhub, nonhub_scan, V, stemp, st);
    k_finish_perm<<<grid_for(V), 256, 0, st>>>(V, h, nonhub, nonhub_scan, off_old, din, g->new_id_d,
                                              g->old_of_d, deg2, g->din_d);
    exclusive_scan<uint64_t, uint64_t>(deg2, g->off_d, V + 1, stemp, st);
    phase("  permutation + new offsets");
    if (g->world == 1 && off_host) {
        // one rank serves every edge: the store range is known without the host copy
        // of the offsets, which rows_phase fetches while the relabel runs
        HYT_CUDA(cudaStreamSynchronize(st));
        g->store_v_lo = 0;
        g->store_v_hi = V;
        g->off_h_pending = true;
    } else {
        fetch_host_offsets(g, st);
        rank_vertex_range(g->off_h, g->world, g->rank, &g->store_v_lo, &g->store_v_hi);
    }
    phase("hub sort + new offsets");
}

// bits of the largest vertex id (the shift of a packed record's weight)
static uint32_t id_bits(uint64_t V) {
    uint32_t b = 1;
    while (b < 64 && (V - 1) >> b) ++b;
    return b;
}
// packed SSSP records are tried when asked for and an id leaves >= 1 bit of a u32
static bool pack_planned(const hyt_graph *g, uint64_t V, bool weighted) {
    return weighted && g->prm.pack_weights && id_bits(V) < 32;
}

// The pinned mapped edge store of this rank's vertex range (the whole
// graph at world 1), from a 16-byte chunk boundary, 16-B padded so chunk loads
// never overrun.  row_start: null = full caller arrays (indexed by off_old),
// else the device copy of the caller's local row offsets.  adopt_ids: the
// caller's local id array IS the u32 store (HYT_ADOPT_HOST, no relabel).
static void rows_phase(hyt_graph *g, const uint64_t *row_start, const uint32_t *nbr_dev, const uint32_t *w_dev,
                       bool weighted, EarlyStore *early, const uint32_t *adopt_ids, Phase &phase) {
    cudaStream_t st = g->main;
    const uint64_t V = g->V;
    g->weighted = weighted;
    const uint64_t e_lo = g->off_h_pending ? 0 : g->off_h[g->store_v_lo];
    const uint64_t e_hi = g->off_h_pending ? g->E : g->off_h[g->store_v_hi];
    g->store_c0[0] = e_lo / 4;                          // first chunk of u32 ids
    g->store_c0[1] = e_lo / 2;                          // first chunk of u64 records
    const uint64_t nbase = g->store_c0[0] * 4, wbase = g->store_c0[1] * 2;
    const uint64_t nbytes = (((e_hi - nbase) * 4 + 15) & ~15ull) + 32;
    const bool pack = pack_planned(g, V, weighted);
    // packed records share the ids' chunk geometry (4 B per edge)
    const uint64_t wbytes = pack ? nbytes : (((e_hi - wbase) * 8 + 15) & ~15ull) + 32;
    g->wshift = pack ? id_bits(V) : 0;
    if (adopt_ids) {
        g->nbr_h = const_cast<uint32_t *>(adopt_ids);
        g->nbr_adopted = true;
    }
    if (early && early->th.joinable()) {
        early->th.join();
        if (early->err) std::rethrow_exception(early->err);
        HYT_REQUIRE((adopt_ids || nbytes == early->nbytes) && (!weighted || wbytes == early->wbytes), HYT_ESTATE,
                    "edge store size mismatch");
        if (!adopt_ids) { g->nbr_h = (uint32_t *)early->n; early->n = nullptr; }   // ownership moves
        if (pack) g->pw_h = (uint32_t *)early->w;
        else g->ew_h = (uint64_t *)early->w;
        early->w = nullptr;
    } else {
        if (!adopt_ids) g->nbr_h = (uint32_t *)pinned_alloc(nbytes);   // zero-filled (padding included)
        if (weighted && pack) g->pw_h = (uint32_t *)pinned_alloc(wbytes);
        else if (weighted) g->ew_h = (uint64_t *)pinned_alloc(wbytes);
    }
    g->store_bytes = (adopt_ids ? 0 : nbytes) + (weighted ? wbytes : 0);
    uint32_t *nbr_out = nullptr, *pw_out = nullptr;
    uint64_t *ew_out = nullptr;
    if (!adopt_ids) HYT_CUDA(cudaHostGetDevicePointer((void **)&nbr_out, g->nbr_h, 0));
    if (weighted && pack) HYT_CUDA(cudaHostGetDevicePointer((void **)&pw_out, g->pw_h, 0));
    else if (weighted) HYT_CUDA(cudaHostGetDevicePointer((void **)&ew_out, g->ew_h, 0));
    phase("pin edge store");
    Temps T(g->arena);
    uint32_t *bad = (uint32_t *)T.get(16, "load: flag");
    uint32_t *wbig = (uint32_t *)T.get(16, "load: weight flag");
    HYT_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    HYT_CUDA(cudaMemsetAsync(wbig, 0, 4, st));
    if (e_hi > e_lo && (nbr_out || ew_out || pw_out || row_start)) {
        k_relabel_tiles<<<num_sms() * 4, 512, 0, st>>>(V, e_lo, e_hi, g->ld_off_old, g->off_d, g->old_of_d, g->new_id_d,
                                                      row_start, g->store_v_lo, g->store_v_hi, nbr_dev, w_dev,
                                                      nbr_out ? nbr_out - nbase : nullptr,
                                                      ew_out ? ew_out - wbase : nullptr,
                                                      pw_out ? pw_out - nbase : nullptr, g->wshift, wbig, bad);
    }
    if (g->off_h_pending) {   // the host offsets while the relabel kernel runs (its own stream)
        cudaStream_t side = nullptr;
        HYT_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        try {
            fetch_host_offsets(g, side);
        } catch (...) {
            cudaStreamDestroy(side);
            throw;
        }
        cudaStreamDestroy(side);
    }
    HYT_REQUIRE(read_flag(bad, st) == 0, HYT_EINVAL, "neighbour id >= V");
    HYT_CUDA(cudaGetLastError());
    if (pw_out && read_flag(wbig, st)) {
        // a weight does not fit beside the id: the unpacked u64 records instead
        pinned_free(g->pw_h);
        g->pw_h = nullptr;
        g->wshift = 0;
        const uint64_t wb = (((e_hi - wbase) * 8 + 15) & ~15ull) + 32;
        g->ew_h = (uint64_t *)pinned_alloc(wb);
        g->store_bytes = (adopt_ids ? 0 : nbytes) + wb;
        HYT_CUDA(cudaHostGetDevicePointer((void **)&ew_out, g->ew_h, 0));
        k_relabel_tiles<<<num_sms() * 4, 512, 0, st>>>(V, e_lo, e_hi, g->ld_off_old, g->off_d, g->old_of_d, g->new_id_d,
                                                      row_start, g->store_v_lo, g->store_v_hi, nbr_dev, w_dev,
                                                      nullptr, ew_out - wbase, nullptr, 0, wbig, bad);
        HYT_CUDA(cudaStreamSynchronize(st));
        HYT_CUDA(cudaGetLastError());
    }
    phase("relabel edges (zero-copy)");
}

static void load_done(hyt_graph *g) {
    g->arena.release(g->ld_off_old);
    g->ld_off_old = nullptr;
    g->planned = false;
    g->loaded = true;
}

static void load_fail(hyt_graph *g) {
    cudaStreamSynchronize(g->main);
    g->off_h_pending = false;
    if (g->ld_off_old) g->arena.release(g->ld_off_old);
    g->ld_off_old = nullptr;
    g->planned = false;
}

static void check_offsets(const uint64_t *off, uint64_t V, uint64_t E) {
    HYT_REQUIRE(off[0] == 0, HYT_EINVAL, "off[0] != 0");
    HYT_REQUIRE(off[V] == E, HYT_EINVAL, "off[V] != E");
    // monotonicity is checked on the GPU (k_check_offsets) once the offsets are there
}

void load_graph(hyt_graph *g, uint64_t V, uint64_t E, const uint64_t *off, const uint32_t *nbr,
                const uint32_t *w, uint32_t flags) {
    Phase phase{g};
    HYT_REQUIRE(!g->loaded && !g->planned, HYT_ESTATE, "graph already loaded");
    HYT_REQUIRE(V > 0 && V < (1ull << 32), HYT_EINVAL, "V must be in [1, 2^32)");
    HYT_REQUIRE(off != nullptr && (E == 0 || nbr != nullptr), HYT_EINVAL, "null CSR array");
    check_offsets(off, V, E);
    const bool adopt = (flags & HYT_ADOPT_HOST) != 0;
    HYT_REQUIRE(!adopt || (flags & HYT_NO_HUBSORT), HYT_EINVAL, "HYT_ADOPT_HOST needs HYT_NO_HUBSORT");
    HYT_REQUIRE(!adopt || ((uintptr_t)nbr & 15) == 0, HYT_EINVAL, "HYT_ADOPT_HOST needs a 16-byte aligned id array");
    HYT_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = g->main;
    phase("validate");
    EarlyStore early;
    if (g->world == 1) {
        const int dev = g->device;
        const bool weighted = w != nullptr;
        early.nbytes = ((E * 4 + 15) & ~15ull) + 32;
        early.wbytes = pack_planned(g, V, weighted) ? early.nbytes : ((E * 8 + 15) & ~15ull) + 32;
        early.th = std::thread([&early, dev, weighted, adopt] {
            try {
                cudaSetDevice(dev);
                if (!adopt) early.n = pinned_alloc(early.nbytes);
                if (weighted) early.w = pinned_alloc(early.wbytes);
            } catch (...) {
                early.err = std::current_exception();
            }
        });
    }
    HostView vn, vw;
    try {
        // an adopted id array is the store: register it up to its last 16-byte chunk
        // (filter copies and chunk loads read whole chunks; the base is 16-B aligned,
        // so the rounded end stays inside the last element's page)
        vn.open(nbr, adopt ? ((E * 4 + 15) & ~15ull) : E * 4);
        if (w) vw.open(w, E * 4);
        HYT_REQUIRE(!adopt || !vn.tmp, HYT_ENOMEM, "HYT_ADOPT_HOST: the id array could not be registered in place");
        phase("map caller arrays");
        plan_phase(g, V, E, off, nullptr, nullptr, (const uint32_t *)vn.dev, flags, phase);
        const uint32_t *adopt_ids = nullptr;
        if (adopt) {
            const uint64_t first = g->off_h_pending ? 0 : g->off_h[g->store_v_lo];
            HYT_REQUIRE(first % 4 == 0, HYT_EINVAL,
                        "HYT_ADOPT_HOST: this rank's first edge is not on a 16-byte chunk boundary");
            adopt_ids = nbr + first;
        }
        rows_phase(g, nullptr, (const uint32_t *)vn.dev, (const uint32_t *)vw.dev, w != nullptr, &early, adopt_ids,
                   phase);
        HYT_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        load_fail(g);
        vn.close(); vw.close();
        throw;
    }
    if (adopt) {   // the caller's ids stay mapped for the handle's lifetime
        g->adopt_key = vn.reg;
        g->adopt_dev = vn.dev;
        vn.reg = nullptr;
    }
    vn.close(); vw.close();
    load_done(g);
    phase("unmap + release");
}

void load_shard_begin(hyt_graph *g, uint64_t V, const uint32_t *out_deg, const uint32_t *in_deg, uint32_t flags,
                      uint64_t *row_lo, uint64_t *row_hi, uint64_t *edges) {
    Phase phase{g};
    HYT_REQUIRE(!g->loaded && !g->planned, HYT_ESTATE, "graph already loaded");
    HYT_REQUIRE(V > 0 && V < (1ull << 32), HYT_EINVAL, "V must be in [1, 2^32)");
    HYT_REQUIRE(out_deg && in_deg, HYT_EINVAL, "null degree array");
    HYT_REQUIRE(!(flags & HYT_ADOPT_HOST) || (flags & HYT_NO_HUBSORT), HYT_EINVAL,
                "HYT_ADOPT_HOST needs HYT_NO_HUBSORT");
    HYT_CUDA(cudaSetDevice(g->device));
    HostView vo, vi;
    try {
        vo.open(out_deg, V * 4);
        vi.open(in_deg, V * 4);
        plan_phase(g, V, 0, nullptr, out_deg, in_deg, nullptr, flags, phase);
        HYT_CUDA(cudaStreamSynchronize(g->main));
    } catch (...) {
        load_fail(g);
        vo.close(); vi.close();
        throw;
    }
    vo.close(); vi.close();
    g->ld_flags = flags;
    g->planned = true;
    *row_lo = g->store_v_lo;
    *row_hi = g->store_v_hi;
    *edges = g->off_h[g->store_v_hi] - g->off_h[g->store_v_lo];
}

void shard_rows(hyt_graph *g, uint32_t *rows, uint64_t n) {
    HYT_REQUIRE(g->planned || g->loaded, HYT_ESTATE, "call hyt_load_shard_begin first");
    HYT_REQUIRE(n == g->store_v_hi - g->store_v_lo, HYT_EINVAL, "row count != row_hi - row_lo");
    HYT_CUDA(cudaSetDevice(g->device));
    if (n) HYT_CUDA(copy_sync(rows, g->old_of_d + g->store_v_lo, n * 4, g->main));
}

void load_shard_rows(hyt_graph *g, uint64_t nrows, const uint64_t *row_off, const uint32_t *nbr,
                     const uint32_t *w) {
    Phase phase{g};
    HYT_REQUIRE(g->planned, HYT_ESTATE, "call hyt_load_shard_begin first");
    HYT_REQUIRE(nrows == g->store_v_hi - g->store_v_lo, HYT_EINVAL, "row count != row_hi - row_lo");
    HYT_REQUIRE(row_off != nullptr, HYT_EINVAL, "null row offsets");
    HYT_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = g->main;
    const uint64_t e_lo = g->off_h[g->store_v_lo], e_hi = g->off_h[g->store_v_hi], n_e = e_hi - e_lo;
    HYT_REQUIRE(row_off[0] == 0 && row_off[nrows] == n_e, HYT_EINVAL,
                "row offsets must start at 0 and end at this rank's edge count");
    HYT_REQUIRE(n_e == 0 || nbr != nullptr, HYT_EINVAL, "null id array");
    // every row's degree must be the one the plan used (the internal offsets)
    for (uint64_t i = 0; i < nrows; ++i)
        HYT_REQUIRE(row_off[i + 1] - row_off[i] == g->off_h[g->store_v_lo + i + 1] - g->off_h[g->store_v_lo + i],
                    HYT_EINVAL, "row " + std::to_string(i) + ": degree differs from the out-degree given to begin");
    const bool adopt = (g->ld_flags & HYT_ADOPT_HOST) != 0;
    HYT_REQUIRE(!adopt || (e_lo % 4 == 0 && ((uintptr_t)nbr & 15) == 0), HYT_EINVAL,
                "HYT_ADOPT_HOST needs a 16-byte aligned id array starting on a 16-byte chunk boundary of the "
                "global edge order");
    HostView vn, vw;
    Temps T(g->arena);
    try {
        vn.open(nbr, adopt ? ((n_e * 4 + 15) & ~15ull) : n_e * 4);
        if (w) vw.open(w, n_e * 4);
        HYT_REQUIRE(!adopt || !vn.tmp, HYT_ENOMEM, "HYT_ADOPT_HOST: the id array could not be registered in place");
        uint64_t *rs = (uint64_t *)T.get((nrows + 1) * 8 + 16, "load: row starts");
        HYT_CUDA(copy_sync(rs, row_off, (nrows + 1) * 8, st));
        rows_phase(g, rs, (const uint32_t *)vn.dev, (const uint32_t *)vw.dev, w != nullptr, nullptr,
                   adopt ? nbr : nullptr, phase);
        HYT_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        vn.close(); vw.close();
        throw;
    }
    if (adopt) {
        g->adopt_key = vn.reg;
        g->adopt_dev = vn.dev;
        vn.reg = nullptr;
    }
    vn.close(); vw.close();
    load_done(g);
}

// Drop the registration of an adopted id array (hyt_free).
void release_adopted(hyt_graph *g) {
    if (!g->nbr_adopted) return;
    if (g->adopt_key) {
        std::lock_guard<std::mutex> l(g_reg_mu);
        auto it = g_reg.find(g->adopt_key);
        if (it != g_reg.end() && --it->second.refs == 0) {
            cudaHostUnregister((void *)g->adopt_key);
            g_reg.erase(it);
        }
    }
    g->adopt_key = nullptr;
    g->nbr_h = nullptr;
    g->nbr_adopted = false;
}

}  // namespace hyt
