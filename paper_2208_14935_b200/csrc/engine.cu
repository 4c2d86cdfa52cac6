// engine.cu -- hyt_run: the per-iteration hybrid-transfer loop.
//
// One iteration:
//   1. plan kernels on the GPU: activity + engine selection per partition
//      (Alg. 1 L2-12) and the per-engine queues ("pre-combine on GPU");
//   2. ONE device->host copy of the plan + one sync (Alg. 1 L13);
//   3. host: task combination into <= k-partition filter units (Alg. 1
//      L14-24, corrected loop SURVEY C9) and contribution-driven ordering
//      (hub-driven or delta-driven);
//   4. multi-stream dispatch: filter units first, in priority
//      order, each = async bulk copy + relax + one recompute pass;
//      then the merged zero-copy task (one kernel over Vz); then the
//      merged compaction task (host gather overlapping the GPU work, bulk copy,
//      relax over the compacted lists).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <numeric>
#include <thread>
#include "graph.h"

namespace hyt {

// ---------------------------------------------------------------------------
// arena
// ---------------------------------------------------------------------------
void *Arena::alloc(uint64_t bytes, const char *what) {
    bytes = (bytes + 255) & ~255ull;
    if (budget && used + bytes > budget)
        throw Err{HYT_ENOMEM, std::string("device budget exceeded allocating ") + what + " (" +
                                  std::to_string(bytes) + " B; used " + std::to_string(used) + " of " +
                                  std::to_string(budget) + ")"};
    void *p = nullptr;
    uint64_t top_before = ext_top;
    if (ext) {
        if (ext_top + bytes > ext_size) throw Err{HYT_ENOMEM, std::string("device arena exhausted: ") + what};
        p = ext + ext_top;
        ext_top += bytes;
    } else {
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw Err{HYT_ENOMEM, std::string("cudaMalloc failed for ") + what + ": " + cudaGetErrorString(e)};
        }
    }
    used += bytes;
    if (used > peak) peak = used;
    blocks.push_back({p, bytes, top_before, true});
    return p;
}

void Arena::release(void *p) {
    if (!p) return;
    for (auto it = blocks.rbegin(); it != blocks.rend(); ++it) {
        if (it->p == p && it->live) {
            it->live = false;
            used -= it->bytes;
            if (!ext) cudaFree(p);
            break;
        }
    }
    // pop dead blocks from the top (stack discipline for the external arena)
    while (!blocks.empty() && !blocks.back().live) {
        if (ext) ext_top = blocks.back().top_before;
        blocks.pop_back();
    }
}

void Arena::release_all() {
    for (auto &b : blocks)
        if (b.live && !ext) cudaFree(b.p);
    blocks.clear();
    used = 0;
    ext_top = 0;
}

CostParams make_cost(const Params &p, uint32_t d1, double cpu_ratio, double zr_rtt, double zs_rtt) {
    CostParams c;
    c.d1 = d1; c.d2 = p.d2; c.m = p.m; c.mr = p.mr;
    const uint64_t den = 1000000;
    c.an = (uint64_t)(p.alpha * den + 0.5); c.ad = den;
    c.bn = (uint64_t)(p.beta * den + 0.5); c.bd = den;
    c.gn = (uint64_t)(p.gamma * den + 0.5); c.gd = den;
    c.m_shift = -1;
    for (int k = 0; k < 63; ++k)
        if ((1ull << k) == p.m) c.m_shift = k;
    c.cd = 1000;
    c.cn = cpu_ratio > 0 ? (uint64_t)(cpu_ratio * 1000 + 0.5) : 0;
    c.zd = 1000;
    c.zn = (uint64_t)(p.zc_weight * 1000 + 0.5);
    c.zden = 1000000;
    c.zr = zr_rtt > 0 ? std::max<uint64_t>(1, (uint64_t)(zr_rtt * 1e6 + 0.5)) : 0;
    c.zs = zs_rtt > 0 ? (uint64_t)(zs_rtt * 1e6 + 0.5) : 0;
    return c;
}

// ---------------------------------------------------------------------------
// host partitioner and task combination
// ---------------------------------------------------------------------------
static void greedy_bounds(const std::vector<uint64_t> &off, uint64_t lo, uint64_t end, uint64_t d1, uint64_t target,
                          std::vector<uint64_t> &b) {
    // greedy sweep over [lo, end) (close a partition when the next vertex would
    // exceed target, unless empty), realised by binary search on the offsets
    while (lo < end) {
        // largest hi with (off[hi] - off[lo]) * d1 <= target, at least lo + 1
        const uint64_t lim = off[lo] + target / d1;
        uint64_t hi = std::upper_bound(off.begin() + lo + 1, off.begin() + end + 1, lim) - off.begin() - 1;
        if (hi <= lo) hi = lo + 1;
        b.push_back(hi);
        lo = hi;
    }
}

std::vector<uint64_t> partition_bounds(const std::vector<uint64_t> &off, uint64_t d1, uint64_t target) {
    std::vector<uint64_t> b{0};
    greedy_bounds(off, 0, off.size() - 1, d1, target, b);
    return b;
}

void rank_vertex_range(const std::vector<uint64_t> &off, int world, int rank, uint64_t *v_lo, uint64_t *v_hi) {
    const uint64_t V = off.size() - 1, E = off[V];
    auto cut = [&](int r) -> uint64_t {
        if (r <= 0) return 0;
        if (r >= world) return V;
        const uint64_t target = (uint64_t)((unsigned __int128)E * (uint64_t)r / (uint64_t)world);
        return std::lower_bound(off.begin(), off.end() - 1, target) - off.begin();
    };
    *v_lo = cut(rank);
    *v_hi = std::max(*v_lo, cut(rank + 1));
}

std::vector<uint64_t> partition_bounds_ranked(const std::vector<uint64_t> &off, uint64_t d1, uint64_t target,
                                              int world) {
    std::vector<uint64_t> b{0};
    for (int r = 0; r < world; ++r) {
        uint64_t lo, hi;
        rank_vertex_range(off, world, r, &lo, &hi);
        greedy_bounds(off, lo, hi, d1, target, b);
    }
    return b;
}

int64_t combine_units(const uint8_t *p, uint64_t n, uint64_t k, uint64_t *units) {
    int64_t nu = 0;
    uint64_t i = 0;
    while (i < n) {
        if (p[i] != ENG_F) { ++i; continue; }
        const uint64_t start = i;
        uint64_t len = 0;
        while (i < n && p[i] == ENG_F && len < k) { ++i; ++len; }
        units[2 * nu] = start;
        units[2 * nu + 1] = i;
        ++nu;
    }
    return nu;
}

// Contribution-driven ordering of the filter units (SURVEY
// C12/C13): a unit's score is the sum of its partitions' scores (hub-driven: sum
// of D_o*D_i over active vertices; delta-driven: sum of delta); units run in
// descending score, ties by unit index (a stable sort of the identity order).
void order_units(int64_t nu, const uint64_t *units, const double *part_score, uint32_t *order) {
    std::vector<double> sc((size_t)std::max<int64_t>(nu, 0), 0.0);
    for (int64_t j = 0; j < nu; ++j) {
        for (uint64_t i = units[2 * j]; i < units[2 * j + 1]; ++i) sc[j] += part_score[i];
        order[j] = (uint32_t)j;
    }
    std::stable_sort(order, order + nu, [&](uint32_t x, uint32_t y) { return sc[x] > sc[y]; });
}

void rank_partitions(const std::vector<uint64_t> &off, const std::vector<uint64_t> &bounds, int world, int rank,
                     uint64_t *p_lo, uint64_t *p_hi) {
    // bounds from partition_bounds_ranked: every rank cut is a partition bound
    uint64_t lo, hi;
    rank_vertex_range(off, world, rank, &lo, &hi);
    *p_lo = std::lower_bound(bounds.begin(), bounds.end(), lo) - bounds.begin();
    *p_hi = std::lower_bound(bounds.begin(), bounds.end(), hi) - bounds.begin();
}

// The store an algorithm's relaxations read: SSSP the packed u32 records (pw_h) or
// the u64 records (ew_h), the others the u32 ids; *c0 = the store's first chunk.
const void *edge_store(const hyt_graph *g, int algo, uint64_t *c0) {
    if (algo == ALGO_SSSP && !g->pw_h) { *c0 = g->store_c0[1]; return g->ew_h; }
    *c0 = g->store_c0[0];
    return algo == ALGO_SSSP ? (const void *)g->pw_h : (const void *)g->nbr_h;
}

const uint4 *host_edges(const hyt_graph *g, int algo) {
    uint64_t c0 = 0;
    const uintptr_t base = (uintptr_t)edge_store(g, algo, &c0);
    return (const uint4 *)(base - c0 * 16);
}

// ---------------------------------------------------------------------------
// host thread pool (compaction gather)
// ---------------------------------------------------------------------------
class Pool {
  public:
    explicit Pool(unsigned n) {
        for (unsigned i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        { std::lock_guard<std::mutex> l(m_); stop_ = true; }
        cv_.notify_all();
        for (auto &t : th_) t.join();
    }
    unsigned size() const { return (unsigned)th_.size(); }
    // run fn(worker) on every worker and wait
    void run(const std::function<void(unsigned)> &fn) {
        {
            std::lock_guard<std::mutex> l(m_);
            fn_ = fn; pending_ = (unsigned)th_.size(); ++gen_;
        }
        cv_.notify_all();
        std::unique_lock<std::mutex> l(m_);
        done_.wait(l, [this] { return pending_ == 0; });
    }

  private:
    void loop(unsigned id) {
        uint64_t seen = 0;
        for (;;) {
            std::function<void(unsigned)> f;
            {
                std::unique_lock<std::mutex> l(m_);
                cv_.wait(l, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                f = fn_;
            }
            f(id);
            {
                std::lock_guard<std::mutex> l(m_);
                if (--pending_ == 0) done_.notify_all();
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    std::function<void(unsigned)> fn_;
    unsigned pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// ---------------------------------------------------------------------------
// run context (cached per handle and edge-record width)
// ---------------------------------------------------------------------------
struct EvPair { cudaEvent_t a, b; int tag; };
enum Tag { TAG_PLAN = 0, TAG_F = 1, TAG_C = 2, TAG_Z = 3, TAG_R = 4, TAG_RECOMP = 5, TAG_COPY = 6, TAG_RQ = 7 };

struct RunCtx {
    uint32_t d1 = 0;
    int algo = -1;
    uint64_t N = 0, p_lo = 0, p_hi = 0;
    std::vector<uint64_t> bounds;
    uint64_t *bounds_d = nullptr, *t_d = nullptr;
    PartIter *parts_d = nullptr, *parts_h = nullptr;
    SegHdr *hdr_d = nullptr, *hdr_h = nullptr;
    Items items{};                // plan items (device)
    std::vector<uint64_t> item_first;   // host copy: partition -> first item
    uint64_t n_items = 0, item_lo = 0, item_hi = 0;
    ItemAgg *iagg = nullptr;
    uint64_t *ibase = nullptr;
    QueueBufs q{};
    uint32_t *val = nullptr, *bm_a = nullptr, *bm_b = nullptr;
    float *rank = nullptr, *delta = nullptr;
    int S = 0;
    uint64_t k_eff = 4;           // filter partitions per unit, reduced under small budgets
    std::vector<uint4 *> slot;
    uint64_t slot_bytes = 0;
    std::vector<RangeBufs> rb;
    uint4 *cbuf[2] = {nullptr, nullptr};
    uint4 *hstage[2] = {nullptr, nullptr};
    uint64_t cbuf_bytes = 0;
    uint32_t *cq_v = nullptr;
    uint64_t *cq_pre = nullptr;
    uint64_t cq_cap = 0;
    uint32_t *snap = nullptr;     // multi-GPU: own-range values before the exchange
    // multi-GPU sparse exchange (§8f #3): full values at iteration start (min-algos),
    // own changed pairs, all ranks' pairs, own pair count
    uint32_t *snapfull = nullptr;
    uint2 *xsend = nullptr, *xrecv = nullptr;
    uint64_t xcap = 0;
    unsigned long long *xcnt = nullptr;
    uint64_t *red = nullptr;      // multi-GPU: device scratch for the active-count reduction
    uint64_t *racc = nullptr;     // recompute statistics accumulators (u64[4])
    uint32_t *outbuf = nullptr;   // u32[V] result staging for hyt_get_values
    uint4 *cache = nullptr;       // resident edge cache: chunks [cache_c0, ...) of partitions [p_lo, cache_hi)
    uint64_t cache_c0 = 0, cache_hi = 0, cache_bytes = 0;
    // fused peer push (exchange = 3): every rank's (values | delta, bitmap a, bitmap b)
    void *peer_ptr[kMaxPeers * 3] = {};
    std::vector<void *> peer_opened;
    uint4 *um = nullptr;          // ImpTM-UM: managed edge copy (cache points here)
    // pull iterations (§8f #4): slices of the lists longer than pull_heavy
    uint32_t *hs_v = nullptr;
    uint64_t *hs_e0 = nullptr, *hs_e1 = nullptr;
    uint64_t n_hs = 0;
    uint32_t *bm_glob = nullptr;  // multi-rank pull BFS: every rank's frontier (OR of own words)
    uint64_t v_lo = 0, v_hi = 0;  // own vertex range
    std::vector<void *> dev;      // arena blocks (released with the context)
    std::vector<void *> pinned;   // cudaHostAlloc blocks
    std::vector<cudaEvent_t> evpool;
    size_t ev_used = 0;
    std::vector<EvPair> pending;
    cudaEvent_t ev_cbuf[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev_done;
    Pool *pool = nullptr;
};

static RunCtx *&ctx_of(hyt_graph *g, int algo) { return *reinterpret_cast<RunCtx **>(&g->ctx[algo]); }

static void destroy_ctx(hyt_graph *g, RunCtx *c) {
    if (!c) return;
    cudaDeviceSynchronize();
    for (auto e : c->evpool) cudaEventDestroy(e);
    for (auto e : c->ev_done) cudaEventDestroy(e);
    for (auto e : c->ev_cbuf) if (e) cudaEventDestroy(e);
    for (auto it = c->dev.rbegin(); it != c->dev.rend(); ++it) g->arena.release(*it);
    for (auto p : c->pinned) pinned_free(p);
    if (c->um) cudaFree(c->um);
    dist_close_peers(c->peer_opened);
    delete c->pool;
    delete c;
}

static cudaEvent_t next_event(RunCtx *c) {
    if (c->ev_used == c->evpool.size()) {
        cudaEvent_t e;
        HYT_CUDA(cudaEventCreate(&e));
        c->evpool.push_back(e);
    }
    return c->evpool[c->ev_used++];
}

static void timed_begin(RunCtx *c, cudaStream_t st, EvPair &ep, int tag) {
    ep.a = next_event(c); ep.b = next_event(c); ep.tag = tag;
    HYT_CUDA(cudaEventRecord(ep.a, st));
}
static void timed_end(RunCtx *c, cudaStream_t st, EvPair &ep) {
    HYT_CUDA(cudaEventRecord(ep.b, st));
    c->pending.push_back(ep);
}

// Accumulate the timings of completed launches (call after a sync).
static void harvest(hyt_graph *g, RunCtx *c) {
    for (auto &ep : c->pending) {
        float ms = 0;
        HYT_CUDA(cudaEventElapsedTime(&ms, ep.a, ep.b));
        EngTime *t = nullptr;
        switch (ep.tag) {
            case TAG_PLAN: t = &g->plan_time; break;
            case TAG_RECOMP: t = &g->recompute_time; break;
            case TAG_COPY: t = &g->copy_time; break;
            case TAG_RQ: t = &g->rq_time; break;
            default: t = &g->eng_time[ep.tag]; break;
        }
        t->ms += ms;
        t->launches += 1;
    }
    c->pending.clear();
    c->ev_used = 0;
}

template <class T> static T *dalloc(hyt_graph *g, RunCtx *c, uint64_t n, const char *what) {
    T *p = arena_new<T>(g->arena, n, what);
    c->dev.push_back(p);
    return p;
}
template <class T> static T *halloc(RunCtx *c, uint64_t n) {
    void *p = pinned_alloc(n * sizeof(T) + 64);
    c->pinned.push_back(p);
    return (T *)p;
}

// Copy the edges of own partitions [p_lo, p_hi_cache) into device memory once;
// the plan then serves them as the resident engine (cost 0, no transfer).
static void fill_cache(hyt_graph *g, RunCtx *c, uint64_t p_hi_cache) {
    const uint64_t c0 = chunk_lo(g->off_h[c->bounds[c->p_lo]], c->d1);
    const uint64_t c1 = chunk_hi(g->off_h[c->bounds[p_hi_cache]], c->d1);
    c->cache = dalloc<uint4>(g, c, c1 - c0 + 1, "resident edge cache");
    HYT_CUDA(copy_sync(c->cache, host_edges(g, c->algo) + c0, (c1 - c0) * 16, g->main));
    c->cache_c0 = c0;
    c->cache_hi = p_hi_cache;
    c->cache_bytes = (c1 - c0) * 16;
}

// ImpTM-UM comparison engine: the own partitions' edges
// in managed memory advised ReadMostly, so the driver migrates (read-duplicates)
// pages on first touch and evicts them under pressure.  Served as engine R: the
// relax kernel dereferences the managed pointer directly.
static void fill_um(hyt_graph *g, RunCtx *c) {
    const uint64_t c0 = chunk_lo(g->off_h[c->bounds[c->p_lo]], c->d1);
    const uint64_t c1 = chunk_hi(g->off_h[c->bounds[c->p_hi]], c->d1);
    const uint64_t bytes = (c1 - c0 + 1) * 16;
    HYT_CUDA(cudaMallocManaged((void **)&c->um, bytes, cudaMemAttachGlobal));
    const char *src = reinterpret_cast<const char *>(host_edges(g, c->algo) + c0);
    char *dst = reinterpret_cast<char *>(c->um);
    const uint64_t n = (c1 - c0) * 16;
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned i = 0; i < nt; ++i)
        th.emplace_back([=]() {
            const uint64_t a = n * i / nt, b = n * (i + 1) / nt;
            if (b > a) std::memcpy(dst + a, src + a, b - a);
        });
    for (auto &t : th) t.join();
    HYT_CUDA(cudaMemAdvise(c->um, bytes, cudaMemAdviseSetReadMostly, g->device));
    c->cache = c->um;
    c->cache_c0 = c0;
    c->cache_hi = c->p_hi;
    c->cache_bytes = n;
}

// Slices of the long lists for pull iterations (one warp per slice).
static void build_pull_slices(hyt_graph *g, RunCtx *c) {
    const uint64_t H = g->prm.pull_heavy, S = 4096;
    std::vector<uint32_t> sv;
    std::vector<uint64_t> e0, e1;
    for (uint64_t v = c->v_lo; v < c->v_hi; ++v) {
        const uint64_t a = g->off_h[v], b = g->off_h[v + 1];
        if (b - a <= H) continue;
        for (uint64_t x = a; x < b; x += S) {
            sv.push_back((uint32_t)v);
            e0.push_back(x);
            e1.push_back(std::min(b, x + S));
        }
    }
    c->n_hs = sv.size();
    if (!c->n_hs) return;
    c->hs_v = dalloc<uint32_t>(g, c, c->n_hs, "pull slice vertices");
    c->hs_e0 = dalloc<uint64_t>(g, c, c->n_hs, "pull slice begin");
    c->hs_e1 = dalloc<uint64_t>(g, c, c->n_hs, "pull slice end");
    HYT_CUDA(copy_sync(c->hs_v, sv.data(), c->n_hs * 4, g->main));
    HYT_CUDA(copy_sync(c->hs_e0, e0.data(), c->n_hs * 8, g->main));
    HYT_CUDA(copy_sync(c->hs_e1, e1.data(), c->n_hs * 8, g->main));
}

// Grow the pinned host copy of the compaction queue to at least n entries (called
// between iterations, when nothing reads the old arrays).
static void ensure_cq(RunCtx *c, uint64_t n) {
    if (n <= c->cq_cap) return;
    const uint64_t cap = std::min<uint64_t>(c->q.cap, std::max<uint64_t>(n, 2 * c->cq_cap));
    for (void *old : {(void *)c->cq_v, (void *)c->cq_pre}) {
        c->pinned.erase(std::find(c->pinned.begin(), c->pinned.end(), old));
        pinned_free(old);
    }
    c->cq_v = nullptr;
    c->cq_pre = nullptr;
    c->cq_cap = 0;
    c->cq_v = halloc<uint32_t>(c, cap);
    c->cq_pre = halloc<uint64_t>(c, cap);
    c->cq_cap = cap;
}

static inline double now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static RunCtx *build_ctx(hyt_graph *g, int algo) {
    const Params &P = g->prm;
    RunCtx *c = new RunCtx();
    const bool verbose = getenv("HYT_VERBOSE") != nullptr;
    double tm = now_ms();
    auto mark = [&](const char *what) {
        if (!verbose) return;
        const double t = now_ms();
        fprintf(stderr, "[hyt ctx]   %-34s %8.1f ms\n", what, t - tm);
        tm = t;
    };
    try {
        c->algo = algo;
        c->d1 = (algo == ALGO_SSSP && !g->pw_h) ? 8 : 4;   // packed SSSP records: 4 B per edge
        const uint64_t V = g->V, W = (V + 31) / 32;
        c->bounds = partition_bounds_ranked(g->off_h, c->d1, P.partition_bytes, g->world);
        c->N = c->bounds.size() - 1;
        // ---- multi-GPU: the partitions of this rank's vertex range (~E/world edges) ----
        rank_partitions(g->off_h, c->bounds, g->world, g->rank, &c->p_lo, &c->p_hi);
        c->v_lo = c->bounds[c->p_lo];
        c->v_hi = c->bounds[c->p_hi];
        c->red = dalloc<uint64_t>(g, c, 2, "reduction scratch");
        c->racc = dalloc<uint64_t>(g, c, 4, "recompute statistics");
        c->outbuf = dalloc<uint32_t>(g, c, V, "result staging");
        if (g->multi && algo != ALGO_PR)
            c->snap = dalloc<uint32_t>(g, c, c->v_hi - c->v_lo + 1, "exchange snapshot");
        if (g->multi && P.exchange && P.exchange != 3) {
            // sparse pays only below V*4 / (8 * world) pairs per rank: size for that
            c->xcap = V / (2 * (uint64_t)g->world) + 1;
            c->xsend = dalloc<uint2>(g, c, c->xcap, "exchange pairs (own)");
            c->xrecv = dalloc<uint2>(g, c, c->xcap * g->world, "exchange pairs (all ranks)");
            c->xcnt = dalloc<unsigned long long>(g, c, 1, "exchange pair count");
            if (algo != ALGO_PR) c->snapfull = dalloc<uint32_t>(g, c, V, "exchange snapshot (full)");
        }
        // ---- vertex state (the paper assumes it fits) ----
        if (algo == ALGO_PR) {
            c->rank = dalloc<float>(g, c, V, "rank");
            c->delta = dalloc<float>(g, c, V, "delta");
        } else {
            c->val = dalloc<uint32_t>(g, c, V, "values");
        }
        mark("bounds + vertex state");
        c->bm_a = dalloc<uint32_t>(g, c, W + 1, "frontier");
        c->bm_b = dalloc<uint32_t>(g, c, W + 1, "next frontier");
        c->bounds_d = dalloc<uint64_t>(g, c, c->N + 1, "partition bounds");
        c->t_d = dalloc<uint64_t>(g, c, c->N, "partition edges");
        c->parts_d = dalloc<PartIter>(g, c, c->N, "partition plan");
        c->hdr_d = dalloc<SegHdr>(g, c, 1, "segment header");
        {   // plan items: <= kItemWords words inside one partition (static per run)
            std::vector<uint32_t> ip;
            std::vector<uint64_t> iw0, iw1;
            c->item_first.assign(c->N + 1, 0);
            for (uint64_t i = 0; i < c->N; ++i) {
                c->item_first[i] = ip.size();
                const uint64_t wl = c->bounds[i] >> 5, wh = (c->bounds[i + 1] + 31) >> 5;
                for (uint64_t w = wl; w < wh; w += kItemWords) {
                    ip.push_back((uint32_t)i);
                    iw0.push_back(w);
                    iw1.push_back(std::min(wh, w + kItemWords));
                }
            }
            c->item_first[c->N] = ip.size();
            c->n_items = ip.size();
            c->item_lo = c->item_first[c->p_lo];
            c->item_hi = c->item_first[c->p_hi];
            uint32_t *dp = dalloc<uint32_t>(g, c, c->n_items, "item partitions");
            uint64_t *d0 = dalloc<uint64_t>(g, c, c->n_items, "item words lo");
            uint64_t *d1w = dalloc<uint64_t>(g, c, c->n_items, "item words hi");
            uint64_t *df = dalloc<uint64_t>(g, c, c->N + 1, "partition first item");
            HYT_CUDA(copy_sync(dp, ip.data(), ip.size() * 4, g->main));
            HYT_CUDA(copy_sync(d0, iw0.data(), iw0.size() * 8, g->main));
            HYT_CUDA(copy_sync(d1w, iw1.data(), iw1.size() * 8, g->main));
            HYT_CUDA(copy_sync(df, c->item_first.data(), (c->N + 1) * 8, g->main));
            c->items.part = dp; c->items.w0 = d0; c->items.w1 = d1w; c->items.first = df;
            c->iagg = dalloc<ItemAgg>(g, c, c->n_items, "item aggregates");
            c->ibase = dalloc<uint64_t>(g, c, 2 * c->n_items, "item bases");
        }
        mark("plan items");
        // queue: at most one entry per vertex with out-edges
        uint64_t vnz = 0, max_part_v = 0;
        for (uint64_t v = 0; v < V; ++v) vnz += g->off_h[v + 1] > g->off_h[v];
        c->q.cap = vnz + 1;
        const uint64_t tot_chunks = chunk_hi(g->E, c->d1) + vnz;
        c->q.tile_cap = tot_chunks / kTile + 8;
        c->q.qv = dalloc<uint32_t>(g, c, c->q.cap, "queue vertices");
        c->q.qpre = dalloc<uint64_t>(g, c, c->q.cap, "queue prefix");
        c->q.qbeg = dalloc<uint64_t>(g, c, c->q.cap, "queue edge begin");
        c->q.qdeg = dalloc<uint32_t>(g, c, c->q.cap, "queue degree");
        c->q.qaux = algo == ALGO_PR ? dalloc<float>(g, c, c->q.cap, "queue contrib") : nullptr;
        c->q.tile = dalloc<uint32_t>(g, c, c->q.tile_cap, "tile map");
        mark("queue");
        // ---- host copies of the plan ----
        c->parts_h = halloc<PartIter>(c, c->N);
        c->hdr_h = halloc<SegHdr>(c, 1);
        std::vector<uint64_t> t(c->N);
        for (uint64_t i = 0; i < c->N; ++i) t[i] = g->off_h[c->bounds[i + 1]] - g->off_h[c->bounds[i]];
        HYT_CUDA(copy_sync(c->bounds_d, c->bounds.data(), (c->N + 1) * 8, g->main));
        HYT_CUDA(copy_sync(c->t_d, t.data(), c->N * 8, g->main));
        // ---- staging for filter units: S slots, each holds the largest unit span ----
        uint64_t k = std::max<uint64_t>(1, P.k);
        uint64_t max_span = 0;
        auto spans = [&](uint64_t kk) {
            max_span = 0; max_part_v = 0;
            for (uint64_t i = 0; i < c->N; ++i) {
                const uint64_t j = std::min(c->N, i + kk);
                const uint64_t c0 = chunk_lo(g->off_h[c->bounds[i]], c->d1);
                const uint64_t c1 = chunk_hi(g->off_h[c->bounds[j]], c->d1);
                max_span = std::max(max_span, (c1 - c0) * 16);
                max_part_v = std::max(max_part_v, c->bounds[j] - c->bounds[i]);
            }
        };
        spans(k);
        if (P.engine_mode == MODE_RESIDENT) {
            // every own partition's edges once into device memory
            fill_cache(g, c, c->p_hi);
        } else if (P.engine_mode == MODE_UM) {
            fill_um(g, c);
        } else {
            const uint64_t rq_bytes_per_v = 28 + 4 + (algo == ALGO_PR ? 8 : 0);
            (void)rq_bytes_per_v;
            auto range_bytes = [&]() {
                return max_part_v * rq_bytes_per_v + (max_span / 16 + max_part_v) / kTile * 4 + 65536;
            };
            const uint64_t cmin = 4ull << 20;
            int S = std::max(1, std::min(P.streams, 8));
            // a small budget first drops streams, then merges fewer partitions per unit
            while (S > 1 && (uint64_t)S * (max_span + range_bytes()) + 2 * cmin > g->arena.avail()) --S;
            while (k > 1 && (uint64_t)S * (max_span + range_bytes()) + 2 * cmin > g->arena.avail()) spans(--k);
            const uint64_t range_b = range_bytes();
            if ((uint64_t)S * (max_span + range_b) + 2 * cmin > g->arena.avail())
                throw Err{HYT_ENOMEM, "device budget too small for one filter staging slot (" +
                                          std::to_string(max_span) + " B)"};
            c->S = S;
            c->k_eff = k;
            c->slot_bytes = max_span;
            for (int s = 0; s < S; ++s) {
                c->slot.push_back(dalloc<uint4>(g, c, max_span / 16 + 2, "filter staging slot"));
                RangeBufs r{};
                r.vcap = max_part_v + 64;
                r.cta_cap = r.vcap / (32 * kItemWords) + 4;
                r.q.cap = r.vcap;
                // a range queue's chunk space can exceed the span: adjacent short lists
                // that share a 16-B chunk each count it (<= one extra chunk per vertex)
                r.q.tile_cap = (max_span / 16 + max_part_v) / kTile + 8;
                r.q.qv = dalloc<uint32_t>(g, c, r.q.cap, "recompute queue");
                r.q.qpre = dalloc<uint64_t>(g, c, r.q.cap, "recompute prefix");
                r.q.qbeg = dalloc<uint64_t>(g, c, r.q.cap, "recompute edge begin");
                r.q.qdeg = dalloc<uint32_t>(g, c, r.q.cap, "recompute degree");
                r.q.qaux = algo == ALGO_PR ? dalloc<float>(g, c, r.q.cap, "recompute contrib") : nullptr;
                r.q.tile = dalloc<uint32_t>(g, c, r.q.tile_cap, "recompute tiles");
                r.taken = dalloc<uint32_t>(g, c, r.vcap / 32 + 4, "recompute taken");
                r.scratch = algo == ALGO_PR ? dalloc<float>(g, c, r.vcap, "recompute delta") : nullptr;
                r.cta_agg = dalloc<uint64_t>(g, c, 2 * r.cta_cap, "recompute aggregates");
                r.total = dalloc<uint64_t>(g, c, 2, "recompute totals");
                r.acc = c->racc;
                c->rb.push_back(r);
            }
            mark("staging slots + range queues");
            // compaction double buffer: what is left (capped), at least cmin
            uint64_t cb = P.compaction_buffer_bytes;
            if (!cb) {
                const uint64_t av = g->arena.avail();
                // with the edge cache on, most of the leftover budget goes to the cache
                const uint64_t div = P.edge_cache ? 16 : 2;
                const uint64_t left = av == UINT64_MAX ? (1ull << 30) : (av > 8192 ? av / div - 4096 : 0);
                cb = std::min<uint64_t>(256ull << 20, left);
            }
            cb = std::max<uint64_t>(cmin, cb) & ~15ull;
            c->cbuf_bytes = cb;
            for (int i = 0; i < 2; ++i) {
                c->cbuf[i] = dalloc<uint4>(g, c, cb / 16, "compaction buffer");
                c->hstage[i] = halloc<uint4>(c, cb / 16);
                HYT_CUDA(cudaEventCreateWithFlags(&c->ev_cbuf[i], cudaEventDisableTiming));
            }
            // host copy of the C queue: grown on demand (ensure_cq); the first 64K
            // entries also serve the Thpt_cpt probe
            c->cq_cap = std::min<uint64_t>(c->q.cap, 1ull << 16);
            c->cq_v = halloc<uint32_t>(c, c->cq_cap);
            c->cq_pre = halloc<uint64_t>(c, c->cq_cap);
            unsigned nt = P.gather_threads > 0 ? (unsigned)P.gather_threads
                                               : std::max(1u, std::thread::hardware_concurrency());
            c->pool = new Pool(nt);
            mark("compaction buffers + gather pool");
            if (P.edge_cache && P.engine_mode == MODE_HYBRID) {
                // partial resident edge cache: the longest prefix of the
                // own partitions in hub order that fits what the budget has left
                const uint64_t av = g->arena.avail();
                const uint64_t reserve = av == UINT64_MAX ? 0 : std::min<uint64_t>(64ull << 20, av / 16);
                uint64_t room = av == UINT64_MAX ? UINT64_MAX : av - reserve;
                if (P.edge_cache_bytes) room = std::min(room, P.edge_cache_bytes);
                const uint64_t c0 = chunk_lo(g->off_h[c->bounds[c->p_lo]], c->d1);
                uint64_t j = c->p_lo;
                while (j < c->p_hi && (chunk_hi(g->off_h[c->bounds[j + 1]], c->d1) - c0) * 16 <= room) ++j;
                if (j > c->p_lo) fill_cache(g, c, j);
            }
        }
        // CC pulls neighbours' labels: across ranks only with an exchange that leaves
        // every rank's copy current (dense / sparse), not with the peer push
        const bool cc_pull = algo == ALGO_CC && (!g->multi || P.exchange != 3);
        if (P.direction && g->symmetric && (algo == ALGO_BFS || cc_pull) && c->cache && c->cache_hi == c->p_hi) {
            build_pull_slices(g, c);
            if (g->multi) c->bm_glob = dalloc<uint32_t>(g, c, W + 2, "global frontier");
        }
        // streams
        const int nst = std::max(c->S, 1) + 2;
        while ((int)g->st.size() < nst) {
            cudaStream_t s;
            HYT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            g->st.push_back(s);
        }
        for (int i = 0; i < nst; ++i) {
            cudaEvent_t e;
            HYT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            c->ev_done.push_back(e);
        }
    } catch (...) {
        destroy_ctx(g, c);
        throw;
    }
    return c;
}

// One cached context per algorithm; when the budget cannot hold another one,
// the others are dropped and the build is retried.

static RunCtx *get_ctx(hyt_graph *g, int algo) {
    RunCtx *&c = ctx_of(g, algo);
    if (c) return c;
    // keep other algorithms' contexts only while the budget is mostly free, so a
    // cached context never shrinks this run's staging
    if (g->arena.budget && g->arena.avail() < g->arena.budget / 2) {
        for (int a = 0; a < 4; ++a)
            if (a != algo && ctx_of(g, a)) { destroy_ctx(g, ctx_of(g, a)); ctx_of(g, a) = nullptr; }
        if (g->last_algo != algo) g->has_result = false;
    }
    try {
        const double t0 = now_ms();
        c = build_ctx(g, algo);
        if (getenv("HYT_VERBOSE")) fprintf(stderr, "[hyt run] context for algo %d built in %.1f ms\n", algo, now_ms() - t0);
    } catch (const Err &e) {
        if (e.code != HYT_ENOMEM) throw;
        for (int a = 0; a < 4; ++a)
            if (a != algo && ctx_of(g, a)) { destroy_ctx(g, ctx_of(g, a)); ctx_of(g, a) = nullptr; }
        if (g->last_algo != algo) g->has_result = false;
        c = build_ctx(g, algo);
    }
    return c;
}

void release_run_ctx(hyt_graph *g) {
    for (int a = 0; a < 4; ++a)
        if (ctx_of(g, a)) { destroy_ctx(g, ctx_of(g, a)); ctx_of(g, a) = nullptr; }
    g->has_result = false;
}

static DevState make_state(hyt_graph *g, RunCtx *c) {
    DevState s{};
    s.V = g->V; s.W = (g->V + 31) / 32;
    s.off = g->off_d; s.din = g->din_d;
    s.val = c->val; s.rank = c->rank; s.delta = c->delta;
    s.bm_cur = c->bm_a; s.bm_next = c->bm_b;
    s.d1 = c->d1; s.algo = c->algo;
    s.wshift = (c->algo == ALGO_SSSP && c->d1 == 4) ? g->wshift : 0;
    s.damping = (float)g->prm.damping;
    s.epsilon = (float)g->prm.epsilon;
    s.hot_v = (uint32_t)g->prm.relax_hot_v;
    s.relax_nt = g->prm.relax_threads;
    s.bands = (uint32_t)g->prm.relax_bands;
    return s;
}

// ---------------------------------------------------------------------------
// compaction gather: chunks [w_lo, w_hi) of the C segment into dst (host)
// ---------------------------------------------------------------------------
void gather_window(RunCtx *c, const uint4 *edges_host, const std::vector<uint64_t> &off, uint64_t n,
                   uint64_t w_lo, uint64_t w_hi, uint4 *dst) {
    // first entry covering w_lo
    const uint64_t *pre = c->cq_pre;
    uint64_t k0 = std::upper_bound(pre, pre + n, w_lo) - pre - 1;
    uint64_t k1 = std::lower_bound(pre, pre + n, w_hi) - pre;   // entries [k0, k1)
    const unsigned nt = c->pool->size();
    c->pool->run([&](unsigned id) {
        const uint64_t a = k0 + (k1 - k0) * id / nt, b = k0 + (k1 - k0) * (id + 1) / nt;
        for (uint64_t k = a; k < b; ++k) {
            const uint32_t v = c->cq_v[k];
            const uint64_t c0 = chunk_lo(off[v], c->d1), c1 = chunk_hi(off[v + 1], c->d1);
            uint64_t lo = pre[k], hi = pre[k] + (c1 - c0);
            const uint64_t s = std::max(lo, w_lo), e = std::min(hi, w_hi);
            if (s >= e) continue;
            std::memcpy(dst + (s - w_lo), edges_host + c0 + (s - lo), (e - s) * 16);
        }
    });
}


// ---------------------------------------------------------------------------
// Cost-model calibration on this box.  Box properties (the DMA
// link rate and the zero-copy request / streamed-line times) are measured once
// per process and device on a dedicated 256 MiB pinned buffer, so they do not
// depend on the graph's size; Thpt_cpt (the host gather) is measured on the
// graph's own lists and then tracked by an EMA of every real gather.
// ---------------------------------------------------------------------------
struct BoxCal { double link_gbs = 0, zc_req_ns = 0, zc_line_ns = 0; };
static std::mutex g_cal_mu;
static BoxCal g_cal[64];

static BoxCal box_calibration(hyt_graph *g) {
    std::lock_guard<std::mutex> lock(g_cal_mu);
    BoxCal &bc = g_cal[g->device & 63];
    if (bc.link_gbs > 0) return bc;
    // Default 4 GiB (cal_probe_bytes): far larger than the host's last-level cache, so
    // random zero-copy requests really go to host DRAM (a 256 MiB probe read 5x too
    // fast).  If the host cannot pin that much, halve down to 256 MiB; if nothing can
    // be pinned and mapped, fall back to the rates measured on this pool
    // (profiles/r01_zc_bench.json) instead of failing the run.
    BoxCal fb;
    fb.link_gbs = 55.5; fb.zc_req_ns = 14.5; fb.zc_line_ns = 2.5;
    uint64_t hbytes = std::max<uint64_t>(g->prm.cal_probe_bytes, 256ull << 20);
    void *h = nullptr;
    while (!h) {
        try {
            h = pinned_alloc(hbytes);
        } catch (const Err &) {
            if (hbytes <= (256ull << 20)) { bc = fb; return bc; }
            hbytes /= 2;
        }
    }
    struct Pin { void *p; ~Pin() { pinned_free(p); } } pin{h};
    uint4 *mapped = nullptr;
    if (cudaHostGetDevicePointer((void **)&mapped, h, 0) != cudaSuccess || !mapped) {
        cudaGetLastError();
        bc = fb;
        return bc;
    }
    // DMA rate: best of 3 trials of 512 MiB into up to 64 MiB of the handle's arena
    const uint64_t av = g->arena.avail();
    const uint64_t dbytes = std::min<uint64_t>(64ull << 20, av == UINT64_MAX ? (64ull << 20) : av / 2) & ~4095ull;
    double link = fb.link_gbs;
    if (dbytes >= (4ull << 20)) {
        void *d = g->arena.alloc(dbytes, "calibration");
        cudaEvent_t a, b;
        HYT_CUDA(cudaEventCreate(&a));
        HYT_CUDA(cudaEventCreate(&b));
        const int reps = (int)std::max<uint64_t>(2, (512ull << 20) / dbytes);
        HYT_CUDA(cudaMemcpyAsync(d, h, dbytes, cudaMemcpyHostToDevice, g->main));
        double best = 0;
        for (int trial = 0; trial < 3; ++trial) {
            HYT_CUDA(cudaEventRecord(a, g->main));
            for (int r = 0; r < reps; ++r)
                HYT_CUDA(cudaMemcpyAsync(d, (const char *)h + (uint64_t)r * dbytes % (hbytes - dbytes), dbytes,
                                         cudaMemcpyHostToDevice, g->main));
            HYT_CUDA(cudaEventRecord(b, g->main));
            HYT_CUDA(cudaEventSynchronize(b));
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (ms > 0) best = std::max(best, (double)dbytes * reps / (ms / 1e3) / 1e9);
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        g->arena.release(d);
        if (best > 0) link = best;
    }
    uint32_t *sink = (uint32_t *)g->arena.alloc(256, "calibration sink");
    uint64_t lines = 0;
    float ms_r = 0, ms_s = 0;
    for (int trial = 0; trial < 2; ++trial) {   // second trial counts (first warms the mapping)
        ms_r = time_zc_probe(mapped, hbytes / 128, 0, sink, &lines, g->main);
    }
    const double req_ns = lines ? ms_r * 1e6 / lines : 0;
    for (int trial = 0; trial < 2; ++trial) ms_s = time_zc_probe(mapped, hbytes / 128, 1, sink, &lines, g->main);
    const double line_ns = lines ? ms_s * 1e6 / lines : 0;
    g->arena.release(sink);
    HYT_CUDA(cudaGetLastError());
    bc.link_gbs = link;
    bc.zc_req_ns = req_ns > 0 ? req_ns : fb.zc_req_ns;
    bc.zc_line_ns = line_ns > 0 ? line_ns : fb.zc_line_ns;
    // sanity: a random request is never cheaper than a streamed line, and a streamed
    // line is never cheaper than the same 128 B by DMA
    bc.zc_line_ns = std::max(bc.zc_line_ns, 128.0 / link);
    bc.zc_req_ns = std::max(bc.zc_req_ns, bc.zc_line_ns);
    return bc;
}

static void calibrate(hyt_graph *g, RunCtx *c) {
    const Params &P = g->prm;
    if (!P.cpu_cost && !P.cost_model) return;
    if (g->est_link_gbs <= 0 || (P.cost_model && g->est_zc_req_ns <= 0)) {
        const BoxCal bc = box_calibration(g);
        if (g->est_link_gbs <= 0) g->est_link_gbs = P.link_gbs > 0 ? P.link_gbs : bc.link_gbs;
        if (g->est_zc_req_ns <= 0) {
            g->est_zc_req_ns = P.zc_req_ns > 0 ? P.zc_req_ns : bc.zc_req_ns;
            g->est_zc_line_ns = P.zc_line_ns > 0 ? P.zc_line_ns : bc.zc_line_ns;
        }
    }
    if (P.thpt_cpt_gbs > 0) g->est_cpt_gbs = P.thpt_cpt_gbs;
    const uint4 *edges_host = host_edges(g, c->algo);
    if (g->est_cpt_gbs <= 0 && c->pool && c->cq_cap > 1 && c->v_hi > c->v_lo) {
        // the lists of up to 64K random own vertices with out-edges, gathered like the C engine
        std::vector<uint32_t> vs;
        uint64_t x = 0x9E3779B97F4A7C15ull;
        for (uint64_t tries = 0; vs.size() < 65536 && tries < 1000000; ++tries) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            const uint64_t v = c->v_lo + x % (c->v_hi - c->v_lo);
            if (g->off_h[v + 1] > g->off_h[v]) vs.push_back((uint32_t)v);
        }
        const uint64_t n = std::min<uint64_t>(vs.size(), c->cq_cap);
        uint64_t pre = 0;
        for (uint64_t k = 0; k < n; ++k) {
            c->cq_v[k] = vs[k];
            c->cq_pre[k] = pre;
            pre += chunk_hi(g->off_h[vs[k] + 1], c->d1) - chunk_lo(g->off_h[vs[k]], c->d1);
        }
        const uint64_t w_hi = std::min<uint64_t>(pre, c->cbuf_bytes / 16);
        if (w_hi >= 4096) {
            gather_window(c, edges_host, g->off_h, n, 0, w_hi, c->hstage[0]);   // warm
            const double t0 = now_ms();
            gather_window(c, edges_host, g->off_h, n, 0, w_hi, c->hstage[0]);
            const double ms = now_ms() - t0;
            if (ms > 0) g->est_cpt_gbs = w_hi * 16 / (ms / 1e3) / 1e9;
        }
        if (g->est_cpt_gbs <= 0) g->est_cpt_gbs = 10.0;   // too few lists to time: order of magnitude measured here
    }
}

// cost_model 1 calibrates the rule for the min-algorithms (BFS / SSSP / CC) and keeps
// the paper's constants for delta-PR; 2 calibrates every algorithm.  The per-iteration
// rule has no term for the recompute pass a filter unit gets (A6): for an
// accumulative algorithm that pass is worth a second relaxation of the unit's
// reactivated vertices, and the calibrated rule, which sends more late partitions to
// zero-copy, was measured 1-2 % slower than the paper's on TW and UK PR
// (profiles/r02_pr_zcw_{tw,uk}.json), where it is 14-19 % faster on SSSP / BFS.
static CostParams cost_for(hyt_graph *g, uint32_t d1, int algo) {
    const Params &P = g->prm;
    const bool cal = P.cost_model == 2 || (P.cost_model == 1 && algo != ALGO_PR);
    double ratio = 0.0, zr = 0.0, zs = 0.0;
    if ((P.cpu_cost || cal) && g->est_link_gbs > 0 && g->est_cpt_gbs > 0)
        ratio = g->est_link_gbs / g->est_cpt_gbs;
    if (cal && g->est_link_gbs > 0 && g->est_zc_req_ns > 0) {
        // RTT = the time of one saturated TLP (m * MR bytes) at the DMA link rate
        const double rtt_ns = (double)(P.m * P.mr) / g->est_link_gbs;
        zr = g->est_zc_req_ns / rtt_ns;
        zs = g->est_zc_line_ns / rtt_ns;
    }
    return make_cost(P, d1, ratio, zr, zs);
}


void run_graph(hyt_graph *g, int algo, uint64_t source) {
    HYT_REQUIRE(g->loaded, HYT_ESTATE, "no graph loaded");
    HYT_REQUIRE(algo >= ALGO_BFS && algo <= ALGO_PR, HYT_EINVAL, "unknown algorithm");
    HYT_REQUIRE(algo == ALGO_CC || algo == ALGO_PR || source < g->V, HYT_EINVAL, "source >= V");
    HYT_REQUIRE(algo != ALGO_SSSP || g->weighted, HYT_EINVAL, "SSSP needs edge weights");
    HYT_CUDA(cudaSetDevice(g->device));
    const Params &P = g->prm;
    const double t0 = now_ms();
    RunCtx *c = get_ctx(g, algo);
    DevState s = make_state(g, c);
    cudaStream_t main = g->main;
    calibrate(g, c);
    const CostParams cp = cost_for(g, c->d1, algo);
    const int mode = P.engine_mode;
    const int prio = P.priority >= 0 ? P.priority : (algo == ALGO_PR ? 2 : 1);
    const int sms = num_sms();
    const int relax_ctas = sms * P.relax_ctas_per_sm, zc_ctas = P.zc_ctas > 0 ? P.zc_ctas : sms * P.zc_ctas_per_sm;
    const uint4 *edges_host = host_edges(g, c->algo);          // indexed by global chunk
    uint64_t store_c0 = 0;
    const void *store = edge_store(g, algo, &store_c0);
    const uint4 *edges_mapped = nullptr;                       // device view of the store's first chunk
    HYT_CUDA(cudaHostGetDevicePointer((void **)&edges_mapped, const_cast<void *>(store), 0));

    // reset statistics
    g->stats = hyt_stats{};
    g->iter_log.clear();
    for (auto &t : g->eng_time) t = EngTime{};
    g->recompute_time = g->copy_time = g->plan_time = g->rq_time = EngTime{};
    for (int i = 0; i < ENG_COUNT; ++i) g->eng_chunks[i] = g->eng_edges[i] = 0;
    g->has_result = false;

    // ImpTM-UM: cold pages, and a balloon so managed pages fit the budget's remainder
    struct Balloon {
        void *p = nullptr;
        ~Balloon() { if (p) cudaFree(p); }
    } balloon;
    if (mode == MODE_UM && c->um) {
        if (P.um_cold) {   // ReadMostly keeps duplicates on a prefetch: drop the hint, migrate, re-advise
            HYT_CUDA(cudaMemAdvise(c->um, c->cache_bytes, cudaMemAdviseUnsetReadMostly, g->device));
            HYT_CUDA(cudaMemPrefetchAsync(c->um, c->cache_bytes, cudaCpuDeviceId, main));
            HYT_CUDA(cudaStreamSynchronize(main));
            HYT_CUDA(cudaMemAdvise(c->um, c->cache_bytes, cudaMemAdviseSetReadMostly, g->device));
        }
        if (P.um_balloon && g->arena.budget) {
            size_t fr = 0, tot = 0;
            HYT_CUDA(cudaMemGetInfo(&fr, &tot));
            const uint64_t room = g->arena.avail();
            if (fr > room + (2ull << 20)) {
                const uint64_t b = (fr - room) & ~((2ull << 20) - 1);
                HYT_CUDA(cudaMalloc(&balloon.p, b));
                g->stats.um_balloon_bytes = b;
            }
        }
    }
    const bool cc_pull = algo == ALGO_CC && (!g->multi || P.exchange != 3);
    bool pull_ok = P.direction && g->symmetric && (algo == ALGO_BFS || cc_pull) && c->cache &&
                   c->cache_hi == c->p_hi && c->d1 == 4 && (!g->multi || c->bm_glob);
    if (g->multi && P.direction && g->symmetric && (algo == ALGO_BFS || cc_pull)) {
        // every rank must take the same branch (the pull gathers the frontier): AND over ranks
        uint32_t f = pull_ok ? 1u : 0u;
        HYT_CUDA(cudaMemcpyAsync(c->red, &f, 4, cudaMemcpyHostToDevice, main));
        dist_allreduce_min_u32(g, (uint32_t *)c->red, 1, main);
        HYT_CUDA(cudaMemcpyAsync(&f, c->red, 4, cudaMemcpyDeviceToHost, main));
        HYT_CUDA(cudaStreamSynchronize(main));
        pull_ok = f != 0;
    }
    // the switch rule uses whole-graph quantities (all ranks decide alike)
    const uint64_t E_own = g->E, V_own = g->V;
    bool pulling = false;
    uint64_t explored = 0;

    // source in internal ids
    uint64_t src_int = 0;
    if (algo == ALGO_BFS || algo == ALGO_SSSP) {
        uint32_t x = 0;
        HYT_CUDA(copy_sync(&x, g->new_id_d + source, 4, main));
        src_int = x;
    }
    launch_init_values(s, src_int, g->old_of_d, main);
    HYT_CUDA(cudaGetLastError());
    if (g->multi && algo == ALGO_PR) {   // only the owner holds a vertex's initial residual
        if (c->v_lo) HYT_CUDA(cudaMemsetAsync(c->delta, 0, c->v_lo * 4, main));
        if (c->v_hi < g->V) HYT_CUDA(cudaMemsetAsync(c->delta + c->v_hi, 0, (g->V - c->v_hi) * 4, main));
    }
    HYT_CUDA(cudaMemsetAsync(c->racc, 0, 4 * sizeof(uint64_t), main));
    g->launches = 1;

    // ---- fused peer push (exchange = 3): publish this rank's arrays, map the others' ----
    const bool peer = g->multi && P.exchange == 3;
    PeerPush pp_it;
    const PeerPush *ppp = nullptr;
    struct PeerGuard {
        RunCtx *c;
        ~PeerGuard() { dist_close_peers(c->peer_opened); }
    } peer_guard{c};
    if (peer) {
        HYT_REQUIRE(g->world <= kMaxPeers, HYT_EINVAL, "exchange = 3 supports at most 8 ranks");
        HYT_REQUIRE(!g->arena.ext, HYT_EINVAL, "exchange = 3 needs library-allocated device memory (no arena)");
        dist_close_peers(c->peer_opened);
        void *mine[3] = {algo == ALGO_PR ? (void *)c->delta : (void *)c->val, (void *)c->bm_a, (void *)c->bm_b};
        // also a barrier: every rank's values are initialised before anyone pushes into them
        dist_share_ptrs(g, mine, 3, c->peer_ptr, c->peer_opened, main);
        pp_it.n = (uint32_t)g->world;
        pp_it.lo = c->v_lo;
        pp_it.hi = c->v_hi;
        for (int r = 0; r <= g->world; ++r) {
            uint64_t lo = 0, hi = 0;
            rank_vertex_range(g->off_h, g->world, std::min(r, g->world - 1), &lo, &hi);
            pp_it.rb[r] = r < g->world ? lo : hi;
        }
        for (int r = 0; r < g->world; ++r) {
            if (algo == ALGO_PR) pp_it.delta[r] = (float *)c->peer_ptr[3 * r];
            else pp_it.val[r] = (uint32_t *)c->peer_ptr[3 * r];
        }
        ppp = &pp_it;
    }

    const uint64_t np = c->p_hi - c->p_lo;
    std::vector<uint8_t> pvec(np);
    std::vector<double> pscore(np);
    std::vector<uint64_t> units(2 * np + 2);
    const uint64_t max_iters = algo == ALGO_PR ? P.max_iters : UINT64_MAX;
    uint64_t it = 0;
    for (; it < max_iters; ++it) {
        const double ti = now_ms();
        EvPair ep;
        timed_begin(c, main, ep, TAG_PLAN);
        if (algo == ALGO_PR) launch_pr_frontier(s, main);
        HYT_CUDA(cudaMemsetAsync(c->hdr_d, 0, sizeof(SegHdr), main));
        HYT_CUDA(cudaMemsetAsync(c->parts_d + c->p_lo, 0, np * sizeof(PartIter), main));
        const PlanBufs pb{c->parts_d, c->iagg, c->ibase, c->hdr_d};
        launch_plan(s, c->bounds_d, c->t_d, c->items, c->item_lo, c->item_hi, c->p_lo, c->p_hi, c->cache_hi, mode, cp,
                    pb, main);
        // with pull possible, the queue is built only for push iterations (after the switch)
        if (!pull_ok) launch_fill(s, c->bounds_d, c->items, c->item_lo, c->item_hi, pb, c->q, main);
        timed_end(c, main, ep);
        if (c->snapfull)   // values at iteration start, for the sparse exchange's change list
            HYT_CUDA(cudaMemcpyAsync(c->snapfull, c->val, g->V * 4, cudaMemcpyDeviceToDevice, main));
        g->launches += ((algo == ALGO_PR) ? 3 : 2) - (pull_ok ? 1 : 0);
        HYT_CUDA(cudaMemcpyAsync(c->parts_h + c->p_lo, c->parts_d + c->p_lo, np * sizeof(PartIter),
                                 cudaMemcpyDeviceToHost, main));
        HYT_CUDA(cudaMemcpyAsync(c->hdr_h, c->hdr_d, sizeof(SegHdr), cudaMemcpyDeviceToHost, main));
        HYT_CUDA(cudaStreamSynchronize(main));
        HYT_CUDA(cudaGetLastError());
        harvest(g, c);
        const SegHdr H = *c->hdr_h;
        uint64_t active = H.active_vertices, active_e = H.active_edges;
        if (g->multi) {   // total active vertices (termination) and edges (direction switch) over all ranks
            HYT_CUDA(cudaMemcpyAsync(c->red, &c->hdr_d->active_vertices, 16, cudaMemcpyDeviceToDevice, main));
            dist_allreduce_sum_u64(g, c->red, 2, main);
            uint64_t a2[2] = {0, 0};
            HYT_CUDA(cudaMemcpyAsync(a2, c->red, 16, cudaMemcpyDeviceToHost, main));
            HYT_CUDA(cudaStreamSynchronize(main));
            active = a2[0];
            active_e = a2[1];
        }
        if (active == 0) break;

        // ---- SEP-Graph direction switch (§8f #4) ----
        bool pull = false;
        if (pull_ok) {
            const double mf = (double)active_e, nf = (double)active;
            if (algo == ALGO_BFS) {   // Beamer's rule
                explored += active_e;
                const double mu = E_own > explored ? (double)(E_own - explored) : 0.0;
                if (P.direction == 2) pulling = true;
                else if (!pulling) pulling = mf * P.pull_alpha > mu;
                else pulling = !(nf * P.pull_beta < (double)V_own);
            } else {
                pulling = P.direction == 2 || mf * P.cc_pull_alpha > (double)E_own;
            }
            pull = pulling;
            if (!pull) {
                EvPair ef;
                timed_begin(c, main, ef, TAG_PLAN);
                launch_fill(s, c->bounds_d, c->items, c->item_lo, c->item_hi, pb, c->q, main);
                timed_end(c, main, ef);
                g->launches += 1;
                HYT_CUDA(cudaStreamWaitEvent(g->st[0], ef.b, 0));
            }
        }

        if (peer && algo != ALGO_PR)   // owners' next bitmaps: all ranks swap in lockstep
            for (int r = 0; r < g->world; ++r) pp_it.bm[r] = (uint32_t *)c->peer_ptr[3 * r + ((it & 1) ? 1 : 2)];

        hyt_iter row{};
        row.iteration = it;
        row.active_vertices = H.active_vertices;
        row.active_edges = H.active_edges;

        // ---- task combination + ordering (host) ----
        for (uint64_t i = 0; i < np; ++i) pvec[i] = (uint8_t)c->parts_h[c->p_lo + i].p;
        const int64_t nu = combine_units(pvec.data(), np, c->k_eff, units.data());
        std::vector<uint32_t> order((size_t)nu);
        std::iota(order.begin(), order.end(), 0u);
        if (prio != 0 && nu > 1) {
            for (uint64_t i = 0; i < np; ++i) {
                const PartIter &pi = c->parts_h[c->p_lo + i];
                pscore[i] = prio == 2 ? pi.dsum : (double)pi.hub;
            }
            order_units(nu, units.data(), pscore.data(), order.data());
        }
        row.parts_f = (uint32_t)H.parts[ENG_F];
        row.parts_c = (uint32_t)H.parts[ENG_C];
        row.parts_z = (uint32_t)H.parts[ENG_Z];
        row.parts_r = (uint32_t)H.parts[ENG_R];
        row.units_f = (uint32_t)nu;

        // C queue to the host (needed by the gather) -- enqueued before the GPU work
        const uint64_t nC = H.ent_count[ENG_C];
        if (nC) {
            ensure_cq(c, nC);
            HYT_CUDA(cudaMemcpyAsync(c->cq_v, c->q.qv + H.ent_base[ENG_C], nC * 4, cudaMemcpyDeviceToHost, main));
            HYT_CUDA(cudaMemcpyAsync(c->cq_pre, c->q.qpre + H.ent_base[ENG_C], nC * 8, cudaMemcpyDeviceToHost, main));
        }

        // ---- filter units, in priority order ----
        const uint64_t fseg_first = H.ent_base[ENG_F], fseg_end = fseg_first + H.ent_count[ENG_F];
        for (int64_t jj = 0; jj < nu; ++jj) {
            const uint32_t j = order[jj];
            const int si = (int)(jj % c->S);
            cudaStream_t stm = g->st[si];
            const uint64_t pa = c->p_lo + units[2 * j], pb = c->p_lo + units[2 * j + 1];
            const uint64_t v_lo = c->bounds[pa], v_hi = c->bounds[pb];
            const uint64_t s0 = chunk_lo(g->off_h[v_lo], c->d1), s1 = chunk_hi(g->off_h[v_hi], c->d1);
            const uint64_t bytes = (s1 - s0) * 16;
            EvPair e1, e2, e3;
            timed_begin(c, stm, e1, TAG_COPY);
            HYT_CUDA(cudaMemcpyAsync(c->slot[si], edges_host + s0, bytes, cudaMemcpyHostToDevice, stm));
            timed_end(c, stm, e1);
            const uint64_t c_lo = c->parts_h[pa].chunk_base;
            const uint64_t c_hi = c->parts_h[pb - 1].chunk_base + c->parts_h[pb - 1].chunks;
            EdgeSrc es{c->slot[si], (int64_t)s0, false};
            if (algo == ALGO_PR) {
                const uint64_t e_lo = fseg_first + c->parts_h[pa].ent_base;
                const uint64_t e_hi = fseg_first + c->parts_h[pb - 1].ent_base + c->parts_h[pb - 1].ent;
                launch_take_delta(s, c->q, e_lo, e_hi, stm);
                g->launches += 1;
            }
            timed_begin(c, stm, e2, TAG_F);
            launch_relax(s, c->q, H.tile_base[ENG_F], fseg_first, fseg_end, H.chunk_total[ENG_F], c_lo, c_hi,
                         nullptr, es, relax_ctas, stm, P.relax_hot, ppp);
            timed_end(c, stm, e2);
            // process the loaded unit once more; recompute > 1 repeats
            // the pass (Subway-style multi-round processing of the staged unit)
            for (int rp = 0; rp < P.recompute; ++rp) {
                EvPair e4;
                timed_begin(c, stm, e4, TAG_RQ);
                launch_range_queue(s, v_lo, v_hi, c->rb[si], stm);
                timed_end(c, stm, e4);
                timed_begin(c, stm, e3, TAG_RECOMP);
                launch_relax(s, c->rb[si].q, 0, 0, 0, 0, 0, 0, c->rb[si].total, es, relax_ctas, stm, P.relax_hot, ppp);
                timed_end(c, stm, e3);
            }
            g->launches += 1 + 3 * P.recompute;
            row.bytes_f += bytes;
            g->eng_chunks[ENG_F] += c_hi - c_lo;
            for (uint64_t i = pa; i < pb; ++i) g->eng_edges[ENG_F] += c->parts_h[i].e;
        }
        // ---- merged zero-copy task: one kernel over Vz ----
        if (H.ent_count[ENG_Z]) {
            cudaStream_t stm = g->st[c->S];
            EvPair e1;
            timed_begin(c, stm, e1, TAG_Z);
            EdgeSrc es{edges_mapped, (int64_t)store_c0, false, true};
            if (algo == ALGO_PR) {
                launch_take_delta(s, c->q, H.ent_base[ENG_Z], H.ent_base[ENG_Z] + H.ent_count[ENG_Z], stm);
                g->launches += 1;
            }
            launch_relax(s, c->q, H.tile_base[ENG_Z], H.ent_base[ENG_Z], H.ent_base[ENG_Z] + H.ent_count[ENG_Z],
                         H.chunk_total[ENG_Z], 0, H.chunk_total[ENG_Z], nullptr, es, zc_ctas, stm, P.relax_hot, ppp);
            timed_end(c, stm, e1);
            g->launches += 1;
            g->eng_chunks[ENG_Z] += H.chunk_total[ENG_Z];
        }
        // ---- pull iteration: topology-driven over the own range (§8f #4) ----
        if (pull) {
            EvPair e1;
            timed_begin(c, main, e1, TAG_R);
            const uint32_t *nbr = reinterpret_cast<const uint32_t *>(c->cache) - c->cache_c0 * 4;
            const uint32_t *front = s.bm_cur;
            if (g->multi) {   // OR of every rank's own frontier words (disjoint bits: a sum)
                launch_own_words(s.bm_cur, c->bm_glob, s.W, c->v_lo, c->v_hi, main);
                HYT_CUDA(cudaMemsetAsync(c->bm_glob + s.W, 0, 8, main));
                dist_allreduce_sum_u64(g, reinterpret_cast<uint64_t *>(c->bm_glob), (s.W + 1) / 2, main);
                front = c->bm_glob;
                g->launches += 1;
            }
            launch_pull(algo, g->off_d, nbr, c->val, front, s.bm_next, c->v_lo, c->v_hi,
                        (uint32_t)std::min<uint64_t>(P.pull_heavy, 0xFFFFFFFFu), c->hs_v, c->hs_e0, c->hs_e1, c->n_hs,
                        (uint32_t)(it + 1), main);
            timed_end(c, main, e1);
            g->launches += c->n_hs ? 2 : 1;
            g->stats.pull_iters += 1;
            row.dir = 1;
        }
        // ---- resident (build extension) ----
        if (H.ent_count[ENG_R] && !pull) {
            HYT_REQUIRE(c->cache != nullptr, HYT_ESTATE, "resident edges missing");
            cudaStream_t stm = g->st[0];
            EvPair e1;
            timed_begin(c, stm, e1, TAG_R);
            EdgeSrc es{c->cache, (int64_t)c->cache_c0, false, mode == MODE_UM};
            if (algo == ALGO_PR) {
                launch_take_delta(s, c->q, H.ent_base[ENG_R], H.ent_base[ENG_R] + H.ent_count[ENG_R], stm);
                g->launches += 1;
            }
            launch_relax(s, c->q, H.tile_base[ENG_R], H.ent_base[ENG_R], H.ent_base[ENG_R] + H.ent_count[ENG_R],
                         H.chunk_total[ENG_R], 0, H.chunk_total[ENG_R], nullptr, es, relax_ctas, stm, P.relax_hot, ppp);
            timed_end(c, stm, e1);
            g->launches += 1;
            g->eng_chunks[ENG_R] += H.chunk_total[ENG_R];
        }
        for (uint64_t i = c->p_lo; i < c->p_hi; ++i) {
            const PartIter &pi = c->parts_h[i];
            if (pi.p == ENG_Z) { row.bytes_z += pi.z * P.m; g->eng_edges[ENG_Z] += pi.e; }
            if (pi.p == ENG_C) g->eng_edges[ENG_C] += pi.e;
            if (pi.p == ENG_R) g->eng_edges[ENG_R] += pi.e;
        }
        // ---- merged compaction task: host gather overlapping the GPU work ----
        if (nC) {
            HYT_CUDA(cudaStreamSynchronize(main));   // C queue on the host
            cudaStream_t stm = g->st[c->S + 1];
            const uint64_t total = H.chunk_total[ENG_C];
            const uint64_t per = c->cbuf_bytes / 16;
            if (algo == ALGO_PR) {
                launch_take_delta(s, c->q, H.ent_base[ENG_C], H.ent_base[ENG_C] + nC, stm);
                g->launches += 1;
            }
            uint64_t b = 0;
            for (uint64_t w_lo = 0; w_lo < total; w_lo += per, ++b) {
                const uint64_t w_hi = std::min(total, w_lo + per);
                const int bi = (int)(b & 1);
                if (b >= 2) HYT_CUDA(cudaEventSynchronize(c->ev_cbuf[bi]));
                const double tg = now_ms();
                gather_window(c, edges_host, g->off_h, nC, w_lo, w_hi, c->hstage[bi]);
                const double gms = now_ms() - tg;
                g->stats.gather_ms += gms;
                if ((P.cpu_cost || P.cost_model) && P.thpt_cpt_gbs <= 0 && gms > 0.5) {   // keep Thpt_cpt current (EMA)
                    const double r = (w_hi - w_lo) * 16 / (gms / 1e3) / 1e9;
                    g->est_cpt_gbs = g->est_cpt_gbs > 0 ? 0.5 * g->est_cpt_gbs + 0.5 * r : r;
                }
                EvPair e1, e2;
                timed_begin(c, stm, e1, TAG_COPY);
                HYT_CUDA(cudaMemcpyAsync(c->cbuf[bi], c->hstage[bi], (w_hi - w_lo) * 16, cudaMemcpyHostToDevice, stm));
                timed_end(c, stm, e1);
                HYT_CUDA(cudaEventRecord(c->ev_cbuf[bi], stm));
                EdgeSrc es{c->cbuf[bi], 0, true};
                timed_begin(c, stm, e2, TAG_C);
                launch_relax(s, c->q, H.tile_base[ENG_C], H.ent_base[ENG_C], H.ent_base[ENG_C] + nC, total, w_lo,
                             w_hi, nullptr, es, relax_ctas, stm, P.relax_hot, ppp);
                timed_end(c, stm, e2);
                g->launches += 1;
            }
            row.bytes_c += total * 16;
            g->eng_chunks[ENG_C] += total;
        }
        // ---- join all streams into main ----
        const int nst = c->S + 2;
        for (int i = 0; i < nst && i < (int)g->st.size(); ++i) {
            HYT_CUDA(cudaEventRecord(c->ev_done[i], g->st[i]));
            HYT_CUDA(cudaStreamWaitEvent(main, c->ev_done[i], 0));
        }
        HYT_CUDA(cudaGetLastError());
        // ---- multi-GPU exchange of pushed values ----
        if (peer) {
            // fused push: remote relaxations already landed in their owners' arrays;
            // a barrier keeps every rank's next plan after every rank's pushes
            HYT_CUDA(cudaMemsetAsync(c->red + 1, 0, 8, main));
            dist_allreduce_max_u64(g, c->red + 1, 1, main);
            g->stats.exch_peer += 1;
        } else if (g->multi) {
            const bool pr = algo == ALGO_PR;
            bool sparse = false;
            uint64_t maxc = 0;
            if (c->xcap) {   // the pairs each rank changed; the largest count decides
                HYT_CUDA(cudaMemsetAsync(c->xcnt, 0, 8, main));
                launch_collect_changed(pr, g->V, c->v_lo, c->v_hi, c->val, c->snapfull, c->delta, c->xsend, c->xcap,
                                       c->xcnt, main);
                HYT_CUDA(cudaMemcpyAsync(c->red + 1, c->xcnt, 8, cudaMemcpyDeviceToDevice, main));
                dist_allreduce_max_u64(g, c->red + 1, 1, main);
                HYT_CUDA(cudaMemcpyAsync(&maxc, c->red + 1, 8, cudaMemcpyDeviceToHost, main));
                HYT_CUDA(cudaStreamSynchronize(main));
                g->launches += 1;
                sparse = maxc <= c->xcap && (P.exchange == 2 || (uint64_t)g->world * maxc * 8 < g->V * 4);
            }
            if (sparse) {
                if (maxc) {
                    launch_pad_pairs(c->xsend, c->xcnt, maxc, main);
                    dist_allgather_u32(g, (const uint32_t *)c->xsend, (uint32_t *)c->xrecv, 2 * maxc, main);
                    launch_apply_pairs(pr, c->xrecv, (uint64_t)g->world * maxc, c->v_lo, c->v_hi, c->val, c->delta,
                                       s.bm_next, main);
                    g->launches += 2;
                }
                g->stats.exch_sparse += 1;
                g->stats.exch_bytes += maxc * 8;
            } else {
                if (pr) {
                    // own entries: residual + every rank's pushes; others: outbox -> zero again
                    dist_allreduce_sum_f32(g, c->delta, g->V, main);
                } else {
                    HYT_CUDA(cudaMemcpyAsync(c->snap, c->val + c->v_lo, (c->v_hi - c->v_lo) * 4,
                                             cudaMemcpyDeviceToDevice, main));
                    dist_allreduce_min_u32(g, c->val, g->V, main);
                    launch_mark_improved(c->val, c->snap, c->v_lo, c->v_hi, s.bm_next, main);
                    g->launches += 1;
                }
                g->stats.exch_dense += 1;
                g->stats.exch_bytes += g->V * 4;
            }
            if (pr) {   // the outbox is empty again
                if (c->v_lo) HYT_CUDA(cudaMemsetAsync(c->delta, 0, c->v_lo * 4, main));
                if (c->v_hi < g->V) HYT_CUDA(cudaMemsetAsync(c->delta + c->v_hi, 0, (g->V - c->v_hi) * 4, main));
            }
        }
        // ---- next frontier ----
        if (algo != ALGO_PR) {
            std::swap(s.bm_cur, s.bm_next);
            std::swap(c->bm_a, c->bm_b);
            HYT_CUDA(cudaMemsetAsync(s.bm_next, 0, s.W * 4, main));
        }
        row.ms = now_ms() - ti;
        g->stats.bytes_filter += row.bytes_f;
        g->stats.bytes_compaction += row.bytes_c;
        g->stats.bytes_zerocopy += row.bytes_z;
        g->stats.parts_filter += row.parts_f;
        g->stats.parts_compaction += row.parts_c;
        g->stats.parts_zerocopy += row.parts_z;
        g->stats.parts_resident += row.parts_r;
        g->stats.units_filter += row.units_f;
        g->stats.edges_relaxed += row.active_edges;
        g->iter_log.push_back(row);
    }
    if (g->multi && algo == ALGO_PR) dist_allreduce_sum_f32(g, c->rank, g->V, main);
    if (peer && algo != ALGO_PR) dist_allreduce_min_u32(g, c->val, g->V, main);   // owners' values everywhere
    HYT_CUDA(cudaStreamSynchronize(main));
    harvest(g, c);
    const double t1 = now_ms();
    g->stats.iterations = it;
    g->stats.time_ns = (uint64_t)((t1 - t0) * 1e6);
    g->stats.num_partitions = c->N;
    g->stats.device_bytes_peak = g->arena.peak;
    double kms = 0;
    for (int i = 1; i < ENG_COUNT; ++i) kms += g->eng_time[i].ms;
    g->stats.kernel_ms = kms + g->recompute_time.ms;
    g->stats.copy_ms = g->copy_time.ms;
    g->stats.plan_ms = g->plan_time.ms;
    g->stats.kernel_launches = g->launches;
    g->stats.cal_link_gbs = g->est_link_gbs;
    g->stats.cal_cpt_gbs = g->est_cpt_gbs;
    g->stats.cal_zc_req_ns = g->est_zc_req_ns;
    g->stats.cal_zc_line_ns = g->est_zc_line_ns;
    g->stats.host_store_bytes = g->store_bytes;
    g->stats.record_bytes = c->d1;
    for (int i = 0; i < 8; ++i) { g->stats.eng_ms[i] = 0; g->stats.eng_launches[i] = 0; g->stats.eng_chunks[i] = 0; g->stats.eng_edges[i] = 0; }
    g->stats.eng_ms[0] = g->plan_time.ms; g->stats.eng_launches[0] = g->plan_time.launches;
    for (int i = 1; i < ENG_COUNT; ++i) {
        g->stats.eng_ms[i] = g->eng_time[i].ms; g->stats.eng_launches[i] = g->eng_time[i].launches;
        g->stats.eng_chunks[i] = g->eng_chunks[i]; g->stats.eng_edges[i] = g->eng_edges[i];
    }
    g->stats.eng_ms[5] = g->recompute_time.ms; g->stats.eng_launches[5] = g->recompute_time.launches;
    {
        uint64_t racc[4] = {0, 0, 0, 0};
        HYT_CUDA(copy_sync(racc, c->racc, sizeof(racc), main));
        g->stats.eng_chunks[5] = racc[1];
        g->stats.eng_edges[5] = racc[2];
    }
    g->stats.eng_ms[6] = g->copy_time.ms; g->stats.eng_launches[6] = g->copy_time.launches;
    g->stats.eng_ms[7] = g->rq_time.ms; g->stats.eng_launches[7] = g->rq_time.launches;
    g->val_d = c->val; g->rank_d = c->rank; g->delta_d = c->delta;
    g->last_algo = algo;
    g->has_result = true;
}

// ---------------------------------------------------------------------------
// results
// ---------------------------------------------------------------------------
void get_values(hyt_graph *g, void *out, uint64_t count) {
    HYT_REQUIRE(g->has_result, HYT_ESTATE, "no result: call hyt_run first");
    HYT_REQUIRE(count == g->V, HYT_EINVAL, "count != V");
    HYT_CUDA(cudaSetDevice(g->device));
    RunCtx *c = ctx_of(g, g->last_algo);
    HYT_REQUIRE(c != nullptr, HYT_ESTATE, "no result: run context was released");
    DevState s = make_state(g, c);
    launch_gather_out(s, g->new_id_d, c->outbuf, g->main);
    HYT_CUDA(cudaMemcpyAsync(out, c->outbuf, g->V * 4, cudaMemcpyDeviceToHost, g->main));
    HYT_CUDA(cudaStreamSynchronize(g->main));
}

// ---------------------------------------------------------------------------
// plan parity hook
// ---------------------------------------------------------------------------
__global__ void k_active_to_bitmap(const uint8_t *__restrict__ act, const uint32_t *__restrict__ new_id,
                                   uint64_t V, uint32_t *__restrict__ bm) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t u = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; u < V; u += stride)
        if (act[u]) {
            const uint32_t v = new_id[u];
            atomicOr(&bm[v >> 5], 1u << (v & 31));
        }
}

void debug_plan(hyt_graph *g, int algo, const uint8_t *active, uint64_t *num_parts, uint64_t *bounds,
                uint64_t *t, uint64_t *e, uint64_t *a, uint64_t *z, uint8_t *p) {
    HYT_REQUIRE(g->loaded, HYT_ESTATE, "no graph loaded");
    HYT_REQUIRE(algo >= ALGO_BFS && algo <= ALGO_PR, HYT_EINVAL, "unknown algorithm");
    HYT_CUDA(cudaSetDevice(g->device));
    const uint32_t d1 = (algo == ALGO_SSSP && !g->pw_h) ? 8 : 4;   // as build_ctx
    std::vector<uint64_t> b = partition_bounds_ranked(g->off_h, d1, g->prm.partition_bytes, g->world);
    const uint64_t N = b.size() - 1;
    *num_parts = N;
    if (!bounds && !t && !p) return;
    RunCtx *c = get_ctx(g, algo);
    DevState s = make_state(g, c);
    uint8_t *act_d = arena_new<uint8_t>(g->arena, g->V, "debug active");
    HYT_CUDA(copy_sync(act_d, active, g->V, g->main));
    HYT_CUDA(cudaMemsetAsync(s.bm_cur, 0, s.W * 4, g->main));
    k_active_to_bitmap<<<num_sms() * 8, 256, 0, g->main>>>(act_d, g->new_id_d, g->V, s.bm_cur);
    if (algo == ALGO_PR) {   // the plan kernel reads delta for priorities only
        HYT_CUDA(cudaMemsetAsync(s.delta, 0, g->V * 4, g->main));
    }
    HYT_CUDA(cudaMemsetAsync(c->hdr_d, 0, sizeof(SegHdr), g->main));
    HYT_CUDA(cudaMemsetAsync(c->parts_d, 0, N * sizeof(PartIter), g->main));
    const PlanBufs pb{c->parts_d, c->iagg, c->ibase, c->hdr_d};
    launch_plan(s, c->bounds_d, c->t_d, c->items, 0, c->n_items, 0, N, c->cache_hi, g->prm.engine_mode,
                cost_for(g, d1, algo), pb, g->main);
    std::vector<PartIter> ph(N);
    HYT_CUDA(cudaMemcpyAsync(ph.data(), c->parts_d, N * sizeof(PartIter), cudaMemcpyDeviceToHost, g->main));
    HYT_CUDA(cudaStreamSynchronize(g->main));
    g->arena.release(act_d);
    for (uint64_t i = 0; i < N; ++i) {
        if (bounds) bounds[i] = b[i];
        if (t) t[i] = g->off_h[b[i + 1]] - g->off_h[b[i]];
        if (e) e[i] = ph[i].e;
        if (a) a[i] = ph[i].a;
        if (z) z[i] = ph[i].z;
        if (p) p[i] = (uint8_t)ph[i].p;
    }
    if (bounds) bounds[N] = b[N];
    g->has_result = false;
}

void free_graph(hyt_graph *g) {
    if (!g) return;
    cudaSetDevice(g->device);
    release_run_ctx(g);
    for (auto s : g->st) cudaStreamDestroy(s);
    if (g->main) cudaStreamDestroy(g->main);
    release_adopted(g);
    pinned_free(g->nbr_h);
    pinned_free(g->ew_h);
    pinned_free(g->pw_h);
    dist_free(g);
    g->arena.release_all();
}

}  // namespace hyt
