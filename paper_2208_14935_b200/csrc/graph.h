// graph.h -- the handle (struct hyt_graph), the device arena and error plumbing.
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/hyt.h"
#include "hyt_internal.h"

namespace hyt {

// thread-local last error
void set_error(const std::string &msg);
const char *get_error();

struct Err {                       // thrown inside the library, caught at the ABI
    int code;
    std::string msg;
};

#define HYT_CUDA(call)                                                                            \
    do {                                                                                          \
        cudaError_t _e = (call);                                                                  \
        if (_e != cudaSuccess)                                                                    \
            throw ::hyt::Err{_e == cudaErrorMemoryAllocation ? HYT_ENOMEM : HYT_ECUDA,            \
                             std::string(#call) + ": " + cudaGetErrorString(_e) + " @" +          \
                                 __FILE__ + ":" + std::to_string(__LINE__)};                      \
    } while (0)

#define HYT_REQUIRE(cond, code, msg)                                                              \
    do {                                                                                          \
        if (!(cond)) throw ::hyt::Err{(code), (msg)};                                              \
    } while (0)

// Device arena: every device byte the handle uses goes through here, so the
// budget is enforced exactly.  Either tracked cudaMalloc blocks or
// a caller-owned block (e.g. a torch tensor) used as a stack.
struct Arena {
    uint64_t budget = 0;       // 0 = no cap
    uint64_t used = 0, peak = 0;
    char *ext = nullptr;
    uint64_t ext_size = 0, ext_top = 0;
    struct Blk { void *p; uint64_t bytes; uint64_t top_before; bool live; };
    std::vector<Blk> blocks;

    void *alloc(uint64_t bytes, const char *what);
    void release(void *p);
    void release_all();
    uint64_t avail() const { return budget ? (budget > used ? budget - used : 0) : UINT64_MAX; }
};

template <class T> T *arena_new(Arena &a, uint64_t n, const char *what) {
    return (T *)a.alloc(n * sizeof(T) + 16, what);
}

struct Params {
    double alpha = 0.8, beta = 0.4, gamma = 0.625;
    uint64_t m = 128, mr = 256, d2 = 4, k = 4;
    uint64_t partition_bytes = 32ull << 20;
    double hub_fraction = 0.08;
    int streams = 4;
    int engine_mode = MODE_HYBRID;
    int priority = -1;
    int recompute = 1;
    double damping = 0.85, epsilon = 1e-5;   // C16 (round 2): eps/(1-d) = 6.7e-5 < 1e-4
    uint64_t max_iters = 1000;
    int gather_threads = 0;
    uint64_t compaction_buffer_bytes = 0;
    int zc_ctas_per_sm = 1;     // 512-thread CTAs
    int zc_ctas = 0;            // > 0: the zero-copy relax grid in 512-thread CTAs (overrides zc_ctas_per_sm)
    int relax_ctas_per_sm = 2;  // 512-thread CTAs
    int exchange = 1;          // multi-GPU: 0 dense, 1 sparse when cheaper (§8f #3), 2 sparse when it fits,
                               // 3 fused peer push (relax writes remote destinations into their owner's memory)
    int relax_hot = 1;         // hub block in smem (PR Δ accumulation / min-algorithm value copy): 0 off, 1 auto, 2 always
    uint64_t relax_hot_v = 16384;   // PR hub-block vertices in shared memory (8 B each: 128 KB; min-algorithms cap at kHotV)
    int relax_bands = 1;            // destination bands for device-resident edges: 1 off (default: measured slower), 0 auto (V*4 / (3/4 L2)), n
    int relax_threads = 0;          // relax CTA size: 0 auto (PR 1024: 1 CTA/SM sharing the hub block; else 512), 512, 1024
    int pack_weights = 1;      // load time: SSSP records as one u32 (id | w << bits(V-1)) when the weights fit
    int edge_cache = 0;        // 1: keep a prefix of partitions resident; 0: paper semantics
    uint64_t edge_cache_bytes = 0;   // cap on the cache (0 = whatever the budget leaves)
    int cpu_cost = 0;          // 1: include Eq. 2's CPU term with Thpt_cpt calibrated on this box
    double thpt_cpt_gbs = 0;   // host gather throughput (0 = measure)
    double link_gbs = 0;       // host->device link rate (0 = measure)
    double zc_weight = 1.0;    // multiplier on Tiz (1 = the paper's Eq. 3)
    int cost_model = 1;        // 1: Eq. 1-3 with costs calibrated on this box for BFS/SSSP/CC, the paper's for PR; 2: calibrated for all; 0: the paper's PCIe-3 constants
    double zc_req_ns = 0;      // zero-copy random 128-B request time (0 = measure)
    double zc_line_ns = 0;     // zero-copy streamed 128-B line time (0 = measure)
    uint64_t cal_probe_bytes = 4ull << 30;   // pinned probe buffer of the box calibration (>= 256 MiB)
    int direction = 1;         // BFS/CC on symmetric resident graphs: 0 push, 1 switch (§8f #4), 2 pull
    double pull_alpha = 14, pull_beta = 24, cc_pull_alpha = 2;
    uint64_t pull_heavy = 1024;
    int um_balloon = 1, um_cold = 1;   // ImpTM-UM comparison mode
};

CostParams make_cost(const Params &p, uint32_t d1, double cpu_ratio = 0.0, double zr_rtt = 0.0,
                     double zs_rtt = 0.0);

// Pinned, mapped host memory: mmap + transparent huge pages + parallel first
// touch + cudaHostRegister.  About 9x faster to create than cudaHostAlloc on the
// B200 box (tools/pin_bench.cu: 0.34 s vs 3.1 s for 8 GB).
void *pinned_alloc(uint64_t bytes);
void pinned_free(void *p);     // keeps the block registered in a bounded cache (HYT_PIN_CACHE_GB)
void pinned_trim();            // release every cached block

// Every host<->device copy and memset runs on one of the library's (non-blocking)
// streams.  A synchronous cudaMemcpy from pageable memory goes through the legacy
// stream and may return before its DMA lands, and the non-blocking streams are
// not ordered after it (the round-1 multi-rank race).  copy_sync: enqueue on st,
// then wait for st, so the copy has landed and later work on st is ordered after it.
inline cudaError_t copy_sync(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
    if (e != cudaSuccess) return e;
    return cudaStreamSynchronize(st);
}

// Engine timing accumulator (CUDA events per launch, read after the iteration).
struct EngTime {
    double ms = 0;
    uint64_t launches = 0;
};

}  // namespace hyt

struct hyt_graph {
    int device = 0;
    hyt::Arena arena;
    hyt::Params prm;
    // ---- graph (internal, hub-sorted order) ----
    bool loaded = false;
    uint64_t V = 0, E = 0;
    bool weighted = false;
    bool symmetric = false;         // HYT_SYMMETRIC: enables pull iterations
    // Edge store: pinned mapped records of this rank's vertex range only
    // [store_v_lo, store_v_hi) (the whole graph when world == 1), starting at the
    // 16-byte chunk store_c0[0] (u32 ids) / store_c0[1] (id | w<<32) of the global
    // edge byte space.  host_edges() returns pointers indexed by GLOBAL chunk.
    uint32_t *nbr_h = nullptr;      // pinned mapped u32 ids (+pad)
    uint64_t *ew_h = nullptr;       // pinned mapped (id | w<<32) u64 (+pad), weighted, unpacked only
    // packed SSSP records (pack_weights): one u32 per edge, id | w << wshift, with
    // wshift = the bits of V-1; used when every weight fits the remaining bits
    uint32_t *pw_h = nullptr;
    uint32_t wshift = 0;
    uint64_t store_v_lo = 0, store_v_hi = 0;
    uint64_t store_c0[2] = {0, 0};
    std::vector<uint64_t> off_h;    // host copy of offsets u64[V+1]
    uint64_t *off_d = nullptr;      // device offsets
    uint32_t *new_id_d = nullptr;   // caller id -> internal id
    uint32_t *old_of_d = nullptr;   // internal id -> caller id
    uint32_t *din_d = nullptr;      // in-degree (internal ids)
    uint64_t store_bytes = 0;       // pinned host bytes this handle owns for its edge store
    bool nbr_adopted = false;       // HYT_ADOPT_HOST: nbr_h is the caller's (registered) array
    const void *adopt_key = nullptr, *adopt_dev = nullptr;
    // ---- two-phase (shard) load state ----
    bool planned = false;           // hyt_load_shard_begin done, rows not yet loaded
    bool off_h_pending = false;     // off_h not yet copied back (one rank: fetched during the relabel)
    uint32_t ld_flags = 0;
    uint64_t *ld_off_old = nullptr; // device: caller offsets (original order), until the rows are loaded
    // ---- streams ----
    cudaStream_t main = nullptr;
    std::vector<cudaStream_t> st;   // worker streams
    // ---- last run ----
    int last_algo = -1;
    bool has_result = false;
    uint32_t *val_d = nullptr;
    float *rank_d = nullptr, *delta_d = nullptr;
    std::vector<void *> run_allocs;  // released at the next run / free
    hyt_stats stats{};
    std::vector<hyt_iter> iter_log;
    hyt::EngTime eng_time[hyt::ENG_COUNT];
    hyt::EngTime recompute_time, copy_time, plan_time, rq_time;
    uint64_t eng_chunks[hyt::ENG_COUNT] = {0, 0, 0, 0, 0};
    uint64_t eng_edges[hyt::ENG_COUNT] = {0, 0, 0, 0, 0};
    uint64_t launches = 0;
    void *ctx[4] = {nullptr, nullptr, nullptr, nullptr};   // cached run contexts, one per algorithm
    double est_link_gbs = 0, est_cpt_gbs = 0;              // calibrated rates (cpu_cost = 1)
    double est_zc_req_ns = 0, est_zc_line_ns = 0;          // zero-copy random request / stream line (cost_model = 1)
    // ---- multi-GPU ----
    int rank = 0, world = 1;
    // joined a group (hyt_init_dist / hyt_init_dist_local): the run takes the
    // multi-rank path (split, exchange, frontier merge) even at world 1, where every
    // collective is an identity -- so the NCCL transport runs on a one-GPU box
    bool multi = false;
    void *nccl_comm = nullptr;
    void *local_group = nullptr;   // in-process group (hyt_init_dist_local) instead of NCCL
    uint64_t local_key = 0;
};

namespace hyt {
void load_graph(hyt_graph *g, uint64_t V, uint64_t E, const uint64_t *off, const uint32_t *nbr,
                const uint32_t *w, uint32_t flags);
void load_shard_begin(hyt_graph *g, uint64_t V, const uint32_t *out_deg, const uint32_t *in_deg, uint32_t flags,
                      uint64_t *row_lo, uint64_t *row_hi, uint64_t *edges);
void shard_rows(hyt_graph *g, uint32_t *rows, uint64_t n);
void load_shard_rows(hyt_graph *g, uint64_t nrows, const uint64_t *row_off, const uint32_t *nbr, const uint32_t *w);
void release_adopted(hyt_graph *g);
void run_graph(hyt_graph *g, int algo, uint64_t source);
void debug_plan(hyt_graph *g, int algo, const uint8_t *active, uint64_t *num_parts, uint64_t *bounds,
                uint64_t *t, uint64_t *e, uint64_t *a, uint64_t *z, uint8_t *p);
void get_values(hyt_graph *g, void *out, uint64_t count);
void free_graph(hyt_graph *g);
void release_run_ctx(hyt_graph *g);   // drop cached run buffers (parameters changed)
// host partitioner: greedy 32-MiB sweep by binary search on offsets
std::vector<uint64_t> partition_bounds(const std::vector<uint64_t> &off, uint64_t d1, uint64_t target);
int64_t combine_units(const uint8_t *p, uint64_t n, uint64_t k, uint64_t *units);
void order_units(int64_t nu, const uint64_t *units, const double *part_score, uint32_t *order);
// multi-GPU split: rank r owns vertices [R_r, R_r+1), R_r = the first vertex whose
// edge offset reaches r*E/world (R_world = V); partitions never cross a rank cut
void rank_vertex_range(const std::vector<uint64_t> &off, int world, int rank, uint64_t *v_lo, uint64_t *v_hi);
std::vector<uint64_t> partition_bounds_ranked(const std::vector<uint64_t> &off, uint64_t d1, uint64_t target,
                                              int world);
void rank_partitions(const std::vector<uint64_t> &off, const std::vector<uint64_t> &bounds, int world, int rank,
                     uint64_t *p_lo, uint64_t *p_hi);
// host pointer to the edge store of record width d1, indexed by GLOBAL 16-byte
// chunk (valid for the chunks of the store's vertex range only)
const void *edge_store(const hyt_graph *g, int algo, uint64_t *c0);
const uint4 *host_edges(const hyt_graph *g, int algo);
// multi-GPU exchange (dist.cu)
void dist_init(hyt_graph *g, int rank, int world, const void *uid);
void dist_init_local(hyt_graph *g, int rank, int world, uint64_t group);
void dist_allreduce_min_u32(hyt_graph *g, uint32_t *buf, uint64_t n, cudaStream_t st);
void dist_allreduce_sum_f32(hyt_graph *g, float *buf, uint64_t n, cudaStream_t st);
void dist_allreduce_sum_u64(hyt_graph *g, uint64_t *buf, uint64_t n, cudaStream_t st);
void dist_allreduce_max_u64(hyt_graph *g, uint64_t *buf, uint64_t n, cudaStream_t st);
void dist_allgather_u32(hyt_graph *g, const uint32_t *send, uint32_t *recv, uint64_t n, cudaStream_t st);
void dist_free(hyt_graph *g);
void dist_share_ptrs(hyt_graph *g, void *const *mine, int nptr, void **all, std::vector<void *> &opened,
                     cudaStream_t st);
void dist_close_peers(std::vector<void *> &opened);
}  // namespace hyt
