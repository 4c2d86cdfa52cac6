// hyt_internal.h -- internal types shared by the host scheduler and the sm_100a kernels.
// Nothing here is part of the ABI (include/hyt.h is).
#pragma once
#include <cstdint>
#include <cstddef>
#include <cuda_runtime.h>

namespace hyt {

// ---------------------------------------------------------------------------
// Edge storage is addressed in 16-byte CHUNKS (one uint4 load).  A vertex v's
// edge records occupy bytes [off[v]*d1, off[v+1]*d1) of the edge array; its
// chunk range is [c0(v), c1(v)) with c0 = off*d1/16 (floor), c1 = ceil.  Every
// engine processes a queue of active vertices whose exclusive chunk prefix
// defines a flat chunk space; 8 consecutive lanes read one aligned 128-byte
// line (the EMOGI "merged and aligned" access).
// ---------------------------------------------------------------------------
constexpr int kChunkBytes = 16;
constexpr int kChunksPerThread = 4;     // 16-byte loads in flight per lane
constexpr int kTile = 32 * kChunksPerThread;   // chunks per WARP tile (2 KiB of edges)
#ifndef HYT_HOTV
#define HYT_HOTV 4096
#endif
constexpr int kHotV = HYT_HOTV;         // PR: pushes to vertices < kHotV (the hub block) go to smem first
constexpr int kItemWords = 256;         // bitmap words (8192 vertices) per plan item
constexpr int kItemThreads = 256;       // threads per plan / fill / range CTA

constexpr uint32_t kInf = 0xFFFFFFFFu;

// SM count of the current device (148 on B200), queried once per device; grid
// caps are multiples of it.
inline int num_sms() {
    static thread_local int cache[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

enum Algo : int { ALGO_BFS = 0, ALGO_SSSP = 1, ALGO_CC = 2, ALGO_PR = 3 };
// k_relax instantiation of SSSP over packed 4-byte records (id | w << wshift)
constexpr int ALGO_SSSP_PACKED = 4;
enum Eng : int { ENG_NONE = 0, ENG_F = 1, ENG_C = 2, ENG_Z = 3, ENG_R = 4, ENG_COUNT = 5 };
enum Mode : int { MODE_HYBRID = 0, MODE_FILTER = 1, MODE_COMPACTION = 2, MODE_ZEROCOPY = 3, MODE_RESIDENT = 4, MODE_UM = 5 };

__host__ __device__ inline uint64_t chunk_lo(uint64_t edge, uint32_t d1) { return (edge * d1) >> 4; }
__host__ __device__ inline uint64_t chunk_hi(uint64_t edge, uint32_t d1) { return (edge * d1 + 15) >> 4; }

// Exact-integer cost-model constants (rationals for alpha/beta/gamma).
struct CostParams {
    uint64_t d1, d2, m, mr;
    uint64_t an, ad, bn, bd, gn, gd;
    int m_shift;                 // log2(m) when m is a power of two, else -1
    uint64_t cn, cd;             // Eq. 2 CPU term: link rate / Thpt_cpt as cn/cd (cn = 0: paper practice)
    uint64_t zn, zd;             // weight on Tiz (zn/zd = 1: the paper's Eq. 3)
    // B200-calibrated Eq. 3 (cost_model = 1): each active list costs one random
    // request (zr) plus its further lines at the stream rate (zs), in RTT units x zden.
    // zr = 0: the paper's Eq. 3 with gamma.
    uint64_t zr, zs, zden;
};

// Section 5.1 engine selection, evaluated identically on host (tests) and device.
// t: partition edges, e: active edges, a: active vertices, z: zero-copy requests.
__host__ __device__ inline int select_engine(uint64_t t, uint64_t e, uint64_t a, uint64_t z, uint64_t r,
                                             const CostParams &c) {
    if (e == 0) return ENG_NONE;
    typedef unsigned __int128 u128;
    const uint64_t tlp = c.m * c.mr;
    const uint64_t Tef = (t * c.d1 + tlp - 1) / tlp;                     // Eq. 1
    uint64_t Tec = (e * c.d1 + a * c.d2 + tlp - 1) / tlp;                // Eq. 2 (transfer term)
    if (c.cn) {   // + (bytes / Thpt_cpt) in TLP-time units (RTT = m*MR bytes at the link rate)
        const u128 b = (u128)(e * c.d1 + a * c.d2) * c.cn;
        const u128 q = (u128)c.cd * tlp;
        Tec += (uint64_t)((b + q - 1) / q);
    }
    const uint64_t nz = (z + c.mr - 1) / c.mr;                            // Eq. 3 TLP count
    // Tiz = nz * RTT_zc, RTT_zc = gamma + (1-gamma) e/t  ->  nz*(gn t + (gd-gn) e) / (gd t)
    u128 num, den;
    if (c.zr) {   // calibrated: (r*zr + (z - r)*zs) / zden
        num = ((u128)r * c.zr + (u128)(z > r ? z - r : 0) * c.zs) * c.zn;
        den = (u128)c.zden * c.zd;
    } else {
        num = (u128)nz * ((u128)c.gn * t + (u128)(c.gd - c.gn) * e) * c.zn;
        den = (u128)c.gd * t * c.zd;
    }
    const bool c1 = (u128)Tec * c.ad < (u128)c.an * Tef;                 // Tec < alpha Tef
    const bool c2 = (u128)Tec * c.bd * den < (u128)c.bn * num;            // Tec < beta Tiz
    if (c1 && c2) return ENG_C;
    if (num < (u128)Tef * den) return ENG_Z;                             // Tiz < Tef
    return ENG_F;                                                        // ties -> F
}

// Per-partition, per-iteration aggregates (written by the activity kernel).
struct PartIter {
    uint64_t e, a, z;          // active edges / vertices / zero-copy requests (Eq. 1-3 inputs)
    uint64_t ent, chunks;      // queue entries (active, degree > 0) and their 16-B chunks
    uint64_t hub;              // sum of D_o*D_i over active vertices (hub priority)
    uint64_t ent_base, chunk_base;   // offsets inside this partition's engine segment
    double dsum;               // sum of delta over active vertices (delta priority)
    uint32_t p, pad;           // engine
};

// Per-iteration segment header (written by the last activity CTA).
struct SegHdr {
    uint64_t ent_base[ENG_COUNT];     // first entry of each engine's segment in the queue
    uint64_t ent_count[ENG_COUNT];
    uint64_t chunk_total[ENG_COUNT];
    uint64_t tile_base[ENG_COUNT];    // first tile-map slot of each segment
    uint64_t parts[ENG_COUNT];
    uint64_t active_vertices, active_edges, zc_requests;
    uint32_t done;                    // CTA completion counter (reset by the last CTA)
    uint32_t pad;
};

// Everything a plan / relax kernel needs about the graph and the run state.
struct DevState {
    uint64_t V, W;              // vertices, bitmap words
    const uint64_t *off;        // u64[V+1] (hub-sorted order)
    const uint32_t *din;        // u32[V] in-degree (hub priority)
    uint32_t *val;              // u32[V] BFS/SSSP/CC
    float *rank, *delta;        // f32[V] PR
    uint32_t *bm_cur, *bm_next; // u32[W]
    uint32_t d1;
    uint32_t wshift;            // SSSP with d1 = 4: packed records, weight = record >> wshift
    int algo;
    float damping, epsilon;
    uint32_t hot_v;             // hub-block size in shared memory (relax_hot_v)
    int relax_nt;               // relax CTA size: 512 or 1024 threads (relax_threads)
    uint32_t bands;             // destination bands for device-resident edges (relax_bands; 0 = auto)
};

// Fused multi-rank push (exchange = 3): a destination outside the own range
// [rb[rank], rb[rank+1]) is relaxed straight into its owner's arrays through
// these peer pointers (same device, or IPC-mapped over NVLink), so no exchange
// collective follows the relax -- only a barrier.
constexpr int kMaxPeers = 8;
struct PeerPush {
    uint32_t n = 0;                       // ranks (0 = off)
    uint64_t lo = 0, hi = 0;              // own range
    uint64_t rb[kMaxPeers + 1] = {};      // rank vertex bounds
    uint32_t *val[kMaxPeers] = {};        // owners' value arrays (min-algorithms)
    uint32_t *bm[kMaxPeers] = {};         // owners' NEXT frontier bitmaps (this iteration)
    float *delta[kMaxPeers] = {};         // owners' delta arrays (PR)
};

struct QueueBufs {
    uint32_t *qv;        // entry -> vertex
    uint64_t *qpre;      // entry -> exclusive chunk prefix within its segment
    uint64_t *qbeg;      // entry -> first edge index off[v]
    uint32_t *qdeg;      // entry -> out-degree
    float *qaux;         // entry -> PR contribution d*delta/D_o
    uint32_t *tile;      // tile -> first entry whose chunks cover the tile start
    uint64_t cap, tile_cap;
};

// Per-stream recompute (range queue) scratch.
struct RangeBufs {
    QueueBufs q;
    uint32_t *taken;     // taken bitmap words of the range
    float *scratch;      // PR: exchanged delta per vertex of the range
    uint64_t *cta_agg;   // per-CTA (entries, chunks)
    uint64_t *total;     // [0] entries, [1] chunks
    uint64_t *acc;       // run statistics: [1] chunks, [2] edges (accumulated)
    uint64_t vcap, cta_cap;
};

// Plan items: runs of <= kItemWords bitmap words inside one partition.
struct Items {
    const uint32_t *part;     // item -> partition
    const uint64_t *w0, *w1;  // item word range
    const uint64_t *first;    // partition -> first item (N+1 entries)
};
struct ItemAgg { uint64_t e, a, z, ent, chunks, hub; double dsum; };
struct PlanBufs {
    PartIter *parts;          // zeroed before every plan
    ItemAgg *iagg;
    uint64_t *ibase;          // item -> (entry base, chunk base) inside its engine segment
    SegHdr *hdr;              // zeroed before every plan
};

// ---- kernel launchers (plan.cu, kernels.cu) ----
void launch_pr_frontier(const DevState &s, cudaStream_t st);
// Partitions [p_lo, cache_hi) have their edges resident in device memory (engine R).
void launch_plan(const DevState &s, const uint64_t *bounds, const uint64_t *t_static, Items it,
                 uint64_t item_lo, uint64_t item_hi, uint64_t p_lo, uint64_t p_hi, uint64_t cache_hi, int mode,
                 const CostParams &cp, PlanBufs pb, cudaStream_t st);
void launch_fill(const DevState &s, const uint64_t *bounds, Items it, uint64_t item_lo, uint64_t item_hi,
                 PlanBufs pb, QueueBufs q, cudaStream_t st);
// Edge source for a relax launch.
struct EdgeSrc {
    const uint4 *base;   // chunk base pointer (device, staging slot, mapped host, compact buffer)
    int64_t shift;       // ABS: address = base + (c0(v) + j - shift)
    bool compact;        // COMPACT: address = base + (c - c_lo)
    bool host = false;   // edges read over the link (zero-copy, managed): never re-read per band
};
// Relax over window [c_lo, c_hi) of the segment whose entries are [seg_first, seg_end)
// with seg_chunks chunks; dev_tot (range queues) overrides seg_end/seg_chunks/c_hi.
void launch_relax(const DevState &s, const QueueBufs &q, uint64_t tile_base, uint64_t seg_first,
                  uint64_t seg_end, uint64_t seg_chunks, uint64_t c_lo, uint64_t c_hi,
                  const uint64_t *dev_tot, EdgeSrc src, int max_ctas, cudaStream_t st, int hot = 1,
                  const PeerPush *peer = nullptr);
void launch_take_delta(const DevState &s, const QueueBufs &q, uint64_t e_lo, uint64_t e_hi, cudaStream_t st);
void launch_range_queue(const DevState &s, uint64_t v_lo, uint64_t v_hi, RangeBufs r, cudaStream_t st);
void launch_init_values(const DevState &s, uint64_t src_internal, const uint32_t *old_of, cudaStream_t st);
// times a zero-copy probe over the mapped edge store (mode 0 random lines, 1 stream)
float time_zc_probe(const uint4 *mapped, uint64_t nlines, int mode, uint32_t *sink, uint64_t *lines_read,
                    cudaStream_t st);
void launch_collect_changed(int pr, uint64_t V, uint64_t lo, uint64_t hi, const uint32_t *val, const uint32_t *snap,
                            const float *delta, uint2 *pairs, uint64_t cap, unsigned long long *cnt,
                            cudaStream_t st);
void launch_pad_pairs(uint2 *pairs, const unsigned long long *cnt, uint64_t n, cudaStream_t st);
void launch_apply_pairs(int pr, const uint2 *pairs, uint64_t n, uint64_t lo, uint64_t hi, uint32_t *val,
                        float *delta, uint32_t *bm_next, cudaStream_t st);
void launch_mark_improved(const uint32_t *val, const uint32_t *snap, uint64_t lo, uint64_t hi, uint32_t *bm,
                          cudaStream_t st);
void launch_gather_out(const DevState &s, const uint32_t *new_id, void *out_dev, cudaStream_t st);

// pull iteration over own vertices [v_lo, v_hi) with device-resident edges (pull.cu);
// slices (sv, e0, e1) cover the lists longer than `heavy`
void launch_pull(int algo, const uint64_t *off, const uint32_t *nbr, uint32_t *val, const uint32_t *bm_cur,
                 uint32_t *bm_next, uint64_t v_lo, uint64_t v_hi, uint32_t heavy, const uint32_t *sv,
                 const uint64_t *e0, const uint64_t *e1, uint64_t ns, uint32_t lvl, cudaStream_t st);
void launch_own_words(const uint32_t *bm, uint32_t *out, uint64_t nw, uint64_t lo, uint64_t hi, cudaStream_t st);

// ---- load-time kernels (load.cu) ----
struct LoadOut;
}  // namespace hyt
