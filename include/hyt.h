/*
 * hyt.h -- C ABI of the B200-native HyTGraph hot path (libhyt.so).
 *
 * The library runs the per-iteration, frontier-driven push of HyTGraph
 * (Wang et al., arXiv 2208.14935; "the paper", PAPER.md line numbers P:n) over a
 * CSR whose vertex data lives on the GPU and whose edges live in pinned host
 * memory.  Each iteration every vertex-range
 * partition with active edges is served by the engine the paper's cost model
 * picks (Eq. 1-3 and the section 5.1 rule; Algorithm 1):
 *   - ExpTM-filter      : whole-partition async bulk copy + relax
 *   - ExpTM-compaction  : host gather of the active edge lists + one bulk copy
 *                         + relax over the compacted lists
 *   - ImpTM-zero-copy   : relax reading edges straight from mapped host memory
 *                         with aligned 128-byte-line loads
 * combined into tasks, ordered by contribution and
 * overlapped on several CUDA streams.
 *
 * Conventions (all calls):
 *   - Every function returns HYT_OK (0) or a negative HYT_E* code; it never
 *     throws across the ABI.  hyt_last_error() returns a thread-local message
 *     describing the most recent failure of this thread.
 *   - Pointers named *_host are host pointers; nothing in this header is a
 *     device pointer except the optional arena of hyt_set_device_arena().
 *   - Vertex ids in every argument and result are the CALLER's ids ("original"
 *     ids); the hub-sorted internal order is never exposed except by
 *     hyt_get_perm().
 *   - A handle is not thread-safe: one thread at a time per handle.
 *   - One handle drives one GPU (the device given to hyt_init); in a multi-GPU
 *     job each process owns one handle and one GPU (hyt_init_dist).
 *   - There is no CPU fallback: if the CUDA device is unavailable every call
 *     that needs it fails with HYT_ECUDA.
 */
#ifndef HYT_H
#define HYT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ---- */
#define HYT_OK        0
#define HYT_EINVAL   -1   /* bad argument or malformed CSR                         */
#define HYT_ENOMEM   -2   /* device budget or pinned host memory exhausted          */
#define HYT_ECUDA    -3   /* CUDA runtime error (message in hyt_last_error)         */
#define HYT_ESTATE   -4   /* call out of order (e.g. run before load)              */
#define HYT_ENCCL    -5   /* NCCL error in the multi-GPU exchange                   */

/* ---- algorithms ---- */
#define HYT_BFS   0       /* levels from source, push lvl+1, merge min (u32)       */
#define HYT_SSSP  1       /* distances from source, push dist+w, merge min (u32)   */
#define HYT_CC    2       /* min original id per component, on symmetric graphs    */
#define HYT_PR    3       /* delta-PageRank, unnormalised, f32             */

/* ---- load flags ---- */
#define HYT_NO_HUBSORT 1u /* keep the caller's vertex order (skip P:452-462)        */
#define HYT_SYMMETRIC  2u /* the caller asserts the edge set is symmetric (every    */
                          /* (u,v) has (v,u), e.g. a symmetrised undirected graph): */
                          /* enables pull iterations for BFS / CC (param direction) */
#define HYT_ADOPT_HOST 4u /* with HYT_NO_HUBSORT: the caller's u32 id array IS the  */
                          /* edge store (the paper keeps edges in host memory,      */
                          /* P:75): it is page-locked and mapped in place,   */
                          /* not copied, so host memory holds one copy of the ids.  */
                          /* The caller keeps it alive and unmodified until         */
                          /* hyt_free.  Needs a 16-byte aligned array whose first   */
                          /* element is on a 16-byte chunk of the global edge order */
                          /* (always true for world 1).  SSSP's packed (id, weight) */
                          /* records are still built in library memory.             */

/* ---- engine modes (hyt_set_param "engine_mode") ---- */
#define HYT_MODE_HYBRID     0  /* the paper: per-partition cost-model selection    */
#define HYT_MODE_FILTER     1  /* every active partition -> ExpTM-filter           */
#define HYT_MODE_COMPACTION 2  /* every active partition -> ExpTM-compaction       */
#define HYT_MODE_ZEROCOPY   3  /* every active partition -> ImpTM-zero-copy        */
#define HYT_MODE_RESIDENT   4  /* edges copied once into device memory (build     */
                               /* extension); needs budget >= edges     */
#define HYT_MODE_UM         5  /* ImpTM-UM comparison mode (Table V):   */
                               /* edges in cudaMallocManaged memory advised         */
                               /* ReadMostly, migrated on demand by the driver; the */
                               /* budget is enforced by a device-memory balloon     */

/* ---- engine ids in plans (hyt_debug_plan) ---- */
#define HYT_ENG_NONE 0
#define HYT_ENG_F    1
#define HYT_ENG_C    2
#define HYT_ENG_Z    3
#define HYT_ENG_R    4

typedef struct hyt_graph hyt_graph;

/* Per-run statistics (hyt_get_stats).  Bytes are algorithmic host-link bytes:
 * filter = whole copied spans (Eq. 1), compaction = copied compacted chunks,
 * zero-copy = touched 128-byte lines (Eq. 3 requests x m). */
typedef struct {
    uint64_t iterations;
    uint64_t time_ns;              /* hyt_run wall time (host clock)              */
    uint64_t edges_relaxed;        /* sum over tasks of active edges pushed       */
    uint64_t edges_reached;        /* sum of out-degrees of vertices with a value */
    uint64_t bytes_filter, bytes_compaction, bytes_zerocopy;
    uint64_t parts_filter, parts_compaction, parts_zerocopy, parts_resident;
    uint64_t units_filter;         /* combined filter tasks                */
    uint64_t device_bytes_peak;    /* arena high-water mark (<= budget)           */
    uint64_t num_partitions;
    double   kernel_ms;            /* sum of relax-kernel times (CUDA events)     */
    double   copy_ms;              /* sum of H2D copy times (CUDA events)         */
    double   plan_ms;              /* activity/selection/fill kernels             */
    double   gather_ms;            /* host compaction gather (wall)               */
    uint64_t kernel_launches;      /* CUDA kernels this library launched in the run */
    /* Per activity tag: 0 plan (activity/selection/fill), 1 filter relax,
     * 2 compaction relax, 3 zero-copy relax, 4 resident relax, 5 filter
     * recompute pass (relax), 6 host-to-device copies, 7 recompute queue
     * building (k_range_count/fill).  Times are sums of per-launch
     * CUDA-event durations on the launching stream. */
    double   eng_ms[8];
    uint64_t eng_launches[8];
    uint64_t eng_chunks[8];        /* 16-byte edge chunks read by the relax launches */
    uint64_t eng_edges[8];         /* active edges pushed by the relax launches      */
    /* cost-model calibration on this box (cpu_cost / cost_model = 1; else 0):
     * DMA link GB/s, host gather GB/s (Thpt_cpt), zero-copy ns per random
     * 128-B request and per streamed 128-B line. */
    double   cal_link_gbs, cal_cpt_gbs, cal_zc_req_ns, cal_zc_line_ns;
    /* multi-GPU exchange (world > 1): iterations that used the
     * sparse pair all-gather / the dense V-entry reduction, and the payload
     * bytes each rank contributed (pairs x 8 B, or V x 4 B). */
    uint64_t exch_sparse, exch_dense, exch_bytes;
    /* SEP-Graph switching: iterations run as pull; ImpTM-UM:   */
    /* device bytes withheld from the driver so managed pages fit the budget     */
    uint64_t pull_iters, um_balloon_bytes;
    uint64_t exch_peer;            /* iterations exchanged by fused peer push (exchange = 3) */
    uint64_t host_store_bytes;     /* pinned host bytes the library owns for this rank's  */
                                   /* edge store (0 for adopted ids, HYT_ADOPT_HOST)      */
    uint64_t record_bytes;         /* bytes per edge record the run read: 4 (ids, or SSSP  */
                                   /* records packed as id | w << bits(V-1)) or 8 (id, w) */
} hyt_stats;

/* One row per iteration (hyt_get_iter_log), the Fig. 7 / Table VI analog. */
typedef struct {
    uint64_t iteration;
    uint64_t active_vertices, active_edges;
    uint32_t parts_f, parts_c, parts_z, parts_r;
    uint32_t units_f;
    uint32_t dir;                  /* 0 push (data-driven), 1 pull (topology-driven) */
    uint64_t bytes_f, bytes_c, bytes_z;
    double   ms;                   /* wall time of the iteration                  */
} hyt_iter;

/* Create a handle bound to CUDA device `device`.  No device memory is
 * allocated until hyt_load_csr.  Errors: HYT_ECUDA (no such device). */
int hyt_init(hyt_graph **g, int device);

/* Cap every device allocation the handle makes (load and run) at `bytes`
 * (budget = vertex state + staging + optional resident edges).
 * 0 = no cap.  Must be called before hyt_load_csr.  The paper assumes vertex
 * data fits: a run whose vertex state exceeds the budget fails with
 * HYT_ENOMEM; staging shrinks to what is left. */
int hyt_set_device_budget(hyt_graph *g, uint64_t bytes);

/* Optional: sub-allocate everything from a caller-owned device block (e.g. a
 * torch tensor) instead of cudaMalloc; sets the budget to `bytes`.  The block
 * must stay alive until hyt_free.  Call before hyt_load_csr. */
int hyt_set_device_arena(hyt_graph *g, void *dptr, uint64_t bytes);

/* Load a CSR graph.
 *   V, E          : vertices (< 2^32) and stored edges.
 *   off_host      : u64[V+1], off[0]=0, non-decreasing, off[V]=E.
 *   nbr_host      : u32[E] neighbour ids (< V).
 *   w_host        : u32[E] edge weights (SSSP) or NULL.
 *   flags         : 0, or HYT_NO_HUBSORT and/or HYT_SYMMETRIC (the caller
 *                   asserts every (u,v) has (v,u).  The load checks the
 *                   necessary condition in-degree = out-degree for every
 *                   vertex (HYT_EINVAL otherwise); a claim that passes it but
 *                   is still false makes pull iterations wrong).
 * The library hub-sorts (top ceil(0.08 V) by D_o*D_i first,
 * descending, ties by id; the rest in natural order), relabels on the GPU and
 * stores the edges in library-owned pinned, mapped host memory (ids u32[E];
 * with weights also packed (id | w<<32) u64[E]).  The caller's arrays are
 * only read during the call; they are page-locked (cudaHostRegister) for its
 * duration, so they must not already be registered by someone else unless
 * they are cudaHostAlloc memory.  Errors: HYT_EINVAL (malformed CSR),
 * HYT_ENOMEM (pinning or budget), HYT_ECUDA, HYT_ESTATE (already loaded). */
int hyt_load_csr(hyt_graph *g, uint64_t V, uint64_t E, const uint64_t *off_host,
                 const uint32_t *nbr_host, const uint32_t *w_host, uint32_t flags);

/* ---- two-phase (shard) load: no process holds the whole graph ----
 * For graphs larger than one host's memory per rank (BASELINE configs[4], RMAT-30
 * over 8 ranks): every rank passes only O(V) global data plus the rows it
 * serves.
 *   1. hyt_load_shard_begin: out_deg_host / in_deg_host are the GLOBAL out- and
 *      in-degrees, u32[V] each, by caller id (e.g. each rank counts a slice of
 *      the edges and the ranks sum them).  The library hub-sorts
 *      exactly as hyt_load_csr would (same permutation on every rank) and
 *      returns this rank's internal vertex range [*row_lo, *row_hi) (the split
 *      of hyt_rank_range) and its edge count *edges.
 *   2. hyt_get_shard_rows: rows_host[i] = the caller id of internal row
 *      row_lo + i (u32[n], n = row_hi - row_lo).
 *   3. hyt_load_shard_rows: the caller passes exactly those rows in that order
 *      as a local CSR: row_off_host u64[nrows+1] (row_off[0] = 0, row_off[nrows]
 *      = *edges), nbr_host u32[*edges] with CALLER neighbour ids, optional
 *      w_host u32[*edges].  Each row's length must equal its out-degree.  The
 *      library relabels them on the GPU into its pinned store (or adopts the id
 *      array with HYT_ADOPT_HOST).
 * Flags as hyt_load_csr, given to begin.  After step 3 the handle is loaded and
 * everything else is unchanged.  Errors: HYT_EINVAL (degree sums differ, a row
 * length or id out of range), HYT_ESTATE (out of order), HYT_ENOMEM. */
int hyt_load_shard_begin(hyt_graph *g, uint64_t V, const uint32_t *out_deg_host, const uint32_t *in_deg_host,
                         uint32_t flags, uint64_t *row_lo, uint64_t *row_hi, uint64_t *edges);
int hyt_get_shard_rows(hyt_graph *g, uint32_t *rows_host, uint64_t n);
int hyt_load_shard_rows(hyt_graph *g, uint64_t nrows, const uint64_t *row_off_host, const uint32_t *nbr_host,
                        const uint32_t *w_host);

/* Set a run parameter.  Keys (defaults in brackets):
 *   alpha [0.8], beta [0.4]; gamma [0.625]; m [128],
 *   mr [256]; d2 [4]; k [4];
 *   partition_bytes [33554432]; hub_fraction [0.08] (load time);
 *   streams [4]; engine_mode [HYT_MODE_HYBRID]; priority [-1 = auto:
 *   delta for PR, hub otherwise; 0 none, 1 hub, 2 delta];
 *   pack_weights [1] (load time, set before hyt_load_csr): store SSSP records as
 *   one u32, id | w << bits(V-1), when every weight fits the remaining bits (else
 *   the (id, w) u64 records); halves SSSP's host-link bytes;
 *   recompute [1] (process a loaded filter unit once more; 0-8 passes,
 *   > 1 is Subway-style multi-round processing, measured slower on PR);
 *   damping [0.85], epsilon [1e-5], max_iters [1000] (PR; the per-vertex
 *   relative truncation error is at most epsilon/(1-d) = 6.7e-5);
 *   gather_threads [0 = all cores]; compaction_buffer_bytes [0 = auto];
 *   edge_cache [0]: 1 keeps the longest hub-order prefix of partitions that fits
 *   the budget left after the run buffers resident in device memory (served as
 *   engine R at no transfer cost, beyond the paper, whose edges
 *   are re-transferred every iteration); edge_cache_bytes [0 = no cap]
 *   caps its size; cpu_cost [0]: 1 adds Eq. 2's CPU-gather term
 *   (bytes / Thpt_cpt) to the compaction cost in selection, with the
 *   link rate and Thpt_cpt calibrated on this box (or set by link_gbs /
 *   thpt_cpt_gbs); the paper omits the term in selection, so 0 is the
 *   paper's rule; zc_weight [1.0] multiplies Tiz (Eq. 3)
 *   before the comparisons (1 = the paper); cost_model [1]: 2 replaces the
 *   PCIe-3 constants by costs measured on this box for every algorithm, 1 does so
 *   for BFS / SSSP / CC and keeps the paper's constants for delta-PR (measured
 *   1-2 % faster there: the rule has no term for a filter unit's recompute pass) -- Eq. 2's CPU term as with
 *   cpu_cost, and Eq. 3 as (active lists x random-request time + further lines
 *   x streamed-line time) / RTT, probed once per process on a pinned buffer
 *   (zc_req_ns / zc_line_ns / link_gbs / thpt_cpt_gbs override the probes;
 *   cal_probe_bytes [4 GiB, >= 256 MiB] sizes the pinned probe buffer, which is
 *   halved down to 256 MiB if the host cannot pin it; if nothing can be pinned
 *   the rates measured on the B200 pool are used and the run proceeds);
 *   0 is the paper's rule with its PCIe-3 constants.
 *   Kernel tuning (no effect on results): relax_ctas_per_sm [2] (in units of
 *   512 threads), zc_ctas_per_sm [1], zc_ctas [0 = zc_ctas_per_sm x SMs]
 *   (the zero-copy relax grid in 512-thread units), relax_threads [0] (relax CTA size: 0 auto
 *   = 1024 for PR, 512 otherwise; 512; 1024), relax_hot [1] (hub block ids <
 *   relax_hot_v in shared memory: PR delta accumulation in fixed point,
 *   min-algorithm value copy; 0 off, 1 auto, 2 always), relax_hot_v [16384]
 *   (PR hub-block vertices, 32..20480, 8 B of dynamic shared memory each;
 *   min-algorithms use at most 4096; the persistent grid is capped at what
 *   stays resident).
 *   exchange [1] (world > 1): 0 always the dense V-entry
 *   all-reduce; 1 per iteration, all-gather the (id, value) pairs each rank
 *   changed when their bytes (world x max pairs x 8) are below the dense
 *   payload (V x 4), else dense; 2 sparse whenever the pairs fit the buffer.
 *   3: fused peer push -- the relax kernels write a remote destination
 *   straight into its owner's value / delta array and next-frontier bitmap
 *   (atomicMin / atomicAdd / atomicOr through peer pointers: the same device
 *   for an in-process group, CUDA IPC over NVLink for an NCCL job), so no
 *   exchange collective follows the relax, only a barrier; one all-reduce of
 *   the values at the end.  Needs <= 8 ranks and no caller arena.
 *   Results are the same either way.
 *   direction [1] (BFS/CC on a graph loaded with HYT_SYMMETRIC
 *   whose own partitions are all device-resident, one rank): 0 push only;
 *   1 switch per iteration -- BFS by Beamer's rule (pull when frontier edges x
 *   pull_alpha [14] > unexplored edges, back to push when frontier vertices x
 *   pull_beta [24] < V), CC pull when frontier edges x cc_pull_alpha [2] > E;
 *   2 pull in every iteration.  pull_heavy [1024]: lists longer than this are
 *   split into slices across warps.  Results are identical either way.
 *   um_balloon [1] (HYT_MODE_UM with a budget): 1 allocates the device memory
 *   the budget leaves unused by others during the run so the driver keeps at
 *   most the budget's remainder of managed pages resident; um_cold [1]: 1
 *   evicts the managed pages to the host before every run (no reuse across
 *   runs, like the paper's per-run measurements).
 * Errors: HYT_EINVAL on an unknown key or out-of-range value. */
int hyt_set_param(hyt_graph *g, const char *key, double value);

/* Run `algo` from `source` (caller id; ignored by CC and PR) to convergence:
 * until no vertex is active, for PR until no delta exceeds epsilon or
 * max_iters.  Blocking; results stay on the device.  Errors: HYT_EINVAL
 * (source >= V, SSSP without weights), HYT_ESTATE (no graph), HYT_ENOMEM
 * (vertex state over budget), HYT_ECUDA, HYT_ENCCL. */
int hyt_run(hyt_graph *g, int algo, uint64_t source);

/* Copy the last run's results, indexed by caller id, into out_host:
 * u32[V] for BFS/SSSP (0xFFFFFFFF = unreachable) and CC (minimum caller id of
 * the component), f32[V] for PR.  count must equal V.  In a multi-GPU job
 * every rank receives all V values.  Errors: HYT_ESTATE (no run yet),
 * HYT_EINVAL (count != V). */
int hyt_get_values(hyt_graph *g, void *out_host, uint64_t count);

/* Statistics of the last run. */
int hyt_get_stats(hyt_graph *g, hyt_stats *s);

/* Per-iteration rows of the last run: copies min(cap, n) rows, sets *n. */
int hyt_get_iter_log(hyt_graph *g, hyt_iter *rows, uint64_t cap, uint64_t *n);

/* The load-time permutation: new_id_host[caller id] = internal id (u32[V]). */
int hyt_get_perm(hyt_graph *g, uint32_t *new_id_host, uint64_t count);

/* Debug/test hook for plan parity: for algorithm `algo` (fixes
 * d1), evaluate Algorithm 1 on the GPU for the frontier given as a u8[V]
 * array in CALLER ids, without running anything.  Outputs, each sized by the
 * partition count (query it first with all output pointers NULL):
 *   *num_parts; bounds_host u64[N+1] (internal vertex ids); t,e,a,z u64[N];
 *   p_host u8[N] (HYT_ENG_*).  Errors as hyt_run. */
int hyt_debug_plan(hyt_graph *g, int algo, const uint8_t *active_host, uint64_t *num_parts,
                   uint64_t *bounds_host, uint64_t *t_host, uint64_t *e_host,
                   uint64_t *a_host, uint64_t *z_host, uint8_t *p_host);

/* Task combination (Alg. 1 L14-24 with the corrected loop), the
 * host routine the scheduler uses, exposed for CPU tests: splits each maximal
 * run of consecutive HYT_ENG_F entries of p[0..n) into units of <= k.
 * units_host receives pairs (first, one-past-last); returns the unit count
 * (>= 0) or HYT_EINVAL.  Needs no GPU. */
int64_t hyt_combine(const uint8_t *p_host, uint64_t n, uint64_t k, uint64_t *units_host);

/* Contribution-driven ordering of the filter units, the host
 * routine the scheduler uses, exposed for CPU tests: units_host holds nu pairs
 * (first, one-past-last partition) as hyt_combine returns them, part_score_host
 * one score per partition (hub-driven: sum of D_o*D_i over its active vertices;
 * delta-driven: sum of their deltas).  order_host[0..nu) receives the unit
 * indices by descending score (sum over the unit's partitions), ties by unit
 * index.  Returns HYT_OK or HYT_EINVAL.  Needs no GPU. */
int hyt_order_units(int64_t nu, const uint64_t *units_host, const double *part_score_host, uint32_t *order_host);

/* Engine selection for one partition (section 5.1), the exact
 * integer rule the GPU selection kernel evaluates, exposed for CPU tests.
 * Inputs: t = sum of out-degrees of the partition, e = active edges,
 * a = active vertices, z = zero-copy requests; d1 bytes per edge record;
 * the remaining constants come from the handle's parameters (or defaults
 * when g == NULL).  Returns HYT_ENG_* or HYT_EINVAL.  Needs no GPU. */
int hyt_select_engine(const hyt_graph *g, uint64_t t, uint64_t e, uint64_t a, uint64_t z,
                      uint64_t d1);

/* ---- multi-GPU (vertex-range sharding, NCCL over NVLink) ----
 * Call after hyt_init and before hyt_load_csr on every rank.  nccl_uid is the
 * 128-byte ncclUniqueId created by rank 0 (hyt_nccl_unique_id) and broadcast
 * by the caller (e.g. torch.distributed).  Every rank then passes the SAME
 * graph to hyt_load_csr.  Each rank computes the same hub order and keeps in
 * pinned host memory only the edges of its own vertex range, about E/world of
 * them (hyt_rank_range).  It serves the partitions of that range.  Once per
 * iteration the ranks exchange pushed values: min for BFS/SSSP/CC, sum for PR
 * deltas.  world = 1 is allowed: the handle gets a one-rank communicator and
 * takes the same multi-rank path (every collective an identity).  The fused
 * peer push (exchange = 3) publishes CUDA IPC handles of the library's own
 * device blocks and refuses a caller arena (hyt_set_device_arena).
 * Errors: HYT_ENCCL, HYT_EINVAL. */
int hyt_nccl_unique_id(void *uid_out_128_bytes);
int hyt_init_dist(hyt_graph *g, int rank, int world, const void *nccl_uid_128_bytes);

/* The same multi-rank protocol with an in-process transport: `world` handles in
 * one process, each driven by its own thread (they may share one GPU), join
 * group `group` (any key the threads agree on).  The reductions go through host
 * memory in rank order.  For testing the multi-rank path on one device; a job
 * uses hyt_init_dist.  Call before hyt_load_csr.  A rank waiting more than
 * 300 s for the others fails with HYT_ENCCL.  Errors: HYT_EINVAL, HYT_ESTATE. */
int hyt_init_dist_local(hyt_graph *g, int rank, int world, uint64_t group);

/* The vertex-range split of a multi-GPU job (host routine the library uses,
 * exposed for CPU tests).  off_host is u64[V+1], the graph as loaded.  Rank r
 * of `world` owns vertices [*v_lo, *v_hi) = [R_r, R_(r+1)), where R_r is the
 * first vertex whose edge offset reaches r*E/world and R_world = V.  A rank's
 * edge count is therefore within the largest out-degree of E/world; a rank
 * may own no vertex when one vertex holds more than E/world edges.  Inside
 * each rank's range, partitions are the greedy `partition_bytes` sweep at
 * record width d1, so no partition crosses a rank cut.  Rank r owns
 * partitions [*p_lo, *p_hi).  The split does not depend on d1 or
 * partition_bytes, so one pinned edge store per rank serves every algorithm.
 * Returns the total partition count (>= 0) or HYT_EINVAL.  Needs no GPU. */
int64_t hyt_rank_range(const uint64_t *off_host, uint64_t V, uint64_t d1, uint64_t partition_bytes, int world,
                       int rank, uint64_t *p_lo, uint64_t *p_hi, uint64_t *v_lo, uint64_t *v_hi);

/* Pinned host memory the library frees (edge stores, staging) stays registered in
 * a process-wide cache and is reused by the next allocation it fits (a new handle's
 * store, a run context's buffers), because pinning costs about a second per 15 GB.
 * The cache holds at most HYT_PIN_CACHE_GB GiB (environment, default 32; 0 turns
 * it off).  hyt_trim_pinned_cache returns every cached block to the OS.  Needs no
 * handle; thread-safe. */
void hyt_trim_pinned_cache(void);

/* Release everything (device arena, pinned host memory -- into the pinned cache --,
 * streams, NCCL). */
void hyt_free(hyt_graph *g);

/* Thread-local message of this thread's last failure ("" if none). */
const char *hyt_last_error(void);

/* Library version string. */
const char *hyt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HYT_H */
