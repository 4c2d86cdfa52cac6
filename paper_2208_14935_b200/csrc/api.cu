// api.cu -- the extern "C" boundary (include/hyt.h).  Every entry point catches
// everything and returns an HYT_E* code; messages go to a thread-local buffer.
#include <cstring>
#include <string>
#include "graph.h"

namespace hyt {
static thread_local std::string t_err;
void set_error(const std::string &msg) { t_err = msg; }
const char *get_error() { return t_err.c_str(); }
}  // namespace hyt

using namespace hyt;

#define HYT_GUARD(...)                                                    \
    try {                                                                  \
        __VA_ARGS__;                                                       \
        return HYT_OK;                                                     \
    } catch (const Err &e) {                                               \
        set_error(e.msg);                                                  \
        return e.code;                                                     \
    } catch (const std::exception &e) {                                   \
        set_error(std::string("internal: ") + e.what());                   \
        return HYT_ECUDA;                                                  \
    } catch (...) {                                                        \
        set_error("internal: unknown exception");                          \
        return HYT_ECUDA;                                                  \
    }

extern "C" {

void hyt_trim_pinned_cache(void) { pinned_trim(); }

const char *hyt_version(void) { return "hyt-b200 0.1 (sm_100a)"; }
const char *hyt_last_error(void) { return get_error(); }

int hyt_init(hyt_graph **out, int device) {
    HYT_GUARD({
        HYT_REQUIRE(out != nullptr, HYT_EINVAL, "null handle pointer");
        *out = nullptr;
        int n = 0;
        HYT_CUDA(cudaGetDeviceCount(&n));
        HYT_REQUIRE(device >= 0 && device < n, HYT_ECUDA, "no CUDA device " + std::to_string(device));
        HYT_CUDA(cudaSetDevice(device));
        hyt_graph *g = new hyt_graph();
        g->device = device;
        cudaError_t e = cudaStreamCreateWithFlags(&g->main, cudaStreamNonBlocking);
        if (e != cudaSuccess) { delete g; HYT_CUDA(e); }
        *out = g;
    })
}

int hyt_set_device_budget(hyt_graph *g, uint64_t bytes) {
    HYT_GUARD({
        HYT_REQUIRE(g, HYT_EINVAL, "null handle");
        HYT_REQUIRE(!g->loaded, HYT_ESTATE, "set the budget before hyt_load_csr");
        HYT_REQUIRE(!g->arena.ext, HYT_ESTATE, "an external arena is set");
        g->arena.budget = bytes;
    })
}

int hyt_set_device_arena(hyt_graph *g, void *dptr, uint64_t bytes) {
    HYT_GUARD({
        HYT_REQUIRE(g && dptr && bytes, HYT_EINVAL, "bad arena");
        HYT_REQUIRE(!g->loaded && g->arena.blocks.empty(), HYT_ESTATE, "set the arena before hyt_load_csr");
        g->arena.ext = (char *)dptr;
        g->arena.ext_size = bytes;
        g->arena.ext_top = 0;
        g->arena.budget = bytes;
    })
}

int hyt_load_csr(hyt_graph *g, uint64_t V, uint64_t E, const uint64_t *off, const uint32_t *nbr,
                 const uint32_t *w, uint32_t flags) {
    HYT_GUARD({
        HYT_REQUIRE(g, HYT_EINVAL, "null handle");
        HYT_REQUIRE((flags & ~(HYT_NO_HUBSORT | HYT_SYMMETRIC | HYT_ADOPT_HOST)) == 0, HYT_EINVAL, "unknown flags");
        load_graph(g, V, E, off, nbr, w, flags);
    })
}

int hyt_load_shard_begin(hyt_graph *g, uint64_t V, const uint32_t *out_deg, const uint32_t *in_deg, uint32_t flags,
                         uint64_t *row_lo, uint64_t *row_hi, uint64_t *edges) {
    HYT_GUARD({
        HYT_REQUIRE(g && row_lo && row_hi && edges, HYT_EINVAL, "null argument");
        HYT_REQUIRE((flags & ~(HYT_NO_HUBSORT | HYT_SYMMETRIC | HYT_ADOPT_HOST)) == 0, HYT_EINVAL, "unknown flags");
        load_shard_begin(g, V, out_deg, in_deg, flags, row_lo, row_hi, edges);
    })
}

int hyt_get_shard_rows(hyt_graph *g, uint32_t *rows, uint64_t n) {
    HYT_GUARD({
        HYT_REQUIRE(g && (rows || n == 0), HYT_EINVAL, "null argument");
        shard_rows(g, rows, n);
    })
}

int hyt_load_shard_rows(hyt_graph *g, uint64_t nrows, const uint64_t *row_off, const uint32_t *nbr,
                        const uint32_t *w) {
    HYT_GUARD({
        HYT_REQUIRE(g, HYT_EINVAL, "null handle");
        load_shard_rows(g, nrows, row_off, nbr, w);
    })
}

int hyt_set_param(hyt_graph *g, const char *key, double v) {
    HYT_GUARD({
        HYT_REQUIRE(g && key, HYT_EINVAL, "null argument");
        Params &p = g->prm;
        const std::string k(key);
        const int old_mode = p.engine_mode;
        auto in = [&](double lo, double hi) {
            HYT_REQUIRE(v >= lo && v <= hi, HYT_EINVAL, k + " out of range");
        };
        auto integral = [&]() { HYT_REQUIRE(v == (double)(int64_t)v, HYT_EINVAL, k + " must be an integer"); };
        if (k == "alpha") { in(1e-6, 1.0); p.alpha = v; }
        else if (k == "beta") { in(1e-6, 1.0); p.beta = v; }
        else if (k == "gamma") { in(1e-6, 1.0); p.gamma = v; }
        else if (k == "m") { integral(); in(1, 1 << 20); p.m = (uint64_t)v; }
        else if (k == "mr") { integral(); in(1, 1 << 20); p.mr = (uint64_t)v; }
        else if (k == "d2") { integral(); in(0, 64); p.d2 = (uint64_t)v; }
        else if (k == "k") { integral(); in(1, 1024); p.k = (uint64_t)v; }
        else if (k == "partition_bytes") { integral(); in(16, 1e12); p.partition_bytes = (uint64_t)v; }
        else if (k == "hub_fraction") { in(0, 1); HYT_REQUIRE(!g->loaded && !g->planned, HYT_ESTATE, "hub_fraction applies at load"); p.hub_fraction = v; }
        else if (k == "streams") { integral(); in(1, 8); p.streams = (int)v; }
        else if (k == "engine_mode") { integral(); in(0, 5); p.engine_mode = (int)v; }
        else if (k == "priority") { integral(); in(-1, 2); p.priority = (int)v; }
        else if (k == "recompute") { integral(); in(0, 8); p.recompute = (int)v; }
        else if (k == "damping") { in(1e-6, 1 - 1e-6); p.damping = v; }
        else if (k == "epsilon") { in(0, 1); p.epsilon = v; }
        else if (k == "pack_weights") { integral(); in(0, 1); p.pack_weights = (int)v; }
        else if (k == "max_iters") { integral(); in(1, 1e9); p.max_iters = (uint64_t)v; }
        else if (k == "gather_threads") { integral(); in(0, 256); p.gather_threads = (int)v; }
        else if (k == "compaction_buffer_bytes") { integral(); in(0, 1e12); p.compaction_buffer_bytes = (uint64_t)v; }
        else if (k == "zc_ctas_per_sm") { integral(); in(1, 32); p.zc_ctas_per_sm = (int)v; }
        else if (k == "zc_ctas") { integral(); in(0, 1 << 16); p.zc_ctas = (int)v; }
        else if (k == "relax_ctas_per_sm") { integral(); in(1, 32); p.relax_ctas_per_sm = (int)v; }
        else if (k == "exchange") { integral(); in(0, 3); p.exchange = (int)v; }
        else if (k == "relax_hot") { integral(); in(0, 2); p.relax_hot = (int)v; }
        else if (k == "relax_hot_v") { integral(); in(32, 20480); p.relax_hot_v = (uint64_t)v; }
        else if (k == "relax_bands") { integral(); in(0, 64); p.relax_bands = (int)v; }
        else if (k == "relax_threads") {
            integral();
            HYT_REQUIRE(v == 0 || v == 512 || v == 1024, HYT_EINVAL, "relax_threads must be 0 (auto), 512 or 1024");
            p.relax_threads = (int)v;
        }
        else if (k == "edge_cache") { integral(); in(0, 1); p.edge_cache = (int)v; }
        else if (k == "edge_cache_bytes") { integral(); in(0, 1e13); p.edge_cache_bytes = (uint64_t)v; }
        else if (k == "cpu_cost") { integral(); in(0, 1); p.cpu_cost = (int)v; }
        else if (k == "zc_weight") { in(0.001, 1000); p.zc_weight = v; }
        else if (k == "cost_model") { integral(); in(0, 2); p.cost_model = (int)v; }
        else if (k == "zc_req_ns") { in(0, 1e6); p.zc_req_ns = v; g->est_zc_req_ns = v; }
        else if (k == "zc_line_ns") { in(0, 1e6); p.zc_line_ns = v; g->est_zc_line_ns = v; }
        else if (k == "cal_probe_bytes") { integral(); in(256.0 * (1 << 20), 1e12); p.cal_probe_bytes = (uint64_t)v; }
        else if (k == "thpt_cpt_gbs") { in(0, 1e6); p.thpt_cpt_gbs = v; g->est_cpt_gbs = v; }
        else if (k == "link_gbs") { in(0, 1e6); p.link_gbs = v; g->est_link_gbs = v; }
        else if (k == "direction") { integral(); in(0, 2); p.direction = (int)v; }
        else if (k == "pull_alpha") { in(1e-3, 1e9); p.pull_alpha = v; }
        else if (k == "pull_beta") { in(1e-3, 1e9); p.pull_beta = v; }
        else if (k == "cc_pull_alpha") { in(1e-3, 1e9); p.cc_pull_alpha = v; }
        else if (k == "pull_heavy") { integral(); in(32, 1 << 30); p.pull_heavy = (uint64_t)v; }
        else if (k == "um_balloon") { integral(); in(0, 1); p.um_balloon = (int)v; }
        else if (k == "um_cold") { integral(); in(0, 1); p.um_cold = (int)v; }
        else throw Err{HYT_EINVAL, "unknown parameter '" + k + "'"};
        // buffers depend on the parameters -- except a switch among the four transfer
        // modes (hybrid / filter / compaction / zero-copy), which share one buffer
        // layout as long as no partial edge cache is built (hybrid only)
        auto transfer = [](int m) { return m >= MODE_HYBRID && m <= MODE_ZEROCOPY; };
        const bool keep = k == "engine_mode" && transfer(old_mode) && transfer(p.engine_mode) && !p.edge_cache;
        if (g->loaded && !keep) release_run_ctx(g);
    })
}

int hyt_run(hyt_graph *g, int algo, uint64_t source) {
    HYT_GUARD({
        HYT_REQUIRE(g, HYT_EINVAL, "null handle");
        run_graph(g, algo, source);
    })
}

int hyt_get_values(hyt_graph *g, void *out, uint64_t count) {
    HYT_GUARD({
        HYT_REQUIRE(g && out, HYT_EINVAL, "null argument");
        get_values(g, out, count);
    })
}

int hyt_get_stats(hyt_graph *g, hyt_stats *s) {
    HYT_GUARD({
        HYT_REQUIRE(g && s, HYT_EINVAL, "null argument");
        *s = g->stats;
    })
}

int hyt_get_iter_log(hyt_graph *g, hyt_iter *rows, uint64_t cap, uint64_t *n) {
    HYT_GUARD({
        HYT_REQUIRE(g && n, HYT_EINVAL, "null argument");
        *n = g->iter_log.size();
        const uint64_t m = std::min<uint64_t>(cap, g->iter_log.size());
        if (rows && m) std::memcpy(rows, g->iter_log.data(), m * sizeof(hyt_iter));
    })
}

int hyt_get_perm(hyt_graph *g, uint32_t *new_id, uint64_t count) {
    HYT_GUARD({
        HYT_REQUIRE(g && new_id, HYT_EINVAL, "null argument");
        HYT_REQUIRE(g->loaded, HYT_ESTATE, "no graph loaded");
        HYT_REQUIRE(count == g->V, HYT_EINVAL, "count != V");
        HYT_CUDA(cudaSetDevice(g->device));
        HYT_CUDA(copy_sync(new_id, g->new_id_d, g->V * 4, g->main));
    })
}

int hyt_debug_plan(hyt_graph *g, int algo, const uint8_t *active, uint64_t *num_parts, uint64_t *bounds,
                   uint64_t *t, uint64_t *e, uint64_t *a, uint64_t *z, uint8_t *p) {
    HYT_GUARD({
        HYT_REQUIRE(g && num_parts, HYT_EINVAL, "null argument");
        HYT_REQUIRE(active || (!bounds && !t && !p), HYT_EINVAL, "null frontier");
        debug_plan(g, algo, active, num_parts, bounds, t, e, a, z, p);
    })
}

int hyt_order_units(int64_t nu, const uint64_t *units, const double *part_score, uint32_t *order) {
    HYT_GUARD({
        HYT_REQUIRE(nu >= 0 && (nu == 0 || (units && part_score && order)), HYT_EINVAL, "bad arguments");
        order_units(nu, units, part_score, order);
    })
}

int64_t hyt_combine(const uint8_t *p, uint64_t n, uint64_t k, uint64_t *units) {
    if ((!p && n) || !units || k == 0) { set_error("bad arguments"); return HYT_EINVAL; }
    return combine_units(p, n, k, units);
}

int hyt_select_engine(const hyt_graph *g, uint64_t t, uint64_t e, uint64_t a, uint64_t z, uint64_t d1) {
    if (d1 == 0 || d1 > 64) { set_error("bad d1"); return HYT_EINVAL; }
    Params def;
    const Params &p = g ? g->prm : def;
    return select_engine(t, e, a, z, a, make_cost(p, (uint32_t)d1));
}

int64_t hyt_rank_range(const uint64_t *off, uint64_t V, uint64_t d1, uint64_t partition_bytes, int world, int rank,
                       uint64_t *p_lo, uint64_t *p_hi, uint64_t *v_lo, uint64_t *v_hi) {
    if (!off || V == 0 || d1 == 0 || partition_bytes == 0 || world < 1 || rank < 0 || rank >= world || !p_lo ||
        !p_hi || !v_lo || !v_hi) {
        set_error("bad arguments");
        return HYT_EINVAL;
    }
    try {
        std::vector<uint64_t> o(off, off + V + 1);
        std::vector<uint64_t> b = partition_bounds_ranked(o, d1, partition_bytes, world);
        rank_partitions(o, b, world, rank, p_lo, p_hi);
        *v_lo = b[*p_lo];
        *v_hi = b[*p_hi];
        return (int64_t)(b.size() - 1);
    } catch (...) {
        set_error("internal error");
        return HYT_EINVAL;
    }
}

int hyt_init_dist(hyt_graph *g, int rank, int world, const void *uid) {
    HYT_GUARD({
        HYT_REQUIRE(g && uid, HYT_EINVAL, "null argument");
        HYT_REQUIRE(world >= 1 && rank >= 0 && rank < world, HYT_EINVAL, "bad rank/world");
        HYT_REQUIRE(!g->loaded, HYT_ESTATE, "call hyt_init_dist before hyt_load_csr");
        dist_init(g, rank, world, uid);
    })
}

int hyt_init_dist_local(hyt_graph *g, int rank, int world, uint64_t group) {
    HYT_GUARD({
        HYT_REQUIRE(g, HYT_EINVAL, "null argument");
        HYT_REQUIRE(world >= 1 && rank >= 0 && rank < world, HYT_EINVAL, "bad rank/world");
        HYT_REQUIRE(!g->loaded, HYT_ESTATE, "call hyt_init_dist_local before hyt_load_csr");
        HYT_REQUIRE(!g->nccl_comm && !g->local_group, HYT_ESTATE, "handle already joined a group");
        dist_init_local(g, rank, world, group);
    })
}

void hyt_free(hyt_graph *g) {
    if (!g) return;
    try { free_graph(g); } catch (...) {}
    delete g;
}

}  // extern "C"
