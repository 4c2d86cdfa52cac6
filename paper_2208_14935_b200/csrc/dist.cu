// dist.cu -- multi-GPU exchange over NCCL: one process per GPU,
// vertex-range sharding, one reduction of the pushed values per iteration
// (min for BFS/SSSP/CC, sum for PR deltas).  NCCL is resolved at run time with
// dlopen (the torch-bundled libnccl.so.2 when torch is loaded), so the library
// has no link-time NCCL dependency.
//
// A second transport, the in-process group (hyt_init_dist_local), runs the same
// reductions through host memory between threads of one process, each thread
// owning one handle (all on one GPU if need be).  It exists so the multi-rank
// path -- split, exchange, frontier merge, termination -- executes on the one GPU
// a test box has; a job uses NCCL.
#include <dlfcn.h>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include "graph.h"

namespace hyt {

typedef struct { char internal[128]; } nccl_uid_t;
typedef void *nccl_comm_t;
enum { ncclUint32 = 3, ncclUint64 = 5, ncclFloat32 = 7 };
enum { ncclSum = 0, ncclMax = 2, ncclMin = 3 };

struct NcclApi {
    void *h = nullptr;
    int (*GetUniqueId)(nccl_uid_t *) = nullptr;
    int (*CommInitRank)(nccl_comm_t *, int, nccl_uid_t, int) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*AllGather)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*CommDestroy)(nccl_comm_t) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
};

static NcclApi &nccl() {
    static NcclApi api;
    if (!api.h) {
        const char *names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char *n : names) {
            api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (api.h) break;
        }
        if (!api.h) {
            const char *env = getenv("HYT_NCCL_LIB");
            if (env) api.h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        }
        HYT_REQUIRE(api.h != nullptr, HYT_ENCCL, "cannot dlopen libnccl.so.2 (set HYT_NCCL_LIB)");
        api.GetUniqueId = (int (*)(nccl_uid_t *))dlsym(api.h, "ncclGetUniqueId");
        api.CommInitRank = (int (*)(nccl_comm_t *, int, nccl_uid_t, int))dlsym(api.h, "ncclCommInitRank");
        api.AllReduce = (int (*)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t))dlsym(api.h, "ncclAllReduce");
        api.AllGather = (int (*)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t))dlsym(api.h, "ncclAllGather");
        api.CommDestroy = (int (*)(nccl_comm_t))dlsym(api.h, "ncclCommDestroy");
        api.GetErrorString = (const char *(*)(int))dlsym(api.h, "ncclGetErrorString");
        HYT_REQUIRE(api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather && api.CommDestroy, HYT_ENCCL,
                    "libnccl is missing symbols");
    }
    return api;
}

#define HYT_NCCL(call)                                                                          \
    do {                                                                                        \
        int _r = (call);                                                                        \
        if (_r != 0)                                                                            \
            throw Err{HYT_ENCCL, std::string(#call) + ": " +                                    \
                                     (nccl().GetErrorString ? nccl().GetErrorString(_r) : "?")}; \
    } while (0)

// ---------------------------------------------------------------------------
// in-process group
// ---------------------------------------------------------------------------
struct LocalGroup {
    int world = 0, members = 0;
    std::mutex mu;
    std::condition_variable cv;
    uint64_t gen = 0;
    int arrived = 0;
    std::vector<std::vector<uint8_t>> slot;
    std::vector<uint8_t> result;
};
static std::mutex g_groups_mu;
static std::map<uint64_t, std::shared_ptr<LocalGroup>> g_groups;

static void local_barrier(LocalGroup &G) {
    std::unique_lock<std::mutex> l(G.mu);
    const uint64_t my = G.gen;
    if (++G.arrived == G.world) {
        G.arrived = 0;
        ++G.gen;
        G.cv.notify_all();
        return;
    }
    // a rank that failed never arrives: fail instead of hanging the others
    if (!G.cv.wait_for(l, std::chrono::seconds(300), [&] { return G.gen != my; }))
        throw Err{HYT_ENCCL, "in-process group: barrier timed out (a rank failed?)"};
}

enum RedOp { RED_MIN_U32, RED_SUM_F32, RED_SUM_U64, RED_MAX_U64 };

static void local_allreduce(hyt_graph *g, void *buf, uint64_t n, RedOp op, cudaStream_t st) {
    LocalGroup &G = *static_cast<LocalGroup *>(g->local_group);
    const uint64_t esz = (op == RED_SUM_U64 || op == RED_MAX_U64) ? 8 : 4, bytes = n * esz;
    HYT_CUDA(cudaStreamSynchronize(st));
    G.slot[g->rank].resize(bytes);
    HYT_CUDA(copy_sync(G.slot[g->rank].data(), buf, bytes, st));
    local_barrier(G);
    if (g->rank == 0) {    // reduce in rank order (a fixed order: f32 sums are reproducible)
        G.result = G.slot[0];
        for (int r = 1; r < G.world; ++r) {
            const uint8_t *x = G.slot[r].data();
            uint8_t *y = G.result.data();
            for (uint64_t i = 0; i < n; ++i) {
                if (op == RED_MIN_U32) {
                    uint32_t a, b; std::memcpy(&a, y + 4 * i, 4); std::memcpy(&b, x + 4 * i, 4);
                    if (b < a) std::memcpy(y + 4 * i, &b, 4);
                } else if (op == RED_SUM_F32) {
                    float a, b; std::memcpy(&a, y + 4 * i, 4); std::memcpy(&b, x + 4 * i, 4);
                    a += b; std::memcpy(y + 4 * i, &a, 4);
                } else {
                    uint64_t a, b; std::memcpy(&a, y + 8 * i, 8); std::memcpy(&b, x + 8 * i, 8);
                    a = op == RED_SUM_U64 ? a + b : (b > a ? b : a);
                    std::memcpy(y + 8 * i, &a, 8);
                }
            }
        }
    }
    local_barrier(G);
    HYT_CUDA(copy_sync(buf, G.result.data(), bytes, st));
    local_barrier(G);      // nobody starts the next reduction before all have read this one
}

// recv = the ranks' send buffers concatenated in rank order (n u32 each)
static void local_allgather(hyt_graph *g, const void *send, void *recv, uint64_t n, cudaStream_t st) {
    LocalGroup &G = *static_cast<LocalGroup *>(g->local_group);
    const uint64_t bytes = n * 4;
    HYT_CUDA(cudaStreamSynchronize(st));
    G.slot[g->rank].resize(bytes);
    HYT_CUDA(copy_sync(G.slot[g->rank].data(), send, bytes, st));
    local_barrier(G);
    for (int r = 0; r < G.world; ++r)
        HYT_CUDA(copy_sync((uint8_t *)recv + (uint64_t)r * bytes, G.slot[r].data(), bytes, st));
    local_barrier(G);
}

// ---------------------------------------------------------------------------
// peer pointers for the fused push exchange (exchange = 3, §8e): every rank
// publishes nptr device pointers; all[r * nptr + i] = rank r's pointer i, valid in
// this process.  In-process group: the raw pointers (one device, or peers in one
// process).  NCCL job: CUDA IPC handles of the cudaMalloc blocks, all-gathered,
// then opened (lazy peer access over NVLink); dist_close_peers unmaps them.
// ---------------------------------------------------------------------------
void dist_share_ptrs(hyt_graph *g, void *const *mine, int nptr, void **all, std::vector<void *> &opened,
                     cudaStream_t st) {
    if (g->local_group) {
        LocalGroup &G = *static_cast<LocalGroup *>(g->local_group);
        HYT_CUDA(cudaStreamSynchronize(st));
        G.slot[g->rank].assign((const uint8_t *)mine, (const uint8_t *)(mine + nptr));
        local_barrier(G);
        for (int r = 0; r < G.world; ++r) std::memcpy(all + r * nptr, G.slot[r].data(), nptr * sizeof(void *));
        local_barrier(G);
        return;
    }
    HYT_REQUIRE(g->nccl_comm, HYT_ESTATE, "peer exchange needs a multi-rank handle");
    // a CUDA IPC handle maps its whole cudaMalloc block: the published arrays must be
    // block bases, which holds for the library's own allocations but not for
    // sub-allocations of a caller-provided arena (hyt_set_device_arena)
    HYT_REQUIRE(!g->arena.ext, HYT_EINVAL,
                "exchange = 3 across processes needs library-allocated device memory (no hyt_set_device_arena)");
    const uint64_t hb = sizeof(cudaIpcMemHandle_t);
    std::vector<cudaIpcMemHandle_t> h(nptr);
    for (int i = 0; i < nptr; ++i) HYT_CUDA(cudaIpcGetMemHandle(&h[i], mine[i]));
    uint8_t *dsend = nullptr, *drecv = nullptr;
    HYT_CUDA(cudaMalloc(&dsend, hb * nptr));
    HYT_CUDA(cudaMalloc(&drecv, hb * nptr * g->world));
    HYT_CUDA(copy_sync(dsend, h.data(), hb * nptr, st));
    HYT_NCCL(nccl().AllGather(dsend, drecv, hb * nptr / 4, ncclUint32, g->nccl_comm, st));
    std::vector<cudaIpcMemHandle_t> hall((size_t)nptr * g->world);
    HYT_CUDA(cudaMemcpyAsync(hall.data(), drecv, hb * nptr * g->world, cudaMemcpyDeviceToHost, st));
    HYT_CUDA(cudaStreamSynchronize(st));
    cudaFree(dsend);
    cudaFree(drecv);
    for (int r = 0; r < g->world; ++r)
        for (int i = 0; i < nptr; ++i) {
            if (r == g->rank) { all[r * nptr + i] = mine[i]; continue; }
            void *p = nullptr;
            HYT_CUDA(cudaIpcOpenMemHandle(&p, hall[(size_t)r * nptr + i], cudaIpcMemLazyEnablePeerAccess));
            opened.push_back(p);
            all[r * nptr + i] = p;
        }
}

void dist_close_peers(std::vector<void *> &opened) {
    for (void *p : opened) cudaIpcCloseMemHandle(p);
    opened.clear();
}

void dist_init_local(hyt_graph *g, int rank, int world, uint64_t group) {
    std::lock_guard<std::mutex> l(g_groups_mu);
    auto &sp = g_groups[group];
    if (!sp) {
        sp = std::make_shared<LocalGroup>();
        sp->world = world;
        sp->slot.resize(world);
    }
    HYT_REQUIRE(sp->world == world, HYT_EINVAL, "in-process group: world size mismatch");
    HYT_REQUIRE(sp->members < world, HYT_EINVAL, "in-process group: more members than world");
    ++sp->members;
    g->rank = rank;
    g->world = world;
    g->local_group = sp.get();
    g->local_key = group;
    g->multi = true;
}

void dist_init(hyt_graph *g, int rank, int world, const void *uid) {
    g->rank = rank;
    g->world = world;
    // a one-rank communicator too: the job's transport is the same at every world size
    nccl_uid_t id;
    std::memcpy(&id, uid, sizeof(id));
    HYT_CUDA(cudaSetDevice(g->device));
    nccl_comm_t comm = nullptr;
    HYT_NCCL(nccl().CommInitRank(&comm, world, id, rank));
    g->nccl_comm = comm;
    g->multi = true;
}

void dist_allreduce_min_u32(hyt_graph *g, uint32_t *buf, uint64_t n, cudaStream_t st) {
    if (g->local_group) return local_allreduce(g, buf, n, RED_MIN_U32, st);
    HYT_NCCL(nccl().AllReduce(buf, buf, n, ncclUint32, ncclMin, g->nccl_comm, st));
}
void dist_allreduce_sum_f32(hyt_graph *g, float *buf, uint64_t n, cudaStream_t st) {
    if (g->local_group) return local_allreduce(g, buf, n, RED_SUM_F32, st);
    HYT_NCCL(nccl().AllReduce(buf, buf, n, ncclFloat32, ncclSum, g->nccl_comm, st));
}
void dist_allreduce_sum_u64(hyt_graph *g, uint64_t *buf, uint64_t n, cudaStream_t st) {
    if (g->local_group) return local_allreduce(g, buf, n, RED_SUM_U64, st);
    HYT_NCCL(nccl().AllReduce(buf, buf, n, ncclUint64, ncclSum, g->nccl_comm, st));
}
void dist_allreduce_max_u64(hyt_graph *g, uint64_t *buf, uint64_t n, cudaStream_t st) {
    if (g->local_group) return local_allreduce(g, buf, n, RED_MAX_U64, st);
    HYT_NCCL(nccl().AllReduce(buf, buf, n, ncclUint64, ncclMax, g->nccl_comm, st));
}
void dist_allgather_u32(hyt_graph *g, const uint32_t *send, uint32_t *recv, uint64_t n, cudaStream_t st) {
    if (g->local_group) return local_allgather(g, send, recv, n, st);
    HYT_NCCL(nccl().AllGather(send, recv, n, ncclUint32, g->nccl_comm, st));
}
void dist_free(hyt_graph *g) {
    if (g->nccl_comm) {
        nccl().CommDestroy(g->nccl_comm);
        g->nccl_comm = nullptr;
    }
    if (g->local_group) {
        std::lock_guard<std::mutex> l(g_groups_mu);
        auto it = g_groups.find(g->local_key);
        if (it != g_groups.end() && --it->second->members == 0) g_groups.erase(it);
        g->local_group = nullptr;
    }
}

}  // namespace hyt

extern "C" int hyt_nccl_unique_id(void *out) {
    using namespace hyt;
    try {
        HYT_REQUIRE(out != nullptr, HYT_EINVAL, "null output");
        hyt::nccl_uid_t id;
        HYT_NCCL(hyt::nccl().GetUniqueId(&id));
        std::memcpy(out, &id, sizeof(id));
        return HYT_OK;
    } catch (const hyt::Err &e) {
        hyt::set_error(e.msg);
        return e.code;
    }
}
