// dist.cu -- multi-GPU exchange over NCCL: one process per GPU,
// vertex-range sharding, one reduction of the pushed values per iteration
// (min for BFS/SSSP/CC, sum for PR deltas).  NCCL is resolved at run time with
// dlopen (the torch-bundled libnccl.so.2 when torch is loaded), so the library
// has no link-time NCCL dependency.
#include <dlfcn.h>
#include <cstring>
#include "graph.h"

namespace hyt {

typedef struct { char internal[128]; } nccl_uid_t;
typedef void *nccl_comm_t;
enum { ncclUint32 = 3, ncclUint64 = 5, ncclFloat32 = 7 };
enum { ncclSum = 0, ncclMin = 3 };

struct NcclApi {
    void *h = nullptr;
    int (*GetUniqueId)(nccl_uid_t *) = nullptr;
    int (*CommInitRank)(nccl_comm_t *, int, nccl_uid_t, int) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
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
        api.CommDestroy = (int (*)(nccl_comm_t))dlsym(api.h, "ncclCommDestroy");
        api.GetErrorString = (const char *(*)(int))dlsym(api.h, "ncclGetErrorString");
        HYT_REQUIRE(api.GetUniqueId && api.CommInitRank && api.AllReduce && api.CommDestroy, HYT_ENCCL,
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

void dist_init(hyt_graph *g, int rank, int world, const void *uid) {
    g->rank = rank;
    g->world = world;
    if (world == 1) return;
    nccl_uid_t id;
    std::memcpy(&id, uid, sizeof(id));
    HYT_CUDA(cudaSetDevice(g->device));
    nccl_comm_t comm = nullptr;
    HYT_NCCL(nccl().CommInitRank(&comm, world, id, rank));
    g->nccl_comm = comm;
}

void dist_allreduce_min_u32(hyt_graph *g, uint32_t *buf, uint64_t n, cudaStream_t st) {
    HYT_NCCL(nccl().AllReduce(buf, buf, n, ncclUint32, ncclMin, g->nccl_comm, st));
}
void dist_allreduce_sum_f32(hyt_graph *g, float *buf, uint64_t n, cudaStream_t st) {
    HYT_NCCL(nccl().AllReduce(buf, buf, n, ncclFloat32, ncclSum, g->nccl_comm, st));
}
void dist_allreduce_sum_u64(hyt_graph *g, uint64_t *buf, uint64_t n, cudaStream_t st) {
    HYT_NCCL(nccl().AllReduce(buf, buf, n, ncclUint64, ncclSum, g->nccl_comm, st));
}
void dist_free(hyt_graph *g) {
    if (g->nccl_comm) {
        nccl().CommDestroy(g->nccl_comm);
        g->nccl_comm = nullptr;
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
