// load.cu -- hyt_load_csr: CSR validation, hub sorting and the
// relabelled copy of the edges into library-owned pinned, mapped host memory
// (the paper's storage split: vertex data on the GPU, edges in host memory,
// P:75).  All per-vertex and per-edge work runs on the GPU; the
// caller's edge arrays are read in place through a temporary host mapping.
#include <cub/cub.cuh>
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

namespace hyt {

// ---------------------------------------------------------------------------
// pinned mapped host memory
// ---------------------------------------------------------------------------
static std::mutex g_pin_mu;
static std::unordered_map<void *, uint64_t> g_pinned;

void *pinned_alloc(uint64_t bytes) {
    const uint64_t huge = 2ull << 20;
    const uint64_t len = (bytes + huge - 1) / huge * huge;
    void *p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) throw Err{HYT_ENOMEM, "mmap of " + std::to_string(len) + " B failed"};
    madvise(p, len, MADV_HUGEPAGE);
    // parallel first touch (the registration pins resident pages)
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
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
    std::lock_guard<std::mutex> l(g_pin_mu);
    g_pinned[p] = len;
    return p;
}

void pinned_free(void *p) {
    if (!p) return;
    uint64_t len = 0;
    {
        std::lock_guard<std::mutex> l(g_pin_mu);
        auto it = g_pinned.find(p);
        if (it == g_pinned.end()) return;
        len = it->second;
        g_pinned.erase(it);
    }
    cudaHostUnregister(p);
    munmap(p, len);
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
__global__ void k_indeg(const uint32_t *__restrict__ nbr, uint64_t E, uint64_t V, uint32_t *__restrict__ din,
                        uint32_t *__restrict__ bad) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += stride) {
        const uint32_t x = nbr[i];
        if (x >= V) { *bad = 1; continue; }
        atomicAdd(&din[x], 1u);
    }
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
__global__ void k_key_hist(const uint64_t *__restrict__ off, const uint32_t *__restrict__ din, uint64_t V,
                           uint64_t prefix, uint64_t mask, int shift, unsigned long long *__restrict__ hist) {
    __shared__ unsigned int sh[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; v < V; v += stride) {
        const uint64_t k = hub_key(off, din, v);
        if ((k & mask) == prefix) atomicAdd(&sh[(k >> shift) & 0xFF], 1u);
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

__global__ void __launch_bounds__(512)
k_relabel_tiles(uint64_t V, uint64_t e_lo, uint64_t e_hi, const uint64_t *__restrict__ off_old,
                const uint64_t *__restrict__ off_new,
                const uint32_t *__restrict__ old_of, const uint32_t *__restrict__ new_id,
                const uint32_t *__restrict__ nbr_in, const uint32_t *__restrict__ w_in,
                uint32_t *__restrict__ nbr_out, uint64_t *__restrict__ ew_out) {
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
                if (i < nr) s_old[i] = off_old[old_of[r0 + i]];
            }
            __syncthreads();
            const uint64_t stop = min(e_end, s_new[nr]);   // edges the staged rows cover
            for (uint64_t x = e + threadIdx.x; x < stop; x += blockDim.x) {
                int lo = 0, hi = (int)nr - 1;              // last staged row starting <= x
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (s_new[mid] <= x) lo = mid; else hi = mid - 1;
                }
                const uint64_t src = s_old[lo] + (x - s_new[lo]);
                const uint32_t y = new_id[nbr_in[src]];
                nbr_out[x] = y;
                if (ew_out) ew_out[x] = (uint64_t)y | ((uint64_t)w_in[src] << 32);
            }
            e = stop;
        }
    }
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
// load
// ---------------------------------------------------------------------------
static double wall_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void load_graph(hyt_graph *g, uint64_t V, uint64_t E, const uint64_t *off, const uint32_t *nbr,
                const uint32_t *w, uint32_t flags) {
    const bool verbose = getenv("HYT_VERBOSE") != nullptr;
    double tph = wall_ms();
    auto phase = [&](const char *name) {
        if (!verbose) return;
        cudaStreamSynchronize(g->main);
        const double t = wall_ms();
        fprintf(stderr, "[hyt load] %-28s %8.1f ms\n", name, t - tph);
        tph = t;
    };
    HYT_REQUIRE(!g->loaded, HYT_ESTATE, "graph already loaded");
    HYT_REQUIRE(V > 0 && V < (1ull << 32), HYT_EINVAL, "V must be in [1, 2^32)");
    HYT_REQUIRE(off != nullptr && (E == 0 || nbr != nullptr), HYT_EINVAL, "null CSR array");
    HYT_REQUIRE(off[0] == 0, HYT_EINVAL, "off[0] != 0");
    HYT_REQUIRE(off[V] == E, HYT_EINVAL, "off[V] != E");
    for (uint64_t v = 0; v < V; ++v)
        HYT_REQUIRE(off[v] <= off[v + 1], HYT_EINVAL, "offsets not non-decreasing at " + std::to_string(v));
    HYT_CUDA(cudaSetDevice(g->device));
    Arena &A = g->arena;
    cudaStream_t st = g->main;
    g->V = V; g->E = E; g->weighted = (w != nullptr); g->symmetric = (flags & HYT_SYMMETRIC) != 0;

    // persistent device arrays
    g->off_d = arena_new<uint64_t>(A, V + 1, "offsets");
    g->new_id_d = arena_new<uint32_t>(A, V, "new_id");
    g->old_of_d = arena_new<uint32_t>(A, V, "old_of");
    g->din_d = arena_new<uint32_t>(A, V, "in_degree");

    // temporaries (released in reverse order)
    std::vector<void *> tmp;
    auto T = [&](uint64_t bytes, const char *what) { void *p = A.alloc(bytes, what); tmp.push_back(p); return p; };
    uint64_t *off_old = (uint64_t *)T((V + 1) * 8, "load: caller offsets");
    uint32_t *din = (uint32_t *)T(V * 4 + 16, "load: in-degree");
    uint32_t *bad = (uint32_t *)T(16, "load: flag");
    uint32_t *nonhub = (uint32_t *)T(V * 4 + 16, "load: non-hub flags");
    uint32_t *nonhub_scan = (uint32_t *)T(V * 4 + 16, "load: non-hub scan");
    HYT_CUDA(cudaMemcpyAsync(off_old, off, (V + 1) * 8, cudaMemcpyHostToDevice, st));
    HYT_CUDA(cudaMemsetAsync(din, 0, V * 4, st));
    HYT_CUDA(cudaMemsetAsync(bad, 0, 4, st));

    phase("validate + device alloc");
    // One rank owns every edge, so the store's size is known now: pin it on a host
    // thread while the GPU computes in-degrees and the hub sort.
    struct EarlyStore {
        std::thread th;
        void *n = nullptr, *w = nullptr;
        std::exception_ptr err;
        ~EarlyStore() {
            if (th.joinable()) th.join();
            pinned_free(n);
            pinned_free(w);
        }
    } early;
    const uint64_t early_nbytes = ((E * 4 + 15) & ~15ull) + 32, early_wbytes = ((E * 8 + 15) & ~15ull) + 32;
    if (g->world == 1) {
        const int dev = g->device;
        const bool weighted = w != nullptr;
        early.th = std::thread([&early, dev, weighted, early_nbytes, early_wbytes] {
            try {
                cudaSetDevice(dev);
                early.n = pinned_alloc(early_nbytes);
                if (weighted) early.w = pinned_alloc(early_wbytes);
            } catch (...) {
                early.err = std::current_exception();
            }
        });
    }
    HostView vn, vw;
    try {
        vn.open(nbr, E * 4);
        if (w) vw.open(w, E * 4);
        phase("map caller arrays");
        if (E) k_indeg<<<grid_for(E), 256, 0, st>>>((const uint32_t *)vn.dev, E, V, din, bad);
        uint32_t bad_h = 0;
        HYT_CUDA(cudaMemcpyAsync(&bad_h, bad, 4, cudaMemcpyDeviceToHost, st));
        HYT_CUDA(cudaStreamSynchronize(st));
        HYT_REQUIRE(bad_h == 0, HYT_EINVAL, "neighbour id >= V");
        if (flags & HYT_SYMMETRIC) {
            k_sym_degrees<<<grid_for(V), 256, 0, st>>>(off_old, din, V, bad);
            HYT_CUDA(cudaMemcpyAsync(&bad_h, bad, 4, cudaMemcpyDeviceToHost, st));
            HYT_CUDA(cudaStreamSynchronize(st));
            HYT_REQUIRE(bad_h == 0, HYT_EINVAL, "HYT_SYMMETRIC: some vertex's in-degree differs from its out-degree");
        }
        phase("in-degrees (zero-copy)");

        // ---- hub sort: top h = ceil(frac*V) by D_o*D_i ----
        const uint64_t fden = 1000000;
        const uint64_t fnum = (uint64_t)(g->prm.hub_fraction * (double)fden + 0.5);
        uint64_t h = (flags & HYT_NO_HUBSORT) ? 0 : (fnum * V + fden - 1) / fden;
        if (h > V) h = V;
        k_fill_u32<<<grid_for(V), 256, 0, st>>>(nonhub, V, 1u);
        if (h > 0) {
            // exact radix select of the h-th largest key T (8 passes of 8 bits), then
            // only the h hubs are sorted: O(V) memory instead of a full-V key sort
            unsigned long long *hist = (unsigned long long *)T(256 * 8, "load: select histogram");
            std::vector<unsigned long long> hh(256);
            uint64_t prefix = 0, mask = 0, kk = h;
            for (int pass = 0; pass < 8; ++pass) {
                const int shift = 56 - 8 * pass;
                HYT_CUDA(cudaMemsetAsync(hist, 0, 256 * 8, st));
                k_key_hist<<<grid_for(V, 256, num_sms() * 8), 256, 0, st>>>(off_old, din, V, prefix, mask, shift, hist);
                HYT_CUDA(cudaMemcpyAsync(hh.data(), hist, 256 * 8, cudaMemcpyDeviceToHost, st));
                HYT_CUDA(cudaStreamSynchronize(st));
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
            const uint64_t Tkey = prefix, ties = kk;      // hubs: key > T, plus `ties` of key == T by id
            k_tie_flags<<<grid_for(V), 256, 0, st>>>(off_old, din, V, Tkey, nonhub);
            size_t t0 = 0;
            HYT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t0, nonhub, nonhub_scan, (int)V, st));
            void *tsc = T(t0 + 16, "load: select scan temp");
            HYT_CUDA(cub::DeviceScan::ExclusiveSum(tsc, t0, nonhub, nonhub_scan, (int)V, st));
            k_hub_flags<<<grid_for(V), 256, 0, st>>>(off_old, din, V, Tkey, ties, nonhub_scan, nonhub);
            HYT_CUDA(cub::DeviceScan::ExclusiveSum(tsc, t0, nonhub, nonhub_scan, (int)V, st));
            uint32_t *hid = (uint32_t *)T(h * 4 + 16, "load: hub ids");
            uint32_t *hid2 = (uint32_t *)T(h * 4 + 16, "load: hub ids sorted");
            uint64_t *hkey = (uint64_t *)T(h * 8 + 16, "load: hub keys");
            uint64_t *hkey2 = (uint64_t *)T(h * 8 + 16, "load: hub keys sorted");
            k_scatter_hubs<<<grid_for(V), 256, 0, st>>>(off_old, din, V, nonhub, nonhub_scan, hid, hkey);
            size_t tb = 0;
            HYT_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, hkey, hkey2, hid, hid2, (int)h, 0, 64, st));
            void *tsort = T(tb + 16, "load: hub sort temp");
            // stable: equal keys keep ascending ids
            HYT_CUDA(cub::DeviceRadixSort::SortPairsDescending(tsort, tb, hkey, hkey2, hid, hid2, (int)h, 0, 64, st));
            k_fill_u32<<<grid_for(V), 256, 0, st>>>(nonhub, V, 1u);
            k_mark_hubs<<<grid_for(h), 256, 0, st>>>(hid2, h, g->new_id_d, nonhub);
            HYT_CUDA(cudaStreamSynchronize(st));
            for (void *q : {(void *)tsort, (void *)hkey2, (void *)hkey, (void *)hid2, (void *)hid, tsc, (void *)hist}) {
                A.release(q);
                tmp.erase(std::find(tmp.begin(), tmp.end(), q));
            }
        }
        uint64_t *deg2 = (uint64_t *)T((V + 1) * 8, "load: degrees");
        size_t ts = 0;
        HYT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, ts, nonhub, nonhub_scan, (int)V, st));
        void *tscan = T(ts + 16, "load: scan temp");
        HYT_CUDA(cub::DeviceScan::ExclusiveSum(tscan, ts, nonhub, nonhub_scan, (int)V, st));
        k_finish_perm<<<grid_for(V), 256, 0, st>>>(V, h, nonhub, nonhub_scan, off_old, din, g->new_id_d,
                                                  g->old_of_d, deg2, g->din_d);
        size_t t2 = 0;
        HYT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t2, deg2, g->off_d, (int)(V + 1), st));
        void *tscan2 = T(t2 + 16, "load: scan temp 2");
        HYT_CUDA(cub::DeviceScan::ExclusiveSum(tscan2, t2, deg2, g->off_d, (int)(V + 1), st));
        g->off_h.resize(V + 1);
        HYT_CUDA(cudaMemcpyAsync(g->off_h.data(), g->off_d, (V + 1) * 8, cudaMemcpyDeviceToHost, st));
        phase("hub sort + new offsets");

        HYT_CUDA(cudaStreamSynchronize(st));   // off_h ready
        // ---- pinned mapped edge store of this rank's vertex range (the
        // whole graph at world 1), from a 16-byte chunk boundary, 16-B padded so chunk
        // loads never overrun ----
        rank_vertex_range(g->off_h, g->world, g->rank, &g->store_v_lo, &g->store_v_hi);
        const uint64_t e_lo = g->off_h[g->store_v_lo], e_hi = g->off_h[g->store_v_hi];
        g->store_c0[0] = e_lo / 4;                          // first chunk of u32 ids
        g->store_c0[1] = e_lo / 2;                          // first chunk of u64 records
        const uint64_t nbase = g->store_c0[0] * 4, wbase = g->store_c0[1] * 2;
        const uint64_t nbytes = (((e_hi - nbase) * 4 + 15) & ~15ull) + 32;
        const uint64_t wbytes = (((e_hi - wbase) * 8 + 15) & ~15ull) + 32;
        if (early.th.joinable()) {
            early.th.join();
            if (early.err) std::rethrow_exception(early.err);
            HYT_REQUIRE(nbytes == early_nbytes && (!w || wbytes == early_wbytes), HYT_ESTATE,
                        "edge store size mismatch");
            g->nbr_h = (uint32_t *)early.n;                 // ownership moves to the handle
            g->ew_h = (uint64_t *)early.w;
            early.n = early.w = nullptr;
        } else {
            g->nbr_h = (uint32_t *)pinned_alloc(nbytes);  // zero-filled (padding included)
            if (w) g->ew_h = (uint64_t *)pinned_alloc(wbytes);
        }
        uint32_t *nbr_out = nullptr;
        uint64_t *ew_out = nullptr;
        HYT_CUDA(cudaHostGetDevicePointer((void **)&nbr_out, g->nbr_h, 0));
        if (w) HYT_CUDA(cudaHostGetDevicePointer((void **)&ew_out, g->ew_h, 0));
        phase("pin edge store");

        if (e_hi > e_lo) {
            k_relabel_tiles<<<num_sms() * 4, 512, 0, st>>>(V, e_lo, e_hi, off_old, g->off_d, g->old_of_d, g->new_id_d,
                                                      (const uint32_t *)vn.dev, (const uint32_t *)vw.dev,
                                                      nbr_out - nbase, ew_out ? ew_out - wbase : nullptr);
        }
        HYT_CUDA(cudaStreamSynchronize(st));
        HYT_CUDA(cudaGetLastError());
        phase("relabel edges (zero-copy)");
    } catch (...) {
        cudaStreamSynchronize(st);
        vn.close(); vw.close();
        for (auto it = tmp.rbegin(); it != tmp.rend(); ++it) A.release(*it);
        throw;
    }
    vn.close(); vw.close();
    for (auto it = tmp.rbegin(); it != tmp.rend(); ++it) A.release(*it);
    phase("unmap + release");
    g->loaded = true;
}

}  // namespace hyt
