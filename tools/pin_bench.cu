// pin_bench.cu -- how fast can this box page-lock host memory?  (load-time cost of
// hyt_load_csr: the edge store is pinned, mapped host memory.)
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
int main(int argc, char **argv) {
    size_t gb = argc > 1 ? atol(argv[1]) : 8;
    size_t n = gb << 30;
    cudaFree(0);
    double t = now();
    void *p = nullptr;
    cudaHostAlloc(&p, n, cudaHostAllocMapped);
    printf("cudaHostAlloc %zu GB: %.2fs\n", gb, now() - t);
    t = now();
    memset(p, 1, n);
    printf("  memset after: %.2fs\n", now() - t);
    cudaFreeHost(p);
    for (int huge = 0; huge < 2; ++huge) {
        t = now();
        void *q = mmap(nullptr, n, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (huge) madvise(q, n, MADV_HUGEPAGE);
        std::vector<std::thread> th;
        int nt = 16;
        for (int i = 0; i < nt; ++i) th.emplace_back([=] { memset((char *)q + n / nt * i, 0, n / nt); });
        for (auto &x : th) x.join();
        double t1 = now();
        cudaError_t e = cudaHostRegister(q, n, cudaHostRegisterMapped);
        double t2 = now();
        printf("mmap%s + parallel touch %.2fs + cudaHostRegister %.2fs (%s)\n", huge ? "+THP" : "", t1 - t, t2 - t1,
               cudaGetErrorString(e));
        // chunked parallel registration of a second region
        cudaHostUnregister(q);
        t = now();
        std::vector<std::thread> th2;
        size_t chunk = n / nt;
        std::vector<cudaError_t> errs(nt);
        for (int i = 0; i < nt; ++i) th2.emplace_back([&, i] { errs[i] = cudaHostRegister((char *)q + chunk * i, chunk, cudaHostRegisterMapped); });
        for (auto &x : th2) x.join();
        printf("   16 parallel chunk registrations: %.2fs (%s)\n", now() - t, cudaGetErrorString(errs[0]));
        for (int i = 0; i < nt; ++i) cudaHostUnregister((char *)q + chunk * i);
        munmap(q, n);
    }
    FILE *f = fopen("/sys/kernel/mm/transparent_hugepage/enabled", "r");
    char buf[256] = {0};
    if (f) { fgets(buf, 255, f); fclose(f); }
    printf("THP: %s\n", buf);
    return 0;
}
