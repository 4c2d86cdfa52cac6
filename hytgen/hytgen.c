/*
 * hytgen.c -- seeded, counter-based synthetic graph INPUT generator.
 *
 * This module is shared by both sides of the parity harness (the CPU oracle
 * under oracle/ and the CUDA library under paper_2208_14935_b200/).  It holds
 * none of HyTGraph's arithmetic: it only produces CSR graphs (the input format
 * the paper assumes, PAPER.md P:142 / P:316) and the SSSP edge weights.
 *
 *  - RMAT edges (Chakrabarti et al.; the paper's synthetic graphs) with
 *    (a,b,c,d) quadrant probabilities, quantised to 1/65536, four levels per
 *    64-bit draw.  Every random number is splitmix64(seed_mix ^ counter), where
 *    the counter encodes (edge index, attempt, draw group), so any thread (or
 *    any rank) can regenerate any edge.
 *  - Rejection to V vertices: an edge whose endpoints fall outside [0,V) is
 *    redrawn with the next attempt counter (up to 255 attempts, then mod V).
 *  - CSR build: degree count, exclusive scan, scatter, then every row sorted
 *    ascending so the CSR is canonical (independent of thread timing).
 *  - Optional symmetrisation (undirected graphs): each generated
 *    edge is stored in both directions.
 *  - Weights: w(u,v) = 1 + splitmix64(seed ^ (min(u,v)<<32 |
 *    max(u,v))) mod 63, i.e. integers in 1..63 (BASELINE.json configs[0]),
 *    symmetric in (u,v) and keyed on ORIGINAL ids.
 *
 * Threads: pthreads, one contiguous edge range per thread.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>
#include <stdio.h>
#include <time.h>
static double now_s(void){struct timespec t;clock_gettime(CLOCK_MONOTONIC,&t);return t.tv_sec+1e-9*t.tv_nsec;}

static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct {
    int scale;
    uint64_t V, E;
    uint32_t thr_a, thr_ab, thr_abc; /* cumulative thresholds on a 16-bit draw */
    uint64_t seed_mix;
} rmat_params;

/* Draw one RMAT edge for edge index e; returns 0 on success. */
static inline void rmat_edge(const rmat_params *p, uint64_t e, uint32_t *su, uint32_t *sv) {
    for (uint64_t attempt = 0; attempt < 256; ++attempt) {
        uint64_t u = 0, v = 0;
        uint64_t word = 0;
        for (int l = 0; l < p->scale; ++l) {
            if ((l & 3) == 0) {
                uint64_t ctr = (e << 12) | (attempt << 4) | (uint64_t)(l >> 2);
                word = splitmix64(p->seed_mix ^ ctr);
            }
            uint32_t r = (uint32_t)(word & 0xFFFFu);
            word >>= 16;
            /* quadrant: r<A:(0,0)  A<=r<AB:(0,1)  AB<=r<ABC:(1,0)  r>=ABC:(1,1) */
            uint64_t ga = r >= p->thr_a, gab = r >= p->thr_ab, gabc = r >= p->thr_abc;
            uint64_t bu = gab, bv = (ga ^ gab) | gabc;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        if (u < p->V && v < p->V) { *su = (uint32_t)u; *sv = (uint32_t)v; return; }
        if (attempt == 255) { *su = (uint32_t)(u % p->V); *sv = (uint32_t)(v % p->V); return; }
    }
}

static void make_params(rmat_params *p, int scale, uint64_t V, uint64_t E,
                        double a, double b, double c, uint64_t seed) {
    p->scale = scale; p->V = V; p->E = E;
    double ca = a, cab = a + b, cabc = a + b + c;
    p->thr_a = (uint32_t)(ca * 65536.0 + 0.5);
    p->thr_ab = (uint32_t)(cab * 65536.0 + 0.5);
    p->thr_abc = (uint32_t)(cabc * 65536.0 + 0.5);
    p->seed_mix = splitmix64(seed);
}

int hytgen_num_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    const char *env = getenv("HYTGEN_THREADS");
    if (env) n = atol(env);
    if (n < 1) n = 1;
    if (n > 256) n = 256;
    return (int)n;
}

/* ---------------- edge-list generation (small graphs, tests) ---------------- */

int hytgen_rmat_edges(int scale, uint64_t V, uint64_t E, double a, double b, double c,
                      uint64_t seed, uint32_t *src, uint32_t *dst) {
    if (scale < 1 || scale > 32 || V == 0 || V > (1ull << scale)) return -1;
    rmat_params p; make_params(&p, scale, V, E, a, b, c, seed);
    for (uint64_t e = 0; e < E; ++e) rmat_edge(&p, e, &src[e], &dst[e]);
    return 0;
}

/* ---------------- multithreaded CSR build ---------------- */

typedef struct {
    const rmat_params *p;
    uint64_t e0, e1;
    int symmetric;
    uint32_t *deg;      /* pass 1: atomic degree counters */
    uint64_t *cursor;   /* pass 2: atomic fill cursors (start = off[v]) */
    uint32_t *nbr;
    int pass;
} csr_job;

static void *csr_worker(void *arg) {
    csr_job *j = (csr_job *)arg;
    for (uint64_t e = j->e0; e < j->e1; ++e) {
        uint32_t u, v;
        rmat_edge(j->p, e, &u, &v);
        if (j->pass == 1) {
            __atomic_fetch_add(&j->deg[u], 1u, __ATOMIC_RELAXED);
            if (j->symmetric) __atomic_fetch_add(&j->deg[v], 1u, __ATOMIC_RELAXED);
        } else {
            uint64_t pos = __atomic_fetch_add(&j->cursor[u], 1ull, __ATOMIC_RELAXED);
            j->nbr[pos] = v;
            if (j->symmetric) {
                pos = __atomic_fetch_add(&j->cursor[v], 1ull, __ATOMIC_RELAXED);
                j->nbr[pos] = u;
            }
        }
    }
    return NULL;
}

static int cmp_u32(const void *x, const void *y) {
    uint32_t a = *(const uint32_t *)x, b = *(const uint32_t *)y;
    return (a > b) - (a < b);
}

typedef struct { const uint64_t *off; uint32_t *nbr; uint64_t v0, v1; } sort_job;

static void *sort_worker(void *arg) {
    sort_job *j = (sort_job *)arg;
    for (uint64_t v = j->v0; v < j->v1; ++v) {
        uint64_t b = j->off[v], e = j->off[v + 1];
        uint64_t n = e - b;
        uint32_t *a = j->nbr + b;
        if (n <= 32) {
            for (uint64_t i = 1; i < n; ++i) {
                uint32_t x = a[i]; uint64_t k = i;
                while (k > 0 && a[k - 1] > x) { a[k] = a[k - 1]; --k; }
                a[k] = x;
            }
        } else {
            qsort(a, n, sizeof(uint32_t), cmp_u32);
        }
    }
    return NULL;
}

/* Rows are sorted by a dynamic split so the hub rows do not serialise one thread. */
static void sort_rows(const uint64_t *off, uint32_t *nbr, uint64_t V, int nt) {
    pthread_t th[256]; sort_job jobs[256];
    uint64_t E = off[V];
    uint64_t v = 0;
    int t = 0;
    for (; t < nt && v < V; ++t) {
        uint64_t target = (E / nt) * (t + 1);
        uint64_t lo = v, hi = V;
        if (t == nt - 1) hi = V;
        else {
            /* first vertex whose offset >= target */
            uint64_t L = v, R = V;
            while (L < R) { uint64_t m = (L + R) / 2; if (off[m] < target) L = m + 1; else R = m; }
            hi = L > v ? L : v + 1;
            if (hi > V) hi = V;
        }
        jobs[t].off = off; jobs[t].nbr = nbr; jobs[t].v0 = lo; jobs[t].v1 = hi;
        pthread_create(&th[t], NULL, sort_worker, &jobs[t]);
        v = hi;
    }
    for (int i = 0; i < t; ++i) pthread_join(th[i], NULL);
}

/*
 * Build the CSR of an RMAT graph.  off: u64[V+1]; nbr: u32[E_stored] where
 * E_stored = E (directed) or 2E (symmetric).  Returns 0 on success.
 */
int hytgen_rmat_csr(int scale, uint64_t V, uint64_t E, double a, double b, double c,
                    uint64_t seed, int symmetric, uint64_t *off, uint32_t *nbr) {
    if (scale < 1 || scale > 32 || V == 0 || V > (1ull << scale)) return -1;
    rmat_params p; make_params(&p, scale, V, E, a, b, c, seed);
    int nt = hytgen_num_threads();
    uint32_t *deg = (uint32_t *)calloc(V, sizeof(uint32_t));
    if (!deg) return -2;
    pthread_t th[256]; csr_job jobs[256];
    int verbose = getenv("HYTGEN_VERBOSE") != NULL;
    double t0 = now_s();
    for (int pass = 1; pass <= 2; ++pass) {
        uint64_t *cursor = NULL;
        if (pass == 2) {
            off[0] = 0;
            for (uint64_t v = 0; v < V; ++v) off[v + 1] = off[v] + deg[v];
            cursor = (uint64_t *)malloc(V * sizeof(uint64_t));
            if (!cursor) { free(deg); return -2; }
            memcpy(cursor, off, V * sizeof(uint64_t));
        }
        for (int t = 0; t < nt; ++t) {
            jobs[t].p = &p; jobs[t].e0 = E * t / nt; jobs[t].e1 = E * (t + 1) / nt;
            jobs[t].symmetric = symmetric; jobs[t].deg = deg; jobs[t].cursor = cursor;
            jobs[t].nbr = nbr; jobs[t].pass = pass;
            pthread_create(&th[t], NULL, csr_worker, &jobs[t]);
        }
        for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
        free(cursor);
        if (verbose) fprintf(stderr, "hytgen pass %d: %.2fs\n", pass, now_s() - t0);
    }
    free(deg);
    sort_rows(off, nbr, V, nt);
    if (verbose) fprintf(stderr, "hytgen sort: %.2fs\n", now_s() - t0);
    return 0;
}

/* ---------------- per-rank (shard) generation, SURVEY §7.2 #6 ----------------
 * A multi-GPU job never materialises the whole graph in one process.  Every
 * edge is a pure function of its index (counter-based draws), so a rank can
 *   1. count the degrees of an edge-index range [e0, e1) (each rank one slice;
 *      the caller sums the slices across ranks: O(V) per rank), and
 *   2. build the rows of ANY vertex subset by regenerating every edge and
 *      keeping those whose source is in the subset (O(E) draws, O(own edges)
 *      memory).  slot[v] = the local row of v, or 0xFFFFFFFF if v is not kept;
 *      rows come out in local-row order, each sorted ascending, identical to
 *      the same rows of hytgen_rmat_csr's full CSR.                            */

typedef struct {
    const rmat_params *p;
    uint64_t e0, e1;
    int symmetric;
    uint32_t *out_deg, *in_deg;
} deg_job;

static void *deg_worker(void *arg) {
    deg_job *j = (deg_job *)arg;
    for (uint64_t e = j->e0; e < j->e1; ++e) {
        uint32_t u, v;
        rmat_edge(j->p, e, &u, &v);
        __atomic_fetch_add(&j->out_deg[u], 1u, __ATOMIC_RELAXED);
        __atomic_fetch_add(&j->in_deg[v], 1u, __ATOMIC_RELAXED);
        if (j->symmetric) {
            __atomic_fetch_add(&j->out_deg[v], 1u, __ATOMIC_RELAXED);
            __atomic_fetch_add(&j->in_deg[u], 1u, __ATOMIC_RELAXED);
        }
    }
    return NULL;
}

/* Adds the stored out-/in-degrees of edges [e0, e1) into out_deg / in_deg (u32[V]). */
int hytgen_rmat_degrees(int scale, uint64_t V, uint64_t E, double a, double b, double c, uint64_t seed,
                        int symmetric, uint64_t e0, uint64_t e1, uint32_t *out_deg, uint32_t *in_deg) {
    if (scale < 1 || scale > 32 || V == 0 || V > (1ull << scale) || e0 > e1 || e1 > E) return -1;
    rmat_params p; make_params(&p, scale, V, E, a, b, c, seed);
    int nt = hytgen_num_threads();
    pthread_t th[256]; deg_job jobs[256];
    for (int t = 0; t < nt; ++t) {
        jobs[t].p = &p; jobs[t].symmetric = symmetric; jobs[t].out_deg = out_deg; jobs[t].in_deg = in_deg;
        jobs[t].e0 = e0 + (e1 - e0) * t / nt; jobs[t].e1 = e0 + (e1 - e0) * (t + 1) / nt;
        pthread_create(&th[t], NULL, deg_worker, &jobs[t]);
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    return 0;
}

typedef struct {
    const rmat_params *p;
    uint64_t e0, e1;
    int symmetric, pass;
    const uint32_t *slot;
    uint32_t *cnt;      /* pass 1 */
    uint64_t *cursor;   /* pass 2 */
    uint32_t *nbr;
} rows_job;

static void *rows_worker(void *arg) {
    rows_job *j = (rows_job *)arg;
    for (uint64_t e = j->e0; e < j->e1; ++e) {
        uint32_t u, v;
        rmat_edge(j->p, e, &u, &v);
        for (int dir = 0; dir < 1 + j->symmetric; ++dir) {
            uint32_t s = dir ? v : u, d = dir ? u : v;
            uint32_t r = j->slot[s];
            if (r == 0xFFFFFFFFu) continue;
            if (j->pass == 1) __atomic_fetch_add(&j->cnt[r], 1u, __ATOMIC_RELAXED);
            else j->nbr[__atomic_fetch_add(&j->cursor[r], 1ull, __ATOMIC_RELAXED)] = d;
        }
    }
    return NULL;
}

/* Rows of the kept vertices: off_local u64[nrows+1]; nbr_local sized by the
 * caller from the global out-degrees (sum over kept vertices), checked here.
 * Returns 0, -1 (bad args), -2 (no memory), -3 (edge count != cap). */
int hytgen_rmat_rows(int scale, uint64_t V, uint64_t E, double a, double b, double c, uint64_t seed,
                     int symmetric, const uint32_t *slot, uint64_t nrows, uint64_t *off_local,
                     uint32_t *nbr_local, uint64_t cap) {
    if (scale < 1 || scale > 32 || V == 0 || V > (1ull << scale)) return -1;
    rmat_params p; make_params(&p, scale, V, E, a, b, c, seed);
    int nt = hytgen_num_threads();
    uint32_t *cnt = (uint32_t *)calloc(nrows ? nrows : 1, sizeof(uint32_t));
    uint64_t *cursor = (uint64_t *)malloc((nrows ? nrows : 1) * sizeof(uint64_t));
    if (!cnt || !cursor) { free(cnt); free(cursor); return -2; }
    pthread_t th[256]; rows_job jobs[256];
    for (int pass = 1; pass <= 2; ++pass) {
        if (pass == 2) {
            off_local[0] = 0;
            for (uint64_t r = 0; r < nrows; ++r) off_local[r + 1] = off_local[r] + cnt[r];
            if (off_local[nrows] != cap) { free(cnt); free(cursor); return -3; }
            memcpy(cursor, off_local, nrows * sizeof(uint64_t));
        }
        for (int t = 0; t < nt; ++t) {
            jobs[t].p = &p; jobs[t].symmetric = symmetric; jobs[t].pass = pass; jobs[t].slot = slot;
            jobs[t].cnt = cnt; jobs[t].cursor = cursor; jobs[t].nbr = nbr_local;
            jobs[t].e0 = E * t / nt; jobs[t].e1 = E * (t + 1) / nt;
            pthread_create(&th[t], NULL, rows_worker, &jobs[t]);
        }
        for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    }
    free(cnt); free(cursor);
    sort_rows(off_local, nbr_local, nrows, nt);
    return 0;
}

/* Weights of local rows: rows[r] = the original id of local row r. */
int hytgen_weights_rows(uint64_t nrows, const uint32_t *rows, const uint64_t *off_local, const uint32_t *nbr,
                        uint64_t seed, uint32_t *w) {
    for (uint64_t r = 0; r < nrows; ++r) {
        uint64_t u = rows[r];
        for (uint64_t k = off_local[r]; k < off_local[r + 1]; ++k) {
            uint64_t v = nbr[k];
            uint64_t lo = u < v ? u : v, hi = u < v ? v : u;
            w[k] = 1u + (uint32_t)(splitmix64(seed ^ ((lo << 32) | hi)) % 63u);
        }
    }
    return 0;
}

/* Build a CSR from an explicit edge list (tests, crafted graphs). Rows sorted. */
int hytgen_csr_from_edges(uint64_t V, uint64_t M, const uint32_t *src, const uint32_t *dst,
                          int symmetric, uint64_t *off, uint32_t *nbr) {
    uint64_t *cnt = (uint64_t *)calloc(V + 1, sizeof(uint64_t));
    if (!cnt) return -2;
    for (uint64_t i = 0; i < M; ++i) {
        if (src[i] >= V || dst[i] >= V) { free(cnt); return -1; }
        cnt[src[i]]++;
        if (symmetric) cnt[dst[i]]++;
    }
    off[0] = 0;
    for (uint64_t v = 0; v < V; ++v) off[v + 1] = off[v] + cnt[v];
    for (uint64_t v = 0; v < V; ++v) cnt[v] = off[v];
    for (uint64_t i = 0; i < M; ++i) {
        nbr[cnt[src[i]]++] = dst[i];
        if (symmetric) nbr[cnt[dst[i]]++] = src[i];
    }
    free(cnt);
    sort_rows(off, nbr, V, 1);
    return 0;
}

/* ---------------- SSSP weights ---------------- */

typedef struct { const uint64_t *off; const uint32_t *nbr; uint32_t *w; uint64_t v0, v1, seed; } w_job;

static void *w_worker(void *arg) {
    w_job *j = (w_job *)arg;
    for (uint64_t u = j->v0; u < j->v1; ++u) {
        for (uint64_t k = j->off[u]; k < j->off[u + 1]; ++k) {
            uint64_t v = j->nbr[k];
            uint64_t lo = u < v ? u : v, hi = u < v ? v : u;
            j->w[k] = 1u + (uint32_t)(splitmix64(j->seed ^ ((lo << 32) | hi)) % 63u);
        }
    }
    return NULL;
}

/* w[k] for every stored edge k = (u, nbr[k]); ids are the generator's (original) ids. */
int hytgen_weights(uint64_t V, const uint64_t *off, const uint32_t *nbr, uint64_t seed, uint32_t *w) {
    int nt = hytgen_num_threads();
    pthread_t th[256]; w_job jobs[256];
    for (int t = 0; t < nt; ++t) {
        jobs[t].off = off; jobs[t].nbr = nbr; jobs[t].w = w; jobs[t].seed = seed;
        jobs[t].v0 = V * t / nt; jobs[t].v1 = V * (t + 1) / nt;
        pthread_create(&th[t], NULL, w_worker, &jobs[t]);
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    return 0;
}

/* Degree histogram (input characterisation): counts of out-degree < 8 and < 32. */
void hytgen_degree_stats(uint64_t V, const uint64_t *off, uint64_t *lt8, uint64_t *lt32,
                         uint64_t *zero, uint64_t *maxdeg) {
    uint64_t a = 0, b = 0, z = 0, m = 0;
    for (uint64_t v = 0; v < V; ++v) {
        uint64_t d = off[v + 1] - off[v];
        a += d < 8; b += d < 32; z += d == 0; if (d > m) m = d;
    }
    *lt8 = a; *lt32 = b; *zero = z; *maxdeg = m;
}
