/*
 * oracle.c -- the CPU ORACLE for the HyTGraph hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The
 * product (paper_2208_14935_b200/) never links, imports or calls it, and it
 * shares no code, header, table or helper with the product: it includes only
 * the C standard library (and POSIX threads for the pull-form Jacobi O4a').
 *
 * Plain, slow, obviously correct, single-threaded; fp64 for floating point.
 * Citations: P:n = /root/reference/PAPER.md line n (the paper), S:n = SPEC.md
 * line n, SURVEY C<n> = the reading listed in DESIGN.md "Readings".
 *
 * Parity status of every function is pinned in tests/test_oracle_*.py:
 *   oracle_bfs / oracle_sssp / oracle_cc / oracle_pr_*   -> brute force, scipy,
 *       closed forms, invariants (see DESIGN.md §Oracle pins)
 *   oracle_hub_sort / oracle_partition / oracle_cost / oracle_plan -> SPEC worked
 *       examples, Fig. 5 counts, an independent Fraction restatement of §5.1.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define INF32 0xFFFFFFFFu

/* ===================================================================== */
/* O1 BFS -- queue BFS over out-edges ("level" = hop count from the  */
/* source, push lvl+1 merged by min).                                 */
/* ===================================================================== */
int oracle_bfs(uint64_t V, const uint64_t *off, const uint32_t *nbr, uint64_t src, uint32_t *level) {
    if (src >= V) return -1;
    for (uint64_t v = 0; v < V; ++v) level[v] = INF32;
    uint32_t *queue = (uint32_t *)malloc(V * sizeof(uint32_t));
    if (!queue) return -2;
    uint64_t head = 0, tail = 0;
    level[src] = 0;
    queue[tail++] = (uint32_t)src;
    while (head < tail) {
        uint32_t u = queue[head++];
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
            uint32_t v = nbr[k];
            if (level[v] == INF32) {
                level[v] = level[u] + 1;
                queue[tail++] = v;
            }
        }
    }
    free(queue);
    return 0;
}

/* ===================================================================== */
/* O2 SSSP -- Dijkstra with a binary heap and lazy deletion, u64 sums     */
/* (Fig. 1 narrative P:153: dist(src)=0, push dist+w, merge = min).        */
/* Returns -3 if a finite distance does not fit u32 (< 0xFFFFFFFF).        */
/* ===================================================================== */
typedef struct { uint64_t d; uint32_t v; } heap_item;

static void heap_push(heap_item *h, uint64_t *n, heap_item x) {
    uint64_t i = (*n)++;
    h[i] = x;
    while (i > 0) {
        uint64_t p = (i - 1) / 2;
        if (h[p].d <= h[i].d) break;
        heap_item t = h[p]; h[p] = h[i]; h[i] = t;
        i = p;
    }
}

static heap_item heap_pop(heap_item *h, uint64_t *n) {
    heap_item top = h[0];
    h[0] = h[--(*n)];
    uint64_t i = 0;
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && h[l].d < h[m].d) m = l;
        if (r < *n && h[r].d < h[m].d) m = r;
        if (m == i) break;
        heap_item t = h[m]; h[m] = h[i]; h[i] = t;
        i = m;
    }
    return top;
}

int oracle_sssp(uint64_t V, const uint64_t *off, const uint32_t *nbr, const uint32_t *w,
                uint64_t src, uint32_t *dist) {
    if (src >= V) return -1;
    uint64_t E = off[V];
    uint64_t *d = (uint64_t *)malloc(V * sizeof(uint64_t));
    heap_item *h = (heap_item *)malloc((E + 1) * sizeof(heap_item));
    if (!d || !h) { free(d); free(h); return -2; }
    for (uint64_t v = 0; v < V; ++v) d[v] = UINT64_MAX;
    uint64_t n = 0;
    d[src] = 0;
    heap_push(h, &n, (heap_item){0, (uint32_t)src});
    while (n > 0) {
        heap_item it = heap_pop(h, &n);
        if (it.d != d[it.v]) continue; /* stale entry */
        uint32_t u = it.v;
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
            uint64_t cand = d[u] + (uint64_t)w[k];
            uint32_t v = nbr[k];
            if (cand < d[v]) {
                d[v] = cand;
                heap_push(h, &n, (heap_item){cand, v});
            }
        }
    }
    int rc = 0;
    for (uint64_t v = 0; v < V; ++v) {
        if (d[v] == UINT64_MAX) dist[v] = INF32;
        else if (d[v] >= INF32) { rc = -3; dist[v] = INF32; }
        else dist[v] = (uint32_t)d[v];
    }
    free(d); free(h);
    return rc;
}

/* ===================================================================== */
/* O3 CC -- union-find (union by min root, path halving).  label(v) = the */
/* minimum vertex id in v's component.  Run on        */
/* symmetrised graphs.                                                     */
/* ===================================================================== */
static uint32_t uf_find(uint32_t *parent, uint32_t x) {
    while (parent[x] != x) {
        parent[x] = parent[parent[x]];
        x = parent[x];
    }
    return x;
}

int oracle_cc(uint64_t V, const uint64_t *off, const uint32_t *nbr, uint32_t *label) {
    uint32_t *parent = (uint32_t *)malloc(V * sizeof(uint32_t));
    if (!parent) return -2;
    for (uint64_t v = 0; v < V; ++v) parent[v] = (uint32_t)v;
    for (uint64_t u = 0; u < V; ++u) {
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
            uint32_t ru = uf_find(parent, (uint32_t)u), rv = uf_find(parent, nbr[k]);
            if (ru == rv) continue;
            if (ru < rv) parent[rv] = ru; else parent[ru] = rv;   /* min id stays root */
        }
    }
    for (uint64_t v = 0; v < V; ++v) label[v] = uf_find(parent, (uint32_t)v);
    free(parent);
    return 0;
}

/* ===================================================================== */
/* O4 PageRank.  Plain definition: r solves            */
/*   r = (1-d)*1 + d * P^T r,  P = D_o^{-1} A, dangling rows zero.         */
/* O4a: Jacobi iteration of that map until max|r_new - r| < tol.           */
/* ===================================================================== */
int oracle_pr_jacobi(uint64_t V, const uint64_t *off, const uint32_t *nbr, double d,
                     double tol, int max_iter, double *rank, int *iters_out) {
    double *acc = (double *)malloc(V * sizeof(double));
    if (!acc) return -2;
    for (uint64_t v = 0; v < V; ++v) rank[v] = 1.0 - d;
    int it = 0;
    for (; it < max_iter; ++it) {
        for (uint64_t v = 0; v < V; ++v) acc[v] = 0.0;
        for (uint64_t u = 0; u < V; ++u) {
            uint64_t deg = off[u + 1] - off[u];
            if (deg == 0) continue;
            double share = rank[u] / (double)deg;
            for (uint64_t k = off[u]; k < off[u + 1]; ++k) acc[nbr[k]] += share;
        }
        double diff = 0.0;
        for (uint64_t v = 0; v < V; ++v) {
            double nv = (1.0 - d) + d * acc[v];
            double dv = fabs(nv - rank[v]);
            if (dv > diff) diff = dv;
            rank[v] = nv;
        }
        if (diff < tol) { ++it; break; }
    }
    if (iters_out) *iters_out = it;
    free(acc);
    return 0;
}

/* O4a': the same Jacobi map in PULL form, for the large parity sizes:      */
/*   r_new[v] = (1-d) + d * sum_{u -> v} r[u] / D_o(u)                      */
/* over a transposed CSR (in-lists, built by a counting sort), with the     */
/* vertex range split across `threads` POSIX threads.  Every r_new[v] is    */
/* written by one thread and summed in in-list order, so the result does    */
/* not depend on the thread count.  Same stopping rule as O4a.              */
#include <pthread.h>
typedef struct {
    uint64_t v0, v1;
    const uint64_t *ioff; const uint32_t *isrc;
    const double *share; double *next; double d;
} pull_job;

static void *pull_range(void *arg) {
    pull_job *j = (pull_job *)arg;
    for (uint64_t v = j->v0; v < j->v1; ++v) {
        double acc = 0.0;
        for (uint64_t k = j->ioff[v]; k < j->ioff[v + 1]; ++k) acc += j->share[j->isrc[k]];
        double nv = (1.0 - j->d) + j->d * acc;
        j->next[v] = nv;
    }
    return NULL;
}

int oracle_pr_jacobi_pull(uint64_t V, const uint64_t *off, const uint32_t *nbr, double d,
                          double tol, int max_iter, int threads, double *rank, int *iters_out) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    const uint64_t E = off[V];
    uint64_t *ioff = (uint64_t *)calloc(V + 1, sizeof(uint64_t));
    uint32_t *isrc = (uint32_t *)malloc((E ? E : 1) * sizeof(uint32_t));
    uint64_t *fill = (uint64_t *)malloc((V ? V : 1) * sizeof(uint64_t));
    double *share = (double *)malloc((V ? V : 1) * sizeof(double));
    double *next = (double *)malloc((V ? V : 1) * sizeof(double));
    pthread_t *th = (pthread_t *)malloc(threads * sizeof(pthread_t));
    pull_job *jobs = (pull_job *)malloc(threads * sizeof(pull_job));
    if (!ioff || !isrc || !fill || !share || !next || !th || !jobs) {
        free(ioff); free(isrc); free(fill); free(share); free(next); free(th); free(jobs);
        return -2;
    }
    /* transpose: in-degree count, exclusive scan, scatter (sources in increasing u) */
    for (uint64_t k = 0; k < E; ++k) ioff[nbr[k] + 1] += 1;
    for (uint64_t v = 0; v < V; ++v) ioff[v + 1] += ioff[v];
    for (uint64_t v = 0; v < V; ++v) fill[v] = ioff[v];
    for (uint64_t u = 0; u < V; ++u)
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) isrc[fill[nbr[k]]++] = (uint32_t)u;
    for (uint64_t v = 0; v < V; ++v) rank[v] = 1.0 - d;
    int it = 0;
    for (; it < max_iter; ++it) {
        for (uint64_t u = 0; u < V; ++u) {
            uint64_t deg = off[u + 1] - off[u];
            share[u] = deg ? rank[u] / (double)deg : 0.0;
        }
        for (int t = 0; t < threads; ++t) {
            jobs[t].v0 = V * (uint64_t)t / (uint64_t)threads;
            jobs[t].v1 = V * (uint64_t)(t + 1) / (uint64_t)threads;
            jobs[t].ioff = ioff; jobs[t].isrc = isrc; jobs[t].share = share;
            jobs[t].next = next; jobs[t].d = d;
            pthread_create(&th[t], NULL, pull_range, &jobs[t]);
        }
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
        double diff = 0.0;
        for (uint64_t v = 0; v < V; ++v) {
            double dv = fabs(next[v] - rank[v]);
            if (dv > diff) diff = dv;
            rank[v] = next[v];
        }
        if (diff < tol) { ++it; break; }
    }
    if (iters_out) *iters_out = it;
    free(ioff); free(isrc); free(fill); free(share); free(next); free(th); free(jobs);
    return 0;
}

/* O4b: sequential delta-PageRank (Maiter-style accumulation,  */
/* S:451-457): rank = 0, delta = 1-d; FIFO worklist of {delta > eps};      */
/* pop u: take delta, rank += delta, push d*delta/D_o(u) to out-neighbours. */
int oracle_pr_delta(uint64_t V, const uint64_t *off, const uint32_t *nbr, double d,
                    double eps, double *rank, uint64_t *pops_out) {
    double *delta = (double *)malloc(V * sizeof(double));
    uint32_t *ring = (uint32_t *)malloc(V * sizeof(uint32_t));
    uint8_t *inq = (uint8_t *)calloc(V, 1);
    if (!delta || !ring || !inq) { free(delta); free(ring); free(inq); return -2; }
    uint64_t head = 0, count = 0, pops = 0;
    for (uint64_t v = 0; v < V; ++v) {
        rank[v] = 0.0;
        delta[v] = 1.0 - d;
        if (delta[v] > eps) { ring[(head + count) % V] = (uint32_t)v; ++count; inq[v] = 1; }
    }
    while (count > 0) {
        uint32_t u = ring[head];
        head = (head + 1) % V; --count; inq[u] = 0; ++pops;
        double du = delta[u];
        delta[u] = 0.0;
        rank[u] += du;
        uint64_t deg = off[u + 1] - off[u];
        if (deg == 0) continue;               /* dangling: absorbs, pushes nothing */
        double share = d * du / (double)deg;
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
            uint32_t v = nbr[k];
            delta[v] += share;
            if (!inq[v] && delta[v] > eps) { ring[(head + count) % V] = v; ++count; inq[v] = 1; }
        }
    }
    if (pops_out) *pops_out = pops;
    free(delta); free(ring); free(inq);
    return 0;
}

/* ===================================================================== */
/* O(E) certificates, usable at any size (SURVEY §8c pins).                */
/* ===================================================================== */

/* BFS level witness: level[src]=0; level[v] <= level[u]+1 on every edge   */
/* from a reached u; every reached v != src has an in-edge from level-1;   */
/* unreached vertices have no in-edge from a reached vertex.               */
int oracle_check_bfs(uint64_t V, const uint64_t *off, const uint32_t *nbr, uint64_t src,
                     const uint32_t *level) {
    if (level[src] != 0) return 1;
    uint8_t *has_parent = (uint8_t *)calloc(V, 1);
    if (!has_parent) return -2;
    int rc = 0;
    for (uint64_t u = 0; u < V && !rc; ++u) {
        if (level[u] == INF32) continue;
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
            uint32_t v = nbr[k];
            if (level[v] == INF32 || level[v] > level[u] + 1) { rc = 2; break; }
            if (level[v] == level[u] + 1) has_parent[v] = 1;
        }
    }
    for (uint64_t v = 0; v < V && !rc; ++v)
        if (v != src && level[v] != INF32 && !has_parent[v]) rc = 3;
    free(has_parent);
    return rc;
}

/* SSSP certificate: dist[src]=0; dist[v] <= dist[u]+w on every edge from a */
/* reached u; every reached v != src has a tight in-edge (parent witness).  */
int oracle_check_sssp(uint64_t V, const uint64_t *off, const uint32_t *nbr, const uint32_t *w,
                      uint64_t src, const uint32_t *dist) {
    if (dist[src] != 0) return 1;
    uint8_t *tight = (uint8_t *)calloc(V, 1);
    if (!tight) return -2;
    int rc = 0;
    for (uint64_t u = 0; u < V && !rc; ++u) {
        if (dist[u] == INF32) continue;
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
            uint32_t v = nbr[k];
            uint64_t cand = (uint64_t)dist[u] + w[k];
            if (dist[v] == INF32 || (uint64_t)dist[v] > cand) { rc = 2; break; }
            if ((uint64_t)dist[v] == cand) tight[v] = 1;
        }
    }
    for (uint64_t v = 0; v < V && !rc; ++v)
        if (v != src && dist[v] != INF32 && !tight[v]) rc = 3;
    free(tight);
    return rc;
}

/* CC certificate on a symmetric graph (label = minimum  */
/* caller id of the component).  Complete, O(V + E):                        */
/*   1. label(u) <= u for every u, and label equal across every edge;       */
/*   2. from every root r (label(r) == r) a BFS over the edges reaches only */
/*      vertices labelled r, and marks them;                                */
/*   3. every vertex is marked.                                             */
/* (2)+(3) make each label class exactly one component (a class split into  */
/* two components leaves the part without its root unmarked -- e.g. the     */
/* merged labelling {0-1},{2-3} -> [0,0,0,0] fails at 3); with (1) the root */
/* is below every member, so it is the component's minimum id.              */
int oracle_check_cc(uint64_t V, const uint64_t *off, const uint32_t *nbr, const uint32_t *label) {
    for (uint64_t u = 0; u < V; ++u) {
        if (label[u] > u) return 1;
        if (label[label[u]] != label[u]) return 2;
        for (uint64_t k = off[u]; k < off[u + 1]; ++k)
            if (label[nbr[k]] != label[u]) return 3;
    }
    uint8_t *seen = (uint8_t *)calloc(V ? V : 1, 1);
    uint32_t *queue = (uint32_t *)malloc((V ? V : 1) * sizeof(uint32_t));
    if (!seen || !queue) { free(seen); free(queue); return -2; }
    int rc = 0;
    for (uint64_t r = 0; r < V && !rc; ++r) {
        if (label[r] != r || seen[r]) continue;
        uint64_t head = 0, tail = 0;
        seen[r] = 1;
        queue[tail++] = (uint32_t)r;
        while (head < tail && !rc) {
            uint32_t u = queue[head++];
            for (uint64_t k = off[u]; k < off[u + 1]; ++k) {
                uint32_t v = nbr[k];
                if (label[v] != r) { rc = 3; break; }
                if (!seen[v]) { seen[v] = 1; queue[tail++] = v; }
            }
        }
    }
    for (uint64_t v = 0; v < V && !rc; ++v)
        if (!seen[v]) rc = 4;
    free(seen);
    free(queue);
    return rc;
}

/* PR: L1 norm of T(r) - r with T(r) = (1-d) + d P^T r, and sum of r.       */
/* ||r* - r||_1 <= ||T(r) - r||_1 / (1-d)  (||P^T||_1 <= 1).                 */
int oracle_pr_residual(uint64_t V, const uint64_t *off, const uint32_t *nbr, double d,
                       const float *r, double *res_l1, double *sum_r, double *max_rel_res) {
    double *acc = (double *)calloc(V, sizeof(double));
    if (!acc) return -2;
    for (uint64_t u = 0; u < V; ++u) {
        uint64_t deg = off[u + 1] - off[u];
        if (!deg) continue;
        double share = (double)r[u] / (double)deg;
        for (uint64_t k = off[u]; k < off[u + 1]; ++k) acc[nbr[k]] += share;
    }
    double l1 = 0, s = 0, mr = 0;
    for (uint64_t v = 0; v < V; ++v) {
        double t = (1.0 - d) + d * acc[v];
        double dv = fabs(t - (double)r[v]);
        l1 += dv; s += r[v];
        double rel = dv / t;
        if (rel > mr) mr = rel;
    }
    *res_l1 = l1; *sum_r = s; *max_rel_res = mr;
    free(acc);
    return 0;
}

/* ===================================================================== */
/* A0 hub sorting.  H(v) = D_o(v)*D_i(v) /        */
/* (D_omax*D_imax); the denominator is common to all v so the order of H  */
/* is the order of the exact integer product D_o*D_i.  The top            */
/* h = ceil(frac_num*V/frac_den) vertices by H (descending, ties by id    */
/* ascending) get new ids 0..h-1 in that order; every other vertex keeps  */
/* its natural order after them.  Output: new_id[old] (old -> new).       */
/* ===================================================================== */
static const uint64_t *g_key;
static int cmp_hub(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    if (g_key[x] != g_key[y]) return g_key[x] > g_key[y] ? -1 : 1;   /* descending H */
    return (x > y) - (x < y);                                           /* ties: id asc */
}

int oracle_hub_sort(uint64_t V, const uint64_t *off, const uint32_t *nbr,
                    uint64_t frac_num, uint64_t frac_den, uint32_t *new_id) {
    uint64_t *din = (uint64_t *)calloc(V, sizeof(uint64_t));
    uint64_t *key = (uint64_t *)malloc(V * sizeof(uint64_t));
    uint32_t *order = (uint32_t *)malloc(V * sizeof(uint32_t));
    uint8_t *is_hub = (uint8_t *)calloc(V, 1);
    if (!din || !key || !order || !is_hub) { free(din); free(key); free(order); free(is_hub); return -2; }
    for (uint64_t k = 0; k < off[V]; ++k) din[nbr[k]]++;
    for (uint64_t v = 0; v < V; ++v) { key[v] = (off[v + 1] - off[v]) * din[v]; order[v] = (uint32_t)v; }
    uint64_t h = (frac_num * V + frac_den - 1) / frac_den;
    if (h > V) h = V;
    g_key = key;
    qsort(order, V, sizeof(uint32_t), cmp_hub);
    for (uint64_t i = 0; i < h; ++i) { new_id[order[i]] = (uint32_t)i; is_hub[order[i]] = 1; }
    uint64_t next = h;
    for (uint64_t v = 0; v < V; ++v) if (!is_hub[v]) new_id[v] = (uint32_t)next++;
    free(din); free(key); free(order); free(is_hub);
    return 0;
}

/* Apply a permutation to a CSR (rows moved, ids remapped, weights travel */
/* with their edge; each new row keeps the old row's edge order).         */
int oracle_relabel(uint64_t V, const uint64_t *off, const uint32_t *nbr, const uint32_t *w,
                   const uint32_t *new_id, uint64_t *off2, uint32_t *nbr2, uint32_t *w2) {
    uint32_t *old_of = (uint32_t *)malloc(V * sizeof(uint32_t));
    if (!old_of) return -2;
    for (uint64_t v = 0; v < V; ++v) old_of[new_id[v]] = (uint32_t)v;
    off2[0] = 0;
    for (uint64_t r = 0; r < V; ++r) {
        uint32_t v = old_of[r];
        uint64_t deg = off[v + 1] - off[v];
        for (uint64_t j = 0; j < deg; ++j) {
            nbr2[off2[r] + j] = new_id[nbr[off[v] + j]];
            if (w && w2) w2[off2[r] + j] = w[off[v] + j];
        }
        off2[r + 1] = off2[r] + deg;
    }
    free(old_of);
    return 0;
}

/* ===================================================================== */
/* A0 chunk-based edge-balanced partitioning:   */
/* greedy sweep in id order; close the partition when adding the next     */
/* vertex would exceed target_bytes (unless the partition is empty).      */
/* bounds[0..N] vertex boundaries.  Returns N.                            */
/* ===================================================================== */
uint64_t oracle_partition(uint64_t V, const uint64_t *off, uint64_t d1, uint64_t target_bytes,
                          uint64_t *bounds) {
    uint64_t N = 0;
    bounds[0] = 0;
    uint64_t cur_bytes = 0, cur_count = 0;
    for (uint64_t v = 0; v < V; ++v) {
        uint64_t b = (off[v + 1] - off[v]) * d1;
        if (cur_count > 0 && cur_bytes + b > target_bytes) {
            bounds[++N] = v;
            cur_bytes = 0; cur_count = 0;
        }
        cur_bytes += b; cur_count++;
    }
    if (V > 0) bounds[++N] = V;
    return N;
}

/* ===================================================================== */
/* §5.1 cost model.  Plain restatement of Eq. 1-3 with RTT = 1, the      */
/* thresholds as exact rationals and every comparison cross-multiplied.  */
/* ===================================================================== */
typedef struct {
    uint64_t d1, d2, m, mr;              /* bytes/edge, bytes/index, request bytes, requests per TLP */
    uint64_t alpha_num, alpha_den;       /* alpha = 0.8 */
    uint64_t beta_num, beta_den;         /* beta  = 0.4 */
    uint64_t gamma_num, gamma_den;       /* gamma = 0.625 */
    uint64_t k;                          /* filter merge width, 4 */
} oracle_cost_cfg;

static uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

/* am(v) (P:368 footnote): 1 if the neighbour span [start, start+len) touches  */
/* one more m-byte line than ceil(len/m).                                       */
uint64_t oracle_am(uint64_t start_byte, uint64_t len_bytes, uint64_t m) {
    if (len_bytes == 0) return 0;
    uint64_t first = start_byte / m, last = (start_byte + len_bytes - 1) / m;
    uint64_t lines = last - first + 1;
    return lines - ceil_div(len_bytes, m);
}

/* Requests of one active vertex for zero-copy: ceil(D_o*d1/m) + am(v) (Eq. 3). */
uint64_t oracle_zc_requests(uint64_t off_v, uint64_t deg, const oracle_cost_cfg *c) {
    if (deg == 0) return 0;
    return ceil_div(deg * c->d1, c->m) + oracle_am(off_v * c->d1, deg * c->d1, c->m);
}

/* Tef = ceil(t*d1/m/MR) (Eq. 1). */
uint64_t oracle_tef(uint64_t t, const oracle_cost_cfg *c) { return ceil_div(t * c->d1, c->m * c->mr); }
/* Tec transfer term = ceil((e*d1 + a*d2)/m/MR) (Eq. 2; selection omits the CPU term). */
uint64_t oracle_tec(uint64_t e, uint64_t a, const oracle_cost_cfg *c) {
    return ceil_div(e * c->d1 + a * c->d2, c->m * c->mr);
}
/* number of zero-copy TLPs ceil(z/MR) (Eq. 3 without the RTT_zc factor). */
uint64_t oracle_nz(uint64_t z, const oracle_cost_cfg *c) { return ceil_div(z, c->mr); }

/* Engine selection, §5.1 prose: C if Tec < alpha*Tef and Tec <    */
/* beta*Tiz; else Z if Tiz < Tef; else F.  Tiz = n_z * RTT_zc, RTT_zc =        */
/* gamma + (1-gamma)*e/t.  Inactive (e == 0) -> 0 (no task).                  */
/* Returns 0 none, 1 F, 2 C, 3 Z.                                              */
int oracle_select(uint64_t t, uint64_t e, uint64_t a, uint64_t z, const oracle_cost_cfg *c) {
    if (e == 0) return 0;
    typedef unsigned __int128 u128;
    uint64_t Tef = oracle_tef(t, c), Tec = oracle_tec(e, a, c), nz = oracle_nz(z, c);
    /* Tiz = nz * (gn*t + (gd-gn)*e) / (gd*t) */
    u128 Q = (u128)c->gamma_num * t + (u128)(c->gamma_den - c->gamma_num) * e;
    u128 tiz_num = (u128)nz * Q, tiz_den = (u128)c->gamma_den * t;
    /* Tec < alpha*Tef  <=>  Tec*an_den < an_num*Tef */
    int c1 = (u128)Tec * c->alpha_den < (u128)c->alpha_num * Tef;
    /* Tec < beta*Tiz   <=>  Tec*bd*tiz_den < bn*tiz_num */
    int c2 = (u128)Tec * c->beta_den * tiz_den < (u128)c->beta_num * tiz_num;
    if (c1 && c2) return 2;
    /* Tiz < Tef <=> tiz_num < Tef*tiz_den */
    if (tiz_num < (u128)Tef * tiz_den) return 3;
    return 1;
}

/* Task combination (Alg. 1 L14-24, with the SURVEY C9 reading: */
/* the printed loop drops the partition that hits length k and creates     */
/* empty units; the intent is to split every maximal run */
/* of consecutive F partitions into units of <= k).  Non-F partitions      */
/* (including inactive ones) break runs.  Returns the number of units.     */
int64_t oracle_combine(uint64_t N, const uint8_t *p, uint64_t k, uint64_t *units) {
    int64_t nu = 0;
    uint64_t i = 0;
    while (i < N) {
        if (p[i] != 1) { ++i; continue; }
        uint64_t start = i, len = 0;
        while (i < N && p[i] == 1 && len < k) { ++i; ++len; }
        units[2 * nu] = start; units[2 * nu + 1] = i; ++nu;
    }
    return nu;
}

/* ===================================================================== */
/* The B200-calibrated variant of the section 5.1 rule (DESIGN.md          */
/* "Calibrated cost model").  All costs are in RTT units,    */
/* RTT = the time of one saturated TLP (m*MR bytes) at the DMA link rate:  */
/*   Tef = ceil(t*d1/(m*MR))                              (Eq. 1)          */
/*   Tec = ceil(B/(m*MR)) + ceil(B * link/Thpt_cpt / (m*MR)),              */
/*         B = e*d1 + a*d2        (Eq. 2 with its CPU term)      */
/*   Tiz = r*zr + (z - r)*zs      (Eq. 3 re-fit: each of the r active lists */
/*         costs one random request zr, each further line a streamed zs)   */
/* with link/Thpt_cpt = cpu_num/cpu_den, zr = zr_num/z_den, zs = zs_num/z_den. */
/* The decision rule itself is unchanged (ties -> F).           */
/* ===================================================================== */
typedef struct { uint64_t cpu_num, cpu_den, zr_num, zs_num, z_den; } oracle_cal;

int oracle_select_cal(uint64_t t, uint64_t e, uint64_t a, uint64_t z, uint64_t r, const oracle_cost_cfg *c,
                      const oracle_cal *k) {
    if (e == 0) return 0;
    typedef unsigned __int128 u128;
    const uint64_t tlp = c->m * c->mr;
    const uint64_t B = e * c->d1 + a * c->d2;
    const uint64_t Tef = ceil_div(t * c->d1, tlp);
    const u128 cpu_n = (u128)B * k->cpu_num, cpu_d = (u128)k->cpu_den * tlp;
    const uint64_t Tec = ceil_div(B, tlp) + (uint64_t)((cpu_n + cpu_d - 1) / cpu_d);
    const u128 tiz_num = (u128)r * k->zr_num + (u128)(z - r) * k->zs_num;   /* / z_den */
    const int c1 = (u128)Tec * c->alpha_den < (u128)c->alpha_num * Tef;
    const int c2 = (u128)Tec * c->beta_den * k->z_den < (u128)c->beta_num * tiz_num;
    if (c1 && c2) return 2;
    if (tiz_num < (u128)Tef * k->z_den) return 3;
    return 1;
}

/* ===================================================================== */
/* Algorithm 1 on a frontier snapshot, step by step.           */
/* Inputs: V, off (the graph the engines see), active[V] (0/1), bounds.    */
/* Per partition i: t_i, e_i, a_i, z_i, hub score (sum D_o*D_i over        */
/* active), p_i.  Task combination (P:416-426 with SURVEY C9): split each  */
/* maximal run of consecutive F partitions into units of <= k partitions.  */
/* units[2*j], units[2*j+1] = first partition, one-past-last partition.    */
/* Returns the number of F units.                                          */
/* ===================================================================== */
int64_t oracle_plan(uint64_t V, const uint64_t *off, const uint64_t *din, const uint8_t *active,
                    uint64_t N, const uint64_t *bounds, const oracle_cost_cfg *c, const oracle_cal *cal,
                    uint64_t *t_out, uint64_t *e_out, uint64_t *a_out, uint64_t *z_out,
                    uint64_t *hub_out, uint8_t *p_out, uint64_t *units) {
    (void)V;
    for (uint64_t i = 0; i < N; ++i) {
        uint64_t t = 0, e = 0, a = 0, z = 0, hub = 0, r = 0;
        for (uint64_t v = bounds[i]; v < bounds[i + 1]; ++v) {
            uint64_t deg = off[v + 1] - off[v];
            t += deg;
            if (!active[v]) continue;
            a += 1;
            e += deg;
            r += deg > 0;
            z += oracle_zc_requests(off[v], deg, c);
            if (din) hub += deg * din[v];
        }
        t_out[i] = t; e_out[i] = e; a_out[i] = a; z_out[i] = z; hub_out[i] = hub;
        p_out[i] = (uint8_t)(cal ? oracle_select_cal(t, e, a, z, r, c, cal) : oracle_select(t, e, a, z, c));
    }
    return oracle_combine(N, p_out, c->k, units);
}
/* ===================================================================== */
/* Contribution-driven ordering of F units (SURVEY      */
/* C12/C13): unit score = sum of its partitions' scores (hub: sum of      */
/* D_o*D_i over active vertices; delta: sum of delta over active          */
/* vertices); order descending, ties by unit index ascending.             */
/* ===================================================================== */
static const double *g_uscore;
static int cmp_unit(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    if (g_uscore[x] != g_uscore[y]) return g_uscore[x] > g_uscore[y] ? -1 : 1;
    return (x > y) - (x < y);
}

void oracle_order_units(int64_t nu, const uint64_t *units, const double *part_score, uint32_t *order) {
    double *us = (double *)malloc((nu > 0 ? nu : 1) * sizeof(double));
    for (int64_t j = 0; j < nu; ++j) {
        double s = 0;
        for (uint64_t i = units[2 * j]; i < units[2 * j + 1]; ++i) s += part_score[i];
        us[j] = s;
        order[j] = (uint32_t)j;
    }
    g_uscore = us;
    qsort(order, nu, sizeof(uint32_t), cmp_unit);
    free(us);
}
