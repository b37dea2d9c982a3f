/*
 * ps_oracle.c -- CPU restatement of the FastPoint sampling kernels.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the CUDA
 * path and the "port" CPU baseline timed by bench.py.  Nothing in the
 * product package (paper_2507_23480_b200/) may link or call it.
 *
 * Each function restates one numba kernel of the reference package
 * (/root/reference/pkg/src/pointsample/_kernels.py, cited as _kernels.py:L)
 * with the same arithmetic: float64 distances accumulated as
 * ((dx*dx + dy*dy) + dz*dz) with no contraction (built with
 * -ffp-contract=off), the same strict comparisons and the same
 * lowest-index tie rules.  Parity with the reference itself is pinned by
 * tests/golden/ (fixtures produced by importing the real reference kernels;
 * see tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define ORA_API __attribute__((visibility("default")))

ORA_API int64_t ora_first_untaken(const uint8_t* taken, int64_t N);
ORA_API int64_t ora_fps_loop(const double* x, const double* y, const double* z,
                             int64_t N, double* md, uint8_t* taken,
                             int64_t* out_idx, double* curve,
                             int64_t k_start, int64_t n_total);

static inline double sqdist(double ax, double ay, double az,
                            double bx, double by, double bz) {
    /* operand order of _kernels.py:55-58 (x[j] - px, ...) */
    double dx = bx - ax;
    double dy = by - ay;
    double dz = bz - az;
    double s = dx * dx;
    s = s + dy * dy;
    s = s + dz * dz;
    return s;
}

/* ------------------------------------------------------------------ */
/* splitmix64, _kernels.py:20-28 / core.py:115-133                      */

#define SM64_GOLDEN 0x9E3779B97F4A7C15ULL
static inline uint64_t sm64_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

ORA_API uint64_t ora_sm64_next(uint64_t* state) {
    *state += SM64_GOLDEN;
    return sm64_mix(*state);
}

/* ------------------------------------------------------------------ */
/* Exact FPS, _kernels.py:35-74.  Iterations k_start..n_total-1 in place. */

ORA_API int64_t ora_fps_loop(const double* x, const double* y, const double* z,
                             int64_t N, double* md, uint8_t* taken,
                             int64_t* out_idx, double* curve,
                             int64_t k_start, int64_t n_total) {
    int64_t evals = 0;
    for (int64_t it = k_start; it < n_total; ++it) {
        const int64_t s = out_idx[it - 1];
        const double px = x[s], py = y[s], pz = z[s];
        double best = -1.0;
        int64_t arg = -1;
        for (int64_t j = 0; j < N; ++j) {
            const double d = sqdist(px, py, pz, x[j], y[j], z[j]);
            if (d < md[j]) md[j] = d;
            if (md[j] > best) { best = md[j]; arg = j; }
        }
        evals += N;
        /* duplicate fallback, _kernels.py:65-70 */
        if (best <= 0.0 || taken[arg]) {
            for (int64_t j = 0; j < N; ++j) {
                if (!taken[j]) { arg = j; best = md[j]; break; }
            }
        }
        out_idx[it] = arg;
        curve[it] = sqrt(best);
        taken[arg] = 1;
    }
    return evals;
}

/* Threaded exact FPS: the reference's multi-worker form (
 * core.workers, core.py:71-101) -- every iteration runs fps_update_chunk
 * (_kernels.py:77-92) on nthreads contiguous slices and merges the slice
 * results by (max md, lowest index: strict > in slice order), then the
 * duplicate fallback through first_untaken (_kernels.py:95-100).  Identical
 * output to ora_fps_loop for any slice count. */
typedef struct {
    const double *x, *y, *z;
    double* md;
    const int64_t* out_idx;
    int64_t N, chunk, k_start, n_total;
    int T;
    double* bests;
    int64_t* args;
    pthread_barrier_t* bar;  /* two waits per iteration: slices done / merge done */
} fps_mt_ctx;

typedef struct { fps_mt_ctx* c; int t; } fps_mt_arg;

static void fps_slice(fps_mt_ctx* c, int t, int64_t it) {
    const int64_t s = c->out_idx[it - 1];
    const double px = c->x[s], py = c->y[s], pz = c->z[s];
    const int64_t lo = t * c->chunk < c->N ? t * c->chunk : c->N;
    const int64_t hi = lo + c->chunk < c->N ? lo + c->chunk : c->N;
    double best = -1.0;
    int64_t arg = -1;
    for (int64_t j = lo; j < hi; ++j) {
        const double d = sqdist(px, py, pz, c->x[j], c->y[j], c->z[j]);
        if (d < c->md[j]) c->md[j] = d;
        if (c->md[j] > best) { best = c->md[j]; arg = j; }
    }
    c->bests[t] = best;
    c->args[t] = arg;
}

static void* fps_mt_worker(void* p) {
    fps_mt_arg* a = (fps_mt_arg*)p;
    for (int64_t it = a->c->k_start; it < a->c->n_total; ++it) {
        fps_slice(a->c, a->t, it);
        pthread_barrier_wait(a->c->bar);  /* slices done */
        pthread_barrier_wait(a->c->bar);  /* thread 0 merged and wrote out_idx[it] */
    }
    return NULL;
}

ORA_API int64_t ora_fps_loop_mt(const double* x, const double* y, const double* z,
                                int64_t N, double* md, uint8_t* taken,
                                int64_t* out_idx, double* curve,
                                int64_t k_start, int64_t n_total, int32_t nthreads) {
    const int T = nthreads > 64 ? 64 : nthreads;
    if (T < 2 || N < 4096 || k_start >= n_total)
        return ora_fps_loop(x, y, z, N, md, taken, out_idx, curve, k_start, n_total);
    double bests[64];
    int64_t args[64];
    pthread_barrier_t bar;
    pthread_barrier_init(&bar, NULL, (unsigned)T);
    fps_mt_ctx c = {x, y, z, md, out_idx, N, (N + T - 1) / T, k_start, n_total, T, bests, args, &bar};
    pthread_t th[64];
    fps_mt_arg wa[64];
    for (int t = 1; t < T; ++t) {
        wa[t].c = &c;
        wa[t].t = t;
        pthread_create(&th[t], NULL, fps_mt_worker, &wa[t]);
    }
    int64_t evals = 0;
    for (int64_t it = k_start; it < n_total; ++it) {
        fps_slice(&c, 0, it);
        pthread_barrier_wait(&bar);
        double best = -1.0;
        int64_t arg = -1;
        for (int t = 0; t < T; ++t)  /* strict > in slice order: lowest index on ties */
            if (bests[t] > best) { best = bests[t]; arg = args[t]; }
        evals += N;
        if (best <= 0.0 || taken[arg]) {  /* _kernels.py:65-70 */
            const int64_t f = ora_first_untaken(taken, N);
            if (f >= 0) { arg = f; best = md[f]; }
        }
        out_idx[it] = arg;
        curve[it] = sqrt(best);
        taken[arg] = 1;
        pthread_barrier_wait(&bar);
    }
    for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
    pthread_barrier_destroy(&bar);
    return evals;
}

/* Slice update + argmax, _kernels.py:77-92. best/arg returned via pointers. */
ORA_API void ora_fps_update_chunk(const double* x, const double* y, const double* z,
                                  double px, double py, double pz, double* md,
                                  int64_t lo, int64_t hi, double* best_out,
                                  int64_t* arg_out) {
    double best = -1.0;
    int64_t arg = -1;
    for (int64_t j = lo; j < hi; ++j) {
        const double d = sqdist(px, py, pz, x[j], y[j], z[j]);
        if (d < md[j]) md[j] = d;
        if (md[j] > best) { best = md[j]; arg = j; }
    }
    *best_out = best;
    *arg_out = arg;
}

/* _kernels.py:95-100 */
ORA_API int64_t ora_first_untaken(const uint8_t* taken, int64_t N) {
    for (int64_t j = 0; j < N; ++j)
        if (!taken[j]) return j;
    return -1;
}

/* ------------------------------------------------------------------ */
/* Exclusion lists: excl_collect + csr_fill + csr_sort_rows              */
/* (_kernels.py:111-219).  One pass over the i<j triangle collects the   */
/* edges (each pair evaluated once), the CSR gets self + both directions, */
/* and rows are ordered by (d2, index).                                   */

typedef struct {
    int64_t N;
    int64_t E;        /* CSR entries including self */
    int64_t evals;    /* pair evaluations of the collect pass: N(N-1)/2 */
    int64_t* indptr;  /* N+1 */
    int64_t* nbr;     /* E */
    double* d2;       /* E */
} ora_csr;

typedef struct { double d; int64_t j; } ora_entry;

static int entry_cmp(const void* a, const void* b) {
    const ora_entry* p = (const ora_entry*)a;
    const ora_entry* q = (const ora_entry*)b;
    if (p->d < q->d) return -1;
    if (p->d > q->d) return 1;
    return (p->j > q->j) - (p->j < q->j);
}

typedef struct { int64_t cap, cnt; int32_t* ei; int32_t* ej; double* ed; } edge_buf;

static void collect_rows(const double* x, const double* y, const double* z, int64_t N, double r2max,
                         int64_t i, edge_buf* b) {
    const double xi = x[i], yi = y[i], zi = z[i];
    for (int64_t j = i + 1; j < N; ++j) {
        /* _kernels.py:149-152: dx = x[jj] - xi */
        const double d = sqdist(xi, yi, zi, x[j], y[j], z[j]);
        if (d < r2max) {
            if (b->cnt == b->cap) {
                b->cap = b->cap ? 2 * b->cap : 1024;
                b->ei = (int32_t*)realloc(b->ei, sizeof(int32_t) * b->cap);
                b->ej = (int32_t*)realloc(b->ej, sizeof(int32_t) * b->cap);
                b->ed = (double*)realloc(b->ed, sizeof(double) * b->cap);
            }
            b->ei[b->cnt] = (int32_t)i; b->ej[b->cnt] = (int32_t)j; b->ed[b->cnt] = d; ++b->cnt;
        }
    }
}

typedef struct { ora_csr* c; int64_t maxrow; int T, t; } sort_arg;

static void* sort_worker(void* p) {
    sort_arg* a = (sort_arg*)p;
    ora_entry* tmp = (ora_entry*)malloc(sizeof(ora_entry) * (size_t)(a->maxrow ? a->maxrow : 1));
    for (int64_t i = a->t; i < a->c->N; i += a->T) {
        const int64_t lo = a->c->indptr[i], m = a->c->indptr[i + 1] - lo;
        if (m < 2) continue;
        for (int64_t q = 0; q < m; ++q) { tmp[q].d = a->c->d2[lo + q]; tmp[q].j = a->c->nbr[lo + q]; }
        qsort(tmp, (size_t)m, sizeof(ora_entry), entry_cmp);
        for (int64_t q = 0; q < m; ++q) { a->c->d2[lo + q] = tmp[q].d; a->c->nbr[lo + q] = tmp[q].j; }
    }
    free(tmp);
    return NULL;
}

static void sort_rows_mt(ora_csr* c, int64_t maxrow, int T) {
    sort_arg sa[64];
    pthread_t th[64];
    for (int t = 0; t < T; ++t) {
        sort_arg v = {c, maxrow, T, t};
        sa[t] = v;
        if (t > 0) pthread_create(&th[t], NULL, sort_worker, &sa[t]);
    }
    sort_worker(&sa[0]);
    for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
}

/* nthreads > 1: the reference's worker split of excl_collect (balanced
 * row-pair tasks k, N-1-k, _kernels.py:103-108, over core.workers) with one
 * edge buffer per worker; the CSR is identical because every row is then
 * ordered by (d2, index), which does not depend on the emission order. */
ORA_API ora_csr* ora_excl_build_mt(const double* x, const double* y, const double* z,
                                   int64_t N, double r2max, int32_t nthreads);

ORA_API ora_csr* ora_excl_build(const double* x, const double* y, const double* z,
                                int64_t N, double r2max) {
    return ora_excl_build_mt(x, y, z, N, r2max, 1);
}

typedef struct {
    const double *x, *y, *z;
    int64_t N, ntask;
    double r2max;
    int T, t;
    edge_buf* b;
} collect_arg;

static void* collect_worker(void* p) {
    collect_arg* a = (collect_arg*)p;
    /* tasks t, t + T, ...: interleaved so every worker gets long and short rows */
    for (int64_t k = a->t; k < a->ntask; k += a->T) {
        collect_rows(a->x, a->y, a->z, a->N, a->r2max, k, a->b);
        if (a->N - 1 - k != k) collect_rows(a->x, a->y, a->z, a->N, a->r2max, a->N - 1 - k, a->b);
    }
    return NULL;
}

ORA_API ora_csr* ora_excl_build_mt(const double* x, const double* y, const double* z,
                                   int64_t N, double r2max, int32_t nthreads) {
    const int T = nthreads < 1 ? 1 : (nthreads > 64 ? 64 : nthreads);
    edge_buf* bufs = (edge_buf*)calloc((size_t)T, sizeof(edge_buf));
    const int64_t ntask = (N + 1) / 2;
    collect_arg ca[64];
    pthread_t th[64];
    for (int t = 0; t < T; ++t) {
        collect_arg v = {x, y, z, N, ntask, r2max, T, t, &bufs[t]};
        ca[t] = v;
        if (t > 0) pthread_create(&th[t], NULL, collect_worker, &ca[t]);
    }
    collect_worker(&ca[0]);
    for (int t = 1; t < T; ++t) pthread_join(th[t], NULL);
    int64_t cnt = 0;
    for (int t = 0; t < T; ++t) cnt += bufs[t].cnt;
    int32_t* ei = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cnt ? cnt : 1));
    int32_t* ej = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cnt ? cnt : 1));
    double* ed = (double*)malloc(sizeof(double) * (size_t)(cnt ? cnt : 1));
    int64_t off = 0;
    for (int t = 0; t < T; ++t) {
        if (bufs[t].cnt) {
            memcpy(ei + off, bufs[t].ei, sizeof(int32_t) * (size_t)bufs[t].cnt);
            memcpy(ej + off, bufs[t].ej, sizeof(int32_t) * (size_t)bufs[t].cnt);
            memcpy(ed + off, bufs[t].ed, sizeof(double) * (size_t)bufs[t].cnt);
        }
        off += bufs[t].cnt;
        free(bufs[t].ei); free(bufs[t].ej); free(bufs[t].ed);
    }
    free(bufs);
    const int64_t evals = N * (N - 1) / 2;
    ora_csr* c = (ora_csr*)calloc(1, sizeof(ora_csr));
    c->N = N;
    c->evals = evals;
    c->indptr = (int64_t*)calloc((size_t)N + 1, sizeof(int64_t));
    int64_t* deg = (int64_t*)calloc((size_t)N, sizeof(int64_t));
    for (int64_t i = 0; i < N; ++i) deg[i] = 1; /* self */
    for (int64_t e = 0; e < cnt; ++e) { deg[ei[e]]++; deg[ej[e]]++; }
    for (int64_t i = 0; i < N; ++i) c->indptr[i + 1] = c->indptr[i] + deg[i];
    c->E = c->indptr[N];
    c->nbr = (int64_t*)malloc(sizeof(int64_t) * (size_t)(c->E ? c->E : 1));
    c->d2 = (double*)malloc(sizeof(double) * (size_t)(c->E ? c->E : 1));
    /* csr_fill, _kernels.py:164-185: self first, then edges in order */
    int64_t* cur = deg; /* reuse as cursor */
    for (int64_t i = 0; i < N; ++i) {
        cur[i] = c->indptr[i];
        c->nbr[cur[i]] = i; c->d2[cur[i]] = 0.0; cur[i]++;
    }
    for (int64_t e = 0; e < cnt; ++e) {
        const int64_t a = ei[e], b = ej[e];
        c->nbr[cur[a]] = b; c->d2[cur[a]] = ed[e]; cur[a]++;
        c->nbr[cur[b]] = a; c->d2[cur[b]] = ed[e]; cur[b]++;
    }
    free(ei); free(ej); free(ed); free(deg);
    /* csr_sort_rows, _kernels.py:188-219: order by (d2, index) */
    int64_t maxrow = 0;
    for (int64_t i = 0; i < N; ++i) {
        int64_t m = c->indptr[i + 1] - c->indptr[i];
        if (m > maxrow) maxrow = m;
    }
    sort_rows_mt(c, maxrow, T);
    return c;
}

ORA_API int64_t ora_csr_N(const ora_csr* c) { return c->N; }
ORA_API int64_t ora_csr_E(const ora_csr* c) { return c->E; }
ORA_API int64_t ora_csr_evals(const ora_csr* c) { return c->evals; }
ORA_API void ora_csr_copy(const ora_csr* c, int64_t* indptr, int64_t* nbr, double* d2) {
    memcpy(indptr, c->indptr, sizeof(int64_t) * (size_t)(c->N + 1));
    memcpy(nbr, c->nbr, sizeof(int64_t) * (size_t)c->E);
    memcpy(d2, c->d2, sizeof(double) * (size_t)c->E);
}
ORA_API void ora_csr_free(ora_csr* c) {
    if (!c) return;
    free(c->indptr); free(c->nbr); free(c->d2); free(c);
}

/* csr_level_counts, _kernels.py:222-234: searchsorted(row, r2, 'left'),
 * i.e. the number of row entries with d2 < r2.  counts is [L][N]. */
ORA_API void ora_level_counts(const int64_t* indptr, const double* d2, int64_t N,
                              const double* r2_levels, int64_t L, int64_t* counts) {
    for (int64_t r = 0; r < N; ++r) {
        const int64_t lo = indptr[r], hi = indptr[r + 1];
        for (int64_t l = 0; l < L; ++l) {
            int64_t a = lo, b = hi; /* first position with d2 >= r2 */
            const double t = r2_levels[l];
            while (a < b) {
                int64_t mid = a + (b - a) / 2;
                if (d2[mid] < t) a = mid + 1; else b = mid;
            }
            counts[l * N + r] = a - lo;
        }
    }
}

/* ------------------------------------------------------------------ */
/* Bitmap sampler, _kernels.py:241-353.                                   */

static void clear_rows(uint8_t* bm, int64_t N, int64_t seg_from, int64_t nseg,
                       const int64_t* seg_level_rows, const int64_t* counts,
                       const int64_t* indptr, const int64_t* nbr, int64_t p) {
    const int64_t base = indptr[p];
    for (int64_t l = seg_from; l < nseg; ++l) {
        const int64_t c = counts[seg_level_rows[l] * N + p];
        for (int64_t u = 0; u < c; ++u) bm[l * N + nbr[base + u]] = 0;
        bm[l * N + p] = 0;
    }
}

static int64_t fill_pool(const uint8_t* row, int64_t N, int64_t* pool) {
    int64_t len = 0;
    for (int64_t j = 0; j < N; ++j)
        if (row[j]) pool[len++] = j;
    return len;
}

/* Returns the count reached; out has n_total slots (-1 filled). */
ORA_API int64_t ora_sample_predicted(const int64_t* indptr, const int64_t* nbr,
                                     const int64_t* counts, const int64_t* seg_level_rows,
                                     const int64_t* boundaries, int64_t nseg,
                                     const int64_t* prefix, int64_t k0, int64_t n_total,
                                     int64_t N, uint64_t* state_io, int32_t pick_lowest,
                                     int64_t* out, int32_t* exhausted_out,
                                     int64_t* entered_out) {
    uint64_t state = *state_io;
    uint8_t* bm = (uint8_t*)malloc((size_t)(nseg * N));
    memset(bm, 1, (size_t)(nseg * N));
    for (int64_t t = 0; t < k0; ++t)
        clear_rows(bm, N, 0, nseg, seg_level_rows, counts, indptr, nbr, prefix[t]);
    for (int64_t t = 0; t < n_total; ++t) out[t] = -1;
    for (int64_t t = 0; t < k0; ++t) out[t] = prefix[t];
    int64_t* pool = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N ? N : 1));
    int64_t i = k0, seg = 0;
    while (seg < nseg && i >= boundaries[seg]) seg++;
    if (seg >= nseg) {
        free(bm); free(pool);
        *exhausted_out = 1; *entered_out = 0;
        return k0;
    }
    int64_t pool_len = fill_pool(bm + seg * N, N, pool);
    int64_t scan = 0, entered = 1;
    int32_t exhausted = 0;
    while (i < n_total) {
        if (i >= boundaries[seg]) {
            while (i >= boundaries[seg]) seg++;
            pool_len = fill_pool(bm + seg * N, N, pool);
            scan = 0;
            entered++;
        }
        int64_t picked = -1;
        if (pick_lowest) {
            for (int64_t j = scan; j < N; ++j)
                if (bm[seg * N + j]) { picked = j; scan = j + 1; break; }
        } else {
            while (pool_len > 0) {
                const uint64_t zv = ora_sm64_next(&state);
                const int64_t pos = (int64_t)(zv % (uint64_t)pool_len);
                const int64_t cand = pool[pos];
                pool[pos] = pool[pool_len - 1];
                pool_len--;
                if (bm[seg * N + cand]) { picked = cand; break; }
            }
        }
        if (picked < 0) {
            seg++;
            if (seg >= nseg) { exhausted = 1; break; }
            pool_len = fill_pool(bm + seg * N, N, pool);
            scan = 0;
            entered++;
            continue;
        }
        out[i] = picked;
        clear_rows(bm, N, seg, nseg, seg_level_rows, counts, indptr, nbr, picked);
        i++;
    }
    free(bm); free(pool);
    *state_io = state;
    *exhausted_out = exhausted;
    *entered_out = entered;
    return i;
}

/* earlyterm_scan, _kernels.py:356-367 */
ORA_API void ora_earlyterm_scan(const int64_t* indptr, const int64_t* nbr, const double* d2,
                                const int64_t* lvl1_counts, const uint8_t* taken,
                                double* md, int64_t lo, int64_t hi) {
    for (int64_t i = lo; i < hi; ++i) {
        const int64_t base = indptr[i], c = lvl1_counts[i];
        double best = md[i];
        for (int64_t u = 0; u < c; ++u) {
            const int64_t j = nbr[base + u];
            if (taken[j] && d2[base + u] < best) best = d2[base + u];
        }
        md[i] = best;
    }
}

/* ------------------------------------------------------------------ */
/* Neighbor-search and quality oracles.        */
/* Ordering key is (d2, index) everywhere.           */

/* ball_query_naive: per centroid all points with d2 < r2 (strict),
 * nearest-first, capped at k.  idx/dist are [n][k] (-1 / NaN padded). */
ORA_API void ora_ball_query_naive(const double* x, const double* y, const double* z,
                                  int64_t N, const int64_t* centroids, int64_t n,
                                  double r2, int64_t k, int64_t* idx, double* dist,
                                  int64_t* cnt) {
    ora_entry* buf = (ora_entry*)malloc(sizeof(ora_entry) * (size_t)(N ? N : 1));
    for (int64_t c = 0; c < n; ++c) {
        const int64_t p = centroids[c];
        int64_t m = 0;
        for (int64_t j = 0; j < N; ++j) {
            const double d = sqdist(x[p], y[p], z[p], x[j], y[j], z[j]);
            if (d < r2) { buf[m].d = d; buf[m].j = j; m++; }
        }
        qsort(buf, (size_t)m, sizeof(ora_entry), entry_cmp);
        const int64_t take = m < k ? m : k;
        for (int64_t t = 0; t < k; ++t) {
            idx[c * k + t] = t < take ? buf[t].j : -1;
            dist[c * k + t] = t < take ? sqrt(buf[t].d) : NAN;
        }
        cnt[c] = take;
    }
    free(buf);
}

/* knn_naive: per query, the k nearest pool members by (d2, index). */
ORA_API void ora_knn_naive(const double* x, const double* y, const double* z,
                           const int64_t* queries, int64_t nq, const int64_t* pool,
                           int64_t npool, int64_t k, int64_t* idx, double* dist,
                           int64_t* cnt) {
    ora_entry* buf = (ora_entry*)malloc(sizeof(ora_entry) * (size_t)(npool ? npool : 1));
    for (int64_t q = 0; q < nq; ++q) {
        const int64_t p = queries[q];
        for (int64_t t = 0; t < npool; ++t) {
            const int64_t j = pool[t];
            buf[t].d = sqdist(x[p], y[p], z[p], x[j], y[j], z[j]);
            buf[t].j = j;
        }
        qsort(buf, (size_t)npool, sizeof(ora_entry), entry_cmp);
        const int64_t take = npool < k ? npool : k;
        for (int64_t t = 0; t < k; ++t) {
            idx[q * k + t] = t < take ? buf[t].j : -1;
            dist[q * k + t] = t < take ? sqrt(buf[t].d) : NAN;
        }
        cnt[q] = take;
    }
    free(buf);
}

/* avg_min_spacing helper: per sample, squared distance to the nearest
 * other sample.  The mean is taken by the caller. */
ORA_API void ora_min_spacing_d2(const double* x, const double* y, const double* z,
                                const int64_t* samples, int64_t n, double* out_d2) {
    for (int64_t a = 0; a < n; ++a) {
        const int64_t p = samples[a];
        double best = INFINITY;
        for (int64_t b = 0; b < n; ++b) {
            if (b == a) continue;
            const int64_t q = samples[b];
            const double d = sqdist(x[p], y[p], z[p], x[q], y[q], z[q]);
            if (d < best) best = d;
        }
        out_d2[a] = best;
    }
}
