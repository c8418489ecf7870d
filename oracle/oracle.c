/*
 * oracle.c — CPU restatement of the reference's pull-PageRank hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h).  Compiled by oracle/Makefile with
 * -O2 -ffp-contract=off and no -march, so every double operation rounds
 * exactly as in the reference's canonical Release build (CMakeLists.txt:7-9,
 * "-O3 -DNDEBUG", no FMA contraction on baseline x86-64).  L1/L2 norms
 * accumulate in x87 `long double` exactly as norms.hpp:57-69 does.
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <time.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* std::mt19937 (32-bit Mersenne Twister, the C++ standard's parameters).   */
/* Used through raw draws by tests/support/graph_gen.hpp:4-6.               */
/* ------------------------------------------------------------------------ */
void orc_mt_seed(orc_mt19937* s, uint32_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 624; ++i)
        s->mt[i] = 1812433253u * (s->mt[i - 1] ^ (s->mt[i - 1] >> 30)) + (uint32_t)i;
    s->idx = 624;
}

uint32_t orc_mt_next(orc_mt19937* s) {
    if (s->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            const uint32_t y = (s->mt[i] & 0x80000000u) | (s->mt[(i + 1) % 624] & 0x7fffffffu);
            uint32_t v = s->mt[(i + 397) % 624] ^ (y >> 1);
            if (y & 1u) v ^= 0x9908b0dfu;
            s->mt[i] = v;
        }
        s->idx = 0;
    }
    uint32_t y = s->mt[s->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* ------------------------------------------------------------------------ */
/* Edge lists                                                               */
/* ------------------------------------------------------------------------ */
orc_edges* orc_edges_new(uint32_t n) {
    orc_edges* e = (orc_edges*)calloc(1, sizeof(orc_edges));
    e->n = n;
    return e;
}

void orc_edges_free(orc_edges* e) {
    if (!e) return;
    free(e->pairs);
    free(e);
}

static void edges_reserve(orc_edges* e, uint64_t cap) {
    if (cap <= e->cap) return;
    e->pairs = (uint32_t*)realloc(e->pairs, (size_t)cap * 2 * sizeof(uint32_t));
    e->cap = cap;
}

static void edges_push(orc_edges* e, uint32_t src, uint32_t dst) {
    if (e->m == e->cap) edges_reserve(e, e->cap ? e->cap * 2 : 64);
    e->pairs[2 * e->m] = src;
    e->pairs[2 * e->m + 1] = dst;
    e->m++;
}

/* std::erase_if(el.edges, [&](e){ return drop[e.first]; }) — stable */
static void edges_drop_sources(orc_edges* e, const char* drop) {
    uint64_t w = 0;
    for (uint64_t i = 0; i < e->m; ++i) {
        const uint32_t s = e->pairs[2 * i], d = e->pairs[2 * i + 1];
        if (drop[s]) continue;
        e->pairs[2 * w] = s;
        e->pairs[2 * w + 1] = d;
        ++w;
    }
    e->m = w;
}

/* graph_gen.hpp:21-37 */
orc_edges* orc_random_digraph(orc_mt19937* rng, uint32_t n, double p, int force_dangling) {
    orc_edges* el = orc_edges_new(n);
    const uint32_t threshold = (uint32_t)(p * 4294967296.0);
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t v = 0; v < n; ++v)
            if (orc_mt_next(rng) < threshold) edges_push(el, u, v);
    if (force_dangling && n > 1) {
        const uint32_t count = 1 + orc_mt_next(rng) % (n / 2 + 1);
        char* drop = (char*)calloc(n, 1);
        for (uint32_t i = 0; i < count; ++i) drop[orc_mt_next(rng) % n] = 1;
        edges_drop_sources(el, drop);
        free(drop);
    }
    return el;
}

/* graph_gen.hpp:41-49 */
orc_edges* orc_regular_ring(uint32_t n, uint32_t k) {
    orc_edges* el = orc_edges_new(n);
    edges_reserve(el, (uint64_t)n * k);
    for (uint32_t v = 0; v < n; ++v)
        for (uint32_t j = 1; j <= k; ++j) edges_push(el, v, (v + j) % n);
    return el;
}

/* graph_gen.hpp:54-85 */
orc_edges* orc_scale_free_web(orc_mt19937* rng, uint32_t n, uint32_t out_links,
                              double dangling_fraction) {
    orc_edges* el = orc_edges_new(n);
    uint64_t pool_n = 0;
    uint32_t* pool = (uint32_t*)malloc(((size_t)n * out_links + n + 1) * sizeof(uint32_t));
    const uint32_t seed_size = out_links + 1 < n ? out_links + 1 : n;
    for (uint32_t v = 0; v < seed_size; ++v) {
        const uint32_t t = (v + 1) % seed_size;
        edges_push(el, v, t);
        pool[pool_n++] = t;
    }
    for (uint32_t v = seed_size; v < n; ++v) {
        for (uint32_t j = 0; j < out_links; ++j) {
            /* 70% preferential, 30% uniform; && short-circuits the 2nd draw */
            uint32_t target;
            if (orc_mt_next(rng) % 10 < 7 && pool_n != 0)
                target = pool[orc_mt_next(rng) % pool_n];
            else
                target = orc_mt_next(rng) % v;
            edges_push(el, v, target);
            pool[pool_n++] = target;
        }
    }
    const uint32_t dangling_count = (uint32_t)(dangling_fraction * n);
    char* drop = (char*)calloc(n ? n : 1, 1);
    for (uint32_t i = 0; i < dangling_count; ++i) drop[orc_mt_next(rng) % n] = 1;
    if (dangling_count > 0) edges_drop_sources(el, drop);
    free(drop);
    free(pool);
    return el;
}

/* ------------------------------------------------------------------------ */
/* Counter-based benchmark generators (spec: DESIGN.md "Synthetic inputs"). */
/* ------------------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

static uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return orc_mix64(seed * 0x9E3779B97F4A7C15ull + stream);
}

uint64_t orc_prob_threshold(double p) {
    if (!(p > 0.0)) return 0;
    const double x = p * 18446744073709551616.0;
    if (x >= 18446744073709551616.0) return UINT64_MAX;
    return (uint64_t)x;
}

uint32_t orc_rmat_perm(uint32_t x32, uint32_t scale, uint64_t seed) {
    const uint64_t mask = (scale >= 32) ? 0xFFFFFFFFull : ((1ull << scale) - 1);
    const uint64_t pk = stream_key(seed, 2);
    const uint32_t hs = (scale + 1) / 2;
    uint64_t x = x32;
    for (uint64_t r = 0; r < 3; ++r) {
        const uint64_t k = orc_mix64(pk + r);
        x = (x * (k | 1ull)) & mask;
        x = (x + (k >> 40)) & mask;
        x ^= x >> hs;
    }
    return (uint32_t)x;
}

void orc_rmat_gen_init(orc_rmat_gen* g, uint32_t scale, double a, double b, double c,
                       uint64_t seed) {
    g->scale = scale;
    g->ta = orc_prob_threshold(a);
    g->tab = orc_prob_threshold(a + b);
    g->tabc = orc_prob_threshold(a + b + c);
    g->kd = stream_key(seed, 1);
    const uint64_t pk = stream_key(seed, 2); /* orc_rmat_perm's keys */
    for (int r = 0; r < 3; ++r) g->pk[r] = orc_mix64(pk + (uint64_t)r);
    g->mask = (scale >= 32) ? 0xFFFFFFFFull : ((1ull << scale) - 1);
    g->hs = (scale + 1) / 2;
}

static uint32_t rmat_gen_perm(const orc_rmat_gen* g, uint32_t x32) {
    uint64_t x = x32;
    for (int r = 0; r < 3; ++r) {
        const uint64_t k = g->pk[r];
        x = (x * (k | 1ull)) & g->mask;
        x = (x + (k >> 40)) & g->mask;
        x ^= x >> g->hs;
    }
    return (uint32_t)x;
}

int orc_rmat_gen_edge(const orc_rmat_gen* g, uint64_t i, uint32_t* src_out, uint32_t* dst_out) {
    uint32_t src = 0, dst = 0;
    for (uint32_t l = 0; l < g->scale; ++l) {
        const uint64_t x = orc_mix64(g->kd ^ ((i << 6) | l));
        const uint32_t bit = 1u << (g->scale - 1 - l);
        if (x < g->ta) {
        } else if (x < g->tab) {
            dst |= bit;
        } else if (x < g->tabc) {
            src |= bit;
        } else {
            src |= bit;
            dst |= bit;
        }
    }
    if (src == dst) return 0; /* self-loops removed (BASELINE.json configs) */
    *src_out = rmat_gen_perm(g, src);
    *dst_out = rmat_gen_perm(g, dst);
    return 1;
}

orc_edges* orc_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                    uint64_t seed) {
    const uint64_t n64 = 1ull << scale;
    orc_edges* el = orc_edges_new((uint32_t)(n64 > 0xFFFFFFFFull ? 0xFFFFFFFFull : n64));
    const uint64_t m = (uint64_t)edge_factor << scale;
    edges_reserve(el, m);
    orc_rmat_gen g;
    orc_rmat_gen_init(&g, scale, a, b, c, seed);
    for (uint64_t i = 0; i < m; ++i) {
        uint32_t src, dst;
        if (orc_rmat_gen_edge(&g, i, &src, &dst)) edges_push(el, src, dst);
    }
    return el;
}

static uint64_t mulhi64(uint64_t x, uint64_t n) {
    return (uint64_t)(((unsigned __int128)x * n) >> 64);
}

orc_edges* orc_grid(uint32_t side, double p, double longrange_frac, uint64_t seed) {
    const uint64_t n = (uint64_t)side * side;
    orc_edges* el = orc_edges_new((uint32_t)n);
    const uint64_t tp = orc_prob_threshold(p);
    const uint64_t kg = stream_key(seed, 3);
    const uint64_t uh = (uint64_t)side * (side - 1); /* horizontal candidates */
    edges_reserve(el, (uint64_t)(2.0 * p * 2 * uh) + 1024);
    for (uint64_t t = 0; t < 2 * uh; ++t) {
        if (!(orc_mix64(kg ^ t) < tp)) continue;
        uint64_t a, b;
        if (t < uh) {
            const uint64_t r = t / (side - 1), cc = t % (side - 1);
            a = r * side + cc;
            b = a + 1;
        } else {
            const uint64_t j = t - uh;
            const uint64_t r = j / side, cc = j % side;
            a = r * side + cc;
            b = a + side;
        }
        edges_push(el, (uint32_t)a, (uint32_t)b);
        edges_push(el, (uint32_t)b, (uint32_t)a);
    }
    const uint64_t L = (uint64_t)(longrange_frac * (double)n);
    const uint64_t kl = stream_key(seed, 4);
    for (uint64_t j = 0; j < L; ++j) {
        const uint64_t s = mulhi64(orc_mix64(kl ^ (2 * j)), n);
        const uint64_t d = mulhi64(orc_mix64(kl ^ (2 * j + 1)), n);
        if (s == d) continue;
        edges_push(el, (uint32_t)s, (uint32_t)d);
    }
    return el;
}

/* ------------------------------------------------------------------------ */
/* build_csr — graph.hpp:204-234                                            */
/* The (dst,src) lexicographic order of graph.hpp:209-212 is the numeric    */
/* order of the 64-bit key dst<<32|src, so an LSD radix sort of that key    */
/* produces the same sequence as the reference's std::sort (total order).   */
/* ------------------------------------------------------------------------ */
static void radix_sort_u64(uint64_t* keys, uint64_t m) {
    if (m < 2) return;
    uint64_t* tmp = (uint64_t*)malloc((size_t)m * sizeof(uint64_t));
    uint64_t* count = (uint64_t*)malloc(65536 * sizeof(uint64_t));
    uint64_t* src = keys;
    uint64_t* dst = tmp;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 16 * pass;
        memset(count, 0, 65536 * sizeof(uint64_t));
        for (uint64_t i = 0; i < m; ++i) count[(src[i] >> shift) & 0xFFFF]++;
        int trivial = 0;
        for (int d = 0; d < 65536; ++d)
            if (count[d] == m) trivial = 1;
        if (trivial) continue;
        uint64_t sum = 0;
        for (int d = 0; d < 65536; ++d) {
            const uint64_t c = count[d];
            count[d] = sum;
            sum += c;
        }
        for (uint64_t i = 0; i < m; ++i) dst[count[(src[i] >> shift) & 0xFFFF]++] = src[i];
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != keys) memcpy(keys, src, (size_t)m * sizeof(uint64_t));
    free(count);
    free(tmp);
}

orc_csr* orc_build_csr(uint32_t n, const uint32_t* pairs, uint64_t m) {
    uint64_t* keys = (uint64_t*)malloc((size_t)(m ? m : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < m; ++i)
        keys[i] = ((uint64_t)pairs[2 * i + 1] << 32) | pairs[2 * i];
    radix_sort_u64(keys, m);
    /* std::unique (graph.hpp:213) */
    uint64_t u = 0;
    for (uint64_t i = 0; i < m; ++i)
        if (i == 0 || keys[i] != keys[u - 1]) keys[u++] = keys[i];

    orc_csr* g = (orc_csr*)calloc(1, sizeof(orc_csr));
    g->n = n;
    g->e = u;
    g->in_offsets = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    g->out_degree = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    g->in_neighbors = (uint32_t*)malloc((size_t)(u ? u : 1) * sizeof(uint32_t));
    /* graph.hpp:220-223 counts, :224 inclusive scan, :226-228 fill */
    for (uint64_t i = 0; i < u; ++i) {
        const uint32_t dst = (uint32_t)(keys[i] >> 32), src = (uint32_t)keys[i];
        g->in_offsets[(size_t)dst + 1]++;
        g->out_degree[src]++;
    }
    for (uint64_t v = 0; v < n; ++v) g->in_offsets[v + 1] += g->in_offsets[v];
    for (uint64_t i = 0; i < u; ++i) g->in_neighbors[i] = (uint32_t)keys[i];
    free(keys);
    /* graph.hpp:230-231 dangling, ascending */
    uint32_t nd = 0;
    for (uint32_t v = 0; v < n; ++v) nd += g->out_degree[v] == 0;
    g->dangling = (uint32_t*)malloc((size_t)(nd ? nd : 1) * sizeof(uint32_t));
    g->ndangling = nd;
    nd = 0;
    for (uint32_t v = 0; v < n; ++v)
        if (g->out_degree[v] == 0) g->dangling[nd++] = v;
    return g;
}

void orc_csr_free(orc_csr* g) {
    if (!g) return;
    free(g->in_offsets);
    free(g->in_neighbors);
    free(g->out_degree);
    free(g->dangling);
    free(g);
}

/* ------------------------------------------------------------------------ */
/* error_norm — norms.hpp:48-78                                             */
/* ------------------------------------------------------------------------ */
double orc_error_norm(int kind, const double* r, const double* s, uint64_t n) {
    switch (kind) {
    case 0: { /* L1, norms.hpp:57-61 */
        long double sum = 0.0L;
        for (uint64_t i = 0; i < n; ++i) sum += fabs(r[i] - s[i]);
        return (double)sum;
    }
    case 1: { /* L2, norms.hpp:62-69 */
        long double sum = 0.0L;
        for (uint64_t i = 0; i < n; ++i) {
            const long double d = r[i] - s[i];
            sum += d * d;
        }
        return (double)sqrtl(sum);
    }
    default: { /* LInf, norms.hpp:70-75 (std::max keeps the first on ties) */
        double max = 0.0;
        for (uint64_t i = 0; i < n; ++i) {
            const double a = fabs(r[i] - s[i]);
            if (max < a) max = a;
        }
        return max;
    }
    }
}

/* ------------------------------------------------------------------------ */
/* pagerank — pagerank.hpp:70-108                                           */
/* ------------------------------------------------------------------------ */
static int config_invalid(double alpha, double tol, int max_iter) {
    /* PageRankConfig::validate, pagerank.hpp:29-39 */
    if (!(alpha >= 0.0 && alpha <= 1.0)) return 1;
    if (!(tol > 0.0)) return 1;
    if (max_iter < 1) return 1;
    return 0;
}

int orc_pagerank(const orc_csr* g, double alpha, double tol, int norm, int max_iter,
                 double* ranks_out, int* iterations, int* converged, double* err_trace) {
    if (config_invalid(alpha, tol, max_iter)) return 1;
    const uint32_t n = g->n;
    if (n == 0) return 1; /* pagerank.hpp:74 */

    double* prev = (double*)malloc((size_t)n * sizeof(double));
    double* next = (double*)malloc((size_t)n * sizeof(double));
    for (uint32_t v = 0; v < n; ++v) prev[v] = 1.0 / n; /* :77 */

    int iteration = 0;
    double err = INFINITY;
    do {
        double dangling_sum = 0.0; /* :85-86, ascending dangling list */
        for (uint32_t i = 0; i < g->ndangling; ++i) dangling_sum += prev[g->dangling[i]];
        const double teleport = (1.0 - alpha) / n + alpha * dangling_sum / n; /* :87 */

        for (uint32_t v = 0; v < n; ++v) { /* :89-93 */
            double acc = 0.0;
            for (uint64_t j = g->in_offsets[v]; j < g->in_offsets[(size_t)v + 1]; ++j) {
                const uint32_t u = g->in_neighbors[j];
                acc += prev[u] / g->out_degree[u];
            }
            next[v] = teleport + alpha * acc;
        }

        err = orc_error_norm(norm, next, prev, n); /* :95 */
        if (err_trace) err_trace[iteration] = err;
        ++iteration;
        double* t = prev; /* :97 swap */
        prev = next;
        next = t;
    } while (err >= tol && iteration < max_iter); /* :99 */

    memcpy(ranks_out, prev, (size_t)n * sizeof(double)); /* :103 */
    *iterations = iteration;
    *converged = err < tol; /* :105 */
    free(prev);
    free(next);
    return 0;
}

/* pagerank.hpp:70-108 with the v-loop (:89-93) split over `threads` host
 * threads.  Each next[v] is computed by exactly the reference's expression in
 * the same ascending-source order, and the dangling sum (:85-86) and the norm
 * (:95) stay sequential on the calling thread, so ranks, errors and
 * iteration counts are BIT-IDENTICAL to orc_pagerank (and to the reference:
 * tests/test_oracle.py) — SPEC.md:194 allows parallelising the vertex loop.
 * The CPU baseline for configs whose single-threaded iteration takes minutes
 * (C4, C5).  elapsed_ms: the loop only, like PageRankResult::elapsed. */
typedef struct {
    const orc_csr* g;
    const double* prev;
    double* next;
    double teleport, alpha;
    uint32_t v0, v1;
} mt_slice;

static void* mt_pull(void* arg) {
    const mt_slice* sl = (const mt_slice*)arg;
    const orc_csr* g = sl->g;
    for (uint32_t v = sl->v0; v < sl->v1; ++v) {
        double acc = 0.0;
        for (uint64_t j = g->in_offsets[v]; j < g->in_offsets[(size_t)v + 1]; ++j) {
            const uint32_t u = g->in_neighbors[j];
            acc += sl->prev[u] / g->out_degree[u];
        }
        sl->next[v] = sl->teleport + sl->alpha * acc;
    }
    return NULL;
}

int orc_pagerank_mt(const orc_csr* g, double alpha, double tol, int norm, int max_iter, int threads,
                    double* ranks_out, int* iterations, int* converged, double* err_trace,
                    double* elapsed_ms) {
    if (config_invalid(alpha, tol, max_iter)) return 1;
    const uint32_t n = g->n;
    if (n == 0) return 1;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    double* prev = (double*)malloc((size_t)n * sizeof(double));
    double* next = (double*)malloc((size_t)n * sizeof(double));
    if (!prev || !next) {
        free(prev);
        free(next);
        return 2;
    }
    for (uint32_t v = 0; v < n; ++v) prev[v] = 1.0 / n;
    for (uint32_t v = 0; v < n; ++v) next[v] = 0.0;
    /* slices of roughly equal edge counts (plus one unit per row) */
    uint32_t cut[257];
    cut[0] = 0;
    const double total = (double)g->in_offsets[n] + n;
    for (int t = 1; t < threads; ++t) {
        const double want = total * t / threads;
        uint32_t lo = cut[t - 1], hi = n;
        while (lo < hi) {
            const uint32_t mid = lo + (hi - lo) / 2;
            if ((double)g->in_offsets[mid] + mid < want) lo = mid + 1;
            else hi = mid;
        }
        cut[t] = lo;
    }
    cut[threads] = n;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    int iteration = 0;
    double err = INFINITY;
    pthread_t tid[256];
    mt_slice sl[256];
    do {
        double dangling_sum = 0.0;
        for (uint32_t i = 0; i < g->ndangling; ++i) dangling_sum += prev[g->dangling[i]];
        const double teleport = (1.0 - alpha) / n + alpha * dangling_sum / n;
        for (int t = 0; t < threads; ++t) {
            sl[t] = (mt_slice){g, prev, next, teleport, alpha, cut[t], cut[t + 1]};
            if (t) pthread_create(&tid[t], NULL, mt_pull, &sl[t]);
        }
        mt_pull(&sl[0]);
        for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
        err = orc_error_norm(norm, next, prev, n);
        if (err_trace) err_trace[iteration] = err;
        ++iteration;
        double* tt = prev;
        prev = next;
        next = tt;
    } while (err >= tol && iteration < max_iter);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (elapsed_ms) *elapsed_ms = (t1.tv_sec - t0.tv_sec) * 1e3 + (t1.tv_nsec - t0.tv_nsec) * 1e-6;
    if (ranks_out) memcpy(ranks_out, prev, (size_t)n * sizeof(double));
    *iterations = iteration;
    *converged = err < tol;
    free(prev);
    free(next);
    return 0;
}

/* One iteration of pagerank.hpp:85-93 for selected rows only, from the full
 * previous rank vector: the dangling sum over ascending ids (:85-86, the
 * dangling list is ascending, graph.hpp:230-231), the teleport (:87), and
 * each row's in-neighbour sum in ascending source order (:89-92).  Lets the
 * tests check a graph too large for a full oracle run (C5) one step at a
 * time against the GPU's own previous iterate. */
double orc_pagerank_step_rows(uint32_t n, const double* prev, const uint32_t* out_degree,
                              double alpha, uint32_t nrows, const uint64_t* off,
                              const uint32_t* nbr, double* out) {
    double dangling_sum = 0.0;
    for (uint32_t v = 0; v < n; ++v)
        if (out_degree[v] == 0) dangling_sum += prev[v];
    const double teleport = (1.0 - alpha) / n + alpha * dangling_sum / n;
    for (uint32_t i = 0; i < nrows; ++i) {
        double acc = 0.0;
        for (uint64_t j = off[i]; j < off[i + 1]; ++j) {
            const uint32_t u = nbr[j];
            acc += prev[u] / out_degree[u];
        }
        out[i] = teleport + alpha * acc;
    }
    return teleport;
}

/* tests/support/dense_oracle.hpp:24-62 */
int orc_dense_pagerank(uint32_t n, const uint32_t* pairs, uint64_t m, double alpha,
                       double tol, int norm, int max_iter, double* ranks_out,
                       int* iterations, int* converged) {
    if (n == 0) return 1;
    char* adj = (char*)calloc((size_t)n * n, 1); /* [source][target] */
    for (uint64_t i = 0; i < m; ++i) adj[(size_t)pairs[2 * i] * n + pairs[2 * i + 1]] = 1;
    uint32_t* out_degree = (uint32_t*)calloc(n, sizeof(uint32_t));
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t v = 0; v < n; ++v)
            if (adj[(size_t)u * n + v]) ++out_degree[u];
    double* prev = (double*)malloc((size_t)n * sizeof(double));
    double* next = (double*)malloc((size_t)n * sizeof(double));
    for (uint32_t v = 0; v < n; ++v) prev[v] = 1.0 / n;
    int iteration = 0;
    double err = 0;
    do {
        double dangling_sum = 0.0;
        for (uint32_t u = 0; u < n; ++u)
            if (out_degree[u] == 0) dangling_sum += prev[u];
        const double teleport = (1.0 - alpha) / n + alpha * dangling_sum / n;
        for (uint32_t v = 0; v < n; ++v) {
            double acc = 0.0;
            for (uint32_t u = 0; u < n; ++u)
                if (adj[(size_t)u * n + v]) acc += prev[u] / out_degree[u];
            next[v] = teleport + alpha * acc;
        }
        err = orc_error_norm(norm, next, prev, n);
        ++iteration;
        double* t = prev;
        prev = next;
        next = t;
    } while (err >= tol && iteration < max_iter);
    memcpy(ranks_out, prev, (size_t)n * sizeof(double));
    *iterations = iteration;
    *converged = err < tol;
    free(adj);
    free(out_degree);
    free(prev);
    free(next);
    return 0;
}

/* pagerank.hpp:113-123 */
int orc_estimate_iterations(double alpha, double tol) {
    if (!(alpha > 0.0 && alpha < 1.0)) return -1;
    if (!(tol > 0.0 && tol < 1.0)) return -1;
    const long estimate = lround(log10(tol) / log10(alpha));
    return (int)(estimate > 1 ? estimate : 1);
}

uint64_t orc_hash64(const void* data, uint64_t nbytes) {
    const unsigned char* p = (const unsigned char*)data;
    uint64_t h = 0x243F6A8885A308D3ull ^ nbytes;
    uint64_t i = 0;
    for (; i + 8 <= nbytes; i += 8) {
        uint64_t w;
        memcpy(&w, p + i, 8);
        h = orc_mix64(h ^ w) + 0x9E3779B97F4A7C15ull;
    }
    if (i < nbytes) {
        uint64_t w = 0;
        memcpy(&w, p + i, (size_t)(nbytes - i));
        h = orc_mix64(h ^ w ^ 0xA5A5A5A5A5A5A5A5ull);
    }
    return orc_mix64(h);
}
