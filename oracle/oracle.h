/*
 * oracle.h — CPU restatement of the reference's pull-PageRank hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (libprgpu.so, the C++
 * drop-in header, the Python mirror) may include, link or call this code.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it, and only as the checker or the timed
 * CPU baseline.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/include/pagerank_lab/*.hpp, tests/support/*.hpp).
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref, built from the reference headers by oracle/Makefile) and
 * against the golden vectors under tests/golden/ (see tests/test_oracle.py).
 */
#ifndef PRGPU_ORACLE_H
#define PRGPU_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- std::mt19937 restated (used by tests/support/graph_gen.hpp:21-85) ---- */
typedef struct {
    uint32_t mt[624];
    int idx;
} orc_mt19937;

void orc_mt_seed(orc_mt19937* s, uint32_t seed);
uint32_t orc_mt_next(orc_mt19937* s);

/* ---- edge lists: graph.hpp:36-39 (interleaved (src,dst) u32 pairs) ---- */
typedef struct {
    uint32_t n;       /* vertex_count */
    uint64_t m;       /* number of pairs */
    uint64_t cap;
    uint32_t* pairs;  /* pairs[2i] = source, pairs[2i+1] = target */
} orc_edges;

orc_edges* orc_edges_new(uint32_t n);
void orc_edges_free(orc_edges* e);

/* graph_gen.hpp:21-37 */
orc_edges* orc_random_digraph(orc_mt19937* rng, uint32_t n, double p, int force_dangling);
/* graph_gen.hpp:41-49 */
orc_edges* orc_regular_ring(uint32_t n, uint32_t k);
/* graph_gen.hpp:54-85 */
orc_edges* orc_scale_free_web(orc_mt19937* rng, uint32_t n, uint32_t out_links,
                              double dangling_fraction);

/* Benchmark generators (BASELINE.json configs; spec in DESIGN.md §Inputs).
 * Counter-based, so the device generator in libprgpu emits the same edges. */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_prob_threshold(double p); /* floor(p * 2^64), saturating */
orc_edges* orc_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                    uint64_t seed);
orc_edges* orc_grid(uint32_t side, double p, double longrange_frac, uint64_t seed);
uint32_t orc_rmat_perm(uint32_t x, uint32_t scale, uint64_t seed);
/* edge i of the RMAT stream by itself (orc_rmat = every i in [0, ef << scale)):
 * lets a builder regenerate the stream in parallel passes instead of holding it */
typedef struct {
    uint32_t scale, hs;
    uint64_t ta, tab, tabc, kd, pk[3], mask;
} orc_rmat_gen;
void orc_rmat_gen_init(orc_rmat_gen* g, uint32_t scale, double a, double b, double c,
                       uint64_t seed);
int orc_rmat_gen_edge(const orc_rmat_gen* g, uint64_t i, uint32_t* src, uint32_t* dst); /* 0: self-loop */

/* ---- reverse CSR: graph.hpp:47-60, build_csr graph.hpp:204-234 ---- */
typedef struct {
    uint32_t n;
    uint64_t e;
    uint64_t* in_offsets;   /* n+1 */
    uint32_t* in_neighbors; /* e */
    uint32_t* out_degree;   /* n */
    uint32_t* dangling;     /* ndangling, ascending */
    uint32_t ndangling;
} orc_csr;

orc_csr* orc_build_csr(uint32_t n, const uint32_t* pairs, uint64_t m);
void orc_csr_free(orc_csr* g);

/* ---- norms.hpp:48-78 (kind 0 = L1, 1 = L2, 2 = LInf) ---- */
double orc_error_norm(int kind, const double* r, const double* s, uint64_t n);

/* ---- pagerank.hpp:70-108.  Returns 0 ok, 1 invalid argument.
 * err_trace (nullable) receives err of every iteration (max_iter slots). */
int orc_pagerank(const orc_csr* g, double alpha, double tol, int norm, int max_iter,
                 double* ranks_out, int* iterations, int* converged, double* err_trace);

/* pagerank.hpp:85-93 for rows off/nbr (reference layout, ascending) from the
 * full prev vector; returns the teleport term.  out[nrows]. */
/* the same run with the vertex loop on `threads` host threads: bit-identical */
int orc_pagerank_mt(const orc_csr* g, double alpha, double tol, int norm, int max_iter, int threads,
                    double* ranks_out, int* iterations, int* converged, double* err_trace,
                    double* elapsed_ms);
double orc_pagerank_step_rows(uint32_t n, const double* prev, const uint32_t* out_degree,
                              double alpha, uint32_t nrows, const uint64_t* off,
                              const uint32_t* nbr, double* out);

/* tests/support/dense_oracle.hpp:24-62 */
int orc_dense_pagerank(uint32_t n, const uint32_t* pairs, uint64_t m, double alpha,
                       double tol, int norm, int max_iter, double* ranks_out,
                       int* iterations, int* converged);

/* pagerank.hpp:113-123; returns -1 where the reference throws */
int orc_estimate_iterations(double alpha, double tol);

/* Golden-file fingerprint: word-wise splitmix hash of a byte range. */
uint64_t orc_hash64(const void* data, uint64_t nbytes);

#ifdef __cplusplus
}
#endif
#endif
