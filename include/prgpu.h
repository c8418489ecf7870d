/*
 * prgpu.h — C ABI of libprgpu.so, the B200-native pull-PageRank engine.
 *
 * The reference (pagerank-lab, /root/reference/proj) has no FFI: its boundary
 * is a set of inline C++ functions in namespace pagerank_lab.  Each entry
 * point below replaces one of them; the C++ drop-in header
 * include/pagerank_b200/pagerank_lab.hpp and the Python mirror
 * paper_2108_02997_b200/pagerank_lab.py bind these and keep the reference's
 * signatures and error behaviour (INTEGRATION.md shows the bindings).
 *
 * Conventions: plain pointers and sizes, no exceptions cross the boundary,
 * every call returns a PRGPU_* status and leaves a message in
 * prgpu_last_error() (thread-local).  Host pointers are ordinary host memory
 * unless a name says "device".  A prgpu_graph is immutable after construction
 * and may be shared by concurrent prgpu_pagerank calls (graph.hpp:44-46,
 * SPEC.md "engine is reentrant"); each call uses its own stream and scratch.
 */
#ifndef PRGPU_H
#define PRGPU_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PRGPU_API __attribute__((visibility("default")))
#else
#define PRGPU_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------- */
#define PRGPU_OK 0
#define PRGPU_EINVAL 1 /* maps to std::invalid_argument / ValueError          */
#define PRGPU_ECUDA 2  /* CUDA runtime or kernel failure                       */
#define PRGPU_ENCCL 3  /* NCCL failure (multi-GPU)                             */
#define PRGPU_ENOMEM 4 /* device allocation failed                             */
#define PRGPU_EPARSE 5 /* MatrixMarket syntax error: MtxParseError(line)       */
#define PRGPU_EIO 6    /* a file cannot be opened / read: std::runtime_error    */

/* ---- norms (norms.hpp:18 NormKind) -------------------------------------- */
#define PRGPU_NORM_L1 0
#define PRGPU_NORM_L2 1
#define PRGPU_NORM_LINF 2

#define PRGPU_MAX_LANES 16 /* batched rank vectors per run (alpha sweep) */

typedef struct prgpu_graph prgpu_graph;
typedef struct prgpu_session prgpu_session;

/* Summary of a device graph. */
typedef struct {
    uint32_t vertex_count;   /* CsrGraph::vertex_count               graph.hpp:48 */
    uint64_t edge_count;     /* CsrGraph::edge_count() after dedup   graph.hpp:59 */
    uint32_t dangling_count; /* |CsrGraph::dangling|                 graph.hpp:52 */
    uint32_t max_in_degree;
    uint32_t hub_rows;       /* rows pulled block-per-vertex */
    uint32_t warp_rows;      /* rows pulled warp-per-vertex */
    uint32_t thread_rows;    /* rows pulled by a lane group (in-degree >= 1) */
    uint32_t empty_rows;     /* in-degree 0: rank = c0 */
    int device;
} prgpu_graph_info;

/* ---- graph construction (replaces build_csr, graph.hpp:204-234) ---------
 * Edges are the reference's EdgeList layout: interleaved (source, target)
 * u32 pairs, duplicates allowed, self-loops kept (graph.hpp:36-39,202-203).
 * The in-CSR is built on the device (sort by (target, source), unique,
 * count, scan), then relabelled for the pull kernel. */
PRGPU_API int prgpu_graph_build(uint32_t n, const uint32_t* edge_pairs, uint64_t m, int device,
                      prgpu_graph** out);
/* Same, from pairs already resident on `device`. */
PRGPU_API int prgpu_graph_build_device(uint32_t n, const uint32_t* d_edge_pairs, uint64_t m, int device,
                             prgpu_graph** out);
/* From a reference-layout CsrGraph on the host (graph.hpp:47-60):
 * in_offsets[n+1], in_neighbors[in_offsets[n]] (ascending per row),
 * out_degree[n].  Validated on the device. */
PRGPU_API int prgpu_graph_from_csr(uint32_t n, const uint64_t* in_offsets, const uint32_t* in_neighbors,
                         const uint32_t* out_degree, int device, prgpu_graph** out);
/* Synthetic benchmark graphs generated on the device (DESIGN.md "Synthetic
 * inputs"; bit-identical to oracle/oracle.c's orc_rmat / orc_grid). */
PRGPU_API int prgpu_graph_generate_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                              uint64_t seed, int device, prgpu_graph** out);
PRGPU_API int prgpu_graph_generate_grid(uint32_t side, double p, double longrange_frac, uint64_t seed,
                              int device, prgpu_graph** out);
/* Rank `rank`'s shard of the same RMAT graph for an `nranks`-rank partition
 * (SURVEY 8e set-up), built without ever holding the whole edge list: every
 * rank generates all edges slab by slab, computes the exact global in- and
 * out-degrees (so the relabelled vertex arrays equal the whole graph's) and
 * keeps the in-edges of its contiguous range of engine rows only (cost-
 * balanced; prgpu_graph_shard_info).  Only prgpu_part_create(rank, nranks)
 * sessions run on it (contiguous rows, every contribution row stored into
 * every peer); downloading its edges is EINVAL. */
PRGPU_API int prgpu_graph_generate_rmat_shard(uint32_t scale, uint32_t edge_factor, double a, double b,
                                              double c, uint64_t seed, int rank, int nranks, int device,
                                              prgpu_graph** out);
/* Device memory held by a graph and/or a session (either may be NULL). */
PRGPU_API int prgpu_device_bytes(const prgpu_graph* g, const prgpu_session* s, uint64_t* graph_bytes,
                                 uint64_t* session_bytes);
/* rank / nranks / engine rows [row_begin, row_end) / edges held (a whole
 * graph: 0, 1, [0, n), its edge count). Any pointer may be NULL. */
PRGPU_API int prgpu_graph_shard_info(const prgpu_graph* g, int* rank, int* nranks, uint32_t* row_begin,
                                     uint32_t* row_end, uint64_t* local_edges);

PRGPU_API int prgpu_graph_get_info(const prgpu_graph* g, prgpu_graph_info* info);
/* Copies the reference-layout CSR back (any pointer may be NULL):
 * in_offsets[n+1], in_neighbors[e], out_degree[n], dangling[dangling_count]. */
PRGPU_API int prgpu_graph_download(const prgpu_graph* g, uint64_t* in_offsets, uint32_t* in_neighbors,
                         uint32_t* out_degree, uint32_t* dangling);
/* In-neighbours of selected rows only (original ids, ascending per row, as
 * in_neighbors): off[nrows+1] is always filled and *total set; nbr is
 * filled when total <= cap.  For graphs too large to download whole (the
 * scale-28 config); no reference counterpart (test/diagnostic call). */
PRGPU_API int prgpu_graph_rows(const prgpu_graph* g, const uint32_t* rows, uint32_t nrows, uint64_t* off,
                     uint32_t* nbr, uint64_t cap, uint64_t* total);
/* ---- MatrixMarket ingest (replaces parse_matrix_market / load_matrix_market /
 * load_csr_graph, graph.hpp:111-199,238-251) -------------------------------
 * Same language and errors as the reference (banner, size line, entries,
 * symmetric expansion, weights validated and discarded, first error in file
 * order with its 1-based line), parsed by `threads` host threads (<= 0: all
 * cores).  On a syntax error: PRGPU_EPARSE, *err_line = the line, and
 * prgpu_last_error() = "line L: what" ("<path>: line L: what" for files);
 * a file that cannot be opened: PRGPU_EIO, "cannot open graph file: <path>".
 * pairs: malloc'd (source, target) u32 pairs, release with prgpu_pairs_free. */
PRGPU_API int prgpu_mtx_parse(const char* text, uint64_t len, int threads, uint32_t* n, uint32_t** pairs,
                    uint64_t* m, uint64_t* err_line);
PRGPU_API int prgpu_mtx_load(const char* path, int threads, uint32_t* n, uint32_t** pairs, uint64_t* m,
                   uint64_t* err_line);
PRGPU_API void prgpu_pairs_free(uint32_t* pairs);
/* load_csr_graph(path): parse in parallel, then build_csr on the device. */
PRGPU_API int prgpu_graph_load_mtx(const char* path, int threads, int device, prgpu_graph** out,
                         uint64_t* err_line);
PRGPU_API void prgpu_graph_free(prgpu_graph* g);

/* ---- engine (replaces pagerank, pagerank.hpp:70-108) --------------------
 * K rank vectors ("lanes") run together, one alpha each; every edge visit
 * feeds all K lanes.  A lane stops when every norm in its stop mask is below
 * its tolerance (strict, pagerank.hpp:99,105) or at max_iterations; its
 * ranks then freeze.  K = 1 with stop_mask = 1 << norm is exactly the
 * reference's pagerank(g, {alpha, tolerance, norm, max_iterations}). */
typedef struct {
    int lanes;                /* K, 1..PRGPU_MAX_LANES */
    const double* alphas;     /* [K] damping factors, each in [0, 1] */
    const double* tolerances; /* [K] (NULL: use `tolerance` for all lanes) */
    double tolerance;         /* > 0 */
    int norm;                 /* PRGPU_NORM_* reported as final_err */
    uint32_t stop_mask;       /* bit i = norm i must be < tolerance; 0 => 1 << norm */
    int max_iterations;       /* >= 1 */
    const double* ref_ranks;  /* optional [n] host, original ids: trace L1 distance to it */
} prgpu_params;

typedef struct {
    double* ranks;            /* optional [K][n] host, original vertex ids */
    int* iterations;          /* optional [K] */
    uint8_t* converged;       /* optional [K] */
    double* final_err;        /* optional [K]: err of the last iteration under `norm` */
    double* err_trace;        /* optional [max_iterations][K][4]: L1, L2, LInf, L1-vs-ref;
                                 entries no iteration wrote (after the lane stopped, or a
                                 quantity the run does not track) are NaN in every entry point */
    double loop_ms;           /* out: device time of the iteration loop (CUDA events) */
    int run_iterations;       /* out: iterations executed (max over lanes) */
} prgpu_result;

/* One-shot run: allocate, iterate on the device (no per-iteration host sync),
 * copy results, free. */
PRGPU_API int prgpu_pagerank(prgpu_graph* g, const prgpu_params* p, prgpu_result* out);

/* Damping sweep as one power series: the same K lanes and results as
 * prgpu_pagerank (iterations, converged, final_err, err_trace L1/L2/LInf,
 * ranks), computed from ONE alpha = 1 chain y_t = M^t y_0 and per-lane
 * weighted sums, since the reference's iterates are exactly
 * r_t = alpha^t y_t + (1 - alpha) sum_{j<t} alpha^j y_j and
 * r_t - r_{t-1} = alpha^t (y_t - y_{t-1}).  One pull per iteration of the
 * slowest lane instead of one per lane-iteration.  ref_ranks unsupported. */
PRGPU_API int prgpu_pagerank_series(prgpu_graph* g, const prgpu_params* p, prgpu_result* out);

/* Per-iteration observer (pagerank.hpp:51-52,98): called after every
 * iteration of lane `lane` with its ranks (original ids) and error.  This
 * path syncs once per iteration and is meant for tests. */
typedef void (*prgpu_observer_fn)(int iteration, int lane, const double* ranks, uint64_t n,
                                  double err, void* user);
PRGPU_API int prgpu_pagerank_observed(prgpu_graph* g, const prgpu_params* p, prgpu_result* out,
                            prgpu_observer_fn fn, void* user);

/* Reusable device session for repeated runs (bench, sweeps): state and the
 * CUDA graph are built once; each run re-initialises ranks on the device. */
PRGPU_API int prgpu_session_create(prgpu_graph* g, const prgpu_params* p, prgpu_session** out);
PRGPU_API int prgpu_session_run(prgpu_session* s, double* loop_ms);
PRGPU_API int prgpu_session_results(prgpu_session* s, prgpu_result* out);
/* Device time of one iteration's pull kernels (the hub-chunk + packed pair,
 * or the single kernel), in ms per iteration: a host-driven run of at most
 * `launches` iterations that launches only the kernels of the lane mode the
 * CUDA graph would run, one CUDA event pair per iteration on the session
 * stream.  x iterations it is at most the graph loop's time. */
PRGPU_API int prgpu_session_time_pull(prgpu_session* s, int launches, double* ms_per_iteration);
/* The last run's per-iteration device time of the pull kernels measured
 * inside the CUDA graph (%globaltimer: the iteration's earliest CTA start to
 * its finalizing CTA's end), ms; *filled = iterations written (<= cap).
 * Single-GPU sessions. */
PRGPU_API int prgpu_session_kernel_times(prgpu_session* s, double* ms_per_iteration, int cap, int* filled);
PRGPU_API void prgpu_session_free(prgpu_session* s);

/* ---- multi-GPU: 1D partition -----------------------------
 * One process per GPU.  Each rank owns a contiguous, cost-balanced range of
 * engine rows (hub rows are never split across ranks) and therefore a
 * contiguous range of source ids.  Per iteration:
 *   prgpu_part_step      local pull over the rank's rows; its new
 *                        contributions land in contrib[parity_out] rows
 *                        [src_begin, src_end) and its partial sums in
 *                        rank_partials[rank]
 *   (caller)             all-gather: every rank's contribution rows and
 *                        partial vector into every rank's buffers (NCCL)
 *   prgpu_part_finalize  reduce the partial vectors in rank order (identical
 *                        on every rank), decide convergence, next teleport
 * Buffers may be supplied by the caller (e.g. torch tensors used by NCCL). */
typedef struct {
    uint32_t row_begin, row_end;   /* engine rows owned */
    uint64_t src_begin, src_end;   /* source ids owned (contiguous) */
    uint32_t task_begin, task_end; /* warp tasks run by the rank */
} prgpu_partition;

typedef struct {
    double* contrib[2];         /* device: contribution buffers, parity 0/1 */
    uint32_t stride;            /* doubles per source row (K padded to 32 B) */
    uint64_t nsrc;              /* source rows per buffer */
    double* rank_partials;      /* device: [nranks][partials_per_rank] */
    uint32_t partials_per_rank;
} prgpu_exchange;

/* Sizes of the buffers a partition session needs (doubles). */
PRGPU_API int prgpu_part_buffer_sizes(prgpu_graph* g, const prgpu_params* p, int nranks,
                                      uint64_t* contrib_doubles, uint64_t* partial_doubles);
/* ext_contrib (optional, device, contrib_doubles) and ext_rank_partials
 * (optional, device, partial_doubles) let the caller own the exchanged memory. */
PRGPU_API int prgpu_part_create(prgpu_graph* g, const prgpu_params* p, int rank, int nranks,
                                double* ext_contrib, double* ext_rank_partials, prgpu_session** out);
PRGPU_API int prgpu_part_plan(prgpu_session* s, prgpu_partition* parts /* [nranks] */);
PRGPU_API int prgpu_part_exchange(prgpu_session* s, prgpu_exchange* ex);
/* Work is enqueued on `stream` (a cudaStream_t; NULL = the session's own). */
PRGPU_API int prgpu_part_set_stream(prgpu_session* s, void* stream);
PRGPU_API int prgpu_part_init(prgpu_session* s);
PRGPU_API int prgpu_part_step(prgpu_session* s, int* parity_out);
PRGPU_API int prgpu_part_finalize(prgpu_session* s);
/* Synchronises the stream; any lane still iterating? */
PRGPU_API int prgpu_part_active(prgpu_session* s, int* any_active);
/* Final ranks of caller lane `lane` for this rank's engine rows [row_begin, row_end). */
PRGPU_API int prgpu_part_local_ranks(prgpu_session* s, int lane, double* out);
/* The same for every lane at once into DEVICE memory, out[lane * ld + i] for
 * row row_begin + i, enqueued on the session's stream (no host sync): for a
 * device-side gather of the ranks across the job. */
PRGPU_API int prgpu_part_local_ranks_device(prgpu_session* s, double* dev_out, uint64_t ld);
/* Fused exchange over peer memory (NVLink / NVSwitch), instead of the
 * caller moving buffers between steps: the peers' contribution buffers,
 * rank-partials buffers (sized 2 x prgpu_part_buffer_sizes' partials: one
 * block per iteration parity) and arrival counters, as device pointers valid
 * in this process (CUDA IPC), `npeers` = nranks - 1 in rank order skipping
 * this rank; `arrive` is this rank's own counter (peers' pointers to it are
 * their peer_arrive).  The pull kernel then stores each contribution row and
 * the rank's partials straight into every peer's buffers and signals arrival;
 * the finalize kernel waits for all ranks.  After prgpu_part_init (and a
 * host barrier across ranks), prgpu_part_launch enqueues the whole loop as
 * one CUDA graph; host-driven prgpu_part_step/_finalize also work.
 * The session must have been created by prgpu_part_create with BOTH
 * ext_contrib and ext_rank_partials (the latter 2 x partial_doubles): those
 * are the buffers the peers map; PRGPU_EINVAL otherwise. */
PRGPU_API int prgpu_part_set_peers(prgpu_session* s, int npeers, double* const* peer_contrib,
                                   double* const* peer_partials, unsigned int* const* peer_arrive,
                                   unsigned int* arrive);
PRGPU_API int prgpu_part_launch(prgpu_session* s);
/* Shard graphs: the needed-only exchange mask is built from every rank's
 * rows, which no rank holds.  prgpu_part_need_local fills dev_bits (device,
 * ceil(nsrc/4)*4 bytes, 4-byte aligned; nsrc = vertices with out-degree > 0)
 * with this rank's bit for every source its rows gather; sum (= OR: the bits
 * are disjoint) the ranks' buffers, e.g. one all-reduce, and hand the result
 * to prgpu_part_set_need before prgpu_part_set_peers.  Without it a shard's
 * fused exchange stores every row into every peer.  At most 8 ranks. */
PRGPU_API int prgpu_part_need_local(prgpu_session* s, uint8_t* dev_bits);
PRGPU_API int prgpu_part_set_need(prgpu_session* s, const uint8_t* dev_bits);
/* Fused exchange volume: contribution rows this rank stores into its peers
 * per iteration while every lane is live (rows of *row_doubles doubles). */
PRGPU_API int prgpu_part_sent_rows(prgpu_session* s, uint64_t* rows, uint32_t* row_doubles);
/* A fused partition deals its work round-robin (prgpu_part_set_peers; the
 * rank's rows are then not one range): *dealt = 1, and every lane's final
 * value of the rows this rank owns is written at its ENGINE row into
 * dev_out[lane * ld + row] (ld >= vertex_count; other entries untouched, so
 * a sum over ranks of zero-initialised buffers gives the whole vector). */
PRGPU_API int prgpu_part_owned_ranks_device(prgpu_session* s, double* dev_out, uint64_t ld, int* dealt);
/* CUDA IPC for the fused exchange's buffers (any pointer inside a device
 * allocation): export a 64-byte handle + offset; open it in another process
 * of the same node (peer access enabled); close with the pointer open gave. */
PRGPU_API int prgpu_ipc_export(const void* dev_ptr, void* handle64, uint64_t* offset);
PRGPU_API int prgpu_ipc_open(const void* handle64, uint64_t offset, int device, void** dev_ptr);
PRGPU_API int prgpu_ipc_close(void* dev_ptr, uint64_t offset);
/* Engine row -> caller vertex id, [n]. */
PRGPU_API int prgpu_graph_permutation(const prgpu_graph* g, uint32_t* old_of_new);

/* ---- norms (replaces error_norm, norms.hpp:48-78) ----------------------- */
PRGPU_API int prgpu_error_norm(int norm, const double* r, const double* s, uint64_t n, int device,
                     double* out);

/* ---- misc ---------------------------------------------------------------- */
PRGPU_API const char* prgpu_last_error(void);
PRGPU_API const char* prgpu_version(void);
/* Number of pull-kernel launches (and other kernels) this process issued. */
PRGPU_API uint64_t prgpu_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
