// capi.cu — extern "C" boundary of libprgpu.so (include/prgpu.h).
// No exception crosses it: every entry point returns a PRGPU_* status and
// leaves a thread-local message for prgpu_last_error().
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "common.cuh"
#include "mtx.h"

#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

namespace prgpu {
std::atomic<uint64_t> g_launches{0};

void pool_init() {
    static std::once_flag once[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::call_once(once[dev & 63], [dev] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            // memory freed back to the pool stays mapped up to this much, so a
            // caller solving graph after graph (the e2e path: C5 maps ~60 GB
            // per build + solve) does not re-map physical memory every call;
            // PRGPU_POOL_KEEP_GB overrides (0: release everything at sync)
            uint64_t keep = kPoolKeepBytes;
            size_t fr = 0, total = 0;
            if (cudaMemGetInfo(&fr, &total) == cudaSuccess) keep = std::max<uint64_t>(keep, total / 2);
            if (const char* k = std::getenv("PRGPU_POOL_KEEP_GB")) keep = (uint64_t)std::atoll(k) << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
    });
}

std::unique_ptr<prgpu_graph> graph_build_device(uint32_t, const uint32_t*, uint64_t, int, cudaStream_t);
std::unique_ptr<prgpu_graph> graph_build_host(uint32_t, const uint32_t*, uint64_t, int, cudaStream_t);
std::unique_ptr<prgpu_graph> graph_from_csr(uint32_t, const uint64_t*, const uint32_t*,
                                            const uint32_t*, int, cudaStream_t);
std::unique_ptr<prgpu_graph> graph_generate_rmat(uint32_t, uint32_t, double, double, double,
                                                 uint64_t, int, cudaStream_t);
std::unique_ptr<prgpu_graph> graph_generate_grid(uint32_t, double, double, uint64_t, int,
                                                 cudaStream_t);
std::unique_ptr<prgpu_graph> graph_generate_rmat_shard(uint32_t, uint32_t, double, double, double, uint64_t, int,
                                                       int, int, cudaStream_t);
void graph_download(const prgpu_graph*, uint64_t*, uint32_t*, uint32_t*, uint32_t*, cudaStream_t);
prgpu_session* session_create(prgpu_graph*, const prgpu_params*, bool, int, int, double*, double*);
void part_sizes(prgpu_graph*, const prgpu_params*, int, uint64_t*, uint64_t*);
uint64_t graph_device_bytes(const prgpu_graph*);
void part_need_local(prgpu_session*, uint8_t*);
int session_kernel_times(prgpu_session*, double*, int);
void part_set_need(prgpu_session*, const uint8_t*);
uint64_t session_device_bytes(const prgpu_session*);
void part_exchange(prgpu_session*, prgpu_exchange*);
int part_step(prgpu_session*);
void part_finalize(prgpu_session*);
void part_local_ranks(prgpu_session*, int, double*);
void part_local_ranks_device(prgpu_session*, double*, uint64_t);
void part_set_peers(prgpu_session*, int, double* const*, double* const*, unsigned int* const*, unsigned int*);
void part_launch(prgpu_session*);
void session_init(prgpu_session*);
int read_any_active(prgpu_session*);
void part_plan_copy(prgpu_session*, prgpu_partition*);
void part_set_stream(prgpu_session*, void*);
void graph_permutation(const prgpu_graph*, uint32_t*);
void part_sent_rows(prgpu_session*, uint64_t*, uint32_t*);
void pagerank_series(prgpu_graph*, const prgpu_params*, prgpu_result*);
void part_owned_ranks_device(prgpu_session*, double*, uint64_t, int*);

uint64_t graph_rows(const prgpu_graph*, const uint32_t*, uint32_t, uint64_t*, uint32_t*, uint64_t, cudaStream_t);
void session_destroy(prgpu_session*);
using SessionPtr = std::unique_ptr<prgpu_session, void (*)(prgpu_session*)>;
double session_run(prgpu_session*);
void session_results(prgpu_session*, prgpu_result*);
void session_solve(prgpu_session*, prgpu_result*);
void session_observed(prgpu_session*, prgpu_result*, prgpu_observer_fn, void*);
double session_time_pull(prgpu_session*, int);
double error_norm_device(int, const double*, const double*, uint64_t, int);
} // namespace prgpu

namespace {
thread_local std::string t_last_error;

template <typename F>
int guarded(F&& f) {
    try {
        t_last_error.clear();
        f();
        return PRGPU_OK;
    } catch (const prgpu::Error& e) {
        t_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        t_last_error = "host allocation failed";
        return PRGPU_ENOMEM;
    } catch (const std::exception& e) {
        t_last_error = e.what();
        return PRGPU_ECUDA;
    } catch (...) {
        t_last_error = "unknown error";
        return PRGPU_ECUDA;
    }
}

void check_device(int device) {
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        prgpu::fail(PRGPU_ECUDA, "no CUDA device available (libprgpu has no CPU fallback)");
    if (device < 0 || device >= count)
        prgpu::fail(PRGPU_EINVAL, "device index out of range: " + std::to_string(device));
}

template <typename Make>
int make_graph(int device, prgpu_graph** out, Make&& make) {
    return guarded([&] {
        if (!out) prgpu::fail(PRGPU_EINVAL, "null output pointer");
        *out = nullptr;
        check_device(device);
        prgpu::DeviceGuard dg(device);
        prgpu::Stream st;
        prgpu::AllocScope scope(st);
        std::unique_ptr<prgpu_graph> g = make((cudaStream_t)st);
        PRGPU_CUDA(cudaStreamSynchronize(st));
        *out = g.release();
    });
}
} // namespace

extern "C" {

int prgpu_graph_build(uint32_t n, const uint32_t* pairs, uint64_t m, int device, prgpu_graph** out) {
    if (m && !pairs) { t_last_error = "null edge_pairs"; return PRGPU_EINVAL; }
    return make_graph(device, out, [&](cudaStream_t st) {
        return prgpu::graph_build_host(n, pairs, m, device, st);
    });
}

int prgpu_graph_build_device(uint32_t n, const uint32_t* d_pairs, uint64_t m, int device,
                             prgpu_graph** out) {
    if (m && !d_pairs) { t_last_error = "null edge_pairs"; return PRGPU_EINVAL; }
    return make_graph(device, out, [&](cudaStream_t st) {
        return prgpu::graph_build_device(n, d_pairs, m, device, st);
    });
}

int prgpu_graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* nbr, const uint32_t* deg,
                         int device, prgpu_graph** out) {
    if (!off || !deg || (n && off[n] && !nbr)) { t_last_error = "null CSR array"; return PRGPU_EINVAL; }
    return make_graph(device, out, [&](cudaStream_t st) {
        return prgpu::graph_from_csr(n, off, nbr, deg, device, st);
    });
}

int prgpu_graph_generate_rmat(uint32_t scale, uint32_t ef, double a, double b, double c,
                              uint64_t seed, int device, prgpu_graph** out) {
    return make_graph(device, out, [&](cudaStream_t st) {
        return prgpu::graph_generate_rmat(scale, ef, a, b, c, seed, device, st);
    });
}

int prgpu_graph_generate_rmat_shard(uint32_t scale, uint32_t ef, double a, double b, double c, uint64_t seed,
                                    int rank, int nranks, int device, prgpu_graph** out) {
    return make_graph(device, out, [&](cudaStream_t st) {
        return prgpu::graph_generate_rmat_shard(scale, ef, a, b, c, seed, rank, nranks, device, st);
    });
}

int prgpu_graph_shard_info(const prgpu_graph* g, int* rank, int* nranks, uint32_t* row_begin, uint32_t* row_end,
                           uint64_t* local_edges) {
    return guarded([&] {
        if (!g) prgpu::fail(PRGPU_EINVAL, "null graph");
        const bool sh = g->shard_n > 1;
        if (rank) *rank = sh ? g->shard_rank : 0;
        if (nranks) *nranks = sh ? g->shard_n : 1;
        if (row_begin) *row_begin = sh ? g->shard_rows[g->shard_rank] : 0u;
        if (row_end) *row_end = sh ? g->shard_rows[g->shard_rank + 1] : g->n;
        if (local_edges) *local_edges = g->local_e;
    });
}

int prgpu_device_bytes(const prgpu_graph* g, const prgpu_session* s, uint64_t* graph_bytes,
                       uint64_t* session_bytes) {
    return guarded([&] {
        if (graph_bytes) *graph_bytes = g ? prgpu::graph_device_bytes(g) : 0;
        if (session_bytes) *session_bytes = s ? prgpu::session_device_bytes(s) : 0;
    });
}

int prgpu_graph_generate_grid(uint32_t side, double p, double lr, uint64_t seed, int device,
                              prgpu_graph** out) {
    return make_graph(device, out, [&](cudaStream_t st) {
        return prgpu::graph_generate_grid(side, p, lr, seed, device, st);
    });
}

int prgpu_graph_get_info(const prgpu_graph* g, prgpu_graph_info* info) {
    return guarded([&] {
        if (!g || !info) prgpu::fail(PRGPU_EINVAL, "null argument");
        info->vertex_count = g->n;
        info->edge_count = g->e;
        info->dangling_count = g->ndangling;
        info->max_in_degree = g->max_in_degree;
        info->hub_rows = g->hub_end;
        info->warp_rows = g->warp_end - g->hub_end;
        info->thread_rows = g->nonempty_end - g->warp_end;
        info->empty_rows = g->n - g->nonempty_end;
        info->device = g->device;
    });
}

int prgpu_graph_download(const prgpu_graph* g, uint64_t* off, uint32_t* nbr, uint32_t* deg,
                         uint32_t* dang) {
    return guarded([&] {
        if (!g) prgpu::fail(PRGPU_EINVAL, "null graph");
        prgpu::DeviceGuard dg(g->device);
        prgpu::Stream st;
        prgpu::AllocScope scope(st);
        prgpu::graph_download(g, off, nbr, deg, dang, st);
    });
}

int prgpu_graph_rows(const prgpu_graph* g, const uint32_t* rows, uint32_t nrows, uint64_t* off,
                     uint32_t* nbr, uint64_t cap, uint64_t* total) {
    return guarded([&] {
        if (!g || (nrows && (!rows || !off))) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::DeviceGuard dg(g->device);
        prgpu::Stream st;
        prgpu::AllocScope scope(st);
        const uint64_t t = prgpu::graph_rows(g, rows, nrows, off, nbr, cap, st);
        if (total) *total = t;
    });
}

// ---- MatrixMarket ingest (graph.hpp:111-199, 238-251) ----------------------------
namespace {
// the file's bytes, mapped read-only (empty files are an empty view)
struct Mapped {
    const char* p = nullptr;
    uint64_t len = 0;
    int fd = -1;
    explicit Mapped(const char* path) {
        fd = ::open(path, O_RDONLY);
        if (fd < 0) prgpu::fail(PRGPU_EIO, std::string("cannot open graph file: ") + path);
        struct stat st {};
        if (::fstat(fd, &st) != 0) prgpu::fail(PRGPU_EIO, std::string("cannot open graph file: ") + path);
        len = (uint64_t)st.st_size;
        if (len) {
            void* m = ::mmap(nullptr, len, PROT_READ, MAP_PRIVATE, fd, 0);
            if (m == MAP_FAILED) prgpu::fail(PRGPU_EIO, std::string("cannot read graph file: ") + path);
            ::madvise(m, len, MADV_SEQUENTIAL);
            p = static_cast<const char*>(m);
        }
    }
    ~Mapped() {
        if (p) ::munmap(const_cast<char*>(p), len);
        if (fd >= 0) ::close(fd);
    }
};

// parse errors: PRGPU_EPARSE, message "line L: what" (MtxParseError::what),
// prefixed with "<path>: " for files (load_matrix_market, graph.hpp:243-246)
prgpu::MtxResult parse_or_fail(const char* text, uint64_t len, int threads, const char* path,
                               uint64_t* err_line) {
    prgpu::MtxResult r = prgpu::mtx_parse(text, len, threads);
    if (r.err_line || !r.err_what.empty()) {
        if (err_line) *err_line = r.err_line;
        std::string msg = "line " + std::to_string(r.err_line) + ": " + r.err_what;
        if (path) msg = std::string(path) + ": " + msg;
        std::free(r.pairs);
        prgpu::fail(r.err_line ? PRGPU_EPARSE : PRGPU_ENOMEM, msg);
    }
    return r;
}
} // namespace

int prgpu_mtx_parse(const char* text, uint64_t len, int threads, uint32_t* n, uint32_t** pairs, uint64_t* m,
                    uint64_t* err_line) {
    return guarded([&] {
        if ((!text && len) || !n || !pairs || !m) prgpu::fail(PRGPU_EINVAL, "null argument");
        if (err_line) *err_line = 0;
        prgpu::MtxResult r = parse_or_fail(text, len, threads, nullptr, err_line);
        *n = r.n;
        *m = r.m;
        *pairs = r.pairs;
    });
}

int prgpu_mtx_load(const char* path, int threads, uint32_t* n, uint32_t** pairs, uint64_t* m,
                   uint64_t* err_line) {
    return guarded([&] {
        if (!path || !n || !pairs || !m) prgpu::fail(PRGPU_EINVAL, "null argument");
        if (err_line) *err_line = 0;
        Mapped f(path);
        prgpu::MtxResult r = parse_or_fail(f.p, f.len, threads, path, err_line);
        *n = r.n;
        *m = r.m;
        *pairs = r.pairs;
    });
}

void prgpu_pairs_free(uint32_t* pairs) { std::free(pairs); }

int prgpu_graph_load_mtx(const char* path, int threads, int device, prgpu_graph** out, uint64_t* err_line) {
    if (!path) { t_last_error = "null path"; return PRGPU_EINVAL; }
    if (err_line) *err_line = 0;
    return make_graph(device, out, [&](cudaStream_t st) {
        Mapped f(path);
        prgpu::MtxResult r = parse_or_fail(f.p, f.len, threads, path, err_line);
        std::unique_ptr<uint32_t, void (*)(void*)> keep(r.pairs, std::free);
        return prgpu::graph_build_host(r.n, r.pairs, r.m, device, st);
    });
}

void prgpu_graph_free(prgpu_graph* g) {
    if (!g) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(g->device);
    {
        // no call may still use the graph: its buffers go back to the pool
        // ordered after everything already queued on the device
        cudaDeviceSynchronize();
        cudaStream_t st = nullptr;
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        {
            prgpu::AllocScope scope(st);
            delete g;
        }
        cudaStreamDestroy(st);
    }
    cudaSetDevice(prev);
}

int prgpu_pagerank(prgpu_graph* g, const prgpu_params* p, prgpu_result* out) {
    return guarded([&] {
        if (!out) prgpu::fail(PRGPU_EINVAL, "null result");
        if (g) check_device(g->device);
        prgpu::SessionPtr s(prgpu::session_create(g, p, true, 0, 0, nullptr, nullptr), prgpu::session_destroy);
        prgpu::session_solve(s.get(), out);
    });
}

int prgpu_pagerank_series(prgpu_graph* g, const prgpu_params* p, prgpu_result* out) {
    return guarded([&] {
        if (!out) prgpu::fail(PRGPU_EINVAL, "null result");
        if (g) check_device(g->device);
        prgpu::pagerank_series(g, p, out);
    });
}

int prgpu_pagerank_observed(prgpu_graph* g, const prgpu_params* p, prgpu_result* out,
                            prgpu_observer_fn fn, void* user) {
    return guarded([&] {
        if (!out) prgpu::fail(PRGPU_EINVAL, "null result");
        if (g) check_device(g->device);
        prgpu::SessionPtr s(prgpu::session_create(g, p, false, 0, 0, nullptr, nullptr), prgpu::session_destroy);
        prgpu::session_observed(s.get(), out, fn, user);
    });
}

int prgpu_session_create(prgpu_graph* g, const prgpu_params* p, prgpu_session** out) {
    return guarded([&] {
        if (!out) prgpu::fail(PRGPU_EINVAL, "null output pointer");
        *out = nullptr;
        if (g) check_device(g->device);
        *out = prgpu::session_create(g, p, true, 0, 0, nullptr, nullptr);
    });
}

int prgpu_session_run(prgpu_session* s, double* loop_ms) {
    return guarded([&] {
        if (!s) prgpu::fail(PRGPU_EINVAL, "null session");
        const double ms = prgpu::session_run(s);
        if (loop_ms) *loop_ms = ms;
    });
}

int prgpu_session_results(prgpu_session* s, prgpu_result* out) {
    return guarded([&] {
        if (!s || !out) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::session_results(s, out);
    });
}

int prgpu_session_time_pull(prgpu_session* s, int launches, double* ms) {
    return guarded([&] {
        if (!s || !ms || launches < 1) prgpu::fail(PRGPU_EINVAL, "bad argument");
        *ms = prgpu::session_time_pull(s, launches);
    });
}

void prgpu_session_free(prgpu_session* s) { prgpu::session_destroy(s); }

int prgpu_error_norm(int norm, const double* r, const double* s, uint64_t n, int device,
                     double* out) {
    return guarded([&] {
        if (!out || (n && (!r || !s))) prgpu::fail(PRGPU_EINVAL, "null argument");
        check_device(device);
        *out = prgpu::error_norm_device(norm, r, s, n, device);
    });
}

int prgpu_part_buffer_sizes(prgpu_graph* g, const prgpu_params* p, int nranks, uint64_t* contrib,
                            uint64_t* partials) {
    return guarded([&] {
        if (!contrib || !partials) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_sizes(g, p, nranks, contrib, partials);
    });
}

int prgpu_part_create(prgpu_graph* g, const prgpu_params* p, int rank, int nranks, double* ext_contrib,
                      double* ext_rank_partials, prgpu_session** out) {
    return guarded([&] {
        if (!out) prgpu::fail(PRGPU_EINVAL, "null output pointer");
        *out = nullptr;
        if (nranks < 1) prgpu::fail(PRGPU_EINVAL, "partition: nranks must be >= 1");
        if (g) check_device(g->device);
        *out = prgpu::session_create(g, p, false, rank, nranks, ext_contrib, ext_rank_partials);
    });
}

int prgpu_part_plan(prgpu_session* s, prgpu_partition* parts) {
    return guarded([&] {
        if (!s || !parts) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_plan_copy(s, parts);
    });
}

int prgpu_part_exchange(prgpu_session* s, prgpu_exchange* ex) {
    return guarded([&] {
        if (!s || !ex) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_exchange(s, ex);
    });
}

int prgpu_part_set_stream(prgpu_session* s, void* stream) {
    return guarded([&] {
        if (!s) prgpu::fail(PRGPU_EINVAL, "null session");
        prgpu::part_set_stream(s, stream);
    });
}

int prgpu_part_init(prgpu_session* s) {
    return guarded([&] {
        if (!s) prgpu::fail(PRGPU_EINVAL, "null session");
        prgpu::session_init(s);
    });
}

int prgpu_part_step(prgpu_session* s, int* parity_out) {
    return guarded([&] {
        if (!s) prgpu::fail(PRGPU_EINVAL, "null session");
        const int par = prgpu::part_step(s);
        if (parity_out) *parity_out = par;
    });
}

int prgpu_part_finalize(prgpu_session* s) {
    return guarded([&] {
        if (!s) prgpu::fail(PRGPU_EINVAL, "null session");
        prgpu::part_finalize(s);
    });
}

int prgpu_part_active(prgpu_session* s, int* any) {
    return guarded([&] {
        if (!s || !any) prgpu::fail(PRGPU_EINVAL, "null argument");
        *any = prgpu::read_any_active(s);
    });
}

int prgpu_part_local_ranks(prgpu_session* s, int lane, double* out) {
    return guarded([&] {
        if (!s || !out) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_local_ranks(s, lane, out);
    });
}

int prgpu_part_local_ranks_device(prgpu_session* s, double* dev_out, uint64_t ld) {
    return guarded([&] {
        if (!s || !dev_out) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_local_ranks_device(s, dev_out, ld);
    });
}

int prgpu_part_set_peers(prgpu_session* s, int npeers, double* const* peer_contrib, double* const* peer_partials,
                         unsigned int* const* peer_arrive, unsigned int* arrive) {
    return guarded([&] {
        if (!s || (npeers > 0 && (!peer_contrib || !peer_partials || !peer_arrive)))
            prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_set_peers(s, npeers, peer_contrib, peer_partials, peer_arrive, arrive);
    });
}

int prgpu_session_kernel_times(prgpu_session* s, double* ms_per_iteration, int cap, int* filled) {
    return guarded([&] {
        if (!s || !ms_per_iteration || !filled) prgpu::fail(PRGPU_EINVAL, "null argument");
        *filled = prgpu::session_kernel_times(s, ms_per_iteration, cap);
    });
}

int prgpu_part_need_local(prgpu_session* s, uint8_t* dev_bits) {
    return guarded([&] {
        if (!s || !dev_bits) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_need_local(s, dev_bits);
    });
}

int prgpu_part_set_need(prgpu_session* s, const uint8_t* dev_bits) {
    return guarded([&] {
        if (!s || !dev_bits) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_set_need(s, dev_bits);
    });
}

int prgpu_part_sent_rows(prgpu_session* s, uint64_t* rows, uint32_t* row_doubles) {
    return guarded([&] {
        if (!s || !rows || !row_doubles) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_sent_rows(s, rows, row_doubles);
    });
}

int prgpu_part_owned_ranks_device(prgpu_session* s, double* dev_out, uint64_t ld, int* dealt) {
    return guarded([&] {
        if (!s || !dealt) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::part_owned_ranks_device(s, dev_out, ld, dealt);
    });
}

int prgpu_part_launch(prgpu_session* s) {
    return guarded([&] {
        if (!s) prgpu::fail(PRGPU_EINVAL, "null session");
        prgpu::part_launch(s);
    });
}

int prgpu_ipc_export(const void* dev_ptr, void* handle64, uint64_t* offset) {
    return guarded([&] {
        if (!dev_ptr || !handle64 || !offset) prgpu::fail(PRGPU_EINVAL, "null argument");
        // the allocation's base through the driver entry point (no libcuda link)
        using AddrRange = int (*)(unsigned long long*, size_t*, unsigned long long);
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        PRGPU_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) prgpu::fail(PRGPU_ECUDA, "cuMemGetAddressRange unavailable");
        unsigned long long base = 0;
        size_t size = 0;
        if (reinterpret_cast<AddrRange>(fn)(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0)
            prgpu::fail(PRGPU_EINVAL, "ipc_export: not a device allocation");
        cudaIpcMemHandle_t h;
        PRGPU_CUDA(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
        std::memcpy(handle64, &h, sizeof(h));
        *offset = (uint64_t)((uintptr_t)dev_ptr - base);
    });
}

int prgpu_ipc_open(const void* handle64, uint64_t offset, int device, void** dev_ptr) {
    return guarded([&] {
        if (!handle64 || !dev_ptr) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::DeviceGuard dg(device);
        cudaIpcMemHandle_t h;
        std::memcpy(&h, handle64, sizeof(h));
        void* base = nullptr;
        PRGPU_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        *dev_ptr = static_cast<char*>(base) + offset;
    });
}

int prgpu_ipc_close(void* dev_ptr, uint64_t offset) {
    return guarded([&] {
        if (!dev_ptr) prgpu::fail(PRGPU_EINVAL, "null argument");
        PRGPU_CUDA(cudaIpcCloseMemHandle(static_cast<char*>(dev_ptr) - offset));
    });
}

int prgpu_graph_permutation(const prgpu_graph* g, uint32_t* old_of_new) {
    return guarded([&] {
        if (!g || !old_of_new) prgpu::fail(PRGPU_EINVAL, "null argument");
        prgpu::graph_permutation(g, old_of_new);
    });
}

const char* prgpu_last_error(void) { return t_last_error.c_str(); }
const char* prgpu_version(void) { return "prgpu 0.1.0 (sm_100a)"; }
uint64_t prgpu_kernel_launch_count(void) { return prgpu::g_launches.load(); }

} // extern "C"
