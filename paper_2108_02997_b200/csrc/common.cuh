// common.cuh — shared internals of libprgpu.so (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/prgpu.h"

namespace prgpu {

// Errors thrown inside the library and turned into status codes at the C ABI.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

inline void check_cuda(cudaError_t e, const char* what, const char* file, int line) {
    if (e == cudaSuccess) return;
    const int code = (e == cudaErrorMemoryAllocation) ? PRGPU_ENOMEM : PRGPU_ECUDA;
    fail(code, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                   std::to_string(line) + ")");
}

#define PRGPU_CUDA(call) ::prgpu::check_cuda((call), #call, __FILE__, __LINE__)
#define PRGPU_LAUNCHED(name)                                                          \
    do {                                                                              \
        ::prgpu::g_launches.fetch_add(1, std::memory_order_relaxed);                  \
        ::prgpu::check_cuda(cudaGetLastError(), name, __FILE__, __LINE__);            \
    } while (0)

extern std::atomic<uint64_t> g_launches;

// Host-side phase timing for tuning (PRGPU_TIMING_LOG=1): syncs the stream at
// each mark and prints the time since the previous one.  Off by default.
struct PhaseLog {
    bool on;
    cudaStream_t st;
    std::chrono::steady_clock::time_point t;
    const char* scope;
    PhaseLog(const char* sc, cudaStream_t s)
        : on(std::getenv("PRGPU_TIMING_LOG") != nullptr), st(s), t(std::chrono::steady_clock::now()),
          scope(sc) {}
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[%s] %-22s %8.3f ms\n", scope, what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// Stream-ordered allocation.  Inside an AllocScope, DevBufs come from the
// device's default memory pool (cudaMallocAsync on the scope's stream) and are
// returned to it stream-ordered, so the many temporaries of a graph build and
// a session cost no cudaMalloc/cudaFree round trips; the pool keeps up to
// kPoolKeepBytes cached across calls.  Outside a scope: plain cudaMalloc/Free.
inline thread_local cudaStream_t t_alloc_stream = nullptr;
constexpr uint64_t kPoolKeepBytes = 8ull << 30;
void pool_init(); // current device, once

struct AllocScope {
    cudaStream_t prev;
    explicit AllocScope(cudaStream_t s) : prev(t_alloc_stream) {
        pool_init();
        t_alloc_stream = s;
    }
    ~AllocScope() { t_alloc_stream = prev; }
    AllocScope(const AllocScope&) = delete;
    AllocScope& operator=(const AllocScope&) = delete;
};

// RAII device buffer.
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    bool pooled = false;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), pooled(o.pooled) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            reset();
            p = o.p; n = o.n; pooled = o.pooled;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { reset(); }
    void alloc(size_t count) {
        reset();
        n = count;
        if (!count) return;
        if (t_alloc_stream) {
            PRGPU_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), t_alloc_stream));
            pooled = true;
        } else {
            PRGPU_CUDA(cudaMalloc(&p, count * sizeof(T)));
            pooled = false;
        }
    }
    void reset() {
        if (p) {
            if (pooled && t_alloc_stream) cudaFreeAsync(p, t_alloc_stream);
            else cudaFree(p); // also valid for pool memory (synchronous)
        }
        p = nullptr;
        n = 0;
    }
    void swap(DevBuf& o) noexcept {
        std::swap(p, o.p); std::swap(n, o.n); std::swap(pooled, o.pooled);
    }
    T* release() { T* q = p; p = nullptr; n = 0; return q; }
    size_t bytes() const { return n * sizeof(T); }
};

struct DeviceGuard {
    int prev = 0;
    explicit DeviceGuard(int dev) {
        PRGPU_CUDA(cudaGetDevice(&prev));
        if (dev != prev) PRGPU_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() { cudaSetDevice(prev); }
};

struct Stream {
    cudaStream_t s = nullptr;
    Stream() { PRGPU_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~Stream() { if (s) cudaStreamDestroy(s); }
    Stream(const Stream&) = delete;
    Stream& operator=(const Stream&) = delete;
    operator cudaStream_t() const { return s; }
};

struct Event {
    cudaEvent_t e = nullptr;
    Event() { PRGPU_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
    ~Event() { if (e) cudaEventDestroy(e); }
    Event(const Event&) = delete;
    Event& operator=(const Event&) = delete;
    operator cudaEvent_t() const { return e; }
};

// Pull-kernel degree bins (rows sorted by in-degree descending).
constexpr uint32_t kHubMinDegree = 4096; // > : block per vertex
constexpr uint32_t kWarpMinDegree = 32;  // > : warp per vertex; else lane group

inline uint32_t bits_for(uint64_t n) { // ceil(log2(n)), >= 1
    uint32_t b = 1;
    while ((1ull << b) < n) ++b;
    return b;
}

// Hot/cold source split of the engine CSR (the split pull):
// every row's in-edges partitioned, in their order, into those whose source
// id is < hot (the most-gathered sources: their contributions stay
// L2-resident while only they are gathered) and the rest, as two CSRs over
// the same rows.  An iteration pulls the hot CSR first (row partials), then
// the cold one (adds the partial, epilogue).
struct SourceSplit {
    uint32_t hot = 0;
    uint64_t e_hot = 0, e_cold = 0;
    DevBuf<uint64_t> off_hot, off_cold; // [n+1]
    DevBuf<uint32_t> col_hot, col_cold; // [e_hot + 16], [e_cold + 16]
};

// Segment plan of the hub rows (the segmented pull, DESIGN.md "Segmented hub
// pull").  The source ids are cut into `S` segments — hot segments of
// `seg_src` sources each (their contribution rows fit L2 together with the
// streams), the last segment the cold rest when the table is longer — and
// the in-edges of the rows with in-degree >= T (a prefix of the engine rows,
// hence a prefix of col) are regrouped into pieces (row, segment): wide
// pieces (> win edges) first, then small ones, each class segment-major,
// rows ascending inside a segment, a piece's edges in their row order.  A
// pull walks the pieces in that order, so at any time every warp gathers from
// the same segment; each piece leaves a partial sum in slot row * S + seg,
// and the row's epilogue adds its slots in segment order.  A hot-segment
// piece of fewer than pmin edges is folded into the row's last-segment piece.
struct SegPlan {
    uint32_t seg_src = 0, S = 0, T = 0, win = 0, pmin = 0;
    uint32_t n_rows = 0;    // segmented rows [0, n_rows)
    uint64_t e_seg = 0;     // their edges: col[0, e_seg)
    uint64_t e_wide = 0;    // edges in wide pieces
    uint32_t n_wp = 0, n_sp = 0;
    DevBuf<uint32_t> col;   // [e_seg + 16]
    DevBuf<uint64_t> off;   // [n_wp + n_sp + 1] piece offsets into col (wide pieces first)
    DevBuf<uint32_t> slot;  // [n_wp + n_sp] row * S + seg
    uint64_t bytes() const { return col.bytes() + off.bytes() + slot.bytes(); }
};

} // namespace prgpu

// The device graph: engine layout (relabelled) + the permutation back to the
// caller's ids.  Immutable after construction.
struct prgpu_graph {
    int device = 0;
    uint32_t n = 0;
    uint64_t e = 0;
    uint32_t ndangling = 0;
    uint32_t max_in_degree = 0;
    uint32_t lg = 1; // bits per vertex id in packed edge keys
    // engine CSR, vertices relabelled by in-degree descending (ties: old id)
    prgpu::DevBuf<uint64_t> row_off;    // [n+1]
    prgpu::DevBuf<uint32_t> col;        // [e + 16] source ids (padding for 128-bit loads)
    prgpu::DevBuf<uint32_t> deg;        // [n] out-degree, engine ids
    prgpu::DevBuf<uint2> rowinfo;       // [n] {out-degree, source id or ~0u if dangling}
    prgpu::DevBuf<uint32_t> row_of_src; // [nsrc] engine row of each source id
    uint32_t nsrc = 0;                  // vertices with out-degree > 0
    prgpu::DevBuf<uint32_t> new_of_old; // [n]
    prgpu::DevBuf<uint32_t> old_of_new; // [n]
    uint32_t hub_end = 0, warp_end = 0, nonempty_end = 0;
    bool locality = false; // rows in the caller's order within classes (low-degree graphs)
    uint32_t sort_end[6] = {0, 0, 0, 0, 0, 0}; // rows with in-degree > 512, 256, 128, 64, 32, 8
    // shard graphs (prgpu_graph_generate_rmat_shard, SURVEY 8e set-up): the
    // vertex arrays are global, `col` holds only the in-edges of engine rows
    // [shard_rows[rank], shard_rows[rank + 1]); kernels index it as
    // col - col_base (col_base = row_off[first row]).  shard_n == 0: whole graph.
    int shard_rank = 0, shard_n = 0;
    std::vector<uint32_t> shard_rows; // [shard_n + 1] engine-row boundaries of every rank
    uint64_t col_base = 0;
    uint64_t local_e = 0;             // edges held (== e unless a shard)
    // source splits built on demand by sessions (graph_source_split), by threshold
    std::mutex split_mu;
    std::map<uint32_t, std::unique_ptr<prgpu::SourceSplit>> splits;
    // segment plans built on demand by sessions (graph_seg_plan), by (seg_src, S, T, win)
    std::map<std::array<uint32_t, 5>, std::unique_ptr<prgpu::SegPlan>> seg_plans;
};

namespace prgpu {
// the graph's hot/cold split at threshold `hot` (built on first use, cached)
const SourceSplit& graph_source_split(prgpu_graph* g, uint32_t hot, cudaStream_t st);
// the graph's segment plan (built on first use, cached); null when no row has T in-edges
const SegPlan* graph_seg_plan(prgpu_graph* g, uint32_t seg_src, uint32_t S, uint32_t T, uint32_t win,
                              uint32_t pmin, cudaStream_t st);
} // namespace prgpu
