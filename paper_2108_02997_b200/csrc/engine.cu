// engine.cu — sessions around the pull kernel (pull.cuh): device state, the
// warp-task tables, the CUDA graph (WHILE node around one pull launch per
// iteration), result extraction, and the device error_norm.
//
// Replaces pagerank() (pagerank.hpp:70-108): init (:72-81), the do/while loop
// (:84-99, one pull_kernel launch per iteration, convergence decided on the
// device), and the result (:100-107).  See pull.cuh for the kernel itself.
#include <cub/cub.cuh>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <mutex>
#include <vector>
#include <chrono>
#include <thread>

#include "common.cuh"
#include "pull.cuh"
#include "lane_cfg.cuh"

namespace prgpu {

// ---- init: uniform ranks 1/N (pagerank.hpp:77), first contributions and c0 ----
template <int KS> // contribution row stride (LaneCfg::KS)
__global__ void init_kernel(Params P, uint32_t ndangling) {
    const size_t n = P.n;
    const double r0 = 1.0 / (double)P.n;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x) {
        const uint2 ri = P.rowinfo[v];
        if (v < P.empty_begin && v >= P.rank_lo && v < P.rank_hi) // a shard's own rows only
            for (uint32_t k = 0; k < P.K; ++k) P.rank[0][v * KS + k] = r0;
        if (ri.x) {
            const double cv = __ddiv_rn(r0, (double)ri.x);
            double* c = caddr<KS>(P, 0, ri.y);
#pragma unroll
            for (int k = 0; k < KS; ++k) c[k] = (k < (int)P.K) ? cv : 0.0;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < P.K) {
        LaneState& L = P.lanes[threadIdx.x];
        const double nd = (double)P.n;
        // sum of the initial dangling ranks: ndangling * (1/N), rounded once
        const double dang = __dmul_rn((double)ndangling, r0);
        const double a = L.alpha;
        L.c0 = __dadd_rn(__ddiv_rn(__dsub_rn(1.0, a), nd), __ddiv_rn(__dmul_rn(a, dang), nd));
        L.c0_used = r0;
        L.prev_empty = r0;
        L.active = 1;
        L.iterations = 0;
        L.converged = 0;
        L.final_err = INFINITY;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.gs->iter = 0;
        P.gs->any_active = 1;
        P.gs->counter = 0;
    }
}

// ---- result extraction: out[k][v_orig] = rank[buf(k)][k][new_of_old[v]] --------
__global__ void extract_ranks(Params P, const uint32_t* __restrict__ new_of_old,
                              double* __restrict__ out, int lane_only, int use_current) {
    const size_t n = P.n;
    const int k0 = lane_only >= 0 ? lane_only : 0;
    const int k1 = lane_only >= 0 ? lane_only + 1 : (int)P.K;
    for (int k = k0; k < k1; ++k) {
        const int buf = use_current ? (P.gs->iter & 1) : (P.lanes[k].iterations & 1);
        const double* src = P.rank[buf] + k; // row-major [row][ks]
        const double c0 = P.lanes[k].c0_used; // rows with no in-edges hold c0
        double* dst = out + (size_t)(k - k0) * n;
        for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
             v += (size_t)gridDim.x * blockDim.x) {
            const uint32_t r = new_of_old[v];
            dst[v] = r >= P.empty_begin ? c0 : src[(size_t)r * P.ks];
        }
    }
}

// trace entries no iteration writes (a lane after it stopped, norms an
// instance does not track) read NaN in every entry point (prgpu.h err_trace)
__global__ void fill_f64(double* __restrict__ p, size_t n, double v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = v;
}

__global__ void strided_copy(const double* __restrict__ src, uint32_t stride, double* __restrict__ dst,
                             uint32_t rows) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < rows; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i * stride];
}

struct LaneMap {
    int user_of[16]; // device slot -> caller lane
};

// every lane of rows [row_begin, row_begin + rows) into out[caller lane][i]
__global__ void local_ranks_kernel(Params P, LaneMap map, uint32_t row_begin, uint32_t rows,
                                   double* __restrict__ out, uint64_t ld) {
    const uint64_t total = (uint64_t)rows * P.K;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = (uint32_t)(x / rows), i = (uint32_t)(x - (uint64_t)k * rows);
        const uint32_t r = row_begin + i;
        const LaneState& L = P.lanes[k];
        const double v = r >= P.empty_begin ? L.c0_used : P.rank[L.iterations & 1][(size_t)r * P.ks + k];
        out[(size_t)map.user_of[k] * ld + i] = v;
    }
}

// dealt partitions: every lane's value of the rows this rank owns, at their
// engine row in out[lane][ld] (other rows untouched)
__global__ void owned_ranks_kernel(Params P, LaneMap map, const uint8_t* __restrict__ owner, int me,
                                   double* __restrict__ out, uint64_t ld) {
    const uint64_t total = (uint64_t)P.n * P.K;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total;
         x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t k = (uint32_t)(x / P.n), r = (uint32_t)(x - (uint64_t)k * P.n);
        if (owner[r] != me) continue;
        const LaneState& L = P.lanes[k];
        const double v = r >= P.empty_begin ? L.c0_used : P.rank[L.iterations & 1][(size_t)r * P.ks + k];
        out[(size_t)map.user_of[k] * ld + r] = v;
    }
}

__global__ void scatter_ref(const double* __restrict__ in, const uint32_t* __restrict__ new_of_old,
                            double* __restrict__ out, uint32_t n) {
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x)
        out[new_of_old[v]] = in[v];
}

// ---- warp-task tables ----------------------------------------------------------
// rows [0, n_long): in-degree > WIN, split into ceil(d / EMAX) chunks
__global__ void count_long_rows(const uint64_t* __restrict__ row_off, uint32_t n, uint32_t win,
                                unsigned int* __restrict__ out) {
    unsigned int c = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        c += (row_off[r + 1] - row_off[r]) > win;
    atomicAdd(out, c);
}

__global__ void chunk_counts(const uint64_t* __restrict__ row_off, uint32_t n_long, uint32_t emax,
                             uint64_t* __restrict__ out) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= n_long; r += gridDim.x * blockDim.x)
        out[r] = (r < n_long) ? (row_off[r + 1] - row_off[r] + emax - 1) / emax : 0;
}

__global__ void chunk_fill(const uint64_t* __restrict__ first, uint32_t n_long,
                           uint32_t* __restrict__ chunk_first, uint32_t* __restrict__ chunk_row) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r <= n_long; r += gridDim.x * blockDim.x) {
        chunk_first[r] = (uint32_t)first[r];
        if (r < n_long)
            for (uint64_t c = first[r]; c < first[r + 1]; ++c) chunk_row[c] = r;
    }
}

// packed rows [lo, hi): cost max(d + 2, cmin); prefix / WIN = task id
__global__ void packed_costs(const uint64_t* __restrict__ row_off, uint32_t lo, uint32_t hi,
                             uint32_t cmin, uint64_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; lo + i <= hi; i += gridDim.x * blockDim.x) {
        const uint32_t r = lo + i;
        const uint64_t c = (r < hi) ? row_off[r + 1] - row_off[r] + 2 : 0;
        out[i] = (r < hi) ? (c > cmin ? c : (uint64_t)cmin) : 0;
    }
}

__global__ void packed_bounds(const uint64_t* __restrict__ excl, uint32_t lo, uint32_t hi,
                              uint32_t win, uint32_t n_packed, uint32_t* __restrict__ r0) {
    const uint32_t rows = hi - lo;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) {
        const uint64_t t = excl[i] / win;
        const int64_t tp = (i == 0) ? -1 : (int64_t)(excl[i - 1] / win);
        for (int64_t x = tp + 1; x <= (int64_t)t; ++x) r0[x] = lo + i;
        if (i == rows - 1)
            for (uint64_t x = t + 1; x <= n_packed; ++x) r0[x] = hi;
    }
}

// One 16-byte record per wide-piece chunk task, so a task costs one load
// instead of the chunk -> piece -> offsets chain: {first edge (lo, hi), edges,
// the piece's slot}; bit 31 of the last word marks a chunk of a multi-chunk
// piece (those go through the hand-off, which looks the piece up itself).
__global__ void seg_task_records(const uint32_t* __restrict__ chunk_row, const uint32_t* __restrict__ chunk_first,
                                 const uint64_t* __restrict__ off, const uint32_t* __restrict__ slot,
                                 uint32_t n_chunk, uint32_t chunk, uint4* __restrict__ rec) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_chunk; t += gridDim.x * blockDim.x) {
        const uint32_t p = chunk_row[t], first = chunk_first[p], nch = chunk_first[p + 1] - first;
        const uint64_t hi = off[p + 1];
        const uint64_t lo = min(off[p] + (uint64_t)(t - first) * chunk, hi);
        const uint32_t len = (uint32_t)min((uint64_t)chunk, hi - lo);
        rec[t] = make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), len, nch == 1 ? slot[p] : 0x80000000u);
    }
}

// One record per packed run (rows or small pieces): {first edge (lo, hi), first
// row, edges | rows << 16}, so the run's offsets and colidx are staged together.
__global__ void run_records(const uint32_t* __restrict__ r0s, const uint64_t* __restrict__ off, uint32_t n_runs,
                            uint4* __restrict__ rec) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_runs; t += gridDim.x * blockDim.x) {
        const uint32_t r0 = r0s[t], r1 = r0s[t + 1];
        const uint64_t e0 = off[r0];
        rec[t] = make_uint4((uint32_t)e0, (uint32_t)(e0 >> 32), r0, (uint32_t)(off[r1] - e0) | ((r1 - r0) << 16));
    }
}

// ---- deterministic device error_norm (norms.hpp:48-78) ------------------------------
// The reference accumulates L1 and L2 in x87 long double (64-bit mantissa,
// norms.hpp:57-69).  The device has no long double: sums are carried as
// double-double pairs (error-free TwoSum; the L2 square split exactly by an
// FMA), i.e. more precise than the reference, so the result is the
// reference's rounded to double, up to the reference's own rounding.
struct DD {
    double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, double b) {
    const double s = a.hi + b, bb = s - a.hi;
    const double e = (a.hi - (s - bb)) + (b - bb);
    const double lo = a.lo + e;
    const double hi = s + lo;
    return DD{hi, lo - (hi - s)};
}
__device__ __forceinline__ DD dd_add(DD a, DD b) { return dd_add(dd_add(a, b.hi), b.lo); }

__global__ void norm_partials(int kind, const double* __restrict__ r, const double* __restrict__ s,
                              uint64_t n, double* __restrict__ out) {
    __shared__ DD red[kNT / 32];
    DD v{0.0, 0.0};
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double d = r[i] - s[i]; // double difference, as the reference
        if (kind == 0) v = dd_add(v, fabs(d));
        else if (kind == 1) {
            const double sq = d * d;
            v = dd_add(dd_add(v, sq), fma(d, d, -sq)); // d^2 exactly
        } else v.hi = fmax(v.hi, fabs(d));
    }
    for (int off = 16; off > 0; off >>= 1) {
        const DD o{__shfl_xor_sync(0xffffffffu, v.hi, off), __shfl_xor_sync(0xffffffffu, v.lo, off)};
        if (kind == 2) v.hi = fmax(v.hi, o.hi);
        else v = dd_add(v, o);
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        DD t{0.0, 0.0};
        for (int w = 0; w < kNT / 32; ++w) {
            if (kind == 2) t.hi = fmax(t.hi, red[w].hi);
            else t = dd_add(t, red[w]);
        }
        out[2 * blockIdx.x] = t.hi;
        out[2 * blockIdx.x + 1] = t.lo;
    }
}

__global__ void norm_final(int kind, const double* __restrict__ parts, int nparts, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    DD t{0.0, 0.0};
    for (int i = 0; i < nparts; ++i) {
        if (kind == 2) t.hi = fmax(t.hi, parts[2 * i]);
        else t = dd_add(t, DD{parts[2 * i], parts[2 * i + 1]});
    }
    if (kind == 1) { // sqrt of the double-double sum, one Newton correction
        const double q = sqrt(t.hi);
        out[0] = q > 0.0 ? q + (fma(-q, q, t.hi) + t.lo) / (2.0 * q) : q;
    } else {
        out[0] = t.hi + t.lo;
    }
}

template <int LG, int W, int WIN, int MINB, int KS = LG * W, int PATHS = 3>
LaneCfg wide_cfg(bool all_q) {
    return all_q ? mk_cfg<LG, W, WIN, 0, MINB, kQmAll, KS, PATHS>()
                 : mk_cfg<LG, W, WIN, 0, MINB, kQmL1, KS, PATHS>();
}

// Defaults measured on B200 (scripts/experiments/gpu_variants*.sh).
// Wide lanes: two doubles per thread (one 16-byte load per edge), LG = KS/2
// threads per edge, rows padded to whole 32-byte sectors; up to four lanes,
// one double per thread (LG = KS).
template <int PATHS>
LaneCfg lane_cfg_t(int K, bool all_q) {
    if (K == 1) return k1_base(); // (PATHS 3: the only base configuration)
    if (K == 2) return wide_cfg<2, 1, 64, 4, 2, PATHS>(all_q);
    if (K <= 4) return wide_cfg<4, 1, kW4, 4, 4, PATHS>(all_q);
    if (K <= 8) return wide_cfg<4, 2, 128, 4, 8, PATHS>(all_q);
    if (K <= 12) return wide_cfg<8, 2, 128, kMinb12, 12, PATHS>(all_q);
    return wide_cfg<8, 2, 128, 4, 16, PATHS>(all_q);
}

// The run's base configuration: one kernel per iteration (PATHS = 3).
inline LaneCfg lane_cfg(int K, bool all_q) { return lane_cfg_t<3>(K, all_q); }

// Lane-width modes of a K > 1 run (Params::mode_id): the same window and task
// tables (an instance's WIN must be >= the run's: its shared-memory stage is
// sized by it); a narrow mode's contribution rows hold
// just its kp lanes (KS = kp), the widest mode's the run's full stride.
// Returns false when (KS, kp) has no instance.
// k1_minb4: a K = 1 run split into its two kernels (win 256), bit PATHS-1
// set: that kernel at 4 CTAs/SM instead of 3.
template <int PATHS>
bool mode_cfg(int KS, int kp, int win, bool all_q, LaneCfg& out, int k1_minb4 = 0) {
    if (win == 256 && KS == 1 && kp == 1) return k1_mode(PATHS, win, all_q, ((k1_minb4 >> (PATHS - 1)) & 1) != 0, out);
    switch (KS * 100 + kp) {
    case 101:
        out = all_q ? mk_cfg<1, 1, 128, 2, 3, kQmAll, 1, PATHS>() : mk_cfg<1, 1, 128, 2, 3, kQmL1, 1, PATHS>();
        return true;
    // two- and four-lane modes: one 8-byte lane per thread (LG = kp), measured
    // -9% per C5 sweep against two lanes per thread (PRGPU_K4CFG=1 /
    // PRGPU_K2CFG=1 select the two-lane-per-thread instances: tuning only)
    case 202:
        if (k_variant("PRGPU_K2CFG") == 1) { out = wide_cfg<1, 2, 128, 4, 2, PATHS>(all_q); return true; }
        out = wide_cfg<2, 1, 128, 4, 2, PATHS>(all_q);
        return true;
    case 404:
        if (k_variant("PRGPU_K4CFG") == 1) { out = wide_cfg<2, 2, 128, 4, 4, PATHS>(all_q); return true; }
        out = wide_cfg<4, 1, kW4, 4, 4, PATHS>(all_q);
        return true;
    case 808: out = wide_cfg<4, 2, 128, 4, 8, PATHS>(all_q); return true;
    case 1216: out = wide_cfg<8, 2, 128, kMinb12, 12, PATHS>(all_q); return true;
    case 1616: out = wide_cfg<8, 2, 128, 4, 16, PATHS>(all_q); return true;
    default: return false;
    }
}

void launch_init(const LaneCfg& c, const Params& P, uint32_t ndangling, cudaStream_t st) {
    const unsigned grid = (unsigned)std::min<uint64_t>((P.n + kNT - 1) / kNT, 148ull * 16);
    switch (c.KS) {
    case 1: init_kernel<1><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 2: init_kernel<2><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 4: init_kernel<4><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 8: init_kernel<8><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 12: init_kernel<12><<<grid, kNT, 0, st>>>(P, ndangling); break;
    default: init_kernel<16><<<grid, kNT, 0, st>>>(P, ndangling); break;
    }
    PRGPU_LAUNCHED("init_kernel");
}

inline unsigned blocks_for(uint64_t n) {
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + kNT - 1) / kNT, 148ull * 16));
}

} // namespace prgpu

using namespace prgpu;

namespace prgpu {
// Host-mapped int slots (the per-lane stop iterations a session's finalizer
// writes for the host): cudaHostAlloc / cudaFreeHost cost ~1 ms each and may
// synchronise, so slots come from a process-wide pool of portable mapped
// blocks (under UVA the device address equals the host address).
constexpr int kSlotInts = 64; // >= PRGPU_MAX_LANES
struct MappedSlots {
    std::mutex mu;
    std::vector<int*> free;
};
inline MappedSlots& mapped_slots() {
    static MappedSlots m;
    return m;
}
inline int* mapped_slot_get() {
    MappedSlots& M = mapped_slots();
    std::lock_guard<std::mutex> lk(M.mu);
    if (M.free.empty()) {
        constexpr int kSlots = 256;
        int* base = nullptr;
        PRGPU_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&base), (size_t)kSlots * kSlotInts * sizeof(int),
                                 cudaHostAllocMapped | cudaHostAllocPortable));
        for (int i = kSlots - 1; i >= 0; --i) M.free.push_back(base + (size_t)i * kSlotInts);
    }
    int* h = M.free.back();
    M.free.pop_back();
    return h;
}
inline void mapped_slot_put(int* h) {
    MappedSlots& M = mapped_slots();
    std::lock_guard<std::mutex> lk(M.mu);
    M.free.push_back(h);
}
} // namespace prgpu

struct prgpu_session {
    prgpu_graph* g = nullptr;
    int K = 1, KP = 1, max_iter = 500;
    LaneCfg cfg{};   // base configuration (window, stride, lanes per row; multi-GPU kernels)
    // the kernels of one iteration, in launch order: one pull kernel, or per
    // lane-width mode a hub-chunk kernel and a packed + empty kernel (only
    // the mode selected by the previous finalizer does work)
    struct Launch {
        KernelFn fn;
        Params P;
        size_t smem;
        bool repack; // repack_kernel(P, nsrc) instead of a pull kernel
    };
    std::vector<Launch> launches;
    int mode0 = 0;   // lane-width mode of the first iteration
    // partition sessions: the lane-mode launch list the fused exchange switches
    // to (prgpu_part_set_peers); the NCCL exchange keeps the widest mode only
    std::vector<Launch> modal_launches;
    Params modal_P{};
    int modal_mode0 = 0;
    bool all_q = true; // every partial quantity tracked (not only the L1 stopping rule)
    Params P{};
    Stream stream;
    DevBuf<double> rank, contrib, partials, trace, ref, chunk_acc;
    DevBuf<double> hot_part; // split pull: [nonempty rows][KS] hot partial sums
    DevBuf<unsigned long long> ktime; // [max_iter][2] in-graph kernel start / end (ns)
    DevBuf<double> mode_contrib[kMaxModes]; // narrow modes' contribution buffers (after `stream`:
                                            // freed on it before it is destroyed)
    DevBuf<LaneState> lanes;
    DevBuf<GlobalState> gs;
    DevBuf<uint32_t> chunk_row, chunk_first, packed_r0;
    DevBuf<unsigned int> row_cnt;
    // segmented hub pull (SegPlan): task tables over the plan's pieces, the
    // wide pieces' chunk hand-off state and the piece partial sums
    const SegPlan* seg = nullptr;
    DevBuf<uint32_t> seg_chunk_row, seg_chunk_first, seg_packed_r0;
    DevBuf<uint4> seg_task; // [wide-piece chunk tasks] one record per task (seg_task_records)
    DevBuf<uint4> seg_run_rec, run_rec; // one record per small-piece run / packed-row run (run_records)
    DevBuf<double> seg_chunk_acc, pacc;
    DevBuf<unsigned int> seg_row_cnt;
    uint32_t seg_n_wchunk = 0, seg_n_runs = 0, seg_n_comb = 0, seg_chunk_t0 = 0;
    std::vector<LaneState> lanes_host; // device slot order
    std::vector<int> user_of;          // caller lane of each device slot
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool use_graph = false;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    double last_loop_ms = 0;
    // multi-GPU partition
    int part_rank = 0, nranks = 1, host_iter = 0;
    uint32_t n_long = 0;        // rows cut into chunk tasks
    bool dealt = false;         // fused partition: work units dealt round-robin (task lists, row owners)
    DevBuf<uint32_t> task_list; // this rank's tasks, ascending: hub chunks, then packed + empty
    DevBuf<uint8_t> row_owner;  // [n] rank owning each row
    uint32_t deal_split = 0, deal_total = 0; // task_list: [0, split) hub chunks, [split, total) the rest
    std::vector<prgpu_partition> parts;
    DevBuf<double> rank_partials;
    uint64_t sent_rows = 0;    // fused exchange: contribution rows stored into peers per iteration
    DevBuf<unsigned int> need; // fused exchange: [ceil(nsrc/4)] one byte per source, bit q = rank q gathers it
    bool need_given = false;   // shards: the ranks' OR-reduced mask (prgpu_part_set_need)
    cudaStream_t ext_stream = nullptr;
    double* ext_contrib_base = nullptr; // caller-provided contribution buffer (partition sessions)
    double* ext_rank_partials = nullptr; // caller-provided rank partials (2 parities for the fused exchange)
    cudaStream_t cur() const { return ext_stream ? ext_stream : (cudaStream_t)stream; }
    // lanes that stopped, written by the device (host-mapped), for copying
    // results out while the other lanes still iterate (session_solve)
    int* host_frozen = nullptr;
    int* dev_frozen = nullptr;
    std::unique_ptr<Stream> aux;

    ~prgpu_session() {
        if (host_frozen) prgpu::mapped_slot_put(host_frozen);
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
    }
};

namespace prgpu {

void validate_params(const prgpu_params* p) {
    if (!p) fail(PRGPU_EINVAL, "pagerank: null params");
    if (p->lanes < 1 || p->lanes > PRGPU_MAX_LANES)
        fail(PRGPU_EINVAL, "pagerank: lanes must be in [1, " + std::to_string(PRGPU_MAX_LANES) + "]");
    if (!p->alphas) fail(PRGPU_EINVAL, "pagerank: null alphas");
    // PageRankConfig::validate (pagerank.hpp:29-39)
    for (int k = 0; k < p->lanes; ++k) {
        const double a = p->alphas[k];
        if (!(a >= 0.0 && a <= 1.0))
            fail(PRGPU_EINVAL, "alpha must be in [0, 1], got " + std::to_string(a));
        const double t = p->tolerances ? p->tolerances[k] : p->tolerance;
        if (!(t > 0.0)) fail(PRGPU_EINVAL, "tolerance must be positive, got " + std::to_string(t));
    }
    if (p->max_iterations < 1)
        fail(PRGPU_EINVAL, "max_iterations must be >= 1, got " + std::to_string(p->max_iterations));
    if (p->norm < 0 || p->norm > 2) fail(PRGPU_EINVAL, "pagerank: unknown norm");
    if (p->stop_mask > 7) fail(PRGPU_EINVAL, "pagerank: stop_mask has unknown bits");
}

__global__ void count_isolated_kernel(const uint64_t* __restrict__ row_off,
                                      const uint2* __restrict__ rowinfo, uint32_t n,
                                      unsigned int* __restrict__ out) {
    unsigned int c = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        c += (row_off[r + 1] == row_off[r]) && rowinfo[r].x == 0;
    atomicAdd(out, c);
}

// rows with neither in- nor out-edges; they sort last (in desc, out desc)
uint32_t count_isolated(const prgpu_graph* g, cudaStream_t st) {
    DevBuf<unsigned int> cnt(1);
    PRGPU_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned int), st));
    count_isolated_kernel<<<blocks_for(g->n), kNT, 0, st>>>(g->row_off.p, g->rowinfo.p, g->n, cnt.p);
    PRGPU_LAUNCHED("count_isolated");
    unsigned int c = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&c, cnt.p, 4, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    return c;
}

// Warp-task tables for one lane configuration (depends only on the graph and WIN).
void build_tasks(prgpu_session* s) {
    const prgpu_graph* g = s->g;
    cudaStream_t st = s->stream;
    // hub rows (in-degree > WIN) are cut into chunk tasks of `emax` edges:
    // large enough to amortise a task's fixed cost (row lookup, the fence and
    // counter that hand the row to its last chunk), small enough to balance
    const uint32_t win = (uint32_t)s->cfg.WIN;
    // measured: 4096 / 2048 edges, 4x that on graphs of >= 2^29
    // edges (C4 -2.6%, C5 -2.2%: fewer hand-offs, still thousands of chunks)
    uint32_t emax = std::max<uint32_t>(2 * win, (s->KP == 1 ? 4096 : 2048) * (s->g->e >= (1ull << 29) ? 4 : 1));
    if (const char* c = std::getenv("PRGPU_CHUNK")) emax = std::max(2 * win, (uint32_t)std::atoi(c));
    s->P.chunk = emax;
    const uint32_t n = g->n;
    // long rows: a prefix, since rows are sorted by in-degree descending
    DevBuf<unsigned int> cnt(1);
    PRGPU_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned int), st));
    count_long_rows<<<blocks_for(n), kNT, 0, st>>>(g->row_off.p, n, win, cnt.p);
    PRGPU_LAUNCHED("count_long_rows");
    unsigned int n_long = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&n_long, cnt.p, 4, cudaMemcpyDeviceToHost, st));
    s->n_long = 0; // set once known (below)
    PRGPU_CUDA(cudaStreamSynchronize(st));

    s->n_long = n_long;
    DevBuf<uint64_t> first((size_t)n_long + 1);
    chunk_counts<<<blocks_for((uint64_t)n_long + 1), kNT, 0, st>>>(g->row_off.p, n_long, emax, first.p);
    PRGPU_LAUNCHED("chunk_counts");
    {
        size_t tmp = 0;
        PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, first.p, first.p, (int64_t)n_long + 1, st));
        DevBuf<char> t(std::max<size_t>(tmp, 1));
        PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, first.p, first.p, (int64_t)n_long + 1, st));
        g_launches.fetch_add(1);
    }
    uint64_t n_chunk = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&n_chunk, first.p + n_long, 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    s->chunk_first.alloc((size_t)n_long + 1);
    s->chunk_row.alloc(std::max<uint64_t>(n_chunk, 1));
    chunk_fill<<<blocks_for((uint64_t)n_long + 1), kNT, 0, st>>>(first.p, n_long, s->chunk_first.p,
                                                                  s->chunk_row.p);
    PRGPU_LAUNCHED("chunk_fill");
    s->chunk_acc.alloc(std::max<uint64_t>(n_chunk, 1) * s->KP);
    s->row_cnt.alloc(std::max<uint32_t>(n_long, 1));
    PRGPU_CUDA(cudaMemsetAsync(s->row_cnt.p, 0, std::max<uint32_t>(n_long, 1) * 4, st));

    // packed rows [n_long, nonempty_end)
    // (rows the segment plan covers beyond the hub rows are pulled as pieces, not as packed rows)
    const uint32_t plo = std::max<uint32_t>(n_long, s->seg ? std::min(s->seg->n_rows, g->nonempty_end) : 0u);
    const uint32_t phi = std::max(plo, g->nonempty_end);
    const uint32_t prow = phi - plo;
    const uint32_t cmin = std::max<uint32_t>(1, (win + 31) / 32);
    uint64_t n_packed = 0;
    if (prow) {
        // runs of rows [a, b): on a shard graph the packed rows are cut at every
        // shard boundary, so no run spans two ranks' rows
        std::vector<uint32_t> cuts{plo};
        if (g->shard_n > 1)
            for (uint32_t x : g->shard_rows)
                if (x > plo && x < phi) cuts.push_back(x);
        cuts.push_back(phi);
        std::vector<std::pair<DevBuf<uint32_t>, uint64_t>> segs;
        for (size_t k = 0; k + 1 < cuts.size(); ++k) {
            const uint32_t a = cuts[k], b = cuts[k + 1], rows = b - a;
            if (!rows) continue;
            DevBuf<uint64_t> cost((size_t)rows + 1);
            packed_costs<<<blocks_for((uint64_t)rows + 1), kNT, 0, st>>>(g->row_off.p, a, b, cmin, cost.p);
            PRGPU_LAUNCHED("packed_costs");
            size_t tmp = 0;
            PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cost.p, cost.p, (int64_t)rows + 1, st));
            DevBuf<char> t(std::max<size_t>(tmp, 1));
            PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, cost.p, cost.p, (int64_t)rows + 1, st));
            g_launches.fetch_add(1);
            uint64_t total = 0;
            PRGPU_CUDA(cudaMemcpyAsync(&total, cost.p + rows, 8, cudaMemcpyDeviceToHost, st));
            PRGPU_CUDA(cudaStreamSynchronize(st));
            const uint64_t np = (total + win - 1) / win;
            DevBuf<uint32_t> r0(np + 1);
            packed_bounds<<<blocks_for(rows), kNT, 0, st>>>(cost.p, a, b, win, (uint32_t)np, r0.p);
            PRGPU_LAUNCHED("packed_bounds");
            PRGPU_CUDA(cudaStreamSynchronize(st));
            n_packed += np;
            segs.emplace_back(std::move(r0), np);
        }
        s->packed_r0.alloc(n_packed + 1);
        uint64_t at = 0; // segment k's runs, then its end row (= the next segment's first)
        for (auto& sg : segs) {
            PRGPU_CUDA(cudaMemcpyAsync(s->packed_r0.p + at, sg.first.p, (sg.second + 1) * 4,
                                       cudaMemcpyDeviceToDevice, st));
            at += sg.second;
        }
        PRGPU_CUDA(cudaStreamSynchronize(st));
    } else {
        s->packed_r0.alloc(1);
    }
    // rows with no in-edges: only those with out-edges need a task (their next
    // contribution c0/d), unless the reference trace needs every row
    const uint32_t er = 8 * (32 / s->cfg.LG);
    const uint32_t iso_begin = std::max(phi, n - count_isolated(g, st));
    const uint32_t n_empty_rows = (s->P.ref ? n : iso_begin) - phi;
    s->P.iso_begin = iso_begin;
    Params& P = s->P;
    P.chunk_row = s->chunk_row.p;
    P.chunk_first = s->chunk_first.p;
    P.packed_r0 = s->packed_r0.p;
    P.run_rec = nullptr;
    if (n_packed && !std::getenv("PRGPU_NO_RUNREC")) { // (PRGPU_NO_RUNREC=1, tuning: bounds -> offsets -> colidx)
        s->run_rec.alloc(n_packed);
        run_records<<<blocks_for(n_packed), kNT, 0, st>>>(s->packed_r0.p, g->row_off.p, (uint32_t)n_packed, s->run_rec.p);
        PRGPU_LAUNCHED("run_records");
        P.run_rec = s->run_rec.p;
    }
    P.chunk_acc = s->chunk_acc.p;
    P.row_cnt = s->row_cnt.p;
    P.n_chunk = (uint32_t)n_chunk;
    P.n_packed = (uint32_t)n_packed;
    P.n_empty_tasks = (n_empty_rows + er - 1) / er;
    P.er = er;
    P.empty_begin = phi;
    P.task_begin = 0;
    P.task_end = P.n_chunk + P.n_packed + P.n_empty_tasks;
    P.part_mode = 0;
    P.part_rank = 0;
    P.nranks = 1;
}

// Segmented hub pull (SegPlan, common.cuh; single-GPU sessions): task tables
// over the plan's pieces.  Wide pieces are cut into chunk tasks exactly like
// hub rows (same chunk size, same hand-off), small pieces are grouped into
// runs exactly like packed rows; the rows' epilogues become combine tasks.
// On by default when the contribution table is at least three segments long
// (measured on B200: C5 620 -> 457 ms per
// sweep, RMAT-24 x 11 lanes -5 %, C4 -3 %; C2's 194 MB table +5 %, off).
// PRGPU_SEG=0/1 forces it off/on, PRGPU_SEG_KB the segment size (KB of the
// run's widest contribution rows), PRGPU_SEG_HOT the number of L2-sized
// segments before the cold rest, PRGPU_SEG_T the least in-degree of a
// segmented row, PRGPU_SEG_PMIN the smallest hot-segment piece kept.
void seg_choose_plan(prgpu_session* s, int nranks) {
    prgpu_graph* g = s->g;
    cudaStream_t st = s->stream;
    if (nranks != 0 || g->shard_n > 1 || g->locality) return;
    auto env_u = [](const char* name, uint64_t dflt) -> uint64_t {
        const char* v = std::getenv(name);
        return v ? (uint64_t)std::atoll(v) : dflt;
    };
    const uint64_t row_bytes = (uint64_t)s->cfg.KS * sizeof(double);
    // 64 MB: the largest slice of the table the L2 keeps (profiles/r1_gather_ceiling.md)
    const uint64_t seg_bytes = std::max<uint64_t>(env_u("PRGPU_SEG_KB", 64u << 10) << 10, row_bytes);
    const uint64_t table = (uint64_t)g->nsrc * row_bytes;
    const char* en = std::getenv("PRGPU_SEG");
    const bool want = en ? std::atoi(en) != 0 : table >= 3 * seg_bytes;
    if (!want) return;
    const uint32_t win = (uint32_t)s->cfg.WIN;
    const uint32_t seg_src = (uint32_t)std::max<uint64_t>(1, seg_bytes / row_bytes);
    const uint32_t hot = (uint32_t)std::min<uint64_t>(63, std::max<uint64_t>(1, env_u("PRGPU_SEG_HOT", 16)));
    const uint32_t s_all = (uint32_t)((table + seg_bytes - 1) / seg_bytes);
    // the last segment is the cold rest: sources past the hot segments, and
    // the hot-segment pieces too small to be worth a partial (pmin)
    if (s_all < 2) return; // the whole table is one segment
    const uint32_t pmin = (uint32_t)env_u("PRGPU_SEG_PMIN", 0); // measured: folding small pieces loses (C5 +1 % at 8, +4 % at 16)
    const uint32_t S = (s_all <= hot && pmin == 0) ? s_all : std::min(s_all, hot) + 1;
    // every hub row by default (C5: T = 512 leaves the rows of 129..511 in-edges to miss: 595 vs 500 ms);
    // a smaller T also segments packed rows (all their pieces are small)
    const uint32_t T = (uint32_t)std::max<uint64_t>(env_u("PRGPU_SEG_T", (uint64_t)win + 1), 2);
    // pieces longer than wmin edges are pulled by a whole warp (chunk tasks), the others by a lane group
    // (measured with the one-load task records: half the packed window; C5 456.3 ms against 459.5 at 3/4
    // and 471.3 at the whole window, RMAT-24 x 11 82.8 / 83.7, C4 111.8 / 112.2; a quarter: 460.2)
    const uint32_t wmin = (uint32_t)std::min<uint64_t>(win, std::max<uint64_t>(1, env_u("PRGPU_SEG_WMIN", win / 2)));
    s->seg = graph_seg_plan(g, seg_src, S, T, wmin, pmin, st);
}

// the plan's task tables (after build_tasks: the chunk size and the hub rows' chunk table)
void build_seg_tasks(prgpu_session* s) {
    const SegPlan* sp = s->seg;
    if (!sp) return;
    cudaStream_t st = s->stream;
    const uint32_t win = (uint32_t)s->cfg.WIN;
    const uint32_t S = sp->S;
    const uint32_t emax = s->P.chunk;
    // chunk tasks of the wide pieces
    const uint32_t nw = sp->n_wp;
    DevBuf<uint64_t> first((size_t)nw + 1);
    chunk_counts<<<blocks_for((uint64_t)nw + 1), kNT, 0, st>>>(sp->off.p, nw, emax, first.p);
    PRGPU_LAUNCHED("chunk_counts");
    {
        size_t tmp = 0;
        PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, first.p, first.p, (int64_t)nw + 1, st));
        DevBuf<char> t(std::max<size_t>(tmp, 1));
        PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, first.p, first.p, (int64_t)nw + 1, st));
        g_launches.fetch_add(1);
    }
    uint64_t n_chunk = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&n_chunk, first.p + nw, 8, cudaMemcpyDeviceToHost, st));
    // the hub rows' own chunk tasks start after the segmented rows'
    PRGPU_CUDA(cudaMemcpyAsync(&s->seg_chunk_t0, s->chunk_first.p + std::min(sp->n_rows, s->n_long), 4,
                               cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    s->seg_chunk_first.alloc((size_t)nw + 1);
    s->seg_chunk_row.alloc(std::max<uint64_t>(n_chunk, 1));
    chunk_fill<<<blocks_for((uint64_t)nw + 1), kNT, 0, st>>>(first.p, nw, s->seg_chunk_first.p, s->seg_chunk_row.p);
    PRGPU_LAUNCHED("chunk_fill");
    s->seg_chunk_acc.alloc(std::max<uint64_t>(n_chunk, 1) * s->KP);
    s->seg_row_cnt.alloc(std::max<uint32_t>(nw, 1));
    PRGPU_CUDA(cudaMemsetAsync(s->seg_row_cnt.p, 0, std::max<uint32_t>(nw, 1) * 4, st));
    s->seg_n_wchunk = (uint32_t)n_chunk;
    s->seg_task.alloc(std::max<uint64_t>(n_chunk, 1));
    if (n_chunk) {
        seg_task_records<<<blocks_for(n_chunk), kNT, 0, st>>>(s->seg_chunk_row.p, s->seg_chunk_first.p, sp->off.p,
                                                               sp->slot.p, (uint32_t)n_chunk, emax, s->seg_task.p);
        PRGPU_LAUNCHED("seg_task_records");
    }
    // runs of small pieces
    const uint32_t lo = nw, hi = nw + sp->n_sp;
    uint64_t np = 0;
    if (hi > lo) {
        const uint32_t rows = hi - lo;
        const uint32_t cmin = std::max<uint32_t>(1, (win + 31) / 32);
        DevBuf<uint64_t> cost((size_t)rows + 1);
        packed_costs<<<blocks_for((uint64_t)rows + 1), kNT, 0, st>>>(sp->off.p, lo, hi, cmin, cost.p);
        PRGPU_LAUNCHED("packed_costs");
        size_t tmp = 0;
        PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cost.p, cost.p, (int64_t)rows + 1, st));
        DevBuf<char> t(std::max<size_t>(tmp, 1));
        PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, cost.p, cost.p, (int64_t)rows + 1, st));
        g_launches.fetch_add(1);
        uint64_t total = 0;
        PRGPU_CUDA(cudaMemcpyAsync(&total, cost.p + rows, 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        np = (total + win - 1) / win;
        s->seg_packed_r0.alloc(np + 1);
        packed_bounds<<<blocks_for(rows), kNT, 0, st>>>(cost.p, lo, hi, win, (uint32_t)np, s->seg_packed_r0.p);
        PRGPU_LAUNCHED("packed_bounds");
        PRGPU_CUDA(cudaStreamSynchronize(st));
    } else {
        s->seg_packed_r0.alloc(1);
    }
    s->seg_n_runs = (uint32_t)np;
    s->seg_run_rec.alloc(std::max<uint64_t>(np, 1));
    if (np) {
        run_records<<<blocks_for(np), kNT, 0, st>>>(s->seg_packed_r0.p, sp->off.p, (uint32_t)np, s->seg_run_rec.p);
        PRGPU_LAUNCHED("run_records");
    }
    // piece partial sums: a slot per (row, segment), zero where a row has no piece
    s->pacc.alloc((size_t)sp->n_rows * S * s->KP);
    PRGPU_CUDA(cudaMemsetAsync(s->pacc.p, 0, s->pacc.bytes(), st));
    const uint32_t cr = 2 * (32 / (uint32_t)s->cfg.LG);
    s->seg_n_comb = (sp->n_rows + cr - 1) / cr;
    Params& P = s->P;
    P.seg_off = sp->off.p;
    P.seg_col = sp->col.p;
    P.seg_slot = sp->slot.p;
    P.seg_task = s->seg_task.p;
    P.seg_run_rec = s->seg_run_rec.p;
    P.seg_chunk_row = s->seg_chunk_row.p;
    P.seg_chunk_first = s->seg_chunk_first.p;
    P.seg_packed_r0 = s->seg_packed_r0.p;
    P.seg_chunk_acc = s->seg_chunk_acc.p;
    P.seg_row_cnt = s->seg_row_cnt.p;
    P.pacc = s->pacc.p;
    P.n_seg_rows = sp->n_rows;
    P.seg_S = S;
    P.pacc_stride = (uint32_t)s->KP;
    P.seg_pre = 0;
    P.seg_cr = cr;
}

// ---- 1D partition (multi-GPU): contiguous task ranges with equal cost, cut at
// row boundaries (a hub row's chunks stay on one rank), so each rank owns a
// contiguous row range and a contiguous source-id range. --------------------------
__global__ void task_costs_kernel(Params P, uint32_t er, uint64_t* __restrict__ cost) {
    const uint32_t T1 = P.n_chunk, T2 = T1 + P.n_packed, T3 = T2 + P.n_empty_tasks;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < T3; t += gridDim.x * blockDim.x) {
        uint64_t c;
        if (t < T1) {
            const uint32_t row = P.chunk_row[t];
            const uint64_t d = P.row_off[row + 1] - P.row_off[row];
            const uint64_t off = (uint64_t)(t - P.chunk_first[row]) * P.chunk;
            c = (d - off < P.chunk ? d - off : P.chunk);
        } else if (t < T2) {
            const uint32_t r0 = P.packed_r0[t - T1], r1 = P.packed_r0[t - T1 + 1];
            c = (P.row_off[r1] - P.row_off[r0]) + 2ull * (r1 - r0);
        } else {
            c = 2ull * er;
        }
        cost[t] = c;
    }
}

__device__ uint32_t row_of_task(const Params& P, uint32_t t, uint32_t er) {
    const uint32_t T1 = P.n_chunk, T2 = T1 + P.n_packed, T3 = T2 + P.n_empty_tasks;
    if (t >= T3) return P.n;
    if (t < T1) return P.chunk_row[t];
    if (t < T2) return P.packed_r0[t - T1];
    const uint64_t r = (uint64_t)P.empty_begin + (uint64_t)(t - T2) * er;
    return r < P.n ? (uint32_t)r : P.n;
}

// bound[b] for b in [0, nranks]: task, row and source boundaries
__global__ void partition_kernel(Params P, const uint64_t* __restrict__ incl, uint32_t er, uint32_t nranks,
                                 const uint32_t* __restrict__ row_of_src, uint32_t nsrc,
                                 uint64_t* __restrict__ bound /* [nranks+1][3] */) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nranks) return;
    const uint32_t T = P.n_chunk + P.n_packed + P.n_empty_tasks;
    uint32_t t;
    if (b == 0) t = 0;
    else if (b == nranks) t = T;
    else {
        const uint64_t total = T ? incl[T - 1] : 0, target = total * b / nranks;
        uint32_t lo = 0, hi = T; // first task whose exclusive prefix >= target
        while (lo < hi) {
            const uint32_t mid = (lo + hi) / 2;
            if ((mid ? incl[mid - 1] : 0) < target) lo = mid + 1; else hi = mid;
        }
        t = lo;
        if (t < P.n_chunk && t != P.chunk_first[P.chunk_row[t]]) t = P.chunk_first[P.chunk_row[t] + 1];
    }
    const uint32_t row = row_of_task(P, t, er);
    uint32_t lo = 0, hi = nsrc; // sources with engine row < row
    while (lo < hi) {
        const uint32_t mid = (lo + hi) / 2;
        if (row_of_src[mid] < row) lo = mid + 1; else hi = mid;
    }
    bound[3 * b + 0] = t;
    bound[3 * b + 1] = row;
    bound[3 * b + 2] = lo;
}

// shard graphs: every rank's tasks are those of its shard's rows (build_tasks
// cut the packed runs at the shard boundaries; empty-row tasks align to them)
__global__ void shard_task_bounds(Params P, uint32_t er, const uint32_t* __restrict__ rows, uint32_t nranks,
                                  const uint32_t* __restrict__ row_of_src, uint32_t nsrc,
                                  uint64_t* __restrict__ bound) {
    const uint32_t b = threadIdx.x;
    if (b > nranks) return;
    const uint32_t T = P.n_chunk + P.n_packed + P.n_empty_tasks, R = rows[b];
    uint32_t lo = 0, hi = T; // first task whose row >= R
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (row_of_task(P, mid, er) < R) lo = mid + 1;
        else hi = mid;
    }
    uint32_t a = 0, z = nsrc; // sources with engine row < R
    while (a < z) {
        const uint32_t mid = (a + z) / 2;
        if (row_of_src[mid] < R) a = mid + 1;
        else z = mid;
    }
    bound[3 * b + 0] = b == nranks ? T : lo;
    bound[3 * b + 1] = R;
    bound[3 * b + 2] = a;
}

void plan_partition(prgpu_session* s, int nranks) {
    const prgpu_graph* g = s->g;
    cudaStream_t st = s->stream;
    Params& P = s->P;
    const uint32_t T = P.n_chunk + P.n_packed + P.n_empty_tasks;
    const uint32_t er = 8 * (32 / s->cfg.LG);
    if (g->shard_n > 1) {
        if (nranks != g->shard_n) fail(PRGPU_EINVAL, "partition: nranks differs from the graph's shard count");
        DevBuf<uint32_t> rows((size_t)nranks + 1);
        DevBuf<uint64_t> bound(3 * ((size_t)nranks + 1));
        PRGPU_CUDA(cudaMemcpyAsync(rows.p, g->shard_rows.data(), ((size_t)nranks + 1) * 4, cudaMemcpyHostToDevice, st));
        shard_task_bounds<<<1, 128, 0, st>>>(P, er, rows.p, (uint32_t)nranks, g->row_of_src.p, g->nsrc, bound.p);
        PRGPU_LAUNCHED("shard_task_bounds");
        std::vector<uint64_t> b(3 * ((size_t)nranks + 1));
        PRGPU_CUDA(cudaMemcpyAsync(b.data(), bound.p, b.size() * 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        s->parts.resize(nranks);
        for (int r = 0; r < nranks; ++r) {
            prgpu_partition& q = s->parts[r];
            q.task_begin = (uint32_t)b[3 * r];
            q.task_end = (uint32_t)b[3 * (r + 1)];
            q.row_begin = (uint32_t)b[3 * r + 1];
            q.row_end = (uint32_t)b[3 * (r + 1) + 1];
            q.src_begin = b[3 * r + 2];
            q.src_end = b[3 * (r + 1) + 2];
        }
        return;
    }
    DevBuf<uint64_t> cost(std::max<uint32_t>(T, 1)), bound(3 * ((size_t)nranks + 1));
    if (T) {
        task_costs_kernel<<<blocks_for(T), kNT, 0, st>>>(P, er, cost.p);
        PRGPU_LAUNCHED("task_costs");
        size_t tmp = 0;
        PRGPU_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cost.p, cost.p, (int64_t)T, st));
        DevBuf<char> t(std::max<size_t>(tmp, 1));
        PRGPU_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, cost.p, cost.p, (int64_t)T, st));
        g_launches.fetch_add(1);
    }
    partition_kernel<<<1, 64, 0, st>>>(P, cost.p, er, (uint32_t)nranks, g->row_of_src.p, g->nsrc, bound.p);
    PRGPU_LAUNCHED("partition");
    std::vector<uint64_t> b(3 * ((size_t)nranks + 1));
    PRGPU_CUDA(cudaMemcpyAsync(b.data(), bound.p, b.size() * 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    for (int r = 1; r <= nranks; ++r) // monotone after the row-boundary adjustment
        for (int f = 0; f < 3; ++f) b[3 * r + f] = std::max(b[3 * r + f], b[3 * (r - 1) + f]);
    s->parts.resize(nranks);
    for (int r = 0; r < nranks; ++r) {
        prgpu_partition& q = s->parts[r];
        q.task_begin = (uint32_t)b[3 * r];
        q.task_end = (uint32_t)b[3 * (r + 1)];
        q.row_begin = (uint32_t)b[3 * r + 1];
        q.row_end = (uint32_t)b[3 * (r + 1) + 1];
        q.src_begin = b[3 * r + 2];
        q.src_end = b[3 * (r + 1) + 2];
    }
}

// Contribution buffer of a partition session (doubles): both parities of the
// run's rows, then of every narrower lane mode a K > 1 run can switch to (the
// fused exchange maps the whole allocation into the peers once).
uint64_t part_contrib_doubles(const prgpu_graph* g, const LaneCfg& c, int K) {
    const uint64_t nsrc = std::max<uint64_t>(g->nsrc, 1);
    uint64_t lanes = (uint64_t)c.KS;
    if (K > 1)
        for (int kp = 1; kp < c.KP(); kp *= 2) lanes += (uint64_t)kp;
    return 2 * nsrc * lanes;
}

prgpu_session* session_create(prgpu_graph* g, const prgpu_params* p, bool build_graph, int rank = 0,
                              int nranks = 0, double* ext_contrib = nullptr, double* ext_rp = nullptr) {
    validate_params(p);
    if (!g || g->n == 0) fail(PRGPU_EINVAL, "pagerank: graph has no vertices");
    if (g->shard_n > 1 && (nranks != g->shard_n || rank != g->shard_rank))
        fail(PRGPU_EINVAL, "shard graph: only rank " + std::to_string(g->shard_rank) + " of a " +
                               std::to_string(g->shard_n) + "-rank partition can run on it");
    DeviceGuard dg(g->device);
    auto s = std::make_unique<prgpu_session>();
    AllocScope scope(s->stream);
    s->g = g;
    s->K = p->lanes;
    {
        const uint32_t mask = p->stop_mask ? p->stop_mask : (1u << p->norm);
        const bool l1_only = mask == 1u && p->norm == PRGPU_NORM_L1 && !p->ref_ranks;
        s->cfg = lane_cfg(s->K, !l1_only);
        s->all_q = !l1_only;
    }
    s->KP = s->cfg.KP();
    s->max_iter = p->max_iterations;
    const size_t n = g->n, nsrc = std::max<size_t>(g->nsrc, 1);
    const int K = s->K, KP = s->KP;
    cudaStream_t st = s->stream;
    PhaseLog ph("session", st);

    const int KS = s->cfg.KS;
    // rank rows: a shard keeps its own rows' only (indexed from its first row)
    const uint32_t rank_lo = g->shard_n > 1 ? g->shard_rows[g->shard_rank] : 0u;
    const uint32_t rank_hi = g->shard_n > 1 ? g->shard_rows[g->shard_rank + 1] : (uint32_t)n;
    // rows without in-edges never store a rank (their value is c0): rows
    // [rank_lo, min(rank_hi, nonempty_end)) only (C5: 99.5M of 268M rows)
    const uint32_t rank_top = std::min<uint32_t>(rank_hi, g->nonempty_end);
    const size_t rank_rows = std::max<size_t>(rank_top > rank_lo ? rank_top - rank_lo : 0, 1);
    s->rank.alloc(2 * (size_t)KS * rank_rows);
    double* cbase = ext_contrib;
    s->ext_contrib_base = ext_contrib;
    s->ext_rank_partials = ext_rp;
    if (!cbase) { // partitions: room for the narrow lane modes' buffers too (part_contrib_doubles)
        s->contrib.alloc(nranks >= 1 ? part_contrib_doubles(g, s->cfg, K) : 2 * nsrc * KS);
        cbase = s->contrib.p;
    }
    PRGPU_CUDA(cudaMemsetAsync(cbase, 0, 2 * nsrc * KS * sizeof(double), st));
    s->trace.alloc((size_t)s->max_iter * K * 4);
    {
        const size_t nt = (size_t)s->max_iter * K * 4;
        fill_f64<<<(unsigned)std::min<size_t>((nt + 255) / 256, 1024), 256, 0, st>>>(s->trace.p, nt, NAN);
        PRGPU_CUDA(cudaGetLastError());
    }
    s->lanes.alloc(K);
    s->gs.alloc(1);

    ph.mark("alloc");
    // device slots hold lanes by alpha descending (slowest-converging first),
    // so the lanes still live late in a sweep share the leading sectors of each
    // contribution row; results are mapped back to the caller's order
    s->user_of.resize(K);
    for (int k = 0; k < K; ++k) s->user_of[k] = k;
    std::stable_sort(s->user_of.begin(), s->user_of.end(),
                     [&](int a, int b) { return p->alphas[a] > p->alphas[b]; });
    s->lanes_host.resize(K);
    for (int k = 0; k < K; ++k) {
        const int u = s->user_of[k];
        LaneState& L = s->lanes_host[k];
        L = LaneState{};
        L.alpha = p->alphas[u];
        L.tol = p->tolerances ? p->tolerances[u] : p->tolerance;
        L.stop_mask = p->stop_mask ? p->stop_mask : (1u << p->norm);
        L.report_norm = p->norm;
    }
    PRGPU_CUDA(cudaMemcpyAsync(s->lanes.p, s->lanes_host.data(), K * sizeof(LaneState),
                               cudaMemcpyHostToDevice, st));
    GlobalState gsh{0, 1, 0u, s->max_iter, s->mode0, s->mode0};
    PRGPU_CUDA(cudaMemcpyAsync(s->gs.p, &gsh, sizeof(gsh), cudaMemcpyHostToDevice, st));

    if (p->ref_ranks) {
        DevBuf<double> tmp(n);
        s->ref.alloc(n);
        PRGPU_CUDA(cudaMemcpyAsync(tmp.p, p->ref_ranks, n * 8, cudaMemcpyHostToDevice, st));
        scatter_ref<<<blocks_for(n), kNT, 0, st>>>(tmp.p, g->new_of_old.p, s->ref.p, g->n);
        PRGPU_LAUNCHED("scatter_ref");
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }

    Params& P = s->P;
    P.n = g->n;
    P.K = K;
    P.row_off = g->row_off.p;
    P.col = g->col.p - g->col_base; // a shard's edges, indexed by the global row offsets
    P.rowinfo = g->rowinfo.p;
    P.rank[0] = s->rank.p - (size_t)rank_lo * KS;
    P.rank[1] = s->rank.p + (size_t)KS * rank_rows - (size_t)rank_lo * KS;
    P.rank_lo = rank_lo;
    P.rank_hi = rank_hi;
    P.ks = (uint32_t)s->cfg.KS;
    P.ref = s->ref.p;
    P.trace = s->trace.p;
    P.lanes = s->lanes.p;
    P.gs = s->gs.p;
    P.use_cond = 0;
    P.frozen_at = nullptr;
    P.fused = 0;
    P.npeers = 0;
    P.arrive = nullptr;
    if (nranks == 0) {
        s->host_frozen = mapped_slot_get();
        std::fill(s->host_frozen, s->host_frozen + K, 0);
        PRGPU_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->dev_frozen), s->host_frozen, 0));
        P.frozen_at = s->dev_frozen;
    }
    P.skip_mask = 0;
    if (const char* sk = std::getenv("PRGPU_SKIP")) P.skip_mask = (uint32_t)std::atoi(sk);
    // streams (colidx, offsets, row info) are loaded evict_first (l2mode 0);
    // PRGPU_L2MODE=2 turns the hints off (tuning).  Contributions: two
    // ping-pong buffers [parity][src][KS].
    P.l2mode = 0;
    if (const char* m = std::getenv("PRGPU_L2MODE")) P.l2mode = (uint32_t)std::atoi(m);
    P.pf = 0;
    if (const char* pf = std::getenv("PRGPU_PF")) P.pf = (uint32_t)std::atoi(pf);
    P.split = 0;
    P.hp = nullptr;
    P.ktime = nullptr;
    if (nranks == 0) { // single GPU: the in-graph kernel clock (finalize is the pull kernel's)
        s->ktime.alloc(2 * (size_t)s->max_iter);
        P.ktime = s->ktime.p;
    }
    P.gpol = 0;
    if (const char* gp = std::getenv("PRGPU_GPOL")) P.gpol = (uint32_t)std::atoi(gp);
    P.hot_src = 0;
    if (const char* h = std::getenv("PRGPU_HOT_MB")) // tuning: L2-resident source rows
        P.hot_src = (uint32_t)std::min<uint64_t>(nsrc, ((uint64_t)std::atoi(h) << 20) / (KS * sizeof(double)));
    P.cbase = cbase;
    P.cold_off[0] = 0;
    P.cold_off[1] = nsrc;
    ph.mark("params");
    try {
        seg_choose_plan(s.get(), nranks);
    } catch (const Error& e) { // no room for the plan (C5: 13 GB + 10 GB of temporaries): the unsegmented pull
        if (e.code != PRGPU_ENOMEM) throw;
        cudaGetLastError();
        s->seg = nullptr;
    }
    ph.mark("seg plan");
    build_tasks(s.get());
    ph.mark("tasks");
    try {
        build_seg_tasks(s.get());
    } catch (const Error& e) {
        if (e.code != PRGPU_ENOMEM) throw;
        cudaGetLastError();
        prgpu_session* q = s.get();
        q->seg = nullptr;
        q->seg_chunk_row.reset(); q->seg_chunk_first.reset(); q->seg_packed_r0.reset(); q->seg_task.reset(); q->seg_run_rec.reset();
        q->seg_chunk_acc.reset(); q->pacc.reset(); q->seg_row_cnt.reset();
        build_tasks(q); // packed runs over every packed row again
    }
    ph.mark("seg tasks");
    if (nranks >= 1) { // partition session (nranks == 0: the fused single-GPU run)
        if (rank < 0 || rank >= nranks) fail(PRGPU_EINVAL, "partition: rank out of range");
        plan_partition(s.get(), nranks);
        const prgpu_partition& me = s->parts[rank];
        s->part_rank = rank;
        s->nranks = nranks;
        P.task_begin = me.task_begin;
        P.task_end = me.task_end;
        P.part_mode = 1;
        P.part_rank = (uint32_t)rank;
        P.nranks = (uint32_t)nranks;
        double* rp = ext_rp;
        if (!rp) {
            // both parity blocks, so the layout is the fused exchange's too
            s->rank_partials.alloc(2 * (size_t)nranks * kNQ * KP);
            rp = s->rank_partials.p;
        }
        P.rank_partials = rp;
        build_graph = false;
    }

    ph.mark("init + tasks");
    // persistent grids: resident CTAs, but at least ~4 tasks per warp
    int dev_sms = 0;
    PRGPU_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, g->device));
    auto grid_for_cfg = [&](const LaneCfg& c, uint64_t tasks, size_t& smem) -> uint32_t {
        smem = c.smem();
        PRGPU_CUDA(cudaFuncSetAttribute((const void*)c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        PRGPU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)c.fn, kNT, smem));
        per_sm = std::max(1, per_sm);
        const uint64_t want = (tasks + kWarps * 4 - 1) / (kWarps * 4);
        return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)dev_sms * per_sm, want));
    };
    // the iteration's kernels.  Single-GPU runs with K > 1 get one kernel
    // pair per lane-width mode (narrowest first): a hub-chunk kernel that only
    // leaves CTA partials and a packed + empty kernel that finalizes; once the
    // live lanes fit a narrower mode the wide pairs exit at once.  Multi-GPU
    // partitions run the one base kernel; K = 1 see below.
    using ModeList = std::vector<std::pair<int, std::pair<LaneCfg, LaneCfg>>>; // kp, (chunk, packed)
    ModeList modes;
    // segmented sessions, per mode: wide-piece chunks + hub chunks, small-piece
    // runs, combine + packed + empty (pull_kernel PATHS 5, 8, 18)
    std::vector<std::array<LaneCfg, 3>> seg_cfgs;
    {
        const char* sp = std::getenv("PRGPU_SPLIT");   // =0: base kernel only (tuning)
        const char* mm = std::getenv("PRGPU_MODES");   // =0: widest mode only (tuning)
        // K = 1 splits into the hub-chunk and packed kernels on large graphs
        // (measured C4 -4%) and on graphs without hub rows, where the packed
        // kernel then runs at 4 CTAs/SM (C3 -19%); on C2's graph (-2.5%) and
        // small graphs (launch-bound) the one kernel wins.  PRGPU_K1SPLIT=0/1
        // and PRGPU_K1MINB (bit 0 hub, bit 1 packed kernel) override (tuning).
        const char* ks1 = std::getenv("PRGPU_K1SPLIT");
        const bool k1auto = P.n_chunk == 0 ? g->e >= (1ull << 24) : g->e >= (1ull << 29);
        const bool k1split = s->K == 1 && (s->seg || (ks1 ? std::atoi(ks1) == 1 : k1auto));
        const char* km = std::getenv("PRGPU_K1MINB");
        const int k1_minb4 = km ? std::atoi(km) : (P.n_chunk == 0 ? 2 : 0);
        const bool modal = (s->K > 1 || k1split) && !(sp && std::atoi(sp) == 0);
        if (modal) {
            const int wide = s->cfg.KP(); // (measured: 12 lanes as 4 threads x 3 lost 30%)
            for (int kp = 1; kp <= wide; kp *= 2) {
                if (kp < wide && mm && std::atoi(mm) == 0) continue;
                LaneCfg a, b;
                const int ks = kp == wide ? s->cfg.KS : kp;
                if (mode_cfg<1>(ks, kp, s->cfg.WIN, s->all_q, a, k1_minb4) &&
                    mode_cfg<2>(ks, kp, s->cfg.WIN, s->all_q, b, k1_minb4)) {
                    modes.push_back({kp, {a, b}});
                    if (s->seg) {
                        std::array<LaneCfg, 3> sc;
                        mode_cfg<5>(ks, kp, s->cfg.WIN, s->all_q, sc[0], k1_minb4);
                        mode_cfg<8>(ks, kp, s->cfg.WIN, s->all_q, sc[1], k1_minb4);
                        mode_cfg<18>(ks, kp, s->cfg.WIN, s->all_q, sc[2], k1_minb4);
                        seg_cfgs.push_back(sc);
                    }
                }
            }
            if (modes.empty() || modes.back().first != wide) modes.clear(); // no instances: base kernel
        }
        if (modes.empty() && s->seg) { // the segmented pull needs the split iteration
            const bool took_packed_rows = s->seg->n_rows > s->n_long;
            s->seg = nullptr;
            if (took_packed_rows) build_tasks(s.get()); // packed runs over every packed row again
        }
    }
    P.part_kp = (uint32_t)KP;
    // contribution buffers of the narrow modes: after the run's own buffers
    // in the same allocation for partitions (one IPC mapping covers them all),
    // separate buffers otherwise
    double* narrow_base = cbase + 2 * nsrc * KS;
    std::vector<double*> narrow_cbase;
    for (int m = 0; m + 1 < (int)modes.size(); ++m) {
        const int kp = modes[m].first;
        double* b = nullptr;
        if (nranks >= 1) {
            b = narrow_base;
            narrow_base += 2 * nsrc * kp;
        } else {
            s->mode_contrib[m].alloc(2 * nsrc * kp);
            b = s->mode_contrib[m].p;
        }
        PRGPU_CUDA(cudaMemsetAsync(b, 0, 2 * nsrc * kp * sizeof(double), st));
        narrow_cbase.push_back(b);
    }
    // one iteration's launches for a list of modes (narrowest first); fills the
    // mode table of `Q` and returns the widest partial-column need
    auto build_launches = [&](const ModeList& ml, Params& Q, std::vector<prgpu_session::Launch>& out,
                              int& mode0) -> size_t {
        Q.nmodes = ml.empty() ? 1 : (int)ml.size();
        for (int m = 0; m < kMaxModes; ++m)
            Q.mode_kp[m] = ml.empty() ? KP : (m < (int)ml.size() ? ml[m].first : KP);
        mode0 = 0;
        for (int m = Q.nmodes - 1; m >= 0; --m)
            if (Q.mode_kp[m] > K - 1) mode0 = m; // narrowest mode covering every lane
        Q.no_finalize = 0;
        // contribution buffers per mode: the widest mode uses the run's buffers
        for (int m = 0; m < kMaxModes; ++m) {
            Q.mode_cbase[m] = Q.cbase;
            Q.mode_cold_off[m][0] = Q.cold_off[0];
            Q.mode_cold_off[m][1] = Q.cold_off[1];
            Q.mode_ks[m] = s->cfg.KS;
        }
        for (int m = 0; m + 1 < (int)ml.size(); ++m) {
            const int kp = ml[m].first;
            int j = 0; // its buffer among the run's narrow modes
            while (j + 1 < (int)modes.size() && modes[j].first != kp) ++j;
            Q.mode_cbase[m] = narrow_cbase[j];
            Q.mode_cold_off[m][0] = 0;
            Q.mode_cold_off[m][1] = nsrc;
            Q.mode_ks[m] = kp;
        }
        size_t cols = 0; // partials: max over modes of kNQ * kp * columns
        out.clear();
        if (ml.empty()) {
            size_t smem = 0;
            Q.G = grid_for_cfg(s->cfg, (uint64_t)Q.task_end - Q.task_begin, smem);
            Q.gtot = Q.G;
            Q.pcol0 = 0;
            Q.mode_id = 0;
            out.push_back({s->cfg.fn, Q, smem, false});
            return (size_t)kNQ * KP * Q.gtot;
        }
        // this rank's tasks [task_begin, task_end): its hub chunks go to the
        // first kernel, its packed + empty tasks to the second
        const uint32_t T1 = Q.n_chunk;
        const uint32_t a0 = std::min(Q.task_begin, T1), a1 = std::min(Q.task_end, T1);
        const uint32_t b0 = std::max(Q.task_begin, T1), b1 = std::max(Q.task_end, b0);
        for (int m = 0; m < (int)ml.size(); ++m) {
            if (s->seg) { // segmented: wide pieces + the other hub rows' chunks; small pieces; the rest
                const LaneCfg& A = seg_cfgs[m][0];
                const LaneCfg& A2 = seg_cfgs[m][1];
                const LaneCfg& B = seg_cfgs[m][2];
                size_t sa = 0, sa2 = 0, sb = 0;
                const uint32_t t0 = std::min(s->seg_chunk_t0, T1);
                const uint32_t GA = grid_for_cfg(A, (uint64_t)s->seg_n_wchunk + (T1 - t0), sa);
                const uint32_t GA2 = s->seg_n_runs ? grid_for_cfg(A2, s->seg_n_runs, sa2) : 0;
                const uint32_t GB = grid_for_cfg(B, (uint64_t)s->seg_n_comb + (b1 - b0), sb);
                Params PM = Q;
                PM.mode_id = m;
                PM.cbase = Q.mode_cbase[m];
                PM.cold_off[0] = Q.mode_cold_off[m][0];
                PM.cold_off[1] = Q.mode_cold_off[m][1];
                if (m + 1 < (int)ml.size()) { // narrow mode: repack on entry
                    PM.G = (uint32_t)dev_sms * 8;
                    out.push_back({nullptr, PM, 0, true});
                }
                Params PA = PM, PA2 = PM, PB = PM;
                PA.gtot = PA2.gtot = PB.gtot = GA + GB;
                PA.task_begin = t0;
                PA.task_end = T1;
                PA.seg_pre = s->seg_n_wchunk;
                PA.seg_grab = 2; // (measured: 1 / 2 / 4 -> C5 482.7 / 468.6 / 467.6 ms, RMAT-24 x 11 82.6 / 83.1 / 85.4)
                if (const char* gr = std::getenv("PRGPU_SEG_GRABW")) PA.seg_grab = (uint32_t)std::min(32, std::max(1, std::atoi(gr)));
                PA2.seg_grab = 4;
                if (const char* gr = std::getenv("PRGPU_SEG_GRAB")) PA2.seg_grab = (uint32_t)std::max(1, std::atoi(gr));
                PA.G = GA;
                PA.pcol0 = 0;
                PA.no_finalize = 1;
                out.push_back({A.fn, PA, sa, false});
                if (GA2) {
                    PA2.task_begin = PA2.task_end = 0;
                    PA2.seg_pre = s->seg_n_runs;
                    PA2.G = GA2;
                    PA2.pcol0 = 0;
                    PA2.no_finalize = 1;
                    out.push_back({A2.fn, PA2, sa2, false});
                }
                PB.task_begin = b0;
                PB.task_end = b1;
                PB.seg_pre = s->seg_n_comb;
                PB.G = GB;
                PB.pcol0 = GA;
                out.push_back({B.fn, PB, sb, false});
                cols = std::max(cols, (size_t)kNQ * ml[m].first * (GA + GB));
                continue;
            }
            const LaneCfg& A = ml[m].second.first;
            const LaneCfg& B = ml[m].second.second;
            size_t sa = 0, sb = 0;
            // partitions keep a hub-chunk kernel even for an empty range: a
            // dealt plan (deal_tasks) may hand this rank hub rows later
            const uint32_t na = a1 > a0 ? a1 - a0 : (nranks >= 1 && T1 ? std::max(1u, T1 / (uint32_t)nranks) : 0u);
            const uint32_t GA = na ? grid_for_cfg(A, na, sa) : 0;
            const uint32_t GB = grid_for_cfg(B, std::max(1u, b1 - b0), sb);
            Params PM = Q;
            PM.mode_id = m;
            PM.cbase = Q.mode_cbase[m];
            PM.cold_off[0] = Q.mode_cold_off[m][0];
            PM.cold_off[1] = Q.mode_cold_off[m][1];
            if (m + 1 < (int)ml.size()) { // narrow mode: repack on entry
                PM.G = (uint32_t)dev_sms * 8;
                out.push_back({nullptr, PM, 0, true});
            }
            Params PA = PM, PB = PM;
            PA.mode_id = PB.mode_id = m;
            PA.gtot = PB.gtot = GA + GB;
            if (GA) {
                PA.task_begin = a0;
                PA.task_end = a1;
                PA.G = GA;
                PA.pcol0 = 0;
                PA.no_finalize = 1;
                out.push_back({A.fn, PA, sa, false});
            }
            PB.task_begin = b0;
            PB.task_end = b1;
            PB.G = GB;
            PB.pcol0 = GA;
            out.push_back({B.fn, PB, sb, false});
            cols = std::max(cols, (size_t)kNQ * ml[m].first * (GA + GB));
        }
        return cols;
    };
    ph.mark("modes");
    size_t part_cols = 0;
    if (nranks >= 1 && modes.size() > 1) {
        // partitions: the full mode list for the fused exchange, kept aside;
        // the widest mode alone is what runs until prgpu_part_set_peers
        s->modal_P = P;
        part_cols = build_launches(modes, s->modal_P, s->modal_launches, s->modal_mode0);
        modes.erase(modes.begin(), modes.end() - 1);
    }
    part_cols = std::max(part_cols, build_launches(modes, P, s->launches, s->mode0));
    // Split pull (single GPU): each iteration pulls the hot-source CSR first
    // (sources [0, hot): their contribution rows, the most gathered ones,
    // stay L2-resident while nothing else is gathered; row sums kept in
    // hot_part), then the cold-source CSR, whose epilogue adds the hot
    // partial.  Every pull launch of a mode becomes a hot copy (no partials,
    // no finalize) ahead of the cold original.  PRGPU_SPLIT_MB = the hot
    // table's size in the run's widest rows (0: one pass).
    const uint32_t split_hot = [&]() -> uint32_t {
        if (!kExp || nranks >= 1) return 0;
        const char* sm = std::getenv("PRGPU_SPLIT_MB");
        const uint64_t mb = sm ? (uint64_t)std::atoll(sm) : 0;
        if (!mb) return 0;
        const uint64_t h = (mb << 20) / ((uint64_t)KS * sizeof(double));
        return h >= g->nsrc ? 0u : (uint32_t)h; // everything hot: one pass
    }();
    if (split_hot && g->nonempty_end) {
        const SourceSplit& sp = graph_source_split(g, split_hot, st);
        s->hot_part.alloc((size_t)g->nonempty_end * KS);
        std::vector<prgpu_session::Launch> ls;
        for (size_t i = 0; i < s->launches.size();) {
            size_t j = i; // [i, j): one mode's launches
            while (j < s->launches.size() && s->launches[j].P.mode_id == s->launches[i].P.mode_id) ++j;
            for (size_t k = i; k < j; ++k)
                if (s->launches[k].repack) ls.push_back(s->launches[k]);
            for (size_t k = i; k < j; ++k) {
                if (s->launches[k].repack) continue;
                prgpu_session::Launch h = s->launches[k];
                h.P.split = 1;
                h.P.row_off = sp.off_hot.p;
                h.P.col = sp.col_hot.p;
                h.P.hp = s->hot_part.p;
                h.P.no_finalize = 1;
                ls.push_back(h);
            }
            for (size_t k = i; k < j; ++k) {
                if (s->launches[k].repack) continue;
                prgpu_session::Launch c = s->launches[k];
                c.P.split = 2;
                c.P.row_off = sp.off_cold.p;
                c.P.col = sp.col_cold.p;
                c.P.hp = s->hot_part.p;
                ls.push_back(c);
            }
            i = j;
        }
        s->launches = std::move(ls);
    }
    s->partials.alloc(part_cols);
    P.partials = s->partials.p;
    s->modal_P.partials = s->partials.p;
    for (auto& l : s->launches) l.P.partials = s->partials.p;
    for (auto& l : s->modal_launches) l.P.partials = s->partials.p;
    P.G = s->launches.back().P.G;
    P.gtot = s->launches.back().P.gtot;

    PRGPU_CUDA(cudaEventCreate(&s->e0));
    PRGPU_CUDA(cudaEventCreate(&s->e1));

    // PRGPU_NO_GRAPH=1: host-driven speculative launches instead of the graph
    // (ncu cannot profile kernel nodes under a conditional node)
    if (const char* ng = std::getenv("PRGPU_NO_GRAPH")) build_graph = build_graph && std::atoi(ng) == 0;
    if (build_graph) {
        // graph: WHILE(cond) { pull_kernel } — cond defaults to 1 at every launch
        PRGPU_CUDA(cudaGraphCreate(&s->graph, 0));
        cudaGraphConditionalHandle h;
        PRGPU_CUDA(cudaGraphConditionalHandleCreate(&h, s->graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        PRGPU_CUDA(cudaGraphAddNode(&cnode, s->graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        // body: per lane-width mode an IF node (narrowest first) around that
        // mode's kernels; only the mode armed by the previous finalizer runs
        uint32_t nsrc32 = (uint32_t)nsrc;
        const int nm = P.nmodes;
        cudaGraphConditionalHandle mh[kMaxModes] = {};
        cudaGraph_t mbody[kMaxModes] = {};
        cudaGraphNode_t prev_if = nullptr;
        if (nm > 1) {
            for (int m = 0; m < nm; ++m) {
                PRGPU_CUDA(cudaGraphConditionalHandleCreate(&mh[m], body, m == s->mode0 ? 1u : 0u,
                                                            cudaGraphCondAssignDefault));
                cudaGraphNodeParams ip = {};
                ip.type = cudaGraphNodeTypeConditional;
                ip.conditional.handle = mh[m];
                ip.conditional.type = cudaGraphCondTypeIf;
                ip.conditional.size = 1;
                cudaGraphNode_t inode;
                PRGPU_CUDA(cudaGraphAddNode(&inode, body, prev_if ? &prev_if : nullptr, prev_if ? 1 : 0, &ip));
                mbody[m] = ip.conditional.phGraph_out[0];
                prev_if = inode;
            }
        }
        cudaGraphNode_t prev[kMaxModes] = {};
        for (const auto& l : s->launches) {
            Params PG = l.P;
            PG.use_cond = 1;
            PG.cond = h;
            PG.use_mode_cond = nm > 1;
            for (int m = 0; m < kMaxModes; ++m) PG.mode_cond[m] = mh[m];
            const int m = nm > 1 ? PG.mode_id : 0;
            cudaGraph_t tgt = nm > 1 ? mbody[m] : body;
            cudaKernelNodeParams kp = {};
            kp.func = l.repack ? (void*)repack_kernel : (void*)l.fn;
            kp.gridDim = dim3(PG.G);
            kp.blockDim = dim3(kNT);
            kp.sharedMemBytes = (unsigned)l.smem;
            void* args[] = {&PG, &nsrc32};
            kp.kernelParams = args;
            cudaGraphNode_t node;
            PRGPU_CUDA(cudaGraphAddKernelNode(&node, tgt, prev[m] ? &prev[m] : nullptr, prev[m] ? 1 : 0, &kp));
            prev[m] = node;
        }
        PRGPU_CUDA(cudaGraphInstantiate(&s->exec, s->graph, 0));
        s->use_graph = true;
    }
    PRGPU_CUDA(cudaStreamSynchronize(st));
    ph.mark("graph");
    return s.release();
}

void part_plan_copy(prgpu_session* s, prgpu_partition* parts) {
    if (s->parts.empty()) fail(PRGPU_EINVAL, "not a partition session");
    std::copy(s->parts.begin(), s->parts.end(), parts);
}

void part_set_stream(prgpu_session* s, void* stream) { s->ext_stream = (cudaStream_t)stream; }

// need[src] bit q: some row of rank q has source src as an in-neighbour (one
// warp per row; rows of rank q are [bound[q], bound[q+1]))
__global__ void need_kernel(const uint64_t* __restrict__ row_off, const uint32_t* __restrict__ col,
                            uint32_t rows, const uint32_t* __restrict__ bound, const uint8_t* __restrict__ owner,
                            int nranks, unsigned int* __restrict__ need) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += (gridDim.x * blockDim.x) >> 5) {
        int q = 0;
        if (owner) q = owner[r];
        else
            while (q + 1 < nranks && r >= bound[q + 1]) ++q;
        const uint32_t bit = 1u << q;
        for (uint64_t j = row_off[r] + lane; j < row_off[r + 1]; j += 32) {
            const uint32_t src = col[j];
            atomicOr(need + (src >> 2), bit << (8 * (src & 3)));
        }
    }
}

// Dealt partition (fused exchange): the work units — a hub row with all its
// chunk tasks, a packed run, an empty-row task — go to the ranks snake-wise
// (0..N-1, N-1..0, ...) within each kind, so every rank pulls a similar
// share of the hottest rows and, above all, publishes a similar share of the
// most-gathered sources (contiguous cost ranges put all hub rows, whose
// sources every rank gathers, on the first ranks: its NVLink egress bounded
// the iteration).  Each rank gets its ascending task list and every row's
// owner.  Needs the split iteration (hub-chunk and packed kernels) and
// PRGPU_DEAL != 0.
__global__ void fill_owner(uint8_t* __restrict__ owner, uint32_t lo, uint32_t hi, uint8_t q) {
    for (uint32_t r = lo + blockIdx.x * blockDim.x + threadIdx.x; r < hi; r += gridDim.x * blockDim.x) owner[r] = q;
}

void deal_tasks(prgpu_session* s) {
    s->dealt = false;
    Params& P = s->P;
    P.task_list = nullptr;
    P.row_owner = nullptr;
    const char* dv = std::getenv("PRGPU_DEAL");
    const int N = s->nranks;
    bool split = false;
    for (const auto& l : s->launches) split |= l.P.no_finalize != 0;
    if (N < 2 || (dv && std::atoi(dv) == 0) || !split) return;
    if (s->g->shard_n > 1) return; // a shard holds one contiguous row range's edges
    cudaStream_t st = s->stream;
    const uint32_t n = s->g->n, nl = s->n_long, T1 = P.n_chunk, np = P.n_packed, ne = P.n_empty_tasks;
    std::vector<uint32_t> cf((size_t)nl + 1), pr((size_t)np + 1);
    PRGPU_CUDA(cudaMemcpyAsync(cf.data(), s->chunk_first.p, cf.size() * 4, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaMemcpyAsync(pr.data(), s->packed_r0.p, pr.size() * 4, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    auto snake = [N](uint32_t u) { const uint32_t r = u / N, q = u % N; return (r & 1) ? N - 1 - q : q; };
    const int me = s->part_rank;
    std::vector<uint32_t> list;
    std::vector<uint8_t> owner(n, 0); // rows without a task (isolated) stay on rank 0
    for (uint32_t u = 0; u < nl; ++u) {
        const uint32_t q = snake(u);
        owner[u] = (uint8_t)q;
        if ((int)q == me)
            for (uint32_t t = cf[u]; t < cf[u + 1]; ++t) list.push_back(t);
    }
    const uint32_t split_at = (uint32_t)list.size();
    for (uint32_t k = 0; k < np; ++k) {
        const uint32_t q = snake(k);
        std::fill(owner.begin() + pr[k], owner.begin() + pr[k + 1], (uint8_t)q);
        if ((int)q == me) list.push_back(T1 + k);
    }
    for (uint32_t e = 0; e < ne; ++e) {
        const uint32_t q = snake(e);
        const uint64_t lo = (uint64_t)P.empty_begin + (uint64_t)e * P.er, hi = std::min<uint64_t>(lo + P.er, n);
        std::fill(owner.begin() + lo, owner.begin() + hi, (uint8_t)q);
        if ((int)q == me) list.push_back(T1 + np + e);
    }
    s->task_list.alloc(std::max<size_t>(list.size(), 1));
    s->row_owner.alloc(n);
    if (!list.empty())
        PRGPU_CUDA(cudaMemcpyAsync(s->task_list.p, list.data(), list.size() * 4, cudaMemcpyHostToDevice, st));
    PRGPU_CUDA(cudaMemcpyAsync(s->row_owner.p, owner.data(), n, cudaMemcpyHostToDevice, st));
    PRGPU_CUDA(cudaStreamSynchronize(st)); // host vectors go out of scope
    s->deal_split = split_at;
    s->deal_total = (uint32_t)list.size();
    P.task_list = s->task_list.p;
    P.row_owner = s->row_owner.p;
    s->dealt = true;
}

// rows this rank stores into peers per iteration (widest mode): for each
// source of its rows, the peers that gather it (all peers without a mask)
__global__ void sent_rows_kernel(const uint2* __restrict__ rowinfo, uint32_t row_begin, uint32_t row_end,
                                 const uint8_t* __restrict__ owner, int me, const uint8_t* __restrict__ need,
                                 uint32_t others, int npeers, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (uint32_t r = row_begin + blockIdx.x * blockDim.x + threadIdx.x; r < row_end; r += gridDim.x * blockDim.x) {
        const uint2 ri = rowinfo[r];
        if (ri.x && (!owner || owner[r] == me))
            c += need ? (unsigned long long)__popc(need[ri.y] & others) : (unsigned long long)npeers;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// this rank's bit of the exchange mask from its own rows only (a shard sees
// no other rows): bits[src] |= 1 << rank for every source its rows gather
__global__ void need_local_kernel(const uint64_t* __restrict__ row_off, const uint32_t* __restrict__ col,
                                  uint32_t r0, uint32_t r1, uint32_t bit, unsigned int* __restrict__ need) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t r = r0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); r < r1;
         r += (gridDim.x * blockDim.x) >> 5)
        for (uint64_t j = row_off[r] + lane; j < row_off[r + 1]; j += 32) {
            const uint32_t src = col[j];
            atomicOr(need + (src >> 2), bit << (8 * (src & 3)));
        }
}

void part_need_local(prgpu_session* s, uint8_t* dev_bits) {
    DeviceGuard dg(s->g->device);
    if (s->parts.empty()) fail(PRGPU_EINVAL, "not a partition session");
    if (s->nranks > 8) fail(PRGPU_EINVAL, "need mask: at most 8 ranks (one byte per source)");
    const uint32_t nsrc = std::max<uint32_t>(s->g->nsrc, 1);
    if (reinterpret_cast<uintptr_t>(dev_bits) % 4) fail(PRGPU_EINVAL, "need mask: buffer must be 4-byte aligned");
    PRGPU_CUDA(cudaMemsetAsync(dev_bits, 0, (size_t)(nsrc + 3) / 4 * 4, s->cur()));
    const prgpu_partition& me = s->parts[s->part_rank];
    const uint32_t r1 = std::min(me.row_end, s->P.empty_begin);
    if (r1 > me.row_begin) {
        need_local_kernel<<<(unsigned)std::min<uint64_t>(((uint64_t)(r1 - me.row_begin) * 32 + kNT - 1) / kNT,
                                                         148ull * 64),
                            kNT, 0, s->cur()>>>(s->P.row_off, s->P.col, me.row_begin, r1, 1u << s->part_rank,
                                                reinterpret_cast<unsigned int*>(dev_bits));
        PRGPU_LAUNCHED("need_local");
    }
    PRGPU_CUDA(cudaStreamSynchronize(s->cur()));
}

void part_set_need(prgpu_session* s, const uint8_t* dev_bits) {
    DeviceGuard dg(s->g->device);
    if (s->parts.empty()) fail(PRGPU_EINVAL, "not a partition session");
    const uint32_t nsrc = std::max<uint32_t>(s->g->nsrc, 1);
    s->need.alloc((nsrc + 3) / 4);
    PRGPU_CUDA(cudaMemcpyAsync(s->need.p, dev_bits, (size_t)(nsrc + 3) / 4 * 4, cudaMemcpyDeviceToDevice, s->cur()));
    PRGPU_CUDA(cudaStreamSynchronize(s->cur()));
    s->need_given = true;
}

// Fused exchange over peer memory (Params::fused): the peers' buffers as
// device pointers valid in this process (CUDA IPC or same-device buffers),
// and the iteration loop as a CUDA graph WHILE { pull ; finalize } that runs
// with no host involvement until every lane has stopped.
void part_set_peers(prgpu_session* s, int npeers, double* const* peer_contrib, double* const* peer_rp,
                    unsigned int* const* peer_arrive, unsigned int* arrive) {
    DeviceGuard dg(s->g->device);
    if (s->parts.empty()) fail(PRGPU_EINVAL, "not a partition session");
    if (npeers < 0 || npeers > kMaxPeers || npeers != s->nranks - 1)
        fail(PRGPU_EINVAL, "set_peers: npeers must be nranks - 1 (<= " + std::to_string(kMaxPeers) + ")");
    if (!arrive) fail(PRGPU_EINVAL, "set_peers: null arrival counter");
    if (!s->ext_contrib_base || !s->ext_rank_partials)
        fail(PRGPU_EINVAL, "set_peers: the session needs caller-provided contribution and rank-partial buffers "
                           "(prgpu_part_session_create ext_contrib / ext_rank_partials, sized by "
                           "prgpu_part_buffer_sizes)");
    // the fused exchange runs the lane-width modes (their buffers live in the
    // same caller allocation, mapped by the peers at the same offsets);
    // PRGPU_PART_MODES=0 keeps the widest mode only (tuning)
    const char* pm = std::getenv("PRGPU_PART_MODES");
    if (!s->modal_launches.empty() && !(pm && std::atoi(pm) == 0)) {
        Params& M = s->modal_P;
        Params& P0 = s->P;
        P0.nmodes = M.nmodes;
        for (int m = 0; m < kMaxModes; ++m) {
            P0.mode_kp[m] = M.mode_kp[m];
            P0.mode_cbase[m] = M.mode_cbase[m];
            P0.mode_cold_off[m][0] = M.mode_cold_off[m][0];
            P0.mode_cold_off[m][1] = M.mode_cold_off[m][1];
            P0.mode_ks[m] = M.mode_ks[m];
        }
        s->launches = s->modal_launches;
        s->mode0 = s->modal_mode0;
        s->modal_launches.clear();
    }
    Params& P = s->P;
    P.fused = 1;
    P.npeers = npeers;
    for (int q = 0; q < npeers; ++q)
        if (!peer_contrib[q] || !peer_rp[q] || !peer_arrive[q]) fail(PRGPU_EINVAL, "set_peers: null peer pointer");
    P.arrive = arrive;
    deal_tasks(s); // before the exchange mask: it decides which rank owns each row
    // only the peers that gather a source receive its row (PRGPU_NEED=0: all)
    P.need = nullptr;
    const char* nv = std::getenv("PRGPU_NEED");
    if (s->need_given && npeers > 0 && !(nv && std::atoi(nv) == 0))
        P.need = reinterpret_cast<const uint8_t*>(s->need.p); // a shard's, OR-reduced over the ranks
    // (a shard sees only its own rows' in-neighbours: every row goes to every peer)
    if (npeers > 0 && !(nv && std::atoi(nv) == 0) && s->g->shard_n <= 1) {
        const uint32_t nsrc = std::max<uint32_t>(s->g->nsrc, 1);
        s->need.alloc((nsrc + 3) / 4);
        PRGPU_CUDA(cudaMemsetAsync(s->need.p, 0, (size_t)(nsrc + 3) / 4 * 4, s->stream));
        std::vector<uint32_t> hb(s->nranks + 1);
        for (int q = 0; q < s->nranks; ++q) hb[q] = s->parts[q].row_begin;
        hb[s->nranks] = s->parts[s->nranks - 1].row_end;
        DevBuf<uint32_t> bound(hb.size());
        PRGPU_CUDA(cudaMemcpyAsync(bound.p, hb.data(), hb.size() * 4, cudaMemcpyHostToDevice, s->stream));
        const uint32_t rows = s->P.empty_begin; // rows with in-edges
        if (rows) {
            need_kernel<<<(unsigned)std::min<uint64_t>(((uint64_t)rows * 32 + kNT - 1) / kNT, 148ull * 64), kNT, 0,
                          s->stream>>>(s->g->row_off.p, s->g->col.p, rows, bound.p, P.row_owner, s->nranks,
                                       s->need.p);
            PRGPU_LAUNCHED("need");
        }
        PRGPU_CUDA(cudaStreamSynchronize(s->stream));
        P.need = reinterpret_cast<const uint8_t*>(s->need.p);
    }
    // every launch: the shared fields, its own grid / tasks / mode buffers, and
    // the peers' copy of its buffers (same offset in the peers' allocation)
    for (auto& l : s->launches) {
        Params keep = l.P;
        l.P = P;
        l.P.G = keep.G;
        l.P.gtot = keep.gtot;
        l.P.pcol0 = keep.pcol0;
        l.P.task_begin = keep.task_begin;
        l.P.task_end = keep.task_end;
        l.P.no_finalize = keep.no_finalize; // split: hub-chunk kernel, then packed + finalize
        l.P.mode_id = keep.mode_id;
        if (s->dealt) { // hub-chunk kernels take the list's chunk tasks, the others the rest
            const bool hub = keep.no_finalize != 0; // the split iteration's first kernel
            l.P.list_begin = hub ? 0u : s->deal_split;
            l.P.list_end = hub ? s->deal_split : s->deal_total;
        }
        l.P.cbase = keep.cbase;
        l.P.cold_off[0] = keep.cold_off[0];
        l.P.cold_off[1] = keep.cold_off[1];
        for (int q = 0; q < npeers; ++q) {
            l.P.peer_cbase[q] = peer_contrib[q] + (l.P.cbase - s->ext_contrib_base);
            l.P.peer_rp[q] = peer_rp[q];
            l.P.peer_arrive[q] = peer_arrive[q];
        }
    }
    for (int q = 0; q < npeers; ++q) {
        P.peer_cbase[q] = peer_contrib[q] + (P.cbase - s->ext_contrib_base);
        P.peer_rp[q] = peer_rp[q];
        P.peer_arrive[q] = peer_arrive[q];
    }
    {
        const prgpu_partition& me = s->parts[s->part_rank];
        const uint32_t others = ((1u << s->nranks) - 1u) & ~(1u << s->part_rank);
        DevBuf<unsigned long long> cnt(1);
        PRGPU_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), s->stream));
        const uint32_t rb = s->dealt ? 0u : me.row_begin, re = s->dealt ? s->g->n : me.row_end;
        if (re > rb)
            sent_rows_kernel<<<blocks_for(re - rb), kNT, 0, s->stream>>>(
                s->g->rowinfo.p, rb, re, P.row_owner, s->part_rank, P.need, others, npeers, cnt.p);
        PRGPU_LAUNCHED("sent_rows");
        unsigned long long c = 0;
        PRGPU_CUDA(cudaMemcpyAsync(&c, cnt.p, sizeof(c), cudaMemcpyDeviceToHost, s->stream));
        PRGPU_CUDA(cudaStreamSynchronize(s->stream));
        s->sent_rows = c;
    }
    if (s->exec) { cudaGraphExecDestroy(s->exec); s->exec = nullptr; }
    if (s->graph) { cudaGraphDestroy(s->graph); s->graph = nullptr; }
    // WHILE { per mode an IF node (narrowest first) around its kernels ; finalize }
    PRGPU_CUDA(cudaGraphCreate(&s->graph, 0));
    cudaGraphConditionalHandle h;
    PRGPU_CUDA(cudaGraphConditionalHandleCreate(&h, s->graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cnode;
    PRGPU_CUDA(cudaGraphAddNode(&cnode, s->graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    const int nm = P.nmodes;
    cudaGraphConditionalHandle mh[kMaxModes] = {};
    cudaGraph_t mbody[kMaxModes] = {};
    cudaGraphNode_t last = nullptr; // the node the finalize kernel follows
    if (nm > 1) {
        for (int m = 0; m < nm; ++m) {
            PRGPU_CUDA(cudaGraphConditionalHandleCreate(&mh[m], body, m == s->mode0 ? 1u : 0u,
                                                        cudaGraphCondAssignDefault));
            cudaGraphNodeParams ip = {};
            ip.type = cudaGraphNodeTypeConditional;
            ip.conditional.handle = mh[m];
            ip.conditional.type = cudaGraphCondTypeIf;
            ip.conditional.size = 1;
            cudaGraphNode_t inode;
            PRGPU_CUDA(cudaGraphAddNode(&inode, body, last ? &last : nullptr, last ? 1 : 0, &ip));
            mbody[m] = ip.conditional.phGraph_out[0];
            last = inode;
        }
    }
    uint32_t nsrc32 = std::max<uint32_t>(s->g->nsrc, 1);
    cudaGraphNode_t prev[kMaxModes] = {};
    for (const auto& l : s->launches) {
        Params PG = l.P;
        PG.use_cond = 1;
        PG.cond = h;
        PG.use_mode_cond = 0; // the finalize kernel arms the next mode
        const int m = nm > 1 ? PG.mode_id : 0;
        cudaGraph_t tgt = nm > 1 ? mbody[m] : body;
        cudaGraphNode_t* dep = nm > 1 ? (prev[m] ? &prev[m] : nullptr) : (last ? &last : nullptr);
        cudaKernelNodeParams kp = {};
        kp.func = l.repack ? (void*)repack_kernel : (void*)l.fn;
        kp.gridDim = dim3(PG.G);
        kp.blockDim = dim3(kNT);
        kp.sharedMemBytes = (unsigned)l.smem;
        void* args[] = {&PG, &nsrc32};
        kp.kernelParams = args;
        cudaGraphNode_t node;
        PRGPU_CUDA(cudaGraphAddKernelNode(&node, tgt, dep, dep ? 1 : 0, &kp));
        if (nm > 1) prev[m] = node;
        else last = node;
    }
    {
        Params PF = P;
        PF.use_cond = 1;
        PF.cond = h;
        PF.use_mode_cond = nm > 1;
        for (int m = 0; m < kMaxModes; ++m) PF.mode_cond[m] = mh[m];
        cudaKernelNodeParams kp = {};
        kp.func = (void*)s->cfg.fin;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(kNT);
        void* args[] = {&PF};
        kp.kernelParams = args;
        cudaGraphNode_t node;
        PRGPU_CUDA(cudaGraphAddKernelNode(&node, body, last ? &last : nullptr, last ? 1 : 0, &kp));
    }
    PRGPU_CUDA(cudaGraphInstantiate(&s->exec, s->graph, 0));
    s->use_graph = true;
}

void part_sent_rows(prgpu_session* s, uint64_t* rows, uint32_t* row_doubles) {
    if (s->parts.empty()) fail(PRGPU_EINVAL, "not a partition session");
    *rows = s->sent_rows;
    *row_doubles = (uint32_t)s->cfg.KS;
}

// the whole fused partitioned loop, enqueued on the session's stream
void part_launch(prgpu_session* s) {
    DeviceGuard dg(s->g->device);
    if (!s->P.fused || !s->exec) fail(PRGPU_EINVAL, "part_launch: call prgpu_part_set_peers first");
    PRGPU_CUDA(cudaGraphLaunch(s->exec, s->cur()));
    g_launches.fetch_add(1);
}

void graph_permutation(const prgpu_graph* g, uint32_t* old_of_new) {
    DeviceGuard dg(g->device);
    PRGPU_CUDA(cudaMemcpy(old_of_new, g->old_of_new.p, (size_t)g->n * 4, cudaMemcpyDeviceToHost));
}

void part_sizes(prgpu_graph* g, const prgpu_params* p, int nranks, uint64_t* contrib, uint64_t* partials) {
    validate_params(p);
    if (!g || nranks < 1) fail(PRGPU_EINVAL, "partition: bad graph or nranks");
    const uint32_t mask = p->stop_mask ? p->stop_mask : (1u << p->norm);
    const bool l1_only = mask == 1u && p->norm == PRGPU_NORM_L1 && !p->ref_ranks;
    const LaneCfg c = lane_cfg(p->lanes, !l1_only);
    *contrib = part_contrib_doubles(g, c, p->lanes);
    *partials = (uint64_t)nranks * kNQ * c.KP();
}

void session_destroy(prgpu_session* s) {
    if (!s) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->g->device);
    // buffers return to the pool on the session's own stream (destroyed after
    // them) once all queued work — ours and a partition caller's — is done
    cudaStreamSynchronize(s->cur());
    cudaStreamSynchronize(s->stream);
    {
        AllocScope scope(s->stream);
        delete s;
    }
    cudaSetDevice(prev);
}

void session_init(prgpu_session* s) {
    // pageable host sources: the copies are staged before the call returns
    PRGPU_CUDA(cudaMemcpyAsync(s->lanes.p, s->lanes_host.data(), s->K * sizeof(LaneState),
                               cudaMemcpyHostToDevice, s->cur()));
    GlobalState gsh{0, 1, 0u, s->max_iter, s->mode0, s->mode0};
    PRGPU_CUDA(cudaMemcpyAsync(s->gs.p, &gsh, sizeof(gsh), cudaMemcpyHostToDevice, s->cur()));
    launch_init(s->cfg, s->P, s->g->ndangling, s->cur());
    s->host_iter = 0;
    if (s->P.fused && s->P.arrive) // peers add to it only after the caller's barrier
        PRGPU_CUDA(cudaMemsetAsync(s->P.arrive, 0, sizeof(unsigned int), s->cur()));
    if (s->host_frozen) std::fill(s->host_frozen, s->host_frozen + s->K, 0); // no kernel in flight
    if (s->ktime.p) // starts = max (atomicMin), ends = 0
        PRGPU_CUDA(cudaMemsetAsync(s->ktime.p, 0xFF, s->ktime.bytes(), s->cur()));
}

// per-iteration device time of the last run's pull kernels, measured inside
// the CUDA graph (earliest CTA start to the finalizing CTA's end, ns clock):
// returns the iterations filled
int session_kernel_times(prgpu_session* s, double* ms, int cap) {
    DeviceGuard dg(s->g->device);
    if (!s->ktime.p) fail(PRGPU_EINVAL, "kernel_times: single-GPU sessions only");
    std::vector<unsigned long long> t(s->ktime.n);
    PRGPU_CUDA(cudaMemcpyAsync(t.data(), s->ktime.p, s->ktime.bytes(), cudaMemcpyDeviceToHost, s->cur()));
    PRGPU_CUDA(cudaStreamSynchronize(s->cur()));
    int n = 0;
    for (int i = 0; i < s->max_iter && n < cap; ++i) {
        if (t[2 * i] == ~0ull || t[2 * i + 1] == ~0ull || t[2 * i + 1] < t[2 * i]) break;
        ms[n++] = (double)(t[2 * i + 1] - t[2 * i]) * 1e-6;
    }
    return n;
}

void launch_pull(prgpu_session* s) {
    const uint32_t nsrc = std::max<uint32_t>(s->g->nsrc, 1);
    for (const auto& l : s->launches) {
        Params P = l.P;
        P.use_cond = 0;
        if (l.repack) repack_kernel<<<P.G, kNT, 0, s->cur()>>>(P, nsrc);
        else l.fn<<<P.G, kNT, l.smem, s->cur()>>>(P);
        PRGPU_LAUNCHED("pull_kernel");
    }
}

int read_any_active(prgpu_session* s) {
    GlobalState gsh;
    PRGPU_CUDA(cudaMemcpyAsync(&gsh, s->gs.p, sizeof(gsh), cudaMemcpyDeviceToHost, s->cur()));
    PRGPU_CUDA(cudaStreamSynchronize(s->cur()));
    return gsh.any_active;
}

// ---- partition sessions ----------------------------------------------------------
void part_exchange(prgpu_session* s, prgpu_exchange* ex) {
    const int KS = s->cfg.KS;
    ex->contrib[0] = s->P.cbase + s->P.cold_off[0] * KS;
    ex->contrib[1] = s->P.cbase + s->P.cold_off[1] * KS;
    ex->stride = (uint32_t)KS;
    ex->nsrc = std::max<uint64_t>(s->g->nsrc, 1);
    ex->rank_partials = s->P.rank_partials;
    ex->partials_per_rank = (uint32_t)(kNQ * s->KP);
}

int part_step(prgpu_session* s) {
    DeviceGuard dg(s->g->device);
    launch_pull(s);
    return ++s->host_iter & 1; // the buffer this iteration wrote
}

void part_finalize(prgpu_session* s) {
    DeviceGuard dg(s->g->device);
    s->cfg.fin<<<1, kNT, 0, s->cur()>>>(s->P); // fused: waits for the peers' arrivals
    PRGPU_LAUNCHED("part_finalize");
}

void part_local_ranks_device(prgpu_session* s, double* out, uint64_t ld) {
    DeviceGuard dg(s->g->device);
    if (s->parts.empty()) fail(PRGPU_EINVAL, "not a partition session");
    const prgpu_partition& me = s->parts[s->part_rank];
    const uint32_t rows = me.row_end - me.row_begin;
    if (ld < rows) fail(PRGPU_EINVAL, "local_ranks_device: ld smaller than the rank's row count");
    LaneMap map{};
    for (int k = 0; k < s->K; ++k) map.user_of[k] = s->user_of[k];
    if (rows) {
        local_ranks_kernel<<<blocks_for((uint64_t)rows * s->K), kNT, 0, s->cur()>>>(s->P, map, me.row_begin, rows,
                                                                                  out, ld);
        PRGPU_LAUNCHED("local_ranks_kernel");
    }
}

void part_owned_ranks_device(prgpu_session* s, double* out, uint64_t ld, int* dealt) {
    DeviceGuard dg(s->g->device);
    if (s->parts.empty()) fail(PRGPU_EINVAL, "not a partition session");
    *dealt = s->dealt ? 1 : 0;
    if (!s->dealt || !out) return;
    if (ld < s->g->n) fail(PRGPU_EINVAL, "owned_ranks_device: ld smaller than vertex_count");
    LaneMap map{};
    for (int k = 0; k < s->K; ++k) map.user_of[k] = s->user_of[k];
    owned_ranks_kernel<<<blocks_for((uint64_t)s->g->n * s->K), kNT, 0, s->cur()>>>(s->P, map, s->row_owner.p,
                                                                                  s->part_rank, out, ld);
    PRGPU_LAUNCHED("owned_ranks_kernel");
}

void part_local_ranks(prgpu_session* s, int user_lane, double* out) {
    DeviceGuard dg(s->g->device);
    int slot = -1;
    for (int k = 0; k < s->K; ++k)
        if (s->user_of[k] == user_lane) slot = k;
    if (slot < 0) fail(PRGPU_EINVAL, "local_ranks: lane out of range");
    LaneState L;
    PRGPU_CUDA(cudaMemcpyAsync(&L, s->lanes.p + slot, sizeof(L), cudaMemcpyDeviceToHost, s->cur()));
    PRGPU_CUDA(cudaStreamSynchronize(s->cur()));
    const prgpu_partition& me = s->parts[s->part_rank];
    const uint32_t stored_end = std::min(me.row_end, s->P.empty_begin);
    if (stored_end > me.row_begin)
    {
        // one lane's column of the row-major ranks, made contiguous on the device
        AllocScope scope(s->cur());
        const uint32_t rows = stored_end - me.row_begin;
        DevBuf<double> tmp(rows);
        strided_copy<<<blocks_for(rows), kNT, 0, s->cur()>>>(
            s->P.rank[L.iterations & 1] + (size_t)me.row_begin * s->P.ks + slot, s->P.ks, tmp.p, rows);
        PRGPU_LAUNCHED("strided_copy");
        PRGPU_CUDA(cudaMemcpyAsync(out, tmp.p, (size_t)rows * 8, cudaMemcpyDeviceToHost, s->cur()));
        PRGPU_CUDA(cudaStreamSynchronize(s->cur()));
    }
    PRGPU_CUDA(cudaStreamSynchronize(s->cur()));
    for (uint32_t r = std::max(me.row_begin, stored_end); r < me.row_end; ++r) out[r - me.row_begin] = L.c0_used;
}

double session_run(prgpu_session* s) {
    DeviceGuard dg(s->g->device);
    session_init(s);
    PRGPU_CUDA(cudaEventRecord(s->e0, s->stream));
    if (s->use_graph) {
        PRGPU_CUDA(cudaGraphLaunch(s->exec, s->stream));
        g_launches.fetch_add(1);
    } else {
        // speculative windows: kernels early-exit once every lane has stopped
        for (int done = 0; done < s->max_iter;) {
            const int w = std::min(8, s->max_iter - done);
            for (int i = 0; i < w; ++i) launch_pull(s);
            done += w;
            if (!read_any_active(s)) break;
        }
    }
    PRGPU_CUDA(cudaEventRecord(s->e1, s->stream));
    PRGPU_CUDA(cudaEventSynchronize(s->e1));
    float ms = 0;
    PRGPU_CUDA(cudaEventElapsedTime(&ms, s->e0, s->e1));
    s->last_loop_ms = ms;
    return ms;
}

void session_results(prgpu_session* s, prgpu_result* out) {
    DeviceGuard dg(s->g->device);
    cudaStream_t st = s->stream;
    AllocScope scope(st);
    PhaseLog ph("results", st);
    std::vector<LaneState> L(s->K);
    PRGPU_CUDA(cudaMemcpyAsync(L.data(), s->lanes.p, s->K * sizeof(LaneState),
                               cudaMemcpyDeviceToHost, st));
    GlobalState gsh;
    PRGPU_CUDA(cudaMemcpyAsync(&gsh, s->gs.p, sizeof(gsh), cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    const size_t n = s->g->n;
    const int K = s->K;
    if (out->ranks) {
        DevBuf<double> tmp((size_t)K * n);
        extract_ranks<<<blocks_for(n), kNT, 0, st>>>(s->P, s->g->new_of_old.p, tmp.p, -1, 0);
        PRGPU_LAUNCHED("extract_ranks");
        for (int k = 0; k < K; ++k) // device slot -> caller lane
            PRGPU_CUDA(cudaMemcpyAsync(out->ranks + (size_t)s->user_of[k] * n, tmp.p + (size_t)k * n,
                                       n * 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        ph.mark("ranks d2h");
    }
    if (out->err_trace) {
        std::vector<double> tr((size_t)s->max_iter * K * 4);
        PRGPU_CUDA(cudaMemcpyAsync(tr.data(), s->trace.p, tr.size() * sizeof(double),
                                   cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        for (int it = 0; it < s->max_iter; ++it)
            for (int k = 0; k < K; ++k)
                for (int q = 0; q < 4; ++q)
                    out->err_trace[((size_t)it * K + s->user_of[k]) * 4 + q] = tr[((size_t)it * K + k) * 4 + q];
    }
    for (int k = 0; k < K; ++k) {
        const int u = s->user_of[k];
        if (out->iterations) out->iterations[u] = L[k].iterations;
        if (out->converged) out->converged[u] = (uint8_t)L[k].converged;
        if (out->final_err) out->final_err[u] = L[k].final_err;
    }
    out->run_iterations = gsh.iter;
    out->loop_ms = s->last_loop_ms;
}

// run + results with the rank copy-out overlapped: while the CUDA graph
// iterates, every lane the device reports stopped (frozen_at) is permuted to
// caller ids on a side stream and copied to the host by the copy engine, so
// only the lanes stopping at the last iteration are copied after the loop.
void session_solve(prgpu_session* s, prgpu_result* out) {
    if (!out->ranks || !s->use_graph || !s->host_frozen) {
        session_run(s);
        session_results(s, out);
        return;
    }
    DeviceGuard dg(s->g->device);
    AllocScope scope(s->stream);
    const size_t n = s->g->n;
    const int K = s->K;
    if (!s->aux) s->aux = std::make_unique<Stream>();
    cudaStream_t ax = *s->aux;
    DevBuf<double> tmp((size_t)K * n);
    Event tmp_ready;
    PRGPU_CUDA(cudaEventRecord(tmp_ready, s->stream));
    PRGPU_CUDA(cudaStreamWaitEvent(ax, tmp_ready, 0));
    session_init(s);
    PRGPU_CUDA(cudaEventRecord(s->e0, s->stream));
    PRGPU_CUDA(cudaGraphLaunch(s->exec, s->stream));
    g_launches.fetch_add(1);
    PRGPU_CUDA(cudaEventRecord(s->e1, s->stream));
    uint32_t copied = 0;
    auto copy_out = [&](int k) {
        extract_ranks<<<blocks_for(n), kNT, 0, ax>>>(s->P, s->g->new_of_old.p, tmp.p + (size_t)k * n, k, 0);
        PRGPU_LAUNCHED("extract_ranks");
        PRGPU_CUDA(cudaMemcpyAsync(out->ranks + (size_t)s->user_of[k] * n, tmp.p + (size_t)k * n, n * 8,
                                   cudaMemcpyDeviceToHost, ax));
        copied |= 1u << k;
    };
    for (;;) {
        const cudaError_t q = cudaEventQuery(s->e1);
        if (q != cudaSuccess && q != cudaErrorNotReady) PRGPU_CUDA(q);
        for (int k = 0; k < K; ++k)
            if (!((copied >> k) & 1u) && *(volatile int*)(s->host_frozen + k)) copy_out(k);
        if (q == cudaSuccess) break;
        std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
    for (int k = 0; k < K; ++k) // lanes not reported (defensive): copy after the loop
        if (!((copied >> k) & 1u)) copy_out(k);
    float ms = 0;
    PRGPU_CUDA(cudaEventElapsedTime(&ms, s->e0, s->e1));
    s->last_loop_ms = ms;
    PRGPU_CUDA(cudaStreamSynchronize(ax));
    Event done;
    PRGPU_CUDA(cudaEventRecord(done, ax));
    PRGPU_CUDA(cudaStreamWaitEvent(s->stream, done, 0)); // tmp is freed on s->stream
    prgpu_result rest = *out;
    rest.ranks = nullptr;
    session_results(s, &rest);
    out->run_iterations = rest.run_iterations;
    out->loop_ms = rest.loop_ms;
}

// ---- damping sweep as one power series ---------------------------------------------
// The reference iterates every alpha separately: r_t = alpha * M r_{t-1} +
// (1 - alpha)/N * 1 with M the column-stochastic link matrix whose dangling
// columns spread 1/N (pagerank.hpp:85-92: c0 = (1-alpha)/N + alpha*D/N).
// With r_0 = y_0 = 1/N and y_j = M^j y_0 that sequence is, exactly,
//   r_t = alpha^t y_t + (1 - alpha) sum_{j<t} alpha^j y_j,
//   r_t - r_{t-1} = alpha^t (y_t - y_{t-1}),
// so every lane's iterates and every norm of its change (the stopping rule,
// norms.hpp) follow from ONE chain y_t (an alpha = 1 run) plus per-lane
// weighted sums of it.  The chain runs until the last lane stops; each lane
// stops at the first t where alpha^t * ||y_t - y_{t-1}|| < tau for every norm
// of its stop mask (or at max_iterations), and its ranks are the weighted sum
// up to there.  Arithmetic differs from the reference's only in rounding
// (summation order), like the batched run's.
// y_t kept (rows with in-edges, in blocks of kHistBlock vectors; rows without
// hold the scalar c0 of step t) and every lane's ranks formed once at the
// end, in engine row order (coalesced), all lanes per pass: acc_k = sum_j
// w[k][j] * y_j in the order j = 0..T_k, w = (1-alpha) alpha^j for j < T_k and
// alpha^T_k at j = T_k (0 beyond).  hist[j] points at y_j.
constexpr int kHistBlock = 16;
__global__ void series_combine(const double* const* __restrict__ hist, const double* __restrict__ yempty,
                               const double* __restrict__ w /*[K][T+1]*/, int T, int K, uint32_t rows, uint32_t n,
                               double* __restrict__ acc /*[K][n] engine rows*/) {
    for (size_t r = blockIdx.x * (size_t)blockDim.x + threadIdx.x; r < n; r += (size_t)gridDim.x * blockDim.x) {
        double a[PRGPU_MAX_LANES];
#pragma unroll
        for (int k = 0; k < PRGPU_MAX_LANES; ++k) a[k] = 0.0;
        for (int j = 0; j <= T; ++j) {
            const double y = r < rows ? hist[j][r] : yempty[j];
#pragma unroll
            for (int k = 0; k < PRGPU_MAX_LANES; ++k) {
                if (k >= K) break;
                const double c = w[(size_t)k * (T + 1) + j];
                if (c != 0.0) a[k] = __dadd_rn(a[k], __dmul_rn(c, y));
            }
        }
#pragma unroll
        for (int k = 0; k < PRGPU_MAX_LANES; ++k)
            if (k < K) acc[(size_t)k * n + r] = a[k];
    }
}

// large graphs (history would not stay in the memory pool): the weighted
// sums accumulated as the chain runs, acc_k += coef_k * y_t (coef 0: lane done)
__global__ void series_accumulate(const double* __restrict__ y, uint32_t rows, double y_empty, uint32_t n,
                                  const double* __restrict__ coef, int K, double* __restrict__ acc) {
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n; v += (size_t)gridDim.x * blockDim.x) {
        const double yv = v < rows ? y[v] : y_empty;
        for (int k = 0; k < K; ++k) {
            const double c = coef[k];
            if (c != 0.0) acc[(size_t)k * n + v] = __dadd_rn(acc[(size_t)k * n + v], __dmul_rn(c, yv));
        }
    }
}

__global__ void series_permute(const double* __restrict__ acc, const uint32_t* __restrict__ new_of_old, uint32_t n,
                               double* __restrict__ out) { // out[v_orig] = acc[new_of_old[v]]
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n; v += (size_t)gridDim.x * blockDim.x)
        out[v] = acc[new_of_old[v]];
}

void pagerank_series(prgpu_graph* g, const prgpu_params* p, prgpu_result* out) {
    validate_params(p);
    if (p->ref_ranks) fail(PRGPU_EINVAL, "pagerank_series: ref_ranks not supported");
    if (!g || g->n == 0) fail(PRGPU_EINVAL, "pagerank: graph has no vertices");
    DeviceGuard dg(g->device);
    const int K = p->lanes;
    const uint32_t n = g->n;
    // the chain: one lane, alpha = 1, every norm traced, never stopping early
    const double one = 1.0;
    prgpu_params q{};
    q.lanes = 1;
    q.alphas = &one;
    q.tolerance = 1e-300;
    q.norm = PRGPU_NORM_L1;
    q.stop_mask = 7u;
    q.max_iterations = p->max_iterations;
    std::unique_ptr<prgpu_session, void (*)(prgpu_session*)> s(session_create(g, &q, false), session_destroy);
    cudaStream_t st = s->stream;
    AllocScope scope(st);
    const uint32_t rows = s->P.empty_begin; // rows the chain stores (the rest hold c0)
    std::vector<double> alpha(K), tol(K);
    std::vector<uint32_t> mask(K);
    std::vector<int> its(K, 0), conv(K, 0);
    std::vector<double> ferr(K, INFINITY);
    for (int k = 0; k < K; ++k) {
        alpha[k] = p->alphas[k];
        tol[k] = p->tolerances ? p->tolerances[k] : p->tolerance;
        mask[k] = p->stop_mask ? p->stop_mask : (1u << p->norm);
    }
    std::vector<double> trace((size_t)p->max_iterations * K * 4, NAN);
    std::vector<DevBuf<double>> blocks; // y_0, y_1, ... (rows with in-edges), kHistBlock per block
    std::vector<const double*> hist;
    std::vector<double> yempty;
    const size_t hrows = std::max<uint32_t>(rows, 1);
    // keep the chain (one combine at the end) while a block of it is small;
    // on large graphs accumulate every lane as the chain runs instead
    const char* sk = std::getenv("PRGPU_SERIES_KEEP"); // =0/1 forces the variant (tests)
    // the whole chain may reach ceil((max_iterations + 2) / kHistBlock) blocks:
    // keep it only if that many fit in half the free device memory now
    size_t free_b = 0, total_b = 0;
    PRGPU_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t block_b = hrows * kHistBlock * sizeof(double);
    const size_t max_blocks = ((size_t)p->max_iterations + 2 + kHistBlock - 1) / kHistBlock;
    const bool keep_chain = sk ? std::atoi(sk) != 0
                               : block_b <= (2ull << 30) && max_blocks * block_b <= free_b / 2;
    DevBuf<double> acc((size_t)K * n), coef(K);
    std::vector<double> pw_run(K, 1.0);
    std::vector<int> done_at(K, 0);
    if (!keep_chain) PRGPU_CUDA(cudaMemsetAsync(acc.p, 0, (size_t)K * n * sizeof(double), st));
    auto keep = [&](int parity, double y_empty) {
        if (!keep_chain) return;
        const size_t j = hist.size();
        if (j % kHistBlock == 0) blocks.emplace_back(hrows * kHistBlock);
        double* dst = blocks.back().p + (j % kHistBlock) * hrows;
        if (rows)
            PRGPU_CUDA(cudaMemcpyAsync(dst, s->P.rank[parity], (size_t)rows * sizeof(double),
                                       cudaMemcpyDeviceToDevice, st)); // K = 1: rank rows are contiguous
        hist.push_back(dst);
        yempty.push_back(y_empty);
    };
    // Host staging in pinned (mapped-pool) memory, so nothing below blocks
    // the host: per parity the chain's trace row and LaneState after a step,
    // and the in-loop variant's per-lane coefficients.
    struct StepOut {
        double tr[4];
        LaneState L;
    };
    static_assert(sizeof(StepOut) <= kSlotInts * sizeof(int), "slot too small");
    static_assert(2 * PRGPU_MAX_LANES * sizeof(double) <= kSlotInts * sizeof(int), "slot too small");
    struct SlotHold { // returned only once no copy of `st` can still target them (error paths too)
        int* p[3];
        cudaStream_t st;
        explicit SlotHold(cudaStream_t s) : st(s) { for (auto& x : p) x = mapped_slot_get(); }
        ~SlotHold() {
            cudaStreamSynchronize(st);
            for (auto* x : p) mapped_slot_put(x);
        }
    } slots(st);
    StepOut* hout[2] = {reinterpret_cast<StepOut*>(slots.p[0]), reinterpret_cast<StepOut*>(slots.p[1])};
    double* hcoef = reinterpret_cast<double*>(slots.p[2]); // [2][PRGPU_MAX_LANES]
    Event landed[2];
    // the in-loop variant: after step t every live lane adds (1 - alpha) alpha^t y_t,
    // a lane stopping at t adds alpha^t y_t and is done.  The coefficient row
    // of parity t&1 is rewritten two steps later, after the host has waited
    // for an event recorded behind this step's copy.
    auto accumulate = [&](int parity, double y_empty, int step) {
        if (keep_chain) return;
        double* cr = hcoef + (step & 1) * PRGPU_MAX_LANES;
        for (int k = 0; k < K; ++k) {
            cr[k] = 0.0;
            if (done_at[k] && done_at[k] < step) continue;
            cr[k] = (done_at[k] == step && step > 0) ? pw_run[k] : (1.0 - alpha[k]) * pw_run[k];
        }
        PRGPU_CUDA(cudaMemcpyAsync(coef.p, cr, K * sizeof(double), cudaMemcpyHostToDevice, st));
        series_accumulate<<<blocks_for(n), kNT, 0, st>>>(s->P.rank[parity], rows, y_empty, n, coef.p, K, acc.p);
        PRGPU_LAUNCHED("series_accumulate");
        for (int k = 0; k < K; ++k) pw_run[k] = pw_run[k] * alpha[k];
    };
    // step t (1-based): y_t into rank[t&1], its trace row and lane state
    // staged for the host, y_t kept; the host reads them after landed[t&1]
    auto enqueue = [&](int step) {
        launch_pull(s.get()); // y_t into rank[t&1]; trace[t-1] = norms of y_t - y_{t-1}
        StepOut* o = hout[step & 1];
        PRGPU_CUDA(cudaMemcpyAsync(o->tr, s->trace.p + (size_t)(step - 1) * 4, sizeof(o->tr),
                                   cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaMemcpyAsync(&o->L, s->lanes.p, sizeof(LaneState), cudaMemcpyDeviceToHost, st));
        keep(step & 1, 0.0);
        PRGPU_CUDA(cudaEventRecord(landed[step & 1], st));
    };
    session_init(s.get());
    cudaEvent_t e0 = s->e0, e1 = s->e1;
    PRGPU_CUDA(cudaEventRecord(e0, st));
    keep(0, 1.0 / (double)n); // y_0 = 1/N everywhere
    accumulate(0, 1.0 / (double)n, 0);
    int live = K, t = 0;
    std::vector<double> pw(K, 1.0); // alpha^t
    // One step of lookahead: step t+1 is enqueued before the host decides on
    // step t, so the GPU never waits for the host; it is skipped when the
    // chain's last decay ratio predicts every live lane is within 2x of its
    // tolerance at t (a wrong guess costs one unused pull, or one host round
    // trip: the margin favours the round trip, a pull is 36 ms on C5).
    double d1 = 0.0, d2 = 0.0; // the stop norm of the chain at t-1, t-2 (lane-independent)
    bool queued = false;       // step t+1 already enqueued
    if (p->max_iterations > 0) enqueue(1);
    while (live > 0 && t < p->max_iterations) {
        ++t;
        if (!queued && t > 1) enqueue(t);
        queued = false;
        if (t < p->max_iterations) {
            bool predict_done = false;
            if (d1 > 0.0 && d2 > 0.0) {
                const double rho = d1 / d2;
                predict_done = true;
                for (int k = 0; k < K && predict_done; ++k)
                    if (!its[k]) predict_done = pw[k] * alpha[k] * d1 * rho < 2.0 * tol[k];
            }
            if (!predict_done) {
                enqueue(t + 1);
                queued = true;
            }
        }
        PRGPU_CUDA(cudaEventSynchronize(landed[t & 1]));
        const StepOut& o = *hout[t & 1];
        const double tr[4] = {o.tr[0], o.tr[1], o.tr[2], o.tr[3]};
        const LaneState L = o.L;
        if (keep_chain) yempty[t] = L.c0_used;
        // a chain that reached a fixed point stops iterating: its later
        // differences are exactly zero
        const bool ran = t - 1 < L.iterations;
        const double e[3] = {ran ? tr[0] : 0.0, ran ? tr[1] : 0.0, ran ? tr[2] : 0.0};
        d2 = d1;
        d1 = e[p->norm];
        for (int k = 0; k < K; ++k) {
            if (its[k]) continue; // stopped earlier
            pw[k] = pw[k] * alpha[k];
            double err[3];
            for (int qn = 0; qn < 3; ++qn) err[qn] = pw[k] * e[qn];
            for (int qn = 0; qn < 3; ++qn) trace[((size_t)(t - 1) * K + k) * 4 + qn] = err[qn];
            bool stop = true; // every norm of the lane's stop mask strictly below tau (pagerank.hpp:99)
            for (int qn = 0; qn < 3; ++qn)
                if ((mask[k] >> qn) & 1u) stop = stop && err[qn] < tol[k];
            if (stop || t >= p->max_iterations) {
                its[k] = t;
                conv[k] = stop;
                ferr[k] = err[p->norm];
                done_at[k] = t;
                --live;
            }
        }
        accumulate(t & 1, L.c0_used, t);
    }
    // weights: (1-alpha) alpha^j for j < T_k, alpha^T_k at T_k
    const int T = t;
    std::vector<double> w((size_t)K * (T + 1), 0.0);
    for (int k = 0; k < K; ++k) {
        double a = 1.0;
        for (int j = 0; j <= its[k]; ++j) {
            w[(size_t)k * (T + 1) + j] = j < its[k] ? (1.0 - alpha[k]) * a : a;
            a = a * alpha[k];
        }
    }
    DevBuf<double> res((size_t)K * n);
    if (keep_chain) {
        DevBuf<const double*> d_hist(hist.size());
        DevBuf<double> d_w(w.size()), d_ye(yempty.size());
        PRGPU_CUDA(cudaMemcpyAsync(d_hist.p, hist.data(), hist.size() * sizeof(const double*),
                                   cudaMemcpyHostToDevice, st));
        PRGPU_CUDA(cudaMemcpyAsync(d_w.p, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        PRGPU_CUDA(cudaMemcpyAsync(d_ye.p, yempty.data(), yempty.size() * sizeof(double), cudaMemcpyHostToDevice, st));
        series_combine<<<blocks_for(n), kNT, 0, st>>>(d_hist.p, d_ye.p, d_w.p, T, K, rows, n, acc.p);
        PRGPU_LAUNCHED("series_combine");
        PRGPU_CUDA(cudaStreamSynchronize(st)); // host staging vectors
    }
    for (int k = 0; k < K; ++k) {
        series_permute<<<blocks_for(n), kNT, 0, st>>>(acc.p + (size_t)k * n, g->new_of_old.p, n,
                                                      res.p + (size_t)k * n);
        PRGPU_LAUNCHED("series_permute");
    }
    PRGPU_CUDA(cudaEventRecord(e1, st));
    PRGPU_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    PRGPU_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    if (out->ranks)
        PRGPU_CUDA(cudaMemcpyAsync(out->ranks, res.p, (size_t)K * n * sizeof(double), cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st)); // ptrs, w, yempty are host vectors
    for (int k = 0; k < K; ++k) {
        if (out->iterations) out->iterations[k] = its[k];
        if (out->converged) out->converged[k] = (uint8_t)conv[k];
        if (out->final_err) out->final_err[k] = ferr[k];
    }
    if (out->err_trace)
        for (size_t i = 0; i < trace.size(); ++i) out->err_trace[i] = trace[i];
    out->run_iterations = t;
    out->loop_ms = ms;
    PRGPU_CUDA(cudaStreamSynchronize(st));
}

void session_observed(prgpu_session* s, prgpu_result* out, prgpu_observer_fn fn, void* user) {
    DeviceGuard dg(s->g->device);
    cudaStream_t st = s->stream;
    const size_t n = s->g->n;
    session_init(s);
    DevBuf<double> tmp(n);
    std::vector<double> host(n);
    std::vector<LaneState> L(s->K), before(s->K);
    PRGPU_CUDA(cudaEventRecord(s->e0, st));
    for (int it = 0; it < s->max_iter; ++it) {
        PRGPU_CUDA(cudaMemcpyAsync(before.data(), s->lanes.p, s->K * sizeof(LaneState),
                                   cudaMemcpyDeviceToHost, st));
        launch_pull(s);
        PRGPU_CUDA(cudaMemcpyAsync(L.data(), s->lanes.p, s->K * sizeof(LaneState),
                                   cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < s->K; ++k) {
            if (!before[k].active || !fn) continue;
            extract_ranks<<<blocks_for(n), kNT, 0, st>>>(s->P, s->g->new_of_old.p, tmp.p, k, 1);
            PRGPU_LAUNCHED("extract_ranks");
            PRGPU_CUDA(cudaMemcpyAsync(host.data(), tmp.p, n * 8, cudaMemcpyDeviceToHost, st));
            PRGPU_CUDA(cudaStreamSynchronize(st));
            fn(L[k].iterations, s->user_of[k], host.data(), n, L[k].final_err, user);
        }
        if (!read_any_active(s)) break;
    }
    PRGPU_CUDA(cudaEventRecord(s->e1, st));
    PRGPU_CUDA(cudaEventSynchronize(s->e1));
    float ms = 0;
    PRGPU_CUDA(cudaEventElapsedTime(&ms, s->e0, s->e1));
    s->last_loop_ms = ms;
    session_results(s, out);
}

// device memory held by a graph / a session (its DevBufs)
uint64_t graph_device_bytes(const prgpu_graph* g) {
    uint64_t b = g->row_off.bytes() + g->col.bytes() + g->deg.bytes() + g->rowinfo.bytes() + g->row_of_src.bytes() +
                 g->new_of_old.bytes() + g->old_of_new.bytes();
    for (const auto& kv : g->splits)
        b += kv.second->off_hot.bytes() + kv.second->off_cold.bytes() + kv.second->col_hot.bytes() +
             kv.second->col_cold.bytes();
    for (const auto& kv : g->seg_plans) b += kv.second->bytes();
    return b;
}
uint64_t session_device_bytes(const prgpu_session* s) {
    uint64_t b = s->rank.bytes() + s->contrib.bytes() + s->partials.bytes() + s->trace.bytes() + s->ref.bytes() +
                 s->chunk_acc.bytes() + s->hot_part.bytes() + s->lanes.bytes() + s->gs.bytes() +
                 s->chunk_row.bytes() + s->chunk_first.bytes() + s->packed_r0.bytes() + s->row_cnt.bytes() +
                 s->task_list.bytes() + s->row_owner.bytes() + s->rank_partials.bytes() + s->need.bytes() +
                 s->ktime.bytes() + s->seg_chunk_row.bytes() + s->seg_chunk_first.bytes() + s->seg_task.bytes() + s->seg_run_rec.bytes() + s->run_rec.bytes() +
                 s->seg_packed_r0.bytes() + s->seg_chunk_acc.bytes() + s->pacc.bytes() + s->seg_row_cnt.bytes();
    for (const auto& m : s->mode_contrib) b += m.bytes();
    return b;
}

double session_time_pull(prgpu_session* s, int launches) {
    // Device time of one iteration's pull kernels, as the CUDA graph runs
    // them: a host-driven pass to convergence (at most `launches`
    // iterations) that launches, per iteration, only the kernels of the lane
    // mode the finalizer armed (plus its repack on a mode change) — the
    // graph's IF nodes skip the others — between ONE event pair.  Mean over
    // the iterations; x iterations it is below the graph loop's time (which
    // adds the conditional-node overhead).
    DeviceGuard dg(s->g->device);
    session_init(s);
    cudaStream_t st = s->cur();
    const uint32_t nsrc = std::max<uint32_t>(s->g->nsrc, 1);
    std::vector<cudaEvent_t> ev(2 * (size_t)launches);
    for (auto& e : ev) PRGPU_CUDA(cudaEventCreate(&e));
    int done = 0;
    GlobalState gsh;
    PRGPU_CUDA(cudaMemcpyAsync(&gsh, s->gs.p, sizeof(gsh), cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    // PRGPU_PERSIST_MB (tuning, host-driven runs only): an L2 persisting
    // access-policy window over the first X MB of the parity this iteration
    // gathers from (the hottest sources, ids in degree order)
    const char* pmb = std::getenv("PRGPU_PERSIST_MB");
    const size_t persist_b = (kExp && pmb) ? ((size_t)std::atoi(pmb) << 20) : 0;
    if (persist_b) {
        int maxp = 0;
        PRGPU_CUDA(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, s->g->device));
        PRGPU_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(persist_b, (size_t)maxp)));
    }
    for (; done < launches && gsh.any_active; ++done) {
        if (persist_b) {
            const Params& P0 = s->P;
            const int par = gsh.iter & 1;
            int mode = gsh.mode;
            const double* base = P0.mode_cbase[mode] + P0.mode_cold_off[mode][par] * P0.mode_ks[mode];
            cudaStreamAttrValue av = {};
            av.accessPolicyWindow.base_ptr = (void*)base;
            av.accessPolicyWindow.num_bytes = persist_b;
            av.accessPolicyWindow.hitRatio = 1.0f;
            av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            PRGPU_CUDA(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
        }
        PRGPU_CUDA(cudaEventRecord(ev[2 * done], st));
        for (const auto& l : s->launches) {
            if (l.P.mode_id != gsh.mode) continue;
            if (l.repack && gsh.layout == gsh.mode) continue;
            Params P = l.P;
            P.use_cond = 0;
            if (l.repack) repack_kernel<<<P.G, kNT, 0, st>>>(P, nsrc);
            else l.fn<<<P.G, kNT, l.smem, st>>>(P);
            PRGPU_LAUNCHED("pull_kernel");
        }
        PRGPU_CUDA(cudaEventRecord(ev[2 * done + 1], st));
        PRGPU_CUDA(cudaMemcpyAsync(&gsh, s->gs.p, sizeof(gsh), cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
    if (persist_b) {
        cudaStreamAttrValue av = {};
        av.accessPolicyWindow.num_bytes = 0;
        PRGPU_CUDA(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
        PRGPU_CUDA(cudaCtxResetPersistingL2Cache());
    }
    double total = 0;
    const bool log = std::getenv("PRGPU_TIMING_LOG") != nullptr; // per-iteration times (tuning)
    for (int i = 0; i < done; ++i) {
        float ms = 0;
        PRGPU_CUDA(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        total += ms;
        if (log) std::fprintf(stderr, "iteration %d: %.4f ms\n", i + 1, ms);
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return done ? total / done : 0.0;
}

double error_norm_device(int kind, const double* r, const double* s, uint64_t n, int device) {
    if (kind < 0 || kind > 2) fail(PRGPU_EINVAL, "error_norm: unknown norm");
    if (n == 0) fail(PRGPU_EINVAL, "error_norm: empty vectors");
    DeviceGuard dg(device);
    Stream st;
    DevBuf<double> dr(n), ds(n), parts(2 * 296), out(1);
    PRGPU_CUDA(cudaMemcpyAsync(dr.p, r, n * 8, cudaMemcpyHostToDevice, st));
    PRGPU_CUDA(cudaMemcpyAsync(ds.p, s, n * 8, cudaMemcpyHostToDevice, st));
    const int blocks = (int)std::min<uint64_t>(296, (n + kNT - 1) / kNT);
    norm_partials<<<blocks, kNT, 0, st>>>(kind, dr.p, ds.p, n, parts.p);
    PRGPU_LAUNCHED("norm_partials");
    norm_final<<<1, 32, 0, st>>>(kind, parts.p, blocks, out.p);
    PRGPU_LAUNCHED("norm_final");
    double v = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&v, out.p, 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    return v;
}

} // namespace prgpu
