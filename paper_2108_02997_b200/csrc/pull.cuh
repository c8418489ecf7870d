// pull.cuh — the per-iteration pull kernel (pagerank.hpp:84-99) for sm_100a.
//
// One launch = one iteration of the reference's do/while loop for K rank
// vectors ("lanes", one alpha each):
//
//   acc_k[v]  = sum_{u in in(v)} contrib_k[u]                  pagerank.hpp:89-91
//   next_k[v] = c0_k + alpha_k * acc_k[v]                                   :92
//   fused epilogue: |delta|, delta^2, max|delta| partials (norms.hpp:56-75),
//   the next dangling sum (:85-86), contrib'_k[src(v)] = next_k[v] / d[v]
//   (the per-edge division of :91 done once per vertex: the same IEEE value).
//   The last CTA to finish reduces the CTA partials in a fixed order, decides
//   convergence per lane (:95-99), computes the next teleport c0 (:87) and
//   sets the CUDA-graph WHILE condition: no per-iteration host sync.
//
// Work decomposition.  Rows are sorted by (in-degree desc, out-degree desc),
// so the degree bins are contiguous row ranges and every warp task costs about
// the same:
//   chunk task  (hub rows, in-degree > WIN): one warp pulls a 2*WIN-edge chunk
//               of a long row with 128-bit colidx loads; the warp finishing the
//               row's last chunk sums the chunk partials in chunk order and
//               runs the epilogue (hub rows are split across warps and SMs).
//   packed task (in-degree 1..WIN): a warp takes a run of consecutive rows
//               holding < 2*WIN edges.  K = 1: every gather of the run is in
//               flight at once (128-bit colidx loads), staged in shared memory,
//               then each row is reduced in ascending source order.  K > 1: one
//               lane group per row, accumulating in registers.
//   empty task  (in-degree 0): such a row's rank is exactly c0 every
//               iteration, so it is never stored: its |delta| terms are added
//               analytically by the finalizer (n_empty * |c0_t - c0_{t-1}|,
//               n_isolated * c0 for the dangling sum) and the task only writes
//               the row's next contribution c0/d when it has out-edges.
// Warps take tasks round-robin (task t -> warp t mod #warps): a static
// assignment, so every partial sum has a fixed order and runs are
// bit-reproducible (sweep.hpp:176-179, acceptance.cpp:331-366).  No
// floating-point atomics anywhere.
//
// Segmented hub pull (graphs whose contribution table exceeds L2, SegPlan in
// common.cuh): the hub rows' in-edges are regrouped into (row, source
// segment) pieces, pulled segment by segment — wide pieces as chunk tasks,
// small pieces as packed runs, both handed out in order from a device counter
// (a piece's sum does not depend on the warp that computes it) — and a
// combine task adds a row's piece sums in segment order before its epilogue.
//
// K lanes share every edge visit: a lane group of LG threads owns an edge (or
// a row), thread j of the group carrying W of the lanes, so the source's K
// contributions ([src][KS] rows) are fetched together.
//
// Contribution layout (HBM): the hottest sources (src < hot_src, the most
// gathered ones, packed at the front by the relabelling) keep both parities
// of their contribution row adjacent, [src][parity][KS], so the hot region of
// BOTH ping-pong buffers is one contiguous range that an L2 persisting window
// (or evict_last hints) keeps resident across iterations; colder sources are
// stored per parity after it.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace prgpu {

constexpr int kNT = 256; // threads per CTA
constexpr int kWarps = kNT / 32;
#ifdef PRGPU_NO_BCAST
constexpr bool kBcast = false; // tuning builds only
#else
constexpr bool kBcast = true;
#endif
// Tuning experiments compiled in only with -DPRGPU_EXPERIMENTS (make
// EXPERIMENTS=1 -> build_alt/libprgpu_exp.so): gather L2 policies
// (Params::gpol), L2 prefetch (pf) and the split pull (split).  All measured
// slower or no better on B200 (profiles/r2_c5_l2_experiments.md); their
// runtime branches alone cost 4-36 % in the hot loops, so the default build
// compiles them out.
#ifdef PRGPU_EXPERIMENTS
constexpr bool kExp = true;
#else
constexpr bool kExp = false;
#endif
constexpr int kNQ = 5;
constexpr int kPackOff = 40; // staged row offsets per packed run (>= rows per run + 1) // partials: L1, L2^2, Linf, dangling sum, L1-vs-ref

struct LaneState {
    double alpha;
    double tol;
    double c0;         // teleport for the next iteration
    double c0_used;    // teleport of the last completed iteration (= rank of empty rows)
    double prev_empty; // rank of empty rows before the current iteration
    double final_err;
    uint32_t stop_mask;
    int report_norm;
    int active;
    int iterations;
    int converged;
    int pad;
};

struct GlobalState {
    int iter;
    int any_active;
    unsigned int counter;
    int max_iter;
    int mode;   // lane-width mode of the next iteration (see Params::mode_id)
    int layout; // mode whose contribution buffer holds the current contributions
    // segmented pull: next piece task of the wide-piece and the small-piece
    // kernels (handed out in order, so every warp works in the same source
    // segment at any time); the finalizer resets them
    unsigned int seg_next[2];
};

constexpr int kMaxModes = 5;
constexpr int kMaxPeers = 7; // up to 8 GPUs of one NVSwitch domain

struct Params {
    uint32_t n, K;
    const uint64_t* __restrict__ row_off;
    const uint32_t* __restrict__ col;  // source ids
    const uint2* __restrict__ rowinfo; // {out-degree, source id}
    double* rank[2];                   // [n][ks] row-major, K lanes per row (rows < empty_begin only)
    uint32_t rank_lo, rank_hi;         // rows whose ranks this session holds (a shard's; else 0..n)
    uint32_t ks;                       // rank / contribution row stride (doubles)
    double* cbase;                     // contributions [parity][src][KS], see caddr()
    uint64_t cold_off[2];              // first row of each parity buffer (in rows of KS)
    const double* ref;                 // [n] engine ids, or null
    double* partials;                  // [kNQ*KP][G]
    double* trace;                     // [max_iter][K][4]
    LaneState* lanes;                  // [K]
    GlobalState* gs;
    // tasks
    const uint32_t* chunk_row;   // [n_chunk]
    const uint32_t* chunk_first; // [n_long + 1]
    const uint32_t* packed_r0;   // [n_packed + 1]
    double* chunk_acc;           // [n_chunk][KP]
    unsigned int* row_cnt;       // [n_long]
    uint32_t n_chunk, n_packed, n_empty_tasks;
    uint32_t chunk;              // edges per chunk task
    uint32_t empty_begin;        // first row with in-degree 0
    uint32_t iso_begin;          // first row with in- and out-degree 0
    uint32_t G;
    uint32_t hot_src;            // sources [0, hot_src) in the L2-resident region
    uint32_t l2mode;             // 0 evict hints, 2 no hints (streams); >= 3 contribution-write hints
    uint32_t pf;                 // L2 prefetch of upcoming gathers: 0 off, 1 on (PRGPU_PF)
    // split pull (SourceSplit): 1 = hot pass (row_off/col are the hot CSR;
    // each row's sum goes to hp, no epilogue), 2 = cold pass (the row's hot
    // partial hp + the cold sum, then the epilogue), 0 = one pass
    int split;
    double* hp;                  // [nonempty rows][ks] hot partial sums
    // in-graph kernel time per iteration (%globaltimer, ns): [iter][0] the
    // earliest start of a CTA of the iteration's pull kernels, [iter][1] the
    // finalizing CTA's end (single-GPU runs; prgpu_session_kernel_times)
    unsigned long long* ktime;
    uint32_t gpol;               // gather L2 policy (tuning): 0 plain; 1 hot evict_last / cold
                                 // evict_first; 2 hot normal / cold evict_first; 3 hot evict_last / cold normal
    uint32_t skip_mask;          // profiling only (PRGPU_SKIP): 1 chunk, 2 packed, 4 empty tasks,
                                 // 8 rank stores, 16 rank loads, 32 contribution stores
    // multi-GPU partition (1D row ranges): this rank runs tasks [task_begin, task_end)
    // and leaves its partial vector in rank_partials[part_rank]; a separate
    // finalize reduces all ranks' vectors in rank order after the exchange
    uint32_t task_begin, task_end;
    int part_mode;
    uint32_t part_rank, nranks;
    double* rank_partials;       // [nranks][kNQ*KP]
    int use_cond;
    cudaGraphConditionalHandle cond;
    int* frozen_at; // host-mapped [K]: iteration at which each lane stopped (0: live), or null
    // split iteration (single GPU): the hub-chunk tasks run as a first kernel
    // that only leaves its CTA partials (no_finalize), the packed and empty
    // tasks as a second kernel whose last CTA reduces both kernels' columns.
    // partials is [kNQ*KP][gtot]; this kernel's CTAs own columns pcol0 + blockIdx.x
    uint32_t pcol0, gtot;
    int no_finalize;
    // lane-width modes: one kernel pair per mode m covering lanes [0, mode_kp[m]);
    // an instance runs only when gs->mode == mode_id, and the finalizer picks
    // the narrowest mode covering the highest still-active lane for the next
    // iteration (lanes are stored slowest first, so the live ones are a prefix)
    int mode_id, nmodes;
    int mode_kp[kMaxModes];
    // each mode gathers from its own contribution buffers, rows of mode_ks
    // doubles (narrow modes: just their lanes, so the table is small enough to
    // stay in L2); repack_kernel converts on a mode change
    double* mode_cbase[kMaxModes];
    uint64_t mode_cold_off[kMaxModes][2];
    int mode_ks[kMaxModes];
    // CUDA-graph runs: one IF node per mode; the finalizer arms the next mode's
    int use_mode_cond;
    cudaGraphConditionalHandle mode_cond[kMaxModes];
    uint32_t er; // rows per empty task
    // fused multi-GPU exchange over peer memory (NVLink/NVSwitch): every
    // contribution row this rank computes is also stored into each peer's
    // buffer (same layout), the rank's partial vector into each peer's
    // rank_partials slot [parity][rank], and the last CTA then bumps every
    // rank's arrival counter; part_finalize_kernel waits for nranks arrivals
    // per iteration.  No host round trip, no collective call.
    int fused;
    int npeers;
    double* peer_cbase[kMaxPeers];
    double* peer_rp[kMaxPeers];
    unsigned int* peer_arrive[kMaxPeers];
    unsigned int* arrive; // this rank's arrival counter (peers add to it)
    const uint8_t* need;  // [src] bit r: rank r gathers the source (null: every peer)
    uint32_t part_kp;     // lane stride of rank_partials (the run's widest mode)
    // dealt partition (fused exchange): this rank runs the tasks
    // task_list[list_begin, list_end) instead of [task_begin, task_end), and
    // row_owner[row] is the rank that owns (pulls and publishes) each row
    const uint32_t* task_list;
    uint32_t list_begin, list_end;
    const uint8_t* row_owner;
    // segmented hub pull (SegPlan, common.cuh): the in-edges of rows [0,
    // n_seg_rows) regrouped into (row, source segment) pieces that are pulled
    // segment by segment, so the contribution rows gathered at any time are
    // one L2-sized slice of the table.  A piece leaves its partial sum in
    // pacc[slot]; the rows' epilogues (combine tasks) add their slots in
    // segment order.  seg_pre: the kernel's leading seg tasks (PATHS 4: chunks
    // of wide pieces, 8: runs of small pieces, 16: combine tasks).
    const uint64_t* seg_off;       // [pieces + 1] into seg_col (wide pieces first)
    const uint32_t* seg_col;
    const uint32_t* seg_slot;      // [pieces] row * seg_S + segment
    const uint4* seg_task;         // [seg chunks] {edge lo, hi, edges, slot | multi-chunk flag} per task
    const uint4* seg_run_rec;      // [runs] {first edge lo, hi, first piece, edges | pieces << 16} per run
    const uint4* run_rec;          // [n_packed] the same for the packed rows' runs (null: not built)
    const uint32_t* seg_chunk_row; // [seg chunks] wide piece of each chunk task
    const uint32_t* seg_chunk_first; // [wide pieces + 1]
    const uint32_t* seg_packed_r0; // [runs + 1] piece ranges of the small-piece runs
    double* seg_chunk_acc;         // [seg chunks][KP]
    unsigned int* seg_row_cnt;     // [wide pieces]
    double* pacc;                  // [n_seg_rows * seg_S][pacc_stride]
    uint32_t n_seg_rows, seg_S, pacc_stride, seg_pre, seg_cr, seg_grab;
};


// ---- L2 residency control -------------------------------------------------------
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// streams touched once per iteration (colidx, row offsets, row info)
__device__ __forceinline__ uint64_t stream_policy(const Params& P) {
    return P.l2mode == 2 ? policy_evict_normal() : policy_evict_first();
}
// contribution of source `src`: hot ones evict_last under the hint mode
__device__ __forceinline__ uint64_t contrib_policy(const Params& P, uint32_t src) {
    if (P.l2mode == 0) return src < P.hot_src ? policy_evict_last() : policy_evict_first();
    return policy_evict_normal();
}

template <int KS>
__device__ __forceinline__ double* caddr(const Params& P, int par, uint32_t src) {
    return P.cbase + (P.cold_off[par] + src) * KS;
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint32_t* p, uint64_t pol) {
    uint4 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
        : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
        : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ uint64_t ld_stream_u64(const uint64_t* p, uint64_t pol) {
    uint64_t r;
    asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
    uint32_t r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ uint2 ld_stream_u2(const uint2* p, uint64_t pol) {
    uint2 r;
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
        : "=r"(r.x), "=r"(r.y)
        : "l"(p), "l"(pol));
    return r;
}

// asynchronous 16-byte global -> shared copies (LDGSTS): gathers in flight
// without holding registers
__device__ __forceinline__ void cp_async16(void* smem, const void* g) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}
// L2-only 16-byte copies (rows gathered once per iteration: no L1 allocation)
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* g) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Hub chunks of the 2- and 4-lane instances (16- and 32-byte contribution
// rows) gather through shared memory with cp.async instead of registers:
// per warp a ring of two 128-edge blocks, the next block's rows in flight
// while the current one is summed (8x the rows in flight per warp of the
// register path, which the hub kernel's DRAM-latency stalls call for).  The
// summation order is the register path's, so results are bit-identical.
// Measured slower on C5 (hub kernel 36.6 -> 46.1 ms: the 74 KB ring halves the
// resident warps and the 16-byte halves of a row are two L2 requests; DRAM
// bytes 186 -> 208 GB): tuning build only.
#ifndef PRGPU_ASYNC_HUB
#define PRGPU_ASYNC_HUB 1
#endif
constexpr bool kAsyncHub = kExp && PRGPU_ASYNC_HUB != 0;
// Packed runs of the 4-lane instance staged in shared memory like K = 1
// (every gather of the run in flight, then per-row sums in edge order)
// instead of one lane group walking each row (packed_pipe).  Tuning switch.
#ifndef PRGPU_STAGED_WIDE
#define PRGPU_STAGED_WIDE 0
#endif
constexpr bool kStagedWide = PRGPU_STAGED_WIDE != 0;
constexpr int kAsyncBlock = 128; // edges per ring block
template <int LG, int KS>
constexpr bool async_hub() { return kAsyncHub && LG > 1 && (KS == 2 || KS == 4); }

// gathers: plain read-only loads (measured: L2 residency hints on the
// contributions did not pay, and the policy/address arithmetic per edge did)
// PRGPU_GATHER_LTC (tuning builds: 64 / 128 / 256): the gathers carry an L2
// prefetch-size qualifier.  A missed 32-byte row moves 128 bytes of DRAM with
// a plain load and 64 with .L2::64B (scripts/microbench_fetch_size.cu); the
// random-row rate itself (~36 G rows/s) does not change.
#ifndef PRGPU_GATHER_LTC
#define PRGPU_GATHER_LTC 0
#endif
#define PRGPU_STR2(x) #x
#define PRGPU_STR(x) PRGPU_STR2(x)
template <int W>
__device__ __forceinline__ void load_w(const double* __restrict__ p, double (&v)[W]) {
#if PRGPU_GATHER_LTC != 0
    if constexpr (W % 2 == 0) {
#pragma unroll
        for (int w = 0; w < W; w += 2)
            asm("ld.global.nc.L2::" PRGPU_STR(PRGPU_GATHER_LTC) "B.v2.f64 {%0,%1}, [%2];"
                : "=d"(v[w]), "=d"(v[w + 1])
                : "l"(p + w));
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w)
            asm("ld.global.nc.L2::" PRGPU_STR(PRGPU_GATHER_LTC) "B.f64 %0, [%1];" : "=d"(v[w]) : "l"(p + w));
    }
    return;
#endif
    if constexpr (W % 2 == 0) {
#pragma unroll
        for (int w = 0; w < W; w += 2) {
            const double2 x = __ldg(reinterpret_cast<const double2*>(p + w));
            v[w] = x.x;
            v[w + 1] = x.y;
        }
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w) v[w] = __ldg(p + w);
    }
}

template <int W>
__device__ __forceinline__ void load_w_pol(const double* __restrict__ p, double (&v)[W], uint64_t pol) {
    if constexpr (W % 2 == 0) {
#pragma unroll
        for (int w = 0; w < W; w += 2)
            asm("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                : "=d"(v[w]), "=d"(v[w + 1])
                : "l"(p + w), "l"(pol));
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w)
            asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[w]) : "l"(p + w), "l"(pol));
    }
}

template <int W>
__device__ __forceinline__ void store_w(double* p, const double (&v)[W]) {
    if constexpr (W % 2 == 0) {
#pragma unroll
        for (int w = 0; w < W; w += 2) *reinterpret_cast<double2*>(p + w) = make_double2(v[w], v[w + 1]);
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w) p[w] = v[w];
    }
}

template <int W>
__device__ __forceinline__ void store_w_pol(double* p, const double (&v)[W], uint64_t pol) {
    if constexpr (W % 2 == 0) {
#pragma unroll
        for (int w = 0; w < W; w += 2)
            asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" ::"l"(p + w),
                         "d"(v[w]), "d"(v[w + 1]), "l"(pol)
                         : "memory");
    } else {
#pragma unroll
        for (int w = 0; w < W; ++w)
            asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p + w), "d"(v[w]), "l"(pol)
                         : "memory");
    }
}

// Partial quantities a kernel instance accumulates (bitmask): L1 = 1, L2 = 2,
// Linf = 4, dangling = 8 (always), L1-vs-ref = 16.  Trimming them frees
// registers for the wide-lane (K > 1) instances; a norm that is not computed
// reads NaN in the trace.
constexpr int kQmAll = 31;
constexpr int kQmL1 = 1 | 8;

constexpr int popc_c(int x) { return x ? (x & 1) + popc_c(x >> 1) : 0; }

// Per-thread partial sums.  Narrow lanes keep them in registers; a thread that
// carries many lanes (W >= 6) keeps them in its own shared-memory column
// (thread-strided, conflict-free) so the gather path keeps its registers.
template <int W, int QM, bool SMEMP>
struct Partials {
    static constexpr int NQU = popc_c(QM);
    static constexpr int qidx(int q) { return popc_c(QM & ((1 << q) - 1)); }
    double reg[SMEMP ? 1 : kNQ][SMEMP ? 1 : W];
    double* sp;
    __device__ void init(double* smem_cols, int tid) {
        if constexpr (SMEMP) {
            sp = smem_cols + tid;
#pragma unroll
            for (int i = 0; i < NQU * W; ++i) sp[i * kNT] = 0.0;
        } else {
#pragma unroll
            for (int q = 0; q < kNQ; ++q)
#pragma unroll
                for (int w = 0; w < W; ++w) reg[q][w] = 0.0;
        }
    }
    __device__ __forceinline__ double& at(int q, int w) {
        if constexpr (SMEMP) return sp[(qidx(q) * W + w) * kNT];
        else return reg[q][w];
    }
    __device__ __forceinline__ void add(int q, int w, double x) {
        if ((QM >> q) & 1) at(q, w) += x;
    }
    __device__ __forceinline__ void max(int q, int w, double x) {
        if ((QM >> q) & 1) at(q, w) = fmax(at(q, w), x);
    }
    __device__ __forceinline__ double get(int q, int w) {
        return ((QM >> q) & 1) ? at(q, w) : 0.0;
    }
};

template <int LG, int W, int WIN, int QJ_ = 0, int KS_ = 0>
struct PullCfg {
    static constexpr int KP = LG * W;
    // contribution row stride in doubles (K rounded up to a sector multiple when
    // the lane group is wider than K: lanes slice*W >= KS idle on loads/stores)
    static constexpr int KS = KS_ ? KS_ : KP;
    static constexpr int ES = 32 / LG;   // edge slots (or lane groups) per warp
    static constexpr int EMAX = 2 * WIN; // edges per packed task / chunk
    static constexpr int QJ = QJ_ ? QJ_ : ((4 * W <= 4) ? 4 : (4 * W <= 8 ? 2 : 1)); // quads per slot per round
    static constexpr int ER = 8 * ES;    // rows per empty task
    // K = 1 stages every gathered value of a run in shared memory; wider lanes
    // accumulate in registers (staging would double the bytes moved per edge)
    static constexpr bool STAGED = (KP == 1); // measured: staging wide lanes' values lost
    static constexpr int SMEM_WARP = STAGED ? EMAX * KS : 0; // doubles per warp
};

template <int LG, int W, int WIN, int QJ_ = 0, int QM = kQmAll, int KS_ = 0, bool SMEMP_ = (W >= 6)>
struct Warp {
    using C = PullCfg<LG, W, WIN, QJ_, KS_>;
    static constexpr int KP = C::KP, ES = C::ES, KS = C::KS;
    const Params& P;
    const int lane, slot, slice, par;
    const double* __restrict__ rp;
    const double* __restrict__ cpl; // contributions read by this thread: buffer par, + slice*W
    double* __restrict__ rn;
    const double* s_alpha;
    const double* s_c0;
    const int* s_active;
    static constexpr bool SMEMP = SMEMP_; // partials in a shared-memory column (frees registers)
    Partials<W, QM, SMEMP> part;
    uint64_t pol_hot = 0, pol_cold = 0; // gather policies (P.gpol)

    __device__ Warp(const Params& p, int parity, int ln, const double* a, const double* c0,
                    const int* act, double* smem_cols, int tid)
        : P(p), lane(ln), slot(ln / LG), slice(ln % LG), par(parity), rp(p.rank[parity]),
          rn(p.rank[parity ^ 1]), cpl(p.cbase + p.cold_off[parity] * KS + (ln % LG) * W), s_alpha(a),
          s_c0(c0), s_active(act) {
        part.init(smem_cols, tid);
        if (kExp && p.gpol) {
            pol_hot = (p.gpol == 2) ? policy_evict_normal() : policy_evict_last();
            pol_cold = (p.gpol == 3) ? policy_evict_normal() : policy_evict_first();
        }
        // gpol 4: cold rows __ldcs; 5: cold rows L1::no_allocate + L2 evict_first
    }

    // L2 prefetch of a source's contribution row (no register held: the
    // later gather of the row then hits L2 instead of waiting on DRAM)
    __device__ __forceinline__ void prefetch_row(uint32_t src) const {
        const double* a = P.cbase + (P.cold_off[par] + src) * KS;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }

    // one source's contribution row slice (the gather of pagerank.hpp:91)
    __device__ __forceinline__ void gather(uint32_t src, double (&v)[W]) const {
        const double* a = cpl + (size_t)src * KS;
        if (!kExp) {
            load_w<W>(a, v);
        } else if (P.gpol == 4 || P.gpol == 5) { // cold rows streamed (.cs / L1 no-allocate + evict_first)
            if (src < P.hot_src) load_w<W>(a, v);
            else if (P.gpol == 4) {
#pragma unroll
                for (int w = 0; w < W; ++w) v[w] = __ldcs(a + w);
            } else {
#pragma unroll
                for (int w = 0; w < W; ++w)
                    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                        : "=d"(v[w]) : "l"(a + w), "l"(pol_cold));
            }
        } else if (P.gpol) load_w_pol<W>(a, v, src < P.hot_src ? pol_hot : pol_cold);
        else load_w<W>(a, v);
    }

    __device__ __forceinline__ bool lane_ok(int sl) const { return KS == KP || sl * W < KS; }

    // this thread's slice holds a lane that is still iterating: frozen lanes
    // are not gathered (lanes are ordered slowest-converging first, so the
    // live ones share the leading sectors of each contribution row)
    __device__ __forceinline__ bool slice_live() const {
        if (!lane_ok(slice)) return false;
        bool live = false;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const int k = slice * W + w;
            live |= (k < KP) && s_active[k];
        }
        return live;
    }

    // l2mode >= 3 (tuning): hot sources' rows (src < hot_src, next iteration's
    // most-gathered) written evict_last (3) / evict_normal (4), the rest
    // evict_first; 5: every row evict_first
    __device__ __forceinline__ void write_contrib(uint32_t src, int sl, const double (&cv)[W]) {
        double* dst = caddr<KS>(P, par ^ 1, src) + sl * W;
        if (P.l2mode >= 3) {
            const uint64_t pol = (P.l2mode == 5 || src >= P.hot_src) ? policy_evict_first()
                                 : P.l2mode == 3                   ? policy_evict_last()
                                                                   : policy_evict_normal();
            store_w_pol<W>(dst, cv, pol);
        } else {
            store_w<W>(dst, cv);
        }
        if (P.fused) { // the same row into the peers that gather it (NVLink stores)
            const size_t off = (size_t)(dst - P.cbase);
            const uint32_t m = P.need ? P.need[src] : 0xffu;
            for (int q = 0; q < P.npeers; ++q)
                if ((m >> (q < (int)P.part_rank ? q : q + 1)) & 1u) store_w<W>(P.peer_cbase[q] + off, cv);
        }
    }

    // split pull, hot pass: the row's hot-source sum is kept for the cold pass
    __device__ __forceinline__ void store_hot(uint32_t v, int sl, const double (&acc)[W]) {
        if (!lane_ok(sl)) return;
        double* h = P.hp + (size_t)v * P.ks + sl * W;
#pragma unroll
        for (int w = 0; w < W; ++w) __stcs(h + w, acc[w]);
    }

    // fused epilogue for row v, lanes [sl*W, sl*W + W)
    __device__ __forceinline__ void epilogue(uint32_t v, int sl, const double (&acc)[W]) {
        if (kExp && P.split == 1) {
            store_hot(v, sl, acc);
            return;
        }
        const uint2 ri = ld_stream_u2(P.rowinfo + v, stream_policy(P));
        epilogue_with<true>(v, sl, acc, ri, acc);
    }

    // the epilogue with the row's info and previous ranks already at hand.
    // Ranks are row-major [row][KS]: a lane group reads and writes one
    // contiguous row (3 sectors at K = 11) instead of K scattered words.
    template <bool LOAD_PREV = false>
    __device__ __forceinline__ void epilogue_with(uint32_t v, int sl, const double (&acc_in)[W], uint2 ri,
                                                  const double (&o_in)[W]) {
        if (kExp && P.split == 1) {
            store_hot(v, sl, acc_in);
            return;
        }
        double acc[W];
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] = acc_in[w];
        if (kExp && P.split == 2 && lane_ok(sl)) { // hot partial first, then the cold sum (a fixed order)
            const double* h = P.hp + (size_t)v * P.ks + sl * W;
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = __dadd_rn(__ldcs(h + w), acc[w]);
        }
        const uint32_t d = ri.x;
        double o[W];
        if constexpr (LOAD_PREV) {
#pragma unroll
            for (int w = 0; w < W; ++w) o[w] = 0.0;
            if (lane_ok(sl) && !(P.skip_mask & 16)) {
                const double* rr = rp + (size_t)v * P.ks + sl * W; // rank rows: stride ks
                if constexpr (W % 2 == 0) {
#pragma unroll
                    for (int w = 0; w < W; w += 2) {
                        const double2 x = __ldcs(reinterpret_cast<const double2*>(rr + w));
                        o[w] = x.x;
                        o[w + 1] = x.y;
                    }
                } else {
#pragma unroll
                    for (int w = 0; w < W; ++w) o[w] = __ldcs(rr + w);
                }
            }
        } else {
#pragma unroll
            for (int w = 0; w < W; ++w) o[w] = o_in[w];
        }
        double cv[W], nr[W];
        bool act[W];
        bool any = false;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const int k = sl * W + w;
            cv[w] = 0.0;
            nr[w] = 0.0;
            act[w] = k < (int)P.K && s_active[k];
            if (act[w]) {
                any = true;
                // next[v] = teleport + alpha*acc, two roundings (pagerank.hpp:92)
                const double r = __dadd_rn(s_c0[k], __dmul_rn(s_alpha[k], acc[w]));
                const double df = __dsub_rn(r, o[w]);
                const double ad = fabs(df);
                part.add(0, w, ad);
                part.add(1, w, df * df);
                part.max(2, w, ad);
                if (d == 0) part.add(3, w, r);
                if constexpr ((QM & 16) != 0)
                    if (P.ref) part.add(4, w, fabs(__dsub_rn(r, __ldg(P.ref + v))));
                nr[w] = r;
                if (d) cv[w] = __ddiv_rn(r, (double)d); // prev[u]/out_degree[u] (:91)
            }
        }
        if (any && !(P.skip_mask & 8)) { // frozen lanes keep their final value: masked stores
            double* rw = rn + (size_t)v * P.ks + sl * W;
            if constexpr (W % 2 == 0) {
#pragma unroll
                for (int w = 0; w < W; w += 2) {
                    if (act[w] && act[w + 1]) __stcs(reinterpret_cast<double2*>(rw + w), make_double2(nr[w], nr[w + 1]));
                    else {
                        if (act[w]) __stcs(rw + w, nr[w]);
                        if (act[w + 1]) __stcs(rw + w + 1, nr[w + 1]);
                    }
                }
            } else {
#pragma unroll
                for (int w = 0; w < W; ++w)
                    if (act[w]) __stcs(rw + w, nr[w]);
            }
        }
        if (d && any && lane_ok(sl) && !(P.skip_mask & 32)) write_contrib(ri.y, sl, cv);
    }

    // Accumulate edges [lo, hi) into acc with 128-bit colidx loads; slot s
    // takes quads s, s+ES, ... (fixed order: quad-major, then position).
    __device__ __forceinline__ void accumulate(const uint32_t* __restrict__ col, uint64_t lo, uint64_t hi,
                                               double (&acc)[W]) const {
        const uint64_t sp = stream_policy(P);
        const uint32_t* __restrict__ cb = col + (lo & ~3ull);
        const uint32_t off0 = (uint32_t)(lo & 3ull);
        const uint32_t ne = (uint32_t)(hi - lo) + off0; // <= 2*WIN + 3
        const bool ok = slice_live();
        // two quads (8 edges) per step; an edge outside [lo, hi) or an idle lane
        // adds +0.0, which leaves the (non-negative) sum exact.  Narrow lanes
        // issue all 8 gathers before the adds; wide lanes (W >= 6) consume
        // each edge's row as it arrives (register budget).
        constexpr int EF = (W >= 6) ? 1 : 8; // gathers held in flight per thread
        // software pipeline: the next step's colidx quads are loaded before
        // this step's gathers are consumed, so each step costs one round trip
        uint32_t q = 4u * slot;
        uint4 na = (q < ne) ? ld_stream_u4(cb + q, sp) : make_uint4(0, 0, 0, 0);
        uint4 nb = (q + 4u * ES < ne) ? ld_stream_u4(cb + q + 4u * ES, sp) : make_uint4(0, 0, 0, 0);
        for (; q < ne; q += 8u * ES) {
            const uint32_t q2 = q + 4u * ES;
            const uint4 a = na, b = nb;
            const uint32_t qn = q + 8u * ES;
            if (qn < ne) na = ld_stream_u4(cb + qn, sp);
            if (qn + 4u * ES < ne) nb = ld_stream_u4(cb + qn + 4u * ES, sp);
            const uint32_t us[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int j0 = 0; j0 < 8; j0 += EF) {
                double v[EF][W];
#pragma unroll
                for (int j = 0; j < EF; ++j) {
                    const uint32_t pos = ((j0 + j) < 4 ? q : q2) + ((j0 + j) & 3);
#pragma unroll
                    for (int w = 0; w < W; ++w) v[j][w] = 0.0;
                    if (ok && pos >= off0 && pos < ne)
                        gather(us[j0 + j], v[j]);
                }
#pragma unroll
                for (int j = 0; j < EF; ++j)
#pragma unroll
                    for (int w = 0; w < W; ++w) acc[w] += v[j][w];
            }
        }
    }

    // Wide lanes (LG > 1): every lane loads distinct colidx (128 edges per
    // block, coalesced) and each edge's source id is broadcast to its lane
    // group with one shuffle, so the index work is not repeated LG times.
    // Slot s sums edges s, s+ES, s+2ES, ... of the block, in order.
    __device__ __forceinline__ void accumulate_bcast(const uint32_t* __restrict__ col, uint64_t lo, uint64_t hi,
                                                     double (&acc)[W]) const {
        const uint64_t sp = stream_policy(P);
        const uint32_t ne = (uint32_t)(hi - lo);
        const uint32_t* __restrict__ cb = col + lo;
        const bool ok = slice_live();
        constexpr int STEPS = 32 / ES; // steps per 32-edge group
        constexpr int SB = STEPS < 4 ? STEPS : 4; // gathers in flight per sub-batch (registers)
        // P.pf: colidx is loaded two 128-edge blocks ahead and the rows of
        // block b+1 are prefetched into L2 before block b is gathered, so
        // gathers mostly hit L2 (the kernel is DRAM-latency bound: this
        // raises the rows in flight per warp without holding registers)
        const bool pf = kExp && P.pf != 0; // warp-uniform (every lane holds colidx for the shuffles)
        auto ld_block = [&](uint32_t base, uint32_t (&c)[4]) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t e = base + lane + 32u * j;
                c[j] = e < ne ? ld_stream_u32(cb + e, sp) : 0u;
            }
        };
        auto pf_block = [&](uint32_t base, const uint32_t (&c)[4]) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (base + lane + 32u * j < ne) prefetch_row(c[j]);
        };
        // the next block's colidx is loaded before this block's rows are
        // gathered, so a block costs one round trip (the gathers'), not two
        // (once the rows come from L2 — the segmented pull — the colidx
        // stream's DRAM latency is the longer of the two)
        uint32_t cn[4], cnn[4];
        ld_block(0, cn);
        if (pf) {
            ld_block(128, cnn);
            pf_block(0, cn);
        }
        for (uint32_t base = 0; base < ne; base += 128) {
            uint32_t c[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) c[j] = cn[j];
            if (pf) {
#pragma unroll
                for (int j = 0; j < 4; ++j) cn[j] = cnn[j];
                pf_block(base + 128, cn);
                if (base + 256 < ne) ld_block(base + 256, cnn);
            } else if (base + 128 < ne) {
                ld_block(base + 128, cn);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
#pragma unroll
                for (int i0 = 0; i0 < STEPS; i0 += SB) {
                    double v[SB][W];
#pragma unroll
                    for (int i = 0; i < SB; ++i) {
                        const uint32_t src = __shfl_sync(0xffffffffu, c[j], (i0 + i) * ES + slot);
                        const uint32_t e = base + 32u * j + (i0 + i) * ES + slot;
#pragma unroll
                        for (int w = 0; w < W; ++w) v[i][w] = 0.0;
                        if (ok && e < ne) gather(src, v[i]);
                    }
#pragma unroll
                    for (int i = 0; i < SB; ++i)
#pragma unroll
                        for (int w = 0; w < W; ++w) acc[w] += v[i][w];
                }
            }
        }
    }

    // cp.async ring (async_hub): see kAsyncHub.  `stage` = this warp's
    // 2 * kAsyncBlock * KS doubles.
    __device__ __forceinline__ void accumulate_async(const uint32_t* __restrict__ col, uint64_t lo, uint64_t hi,
                                                     double (&acc)[W], double* __restrict__ stage) const {
        const uint64_t sp = stream_policy(P);
        const uint32_t ne = (uint32_t)(hi - lo);
        const uint32_t* __restrict__ cb = col + lo;
        const bool ok = slice_live();
        constexpr int NP = KS / 2; // 16-byte pieces per row
        constexpr uint32_t B = kAsyncBlock;
        const double* __restrict__ ctab = P.cbase + P.cold_off[par] * KS;
        auto ld_block = [&](uint32_t base, uint32_t (&c)[4]) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t e = base + lane + 32u * j;
                c[j] = e < ne ? ld_stream_u32(cb + e, sp) : 0u;
            }
        };
        auto issue = [&](uint32_t base, const uint32_t (&c)[4], uint32_t ring) {
            double* dst = stage + (size_t)ring * B * KS;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t i = lane + 32u * j;
                if (base + i < ne) {
                    const double* src = ctab + (size_t)c[j] * KS;
#pragma unroll
                    for (int q = 0; q < NP; ++q) cp_async16_cg(dst + (size_t)i * KS + 2 * q, src + 2 * q);
                }
            }
            cp_async_commit();
        };
        const uint32_t nb = (ne + B - 1) / B;
        uint32_t cn[4];
        {
            uint32_t c0[4];
            ld_block(0, c0);
            if (nb > 1) ld_block(B, cn);
            issue(0, c0, 0);
        }
        for (uint32_t b = 0; b < nb; ++b) {
            if (b + 1 < nb) issue((b + 1) * B, cn, (b + 1) & 1);
            else cp_async_commit(); // an empty group keeps the wait count uniform
            if (b + 2 < nb) ld_block((b + 2) * B, cn);
            cp_async_wait<1>(); // block b has landed (block b+1 may be in flight)
            __syncwarp();
            if (ok) {
                const double* blk = stage + (size_t)(b & 1) * B * KS + slice * W;
                const uint32_t cnt = min(B, ne - b * B);
                // slot s sums edges s, s+ES, ... in order: accumulate_bcast's order
                for (uint32_t i = slot; i < cnt; i += ES)
#pragma unroll
                    for (int w = 0; w < W; ++w) acc[w] += blk[(size_t)i * KS + w];
            }
            __syncwarp(); // the ring slot is refilled next iteration
        }
        cp_async_wait<0>();
    }

    __device__ __forceinline__ void reduce_slots(double (&acc)[W]) const {
#pragma unroll
        for (int off = LG; off < 32; off <<= 1)
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] += __shfl_xor_sync(0xffffffffu, acc[w], off);
    }

    // a piece's partial sum (segmented pull): slot `sl` of the piece's row
    __device__ __forceinline__ void piece_store(uint32_t slot_id, int sl, const double (&acc)[W]) {
        if (lane_ok(sl)) store_w<W>(P.pacc + (size_t)slot_id * P.pacc_stride + sl * W, acc);
    }

    // ---- chunk of a long (hub) row, or (PIECE) of a wide piece ------------------------
    template <bool PIECE = false>
    __device__ void chunk_task(uint32_t t, double* __restrict__ stage = nullptr) {
        // the tables a chunk task reads: the hub rows' own, or the wide pieces'
        struct {
            const uint32_t* __restrict__ chunk_row;
            const uint32_t* __restrict__ chunk_first;
            const uint64_t* __restrict__ off;
            const uint32_t* __restrict__ col;
            double* acc;
            unsigned int* cnt;
        } T;
        if constexpr (PIECE) {
            T.chunk_row = P.seg_chunk_row; T.chunk_first = P.seg_chunk_first; T.off = P.seg_off;
            T.col = P.seg_col; T.acc = P.seg_chunk_acc; T.cnt = P.seg_row_cnt;
        } else {
            T.chunk_row = P.chunk_row; T.chunk_first = P.chunk_first; T.off = P.row_off;
            T.col = P.col; T.acc = P.chunk_acc; T.cnt = P.row_cnt;
        }
        const uint64_t sp = stream_policy(P);
        const uint32_t row = T.chunk_row[t];
        const uint32_t first = T.chunk_first[row];
        const uint32_t nch = T.chunk_first[row + 1] - first;
        const uint64_t rlo = ld_stream_u64(T.off + row, sp), rhi = ld_stream_u64(T.off + row + 1, sp);
        // (a split pass's part of the row can end before this chunk: empty range)
        const uint64_t lo = min(rlo + (uint64_t)(t - first) * P.chunk, rhi);
        const uint64_t hi = min(lo + P.chunk, rhi);
        double acc[W];
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] = 0.0;
        if constexpr (async_hub<LG, KS>()) {
            if (stage) accumulate_async(T.col, lo, hi, acc, stage);
            else accumulate_bcast(T.col, lo, hi, acc);
        } else if constexpr (LG > 1 && kBcast) accumulate_bcast(T.col, lo, hi, acc);
        else accumulate(T.col, lo, hi, acc);
        reduce_slots(acc);
        if (nch == 1) { // the whole row was this chunk: no hand-off needed
            if (lane < LG) {
                if constexpr (PIECE) piece_store(P.seg_slot[row], slice, acc);
                else epilogue(row, slice, acc);
            }
            return;
        }
        if (lane < LG) store_w<W>(T.acc + (size_t)t * KP + slice * W, acc);
        __threadfence();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) last = (atomicAdd(T.cnt + row, 1u) == nch - 1);
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) return;
        __threadfence();
        // the row's chunk partials, in chunk order per slot, then slot tree
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] = 0.0;
        for (uint32_t c = slot; c < nch; c += ES) {
            const double* p = T.acc + (size_t)(first + c) * KP + slice * W;
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] += __ldcg(p + w);
        }
        reduce_slots(acc);
        if (lane < LG) {
            if constexpr (PIECE) piece_store(P.seg_slot[row], slice, acc);
            else epilogue(row, slice, acc);
        }
        if (lane == 0) T.cnt[row] = 0;
    }

    // a whole wide piece in one chunk task: its record gives the edge range and the slot
    __device__ __forceinline__ void piece_chunk(uint64_t lo, uint32_t len, uint32_t slot_id) {
        double acc[W];
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] = 0.0;
        if constexpr (LG > 1 && kBcast) accumulate_bcast(P.seg_col, lo, lo + len, acc);
        else accumulate(P.seg_col, lo, lo + len, acc);
        reduce_slots(acc);
        if (lane < LG) piece_store(slot_id, slice, acc);
    }

    // ---- epilogues of the segmented rows: a row's piece partials in segment order --------
    __device__ void combine_task(uint32_t t) {
        const uint32_t base = t * P.seg_cr;
        const uint32_t end = min(base + P.seg_cr, P.n_seg_rows);
        const uint32_t S = P.seg_S;
        const bool lok = lane_ok(slice);
        for (uint32_t v = base + slot; v < end; v += ES) {
            double acc[W];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = 0.0;
            if (lok) {
                const double* p = P.pacc + (size_t)v * S * P.pacc_stride + slice * W;
#pragma unroll 4
                for (uint32_t j = 0; j < S; ++j) {
#pragma unroll
                    for (int w = 0; w < W; ++w) acc[w] += __ldcs(p + (size_t)j * P.pacc_stride + w);
                }
            }
            epilogue(v, slice, acc);
        }
    }

    // ---- packed run of rows, K = 1: all gathers in flight, staged in smem ----------------
    // PIECE: the run's "rows" are small pieces (segmented pull): offsets and
    // colidx from the segment plan, a piece's sum stored to its slot
    template <bool PIECE = false>
    __device__ void packed_task(uint32_t t, double* __restrict__ sv) {
        const uint64_t sp = stream_policy(P);
        const uint32_t* __restrict__ pr = PIECE ? P.seg_packed_r0 : P.packed_r0;
        const uint64_t* __restrict__ roff = PIECE ? P.seg_off : P.row_off;
        const uint32_t* __restrict__ colp = PIECE ? P.seg_col : P.col;
        const uint32_t r0 = pr[t], r1 = pr[t + 1];
        const int R = (int)(r1 - r0); // <= 32
        if (R <= 0) return;
        const uint64_t e0 = ld_stream_u64(roff + r0, sp);
        const uint64_t e1 = ld_stream_u64(roff + r1, sp);
        // row bounds relative to e0 (a run holds < 2*WIN edges: 32-bit is enough)
        const uint32_t mylo = (lane < R) ? (uint32_t)(ld_stream_u64(roff + r0 + lane, sp) - e0) : 0;
        const uint32_t myhi = (lane < R) ? (uint32_t)(ld_stream_u64(roff + r0 + lane + 1, sp) - e0) : 0;
        // the epilogue's row info and previous rank of row r0 + lane, in flight
        // during the gathers (handed to the reducing lane by a shuffle)
        uint2 my_ri = make_uint2(0, 0);
        double my_prev = 0.0;
        if constexpr (PIECE) {
            if (lane < R) my_ri.x = ld_stream_u32(P.seg_slot + r0 + lane, sp);
        } else if constexpr (KP == 1) {
            if (lane < R) {
                my_ri = ld_stream_u2(P.rowinfo + r0 + lane, sp);
                if (!(P.skip_mask & 16)) my_prev = __ldcs(rp + (size_t)(r0 + lane) * P.ks);
            }
        }
        // cb is the 16-byte aligned colidx base; valid positions [off0, ne).
        const uint32_t* __restrict__ cb = colp + (e0 & ~3ull);
        const uint32_t off0 = (uint32_t)(e0 & 3ull);
        const uint32_t ne = (uint32_t)(e1 - e0) + off0;
        const bool live = slice_live();
        for (uint32_t qb = 4u * slot; qb < ne; qb += 4u * ES * C::QJ) {
            uint32_t us[C::QJ][4];
#pragma unroll
            for (int j = 0; j < C::QJ; ++j) {
                const uint32_t q = qb + 4u * ES * j;
                const uint4 c4 = (q < ne) ? ld_stream_u4(cb + q, sp) : make_uint4(0, 0, 0, 0);
                us[j][0] = c4.x; us[j][1] = c4.y; us[j][2] = c4.z; us[j][3] = c4.w;
            }
            double v[C::QJ][4][W];
#pragma unroll
            for (int j = 0; j < C::QJ; ++j)
#pragma unroll
                for (int tq = 0; tq < 4; ++tq) {
                    const uint32_t e = qb + 4u * ES * j + tq;
                    if (live && e >= off0 && e < ne)
                        gather(us[j][tq], v[j][tq]);
                }
#pragma unroll
            for (int j = 0; j < C::QJ; ++j)
#pragma unroll
                for (int tq = 0; tq < 4; ++tq) {
                    const uint32_t e = qb + 4u * ES * j + tq;
                    if (live && e >= off0 && e < ne) store_w<W>(sv + (e - off0) * KS + slice * W, v[j][tq]);
                }
        }
        __syncwarp();
        // per-row reduction in ascending source order, gs lanes per (row, slice)
        const int np2 = R <= 1 ? 1 : (R <= 2 ? 2 : (R <= 4 ? 4 : (R <= 8 ? 8 : (R <= 16 ? 16 : 32))));
        const int rows_per_round = 32 / LG;
        const int gs = (np2 <= rows_per_round) ? rows_per_round / np2 : 1;
        const int rounds = (np2 <= rows_per_round) ? 1 : (R + rows_per_round - 1) / rows_per_round;
        const int sub = (lane / LG) % gs;
        for (int rd = 0; rd < rounds; ++rd) {
            const int i = rd * rows_per_round + (lane / LG) / gs;
            const int src = i < R ? i : 0;
            const uint32_t lo = __shfl_sync(0xffffffffu, mylo, src);
            const uint32_t hi = __shfl_sync(0xffffffffu, myhi, src);
            double acc[W];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = 0.0;
            if (i < R) {
                for (uint32_t j = lo + sub; j < hi; j += gs) {
                    const double* p = sv + j * KS + slice * W;
#pragma unroll
                    for (int w = 0; w < W; ++w) acc[w] += p[w];
                }
            }
            for (int off = LG; off < LG * gs; off <<= 1)
#pragma unroll
                for (int w = 0; w < W; ++w) acc[w] += __shfl_xor_sync(0xffffffffu, acc[w], off);
            if constexpr (PIECE) {
                const uint32_t sl_id = __shfl_sync(0xffffffffu, my_ri.x, src);
                if (i < R && sub == 0) piece_store(sl_id, slice, acc);
            } else if constexpr (KP == 1) {
                const uint2 ri = make_uint2(__shfl_sync(0xffffffffu, my_ri.x, src),
                                            __shfl_sync(0xffffffffu, my_ri.y, src));
                const double o[1] = {__shfl_sync(0xffffffffu, my_prev, src)};
                if (i < R && sub == 0) epilogue_with<false>(r0 + i, slice, acc, ri, o);
            } else {
                if (i < R && sub == 0) epilogue(r0 + i, slice, acc);
            }
        }
        __syncwarp();
    }

    // ---- packed run, K > 1: one lane group per row, register accumulation ------------
    // Group g takes rows g, g+ES, ... of the run; each row is summed in
    // ascending source order with 128-bit colidx loads, two quads in flight.
    __device__ void packed_direct(uint32_t t) {
        const uint64_t sp = stream_policy(P);
        const uint32_t r0 = P.packed_r0[t], r1 = P.packed_r0[t + 1];
        const uint32_t R = r1 - r0;
        for (uint32_t i = slot; i < R; i += ES) {
            const uint32_t v = r0 + i;
            double acc[W];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = 0.0;
            // accumulate() with a single slot of this group: quads 0, 1, 2, ...
            const uint64_t lo = ld_stream_u64(P.row_off + v, sp), hi = ld_stream_u64(P.row_off + v + 1, sp);
            const uint32_t* __restrict__ cb = P.col + (lo & ~3ull);
            const uint32_t off0 = (uint32_t)(lo & 3ull);
            const uint32_t ne = (uint32_t)(hi - lo) + off0;
            const bool ok = slice_live();
            for (uint32_t q = 0; q < ne; q += 8) {
                const uint4 a = ld_stream_u4(cb + q, sp);
                const uint4 b = (q + 4 < ne) ? ld_stream_u4(cb + q + 4, sp) : make_uint4(0, 0, 0, 0);
                const uint32_t us[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
                constexpr int EF = (W >= 6) ? 1 : 8; // see accumulate()
#pragma unroll
                for (int j0 = 0; j0 < 8; j0 += EF) {
                    double vals[EF][W];
#pragma unroll
                    for (int j = 0; j < EF; ++j) {
#pragma unroll
                        for (int w = 0; w < W; ++w) vals[j][w] = 0.0;
                        if (ok && q + j0 + j >= off0 && q + j0 + j < ne)
                            gather(us[j0 + j], vals[j]);
                    }
#pragma unroll
                    for (int j = 0; j < EF; ++j)
#pragma unroll
                        for (int w = 0; w < W; ++w) acc[w] += vals[j][w];
                }
            }
            epilogue(v, slice, acc);
        }
    }

    // K > 1 packed run.  The warp stages the run's row offsets and colidx in
    // shared memory with coalesced loads (two round trips for the whole run);
    // then each slot walks its rows issuing the next row's row info and
    // previous ranks before gathering the current one, so a row costs a
    // single gather round trip.
    template <bool PIECE = false>
    __device__ void packed_pipe(uint32_t t, double* __restrict__ stage, bool have_rec = false,
                                uint4 rec = make_uint4(0, 0, 0, 0)) {
        constexpr int WIN_ = C::EMAX / 2;
        const uint64_t sp = stream_policy(P);
        const uint32_t* __restrict__ pr = PIECE ? P.seg_packed_r0 : P.packed_r0;
        const uint64_t* __restrict__ roff = PIECE ? P.seg_off : P.row_off;
        const uint32_t* __restrict__ colp = PIECE ? P.seg_col : P.col;
        const uint4* __restrict__ recs = PIECE ? P.seg_run_rec : P.run_rec;
        uint64_t* s_off = reinterpret_cast<uint64_t*>(stage);                 // [kPackOff]
        uint32_t* s_col = reinterpret_cast<uint32_t*>(s_off + kPackOff);     // [2*WIN + 8]
        uint32_t r0, R, ne_all; // R <= 2*WIN / max(1, WIN/32) + 1
        uint64_t e0;
        if (recs != nullptr && !(kExp && P.split)) {
            // the run's record {first edge, first row, edges | rows << 16}: the row
            // offsets and the colidx are staged in ONE round trip instead of
            // bounds -> offsets -> colidx
            const uint4 rc = have_rec ? rec : __ldg(recs + t);
            e0 = ((uint64_t)rc.y << 32) | rc.x;
            r0 = rc.z;
            ne_all = rc.w & 0xffffu;
            R = rc.w >> 16;
            for (uint32_t x = lane; x <= R; x += 32) s_off[x] = ld_stream_u64(roff + r0 + x, sp);
            for (uint32_t x = lane; x < ne_all; x += 32) s_col[x] = ld_stream_u32(colp + e0 + x, sp);
            __syncwarp();
        } else {
            r0 = pr[t];
            R = pr[t + 1] - r0;
            for (uint32_t x = lane; x <= R; x += 32) s_off[x] = ld_stream_u64(roff + r0 + x, sp);
            __syncwarp();
            e0 = s_off[0];
            ne_all = (uint32_t)(s_off[R] - e0);
            for (uint32_t x = lane; x < ne_all; x += 32) s_col[x] = ld_stream_u32(colp + e0 + x, sp);
            __syncwarp();
        }
        if (kExp && P.pf) // every row of the run in flight to L2 at once (the walk below is one row per slot)
            for (uint32_t x = lane; x < ne_all; x += 32) prefetch_row(s_col[x]);
        uint32_t i = slot;
        if (i < R) {
            const bool ok = slice_live();
            const bool lok = lane_ok(slice);
            auto load_prev = [&](uint32_t v, double (&o)[W]) {
#pragma unroll
                for (int w = 0; w < W; ++w) o[w] = 0.0;
                if (lok && !PIECE) {
                    const double* rr = rp + (size_t)v * P.ks + slice * W;
                    if constexpr (W % 2 == 0) {
#pragma unroll
                        for (int w = 0; w < W; w += 2) {
                            const double2 x = __ldcs(reinterpret_cast<const double2*>(rr + w));
                            o[w] = x.x;
                            o[w + 1] = x.y;
                        }
                    } else {
#pragma unroll
                        for (int w = 0; w < W; ++w) o[w] = __ldcs(rr + w);
                    }
                }
            };
            uint32_t v = r0 + i;
            // (PIECE: ri.x is the piece's slot)
            uint2 ri = PIECE ? make_uint2(ld_stream_u32(P.seg_slot + v, sp), 0u) : ld_stream_u2(P.rowinfo + v, sp);
            double o[W];
            load_prev(v, o);
            for (;;) {
                const uint32_t in = i + ES;
                const bool more = in < R;
                const uint32_t vn = r0 + (more ? in : i);
                // next row's info and previous ranks, in flight during this row's gathers
                const uint2 nri =
                    PIECE ? make_uint2(ld_stream_u32(P.seg_slot + vn, sp), 0u) : ld_stream_u2(P.rowinfo + vn, sp);
                double no[W];
                load_prev(vn, no);
                double acc[W];
#pragma unroll
                for (int w = 0; w < W; ++w) acc[w] = 0.0;
                const uint32_t lo = (uint32_t)(s_off[i] - e0), hi = (uint32_t)(s_off[i + 1] - e0);
                for (uint32_t q = lo; q < hi; q += 8) {
                    const uint32_t nv = min(8u, hi - q);
                    const uint32_t vb = ok ? ((1u << nv) - 1u) : 0u; // valid positions as a bit mask
                    double vals[8][W];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
#pragma unroll
                        for (int w = 0; w < W; ++w) vals[j][w] = 0.0;
                        if (vb & (1u << j)) gather(s_col[q + j], vals[j]);
                    }
#pragma unroll
                    for (int j = 0; j < 8; ++j)
#pragma unroll
                        for (int w = 0; w < W; ++w) acc[w] += vals[j][w];
                }
                if constexpr (PIECE) piece_store(ri.x, slice, acc);
                else epilogue_with<false>(v, slice, acc, ri, o);
                if (!more) break;
                i = in;
                v = vn;
                ri = nri;
#pragma unroll
                for (int w = 0; w < W; ++w) o[w] = no[w];
            }
        }
        __syncwarp(); // the next task reuses the stage
    }

    // ---- rows with no in-edges: rank = c0; write c0/d for rows with out-edges,
    //      and (sweep mode) the L1 distance to the reference -------------------------
    __device__ void empty_task(uint32_t t) {
        if (kExp && P.split == 1) return; // no in-edges: nothing for the hot pass
        const uint64_t sp = stream_policy(P);
        const uint32_t base = P.empty_begin + t * P.er;
        const uint32_t end = min(base + P.er, P.n);
#pragma unroll 2
        for (uint32_t v = base + slot; v < end; v += ES) {
            const uint2 ri = ld_stream_u2(P.rowinfo + v, sp);
            double cv[W];
            bool any = false;
#pragma unroll
            for (int w = 0; w < W; ++w) {
                const int k = slice * W + w;
                cv[w] = 0.0;
                if (k < (int)P.K && s_active[k]) {
                    any = true;
                    const double r = s_c0[k];
                    if constexpr ((QM & 16) != 0)
                        if (P.ref) part.add(4, w, fabs(__dsub_rn(r, __ldg(P.ref + v))));
                    if (ri.x) cv[w] = __ddiv_rn(r, (double)ri.x);
                }
            }
            if (ri.x && any && lane_ok(slice)) write_contrib(ri.y, slice, cv);
        }
    }
};

// Per-lane convergence and the next teleport from the reduced partials
// (pagerank.hpp:87, :95-99); thread k < K handles lane k, thread 0 the loop flag.
// `layout`: the lane-width mode whose contribution buffers this iteration wrote
template <int KP, int QM>
__device__ void finalize_lanes(const Params& P, const double* s_tot, const double* s_c0,
                               const int* s_active, int iter, int layout) {
    const int tid = threadIdx.x;
    if (tid < (int)P.K && tid < KP && s_active[tid]) { // lanes >= KP are frozen in this mode
        const int k = tid;
        LaneState& L = P.lanes[k];
        // rows with no in-edges all moved from prev_empty to c0 (exactly); add
        // their terms once instead of per row
        const double c0 = s_c0[k];
        const double de = __dsub_rn(c0, L.prev_empty);
        const double ade = fabs(de);
        const double n_empty = (double)(P.n - P.empty_begin), n_iso = (double)(P.n - P.iso_begin);
        double l1s = s_tot[0 * KP + k], l2s = s_tot[1 * KP + k], linf = s_tot[2 * KP + k];
        double dang = s_tot[3 * KP + k];
        if (P.n > P.empty_begin) {
            l1s = __dadd_rn(l1s, __dmul_rn(n_empty, ade));
            l2s = __dadd_rn(l2s, __dmul_rn(n_empty, __dmul_rn(de, de)));
            linf = fmax(linf, ade);
            dang = __dadd_rn(dang, __dmul_rn(n_iso, c0));
        }
        const double l2 = sqrt(l2s);
        double* tr = P.trace + ((size_t)iter * P.K + k) * 4;
        tr[0] = (QM & 1) ? l1s : NAN;
        tr[1] = (QM & 2) ? l2 : NAN;
        tr[2] = (QM & 4) ? linf : NAN;
        tr[3] = (QM & 16) ? s_tot[4 * KP + k] : NAN;
        const double errs[3] = {l1s, l2, linf};
        const int done = iter + 1;
        L.iterations = done;
        L.final_err = errs[L.report_norm];
        L.c0_used = c0;
        L.prev_empty = c0;
        bool stop = true; // every norm in the mask strictly below tau (pagerank.hpp:99)
        for (int q = 0; q < 3; ++q)
            if ((L.stop_mask >> q) & 1u) stop = stop && (errs[q] < L.tol);
        if (stop) {
            L.converged = 1;
            L.active = 0;
        } else if (done >= P.gs->max_iter) {
            L.active = 0;
        }
        // teleport = (1 - alpha)/n + alpha*dangling_sum/n   (pagerank.hpp:87)
        const double a = L.alpha, nd = (double)P.n;
        L.c0 = __dadd_rn(__ddiv_rn(__dsub_rn(1.0, a), nd), __ddiv_rn(__dmul_rn(a, dang), nd));
        if (!L.active && P.frozen_at) { // the host may now copy this lane out
            __threadfence_system();
            *(volatile int*)(P.frozen_at + k) = done;
        }
    }
    __syncthreads();
    if (tid == 0) {
        int any = 0, top = -1;
        for (uint32_t k = 0; k < P.K; ++k)
            if (P.lanes[k].active) { any = 1; top = (int)k; }
        int mode = P.nmodes - 1; // narrowest mode that still covers every live lane
        for (int m = P.nmodes - 1; m >= 0; --m)
            if (P.mode_kp[m] > top) mode = m;
        P.gs->mode = mode;
        if (P.use_cond && P.use_mode_cond)
            for (int m = 0; m < P.nmodes; ++m) cudaGraphSetConditional(P.mode_cond[m], m == mode ? 1u : 0u);
        P.gs->layout = layout; // this iteration wrote that mode's buffers
        P.gs->iter = iter + 1;
        P.gs->any_active = any;
        P.gs->counter = 0;
        P.gs->seg_next[0] = 0;
        P.gs->seg_next[1] = 0;
        __threadfence();
        if (P.use_cond) cudaGraphSetConditional(P.cond, any ? 1u : 0u);
    }
}

// PATHS: which task kinds this instance compiles (1 hub chunks, 2 packed +
// empty); a split iteration runs a PATHS=1 and a PATHS=2 instance, each with
// only its own path's register pressure.
// CTAs per SM the small-piece instances (PATHS 8) are compiled for (tuning
// builds: -DPRGPU_A2_MINB=6; 0: the instance's own MINB)
#ifndef PRGPU_A2_MINB
#define PRGPU_A2_MINB 0
#endif
#ifndef PRGPU_A_MINB // likewise the wide-piece instances (PATHS 5)
#define PRGPU_A_MINB 0
#endif
template <int LG, int W, int WIN, int QJ_, int MINB, int QM = kQmAll, int KS_ = 0, int PATHS = 3>
__global__ void __launch_bounds__(kNT, (PATHS == 8 && PRGPU_A2_MINB) ? PRGPU_A2_MINB : (PATHS == 5 && PRGPU_A_MINB) ? PRGPU_A_MINB : MINB) pull_kernel(const Params P) {
    using C = PullCfg<LG, W, WIN, QJ_, KS_>;
    constexpr int KP = C::KP;
    __shared__ double s_alpha[KP], s_c0[KP];
    __shared__ int s_active[KP];
    __shared__ int s_iter, s_flag;
    extern __shared__ __align__(16) double s_dyn[]; // [kWarps][SMEM_WARP] gathered values
    __shared__ double s_red[kWarps][kNQ * KP];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_iter = P.gs->iter;
        // not this instance's lane-width mode, or a speculative launch after convergence
        s_flag = P.gs->any_active && P.gs->mode == P.mode_id;
    }
    if (tid < KP) {
        const bool real = tid < (int)P.K;
        s_alpha[tid] = real ? P.lanes[tid].alpha : 0.0;
        s_c0[tid] = real ? P.lanes[tid].c0 : 0.0;
        s_active[tid] = real ? P.lanes[tid].active : 0;
    }
    __syncthreads();
    if (!s_flag) return;
    if (P.ktime && tid == 0 && s_iter < P.gs->max_iter) atomicMin(P.ktime + 2 * s_iter, global_ns());

    // dynamic smem: [kWarps][SMEM_WARP + ASYNC_WARP] staged gathers, then the per-thread
    // partial columns when W >= 6
    // K > 1 packed runs (PATHS == 2): staged row offsets + colidx, in doubles
    // PATHS bits: 1 hub chunks, 2 packed + empty; segmented pull: 4 chunks
    // of wide pieces, 8 runs of small pieces, 16 combine tasks (the seg
    // tasks lead the kernel's task range: Params::seg_pre of them)
    constexpr bool PACKS = (PATHS & (2 | 8)) != 0;
    constexpr bool WSTAGE = (PATHS == 2) && kStagedWide && LG == 4 && C::KS == 4 && !C::STAGED;
    constexpr int PACK_WARP = (PACKS && PATHS != 3 && !C::STAGED) ? (WSTAGE ? C::EMAX * C::KS : kPackOff + (2 * WIN + 8) / 2) : 0;
    // hub-chunk instances of 2/4 lanes: the cp.async ring (kAsyncHub)
    constexpr bool ASYNC = (PATHS == 1) && async_hub<LG, C::KS>();
    constexpr int ASYNC_WARP = ASYNC ? 2 * kAsyncBlock * C::KS : 0;
    constexpr int PER_WARP = C::SMEM_WARP + PACK_WARP + ASYNC_WARP;
    // the instances of a split iteration keep their partials in shared
    // memory: the registers go to gathers in flight
    constexpr bool SMEMP = (W >= 6) || (PATHS != 3 && C::KP > 1);
    Warp<LG, W, WIN, QJ_, QM, KS_, SMEMP> w(P, s_iter & 1, lane, s_alpha, s_c0, s_active,
                                     s_dyn + (size_t)kWarps * PER_WARP, tid);
    double* sv = s_dyn + (size_t)warp * PER_WARP;
    const uint32_t TW = P.G * kWarps;
    const uint32_t T1 = P.n_chunk, T2 = T1 + P.n_packed;
    const bool listed = P.task_list != nullptr;
    const uint32_t i0 = listed ? P.list_begin : P.task_begin, i1 = listed ? P.list_end : P.task_end;
    uint32_t istart = i0 + blockIdx.x * kWarps + warp;
    if constexpr ((PATHS & (4 | 8)) != 0) {
        // piece tasks are handed out in order from a device counter, Params::seg_grab
        // at a time: the warps stay within a few thousand tasks of each other,
        // i.e. inside one source segment (a static deal drifts apart by more
        // than a segment over a kernel).  A piece's sum does not depend on
        // which warp computes it, so runs stay bit-reproducible.
        const uint32_t GRAB = P.seg_grab;
        const uint32_t pre = P.seg_pre;
        unsigned int* ctr = &P.gs->seg_next[(PATHS & 4) ? 0 : 1];
        for (;;) {
            uint32_t b = 0;
            if (lane == 0) b = atomicAdd(ctr, GRAB);
            b = __shfl_sync(0xffffffffu, b, 0);
            if (b >= pre) break;
            const uint32_t e = min(b + GRAB, pre);
            if constexpr ((PATHS & 4) != 0) {
                // the grabbed tasks' records in one round trip (lane i holds task b + i's)
                uint4 rec = make_uint4(0, 0, 0, 0);
                if (b + lane < e) rec = __ldg(P.seg_task + b + lane);
                for (uint32_t i = b; i < e; ++i) {
                    const uint32_t lo_l = __shfl_sync(0xffffffffu, rec.x, i - b), lo_h = __shfl_sync(0xffffffffu, rec.y, i - b);
                    const uint32_t len = __shfl_sync(0xffffffffu, rec.z, i - b), sl = __shfl_sync(0xffffffffu, rec.w, i - b);
                    if (sl & 0x80000000u) w.template chunk_task<true>(i); // a chunk of a multi-chunk piece: hand-off
                    else w.piece_chunk(((uint64_t)lo_h << 32) | lo_l, len, sl);
                }
            } else {
                if constexpr (C::STAGED) {
                    for (uint32_t i = b; i < e; ++i) w.template packed_task<true>(i, sv);
                } else { // the grabbed runs' records in one round trip (lane i holds run b + i's)
                    const bool hr = P.seg_run_rec != nullptr;
                    uint4 rec = make_uint4(0, 0, 0, 0);
                    if (hr && b + lane < e) rec = __ldg(P.seg_run_rec + b + lane);
                    for (uint32_t i = b; i < e; ++i) {
                        const uint4 rc = make_uint4(__shfl_sync(0xffffffffu, rec.x, i - b), __shfl_sync(0xffffffffu, rec.y, i - b),
                                                    __shfl_sync(0xffffffffu, rec.z, i - b), __shfl_sync(0xffffffffu, rec.w, i - b));
                        w.template packed_pipe<true>(i, sv, hr, rc);
                    }
                }
            }
        }
    } else if constexpr ((PATHS & 16) != 0) { // combine tasks lead, then the round-robin carries on
        const uint32_t pre = P.seg_pre;
        uint32_t i = blockIdx.x * kWarps + warp;
        for (; i < pre; i += TW) w.combine_task(i);
        istart = i0 + (i - pre);
    }
    for (uint32_t i = istart; i < i1; i += TW) {
        const uint32_t t = listed ? __ldg(P.task_list + i) : i;
        if (t < T1) {
            if constexpr ((PATHS & 1) != 0)
                if (!(P.skip_mask & 1)) w.chunk_task(t, ASYNC ? sv : nullptr);
        } else if constexpr ((PATHS & 2) != 0) {
            if (t < T2) {
                if (!(P.skip_mask & 2)) {
                    if constexpr (C::STAGED || WSTAGE) w.packed_task(t - T1, sv);
                    else if constexpr (PATHS != 3) w.packed_pipe(t - T1, sv);
                    else w.packed_direct(t - T1);
                }
            } else if (!(P.skip_mask & 4)) {
                w.empty_task(t - T2);
            }
        }
    }

    if constexpr (PATHS == 8) return; // piece sums only: no epilogue ran, no partials
    if (kExp && P.split == 1) return; // hot pass: row sums only, no partials

    // ---- CTA partials, fixed order ------------------------------------------------
#pragma unroll
    for (int q = 0; q < kNQ; ++q)
#pragma unroll
        for (int wv = 0; wv < W; ++wv) {
            double v = w.part.get(q, wv);
#pragma unroll
            for (int off = LG; off < 32; off <<= 1) {
                const double o = __shfl_xor_sync(0xffffffffu, v, off);
                v = (q == 2) ? fmax(v, o) : v + o;
            }
            if (lane < LG) s_red[warp][q * KP + w.slice * W + wv] = v;
        }
    __syncthreads();
    for (int t = tid; t < kNQ * KP; t += kNT) {
        const int q = t / KP;
        double v = 0.0;
#pragma unroll
        for (int wp = 0; wp < kWarps; ++wp) v = (q == 2) ? fmax(v, s_red[wp][t]) : v + s_red[wp][t];
        P.partials[(size_t)t * P.gtot + P.pcol0 + blockIdx.x] = v;
    }

    // ---- last CTA: reduce partials, convergence, next teleport --------------------------
    if (P.fused) __threadfence_system(); // this CTA's peer stores before its ticket
    else __threadfence();
    if (P.no_finalize) return; // first kernel of a split iteration
    __syncthreads();
    if (tid == 0) s_flag = (atomicAdd(&P.gs->counter, 1u) == P.G - 1);
    __syncthreads();
    if (!s_flag) return;
    __threadfence();

    __shared__ double s_tot[kNQ * KP];
    for (int t = tid; t < kNQ * KP; t += kNT) s_tot[t] = 0.0;
    __syncthreads();
    // only the quantities this instance tracks, only real lanes; each warp
    // streams one quantity's CTA column with 4 loads in flight per lane
    for (int t = warp; t < kNQ * KP; t += kWarps) {
        const int q = t / KP;
        if (!((QM >> q) & 1) || (t % KP) >= (int)P.K) continue;
        double v = 0.0;
        const double* col = P.partials + (size_t)t * P.gtot;
        uint32_t b = lane;
        for (; b + 96 < P.gtot; b += 128) {
            const double x0 = __ldcg(col + b), x1 = __ldcg(col + b + 32), x2 = __ldcg(col + b + 64),
                         x3 = __ldcg(col + b + 96);
            v = (q == 2) ? fmax(fmax(fmax(fmax(v, x0), x1), x2), x3) : (((v + x0) + x1) + x2) + x3;
        }
        for (; b < P.gtot; b += 32) {
            const double x = __ldcg(col + b);
            v = (q == 2) ? fmax(v, x) : v + x;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const double o = __shfl_xor_sync(0xffffffffu, v, off);
            v = (q == 2) ? fmax(v, o) : v + o;
        }
        if (lane == 0) s_tot[t] = v;
    }
    __syncthreads();
    if (P.part_mode) { // multi-GPU: publish this rank's vector; finalize runs after the exchange
        // in the run's layout [q][part_kp] (a narrow mode fills its first KP lanes)
        const uint32_t pkp = P.part_kp;
        const size_t slot = ((P.fused ? (size_t)(s_iter & 1) * P.nranks : 0) + P.part_rank) * kNQ * pkp;
        for (int t = tid; t < kNQ * KP; t += kNT) {
            const size_t at = slot + (size_t)(t / KP) * pkp + t % KP;
            P.rank_partials[at] = s_tot[t];
            if (P.fused)
                for (int q = 0; q < P.npeers; ++q) P.peer_rp[q][at] = s_tot[t];
        }
        __syncthreads();
        if (tid == 0) {
            P.gs->counter = 0;
            if (P.fused) { // every CTA's rows and this vector are out: arrive everywhere
                __threadfence_system();
                for (int q = 0; q < P.npeers; ++q) atomicAdd_system(P.peer_arrive[q], 1u);
                atomicAdd_system(P.arrive, 1u);
            }
        }
        return;
    }
    finalize_lanes<KP, QM>(P, s_tot, s_c0, s_active, s_iter, P.mode_id);
    if (P.ktime && tid == 0 && s_iter < P.gs->max_iter) P.ktime[2 * s_iter + 1] = global_ns();
}

// Mode change (Params::mode_id): copy the current contributions (parity of
// this iteration) of lanes [0, mode_ks[m]) from the buffer of the mode that
// wrote them into this mode's narrower buffer.  A no-op launch otherwise.
static __global__ void __launch_bounds__(kNT) repack_kernel(const Params P, uint32_t nsrc) {
    __shared__ int s_go, s_from, s_par;
    if (threadIdx.x == 0) {
        const int mode = P.gs->mode, from = P.gs->layout;
        s_go = P.gs->any_active && mode == P.mode_id && from != P.mode_id;
        s_from = from;
        s_par = P.gs->iter & 1;
    }
    __syncthreads();
    if (!s_go) return;
    const int m = P.mode_id, f = s_from, par = s_par;
    const int ks_t = P.mode_ks[m], ks_f = P.mode_ks[f];
    const double* __restrict__ src = P.mode_cbase[f] + P.mode_cold_off[f][par] * ks_f;
    double* __restrict__ dst = P.mode_cbase[m] + P.mode_cold_off[m][par] * ks_t;
    const uint64_t total = (uint64_t)nsrc * ks_t;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t u = i / ks_t, k = i - u * ks_t;
        dst[i] = src[u * ks_f + k];
    }
}

// Multi-GPU finalize (one CTA, identical on every rank): the ranks' partial
// vectors reduced in rank order, then the same lane update as the fused path.
template <int LG, int W, int WIN, int QJ_, int MINB, int QM = kQmAll, int KS_ = 0>
__global__ void __launch_bounds__(kNT) part_finalize_kernel(const Params P) {
    constexpr int KP = PullCfg<LG, W, WIN, QJ_, KS_>::KP;
    __shared__ double s_c0[KP], s_tot[kNQ * KP];
    __shared__ int s_active[KP];
    __shared__ int s_iter;
    const int tid = threadIdx.x;
    if (tid == 0) s_iter = P.gs->iter;
    if (tid < KP) {
        const bool real = tid < (int)P.K;
        s_c0[tid] = real ? P.lanes[tid].c0 : 0.0;
        s_active[tid] = real ? P.lanes[tid].active : 0;
    }
    __shared__ int s_go, s_mode;
    if (tid == 0) {
        s_go = P.gs->any_active;
        s_mode = P.gs->mode; // the mode this iteration ran in (finalize picks the next)
    }
    __syncthreads();
    if (!s_go) return; // speculative launch after convergence
    if (P.fused && tid == 0) {
        // every rank's rows and partials for this iteration have landed once
        // nranks arrivals are counted (a bounded wait: a lost peer traps
        // instead of hanging the device)
        const unsigned target = P.nranks * (unsigned)(s_iter + 1);
        const long long t0 = clock64();
        unsigned seen;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(seen) : "l"(P.arrive) : "memory");
            if (seen >= target) break;
            __nanosleep(256);
            if (clock64() - t0 > 40000000000ll) __trap(); // ~20 s
        }
    }
    __syncthreads();
    const size_t pbase = P.fused ? (size_t)(s_iter & 1) * P.nranks * kNQ * KP : 0;
    for (int t = tid; t < kNQ * KP; t += kNT) {
        const int q = t / KP;
        double v = 0.0;
        for (uint32_t r = 0; r < P.nranks; ++r) {
            const double x = __ldcg(P.rank_partials + pbase + (size_t)r * kNQ * KP + t);
            v = (q == 2) ? fmax(v, x) : v + x;
        }
        s_tot[t] = v;
    }
    __syncthreads();
    finalize_lanes<KP, QM>(P, s_tot, s_c0, s_active, s_iter, s_mode);
}

} // namespace prgpu
