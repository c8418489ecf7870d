// engine.cu — the pull power-iteration hot path (pagerank.hpp:70-108) for sm_100a.
//
// One launch of `pull_kernel` is one iteration of the reference's do/while
// loop (pagerank.hpp:84-99) for K rank vectors ("lanes", one alpha each):
//
//   acc_k[v]  = sum_{u in in(v)} contrib_k[u]          pagerank.hpp:89-91
//   next_k[v] = c0_k + alpha_k * acc_k[v]                           :92
//   fused epilogue: |delta|, delta^2, max|delta| partials (norms.hpp:56-75),
//   the next dangling sum (:85-86), and contrib'_k[v] = next_k[v]/d[v]
//   (the per-edge division of :91, done once per vertex: same IEEE value).
//   The last CTA to finish reduces all CTA partials in a fixed order and
//   decides convergence per lane (:95-99), computes the next teleport c0
//   (:87), and sets the CUDA-graph WHILE condition — no per-iteration host
//   synchronisation.
//
// Work decomposition: rows are sorted by in-degree
// descending, so the degree bins are contiguous row ranges:
//   hub rows   (deg > 4096): one CTA per row, 128-bit colidx loads
//   warp rows  (deg > 32)  : one warp per row, 128-bit colidx loads + shuffle reduce
//   thread rows(deg <= 32) : one lane group (LG threads) per row, colidx staged
//                            per warp in shared memory with 128-bit loads
// A lane group of LG threads owns one row; thread j of the group carries W of
// the K lanes, so each edge visit loads the source's K contributions once
// (interleaved [v][KP] layout) and feeds all K lanes.
//
// The grid is persistent: CTA b processes a contiguous, cost-balanced range
// of work items (computed once per session), so every partial sum has a
// fixed summation order and results are run-to-run bit-identical (required by
// sweep.hpp:176-179 and acceptance.cpp:331-366).  No floating-point atomics.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <memory>
#include <vector>

#include "common.cuh"

namespace prgpu {

constexpr int kNT = 256;     // threads per CTA
constexpr int kNQ = 5;       // partial quantities: L1, L2^2, Linf, dangling, L1-vs-ref
constexpr int kRowCost = 3;  // scheduling cost of a row, in edges
constexpr int kWarpStage = 32 * kWarpMinDegree + 4; // staged colidx per warp (thread bin)

struct LaneState {
    double alpha;
    double tol;
    double c0;
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
};

struct Params {
    uint32_t n, K;
    const uint64_t* __restrict__ row_off;
    const uint32_t* __restrict__ col;
    const uint32_t* __restrict__ deg;
    double* rank[2];    // [K][n]
    double* contrib[2]; // [n][KP]
    const double* ref;  // [n] engine ids, or null
    double* partials;   // [kNQ*KP][G]
    double* trace;      // [max_iter][K][4]
    LaneState* lanes;   // [K]
    GlobalState* gs;
    const uint32_t* block_begin; // [G+1]
    uint32_t hub_end, warp_end;
    uint32_t items_hub, items_warp;
    uint32_t G;
    int use_cond;
    cudaGraphConditionalHandle cond;
};

// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream_u4(const uint32_t* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <int W>
__device__ __forceinline__ void gather_add(const double* __restrict__ p, double (&acc)[W]) {
    if constexpr (W == 1) {
        acc[0] += __ldg(p);
    } else {
#pragma unroll
        for (int w = 0; w < W; w += 2) {
            const double2 v = __ldg(reinterpret_cast<const double2*>(p + w));
            acc[w] += v.x;
            acc[w + 1] += v.y;
        }
    }
}

template <int LG, int W>
struct Ctx {
    static constexpr int KP = LG * W;
    const Params& P;
    const double* __restrict__ rp; // ranks read
    double* __restrict__ rn;       // ranks written
    const double* __restrict__ cp; // contributions read
    double* __restrict__ cn;       // contributions written
    const double* s_alpha;
    const double* s_c0;
    const int* s_active;
    double part[kNQ][W];

    __device__ Ctx(const Params& p, int par, const double* a, const double* c0, const int* act)
        : P(p), rp(p.rank[par]), rn(p.rank[par ^ 1]), cp(p.contrib[par]), cn(p.contrib[par ^ 1]),
          s_alpha(a), s_c0(c0), s_active(act) {
#pragma unroll
        for (int q = 0; q < kNQ; ++q)
#pragma unroll
            for (int w = 0; w < W; ++w) part[q][w] = 0.0;
    }

    __device__ __forceinline__ void gather(uint32_t u, int slice, double (&acc)[W]) const {
        gather_add<W>(cp + (size_t)u * KP + slice * W, acc);
    }

    // fused epilogue for row v, lanes [slice*W, slice*W+W)
    __device__ __forceinline__ void epilogue(uint32_t v, int slice, const double (&acc)[W]) {
        const uint32_t d = __ldg(P.deg + v);
        const double dd = (double)d;
        const size_t n = P.n;
        double cv[W];
        bool any = false;
#pragma unroll
        for (int w = 0; w < W; ++w) {
            const int k = slice * W + w;
            cv[w] = 0.0;
            if (k < (int)P.K && s_active[k]) {
                any = true;
                // next[v] = teleport + alpha * acc, rounded separately (pagerank.hpp:92)
                const double r = __dadd_rn(s_c0[k], __dmul_rn(s_alpha[k], acc[w]));
                const double o = __ldcs(rp + (size_t)k * n + v);
                const double df = __dsub_rn(r, o);
                const double ad = fabs(df);
                part[0][w] += ad;
                part[1][w] += df * df;
                part[2][w] = fmax(part[2][w], ad);
                if (d == 0) part[3][w] += r;
                if (P.ref) part[4][w] += fabs(__dsub_rn(r, __ldg(P.ref + v)));
                __stcs(rn + (size_t)k * n + v, r);
                if (d) cv[w] = __ddiv_rn(r, dd); // prev[u]/out_degree[u], pagerank.hpp:91
            }
        }
        if (d && any) {
            double* dst = cn + (size_t)v * KP + slice * W;
            if constexpr (W == 1) {
                dst[0] = cv[0];
            } else {
#pragma unroll
                for (int w = 0; w < W; w += 2)
                    *reinterpret_cast<double2*>(dst + w) = make_double2(cv[w], cv[w + 1]);
            }
        }
    }
};

// Strided accumulation over [lo, hi) with 128-bit colidx loads: `slot` of
// `nslots` handles quads q = align4(lo) + 4*slot, +4*nslots, ...
template <int LG, int W>
__device__ __forceinline__ void accumulate_strided(const Ctx<LG, W>& c, uint64_t lo, uint64_t hi,
                                                   int slot, int nslots, int slice,
                                                   double (&acc)[W]) {
    const uint32_t* __restrict__ col = c.P.col;
    uint64_t q = (lo & ~3ull) + 4ull * slot;
    const uint64_t step = 4ull * nslots;
#pragma unroll 2
    for (; q < hi; q += step) {
        const uint4 c4 = ld_stream_u4(col + q);
        const uint32_t us[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint64_t j = q + t;
            if (j >= lo && j < hi) c.gather(us[t], slice, acc);
        }
    }
}

template <int LG, int W>
__device__ __forceinline__ void reduce_slots_warp(double (&acc)[W]) {
#pragma unroll
    for (int off = LG; off < 32; off <<= 1)
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] += __shfl_xor_sync(0xffffffffu, acc[w], off);
}

template <int LG, int W>
__global__ void __launch_bounds__(kNT) pull_kernel(const Params P) {
    constexpr int KP = LG * W;
    constexpr int RW = 32 / LG;   // rows per warp in the thread bin
    constexpr int TR = kNT / LG;  // rows per thread-bin item
    __shared__ double s_alpha[KP], s_c0[KP];
    __shared__ int s_active[KP];
    __shared__ int s_iter, s_last;
    __shared__ double s_red[kNT / 32][kNQ * KP];
    __shared__ uint32_t s_col[kNT / 32][kWarpStage];

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_iter = P.gs->iter;
        s_last = P.gs->any_active;
    }
    if (tid < KP) {
        const bool real = tid < (int)P.K;
        s_alpha[tid] = real ? P.lanes[tid].alpha : 0.0;
        s_c0[tid] = real ? P.lanes[tid].c0 : 0.0;
        s_active[tid] = real ? P.lanes[tid].active : 0;
    }
    __syncthreads();
    if (!s_last) return; // speculative launch after convergence (host-loop mode)

    Ctx<LG, W> c(P, s_iter & 1, s_alpha, s_c0, s_active);
    const uint32_t n = P.n;
    const uint32_t ib = P.block_begin[blockIdx.x], ie = P.block_begin[blockIdx.x + 1];

    for (uint32_t it = ib; it < ie; ++it) {
        if (it < P.items_hub) {
            // ---- hub row: the whole CTA ------------------------------------
            const uint32_t row = it;
            const uint64_t lo = P.row_off[row], hi = P.row_off[row + 1];
            const int slot = tid / LG, slice = tid % LG;
            double acc[W];
#pragma unroll
            for (int w = 0; w < W; ++w) acc[w] = 0.0;
            accumulate_strided<LG, W>(c, lo, hi, slot, kNT / LG, slice, acc);
            reduce_slots_warp<LG, W>(acc);
            if (lane < LG)
#pragma unroll
                for (int w = 0; w < W; ++w) s_red[warp][lane * W + w] = acc[w];
            __syncthreads();
            if (tid < LG) {
#pragma unroll
                for (int w = 0; w < W; ++w) {
                    double s = 0.0;
#pragma unroll
                    for (int wp = 0; wp < kNT / 32; ++wp) s += s_red[wp][tid * W + w];
                    acc[w] = s;
                }
                c.epilogue(row, tid, acc);
            }
            __syncthreads();
        } else if (it < P.items_hub + P.items_warp) {
            // ---- warp rows: one row per warp ---------------------------------
            const uint32_t row = P.hub_end + (it - P.items_hub) * (kNT / 32) + warp;
            if (row < P.warp_end) {
                const uint64_t lo = P.row_off[row], hi = P.row_off[row + 1];
                const int slot = lane / LG, slice = lane % LG;
                double acc[W];
#pragma unroll
                for (int w = 0; w < W; ++w) acc[w] = 0.0;
                accumulate_strided<LG, W>(c, lo, hi, slot, 32 / LG, slice, acc);
                reduce_slots_warp<LG, W>(acc);
                if (lane < LG) c.epilogue(row, lane, acc);
            }
        } else {
            // ---- thread rows: one lane group per row, colidx staged per warp --
            const uint32_t base = P.warp_end + (it - P.items_hub - P.items_warp) * TR + warp * RW;
            if (base < n) {
                const uint32_t wend = min(base + RW, n);
                const uint64_t wlo = P.row_off[base], whi = P.row_off[wend];
                const uint64_t alo = wlo & ~3ull;
                const uint32_t cnt = (uint32_t)(whi - alo);
                for (uint32_t p = lane * 4; p < cnt; p += 128)
                    *reinterpret_cast<uint4*>(&s_col[warp][p]) = ld_stream_u4(P.col + alo + p);
                __syncwarp();
                const uint32_t row = base + lane / LG;
                const int slice = lane % LG;
                if (row < n) {
                    const uint32_t lo = (uint32_t)(P.row_off[row] - alo);
                    const uint32_t hi = (uint32_t)(P.row_off[row + 1] - alo);
                    double acc[W];
#pragma unroll
                    for (int w = 0; w < W; ++w) acc[w] = 0.0;
#pragma unroll 4
                    for (uint32_t j = lo; j < hi; ++j) c.gather(s_col[warp][j], slice, acc);
                    c.epilogue(row, slice, acc);
                }
                __syncwarp();
            }
        }
    }

    // ---- CTA partials, fixed order ------------------------------------------
    {
        const int slice = lane % LG;
#pragma unroll
        for (int q = 0; q < kNQ; ++q)
#pragma unroll
            for (int w = 0; w < W; ++w) {
                double v = c.part[q][w];
#pragma unroll
                for (int off = LG; off < 32; off <<= 1) {
                    const double o = __shfl_xor_sync(0xffffffffu, v, off);
                    v = (q == 2) ? fmax(v, o) : v + o;
                }
                if (lane < LG) s_red[warp][q * KP + slice * W + w] = v;
            }
        __syncthreads();
        for (int t = tid; t < kNQ * KP; t += kNT) {
            const int q = t / KP;
            double v = 0.0;
#pragma unroll
            for (int wp = 0; wp < kNT / 32; ++wp)
                v = (q == 2) ? fmax(v, s_red[wp][t]) : v + s_red[wp][t];
            P.partials[(size_t)t * P.G + blockIdx.x] = v;
        }
    }

    // ---- last CTA: reduce partials, convergence, next teleport -------------------
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&P.gs->counter, 1u) == P.G - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();

    __shared__ double s_tot[kNQ * KP];
    for (int t = warp; t < kNQ * KP; t += kNT / 32) {
        const int q = t / KP;
        double v = 0.0;
        for (uint32_t b = lane; b < P.G; b += 32) {
            const double x = __ldcg(P.partials + (size_t)t * P.G + b);
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
    const int iter = s_iter; // iterations completed before this launch
    if (tid < (int)P.K && s_active[tid]) {
        const int k = tid;
        LaneState& L = P.lanes[k];
        const double l1 = s_tot[0 * KP + k];
        const double l2 = sqrt(s_tot[1 * KP + k]);
        const double linf = s_tot[2 * KP + k];
        const double dang = s_tot[3 * KP + k];
        double* tr = P.trace + ((size_t)iter * P.K + k) * 4;
        tr[0] = l1;
        tr[1] = l2;
        tr[2] = linf;
        tr[3] = s_tot[4 * KP + k];
        const double errs[3] = {l1, l2, linf};
        const int done = iter + 1;
        L.iterations = done;
        L.final_err = errs[L.report_norm];
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
        const double a = L.alpha, nd = (double)n;
        L.c0 = __dadd_rn(__ddiv_rn(__dsub_rn(1.0, a), nd), __ddiv_rn(__dmul_rn(a, dang), nd));
    }
    __syncthreads();
    if (tid == 0) {
        int any = 0;
        for (uint32_t k = 0; k < P.K; ++k) any |= P.lanes[k].active;
        P.gs->iter = iter + 1;
        P.gs->any_active = any;
        P.gs->counter = 0;
        __threadfence();
        if (P.use_cond) cudaGraphSetConditional(P.cond, any ? 1u : 0u);
    }
}

// ---- init: uniform ranks 1/N (pagerank.hpp:77), first contributions and c0 ----
template <int KP>
__global__ void init_kernel(Params P, uint32_t ndangling) {
    const size_t n = P.n;
    const double r0 = 1.0 / (double)P.n;
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x) {
        const uint32_t d = P.deg[v];
        for (uint32_t k = 0; k < P.K; ++k) P.rank[0][k * n + v] = r0;
        const double cv = d ? __ddiv_rn(r0, (double)d) : 0.0;
#pragma unroll
        for (int k = 0; k < KP; ++k) P.contrib[0][v * KP + k] = (k < (int)P.K) ? cv : 0.0;
    }
    if (blockIdx.x == 0 && threadIdx.x < P.K) {
        LaneState& L = P.lanes[threadIdx.x];
        const double nd = (double)P.n;
        // sum of the initial dangling ranks: ndangling * (1/N), rounded once
        const double dang = __dmul_rn((double)ndangling, r0);
        const double a = L.alpha;
        L.c0 = __dadd_rn(__ddiv_rn(__dsub_rn(1.0, a), nd), __ddiv_rn(__dmul_rn(a, dang), nd));
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

// ---- result extraction: out[k][v_orig] = rank[final_buf(k)][k][new_of_old[v]] ----
__global__ void extract_ranks(Params P, const uint32_t* __restrict__ new_of_old,
                              double* __restrict__ out, int lane_only, int use_current) {
    const size_t n = P.n;
    const int k0 = lane_only >= 0 ? lane_only : 0;
    const int k1 = lane_only >= 0 ? lane_only + 1 : (int)P.K;
    for (int k = k0; k < k1; ++k) {
        const int buf = use_current ? (P.gs->iter & 1) : (P.lanes[k].iterations & 1);
        const double* src = P.rank[buf] + (size_t)k * n;
        double* dst = out + (size_t)(k - k0) * n;
        for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
             v += (size_t)gridDim.x * blockDim.x)
            dst[v] = src[new_of_old[v]];
    }
}

__global__ void scatter_ref(const double* __restrict__ in, const uint32_t* __restrict__ new_of_old,
                            double* __restrict__ out, uint32_t n) {
    for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < n;
         v += (size_t)gridDim.x * blockDim.x)
        out[new_of_old[v]] = in[v];
}

// ---- work-item costs and the balanced CTA ranges --------------------------------
__global__ void item_costs(const uint64_t* __restrict__ row_off, uint32_t n, uint32_t hub_end,
                           uint32_t warp_end, uint32_t items_hub, uint32_t items_warp,
                           uint32_t items_total, uint32_t tr, uint64_t* __restrict__ cost) {
    for (uint32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < items_total;
         it += gridDim.x * blockDim.x) {
        uint32_t r0, r1;
        if (it < items_hub) {
            r0 = it;
            r1 = it + 1;
        } else if (it < items_hub + items_warp) {
            r0 = hub_end + (it - items_hub) * (kNT / 32);
            r1 = min(r0 + kNT / 32, warp_end);
        } else {
            r0 = warp_end + (it - items_hub - items_warp) * tr;
            r1 = min(r0 + tr, n);
        }
        cost[it] = (row_off[r1] - row_off[r0]) + (uint64_t)kRowCost * (r1 - r0);
    }
}

__global__ void block_ranges(const uint64_t* __restrict__ incl, uint32_t items, uint32_t G,
                             uint32_t* __restrict__ begin) {
    const uint64_t total = items ? incl[items - 1] : 0;
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b <= G; b += gridDim.x * blockDim.x) {
        if (b == G) { begin[b] = items; continue; }
        const uint64_t target = (total * b) / G; // first item whose exclusive prefix >= target
        uint32_t lo = 0, hi = items;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) / 2;
            const uint64_t excl = mid ? incl[mid - 1] : 0;
            if (excl < target) lo = mid + 1; else hi = mid;
        }
        begin[b] = lo;
    }
}

// ---- deterministic device error_norm (norms.hpp:48-78) ----------------------------
__global__ void norm_partials(int kind, const double* __restrict__ r, const double* __restrict__ s,
                              uint64_t n, double* __restrict__ out) {
    __shared__ double red[kNT / 32];
    double v = 0.0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double d = r[i] - s[i];
        if (kind == 0) v += fabs(d);
        else if (kind == 1) v += d * d;
        else v = fmax(v, fabs(d));
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, v, off);
        v = kind == 2 ? fmax(v, o) : v + o;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kNT / 32; ++w) t = kind == 2 ? fmax(t, red[w]) : t + red[w];
        out[blockIdx.x] = t;
    }
}

__global__ void norm_final(int kind, const double* __restrict__ parts, int nparts, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double t = 0.0;
    for (int i = 0; i < nparts; ++i) t = kind == 2 ? fmax(t, parts[i]) : t + parts[i];
    out[0] = kind == 1 ? sqrt(t) : t;
}

// ============================================================================
// Session: device state + the CUDA graph (WHILE node around one pull launch).
// ============================================================================
struct LaneCfg {
    int LG, W;
};

inline LaneCfg lane_cfg(int K) {
    if (K == 1) return {1, 1};
    if (K == 2) return {1, 2};
    if (K <= 4) return {2, 2};
    if (K <= 8) return {4, 2};
    if (K <= 12) return {2, 6};
    return {4, 4};
}

using KernelFn = void (*)(const Params);

template <int LG, int W>
KernelFn pull_fn() { return pull_kernel<LG, W>; }

KernelFn pick_pull(LaneCfg c) {
    if (c.LG == 1 && c.W == 1) return pull_fn<1, 1>();
    if (c.LG == 1 && c.W == 2) return pull_fn<1, 2>();
    if (c.LG == 2 && c.W == 2) return pull_fn<2, 2>();
    if (c.LG == 4 && c.W == 2) return pull_fn<4, 2>();
    if (c.LG == 2 && c.W == 6) return pull_fn<2, 6>();
    return pull_fn<4, 4>();
}

void launch_init(LaneCfg c, const Params& P, uint32_t ndangling, cudaStream_t st) {
    const unsigned grid = (unsigned)std::min<uint64_t>((P.n + kNT - 1) / kNT, 148ull * 16);
    const int KP = c.LG * c.W;
    switch (KP) {
    case 1: init_kernel<1><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 2: init_kernel<2><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 4: init_kernel<4><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 8: init_kernel<8><<<grid, kNT, 0, st>>>(P, ndangling); break;
    case 12: init_kernel<12><<<grid, kNT, 0, st>>>(P, ndangling); break;
    default: init_kernel<16><<<grid, kNT, 0, st>>>(P, ndangling); break;
    }
    PRGPU_LAUNCHED("init_kernel");
}

} // namespace prgpu

using namespace prgpu;

struct prgpu_session {
    prgpu_graph* g = nullptr;
    int K = 1, KP = 1, max_iter = 500;
    LaneCfg cfg{1, 1};
    KernelFn pull = nullptr;
    Params P{};
    Stream stream;
    DevBuf<double> rank, contrib, partials, trace, ref;
    DevBuf<LaneState> lanes;
    DevBuf<GlobalState> gs;
    DevBuf<uint32_t> block_begin;
    std::vector<LaneState> lanes_host;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool use_graph = false;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    double last_loop_ms = 0;

    ~prgpu_session() {
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

prgpu_session* session_create(prgpu_graph* g, const prgpu_params* p, bool build_graph) {
    validate_params(p);
    if (!g || g->n == 0) fail(PRGPU_EINVAL, "pagerank: graph has no vertices");
    DeviceGuard dg(g->device);
    auto s = std::make_unique<prgpu_session>();
    s->g = g;
    s->K = p->lanes;
    s->cfg = lane_cfg(s->K);
    s->KP = s->cfg.LG * s->cfg.W;
    s->max_iter = p->max_iterations;
    s->pull = pick_pull(s->cfg);
    const size_t n = g->n;
    const int K = s->K, KP = s->KP;
    cudaStream_t st = s->stream;

    s->rank.alloc(2 * (size_t)K * n);
    s->contrib.alloc(2 * n * KP);
    PRGPU_CUDA(cudaMemsetAsync(s->contrib.p, 0, 2 * n * KP * sizeof(double), st));
    s->trace.alloc((size_t)s->max_iter * K * 4);
    PRGPU_CUDA(cudaMemsetAsync(s->trace.p, 0, (size_t)s->max_iter * K * 4 * sizeof(double), st));
    s->lanes.alloc(K);
    s->gs.alloc(1);

    s->lanes_host.resize(K);
    for (int k = 0; k < K; ++k) {
        LaneState& L = s->lanes_host[k];
        L = LaneState{};
        L.alpha = p->alphas[k];
        L.tol = p->tolerances ? p->tolerances[k] : p->tolerance;
        L.stop_mask = p->stop_mask ? p->stop_mask : (1u << p->norm);
        L.report_norm = p->norm;
    }
    PRGPU_CUDA(cudaMemcpyAsync(s->lanes.p, s->lanes_host.data(), K * sizeof(LaneState),
                               cudaMemcpyHostToDevice, st));
    GlobalState gsh{0, 1, 0u, s->max_iter};
    PRGPU_CUDA(cudaMemcpyAsync(s->gs.p, &gsh, sizeof(gsh), cudaMemcpyHostToDevice, st));

    if (p->ref_ranks) {
        DevBuf<double> tmp(n);
        s->ref.alloc(n);
        PRGPU_CUDA(cudaMemcpyAsync(tmp.p, p->ref_ranks, n * 8, cudaMemcpyHostToDevice, st));
        scatter_ref<<<(unsigned)std::min<size_t>((n + kNT - 1) / kNT, 148 * 16), kNT, 0, st>>>(
            tmp.p, g->new_of_old.p, s->ref.p, g->n);
        PRGPU_LAUNCHED("scatter_ref");
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }

    // persistent grid and the cost-balanced item ranges
    int dev_sms = 0, per_sm = 0;
    PRGPU_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, g->device));
    PRGPU_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)s->pull, kNT, 0));
    per_sm = std::max(1, per_sm);
    const uint32_t TR = kNT / s->cfg.LG;
    const uint32_t items_hub = g->hub_end;
    const uint32_t items_warp = (g->warp_end - g->hub_end + (kNT / 32) - 1) / (kNT / 32);
    const uint32_t items_thread = (uint32_t)((n - g->warp_end + TR - 1) / TR);
    const uint32_t items = items_hub + items_warp + items_thread;
    // enough work per CTA to amortise the partial reduction
    const uint64_t work = g->e + (uint64_t)kRowCost * n;
    uint32_t G = (uint32_t)std::min<uint64_t>((uint64_t)dev_sms * per_sm,
                                              std::max<uint64_t>(1, work / 2048));
    G = std::max(1u, std::min(G, std::max(1u, items)));
    s->partials.alloc((size_t)kNQ * KP * G);
    s->block_begin.alloc(G + 1);
    {
        DevBuf<uint64_t> cost(std::max(1u, items));
        item_costs<<<std::max(1u, std::min((items + kNT - 1) / kNT, 148u * 16)), kNT, 0, st>>>(
            g->row_off.p, g->n, g->hub_end, g->warp_end, items_hub, items_warp, items, TR, cost.p);
        PRGPU_LAUNCHED("item_costs");
        size_t tmp = 0;
        PRGPU_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cost.p, cost.p, (int64_t)items, st));
        DevBuf<char> t(std::max<size_t>(tmp, 1));
        PRGPU_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, cost.p, cost.p, (int64_t)items, st));
        g_launches.fetch_add(1);
        block_ranges<<<(G + kNT) / kNT, kNT, 0, st>>>(cost.p, items, G, s->block_begin.p);
        PRGPU_LAUNCHED("block_ranges");
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }

    Params& P = s->P;
    P.n = g->n;
    P.K = K;
    P.row_off = g->row_off.p;
    P.col = g->col.p;
    P.deg = g->deg.p;
    P.rank[0] = s->rank.p;
    P.rank[1] = s->rank.p + (size_t)K * n;
    P.contrib[0] = s->contrib.p;
    P.contrib[1] = s->contrib.p + n * KP;
    P.ref = s->ref.p;
    P.partials = s->partials.p;
    P.trace = s->trace.p;
    P.lanes = s->lanes.p;
    P.gs = s->gs.p;
    P.block_begin = s->block_begin.p;
    P.hub_end = g->hub_end;
    P.warp_end = g->warp_end;
    P.items_hub = items_hub;
    P.items_warp = items_warp;
    P.G = G;
    P.use_cond = 0;

    PRGPU_CUDA(cudaEventCreate(&s->e0));
    PRGPU_CUDA(cudaEventCreate(&s->e1));

    if (build_graph) {
        // graph: WHILE(cond) { pull_kernel }  — cond defaults to 1 at every launch
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
        P.use_cond = 1;
        P.cond = h;
        cudaKernelNodeParams kp = {};
        kp.func = (void*)s->pull;
        kp.gridDim = dim3(G);
        kp.blockDim = dim3(kNT);
        kp.sharedMemBytes = 0;
        void* args[] = {&s->P};
        kp.kernelParams = args;
        cudaGraphNode_t knode;
        PRGPU_CUDA(cudaGraphAddKernelNode(&knode, body, nullptr, 0, &kp));
        PRGPU_CUDA(cudaGraphInstantiate(&s->exec, s->graph, 0));
        s->use_graph = true;
    }
    return s.release();
}

void session_destroy(prgpu_session* s) {
    if (!s) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(s->g->device);
    delete s;
    cudaSetDevice(prev);
}

void session_init(prgpu_session* s) {
    PRGPU_CUDA(cudaMemcpyAsync(s->lanes.p, s->lanes_host.data(), s->K * sizeof(LaneState),
                               cudaMemcpyHostToDevice, s->stream));
    GlobalState gsh{0, 1, 0u, s->max_iter};
    PRGPU_CUDA(cudaMemcpyAsync(s->gs.p, &gsh, sizeof(gsh), cudaMemcpyHostToDevice, s->stream));
    launch_init(s->cfg, s->P, s->g->ndangling, s->stream);
}

void launch_pull(prgpu_session* s) {
    Params P = s->P;
    P.use_cond = 0;
    s->pull<<<P.G, kNT, 0, s->stream>>>(P);
    PRGPU_LAUNCHED("pull_kernel");
}

int read_any_active(prgpu_session* s) {
    GlobalState gsh;
    PRGPU_CUDA(cudaMemcpyAsync(&gsh, s->gs.p, sizeof(gsh), cudaMemcpyDeviceToHost, s->stream));
    PRGPU_CUDA(cudaStreamSynchronize(s->stream));
    return gsh.any_active;
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
    std::vector<LaneState> L(s->K);
    PRGPU_CUDA(cudaMemcpyAsync(L.data(), s->lanes.p, s->K * sizeof(LaneState),
                               cudaMemcpyDeviceToHost, st));
    GlobalState gsh;
    PRGPU_CUDA(cudaMemcpyAsync(&gsh, s->gs.p, sizeof(gsh), cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    const size_t n = s->g->n;
    if (out->ranks) {
        DevBuf<double> tmp((size_t)s->K * n);
        extract_ranks<<<(unsigned)std::min<size_t>((n + kNT - 1) / kNT, 148 * 16), kNT, 0, st>>>(
            s->P, s->g->new_of_old.p, tmp.p, -1, 0);
        PRGPU_LAUNCHED("extract_ranks");
        PRGPU_CUDA(cudaMemcpyAsync(out->ranks, tmp.p, (size_t)s->K * n * 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
    if (out->err_trace) {
        PRGPU_CUDA(cudaMemcpyAsync(out->err_trace, s->trace.p,
                                   (size_t)s->max_iter * s->K * 4 * sizeof(double),
                                   cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
    int maxit = 0;
    for (int k = 0; k < s->K; ++k) {
        if (out->iterations) out->iterations[k] = L[k].iterations;
        if (out->converged) out->converged[k] = (uint8_t)L[k].converged;
        if (out->final_err) out->final_err[k] = L[k].final_err;
        maxit = std::max(maxit, L[k].iterations);
    }
    out->run_iterations = gsh.iter;
    out->loop_ms = s->last_loop_ms;
    (void)maxit;
}

void session_observed(prgpu_session* s, prgpu_result* out, prgpu_observer_fn fn, void* user) {
    DeviceGuard dg(s->g->device);
    cudaStream_t st = s->stream;
    const size_t n = s->g->n;
    session_init(s);
    DevBuf<double> tmp(n);
    std::vector<double> host(n);
    std::vector<LaneState> L(s->K);
    PRGPU_CUDA(cudaEventRecord(s->e0, st));
    for (int it = 0; it < s->max_iter; ++it) {
        std::vector<LaneState> before(s->K);
        PRGPU_CUDA(cudaMemcpyAsync(before.data(), s->lanes.p, s->K * sizeof(LaneState),
                                   cudaMemcpyDeviceToHost, st));
        launch_pull(s);
        PRGPU_CUDA(cudaMemcpyAsync(L.data(), s->lanes.p, s->K * sizeof(LaneState),
                                   cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < s->K; ++k) {
            if (!before[k].active) continue;
            if (fn) {
                extract_ranks<<<(unsigned)std::min<size_t>((n + kNT - 1) / kNT, 148 * 16), kNT, 0,
                                st>>>(s->P, s->g->new_of_old.p, tmp.p, k, 1);
                PRGPU_LAUNCHED("extract_ranks");
                PRGPU_CUDA(cudaMemcpyAsync(host.data(), tmp.p, n * 8, cudaMemcpyDeviceToHost, st));
                PRGPU_CUDA(cudaStreamSynchronize(st));
                fn(L[k].iterations, k, host.data(), n, L[k].final_err, user);
            }
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

double session_time_pull(prgpu_session* s, int launches) {
    // host-loop run with an event pair per launch; mean device time per launch
    DeviceGuard dg(s->g->device);
    session_init(s);
    cudaStream_t st = s->stream;
    std::vector<cudaEvent_t> ev(2 * (size_t)launches);
    for (auto& e : ev) PRGPU_CUDA(cudaEventCreate(&e));
    int done = 0;
    for (; done < launches; ++done) {
        PRGPU_CUDA(cudaEventRecord(ev[2 * done], st));
        launch_pull(s);
        PRGPU_CUDA(cudaEventRecord(ev[2 * done + 1], st));
        if (!read_any_active(s)) { ++done; break; }
    }
    double total = 0;
    for (int i = 0; i < done; ++i) {
        float ms = 0;
        PRGPU_CUDA(cudaEventElapsedTime(&ms, ev[2 * i], ev[2 * i + 1]));
        total += ms;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return done ? total / done : 0.0;
}

double error_norm_device(int kind, const double* r, const double* s, uint64_t n, int device) {
    if (kind < 0 || kind > 2) fail(PRGPU_EINVAL, "error_norm: unknown norm");
    if (n == 0) fail(PRGPU_EINVAL, "error_norm: empty vectors");
    DeviceGuard dg(device);
    Stream st;
    DevBuf<double> dr(n), ds(n), parts(296), out(1);
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
