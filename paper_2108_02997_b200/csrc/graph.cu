// graph.cu — K0: device in-CSR (transpose) construction, relabelling, the
// synthetic benchmark generators, and the reference-layout download.
//
// Replaces build_csr (graph.hpp:204-234): sort edges by (target, source)
// (:209-212), drop exact duplicates (:213), count in/out degrees (:220-223),
// scan (:224), fill in-neighbours (:226-228), dangling list (:230-231).
// Here the sort is a CUB radix sort of the packed key target<<lg | source
// (same total order), the counts are integer atomics (order-free, so the
// arrays are bit-identical to the reference's), and the scan is a device scan.
//
// The engine then relabels vertices by in-degree descending (ties: original
// id ascending) so the degree bins of the pull kernel are contiguous row
// ranges and the hottest rows/sources are packed at the front.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <type_traits>
#include <vector>

#include "common.cuh"

namespace prgpu {

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kLocalityMaxDeg = 8; // graphs up to this in-degree keep the caller's order (relabel)

inline unsigned grid_for(uint64_t n, int threads = kThreads) {
    uint64_t b = (n + threads - 1) / threads;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 64));
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

inline uint64_t mix64_host(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return mix64_host(seed * 0x9E3779B97F4A7C15ull + stream);
}

inline uint64_t prob_threshold(double p) {
    if (!(p > 0.0)) return 0;
    const double x = p * 18446744073709551616.0;
    if (x >= 18446744073709551616.0) return UINT64_MAX;
    return (uint64_t)x;
}

constexpr uint64_t kSentinel = ~0ull;

// ---- packing -----------------------------------------------------------------
__global__ void pairs_to_keys(const uint32_t* __restrict__ pairs, uint64_t m, uint32_t n,
                              uint32_t lg, uint64_t* __restrict__ keys, int* bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 p = reinterpret_cast<const uint2*>(pairs)[i];
        if (p.x >= n || p.y >= n) *bad = 1;
        keys[i] = ((uint64_t)p.y << lg) | p.x;
    }
}

// ---- synthetic generators (spec: DESIGN.md; host twin: oracle/oracle.c) -------
struct PermKeys {
    uint64_t k[3];
    uint64_t mask;
    uint32_t hs;
};

__device__ __forceinline__ uint32_t perm_apply(uint32_t x32, const PermKeys& pk) {
    uint64_t x = x32;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        x = (x * (pk.k[r] | 1ull)) & pk.mask;
        x = (x + (pk.k[r] >> 40)) & pk.mask;
        x ^= x >> pk.hs;
    }
    return (uint32_t)x;
}

__global__ void rmat_keys(uint64_t m, uint32_t scale, uint64_t kd, uint64_t ta, uint64_t tab,
                          uint64_t tabc, PermKeys pk, uint64_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t src = 0, dst = 0;
        for (uint32_t l = 0; l < scale; ++l) {
            const uint64_t x = mix64(kd ^ ((i << 6) | l));
            const uint32_t bit = 1u << (scale - 1 - l);
            if (x < ta) {
            } else if (x < tab) {
                dst |= bit;
            } else if (x < tabc) {
                src |= bit;
            } else {
                src |= bit;
                dst |= bit;
            }
        }
        keys[i] = (src == dst) ? kSentinel
                               : (((uint64_t)perm_apply(dst, pk) << scale) | perm_apply(src, pk));
    }
}

// rmat_keys restricted to edges whose (permuted) target lies in [dlo, dhi):
// appended in any order at a block-aggregated cursor (the slab is sorted
// afterwards); keys past `cap` are counted, not written (caller retries)
__global__ void __launch_bounds__(256) rmat_keys_slab(uint64_t m, uint32_t scale, uint64_t kd, uint64_t ta,
                                                      uint64_t tab, uint64_t tabc, PermKeys pk, uint32_t dlo,
                                                      uint32_t dhi, uint64_t* __restrict__ keys, uint64_t cap,
                                                      unsigned long long* __restrict__ cnt) {
    __shared__ unsigned s_w[8];
    __shared__ unsigned long long s_base;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < m; i0 += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = i0 + threadIdx.x;
        bool keep = false;
        uint64_t key = 0;
        if (i < m) {
            uint32_t src = 0, dst = 0;
            for (uint32_t l = 0; l < scale; ++l) {
                const uint64_t x = mix64(kd ^ ((i << 6) | l));
                const uint32_t bit = 1u << (scale - 1 - l);
                if (x < ta) {
                } else if (x < tab) {
                    dst |= bit;
                } else if (x < tabc) {
                    src |= bit;
                } else {
                    src |= bit;
                    dst |= bit;
                }
            }
            if (src != dst) {
                const uint32_t d = perm_apply(dst, pk);
                keep = d >= dlo && d < dhi;
                key = ((uint64_t)d << scale) | perm_apply(src, pk);
            }
        }
        const unsigned b = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_w[warp] = __popc(b);
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < 8; ++w) t += s_w[w];
            s_base = t ? atomicAdd(cnt, t) : 0ull;
        }
        __syncthreads();
        unsigned before = 0;
        for (uint32_t w = 0; w < warp; ++w) before += s_w[w];
        const uint64_t at = s_base + before + __popc(b & ((1u << lane) - 1u));
        if (keep && at < cap) keys[at] = key;
        __syncthreads();
    }
}

// shard boundaries: cost of engine row r (in-degree + 2 for rows with
// in-edges, 1 for the rest)
__global__ void shard_costs(const uint64_t* __restrict__ row_off, uint32_t n, uint32_t nonempty_end,
                            uint64_t* __restrict__ cost) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x)
        cost[r] = r < nonempty_end ? (row_off[r + 1] - row_off[r]) + 2 : 1;
}
__global__ void shard_search(const uint64_t* __restrict__ excl, uint32_t n, uint32_t nranks,
                             uint32_t* __restrict__ out) {
    const uint32_t b = threadIdx.x;
    if (b > nranks) return;
    if (b == 0 || b == nranks) {
        out[b] = b ? n : 0;
        return;
    }
    const uint64_t target = excl[n] * b / nranks;
    uint32_t lo = 0, hi = n; // first row whose exclusive prefix >= target
    while (lo < hi) {
        const uint32_t mid = lo + (hi - lo) / 2;
        if (excl[mid] < target) lo = mid + 1;
        else hi = mid;
    }
    out[b] = lo;
}

__global__ void grid_keys(uint32_t side, uint64_t uh, uint64_t tp, uint64_t kg, uint64_t L,
                          uint64_t kl, uint64_t n, uint32_t lg, uint64_t* __restrict__ keys) {
    const uint64_t total = 2 * uh; // candidates
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < total + L;
         t += (uint64_t)gridDim.x * blockDim.x) {
        if (t < total) {
            uint64_t a, b;
            if (t < uh) {
                const uint64_t r = t / (side - 1), c = t % (side - 1);
                a = r * side + c;
                b = a + 1;
            } else {
                const uint64_t j = t - uh;
                const uint64_t r = j / side, c = j % side;
                a = r * side + c;
                b = a + side;
            }
            const bool keep = mix64(kg ^ t) < tp;
            keys[2 * t] = keep ? ((b << lg) | a) : kSentinel;     // a -> b
            keys[2 * t + 1] = keep ? ((a << lg) | b) : kSentinel; // b -> a
        } else {
            const uint64_t j = t - total;
            const uint64_t s = __umul64hi(mix64(kl ^ (2 * j)), n);
            const uint64_t d = __umul64hi(mix64(kl ^ (2 * j + 1)), n);
            keys[2 * total + j] = (s == d) ? kSentinel : ((d << lg) | s);
        }
    }
}

// ---- CSR assembly ---------------------------------------------------------------
__global__ void count_degrees(const uint64_t* __restrict__ keys, uint64_t u, uint32_t lg,
                              uint32_t* __restrict__ in_deg, uint32_t* __restrict__ out_deg) {
    const uint64_t mask = (1ull << lg) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < u;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        atomicAdd(&in_deg[k >> lg], 1u);
        atomicAdd(&out_deg[k & mask], 1u);
    }
}

__global__ void iota_u32(uint32_t* __restrict__ v, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        v[i] = (uint32_t)i;
}

__global__ void degree_keys(const uint32_t* __restrict__ in_deg, const uint32_t* __restrict__ out_deg,
                            uint64_t* __restrict__ out, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = ((uint64_t)(~in_deg[i]) << 32) | (uint32_t)(~out_deg[i]);
}

// low-degree graphs (max in-degree <= kLocalityMaxDeg): keep the caller's
// order inside three classes — rows with in-edges, rows with only out-edges,
// isolated rows — so neighbouring ids stay neighbours (road/grid graphs)
__global__ void locality_keys(const uint32_t* __restrict__ in_deg, const uint32_t* __restrict__ out_deg,
                              uint64_t* __restrict__ out, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint64_t)(in_deg[i] ? 0u : (out_deg[i] ? 1u : 2u)) << 32;
}

__global__ void max_u32(const uint32_t* __restrict__ x, uint32_t n, unsigned int* __restrict__ out) {
    uint32_t m = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        m = max(m, x[i]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void invert_perm(const uint32_t* __restrict__ old_of_new, uint32_t* __restrict__ new_of_old,
                            uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        new_of_old[old_of_new[i]] = (uint32_t)i;
}

__global__ void relabel_keys(uint64_t* __restrict__ keys, uint64_t u, uint32_t lg,
                             const uint32_t* __restrict__ map) {
    const uint64_t mask = (1ull << lg) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < u;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = keys[i];
        keys[i] = ((uint64_t)map[k >> lg] << lg) | map[k & mask];
    }
}

// out[i] = (u64) src[perm[i]]  (perm may be null: identity); out[n] = 0
__global__ void gather_deg_u64(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm,
                               uint64_t* __restrict__ out, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (i < n) ? (uint64_t)src[perm ? perm[i] : i] : 0ull;
}

__global__ void gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm,
                           uint32_t* __restrict__ out, uint32_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = src[perm[i]];
}

__global__ void keys_low(const uint64_t* __restrict__ keys, uint64_t u, uint32_t lg,
                         uint32_t* __restrict__ col) {
    const uint64_t mask = (1ull << lg) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < u;
         i += (uint64_t)gridDim.x * blockDim.x)
        col[i] = (uint32_t)(keys[i] & mask);
}

template <typename T>
__device__ __forceinline__ void block_add(T v, unsigned long long* dst) {
    __shared__ unsigned long long s_sum[kThreads / 32];
    unsigned long long x = (unsigned long long)v;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
    if ((threadIdx.x & 31) == 0) s_sum[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += s_sum[w];
        if (t) atomicAdd(dst, t);
    }
    __syncthreads();
}

// bins over rows sorted by in-degree descending: counts of rows above thresholds
// counts[0..2]: rows with in-degree > 4096, > 32, > 0; counts[4..6]: > 512, > 128, > 8
__global__ void bin_counts(const uint64_t* __restrict__ row_off, uint32_t n,
                           unsigned long long* __restrict__ counts /*9*/) {
    unsigned long long c0 = 0, c1 = 0, c2 = 0, c4 = 0, c5 = 0, c6 = 0, c7 = 0, c8 = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t d = row_off[i + 1] - row_off[i];
        c0 += d > kHubMinDegree;
        c1 += d > kWarpMinDegree;
        c2 += d > 0;
        c4 += d > 512;
        c5 += d > 256;
        c6 += d > 128;
        c7 += d > 64;
        c8 += d > 8;
    }
    block_add(c0, &counts[0]);
    block_add(c1, &counts[1]);
    block_add(c2, &counts[2]);
    block_add(c4, &counts[4]);
    block_add(c5, &counts[5]);
    block_add(c6, &counts[6]);
    block_add(c7, &counts[7]);
    block_add(c8, &counts[8]);
}

__global__ void count_zero(const uint32_t* __restrict__ v, uint32_t n,
                           unsigned long long* __restrict__ count) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        c += v[i] == 0;
    block_add(c, count);
}

// ---- edge-parallel CSR passes ------------------------------------------------------
// Block b covers edges [b*kEdgeChunk, (b+1)*kEdgeChunk); the row of an edge is
// the last row o with off[o] <= j, found by binary search inside the rows the
// chunk spans (so hub rows are split across blocks: no per-row stragglers).
constexpr uint32_t kEdgeChunk = 4096;

__device__ __forceinline__ uint32_t last_row_le(const uint64_t* __restrict__ off, uint32_t lo, uint32_t hi,
                                                uint64_t j) {
    while (lo < hi) { // largest o in [lo, hi] with off[o] <= j
        const uint32_t mid = lo + (hi - lo + 1) / 2;
        if (off[mid] <= j) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__device__ __forceinline__ void chunk_rows(const uint64_t* __restrict__ off, uint32_t n, uint64_t j0,
                                           uint64_t j1, uint32_t& r0, uint32_t& r1) {
    __shared__ uint32_t s_r[2];
    if (threadIdx.x == 0) {
        s_r[0] = last_row_le(off, 0, n - 1, j0);
        s_r[1] = last_row_le(off, 0, n - 1, j1 - 1);
    }
    __syncthreads();
    r0 = s_r[0];
    r1 = s_r[1];
}

// offsets monotone (off[0] == 0 is checked on the host)
__global__ void check_offsets(const uint64_t* __restrict__ off, uint32_t n, uint64_t e, int* bad) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        if (off[v + 1] < off[v] || off[v + 1] > e) *bad = 1;
}

// Engine CSR fill for edges [jb, je) of the original CSR: edge j of original
// row o lands at row_off[new(o)] + (j - off[o]) as the engine source id of
// its in-neighbour (rows keep the caller's neighbour order until sorted).
// With `bad` (graph_from_csr), also validates what pagerank() needs of a
// hand-filled CsrGraph: in-neighbours in range (graph.hpp:56-59) and with a
// nonzero caller out-degree (pagerank.hpp:91 divides by it).  Like the
// reference, rows may hold duplicates and any order, and out_degree is used
// as given (it need not equal the in-neighbour histogram).
__global__ void place_edges(const uint64_t* __restrict__ off, const uint32_t* __restrict__ nbr, uint32_t n,
                            uint64_t jb, uint64_t je, const uint32_t* __restrict__ new_of_old,
                            const uint64_t* __restrict__ row_off, const uint32_t* __restrict__ src_of_old,
                            uint32_t* __restrict__ col, const uint32_t* __restrict__ out_deg, int* bad,
                            uint32_t rb = 0, uint32_t re = 0xFFFFFFFFu, uint64_t col_base = 0) {
    const uint64_t j0 = jb + (uint64_t)blockIdx.x * kEdgeChunk, j1 = min(j0 + kEdgeChunk, je);
    uint32_t r0, r1;
    chunk_rows(off, n, j0, j1, r0, r1);
    for (uint64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) {
        const uint32_t u = nbr[j];
        const uint32_t o = last_row_le(off, r0, r1, j);
        if (bad) {
            if (u >= n) { *bad = 1; continue; }
            if (out_deg[u] == 0) { *bad = 2; continue; }
        }
        const uint32_t r = new_of_old[o];
        if (r < rb || r >= re) continue; // a shard keeps its own rows only
        col[row_off[r] + (j - off[o]) - col_base] = src_of_old[u];
    }
}

__global__ void in_deg_from_off(const uint64_t* __restrict__ off, uint32_t n, uint32_t* __restrict__ d) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        d[v] = (uint32_t)(off[v + 1] - off[v]);
}

__global__ void src_of_old_kernel(const uint2* __restrict__ rowinfo, const uint32_t* __restrict__ new_of_old,
                                  uint32_t n, uint32_t* __restrict__ out) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        out[v] = rowinfo[new_of_old[v]].y;
}

// engine CSR -> original-id keys (for download)
__global__ void engine_to_orig_keys(const uint64_t* __restrict__ row_off,
                                    const uint32_t* __restrict__ col,
                                    const uint32_t* __restrict__ row_of_src,
                                    const uint32_t* __restrict__ old_of_new, uint32_t n,
                                    uint32_t lg, uint64_t* __restrict__ keys) {
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < n;
         r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t dst = old_of_new[r];
        for (uint64_t j = row_off[r]; j < row_off[r + 1]; ++j)
            keys[j] = (dst << lg) | old_of_new[row_of_src[col[j]]];
    }
}

// in-degrees of requested original rows (graph_rows)
__global__ void rows_deg(const uint64_t* __restrict__ row_off, const uint32_t* __restrict__ new_of_old,
                         const uint32_t* __restrict__ rows, uint32_t nrows, uint64_t* __restrict__ cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nrows; i += gridDim.x * blockDim.x) {
        const uint32_t r = new_of_old[rows[i]];
        cnt[i] = row_off[r + 1] - row_off[r];
    }
}

// in-neighbours (original ids, engine order) of requested rows: one warp per row
__global__ void rows_fill(const uint64_t* __restrict__ row_off, const uint32_t* __restrict__ col,
                          const uint32_t* __restrict__ row_of_src, const uint32_t* __restrict__ old_of_new,
                          const uint32_t* __restrict__ new_of_old, const uint32_t* __restrict__ rows,
                          uint32_t nrows, const uint64_t* __restrict__ out_off, uint32_t* __restrict__ out) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < nrows;
         i += (gridDim.x * blockDim.x) >> 5) {
        const uint32_t r = new_of_old[rows[i]];
        const uint64_t lo = row_off[r], d = row_off[r + 1] - lo;
        for (uint64_t j = lane; j < d; j += 32) out[out_off[i] + j] = old_of_new[row_of_src[col[lo + j]]];
    }
}

__global__ void in_deg_orig(const uint64_t* __restrict__ row_off,
                            const uint32_t* __restrict__ new_of_old, uint32_t n,
                            uint64_t* __restrict__ out) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        if (v == n) { out[v] = 0; continue; }
        const uint32_t r = new_of_old[v];
        out[v] = row_off[r + 1] - row_off[r];
    }
}

__global__ void src_flags(const uint32_t* __restrict__ deg, uint32_t n, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= n;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (i < n && deg[i] > 0) ? 1ull : 0ull;
}

// rowinfo[i] = {deg, src id}; row_of_src[src] = i
__global__ void src_maps(const uint32_t* __restrict__ deg, const uint64_t* __restrict__ excl,
                         uint32_t n, uint2* __restrict__ rowinfo, uint32_t* __restrict__ row_of_src) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t d = deg[i];
        const uint32_t s = (uint32_t)excl[i];
        rowinfo[i] = make_uint2(d, d ? s : 0xFFFFFFFFu);
        if (d) row_of_src[s] = (uint32_t)i;
    }
}

// ---- sources ascending within rows --------------------------------------------------
// The scatter leaves each row in the caller's neighbour order; sorting rows by
// engine source id makes the gathers of a warp task walk the contribution
// table monotonically (measured: -6% pull time on C2, -8% on C4; hub rows
// (> 4096 in-edges) and rows of <= 8 gain nothing and are left as they are).
// Rows are sorted by in-degree, so each size class is a contiguous row range.
template <int ITEMS>
__global__ void __launch_bounds__(256) sort_rows_warp(const uint64_t* __restrict__ row_off, uint32_t r0,
                                                     uint32_t r1, uint32_t* __restrict__ col) {
    using Sort = cub::WarpMergeSort<uint32_t, ITEMS, 32>;
    __shared__ typename Sort::TempStorage tmp[8];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t r = r0 + blockIdx.x * 8 + warp;
    if (r >= r1) return;
    const uint64_t lo = row_off[r];
    const int d = (int)(row_off[r + 1] - lo);
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int j = lane * ITEMS + i;
        k[i] = j < d ? col[lo + j] : 0xFFFFFFFFu;
    }
    Sort(tmp[warp]).Sort(k, [](uint32_t a, uint32_t b) { return a < b; });
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int j = lane * ITEMS + i;
        if (j < d) col[lo + j] = k[i];
    }
}

__global__ void __launch_bounds__(256) sort_rows_block(const uint64_t* __restrict__ row_off, uint32_t r0,
                                                      int end_bit, uint32_t* __restrict__ col) {
    using Sort = cub::BlockRadixSort<uint32_t, 256, 16>;
    __shared__ typename Sort::TempStorage tmp;
    const uint32_t r = r0 + blockIdx.x;
    const uint64_t lo = row_off[r];
    const int d = (int)(row_off[r + 1] - lo);
    uint32_t k[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int j = threadIdx.x * 16 + i;
        k[i] = j < d ? col[lo + j] : 0xFFFFFFFFu;
    }
    Sort(tmp).Sort(k, 0, end_bit);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const int j = threadIdx.x * 16 + i;
        if (j < d) col[lo + j] = k[i];
    }
}

// Per-slice variant for graph_from_csr: the caller's rows [v0, v1) (original
// ids) whose edges have all been placed, one warp per row, each sorted at
// the width of its length band; rows of 513..4096 are appended to `big` for
// sort_rows_listed (one block per row).
template <int ITEMS>
__device__ __forceinline__ void warp_sort_row(uint32_t* col, uint64_t lo, int d, int lane, void* tmp) {
    using Sort = cub::WarpMergeSort<uint32_t, ITEMS, 32>;
    uint32_t k[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int j = lane * ITEMS + i;
        k[i] = j < d ? col[lo + j] : 0xFFFFFFFFu;
    }
    Sort(*reinterpret_cast<typename Sort::TempStorage*>(tmp)).Sort(k, [](uint32_t a, uint32_t b) { return a < b; });
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const int j = lane * ITEMS + i;
        if (j < d) col[lo + j] = k[i];
    }
}

__global__ void __launch_bounds__(256) sort_rows_orig(const uint64_t* __restrict__ row_off,
                                                     const uint32_t* __restrict__ new_of_old, uint32_t v0,
                                                     uint32_t v1, uint32_t* __restrict__ big,
                                                     unsigned* __restrict__ nbig, uint32_t* __restrict__ col) {
    constexpr size_t kTmp = sizeof(typename cub::WarpMergeSort<uint32_t, 16, 32>::TempStorage);
    __shared__ __align__(16) unsigned char tmp[8][kTmp];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t v = v0 + (uint64_t)blockIdx.x * 8 + warp;
    if (v >= v1) return;
    const uint32_t r = new_of_old[v];
    const uint64_t lo = row_off[r];
    const int d = (int)(row_off[r + 1] - lo);
    if (d <= 8 || d > (int)kHubMinDegree) return;
    if (d > 512) {
        if (lane == 0) big[atomicAdd(nbig, 1u)] = r;
        return;
    }
    if (d <= 32) warp_sort_row<1>(col, lo, d, lane, tmp[warp]);
    else if (d <= 64) warp_sort_row<2>(col, lo, d, lane, tmp[warp]);
    else if (d <= 128) warp_sort_row<4>(col, lo, d, lane, tmp[warp]);
    else if (d <= 256) warp_sort_row<8>(col, lo, d, lane, tmp[warp]);
    else warp_sort_row<16>(col, lo, d, lane, tmp[warp]);
}

// the rows appended since the last call: big[done[0] .. nbig), block per row
__global__ void __launch_bounds__(256) sort_rows_listed(const uint64_t* __restrict__ row_off,
                                                       const uint32_t* __restrict__ big,
                                                       const unsigned* __restrict__ nbig,
                                                       const unsigned* __restrict__ done, int end_bit,
                                                       uint32_t* __restrict__ col) {
    using Sort = cub::BlockRadixSort<uint32_t, 256, 16>;
    __shared__ typename Sort::TempStorage tmp;
    const unsigned e = *nbig;
    for (unsigned i = done[0] + blockIdx.x; i < e; i += gridDim.x) {
        const uint32_t r = big[i];
        const uint64_t lo = row_off[r];
        const int d = (int)(row_off[r + 1] - lo);
        uint32_t k[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int j = threadIdx.x * 16 + q;
            k[q] = j < d ? col[lo + j] : 0xFFFFFFFFu;
        }
        Sort(tmp).Sort(k, 0, end_bit);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const int j = threadIdx.x * 16 + q;
            if (j < d) col[lo + j] = k[q];
        }
        __syncthreads(); // tmp is reused by the next row
    }
}

__global__ void mark_listed(const unsigned* __restrict__ nbig, unsigned* __restrict__ done) { done[0] = *nbig; }

// source ids in original-id order (tuning: PRGPU_SRC_ORDER=1)
__global__ void src_maps_orig(const uint32_t* __restrict__ deg, const uint64_t* __restrict__ excl_old,
                              const uint32_t* __restrict__ old_of_new, uint32_t n,
                              uint2* __restrict__ rowinfo, uint32_t* __restrict__ row_of_src) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t d = deg[i];
        const uint32_t s = (uint32_t)excl_old[old_of_new[i]];
        rowinfo[i] = make_uint2(d, d ? s : 0xFFFFFFFFu);
        if (d) row_of_src[s] = (uint32_t)i;
    }
}

// col: engine row ids -> source ids (every in-neighbour has out-degree >= 1)
__global__ void col_to_src(uint32_t* __restrict__ col, uint64_t e, const uint2* __restrict__ rowinfo) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < e;
         j += (uint64_t)gridDim.x * blockDim.x)
        col[j] = rowinfo[col[j]].y;
}

struct IsZero {
    const uint32_t* deg;
    __device__ bool operator()(uint32_t v) const { return deg[v] == 0; }
};

// ---- host helpers -----------------------------------------------------------------
void sort_keys(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& alt, uint64_t m, int end_bit,
               cudaStream_t st) {
    if (m < 2) return;
    cub::DoubleBuffer<uint64_t> db(keys.p, alt.p);
    size_t tmp = 0;
    PRGPU_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, m, 0, end_bit, st));
    DevBuf<char> t(tmp);
    PRGPU_CUDA(cub::DeviceRadixSort::SortKeys(t.p, tmp, db, m, 0, end_bit, st));
    g_launches.fetch_add(1);
    if (db.Current() != keys.p) std::swap(keys, alt);
}

uint64_t unique_keys(DevBuf<uint64_t>& keys, DevBuf<uint64_t>& alt, uint64_t m, cudaStream_t st) {
    if (m == 0) return 0;
    DevBuf<long long> nsel(1);
    size_t tmp = 0;
    PRGPU_CUDA(cub::DeviceSelect::Unique(nullptr, tmp, keys.p, alt.p, nsel.p, (int64_t)m, st));
    DevBuf<char> t(tmp);
    PRGPU_CUDA(cub::DeviceSelect::Unique(t.p, tmp, keys.p, alt.p, nsel.p, (int64_t)m, st));
    g_launches.fetch_add(1);
    long long u = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&u, nsel.p, sizeof(u), cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    std::swap(keys, alt);
    return (uint64_t)u;
}

void exclusive_scan_u64(uint64_t* data, uint64_t count, cudaStream_t st) {
    size_t tmp = 0;
    PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, data, data, (int64_t)count, st));
    DevBuf<char> t(tmp);
    PRGPU_CUDA(cub::DeviceScan::ExclusiveSum(t.p, tmp, data, data, (int64_t)count, st));
    g_launches.fetch_add(1);
}

int read_flag(const DevBuf<int>& f, cudaStream_t st) {
    int v = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&v, f.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    return v;
}

// Original-label CSR on the device (off[n+1], nbr[e] ascending per row,
// out-degrees) -> engine graph, in two halves: the vertex side (relabelling,
// row offsets, source ids) needs only off and the degrees, so graph_from_csr
// runs it while the neighbour array is still in flight from the host.
// The inputs are not modified.
std::unique_ptr<prgpu_graph> assemble_vertices(uint32_t n, const uint64_t* off, uint64_t e,
                                               const uint32_t* out_deg, uint32_t lg, int device,
                                               cudaStream_t st) {
    PhaseLog ph("assemble", st);
    auto g = std::make_unique<prgpu_graph>();
    g->device = device;
    g->n = n;
    g->e = e;
    g->lg = lg;

    DevBuf<uint32_t> in_deg(n);
    in_deg_from_off<<<grid_for(n), kThreads, 0, st>>>(off, n, in_deg.p);
    PRGPU_LAUNCHED("in_deg_from_off");

    // relabel: stable sort of vertices by (in-degree desc, out-degree desc, id):
    // degree bins become contiguous row ranges, and within each in-degree class
    // the most-gathered sources (high out-degree) are packed together.  Graphs
    // whose in-degrees are all small (no hub rows, no row to sort) keep the
    // caller's order within the nonempty / out-only / isolated classes instead:
    // their gathers then follow the caller's locality (measured C3 grid: the
    // degree order costs +5% pull time).  PRGPU_LOCALITY=0/1 overrides.
    uint32_t max_in = 0;
    {
        DevBuf<unsigned int> mx(1);
        PRGPU_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned int), st));
        max_u32<<<grid_for(n), kThreads, 0, st>>>(in_deg.p, n, mx.p);
        PRGPU_LAUNCHED("max_u32");
        PRGPU_CUDA(cudaMemcpyAsync(&max_in, mx.p, sizeof(max_in), cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
    bool locality = max_in <= kLocalityMaxDeg;
    if (const char* lv = std::getenv("PRGPU_LOCALITY")) locality = locality && std::atoi(lv) != 0;
    g->locality = locality;
    {
        DevBuf<uint64_t> kin(n), kout(n);
        DevBuf<uint32_t> vin(n);
        g->old_of_new.alloc(n);
        if (locality) locality_keys<<<grid_for(n), kThreads, 0, st>>>(in_deg.p, out_deg, kin.p, n);
        else degree_keys<<<grid_for(n), kThreads, 0, st>>>(in_deg.p, out_deg, kin.p, n);
        PRGPU_LAUNCHED("degree_keys");
        iota_u32<<<grid_for(n), kThreads, 0, st>>>(vin.p, n);
        PRGPU_LAUNCHED("iota_u32");
        const int b0 = locality ? 32 : 0, b1 = locality ? 34 : 64;
        size_t tmp = 0;
        PRGPU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin.p, kout.p, vin.p,
                                                   g->old_of_new.p, (int64_t)n, b0, b1, st));
        DevBuf<char> t(tmp);
        PRGPU_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kin.p, kout.p, vin.p,
                                                   g->old_of_new.p, (int64_t)n, b0, b1, st));
        g_launches.fetch_add(1);
        g->new_of_old.alloc(n);
        invert_perm<<<grid_for(n), kThreads, 0, st>>>(g->old_of_new.p, g->new_of_old.p, n);
        PRGPU_LAUNCHED("invert_perm");
    }
    ph.mark("relabel sort");

    g->row_off.alloc((size_t)n + 1);
    gather_deg_u64<<<grid_for((uint64_t)n + 1), kThreads, 0, st>>>(in_deg.p, g->old_of_new.p,
                                                                    g->row_off.p, n);
    PRGPU_LAUNCHED("gather_deg_u64");
    exclusive_scan_u64(g->row_off.p, (uint64_t)n + 1, st);
    g->deg.alloc(n);
    gather_u32<<<grid_for(n), kThreads, 0, st>>>(out_deg, g->old_of_new.p, g->deg.p, n);
    PRGPU_LAUNCHED("gather_u32");

    // compact source ids: contributions are stored for out-degree > 0 only
    {
        DevBuf<uint64_t> flags((size_t)n + 1);
        const char* so = std::getenv("PRGPU_SRC_ORDER");
        const bool orig = so && std::atoi(so) == 1;
        src_flags<<<grid_for((uint64_t)n + 1), kThreads, 0, st>>>(orig ? out_deg : g->deg.p, n, flags.p);
        PRGPU_LAUNCHED("src_flags");
        exclusive_scan_u64(flags.p, (uint64_t)n + 1, st);
        uint64_t nsrc = 0;
        PRGPU_CUDA(cudaMemcpyAsync(&nsrc, flags.p + n, 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        g->nsrc = (uint32_t)nsrc;
        g->rowinfo.alloc(n);
        g->row_of_src.alloc(std::max<uint64_t>(nsrc, 1));
        if (orig)
            src_maps_orig<<<grid_for(n), kThreads, 0, st>>>(g->deg.p, flags.p, g->old_of_new.p, n, g->rowinfo.p,
                                                            g->row_of_src.p);
        else
            src_maps<<<grid_for(n), kThreads, 0, st>>>(g->deg.p, flags.p, n, g->rowinfo.p,
                                                       g->row_of_src.p);
        PRGPU_LAUNCHED("src_maps");
    }
    ph.mark("row_off + source ids");
    DevBuf<unsigned long long> counts(9);
    PRGPU_CUDA(cudaMemsetAsync(counts.p, 0, 9 * sizeof(unsigned long long), st));
    bin_counts<<<grid_for(n), kThreads, 0, st>>>(g->row_off.p, n, counts.p);
    PRGPU_LAUNCHED("bin_counts");
    count_zero<<<grid_for(n), kThreads, 0, st>>>(out_deg, n, counts.p + 3);
    PRGPU_LAUNCHED("count_zero");
    unsigned long long c[9];
    uint64_t first_two[2];
    PRGPU_CUDA(cudaMemcpyAsync(c, counts.p, sizeof(c), cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaMemcpyAsync(first_two, g->row_off.p, sizeof(first_two),
                               cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    g->hub_end = (uint32_t)c[0];
    g->warp_end = (uint32_t)c[1];
    g->nonempty_end = (uint32_t)c[2];
    g->ndangling = (uint32_t)c[3];
    g->sort_end[0] = (uint32_t)c[4];
    g->sort_end[1] = (uint32_t)c[5];
    g->sort_end[2] = (uint32_t)c[6];
    g->sort_end[3] = (uint32_t)c[7];
    g->sort_end[4] = g->warp_end;
    g->sort_end[5] = (uint32_t)c[8];
    g->max_in_degree = max_in;
    (void)first_two;
    return g;
}

// Second half: the engine edge array, filled in edge ranges (graph_from_csr
// places each slice of the neighbour array as it lands), then rows sorted.
struct EdgeFill {
    prgpu_graph* g;
    DevBuf<uint32_t> src_of_old;
    uint32_t rb = 0, re = 0xFFFFFFFFu; // engine rows whose edges are kept (a shard's)
    // rows [r_begin, r_end) only (a shard): col holds their edges, from col_base
    EdgeFill(prgpu_graph* gr, cudaStream_t st, uint32_t r_begin = 0, uint32_t r_end = 0xFFFFFFFFu) : g(gr) {
        uint64_t n_alloc = g->e; // col entries: [col_base, col_base + n_alloc)
        g->col_base = 0;
        g->local_e = g->e;
        if (r_end != 0xFFFFFFFFu) {
            rb = r_begin;
            re = r_end;
            uint64_t lo = 0, hi = 0;
            PRGPU_CUDA(cudaMemcpyAsync(&lo, g->row_off.p + rb, 8, cudaMemcpyDeviceToHost, st));
            PRGPU_CUDA(cudaMemcpyAsync(&hi, g->row_off.p + re, 8, cudaMemcpyDeviceToHost, st));
            PRGPU_CUDA(cudaStreamSynchronize(st));
            // the kernels load colidx 128 bits at a time from global indices
            // that are multiples of 4: the shard's array starts at one
            g->col_base = lo & ~3ull;
            g->local_e = hi - lo;
            n_alloc = hi - g->col_base;
        }
        // engine edges (+16 zero pad for the kernels' 128-bit colidx loads)
        g->col.alloc(n_alloc + 16);
        PRGPU_CUDA(cudaMemsetAsync(g->col.p + n_alloc, 0, 16 * sizeof(uint32_t), st));
        if (n_alloc > g->local_e) // the (< 4) alignment slots ahead of a shard's first edge
            PRGPU_CUDA(cudaMemsetAsync(g->col.p, 0, (n_alloc - g->local_e) * sizeof(uint32_t), st));
        src_of_old.alloc(g->n);
        src_of_old_kernel<<<grid_for(g->n), kThreads, 0, st>>>(g->rowinfo.p, g->new_of_old.p, g->n,
                                                               src_of_old.p);
        PRGPU_LAUNCHED("src_of_old");
    }
    void place(const uint64_t* off, const uint32_t* nbr, uint64_t jb, uint64_t je, const uint32_t* deg, int* bad,
               cudaStream_t st) {
        if (je <= jb) return;
        const uint64_t blocks = (je - jb + kEdgeChunk - 1) / kEdgeChunk;
        place_edges<<<(unsigned)blocks, kThreads, 0, st>>>(off, nbr, g->n, jb, je, g->new_of_old.p,
                                                           g->row_off.p, src_of_old.p, g->col.p, deg, bad, rb,
                                                           re, g->col_base);
        PRGPU_LAUNCHED("place_edges");
    }
    // graph_from_csr: sort the caller's rows [v0, v1) (complete once their
    // slice is placed) while later slices are still in flight
    DevBuf<uint32_t> big;
    DevBuf<unsigned> nbig; // [0] appended, [1] sorted
    bool sliced = false;
    void sort_slice(uint32_t v0, uint32_t v1, cudaStream_t st) {
        if (!sliced) {
            sliced = true;
            big.alloc(std::max<uint32_t>(g->sort_end[0] - g->hub_end, 1));
            nbig.alloc(2);
            PRGPU_CUDA(cudaMemsetAsync(nbig.p, 0, 2 * sizeof(unsigned), st));
        }
        if (v1 <= v0) return;
        sort_rows_orig<<<(v1 - v0 + 7) / 8, 256, 0, st>>>(g->row_off.p, g->new_of_old.p, v0, v1, big.p, nbig.p,
                                                           g->col.p);
        PRGPU_LAUNCHED("sort_rows_orig");
        if (g->sort_end[0] > g->hub_end) {
            sort_rows_listed<<<2 * 148, 256, 0, st>>>(g->row_off.p, big.p, nbig.p, nbig.p + 1,
                                                      (int)bits_for(std::max(g->nsrc, 2u)), g->col.p);
            PRGPU_LAUNCHED("sort_rows_listed");
            mark_listed<<<1, 1, 0, st>>>(nbig.p, nbig.p + 1);
            PRGPU_LAUNCHED("mark_listed");
        }
    }
    void finish(cudaStream_t st) {
        src_of_old.reset();
        if (sliced) return; // sorted slice by slice
        const char* rs = std::getenv("PRGPU_ROW_SORT"); // =0: leave rows unsorted (tuning)
        if (rs && std::atoi(rs) == 0) return;
        // one class per power-of-two length band, each sorted at its own
        // width (a row is padded to the class's width, so bands halve the
        // padding of the wide ones)
        // a shard sorts its own rows only (col indexed from col_base)
        uint32_t* colv = g->col.p - g->col_base;
        const uint32_t lo_r = rb, hi_r = std::min<uint32_t>(re, g->n);
        const uint32_t h = std::max(g->hub_end, lo_r), m512 = std::min(g->sort_end[0], hi_r);
        if (m512 > h) {
            sort_rows_block<<<m512 - h, 256, 0, st>>>(g->row_off.p, h, (int)bits_for(std::max(g->nsrc, 2u)),
                                                      colv);
            PRGPU_LAUNCHED("sort_rows_block");
        }
        auto warp_sort = [&](auto items, int c) {
            constexpr int I = decltype(items)::value;
            const uint32_t r0 = std::max(g->sort_end[c], lo_r), r1 = std::min(g->sort_end[c + 1], hi_r);
            if (r1 <= r0) return;
            sort_rows_warp<I><<<(r1 - r0 + 7) / 8, 256, 0, st>>>(g->row_off.p, r0, r1, colv);
            PRGPU_LAUNCHED("sort_rows_warp");
        };
        warp_sort(std::integral_constant<int, 16>{}, 0); // 257..512
        warp_sort(std::integral_constant<int, 8>{}, 1);  // 129..256
        warp_sort(std::integral_constant<int, 4>{}, 2);  // 65..128
        warp_sort(std::integral_constant<int, 2>{}, 3);  // 33..64
        warp_sort(std::integral_constant<int, 1>{}, 4);  // 9..32
    }
};

// Sorted unique original-id keys (target << lg | source) -> engine graph.
// Consumes `keys`.
std::unique_ptr<prgpu_graph> assemble(DevBuf<uint64_t>&& keys_in, uint64_t u, uint32_t n,
                                      uint32_t lg, int device, cudaStream_t st) {
    DevBuf<uint64_t> keys(std::move(keys_in));
    DevBuf<uint32_t> in_deg(n), out_deg(n);
    PRGPU_CUDA(cudaMemsetAsync(in_deg.p, 0, n * sizeof(uint32_t), st));
    PRGPU_CUDA(cudaMemsetAsync(out_deg.p, 0, n * sizeof(uint32_t), st));
    if (u) {
        count_degrees<<<grid_for(u), kThreads, 0, st>>>(keys.p, u, lg, in_deg.p, out_deg.p);
        PRGPU_LAUNCHED("count_degrees");
    }
    DevBuf<uint64_t> off((size_t)n + 1);
    gather_deg_u64<<<grid_for((uint64_t)n + 1), kThreads, 0, st>>>(in_deg.p, nullptr, off.p, n);
    PRGPU_LAUNCHED("gather_deg_u64");
    exclusive_scan_u64(off.p, (uint64_t)n + 1, st);
    DevBuf<uint32_t> nbr(std::max<uint64_t>(u, 1));
    if (u) {
        keys_low<<<grid_for(u), kThreads, 0, st>>>(keys.p, u, lg, nbr.p);
        PRGPU_LAUNCHED("keys_low");
    }
    keys.reset();
    in_deg.reset();
    auto g = assemble_vertices(n, off.p, u, out_deg.p, lg, device, st);
    EdgeFill fill(g.get(), st);
    fill.place(off.p, nbr.p, 0, u, nullptr, nullptr, st);
    fill.finish(st);
    return g;
}

} // namespace

// vertex_count 0: no device arrays; every solve entry point rejects it
std::unique_ptr<prgpu_graph> empty_graph(int device) {
    auto g = std::make_unique<prgpu_graph>();
    g->device = device;
    g->lg = 1;
    return g;
}

std::unique_ptr<prgpu_graph> graph_build_device(uint32_t n, const uint32_t* d_pairs, uint64_t m,
                                                int device, cudaStream_t st) {
    if (n == 0) { // graph.hpp:204-234 returns an empty graph; pagerank() then throws (pagerank.hpp:74)
        if (m) fail(PRGPU_EINVAL, "build_csr: edge endpoint >= vertex_count");
        return empty_graph(device);
    }
    const uint32_t lg = bits_for(n);
    DevBuf<uint64_t> keys(std::max<uint64_t>(m, 1));
    if (m) {
        DevBuf<int> bad(1);
        PRGPU_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        pairs_to_keys<<<grid_for(m), kThreads, 0, st>>>(d_pairs, m, n, lg, keys.p, bad.p);
        PRGPU_LAUNCHED("pairs_to_keys");
        if (read_flag(bad, st)) fail(PRGPU_EINVAL, "build_csr: edge endpoint >= vertex_count");
        DevBuf<uint64_t> alt(m);
        sort_keys(keys, alt, m, 2 * (int)lg, st);
        m = unique_keys(keys, alt, m, st);
    }
    return assemble(std::move(keys), m, n, lg, device, st);
}

std::unique_ptr<prgpu_graph> graph_build_host(uint32_t n, const uint32_t* pairs, uint64_t m,
                                              int device, cudaStream_t st) {
    DevBuf<uint32_t> d(std::max<uint64_t>(2 * m, 2));
    if (m)
        PRGPU_CUDA(cudaMemcpyAsync(d.p, pairs, 2 * m * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    return graph_build_device(n, d.p, m, device, st);
}

std::unique_ptr<prgpu_graph> graph_from_csr(uint32_t n, const uint64_t* off, const uint32_t* nbr,
                                            const uint32_t* out_degree, int device,
                                            cudaStream_t st) {
    if (off[0] != 0) fail(PRGPU_EINVAL, "graph_from_csr: in_offsets[0] != 0");
    if (n == 0) return empty_graph(device); // pagerank() throws on it (pagerank.hpp:74)
    const uint64_t e = off[n];
    const uint32_t lg = bits_for(n);
    PhaseLog ph("from_csr", st);
    DevBuf<uint64_t> d_off((size_t)n + 1);
    DevBuf<uint32_t> d_nbr(std::max<uint64_t>(e, 1)), d_deg(n);
    // offsets and degrees first; the neighbour array (the bulk) follows on a
    // side stream in slices, while `st` runs the vertex half of the build and
    // then places each slice as it lands
    PRGPU_CUDA(cudaMemcpyAsync(d_off.p, off, ((size_t)n + 1) * 8, cudaMemcpyHostToDevice, st));
    PRGPU_CUDA(cudaMemcpyAsync(d_deg.p, out_degree, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    Stream side;
    Event meta;
    PRGPU_CUDA(cudaEventRecord(meta, st)); // also orders d_nbr's allocation
    PRGPU_CUDA(cudaStreamWaitEvent(side, meta, 0));
    const uint64_t slice = std::max<uint64_t>(8ull << 20, (e + 7) / 8);
    std::vector<std::unique_ptr<Event>> landed;
    for (uint64_t j = 0; j < e; j += slice) {
        const uint64_t k = std::min(slice, e - j);
        PRGPU_CUDA(cudaMemcpyAsync(d_nbr.p + j, nbr + j, k * 4, cudaMemcpyHostToDevice, side));
        landed.emplace_back(std::make_unique<Event>());
        PRGPU_CUDA(cudaEventRecord(*landed.back(), side));
    }
    DevBuf<int> bad(1);
    PRGPU_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
    check_offsets<<<grid_for(n), kThreads, 0, st>>>(d_off.p, n, e, bad.p);
    PRGPU_LAUNCHED("check_offsets");
    if (read_flag(bad, st)) {
        cudaStreamSynchronize(side);
        fail(PRGPU_EINVAL, "graph_from_csr: offsets not monotone");
    }
    ph.mark("offsets h2d + check");
    std::unique_ptr<prgpu_graph> g;
    try {
        g = assemble_vertices(n, d_off.p, e, d_deg.p, lg, device, st);
        ph.mark("vertex half");
        EdgeFill fill(g.get(), st);
        const char* rs = std::getenv("PRGPU_ROW_SORT"); // =0: leave rows unsorted (tuning)
        const bool sort_rows = !(rs && std::atoi(rs) == 0);
        uint32_t v_done = 0; // caller rows [0, v_done) complete and sorted
        for (size_t c = 0; c < landed.size(); ++c) {
            PRGPU_CUDA(cudaStreamWaitEvent(st, *landed[c], 0));
            const uint64_t j = c * slice, je = std::min(e, j + slice);
            fill.place(d_off.p, d_nbr.p, j, je, d_deg.p, bad.p, st);
            if (!sort_rows) continue;
            // rows whose last edge is before je (the last slice: every row)
            const uint32_t v_end = c + 1 == landed.size()
                                       ? n
                                       : (uint32_t)(std::upper_bound(off + 1, off + n + 1, je) - (off + 1));
            fill.sort_slice(v_done, v_end, st);
            v_done = v_end;
        }
        const int why = read_flag(bad, st);
        if (why == 1) fail(PRGPU_EINVAL, "graph_from_csr: in-neighbour >= vertex_count");
        if (why) fail(PRGPU_EINVAL, "graph_from_csr: an in-neighbour has out_degree 0 (pagerank.hpp:91 would divide by zero)");
        ph.mark("edges placed");
        fill.finish(st);
        ph.mark("rows sorted");
    } catch (...) {
        cudaStreamSynchronize(side); // no copy may still target d_nbr
        throw;
    }
    return g;
}

// ---- hot/cold source split (SourceSplit) ----------------------------------------
// Per row, its in-edges with source id < hot, counted (split_count) and then
// placed (split_place) in their order into the hot CSR, the rest into the
// cold one.  Rows with more than kHubMinDegree in-edges get a CTA (256-edge
// windows, a CTA-wide prefix of the warps' hot counts keeps the order), the
// others a warp (32-edge windows, ballot prefix).
template <bool PLACE>
__global__ void split_rows_warp(const uint64_t* __restrict__ off, const uint32_t* __restrict__ col, uint32_t r0,
                                uint32_t r1, uint32_t hot, uint64_t* __restrict__ cnt_hot,
                                const uint64_t* __restrict__ off_hot, const uint64_t* __restrict__ off_cold,
                                uint32_t* __restrict__ col_hot, uint32_t* __restrict__ col_cold) {
    const uint32_t lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t r = r0 + ((blockIdx.x * blockDim.x + threadIdx.x) >> 5); r < r1;
         r += (gridDim.x * blockDim.x) >> 5) {
        const uint64_t lo = off[r], hi = off[r + 1];
        uint64_t h = PLACE ? off_hot[r] : 0, c = PLACE ? off_cold[r] : 0;
        for (uint64_t j = lo; j < hi; j += 32) {
            const bool in = j + lane < hi;
            const uint32_t src = in ? col[j + lane] : 0u;
            const bool is_hot = in && src < hot;
            const unsigned bh = __ballot_sync(0xffffffffu, is_hot), bc = __ballot_sync(0xffffffffu, in && !is_hot);
            if (PLACE) {
                if (is_hot) col_hot[h + __popc(bh & lt)] = src;
                else if (in) col_cold[c + __popc(bc & lt)] = src;
                c += __popc(bc);
            }
            h += __popc(bh);
        }
        if (!PLACE && lane == 0) cnt_hot[r] = h;
    }
}

template <bool PLACE>
__global__ void __launch_bounds__(256) split_rows_block(const uint64_t* __restrict__ off,
                                                        const uint32_t* __restrict__ col, uint32_t hot,
                                                        uint64_t* __restrict__ cnt_hot,
                                                        const uint64_t* __restrict__ off_hot,
                                                        const uint64_t* __restrict__ off_cold,
                                                        uint32_t* __restrict__ col_hot,
                                                        uint32_t* __restrict__ col_cold) {
    __shared__ unsigned s_h[8], s_c[8];
    const uint32_t r = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = (1u << lane) - 1u;
    const uint64_t lo = off[r], hi = off[r + 1];
    uint64_t h = PLACE ? off_hot[r] : 0, c = PLACE ? off_cold[r] : 0;
    for (uint64_t j0 = lo; j0 < hi; j0 += 256) {
        const uint64_t j = j0 + threadIdx.x;
        const bool in = j < hi;
        const uint32_t src = in ? col[j] : 0u;
        const bool is_hot = in && src < hot;
        const unsigned bh = __ballot_sync(0xffffffffu, is_hot), bc = __ballot_sync(0xffffffffu, in && !is_hot);
        if (lane == 0) {
            s_h[warp] = __popc(bh);
            s_c[warp] = __popc(bc);
        }
        __syncthreads();
        uint64_t ph = 0, pc = 0, th = 0, tc = 0;
        for (uint32_t w = 0; w < 8; ++w) {
            if (w < warp) {
                ph += s_h[w];
                pc += s_c[w];
            }
            th += s_h[w];
            tc += s_c[w];
        }
        if (PLACE) {
            if (is_hot) col_hot[h + ph + __popc(bh & lt)] = src;
            else if (in) col_cold[c + pc + __popc(bc & lt)] = src;
        }
        h += th;
        c += tc;
        __syncthreads();
    }
    if (!PLACE && threadIdx.x == 0) cnt_hot[r] = h;
}

__global__ void split_cold_off(const uint64_t* __restrict__ off, const uint64_t* __restrict__ off_hot, uint32_t n,
                               uint64_t* __restrict__ off_cold) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= n; v += (uint64_t)gridDim.x * blockDim.x)
        off_cold[v] = off[v] - off_hot[v];
}

const SourceSplit& graph_source_split(prgpu_graph* g, uint32_t hot, cudaStream_t st) {
    std::lock_guard<std::mutex> lock(g->split_mu);
    auto it = g->splits.find(hot);
    if (it != g->splits.end()) return *it->second;
    AllocScope scope(st); // the split's buffers come from the pool like the graph's own
    auto sp = std::make_unique<SourceSplit>();
    sp->hot = hot;
    const uint32_t n = g->n, hub = g->hub_end, rows = g->nonempty_end;
    const unsigned wgrid = rows > hub ? grid_for((uint64_t)(rows - hub) * 32) : 0;
    sp->off_hot.alloc((size_t)n + 1);
    PRGPU_CUDA(cudaMemsetAsync(sp->off_hot.p, 0, ((size_t)n + 1) * 8, st));
    if (hub) {
        split_rows_block<false><<<hub, 256, 0, st>>>(g->row_off.p, g->col.p, hot, sp->off_hot.p, nullptr, nullptr,
                                                     nullptr, nullptr);
        PRGPU_LAUNCHED("split_rows_block");
    }
    if (wgrid) {
        split_rows_warp<false><<<wgrid, kThreads, 0, st>>>(g->row_off.p, g->col.p, hub, rows, hot, sp->off_hot.p,
                                                           nullptr, nullptr, nullptr, nullptr);
        PRGPU_LAUNCHED("split_rows_warp");
    }
    exclusive_scan_u64(sp->off_hot.p, (uint64_t)n + 1, st); // hot counts -> hot row offsets
    PRGPU_CUDA(cudaMemcpyAsync(&sp->e_hot, sp->off_hot.p + n, 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    sp->e_cold = g->e - sp->e_hot;
    sp->off_cold.alloc((size_t)n + 1);
    split_cold_off<<<grid_for((uint64_t)n + 1), kThreads, 0, st>>>(g->row_off.p, sp->off_hot.p, n, sp->off_cold.p);
    PRGPU_LAUNCHED("split_cold_off");
    sp->col_hot.alloc(sp->e_hot + 16);
    sp->col_cold.alloc(sp->e_cold + 16);
    PRGPU_CUDA(cudaMemsetAsync(sp->col_hot.p + sp->e_hot, 0, 16 * 4, st));
    PRGPU_CUDA(cudaMemsetAsync(sp->col_cold.p + sp->e_cold, 0, 16 * 4, st));
    if (hub) {
        split_rows_block<true><<<hub, 256, 0, st>>>(g->row_off.p, g->col.p, hot, nullptr, sp->off_hot.p,
                                                    sp->off_cold.p, sp->col_hot.p, sp->col_cold.p);
        PRGPU_LAUNCHED("split_rows_block");
    }
    if (wgrid) {
        split_rows_warp<true><<<wgrid, kThreads, 0, st>>>(g->row_off.p, g->col.p, hub, rows, hot, nullptr,
                                                          sp->off_hot.p, sp->off_cold.p, sp->col_hot.p,
                                                          sp->col_cold.p);
        PRGPU_LAUNCHED("split_rows_warp");
    }
    PRGPU_CUDA(cudaStreamSynchronize(st));
    return *(g->splits[hot] = std::move(sp));
}

// ---- segment plan (SegPlan, common.cuh) ------------------------------------------
constexpr uint32_t kSegSlab = 32768; // edges per CTA of the counting / key passes

__device__ __forceinline__ uint32_t seg_of(uint32_t src, uint32_t seg_src, uint32_t S) {
    const uint32_t q = src / seg_src;
    return q < S ? q : S - 1;
}

// One CTA per slab of col[0, e_seg): for every row crossing the slab, the
// number of its edges per segment (COUNT: added to cnt[seg][row], integer
// atomics) or, once the counts are complete, every edge's sort key
// class * S + seg (class 1: the edge's piece has <= win edges).
template <bool KEYS>
__global__ void __launch_bounds__(256) seg_slab_kernel(const uint64_t* __restrict__ row_off,
                                                       const uint32_t* __restrict__ col, uint32_t n_rows,
                                                       uint64_t e_seg, uint32_t seg_src, uint32_t S, uint32_t win,
                                                       uint32_t* __restrict__ cnt, uint8_t* __restrict__ keys,
                                                       const uint64_t* __restrict__ merged) {
    __shared__ uint32_t s_h[64];
    __shared__ uint32_t s_row;
    const uint64_t lo = (uint64_t)blockIdx.x * kSegSlab, hi = min(lo + kSegSlab, e_seg);
    if (threadIdx.x == 0) { // the row holding edge lo: last r with row_off[r] <= lo
        uint32_t a = 0, b = n_rows;
        while (b - a > 1) {
            const uint32_t m = a + (b - a) / 2;
            if (row_off[m] <= lo) a = m;
            else b = m;
        }
        s_row = a;
    }
    __syncthreads();
    for (uint32_t r = s_row; r < n_rows; ++r) {
        const uint64_t r0 = row_off[r], r1 = row_off[r + 1];
        if (r0 >= hi) break;
        const uint64_t a = max(r0, lo), b = min(r1, hi);
        const uint64_t mm = KEYS ? merged[r] : 0ull; // segments whose (small) piece went to the cold piece
        if (threadIdx.x < 64)
            s_h[threadIdx.x] = (KEYS && threadIdx.x < S && cnt[(size_t)threadIdx.x * n_rows + r] <= win) ? S : 0u;
        __syncthreads();
        for (uint64_t j = a + threadIdx.x; j < b; j += 256) {
            uint32_t sg = seg_of(col[j], seg_src, S);
            if (KEYS && ((mm >> sg) & 1ull)) sg = S - 1;
            if (KEYS) keys[j] = (uint8_t)(sg + s_h[sg]);
            else atomicAdd(&s_h[sg], 1u);
        }
        __syncthreads();
        if (!KEYS && threadIdx.x < S && s_h[threadIdx.x])
            atomicAdd(&cnt[(size_t)threadIdx.x * n_rows + r], s_h[threadIdx.x]);
        __syncthreads();
    }
}

// A hot-segment piece of fewer than pmin edges costs more (its offsets, its
// partial's round trip) than the misses it saves: its edges join the row's
// piece in the last (cold) segment; merged[row] keeps the segments folded.
__global__ void seg_merge_small(uint32_t* __restrict__ cnt, uint32_t n_rows, uint32_t S, uint32_t pmin,
                                uint64_t* __restrict__ merged) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        uint64_t m = 0;
        uint32_t cold = 0;
        for (uint32_t sg = 0; sg + 1 < S; ++sg) {
            const uint32_t c = cnt[(size_t)sg * n_rows + r];
            if (c && c < pmin) {
                cold += c;
                cnt[(size_t)sg * n_rows + r] = 0;
                m |= 1ull << sg;
            }
        }
        if (cold) cnt[(size_t)(S - 1) * n_rows + r] += cold;
        merged[r] = m;
    }
}

// flattened pieces f = (class * S + seg) * n_rows + row, f in [0, 2F]: length
// and presence (element 2F is the sentinel that receives the totals)
__global__ void seg_piece_len(const uint32_t* __restrict__ cnt, uint64_t F, uint32_t win,
                              uint64_t* __restrict__ len, uint64_t* __restrict__ flag) {
    for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f <= 2 * F;
         f += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        if (f < 2 * F) {
            c = cnt[f < F ? f : f - F];
            const bool small = c <= win;
            if (small != (f >= F)) c = 0;
        }
        len[f] = c;
        flag[f] = c != 0;
    }
}

__global__ void seg_piece_fill(const uint64_t* __restrict__ start, const uint64_t* __restrict__ pidx,
                               const uint32_t* __restrict__ cnt, uint64_t F, uint32_t n_rows, uint32_t S,
                               uint32_t win, uint64_t* __restrict__ off, uint32_t* __restrict__ slot) {
    for (uint64_t f = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; f <= 2 * F;
         f += (uint64_t)gridDim.x * blockDim.x) {
        if (f == 2 * F) {
            off[pidx[f]] = start[f];
            continue;
        }
        const uint64_t g = f < F ? f : f - F;
        const uint32_t c = cnt[g];
        if (c == 0 || ((c <= win) != (f >= F))) continue;
        const uint64_t p = pidx[f];
        off[p] = start[f];
        slot[p] = (uint32_t)(g % n_rows) * S + (uint32_t)(g / n_rows);
    }
}

__global__ void count_rows_ge(const uint64_t* __restrict__ row_off, uint32_t n, uint32_t T,
                              unsigned int* __restrict__ out) {
    unsigned int c = 0;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        c += (row_off[r + 1] - row_off[r]) >= T;
    if (c) atomicAdd(out, c);
}

const SegPlan* graph_seg_plan(prgpu_graph* g, uint32_t seg_src, uint32_t S, uint32_t T, uint32_t win,
                              uint32_t pmin, cudaStream_t st) {
    if (S < 1 || S > 64 || seg_src == 0 || T < 2) fail(PRGPU_EINVAL, "segment plan: bad parameters");
    if (g->shard_n > 1 || g->locality) return nullptr; // rows not in degree order / col not whole
    std::lock_guard<std::mutex> lock(g->split_mu);
    const std::array<uint32_t, 5> key{seg_src, S, T, win, pmin};
    auto it = g->seg_plans.find(key);
    if (it != g->seg_plans.end()) return it->second->n_rows ? it->second.get() : nullptr;
    AllocScope scope(st);
    PhaseLog ph("segplan", st);
    auto sp = std::make_unique<SegPlan>();
    sp->seg_src = seg_src;
    sp->S = S;
    sp->T = T;
    sp->win = win;
    sp->pmin = pmin;
    // rows are in in-degree order: the rows with >= T in-edges are a prefix
    {
        DevBuf<unsigned int> c(1);
        PRGPU_CUDA(cudaMemsetAsync(c.p, 0, 4, st));
        count_rows_ge<<<grid_for(g->n), kThreads, 0, st>>>(g->row_off.p, g->n, T, c.p);
        PRGPU_LAUNCHED("count_rows_ge");
        PRGPU_CUDA(cudaMemcpyAsync(&sp->n_rows, c.p, 4, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
    // (slots row * S + seg are 32-bit: only a far-too-small T could overflow them)
    if (sp->n_rows == 0 || (uint64_t)sp->n_rows * S >= (1ull << 32)) {
        sp->n_rows = 0;
        g->seg_plans[key] = std::move(sp);
        return nullptr;
    }
    const uint32_t nr = sp->n_rows;
    PRGPU_CUDA(cudaMemcpyAsync(&sp->e_seg, g->row_off.p + nr, 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    const uint64_t es = sp->e_seg, F = (uint64_t)S * nr;
    const unsigned slabs = (unsigned)((es + kSegSlab - 1) / kSegSlab);
    DevBuf<uint32_t> cnt(F);
    PRGPU_CUDA(cudaMemsetAsync(cnt.p, 0, F * 4, st));
    seg_slab_kernel<false><<<slabs, 256, 0, st>>>(g->row_off.p, g->col.p, nr, es, seg_src, S, win, cnt.p, nullptr,
                                                  nullptr);
    PRGPU_LAUNCHED("seg_slab_kernel<count>");
    DevBuf<uint64_t> merged(nr);
    seg_merge_small<<<grid_for(nr), kThreads, 0, st>>>(cnt.p, nr, S, pmin, merged.p);
    PRGPU_LAUNCHED("seg_merge_small");
    ph.mark("count");
    {
        DevBuf<uint8_t> kin(es), kout(es);
        seg_slab_kernel<true><<<slabs, 256, 0, st>>>(g->row_off.p, g->col.p, nr, es, seg_src, S, win, cnt.p, kin.p,
                                                     merged.p);
        PRGPU_LAUNCHED("seg_slab_kernel<keys>");
        sp->col.alloc(es + 16);
        PRGPU_CUDA(cudaMemsetAsync(sp->col.p + es, 0, 16 * 4, st));
        // one stable radix pass over the (class, segment) key keeps rows, and
        // each row's edge order, inside every (class, segment) group
        const int bits = (int)bits_for(2ull * S);
        size_t tmp = 0;
        PRGPU_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, kin.p, kout.p, g->col.p, sp->col.p, (int64_t)es, 0,
                                                   bits, st));
        DevBuf<char> t(std::max<size_t>(tmp, 1));
        PRGPU_CUDA(cub::DeviceRadixSort::SortPairs(t.p, tmp, kin.p, kout.p, g->col.p, sp->col.p, (int64_t)es, 0,
                                                   bits, st));
        g_launches.fetch_add(1);
        ph.mark("keys + sort");
    }
    {
        DevBuf<uint64_t> len(2 * F + 1), flag(2 * F + 1);
        seg_piece_len<<<grid_for(2 * F + 1), kThreads, 0, st>>>(cnt.p, F, win, len.p, flag.p);
        PRGPU_LAUNCHED("seg_piece_len");
        exclusive_scan_u64(len.p, 2 * F + 1, st);
        exclusive_scan_u64(flag.p, 2 * F + 1, st);
        uint64_t np = 0, nw = 0;
        PRGPU_CUDA(cudaMemcpyAsync(&np, flag.p + 2 * F, 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaMemcpyAsync(&nw, flag.p + F, 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaMemcpyAsync(&sp->e_wide, len.p + F, 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        sp->n_wp = (uint32_t)nw;
        sp->n_sp = (uint32_t)(np - nw);
        sp->off.alloc(np + 1);
        sp->slot.alloc(std::max<uint64_t>(np, 1));
        seg_piece_fill<<<grid_for(2 * F + 1), kThreads, 0, st>>>(len.p, flag.p, cnt.p, F, nr, S, win, sp->off.p,
                                                                  sp->slot.p);
        PRGPU_LAUNCHED("seg_piece_fill");
        PRGPU_CUDA(cudaStreamSynchronize(st));
        ph.mark("pieces");
    }
    if (std::getenv("PRGPU_TIMING_LOG"))
        std::fprintf(stderr, "[segplan] rows %u edges %llu (%.1f%% of E) S %u seg_src %u wide pieces %u (%llu edges) small %u\n",
                     nr, (unsigned long long)es, 100.0 * (double)es / (double)std::max<uint64_t>(g->e, 1), S, seg_src,
                     sp->n_wp, (unsigned long long)sp->e_wide, sp->n_sp);
    SegPlan* out = sp.get();
    g->seg_plans[key] = std::move(sp);
    return out;
}

std::unique_ptr<prgpu_graph> graph_generate_rmat(uint32_t scale, uint32_t ef, double a, double b,
                                                 double c, uint64_t seed, int device,
                                                 cudaStream_t st) {
    if (scale < 1 || scale > 30) fail(PRGPU_EINVAL, "rmat: scale must be in [1, 30]");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
        fail(PRGPU_EINVAL, "rmat: probabilities must be >= 0 with a+b+c <= 1");
    const uint32_t n = 1u << scale;
    const uint64_t m = (uint64_t)ef << scale;
    PermKeys pk;
    const uint64_t pkey = stream_key(seed, 2);
    for (int r = 0; r < 3; ++r) pk.k[r] = mix64_host(pkey + (uint64_t)r);
    pk.mask = (1ull << scale) - 1;
    pk.hs = (scale + 1) / 2;
    DevBuf<uint64_t> keys(std::max<uint64_t>(m, 1));
    if (m) {
        rmat_keys<<<grid_for(m), kThreads, 0, st>>>(m, scale, stream_key(seed, 1), prob_threshold(a),
                                                    prob_threshold(a + b), prob_threshold(a + b + c),
                                                    pk, keys.p);
        PRGPU_LAUNCHED("rmat_keys");
    }
    uint64_t u = 0;
    if (m) {
        DevBuf<uint64_t> alt(m);
        sort_keys(keys, alt, m, 2 * (int)scale, st);
        u = unique_keys(keys, alt, m, st);
        uint64_t last = 0;
        PRGPU_CUDA(cudaMemcpyAsync(&last, keys.p + (u - 1), 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        if (last == kSentinel) --u; // self-loop slots
    }
    return assemble(std::move(keys), u, n, scale, device, st);
}

// One rank's shard of the RMAT graph (SURVEY 8e set-up), never holding the
// whole edge list: every rank generates all edges, in slabs of target ids —
//   pass 1: per slab, the slab's keys sorted + deduplicated, counted into the
//           global in- and out-degrees (exact: a (source, target) duplicate
//           lies in one slab), so every rank computes the same vertex half
//           (relabel, row offsets, source ids) as the whole-graph build;
//   shard rows: contiguous engine-row ranges of equal cost (in-degree + 2
//           per row, 1 per row without in-edges; cuts among those rows on
//           multiples of 256 so no empty-row task spans two ranks);
//   pass 2: per slab again, the slab's edges (= its range of the original
//           CSR) placed into col if their engine row is this rank's; rows
//           then sorted by source id as in the whole build.
// Slabs are sized so a slab's keys (+ the sort buffer) stay under ~16 GB.
std::unique_ptr<prgpu_graph> graph_generate_rmat_shard(uint32_t scale, uint32_t ef, double a, double b, double c,
                                                       uint64_t seed, int rank, int nranks, int device,
                                                       cudaStream_t st) {
    if (scale < 1 || scale > 30) fail(PRGPU_EINVAL, "rmat: scale must be in [1, 30]");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
        fail(PRGPU_EINVAL, "rmat: probabilities must be >= 0 with a+b+c <= 1");
    if (nranks < 1 || nranks > 64 || rank < 0 || rank >= nranks) fail(PRGPU_EINVAL, "shard: bad rank / nranks");
    const uint32_t n = 1u << scale;
    const uint64_t m = (uint64_t)ef << scale;
    PermKeys pk;
    const uint64_t pkey = stream_key(seed, 2);
    for (int r = 0; r < 3; ++r) pk.k[r] = mix64_host(pkey + (uint64_t)r);
    pk.mask = (1ull << scale) - 1;
    pk.hs = (scale + 1) / 2;
    const uint64_t kd = stream_key(seed, 1), ta = prob_threshold(a), tab = prob_threshold(a + b),
                   tabc = prob_threshold(a + b + c);
    const char* sb = std::getenv("PRGPU_SLAB_KEYS"); // keys per slab (tests: small slabs)
    const uint64_t slab_keys = sb ? std::max<uint64_t>(1024, (uint64_t)std::atoll(sb)) : (1ull << 30);
    const uint32_t S = (uint32_t)std::min<uint64_t>(n, std::max<uint64_t>(1, (m + slab_keys - 1) / slab_keys));
    auto slab_lo = [&](uint32_t s) { return (uint32_t)(((uint64_t)n * s) / S); };
    DevBuf<unsigned long long> cnt(1);
    // one slab's sorted unique keys (target << scale | source) into `keys`
    auto slab = [&](uint32_t s, DevBuf<uint64_t>& keys) -> uint64_t {
        uint64_t cap = (m / S) + (m / S) / 4 + 4096;
        for (;;) {
            keys.alloc(cap);
            PRGPU_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
            rmat_keys_slab<<<grid_for(m), 256, 0, st>>>(m, scale, kd, ta, tab, tabc, pk, slab_lo(s), slab_lo(s + 1),
                                                        keys.p, cap, cnt.p);
            PRGPU_LAUNCHED("rmat_keys_slab");
            unsigned long long got = 0;
            PRGPU_CUDA(cudaMemcpyAsync(&got, cnt.p, sizeof(got), cudaMemcpyDeviceToHost, st));
            PRGPU_CUDA(cudaStreamSynchronize(st));
            if (got <= cap) {
                if (!got) return 0;
                DevBuf<uint64_t> alt(got);
                sort_keys(keys, alt, got, 2 * (int)scale, st);
                return unique_keys(keys, alt, got, st);
            }
            cap = got + 4096; // a heavier slab than expected: once more at its size
        }
    };
    // pass 1: exact degrees
    DevBuf<uint32_t> in_deg(n), out_deg(n);
    PRGPU_CUDA(cudaMemsetAsync(in_deg.p, 0, (size_t)n * 4, st));
    PRGPU_CUDA(cudaMemsetAsync(out_deg.p, 0, (size_t)n * 4, st));
    uint64_t e = 0;
    for (uint32_t s = 0; s < S; ++s) {
        DevBuf<uint64_t> keys;
        const uint64_t u = slab(s, keys);
        if (u) {
            count_degrees<<<grid_for(u), kThreads, 0, st>>>(keys.p, u, scale, in_deg.p, out_deg.p);
            PRGPU_LAUNCHED("count_degrees");
        }
        e += u;
    }
    DevBuf<uint64_t> off((size_t)n + 1);
    gather_deg_u64<<<grid_for((uint64_t)n + 1), kThreads, 0, st>>>(in_deg.p, nullptr, off.p, n);
    PRGPU_LAUNCHED("gather_deg_u64");
    exclusive_scan_u64(off.p, (uint64_t)n + 1, st);
    in_deg.reset();
    auto g = assemble_vertices(n, off.p, e, out_deg.p, scale, device, st);
    // shard rows
    {
        DevBuf<uint64_t> cost((size_t)n + 1);
        PRGPU_CUDA(cudaMemsetAsync(cost.p + n, 0, 8, st));
        shard_costs<<<grid_for(n), kThreads, 0, st>>>(g->row_off.p, n, g->nonempty_end, cost.p);
        PRGPU_LAUNCHED("shard_costs");
        exclusive_scan_u64(cost.p, (uint64_t)n + 1, st);
        DevBuf<uint32_t> bnd((size_t)nranks + 1);
        shard_search<<<1, 128, 0, st>>>(cost.p, n, (uint32_t)nranks, bnd.p);
        PRGPU_LAUNCHED("shard_search");
        g->shard_rows.resize((size_t)nranks + 1);
        PRGPU_CUDA(cudaMemcpyAsync(g->shard_rows.data(), bnd.p, ((size_t)nranks + 1) * 4, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
        const uint32_t eb = g->nonempty_end;
        for (int r = 1; r < nranks; ++r) {
            uint32_t x = g->shard_rows[r];
            if (x > eb) x = eb + ((x - eb) & ~255u); // empty-row tasks never straddle two ranks
            g->shard_rows[r] = std::max(x, g->shard_rows[r - 1]);
        }
    }
    g->shard_rank = rank;
    g->shard_n = nranks;
    // pass 2: this rank's edges
    EdgeFill fill(g.get(), st, g->shard_rows[rank], g->shard_rows[rank + 1]);
    std::vector<uint64_t> offh((size_t)S + 1);
    for (uint32_t s = 0; s <= S; ++s)
        PRGPU_CUDA(cudaMemcpyAsync(&offh[s], off.p + slab_lo(s), 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    for (uint32_t s = 0; s < S; ++s) {
        if (offh[s + 1] == offh[s]) continue;
        DevBuf<uint64_t> keys;
        const uint64_t u = slab(s, keys);
        if (u != offh[s + 1] - offh[s]) fail(PRGPU_ECUDA, "shard: slab edge count changed between passes");
        DevBuf<uint32_t> nbr(u);
        keys_low<<<grid_for(u), kThreads, 0, st>>>(keys.p, u, scale, nbr.p);
        PRGPU_LAUNCHED("keys_low");
        keys.reset();
        // the slab is the original CSR's edges [offh[s], offh[s+1]): nbr indexed by global edge index
        fill.place(off.p, nbr.p - offh[s], offh[s], offh[s + 1], nullptr, nullptr, st);
        PRGPU_CUDA(cudaStreamSynchronize(st)); // nbr is freed next
    }
    fill.finish(st);
    PRGPU_CUDA(cudaStreamSynchronize(st));
    return g;
}

std::unique_ptr<prgpu_graph> graph_generate_grid(uint32_t side, double p, double lr, uint64_t seed,
                                                 int device, cudaStream_t st) {
    if (side < 2 || (uint64_t)side * side > 0xFFFFFFFFull)
        fail(PRGPU_EINVAL, "grid: side must be >= 2 and side^2 < 2^32");
    const uint64_t n = (uint64_t)side * side;
    const uint32_t lg = bits_for(n);
    const uint64_t uh = (uint64_t)side * (side - 1);
    const uint64_t L = (uint64_t)(lr * (double)n);
    const uint64_t m = 4 * uh + L;
    DevBuf<uint64_t> keys(m);
    grid_keys<<<grid_for(2 * uh + L), kThreads, 0, st>>>(side, uh, prob_threshold(p),
                                                         stream_key(seed, 3), L, stream_key(seed, 4),
                                                         n, lg, keys.p);
    PRGPU_LAUNCHED("grid_keys");
    DevBuf<uint64_t> alt(m);
    sort_keys(keys, alt, m, 2 * (int)lg, st);
    uint64_t u = unique_keys(keys, alt, m, st);
    alt.reset();
    uint64_t last = 0;
    PRGPU_CUDA(cudaMemcpyAsync(&last, keys.p + (u - 1), 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    if (last == kSentinel) --u;
    return assemble(std::move(keys), u, (uint32_t)n, lg, device, st);
}

void graph_download(const prgpu_graph* g, uint64_t* h_off, uint32_t* h_nbr, uint32_t* h_deg,
                    uint32_t* h_dang, cudaStream_t st) {
    if (g->shard_n > 1 && h_nbr) fail(PRGPU_EINVAL, "graph_download: a shard graph holds one rank's edges only");
    const uint32_t n = g->n;
    const uint64_t e = g->e;
    if (n == 0) { // the empty graph: in_offsets = {0}
        if (h_off) h_off[0] = 0;
        return;
    }
    if (h_deg || h_dang) {
        DevBuf<uint32_t> deg(n);
        gather_u32<<<grid_for(n), kThreads, 0, st>>>(g->deg.p, g->new_of_old.p, deg.p, n);
        PRGPU_LAUNCHED("gather_u32");
        if (h_deg)
            PRGPU_CUDA(cudaMemcpyAsync(h_deg, deg.p, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
        if (h_dang && g->ndangling) {
            DevBuf<uint32_t> out(g->ndangling);
            DevBuf<long long> nsel(1);
            cub::CountingInputIterator<uint32_t> it(0);
            IsZero pred{deg.p};
            size_t tmp = 0;
            PRGPU_CUDA(cub::DeviceSelect::If(nullptr, tmp, it, out.p, nsel.p, (int64_t)n, pred, st));
            DevBuf<char> t(tmp);
            PRGPU_CUDA(cub::DeviceSelect::If(t.p, tmp, it, out.p, nsel.p, (int64_t)n, pred, st));
            g_launches.fetch_add(1);
            PRGPU_CUDA(cudaMemcpyAsync(h_dang, out.p, (size_t)g->ndangling * 4,
                                       cudaMemcpyDeviceToHost, st));
            PRGPU_CUDA(cudaStreamSynchronize(st));
        }
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
    if (h_off) {
        DevBuf<uint64_t> off((size_t)n + 1);
        in_deg_orig<<<grid_for((uint64_t)n + 1), kThreads, 0, st>>>(g->row_off.p, g->new_of_old.p,
                                                                    n, off.p);
        PRGPU_LAUNCHED("in_deg_orig");
        exclusive_scan_u64(off.p, (uint64_t)n + 1, st);
        PRGPU_CUDA(cudaMemcpyAsync(h_off, off.p, ((size_t)n + 1) * 8, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
    if (h_nbr && e) {
        DevBuf<uint64_t> keys(e), alt(e);
        engine_to_orig_keys<<<grid_for(n), kThreads, 0, st>>>(g->row_off.p, g->col.p,
                                                              g->row_of_src.p, g->old_of_new.p, n,
                                                              g->lg, keys.p);
        PRGPU_LAUNCHED("engine_to_orig_keys");
        sort_keys(keys, alt, e, 2 * (int)g->lg, st);
        DevBuf<uint32_t> nb(e);
        keys_low<<<grid_for(e), kThreads, 0, st>>>(keys.p, e, g->lg, nb.p);
        PRGPU_LAUNCHED("keys_low");
        PRGPU_CUDA(cudaMemcpyAsync(h_nbr, nb.p, e * 4, cudaMemcpyDeviceToHost, st));
        PRGPU_CUDA(cudaStreamSynchronize(st));
    }
}

// In-neighbours of selected original rows in the reference layout (ascending
// per row): off[nrows+1] always filled; nbr (capacity cap) filled when it fits.
// Test tooling for graphs too large to download whole (C5).
uint64_t graph_rows(const prgpu_graph* g, const uint32_t* h_rows, uint32_t nrows, uint64_t* h_off,
                    uint32_t* h_nbr, uint64_t cap, cudaStream_t st) {
    if (g->shard_n > 1) fail(PRGPU_EINVAL, "graph_rows: a shard graph holds one rank's edges only");
    for (uint32_t i = 0; i < nrows; ++i)
        if (h_rows[i] >= g->n) fail(PRGPU_EINVAL, "graph_rows: row >= vertex_count");
    h_off[0] = 0;
    if (nrows == 0) return 0;
    DevBuf<uint32_t> rows(nrows);
    DevBuf<uint64_t> cnt((size_t)nrows + 1);
    PRGPU_CUDA(cudaMemcpyAsync(rows.p, h_rows, (size_t)nrows * 4, cudaMemcpyHostToDevice, st));
    rows_deg<<<grid_for(nrows), kThreads, 0, st>>>(g->row_off.p, g->new_of_old.p, rows.p, nrows, cnt.p);
    PRGPU_LAUNCHED("rows_deg");
    PRGPU_CUDA(cudaMemcpyAsync(h_off + 1, cnt.p, (size_t)nrows * 8, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    for (uint32_t i = 0; i < nrows; ++i) h_off[i + 1] += h_off[i];
    const uint64_t total = h_off[nrows];
    if (!h_nbr || total > cap || total == 0) return total;
    PRGPU_CUDA(cudaMemcpyAsync(cnt.p, h_off, ((size_t)nrows + 1) * 8, cudaMemcpyHostToDevice, st));
    DevBuf<uint32_t> out(total);
    rows_fill<<<grid_for((uint64_t)nrows * 32), kThreads, 0, st>>>(g->row_off.p, g->col.p, g->row_of_src.p,
                                                                    g->old_of_new.p, g->new_of_old.p, rows.p,
                                                                    nrows, cnt.p, out.p);
    PRGPU_LAUNCHED("rows_fill");
    PRGPU_CUDA(cudaMemcpyAsync(h_nbr, out.p, total * 4, cudaMemcpyDeviceToHost, st));
    PRGPU_CUDA(cudaStreamSynchronize(st));
    for (uint32_t i = 0; i < nrows; ++i) std::sort(h_nbr + h_off[i], h_nbr + h_off[i + 1]);
    return total;
}

} // namespace prgpu
