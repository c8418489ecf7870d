// microbench_tma_gather.cu — random row gathers on B200: per-thread LDG
// (the current pull kernel's way) against TMA tile::gather4 into shared
// memory (cp.async.bulk.tensor.2d ... tile::gather4, mbarrier completion),
// index-driven like the pull kernel (a u32 index stream + one row per index).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a scripts/microbench_tma_gather.cu -lcuda -o /tmp/mtg
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; return z ^ (z >> 31);
}

__global__ void fill_idx(uint32_t* idx, uint64_t m, uint64_t rows, int skew) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix(i + 77);
        if (skew) {
            const double u = (h >> 11) * (1.0 / 9007199254740992.0);
            idx[i] = (uint32_t)(u * u * u * rows);
        } else idx[i] = (uint32_t)(h % rows);
    }
}

__global__ void hotcold_idx(uint32_t* idx, uint64_t m, uint64_t hot, uint64_t rows, double hf, int split) {
    const uint64_t nh = (uint64_t)(hf * m);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix(i + 99), h2 = mix(h);
        const bool is_hot = split ? (i < nh) : ((h2 >> 11) * (1.0 / 9007199254740992.0) < hf);
        idx[i] = is_hot ? (uint32_t)(h % hot) : (uint32_t)(hot + h % (rows - hot));
    }
}

// LDG: LG threads per row, 16 bytes each (RB = row bytes), 8 rows in flight per thread
template <int RB>
__global__ void __launch_bounds__(256) ldg_rows(const double* __restrict__ t, const uint32_t* __restrict__ idx, uint64_t m,
                                                double* out) {
    constexpr int LG = RB >= 16 ? RB / 16 : 1;
    constexpr int ES = 32 / LG;
    const int lane = threadIdx.x & 31, slot = lane / LG, slice = lane % LG;
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
    double acc = 0;
    constexpr int RD = RB / 8; // doubles per row
    for (uint64_t e = w * ES + slot; e + 7 * warps * ES < m; e += 8 * warps * ES) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint64_t r = idx[e + u * warps * ES];
            if constexpr (RB == 8) v[u] = make_double2(__ldg(t + r), 0.0);
            else v[u] = __ldg(reinterpret_cast<const double2*>(t + r * RD + slice * 2));
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 12345.0) out[0] = acc;
}

// 96-byte rows with lane groups of 8 (6 active, 4 rows per warp instruction:
// the pull kernel's K = 11 layout) against ldg_rows<96> (groups of 6, 5 rows)
__global__ void __launch_bounds__(256) ldg_rows96_lg8(const double* __restrict__ t, const uint32_t* __restrict__ idx,
                                                      uint64_t m, double* out) {
    const int lane = threadIdx.x & 31, slot = lane / 8, slice = lane % 8;
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
    double acc = 0;
    for (uint64_t e = w * 4 + slot; e + 7 * warps * 4 < m; e += 8 * warps * 4) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint64_t r = idx[e + u * warps * 4];
            v[u] = slice < 6 ? __ldg(reinterpret_cast<const double2*>(t + r * 12 + slice * 2)) : make_double2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 12345.0) out[0] = acc;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// TMA gather4: each warp owns D stages of 4 rows; lane 0 issues, all lanes consume
template <int RB, int D>
__global__ void __launch_bounds__(128) tma_rows(const __grid_constant__ CUtensorMap map, const uint32_t* __restrict__ idx,
                                                uint64_t m, double* out) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    constexpr int STAGE = 4 * RB;                     // bytes landed per stage
    constexpr int SP = (STAGE + 127) / 128 * 128;     // TMA destinations 128-byte aligned
    unsigned char* buf = smem + (size_t)wib * (D * SP + 128 * ((D * 8 + 127) / 128));
    uint64_t* bar = reinterpret_cast<uint64_t*>(buf + D * SP);
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + wib;
    const uint64_t groups = m / 4;
    if (lane == 0)
        for (int s = 0; s < D; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    auto issue = [&](uint64_t g, int s) {
        const uint4 r = *reinterpret_cast<const uint4*>(idx + 4 * g);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar + s)), "r"(STAGE) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(buf + s * SP)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w),
            "r"(su32(bar + s))
            : "memory");
    };
    if (lane == 0)
        for (int s = 0; s < D; ++s)
            if (w + s * nw < groups) issue(w + s * nw, s);
    double acc = 0;
    int it = 0;
    for (uint64_t g = w; g < groups; g += nw, ++it) {
        const int s = it % D;
        const uint32_t par = (it / D) & 1;
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                         : "=r"(ok) : "r"(su32(bar + s)), "r"(par) : "memory");
        const double* rows = reinterpret_cast<const double*>(buf + s * SP);
        for (int j = lane; j < STAGE / 8; j += 32) acc += rows[j];
        __syncwarp();
        if (lane == 0 && g + D * nw < groups) issue(g + D * nw, s);
    }
    if (acc == 12345.0) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no cuTensorMapEncodeTiled\n"); return 1; }
    const uint64_t m = 64ull << 20;
    double* t; uint32_t* idx; double* out;
    cudaMalloc(&t, 4ull << 30); cudaMemset(t, 0, 4ull << 30);
    cudaMalloc(&idx, m * 4); cudaMalloc(&out, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int nsm = 148;
    // L2 capacity sweep: uniform 8-byte and 32-byte gathers, LDG only
    for (int rb : {8, 32})
        for (size_t mb : {16, 32, 48, 56, 64, 72, 80, 96, 112, 128, 160, 256}) {
            const uint64_t rows = (mb << 20) / rb;
            fill_idx<<<1024, 256>>>(idx, m, rows, 0);
            float ms = 0;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (rb == 8) ldg_rows<8><<<nsm * 8, 256>>>(t, idx, m, out);
                else ldg_rows<32><<<nsm * 8, 256>>>(t, idx, m, out);
                cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
            }
            printf("L2 sweep: unif table %4zu MB rows %2d B: %.3f ms  %.1f Grows/s\n", mb, rb, ms, m / ms / 1e6);
        }
    if (getenv("LG_ONLY")) {
        for (int skew = 0; skew < 2; ++skew)
            for (size_t mb : {48, 96, 194, 512}) {
                const uint64_t rows = (mb << 20) / 96;
                fill_idx<<<1024, 256>>>(idx, m, rows, skew);
                float a6 = 0, a8 = 0;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a); ldg_rows<96><<<nsm * 8, 256>>>(t, idx, m, out); cudaEventRecord(b);
                    cudaEventSynchronize(b); cudaEventElapsedTime(&a6, a, b);
                    cudaEventRecord(a); ldg_rows96_lg8<<<nsm * 8, 256>>>(t, idx, m, out); cudaEventRecord(b);
                    cudaEventSynchronize(b); cudaEventElapsedTime(&a8, a, b);
                }
                printf("%s 96 B rows table %4zu MB: groups of 6 (5 rows/warp) %.1f G rows/s | groups of 8 (4 rows/warp) %.1f G rows/s\n",
                       skew ? "skew" : "unif", mb, m / a6 / 1e6, m / a8 / 1e6);
            }
        return 0;
    }
    if (getenv("SWEEP_ONLY")) return 0;
    // hot/cold split: a fraction `hf` of the gathers hits the hottest `hot_mb`
    // of a `tab_mb` table (96-byte rows, like C2); mixed in one stream, or
    // hot-first then cold (two passes over separated streams)
    if (getenv("HOTCOLD")) {
        for (int rb : {96, 32, 8})
            for (double hf : {0.85, 0.95})
                for (size_t hot_mb : {32, 48, 64}) {
                    const size_t tab_mb = rb == 96 ? 194 : (rb == 32 ? 3072 : 216);
                    const uint64_t rows = (tab_mb << 20) / rb, hot = (hot_mb << 20) / rb;
                    const uint64_t nh = (uint64_t)(hf * m);
                    hotcold_idx<<<1024, 256>>>(idx, m, hot, rows, hf, 0);
                    float ms_mix = 0, ms_a = 0, ms_b = 0;
                    for (int rep = 0; rep < 3; ++rep) {
                        cudaEventRecord(a);
                        if (rb == 96) ldg_rows<96><<<nsm * 8, 256>>>(t, idx, m, out);
                        else if (rb == 32) ldg_rows<32><<<nsm * 8, 256>>>(t, idx, m, out);
                        else ldg_rows<8><<<nsm * 8, 256>>>(t, idx, m, out);
                        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms_mix, a, b);
                    }
                    hotcold_idx<<<1024, 256>>>(idx, m, hot, rows, hf, 1); // hot first, then cold
                    for (int rep = 0; rep < 3; ++rep) {
                        cudaEventRecord(a);
                        if (rb == 96) ldg_rows<96><<<nsm * 8, 256>>>(t, idx, nh, out);
                        else if (rb == 32) ldg_rows<32><<<nsm * 8, 256>>>(t, idx, nh, out);
                        else ldg_rows<8><<<nsm * 8, 256>>>(t, idx, nh, out);
                        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms_a, a, b);
                        cudaEventRecord(a);
                        if (rb == 96) ldg_rows<96><<<nsm * 8, 256>>>(t, idx + nh, m - nh, out);
                        else if (rb == 32) ldg_rows<32><<<nsm * 8, 256>>>(t, idx + nh, m - nh, out);
                        else ldg_rows<8><<<nsm * 8, 256>>>(t, idx + nh, m - nh, out);
                        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms_b, a, b);
                    }
                    printf("hotcold rows %2d B table %4zu MB hot %2zu MB frac %.2f: mixed %.3f ms | hot pass %.3f + cold pass %.3f = %.3f ms (%.2fx)\n",
                           rb, tab_mb, hot_mb, hf, ms_mix, ms_a, ms_b, ms_a + ms_b, ms_mix / (ms_a + ms_b));
                }
        return 0;
    }
    for (int skew = 0; skew < 2; ++skew)
        for (size_t bytes : {48ull << 20, 256ull << 20, 3072ull << 20})
            for (int rb : {16, 32, 96}) {
                const uint64_t rows = bytes / rb;
                fill_idx<<<1024, 256>>>(idx, m, rows, skew);
                float ms_l = 0, ms_t[3] = {0, 0, 0};
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    if (rb == 16) ldg_rows<16><<<nsm * 8, 256>>>(t, idx, m, out);
                    if (rb == 32) ldg_rows<32><<<nsm * 8, 256>>>(t, idx, m, out);
                    if (rb == 96) ldg_rows<96><<<nsm * 8, 256>>>(t, idx, m, out);
                    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms_l, a, b);
                }
                CUtensorMap map;
                cuuint64_t dims[2] = {(cuuint64_t)rb / 8, rows};
                cuuint64_t strides[1] = {(cuuint64_t)rb};
                cuuint32_t box[2] = {(cuuint32_t)rb / 8, 1};
                cuuint32_t es[2] = {1, 1};
                CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, t, dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
                if (r != CUDA_SUCCESS) { printf("encode failed %d (rb %d)\n", (int)r, rb); continue; }
                const int Ds[3] = {8, 16, 32};
                for (int di = 0; di < 3; ++di) {
                    const int D = Ds[di];
                    const size_t sp = (4 * rb + 127) / 128 * 128;
                    const size_t sm = 4 * (size_t)(D * sp + 128 * ((D * 8 + 127) / 128)) + 128;
                    for (int rep = 0; rep < 3; ++rep) {
                        cudaEventRecord(a);
#define L(RB, DD) if (rb == RB && D == DD) { cudaFuncSetAttribute(tma_rows<RB, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
                        tma_rows<RB, DD><<<nsm * 8, 128, sm>>>(map, idx, m, out); }
                        L(16, 8) L(16, 16) L(16, 32) L(32, 8) L(32, 16) L(32, 32) L(96, 8) L(96, 16) L(96, 32)
                        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms_t[di], a, b);
                    }
                }
                cudaError_t e = cudaGetLastError();
                printf("%s table %5zu MB rows %3d B: ldg %.3f ms (%.1f Grows/s) | tma D8 %.3f D16 %.3f D32 %.3f ms (best %.1f Grows/s) %s\n",
                       skew ? "skew" : "unif", bytes >> 20, rb, ms_l, m / ms_l / 1e6, ms_t[0], ms_t[1], ms_t[2],
                       m / fminf(ms_t[0], fminf(ms_t[1], ms_t[2])) / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    return 0;
}
