// microbench_fetch_size.cu — does a load's L2 prefetch-size qualifier change
// the DRAM bytes moved per missed random 32-byte row (128 bytes with plain
// loads, profiles/r2_random_rows.md) or the random-row rate?  Same set-up as
// microbench_random_rows.cu: 1 G uniform indices over a 3.2 GB table.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/microbench_fetch_size.cu -o build_alt/mfs
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void fill_idx(uint32_t* idx, uint64_t m, uint64_t rows, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull + seed;
        z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31;
        idx[i] = (uint32_t)(z % rows);
    }
}

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
    double v;
    if constexpr (MODE == 0) v = __ldg(p);
    else if constexpr (MODE == 1) asm volatile("ld.global.nc.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (MODE == 2) asm volatile("ld.global.nc.L2::128B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (MODE == 3) asm volatile("ld.global.nc.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (MODE == 4) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (MODE == 5) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (MODE == 6) asm volatile("ld.global.cs.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else if constexpr (MODE == 7) asm volatile("ld.global.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
    else asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int MODE, int LG, int U>
__global__ void __launch_bounds__(256) gather(const double* __restrict__ t, const uint32_t* __restrict__ idx,
                                              uint64_t m, double* out) {
    const int lane = threadIdx.x & 31, slot = lane / LG, slice = lane % LG;
    constexpr int ES = 32 / LG;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0;
    for (uint64_t base = warp * ES * U; base < m; base += warps * ES * U) {
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t e = base + u * ES + slot;
            v[u] = e < m ? ld<MODE>(t + (uint64_t)__ldg(idx + e) * 4 + slice) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 12345.0) out[0] = acc;
}

template <int MODE>
void run(const char* name, const double* t, const uint32_t* idx, uint64_t m, double* out) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<MODE, 4, 8><<<grid, 256>>>(t, idx, m, out);
    float best = 1e30f;
    for (int r = 0; r < 2; ++r) {
        cudaEventRecord(a);
        gather<MODE, 4, 8><<<grid, 256>>>(t, idx, m, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    printf("mode %d %-34s %.2f ms  %.1f G rows/s  err %s\n", MODE, name, best, m / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    const uint64_t rows = 100'000'000ull;
    const uint64_t m = 1ull << (argc > 1 ? atoi(argv[1]) : 30);
    double *t, *out;
    uint32_t* idx;
    cudaMalloc(&t, rows * 32);
    cudaMalloc(&idx, m * 4);
    cudaMalloc(&out, 8);
    cudaMemset(t, 0, rows * 32);
    fill_idx<<<4096, 256>>>(idx, m, rows, 7);
    cudaDeviceSynchronize();
    run<0>("__ldg", t, idx, m, out);
    run<1>("ld.global.nc.L2::64B", t, idx, m, out);
    run<2>("ld.global.nc.L2::128B", t, idx, m, out);
    run<3>("ld.global.nc.L2::256B", t, idx, m, out);
    run<4>("ld.global.nc.L1::no_allocate", t, idx, m, out);
    run<5>("ld.global.cg", t, idx, m, out);
    run<6>("ld.global.cs", t, idx, m, out);
    run<7>("ld.global.L1::no_allocate.L2::64B", t, idx, m, out);
    run<8>("ld.volatile.global", t, idx, m, out);
    return 0;
}
