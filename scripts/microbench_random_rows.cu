// microbench_random_rows.cu — the DRAM rate for random 32-byte rows on this
// B200: a precomputed index stream (uniform over the table, no hashing in
// the timed loop) and one 32-byte row gathered per index, many rows in
// flight.  Settles whether C5's hub kernel (~74 G misses/s, ~5 TB/s of
// 64-byte DRAM atoms) sits at the hardware's random-access rate.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/microbench_random_rows.cu -o /tmp/mbr
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__global__ void fill_idx(uint32_t* idx, uint64_t m, uint64_t rows, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull + seed;
        z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31;
        idx[i] = (uint32_t)(z % rows);
    }
}

// LG threads per row (8 B each, like the pull kernel's 4-lane instance),
// U rows in flight per thread per step
template <int LG, int U>
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
            v[u] = e < m ? __ldg(t + (uint64_t)__ldg(idx + e) * 4 + slice) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 12345.0) out[0] = acc;
}

template <int LG, int U>
void run(const char* name, const double* t, const uint32_t* idx, uint64_t m, double* out, int ctas_per_sm) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = sms * ctas_per_sm;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    gather<LG, U><<<grid, 256>>>(t, idx, m, out);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(a);
        gather<LG, U><<<grid, 256>>>(t, idx, m, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    printf("%-28s LG=%d U=%2d CTAs/SM=%d: %.2f ms  %.1f G rows/s  (%.2f TB/s at 64 B per row)\n", name, LG, U,
           ctas_per_sm, best, m / (best * 1e-3) / 1e9, m * 64.0 / (best * 1e-3) / 1e12);
}

int main() {
    const uint64_t rows = 100'000'000ull; // 3.2 GB of 32-byte rows (C5's table)
    const uint64_t m = 1ull << 30;         // 1 G gathers
    double* t;
    uint32_t* idx;
    double* out;
    cudaMalloc(&t, rows * 32);
    cudaMalloc(&idx, m * 4);
    cudaMalloc(&out, 8);
    cudaMemset(t, 0, rows * 32);
    fill_idx<<<4096, 256>>>(idx, m, rows, 7);
    cudaDeviceSynchronize();
    size_t g0 = 0;
    cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity);
    printf("default cudaLimitMaxL2FetchGranularity = %zu\n", g0);
    for (size_t gr : {32, 64, 128}) {
        const cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gr);
        size_t got = 0;
        cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity);
        printf("set %zu -> %s, now %zu\n", gr, cudaGetErrorString(e), got);
        run<4, 8>("uniform 3.2 GB", t, idx, m, out, 4);
    }
    cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g0);
    run<4, 4>("uniform 3.2 GB", t, idx, m, out, 4);
    run<4, 8>("uniform 3.2 GB", t, idx, m, out, 4);
    run<4, 8>("uniform 3.2 GB", t, idx, m, out, 8);
    run<4, 16>("uniform 3.2 GB", t, idx, m, out, 4);
    run<1, 4>("uniform 3.2 GB (1 thr/row)", t, idx, m, out, 8);
    run<1, 8>("uniform 3.2 GB (1 thr/row)", t, idx, m, out, 8);
    // a sequential copy for reference
    {
        double* d;
        cudaMalloc(&d, rows * 32);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaMemcpy(d, t, rows * 32, cudaMemcpyDeviceToDevice);
        cudaEventRecord(a);
        cudaMemcpy(d, t, rows * 32, cudaMemcpyDeviceToDevice);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        printf("copy 3.2 GB: %.2f ms = %.2f TB/s (read + write)\n", ms, 2.0 * rows * 32 / (ms * 1e-3) / 1e12);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
