// microbench_die_local.cu — does confining each die's SMs to one half of a
// gathered table double the L2 that gathers see?
//  1. SM -> die map: every SM times L2-hit loads of 512 lines spread over
//     memory (~2 KB apart, so their home dies are mixed); SMs on one die see
//     the same near/far pattern, so SMs are clustered by the correlation of
//     their latency profiles (2 clusters, seeded by SM 0's profile).
//  2. Gather rate, one 32-byte row per random index (4 threads x 8 B), from a
//     table of T MB: (a) every SM over the whole table, (b) die d's SMs only
//     over half d (same rows gathered per SM, same table).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/microbench_die_local.cu -o build_alt/mbd
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

constexpr int kLines = 512;

// one CTA per SM (grid = many, keep the first CTA seen per SM): latency per line
__global__ void probe(const uint32_t* __restrict__ buf, uint64_t stride_words, float* __restrict__ lat,
                      int* __restrict__ taken) {
    if (threadIdx.x != 0) return;
    const uint32_t s = smid();
    if (atomicCAS(taken + s, 0, 1) != 0) return;
    uint32_t sink = 0;
    for (int j = 0; j < kLines; ++j) sink += __ldcg(buf + j * stride_words); // warm L2
    for (int j = 0; j < kLines; ++j) {
        // a chain of 32 loads of the same L2-resident line, each address
        // depending on the previous value (which is 0): 31 latencies between
        // the two clock reads, whatever the compiler schedules
        const uint32_t* p = buf + j * stride_words;
        long long t0, t1;
        uint32_t v = 0;
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t0)::"memory");
#pragma unroll
        for (int r = 0; r < 32; ++r) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(p + v) : "memory");
        asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1)::"memory");
        sink += v;
        lat[s * kLines + j] = (float)(t1 - t0) / 31.0f;
    }
    if (sink == 0xdeadbeef) taken[0] = 2;
}

__global__ void fill_idx(uint32_t* idx, uint64_t m, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9E3779B97F4A7C15ull + seed;
        z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; z ^= z >> 31;
        idx[i] = (uint32_t)z;
    }
}

// persistent: each warp takes gathers; row = idx % rows (whole table) or
// die-local: half (die) of the table
__global__ void __launch_bounds__(256) gather(const double* __restrict__ t, const uint32_t* __restrict__ idx,
                                              uint64_t m, uint32_t rows, const int8_t* __restrict__ die,
                                              int local, double* out) {
    const int lane = threadIdx.x & 31, slot = lane / 4, slice = lane % 4;
    const uint32_t d = local ? (uint32_t)die[smid()] : 0u;
    const uint32_t half = rows / 2;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0;
    for (uint64_t base = warp * 32; base < m; base += warps * 32) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint64_t e = base + u * 8 + slot;
            const uint32_t x = __ldg(idx + e);
            const uint32_t r = local ? d * half + x % half : x % rows;
            v[u] = __ldg(t + (uint64_t)r * 4 + slice);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += v[u];
    }
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    // 1. SM -> die
    const uint64_t stride_words = 2048 / 4 + 8; // ~2 KB apart
    uint32_t* buf;
    cudaMalloc(&buf, kLines * stride_words * 4 + 4096);
    cudaMemset(buf, 0, kLines * stride_words * 4 + 4096);
    float* lat;
    int* taken;
    cudaMalloc(&lat, 256 * kLines * sizeof(float));
    cudaMalloc(&taken, 256 * sizeof(int));
    cudaMemset(taken, 0, 256 * sizeof(int));
    probe<<<sms * 8, 32>>>(buf, stride_words, lat, taken);
    cudaDeviceSynchronize();
    std::vector<float> L(256 * kLines);
    std::vector<int> tk(256);
    cudaMemcpy(L.data(), lat, L.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(tk.data(), taken, tk.size() * 4, cudaMemcpyDeviceToHost);
    std::vector<int8_t> die(256, 0);
    int found = 0;
    for (int s = 0; s < 256; ++s) found += tk[s] == 1;
    // correlation of each SM's profile with SM 0's (centred)
    auto prof = [&](int s) {
        std::vector<double> p(kLines);
        double mu = 0;
        for (int j = 0; j < kLines; ++j) mu += p[j] = L[s * kLines + j];
        mu /= kLines;
        for (auto& x : p) x -= mu;
        return p;
    };
    const auto p0 = prof(0);
    int n0 = 0, n1 = 0;
    double cmin = 1, cmax = -1;
    for (int s = 0; s < sms; ++s) {
        const auto p = prof(s);
        double num = 0, a = 0, b = 0;
        for (int j = 0; j < kLines; ++j) num += p[j] * p0[j], a += p[j] * p[j], b += p0[j] * p0[j];
        const double c = num / std::sqrt(a * b + 1e-30);
        cmin = std::min(cmin, c);
        cmax = std::max(cmax, c);
        die[s] = c > 0 ? 0 : 1;
        (die[s] ? n1 : n0)++;
    }
    double near = 0, far = 0;
    int nn = 0, nf = 0;
    for (int j = 0; j < kLines; ++j) { // per line: SM0's die vs the other die's mean latency
        double a = 0, b = 0;
        int ca = 0, cb = 0;
        for (int s = 0; s < sms; ++s) (die[s] ? (b += L[s * kLines + j], ++cb) : (a += L[s * kLines + j], ++ca));
        if (ca && cb) { near += std::min(a / ca, b / cb); far += std::max(a / ca, b / cb); ++nn; ++nf; }
    }
    printf("SMs probed %d of %d; clusters %d / %d; profile correlation with SM 0 in [%.2f, %.2f]; "
           "L2 hit latency near %.0f / far %.0f cycles (per-line min / max of the two clusters' means)\n",
           found, sms, n0, n1, cmin, cmax, near / nn, far / nf);
    printf("SM 0 latencies (first 16 lines):");
    for (int j = 0; j < 16; ++j) printf(" %.0f", L[j]);
    printf("\nSM 100 latencies (first 16 lines):");
    for (int j = 0; j < 16; ++j) printf(" %.0f", L[100 * kLines + j]);
    printf("\ndie map:");
    for (int s = 0; s < sms; ++s) printf("%d", die[s]);
    printf("\n");
    int8_t* ddie;
    cudaMalloc(&ddie, 256);
    cudaMemcpy(ddie, die.data(), 256, cudaMemcpyHostToDevice);
    // 2. gathers
    const uint64_t m = 1ull << 28;
    uint32_t* idx;
    cudaMalloc(&idx, m * 4);
    fill_idx<<<4096, 256>>>(idx, m, 11);
    double* out;
    cudaMalloc(&out, 8);
    double* t;
    const uint64_t max_rows = (256ull << 20) / 32;
    cudaMalloc(&t, max_rows * 32);
    cudaMemset(t, 0, max_rows * 32);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mb : {32, 48, 64, 80, 96, 112, 128, 160, 192, 256}) {
        const uint32_t rows = (uint32_t)(((uint64_t)mb << 20) / 32);
        float res[2];
        for (int local = 0; local < 2; ++local) {
            gather<<<sms * 4, 256>>>(t, idx, m, rows, ddie, local, out);
            float best = 1e30f;
            for (int r = 0; r < 3; ++r) {
                cudaEventRecord(e0);
                gather<<<sms * 4, 256>>>(t, idx, m, rows, ddie, local, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                best = std::min(best, ms);
            }
            res[local] = m / (best * 1e-3) / 1e9;
        }
        printf("table %3d MB: whole table %6.1f G rows/s, die-local halves %6.1f G rows/s (x%.2f)\n", mb, res[0],
               res[1], res[1] / res[0]);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
