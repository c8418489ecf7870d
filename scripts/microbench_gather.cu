// microbench_gather.cu — hardware ceiling of random gathers on this GPU:
// sectors/s for (a) 8-byte gathers and (b) 96-byte row gathers, from an
// L2-resident table and from an HBM-sized table.  Used to decide whether the
// pull kernel is bound by the memory system or by its own structure.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/microbench_gather.cu -o /tmp/mbg
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 27; z *= 0x94D049BB133111EBull; return z ^ (z >> 31);
}

// each thread: `per` gathers of one double at random rows of `rows` rows of stride `stride` doubles
template <int UNROLL>
__global__ void g8(const double* __restrict__ t, uint64_t rows, int stride, int per, double* out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    double acc = 0;
    uint64_t s = mix(tid + 1);
    for (int i = 0; i < per; i += UNROLL) {
        double v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            s = mix(s + u);
            v[u] = __ldg(t + (s % rows) * stride);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u];
    }
    if (acc == 12345.0) out[0] = acc;
}

// 96-byte rows: 6 threads per row, double2 each (the K=11 layout)
template <int UNROLL>
__global__ void g96(const double* __restrict__ t, uint64_t rows, int per, double* out) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, slot = lane / 8, slice = lane % 8;
    double acc = 0;
    uint64_t s = mix((tid >> 3) + 1);
    for (int i = 0; i < per; i += UNROLL) {
        double2 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            s = mix(s + u);
            v[u] = slice < 6 ? __ldg(reinterpret_cast<const double2*>(t + (s % rows) * 12 + slice * 2))
                             : make_double2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) acc += v[u].x + v[u].y;
    }
    (void)slot;
    if (acc == 12345.0) out[0] = acc;
}

// index-driven (like the pull kernel: colidx stream + gather), no hashing
__global__ void gi8(const double* __restrict__ t, const uint32_t* __restrict__ idx, uint64_t m, double* out) {
    double acc = 0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    for (; i + 7 * stride < m; i += 8 * stride) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(t + idx[i + u * stride]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u];
    }
    if (acc == 12345.0) out[0] = acc;
}
__global__ void gi96(const double* __restrict__ t, const uint32_t* __restrict__ idx, uint64_t m, double* out) {
    // 8 threads per edge, 6 active (double2 each): K = 11 layout
    const int lane = threadIdx.x & 31, slot = lane / 8, slice = lane % 8;
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / 32;
    double acc = 0;
    for (uint64_t e = w * 4 + slot; e + 7 * warps * 4 < m; e += 8 * warps * 4) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
            v[u] = slice < 6 ? __ldg(reinterpret_cast<const double2*>(t + (uint64_t)idx[e + u * warps * 4] * 12 + slice * 2))
                             : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y;
    }
    if (acc == 12345.0) out[0] = acc;
}

__global__ void fill_idx(uint32_t* idx, uint64_t m, uint64_t rows, int skew) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t h = mix(i + 77);
        if (skew) { // power-law-ish: square of a uniform -> more mass at low ids
            const double u = (h >> 11) * (1.0 / 9007199254740992.0);
            idx[i] = (uint32_t)(u * u * u * rows);
        } else idx[i] = (uint32_t)(h % rows);
    }
}

int main() {
    {
        double* t; uint32_t* idx; double* out;
        const uint64_t m = 64ull << 20;
        cudaMalloc(&t, 4ull << 30); cudaMemset(t, 0, 4ull << 30);
        cudaMalloc(&idx, m * 4); cudaMalloc(&out, 8);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int skew = 0; skew < 2; ++skew)
        for (size_t bytes : {16ull << 20, 96ull << 20, 256ull << 20, 2048ull << 20}) {
            for (int kind = 0; kind < 2; ++kind) {
                const uint64_t rows = kind == 0 ? bytes / 8 : bytes / 96;
                fill_idx<<<1024, 256>>>(idx, m, rows, skew);
                float ms = 0;
                for (int rep = 0; rep < 3; ++rep) {
                    cudaEventRecord(a);
                    if (kind == 0) gi8<<<148 * 8, 256>>>(t, idx, m, out);
                    else gi96<<<148 * 8, 256>>>(t, idx, m, out);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    cudaEventElapsedTime(&ms, a, b);
                }
                printf("idx-%s %s table %5zu MB: %.3f ms  %.1f G gathers/s  %.2f TB/s incl. idx\n",
                       kind == 0 ? "g8 " : "g96", skew ? "skew" : "unif", bytes >> 20, ms, m / ms / 1e6,
                       m * (kind == 0 ? 36.0 : 100.0) / ms / 1e9);
            }
        }
        cudaFree(t); cudaFree(idx); cudaFree(out);
    }
    double* t;
    const size_t big = 512ull << 20; // 4 GB of doubles? no: 512M doubles = 4 GB
    cudaMalloc(&t, big * sizeof(double));
    cudaMemset(t, 0, big * sizeof(double));
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256, per = 256;
    for (size_t bytes : {16ull << 20, 64ull << 20, 256ull << 20, 2048ull << 20}) {
        // 8-byte gathers, stride 1 (each gather one sector)
        const uint64_t rows8 = bytes / 8;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            g8<8><<<blocks, threads>>>(t, rows8, 1, per, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double n = (double)blocks * threads * per;
        printf("g8   table %5zu MB: %.3f ms  %.1f Ggathers/s  %.2f TB/s of sectors\n", bytes >> 20, ms,
               n / ms / 1e6, n * 32 / ms / 1e9);
        const uint64_t rows96 = bytes / 96;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            g96<8><<<blocks, threads>>>(t, rows96, per, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms, a, b);
        const double rows_g = (double)blocks * threads / 8 * per; // row gathers
        printf("g96  table %5zu MB: %.3f ms  %.1f Grows/s     %.2f TB/s of sectors\n", bytes >> 20, ms,
               rows_g / ms / 1e6, rows_g * 96 / ms / 1e9);
    }
    return 0;
}
