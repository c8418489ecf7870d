// lane_cfg.cuh — a pull_kernel instance and its launch shape (shared by
// engine.cu and engine_k1.cu: the one-lane instances are compiled in a
// translation unit of their own, so nvcc's output for them does not shift
// with the wide-lane code of the other instances — DESIGN.md "Tuning log").
#pragma once

#include <cstdlib>

#include "common.cuh"
#include "pull.cuh"

namespace prgpu {

// ============================================================================
// Lane configurations: K lanes -> (LG threads per edge/row, W lanes per thread,
// WIN edge window per packed task).  Shared memory per warp = 2*WIN*KP doubles.
// ============================================================================
using KernelFn = void (*)(const Params);

struct LaneCfg {
    int LG, W, WIN, KS; // KS: contribution row stride (doubles)
    KernelFn fn;        // pull_kernel instance
    int QM = kQmAll;
    KernelFn fin = nullptr; // matching part_finalize_kernel (multi-GPU)
    int paths = 3;          // task kinds compiled in (pull_kernel PATHS)
    int KP() const { return LG * W; }
    size_t smem() const {
        const bool async = paths == 1 && kAsyncHub && LG > 1 && (KS == 2 || KS == 4); // pull.cuh async_hub
        const bool packs = paths != 3 && (paths & (2 | 8)) != 0; // packed_pipe instances (pull.cuh PACKS)
        const size_t staged = KP() == 1 ? (size_t)kWarps * 2 * WIN * sizeof(double) // STAGED
                              : packs ? (size_t)kWarps *
                                                 ((kStagedWide && LG == 4 && KS == 4) ? 2 * WIN * KS
                                                                                     : kPackOff + (2 * WIN + 8) / 2) *
                                                 sizeof(double)
                              : async      ? (size_t)kWarps * 2 * kAsyncBlock * KS * sizeof(double)
                                           : 0; // packed_pipe stage / cp.async ring
        const bool smemp = W >= 6 || (paths != 3 && KP() > 1);
        const size_t cols = smemp ? (size_t)popc_c(QM) * W * kNT * sizeof(double) : 0;     // Partials
        return staged + cols;
    }
};

// CTAs per SM the 11/12-lane instances are compiled for (tuning builds:
// -DPRGPU_K12_MINB=5/6 trade registers for resident warps)
#ifndef PRGPU_K12_MINB
#define PRGPU_K12_MINB 4
#endif
constexpr int kMinb12 = PRGPU_K12_MINB;

// packed-row window of the 3/4-lane instances (tuning builds: -DPRGPU_W4=64 / 32)
#ifndef PRGPU_W4
#define PRGPU_W4 128
#endif
constexpr int kW4 = PRGPU_W4;

// per-mode instance alternatives (tuning only)
inline int k_variant(const char* name) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : 0;
}

// `all_q`: the run needs every partial (all norms / the reference trace);
// otherwise only L1 + dangling (the damping sweep's stopping rule).
template <int LG, int W, int WIN, int QJ, int MINB, int QM, int KS, int PATHS = 3>
LaneCfg mk_cfg() {
    return LaneCfg{LG, W, WIN, KS ? KS : LG * W, pull_kernel<LG, W, WIN, QJ, MINB, QM, KS, PATHS>, QM,
                   part_finalize_kernel<LG, W, WIN, QJ, MINB, QM, KS>, PATHS};
}

// the one-lane (LG = 1, W = 1) instances, engine_k1.cu.  k1_base: the run's
// base configuration (one kernel per iteration); k1_mode: the kernels of a
// split iteration (paths: pull_kernel PATHS), win 256 (minb4: 4 CTAs/SM
// instead of 3); false for another window (the one-lane mode of a wider run is engine.cu's)
LaneCfg k1_base();
bool k1_mode(int paths, int win, bool all_q, bool minb4, LaneCfg& out);

} // namespace prgpu
