// engine_k1.cu — the pull_kernel instances of one-lane runs (LG = 1, W = 1,
// window 256: staged packed runs), in a translation unit of their own (lane_cfg.cuh).
#include "lane_cfg.cuh"

namespace prgpu {

LaneCfg k1_base() { return mk_cfg<1, 1, 256, 2, 3, kQmAll, 0, 3>(); }

namespace {
template <int PATHS>
bool k1_mode_t(int win, bool all_q, bool minb4, LaneCfg& out) {
    if (win == 256) {
        if (minb4) out = mk_cfg<1, 1, 256, 2, 4, kQmAll, 1, PATHS>();
        else out = mk_cfg<1, 1, 256, 2, 3, kQmAll, 1, PATHS>();
        return true;
    }
    return false; // (the one-lane mode of a wider run, win 128: engine.cu)
}
} // namespace

bool k1_mode(int paths, int win, bool all_q, bool minb4, LaneCfg& out) {
    switch (paths) {
    case 1: return k1_mode_t<1>(win, all_q, minb4, out);
    case 2: return k1_mode_t<2>(win, all_q, minb4, out);
    case 5: return k1_mode_t<5>(win, all_q, minb4, out);
    case 8: return k1_mode_t<8>(win, all_q, minb4, out);
    case 18: return k1_mode_t<18>(win, all_q, minb4, out);
    default: return false;
    }
}

} // namespace prgpu
