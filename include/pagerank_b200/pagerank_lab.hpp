// pagerank_b200/pagerank_lab.hpp — C++20 drop-in for the reference's
// pagerank_lab headers (graph.hpp, norms.hpp, pagerank.hpp, sweep.hpp), backed
// by libprgpu.so (include/prgpu.h) on a B200.
//
// Same type names, signatures, argument meaning and exceptions as the
// reference, in namespace pagerank_lab::cuda (so it can sit in one binary next
// to the reference headers).  `#include <pagerank_b200/dropin.hpp>` instead
// makes them visible as pagerank_lab::... for an unmodified caller.
//
//   build_csr      graph.hpp:204-234   device sort/unique/count/scan; the host
//                                      arrays are downloaded bit-identical
//   pagerank       pagerank.hpp:70-108 device loop, convergence on the device
//   error_norm     norms.hpp:48-78     device reduction
//   run_sweep      sweep.hpp:146-243   alphas batched as lanes, every (tau,
//                                      norm) cell read off one run's norm trace
// Host-only pieces (MatrixMarket text parsing, estimate_iterations, grids,
// CSV formatting, detect_sensitivity) stay on the host, as in the reference.
// Link with -lprgpu (paper_2108_02997_b200/libprgpu.so).
#pragma once

#include <prgpu.h>

#include <algorithm>
#include <array>
#include <cctype>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <filesystem>
#include <iterator>
#include <fstream>
#include <functional>
#include <istream>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace pagerank_lab::cuda {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
namespace b200_detail {
inline void check(int status, const char* what) {
    if (status == PRGPU_OK) return;
    std::string msg = std::string(what) + ": " + prgpu_last_error();
    if (status == PRGPU_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline int default_device() {
    if (const char* v = std::getenv("PRGPU_DEVICE")) return std::atoi(v);
    if (const char* v = std::getenv("LOCAL_RANK")) return std::atoi(v);
    return 0;
}
} // namespace b200_detail

// ---------------------------------------------------------------------------
// norms.hpp:18-78
// ---------------------------------------------------------------------------
enum class NormKind { L1, L2, LInf };

inline constexpr std::array<NormKind, 3> all_norms = {NormKind::L1, NormKind::L2, NormKind::LInf};

constexpr std::string_view norm_name(NormKind kind) {
    switch (kind) {
    case NormKind::L1: return "l1";
    case NormKind::L2: return "l2";
    case NormKind::LInf: return "linf";
    }
    return "?";
}

inline std::optional<NormKind> parse_norm(std::string_view token) {
    std::string t(token);
    for (char& c : t) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    if (t == "l1") return NormKind::L1;
    if (t == "l2") return NormKind::L2;
    if (t == "linf") return NormKind::LInf;
    return std::nullopt;
}

/// Distance between two equal-length vectors, reduced on the device in a
/// fixed order (run-to-run identical).
inline double error_norm(NormKind kind, std::span<const double> r, std::span<const double> s) {
    if (r.size() != s.size())
        throw std::invalid_argument("error_norm: vector lengths differ (" + std::to_string(r.size()) +
                                    " vs " + std::to_string(s.size()) + ")");
    if (r.empty()) throw std::invalid_argument("error_norm: empty vectors");
    double out = 0;
    b200_detail::check(prgpu_error_norm(static_cast<int>(kind), r.data(), s.data(), r.size(),
                                   b200_detail::default_device(), &out),
                  "error_norm");
    return out;
}

// ---------------------------------------------------------------------------
// graph.hpp
// ---------------------------------------------------------------------------
class MtxParseError : public std::runtime_error {
public:
    MtxParseError(std::size_t line, const std::string& what)
        : std::runtime_error("line " + std::to_string(line) + ": " + what), line_(line) {}
    std::size_t line() const noexcept { return line_; }

private:
    std::size_t line_;
};

struct EdgeList {
    std::uint32_t vertex_count = 0;
    std::vector<std::pair<std::uint32_t, std::uint32_t>> edges; // (source, target)
};

/// Reverse CSR in the reference layout (graph.hpp:47-60) plus the device
/// graph it came from.  Copies share the device graph; it is immutable and
/// safe to use from several threads.
struct CsrGraph {
    std::uint32_t vertex_count = 0;
    std::vector<std::uint64_t> in_offsets;
    std::vector<std::uint32_t> in_neighbors;
    std::vector<std::uint32_t> out_degree;
    std::vector<std::uint32_t> dangling;

    std::span<const std::uint32_t> in_edges(std::uint32_t v) const {
        return {in_neighbors.data() + in_offsets[v], in_neighbors.data() + in_offsets[v + 1]};
    }
    std::uint64_t edge_count() const { return in_neighbors.size(); }

    /// The device graph; built from the host arrays on first use when this
    /// CsrGraph was filled by hand.
    prgpu_graph* device_graph() const {
        std::lock_guard<std::mutex> lock(state_->mutex);
        if (!state_->graph) {
            if (vertex_count == 0) throw std::invalid_argument("pagerank: graph has no vertices");
            prgpu_graph* g = nullptr;
            b200_detail::check(prgpu_graph_from_csr(vertex_count, in_offsets.data(), in_neighbors.data(),
                                               out_degree.data(), b200_detail::default_device(), &g),
                          "graph_from_csr");
            state_->graph.reset(g, prgpu_graph_free);
        }
        return state_->graph.get();
    }

    void attach(prgpu_graph* g) { state_->graph.reset(g, prgpu_graph_free); }

private:
    struct State {
        std::mutex mutex;
        std::shared_ptr<prgpu_graph> graph;
    };
    std::shared_ptr<State> state_ = std::make_shared<State>();
};

namespace b200_detail {
// pairs from prgpu_mtx_parse / prgpu_mtx_load into an EdgeList
inline EdgeList take_pairs(std::uint32_t n, std::uint32_t* pairs, std::uint64_t m) {
    EdgeList el;
    el.vertex_count = n;
    el.edges.resize(m);
    static_assert(sizeof(std::pair<std::uint32_t, std::uint32_t>) == 8);
    if (m) std::memcpy(static_cast<void*>(el.edges.data()), pairs, m * 8);
    prgpu_pairs_free(pairs);
    return el;
}
} // namespace b200_detail

/// graph.hpp:111-199: the library's multi-threaded MatrixMarket parser
/// (prgpu_mtx_parse), same language, same MtxParseError lines and messages.
inline EdgeList parse_matrix_market(std::istream& in) {
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::uint32_t n = 0, *pairs = nullptr;
    std::uint64_t m = 0, line = 0;
    const int st = prgpu_mtx_parse(text.data(), text.size(), 0, &n, &pairs, &m, &line);
    if (st == PRGPU_EPARSE) {
        const std::string msg = prgpu_last_error(), prefix = "line " + std::to_string(line) + ": ";
        throw MtxParseError(line, msg.rfind(prefix, 0) == 0 ? msg.substr(prefix.size()) : msg);
    }
    b200_detail::check(st, "parse_matrix_market");
    return b200_detail::take_pairs(n, pairs, m);
}

namespace b200_detail {
inline CsrGraph download(prgpu_graph* g) {
    prgpu_graph_info info{};
    check(prgpu_graph_get_info(g, &info), "graph info");
    CsrGraph out;
    out.vertex_count = info.vertex_count;
    out.in_offsets.resize(static_cast<std::size_t>(info.vertex_count) + 1);
    out.in_neighbors.resize(info.edge_count);
    out.out_degree.resize(info.vertex_count);
    out.dangling.resize(info.dangling_count);
    check(prgpu_graph_download(g, out.in_offsets.data(), out.in_neighbors.data(), out.out_degree.data(),
                               out.dangling.data()),
          "graph download");
    out.attach(g);
    return out;
}
} // namespace b200_detail

/// graph.hpp:204-234 on the device.  The returned host arrays are identical
/// to the reference build_csr's; the device copy is kept for pagerank().
inline CsrGraph build_csr(EdgeList el) {
    // vertex_count 0 gives the empty graph, as graph.hpp:204-234 does;
    // pagerank() then throws (pagerank.hpp:74)
    static_assert(sizeof(std::pair<std::uint32_t, std::uint32_t>) == 8);
    prgpu_graph* g = nullptr;
    b200_detail::check(prgpu_graph_build(el.vertex_count, reinterpret_cast<const std::uint32_t*>(el.edges.data()),
                                    el.edges.size(), b200_detail::default_device(), &g),
                  "build_csr");
    return b200_detail::download(g);
}

/// graph.hpp:238-247: file parsed in place (mmap) by all host threads;
/// errors name the file (std::runtime_error).
inline EdgeList load_matrix_market(const std::filesystem::path& path) {
    std::uint32_t n = 0, *pairs = nullptr;
    std::uint64_t m = 0, line = 0;
    const int st = prgpu_mtx_load(path.string().c_str(), 0, &n, &pairs, &m, &line);
    if (st == PRGPU_EPARSE || st == PRGPU_EIO) throw std::runtime_error(prgpu_last_error());
    b200_detail::check(st, "load_matrix_market");
    return b200_detail::take_pairs(n, pairs, m);
}

/// graph.hpp:249-251: parallel parse, build_csr on the device.
inline CsrGraph load_csr_graph(const std::filesystem::path& path) {
    prgpu_graph* g = nullptr;
    std::uint64_t line = 0;
    const int st = prgpu_graph_load_mtx(path.string().c_str(), 0, b200_detail::default_device(), &g, &line);
    if (st == PRGPU_EPARSE || st == PRGPU_EIO) throw std::runtime_error(prgpu_last_error());
    b200_detail::check(st, "load_csr_graph");
    return b200_detail::download(g);
}

// ---------------------------------------------------------------------------
// pagerank.hpp
// ---------------------------------------------------------------------------
using RankVector = std::vector<double>;

struct PageRankConfig {
    double alpha = 0.85;
    double tolerance = 1e-6;
    NormKind norm = NormKind::L1;
    int max_iterations = 500;

    void validate() const {
        if (!(alpha >= 0.0 && alpha <= 1.0))
            throw std::invalid_argument("alpha must be in [0, 1], got " + std::to_string(alpha));
        if (!(tolerance > 0.0))
            throw std::invalid_argument("tolerance must be positive, got " + std::to_string(tolerance));
        if (max_iterations < 1)
            throw std::invalid_argument("max_iterations must be >= 1, got " + std::to_string(max_iterations));
    }
};

struct PageRankResult {
    RankVector ranks;
    int iterations = 0;
    bool converged = false;
    std::chrono::duration<double, std::milli> elapsed{}; // device loop time (CUDA events)
};

using IterationObserver = std::function<void(int iteration, std::span<const double> ranks, double error)>;

namespace b200_detail {
inline void observer_trampoline(int it, int, const double* ranks, std::uint64_t n, double err, void* user) {
    auto* obs = static_cast<const IterationObserver*>(user);
    (*obs)(it, std::span<const double>(ranks, n), err);
}
} // namespace b200_detail

/// pagerank.hpp:70-108: the pull power iteration, run to convergence on the
/// device.  `elapsed` is the device time of the iteration loop.
inline PageRankResult pagerank(const CsrGraph& g, const PageRankConfig& cfg,
                               const IterationObserver& on_iteration = {}) {
    cfg.validate();
    if (g.vertex_count == 0) throw std::invalid_argument("pagerank: graph has no vertices");
    prgpu_graph* dg = g.device_graph();
    const double alpha = cfg.alpha;
    prgpu_params p{};
    p.lanes = 1;
    p.alphas = &alpha;
    p.tolerance = cfg.tolerance;
    p.norm = static_cast<int>(cfg.norm);
    p.max_iterations = cfg.max_iterations;
    PageRankResult r;
    r.ranks.resize(g.vertex_count);
    int iters = 0;
    std::uint8_t conv = 0;
    prgpu_result out{};
    out.ranks = r.ranks.data();
    out.iterations = &iters;
    out.converged = &conv;
    if (on_iteration)
        b200_detail::check(prgpu_pagerank_observed(dg, &p, &out, b200_detail::observer_trampoline,
                                              const_cast<IterationObserver*>(&on_iteration)),
                      "pagerank");
    else
        b200_detail::check(prgpu_pagerank(dg, &p, &out), "pagerank");
    r.iterations = iters;
    r.converged = conv != 0;
    r.elapsed = std::chrono::duration<double, std::milli>(out.loop_ms);
    return r;
}

inline int estimate_iterations(double alpha, double tolerance) {
    if (!(alpha > 0.0 && alpha < 1.0))
        throw std::invalid_argument("estimate_iterations: alpha must be in (0, 1), got " + std::to_string(alpha));
    if (!(tolerance > 0.0 && tolerance < 1.0))
        throw std::invalid_argument("estimate_iterations: tolerance must be in (0, 1), got " +
                                    std::to_string(tolerance));
    const long e = std::lround(std::log10(tolerance) / std::log10(alpha));
    return static_cast<int>(std::max(1L, e));
}

constexpr PageRankConfig reference_config() {
    return {.alpha = 0.85, .tolerance = 1e-6, .norm = NormKind::L1, .max_iterations = 500};
}

inline RankVector reference_ranks(const CsrGraph& g) { return pagerank(g, reference_config()).ranks; }

inline double reference_error(const CsrGraph& g, std::span<const double> ranks) {
    const RankVector ref = reference_ranks(g);
    return error_norm(NormKind::L1, ranks, ref);
}

/// K runs that share every edge visit (one alpha each); per-lane results plus
/// the per-iteration norm trace [iteration][lane][L1, L2, LInf, L1-vs-ref].
struct BatchedRun {
    std::vector<PageRankResult> results;
    std::vector<double> trace;
    int run_iterations = 0;
    double loop_ms = 0;
};

inline BatchedRun pagerank_batched(const CsrGraph& g, std::span<const double> alphas, double tolerance,
                                   NormKind norm, int max_iterations, std::uint32_t stop_mask = 0,
                                   const RankVector* ref = nullptr, bool want_ranks = true,
                                   bool series = false) {
    // series: the same results from one alpha = 1 chain and per-lane weighted
    // sums (prgpu_pagerank_series; no ref trace)
    const int K = static_cast<int>(alphas.size());
    if (K < 1 || K > PRGPU_MAX_LANES) throw std::invalid_argument("pagerank_batched: 1..16 alphas");
    prgpu_params p{};
    p.lanes = K;
    p.alphas = alphas.data();
    p.tolerance = tolerance;
    p.norm = static_cast<int>(norm);
    p.stop_mask = stop_mask;
    p.max_iterations = max_iterations;
    p.ref_ranks = ref ? ref->data() : nullptr;
    BatchedRun b;
    std::vector<double> ranks(want_ranks ? static_cast<std::size_t>(K) * g.vertex_count : 0);
    std::vector<int> its(K);
    std::vector<std::uint8_t> conv(K);
    b.trace.assign(static_cast<std::size_t>(max_iterations) * K * 4, 0.0);
    prgpu_result out{};
    out.ranks = want_ranks ? ranks.data() : nullptr;
    out.iterations = its.data();
    out.converged = conv.data();
    out.err_trace = b.trace.data();
    if (series && ref) throw std::invalid_argument("pagerank_batched: series runs take no reference ranks");
    b200_detail::check(series ? prgpu_pagerank_series(g.device_graph(), &p, &out)
                              : prgpu_pagerank(g.device_graph(), &p, &out),
                       "pagerank");
    b.run_iterations = out.run_iterations;
    b.loop_ms = out.loop_ms;
    for (int k = 0; k < K; ++k) {
        PageRankResult r;
        if (want_ranks)
            r.ranks.assign(ranks.begin() + static_cast<std::ptrdiff_t>(k) * g.vertex_count,
                           ranks.begin() + static_cast<std::ptrdiff_t>(k + 1) * g.vertex_count);
        r.iterations = its[k];
        r.converged = conv[k] != 0;
        r.elapsed = std::chrono::duration<double, std::milli>(out.loop_ms);
        b.results.push_back(std::move(r));
    }
    return b;
}

// ---------------------------------------------------------------------------
// csv.hpp (host formatting used by sweep rows)
// ---------------------------------------------------------------------------
inline std::string format_double(double x) {
    char buf[32];
    const auto r = std::to_chars(buf, buf + sizeof buf, x);
    return std::string(buf, r.ptr);
}

inline std::string csv_escape(std::string_view field) {
    if (field.find_first_of(",\"\n") == std::string_view::npos) return std::string(field);
    std::string out = "\"";
    for (const char c : field) {
        out += c;
        if (c == '"') out += '"';
    }
    return out + '"';
}

// ---------------------------------------------------------------------------
// sweep.hpp
// ---------------------------------------------------------------------------
struct SweepPlan {
    std::vector<std::filesystem::path> graphs;
    std::vector<double> alphas{0.85};
    std::vector<double> tolerances{1e-6};
    std::vector<NormKind> norms{NormKind::L1};
    int repeats = 5;
    int max_iterations = 500;
    /// Not in the reference: run all alphas of a graph as batched lanes and
    /// read every (tau, norm) cell off the per-iteration norm trace of one run
    /// (the iterate sequence does not depend on tau or norm).  false runs each
    /// cell on its own exactly like the reference.
    bool fuse = true;

    void validate() const {
        if (graphs.empty()) throw std::invalid_argument("sweep: no graphs");
        if (alphas.empty()) throw std::invalid_argument("sweep: no alphas");
        if (tolerances.empty()) throw std::invalid_argument("sweep: no tolerances");
        if (norms.empty()) throw std::invalid_argument("sweep: no norms");
        if (repeats < 1) throw std::invalid_argument("sweep: repeats must be >= 1");
        if (max_iterations < 1) throw std::invalid_argument("sweep: max_iterations must be >= 1");
        for (const double a : alphas)
            if (!(a >= 0.0 && a <= 1.0)) throw std::invalid_argument("sweep: alpha out of [0, 1]: " + std::to_string(a));
        for (const double t : tolerances)
            if (!(t > 0.0)) throw std::invalid_argument("sweep: tolerance must be positive: " + std::to_string(t));
    }
};

struct SweepRecord {
    std::string graph;
    std::uint32_t vertices = 0;
    std::uint64_t edges = 0;
    double alpha = 0;
    double tolerance = 0;
    NormKind norm = NormKind::L1;
    int iterations = 0;
    bool converged = false;
    double time_ms = 0;    // fused: per-iteration cost of the batched run x iterations
    double err_vs_ref = 0; // L1 distance from alpha=0.85 reference ranks
};

inline constexpr std::string_view sweep_csv_header =
    "graph,vertices,edges,alpha,tolerance,norm,iterations,converged,time_ms,err_vs_ref";

inline std::string sweep_csv_row(const SweepRecord& r) {
    std::string row = csv_escape(r.graph);
    for (const std::string& f :
         {std::to_string(r.vertices), std::to_string(r.edges), format_double(r.alpha),
          format_double(r.tolerance), std::string(norm_name(r.norm)), std::to_string(r.iterations),
          std::string(r.converged ? "true" : "false"), format_double(r.time_ms), format_double(r.err_vs_ref)}) {
        row += ',';
        row += f;
    }
    return row;
}

inline void write_sweep_csv(std::ostream& os, std::span<const SweepRecord> records) {
    os << sweep_csv_header << '\n';
    for (const SweepRecord& r : records) os << sweep_csv_row(r) << '\n';
}

inline std::vector<double> default_damping_grid() {
    return {0.50, 0.55, 0.60, 0.65, 0.70, 0.75, 0.80, 0.85, 0.90, 0.95, 1.00};
}

inline std::vector<double> default_tolerance_grid() {
    return {1e0,  5e-1, 1e-1, 5e-2, 1e-2, 5e-3, 1e-3, 5e-4, 1e-4, 5e-5, 1e-5,
            5e-6, 1e-6, 5e-7, 1e-7, 5e-8, 1e-8, 5e-9, 1e-9, 5e-10, 1e-10};
}

namespace b200_detail {
inline void sweep_graph(const SweepPlan& plan, const CsrGraph& g, const std::string& label,
                        std::vector<SweepRecord>& out, std::ostream* log) {
    const RankVector ref = reference_ranks(g); // untimed warm-up (sweep.hpp:160-161)
    auto emit = [&](SweepRecord rec) {
        if (log) *log << sweep_csv_row(rec) << '\n';
        out.push_back(std::move(rec));
    };
    if (!plan.fuse) {
        for (const NormKind norm : plan.norms)
            for (const double alpha : plan.alphas)
                for (const double tol : plan.tolerances) {
                    const PageRankConfig cfg{alpha, tol, norm, plan.max_iterations};
                    PageRankResult result;
                    double total = 0;
                    for (int rep = 0; rep < plan.repeats; ++rep) {
                        PageRankResult r = pagerank(g, cfg);
                        total += r.elapsed.count();
                        if (rep > 0 && r.iterations != result.iterations)
                            throw std::logic_error("sweep: iteration count changed between repeats on " + label);
                        result = std::move(r);
                    }
                    emit({label, g.vertex_count, g.edge_count(), alpha, tol, norm, result.iterations,
                          result.converged, total / plan.repeats, error_norm(NormKind::L1, result.ranks, ref)});
                }
        return;
    }
    std::uint32_t mask = 0;
    for (const NormKind nm : plan.norms) mask |= 1u << static_cast<int>(nm);
    const double tau_min = *std::min_element(plan.tolerances.begin(), plan.tolerances.end());
    for (std::size_t c0 = 0; c0 < plan.alphas.size(); c0 += PRGPU_MAX_LANES) {
        const std::size_t kn = std::min<std::size_t>(PRGPU_MAX_LANES, plan.alphas.size() - c0);
        const std::span<const double> chunk(plan.alphas.data() + c0, kn);
        BatchedRun first;
        double total_ms = 0;
        for (int rep = 0; rep < plan.repeats; ++rep) {
            BatchedRun b = pagerank_batched(g, chunk, tau_min, plan.norms.front(), plan.max_iterations,
                                            mask, &ref, false);
            total_ms += b.loop_ms;
            // bitwise: NaN entries (prgpu.h err_trace) compare equal to themselves
            if (rep > 0 && (b.trace.size() != first.trace.size() ||
                            std::memcmp(b.trace.data(), first.trace.data(), b.trace.size() * sizeof(double)) != 0))
                throw std::logic_error("sweep: iteration trace changed between repeats on " + label);
            if (rep == 0) first = std::move(b);
        }
        const double per_iter = total_ms / plan.repeats / std::max(1, first.run_iterations);
        const int K = static_cast<int>(kn);
        for (const NormKind norm : plan.norms)
            for (int k = 0; k < K; ++k)
                for (const double tol : plan.tolerances) {
                    const int lane_its = first.results[k].iterations;
                    int t = std::min(lane_its, plan.max_iterations);
                    bool conv = false;
                    for (int i = 0; i < lane_its; ++i)
                        if (first.trace[(static_cast<std::size_t>(i) * K + k) * 4 + static_cast<int>(norm)] < tol) {
                            t = i + 1;
                            conv = true;
                            break;
                        }
                    emit({label, g.vertex_count, g.edge_count(), chunk[k], tol, norm, t, conv, per_iter * t,
                          first.trace[(static_cast<std::size_t>(t - 1) * K + k) * 4 + 3]});
                }
    }
}
} // namespace b200_detail

/// sweep.hpp:146-243.  Graphs run one after another on the GPU; records come
/// back sorted by (graph, norm, alpha, tolerance descending).
inline std::vector<SweepRecord> run_sweep(const SweepPlan& plan, std::ostream* log = nullptr) {
    plan.validate();
    std::vector<SweepRecord> records;
    for (const auto& path : plan.graphs) {
        const CsrGraph g = load_csr_graph(path);
        b200_detail::sweep_graph(plan, g, path.stem().string(), records, log);
    }
    std::sort(records.begin(), records.end(), [](const SweepRecord& a, const SweepRecord& b) {
        if (a.graph != b.graph) return a.graph < b.graph;
        if (a.norm != b.norm) return static_cast<int>(a.norm) < static_cast<int>(b.norm);
        if (a.alpha != b.alpha) return a.alpha < b.alpha;
        return a.tolerance > b.tolerance;
    });
    return records;
}

struct SensitivityFinding {
    std::string graph;
    NormKind norm = NormKind::L1;
    std::optional<double> first_failing_tolerance;
    std::vector<double> single_iteration_tolerances;
};

using SensitivityReport = std::vector<SensitivityFinding>;

/// sweep.hpp:262-310 (host post-processing).
inline SensitivityReport detect_sensitivity(std::span<const SweepRecord> records) {
    if (records.empty()) throw std::invalid_argument("detect_sensitivity: no records");
    std::map<std::pair<std::string, int>, std::vector<const SweepRecord*>> groups;
    std::vector<double> grid;
    for (const SweepRecord& r : records) {
        groups[{r.graph, static_cast<int>(r.norm)}].push_back(&r);
        grid.push_back(r.tolerance);
    }
    std::sort(grid.begin(), grid.end(), std::greater<>());
    grid.erase(std::unique(grid.begin(), grid.end()), grid.end());
    SensitivityReport report;
    for (auto& [key, cells] : groups) {
        std::sort(cells.begin(), cells.end(), [](auto* a, auto* b) { return a->tolerance > b->tolerance; });
        const std::string name = key.first + "/" + std::string(norm_name(NormKind(key.second)));
        if (cells.size() != grid.size())
            throw std::invalid_argument("detect_sensitivity: tolerance grid for " + name + " has gaps or duplicate cells");
        for (std::size_t i = 0; i < cells.size(); ++i)
            if (cells[i]->tolerance != grid[i])
                throw std::invalid_argument("detect_sensitivity: tolerance grid for " + name + " has gaps");
        SensitivityFinding f;
        f.graph = key.first;
        f.norm = NormKind(key.second);
        std::size_t tail = cells.size();
        while (tail > 0 && !cells[tail - 1]->converged) --tail;
        if (tail < cells.size()) f.first_failing_tolerance = cells[tail]->tolerance;
        for (const auto* c : cells)
            if (c->iterations == 1) f.single_iteration_tolerances.push_back(c->tolerance);
        report.push_back(std::move(f));
    }
    return report;
}

} // namespace pagerank_lab::cuda
