// pagerank-lab command line over the B200 path.
//
// Same subcommands, flags, outputs and exit codes as the reference CLI
// (/root/reference/proj/tools/main.cpp): run, sweep-damping,
// sweep-tolerance, compare-norms, ratios, estimate, chart.  The PageRank
// work goes through the drop-in (<pagerank_b200/dropin.hpp>: device
// build_csr, batched lanes, fused tau x norm sweeps); the host-only
// reporting comes from the reference's own stats.hpp / csv.hpp / chart.hpp,
// unchanged (compiled in from the reference include tree, see
// tools/Makefile).  The reference's CLI11 dependency is not in the image,
// so the flags are parsed here by a small table-driven parser with CLI11's
// observable behaviour for this CLI: `--opt value` and `--opt=value`,
// multi-value `--graphs a b c`, comma lists for --tol-grid / --norms,
// required options, unknown flags and bad numbers -> exit 2.
//
// Exit codes (main.cpp:1-8): 0 success, 1 parse/IO error, 2 invalid flags
// or values, 3 `run` finished without converging.
//
// Timing column: sweeps run fused by default (all alphas of a graph as
// batched lanes, every (tau, norm) cell read off one run's norm trace), and
// time_ms is then the batched loop's per-iteration cost x the cell's
// iterations; `--per-cell-timing` runs and times every cell on its own, as
// the reference does (sweep.hpp:173-192).  All other columns are identical.
#include <pagerank_b200/dropin.hpp>
#include <pagerank_lab/chart.hpp>
#include <pagerank_lab/csv.hpp>
#include <pagerank_lab/stats.hpp>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace {

using namespace pagerank_lab;

// ---- flag parsing ---------------------------------------------------------

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Flag {
    std::vector<std::string> names; // first is canonical
    enum Kind { Value, Multi, List, Switch } kind = Value;
    bool required = false;
    std::string help;
    std::vector<std::string> values; // as given
    bool seen = false;
};

class Command {
public:
    Command(std::string name, std::string help) : name_(std::move(name)), help_(std::move(help)) {}
    Command& value(std::vector<std::string> names, std::string help, bool required = false) {
        return add(std::move(names), Flag::Value, std::move(help), required);
    }
    Command& multi(std::vector<std::string> names, std::string help, bool required = false) {
        return add(std::move(names), Flag::Multi, std::move(help), required);
    }
    Command& list(std::vector<std::string> names, std::string help) {
        return add(std::move(names), Flag::List, std::move(help), false);
    }
    Command& flag(std::vector<std::string> names, std::string help) {
        return add(std::move(names), Flag::Switch, std::move(help), false);
    }

    // returns false when help was requested
    bool parse(const std::vector<std::string>& args) {
        for (std::size_t i = 0; i < args.size(); ++i) {
            std::string tok = args[i];
            if (tok == "-h" || tok == "--help") return false;
            std::optional<std::string> inline_val;
            if (const auto eq = tok.find('='); tok.rfind("--", 0) == 0 && eq != std::string::npos) {
                inline_val = tok.substr(eq + 1);
                tok = tok.substr(0, eq);
            }
            Flag* f = find(tok);
            if (!f) throw UsageError("The following argument was not expected: " + args[i]);
            f->seen = true;
            if (f->kind == Flag::Switch) {
                if (inline_val) throw UsageError(tok + " does not take a value");
                continue;
            }
            std::vector<std::string> got;
            if (inline_val) got.push_back(*inline_val);
            while (i + 1 < args.size() && !is_flag(args[i + 1]) &&
                   (got.empty() || f->kind == Flag::Multi))
                got.push_back(args[++i]);
            if (got.empty()) throw UsageError(tok + " requires an argument");
            if (f->kind == Flag::Value) f->values = {got.back()};
            for (const auto& g : got) {
                if (f->kind == Flag::Multi) f->values.push_back(g);
                if (f->kind == Flag::List) {
                    std::stringstream ss(g);
                    for (std::string part; std::getline(ss, part, ',');)
                        if (!part.empty()) f->values.push_back(part);
                }
            }
        }
        for (const auto& f : flags_)
            if (f.required && !f.seen) throw UsageError(f.names.front() + " is required");
        return true;
    }

    const Flag& get(const std::string& name) const {
        for (const auto& f : flags_)
            for (const auto& n : f.names)
                if (n == name) return f;
        throw std::logic_error("no flag " + name);
    }
    std::optional<std::string> str(const std::string& name) const {
        const Flag& f = get(name);
        if (f.values.empty()) return std::nullopt;
        return f.values.back();
    }
    std::optional<double> num(const std::string& name) const {
        const auto s = str(name);
        if (!s) return std::nullopt;
        try {
            return parse_double(*s);
        } catch (const std::exception&) {
            throw UsageError(name + ": '" + *s + "' is not a number");
        }
    }
    std::optional<int> integer(const std::string& name) const {
        const auto s = str(name);
        if (!s) return std::nullopt;
        int v = 0;
        const auto r = std::from_chars(s->data(), s->data() + s->size(), v);
        if (r.ec != std::errc{} || r.ptr != s->data() + s->size())
            throw UsageError(name + ": '" + *s + "' is not an integer");
        return v;
    }
    std::vector<double> nums(const std::string& name) const {
        std::vector<double> out;
        for (const auto& s : get(name).values) {
            try {
                out.push_back(parse_double(s));
            } catch (const std::exception&) {
                throw UsageError(name + ": '" + s + "' is not a number");
            }
        }
        return out;
    }
    bool on(const std::string& name) const { return get(name).seen; }

    void usage(std::ostream& os) const {
        os << name_ << ": " << help_ << "\nOptions:\n";
        for (const auto& f : flags_) {
            std::string names;
            for (const auto& n : f.names) names += (names.empty() ? "" : ",") + n;
            os << "  " << names << (f.required ? " (required)" : "") << "  " << f.help << '\n';
        }
    }
    const std::string& name() const { return name_; }
    const std::string& help() const { return help_; }

private:
    Command& add(std::vector<std::string> names, Flag::Kind kind, std::string help, bool required) {
        Flag f;
        f.names = std::move(names);
        f.kind = kind;
        f.help = std::move(help);
        f.required = required;
        flags_.push_back(std::move(f));
        return *this;
    }
    static bool is_flag(const std::string& s) { return s.size() > 2 && s.rfind("--", 0) == 0; }
    Flag* find(const std::string& tok) {
        for (auto& f : flags_)
            for (const auto& n : f.names)
                if (n == tok) return &f;
        return nullptr;
    }
    std::string name_, help_;
    std::vector<Flag> flags_;
};

// ---- shared helpers -------------------------------------------------------

NormKind norm_of(const std::string& token) {
    const auto k = parse_norm(token);
    if (!k) throw std::invalid_argument("unknown norm '" + token + "' (want l1, l2 or linf)");
    return *k;
}

std::vector<NormKind> norms_of(const std::vector<std::string>& tokens) {
    std::vector<NormKind> out;
    for (const auto& t : tokens) out.push_back(norm_of(t));
    return out;
}

// alpha grid from..to by step, the endpoint clamped (step counted by lround)
std::vector<double> alpha_range(double from, double to, double step) {
    if (!(step > 0.0)) throw std::invalid_argument("--alpha-step must be positive");
    if (from > to) throw std::invalid_argument("--alpha-from exceeds --alpha-to");
    std::vector<double> out;
    const long count = std::lround((to - from) / step);
    for (long i = 0; i <= count; ++i) {
        const double a = from + static_cast<double>(i) * step;
        if (a <= to + step * 1e-9) out.push_back(a < to ? a : to);
    }
    return out;
}

void save_records(const std::string& path, const std::vector<SweepRecord>& recs) {
    std::ofstream f(path);
    if (!f) throw std::runtime_error("cannot open output file: " + path);
    write_sweep_csv(f, recs);
    if (!f) throw std::runtime_error("failed writing output file: " + path);
}

std::string two_decimals(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.2f", v);
    return b;
}

// ---- subcommands ----------------------------------------------------------

int run_cmd(const Command& c) {
    SweepPlan plan;
    plan.graphs = {*c.str("--graph")};
    plan.alphas = {c.num("--alpha").value_or(0.85)};
    plan.tolerances = {c.num("--tolerance").value_or(1e-6)};
    plan.norms = {norm_of(c.str("--norm").value_or("l1"))};
    plan.max_iterations = c.integer("--max-iter").value_or(500);
    plan.repeats = c.integer("--repeat").value_or(5);
    plan.fuse = false; // one cell: time it as the reference does
    const auto recs = run_sweep(plan);
    std::cout << sweep_csv_row(recs.front()) << '\n';
    return recs.front().converged ? 0 : 3;
}

enum class Sweep { Damping, Tolerance, Norms };

int sweep_cmd(const Command& c, Sweep kind) {
    SweepPlan plan;
    for (const auto& g : c.get("--graphs").values) plan.graphs.emplace_back(g);
    plan.repeats = c.integer("--repeat").value_or(5);
    plan.max_iterations = c.integer("--max-iter").value_or(500);
    plan.fuse = !c.on("--per-cell-timing");
    const std::vector<double> tol_grid = c.nums("--tol-grid");
    const std::vector<std::string> norm_tokens = c.get("--norms").values;
    const std::vector<NormKind> every_norm(all_norms.begin(), all_norms.end());
    if (kind == Sweep::Damping) {
        const auto from = c.num("--alpha-from"), to = c.num("--alpha-to"), step = c.num("--alpha-step");
        if (from || to || step) {
            if (!(from && to && step))
                throw std::invalid_argument("--alpha-from/--alpha-to/--alpha-step must be given together");
            plan.alphas = alpha_range(*from, *to, *step);
        } else {
            const auto a = c.num("--alpha");
            plan.alphas = a ? std::vector<double>{*a} : default_damping_grid();
        }
        plan.tolerances = tol_grid.empty() ? std::vector<double>{c.num("--tolerance").value_or(1e-6)} : tol_grid;
        plan.norms = norm_tokens.empty() ? std::vector<NormKind>{NormKind::L1} : norms_of(norm_tokens);
    } else {
        plan.alphas = {c.num("--alpha").value_or(0.85)};
        if (kind == Sweep::Tolerance)
            plan.tolerances = tol_grid.empty() ? default_tolerance_grid() : tol_grid;
        else
            plan.tolerances =
                tol_grid.empty() ? std::vector<double>{c.num("--tolerance").value_or(1e-6)} : tol_grid;
        plan.norms = norm_tokens.empty() ? every_norm : norms_of(norm_tokens);
    }
    std::cout << sweep_csv_header << '\n';
    const auto recs = run_sweep(plan, &std::cout);
    save_records(*c.str("--csv"), recs);
    return 0;
}

// sweep CSV -> approaches (norms) x cases (graph, alpha, tolerance) of one metric
MeasurementMatrix measurements(const CsvTable& t, const std::string& metric) {
    const std::size_t cn = t.column("norm"), cm = t.column(metric), cg = t.column("graph"),
                      ca = t.column("alpha"), ct = t.column("tolerance");
    const bool conv = t.has_column("converged");
    const std::size_t cc = conv ? t.column("converged") : 0;
    std::map<std::pair<std::string, std::string>, double> cell;
    std::set<std::string> approaches, cases;
    std::size_t unconverged = 0;
    for (const auto& row : t.rows) {
        const std::string who = row[cn];
        const std::string where = row[cg] + " a=" + row[ca] + " t=" + row[ct];
        if (!cell.emplace(std::make_pair(who, where), parse_double(row[cm])).second)
            throw std::runtime_error("duplicate cell for " + who + ", " + where);
        approaches.insert(who);
        cases.insert(where);
        if (conv && row[cc] == "false") ++unconverged;
    }
    MeasurementMatrix m;
    m.approaches.assign(approaches.begin(), approaches.end());
    m.cases.assign(cases.begin(), cases.end());
    std::string missing;
    for (const auto& a : m.approaches)
        for (const auto& w : m.cases) {
            const auto it = cell.find({a, w});
            if (it == cell.end()) missing += "\n  " + a + ", " + w;
            else m.values.push_back(it->second);
        }
    if (!missing.empty()) throw std::runtime_error("incomplete measurement matrix; missing cells:" + missing);
    if (unconverged)
        std::cerr << "warning: " << unconverged << " non-converged cell(s) included in ratio computation\n";
    return m;
}

int ratios_cmd(const Command& c) {
    const std::string metric = c.str("--metric").value_or("iterations");
    if (metric != "iterations" && metric != "time_ms")
        throw std::invalid_argument("--metric must be iterations or time_ms");
    const std::string input = *c.str("--input");
    std::ifstream in(input);
    if (!in) throw std::runtime_error("cannot open input file: " + input);
    const MeasurementMatrix m = measurements(read_csv(in), metric);
    const std::string which = c.str("--method").value_or("all");
    std::vector<RatioMethod> methods;
    if (which == "all") {
        methods.assign(all_ratio_methods.begin(), all_ratio_methods.end());
    } else if (const auto one = parse_ratio_method(which)) {
        methods.push_back(*one);
    } else {
        throw std::invalid_argument("unknown method '" + which +
                                    "' (want ratio-am, ratio-gm, ratio-hm, am-ratio, gm-ratio, hm-ratio or all)");
    }
    std::string head = "method,baseline";
    for (const auto& a : m.approaches) head += ",mean:" + a;
    for (const auto& a : m.approaches) head += ",ratio:" + a;
    std::cout << head << '\n';
    const std::string baseline = c.str("--baseline").value_or("l1");
    for (const RatioMethod method : methods) {
        const RatioTable t = compute_ratio_table(m, baseline, method);
        std::ostringstream line;
        line << ratio_method_name(method) << ',' << t.baseline;
        // only the mean-then-ratio family reports per-approach means
        for (const double mu : t.means) line << ',' << (is_mean_then_ratio(method) ? two_decimals(mu) : "");
        for (const double r : t.ratios) line << ',' << two_decimals(r);
        std::cout << line.str() << '\n';
    }
    return 0;
}

int estimate_cmd(const Command& c) {
    std::cout << estimate_iterations(*c.num("--alpha"), *c.num("--tolerance")) << '\n';
    return 0;
}

int chart_cmd(const Command& c) {
    const std::string input = *c.str("--input"), out_path = *c.str("--out");
    std::ifstream in(input);
    if (!in) throw std::runtime_error("cannot open input file: " + input);
    const CsvTable table = read_csv(in);
    ChartOptions opt;
    opt.x_column = *c.str("--x");
    opt.y_column = *c.str("--y");
    opt.series_column = c.str("--series").value_or("");
    opt.log_x = c.on("--log-x");
    opt.title = opt.y_column + " by " + opt.x_column;
    std::ostringstream svg;
    write_line_chart_svg(svg, table, opt);
    std::ofstream out(out_path);
    if (!out) throw std::runtime_error("cannot open output file: " + out_path);
    out << svg.str();
    if (!out) throw std::runtime_error("failed writing output file: " + out_path);
    return 0;
}

Command sweep_command(const std::string& name, const std::string& help, bool damping) {
    Command c(name, help);
    c.multi({"--graphs", "--graph"}, "input .mtx graph files", true)
        .value({"--csv"}, "output CSV path", true)
        .value({"--alpha"}, "damping factor");
    if (damping)
        c.value({"--alpha-from"}, "damping grid start")
            .value({"--alpha-to"}, "damping grid end")
            .value({"--alpha-step"}, "damping grid step");
    c.value({"--tolerance"}, "convergence tolerance")
        .list({"--tol-grid"}, "comma-separated tolerance grid override")
        .list({"--norms", "--norm"}, "convergence norms (l1, l2, linf)")
        .value({"--repeat"}, "timed repeats per cell")
        .value({"--max-iter"}, "iteration cap")
        .flag({"--per-cell-timing"}, "run and time every cell on its own (reference time_ms semantics)");
    return c;
}

} // namespace

int main(int argc, char** argv) {
    using Handler = std::function<int(const Command&)>;
    std::vector<std::pair<Command, Handler>> cmds;
    {
        Command c("run", "run PageRank once and print one CSV record");
        c.value({"--graph"}, "input .mtx graph file", true)
            .value({"--alpha"}, "damping factor")
            .value({"--tolerance"}, "convergence tolerance")
            .value({"--norm"}, "convergence norm (l1, l2, linf)")
            .value({"--max-iter"}, "iteration cap")
            .value({"--repeat"}, "timed repeats");
        cmds.emplace_back(c, run_cmd);
    }
    cmds.emplace_back(sweep_command("sweep-damping", "sweep the damping factor 0.50 .. 1.00 in steps of 0.05", true),
                      [](const Command& c) { return sweep_cmd(c, Sweep::Damping); });
    cmds.emplace_back(sweep_command("sweep-tolerance", "sweep the tolerance 1e0 .. 1e-10 under all three norms", false),
                      [](const Command& c) { return sweep_cmd(c, Sweep::Tolerance); });
    cmds.emplace_back(sweep_command("compare-norms", "run all three norms at fixed alpha and tolerance", false),
                      [](const Command& c) { return sweep_cmd(c, Sweep::Norms); });
    {
        Command c("ratios", "aggregate a sweep CSV into composite ratios");
        c.value({"--input"}, "sweep CSV to aggregate", true)
            .value({"--metric"}, "iterations or time_ms")
            .value({"--baseline"}, "baseline approach (norm)")
            .value({"--method"}, "ratio-am, ratio-gm, ratio-hm, am-ratio, gm-ratio, hm-ratio or all");
        cmds.emplace_back(c, ratios_cmd);
    }
    {
        Command c("estimate", "estimated iterations to converge at (alpha, tau)");
        c.value({"--alpha"}, "damping factor in (0, 1)", true).value({"--tolerance"}, "tolerance in (0, 1)", true);
        cmds.emplace_back(c, estimate_cmd);
    }
    {
        Command c("chart", "emit an SVG line chart from a sweep CSV");
        c.value({"--input"}, "CSV to plot", true)
            .value({"--x"}, "x column", true)
            .value({"--y"}, "y column", true)
            .value({"--series"}, "series column (one line per value)")
            .flag({"--log-x"}, "log10-scale the x axis")
            .value({"--out"}, "output SVG path", true);
        cmds.emplace_back(c, chart_cmd);
    }
    auto overview = [&](std::ostream& os) {
        os << "pagerank-lab (B200): PageRank parameter-study toolkit\nSubcommands:\n";
        for (const auto& [c, h] : cmds) os << "  " << c.name() << "  " << c.help() << '\n';
    };
    const std::vector<std::string> args(argv + 1, argv + argc);
    if (args.empty()) {
        overview(std::cerr);
        std::cerr << "A subcommand is required\n";
        return 2;
    }
    if (args[0] == "-h" || args[0] == "--help") {
        overview(std::cout);
        return 0;
    }
    for (auto& [cmd, handler] : cmds) {
        if (cmd.name() != args[0]) continue;
        try {
            if (!cmd.parse({args.begin() + 1, args.end()})) {
                cmd.usage(std::cout);
                return 0;
            }
            return handler(cmd);
        } catch (const UsageError& e) {
            std::cerr << e.what() << '\n';
            cmd.usage(std::cerr);
            return 2;
        } catch (const std::invalid_argument& e) {
            std::cerr << "error: " << e.what() << '\n';
            return 2;
        } catch (const std::exception& e) {
            std::cerr << "error: " << e.what() << '\n';
            return 1;
        }
    }
    std::cerr << "The following argument was not expected: " << args[0] << '\n';
    overview(std::cerr);
    return 2;
}
