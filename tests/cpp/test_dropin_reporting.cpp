// test_dropin_reporting.cpp — the drop-in next to the reference's own host-only
// reporting headers (stats.hpp: mean-ratio tables, csv.hpp, chart.hpp), as a
// reference caller would combine them: the GPU path's names and the
// reporting names resolve without ambiguity.  Host-only at run time (no GPU
// call): the sweep CSV rows this header writes are read back by csv.hpp and
// fed to the ratio tables and the chart writer.
#include <pagerank_b200/dropin.hpp>
#include <pagerank_lab/chart.hpp>
#include <pagerank_lab/csv.hpp>
#include <pagerank_lab/stats.hpp>

#include <cmath>
#include <cstdio>
#include <sstream>
#include <vector>

using namespace pagerank_lab;

int main() {
    // sweep records as run_sweep returns them, written with the drop-in
    std::vector<SweepRecord> recs;
    for (double a : {0.75, 0.85, 0.95})
        recs.push_back(SweepRecord{"g", 10, 20, a, 1e-6, NormKind::L1, int(a * 20), true, a * 3.0, 0.0});
    std::ostringstream os;
    write_sweep_csv(os, recs);
    // the reference's csv reader and mean-ratio reporting on them
    const auto lines = os.str();
    std::istringstream in(lines);
    std::string header;
    std::getline(in, header);
    const auto fields = split_csv_line(header);
    MeasurementMatrix m;
    m.approaches = {"cpu", "b200"};
    m.cases = {"a", "b", "c"};
    m.values = {3.0, 6.0, 9.0, 0.01, 0.02, 0.03};
    const RatioTable t = compute_ratio_table(m, "cpu", RatioMethod::GmRatio);
    const double gm = mean(MeanKind::Geometric, std::vector<double>{1.0, 4.0});
    std::ostringstream csv;
    write_csv_row(csv, std::vector<std::string>{"x", format_double(0.5)});
    const bool ok = fields.size() == 10 && std::abs(gm - 2.0) < 1e-12 && t.ratios.size() == 2 && std::abs(t.ratio_of("cpu") - 1.0) < 1e-12 &&
                    parse_norm("l2") == NormKind::L2 && estimate_iterations(0.85, 1e-6) == 85;
    std::printf("%s\n", ok ? "PASS" : "FAIL");
    return ok ? 0 : 1;
}
