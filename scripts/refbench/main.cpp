// Report emitter of the reference benchmark: the reference's
// own bench.cpp (bench_cfar / bench_pipeline and its text / CSV / JSON
// renderers, compiled unchanged where it lies) linked either against the B200
// drop-in (libuwbvital.so: every timed call runs on the GPU) or against the
// reference library itself (oracle/_ref), so both reports share one schema.
// The B200 build (REFBENCH_GPU) adds the GPU columns of gpu_columns.hpp.
//
//   refbench {cfar|pipeline} {text|csv|json} [repetitions]
//   refbench parse {cfar|pipeline} {csv|json} FILE   (reference parsers;
//       prints the rows it read - the augmented CSV is cut to the reference's
//       columns first, the augmented JSON is read as it is)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "uwbvital/bench.hpp"
#include "uwbvital/synth.hpp"
#ifdef REFBENCH_GPU
#include "gpu_columns.hpp"
#endif

namespace {

std::string read_file(const char* path) {
    std::ifstream f(path);
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

// keep the first n comma-separated fields of every line (no quoted commas in
// the leading columns of either schema)
std::string cut_csv(const std::string& csv, std::size_t n) {
    std::istringstream in(csv);
    std::string ln, out;
    while (std::getline(in, ln)) {
        std::size_t pos = 0, k = 0;
        bool quoted = false;
        for (; pos < ln.size(); ++pos) {
            if (ln[pos] == '"') quoted = !quoted;
            if (ln[pos] == ',' && !quoted && ++k == n) break;
        }
        out += ln.substr(0, pos) + "\n";
    }
    return out;
}

int parse_mode(const std::string& mode, const std::string& fmt, const char* path) {
    const std::string text = read_file(path);
    if (mode == "cfar") {
        const auto r = fmt == "csv" ? uwbvital::cfar_report_from_csv(cut_csv(text, 7))
                                    : uwbvital::cfar_report_from_json(text);
        for (const auto& row : r.rows)
            std::printf("%d %d %.9g %.9g %.9g\n", row.guard, row.background, row.naive.mean_s, row.integral.mean_s,
                        row.ratio);
    } else {
        const auto r = fmt == "csv" ? uwbvital::pipeline_report_from_csv(cut_csv(text, 5))
                                    : uwbvital::pipeline_report_from_json(text);
        for (const auto& row : r.rows)
            std::printf("%s|%.9g|%.9g\n", row.name.c_str(), row.naive ? row.naive->mean_s : -1.0,
                        row.integral ? row.integral->mean_s : -1.0);
    }
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cfar";
    const std::string fmt = argc > 2 ? argv[2] : "text";
    try {
        if (mode == "parse") {
            if (argc < 5) {
                std::fprintf(stderr, "usage: refbench parse {cfar|pipeline} {csv|json} FILE\n");
                return 2;
            }
            return parse_mode(argv[2], argv[3], argv[4]);
        }
        const std::size_t reps = argc > 3 ? static_cast<std::size_t>(std::atoi(argv[3])) : 10;
        if (mode == "cfar") {
            uwbvital::BenchSpec spec; // 1024 x 600, Table I grid, pfa 1e-3 (bench.hpp:14-23)
            spec.repetitions = reps;
            const auto r = uwbvital::bench_cfar(spec, 1, 1);
            std::string out = fmt == "csv" ? uwbvital::to_csv(r) : fmt == "json" ? uwbvital::to_json(r)
                                                                                 : uwbvital::render_text(r);
#ifdef REFBENCH_GPU
            std::vector<refbench::DevTimes> dev;
            std::vector<double> frac, e2e;
            std::string src;
            const double peak = refbench::hbm_peak_gbs(&src);
            const double cells = static_cast<double>(spec.map_rows * spec.map_cols);
            for (const auto& [g, b] : spec.param_grid) {
                dev.push_back(refbench::time_cfar_device(spec.map_rows, spec.map_cols, g, b, spec.pfa, reps));
                frac.push_back(17.0 * cells / dev.back().integral_s / 1e9 / peak);
            }
            for (const auto& row : r.rows) e2e.push_back(row.integral.mean_s);
            out = fmt == "csv"    ? refbench::cfar_csv_with_gpu(out, dev, frac)
                  : fmt == "json" ? refbench::cfar_json_with_gpu(out, dev, frac, src)
                                  : refbench::cfar_text_with_gpu(out, spec.param_grid, dev, frac, e2e);
#endif
            std::fputs(out.c_str(), stdout);
        } else {
            const uwbvital::Scene scene = uwbvital::generate_scene(uwbvital::SceneConfig{});
            const uwbvital::PipelineConfig cfg{};
            const auto r = uwbvital::bench_pipeline(scene.frame, cfg, reps, 2, 1);
            std::string out = fmt == "csv" ? uwbvital::to_csv(r) : fmt == "json" ? uwbvital::to_json(r)
                                                                                 : uwbvital::render_text(r);
#ifdef REFBENCH_GPU
            const auto& f = scene.frame;
            const std::size_t m = f.data.rows(), n = f.data.cols();
            const std::vector<double> frame(f.data.values().begin(), f.data.values().end());
            const auto dev = refbench::time_detect_device(
                frame, m, n, f.fast_rate, f.prf, cfg.mean_filter_window, cfg.fft_length, cfg.band_low_hz,
                cfg.band_high_hz, static_cast<int>(cfg.cfar.guard_radius), static_cast<int>(cfg.cfar.background_radius),
                cfg.cfar.pfa, reps);
            out = fmt == "csv"    ? refbench::pipeline_csv_with_gpu(out, dev)
                  : fmt == "json" ? refbench::pipeline_json_with_gpu(out, dev)
                                  : refbench::pipeline_text_with_gpu(out, dev);
#endif
            std::fputs(out.c_str(), stdout);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "refbench: %s\n", e.what());
        return 1;
    }
    return 0;
}
