// Report emitter of the reference benchmark: the reference's
// own bench.cpp (bench_cfar / bench_pipeline and its text / CSV / JSON
// renderers, compiled unchanged where it lies) linked either against the B200
// drop-in (libuwbvital.so: every timed call runs on the GPU) or against the
// reference library itself (oracle/_ref), so both reports share one schema.
//
//   refbench {cfar|pipeline} {text|csv|json} [repetitions]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "uwbvital/bench.hpp"
#include "uwbvital/synth.hpp"

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "cfar";
    const std::string fmt = argc > 2 ? argv[2] : "text";
    const std::size_t reps = argc > 3 ? static_cast<std::size_t>(std::atoi(argv[3])) : 10;
    try {
        if (mode == "cfar") {
            uwbvital::BenchSpec spec; // 1024 x 600, Table I grid, pfa 1e-3 (bench.hpp:14-23)
            spec.repetitions = reps;
            const auto r = uwbvital::bench_cfar(spec, 1, 1);
            const std::string out = fmt == "csv" ? uwbvital::to_csv(r) : fmt == "json" ? uwbvital::to_json(r)
                                                                                      : uwbvital::render_text(r);
            std::fputs(out.c_str(), stdout);
        } else {
            const uwbvital::Scene scene = uwbvital::generate_scene(uwbvital::SceneConfig{});
            const auto r = uwbvital::bench_pipeline(scene.frame, uwbvital::PipelineConfig{}, reps, 2, 1);
            const std::string out = fmt == "csv" ? uwbvital::to_csv(r) : fmt == "json" ? uwbvital::to_json(r)
                                                                                      : uwbvital::render_text(r);
            std::fputs(out.c_str(), stdout);
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "refbench: %s\n", e.what());
        return 1;
    }
    return 0;
}
