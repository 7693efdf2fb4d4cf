// GPU columns for the reference benchmark reports: see gpu_columns.hpp.
#include "gpu_columns.hpp"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>

#include <json.hpp>

#include "uwbvital_b200.h"

namespace refbench {

namespace {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void check(uwb_status s, const char* what) {
    if (s != UWB_OK) throw std::runtime_error(std::string(what) + ": " + uwb_last_error());
}

struct Dev {
    void* p = nullptr;
    explicit Dev(size_t bytes) { check(cudaMalloc(&p, bytes ? bytes : 16), "cudaMalloc"); }
    ~Dev() { cudaFree(p); }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// mean seconds per call of fn() over reps calls, CUDA events on `s`
template <typename F>
double event_time(F&& fn, std::size_t reps, cudaStream_t s) {
    fn(); // warm-up
    check(cudaStreamSynchronize(s), "warm-up");
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (std::size_t i = 0; i < reps; ++i) fn();
    cudaEventRecord(b, s);
    check(cudaEventSynchronize(b), "timed calls");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / 1e3 / static_cast<double>(reps);
}

std::string fmt(double v) {
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%.9g", v);
    return buf;
}

std::vector<std::string> lines_of(const std::string& text) {
    std::vector<std::string> out;
    std::istringstream in(text);
    std::string ln;
    while (std::getline(in, ln))
        if (!ln.empty()) out.push_back(ln);
    return out;
}

// Device-resident CFAR of one map with the drop-in's outputs.
struct CfarDev {
    uwb_map_batch batch{};
    uwb_cfar_params params{};
    uwb_cfar_outputs out{};
    std::unique_ptr<Dev> alpha, ws, bits, mask, thr, dets, cnt, bad;
    uint64_t ws_bytes = 0;
    CfarDev(const double* map_dev, std::size_t rows, std::size_t cols, int g, int b, double pfa) {
        batch.maps = map_dev;
        batch.dtype = UWB_F64;
        batch.n_maps = 1;
        batch.rows = rows;
        batch.cols = cols;
        batch.ld = cols;
        batch.map_stride = rows * cols;
        params = uwb_cfar_params{g, g, b, b, pfa};
        const uint64_t n_int = uwb_interior_train_count(&params);
        std::vector<double> a(n_int + 1);
        check(uwb_alpha_table(&params, a.data(), a.size()), "uwb_alpha_table");
        alpha = std::make_unique<Dev>(sizeof(double) * a.size());
        check(cudaMemcpy(alpha->p, a.data(), sizeof(double) * a.size(), cudaMemcpyHostToDevice), "alpha H2D");
        const uint64_t cap = rows * cols;
        ws_bytes = uwb_dev_cfar2d_workspace(&batch, &params, UWB_SAT_GLOBAL, 0, cap);
        ws = std::make_unique<Dev>(ws_bytes);
        const uint64_t words = (cols + 31) / 32;
        bits = std::make_unique<Dev>(4 * words * rows);
        mask = std::make_unique<Dev>(rows * cols);
        thr = std::make_unique<Dev>(8 * rows * cols);
        dets = std::make_unique<Dev>(sizeof(uwb_detection) * cap);
        cnt = std::make_unique<Dev>(8);
        bad = std::make_unique<Dev>(16);
        out.mask_bits = bits->as<uint32_t>();
        out.words_per_row = words;
        out.mask_map_stride = words * rows;
        out.mask_u8 = mask->as<uint8_t>();
        out.thresholds = thr->as<double>();
        out.dets = dets->as<uwb_detection>();
        out.det_capacity = cap;
        out.det_counts = cnt->as<uint64_t>();
        out.first_bad = bad->as<uint64_t>();
    }
    void run(bool naive, cudaStream_t s) {
        check(uwb_dev_cfar2d(&batch, &params, alpha->as<double>(), UWB_SAT_GLOBAL, 0, &out, ws->p, ws_bytes,
                             naive ? 8u : 0u, s),
              "uwb_dev_cfar2d");
    }
};

} // namespace

double hbm_peak_gbs(std::string* source) {
    for (const char* path : {"MEASURED_PEAKS.json", "../MEASURED_PEAKS.json"}) {
        std::ifstream f(path);
        if (!f) continue;
        try {
            const auto j = nlohmann::json::parse(f);
            if (j.contains("hbm_gbs")) {
                if (source) *source = "measured (MEASURED_PEAKS.json hbm_gbs)";
                return j.at("hbm_gbs").get<double>();
            }
        } catch (...) {
        }
    }
    if (source) *source = "fallback (B200_PROFILING.md 6.65 TB/s)";
    return 6650.0;
}

DevTimes time_cfar_device(std::size_t rows, std::size_t cols, int guard, int background, double pfa,
                          std::size_t reps) {
    std::mt19937_64 gen(12345);
    std::exponential_distribution<double> ex(1.0);
    std::vector<double> host(rows * cols);
    for (auto& v : host) v = ex(gen);
    Dev map(8 * host.size());
    check(cudaMemcpy(map.p, host.data(), 8 * host.size(), cudaMemcpyHostToDevice), "map H2D");
    cudaStream_t s;
    check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    CfarDev c(map.as<double>(), rows, cols, guard, background, pfa);
    DevTimes t;
    t.naive_s = event_time([&] { c.run(true, s); }, reps, s);
    t.integral_s = event_time([&] { c.run(false, s); }, reps, s);
    cudaStreamDestroy(s);
    return t;
}

DetectDevTimes time_detect_device(const std::vector<double>& frame, std::size_t m, std::size_t n, double fast_rate,
                                  double prf, std::size_t mean_filter_window, std::size_t fft_length,
                                  double band_low, double band_high, int guard, int background, double pfa,
                                  std::size_t reps) {
    cudaStream_t s;
    check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    Dev rec(8 * m * n);
    check(cudaMemcpy(rec.p, frame.data(), 8 * m * n, cudaMemcpyHostToDevice), "record H2D");
    uwb_pipeline_config cfg{};
    cfg.mean_filter_window = mean_filter_window;
    cfg.fft_length = fft_length;
    cfg.band_low_hz = band_low;
    cfg.band_high_hz = band_high;
    cfg.cfar = uwb_cfar_params{guard, guard, background, background, pfa};
    cfg.mean_filter_mode = 0;
    cfg.normalization_epsilon = 1e-12;
    DetectDevTimes t;
    uint64_t kept = 0;
    uwb_cfar_outputs none{};
    for (int backend : {UWB_NAIVE, UWB_INTEGRAL}) {
        cfg.backend = backend;
        check(uwb_dev_detect_batch(nullptr, UWB_F64, 0, m, n, fast_rate, prf, &cfg, nullptr, &kept, &none, nullptr, 0,
                                   0, s),
              "detect plan");
        const uint64_t cap = m * kept;
        const uint64_t ws_bytes = uwb_dev_detect_batch_workspace(1, m, n, prf, &cfg, cap);
        Dev ws(ws_bytes), band(8 * m * kept), bits(4 * ((kept + 31) / 32) * m), dets(sizeof(uwb_detection) * cap),
            cnt(8), bad(16);
        uwb_cfar_outputs o{};
        o.mask_bits = bits.as<uint32_t>();
        o.words_per_row = (kept + 31) / 32;
        o.mask_map_stride = o.words_per_row * m;
        o.dets = dets.as<uwb_detection>();
        o.det_capacity = cap;
        o.det_counts = cnt.as<uint64_t>();
        o.first_bad = bad.as<uint64_t>();
        const double total = event_time(
            [&] {
                check(uwb_dev_detect_batch(rec.p, UWB_F64, 1, m, n, fast_rate, prf, &cfg, band.as<double>(), &kept, &o,
                                           ws.p, ws_bytes, 0, s),
                      "uwb_dev_detect_batch");
            },
            reps, s);
        // the threshold step alone on the band map (the drop-in's cfar2d outputs)
        CfarDev c(band.as<double>(), m, kept, guard, background, pfa);
        const double thr = event_time([&] { c.run(backend == UWB_NAIVE, s); }, reps, s);
        if (backend == UWB_NAIVE) {
            t.total.naive_s = total;
            t.threshold.naive_s = thr;
        } else {
            t.total.integral_s = total;
            t.threshold.integral_s = thr;
        }
    }
    cudaStreamDestroy(s);
    return t;
}

std::string cfar_csv_with_gpu(const std::string& ref_csv, const std::vector<DevTimes>& dev,
                              const std::vector<double>& hbm_frac) {
    const auto ls = lines_of(ref_csv);
    std::string out = ls.at(0) + ",dev_naive_s,dev_ii_s,dev_ratio,dev_ii_hbm_frac\n";
    for (std::size_t i = 1; i < ls.size(); ++i) {
        const DevTimes& d = dev.at(i - 1);
        out += ls[i] + "," + fmt(d.naive_s) + "," + fmt(d.integral_s) + "," + fmt(d.naive_s / d.integral_s) + "," +
               fmt(hbm_frac.at(i - 1)) + "\n";
    }
    return out;
}

std::string cfar_json_with_gpu(const std::string& ref_json, const std::vector<DevTimes>& dev,
                               const std::vector<double>& hbm_frac, const std::string& peak_source) {
    auto j = nlohmann::ordered_json::parse(ref_json);
    auto& rows = j.at("rows");
    for (std::size_t i = 0; i < rows.size(); ++i) {
        const DevTimes& d = dev.at(i);
        rows[i]["dev_naive_s"] = d.naive_s;
        rows[i]["dev_ii_s"] = d.integral_s;
        rows[i]["dev_ratio"] = d.naive_s / d.integral_s;
        rows[i]["dev_ii_hbm_frac"] = hbm_frac.at(i);
        rows[i]["e2e_ii_s"] = rows[i].at("ii_mean_s");
    }
    j["gpu_note"] = "dev_*: device-resident calls through the C ABI timed with CUDA events; dev_ii_hbm_frac: 17 "
                    "B/cell (map in, threshold map + mask out) over dev_ii_s, HBM peak " +
                    peak_source + "; e2e_ii_s / *_mean_s: the drop-in call from host buffers";
    return j.dump(2) + "\n";
}

std::string cfar_text_with_gpu(const std::string& ref_text, const std::vector<std::pair<int, int>>& grid,
                               const std::vector<DevTimes>& dev, const std::vector<double>& hbm_frac,
                               const std::vector<double>& e2e_ii_s) {
    std::string out = ref_text;
    out += "GPU columns (device-resident, CUDA events)\n";
    out += "guard  bkgnd  dev naive (s)   dev ii (s)      dev ratio  ii HBM frac  e2e ii (s)\n";
    for (std::size_t i = 0; i < dev.size(); ++i) {
        char line[200];
        std::snprintf(line, sizeof(line), "%-6d %-6d %-15.9f %-15.9f %6.2f:1   %-12.4f %-12.9f\n", grid.at(i).first,
                      grid.at(i).second, dev[i].naive_s, dev[i].integral_s, dev[i].naive_s / dev[i].integral_s,
                      hbm_frac.at(i), e2e_ii_s.at(i));
        out += line;
    }
    return out;
}

namespace {
// device columns of the pipeline rows (bench.cpp:302-308): {naive, integral} or -1 for none
void pipeline_dev_row(std::size_t i, const DetectDevTimes& d, double& ca, double& ii) {
    ca = ii = -1.0;
    if (i == 2) ca = d.threshold.naive_s;
    if (i == 3) ii = d.threshold.integral_s;
    if (i == 4) {
        ca = d.total.naive_s;
        ii = d.total.integral_s;
    }
}
} // namespace

std::string pipeline_csv_with_gpu(const std::string& ref_csv, const DetectDevTimes& dev) {
    const auto ls = lines_of(ref_csv);
    std::string out = ls.at(0) + ",dev_ca_s,dev_ii_s\n";
    for (std::size_t i = 1; i < ls.size(); ++i) {
        double ca, ii;
        pipeline_dev_row(i - 1, dev, ca, ii);
        out += ls[i] + "," + (ca >= 0 ? fmt(ca) : "") + "," + (ii >= 0 ? fmt(ii) : "") + "\n";
    }
    return out;
}

std::string pipeline_json_with_gpu(const std::string& ref_json, const DetectDevTimes& dev) {
    auto j = nlohmann::ordered_json::parse(ref_json);
    auto& rows = j.at("rows");
    for (std::size_t i = 0; i < rows.size(); ++i) {
        double ca, ii;
        pipeline_dev_row(i, dev, ca, ii);
        rows[i]["dev_ca_s"] = ca >= 0 ? nlohmann::ordered_json(ca) : nlohmann::ordered_json(nullptr);
        rows[i]["dev_ii_s"] = ii >= 0 ? nlohmann::ordered_json(ii) : nlohmann::ordered_json(nullptr);
    }
    j["gpu_note"] = "dev_*: device-resident detect() / cfar2d through the C ABI, CUDA events";
    return j.dump(2) + "\n";
}

std::string pipeline_text_with_gpu(const std::string& ref_text, const DetectDevTimes& dev) {
    std::string out = ref_text;
    char buf[512];
    std::snprintf(buf, sizeof(buf),
                  "GPU columns (device-resident, CUDA events)\n"
                  "%-34s %-26s %-26s\n%-34s %-26.9f %-26s\n%-34s %-26s %-26.9f\n%-34s %-26.9f %-26.9f\n",
                  "step", "CA-CFAR dev (s)", "II CA-CFAR dev (s)", "Signal Threshold (CA-CFAR)", dev.threshold.naive_s,
                  "-", "Signal Threshold (II CA-CFAR)", "-", dev.threshold.integral_s, "Total", dev.total.naive_s,
                  dev.total.integral_s);
    out += buf;
    return out;
}

} // namespace refbench
