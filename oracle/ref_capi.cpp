// TEST INFRASTRUCTURE ONLY (oracle/): a C shim over the REFERENCE library,
// compiled together with the unmodified reference sources
// /root/reference/proj/src/{sat,cfar,pipeline,synth}.cpp by oracle/Makefile into
// oracle/_ref/libuwbref.so. The namespace is renamed at build time
// (-Duwbvital=uwbvital_ref) so the reference links beside the B200 drop-in.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load this library, and only as the checker / the
// timed CPU baseline.
//
// Every function returns an error code: 0 ok, 1 DimensionError, 2 InputError,
// 3 ParameterError, 4 BoundsError, 5 ConfigurationError, 9 other; the
// exception text is copied into errbuf.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "uwbvital/cfar.hpp"
#include "uwbvital/errors.hpp"
#include "uwbvital/frame_io.hpp"
#include "uwbvital/pipeline.hpp"
#include "uwbvital/sat.hpp"
#include "uwbvital/synth.hpp"

namespace R = uwbvital;

namespace {

void put_msg(char* buf, std::size_t len, const char* msg) {
    if (!buf || len == 0) return;
    std::strncpy(buf, msg, len - 1);
    buf[len - 1] = '\0';
}

template <typename F>
int guarded(char* errbuf, std::size_t errlen, F&& f) {
    try {
        f();
        put_msg(errbuf, errlen, "");
        return 0;
    } catch (const R::DimensionError& e) {
        put_msg(errbuf, errlen, e.what());
        return 1;
    } catch (const R::InputError& e) {
        put_msg(errbuf, errlen, e.what());
        return 2;
    } catch (const R::ParameterError& e) {
        put_msg(errbuf, errlen, e.what());
        return 3;
    } catch (const R::BoundsError& e) {
        put_msg(errbuf, errlen, e.what());
        return 4;
    } catch (const R::ConfigurationError& e) {
        put_msg(errbuf, errlen, e.what());
        return 5;
    } catch (const R::FormatError& e) {
        put_msg(errbuf, errlen, e.what());
        return 7;
    } catch (const std::exception& e) {
        put_msg(errbuf, errlen, e.what());
        return 9;
    }
}

R::Matrix to_matrix(const double* p, std::size_t rows, std::size_t cols) {
    R::Matrix m(rows, cols);
    if (rows * cols) std::memcpy(m.values().data(), p, sizeof(double) * rows * cols);
    return m;
}

void from_matrix(const R::Matrix& m, double* out) {
    if (m.size()) std::memcpy(out, m.values().data(), sizeof(double) * m.size());
}

R::CfarParams make_params(int g, int b, double pfa) {
    R::CfarParams p;
    p.guard_radius = g;
    p.background_radius = b;
    p.pfa = pfa;
    return p;
}

void export_result(const R::DetectionResult& r, std::uint8_t* mask, double* thr,
                   std::uint64_t* n_det, std::uint64_t det_cap, std::uint64_t* det_rows,
                   std::uint64_t* det_cols, double* det_val, double* det_thr) {
    if (mask && r.mask.size()) std::memcpy(mask, r.mask.values().data(), r.mask.size());
    if (thr) from_matrix(r.threshold_map, thr);
    *n_det = r.detections.size();
    const std::size_t n = std::min<std::size_t>(r.detections.size(), det_cap);
    for (std::size_t i = 0; i < n; ++i) {
        const R::Detection& d = r.detections[i];
        if (det_rows) det_rows[i] = d.row;
        if (det_cols) det_cols[i] = d.col;
        if (det_val) det_val[i] = d.value;
        if (det_thr) det_thr[i] = d.threshold;
    }
}

R::RadarFrame make_frame(const double* data, std::size_t m, std::size_t n, double fast_rate,
                         double prf) {
    R::RadarFrame f;
    f.data = to_matrix(data, m, n);
    f.fast_rate = fast_rate;
    f.prf = prf;
    return f;
}

} // namespace

extern "C" {

int uwbref_build_sat(const double* src, std::uint64_t rows, std::uint64_t cols, double* table,
                     char* errbuf, std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const R::SummedAreaTable sat = R::build_sat(to_matrix(src, rows, cols));
        from_matrix(sat.table(), table);
    });
}

int uwbref_region_sum(const double* src, std::uint64_t rows, std::uint64_t cols,
                      std::uint64_t r0, std::uint64_t r1, std::uint64_t c0, std::uint64_t c1,
                      double* out, char* errbuf, std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const R::SummedAreaTable sat = R::build_sat(to_matrix(src, rows, cols));
        *out = sat.region_sum(r0, r1, c0, c1);
    });
}

int uwbref_alpha_factor(std::uint64_t n_train, double pfa, double* out, char* errbuf,
                        std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] { *out = R::alpha_factor(n_train, pfa); });
}

int uwbref_interior_train_count(int g, int b, std::uint64_t* out) {
    *out = make_params(g, b, 0.5).interior_train_count();
    return 0;
}

// out: outer r0 r1 c0 c1, guard r0 r1 c0 c1, n_train
int uwbref_training_window(int g, int b, double pfa, std::uint64_t row, std::uint64_t col,
                           std::uint64_t rows, std::uint64_t cols, std::uint64_t* out,
                           char* errbuf, std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const R::TrainingWindow w = R::training_window(make_params(g, b, pfa), row, col, rows, cols);
        out[0] = w.outer.r0; out[1] = w.outer.r1; out[2] = w.outer.c0; out[3] = w.outer.c1;
        out[4] = w.guard.r0; out[5] = w.guard.r1; out[6] = w.guard.c0; out[7] = w.guard.c1;
        out[8] = w.n_train;
    });
}

// backend: 0 naive, 1 integral image
int uwbref_cfar2d(int backend, const double* map, std::uint64_t rows, std::uint64_t cols, int g,
                  int b, double pfa, unsigned threads, std::uint8_t* mask, double* thr,
                  std::uint64_t* n_det, std::uint64_t det_cap, std::uint64_t* det_rows,
                  std::uint64_t* det_cols, double* det_val, double* det_thr, char* errbuf,
                  std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const R::Matrix m = to_matrix(map, rows, cols);
        const R::CfarParams p = make_params(g, b, pfa);
        const R::DetectionResult r =
            backend == 0 ? R::cfar2d_naive(m, p, threads) : R::cfar2d_integral(m, p, threads);
        export_result(r, mask, thr, n_det, det_cap, det_rows, det_cols, det_val, det_thr);
    });
}

// Times cfar2d_integral over a batch of fp32 maps (widened to double outside
// the timer, bench.hpp:70-72) on `workers` host threads, each running the
// reference with threads=1 on whole maps (way (ii)); or, with
// workers == 1 and ref_threads > 1, the reference's own row split.
// Returns total seconds; detection counts per map go to counts.
int uwbref_time_cfar_batch(const float* maps, std::uint64_t n_maps, std::uint64_t rows,
                           std::uint64_t cols, int g, int b, double pfa, unsigned workers,
                           unsigned ref_threads, std::uint64_t* counts, double* seconds,
                           char* errbuf, std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const std::size_t cells = rows * cols;
        std::vector<R::Matrix> widened(n_maps, R::Matrix(rows, cols));
        for (std::size_t i = 0; i < n_maps; ++i) {
            double* d = widened[i].values().data();
            const float* s = maps + i * cells;
            for (std::size_t k = 0; k < cells; ++k) d[k] = static_cast<double>(s[k]);
        }
        const R::CfarParams p = make_params(g, b, pfa);
        const auto t0 = std::chrono::steady_clock::now();
        if (workers <= 1) {
            for (std::size_t i = 0; i < n_maps; ++i)
                counts[i] = R::cfar2d_integral(widened[i], p, ref_threads).detections.size();
        } else {
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < workers; ++w) {
                pool.emplace_back([&, w] {
                    for (std::size_t i = w; i < n_maps; i += workers)
                        counts[i] = R::cfar2d_integral(widened[i], p, 1).detections.size();
                });
            }
            for (auto& t : pool) t.join();
        }
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
    });
}

// ---- front-end stages (pipeline.cpp) ----
// op: 0 remove_dc, 1 detrend_linear, 2 mean_filter_slow(window),
//     3 subtract_slow_time_mean, 4 normalize_slow(epsilon)
int uwbref_frame_stage(int op, const double* data, std::uint64_t m, std::uint64_t n,
                       std::uint64_t window, double epsilon, double* out, char* errbuf,
                       std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const R::RadarFrame f = make_frame(data, m, n, 39e9, 68.6);
        R::RadarFrame o;
        switch (op) {
            case 0: o = R::remove_dc(f); break;
            case 1: o = R::detrend_linear(f); break;
            case 2: o = R::mean_filter_slow(f, window); break;
            case 3: o = R::subtract_slow_time_mean(f); break;
            case 4: o = R::normalize_slow(f, epsilon); break;
            default: throw std::runtime_error("bad op");
        }
        from_matrix(o.data, out);
    });
}

int uwbref_slow_time_spectrum(const double* data, std::uint64_t m, std::uint64_t n, double fast_rate,
                              double prf, std::uint64_t fft_length, double* power,
                              double* freq_axis, double* range_axis, char* errbuf,
                              std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const R::RangeFrequencyMap map =
            R::slow_time_spectrum(make_frame(data, m, n, fast_rate, prf), fft_length);
        from_matrix(map.power, power);
        std::memcpy(freq_axis, map.freq_axis.data(), sizeof(double) * map.freq_axis.size());
        std::memcpy(range_axis, map.range_axis.data(), sizeof(double) * map.range_axis.size());
    });
}

// band_select on a full spectrum; outputs the kept bin range [first, first+kept).
int uwbref_band_select(const double* power, std::uint64_t m, std::uint64_t bins,
                       const double* freq_axis, double low, double high, double* out_power,
                       double* out_freq, std::uint64_t* kept, char* errbuf, std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        R::RangeFrequencyMap in;
        in.power = to_matrix(power, m, bins);
        in.freq_axis.assign(freq_axis, freq_axis + bins);
        in.range_axis.assign(m, 0.0);
        const R::RangeFrequencyMap o = R::band_select(in, low, high);
        *kept = o.freq_axis.size();
        if (out_power) from_matrix(o.power, out_power);
        if (out_freq) std::memcpy(out_freq, o.freq_axis.data(), sizeof(double) * o.freq_axis.size());
    });
}

struct uwbref_pipeline_config {
    std::uint64_t mean_filter_window;
    std::uint64_t fft_length;
    double band_low_hz;
    double band_high_hz;
    int guard_radius;
    int background_radius;
    double pfa;
    int backend; // 0 naive, 1 integral
    double normalization_epsilon;
    int mean_filter_mode; // 0 smoothing, 1 subtract mean
};

// detect(); band map capacity is m * band_cap columns. Outputs the band width
// and the band's first frequency index so callers can size buffers.
int uwbref_detect(const double* data, std::uint64_t m, std::uint64_t n, double fast_rate, double prf,
                  const uwbref_pipeline_config* cfg, unsigned threads, std::uint64_t band_cap,
                  double* band_power, double* band_freq, double* range_axis,
                  std::uint64_t* band_cols, std::uint8_t* mask, double* thr, std::uint64_t* n_det,
                  std::uint64_t det_cap, std::uint64_t* det_rows, std::uint64_t* det_cols,
                  double* det_val, double* det_thr, char* errbuf, std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        R::PipelineConfig c;
        c.mean_filter_window = cfg->mean_filter_window;
        c.fft_length = cfg->fft_length;
        c.band_low_hz = cfg->band_low_hz;
        c.band_high_hz = cfg->band_high_hz;
        c.cfar = make_params(cfg->guard_radius, cfg->background_radius, cfg->pfa);
        c.backend = cfg->backend == 0 ? R::CfarBackend::Naive : R::CfarBackend::IntegralImage;
        c.normalization_epsilon = cfg->normalization_epsilon;
        c.mean_filter_mode = cfg->mean_filter_mode == 0 ? R::MeanFilterMode::Smoothing
                                                        : R::MeanFilterMode::SubtractMean;
        const R::DetectOutput o = R::detect(make_frame(data, m, n, fast_rate, prf), c, threads);
        const std::size_t k = o.band_map.freq_axis.size();
        *band_cols = k;
        if (k > band_cap) throw std::runtime_error("band_cap too small");
        if (band_power) from_matrix(o.band_map.power, band_power);
        if (band_freq) std::memcpy(band_freq, o.band_map.freq_axis.data(), sizeof(double) * k);
        if (range_axis)
            std::memcpy(range_axis, o.band_map.range_axis.data(), sizeof(double) * m);
        export_result(o.detections, mask, thr, n_det, det_cap, det_rows, det_cols, det_val,
                      det_thr);
    });
}

// Reference scene synthesiser (synth.cpp), used only to generate test inputs
// for the reference's own detect() scene tests (test_pipeline.cpp:294-412).
struct uwbref_scene_config {
    std::uint64_t m_samples;
    std::uint64_t n_traces;
    double fast_rate;
    double prf;
    double target_range_m;
    double resp_freq_hz;
    double resp_displacement_m;
    double wall_range_m;
    double wall_amplitude;
    double noise_sigma;
    double pulse_center_hz;
    double pulse_bandwidth_hz;
    double target_attenuation;
    std::uint64_t seed;
};

void uwbref_default_scene_config(uwbref_scene_config* out) {
    const R::SceneConfig d;
    out->m_samples = d.m_samples;
    out->n_traces = d.n_traces;
    out->fast_rate = d.fast_rate;
    out->prf = d.prf;
    out->target_range_m = d.target_range_m;
    out->resp_freq_hz = d.resp_freq_hz;
    out->resp_displacement_m = d.resp_displacement_m;
    out->wall_range_m = d.wall_range_m;
    out->wall_amplitude = d.wall_amplitude;
    out->noise_sigma = d.noise_sigma;
    out->pulse_center_hz = d.pulse_center_hz;
    out->pulse_bandwidth_hz = d.pulse_bandwidth_hz;
    out->target_attenuation = d.target_attenuation;
    out->seed = d.seed;
}

int uwbref_generate_scene(const uwbref_scene_config* in, double* data, std::uint64_t* truth_bin,
                          double* truth_freq, char* errbuf, std::uint64_t errlen) {
    return guarded(errbuf, errlen, [&] {
        R::SceneConfig c;
        c.m_samples = in->m_samples;
        c.n_traces = in->n_traces;
        c.fast_rate = in->fast_rate;
        c.prf = in->prf;
        c.target_range_m = in->target_range_m;
        c.resp_freq_hz = in->resp_freq_hz;
        c.resp_displacement_m = in->resp_displacement_m;
        c.wall_range_m = in->wall_range_m;
        c.wall_amplitude = in->wall_amplitude;
        c.noise_sigma = in->noise_sigma;
        c.pulse_center_hz = in->pulse_center_hz;
        c.pulse_bandwidth_hz = in->pulse_bandwidth_hz;
        c.target_attenuation = in->target_attenuation;
        c.seed = in->seed;
        const R::Scene s = R::generate_scene(c);
        from_matrix(s.frame.data, data);
        *truth_bin = s.truth.target_range_bin;
        *truth_freq = s.truth.resp_freq_hz;
    });
}

// ---- frame_io.cpp:69-122 read_frame (RFRM files) ----
// data: m x n doubles (range-major, as RadarFrame::data) when capacity allows.
int uwbref_read_frame(const char* path, double* data, std::uint64_t capacity, std::uint32_t* m, std::uint32_t* n,
                      double* fast_rate, double* prf, char* errbuf, std::size_t errlen) {
    return guarded(errbuf, errlen, [&] {
        const R::RadarFrame f = R::read_frame_file(path);
        *m = static_cast<std::uint32_t>(f.samples());
        *n = static_cast<std::uint32_t>(f.traces());
        *fast_rate = f.fast_rate;
        *prf = f.prf;
        if (data && capacity >= f.samples() * f.traces())
            std::memcpy(data, f.data.values().data(), sizeof(double) * f.samples() * f.traces());
    });
}

} // extern "C"
