// The uwbvital:: C++ API (include/uwbvital/*.hpp) implemented over the C ABI of
// include/uwbvital_b200.h. This is what a C++ caller of the reference links
// instead of uwbvital_core: same headers, same functions, same exceptions and
// messages; the arithmetic runs on the B200.
#include <cstring>
#include <string>

#include "uwbvital/cfar.hpp"
#include "uwbvital/errors.hpp"
#include "uwbvital/pipeline.hpp"
#include "uwbvital/sat.hpp"
#include "uwbvital_b200.h"

namespace uwbvital {

namespace {

[[noreturn]] void raise(uwb_status s) {
    const std::string msg = uwb_last_error();
    switch (s) {
        case UWB_DIMENSION_ERROR: throw DimensionError(msg);
        case UWB_INPUT_ERROR: throw InputError(msg);
        case UWB_PARAMETER_ERROR: throw ParameterError(msg);
        case UWB_BOUNDS_ERROR: throw BoundsError(msg);
        case UWB_CONFIGURATION_ERROR: throw ConfigurationError(msg);
        default: throw Error("uwbvital_b200: " + msg);
    }
}

void check(uwb_status s) {
    if (s != UWB_OK) raise(s);
}

uwb_cfar_params to_c(const CfarParams& p) {
    return uwb_cfar_params{p.guard_radius, p.guard_radius, p.background_radius, p.background_radius,
                           p.pfa};
}

DetectionResult run_cfar(uwb_backend backend, const Matrix& map, const CfarParams& params) {
    const uwb_cfar_params cp = to_c(params);
    DetectionResult res;
    res.mask = Mask(map.rows(), map.cols(), 0);
    res.threshold_map = Matrix(map.rows(), map.cols(), 0.0);
    uint64_t n = 0;
    std::vector<uwb_detection> buf(std::max<std::size_t>(1, std::min<std::size_t>(map.size(), 4096)));
    uwb_status s = uwb_cfar2d(backend, map.values().data(), map.rows(), map.cols(), &cp,
                              res.mask.values().data(), res.threshold_map.values().data(), buf.data(),
                              buf.size(), &n);
    if (s == UWB_CAPACITY_ERROR) {
        buf.resize(n);
        s = uwb_cfar2d(backend, map.values().data(), map.rows(), map.cols(), &cp, res.mask.values().data(),
                       res.threshold_map.values().data(), buf.data(), buf.size(), &n);
    }
    check(s);
    res.detections.resize(n);
    for (std::size_t i = 0; i < n; ++i)
        res.detections[i] = Detection{buf[i].row, buf[i].col, buf[i].value, buf[i].threshold};
    return res;
}

RadarFrame stage(const RadarFrame& f,
                 uwb_status (*fn)(const double*, uint64_t, uint64_t, double*)) {
    RadarFrame out = f;
    check(fn(f.data.values().data(), f.samples(), f.traces(), out.data.values().data()));
    return out;
}

} // namespace

// ----------------------------------------------------------------- frame ---

void RadarFrame::validate() const {
    if (data.rows() < 2 || data.cols() < 2)
        throw DimensionError("RadarFrame: need at least 2x2 samples, got " + std::to_string(data.rows()) +
                             "x" + std::to_string(data.cols()));
    if (!(fast_rate > 0.0) || !(prf > 0.0))
        throw ParameterError("RadarFrame: fast_rate and prf must be positive");
    if (!all_finite(data)) throw InputError("RadarFrame: non-finite sample");
}

// ------------------------------------------------------------------- SAT ---

SummedAreaTable build_sat(const Matrix& source) {
    SummedAreaTable sat;
    sat.src_rows_ = source.rows();
    sat.src_cols_ = source.cols();
    if (!source.empty()) sat.padded_ = Matrix(source.rows() + 1, source.cols() + 1, 0.0);
    check(uwb_build_sat(source.values().data(), source.rows(), source.cols(), sat.padded_.values().data()));
    return sat;
}

double SummedAreaTable::region_sum(std::size_t r0, std::size_t r1, std::size_t c0, std::size_t c1) const {
    if (r0 > r1 || c0 > c1 || r1 >= src_rows_ || c1 >= src_cols_) {
        throw BoundsError("region_sum: invalid rectangle [" + std::to_string(r0) + ".." + std::to_string(r1) +
                          "] x [" + std::to_string(c0) + ".." + std::to_string(c1) + "] on " +
                          std::to_string(src_rows_) + "x" + std::to_string(src_cols_) + " table");
    }
    return region_sum_unchecked(r0, r1, c0, c1);
}

// ------------------------------------------------------------------ CFAR ---

void CfarParams::validate() const {
    const uwb_cfar_params p = to_c(*this);
    check(uwb_cfar_params_validate(&p));
}

std::size_t CfarParams::interior_train_count() const {
    const uwb_cfar_params p = to_c(*this);
    return uwb_interior_train_count(&p);
}

double alpha_factor(std::size_t n_train, double pfa) {
    double a = 0.0;
    check(uwb_alpha_factor(n_train, pfa, &a));
    return a;
}

TrainingWindow training_window(const CfarParams& params, std::size_t row, std::size_t col, std::size_t rows,
                               std::size_t cols) {
    const uwb_cfar_params p = to_c(params);
    uint64_t o[9];
    check(uwb_training_window(&p, row, col, rows, cols, o));
    TrainingWindow w;
    w.outer = CellRect{o[0], o[1], o[2], o[3]};
    w.guard = CellRect{o[4], o[5], o[6], o[7]};
    w.n_train = o[8];
    return w;
}

DetectionResult cfar2d_naive(const Matrix& power_map, const CfarParams& params, unsigned) {
    return run_cfar(UWB_NAIVE, power_map, params);
}

DetectionResult cfar2d_integral(const Matrix& power_map, const CfarParams& params, unsigned) {
    return run_cfar(UWB_INTEGRAL, power_map, params);
}

// -------------------------------------------------------------- pipeline ---

std::size_t PipelineConfig::effective_fft_length(std::size_t n_traces) const {
    if (fft_length != 0) return fft_length;
    std::size_t p = 1;
    while (p < n_traces) p <<= 1;
    return p;
}

void PipelineConfig::validate() const {
    if (mean_filter_window == 0 || mean_filter_window % 2 == 0)
        throw ParameterError("PipelineConfig: mean_filter_window must be odd and positive, got " +
                             std::to_string(mean_filter_window));
    if (!(band_low_hz > 0.0) || !(band_low_hz < band_high_hz))
        throw ParameterError("PipelineConfig: need 0 < band_low_hz < band_high_hz");
    if (!(normalization_epsilon > 0.0))
        throw ParameterError("PipelineConfig: normalization_epsilon must be positive");
    cfar.validate();
}

RadarFrame remove_dc(const RadarFrame& frame) { return stage(frame, uwb_remove_dc); }
RadarFrame detrend_linear(const RadarFrame& frame) { return stage(frame, uwb_detrend_linear); }
RadarFrame subtract_slow_time_mean(const RadarFrame& frame) { return stage(frame, uwb_subtract_slow_time_mean); }

RadarFrame mean_filter_slow(const RadarFrame& frame, std::size_t window) {
    RadarFrame out = frame;
    check(uwb_mean_filter_slow(frame.data.values().data(), frame.samples(), frame.traces(), window,
                               out.data.values().data()));
    return out;
}

RadarFrame normalize_slow(const RadarFrame& frame, double epsilon) {
    RadarFrame out = frame;
    check(uwb_normalize_slow(frame.data.values().data(), frame.samples(), frame.traces(), epsilon,
                             out.data.values().data()));
    return out;
}

RangeFrequencyMap slow_time_spectrum(const RadarFrame& frame, std::size_t fft_length) {
    RangeFrequencyMap map;
    const std::size_t bins = fft_length / 2 + 1;
    if (fft_length >= frame.traces()) {
        map.power = Matrix(frame.samples(), bins, 0.0);
        map.freq_axis.resize(bins);
        map.range_axis.resize(frame.samples());
    }
    check(uwb_slow_time_spectrum(frame.data.values().data(), frame.samples(), frame.traces(), frame.fast_rate,
                                 frame.prf, fft_length, map.power.values().data(), map.freq_axis.data(),
                                 map.range_axis.data()));
    return map;
}

RangeFrequencyMap band_select(const RangeFrequencyMap& map, double band_low_hz, double band_high_hz) {
    uint64_t first = 0, kept = 0;
    check(uwb_band_select(map.power.values().data(), map.power.rows(), map.freq_axis.size(),
                          map.freq_axis.data(), band_low_hz, band_high_hz, &first, &kept, nullptr, nullptr));
    RangeFrequencyMap out;
    out.power = Matrix(map.power.rows(), kept, 0.0);
    out.freq_axis.resize(kept);
    check(uwb_band_select(map.power.values().data(), map.power.rows(), map.freq_axis.size(),
                          map.freq_axis.data(), band_low_hz, band_high_hz, &first, &kept,
                          out.power.values().data(), out.freq_axis.data()));
    out.range_axis = map.range_axis;
    return out;
}

DetectOutput detect(const RadarFrame& frame, const PipelineConfig& config, unsigned) {
    uwb_pipeline_config c{};
    c.mean_filter_window = config.mean_filter_window;
    c.fft_length = config.fft_length;
    c.band_low_hz = config.band_low_hz;
    c.band_high_hz = config.band_high_hz;
    c.cfar = to_c(config.cfar);
    c.backend = config.backend == CfarBackend::Naive ? UWB_NAIVE : UWB_INTEGRAL;
    c.mean_filter_mode = config.mean_filter_mode == MeanFilterMode::Smoothing ? 0 : 1;
    c.normalization_epsilon = config.normalization_epsilon;
    const std::size_t m = frame.samples(), n = frame.traces();
    const std::size_t L = config.effective_fft_length(n);
    const std::size_t cap = L / 2 + 1;
    std::vector<double> band(m * cap), freq(cap), range(m), thr(m * cap);
    std::vector<uint8_t> mask(m * cap);
    std::vector<uwb_detection> dets(std::max<std::size_t>(1, m * cap));
    uint64_t kept = 0, nd = 0;
    check(uwb_detect(frame.data.values().data(), m, n, frame.fast_rate, frame.prf, &c, cap, band.data(),
                     freq.data(), range.data(), &kept, mask.data(), thr.data(), dets.data(), dets.size(), &nd));
    DetectOutput out;
    out.band_map.power = Matrix(m, kept, 0.0);
    std::memcpy(out.band_map.power.values().data(), band.data(), sizeof(double) * m * kept);
    out.band_map.freq_axis.assign(freq.begin(), freq.begin() + static_cast<std::ptrdiff_t>(kept));
    out.band_map.range_axis = range;
    out.detections.mask = Mask(m, kept, 0);
    std::memcpy(out.detections.mask.values().data(), mask.data(), m * kept);
    out.detections.threshold_map = Matrix(m, kept, 0.0);
    std::memcpy(out.detections.threshold_map.values().data(), thr.data(), sizeof(double) * m * kept);
    out.detections.detections.resize(nd);
    for (std::size_t i = 0; i < nd; ++i)
        out.detections.detections[i] = Detection{dets[i].row, dets[i].col, dets[i].value, dets[i].threshold};
    return out;
}

} // namespace uwbvital
