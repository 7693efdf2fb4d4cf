// GPU columns for the reference benchmark reports.
//
// The reference's renderers (bench.cpp:318-430, compiled unchanged) report the
// wall time of each call; linked against the drop-in that is the end-to-end
// time of the call (host buffers, H2D, kernels, D2H). These helpers measure the
// same work device-resident through the C ABI (uwb_dev_cfar2d /
// uwb_dev_detect_batch on device buffers, CUDA events on the launching stream)
// and append it to the reports:
//   dev_naive_s / dev_ii_s    device time per call (naive / integral backend)
//   dev_ratio                 dev_naive_s / dev_ii_s
//   dev_ii_hbm_frac           the integral call's required bytes (map in,
//                             threshold map + mask out: 17 B/cell) over its
//                             device time, as a fraction of the HBM peak
//   e2e_ii_s                  the reference column itself (the drop-in call)
// CSV rows keep the reference's seven / five columns first and add these after
// them; JSON rows keep every reference key (the reference's parsers read the
// augmented JSON unchanged); the text report gains a "GPU columns" block.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace refbench {

struct DevTimes {
    double naive_s = 0.0;
    double integral_s = 0.0;
};

// Per-call device time of cfar2d on a rows x cols Exp(1) fp64 map with the
// drop-in's outputs (u8 mask + threshold map + sorted list).
DevTimes time_cfar_device(std::size_t rows, std::size_t cols, int guard, int background, double pfa,
                          std::size_t reps);

// Per-call device time of detect() (front end + CFAR) on one record, and of the
// threshold step alone on its band map, for both backends.
struct DetectDevTimes {
    DevTimes total, threshold;
};
DetectDevTimes time_detect_device(const std::vector<double>& frame, std::size_t m, std::size_t n, double fast_rate,
                                  double prf, std::size_t mean_filter_window, std::size_t fft_length,
                                  double band_low, double band_high, int guard, int background, double pfa,
                                  std::size_t reps);

double hbm_peak_gbs(std::string* source);

// Report augmentation (see the header comment).
std::string cfar_csv_with_gpu(const std::string& ref_csv, const std::vector<DevTimes>& dev,
                              const std::vector<double>& hbm_frac);
std::string cfar_json_with_gpu(const std::string& ref_json, const std::vector<DevTimes>& dev,
                               const std::vector<double>& hbm_frac, const std::string& peak_source);
std::string cfar_text_with_gpu(const std::string& ref_text, const std::vector<std::pair<int, int>>& grid,
                               const std::vector<DevTimes>& dev, const std::vector<double>& hbm_frac,
                               const std::vector<double>& e2e_ii_s);
// Pipeline rows (bench.cpp:302-308): fast time, slow time, threshold (naive),
// threshold (II), total. Device columns on the threshold and total rows.
std::string pipeline_csv_with_gpu(const std::string& ref_csv, const DetectDevTimes& dev);
std::string pipeline_json_with_gpu(const std::string& ref_json, const DetectDevTimes& dev);
std::string pipeline_text_with_gpu(const std::string& ref_text, const DetectDevTimes& dev);

} // namespace refbench
