// uwbvital B200 drop-in: raw radar record (rows = fast-time samples, cols =
// slow-time traces). Same fields and defaults as the reference's frame.hpp.
#pragma once

#include "uwbvital/grid.hpp"

namespace uwbvital {

struct RadarFrame {
    Matrix data;
    double fast_rate = 39e9; // Hz, within-trace sampling rate
    double prf = 68.6;       // Hz, trace repetition rate

    std::size_t samples() const { return data.rows(); }
    std::size_t traces() const { return data.cols(); }

    // >= 2x2 (DimensionError), positive rates (ParameterError), finite (InputError).
    void validate() const;
};

} // namespace uwbvital
