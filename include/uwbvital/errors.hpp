// uwbvital B200 drop-in: exception taxonomy (same classes and base as the
// reference's errors.hpp, so existing catch sites and exit-code mappings work).
// The C ABI reports these as uwb_status codes 1..5 (include/uwbvital_b200.h).
#pragma once

#include <stdexcept>
#include <string>

namespace uwbvital {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct DimensionError : Error { using Error::Error; };     // empty / mis-shaped input
struct InputError : Error { using Error::Error; };         // non-finite or negative data
struct ParameterError : Error { using Error::Error; };     // scalar out of domain
struct BoundsError : Error { using Error::Error; };        // rectangle or cell out of range
struct ConfigurationError : Error { using Error::Error; }; // config incompatible with data
struct FormatError : Error { using Error::Error; };        // on-disk format violation
struct GateError : Error { using Error::Error; };          // benchmark correctness gate

} // namespace uwbvital
