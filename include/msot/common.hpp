// msot/common.hpp — error types of the msot:: API.
//
// Same types and meaning as the reference (proj/include/msot/common.hpp:10-19):
// DataError for malformed or inconsistent input, NumericError for numerical
// breakdown.  The GPU front-end adds DeviceError for CUDA/NCCL failures
// (C ABI status MSOT_ECUDA), which the reference, being CPU-only, lacks.
#pragma once

#include <stdexcept>
#include <string>

namespace msot {

class DataError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class NumericError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// Maps a C ABI status (include/msot_gpu.h) to the exception above; status 2
// (usage) is reported as DataError like the reference's parameter checks.
void throw_on_status(int status, const std::string& what);

}  // namespace msot
