// msot/numeric.hpp — deterministic summation of the msot:: API.
//
// Same declarations and contract as the reference (proj/include/msot/
// numeric.hpp:9-15), implemented host-side in libmsot_b200.so
// (csrc/host_runtime.cpp).  pairwise_sum / pairwise_dot use the reference's
// summation tree (halving split, serial leaves of <= 32 terms), so their
// results are bitwise those of the reference build; the device analogue is
// the fixed-order float64 reduction of loss.cu.
#pragma once

#include <cstddef>
#include <span>

namespace msot {

// Compensated (Kahan) summation.
double kahan_sum(std::span<const double> values);

// Fixed-order cascade summation: bitwise deterministic.
double pairwise_sum(std::span<const double> values);

// <a, b> over the shorter length, with the same summation tree.
double pairwise_dot(std::span<const double> a, std::span<const double> b);

}  // namespace msot
