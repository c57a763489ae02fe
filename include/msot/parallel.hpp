// msot/parallel.hpp — the host thread pool of the msot:: API.
//
// Same declarations and contract as the reference (proj/include/msot/
// parallel.hpp:10-17), implemented in libmsot_b200.so (csrc/host_runtime.cpp).
// On the GPU build the solver's data parallelism is the CUDA grid and one
// process per GPU; this pool serves the host-side preparation of the
// front-end and CLI (file parsing, fibre encoding, flip resolution), and
// callers that used it with the reference keep working unchanged.
#pragma once

#include <cstddef>
#include <functional>

namespace msot::parallel {

// Worker threads used by the host-side data-parallel loops (default: the
// hardware concurrency; 1 runs everything on the caller's thread).
int threads();
void set_threads(int n);

// fn(begin, end) over a static partition of [0, n) into contiguous chunks of
// ceil(n / threads()) indices, one per thread; returns when all are done.
void for_ranges(std::size_t n, const std::function<void(std::size_t, std::size_t)>& fn);

}  // namespace msot::parallel
