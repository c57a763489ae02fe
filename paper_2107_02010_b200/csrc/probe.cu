// probe.cu — on-box measurement of the softmin roofline denominator: the
// MUFU.EX2 issue rate of the whole GPU (SURVEY.md §2.3 assumes 16/clk/SM;
// this kernel measures it, with the same ex2.approx.ftz.f32 the softmin
// issues).  Every thread runs 8 independent ex2 chains so the pipe, not the
// latency, is the limit.
#include "prims.cuh"

namespace msot_dev {

__global__ void __launch_bounds__(256) ex2_probe_kernel(int iters, float seed, float* sink) {
  float v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = seed * (threadIdx.x + k) * 1e-7f - 1.0f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ex2_approx(v[k]) - 1.5f;
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += v[k];
  if (s == 12345.f) sink[threadIdx.x] = s;
}

cudaError_t ex2_probe(int n_sm, int iters, float* sink, double* ex2_per_launch, int* blocks,
                      cudaStream_t st) {
  const int b = n_sm * 8;  // 8 x 256 threads per SM
  *blocks = b;
  *ex2_per_launch = static_cast<double>(b) * 256.0 * 8.0 * iters;
  ++g_launches;
  ex2_probe_kernel<<<b, 256, 0, st>>>(iters, 1.0f, sink);
  return cudaGetLastError();
}

}  // namespace msot_dev
