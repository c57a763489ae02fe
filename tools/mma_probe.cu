// mma_probe.cu — dev microbenchmark: legacy mma.sync m16n8k8 tf32 issue rate on
// sm_100a, alone and interleaved with MUFU.EX2 at the 4:1 ratio of the
// evaluate-once column reduction (K4s).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int MODE>
__global__ void __launch_bounds__(256) probe(int iters, float seed, float* sink) {
  float d[4][4] = {};
  unsigned a[4], b[2];
  for (int k = 0; k < 4; ++k) a[k] = __float_as_uint(seed * (threadIdx.x + k));
  b[0] = __float_as_uint(1.f);
  b[1] = __float_as_uint(1.f);
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = seed * (threadIdx.x + k) * 1e-7f - 1.0f;
  for (int i = 0; i < iters; ++i) {
    if (MODE != 1) {  // 16 ex2 per lane
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = ex2(v[k]) - 1.5f;
    }
    if (MODE != 0) {  // 4 mma per warp
#pragma unroll
      for (int c = 0; c < 4; ++c) mma_tf32(d[c], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += v[k];
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 12345.f) sink[threadIdx.x] = s;
}

template <int MODE>
float run(int iters) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  float* sink;
  cudaMalloc(&sink, 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  probe<MODE><<<nsm * 8, 256>>>(iters, 1.f, sink);
  cudaEventRecord(e0);
  probe<MODE><<<nsm * 8, 256>>>(iters, 1.f, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = nsm * 8.0 * 8.0;
  const double ex2s = MODE == 1 ? 0 : warps * 32 * 16.0 * iters;
  const double mmas = MODE == 0 ? 0 : warps * 4.0 * iters;
  printf("mode %d: %.3f ms  ex2 %.3e/s  mma %.3e/s (%.1f TFLOP/s tf32)\n", MODE, ms, ex2s / (ms * 1e-3),
         mmas / (ms * 1e-3), mmas * 2.0 * 16 * 8 * 8 / (ms * 1e-3) / 1e12);
  cudaFree(sink);
  return ms;
}

int main() {
  run<0>(4000);
  run<1>(4000);
  run<2>(4000);
  return 0;
}
