// loss.cu — K7: the debiased divergence from the four potentials.
//
// Balanced (reach = inf):
//   S = <a, b_yx - a_xx> + <b, a_xy - b_yy> + (eps/2)(sum a - sum b)^2
// Unbalanced (Eq. 6, plus the Eq. 5 mass term):
//   S = -(rho + eps/2) [<a, e^{-b_yx/rho} - e^{-a_xx/rho}> + <b, e^{-a_xy/rho} - e^{-b_yy/rho}>]
//       + (eps/2)(sum a - sum b)^2
// float64 accumulation with a fixed reduction tree (fixed grid, fixed block,
// fixed order), computed on the full gathered vectors: the value does not
// depend on the number of GPUs.
#include "prims.cuh"

namespace msot_dev {

constexpr int kLossThreads = 256;

__device__ __forceinline__ double term(double w, float f_cross, float f_self, double rho) {
  if (rho <= 0.0) return w * (static_cast<double>(f_cross) - static_cast<double>(f_self));
  return w * (exp(-static_cast<double>(f_cross) / rho) - exp(-static_cast<double>(f_self) / rho));
}

__global__ void divergence_partial_kernel(const double* a, const double* b, int64_t n, int64_t m,
                                          const float* a_xx, const float* b_yy, const float* a_xy,
                                          const float* b_yx, double rho, double* partials) {
  __shared__ double sh[3][kLossThreads / 32];
  const int64_t total = n + m;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(total, lo + per);
  double S = 0.0, A = 0.0, B = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    if (i < n) {
      S += term(a[i], b_yx[i], a_xx[i], rho);
      A += a[i];
    } else {
      const int64_t j = i - n;
      S += term(b[j], a_xy[j], b_yy[j], rho);
      B += b[j];
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    S += __shfl_xor_sync(0xffffffffu, S, o);
    A += __shfl_xor_sync(0xffffffffu, A, o);
    B += __shfl_xor_sync(0xffffffffu, B, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sh[0][w] = S;
    sh[1][w] = A;
    sh[2][w] = B;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int k = 0; k < kLossThreads / 32; ++k) v += sh[threadIdx.x][k];
    partials[3 * blockIdx.x + threadIdx.x] = v;
  }
}

__global__ void divergence_final_kernel(const double* partials, int nb, double eps, double rho,
                                        double* out) {
  if (threadIdx.x != 0) return;
  double S = 0.0, A = 0.0, B = 0.0;
  for (int k = 0; k < nb; ++k) {
    S += partials[3 * k];
    A += partials[3 * k + 1];
    B += partials[3 * k + 2];
  }
  const double mass = 0.5 * eps * (A - B) * (A - B);
  out[0] = (rho <= 0.0 ? S : -(rho + 0.5 * eps) * S) + mass;
  out[1] = A;
  out[2] = B;
}

cudaError_t divergence_partial(const double* a, const double* b, int64_t n, int64_t m,
                               const float* a_xx, const float* b_yy, const float* a_xy,
                               const float* b_yx, double rho, double* partials, int nblocks,
                               cudaStream_t st) {
  ++g_launches; divergence_partial_kernel<<<nblocks, kLossThreads, 0, st>>>(a, b, n, m, a_xx, b_yy, a_xy, b_yx,
                                                              rho, partials);
  return cudaGetLastError();
}

cudaError_t divergence_final(const double* partials, int nblocks, double eps, double rho,
                             double* out, cudaStream_t st) {
  ++g_launches; divergence_final_kernel<<<1, 32, 0, st>>>(partials, nblocks, eps, rho, out);
  return cudaGetLastError();
}

__global__ void scatter_unsort_kernel(const float* v, const int32_t* perm, int64_t n, double* out) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s < n) out[perm ? perm[s] : s] = static_cast<double>(v[s]);
}

cudaError_t scatter_unsort(const float* v, const int32_t* perm, int64_t n, double* out,
                           cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; scatter_unsort_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(v, perm, n, out);
  return cudaGetLastError();
}

}  // namespace msot_dev
