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
constexpr int kLossAcc = 5;

__device__ __forceinline__ double term(double w, float f_cross, float f_self, double rho) {
  if (rho <= 0.0) return w * (static_cast<double>(f_cross) - static_cast<double>(f_self));
  return w * (exp(-static_cast<double>(f_cross) / rho) - exp(-static_cast<double>(f_self) / rho));
}

__global__ void divergence_partial_kernel(const double* a, const double* b, int64_t n, int64_t m,
                                          const float* a_xx, const float* b_yy, const float* a_xy,
                                          const float* b_yx, double rho, double* partials) {
  // accumulators: S (dual objective), A = sum a, B = sum b,
  //               Pa = <a, b_yx>, Pb = <b, a_xy> (for the gauge, balanced case)
  __shared__ double sh[kLossAcc][kLossThreads / 32];
  const int64_t total = n + m;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = min(total, lo + per);
  double v[kLossAcc] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    if (i < n) {
      v[0] += term(a[i], b_yx[i], a_xx[i], rho);
      v[1] += a[i];
      v[3] += a[i] * static_cast<double>(b_yx[i]);
    } else {
      const int64_t j = i - n;
      v[0] += term(b[j], a_xy[j], b_yy[j], rho);
      v[2] += b[j];
      v[4] += b[j] * static_cast<double>(a_xy[j]);
    }
  }
#pragma unroll
  for (int q = 0; q < kLossAcc; ++q)
    for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int q = 0; q < kLossAcc; ++q) sh[q][w] = v[q];
  __syncthreads();
  if (threadIdx.x < kLossAcc) {
    double s = 0.0;
    for (int k = 0; k < kLossThreads / 32; ++k) s += sh[threadIdx.x][k];
    partials[kLossAcc * blockIdx.x + threadIdx.x] = s;
  }
}

// out = {S_eps, sum a, sum b, gauge c}.  Balanced potentials are defined up
// to (b_yx + c, a_xy - c) — a direction the averaged iteration never damps,
// so float rounding random-walks along it.  Both the oracle and this solver
// return the canonical representative <a, b_yx> = <b, a_xy>; the loss is
// evaluated on it (identical to the raw value when the masses are equal).
__global__ void divergence_final_kernel(const double* partials, int nb, double eps, double rho,
                                        double* out) {
  if (threadIdx.x != 0) return;
  double v[kLossAcc] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < nb; ++k)
    for (int q = 0; q < kLossAcc; ++q) v[q] += partials[kLossAcc * k + q];
  const double A = v[1], B = v[2];
  double S = v[0], c = 0.0;
  if (rho <= 0.0) {
    c = (v[4] - v[3]) / (A + B);
    S += c * (A - B);
  } else {
    S = -(rho + 0.5 * eps) * S;
  }
  out[0] = S + 0.5 * eps * (A - B) * (A - B);
  out[1] = A;
  out[2] = B;
  out[3] = c;
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

// out[perm[s]] = v[s] + sign * (*shift)  (shift nullable)
__global__ void scatter_unsort_kernel(const float* v, const int32_t* perm, int64_t n,
                                      const double* shift, double sign, double* out) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int64_t i = perm ? perm[s] : s;
  if (i >= 0)  // padding slots of the high-D multiscale layout carry a negative index
    out[i] = static_cast<double>(v[s]) + (shift ? sign * *shift : 0.0);
}

cudaError_t scatter_unsort(const float* v, const int32_t* perm, int64_t n, const double* shift,
                           double sign, double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; scatter_unsort_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(v, perm, n, shift, sign, out);
  return cudaGetLastError();
}

}  // namespace msot_dev

namespace msot_dev {

// grad_positions, envelope theorem with the final
// potentials: d S / d x_i = sum_j pi^xy_ij (x_i - y_j) - sum_k pi^xx_ik (x_i - x_k)
// (the self term of -1/2 OT(a,a) counts twice), i.e.
//   a_i [ (m^xy_i - m^xx_i) x_i - (u^xy_i - u^xx_i) ]
// with m, u the per-row plan sums of plan_kernel (pi / a_i, payload = coordinates).
__global__ void grad_positions_kernel(const float4* pts, const double* w64, const float4* pxy,
                                      const float4* pxx, const int32_t* perm, int64_t n, int d,
                                      double* grad) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const float4 x = pts[s], a = pxy[s], b = pxx[s];
  const double dm = static_cast<double>(a.x) - static_cast<double>(b.x);
  const double g[3] = {dm * x.x - (static_cast<double>(a.y) - b.y),
                       dm * x.y - (static_cast<double>(a.z) - b.z),
                       dm * x.z - (static_cast<double>(a.w) - b.w)};
  const int64_t i = perm ? perm[s] : s;
  for (int k = 0; k < d; ++k) grad[i * d + k] = w64[s] * g[k];
}

cudaError_t grad_positions(const float4* pts, const double* w64, const float4* plan_xy,
                           const float4* plan_xx, const int32_t* perm, int64_t n, int d,
                           double* grad, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  grad_positions_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
      pts, w64, plan_xy, plan_xx, perm, n, d, grad);
  return cudaGetLastError();
}

}  // namespace msot_dev

namespace msot_dev {

// field += scale * grad   (float64, n*d)
__global__ void axpy_kernel(double* field, const double* grad, double scale, int64_t len) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < len) field[i] += scale * grad[i];
}

// x_new = x - step * field / a   (barycenter descent on the positions with the
// displacement field grad / a_i)
__global__ void bary_step_kernel(double* x_new, const double* x, const double* field,
                                 const double* a, double step, int64_t n, int d) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n * d) return;
  x_new[g] = x[g] - step * field[g] / a[g / d];
}

cudaError_t field_accumulate(double* field, const double* grad, double scale, int64_t len,
                             cudaStream_t st) {
  if (len <= 0) return cudaSuccess;
  ++g_launches;
  axpy_kernel<<<static_cast<unsigned>((len + 255) / 256), 256, 0, st>>>(field, grad, scale, len);
  return cudaGetLastError();
}

cudaError_t bary_step(double* x_new, const double* x, const double* field, const double* a,
                      double step, int64_t n, int d, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  bary_step_kernel<<<static_cast<unsigned>((n * d + 255) / 256), 256, 0, st>>>(x_new, x, field, a,
                                                                               step, n, d);
  return cudaGetLastError();
}

}  // namespace msot_dev
