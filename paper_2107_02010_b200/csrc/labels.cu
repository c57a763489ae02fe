// labels.cu — K9: label transfer through the implicit transport plan
// (eq. 7, config 4 "with label transfer"):
//
//   Lab_i[l] = sum_{j : label_j = l} b_j exp((f_i + g_j - C_ij) / eps)   ( = (pi l)_i / a_i )
//
// The reduction is the softmin's own (softmin_kernel / softmin_hd_kernel)
// with est = f, h = g and lambda = 1: each partial sum is then
// sum_j pi_ij / a_i over a run of columns.  The columns are re-ordered by
// label (stable), each label segment padded to the kernel's column block,
// and the work items are cut at segment boundaries, so every partial belongs
// to exactly one (row tile, label); label_finalize sums them in a fixed
// order into float64 scores.  One-hot label vectors are never materialised
// and the plan never is either: memory stays linear in N + M (+ N x L out).
#include "prims.cuh"

namespace msot_dev {

// Columns in label order: src[p] = source column (solver order) or -1 for
// padding (weight 0 -> log2 w = -inf, contributes exactly 0).
__global__ void gather_label_cols_kernel(const float4* pts, const float* lw2, const float* h,
                                         const int32_t* src, int64_t mpad, float4* cols,
                                         float* lw_out, float* h_out) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= mpad) return;
  const int32_t s = src[p];
  if (s >= 0) {
    if (cols) cols[p] = pts[s];
    lw_out[p] = lw2[s];
    h_out[p] = h[s];
  } else {
    if (cols) cols[p] = make_float4(0.f, 0.f, 0.f, 0.f);
    lw_out[p] = __int_as_float(0xff800000);
    h_out[p] = 0.f;
  }
}

cudaError_t gather_label_cols(const float4* pts, const float* lw2, const float* h,
                              const int32_t* src, int64_t mpad, float4* cols, float* lw_out,
                              float* h_out, cudaStream_t st) {
  if (mpad <= 0) return cudaSuccess;
  ++g_launches;
  gather_label_cols_kernel<<<static_cast<unsigned>((mpad + 255) / 256), 256, 0, st>>>(
      pts, lw2, h, src, mpad, cols, lw_out, h_out);
  return cudaGetLastError();
}

// float64 rows x (row-major, d per row) in label order (high-D operands are
// packed from these); padding rows are zero.
__global__ void gather_rows_f64_kernel(const double* x, int d, const int32_t* src, int64_t mpad,
                                       double* out) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= mpad * d) return;
  const int64_t p = g / d;
  const int k = static_cast<int>(g - p * d);
  const int32_t s = src[p];
  out[g] = s >= 0 ? x[static_cast<int64_t>(s) * d + k] : 0.0;
}

cudaError_t gather_rows_f64(const double* x, int d, const int32_t* src, int64_t mpad, double* out,
                            cudaStream_t st) {
  if (mpad <= 0) return cudaSuccess;
  ++g_launches;
  const int64_t tot = mpad * d;
  gather_rows_f64_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(x, d, src,
                                                                                   mpad, out);
  return cudaGetLastError();
}

// One CTA per row tile, one thread per row: scores[row][l] = sum of the
// partials of the tile's items of label l (item order = column order, fixed),
// row_mass = sum over l in order.  Outputs in the caller's row order.
__global__ void label_finalize_kernel(const float* part, const int32_t* lbase,
                                      const int32_t* tile_start, int n_classes,
                                      const int32_t* perm, double* scores, double* mass) {
  const int t = blockIdx.x;
  const int lr = threadIdx.x;
  const int row = tile_start[t] + lr;
  if (row >= tile_start[t + 1]) return;
  const int64_t out = perm ? perm[row] : row;
  if (out < 0) return;  // padding slot of the high-D multiscale layout
  double m = 0.0;
  const int32_t* lb = lbase + static_cast<int64_t>(t) * n_classes;
  for (int l = 0; l < n_classes; ++l) {
    double s = 0.0;
    for (int32_t it = lb[l]; it < lb[l + 1]; ++it)
      s += static_cast<double>(part[static_cast<int64_t>(it) * kTileRows + lr]);
    scores[out * n_classes + l] = s;
    m += s;
  }
  mass[out] = m;
}

cudaError_t label_finalize(const float* part, const int32_t* lbase, const int32_t* tile_start,
                           int64_t n_tiles, int n_classes, const int32_t* perm, double* scores,
                           double* mass, cudaStream_t st) {
  if (n_tiles <= 0) return cudaSuccess;
  ++g_launches;
  label_finalize_kernel<<<static_cast<unsigned>(n_tiles), kTileRows, 0, st>>>(
      part, lbase, tile_start, n_classes, perm, scores, mass);
  return cudaGetLastError();
}

}  // namespace msot_dev
