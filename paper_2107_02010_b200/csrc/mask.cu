// mask.cu — K3: kernel truncation and the
// ranges that feed the block-sparse softmin.
//
// Test per cluster pair (a per-pair distance bound in
// place of SPEC.md:283's Lipschitz margin p (r_I + r_J) d^{p-1}):
//   keep (I,J)  iff  F_I + G_J - (1/2) max(0, |X_I - Y_J| - r_I - r_J)^2 >= -theta eps
// where F, G are per-cluster maxima of the current fine potentials, so the
// left side bounds f_i + g_j - C(x_i, y_j) from above for every member pair:
// a dropped block carries plan mass <= alpha_i beta_j e^{-theta} per pair.
// Evaluated in float64 with explicitly rounded operations (no FMA) on
// float32 inputs: bit-identical to oracle.cpp:pair_slack on the same inputs.
#include "prims.cuh"

namespace msot_dev {

__device__ __forceinline__ double pair_slack(float4 X, float rI, float F, float4 Y, float rJ,
                                             float G, int d) {
  double s = 0.0;
  double t = __dsub_rn(static_cast<double>(X.x), static_cast<double>(Y.x));
  s = __dadd_rn(s, __dmul_rn(t, t));
  if (d > 1) {
    t = __dsub_rn(static_cast<double>(X.y), static_cast<double>(Y.y));
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  if (d > 2) {
    t = __dsub_rn(static_cast<double>(X.z), static_cast<double>(Y.z));
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  double lb = __dsub_rn(__dsqrt_rn(s), static_cast<double>(rI));
  lb = __dsub_rn(lb, static_cast<double>(rJ));
  if (lb < 0.0) lb = 0.0;
  const double c = __dmul_rn(0.5, __dmul_rn(lb, lb));
  const double fg = __dadd_rn(static_cast<double>(F), static_cast<double>(G));
  return __dsub_rn(fg, c);
}

__global__ void mask_kernel(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                            const float* fx, const float4* cy, const float* ry, const float* gy,
                            double thr, int self, uint8_t* mask) {
  const int32_t J = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t I = blockIdx.y;
  if (J >= ky) return;
  const double v = pair_slack(cx[I], rx[I], fx[I], cy[J], ry[J], gy[J], d);
  mask[static_cast<int64_t>(I) * ky + J] = (v >= thr || (self && I == J)) ? 1 : 0;
}

// best pair of each row (ties -> lowest J) and of each column (ties -> lowest I)
__global__ void best_kernel(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                            const float* fx, const float4* cy, const float* ry, const float* gy,
                            int by_col, uint8_t* mask) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int32_t nw = by_col ? ky : kx, nl = by_col ? kx : ky;
  if (w >= nw) return;
  double best = -INFINITY;
  int32_t arg = 0x7fffffff;
  for (int32_t q = lane; q < nl; q += 32) {
    const int32_t I = by_col ? q : static_cast<int32_t>(w);
    const int32_t J = by_col ? static_cast<int32_t>(w) : q;
    const double v = pair_slack(cx[I], rx[I], fx[I], cy[J], ry[J], gy[J], d);
    if (v > best) { best = v; arg = q; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
    const int32_t a2 = __shfl_xor_sync(0xffffffffu, arg, o);
    if (b2 > best || (b2 == best && a2 < arg)) { best = b2; arg = a2; }
  }
  if (lane == 0 && arg != 0x7fffffff) {
    const int64_t I = by_col ? arg : w, J = by_col ? w : arg;
    mask[I * ky + J] = 1;
  }
}

cudaError_t truncation_mask(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                            const float* fx, const float4* cy, const float* ry, const float* gy,
                            double eps, double theta, int self, uint8_t* mask, cudaStream_t st) {
  if (kx <= 0 || ky <= 0) return cudaSuccess;
  const double thr = -(theta * eps);
  dim3 grid((ky + 255) / 256, kx);
  ++g_launches; mask_kernel<<<grid, 256, 0, st>>>(kx, ky, d, cx, rx, fx, cy, ry, gy, thr, self, mask);
  ++g_launches; best_kernel<<<static_cast<unsigned>((static_cast<int64_t>(kx) * 32 + 255) / 256), 256, 0, st>>>(
      kx, ky, d, cx, rx, fx, cy, ry, gy, 0, mask);
  ++g_launches; best_kernel<<<static_cast<unsigned>((static_cast<int64_t>(ky) * 32 + 255) / 256), 256, 0, st>>>(
      kx, ky, d, cx, rx, fx, cy, ry, gy, 1, mask);
  return cudaGetLastError();
}

__global__ void transpose_kernel(const uint8_t* m, int32_t kx, int32_t ky, uint8_t* mt) {
  __shared__ uint8_t t[32][33];
  const int32_t bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int32_t I = by + r, J = bx + threadIdx.x;
    if (I < kx && J < ky) t[r][threadIdx.x] = m[static_cast<int64_t>(I) * ky + J];
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int32_t J = bx + r, I = by + threadIdx.x;
    if (I < kx && J < ky) mt[static_cast<int64_t>(J) * kx + I] = t[threadIdx.x][r];
  }
}

cudaError_t transpose_mask(const uint8_t* m, int32_t kx, int32_t ky, uint8_t* mt,
                           cudaStream_t st) {
  if (kx <= 0 || ky <= 0) return cudaSuccess;
  dim3 grid((ky + 31) / 32, (kx + 31) / 32), block(32, 8);
  ++g_launches; transpose_kernel<<<grid, block, 0, st>>>(m, kx, ky, mt);
  return cudaGetLastError();
}

// ---- ranges per row tile -------------------------------------------------
// One warp per tile: OR the mask rows of the clusters the tile touches, then
// turn runs of kept column clusters into sorted-column ranges [co[J0], co[J1+1]).
__device__ __forceinline__ bool tile_keep(const uint8_t* mask, int32_t ky, int32_t I0, int32_t I1,
                                          int32_t J) {
  if (J >= ky) return false;
  for (int32_t I = I0; I <= I1; ++I)
    if (mask[static_cast<int64_t>(I) * ky + J]) return true;
  return false;
}

template <bool kWrite>
__global__ void tile_ranges_kernel(const int32_t* rl, const int32_t* ts, int64_t n_tiles,
                                   const int32_t* co, int32_t ky, const uint8_t* mask,
                                   int64_t* n_ranges, int64_t* n_cols, const int64_t* rptr,
                                   int2* ranges) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= n_tiles) return;
  const int32_t I0 = rl[ts[t]];
  const int32_t I1 = rl[ts[t + 1] - 1];
  const unsigned lt = (1u << lane) - 1u;
  int64_t nr = 0, nc = 0;
  int64_t base = kWrite ? rptr[t] : 0;
  int64_t ns = 0, ne = 0;  // starts / ends written so far
  bool prev = false;       // keep[J0 - 1]
  for (int32_t J0 = 0; J0 < ky; J0 += 32) {
    const int32_t J = J0 + lane;
    const bool k = tile_keep(mask, ky, I0, I1, J);
    const unsigned b = __ballot_sync(0xffffffffu, k);
    const bool next = (lane < 31) ? ((b >> (lane + 1)) & 1u) : tile_keep(mask, ky, I0, I1, J0 + 32);
    const bool left = (lane > 0) ? ((b >> (lane - 1)) & 1u) : prev;
    const bool is_start = k && !left, is_end = k && !next;
    const unsigned bs = __ballot_sync(0xffffffffu, is_start);
    const unsigned be = __ballot_sync(0xffffffffu, is_end);
    if (kWrite) {
      if (is_start) ranges[base + ns + __popc(bs & lt)].x = co[J];
      if (is_end) ranges[base + ne + __popc(be & lt)].y = co[J + 1];
    }
    ns += __popc(bs);
    ne += __popc(be);
    if (!kWrite && k) nc += co[J + 1] - co[J];
    prev = __shfl_sync(0xffffffffu, k, 31);
  }
  nr = ns;
  if (!kWrite) {
    for (int o = 16; o > 0; o >>= 1) nc += __shfl_xor_sync(0xffffffffu, nc, o);
    if (lane == 0) {
      n_ranges[t] = nr;
      n_cols[t] = nc;
    }
  }
}

cudaError_t tile_range_count(const int32_t* row_labels, const int32_t* tile_start, int64_t nt,
                             const int32_t* col_offsets, int32_t ky, const uint8_t* mask,
                             int64_t* n_ranges, int64_t* n_cols, cudaStream_t st) {
  if (nt <= 0) return cudaSuccess;
  ++g_launches; tile_ranges_kernel<false><<<static_cast<unsigned>((nt * 32 + 255) / 256), 256, 0, st>>>(
      row_labels, tile_start, nt, col_offsets, ky, mask, n_ranges, n_cols, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t tile_range_write(const int32_t* row_labels, const int32_t* tile_start, int64_t nt,
                             const int32_t* col_offsets, int32_t ky, const uint8_t* mask,
                             const int64_t* rptr, int2* ranges, cudaStream_t st) {
  if (nt <= 0) return cudaSuccess;
  ++g_launches; tile_ranges_kernel<true><<<static_cast<unsigned>((nt * 32 + 255) / 256), 256, 0, st>>>(
      row_labels, tile_start, nt, col_offsets, ky, mask, nullptr, nullptr, rptr, ranges);
  return cudaGetLastError();
}

__global__ void dense_ranges_kernel(int64_t nt, int32_t m, int64_t* rptr, int2* ranges,
                                    int64_t* tile_cols) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t > nt) return;
  rptr[t] = t;
  if (t < nt) {
    ranges[t] = make_int2(0, m);
    if (tile_cols) tile_cols[t] = m;
  }
}

cudaError_t dense_ranges(int64_t n_tiles, int32_t n_cols, int64_t* rptr, int2* ranges,
                         int64_t* tile_cols, cudaStream_t st) {
  ++g_launches; dense_ranges_kernel<<<static_cast<unsigned>((n_tiles + 1 + 255) / 256), 256, 0, st>>>(
      n_tiles, n_cols, rptr, ranges, tile_cols);
  return cudaGetLastError();
}

// ---- work items ----------------------------------------------------------
__global__ void item_counts_kernel(const int64_t* tc, int64_t nt, int64_t chunk, int32_t* cnt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int64_t c = (tc[t] + chunk - 1) / chunk;
  cnt[t] = static_cast<int32_t>(c < 1 ? 1 : c);
}

cudaError_t item_counts(const int64_t* tile_cols, int64_t n_tiles, int64_t chunk, int32_t* cnt,
                        cudaStream_t st) {
  if (n_tiles <= 0) return cudaSuccess;
  ++g_launches; item_counts_kernel<<<static_cast<unsigned>((n_tiles + 255) / 256), 256, 0, st>>>(tile_cols,
                                                                                   n_tiles, chunk, cnt);
  return cudaGetLastError();
}

// ibase is indexed by tile (valid on [t0, t1]); items are split evenly over
// the tile's concatenated column list.
__global__ void item_write_kernel(const int64_t* tc, int64_t t0, int64_t t1, const int32_t* ibase,
                                  int problem, int4* items) {
  const int64_t t = t0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= t1) return;
  const int32_t b = ibase[t], nch = ibase[t + 1] - b;
  const int64_t L = tc[t];
  for (int32_t c = 0; c < nch; ++c)
    items[b + c] = make_int4(problem, static_cast<int32_t>(t), static_cast<int32_t>(c * L / nch),
                             static_cast<int32_t>((c + 1) * L / nch));
}

cudaError_t item_write(const int64_t* tile_cols, int64_t t0, int64_t t1, int64_t chunk,
                       const int32_t* ibase, int problem, int4* items, cudaStream_t st) {
  (void)chunk;
  if (t1 <= t0) return cudaSuccess;
  ++g_launches; item_write_kernel<<<static_cast<unsigned>((t1 - t0 + 255) / 256), 256, 0, st>>>(
      tile_cols, t0, t1, ibase, problem, items);
  return cudaGetLastError();
}

}  // namespace msot_dev
