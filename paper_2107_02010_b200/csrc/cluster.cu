// cluster.cu — K2: voxel-grid clustering (north star; stands in for the
// K-means coarsening of SPEC.md:260-268, ClusterTree fields SPEC.md:249-252).
//
//   cube id   floor((x - origin) / cell) per axis in float64 (one rounded
//             subtraction + one rounded division: bit-identical to the host
//             rule in policy.h), Morton-interleaved so consecutive cubes are
//             spatial neighbours and a 256-row tile stays compact;
//   sort      stable LSD radix sort of (cube id, atom index) (prims.cu);
//   segments  flags where the id changes -> inclusive scan -> labels, offsets;
//   stats     one warp per cluster: weight, mass-weighted centroid, radius
//             (max distance to the centroid, rounded up to float32).
#include "prims.cuh"

namespace msot_dev {

__global__ void cube_keys_kernel(const double* x, int64_t n, GridSpec g, uint32_t* keys,
                                 int32_t* iota) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = msot_cube_key(x + i * g.d, g.d, g.origin, g.cell);
  iota[i] = static_cast<int32_t>(i);
}

cudaError_t cube_keys(const double* x, int64_t n, GridSpec g, uint32_t* keys, int32_t* iota,
                      cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; cube_keys_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(x, n, g, keys, iota);
  return cudaGetLastError();
}

// Sorted, centred float32 atoms {x, y, z, 0}, log2 weights, float64 weights.
__global__ void gather_points_kernel(const double* x, const double* w, int64_t n, int d,
                                     GridSpec g, const int32_t* perm, float4* pts, float* lw2,
                                     double* w64, int32_t* nonuniform) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in = s < n;
  const int64_t i = in ? (perm ? perm[s] : s) : 0;
  const double wi = w[i];
  // weights not all equal (one atomic per warp)
  const bool diff = in && wi != w[0];
  if (nonuniform && __any_sync(0xffffffffu, diff) && (threadIdx.x & 31) == 0) atomicOr(nonuniform, 1);
  if (!in) return;
  float c[3] = {0.f, 0.f, 0.f};
  for (int k = 0; k < d && k < 3; ++k) c[k] = __double2float_rn(x[i * d + k] - g.center[k]);
  pts[s] = make_float4(c[0], c[1], c[2], 0.f);
  lw2[s] = __double2float_rn(log2(wi));
  w64[s] = wi;
}

cudaError_t gather_points(const double* x, const double* w, int64_t n, int d, GridSpec g,
                          const int32_t* perm, float4* pts, float* lw2, double* w64,
                          int32_t* nonuniform, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; gather_points_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(x, w, n, d, g, perm,
                                                                               pts, lw2, w64, nonuniform);
  return cudaGetLastError();
}

__global__ void segment_flags_kernel(const uint32_t* k, int64_t n, uint8_t* flags) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  flags[s] = (s == 0 || k[s] != k[s - 1]) ? 1 : 0;
}

cudaError_t segment_flags(const uint32_t* sorted_keys, int64_t n, uint8_t* flags,
                          cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; segment_flags_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(sorted_keys, n,
                                                                               flags);
  return cudaGetLastError();
}

// labels arrive as an inclusive scan of the flags; make them 0-based and
// record each cluster's first sorted position (offsets[K] = n).
__global__ void segment_offsets_kernel(int32_t* labels, const uint8_t* flags, int64_t n,
                                       int32_t* offsets) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const int32_t l = labels[s] - 1;
  labels[s] = l;
  if (flags[s]) offsets[l] = static_cast<int32_t>(s);
  if (s == n - 1) offsets[l + 1] = static_cast<int32_t>(n);
}

cudaError_t segment_offsets(const int32_t* labels, const uint8_t* flags, int64_t n,
                            int32_t* offsets, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; segment_offsets_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
      const_cast<int32_t*>(labels), flags, n, offsets);
  return cudaGetLastError();
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void cluster_stats_kernel(const float4* pts, const double* w64, const int32_t* off,
                                     int32_t k, int d, float4* cen, float* clw2, double* cw64,
                                     float* radii, float4* box_lo, float4* box_hi) {
  const int lane = threadIdx.x & 31;
  const int64_t I = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (I >= k) return;
  const int32_t s0 = off[I], s1 = off[I + 1];
  double W = 0.0, a0 = 0.0, a1 = 0.0, a2 = 0.0;
  for (int32_t s = s0 + lane; s < s1; s += 32) {
    const double wi = w64[s];
    const float4 p = pts[s];
    W += wi;
    a0 += wi * static_cast<double>(p.x);
    a1 += wi * static_cast<double>(p.y);
    a2 += wi * static_cast<double>(p.z);
  }
  W = warp_sum(W);
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  a2 = warp_sum(a2);
  const double c0 = a0 / W, c1 = d > 1 ? a1 / W : 0.0, c2 = d > 2 ? a2 / W : 0.0;
  const float4 cf = make_float4(__double2float_rn(c0), __double2float_rn(c1),
                                __double2float_rn(c2), 0.f);
  double r = 0.0;
  // member box: the float-to-double differences are exact, min/max too
  double l0 = 0.0, l1 = 0.0, l2 = 0.0, h0 = 0.0, h1 = 0.0, h2 = 0.0;
  for (int32_t s = s0 + lane; s < s1; s += 32) {
    const float4 p = pts[s];
    const double t0 = static_cast<double>(p.x) - cf.x, t1 = static_cast<double>(p.y) - cf.y,
                 t2 = static_cast<double>(p.z) - cf.z;
    r = fmax(r, sqrt(t0 * t0 + t1 * t1 + t2 * t2));
    l0 = fmin(l0, t0); l1 = fmin(l1, t1); l2 = fmin(l2, t2);
    h0 = fmax(h0, t0); h1 = fmax(h1, t1); h2 = fmax(h2, t2);
  }
  r = warp_max(r);
  for (int o = 16; o > 0; o >>= 1) {
    l0 = fmin(l0, __shfl_xor_sync(0xffffffffu, l0, o));
    l1 = fmin(l1, __shfl_xor_sync(0xffffffffu, l1, o));
    l2 = fmin(l2, __shfl_xor_sync(0xffffffffu, l2, o));
    h0 = fmax(h0, __shfl_xor_sync(0xffffffffu, h0, o));
    h1 = fmax(h1, __shfl_xor_sync(0xffffffffu, h1, o));
    h2 = fmax(h2, __shfl_xor_sync(0xffffffffu, h2, o));
  }
  if (lane == 0) {
    cen[I] = cf;
    cw64[I] = W;
    clw2[I] = __double2float_rn(log2(W));
    radii[I] = __double2float_ru(r);
    if (box_lo) {
      box_lo[I] = make_float4(__double2float_rd(l0), __double2float_rd(l1), __double2float_rd(l2), 0.f);
      box_hi[I] = make_float4(__double2float_ru(h0), __double2float_ru(h1), __double2float_ru(h2), 0.f);
    }
  }
}

cudaError_t cluster_stats(const float4* pts, const double* w64, const int32_t* offsets, int32_t k,
                          int d, float4* cen, float* clw2, double* cw64, float* radii,
                          cudaStream_t st, float4* box_lo, float4* box_hi) {
  if (k <= 0) return cudaSuccess;
  const int64_t threads = static_cast<int64_t>(k) * 32;
  ++g_launches; cluster_stats_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
      pts, w64, offsets, k, d, cen, clw2, cw64, radii, box_lo, box_hi);
  return cudaGetLastError();
}

// Per-cluster bound inputs of the truncation test (mask.cu) from a fine
// potential f over the cluster's members u_i = x_i - X_I:
//   fmax  = max_i f_i
//   grad  = {G, F'}: G the w-weighted least-squares slope of f in u (float),
//           F' = max_i (f_i - <G, u_i>) in float64, rounded up.
// Any G gives a valid bound; the fitted slope makes the margin small.
__device__ __forceinline__ void solve3(double m00, double m01, double m02, double m11, double m12,
                                       double m22, double b0, double b1, double b2, double* g) {
  const double tr = m00 + m11 + m22;
  const double reg = 1e-9 * tr + 1e-300;
  m00 += reg;
  m11 += reg;
  m22 += reg;
  const double c00 = m11 * m22 - m12 * m12, c01 = m02 * m12 - m01 * m22,
               c02 = m01 * m12 - m02 * m11;
  const double det = m00 * c00 + m01 * c01 + m02 * c02;
  if (!(det > 0.0) || !isfinite(det)) {
    g[0] = g[1] = g[2] = 0.0;
    return;
  }
  const double c11 = m00 * m22 - m02 * m02, c12 = m01 * m02 - m00 * m12,
               c22 = m00 * m11 - m01 * m01;
  g[0] = (c00 * b0 + c01 * b1 + c02 * b2) / det;
  g[1] = (c01 * b0 + c11 * b1 + c12 * b2) / det;
  g[2] = (c02 * b0 + c12 * b1 + c22 * b2) / det;
}

__global__ void cluster_bound_kernel(const float4* pts, const double* w64, const float* f,
                                     const int32_t* off, const float4* cen, int32_t k,
                                     float* fmax_out, float4* grad) {
  const int lane = threadIdx.x & 31;
  const int64_t I = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (I >= k) return;
  const int32_t s0 = off[I], s1 = off[I + 1];
  const float4 X = cen[I];
  double m[6] = {0, 0, 0, 0, 0, 0}, b[3] = {0, 0, 0}, W = 0.0, wf = 0.0;
  for (int32_t s = s0 + lane; s < s1; s += 32) {
    const float4 p = pts[s];
    const double w = w64[s], fv = f[s];
    const double u0 = static_cast<double>(p.x) - X.x, u1 = static_cast<double>(p.y) - X.y,
                 u2 = static_cast<double>(p.z) - X.z;
    m[0] += w * u0 * u0; m[1] += w * u0 * u1; m[2] += w * u0 * u2;
    m[3] += w * u1 * u1; m[4] += w * u1 * u2; m[5] += w * u2 * u2;
    W += w;
    wf += w * fv;
    b[0] += w * u0 * fv; b[1] += w * u1 * fv; b[2] += w * u2 * fv;
  }
  for (int o = 16; o > 0; o >>= 1) {
    for (int q = 0; q < 6; ++q) m[q] += __shfl_xor_sync(0xffffffffu, m[q], o);
    for (int q = 0; q < 3; ++q) b[q] += __shfl_xor_sync(0xffffffffu, b[q], o);
    W += __shfl_xor_sync(0xffffffffu, W, o);
    wf += __shfl_xor_sync(0xffffffffu, wf, o);
  }
  // centre f on its mean: sum w u (f - fbar) = sum w u f - fbar sum w u
  double mu[3] = {0, 0, 0};
  for (int32_t s = s0 + lane; s < s1; s += 32) {
    const float4 p = pts[s];
    const double w = w64[s];
    mu[0] += w * (static_cast<double>(p.x) - X.x);
    mu[1] += w * (static_cast<double>(p.y) - X.y);
    mu[2] += w * (static_cast<double>(p.z) - X.z);
  }
  for (int o = 16; o > 0; o >>= 1)
    for (int q = 0; q < 3; ++q) mu[q] += __shfl_xor_sync(0xffffffffu, mu[q], o);
  const double fbar = wf / W;
  double g[3];
  solve3(m[0], m[1], m[2], m[3], m[4], m[5], b[0] - fbar * mu[0], b[1] - fbar * mu[1],
         b[2] - fbar * mu[2], g);
  const float4 G = make_float4(__double2float_rn(g[0]), __double2float_rn(g[1]),
                               __double2float_rn(g[2]), 0.f);
  float fm = -INFINITY;
  double fp = -INFINITY;
  for (int32_t s = s0 + lane; s < s1; s += 32) {
    const float4 p = pts[s];
    const float fv = f[s];
    fm = fmaxf(fm, fv);
    const double lin = static_cast<double>(G.x) * (static_cast<double>(p.x) - X.x) +
                       static_cast<double>(G.y) * (static_cast<double>(p.y) - X.y) +
                       static_cast<double>(G.z) * (static_cast<double>(p.z) - X.z);
    fp = fmax(fp, static_cast<double>(fv) - lin);
  }
  for (int o = 16; o > 0; o >>= 1) {
    fm = fmaxf(fm, __shfl_xor_sync(0xffffffffu, fm, o));
    fp = fmax(fp, __shfl_xor_sync(0xffffffffu, fp, o));
  }
  if (lane == 0) {
    fmax_out[I] = fm;
    grad[I] = make_float4(G.x, G.y, G.z, __double2float_ru(fp));
  }
}

cudaError_t cluster_bound(const float4* pts, const double* w64, const float* f,
                          const int32_t* offsets, const float4* cen, int32_t k, float* fmax,
                          float4* grad, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  const int64_t threads = static_cast<int64_t>(k) * 32;
  ++g_launches; cluster_bound_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(
      pts, w64, f, offsets, cen, k, fmax, grad);
  return cudaGetLastError();
}

// coarse_duals_to_fine by inheritance: used as the
// expansion reference of the extrapolation softmin.
// Super-voxel key of every cluster: the key of its first sorted atom >> bits.
__global__ void super_keys_kernel(const uint32_t* sorted_keys, const int32_t* offsets, int32_t k,
                                  int bits, uint32_t* out) {
  const int32_t I = blockIdx.x * blockDim.x + threadIdx.x;
  if (I < k) out[I] = sorted_keys[offsets[I]] >> bits;
}

cudaError_t super_keys(const uint32_t* sorted_keys, const int32_t* offsets, int32_t k, int bits,
                       uint32_t* out, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  ++g_launches;
  super_keys_kernel<<<(k + 255) / 256, 256, 0, st>>>(sorted_keys, offsets, k, bits, out);
  return cudaGetLastError();
}

// dst[s] = src[idx[s]] / dst[idx[s]] = src[s] (float4, float): moves between a
// solve's sorted order and the caller's (idx = the sort permutation).
__global__ void gather_f4_kernel(const float4* src, const int32_t* idx, int64_t n, float4* dst) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s < n) dst[s] = src[idx[s]];
}
__global__ void scatter_f4_kernel(const float4* src, const int32_t* idx, int64_t n, float4* dst) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s < n) dst[idx[s]] = src[s];
}
__global__ void scatter_f32_kernel(const float* src, const int32_t* idx, int64_t n, float* dst) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s < n) dst[idx[s]] = src[s];
}
cudaError_t gather_f4(const float4* src, const int32_t* idx, int64_t n, float4* dst, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  gather_f4_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(src, idx, n, dst);
  return cudaGetLastError();
}
cudaError_t scatter_f4(const float4* src, const int32_t* idx, int64_t n, float4* dst, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  scatter_f4_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(src, idx, n, dst);
  return cudaGetLastError();
}
cudaError_t scatter_f32(const float* src, const int32_t* idx, int64_t n, float* dst, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  scatter_f32_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(src, idx, n, dst);
  return cudaGetLastError();
}

// payload {w, sx, sy, sz} += w * (cx, cy, cz): a plan payload's weighted
// coordinate sums moved to another origin.
__global__ void shift_payload_kernel(float4* p, int64_t n, double cx, double cy, double cz) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  float4 v = p[s];
  const double w = v.x;
  v.y = static_cast<float>(v.y + w * cx);
  v.z = static_cast<float>(v.z + w * cy);
  v.w = static_cast<float>(v.w + w * cz);
  p[s] = v;
}
cudaError_t shift_payload(float4* p, int64_t n, double cx, double cy, double cz, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  shift_payload_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(p, n, cx, cy, cz);
  return cudaGetLastError();
}

__global__ void inherit_kernel(const float* coarse, const int32_t* labels, int64_t n, float* fine) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s < n) fine[s] = coarse[labels[s]];
}

cudaError_t inherit(const float* coarse, const int32_t* labels, int64_t n, float* fine,
                    cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches; inherit_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(coarse, labels, n, fine);
  return cudaGetLastError();
}

}  // namespace msot_dev
