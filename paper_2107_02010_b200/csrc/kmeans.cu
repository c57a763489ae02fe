// kmeans.cu — K-means coarsening of high-dimensional measures
// (kmeans_coarsen; "a simple K-means
// algorithm"): the coarse measure of the multiscale solver when the voxel
// grid does not apply (D > 3, the D = 60 fibre features of config 4).
//
//   seeding   farthest-point: the first centre is atom (seed mod N), then
//             repeatedly the atom farthest from all chosen centres (ties to
//             the lowest index)
//   Lloyd     assign every atom to its nearest centre (ties to the lowest
//             centre), mass-weighted centroids, until the largest centre
//             move is below 1e-9 d or 100 iterations
//
// Every distance is sum_k (x_k - c_k)^2 in float64 in a fixed order with
// explicitly rounded operations (no FMA), and every centroid sum runs
// sequentially over the cluster's atoms in index order, so labels, centroids
// and radii are bit-identical to oracle.cpp:kmeans on the same input.
#include "prims.cuh"

namespace msot_dev {

constexpr int kKmDmax = 64;

__device__ __forceinline__ double km_dist2(const double* x, const double* c, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = __dsub_rn(x[k], c[k]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  return s;
}

// farthest-point step: mind_i = min(mind_i, |x_i - c|^2); per-block argmax
// (largest, then lowest index).  asg_i = the centre that attains mind_i,
// dnew[a] = |c_a - c|^2 (fps_ccdist_kernel): when |c_asg - c| >= 2 sqrt(mind_i)
// the triangle inequality puts c no closer than the current minimum, so the
// atom's row is not read at all (margin 1e-9 against the float64 rounding of
// the three distances, ~1e-14 relative) — mind is exactly what the full scan
// computes, and most atoms skip once the centres are dense.
__global__ void fps_update_kernel(const double* x, int64_t n, int d, const double* c, int kc,
                                  double* mind, int32_t* asg, const double* dnew, int first,
                                  double* bval, int64_t* bidx) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double m = -1.0;
  int64_t mi = INT64_MAX;
  if (i < n) {
    if (first) {
      m = km_dist2(x + i * d, c, d);
      mind[i] = m;
      asg[i] = kc;
    } else {
      m = mind[i];
      if (!(dnew[asg[i]] >= 4.0 * m * (1.0 + 1e-9))) {
        const double dd = km_dist2(x + i * d, c, d);
        if (dd < m) {  // fmin(m, dd)
          m = dd;
          mind[i] = m;
          asg[i] = kc;
        }
      }
    }
    mi = i;
  }
  sv[threadIdx.x] = m;
  si[threadIdx.x] = mi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = sv[threadIdx.x + o];
      const int64_t i2 = si[threadIdx.x + o];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bval[blockIdx.x] = sv[0];
    bidx[blockIdx.x] = si[0];
  }
}

// global argmax over the blocks; the winner becomes centre k
__global__ void fps_select_kernel(const double* bval, const int64_t* bidx, int nb, const double* x,
                                  int d, double* centers, int k) {
  __shared__ double sv[256];
  __shared__ int64_t si[256];
  double m = -2.0;
  int64_t mi = INT64_MAX;
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (bval[b] > m || (bval[b] == m && bidx[b] < mi)) {
      m = bval[b];
      mi = bidx[b];
    }
  sv[threadIdx.x] = m;
  si[threadIdx.x] = mi;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      const double v2 = sv[threadIdx.x + o];
      const int64_t i2 = si[threadIdx.x + o];
      if (v2 > sv[threadIdx.x] || (v2 == sv[threadIdx.x] && i2 < si[threadIdx.x])) {
        sv[threadIdx.x] = v2;
        si[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  const int64_t w = si[0];
  for (int q = threadIdx.x; q < d; q += blockDim.x) centers[static_cast<int64_t>(k) * d + q] = x[w * d + q];
}

// distances of the earlier centres to the newest one, centre k
// (fps_update_kernel's skip; a bound with a margin, so any summation order):
// one warp per earlier centre, spread over the SMs
__global__ void fps_ccdist_kernel(const double* centers, int d, int k, double* dnew) {
  const int lane = threadIdx.x & 31;
  const int a = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  if (a >= k) return;
  const double* ca = centers + static_cast<int64_t>(a) * d;
  const double* ck = centers + static_cast<int64_t>(k) * d;
  double s = 0.0;
  for (int q = lane; q < d; q += 32) {
    const double t = ca[q] - ck[q];
    s = fma(t, t, s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) dnew[a] = s;
}

__global__ void copy_center_kernel(const double* x, int64_t i, int d, double* c) {
  for (int q = threadIdx.x; q < d; q += blockDim.x) c[q] = x[i * d + q];
}

// nearest centre of every atom (ties to the lowest centre); centres staged
// through shared memory in chunks, the atom's coordinates in registers
// list (nullable): scan only the atoms list[0 .. *count) (km_bounds_kernel).
// ub / lb (nullable): the distance to the nearest centre and to the second
// nearest (Hamerly bounds for the next iteration).
template <int DM>
__global__ void __launch_bounds__(128) km_assign_kernel(const double* x, int64_t n, int d,
                                                        const double* centers, int K,
                                                        uint32_t* labels, const int32_t* list,
                                                        const int32_t* count, double* ub,
                                                        double* lb) {
  constexpr int kChunk = 32;
  __shared__ double cs[kChunk * DM];
  const int64_t slot = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t m = list ? *count : n;
  if (static_cast<int64_t>(blockIdx.x) * blockDim.x >= m) return;  // whole block idle
  const int64_t i = slot < m ? (list ? list[slot] : slot) : n;
  double xr[DM];
#pragma unroll
  for (int k = 0; k < DM; ++k) xr[k] = (i < n && k < d) ? x[i * d + k] : 0.0;
  double best = INFINITY, second = INFINITY;
  int bl = 0;
  for (int c0 = 0; c0 < K; c0 += kChunk) {
    const int nc = min(kChunk, K - c0);
    __syncthreads();
    for (int q = threadIdx.x; q < nc * d; q += blockDim.x)
      cs[(q / d) * DM + (q % d)] = centers[static_cast<int64_t>(c0) * d + q];
    __syncthreads();
    // 4 centres at a time: independent float64 chains (same per-centre
    // operation order, so the distances are bitwise those of one at a time)
    int c = 0;
    for (; c + 4 <= nc; c += 4) {
      const double* cc = cs + c * DM;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (k < d) {
          const double t0 = __dsub_rn(xr[k], cc[k]);
          const double t1 = __dsub_rn(xr[k], cc[DM + k]);
          const double t2 = __dsub_rn(xr[k], cc[2 * DM + k]);
          const double t3 = __dsub_rn(xr[k], cc[3 * DM + k]);
          s0 = __dadd_rn(s0, __dmul_rn(t0, t0));
          s1 = __dadd_rn(s1, __dmul_rn(t1, t1));
          s2 = __dadd_rn(s2, __dmul_rn(t2, t2));
          s3 = __dadd_rn(s3, __dmul_rn(t3, t3));
        }
      // strict: ties keep the lowest centre (and make second == best)
      if (s0 < best) { second = best; best = s0; bl = c0 + c; } else second = fmin(second, s0);
      if (s1 < best) { second = best; best = s1; bl = c0 + c + 1; } else second = fmin(second, s1);
      if (s2 < best) { second = best; best = s2; bl = c0 + c + 2; } else second = fmin(second, s2);
      if (s3 < best) { second = best; best = s3; bl = c0 + c + 3; } else second = fmin(second, s3);
    }
    for (; c < nc; ++c) {
      const double* cc = cs + c * DM;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < DM; ++k)
        if (k < d) {
          const double t = __dsub_rn(xr[k], cc[k]);
          s = __dadd_rn(s, __dmul_rn(t, t));
        }
      if (s < best) {
        second = best;
        best = s;
        bl = c0 + c;
      } else {
        second = fmin(second, s);
      }
    }
  }
  if (i < n) {
    labels[i] = static_cast<uint32_t>(bl);
    if (ub) {
      ub[i] = sqrt(best);
      lb[i] = sqrt(second);
    }
  }
}

// Hamerly's test before an assignment (labels, ub, lb from the previous one;
// the centres then moved by move[c], at most mmax): the nearest centre stays
// the same when ub + move[a] < max(lb - mmax, half the distance from c_a to
// its nearest other centre) — every other centre is then strictly farther,
// so the full scan (ties to the lowest index) would keep a.  An atom that
// fails is retried with its exact distance to c_a as the upper bound.  Margins
// of 1e-9 relative cover the float64 rounding of the distances (~1e-14).
// Atoms that still fail are listed for km_assign_kernel; the others keep
// their label, with the moved bounds.
__global__ void km_bounds_kernel(const double* x, int64_t n, int d, const double* centers,
                                 const uint32_t* labels, const double* move, const double* mmax,
                                 const double* half, double* ub, double* lb, int32_t* list,
                                 int32_t* count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t a = labels[i];
  double u = (ub[i] + move[a]) * (1.0 + 1e-9);
  const double l = (lb[i] - *mmax) * (1.0 - 1e-9);
  const double bound = fmax(l, half[a] * (1.0 - 1e-9));
  if (!(u < bound))  // tighten: the distance to the assigned centre itself
    u = sqrt(km_dist2(x + i * d, centers + static_cast<int64_t>(a) * d, d)) * (1.0 + 1e-9);
  if (u < bound) {
    ub[i] = u;
    lb[i] = l;
  } else {
    list[atomicAdd(count, 1)] = static_cast<int32_t>(i);
  }
}

// per-centre move |c_new - c_old| and its maximum; half the distance from
// each (new) centre to its nearest other centre.  One warp per centre.
__global__ void km_centre_geom_kernel(const double* old_c, const double* new_c, int K, int d,
                                      double* move, double* half, unsigned long long* mmax_bits) {
  const int lane = threadIdx.x & 31;
  const int c = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  if (c >= K) return;
  const double* cc = new_c + static_cast<int64_t>(c) * d;
  double mv = 0.0;
  for (int q = lane; q < d; q += 32) {
    const double t = cc[q] - old_c[static_cast<int64_t>(c) * d + q];
    mv = fma(t, t, mv);
  }
  for (int o = 16; o > 0; o >>= 1) mv += __shfl_xor_sync(0xffffffffu, mv, o);
  double nn = INFINITY;
  for (int e = 0; e < K; ++e) {
    if (e == c) continue;
    const double* ce = new_c + static_cast<int64_t>(e) * d;
    double s = 0.0;
    for (int q = lane; q < d; q += 32) {
      const double t = cc[q] - ce[q];
      s = fma(t, t, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    nn = fmin(nn, s);
  }
  if (lane == 0) {
    const double m = sqrt(mv);
    move[c] = m;
    half[c] = 0.5 * sqrt(nn);
    // non-negative doubles order as their bit patterns
    atomicMax(mmax_bits, static_cast<unsigned long long>(__double_as_longlong(m)));
  }
}

// mass-weighted centroids: one thread per (cluster, coordinate), sequential
// over the cluster's atoms (sorted by label, stable: index order); empty
// clusters keep their centre.  move[I] = |c_new - c_old|^2 (coordinate 0's
// thread, after the others finished via a second kernel).
__global__ void km_centroid_kernel(const double* x, const double* w, const int32_t* perm,
                                   const int32_t* off, int K, int d, const double* old_c,
                                   double* new_c, double* cw) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= static_cast<int64_t>(K) * d) return;
  const int I = static_cast<int>(g / d), q = static_cast<int>(g % d);
  const int32_t s0 = off[I], s1 = off[I + 1];
  if (s1 <= s0) {
    new_c[g] = old_c[g];
    if (q == 0) cw[I] = 0.0;
    return;
  }
  double W = 0.0, S = 0.0;
  for (int32_t s = s0; s < s1; ++s) {
    const int64_t i = perm[s];
    W = __dadd_rn(W, w[i]);
    S = __dadd_rn(S, __dmul_rn(w[i], x[i * d + q]));
  }
  new_c[g] = __ddiv_rn(S, W);
  if (q == 0) cw[I] = W;
}

__global__ void km_move_kernel(const double* a, const double* b, int K, int d, double* out) {
  __shared__ double sm[256];
  double m = 0.0;
  for (int I = threadIdx.x; I < K; I += blockDim.x) m = fmax(m, km_dist2(a + static_cast<int64_t>(I) * d, b + static_cast<int64_t>(I) * d, d));
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

// radius of each cluster: max |x - c| over its atoms, rounded up to float
__global__ void km_radius_kernel(const double* x, const int32_t* perm, const int32_t* off, int K,
                                 int d, const double* c, float* radii) {
  const int lane = threadIdx.x & 31;
  const int64_t I = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (I >= K) return;
  double r = 0.0;
  for (int32_t s = off[I] + lane; s < off[I + 1]; s += 32)
    r = fmax(r, km_dist2(x + static_cast<int64_t>(perm[s]) * d, c + I * d, d));
  for (int o = 16; o > 0; o >>= 1) r = fmax(r, __shfl_xor_sync(0xffffffffu, r, o));
  if (lane == 0) {
    const double rr = __dsqrt_ru(r);
    float f = __double2float_ru(rr);
    radii[I] = f;
  }
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

// offsets of the label-sorted atoms: off[I] = first sorted position of label I
__global__ void km_offsets_kernel(const uint32_t* sorted_labels, int64_t n, int K, int32_t* off) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const uint32_t l = sorted_labels[s];
  const uint32_t prev = s == 0 ? 0xffffffffu : sorted_labels[s - 1];
  if (s == 0)
    for (uint32_t q = 0; q <= l; ++q) off[q] = 0;
  else if (l != prev)
    for (uint32_t q = prev + 1; q <= l; ++q) off[q] = static_cast<int32_t>(s);
  if (s == n - 1)
    for (uint32_t q = l + 1; q <= static_cast<uint32_t>(K); ++q) off[q] = static_cast<int32_t>(n);
}

// scratch: see kmeans_ws_bytes
cudaError_t kmeans(const double* x, const double* w, int64_t n, int d, int K, uint64_t seed,
                   double tol2, int max_iter, void* ws, int32_t* perm, int32_t* off,
                   uint32_t* labels, double* centers, double* cw, float* radii, int* iters,
                   cudaStream_t st) {
  if (n <= 0 || K <= 0 || K > n || d < 1 || d > kKmDmax) return cudaErrorInvalidValue;
  const int nb = static_cast<int>((n + 255) / 256);
  char* p = static_cast<char*>(ws);
  double* mind = reinterpret_cast<double*>(p);
  p += n * sizeof(double);
  double* bval = reinterpret_cast<double*>(p);
  p += nb * sizeof(double);
  int64_t* bidx = reinterpret_cast<int64_t*>(p);
  p += nb * sizeof(int64_t);
  double* c2 = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(K) * d * sizeof(double);
  double* mv = reinterpret_cast<double*>(p);
  p += 2 * sizeof(double);
  uint32_t* keys = reinterpret_cast<uint32_t*>(p);
  p += n * sizeof(uint32_t);
  // Hamerly bounds: distance to the nearest / second-nearest centre, the
  // centres' moves and half nearest-centre distances, the list of atoms to
  // rescan and its length, the largest move (as ordered bits)
  p += (16 - reinterpret_cast<uintptr_t>(p) % 16) % 16;
  double* ub = reinterpret_cast<double*>(p);
  p += n * sizeof(double);
  double* lb = reinterpret_cast<double*>(p);
  p += n * sizeof(double);
  double* cmove = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(K) * sizeof(double);
  double* chalf = reinterpret_cast<double*>(p);
  p += static_cast<size_t>(K) * sizeof(double);
  unsigned long long* mmax = reinterpret_cast<unsigned long long*>(p);
  p += sizeof(unsigned long long);
  int32_t* cnt = reinterpret_cast<int32_t*>(p);
  p += 2 * sizeof(int32_t);
  int32_t* list = reinterpret_cast<int32_t*>(p);
  p += n * sizeof(int32_t);
  p += (256 - reinterpret_cast<uintptr_t>(p) % 256) % 256;
  void* rtmp = p;
  // farthest-point seeding (the atoms' nearest-centre index lives in `keys`,
  // the new centre's distances to the earlier ones in `c2`, both free until
  // Lloyd)
  int32_t* asg = reinterpret_cast<int32_t*>(keys);
  double* dnew = c2;
  ++g_launches;
  copy_center_kernel<<<1, 64, 0, st>>>(x, static_cast<int64_t>(seed % static_cast<uint64_t>(n)), d,
                                       centers);
  for (int k = 1; k < K; ++k) {
    ++g_launches;
    fps_update_kernel<<<nb, 256, 0, st>>>(x, n, d, centers + static_cast<int64_t>(k - 1) * d, k - 1,
                                          mind, asg, dnew, k == 1, bval, bidx);
    ++g_launches;
    fps_select_kernel<<<1, 256, 0, st>>>(bval, bidx, nb, x, d, centers, k);
    if (k + 1 < K) {
      ++g_launches;
      fps_ccdist_kernel<<<(k + 7) / 8, 256, 0, st>>>(centers, d, k, dnew);
    }
  }
  const int kb = static_cast<int>((static_cast<int64_t>(K) * d + 255) / 256);
  int it = 0;
  const int key_bits = K <= 1 ? 1 : 32 - __builtin_clz(static_cast<unsigned>(K - 1));
  for (;;) {
    // assignment to the current centres (after the first: only the atoms
    // Hamerly's test cannot keep), then the clusters in index order
    const int32_t* sl = nullptr;
    if (it > 0) {
      cudaError_t e0 = cudaMemsetAsync(cnt, 0, sizeof(int32_t), st);
      if (e0 != cudaSuccess) return e0;
      ++g_launches;
      km_bounds_kernel<<<nb, 256, 0, st>>>(x, n, d, centers, labels, cmove,
                                           reinterpret_cast<const double*>(mmax), chalf, ub, lb,
                                           list, cnt);
      sl = list;
    }
    const unsigned ab = static_cast<unsigned>((n + 127) / 128);
    ++g_launches;
    if (d <= 16)
      km_assign_kernel<16><<<ab, 128, 0, st>>>(x, n, d, centers, K, labels, sl, cnt, ub, lb);
    else if (d <= 32)
      km_assign_kernel<32><<<ab, 128, 0, st>>>(x, n, d, centers, K, labels, sl, cnt, ub, lb);
    else
      km_assign_kernel<64><<<ab, 128, 0, st>>>(x, n, d, centers, K, labels, sl, cnt, ub, lb);
    cudaError_t e = cudaMemcpyAsync(keys, labels, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    ++g_launches;
    iota_kernel<<<nb, 256, 0, st>>>(perm, n);
    e = radix_sort_pairs(keys, perm, n, key_bits, rtmp, st);
    if (e != cudaSuccess) return e;
    ++g_launches;
    km_offsets_kernel<<<nb, 256, 0, st>>>(keys, n, K, off);
    ++it;
    // mass-weighted means of this assignment become the centres
    ++g_launches;
    km_centroid_kernel<<<kb, 256, 0, st>>>(x, w, perm, off, K, d, centers, c2, cw);
    ++g_launches;
    km_move_kernel<<<1, 256, 0, st>>>(centers, c2, K, d, mv);
    // the moves and centre spacing the next assignment's bounds need
    e = cudaMemsetAsync(mmax, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    ++g_launches;
    km_centre_geom_kernel<<<static_cast<unsigned>((static_cast<int64_t>(K) * 32 + 255) / 256), 256, 0,
                            st>>>(centers, c2, K, d, cmove, chalf, mmax);
    e = cudaMemcpyAsync(centers, c2, static_cast<size_t>(K) * d * sizeof(double),
                        cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
    double hm = 0.0;
    e = cudaMemcpyAsync(&hm, mv, sizeof(double), cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    if (hm < tol2 || it >= max_iter) break;
  }
  ++g_launches;
  km_radius_kernel<<<static_cast<unsigned>((static_cast<int64_t>(K) * 32 + 255) / 256), 256, 0, st>>>(
      x, perm, off, K, d, centers, radii);
  if (iters) *iters = it;
  return cudaGetLastError();
}

// ---- padded cluster layout of the high-D multiscale solver ---------------
// Cluster I occupies rows [poff[I], poff[I+1]) (its atoms in index order, then
// padding up to a multiple of 128 — the tcgen05 kernel's column block).
// src[p] = caller index of slot p, or -(I+1) for a padding slot of cluster I,
// which takes the centroid's coordinates (finite, harmless sums) and weight 0.
__global__ void hd_gather_padded_kernel(const double* x, const double* centers, const int32_t* src,
                                        int64_t npad, int d, double* out) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= npad * d) return;
  const int64_t p = g / d;
  const int q = static_cast<int>(g - p * d);
  const int32_t s = src[p];
  out[g] = s >= 0 ? x[static_cast<int64_t>(s) * d + q] : centers[static_cast<int64_t>(-s - 1) * d + q];
}

__global__ void hd_padded_weights_kernel(const double* w, const int32_t* src, int64_t npad,
                                         float* lw2, double* w64) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= npad) return;
  const int32_t s = src[p];
  const double wi = s >= 0 ? w[s] : 0.0;
  lw2[p] = s >= 0 ? __double2float_rn(log2(wi)) : __int_as_float(0xff800000);
  w64[p] = wi;
}

// per-cluster max of a potential over the cluster's real atoms (weight > 0)
__global__ void hd_cluster_fmax_kernel(const float* f, const double* w64, const int32_t* off, int K,
                                       float* fmax) {
  const int lane = threadIdx.x & 31;
  const int64_t I = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (I >= K) return;
  float m = -INFINITY;
  for (int32_t s = off[I] + lane; s < off[I + 1]; s += 32)
    if (w64[s] > 0.0) m = fmaxf(m, f[s]);
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) fmax[I] = m;
}

cudaError_t hd_gather_padded(const double* x, const double* centers, const int32_t* src,
                             int64_t npad, int d, double* out, cudaStream_t st) {
  if (npad <= 0) return cudaSuccess;
  ++g_launches;
  hd_gather_padded_kernel<<<static_cast<unsigned>((npad * d + 255) / 256), 256, 0, st>>>(
      x, centers, src, npad, d, out);
  return cudaGetLastError();
}

cudaError_t hd_padded_weights(const double* w, const int32_t* src, int64_t npad, float* lw2,
                              double* w64, cudaStream_t st) {
  if (npad <= 0) return cudaSuccess;
  ++g_launches;
  hd_padded_weights_kernel<<<static_cast<unsigned>((npad + 255) / 256), 256, 0, st>>>(w, src, npad,
                                                                                     lw2, w64);
  return cudaGetLastError();
}

cudaError_t hd_cluster_fmax(const float* f, const double* w64, const int32_t* off, int K,
                            float* fmax, cudaStream_t st) {
  if (K <= 0) return cudaSuccess;
  ++g_launches;
  hd_cluster_fmax_kernel<<<static_cast<unsigned>((static_cast<int64_t>(K) * 32 + 255) / 256), 256, 0,
                           st>>>(f, w64, off, K, fmax);
  return cudaGetLastError();
}

size_t kmeans_ws_bytes(int64_t n, int d, int K) {
  const int64_t nb = (n + 255) / 256;
  return static_cast<size_t>(n) * sizeof(double) + nb * (sizeof(double) + sizeof(int64_t)) +
         static_cast<size_t>(K) * d * sizeof(double) + 2 * sizeof(double) +
         static_cast<size_t>(n) * sizeof(uint32_t) +
         // Hamerly bounds, moves, half spacings, max move, count, rescan list
         2 * static_cast<size_t>(n) * sizeof(double) + 2 * static_cast<size_t>(K) * sizeof(double) +
         sizeof(unsigned long long) + 2 * sizeof(int32_t) + static_cast<size_t>(n) * sizeof(int32_t) +
         256 + radix_temp_bytes(n) + 256;
}

}  // namespace msot_dev
