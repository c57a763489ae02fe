// prims.cu — device primitives: prefix scans, bounding box, stable LSD radix
// sort.  Hand-written (no CUB): the voxel-grid clustering of the north star
// is "a radix sort by cube id" and must be bit-reproducible.
#include <cfloat>

#include "common.cuh"
#include "prims.cuh"

namespace msot_dev {

// ---------------------------------------------------------------- scans ---
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

template <typename T>
__device__ T block_exclusive_scan(T v, T* sh, T* total) {
  // warp inclusive
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    T w = lane < nw ? sh[lane] : T(0);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < nw) sh[lane] = w;
  }
  __syncthreads();
  const T wpre = warp > 0 ? sh[warp - 1] : T(0);
  if (total) *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return wpre + x - v;
}

template <typename TI, typename TO>
__global__ void scan_reduce(const TI* in, int64_t n, TO* sums) {
  __shared__ TO sh[32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  TO acc = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t g = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    if (g < n) acc += static_cast<TO>(in[g]);
  }
  TO tot;
  block_exclusive_scan<TO>(acc, sh, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

template <typename TO>
__global__ void scan_sums(TO* sums, int64_t nb, TO* total_out) {
  __shared__ TO sh[32];
  __shared__ TO carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += blockDim.x) {
    const int64_t g = base + threadIdx.x;
    TO v = g < nb ? sums[g] : TO(0);
    TO tot;
    TO ex = block_exclusive_scan<TO>(v, sh, &tot);
    if (g < nb) sums[g] = ex + carry;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && total_out) *total_out = carry;
}

template <typename TI, typename TO>
__global__ void scan_apply(const TI* in, int64_t n, const TO* sums, TO* out, int inclusive) {
  __shared__ TO sh[32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
  TO v[kScanItems];
  TO acc = 0;
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t g = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    v[i] = g < n ? static_cast<TO>(in[g]) : TO(0);
    acc += v[i];
  }
  TO pre = block_exclusive_scan<TO>(acc, sh, nullptr) + sums[blockIdx.x];
  for (int i = 0; i < kScanItems; ++i) {
    const int64_t g = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
    if (inclusive) pre += v[i];
    if (g < n) out[g] = pre;
    if (!inclusive) pre += v[i];
  }
}

// Small inputs (<= kScanSingleTiles tiles): one block walks the tiles in
// order with a running carry — one launch instead of three (the pair-set
// builds scan many short per-tile arrays).  Same integer sums.
constexpr int64_t kScanSingleTiles = 16;
template <typename TI, typename TO>
__global__ void __launch_bounds__(kScanThreads) scan_single(const TI* in, int64_t n, TO* out,
                                                            int inclusive, TO* total) {
  __shared__ TO sh[32];
  TO carry = 0;
  for (int64_t base = 0; base < n; base += kScanTile) {
    TO v[kScanItems];
    TO acc = 0;
    for (int i = 0; i < kScanItems; ++i) {
      const int64_t g = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
      v[i] = g < n ? static_cast<TO>(in[g]) : TO(0);
      acc += v[i];
    }
    TO tot;
    TO pre = block_exclusive_scan<TO>(acc, sh, &tot) + carry;
    for (int i = 0; i < kScanItems; ++i) {
      const int64_t g = base + static_cast<int64_t>(threadIdx.x) * kScanItems + i;
      if (inclusive) pre += v[i];
      if (g < n) out[g] = pre;
      if (!inclusive) pre += v[i];
    }
    carry += tot;
  }
  if (threadIdx.x == 0 && total) *total = carry;
}

size_t scan_temp_elems(int64_t n) { return static_cast<size_t>((n + kScanTile - 1) / kScanTile) + 1; }

template <typename TI, typename TO>
cudaError_t scan(const TI* in, TO* out, int64_t n, bool inclusive, TO* tmp, TO* total,
                 cudaStream_t st) {
  if (n <= 0) {
    if (total) return cudaMemsetAsync(total, 0, sizeof(TO), st);
    return cudaSuccess;
  }
  const int64_t nb = (n + kScanTile - 1) / kScanTile;
  if (nb <= kScanSingleTiles) {
    ++g_launches;
    scan_single<TI, TO><<<1, kScanThreads, 0, st>>>(in, n, out, inclusive ? 1 : 0, total);
    return cudaGetLastError();
  }
  ++g_launches; scan_reduce<TI, TO><<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(in, n, tmp);
  ++g_launches; scan_sums<TO><<<1, 1024, 0, st>>>(tmp, nb, total);
  ++g_launches; scan_apply<TI, TO><<<static_cast<unsigned>(nb), kScanThreads, 0, st>>>(in, n, tmp, out,
                                                                           inclusive ? 1 : 0);
  return cudaGetLastError();
}

template cudaError_t scan<int32_t, int32_t>(const int32_t*, int32_t*, int64_t, bool, int32_t*,
                                            int32_t*, cudaStream_t);
template cudaError_t scan<int32_t, int64_t>(const int32_t*, int64_t*, int64_t, bool, int64_t*,
                                            int64_t*, cudaStream_t);
template cudaError_t scan<int64_t, int64_t>(const int64_t*, int64_t*, int64_t, bool, int64_t*,
                                            int64_t*, cudaStream_t);
template cudaError_t scan<uint8_t, int32_t>(const uint8_t*, int32_t*, int64_t, bool, int32_t*,
                                            int32_t*, cudaStream_t);

// ----------------------------------------------------------- bounding box --
// float64 min/max are exact, so the joint bounding box is
// bit-identical to the host's.  Ordered-int64 atomics make it order-free.
__device__ __forceinline__ long long dkey(double v) {
  long long b = __double_as_longlong(v);
  return b >= 0 ? b : (b ^ 0x7fffffffffffffffLL);
}
__host__ __device__ inline double dkey_inv(long long k) {
  long long b = k >= 0 ? k : (k ^ 0x7fffffffffffffffLL);
  double v;
  memcpy(&v, &b, sizeof(v));
  return v;
}

__global__ void bbox_kernel(const double* x, int64_t n, int d, long long* lohi) {
  // lohi[2k] = min key of dim k, lohi[2k+1] = max key
  for (int k = 0; k < d; ++k) {
    double lo = DBL_MAX, hi = -DBL_MAX;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
      const double v = x[i * d + k];
      if (!isfinite(v)) {  // non-finite input: the box becomes [-inf, inf] (DataError)
        lo = -INFINITY;
        hi = INFINITY;
      }
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&lohi[2 * k], dkey(lo));
      atomicMax(&lohi[2 * k + 1], dkey(hi));
    }
  }
}

__global__ void bbox_init(long long* lohi, int d) {
  for (int k = threadIdx.x; k < d; k += blockDim.x) {
    lohi[2 * k] = 0x7fffffffffffffffLL;
    lohi[2 * k + 1] = -0x7fffffffffffffffLL - 1;
  }
}

cudaError_t bbox(const double* x, int64_t n, int d, long long* lohi_dev, bool init,
                 cudaStream_t st) {
  if (init) { ++g_launches; bbox_init<<<1, 32, 0, st>>>(lohi_dev, d); }
  if (n > 0) {
    int64_t nb0 = (n + 255) / 256;
    int blocks = static_cast<int>(nb0 < 592 ? nb0 : 592);
    ++g_launches; bbox_kernel<<<blocks, 256, 0, st>>>(x, n, d, lohi_dev);
  }
  return cudaGetLastError();
}

// Weights that are not finite and > 0 (counted into *bad).
__global__ void bad_weights_kernel(const double* w, int64_t n, int32_t* bad) {
  int32_t c = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += !(w[i] > 0.0 && isfinite(w[i]));
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, c);
}

cudaError_t count_bad_weights(const double* w, int64_t n, int32_t* bad, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t nb0 = (n + 255) / 256;
  ++g_launches;
  bad_weights_kernel<<<static_cast<int>(nb0 < 592 ? nb0 : 592), 256, 0, st>>>(w, n, bad);
  return cudaGetLastError();
}

void bbox_decode(const long long* lohi_host, int d, double* lo, double* hi) {
  for (int k = 0; k < d; ++k) {
    lo[k] = dkey_inv(lohi_host[2 * k]);
    hi[k] = dkey_inv(lohi_host[2 * k + 1]);
  }
}

// ------------------------------------------------------- LSD radix sort ---
// Stable sort of (key, value) pairs by 8-bit digits.  Per pass: digit
// histogram per block, one exclusive scan over the digit-major histogram,
// then an order-preserving scatter (warp match for ranks inside a warp, warp
// counts in shared memory for ranks across warps, a running per-digit offset
// across the block's rounds).
constexpr int kRsThreads = 256;
constexpr int kRsRounds = 16;
constexpr int kRsTile = kRsThreads * kRsRounds;  // keys per block
constexpr int kRsWarps = kRsThreads / 32;

__global__ void rs_hist(const uint32_t* keys, int64_t n, int shift, int32_t* hist, int nblocks) {
  __shared__ int32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t g = base + r * kRsThreads + threadIdx.x;
    if (g < n) atomicAdd(&h[(keys[g] >> shift) & 255u], 1);
  }
  __syncthreads();
  hist[static_cast<int64_t>(threadIdx.x) * nblocks + blockIdx.x] = h[threadIdx.x];
}

__global__ void rs_scatter(const uint32_t* kin, const int32_t* vin, uint32_t* kout,
                           int32_t* vout, int64_t n, int shift, const int32_t* offs,
                           int nblocks) {
  __shared__ int32_t run[256];
  __shared__ int32_t wcnt[kRsWarps][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  run[threadIdx.x] = offs[static_cast<int64_t>(threadIdx.x) * nblocks + blockIdx.x];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kRsTile;
  for (int r = 0; r < kRsRounds; ++r) {
    for (int w = 0; w < kRsWarps; ++w) wcnt[w][threadIdx.x] = 0;
    __syncthreads();
    const int64_t g = base + r * kRsThreads + threadIdx.x;
    const bool valid = g < n;
    const uint32_t key = valid ? kin[g] : 0xffffffffu;
    const int32_t val = valid ? vin[g] : 0;
    const unsigned dg = valid ? ((key >> shift) & 255u) : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, dg);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank == 0) wcnt[warp][dg] = __popc(peers);
    __syncthreads();
    if (valid) {
      int pos = run[dg] + rank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][dg];
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    int add = 0;
    for (int w = 0; w < kRsWarps; ++w) add += wcnt[w][threadIdx.x];
    run[threadIdx.x] += add;
    __syncthreads();
  }
}

size_t radix_temp_bytes(int64_t n) {
  const int64_t nb = (n + kRsTile - 1) / kRsTile;
  const int64_t hn = 256 * nb;
  return static_cast<size_t>(hn) * sizeof(int32_t) * 2 + scan_temp_elems(hn) * sizeof(int32_t) +
         static_cast<size_t>(n) * (sizeof(uint32_t) + sizeof(int32_t)) + 256;
}

cudaError_t radix_sort_pairs(uint32_t* keys, int32_t* vals, int64_t n, int key_bits, void* temp,
                             cudaStream_t st) {
  if (n <= 1) return cudaSuccess;
  const int nb = static_cast<int>((n + kRsTile - 1) / kRsTile);
  const int64_t hn = 256LL * nb;
  char* p = static_cast<char*>(temp);
  int32_t* hist = reinterpret_cast<int32_t*>(p);
  p += hn * sizeof(int32_t);
  int32_t* offs = reinterpret_cast<int32_t*>(p);
  p += hn * sizeof(int32_t);
  int32_t* stmp = reinterpret_cast<int32_t*>(p);
  p += scan_temp_elems(hn) * sizeof(int32_t);
  uint32_t* k2 = reinterpret_cast<uint32_t*>(p);
  p += n * sizeof(uint32_t);
  int32_t* v2 = reinterpret_cast<int32_t*>(p);
  uint32_t *ka = keys, *kb = k2;
  int32_t *va = vals, *vb = v2;
  int passes = 0;
  for (int shift = 0; shift < key_bits; shift += 8, ++passes) {
    ++g_launches; rs_hist<<<nb, kRsThreads, 0, st>>>(ka, n, shift, hist, nb);
    cudaError_t e = scan<int32_t, int32_t>(hist, offs, hn, false, stmp, nullptr, st);
    if (e != cudaSuccess) return e;
    ++g_launches; rs_scatter<<<nb, kRsThreads, 0, st>>>(ka, va, kb, vb, n, shift, offs, nb);
    uint32_t* tk = ka; ka = kb; kb = tk;
    int32_t* tv = va; va = vb; vb = tv;
  }
  if (passes & 1) {
    cudaMemcpyAsync(keys, ka, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(vals, va, n * sizeof(int32_t), cudaMemcpyDeviceToDevice, st);
  }
  return cudaGetLastError();
}

}  // namespace msot_dev
