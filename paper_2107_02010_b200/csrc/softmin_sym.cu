// softmin_sym.cu — K4s: the evaluate-once block-sparse softmin.  Each kept
// pair (i, j) is exponentiated once and feeds both potentials it belongs to:
//
//   row i    s_i = sum_j w_j 2^{E_ij}                       (the K4 row sum)
//   column j t_j = sum_i a_i 2^{E'_ij},  E'_ij - E_ij = (lw2_i - ell (est_i - est_mid))
//                                                     + (ell (h_j - est_mid) - lw2_j)
//
// with E_ij the row exponent of softmin.cu (reference est_i / lambda) and E'_ij
// the exponent of pair (j, i) in the transposed problem (reference h_j /
// lambda); ell = (1/lambda - 1) / (eps ln2) (0 for reach = inf).  The two
// differ by a row factor and a column factor, so one MUFU.EX2 per pair serves
// both updates (the cross pair a_xy / b_yx shares its
// kernel matrix, and the self kernels are symmetric).  This halves the MUFU
// work that bounds the solver.
//
// Per 16 columns a warp reduces its 32 x 2 rows with a 5-step transpose
// butterfly (one shuffle per column per warp), the 4 warps combine through
// shared memory in a fixed order, and thread c writes column c's CTA partial
// to its (tile, position) slot.  Column totals are formed by
// sym_colsum_kernel in tile order (deterministic for a fixed GPU count).
#include "prims.cuh"
#include "softmin_inner.cuh"

namespace msot_dev {

// Sum over the 32 lanes of 16 per-lane values.  Lane l returns the warp
// total of value q(l) = 8 b4 + 4 b3 + 2 b2 + b1 (bits of l; l, l^1 agree).
__device__ __forceinline__ float warp_sum16(float (&v)[16], int lane) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const bool up = lane & 16;
    const float send = up ? v[i] : v[i + 8];
    const float keep = up ? v[i + 8] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = lane & 8;
    const float send = up ? v[i] : v[i + 4];
    const float keep = up ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = lane & 4;
    const float send = up ? v[i] : v[i + 2];
    const float keep = up ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool up = lane & 2;
    const float send = up ? v[0] : v[1];
    const float keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__device__ __forceinline__ int warp_sum16_col(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}

// One CTA = one work item (256 rows x a run of the tile's columns), 64
// threads with 4 rows each: a staged column pair is read once per 4 rows and
// the column butterfly is shared by 128 rows per warp.
constexpr int kSymThreads = 64;
constexpr int kSymRows = kTileRows / kSymThreads;  // 4
constexpr int kSymColsPerThread = 2;
constexpr int kSymCols = kSymThreads * kSymColsPerThread;  // columns staged per buffer
static_assert(kSymRows == 4, "softmin_sym_kernel is written for 4 rows per thread");

// kUni: every row weight equal and lambda = 1, so the row factor is one
// constant per CTA, applied at the column write-out (the column partial of a
// column pair is the packed sum of the 4 rows' terms).
// (All exponentials on the MUFU: moving 2/16 of them to the FMA pipe, which
// pays +1.4% in the row-wise softmin_kernel, costs 8% here — the FMA pipe
// carries the column sums.)
template <int D, bool kUni>
__global__ void __launch_bounds__(kSymThreads)
softmin_sym_kernel(const __grid_constant__ Group G) {
  __shared__ __align__(16) float smem[2][kSymCols * 4];
  __shared__ float colacc[kSymThreads / 32][kSymCols];
  const int it = blockIdx.x;
  if (it >= G.n_items) return;
  const int4 item = G.items[it];
  const Problem& P = G.P[item.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row_base = P.tile_start[item.y];
  const int row_end = P.tile_start[item.y + 1];
  const int mid = (row_base + row_end) >> 1;
  const float4 o = P.rows[mid];
  const float est_mid = P.row_est ? P.row_est[mid] : 0.f;
  const float R = est_mid * P.inv_lam_eps_ln2;  // tile reference (softmin.cu)

  RowState rs[kSymRows];
  float2 W[kSymRows];
#pragma unroll
  for (int q = 0; q < kSymRows; ++q) {
    const int r = row_base + tid + q * kSymThreads;
    load_row<D>(P, r, row_end, o, R, rs[q]);
    // padding rows contribute exactly 0 (rows and columns)
    if (r >= row_end) rs[q].r = __int_as_float(0xff800000);
    float wq = 0.f;
    if (!kUni && r < row_end) {
      // column-sum row factor a_i 2^{-ell (est_i - est_mid)}
      const float est = P.row_est ? P.row_est[r] : 0.f;
      wq = exp2f(P.row_lw2[r] - P.ell * (est - est_mid));
    }
    W[q] = make_float2(wq, wq);
  }
  const float wu = kUni ? exp2f(P.row_lw2[row_base]) : 0.f;

  ColWalker w{P.ranges, P.tile_rptr[item.y], P.tile_rptr[item.y + 1], 0};
  const int32_t pos_begin = item.z, pos_end = item.w;
  float* colout = P.colpart + P.tile_slot[item.y];

  // each thread fetches and stages columns tid + 64 q of every 128-column stage
  float4 cv[kSymColsPerThread];
  float ch[kSymColsPerThread], cl[kSymColsPerThread];
  bool cvalid[kSymColsPerThread];
  auto fetch = [&](int32_t tile_pos) {
#pragma unroll
    for (int q = 0; q < kSymColsPerThread; ++q) {
      const int32_t pos = tile_pos + tid + q * kSymThreads;
      cvalid[q] = false;
      if (pos < pos_end) {
        const int j = w.col(pos);
        if (j >= 0) {
          cv[q] = __ldg(P.cols + j);
          cl[q] = __ldg(P.col_lw2 + j);
          ch[q] = __ldg(P.col_h + j);
          cvalid[q] = true;
        }
      }
    }
  };
  float cfac[kSymColsPerThread];  // column factors of the columns this thread staged
  auto stage = [&](float* buf) {
#pragma unroll
    for (int q = 0; q < kSymColsPerThread; ++q) {
      const int cidx = tid + q * kSymThreads;
      float* rec = buf + (cidx >> 1) * 8 + (cidx & 1);
      if (cvalid[q]) {
        const float a = (cv[q].x - o.x) * P.sc;
        const float b = D > 1 ? (cv[q].y - o.y) * P.sc : 0.f;
        const float c = D > 2 ? (cv[q].z - o.z) * P.sc : 0.f;
        rec[0] = a;
        rec[2] = b;
        rec[4] = c;
        rec[6] = (fmaf(ch[q], P.inv_eps_ln2, R) + cl[q]) - fmaf(a, a, fmaf(b, b, c * c));
        cfac[q] = exp2f(P.ell * (ch[q] - est_mid) - cl[q]);
      } else {
        rec[0] = 0.f;
        rec[2] = 0.f;
        rec[4] = 0.f;
        rec[6] = __int_as_float(0xff800000);  // -inf -> exp2(-inf) = 0
        cfac[q] = 0.f;
      }
    }
  };

  float2 sum[kSymRows];
#pragma unroll
  for (int q = 0; q < kSymRows; ++q) sum[q] = make_float2(0.f, 0.f);
  int buf = 0;
  fetch(pos_begin);
  for (int32_t tp = pos_begin; tp < pos_end; tp += kSymCols) {
    stage(smem[buf]);
    __syncthreads();
    if (tp + kSymCols < pos_end) fetch(tp + kSymCols);
    const float4* s4 = reinterpret_cast<const float4*>(smem[buf]);
#pragma unroll 2  // (1: +1% time; 4: 110 registers, +3%)
    for (int c0 = 0; c0 < kSymCols / 2; c0 += 8) {
      float v[16];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = c0 + k;
        const float4 A = s4[2 * c], B = s4[2 * c + 1];
        const float2 Y0 = make_float2(A.x, A.y);
        const float2 Y1 = make_float2(A.z, A.w);
        const float2 Y2 = make_float2(B.x, B.y);
        const float2 C = make_float2(B.z, B.w);
        float2 e[kSymRows];
#pragma unroll
        for (int q = 0; q < kSymRows; ++q) {
          e[q] = pair_terms<D, false>(rs[q], Y0, Y1, Y2, C);
          sum[q] = __fadd2_rn(sum[q], e[q]);
        }
        float2 cp;
        if (kUni) {
          cp = __fadd2_rn(__fadd2_rn(e[0], e[1]), __fadd2_rn(e[2], e[3]));
        } else {
          cp = __fmul2_rn(W[0], e[0]);
          cp = __ffma2_rn(W[1], e[1], cp);
          cp = __ffma2_rn(W[2], e[2], cp);
          cp = __ffma2_rn(W[3], e[3], cp);
        }
        v[2 * k] = cp.x;
        v[2 * k + 1] = cp.y;
      }
      const float cs = warp_sum16(v, lane);
      if ((lane & 1) == 0) colacc[warp][2 * c0 + warp_sum16_col(lane)] = cs;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kSymColsPerThread; ++q) {
      const int cidx = tid + q * kSymThreads;
      const int32_t pos = tp + cidx;
      if (pos < pos_end) {
        float s = colacc[0][cidx];
#pragma unroll
        for (int k = 1; k < kSymThreads / 32; ++k) s += colacc[k][cidx];
        colout[pos] = kUni ? s * (cfac[q] * wu) : s * cfac[q];
      }
    }
    buf ^= 1;
  }
  float* out = G.part + static_cast<int64_t>(it) * kTileRows;
#pragma unroll
  for (int q = 0; q < kSymRows; ++q) out[tid + q * kSymThreads] = sum[q].x + sum[q].y;
}

// Column totals (ColSum, prims.cuh): for every column j (cluster J =
// labels[j], offset j - co[J]), the sum over the cluster's entries (tiles in
// ascending order, this rank's tiles [t0, t1) only; self problems: only
// tiles that end at or before j) of colpart[eslot + offset], in float64.
// Batched (bounded colpart): [t0, t1) is the batch's tile
// range, found in the cluster's tile-ordered entries by binary search, and
// the float64 running total carries across batches in `acc` — the same
// additions in the same order as one pass, so the bits do not depend on
// the batch size.
__global__ void sym_colsum_kernel(const __grid_constant__ ColSumGroup g) {
  const ColSum& a = g.c[blockIdx.y];
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n_cols) return;
  const int32_t J = a.labels[j];
  const int32_t off = j - a.co[J];
  int64_t e = a.eptr[static_cast<int64_t>(J) * kEntryChunks];
  int64_t e1 = a.eptr[static_cast<int64_t>(J + 1) * kEntryChunks];
  {  // first entry with tile >= t0, then stop at tile >= t1
    int64_t lo = e, hi = e1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (a.etile[mid] < a.t0) lo = mid + 1; else hi = mid;
    }
    e = lo;
  }
  double s = (a.acc && !a.first) ? a.acc[j] : 0.0;
  // entries are in ascending tile order, so both stopping rules end the
  // walk: tile >= t1 (batch end), and for self problems the first tile that
  // ends after j (so do all later ones).  Eight entries' loads in flight per
  // step, added in entry order (the bits of the one-at-a-time loop).
  const int32_t tend = a.t1;
  auto stop = [&](int32_t t) { return t >= tend || (a.self && a.tile_start[t + 1] > j); };
  constexpr int kAhead = 8;
  for (; e + kAhead <= e1; e += kAhead) {
    if (stop(a.etile[e + kAhead - 1])) break;  // the last decides for all (ascending)
    float v[kAhead];
#pragma unroll
    for (int u = 0; u < kAhead; ++u) v[u] = a.colpart[a.eslot[e + u] + off];
#pragma unroll
    for (int u = 0; u < kAhead; ++u) s += static_cast<double>(v[u]);
  }
  for (; e < e1; ++e) {
    if (stop(a.etile[e])) break;
    s += static_cast<double>(a.colpart[a.eslot[e] + off]);
  }
  // (tot null: a multi-rank group keeps the float64 total for the exchange)
  if ((a.last || !a.acc) && a.tot) a.tot[j] = static_cast<float>(s);
  else a.acc[j] = s;
}

// Column totals exchanged in float64 (multi-rank): tot = float(acc) after the
// all-reduce, the one rounding a single-rank solve makes.
__global__ void totals_f32_kernel(const double* acc, float* tot, int32_t n) {
  const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n) tot[j] = static_cast<float>(acc[j]);
}

cudaError_t totals_f32(const double* acc, float* tot, int32_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  ++g_launches;
  totals_f32_kernel<<<(n + 255) / 256, 256, 0, st>>>(acc, tot, n);
  return cudaGetLastError();
}

cudaError_t launch_colsum(const ColSum* c, int n, cudaStream_t st) {
  ColSumGroup g{};
  int32_t mx = 0;
  for (int k = 0; k < n; ++k) {
    g.c[k] = c[k];
    mx = max(mx, c[k].n_cols);
  }
  g.n = n;
  if (n <= 0 || mx <= 0) return cudaSuccess;
  ++g_launches;
  sym_colsum_kernel<<<dim3((mx + 255) / 256, n), 256, 0, st>>>(g);
  return cudaGetLastError();
}

// Exact online-max LSE for the rows the fixed-reference path rejected.  In
// the fine phase (P.fb_mask set) a row sums the columns of the clusters its
// own cluster keeps in the problem's mask (a subset of its pair set that
// holds every term above e^-theta; the pair set's extra terms are below
// that), so the cost is the row's neighbourhood, not all M columns.  Without
// a mask (dense pair sets) it sums all columns.  One warp per row.
template <int D>
__device__ __forceinline__ void fb_term(const Problem& P, float4 xv, int j, float& m, float& s) {
  const float4 yv = P.cols[j];
  float dx = xv.x - yv.x, c = dx * dx;
  if (D > 1) { const float dy = xv.y - yv.y; c = fmaf(dy, dy, c); }
  if (D > 2) { const float dz = xv.z - yv.z; c = fmaf(dz, dz, c); }
  const float z = P.col_lw2[j] + (P.col_h[j] - 0.5f * c) * P.inv_eps_ln2;
  if (z > m) { s = s * ex2_approx(m - z) + 1.f; m = z; }
  else s += ex2_approx(z - m);
}

template <int D>
__global__ void softmin_fallback_dense(const __grid_constant__ Group G) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int cnt = min(*G.fb_count, G.fb_cap);
  for (int q = warp; q < cnt; q += nwarps) {
    const int4 pr = G.fb_list[q];
    const Problem& P = G.P[pr.x];
    const int r = pr.y;
    const float4 xv = P.rows[r];
    float m = -INFINITY, s = 0.f;
    if (!P.fb_mask) {
      for (int j = lane; j < P.n_cols; j += 32) fb_term<D>(P, xv, j, m, s);
    } else if (!P.fb_trans) {  // mask row of the row's cluster: kept column clusters
      const int I = P.fb_rlab[r];
      const uint32_t* mrow = P.fb_mask + static_cast<int64_t>(I) * P.fb_words;
      // an upper-half self mask: clusters below the diagonal word from their
      // own rows (the mask is symmetric), the rest from row I
      const int wlo = P.fb_upper ? (I >> 5) : 0;
      for (int J0 = 0; J0 < wlo * 32; J0 += 32) {
        const int J = J0 + lane;
        const bool keep = (P.fb_mask[static_cast<int64_t>(J) * P.fb_words + (I >> 5)] >> (I & 31)) & 1u;
        uint32_t b = __ballot_sync(0xffffffffu, keep);
        while (b) {
          const int Jk = J0 + __ffs(b) - 1;
          b &= b - 1;
          for (int j = P.fb_co[Jk] + lane; j < P.fb_co[Jk + 1]; j += 32) fb_term<D>(P, xv, j, m, s);
        }
      }
      for (int w0 = wlo; w0 < P.fb_words; w0 += 32) {
        const uint32_t bits = (w0 + lane < P.fb_words) ? mrow[w0 + lane] : 0u;
        for (int src = 0; src < 32; ++src) {
          uint32_t b = __shfl_sync(0xffffffffu, bits, src);
          while (b) {
            const int J = (w0 + src) * 32 + __ffs(b) - 1;
            b &= b - 1;
            for (int j = P.fb_co[J] + lane; j < P.fb_co[J + 1]; j += 32) fb_term<D>(P, xv, j, m, s);
          }
        }
      }
    } else {  // transposed: column fb_rlab[r] of the mask, over its kc rows
      const int I = P.fb_rlab[r];
      for (int J0 = 0; J0 < P.fb_kc; J0 += 32) {
        const int J = J0 + lane;
        const bool keep =
            J < P.fb_kc && ((P.fb_mask[static_cast<int64_t>(J) * P.fb_words + (I >> 5)] >> (I & 31)) & 1u);
        uint32_t b = __ballot_sync(0xffffffffu, keep);
        while (b) {
          const int Jk = J0 + __ffs(b) - 1;
          b &= b - 1;
          for (int j = P.fb_co[Jk] + lane; j < P.fb_co[Jk + 1]; j += 32) fb_term<D>(P, xv, j, m, s);
        }
      }
    }
    for (int off = 16; off > 0; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
      const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
      const float mm = fmaxf(m, m2);
      s = (m == -INFINITY ? 0.f : s * exp2f(m - mm)) + (m2 == -INFINITY ? 0.f : s2 * exp2f(m2 - mm));
      m = mm;
    }
    if (lane == 0) {
      const float est = P.row_est ? P.row_est[r] : 0.f;
      const float ft = -P.lam_eps * kLn2 * (m + log2f(s));
      store_potential(G, P.row_out, r, (1.f - P.mixw) * est + P.mixw * ft);
    }
  }
}

template <int D, bool kUni>
static void launch_sym_d(const Group& g, cudaStream_t st) {
  ++g_launches;
  softmin_sym_kernel<D, kUni><<<g.n_items, kSymThreads, 0, st>>>(g);
}

cudaError_t launch_softmin_sym(const Group& g, int d, bool uniform, cudaStream_t st) {
  if (g.n_items <= 0) return cudaSuccess;
  if (uniform) {
    switch (d) {
      case 1: launch_sym_d<1, true>(g, st); break;
      case 2: launch_sym_d<2, true>(g, st); break;
      default: launch_sym_d<3, true>(g, st); break;
    }
  } else {
    switch (d) {
      case 1: launch_sym_d<1, false>(g, st); break;
      case 2: launch_sym_d<2, false>(g, st); break;
      default: launch_sym_d<3, false>(g, st); break;
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_fallback_dense(const Group& g, int d, int n_sm, cudaStream_t st) {
  ++g_launches;
  // 8 warps x 8 CTAs per SM: one warp per queued row, latency-bound gathers
  const int grid = n_sm * 8;
  switch (d) {
    case 1: softmin_fallback_dense<1><<<grid, 256, 0, st>>>(g); break;
    case 2: softmin_fallback_dense<2><<<grid, 256, 0, st>>>(g); break;
    default: softmin_fallback_dense<3><<<grid, 256, 0, st>>>(g); break;
  }
  return cudaGetLastError();
}

}  // namespace msot_dev
