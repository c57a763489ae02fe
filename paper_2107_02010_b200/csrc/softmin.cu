// softmin.cu — K1/K4: the online log-sum-exp softmin of the Sinkhorn loop.
//
//   f_i = -lambda eps log sum_j w_j exp((h_j - |x_i - y_j|^2 / 2) / eps)
// (the four lines of the Algorithm).
//
// Design: one CTA = one work item = a 256-row tile (rows
// sorted by voxel cube, 2 rows per thread) against a chunk of that tile's
// kept columns (dense = one range per tile; block-sparse = the ranges of the
// truncation mask).  Columns stream through a double-buffered shared-memory
// tile, stored as float32 *pairs* so the inner loop runs on the packed
// FADD2/FFMA2 pipe: 5 packed ops per two pairs (the FMA pipe runs a packed
// op in 2 cycles, so this is 5 FP32 lane-ops per pair against the 8 per ex2
// the pipes balance at) next to the one MUFU.EX2 per pair that bounds it
// (roofline: 16 ex2/clk/SM, measured by probe.cu).
//
// Fixed-reference expansion: instead of a running max, every row is
// expanded around m_i = -est_i / (lambda eps ln2), its previous potential in
// log2 units, so s_i = sum_j 2^{z_ij - m_i} is additive across column chunks
// and the update is f_i = est_i - lambda eps ln(s_i).  Since the LSE is
// bounded by [max, max + log M], a reference within ~60 nats of the truth
// keeps s_i in [2^-60, 2^100]; rows outside that window are recomputed by the
// exact online-max kernel (softmin_fallback), so the result never depends on
// the reference being good.
//
// Precision: coordinates are re-centred on the tile's middle row before
// scaling, so |x^ - y^|^2 is formed from small, exactly-subtracted numbers.
#include "softmin_inner.cuh"

namespace msot_dev {


template <int D, int kPoly16>
__global__ void __launch_bounds__(kSoftminThreads)
softmin_kernel(const __grid_constant__ Group G) {
  __shared__ __align__(16) float smem[2][kColTile * 4];
  const int it = blockIdx.x;
  if (it >= G.n_items) return;
  const int4 item = G.items[it];
  const Problem& P = G.P[item.x];
  const int tid = threadIdx.x;
  const int row_base = P.tile_start[item.y];
  const int row_end = P.tile_start[item.y + 1];
  const int mid = (row_base + row_end) >> 1;
  const float4 o = P.rows[mid];
  // Tile reference R (log2 units): the row constant est/(lambda eps ln2) and
  // the column constant h/(eps ln2) are ~|f|/eps (10^2..10^4) and cancel on
  // the pairs that matter; shifting both by R inside an FMA keeps each to one
  // rounding of a small number instead of two roundings of large ones.
  const float R = P.row_est ? P.row_est[mid] * P.inv_lam_eps_ln2 : 0.f;

  RowState ra, rb;
  load_row<D>(P, row_base + tid, row_end, o, R, ra);
  load_row<D>(P, row_base + tid + kSoftminThreads, row_end, o, R, rb);

  ColWalker w{P.ranges, P.tile_rptr[item.y], P.tile_rptr[item.y + 1], 0};
  const int32_t pos_begin = item.z, pos_end = item.w;

  // raw column prefetch registers
  float4 cv = make_float4(0.f, 0.f, 0.f, 0.f);
  float ch = 0.f, cl = 0.f;
  bool cvalid = false;
  auto fetch = [&](int32_t tile_pos) {
    const int32_t pos = tile_pos + tid;
    cvalid = false;
    if (pos < pos_end) {
      const int j = w.col(pos);
      if (j >= 0) {
        cv = __ldg(P.cols + j);
        cl = __ldg(P.col_lw2 + j);
        ch = __ldg(P.col_h + j);
        cvalid = true;
      }
    }
  };
  auto stage = [&](float* buf) {
    // pair record layout: [y0a, y0b, y1a, y1b, y2a, y2b, ca, cb]
    float* rec = buf + (tid >> 1) * 8 + (tid & 1);
    if (cvalid) {
      const float a = (cv.x - o.x) * P.sc;
      const float b = D > 1 ? (cv.y - o.y) * P.sc : 0.f;
      const float c = D > 2 ? (cv.z - o.z) * P.sc : 0.f;
      rec[0] = a;
      rec[2] = b;
      rec[4] = c;
      rec[6] = (fmaf(ch, P.inv_eps_ln2, R) + cl) - fmaf(a, a, fmaf(b, b, c * c));
    } else {
      rec[0] = 0.f;
      rec[2] = 0.f;
      rec[4] = 0.f;
      rec[6] = __int_as_float(0xff800000);  // -inf -> exp2(-inf) = 0
    }
  };

  float2 sa = make_float2(0.f, 0.f), sb = make_float2(0.f, 0.f);
  int buf = 0;
  fetch(pos_begin);
  for (int32_t tp = pos_begin; tp < pos_end; tp += kColTile) {
    stage(smem[buf]);
    __syncthreads();
    if (tp + kColTile < pos_end) fetch(tp + kColTile);
    const float4* s4 = reinterpret_cast<const float4*>(smem[buf]);
#pragma unroll 2
    for (int c0 = 0; c0 < kColTile / 2; c0 += 8) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int c = c0 + k;
        const float4 A = s4[2 * c], B = s4[2 * c + 1];
        const float2 Y0 = make_float2(A.x, A.y);
        const float2 Y1 = make_float2(A.z, A.w);
        const float2 Y2 = make_float2(B.x, B.y);
        const float2 C = make_float2(B.z, B.w);
        if (poly_slot(2 * k, kPoly16))
          sa = __fadd2_rn(sa, pair_terms<D, true>(ra, Y0, Y1, Y2, C));
        else
          sa = __fadd2_rn(sa, pair_terms<D, false>(ra, Y0, Y1, Y2, C));
        if (poly_slot(2 * k + 1, kPoly16))
          sb = __fadd2_rn(sb, pair_terms<D, true>(rb, Y0, Y1, Y2, C));
        else
          sb = __fadd2_rn(sb, pair_terms<D, false>(rb, Y0, Y1, Y2, C));
      }
    }
    buf ^= 1;
  }
  float* out = G.part + static_cast<int64_t>(it) * kTileRows;
  out[tid] = sa.x + sa.y;
  out[tid + kSoftminThreads] = sb.x + sb.y;
}

// Implicit transport plan applied to column payloads (SPEC.md:204-212,
// PAPER.md eq. 4): with est = f (final row potential), h = g and lambda = 1
// the exponent is log2 of pi_ij / alpha_i = beta_j exp((f_i + g_j - C_ij)/eps),
// so one pass gives, per row, m_i = sum_j pi_ij / alpha_i and
// u_i = sum_j pi_ij v_j / alpha_i for a float4 payload v (the column
// coordinates for the barycentric map / grad_positions).
// Partials: part[item][4][256] = {m, u.x, u.y, u.z}.
template <int D>
__global__ void __launch_bounds__(kSoftminThreads)
plan_kernel(const __grid_constant__ Group G) {
  __shared__ __align__(16) float smem[2][kColTile * 4];
  __shared__ __align__(16) float spay[2][kColTile * 4];
  const int it = blockIdx.x;
  if (it >= G.n_items) return;
  const int4 item = G.items[it];
  const Problem& P = G.P[item.x];
  const int tid = threadIdx.x;
  const int row_base = P.tile_start[item.y];
  const int row_end = P.tile_start[item.y + 1];
  const int mid = (row_base + row_end) >> 1;
  const float4 o = P.rows[mid];
  const float R = P.row_est ? P.row_est[mid] * P.inv_lam_eps_ln2 : 0.f;
  RowState ra, rb;
  load_row<D>(P, row_base + tid, row_end, o, R, ra);
  load_row<D>(P, row_base + tid + kSoftminThreads, row_end, o, R, rb);
  ColWalker w{P.ranges, P.tile_rptr[item.y], P.tile_rptr[item.y + 1], 0};
  const int32_t pos_begin = item.z, pos_end = item.w;
  float4 cv = make_float4(0.f, 0.f, 0.f, 0.f), pv = cv;
  float ch = 0.f, cl = 0.f;
  bool cvalid = false;
  auto fetch = [&](int32_t tile_pos) {
    const int32_t pos = tile_pos + tid;
    cvalid = false;
    if (pos < pos_end) {
      const int j = w.col(pos);
      if (j >= 0) {
        cv = __ldg(P.cols + j);
        pv = __ldg(P.col_pay + j);
        cl = __ldg(P.col_lw2 + j);
        ch = __ldg(P.col_h + j);
        cvalid = true;
      }
    }
  };
  auto stage = [&](float* buf, float* pbuf) {
    float* rec = buf + (tid >> 1) * 8 + (tid & 1);
    float* prc = pbuf + (tid >> 1) * 8 + (tid & 1);
    if (cvalid) {
      const float a = (cv.x - o.x) * P.sc;
      const float b = D > 1 ? (cv.y - o.y) * P.sc : 0.f;
      const float c = D > 2 ? (cv.z - o.z) * P.sc : 0.f;
      rec[0] = a;
      rec[2] = b;
      rec[4] = c;
      rec[6] = (fmaf(ch, P.inv_eps_ln2, R) + cl) - fmaf(a, a, fmaf(b, b, c * c));
      prc[0] = pv.x;
      prc[2] = pv.y;
      prc[4] = pv.z;
    } else {
      rec[0] = rec[2] = rec[4] = 0.f;
      rec[6] = __int_as_float(0xff800000);
      prc[0] = prc[2] = prc[4] = 0.f;
    }
  };
  float2 ma = make_float2(0.f, 0.f), mb = ma, a0 = ma, a1 = ma, a2 = ma, b0 = ma, b1 = ma, b2 = ma;
  int buf = 0;
  fetch(pos_begin);
  for (int32_t tp = pos_begin; tp < pos_end; tp += kColTile) {
    stage(smem[buf], spay[buf]);
    __syncthreads();
    if (tp + kColTile < pos_end) fetch(tp + kColTile);
    const float4* s4 = reinterpret_cast<const float4*>(smem[buf]);
    const float4* p4 = reinterpret_cast<const float4*>(spay[buf]);
#pragma unroll 4
    for (int c = 0; c < kColTile / 2; ++c) {
      const float4 A = s4[2 * c], B = s4[2 * c + 1];
      const float4 PA = p4[2 * c], PB = p4[2 * c + 1];
      const float2 Y0 = make_float2(A.x, A.y), Y1 = make_float2(A.z, A.w);
      const float2 Y2 = make_float2(B.x, B.y), C = make_float2(B.z, B.w);
      const float2 V0 = make_float2(PA.x, PA.y), V1 = make_float2(PA.z, PA.w);
      const float2 V2 = make_float2(PB.x, PB.y);
      const float2 ea = pair_terms<D, false>(ra, Y0, Y1, Y2, C);
      const float2 eb = pair_terms<D, false>(rb, Y0, Y1, Y2, C);
      ma = __fadd2_rn(ma, ea);
      mb = __fadd2_rn(mb, eb);
      a0 = __ffma2_rn(ea, V0, a0);
      a1 = __ffma2_rn(ea, V1, a1);
      a2 = __ffma2_rn(ea, V2, a2);
      b0 = __ffma2_rn(eb, V0, b0);
      b1 = __ffma2_rn(eb, V1, b1);
      b2 = __ffma2_rn(eb, V2, b2);
    }
    buf ^= 1;
  }
  float* out = G.part + static_cast<int64_t>(it) * 4 * kTileRows;
  const int r2 = tid + kSoftminThreads;
  out[tid] = ma.x + ma.y;
  out[kTileRows + tid] = a0.x + a0.y;
  out[2 * kTileRows + tid] = a1.x + a1.y;
  out[3 * kTileRows + tid] = a2.x + a2.y;
  out[r2] = mb.x + mb.y;
  out[kTileRows + r2] = b0.x + b0.y;
  out[2 * kTileRows + r2] = b1.x + b1.y;
  out[3 * kTileRows + r2] = b2.x + b2.y;
}

// Sums the plan partials of every row in a fixed chunk order into
// row_plan[r] = {m_r, u_r} (float4).
__global__ void __launch_bounds__(kTileRows) plan_finalize(const __grid_constant__ Group G) {
  const int b = blockIdx.x;
  int p = 0;
  while (p + 1 < G.n_problems && b >= G.tile_prefix[p + 1]) ++p;
  const Problem& P = G.P[p];
  const int t = G.t0[p] + (b - G.tile_prefix[p]);
  const int lr = threadIdx.x;
  const int r = P.tile_start[t] + lr;
  if (r >= P.tile_start[t + 1]) return;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int32_t k = P.tile_ibase[t]; k < P.tile_ibase[t + 1]; ++k) {
    const float* q = G.part + static_cast<int64_t>(k) * 4 * kTileRows + lr;
    s.x += q[0];
    s.y += q[kTileRows];
    s.z += q[2 * kTileRows];
    s.w += q[3 * kTileRows];
  }
  P.row_plan[r] = s;
}

// Sum over a tile's items k0 <= k < k1 of one row's partial (part[(k - i0) *
// kTileRows]): four interleaved running sums (item k0 + 4i + u feeds sum u),
// combined as (s0 + s1) + (s2 + s3) — four loads in flight per step, and the
// same additions whether the items are reduced per batch or at finalize.
__device__ __forceinline__ float sum_items(const float* part, int32_t k0, int32_t k1, int32_t i0) {
  const float* q = part + static_cast<int64_t>(k0 - i0) * kTileRows;
  const int32_t n = k1 - k0;
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  int32_t i = 0;
  for (; i + 3 < n; i += 4, q += 4 * kTileRows) {
    s0 += q[0];
    s1 += q[kTileRows];
    s2 += q[2 * kTileRows];
    s3 += q[3 * kTileRows];
  }
  if (i < n) s0 += q[0];
  if (i + 1 < n) s1 += q[kTileRows];
  if (i + 2 < n) s2 += q[2 * kTileRows];
  return (s0 + s1) + (s2 + s3);
}

// Combines the partial sums of every row (fixed chunk order: deterministic
// and independent of the number of GPUs) and applies the update
//   new = est - mixw * lambda eps ln(s)   (averaging of PAPER.md:293-315).
// Rows whose sum left the safe window are queued for the exact path.
// One CTA per row tile of this rank's shard.
__global__ void __launch_bounds__(kTileRows) softmin_finalize(const __grid_constant__ Group G) {
  const int b = blockIdx.x;
  const int nt = G.tile_prefix[G.n_problems];
  if (b >= nt) {  // the extra blocks: the transposed problem's rows (evaluate-once)
    sym_colfinal_row(G, G.colfinal_p, (b - nt) * kTileRows + static_cast<int32_t>(threadIdx.x));
    return;
  }
  int p = 0;
  while (p + 1 < G.n_problems && b >= G.tile_prefix[p + 1]) ++p;
  const Problem& P = G.P[p];
  const int t = G.t0[p] + (b - G.tile_prefix[p]);
  const int lr = threadIdx.x;
  const int r = P.tile_start[t] + lr;
  if (r >= P.tile_start[t + 1]) return;
  float s = 0.f;
  if (P.row_sum) {  // batched group: the row partials were reduced per batch
    s = P.row_sum[r];
  } else {
    s = sum_items(G.part + lr, P.tile_ibase[t], P.tile_ibase[t + 1], 0);
  }
  if (P.row_add) s += P.row_add[r];  // column side of an evaluate-once self problem
  const float est = P.row_est ? P.row_est[r] : 0.f;
  // window [2^-60, 2^100]: flushed terms (< 2^-126 each) stay below 2^-84 s
  if (!(s >= 8.67361738e-19f && s <= 1.2676506e30f) || G.force_fb) {
    const int slot = atomicAdd(G.fb_count, 1);
    atomicAdd(G.fb_total, 1);
    if (slot < G.fb_cap) G.fb_list[slot] = make_int4(p, r, t, 0);
    return;
  }
  store_potential(G, P.row_out, r, est - P.mixw * P.lam_eps * logf(s));
}

// Row partials of one colpart batch (solver.cu: Plan::Batch): the rows of
// the batch's tiles sum their items' partials (sum_items) — the same float
// additions softmin_finalize makes unbatched — into P.row_sum.  G.part holds
// the batch's items only (item k at k - i0); G.t0 / tile_prefix describe the
// batch's tiles.
__global__ void __launch_bounds__(kTileRows) softmin_rowsum(const __grid_constant__ Group G,
                                                             int32_t i0) {
  const int b = blockIdx.x;
  int p = 0;
  while (p + 1 < G.n_problems && b >= G.tile_prefix[p + 1]) ++p;
  const Problem& P = G.P[p];
  const int t = G.t0[p] + (b - G.tile_prefix[p]);
  const int lr = threadIdx.x;
  const int r = P.tile_start[t] + lr;
  if (r >= P.tile_start[t + 1]) return;
  P.row_sum[r] = sum_items(G.part + lr, P.tile_ibase[t], P.tile_ibase[t + 1], i0);
}

// Exact online-max LSE for the rows the fixed-reference path rejected: one
// warp per row over the same column set, float32 with a running max.
template <int D>
__global__ void softmin_fallback(const __grid_constant__ Group G) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int cnt = min(*G.fb_count, G.fb_cap);
  for (int q = warp; q < cnt; q += nwarps) {
    const int4 pr = G.fb_list[q];
    const Problem& P = G.P[pr.x];
    const int r = pr.y;
    const float4 xv = P.rows[r];
    const int t = pr.z;
    float m = -INFINITY, s = 0.f;
    for (int64_t k = P.tile_rptr[t]; k < P.tile_rptr[t + 1]; ++k) {
      const int2 rg = P.ranges[k];
      for (int j = rg.x + lane; j < rg.y; j += 32) {
        const float4 yv = P.cols[j];
        float dx = xv.x - yv.x, c = dx * dx;
        if (D > 1) { const float dy = xv.y - yv.y; c = fmaf(dy, dy, c); }
        if (D > 2) { const float dz = xv.z - yv.z; c = fmaf(dz, dz, c); }
        const float z = P.col_lw2[j] + (P.col_h[j] - 0.5f * c) * P.inv_eps_ln2;
        if (z > m) { s = s * exp2f(m - z) + 1.f; m = z; }
        else s += exp2f(z - m);
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

// ---- host launchers -------------------------------------------------------

// exp2 split between MUFU and the FMA pipe (see poly_slot); MSOT_POLY16
// overrides for experiments (0 = MUFU only).
static int poly16() {
  static const int v = [] {
    const char* e = getenv("MSOT_POLY16");
    return e ? atoi(e) : kDefaultPoly16;
  }();
  return v;
}

template <int D>
static void launch_d(const Group& g, dim3 grid, dim3 block, cudaStream_t st) {
  ++g_launches;
  switch (poly16()) {
    case 0: softmin_kernel<D, 0><<<grid, block, 0, st>>>(g); break;
    case 2: softmin_kernel<D, 2><<<grid, block, 0, st>>>(g); break;
    case 4: softmin_kernel<D, 4><<<grid, block, 0, st>>>(g); break;
    default: softmin_kernel<D, 3><<<grid, block, 0, st>>>(g); break;
  }
}

cudaError_t launch_softmin(const Group& g, int d, cudaStream_t st) {
  if (g.n_items <= 0) return cudaSuccess;
  dim3 grid(g.n_items), block(kSoftminThreads);
  switch (d) {
    case 1: launch_d<1>(g, grid, block, st); break;
    case 2: launch_d<2>(g, grid, block, st); break;
    default: launch_d<3>(g, grid, block, st); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_plan(const Group& g, int d, cudaStream_t st) {
  if (g.n_items <= 0) return cudaSuccess;
  dim3 grid(g.n_items), block(kSoftminThreads);
  ++g_launches;
  switch (d) {
    case 1: plan_kernel<1><<<grid, block, 0, st>>>(g); break;
    case 2: plan_kernel<2><<<grid, block, 0, st>>>(g); break;
    default: plan_kernel<3><<<grid, block, 0, st>>>(g); break;
  }
  const int tiles = g.tile_prefix[g.n_problems];
  if (tiles > 0) {
    ++g_launches;
    plan_finalize<<<tiles, kTileRows, 0, st>>>(g);
  }
  return cudaGetLastError();
}

cudaError_t launch_finalize(const Group& g, cudaStream_t st) {
  const int tiles = g.tile_prefix[g.n_problems];
  const int extra = g.colfinal_p > 0 ? (g.P[g.colfinal_p].n_rows + kTileRows - 1) / kTileRows : 0;
  if (tiles + extra <= 0) return cudaSuccess;
  ++g_launches; softmin_finalize<<<tiles + extra, kTileRows, 0, st>>>(g);
  return cudaGetLastError();
}

cudaError_t launch_rowsum(const Group& g, int32_t i0, cudaStream_t st) {
  const int tiles = g.tile_prefix[g.n_problems];
  if (tiles <= 0) return cudaSuccess;
  ++g_launches; softmin_rowsum<<<tiles, kTileRows, 0, st>>>(g, i0);
  return cudaGetLastError();
}

cudaError_t launch_fallback(const Group& g, int d, int n_sm, cudaStream_t st) {
  dim3 grid(n_sm), block(256);
  switch (d) {
    case 1: ++g_launches; softmin_fallback<1><<<grid, block, 0, st>>>(g); break;
    case 2: ++g_launches; softmin_fallback<2><<<grid, block, 0, st>>>(g); break;
    default: ++g_launches; softmin_fallback<3><<<grid, block, 0, st>>>(g); break;
  }
  return cudaGetLastError();
}

}  // namespace msot_dev
