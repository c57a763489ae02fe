// common.cuh — shared device/host definitions of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "policy.h"

namespace msot_dev {

constexpr int kTileRows = MSOT_TILE_ROWS;  // rows per block-sparse tile
constexpr int kSoftminThreads = 128;       // threads per softmin CTA
constexpr int kRowsPerThread = kTileRows / kSoftminThreads;
constexpr int kColTile = 128;              // columns staged per smem buffer
// exp2 on the FMA pipe for 2 of 16 pair-of-pairs (softmin.cu).  Measured on
// B200 (C3 + dense 300k): 0 -> 4.31e12 pairs/s, 2 -> 4.37e12, 3 -> 4.16e12,
// 4 -> 3.81e12: the pipes do not co-saturate beyond 2/16.
constexpr int kDefaultPoly16 = 2;
static_assert(kRowsPerThread == 2, "softmin kernel is written for 2 rows per thread");

constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;

// One softmin problem of a launch group (the four updates of PAPER.md:258-290
// share a launch).  Rows/cols are float4 {x, y, z, 0} centred float32 atoms
// in cluster-sorted order; potentials are float32.
struct Problem {
  const float4* rows;
  const float* row_est;   // reference value of the output potential (nullable)
  float* row_out;         // output potential
  const float4* cols;
  const float* col_lw2;   // log2 of column weights
  const float* col_h;     // column potentials
  const int32_t* tile_start; // [n_tiles+1] first row of each (cluster-aligned) tile
  const int64_t* tile_rptr;  // [n_tiles+1] range index per row tile
  const int2* ranges;        // column ranges [begin, end)
  const int32_t* tile_ibase; // [n_tiles+1] work items per row tile (prefix)
  const float4* col_pay;     // plan_kernel: column payload v_j
  float4* row_plan;          // plan_kernel: {m_i, u_i} per row
  // high-dimensional path (softmin_hd.cu): pre-swizzled split-f16 operands
  const uint8_t* a_pack;     // rows, [hi, hi, lo] per 128-row block
  const uint8_t* b_pack;     // cols, [hi, lo, hi] per 128-col block
  const float* row_sq;       // |x_i|^2 (float32 coordinates)
  const float* col_sq;       // |y_j|^2
  const float* col_c;        // per-scale column constants (hd_colconst)
  const float* col_c2;       // evaluate-once: column factor exponents (hd_colconst)
  const float* row_f;        // float32 coordinates, row-major x 64 (exact fallback)
  const float* col_f;
  // evaluate-once (symmetric) groups (softmin_sym.cu)
  const float* row_lw2;      // log2 row weights (column sums weight rows by alpha_i)
  float* colpart;            // column partial of every (tile, position) slot
  const int64_t* tile_slot;  // [n_tiles] first colpart slot of each tile
  const float* row_add;      // column totals added to the row sums (self problems;
                             // the whole sum of the transposed cross problem)
  float* row_sum;            // batched groups: reduced row partials (softmin_rowsum),
                             // read by softmin_finalize instead of G.part
  // exact fallback restricted to the row cluster's mask neighbourhood (fine
  // phase; null = all columns): cluster of each row, column cluster offsets,
  // the problem's cluster mask (kr x words bits, rows = row clusters unless
  // fb_trans, where the row cluster is the mask's column)
  const uint32_t* fb_mask;
  const int32_t* fb_rlab;
  const int32_t* fb_co;
  int32_t fb_words, fb_kc, fb_trans;
  int32_t fb_upper;          // self mask holding its upper half only (mask_mirror)
  float ell;                 // (1/lambda - 1) / (eps ln2): row/column reference shift
  int32_t n_rows, n_cols;
  float sc;                // 1 / sqrt(2 eps ln2): scaled |dx|^2 = C / (eps ln2)
  float inv_eps_ln2;       // 1 / (eps ln 2)
  float inv_lam_eps_ln2;   // 1 / (lambda eps ln 2)
  float lam_eps;           // lambda * eps
  float mixw;              // 1 = assign, 1/2 = averaged update
  float pad_;
};

constexpr int kMaxProblems = 4;

struct Group {
  Problem P[kMaxProblems];
  const int4* items;      // {problem, tile, pos_begin, pos_end}
  int32_t n_items;
  float* part;            // [n_items][kTileRows] partial sums
  int32_t* fb_count;      // fallback row counter (reset per launch)
  int32_t* fb_total;      // fallback rows over the whole solve
  int4* fb_list;          // {problem, row, tile, 0}
  int32_t fb_cap;
  int32_t n_problems;
  int32_t tile_prefix[kMaxProblems + 1];  // finalized tiles per problem (prefix)
  int32_t t0[kMaxProblems];               // first tile this rank finalizes
  int32_t force_fb;       // tests (MSOT_FORCE_FALLBACK): every row takes the exact path
  int32_t* bad_scale;     // first scale that produced a non-finite potential
  int32_t scale;          // index of this launch group's scale
  int32_t colfinal_p;     // > 0: softmin_finalize also updates this problem's rows
                          // from their column totals (evaluate-once, sym_colfinal_row);
                          // 0 (the zero-initialised default): off
};

// Kernel launches issued by this thread (reported as stats.gpu_launches).
extern thread_local int64_t g_launches;

// Writes an updated potential; a non-finite value records the group's scale
// (atomicMin: the first failing scale is reported).
__device__ __forceinline__ void store_potential(const Group& G, float* out, int32_t r, float v) {
  out[r] = v;
  if (!isfinite(v) && G.bad_scale) atomicMin(G.bad_scale, G.scale);
}

// The transposed cross problem of an evaluate-once group (problem p, no
// tiles of its own): its row sum is the column total alone.  Out-of-window
// rows are queued for the exact path.
__device__ __forceinline__ void sym_colfinal_row(const Group& G, int p, int32_t r) {
  const Problem& P = G.P[p];
  if (r >= P.n_rows) return;
  const float s = P.row_add[r];
  const float est = P.row_est ? P.row_est[r] : 0.f;
  if (P.row_lw2 && P.row_lw2[r] == -INFINITY) {  // zero-weight atom (padding): no update
    store_potential(G, P.row_out, r, est);
    return;
  }
  if (!(s >= 8.67361738e-19f && s <= 1.2676506e30f) || G.force_fb) {
    const int slot = atomicAdd(G.fb_count, 1);
    atomicAdd(G.fb_total, 1);
    if (slot < G.fb_cap) G.fb_list[slot] = make_int4(p, r, -1, 0);
    return;
  }
  store_potential(G, P.row_out, r, est - P.mixw * P.lam_eps * logf(s));
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace msot_dev
