// softmin_inner.cuh — the inner-loop pieces shared by the softmin kernels
// (softmin.cu: K1/K4 row sums; softmin_sym.cu: evaluate-once row + column
// sums): row state, the column-range walker, the packed pair exponent and
// the exp2 split between the MUFU and the FMA pipe.
#pragma once

#include "common.cuh"

namespace msot_dev {

struct RowState {
  float x0, x1, x2;  // 2 x scaled, tile-centred coordinates
  float r;           // est/(lambda eps ln2) - R - |x^|^2   (log2 units)
};

template <int D>
__device__ __forceinline__ void load_row(const Problem& P, int r, int r_end, float4 o, float R,
                                         RowState& rs) {
  const bool ok = r < r_end;
  float4 v = ok ? P.rows[r] : o;
  const float a = (v.x - o.x) * P.sc;
  const float b = D > 1 ? (v.y - o.y) * P.sc : 0.f;
  const float c = D > 2 ? (v.z - o.z) * P.sc : 0.f;
  rs.x0 = 2.f * a;
  rs.x1 = 2.f * b;
  rs.x2 = 2.f * c;
  const float est = (P.row_est != nullptr && ok) ? P.row_est[r] : 0.f;
  // one rounding of a small number for the potential part (see R below)
  rs.r = fmaf(est, P.inv_lam_eps_ln2, -R) - fmaf(a, a, fmaf(b, b, c * c));
}

// Walks the concatenated column ranges of one tile: position -> column.
struct ColWalker {
  const int2* rg;
  int64_t k, kend;
  int32_t acc;   // positions before range k
  __device__ __forceinline__ int col(int32_t pos) {
    while (k < kend) {
      int2 r = rg[k];
      int32_t len = r.y - r.x;
      if (pos < acc + len) return r.x + (pos - acc);
      acc += len;
      ++k;
    }
    return -1;
  }
};

// Exponent of pair (i, j) in log2 units, expanded around the tile centre o:
//   E_ij = c_j + r_i + <2 x^_i, y^_j>,  x^ = (x - o) sc, y^ = (y - o) sc,
//   c_j  = log2 w_j + h_j/(eps ln2) + R - |y^_j|^2,
//   r_i  = est_i/(lambda eps ln2) - R - |x^_i|^2
// = log2 w_j + (h_j + est_i/lambda - |x_i - y_j|^2/2)/(eps ln2).  Per column
// pair: one FADD2 + D FFMA2 + one FADD2 accumulate next to two MUFU.EX2.
// 2^e for a pair of exponents on the FMA pipe (the MUFU is the bottleneck and
// the FMA pipe has ~40% headroom): e = j + f with j = round(e) taken from the
// mantissa of e + 1.5*2^23, f in [-1/2, 1/2], 2^f by a degree-5 near-minimax
// polynomial (max relative error 3.4e-7 in float32, ex2.approx: 1.7e-7), and
// 2^j added to the exponent bits.  e is clamped to [-127, 127] so the result
// saturates like MUFU.EX2 (~0 below, >= 2^127 above, which the finalize
// window then rejects to the exact path).
__device__ __forceinline__ float2 exp2_poly(float2 e) {
  e.x = fminf(fmaxf(e.x, -127.f), 127.f);
  e.y = fminf(fmaxf(e.y, -127.f), 127.f);
  const float2 kShift = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = __fadd2_rn(e, kShift);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __fadd2_rn(e, make_float2(-j.x, -j.y));
  float2 p = __ffma2_rn(f, make_float2(1.2915660627186298e-3f, 1.2915660627186298e-3f),
                        make_float2(9.668532758951187e-3f, 9.668532758951187e-3f));
  p = __ffma2_rn(f, p, make_float2(5.5516887456178665e-2f, 5.5516887456178665e-2f));
  p = __ffma2_rn(f, p, make_float2(2.4022264778614044e-1f, 2.4022264778614044e-1f));
  p = __ffma2_rn(f, p, make_float2(6.931464672088623e-1f, 6.931464672088623e-1f));
  p = __ffma2_rn(f, p, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

template <int D, bool kPoly>
__device__ __forceinline__ float2 pair_terms(const RowState& rs, float2 Y0, float2 Y1, float2 Y2,
                                             float2 C) {
  float2 e = __fadd2_rn(make_float2(rs.r, rs.r), C);
  e = __ffma2_rn(make_float2(rs.x0, rs.x0), Y0, e);
  if (D > 1) e = __ffma2_rn(make_float2(rs.x1, rs.x1), Y1, e);
  if (D > 2) e = __ffma2_rn(make_float2(rs.x2, rs.x2), Y2, e);
  if (kPoly) return exp2_poly(e);
  return make_float2(ex2_approx(e.x), ex2_approx(e.y));
}

// Of the 16 pair-of-pairs (8 column pairs x 2 rows) of one unrolled step,
// kPoly16 go through exp2_poly, spread evenly.  On paper the pipes balance
// at kPoly16 = 3 (MUFU: (16-3)/16 ex2 per pair; FMA: 5 + 8*3/16 lane-ops per
// pair against 8 per ex2), a 1.23x ceiling over the MUFU-only roofline; on
// B200 only 2/16 pays (+1.4%, common.cuh kDefaultPoly16) — the MUFU and the
// packed FMA pipe do not both run near 100% with the issue slots at ~85%.
__host__ __device__ constexpr bool poly_slot(int q, int n) { return n > 0 && (q * n) % 16 < n; }

}  // namespace msot_dev
