// mask.cu — K3: kernel truncation and the
// ranges that feed the block-sparse softmin.
//
// Test per cluster pair (per-pair bounds in place of
// SPEC.md:283's Lipschitz margin p (r_I + r_J) d^{p-1}): keep (I,J) iff
//   min(B_a, B_b) >= -theta eps,   D = X_I - Y_J,
//   B_a = F_I + G_J - (1/2) max(0, |D| - (r_I + r_J))^2
//   B_b = F'_I + G'_J + r_I |G_I - D| + r_J |H_J + D| - |D|^2 / 2
// F, G are per-cluster maxima of the current fine potentials; G_I, H_J any
// per-cluster vectors (the fitted slopes of f, g) with F'_I = max_i (f_i -
// <G_I, x_i - X_I>), G'_J likewise.  Both bound f_i + g_j - C(x_i, y_j) from
// above for every member pair (expand |D + u - v|^2, Cauchy-Schwarz), so a
// dropped block carries plan mass <= alpha_i beta_j e^{-theta} per pair.
// B_b's margin vanishes where Y_J sits at the transport image of X_I
// (grad f = x - T(x)), instead of growing with the transport distance.
// With the clusters' axis-aligned member boxes (offsets u_i = x_i - X_I in
// [L_I, H_I], rounded outward) a third bound keeps the -|u - v|^2/2 term B_b
// drops and replaces the balls by the boxes:
//   B_c = F'_I + G'_J - |D|^2/2 + sum_k max_{a in [L_Ik, H_Ik], b in [L_Jk, H_Jk]}
//                                     [(G_I - D)_k a + (H_J + D)_k b - (a - b)^2 / 2]
// — per axis a concave quadratic on a rectangle.  Along a = b it is linear
// with slope (u + v)/2, so for u + v >= 0 the maximum lies on the edge a = H_I
// or b = H_J (else on a = L_I or b = L_J), the free variable at its clamped
// stationary point: two candidates per axis.  The
// test keeps (I, J) iff min(B_a, B_b, B_c) >= -theta eps.  On C3 it removes
// 5-15% of the tile-union pairs per fine update (tools/box_bound_probe.py).
// Evaluated in float64 with explicitly rounded operations (no FMA) on
// float32 inputs; the formula is symmetric in (I, J), so the mask of the
// transposed problem is the exact transpose.  Bit-identical to
// oracle.cpp:pair_slack on the same inputs.
//
// Layout: masks are bit-packed rows, W = ceil(Ky/32) words per row cluster.
// Ranges: per row tile, OR the rows of the tile's clusters (tile_or), then
// turn runs of set bits into sorted-column ranges [co[J0], co[J1+1])
// (tile_runs), one warp per tile, 1024 column clusters per step.
#include "prims.cuh"

namespace msot_dev {

// max over a in [l1, h1], b in [l2, h2] of u a + v b - (a - b)^2 / 2, in
// float64 with explicitly rounded operations (oracle.cpp: box_quad)
__device__ __forceinline__ double quad_edge(double u, double v, double A, double B) {
  const double c = __dsub_rn(A, B);
  return __dsub_rn(__dadd_rn(__dmul_rn(u, A), __dmul_rn(v, B)), __dmul_rn(0.5, __dmul_rn(c, c)));
}
__device__ __forceinline__ double box_quad(double u, double v, double l1, double h1, double l2,
                                           double h2) {
  // the quadratic grows along a = b with slope (u + v)/2: if u + v >= 0 the
  // maximum has a = h1 or b = h2, otherwise a = l1 or b = l2
  const bool up = __dadd_rn(u, v) >= 0.0;
  const double A = up ? h1 : l1, B = up ? h2 : l2;
  const double ca = quad_edge(u, v, A, fmin(fmax(__dadd_rn(A, v), l2), h2));
  const double cb = quad_edge(u, v, fmin(fmax(__dadd_rn(B, u), l1), h1), B);
  return fmax(ca, cb);
}

__device__ __forceinline__ double pair_slack(float4 X, float rI, float F, float4 GI, float4 Y,
                                             float rJ, float G, float4 HJ, int d, bool grad,
                                             bool box = false, float4 LI = float4{},
                                             float4 UI = float4{}, float4 LJ = float4{},
                                             float4 UJ = float4{}, double thr = -INFINITY) {
  const double d0 = __dsub_rn(static_cast<double>(X.x), static_cast<double>(Y.x));
  const double d1 = d > 1 ? __dsub_rn(static_cast<double>(X.y), static_cast<double>(Y.y)) : 0.0;
  const double d2 = d > 2 ? __dsub_rn(static_cast<double>(X.z), static_cast<double>(Y.z)) : 0.0;
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
  // (a) centroid/radius bound
  const double rr = __dadd_rn(static_cast<double>(rI), static_cast<double>(rJ));
  double lb = __dsub_rn(__dsqrt_rn(s), rr);
  if (lb < 0.0) lb = 0.0;
  const double fg = __dadd_rn(static_cast<double>(F), static_cast<double>(G));
  const double va = __dsub_rn(fg, __dmul_rn(0.5, __dmul_rn(lb, lb)));
  if (!grad) return va;
  // (b) slope bound: F'_I + G'_J + r_I |G_I - D| + r_J |H_J + D| - |D|^2 / 2
  const double a0 = __dsub_rn(static_cast<double>(GI.x), d0);
  const double a1 = __dsub_rn(static_cast<double>(GI.y), d1);
  const double a2 = __dsub_rn(static_cast<double>(GI.z), d2);
  const double b0 = __dadd_rn(static_cast<double>(HJ.x), d0);
  const double b1 = __dadd_rn(static_cast<double>(HJ.y), d1);
  const double b2 = __dadd_rn(static_cast<double>(HJ.z), d2);
  const double na = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)), __dmul_rn(a2, a2)));
  const double nb = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(b0, b0), __dmul_rn(b1, b1)), __dmul_rn(b2, b2)));
  const double marg = __dadd_rn(__dmul_rn(static_cast<double>(rI), na), __dmul_rn(static_cast<double>(rJ), nb));
  const double fgp = __dadd_rn(static_cast<double>(GI.w), static_cast<double>(HJ.w));
  const double vb = __dsub_rn(__dadd_rn(fgp, marg), __dmul_rn(0.5, s));
  double v = va < vb ? va : vb;
  // (a caller testing against thr needs B_c only while min(B_a, B_b) keeps
  // the pair: below thr the decision is made, and B_c can only lower v)
  if (!box || v < thr) return v;
  // (c) box bound: sum over axes of the edge maxima (axis order fixed)
  double q = box_quad(a0, b0, LI.x, UI.x, LJ.x, UJ.x);
  if (d > 1) q = __dadd_rn(q, box_quad(a1, b1, LI.y, UI.y, LJ.y, UJ.y));
  if (d > 2) q = __dadd_rn(q, box_quad(a2, b2, LI.z, UI.z, LJ.z, UJ.z));
  const double vc = __dsub_rn(__dadd_rn(fgp, q), __dmul_rn(0.5, s));
  return v < vc ? v : vc;
}

struct MaskIn {
  int32_t kx, ky, d, words;
  const float4 *cx, *cy;
  const float *rx, *ry, *fx, *gy;
  const float4 *gx, *hy;  // {slope, F'} per cluster, both or neither
  // member boxes {lo}, {hi} of x / y clusters (all four or none; only with gx)
  const float4 *lx = nullptr, *ux = nullptr, *ly = nullptr, *uy = nullptr;
  __device__ __forceinline__ bool box() const { return lx != nullptr; }
  __device__ __forceinline__ double slack(int32_t I, int32_t J) const {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    const bool g = gx != nullptr, b = box();
    return pair_slack(cx[I], rx[I], fx[I], g ? gx[I] : z, cy[J], ry[J], gy[J], g ? hy[J] : z, d, g,
                      b, b ? lx[I] : z, b ? ux[I] : z, b ? ly[J] : z, b ? uy[J] : z);
  }
  // float32 upper bound of the exact (float64) slack: B_a evaluated in float
  // plus a margin far above its rounding error (every term's magnitude times
  // 1e-5, ~100x the accumulated relative error of ~10 float operations).
  // Since min(B_a, B_b) <= B_a, a pair with ub < thr is dropped exactly as
  // the float64 test would drop it — the prefilter never changes a bit.
  __device__ __forceinline__ float ub(int32_t I, int32_t J) const {
    const float4 X = cx[I], Y = cy[J];
    const float dx = X.x - Y.x, dy = d > 1 ? X.y - Y.y : 0.f, dz = d > 2 ? X.z - Y.z : 0.f;
    const float s = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
    const float rr = rx[I] + ry[J];
    const float lb = fmaxf(sqrtf(s) - rr, 0.f);
    const float F = fx[I], G = gy[J];
    const float v = (F + G) - 0.5f * lb * lb;
    return v + 1e-5f * (1.f + fabsf(F) + fabsf(G) + 2.f * s + 2.f * rr * rr);
  }
};

// largest |coordinate| of a box {lo}, {hi} (x, y, z)
__device__ __forceinline__ float box_extent(float4 lo, float4 hi) {
  return fmaxf(fmaxf(fmaxf(fabsf(lo.x), fabsf(hi.x)), fmaxf(fabsf(lo.y), fabsf(hi.y))),
               fmaxf(fabsf(lo.z), fabsf(hi.z)));
}

// sqrt.approx (relative error ~2^-23, sqrt(0) = 0): the float32 bounds carry
// a 1e-5 relative margin, so the IEEE square root's fix-up is not needed
__device__ __forceinline__ float sqrt_fast(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Float32 upper bound of the float64 slack for row data already in registers
// (same arithmetic as MaskIn::ub).
__device__ __forceinline__ float ub_regs(float4 X, float rI, float F, float4 Y, float rJ, float G,
                                         int d) {
  const float dx = X.x - Y.x, dy = d > 1 ? X.y - Y.y : 0.f, dz = d > 2 ? X.z - Y.z : 0.f;
  const float s = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  const float rr = rI + rJ;
  const float lb = fmaxf(sqrt_fast(s) - rr, 0.f);
  const float v = (F + G) - 0.5f * lb * lb;
  return v + 1e-5f * (1.f + fabsf(F) + fabsf(G) + 2.f * s + 2.f * rr * rr);
}

// Float32 value of the float64 slack min(B_a, B_b[, B_c]) with an error
// margin (same rule as ub_regs: 1e-5 x the magnitudes of the terms, ~100x the
// float32 rounding of the operations).  A pair with v - m >= thr is kept and
// one with v + m < thr dropped exactly as the float64 test would decide; only
// the pairs in between need it.
__device__ __forceinline__ float quad_edge_f(float u, float v, float A, float B) {
  const float c = A - B;
  return fmaf(u, A, v * B) - 0.5f * c * c;
}
// float32 box_quad (same two candidates; the margin for its terms is added
// once per pair by bounds_regs)
__device__ __forceinline__ float box_quad_f(float u, float v, float l1, float h1, float l2, float h2) {
  const bool up = u + v >= 0.f;
  const float A = up ? h1 : l1, B = up ? h2 : l2;
  const float ca = quad_edge_f(u, v, A, fminf(fmaxf(A + v, l2), h2));
  const float cb = quad_edge_f(u, v, fminf(fmaxf(B + u, l1), h1), B);
  return fmaxf(ca, cb);
}

// float32 value of min(B_a, B_b[, B_c]) and its error margin: lo = v - m is
// a lower bound of the float64 slack, v + m an upper bound.
// (thr: the box term is skipped once min(B_a, B_b) is already certainly
// below the threshold — the pair is dropped whatever B_c says.)
__device__ __forceinline__ float2 bounds_regs(float4 X, float rI, float F, float4 GI, float4 Y,
                                              float rJ, float G, float4 HJ, int d, bool g,
                                              bool box = false, float4 LI = float4{},
                                              float4 UI = float4{}, float4 LJ = float4{},
                                              float4 UJ = float4{}, float thr = -INFINITY) {
  const float dx = X.x - Y.x, dy = d > 1 ? X.y - Y.y : 0.f, dz = d > 2 ? X.z - Y.z : 0.f;
  const float s = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  const float rr = rI + rJ;
  const float lb = fmaxf(sqrt_fast(s) - rr, 0.f);
  float v = (F + G) - 0.5f * lb * lb;
  float mag = 1.f + fabsf(F) + fabsf(G) + 2.f * s + 2.f * rr * rr;
  if (g) {
    const float a0 = GI.x - dx, a1 = GI.y - dy, a2 = GI.z - dz;
    const float b0 = HJ.x + dx, b1 = HJ.y + dy, b2 = HJ.z + dz;
    const float na = sqrt_fast(fmaf(a0, a0, fmaf(a1, a1, a2 * a2)));
    const float nb = sqrt_fast(fmaf(b0, b0, fmaf(b1, b1, b2 * b2)));
    const float marg = fmaf(rI, na, rJ * nb);
    const float vb = ((GI.w + HJ.w) + marg) - 0.5f * s;
    v = fminf(v, vb);
    mag += fabsf(GI.w) + fabsf(HJ.w) + marg;
    if (box && v + 1e-5f * mag >= thr) {
      float q = box_quad_f(a0, b0, LI.x, UI.x, LJ.x, UJ.x);
      if (d > 1) q += box_quad_f(a1, b1, LI.y, UI.y, LJ.y, UJ.y);
      if (d > 2) q += box_quad_f(a2, b2, LI.z, UI.z, LJ.z, UJ.z);
      v = fminf(v, ((GI.w + HJ.w) + q) - 0.5f * s);
      // term magnitudes of the box sums: with e_I, e_J the largest box
      // coordinates, sum_k |u_k a_k| + |v_k b_k| <= sqrt(3) (e_I |u| + e_J |v|)
      // (Cauchy-Schwarz) and sum_k (|a_k| + |b_k|)^2 <= 3 (e_I + e_J)^2
      const float eI = box_extent(LI, UI), eJ = box_extent(LJ, UJ);
      mag += 1.7320508f * (fmaf(eI, na, eJ * nb) + na + nb) + 3.f * (eI + eJ) * (eI + eJ);
    }
  }
  return make_float2(v, 1e-5f * mag);
}

// Column blocks = the 32 clusters of one mask word (Morton-consecutive, so
// spatially compact): centre C_W, radius R_W >= |Y_J - C_W| + r_J (rounded
// up), G_W = max_J G_J.  Since |X_I - Y_J| - r_I - r_J >= |X_I - C_W| - R_W -
// r_I, ub_regs at (C_W, R_W, G_W) bounds B_a — hence the slack — of every
// pair of the block.
__global__ void block_bounds_kernel(const float4* cy, const float* ry, const float* gy,
                                    int32_t ky, int d, float4* blk, float* blkg) {
  const int lane = threadIdx.x & 31;
  const int32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= mask_words(ky)) return;
  const int32_t J = w * 32 + lane;
  const bool v = J < ky;
  const float4 Y = v ? cy[J] : make_float4(0.f, 0.f, 0.f, 0.f);
  const int cnt = __popc(__ballot_sync(0xffffffffu, v));
  float sx = v ? Y.x : 0.f, sy = v ? Y.y : 0.f, sz = v ? Y.z : 0.f;
  float gm = v ? gy[J] : -INFINITY;
  for (int o = 16; o > 0; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
    gm = fmaxf(gm, __shfl_xor_sync(0xffffffffu, gm, o));
  }
  const float cx = sx / cnt, cyy = d > 1 ? sy / cnt : 0.f, cz = d > 2 ? sz / cnt : 0.f;
  float r = 0.f;
  if (v) {
    const double dx = static_cast<double>(Y.x) - cx;
    const double dy = d > 1 ? static_cast<double>(Y.y) - cyy : 0.0;
    const double dz = d > 2 ? static_cast<double>(Y.z) - cz : 0.0;
    r = static_cast<float>(sqrt(dx * dx + dy * dy + dz * dz) + static_cast<double>(ry[J]));
  }
  for (int o = 16; o > 0; o >>= 1) r = fmaxf(r, __shfl_xor_sync(0xffffffffu, r, o));
  if (lane == 0) {
    blk[w] = make_float4(cx, cyy, cz, r * (1.f + 1e-5f) + 1e-6f);
    blkg[w] = gm;
  }
}

// One CTA per row cluster I: every word of row I, and — only when the row
// has no kept pair — its best pair (max slack, ties -> lowest J).  A row with
// a kept pair needs no best pair: the best is then itself kept, so setting its
// bit would change nothing (best[I] = -1).  Pass 1: a warp tests 32 words'
// blocks at a time (one lane per word) against thr, writes 0 to the words that
// fail and walks the others with one lane per column cluster (coalesced loads,
// one ballot per word); per pair the float32 bounds decide (ub < thr: drop,
// lb >= thr: keep) and the float64 slack only settles the pairs in between.
// Words with kept bits are OR-ed into `colany` (nullable).  Pass 2 (rare: no
// kept pair, so no diagonal either) scans every word for the exact arg-max,
// evaluating the float64 slack where the float32 upper bound reaches the
// lane's best so far.
// One warp per row cluster: rows finish at very different times (their kept
// words vary), small CTAs keep the SMs full and need no inter-warp barrier
// (C3 mask phase: 256 threads 34 ms, 128: 31 ms, 64: 30 ms; with the box
// bound, mask_rows alone: 64 threads 21.7 ms, 32: 20.0 ms).
constexpr int kMaskThreads = 32;

// (64 registers: the kernel is latency-bound and needs the occupancy; the
// rare float64 box path spills)
__global__ void __launch_bounds__(kMaskThreads, 1024 / kMaskThreads)
mask_rows_kernel(MaskIn m, const float4* blk, const float* blkg, double thr, int self,
                 uint32_t* mask, int32_t* best, uint32_t* colany, int32_t row0, int upper) {
  __shared__ double sv[kMaskThreads / 32];
  __shared__ int32_t sj[kMaskThreads / 32];
  const int32_t I = row0 + static_cast<int32_t>(blockIdx.x);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const bool g = m.gx != nullptr;
  const float4 X = m.cx[I];
  const float rI = m.rx[I], F = m.fx[I];
  const float4 GI = g ? m.gx[I] : zero;
  const bool bx = m.box();
  const float4 LI = bx ? m.lx[I] : zero, UI = bx ? m.ux[I] : zero;
  uint32_t* row = mask + static_cast<int64_t>(I) * m.words;
  // for a float v, double(v) >= thr  <=>  v >= thrf (the least float >= thr):
  // the float screens compare without conversions
  const float thrf = __double2float_ru(thr);
  bool any = false;
  // pass 1 (upper: a self mask's words from the diagonal word on; the words
  // below, the transpose of other rows' words, are zeroed here and filled by
  // mask_mirror where a consumer needs the whole mask)
  const int32_t wmin = upper ? (I >> 5) : 0;
  for (int32_t w = threadIdx.x; w < wmin; w += kMaskThreads) row[w] = 0u;
  for (int32_t w0 = (wmin & ~31) + warp * 32; w0 < m.words; w0 += kMaskThreads) {
    const int32_t wl = w0 + lane;
    bool need = false;
    if (wl < m.words && wl >= wmin) {
      const float4 B = blk[wl];
      const float u = ub_regs(X, rI, F, B, B.w, blkg[wl], m.d);
      need = u >= thrf || (self && (I >> 5) == wl);
      if (!need) row[wl] = 0u;
    }
    uint32_t todo = __ballot_sync(0xffffffffu, need);
    // two words per step: both words' column loads are in flight together
    auto keep_of = [&](int32_t J, float4 Y, float rJ, float G, float4 HJ) {
      bool keep = self && I == J;  // diagonal of a self mask
      if (ub_regs(X, rI, F, Y, rJ, G, m.d) >= thrf) {
        const float4 LJ = bx ? m.ly[J] : zero, UJ = bx ? m.uy[J] : zero;
        const float2 vm = bounds_regs(X, rI, F, GI, Y, rJ, G, HJ, m.d, g, bx, LI, UI, LJ, UJ, thrf);
        if (vm.x - vm.y >= thrf)
          keep = true;  // float32 lower bound settles it
        else if (vm.x + vm.y >= thrf)  // in between: float64
          keep = keep || pair_slack(X, rI, F, GI, Y, rJ, G, HJ, m.d, g, bx, LI, UI, LJ, UJ, thr) >= thr;
      }
      return keep;
    };
    while (todo) {
      const int32_t wa = w0 + __ffs(todo) - 1;
      todo &= todo - 1;
      int32_t wb = -1;
      if (todo) {
        wb = w0 + __ffs(todo) - 1;
        todo &= todo - 1;
      }
      const int32_t Ja = wa * 32 + lane, Jb = wb * 32 + lane;
      const bool va = Ja < m.ky, vb = wb >= 0 && Jb < m.ky;
      float4 Ya = zero, Yb = zero, Ha = zero, Hb = zero;
      float ra = 0.f, rb = 0.f, Ga = 0.f, Gb = 0.f;
      if (va) { Ya = m.cy[Ja]; ra = m.ry[Ja]; Ga = m.gy[Ja]; if (g) Ha = m.hy[Ja]; }
      if (vb) { Yb = m.cy[Jb]; rb = m.ry[Jb]; Gb = m.gy[Jb]; if (g) Hb = m.hy[Jb]; }
      const bool ka = va && keep_of(Ja, Ya, ra, Ga, Ha);
      const bool kb = vb && keep_of(Jb, Yb, rb, Gb, Hb);
      const uint32_t bits_a = __ballot_sync(0xffffffffu, ka);
      const uint32_t bits_b = __ballot_sync(0xffffffffu, kb);
      if (lane == 0) {
        row[wa] = bits_a;
        if (bits_a && colany) atomicOr(colany + wa, bits_a);
        if (wb >= 0) {
          row[wb] = bits_b;
          if (bits_b && colany) atomicOr(colany + wb, bits_b);
        }
      }
      any = any || bits_a != 0u || bits_b != 0u;
    }
  }
  if (__syncthreads_or(any)) {
    if (threadIdx.x == 0) best[I] = -1;
    return;
  }
  // pass 2: no kept pair — exact arg-max over every column cluster
  double bv = -INFINITY;
  int32_t bj = 0x7fffffff;
  for (int32_t J = threadIdx.x; J < m.ky; J += kMaskThreads) {
    const float4 Y = m.cy[J];
    const float rJ = m.ry[J], G = m.gy[J];
    if (static_cast<double>(ub_regs(X, rI, F, Y, rJ, G, m.d)) >= bv) {
      const double v = pair_slack(X, rI, F, GI, Y, rJ, G, g ? m.hy[J] : zero, m.d, g, bx, LI, UI,
                                  bx ? m.ly[J] : zero, bx ? m.uy[J] : zero);
      if (v > bv) { bv = v; bj = J; }  // J ascending per thread: ties keep the lowest
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int32_t j2 = __shfl_xor_sync(0xffffffffu, bj, o);
    if (v2 > bv || (v2 == bv && j2 < bj)) { bv = v2; bj = j2; }
  }
  if (lane == 0) { sv[warp] = bv; sj[warp] = bj; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < kMaskThreads / 32; ++q)
      if (sv[q] > bv || (sv[q] == bv && sj[q] < bj)) { bv = sv[q]; bj = sj[q]; }
    best[I] = bj == 0x7fffffff ? -1 : bj;
  }
}

// Column best pairs without the transposed mask: for every column cluster J
// with no kept pair (colany bit clear) the exact arg-max over the row clusters
// (ties -> lowest I); -1 for the others.  One CTA per mask word of columns.
__global__ void __launch_bounds__(kMaskThreads)
mask_colbest_kernel(MaskIn m, const uint32_t* colany, int32_t* best) {
  __shared__ double sv[kMaskThreads / 32];
  __shared__ int32_t sj[kMaskThreads / 32];
  const int32_t w = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  const bool g = m.gx != nullptr;
  const uint32_t have = colany[w];
  for (int b = 0; b < 32; ++b) {
    const int32_t J = w * 32 + b;
    if (J >= m.ky) break;
    if (have >> b & 1u) {
      if (threadIdx.x == 0) best[J] = -1;
      continue;
    }
    const float4 Y = m.cy[J];
    const float rJ = m.ry[J], G = m.gy[J];
    const float4 HJ = g ? m.hy[J] : zero;
    double bv = -INFINITY;
    int32_t bi = 0x7fffffff;
    for (int32_t I = threadIdx.x; I < m.kx; I += kMaskThreads) {
      const float4 X = m.cx[I];
      const float rI = m.rx[I], F = m.fx[I];
      if (static_cast<double>(ub_regs(X, rI, F, Y, rJ, G, m.d)) >= bv) {
        const bool bx = m.box();
        const double v = pair_slack(X, rI, F, g ? m.gx[I] : zero, Y, rJ, G, HJ, m.d, g, bx,
                                    bx ? m.lx[I] : zero, bx ? m.ux[I] : zero,
                                    bx ? m.ly[J] : zero, bx ? m.uy[J] : zero);
        if (v > bv) { bv = v; bi = I; }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
      const int32_t i2 = __shfl_xor_sync(0xffffffffu, bi, o);
      if (v2 > bv || (v2 == bv && i2 < bi)) { bv = v2; bi = i2; }
    }
    if (lane == 0) { sv[warp] = bv; sj[warp] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < kMaskThreads / 32; ++q)
        if (sv[q] > bv || (sv[q] == bv && sj[q] < bi)) { bv = sv[q]; bi = sj[q]; }
      best[J] = bi == 0x7fffffff ? -1 : bi;
    }
    __syncthreads();
  }
}

// Best pairs into the masks: row I's best J (br) and column J's best I (bc)
// set (I, J) in `mask` and (J, I) in `maskT` (nullable; == mask for a self
// mask, whose best pairs are symmetric).
__global__ void mask_best_kernel(const int32_t* br, int32_t r0, int32_t r1, const int32_t* bc,
                                 int32_t ky, uint32_t* mask, int32_t wx, uint32_t* maskT,
                                 int32_t wt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nr = r1 - r0;
  int32_t I, J;
  if (t < nr) {
    I = r0 + static_cast<int32_t>(t);
    J = br[I];
  } else if (t < nr + ky) {
    J = static_cast<int32_t>(t - nr);
    I = bc[J];
  } else {
    return;
  }
  if (I < 0 || J < 0) return;
  atomicOr(&mask[static_cast<int64_t>(I) * wx + (J >> 5)], 1u << (J & 31));
  if (maskT) atomicOr(&maskT[static_cast<int64_t>(J) * wt + (I >> 5)], 1u << (I & 31));
}

// Lower half of a self mask from its upper half: the slack is exactly
// symmetric (pair_slack), so bit (I, J) = bit (J, I).  One CTA per 8 x 8
// group of 32 x 32 bit blocks (bi, bj), bj < bi: warp w reads rows
// (8 BJ + w) * 32 + lane, words 8 BI .. 8 BI + 7 (one sector per row), 32
// ballots per block transpose them into shared memory, and each thread then
// writes one row's 8 words of the group (one sector per row).
__global__ void __launch_bounds__(256) mask_mirror_kernel(uint32_t* mask, int32_t k, int32_t words) {
  __shared__ uint32_t T[256][9];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int32_t BI = static_cast<int32_t>(blockIdx.y), BJ = static_cast<int32_t>(blockIdx.x);
  if (BJ > BI) return;
  const int32_t bj = BJ * 8 + w, J = bj * 32 + lane;
  uint32_t vq[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {  // all eight loads in flight
    const int32_t bi = BI * 8 + q;
    vq[q] = (J < k && bi < words) ? mask[static_cast<int64_t>(J) * words + bi] : 0u;
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t v = vq[q];
    uint32_t out = 0u;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      const uint32_t t = __ballot_sync(0xffffffffu, (v >> b) & 1u);
      if (lane == b) out = t;
    }
    T[q * 32 + lane][w] = out;  // row bi * 32 + lane, word bj
  }
  __syncthreads();
  const int32_t I = BI * 256 + static_cast<int32_t>(threadIdx.x);
  if (I >= k) return;
  const int32_t bi = I >> 5;
  uint32_t* row = mask + static_cast<int64_t>(I) * words;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int32_t wj = BJ * 8 + q;
    if (wj < bi) row[wj] = T[threadIdx.x][q];
  }
}

cudaError_t mask_mirror(uint32_t* mask, int32_t k, cudaStream_t st) {
  if (k <= 32) return cudaSuccess;
  const int32_t words = mask_words(k);
  const unsigned g = static_cast<unsigned>((words + 7) / 8);
  ++g_launches;
  mask_mirror_kernel<<<dim3(g, g), 256, 0, st>>>(mask, k, words);
  return cudaGetLastError();
}

cudaError_t truncation_masks(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                             const float* fx, const float4* gx, const float4* cy, const float* ry,
                             const float* gy, const float4* hy, double eps, double theta, int self,
                             uint32_t* mask, uint32_t* maskT, int32_t* best_r, int32_t* best_c,
                             void* blkws, cudaStream_t st, const float4* const* box) {
  if (kx <= 0 || ky <= 0) return cudaSuccess;
  if ((gx == nullptr) != (hy == nullptr)) return cudaErrorInvalidValue;
  if (box && gx == nullptr) return cudaErrorInvalidValue;
  if (self && kx != ky) return cudaErrorInvalidValue;
  const double thr = -(theta * eps);
  MaskIn m{kx, ky, d, mask_words(ky), cx, cy, rx, ry, fx, gy, gx, hy};
  if (box) { m.lx = box[0]; m.ux = box[1]; m.ly = box[2]; m.uy = box[3]; }
  // layout of blkws: float4 blocks of y, float4 blocks of x, the float maxima,
  // then the column-any words
  float4* blk_y = reinterpret_cast<float4*>(blkws);
  float4* blk_x = blk_y + mask_words(ky);
  float* blkg_y = reinterpret_cast<float*>(blk_x + mask_words(kx));
  float* blkg_x = blkg_y + mask_words(ky);
  uint32_t* colany = reinterpret_cast<uint32_t*>(blkg_x + mask_words(kx));
  const bool col_pass = !self && maskT == nullptr;  // column bests without the transpose
  if (col_pass) {
    const cudaError_t e = cudaMemsetAsync(colany, 0, sizeof(uint32_t) * mask_words(ky), st);
    if (e != cudaSuccess) return e;
  }
  ++g_launches;
  block_bounds_kernel<<<static_cast<unsigned>((mask_words(ky) * 32 + 255) / 256), 256, 0, st>>>(
      cy, ry, gy, ky, d, blk_y, blkg_y);
  ++g_launches;
  mask_rows_kernel<<<static_cast<unsigned>(kx), kMaskThreads, 0, st>>>(
      m, blk_y, blkg_y, thr, self, mask, best_r, col_pass ? colany : nullptr, 0, self);
  if (self) {
    const cudaError_t e = mask_mirror(mask, kx, st);
    if (e != cudaSuccess) return e;
    ++g_launches;
    mask_best_kernel<<<static_cast<unsigned>((kx + 255) / 256), 256, 0, st>>>(
        best_r, 0, kx, best_r, 0, mask, m.words, mask, m.words);
    return cudaGetLastError();
  }
  if (col_pass) {
    ++g_launches;
    mask_colbest_kernel<<<static_cast<unsigned>(mask_words(ky)), kMaskThreads, 0, st>>>(m, colany,
                                                                                      best_c);
    ++g_launches;
    mask_best_kernel<<<static_cast<unsigned>((static_cast<int64_t>(kx) + ky + 255) / 256), 256, 0,
                       st>>>(best_r, 0, kx, best_c, ky, mask, m.words, nullptr, 0);
    return cudaGetLastError();
  }
  // the transposed problem: same formula with the roles swapped (pair_slack
  // is exactly symmetric), so maskT is the bitwise transpose of mask
  MaskIn t{ky, kx, d, mask_words(kx), cy, cx, ry, rx, gy, fx, hy, gx};
  if (box) { t.lx = box[2]; t.ux = box[3]; t.ly = box[0]; t.uy = box[1]; }
  ++g_launches;
  block_bounds_kernel<<<static_cast<unsigned>((mask_words(kx) * 32 + 255) / 256), 256, 0, st>>>(
      cx, rx, fx, kx, d, blk_x, blkg_x);
  ++g_launches;
  mask_rows_kernel<<<static_cast<unsigned>(ky), kMaskThreads, 0, st>>>(t, blk_x, blkg_x, thr, 0,
                                                                         maskT, best_c, nullptr, 0, 0);
  ++g_launches;
  mask_best_kernel<<<static_cast<unsigned>((static_cast<int64_t>(kx) + ky + 255) / 256), 256, 0, st>>>(
      best_r, 0, kx, best_c, ky, mask, m.words, maskT, t.words);
  return cudaGetLastError();
}

// Diagnostic (profiling only): sum over kept cluster pairs of n_I * m_J,
// the pair count of the mask at cluster granularity (what the block-sparse
// reduction would evaluate with no tile-level union).
// Row-sharded truncation masks (multi-GPU fine phase): part 1 computes the
// rows [r0, r1) of the mask and their best pairs (rows with no kept pair);
// after the callers exchange the row blocks, part 2 (cross masks only) forms
// each column's any-bit from the whole mask and sets the column best pairs
// of the columns with none — every rank identically.  With [0, kx) and no
// exchange this is bitwise truncation_masks(maskT = nullptr).
// OR of the mask rows per word: blockIdx.y strides the rows, atomicOr merges
// (order-free, so deterministic); colany must be zeroed first.
__global__ void col_any_kernel(const uint32_t* mask, int32_t kx, int32_t words, uint32_t* colany) {
  const int32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= words) return;
  uint32_t a = 0u;
  for (int32_t I = blockIdx.y; I < kx; I += gridDim.y) a |= mask[static_cast<int64_t>(I) * words + w];
  if (a) atomicOr(colany + w, a);
}

cudaError_t truncation_masks_rows(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                                  const float* fx, const float4* gx, const float4* cy,
                                  const float* ry, const float* gy, const float4* hy, double eps,
                                  double theta, int self, int32_t r0, int32_t r1, uint32_t* mask,
                                  int32_t* best_r, void* blkws, cudaStream_t st,
                                  const float4* const* box) {
  if (kx <= 0 || ky <= 0) return cudaSuccess;
  if ((gx == nullptr) != (hy == nullptr)) return cudaErrorInvalidValue;
  if (box && gx == nullptr) return cudaErrorInvalidValue;
  if (self && kx != ky) return cudaErrorInvalidValue;
  const double thr = -(theta * eps);
  MaskIn m{kx, ky, d, mask_words(ky), cx, cy, rx, ry, fx, gy, gx, hy};
  if (box) { m.lx = box[0]; m.ux = box[1]; m.ly = box[2]; m.uy = box[3]; }
  float4* blk_y = reinterpret_cast<float4*>(blkws);
  float4* blk_x = blk_y + mask_words(ky);
  float* blkg_y = reinterpret_cast<float*>(blk_x + mask_words(kx));
  ++g_launches;
  block_bounds_kernel<<<static_cast<unsigned>((mask_words(ky) * 32 + 255) / 256), 256, 0, st>>>(
      cy, ry, gy, ky, d, blk_y, blkg_y);
  if (r1 <= r0) return cudaGetLastError();
  ++g_launches;
  mask_rows_kernel<<<static_cast<unsigned>(r1 - r0), kMaskThreads, 0, st>>>(
      m, blk_y, blkg_y, thr, self, mask, best_r, nullptr, r0, self);
  ++g_launches;
  mask_best_kernel<<<static_cast<unsigned>((r1 - r0 + 255) / 256), 256, 0, st>>>(
      best_r, r0, r1, nullptr, 0, mask, m.words, nullptr, 0);
  return cudaGetLastError();
}

cudaError_t truncation_masks_cols(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                                  const float* fx, const float4* gx, const float4* cy,
                                  const float* ry, const float* gy, const float4* hy, uint32_t* mask,
                                  int32_t* best_c, void* blkws, cudaStream_t st,
                                  const float4* const* box) {
  if (kx <= 0 || ky <= 0) return cudaSuccess;
  if (box && gx == nullptr) return cudaErrorInvalidValue;
  MaskIn m{kx, ky, d, mask_words(ky), cx, cy, rx, ry, fx, gy, gx, hy};
  if (box) { m.lx = box[0]; m.ux = box[1]; m.ly = box[2]; m.uy = box[3]; }
  float4* blk_y = reinterpret_cast<float4*>(blkws);
  float4* blk_x = blk_y + mask_words(ky);
  float* blkg_y = reinterpret_cast<float*>(blk_x + mask_words(kx));
  float* blkg_x = blkg_y + mask_words(ky);
  uint32_t* colany = reinterpret_cast<uint32_t*>(blkg_x + mask_words(kx));
  cudaError_t e = cudaMemsetAsync(colany, 0, sizeof(uint32_t) * m.words, st);
  if (e != cudaSuccess) return e;
  ++g_launches;
  const unsigned ry_blocks = static_cast<unsigned>(kx < 256 ? kx : 256);
  col_any_kernel<<<dim3(static_cast<unsigned>((m.words + 127) / 128), ry_blocks), 128, 0, st>>>(
      mask, kx, m.words, colany);
  ++g_launches;
  mask_colbest_kernel<<<static_cast<unsigned>(m.words), kMaskThreads, 0, st>>>(m, colany, best_c);
  ++g_launches;
  mask_best_kernel<<<static_cast<unsigned>((ky + 255) / 256), 256, 0, st>>>(
      nullptr, 0, 0, best_c, ky, mask, m.words, nullptr, 0);
  return cudaGetLastError();
}

__global__ void mask_pair_count_kernel(const uint32_t* mask, int32_t kx, int32_t ky,
                                       const int32_t* ro, const int32_t* co, double* out) {
  const int32_t I = blockIdx.x;
  const int32_t words = mask_words(ky);
  double s = 0.0;
  for (int32_t w = threadIdx.x; w < words; w += blockDim.x) {
    uint32_t b = mask[static_cast<int64_t>(I) * words + w];
    while (b) {
      const int32_t J = w * 32 + __ffs(b) - 1;
      b &= b - 1;
      s += static_cast<double>(co[J + 1] - co[J]);
    }
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, s * static_cast<double>(ro[I + 1] - ro[I]));
}

cudaError_t mask_pair_count(const uint32_t* mask, int32_t kx, int32_t ky, const int32_t* ro,
                            const int32_t* co, double* out, cudaStream_t st) {
  if (kx <= 0) return cudaSuccess;
  ++g_launches;
  mask_pair_count_kernel<<<kx, 128, 0, st>>>(mask, kx, ky, ro, co, out);
  return cudaGetLastError();
}

// ---- high-D masks (K-means clusters, D <= 64) -----------------------------
// B_a = F_I + G_J - 1/2 max(0, |X_I - Y_J| - (r_I + r_J))^2 with float64
// centroids, |X_I - Y_J|^2 summed in coordinate order, explicitly rounded
// (bit-identical to oracle.cpp:hd_pair_slack).  One CTA per row cluster.
__device__ __forceinline__ double hd_pair_slack(const double* X, float rI, float F, const double* Y,
                                                float rJ, float G, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = __dsub_rn(X[k], Y[k]);
    s = __dadd_rn(s, __dmul_rn(t, t));
  }
  const double rr = __dadd_rn(static_cast<double>(rI), static_cast<double>(rJ));
  double lb = __dsub_rn(__dsqrt_rn(s), rr);
  if (lb < 0.0) lb = 0.0;
  const double fg = __dadd_rn(static_cast<double>(F), static_cast<double>(G));
  return __dsub_rn(fg, __dmul_rn(0.5, __dmul_rn(lb, lb)));
}

__global__ void __launch_bounds__(256)
mask_hd_rows_kernel(const double* cx, const float* rx, const float* fx, const double* cy,
                    const float* ry, const float* gy, int32_t ky, int d, double thr, int self,
                    uint32_t* mask, int32_t* best) {
  __shared__ double X[64];
  __shared__ double sv[8];
  __shared__ int32_t sj[8];
  const int32_t I = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = threadIdx.x; q < d; q += blockDim.x) X[q] = cx[static_cast<int64_t>(I) * d + q];
  __syncthreads();
  const float rI = rx[I], F = fx[I];
  const int32_t words = mask_words(ky);
  double bv = -INFINITY;
  int32_t bj = 0x7fffffff;
  for (int32_t w = warp; w < words; w += 8) {
    const int32_t J = w * 32 + lane;
    bool keep = false;
    if (J < ky) {
      const double v = hd_pair_slack(X, rI, F, cy + static_cast<int64_t>(J) * d, ry[J], gy[J], d);
      keep = (self && I == J) || v >= thr;
      if (v > bv) { bv = v; bj = J; }
    }
    const uint32_t bits = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) mask[static_cast<int64_t>(I) * words + w] = bits;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int32_t j2 = __shfl_xor_sync(0xffffffffu, bj, o);
    if (v2 > bv || (v2 == bv && j2 < bj)) { bv = v2; bj = j2; }
  }
  if (lane == 0) { sv[warp] = bv; sj[warp] = bj; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < 8; ++q)
      if (sv[q] > bv || (sv[q] == bv && sj[q] < bj)) { bv = sv[q]; bj = sj[q]; }
    best[I] = bj == 0x7fffffff ? -1 : bj;
  }
}

cudaError_t truncation_masks_hd(int32_t kx, int32_t ky, int d, const double* cx, const float* rx,
                                const float* fx, const double* cy, const float* ry,
                                const float* gy, double eps, double theta, int self,
                                uint32_t* mask, uint32_t* maskT, int32_t* best_r, int32_t* best_c,
                                cudaStream_t st) {
  if (kx <= 0 || ky <= 0) return cudaSuccess;
  if (d > 64 || (self && kx != ky)) return cudaErrorInvalidValue;
  const double thr = -(theta * eps);
  ++g_launches;
  mask_hd_rows_kernel<<<static_cast<unsigned>(kx), 256, 0, st>>>(cx, rx, fx, cy, ry, gy, ky, d,
                                                                   thr, self, mask, best_r);
  if (self) {
    ++g_launches;
    mask_best_kernel<<<static_cast<unsigned>((kx + 255) / 256), 256, 0, st>>>(
        best_r, 0, kx, best_r, 0, mask, mask_words(ky), mask, mask_words(ky));
    return cudaGetLastError();
  }
  ++g_launches;
  mask_hd_rows_kernel<<<static_cast<unsigned>(ky), 256, 0, st>>>(cy, ry, gy, cx, rx, fx, kx, d,
                                                                   thr, 0, maskT, best_c);
  ++g_launches;
  mask_best_kernel<<<static_cast<unsigned>((static_cast<int64_t>(kx) + ky + 255) / 256), 256, 0, st>>>(
      best_r, 0, kx, best_c, ky, mask, mask_words(ky), maskT, mask_words(kx));
  return cudaGetLastError();
}

__global__ void unpack_kernel(const uint32_t* mask, int32_t kx, int32_t ky, uint8_t* out) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= static_cast<int64_t>(kx) * ky) return;
  const int64_t I = g / ky, J = g % ky;
  out[g] = (mask[I * mask_words(ky) + (J >> 5)] >> (J & 31)) & 1u;
}

cudaError_t unpack_mask(const uint32_t* mask, int32_t kx, int32_t ky, uint8_t* out,
                        cudaStream_t st) {
  const int64_t n = static_cast<int64_t>(kx) * ky;
  if (n <= 0) return cudaSuccess;
  ++g_launches; unpack_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(mask, kx, ky, out);
  return cudaGetLastError();
}

// ---- ranges per row tile -------------------------------------------------
__global__ void tile_or_kernel(const uint32_t* mask, int32_t words, const int32_t* rl,
                               const int32_t* ts, int64_t nt, uint32_t* tbits) {
  const int32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t t = blockIdx.y;
  if (w >= words || t >= nt) return;
  const int32_t I0 = rl[ts[t]], I1 = rl[ts[t + 1] - 1];
  uint32_t b = 0;
  for (int32_t I = I0; I <= I1; ++I) b |= mask[static_cast<int64_t>(I) * words + w];
  tbits[t * words + w] = b;
}

template <bool kWrite>
__global__ void tile_runs_kernel(const uint32_t* tbits, int32_t words, int64_t nt,
                                 const int32_t* co, int64_t* n_ranges, int64_t* n_cols,
                                 const int64_t* rptr, int2* ranges) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= nt) return;
  const uint32_t* tb = tbits + t * words;
  int64_t ns = 0, ne = 0, cols = 0;
  const int64_t base = kWrite ? rptr[t] : 0;
  uint32_t carry = 0;  // top bit of the previous word
  for (int32_t w0 = 0; w0 < words; w0 += 32) {
    const int32_t w = w0 + lane;
    const uint32_t b = w < words ? tb[w] : 0u;
    const uint32_t up = __shfl_up_sync(0xffffffffu, b, 1);
    const uint32_t cin = lane == 0 ? carry : (up >> 31);
    uint32_t dn = __shfl_down_sync(0xffffffffu, b, 1);
    if (lane == 31) dn = (w0 + 32 < words) ? tb[w0 + 32] : 0u;
    const uint32_t starts = b & ~((b << 1) | cin);
    const uint32_t ends = b & ~((b >> 1) | ((dn & 1u) << 31));
    // warp prefix counts (a run may start in one lane and end in another)
    const int ps = __popc(starts), pe = __popc(ends);
    int xs = ps, xe = pe;
    for (int o = 1; o < 32; o <<= 1) {
      const int ys = __shfl_up_sync(0xffffffffu, xs, o);
      const int ye = __shfl_up_sync(0xffffffffu, xe, o);
      if (lane >= o) { xs += ys; xe += ye; }
    }
    int64_t ks = ns + xs - ps, ke = ne + xe - pe;
    uint32_t s = starts, e = ends;
    while (s) {
      const int bpos = __ffs(s) - 1;
      s &= s - 1;
      const int32_t J = w * 32 + bpos;
      if (kWrite) ranges[base + ks].x = co[J];
      else cols -= co[J];
      ++ks;
    }
    while (e) {
      const int bpos = __ffs(e) - 1;
      e &= e - 1;
      const int32_t J = w * 32 + bpos;
      if (kWrite) ranges[base + ke].y = co[J + 1];
      else cols += co[J + 1];
      ++ke;
    }
    ns += __shfl_sync(0xffffffffu, xs, 31);
    ne += __shfl_sync(0xffffffffu, xe, 31);
    carry = __shfl_sync(0xffffffffu, b, 31) >> 31;
  }
  if (!kWrite) {
    for (int o = 16; o > 0; o >>= 1) cols += __shfl_xor_sync(0xffffffffu, cols, o);
    if (lane == 0) {
      n_ranges[t] = ns;
      n_cols[t] = cols;
    }
  }
}

cudaError_t tile_or(const uint32_t* mask, int32_t ky, const int32_t* row_labels,
                    const int32_t* tile_start, int64_t nt, uint32_t* tbits, cudaStream_t st) {
  if (nt <= 0) return cudaSuccess;
  const int32_t words = mask_words(ky);
  dim3 grid((words + 127) / 128, static_cast<unsigned>(nt));
  ++g_launches; tile_or_kernel<<<grid, 128, 0, st>>>(mask, words, row_labels, tile_start, nt, tbits);
  return cudaGetLastError();
}

cudaError_t tile_range_count(const uint32_t* tbits, int32_t ky, int64_t nt,
                             const int32_t* col_offsets, int64_t* n_ranges, int64_t* n_cols,
                             cudaStream_t st) {
  if (nt <= 0) return cudaSuccess;
  ++g_launches; tile_runs_kernel<false><<<static_cast<unsigned>((nt * 32 + 255) / 256), 256, 0, st>>>(
      tbits, mask_words(ky), nt, col_offsets, n_ranges, n_cols, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t tile_range_write(const uint32_t* tbits, int32_t ky, int64_t nt,
                             const int32_t* col_offsets, const int64_t* rptr, int2* ranges,
                             cudaStream_t st) {
  if (nt <= 0) return cudaSuccess;
  ++g_launches; tile_runs_kernel<true><<<static_cast<unsigned>((nt * 32 + 255) / 256), 256, 0, st>>>(
      tbits, mask_words(ky), nt, col_offsets, nullptr, nullptr, rptr, ranges);
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

// ---- evaluate-once pair sets (softmin_sym.cu) -----------------------------
// Every kept pair is evaluated once and feeds its row sum and its column sum.
// Tile t's column list:
//   cross (rows x, cols y): the runs of the tile-OR clusters (as tile_runs);
//   self: a head range [ts, co[I1 + 1]) — the diagonal block plus the rest of
//         the tile's last cluster I1 — then the runs of the tile-OR clusters
//         J > I1.  Columns below te only feed row sums; column k >= te(t) of
//         the list gets tile t's rows as a column sum, which makes the pair
//         set symmetric (oracle.cpp:sym_self).
// posword[t][w] = position of word w's first cluster in tile t's list, so the
// column-major pass can place every (tile, cluster) entry without a sort.

// bits of tile t's word w that are list clusters: self keeps J > I1 only
__device__ __forceinline__ uint32_t list_bits(uint32_t b, int32_t w, int32_t I1, bool self) {
  if (!self) return b;
  const int32_t k = I1 - w * 32;  // clear bits 0..k
  if (k < 0) return b;
  if (k >= 31) return 0u;
  return b & (~0u << (k + 1));
}

template <bool kWrite>
__global__ void sym_runs_kernel(const uint32_t* tbits, int32_t words, int64_t nt,
                                const int32_t* co, const int32_t* ts, const int32_t* rl, int self,
                                int64_t* n_ranges, int64_t* n_cols, int32_t* posword,
                                const int64_t* rptr, int2* ranges) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (t >= nt) return;
  const uint32_t* tb = tbits + t * words;
  const int32_t I1 = self ? rl[ts[t + 1] - 1] : -1;
  const int64_t hn = self ? 1 : 0;  // the head range
  int64_t cols = self ? co[I1 + 1] - ts[t] : 0, ns = 0, ne = 0;
  const int64_t base = kWrite ? rptr[t] : 0;
  if (kWrite && self && lane == 0) ranges[base] = make_int2(ts[t], co[I1 + 1]);
  uint32_t carry = 0;  // top bit of the previous word
  // self: the words below I1's hold no list bits (posword is read only where
  // a word has list bits)
  for (int32_t w0 = self ? ((I1 >> 5) & ~31) : 0; w0 < words; w0 += 32) {
    const int32_t w = w0 + lane;
    const uint32_t b = w < words ? list_bits(tb[w], w, I1, self) : 0u;
    const uint32_t up = __shfl_up_sync(0xffffffffu, b, 1);
    const uint32_t cin = lane == 0 ? carry : (up >> 31);
    uint32_t dn = __shfl_down_sync(0xffffffffu, b, 1);
    if (lane == 31) dn = (w0 + 32 < words) ? list_bits(tb[w0 + 32], w0 + 32, I1, self) : 0u;
    const uint32_t starts = b & ~((b << 1) | cin);
    const uint32_t ends = b & ~((b >> 1) | ((dn & 1u) << 31));
    int64_t contrib = 0;  // columns of the runs: -co[start] + co[end + 1]
    for (uint32_t q = starts; q; q &= q - 1) contrib -= co[w * 32 + __ffs(q) - 1];
    for (uint32_t q = ends; q; q &= q - 1) contrib += co[w * 32 + __ffs(q)];
    const int ps = __popc(starts), pe = __popc(ends);
    int xs = ps, xe = pe;
    int64_t xc = contrib;
    for (int o = 1; o < 32; o <<= 1) {
      const int ys = __shfl_up_sync(0xffffffffu, xs, o);
      const int ye = __shfl_up_sync(0xffffffffu, xe, o);
      const int64_t yc = __shfl_up_sync(0xffffffffu, xc, o);
      if (lane >= o) { xs += ys; xe += ye; xc += yc; }
    }
    if (!kWrite && w < words) {
      // a run open across the word boundary counts up to the boundary
      const int64_t open = (cin && (b & 1u)) ? co[w * 32] : 0;
      posword[t * words + w] = static_cast<int32_t>(cols + xc - contrib + open);
    }
    if (kWrite) {
      int64_t ks = hn + ns + xs - ps, ke = hn + ne + xe - pe;
      for (uint32_t q = starts; q; q &= q - 1) ranges[base + ks++].x = co[w * 32 + __ffs(q) - 1];
      for (uint32_t q = ends; q; q &= q - 1) ranges[base + ke++].y = co[w * 32 + __ffs(q)];
    }
    ns += __shfl_sync(0xffffffffu, xs, 31);
    ne += __shfl_sync(0xffffffffu, xe, 31);
    cols += __shfl_sync(0xffffffffu, xc, 31);
    carry = __shfl_sync(0xffffffffu, b, 31) >> 31;
  }
  if (!kWrite && lane == 0) {
    n_ranges[t] = hn + ns;
    n_cols[t] = cols;
  }
}

// Column-major pass over the (tile, cluster) entries: warp = one word of 32
// column clusters x one chunk of tiles (ascending).  kFill = false counts the
// entries of every (cluster, chunk); kFill writes, in tile order, the colpart
// slot of the cluster's first column in each tile's list.  Self problems add
// the head entry of the tile's last cluster I1 (slot of column co[I1]).
template <bool kFill>
__global__ void sym_entries_kernel(const uint32_t* tbits, int32_t words, int32_t k, int64_t nt,
                                   const int32_t* co, const int32_t* ts, const int32_t* rl,
                                   int self, const int32_t* posword, const int64_t* tslot,
                                   int32_t* cnt, const int64_t* ebase, int64_t* eslot,
                                   int32_t* etile) {
  const int lane = threadIdx.x & 31;
  const int32_t w = static_cast<int32_t>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
  const int ch = blockIdx.y;
  if (w >= words) return;
  const int32_t J = w * 32 + lane;
  const int64_t t0 = nt * ch / kEntryChunks, t1 = nt * (ch + 1) / kEntryChunks;
  const int64_t ncl = J < k ? co[J + 1] - co[J] : 0;
  int64_t e = kFill ? ebase[static_cast<int64_t>(J < k ? J : 0) * kEntryChunks + ch] : 0;
  int32_t c = 0;
  // one tile ahead in flight (the walk is latency-bound)
  int32_t I1n = (self && t0 < t1) ? rl[ts[t0 + 1] - 1] : -1;
  uint32_t bn = t0 < t1 ? tbits[t0 * words + w] : 0u;
  for (int64_t t = t0; t < t1; ++t) {
    const int32_t I1 = I1n;
    // self: I1 grows with t, and past this word neither list bits nor the
    // head entry remain
    if (self && I1 >= (w + 1) * 32) break;
    const uint32_t braw = bn;
    if (t + 1 < t1) {
      I1n = self ? rl[ts[t + 2] - 1] : -1;
      bn = tbits[(t + 1) * words + w];
    }
    const uint32_t b = list_bits(braw, w, I1, self);
    const bool head = self && J == I1;
    const bool mine = J < k && (((b >> lane) & 1u) || head);
    if (!__any_sync(0xffffffffu, mine)) continue;
    if (!kFill) {
      c += mine;
      continue;
    }
    // position of cluster J in tile t's list: word base + list columns of
    // the lower clusters of this word
    int64_t pre = ((b >> lane) & 1u) ? ncl : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    if (mine) {
      const int64_t posJ = head ? static_cast<int64_t>(co[J]) - ts[t]
                                : posword[t * words + w] + pre - ncl;
      eslot[e] = tslot[t] + posJ;
      etile[e] = static_cast<int32_t>(t);
      ++e;
    }
  }
  if (!kFill && J < k) cnt[static_cast<int64_t>(J) * kEntryChunks + ch] = c;
}

cudaError_t sym_ranges(const uint32_t* tbits, int32_t k, int64_t nt, const int32_t* co,
                       const int32_t* ts, const int32_t* rl, int self, int64_t* n_ranges,
                       int64_t* n_cols, int32_t* posword, const int64_t* rptr, int2* ranges,
                       bool write, cudaStream_t st) {
  if (nt <= 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>((nt * 32 + 255) / 256);
  ++g_launches;
  if (write)
    sym_runs_kernel<true><<<grid, 256, 0, st>>>(tbits, mask_words(k), nt, co, ts, rl, self,
                                                 nullptr, nullptr, nullptr, rptr, ranges);
  else
    sym_runs_kernel<false><<<grid, 256, 0, st>>>(tbits, mask_words(k), nt, co, ts, rl, self,
                                                  n_ranges, n_cols, posword, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t sym_entries(const uint32_t* tbits, int32_t k, int64_t nt, const int32_t* co,
                        const int32_t* ts, const int32_t* rl, int self, const int32_t* posword,
                        const int64_t* tslot, int32_t* cnt, const int64_t* ebase, int64_t* eslot,
                        int32_t* etile, bool fill, cudaStream_t st) {
  if (nt <= 0 || k <= 0) return cudaSuccess;
  const int32_t words = mask_words(k);
  dim3 grid(static_cast<unsigned>((static_cast<int64_t>(words) * 32 + 127) / 128), kEntryChunks);
  ++g_launches;
  if (fill)
    sym_entries_kernel<true><<<grid, 128, 0, st>>>(tbits, words, k, nt, co, ts, rl, self, posword,
                                                   tslot, nullptr, ebase, eslot, etile);
  else
    sym_entries_kernel<false><<<grid, 128, 0, st>>>(tbits, words, k, nt, co, ts, rl, self,
                                                    posword, tslot, cnt, nullptr, nullptr, nullptr);
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
