// oracle.cpp — FP64 CPU restatement of the multiscale Sinkhorn hot path.
//
// TEST INFRASTRUCTURE (see oracle.h): the checker for the CUDA path and the
// timed CPU baseline.  Never linked into the product library.
//
// Executor and summation are the reference's own code, built unmodified from
// /root/reference/proj/src/{parallel,numeric}.cpp into oracle/_ref/ by
// oracle/Makefile:
//   msot::parallel::for_ranges  (parallel.hpp:17, parallel.cpp:102-123)
//   msot::pairwise_dot          (numeric.hpp:15,  numeric.cpp:44-47)
//   msot::kahan_sum             (numeric.hpp:9,   numeric.cpp:7-17)
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <span>
#include <string>
#include <vector>

#include "../paper_2107_02010_b200/csrc/policy.h"

// Prototypes of the reference utilities we link against (declared in
// /root/reference/proj/include/msot/{numeric,parallel}.hpp).
namespace msot {
double kahan_sum(std::span<const double> values);
double pairwise_sum(std::span<const double> values);
double pairwise_dot(std::span<const double> a, std::span<const double> b);
namespace parallel {
int threads();
void set_threads(int n);
void for_ranges(std::size_t n, const std::function<void(std::size_t, std::size_t)>& fn);
}  // namespace parallel
}  // namespace msot

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

using Vec = std::vector<double>;

// C(x,y) = (1/p)|x-y|^p  (measure.hpp:18).
inline double cost(const double* x, const double* y, int d, double p) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = x[k] - y[k];
    s += t * t;
  }
  if (p == 2.0) return 0.5 * s;
  return std::pow(std::sqrt(s), p) / p;
}

// A set of columns for a softmin: atoms, log-weights, potentials.
struct Cols {
  const double* pts;
  const double* logw;
  const double* h;
  int64_t m;
};

// Block-sparse structure: column ranges per row tile (nullptr = dense).
struct Ranges {
  std::vector<int64_t> tile_start;  // T+1 row boundaries (policy.h:msot_pack_tiles)
  std::vector<int32_t> row_tile;    // row -> tile
  std::vector<int64_t> tile_ptr;    // T+1 range boundaries
  std::vector<int32_t> r;           // pairs [begin, end)
};

// softmin over rows (PAPER.md:258-290 lines 4-7):
//   out_i = -lam * eps * log sum_k w_k exp((h_k - C(x_i, y_k)) / eps)
// evaluated with a max shift in FP64.  `rg` restricts row i to the column
// ranges of its tile (the block-sparse reduction of SPEC.md:290-298).
// Returns the number of evaluated pairs.
double softmin_rows(const double* xr, int64_t n, int d, const Cols& c, double eps, double lam,
                    double p, const Ranges* rg, double* out) {
  std::vector<double> pairs_per_chunk(std::max(1, msot::parallel::threads()), 0.0);
  msot::parallel::for_ranges(static_cast<std::size_t>(n), [&](std::size_t b, std::size_t e) {
    std::vector<double> z;
    double cnt = 0.0;
    for (std::size_t i = b; i < e; ++i) {
      const double* xi = xr + i * d;
      int64_t r0 = 0, r1 = 1;
      int32_t dense[2] = {0, static_cast<int32_t>(c.m)};
      const int32_t* rr = dense;
      if (rg) {
        const int64_t t = rg->row_tile[i];
        r0 = rg->tile_ptr[t];
        r1 = rg->tile_ptr[t + 1];
        rr = rg->r.data();
      }
      // max-shifted LSE over blocks of kBlock terms: a block is buffered,
      // its max folded into the running max (rescaling the sum), then summed
      // -- one block (every block-sparse row of the tests) is the plain
      // two-pass LSE; dense rows over 1M columns stay in cache
      constexpr std::size_t kBlock = 4096;
      z.clear();
      double zmax = -std::numeric_limits<double>::infinity(), s = 0.0;
      auto flush = [&]() {
        double bmax = -std::numeric_limits<double>::infinity();
        for (double v : z) bmax = std::max(bmax, v);
        if (bmax > zmax) {
          if (s != 0.0) s *= std::exp(zmax - bmax);
          zmax = bmax;
        }
        for (double v : z) {
          const double e = v - zmax;  // exp(e) rounds to +0 below -746: skip the call
          if (e > -746.0) s += std::exp(e);
        }
        cnt += static_cast<double>(z.size());
        z.clear();
      };
      for (int64_t q = r0; q < r1; ++q) {
        for (int32_t k = rr[2 * q]; k < rr[2 * q + 1]; ++k) {
          z.push_back(c.logw[k] + (c.h[k] - cost(xi, c.pts + int64_t(k) * d, d, p)) / eps);
          if (z.size() == kBlock) flush();
        }
      }
      if (!z.empty()) flush();
      out[i] = -lam * eps * (zmax + std::log(s));
    }
    // one chunk per thread slot; slot index recovered from the chunk start
    const std::size_t slots = pairs_per_chunk.size();
    const std::size_t chunk = (static_cast<std::size_t>(n) + slots - 1) / slots;
    pairs_per_chunk[chunk ? b / chunk : 0] += cnt;
  });
  double tot = 0.0;
  for (double v : pairs_per_chunk) tot += v;
  return tot;
}

struct Measure {
  Vec pts, w, logw;
  int64_t n = 0;
};

// The four potentials of SPEC.md:137-140.
struct Duals {
  Vec a_xx, b_yy, a_xy, b_yx;
};

// One symmetric update: all four softmins read the old
// values; averaged (lines 8-9) unless `assign` (the final update of
// SPEC.md:177, :224).
double sym_update(const Measure& X, const Measure& Y, int d, Duals& u, double eps, double lam,
                  double p, bool assign, const Ranges* rxx, const Ranges* ryy,
                  const Ranges* rxy /* rows y, cols x */, const Ranges* ryx /* rows x, cols y */) {
  Vec t_xx(X.n), t_yy(Y.n), t_xy(Y.n), t_yx(X.n);
  double pairs = 0.0;
  pairs += softmin_rows(X.pts.data(), X.n, d, {X.pts.data(), X.logw.data(), u.a_xx.data(), X.n},
                        eps, lam, p, rxx, t_xx.data());
  pairs += softmin_rows(Y.pts.data(), Y.n, d, {Y.pts.data(), Y.logw.data(), u.b_yy.data(), Y.n},
                        eps, lam, p, ryy, t_yy.data());
  pairs += softmin_rows(Y.pts.data(), Y.n, d, {X.pts.data(), X.logw.data(), u.b_yx.data(), X.n},
                        eps, lam, p, rxy, t_xy.data());
  pairs += softmin_rows(X.pts.data(), X.n, d, {Y.pts.data(), Y.logw.data(), u.a_xy.data(), Y.n},
                        eps, lam, p, ryx, t_yx.data());
  auto mix = [&](Vec& a, const Vec& t) {
    for (std::size_t i = 0; i < a.size(); ++i) a[i] = assign ? t[i] : 0.5 * (a[i] + t[i]);
  };
  mix(u.a_xx, t_xx);
  mix(u.b_yy, t_yy);
  mix(u.a_xy, t_xy);
  mix(u.b_yx, t_yx);
  for (const Vec* v : {&u.a_xx, &u.b_yy, &u.a_xy, &u.b_yx})
    for (double q : *v)
      if (!std::isfinite(q)) return -1.0;
  return pairs;
}

// Clustering result in sorted order.
struct Clusters {
  std::vector<int32_t> perm, labels, offsets;
  int32_t k = 0;
  Vec centroids, cweights;
  std::vector<float> radii;
  std::vector<float> box;  // per cluster {lo[3], hi[3]}: members' offsets from the float centroid
};

float round_up_float(double v) {
  float f = static_cast<float>(v);
  if (static_cast<double>(f) < v) f = std::nextafter(f, std::numeric_limits<float>::infinity());
  return f;
}

// Voxel-grid clustering (north star; stands in for kmeans_coarsen,
// SPEC.md:260-268; ClusterTree fields SPEC.md:249-252).
Clusters grid_cluster(const double* x, const double* w, int64_t n, int d, const double* origin,
                      double cell) {
  Clusters c;
  std::vector<uint32_t> key(n);
  for (int64_t i = 0; i < n; ++i) key[i] = msot_cube_key(x + i * d, d, origin, cell);
  c.perm.resize(n);
  std::iota(c.perm.begin(), c.perm.end(), 0);
  std::stable_sort(c.perm.begin(), c.perm.end(),
                   [&](int32_t a, int32_t b) { return key[a] < key[b]; });
  c.labels.resize(n);
  c.offsets.clear();
  for (int64_t s = 0; s < n; ++s) {
    if (s == 0 || key[c.perm[s]] != key[c.perm[s - 1]]) c.offsets.push_back(static_cast<int32_t>(s));
    c.labels[s] = static_cast<int32_t>(c.offsets.size()) - 1;
  }
  c.k = static_cast<int32_t>(c.offsets.size());
  c.offsets.push_back(static_cast<int32_t>(n));
  c.centroids.assign(static_cast<std::size_t>(c.k) * d, 0.0);
  c.cweights.assign(c.k, 0.0);
  c.radii.assign(c.k, 0.0f);
  for (int32_t I = 0; I < c.k; ++I) {
    double W = 0.0;
    std::vector<double> acc(d, 0.0);
    for (int32_t s = c.offsets[I]; s < c.offsets[I + 1]; ++s) {
      const int32_t i = c.perm[s];
      W += w[i];
      for (int k = 0; k < d; ++k) acc[k] += w[i] * x[int64_t(i) * d + k];
    }
    c.cweights[I] = W;
    for (int k = 0; k < d; ++k) c.centroids[int64_t(I) * d + k] = acc[k] / W;
    double r = 0.0;
    for (int32_t s = c.offsets[I]; s < c.offsets[I + 1]; ++s) {
      const int32_t i = c.perm[s];
      double q = 0.0;
      for (int k = 0; k < d; ++k) {
        const double t = x[int64_t(i) * d + k] - c.centroids[int64_t(I) * d + k];
        q += t * t;
      }
      r = std::max(r, std::sqrt(q));
    }
    c.radii[I] = round_up_float(r);
  }
  return c;
}

float round_down_float(double v) { return -round_up_float(-v); }

// Member boxes for the truncation box bound: per axis the min / max of the
// members' float coordinates minus the float centroid (exact in double),
// rounded outward — what cluster_stats does with the same float inputs.
void cluster_boxes(const double* x, int d, Clusters& c) {
  c.box.assign(size_t(c.k) * 6, 0.0f);
  for (int32_t I = 0; I < c.k; ++I) {
    double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int32_t s = c.offsets[I]; s < c.offsets[I + 1]; ++s) {
      const int32_t i = c.perm[s];
      for (int k = 0; k < d; ++k) {
        const double t = static_cast<double>(static_cast<float>(x[int64_t(i) * d + k])) -
                         static_cast<double>(static_cast<float>(c.centroids[int64_t(I) * d + k]));
        lo[k] = std::min(lo[k], t);
        hi[k] = std::max(hi[k], t);
      }
    }
    for (int k = 0; k < 3; ++k) {
      c.box[size_t(I) * 6 + k] = round_down_float(lo[k]);
      c.box[size_t(I) * 6 + 3 + k] = round_up_float(hi[k]);
    }
  }
}

// Slack upper bound of a cluster pair (SURVEY.md §0.1 #3 — the per-pair
// distance bound replacing SPEC.md:283's d^{p-1} margin):
//   F_I + G_J - (1/p) max(0, |X_I - Y_J| - r_I - r_J)^p
// in float64 with every operation explicitly ordered (no contraction).
// max over a in [l1, h1], b in [l2, h2] of u a + v b - (a - b)^2 / 2 (the
// box bound of mask.cu: box_quad, same operations in the same order)
inline double quad_edge(double u, double v, double A, double B) {
  const double c = A - B;
  return (u * A + v * B) - 0.5 * (c * c);
}
inline double box_quad(double u, double v, double l1, double h1, double l2, double h2) {
  // u a + v b - (a - b)^2/2 grows along a = b with slope (u + v)/2, so for
  // u + v >= 0 its maximum over the rectangle has a = h1 or b = h2 (else
  // a = l1 or b = l2), the other variable at its clamped stationary point
  const bool up = u + v >= 0.0;
  const double A = up ? h1 : l1, B = up ? h2 : l2;
  const double ca = quad_edge(u, v, A, std::fmin(std::fmax(A + v, l2), h2));
  const double cb = quad_edge(u, v, std::fmin(std::fmax(B + u, l1), h1), B);
  return std::fmax(ca, cb);
}

// BI / BJ (nullable, only with GI / HJ): member box {lo[3], hi[3]} of the
// cluster's offsets from its centroid, adding the box bound
//   B_c = F'_I + G'_J - |D|^2/2 + sum_k max_{a, b in the boxes}
//         [(G_I - D)_k a + (H_J + D)_k b - (a - b)^2 / 2]
// (mask.cu header: it keeps the -|u - v|^2/2 term the slope bound drops)
inline double pair_slack(const float* X, float rI, float F, const float* GI, const float* Y,
                         float rJ, float G, const float* HJ, int d, double p,
                         const float* BI = nullptr, const float* BJ = nullptr) {
  double dd[3] = {0.0, 0.0, 0.0};
  for (int k = 0; k < d; ++k) dd[k] = static_cast<double>(X[k]) - static_cast<double>(Y[k]);
  const double s = (dd[0] * dd[0] + dd[1] * dd[1]) + dd[2] * dd[2];
  // (a) centroid/radius bound
  const double rr = static_cast<double>(rI) + static_cast<double>(rJ);  // symmetric in (I,J)
  double lb = std::sqrt(s) - rr;
  if (lb < 0.0) lb = 0.0;
  double c;
  if (p == 2.0) {
    const double l2 = lb * lb;
    c = 0.5 * l2;
  } else {
    c = std::pow(lb, p) / p;
  }
  const double fg = static_cast<double>(F) + static_cast<double>(G);
  const double va = fg - c;
  if (!GI || p != 2.0) return va;
  // (b) slope bound F'_I + G'_J + r_I |G_I - D| + r_J |H_J + D| - |D|^2/2
  // (mask.cu header); GI/HJ = {slope[3], F'}
  double a[3], b[3];
  for (int k = 0; k < 3; ++k) {
    a[k] = static_cast<double>(GI[k]) - dd[k];
    b[k] = static_cast<double>(HJ[k]) + dd[k];
  }
  const double na = std::sqrt((a[0] * a[0] + a[1] * a[1]) + a[2] * a[2]);
  const double nb = std::sqrt((b[0] * b[0] + b[1] * b[1]) + b[2] * b[2]);
  const double marg = static_cast<double>(rI) * na + static_cast<double>(rJ) * nb;
  const double fgp = static_cast<double>(GI[3]) + static_cast<double>(HJ[3]);
  const double vb = (fgp + marg) - 0.5 * s;
  const double v = va < vb ? va : vb;
  if (!BI) return v;
  double q = box_quad(a[0], b[0], BI[0], BI[3], BJ[0], BJ[3]);
  if (d > 1) q = q + box_quad(a[1], b[1], BI[1], BI[4], BJ[1], BJ[4]);
  if (d > 2) q = q + box_quad(a[2], b[2], BI[2], BI[5], BJ[2], BJ[5]);
  const double vc = (fgp + q) - 0.5 * s;
  return v < vc ? v : vc;
}

// gx / hy: nullable Kx x 4 / Ky x 4 {slope, F'} per cluster (both or neither)
void truncation_mask(int64_t kx, int64_t ky, int d, const float* cx, const float* rx,
                     const float* fx, const float* gx, const float* cy, const float* ry,
                     const float* gy, const float* hy, double eps, double theta, double p,
                     int self, uint8_t* mask, const float* bx = nullptr,
                     const float* by = nullptr) {
  const double thr = -(theta * eps);
  std::vector<double> rbest(kx, -std::numeric_limits<double>::infinity());
  std::vector<int64_t> rarg(kx, 0);
  std::vector<double> cbest(ky, -std::numeric_limits<double>::infinity());
  std::vector<int64_t> carg(ky, 0);
  const bool g = gx && hy;
  for (int64_t I = 0; I < kx; ++I) {
    for (int64_t J = 0; J < ky; ++J) {
      const double v = pair_slack(cx + I * d, rx[I], fx[I], g ? gx + 4 * I : nullptr, cy + J * d,
                                  ry[J], gy[J], g ? hy + 4 * J : nullptr, d, p,
                                  g && bx ? bx + 6 * I : nullptr, g && bx ? by + 6 * J : nullptr);
      mask[I * ky + J] = (v >= thr) ? 1 : 0;
      if (v > rbest[I]) { rbest[I] = v; rarg[I] = J; }
      if (v > cbest[J]) { cbest[J] = v; carg[J] = I; }
    }
  }
  // Best-pair guarantee: no row or column is empty.
  for (int64_t I = 0; I < kx; ++I) mask[I * ky + rarg[I]] = 1;
  for (int64_t J = 0; J < ky; ++J) mask[carg[J] * ky + J] = 1;
  if (self)
    for (int64_t I = 0; I < std::min(kx, ky); ++I) mask[I * ky + I] = 1;
}

// Slope-bound inputs of one potential over one clustering (csrc/cluster.cu
// cluster_bound): weighted least-squares slope G of f in u = x - X_I (float),
// F' = max (f_i - <G, u_i>) rounded up, centroids as float (mask inputs).
void cluster_bound(const Vec& f, const Measure& M, const Clusters& c,
                   const std::vector<float>& cenf, int d, std::vector<float>& fmax,
                   std::vector<float>& grad) {
  fmax.assign(c.k, 0.0f);
  grad.assign(4 * size_t(c.k), 0.0f);
  for (int32_t I = 0; I < c.k; ++I) {
    double m[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}}, b[3] = {0, 0, 0}, mu[3] = {0, 0, 0};
    double W = 0.0, wf = 0.0;
    for (int32_t s = c.offsets[I]; s < c.offsets[I + 1]; ++s) {
      double u[3] = {0, 0, 0};
      for (int k = 0; k < d; ++k)
        u[k] = static_cast<double>(static_cast<float>(M.pts[int64_t(s) * d + k])) - cenf[size_t(I) * d + k];
      const double w = M.w[s];
      for (int a = 0; a < 3; ++a) {
        for (int q = 0; q < 3; ++q) m[a][q] += w * u[a] * u[q];
        b[a] += w * u[a] * f[s];
        mu[a] += w * u[a];
      }
      W += w;
      wf += w * f[s];
    }
    const double fbar = wf / W;
    for (int a = 0; a < 3; ++a) b[a] -= fbar * mu[a];
    const double tr = m[0][0] + m[1][1] + m[2][2], reg = 1e-9 * tr + 1e-300;
    for (int a = 0; a < 3; ++a) m[a][a] += reg;
    const double c00 = m[1][1] * m[2][2] - m[1][2] * m[1][2], c01 = m[0][2] * m[1][2] - m[0][1] * m[2][2],
                 c02 = m[0][1] * m[1][2] - m[0][2] * m[1][1];
    const double det = m[0][0] * c00 + m[0][1] * c01 + m[0][2] * c02;
    double gg[3] = {0, 0, 0};
    if (det > 0.0 && std::isfinite(det)) {
      const double c11 = m[0][0] * m[2][2] - m[0][2] * m[0][2], c12 = m[0][1] * m[0][2] - m[0][0] * m[1][2],
                   c22 = m[0][0] * m[1][1] - m[0][1] * m[0][1];
      gg[0] = (c00 * b[0] + c01 * b[1] + c02 * b[2]) / det;
      gg[1] = (c01 * b[0] + c11 * b[1] + c12 * b[2]) / det;
      gg[2] = (c02 * b[0] + c12 * b[1] + c22 * b[2]) / det;
    }
    float G[3];
    for (int a = 0; a < 3; ++a) G[a] = static_cast<float>(gg[a]);
    double fm = -std::numeric_limits<double>::infinity(), fp = fm;
    for (int32_t s = c.offsets[I]; s < c.offsets[I + 1]; ++s) {
      double lin = 0.0;
      for (int k = 0; k < d; ++k)
        lin += static_cast<double>(G[k]) *
               (static_cast<double>(static_cast<float>(M.pts[int64_t(s) * d + k])) - cenf[size_t(I) * d + k]);
      fm = std::max(fm, f[s]);
      fp = std::max(fp, f[s] - lin);
    }
    fmax[I] = round_up_float(fm);
    for (int a = 0; a < 3; ++a) grad[4 * size_t(I) + a] = G[a];
    grad[4 * size_t(I) + 3] = round_up_float(fp);
  }
}

// High-D truncation mask (csrc/mask.cu: mask_hd_rows_kernel): B_a with
// float64 centroids, |X - Y|^2 summed in coordinate order, best pairs (ties to
// the lowest index) of every row and column, the diagonal of self masks.
double hd_pair_slack(const double* X, float rI, float F, const double* Y, float rJ, float G, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = X[k] - Y[k];
    s = s + t * t;
  }
  const double rr = static_cast<double>(rI) + static_cast<double>(rJ);
  double lb = std::sqrt(s) - rr;
  if (lb < 0.0) lb = 0.0;
  const double fg = static_cast<double>(F) + static_cast<double>(G);
  return fg - 0.5 * (lb * lb);
}

void hd_mask(int64_t kx, int64_t ky, int d, const double* cx, const float* rx, const float* fx,
             const double* cy, const float* ry, const float* gy, double eps, double theta,
             int self, std::vector<uint8_t>& mask) {
  const double thr = -(theta * eps);
  mask.assign(size_t(kx) * ky, 0);
  std::vector<double> v(size_t(kx) * ky);
  for (int64_t I = 0; I < kx; ++I)
    for (int64_t J = 0; J < ky; ++J) {
      v[I * ky + J] = hd_pair_slack(cx + I * d, rx[I], fx[I], cy + J * d, ry[J], gy[J], d);
      mask[I * ky + J] = (self && I == J) || v[I * ky + J] >= thr;
    }
  for (int64_t I = 0; I < kx; ++I) {
    int64_t bj = -1;
    for (int64_t J = 0; J < ky; ++J)
      if (bj < 0 || v[I * ky + J] > v[I * ky + bj]) bj = J;
    if (bj >= 0 && v[I * ky + bj] > -std::numeric_limits<double>::infinity()) mask[I * ky + bj] = 1;
  }
  for (int64_t J = 0; J < ky; ++J) {
    int64_t bi = -1;
    for (int64_t I = 0; I < kx; ++I)
      if (bi < 0 || v[I * ky + J] > v[bi * ky + J]) bi = I;
    if (bi >= 0 && v[bi * ky + J] > -std::numeric_limits<double>::infinity()) mask[bi * ky + J] = 1;
  }
}

// Column ranges of every cluster-aligned row tile: the union of the kept
// column clusters of the row clusters the tile covers, as runs of sorted
// column indices [co[J0], co[J1+1]).
int64_t tile_ranges(const int32_t* rl, const int32_t* ro, int64_t kx, int64_t n,
                    const int32_t* co, int64_t ky, const uint8_t* mask, Ranges& out) {
  out.tile_start.assign(kx + n / MSOT_TILE_ROWS + 2, 0);
  const int64_t nt = msot_row_tiles(ro, kx, n, MSOT_TILE_ROWS, out.tile_start.data());
  out.tile_start.resize(nt + 1);
  out.row_tile.resize(n);
  for (int64_t t = 0; t < nt; ++t)
    for (int64_t i = out.tile_start[t]; i < out.tile_start[t + 1]; ++i) out.row_tile[i] = int32_t(t);
  out.tile_ptr.assign(nt + 1, 0);
  out.r.clear();
  std::vector<uint8_t> keep(ky);
  for (int64_t t = 0; t < nt; ++t) {
    const int32_t Ilo = rl[out.tile_start[t]];
    const int32_t Ihi = rl[out.tile_start[t + 1] - 1];
    std::fill(keep.begin(), keep.end(), 0);
    for (int32_t I = Ilo; I <= Ihi; ++I)
      for (int64_t J = 0; J < ky; ++J) keep[J] |= mask[I * ky + J];
    int64_t J = 0;
    while (J < ky) {
      if (!keep[J]) { ++J; continue; }
      int64_t J1 = J;
      while (J1 + 1 < ky && keep[J1 + 1]) ++J1;
      out.r.push_back(co[J]);
      out.r.push_back(co[J1 + 1]);
      J = J1 + 1;
    }
    out.tile_ptr[t + 1] = static_cast<int64_t>(out.r.size() / 2);
  }
  return out.tile_ptr[nt];
}

// Per-row ranges (every row its own "tile") from per-row interval lists.
Ranges per_row(std::vector<std::vector<std::pair<int32_t, int32_t>>>& L) {
  Ranges out;
  const int64_t n = static_cast<int64_t>(L.size());
  out.tile_start.resize(n + 1);
  out.row_tile.resize(n);
  out.tile_ptr.assign(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) {
    out.tile_start[i] = i;
    out.row_tile[i] = static_cast<int32_t>(i);
    std::sort(L[i].begin(), L[i].end());
    for (const auto& r : L[i]) {
      out.r.push_back(r.first);
      out.r.push_back(r.second);
    }
    out.tile_ptr[i + 1] = static_cast<int64_t>(out.r.size() / 2);
  }
  out.tile_start[n] = n;
  return out;
}

// The pair sets of the symmetric evaluation (csrc/softmin.cu):
// every kept pair is evaluated once and feeds both its row and its column.
// Self problem with tile ranges R (rows = cols): row i of tile t sums over
//   its own tile's rows [ts, te)                     (diagonal block)
//   R(t) clipped to columns >= te                    (upper part, row side)
//   the rows of every tile t' < t with i in R(t')    (column side)
// which is a symmetric relation containing the cluster mask.
Ranges sym_self(const Ranges& R, int64_t n) {
  std::vector<std::vector<std::pair<int32_t, int32_t>>> L(n);
  const int64_t T = static_cast<int64_t>(R.tile_start.size()) - 1;
  for (int64_t t = 0; t < T; ++t) {
    const int32_t ts = static_cast<int32_t>(R.tile_start[t]), te = static_cast<int32_t>(R.tile_start[t + 1]);
    for (int32_t i = ts; i < te; ++i) L[i].push_back({ts, te});
    for (int64_t q = R.tile_ptr[t]; q < R.tile_ptr[t + 1]; ++q) {
      const int32_t c0 = std::max(R.r[2 * q], te), c1 = R.r[2 * q + 1];
      if (c0 >= c1) continue;
      for (int32_t i = ts; i < te; ++i) L[i].push_back({c0, c1});
      for (int32_t k = c0; k < c1; ++k) L[k].push_back({ts, te});
    }
  }
  return per_row(L);
}

// Cross problem: tile ranges R of rows x over columns y; the y rows sum over
// the transposed relation {i : j in R(tile(i))}.
Ranges transpose_ranges(const Ranges& R, int64_t n_cols) {
  std::vector<std::vector<std::pair<int32_t, int32_t>>> L(n_cols);
  const int64_t T = static_cast<int64_t>(R.tile_start.size()) - 1;
  for (int64_t t = 0; t < T; ++t) {
    const int32_t ts = static_cast<int32_t>(R.tile_start[t]), te = static_cast<int32_t>(R.tile_start[t + 1]);
    for (int64_t q = R.tile_ptr[t]; q < R.tile_ptr[t + 1]; ++q)
      for (int32_t j = R.r[2 * q]; j < R.r[2 * q + 1]; ++j) L[j].push_back({ts, te});
  }
  return per_row(L);
}

double dot(const Vec& a, const Vec& b) { return msot::pairwise_dot(a, b); }

// S_eps,rho from the four potentials: balanced limit or the
// dual form Eq. 6, plus (eps/2)(sum a - sum b)^2 (Eq. 5).
double divergence(const msot_params* prm, double eps, const Vec& a, const Vec& b, const Duals& u) {
  const double ma = msot::kahan_sum(a), mb = msot::kahan_sum(b);
  double s;
  if (msot_reach_is_inf(prm->reach)) {
    Vec dx(a.size()), dy(b.size());
    for (std::size_t i = 0; i < a.size(); ++i) dx[i] = u.b_yx[i] - u.a_xx[i];
    for (std::size_t j = 0; j < b.size(); ++j) dy[j] = u.a_xy[j] - u.b_yy[j];
    s = dot(a, dx) + dot(b, dy);
  } else {
    const double rho = std::pow(prm->reach, prm->p);
    Vec dx(a.size()), dy(b.size());
    for (std::size_t i = 0; i < a.size(); ++i)
      dx[i] = std::exp(-u.b_yx[i] / rho) - std::exp(-u.a_xx[i] / rho);
    for (std::size_t j = 0; j < b.size(); ++j)
      dy[j] = std::exp(-u.a_xy[j] / rho) - std::exp(-u.b_yy[j] / rho);
    s = -(rho + 0.5 * eps) * (dot(a, dx) + dot(b, dy));
  }
  return s + 0.5 * eps * (ma - mb) * (ma - mb);
}

Measure make_measure(const double* x, const double* w, int64_t n, int d) {
  Measure m;
  m.n = n;
  m.pts.assign(x, x + n * d);
  m.w.assign(w, w + n);
  m.logw.resize(n);
  for (int64_t i = 0; i < n; ++i) m.logw[i] = std::log(w[i]);
  return m;
}

Measure permute(const Measure& m, const std::vector<int32_t>& perm, int d) {
  Measure o;
  o.n = m.n;
  o.pts.resize(m.pts.size());
  o.w.resize(m.n);
  o.logw.resize(m.n);
  for (int64_t s = 0; s < m.n; ++s) {
    const int32_t i = perm[s];
    for (int k = 0; k < d; ++k) o.pts[s * d + k] = m.pts[int64_t(i) * d + k];
    o.w[s] = m.w[i];
    o.logw[s] = m.logw[i];
  }
  return o;
}


}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

void oracle_set_threads(int n) { msot::parallel::set_threads(n); }
int oracle_threads(void) { return msot::parallel::threads(); }

int oracle_schedule(double diameter, const msot_params* p, double* sigma, double* eps,
                    double* lam, int cap) {
  const int n = msot_schedule_len(diameter, p->blur, p->scaling);
  if (n > cap) return -n;
  for (int t = 0; t < n; ++t) {
    sigma[t] = msot_schedule_sigma(diameter, p->blur, p->scaling, n, t);
    eps[t] = std::pow(sigma[t], p->p);
    lam[t] = msot_lambda(eps[t], p);
  }
  return n;
}

void oracle_softmin(const double* x, int64_t n, const double* y, int64_t m, int d,
                    const double* logw_y, const double* h, double eps, double lambda, double p,
                    double* f_out) {
  softmin_rows(x, n, d, {y, logw_y, h, m}, eps, lambda, p, nullptr, f_out);
}

// kmeans_coarsen: farthest-point seeding from atom
// (seed mod N), Lloyd iterations with mass-weighted centroids until the
// largest centre move is < 1e-9 d or 100 iterations.  Distances sum
// (x_k - c_k)^2 in coordinate order, centroid sums run over each cluster's
// atoms in index order (the CUDA kernels' exact order, kmeans.cu).
struct KMeans {
  std::vector<int32_t> perm, offsets, labels;
  Vec centroids, cweights;
  std::vector<float> radii;
  int iters = 0;
};

double km_dist2(const double* x, const double* c, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double t = x[k] - c[k];
    s = s + t * t;
  }
  return s;
}

KMeans kmeans(const double* x, const double* w, int64_t n, int d, int K, uint64_t seed,
              int max_iter = 100) {
  KMeans r;
  Vec c(static_cast<std::size_t>(K) * d), mind(n);
  const int64_t s0 = static_cast<int64_t>(seed % static_cast<uint64_t>(n));
  std::copy(x + s0 * d, x + (s0 + 1) * d, c.begin());
  for (int k = 1; k < K; ++k) {
    double best = -1.0;
    int64_t bi = 0;
    for (int64_t i = 0; i < n; ++i) {
      const double dd = km_dist2(x + i * d, c.data() + static_cast<int64_t>(k - 1) * d, d);
      mind[i] = k == 1 ? dd : std::min(mind[i], dd);
      if (mind[i] > best) {  // strict: ties keep the lowest index
        best = mind[i];
        bi = i;
      }
    }
    std::copy(x + bi * d, x + (bi + 1) * d, c.begin() + static_cast<int64_t>(k) * d);
  }
  double diag2 = 0.0;
  for (int q = 0; q < d; ++q) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = 0; i < n; ++i) lo = std::min(lo, x[i * d + q]), hi = std::max(hi, x[i * d + q]);
    diag2 += (hi - lo) * (hi - lo);
  }
  const double tol = 1e-9 * std::sqrt(diag2), tol2 = tol * tol;
  r.labels.assign(n, 0);
  r.cweights.assign(K, 0.0);
  Vec c2(c.size());
  for (;;) {
    msot::parallel::for_ranges(static_cast<std::size_t>(n), [&](std::size_t lo, std::size_t hi) {
      for (std::size_t i = lo; i < hi; ++i) {
        double best = INFINITY;
        int bl = 0;
        for (int I = 0; I < K; ++I) {
          const double dd = km_dist2(x + i * d, c.data() + static_cast<int64_t>(I) * d, d);
          if (dd < best) {
            best = dd;
            bl = I;
          }
        }
        r.labels[i] = bl;
      }
    });
    r.perm.resize(n);
    std::iota(r.perm.begin(), r.perm.end(), 0);
    std::stable_sort(r.perm.begin(), r.perm.end(),
                     [&](int32_t p, int32_t q) { return r.labels[p] < r.labels[q]; });
    r.offsets.assign(K + 1, 0);
    for (int64_t i = 0; i < n; ++i) ++r.offsets[r.labels[i] + 1];
    for (int I = 0; I < K; ++I) r.offsets[I + 1] += r.offsets[I];
    ++r.iters;
    double move = 0.0;
    for (int I = 0; I < K; ++I) {
      const int32_t a = r.offsets[I], b = r.offsets[I + 1];
      for (int q = 0; q < d; ++q) {
        const int64_t g = static_cast<int64_t>(I) * d + q;
        if (b <= a) {
          c2[g] = c[g];
          continue;
        }
        double W = 0.0, S = 0.0;
        for (int32_t s = a; s < b; ++s) {
          const int64_t i = r.perm[s];
          W = W + w[i];
          S = S + w[i] * x[i * d + q];
        }
        c2[g] = S / W;
        if (q == 0) r.cweights[I] = W;
      }
      if (b <= a) r.cweights[I] = 0.0;
      move = std::max(move, km_dist2(c.data() + static_cast<int64_t>(I) * d,
                                     c2.data() + static_cast<int64_t>(I) * d, d));
    }
    c = c2;
    if (move < tol2 || r.iters >= max_iter) break;
  }
  r.centroids = c;
  r.radii.assign(K, 0.0f);
  for (int I = 0; I < K; ++I) {
    double m = 0.0;
    for (int32_t s = r.offsets[I]; s < r.offsets[I + 1]; ++s)
      m = std::max(m, km_dist2(x + static_cast<int64_t>(r.perm[s]) * d, c.data() + static_cast<int64_t>(I) * d, d));
    // sqrt and float conversion rounded up, as __dsqrt_ru / __double2float_ru
    double rr = std::sqrt(m);
    if (std::fma(rr, rr, -m) < 0.0) rr = std::nextafter(rr, INFINITY);  // exact rr^2 < m
    r.radii[I] = round_up_float(rr);
  }
  return r;
}

int oracle_kmeans(const double* x, const double* w, int64_t n, int d, int k, uint64_t seed,
                  int32_t* perm, int32_t* offsets, int32_t* labels, double* centroids,
                  double* cweights, float* radii, int* iters) {
  if (k < 1 || k > n) return fail(MSOT_EDATA, "K must lie in [1, N]");
  KMeans r = kmeans(x, w, n, d, k, seed);
  std::copy(r.perm.begin(), r.perm.end(), perm);
  std::copy(r.offsets.begin(), r.offsets.end(), offsets);
  std::copy(r.labels.begin(), r.labels.end(), labels);
  std::copy(r.centroids.begin(), r.centroids.end(), centroids);
  std::copy(r.cweights.begin(), r.cweights.end(), cweights);
  std::copy(r.radii.begin(), r.radii.end(), radii);
  if (iters) *iters = r.iters;
  return MSOT_OK;
}

int oracle_grid_cluster(const double* x, const double* w, int64_t n, int d, const double* origin,
                        double cell, int32_t* perm, int32_t* labels, int32_t* offsets,
                        int32_t* k_out, double* centroids, double* cweights, float* radii) {
  if (d < 1 || d > 3) return fail(MSOT_EUSAGE, "grid clustering supports D in 1..3");
  Clusters c = grid_cluster(x, w, n, d, origin, cell);
  std::copy(c.perm.begin(), c.perm.end(), perm);
  std::copy(c.labels.begin(), c.labels.end(), labels);
  std::copy(c.offsets.begin(), c.offsets.end(), offsets);
  *k_out = c.k;
  std::copy(c.centroids.begin(), c.centroids.end(), centroids);
  std::copy(c.cweights.begin(), c.cweights.end(), cweights);
  std::copy(c.radii.begin(), c.radii.end(), radii);
  return MSOT_OK;
}

void oracle_truncation_mask(int64_t kx, int64_t ky, int d, const float* cx, const float* rx,
                            const float* fx, const float* gx, const float* cy, const float* ry,
                            const float* gy, const float* hy, double eps, double theta, double p,
                            int self, uint8_t* mask_out) {
  truncation_mask(kx, ky, d, cx, rx, fx, gx, cy, ry, gy, hy, eps, theta, p, self, mask_out);
}

void oracle_truncation_mask_box(int64_t kx, int64_t ky, int d, const float* cx, const float* rx,
                                const float* fx, const float* gx, const float* bx, const float* cy,
                                const float* ry, const float* gy, const float* hy, const float* by,
                                double eps, double theta, double p, int self, uint8_t* mask_out) {
  truncation_mask(kx, ky, d, cx, rx, fx, gx, cy, ry, gy, hy, eps, theta, p, self, mask_out, bx, by);
}

int64_t oracle_tile_ranges(const int32_t* row_labels, const int32_t* row_offsets,
                           int64_t n_rows, int64_t kx, const int32_t* col_offsets, int64_t ky,
                           const uint8_t* mask, int64_t* n_tiles, int64_t* tile_start,
                           int64_t* tile_ptr, int32_t* ranges, int64_t cap) {
  Ranges r;
  const int64_t nr = tile_ranges(row_labels, row_offsets, kx, n_rows, col_offsets, ky, mask, r);
  const int64_t nt = static_cast<int64_t>(r.tile_start.size()) - 1;
  if (n_tiles) *n_tiles = nt;
  if (tile_start) std::copy(r.tile_start.begin(), r.tile_start.end(), tile_start);
  if (tile_ptr) std::copy(r.tile_ptr.begin(), r.tile_ptr.end(), tile_ptr);
  if (ranges && cap >= nr) std::copy(r.r.begin(), r.r.end(), ranges);
  return nr;
}

double oracle_divergence_from_potentials(const msot_params* prm, double eps, const double* a,
                                         int64_t n, const double* b, int64_t m,
                                         const double* a_xx, const double* b_yy,
                                         const double* a_xy, const double* b_yx) {
  Duals u{Vec(a_xx, a_xx + n), Vec(b_yy, b_yy + m), Vec(a_xy, a_xy + m), Vec(b_yx, b_yx + n)};
  return divergence(prm, eps, Vec(a, a + n), Vec(b, b + m), u);
}

// The full solve: symmetric_sinkhorn or
// multiscale_sinkhorn then divergence.
// Schedule diameter override (> 0), set by oracle_barycenter for its shared
// schedule (mirrors msot_ctx::diam_override).
static double g_diam_override = 0.0;

int oracle_sinkhorn(const msot_params* prm, const double* x, const double* a, int64_t n,
                    const double* y, const double* b, int64_t m, int d, double* a_xx,
                    double* b_yy, double* a_xy, double* b_yx, double* loss_out,
                    msot_stats* st) {
  if (n < 1 || m < 1 || d < 1) return fail(MSOT_EDATA, "empty measure");
  if (!(prm->blur > 0) || !(prm->scaling > 0 && prm->scaling < 1) || !(prm->p >= 1 && prm->p <= 2) ||
      !msot_reach_valid(prm->reach))
    return fail(MSOT_EUSAGE, "invalid solver parameters");
  for (int64_t i = 0; i < n; ++i)
    if (!(a[i] > 0)) return fail(MSOT_EDATA, "weights must be > 0");
  for (int64_t j = 0; j < m; ++j)
    if (!(b[j] > 0)) return fail(MSOT_EDATA, "weights must be > 0");
  msot_stats local{};
  msot_stats& S = st ? *st : local;
  std::memset(&S, 0, sizeof(S));
  S.world = 1;

  // diameter_estimate: joint bounding-box diagonal, >= blur.
  std::vector<double> lo(d, std::numeric_limits<double>::infinity()), hi(d, -lo[0]);
  for (int64_t i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) lo[k] = std::min(lo[k], x[i * d + k]), hi[k] = std::max(hi[k], x[i * d + k]);
  for (int64_t j = 0; j < m; ++j)
    for (int k = 0; k < d; ++k) lo[k] = std::min(lo[k], y[j * d + k]), hi[k] = std::max(hi[k], y[j * d + k]);
  double diag2 = 0.0;
  for (int k = 0; k < d; ++k) diag2 += (hi[k] - lo[k]) * (hi[k] - lo[k]);
  const double diam = g_diam_override > 0 ? std::max(g_diam_override, prm->blur)
                                         : std::max(std::sqrt(diag2), prm->blur);
  S.diameter = diam;

  const int ns = msot_schedule_len(diam, prm->blur, prm->scaling);
  if (prm->max_full_iters > 0 && ns > prm->max_full_iters)
    return fail(MSOT_EUSAGE, "schedule longer than max_full_iters");
  Vec sig(ns), eps(ns), lam(ns);
  oracle_schedule(diam, prm, sig.data(), eps.data(), lam.data(), ns);
  S.n_scales = ns;
  const double p = prm->p;

  Measure X = make_measure(x, a, n, d), Y = make_measure(y, b, m, d);
  Duals u{Vec(n, 0.0), Vec(m, 0.0), Vec(m, 0.0), Vec(n, 0.0)};
  const double full = double(n) * n + double(m) * m + 2.0 * double(n) * m;

  std::vector<int32_t> px, py;
  if (prm->multiscale && d > 3) {
    // ---- high-D multiscale (csrc/solver.cu: hd_multiscale): K-means
    // coarsening, every cluster padded to a multiple of 128 atoms (centroid
    // coordinates, weight 0) exactly as the GPU layout, dense coarse phase,
    // inheritance, centroid/radius masks, evaluate-once pair sets.
    if (prm->pair_eval == 0) return fail(MSOT_EUSAGE, "high-D multiscale runs the evaluate-once scheme");
    struct Pad {
      int K = 0;
      int64_t npad = 0;
      std::vector<int32_t> poff, src, labels;
      KMeans km;
      Measure M;
    };
    auto layout = [&](const double* xx, const double* ww, int64_t cnt) {
      Pad P;
      P.K = prm->clusters > 0 ? static_cast<int>(std::min<int64_t>(prm->clusters, cnt))
                              : static_cast<int>(std::ceil(std::sqrt(static_cast<double>(cnt))));
      P.km = kmeans(xx, ww, cnt, d, P.K, static_cast<uint64_t>(prm->seed), MSOT_KMEANS_SOLVER_ITERS);
      P.poff.assign(P.K + 1, 0);
      for (int I = 0; I < P.K; ++I)
        P.poff[I + 1] = P.poff[I] + (P.km.offsets[I + 1] - P.km.offsets[I] + 127) / 128 * 128;
      P.npad = P.poff[P.K];
      P.src.assign(P.npad, 0);
      P.labels.assign(P.npad, 0);
      P.M.n = P.npad;
      P.M.pts.assign(P.npad * d, 0.0);
      P.M.w.assign(P.npad, 0.0);
      P.M.logw.assign(P.npad, -std::numeric_limits<double>::infinity());
      for (int I = 0; I < P.K; ++I) {
        const int32_t c0 = P.km.offsets[I], cn = P.km.offsets[I + 1] - c0;
        for (int32_t q = 0; q < P.poff[I + 1] - P.poff[I]; ++q) {
          const int64_t s = P.poff[I] + q;
          P.labels[s] = I;
          if (q < cn) {
            const int32_t i = P.km.perm[c0 + q];
            P.src[s] = i;
            std::copy(xx + int64_t(i) * d, xx + int64_t(i + 1) * d, P.M.pts.begin() + s * d);
            P.M.w[s] = ww[i];
            P.M.logw[s] = std::log(ww[i]);
          } else {
            P.src[s] = -(I + 1);
            std::copy(P.km.centroids.begin() + int64_t(I) * d,
                      P.km.centroids.begin() + int64_t(I + 1) * d, P.M.pts.begin() + s * d);
          }
        }
      }
      return P;
    };
    Pad PX = layout(x, a, n), PY = layout(y, b, m);
    S.kx = PX.K;
    S.ky = PY.K;
    double rmax = 0.0;
    for (float r : PX.km.radii) rmax = std::max(rmax, double(r));
    for (float r : PY.km.radii) rmax = std::max(rmax, double(r));
    const int tsw = msot_switch_index(sig.data(), ns, rmax, prm->switch_factor);
    S.t_switch = tsw;
    auto coarse_measure = [&](const Pad& P) {
      Measure C;
      C.n = P.K;
      C.pts = P.km.centroids;
      C.w = P.km.cweights;
      C.logw.resize(P.K);
      for (int I = 0; I < P.K; ++I) C.logw[I] = std::log(C.w[I]);
      return C;
    };
    Measure Xc = coarse_measure(PX), Yc = coarse_measure(PY);
    Duals cu{Vec(PX.K, 0.0), Vec(PY.K, 0.0), Vec(PY.K, 0.0), Vec(PX.K, 0.0)};
    for (int t = 0; t < tsw; ++t) {
      const double pr = sym_update(Xc, Yc, d, cu, eps[t], lam[t], p, false, nullptr, nullptr,
                                   nullptr, nullptr);
      if (pr < 0) return fail(MSOT_ENUMERIC, "non-finite potential at scale " + std::to_string(t));
      S.pairs_evaluated += pr;
    }
    Duals fu{Vec(PX.npad, 0.0), Vec(PY.npad, 0.0), Vec(PY.npad, 0.0), Vec(PX.npad, 0.0)};
    if (tsw > 0 && prm->transfer_rule == 1) {  // extrapolation (GeomLoss)
      const int te = tsw - 1;
      const double e = eps[te], l = lam[te];
      S.pairs_evaluated += softmin_rows(PX.M.pts.data(), PX.npad, d, {Xc.pts.data(), Xc.logw.data(), cu.a_xx.data(), PX.K}, e, l, p, nullptr, fu.a_xx.data());
      S.pairs_evaluated += softmin_rows(PY.M.pts.data(), PY.npad, d, {Yc.pts.data(), Yc.logw.data(), cu.b_yy.data(), PY.K}, e, l, p, nullptr, fu.b_yy.data());
      S.pairs_evaluated += softmin_rows(PY.M.pts.data(), PY.npad, d, {Xc.pts.data(), Xc.logw.data(), cu.b_yx.data(), PX.K}, e, l, p, nullptr, fu.a_xy.data());
      S.pairs_evaluated += softmin_rows(PX.M.pts.data(), PX.npad, d, {Yc.pts.data(), Yc.logw.data(), cu.a_xy.data(), PY.K}, e, l, p, nullptr, fu.b_yx.data());
    } else if (tsw > 0) {
      for (int64_t s2 = 0; s2 < PX.npad; ++s2) {
        fu.a_xx[s2] = cu.a_xx[PX.labels[s2]];
        fu.b_yx[s2] = cu.b_yx[PX.labels[s2]];
      }
      for (int64_t s2 = 0; s2 < PY.npad; ++s2) {
        fu.b_yy[s2] = cu.b_yy[PY.labels[s2]];
        fu.a_xy[s2] = cu.a_xy[PY.labels[s2]];
      }
    }
    // per-cluster max of a potential over the real atoms, as float
    auto fmaxv = [&](const Vec& f, const Pad& P) {
      std::vector<float> F(P.K, -std::numeric_limits<float>::infinity());
      for (int I = 0; I < P.K; ++I)
        for (int32_t s2 = P.poff[I]; s2 < P.poff[I + 1]; ++s2)
          if (P.M.w[s2] > 0.0) F[I] = std::max(F[I], static_cast<float>(f[s2]));
      return F;
    };
    Ranges rxx, ryy, rxy, ryx;
    auto build = [&](double e) {
      const double theta = tsw > 0 ? prm->theta : std::numeric_limits<double>::infinity();
      std::vector<float> Fxx = fmaxv(fu.a_xx, PX), Fyx = fmaxv(fu.b_yx, PX);
      std::vector<float> Gyy = fmaxv(fu.b_yy, PY), Gxy = fmaxv(fu.a_xy, PY);
      std::vector<uint8_t> mxx, myy, mxy;
      hd_mask(PX.K, PX.K, d, PX.km.centroids.data(), PX.km.radii.data(), Fxx.data(),
              PX.km.centroids.data(), PX.km.radii.data(), Fxx.data(), e, theta, 1, mxx);
      hd_mask(PY.K, PY.K, d, PY.km.centroids.data(), PY.km.radii.data(), Gyy.data(),
              PY.km.centroids.data(), PY.km.radii.data(), Gyy.data(), e, theta, 1, myy);
      hd_mask(PX.K, PY.K, d, PX.km.centroids.data(), PX.km.radii.data(), Fyx.data(),
              PY.km.centroids.data(), PY.km.radii.data(), Gxy.data(), e, theta, 0, mxy);
      tile_ranges(PX.labels.data(), PX.poff.data(), PX.K, PX.npad, PX.poff.data(), PX.K, mxx.data(), rxx);
      tile_ranges(PY.labels.data(), PY.poff.data(), PY.K, PY.npad, PY.poff.data(), PY.K, myy.data(), ryy);
      tile_ranges(PX.labels.data(), PX.poff.data(), PX.K, PX.npad, PY.poff.data(), PY.K, mxy.data(), ryx);
      rxx = sym_self(rxx, PX.npad);
      ryy = sym_self(ryy, PY.npad);
      rxy = transpose_ranges(ryx, PY.npad);
    };
    for (int t = tsw; t <= ns; ++t) {
      const int tt = std::min(t, ns - 1);
      const bool rebuild = (t == tsw) || (prm->retruncate > 0 && t < ns && (t - tsw) % prm->retruncate == 0);
      if (rebuild) build(eps[tt]);
      const double pr = sym_update(PX.M, PY.M, d, fu, eps[tt], lam[tt], p, t == ns, &rxx, &ryy, &rxy, &ryx);
      if (pr < 0) return fail(MSOT_ENUMERIC, "non-finite potential at scale " + std::to_string(tt));
      S.pairs_evaluated += pr;
      S.pairs_fine += pr;
    }
    auto unpad = [](const Vec& v, const Pad& P, int64_t cnt) {
      Vec o(cnt);
      for (int64_t s2 = 0; s2 < P.npad; ++s2)
        if (P.src[s2] >= 0) o[P.src[s2]] = v[s2];
      return o;
    };
    u.a_xx = unpad(fu.a_xx, PX, n);
    u.b_yx = unpad(fu.b_yx, PX, n);
    u.b_yy = unpad(fu.b_yy, PY, m);
    u.a_xy = unpad(fu.a_xy, PY, m);
  } else if (!prm->multiscale || d > 3) {
    S.t_switch = 0;
    for (int t = 0; t <= ns; ++t) {
      const int tt = std::min(t, ns - 1);
      const double pr = sym_update(X, Y, d, u, eps[tt], lam[tt], p, t == ns, nullptr, nullptr,
                                   nullptr, nullptr);
      if (pr < 0) return fail(MSOT_ENUMERIC, "non-finite potential at scale " + std::to_string(tt));
      S.pairs_evaluated += pr;
      S.pairs_dense += full;
    }
  } else {
    // ---- multiscale_sinkhorn with voxel-grid coarsening.
    double cell = prm->cluster_scale > 0 ? prm->cluster_scale
                                         : msot_auto_cell(lo.data(), hi.data(), d, n, m);
    if (prm->cluster_scale <= 0) {  // policy.h: refine on occupied voxels
      auto occupied = [&](const double* p, int64_t cnt) {
        std::vector<uint32_t> k(cnt);
        for (int64_t i = 0; i < cnt; ++i) k[i] = msot_cube_key(p + i * d, d, lo.data(), cell);
        std::sort(k.begin(), k.end());
        return static_cast<int64_t>(std::unique(k.begin(), k.end()) - k.begin());
      };
      for (int it = 0; it < MSOT_AUTO_REFINE; ++it) {
        const int64_t kk = std::max(occupied(x, n), occupied(y, m));
        cell = msot_refine_cell(cell, kk, n, m, d, lo.data(), hi.data());
      }
    }
    S.cluster_scale = cell;
    Clusters cx = grid_cluster(x, a, n, d, lo.data(), cell);
    Clusters cy = grid_cluster(y, b, m, d, lo.data(), cell);
    cluster_boxes(x, d, cx);
    cluster_boxes(y, d, cy);
    S.kx = cx.k;
    S.ky = cy.k;
    px = cx.perm;
    py = cy.perm;
    Measure Xs = permute(X, cx.perm, d), Ys = permute(Y, cy.perm, d);
    Measure Xc, Yc;  // coarse measures: centroids + cluster weights
    Xc.n = cx.k; Xc.pts = cx.centroids; Xc.w = cx.cweights;
    Yc.n = cy.k; Yc.pts = cy.centroids; Yc.w = cy.cweights;
    for (auto* M : {&Xc, &Yc}) {
      M->logw.resize(M->n);
      for (int64_t i = 0; i < M->n; ++i) M->logw[i] = std::log(M->w[i]);
    }
    double rmax = 0.0;
    for (float r : cx.radii) rmax = std::max(rmax, double(r));
    for (float r : cy.radii) rmax = std::max(rmax, double(r));
    const int tsw = msot_switch_index(sig.data(), ns, rmax, prm->switch_factor);
    S.t_switch = tsw;

    // Coarse phase on the centroid measures, preceded by the super level
    // (policy.h:msot_super_switch): consecutive clusters sharing a super-voxel
    // key, run for t < t2, their duals inherited by the clusters.
    Duals cu{Vec(cx.k, 0.0), Vec(cy.k, 0.0), Vec(cy.k, 0.0), Vec(cx.k, 0.0)};
    const int t2 = tsw > 0 ? msot_super_switch(sig.data(), tsw, cell, d, std::max(cx.k, cy.k),
                                               prm->super_level)
                           : 0;
    if (t2 > 0) {
      auto super = [&](const Clusters& cc, const Measure& Mc, const double* pts,
                       std::vector<int32_t>& lab) {
        Measure S2;
        lab.assign(cc.k, 0);
        std::vector<int32_t> off;
        uint32_t prev = 0;
        for (int32_t I = 0; I < cc.k; ++I) {
          const int64_t i = cc.perm[cc.offsets[I]];
          const uint32_t key = msot_cube_key(pts + i * d, d, lo.data(), cell) >> (d * MSOT_SUPER_SHIFT);
          if (I == 0 || key != prev) off.push_back(I);
          prev = key;
          lab[I] = static_cast<int32_t>(off.size()) - 1;
        }
        S2.n = static_cast<int64_t>(off.size());
        off.push_back(cc.k);
        S2.pts.assign(S2.n * d, 0.0);
        S2.w.assign(S2.n, 0.0);
        S2.logw.assign(S2.n, 0.0);
        for (int64_t J = 0; J < S2.n; ++J) {
          double W = 0.0;
          std::vector<double> acc(d, 0.0);
          for (int32_t I = off[J]; I < off[J + 1]; ++I) {
            W += Mc.w[I];
            for (int k = 0; k < d; ++k) acc[k] += Mc.w[I] * Mc.pts[int64_t(I) * d + k];
          }
          S2.w[J] = W;
          S2.logw[J] = std::log(W);
          for (int k = 0; k < d; ++k) S2.pts[J * d + k] = acc[k] / W;
        }
        return S2;
      };
      std::vector<int32_t> lx, ly;
      const Measure X2 = super(cx, Xc, x, lx), Y2 = super(cy, Yc, y, ly);
      S.t_super = t2;
      S.k_super_x = static_cast<int32_t>(X2.n);
      S.k_super_y = static_cast<int32_t>(Y2.n);
      Duals su{Vec(X2.n, 0.0), Vec(Y2.n, 0.0), Vec(Y2.n, 0.0), Vec(X2.n, 0.0)};
      const double sfull = double(X2.n) * X2.n + double(Y2.n) * Y2.n + 2.0 * double(X2.n) * Y2.n;
      for (int t = 0; t < t2; ++t) {
        const double pr = sym_update(X2, Y2, d, su, eps[t], lam[t], p, false, nullptr, nullptr,
                                     nullptr, nullptr);
        if (pr < 0) return fail(MSOT_ENUMERIC, "non-finite potential at scale " + std::to_string(t));
        S.pairs_evaluated += pr;
        S.pairs_dense += sfull;
      }
      for (int32_t I = 0; I < cx.k; ++I) {
        cu.a_xx[I] = su.a_xx[lx[I]];
        cu.b_yx[I] = su.b_yx[lx[I]];
      }
      for (int32_t I = 0; I < cy.k; ++I) {
        cu.b_yy[I] = su.b_yy[ly[I]];
        cu.a_xy[I] = su.a_xy[ly[I]];
      }
    }
    const double cfull = double(cx.k) * cx.k + double(cy.k) * cy.k + 2.0 * double(cx.k) * cy.k;
    for (int t = t2; t < tsw; ++t) {
      const double pr = sym_update(Xc, Yc, d, cu, eps[t], lam[t], p, false, nullptr, nullptr,
                                   nullptr, nullptr);
      if (pr < 0) return fail(MSOT_ENUMERIC, "non-finite potential at scale " + std::to_string(t));
      S.pairs_evaluated += pr;
      S.pairs_dense += cfull;
    }
    // Coarse -> fine, prm->transfer_rule:
    //   0  coarse_duals_to_fine by inheritance
    //   1  extrapolation: one lambda-damped softmin of every fine atom against
    //      the coarse measure at the last coarse eps (GeomLoss)
    Duals fu{Vec(n, 0.0), Vec(m, 0.0), Vec(m, 0.0), Vec(n, 0.0)};
    if (tsw > 0 && prm->transfer_rule == 1) {
      const int te = tsw - 1;
      const double e = eps[te], l = lam[te];
      S.pairs_evaluated += softmin_rows(Xs.pts.data(), n, d, {Xc.pts.data(), Xc.logw.data(), cu.a_xx.data(), cx.k}, e, l, p, nullptr, fu.a_xx.data());
      S.pairs_evaluated += softmin_rows(Ys.pts.data(), m, d, {Yc.pts.data(), Yc.logw.data(), cu.b_yy.data(), cy.k}, e, l, p, nullptr, fu.b_yy.data());
      S.pairs_evaluated += softmin_rows(Ys.pts.data(), m, d, {Xc.pts.data(), Xc.logw.data(), cu.b_yx.data(), cx.k}, e, l, p, nullptr, fu.a_xy.data());
      S.pairs_evaluated += softmin_rows(Xs.pts.data(), n, d, {Yc.pts.data(), Yc.logw.data(), cu.a_xy.data(), cy.k}, e, l, p, nullptr, fu.b_yx.data());
    } else if (tsw > 0) {
      for (int64_t s = 0; s < n; ++s) {
        fu.a_xx[s] = cu.a_xx[cx.labels[s]];
        fu.b_yx[s] = cu.b_yx[cx.labels[s]];
      }
      for (int64_t s = 0; s < m; ++s) {
        fu.b_yy[s] = cu.b_yy[cy.labels[s]];
        fu.a_xy[s] = cu.a_xy[cy.labels[s]];
      }
    }
    // Fine phase: block-sparse updates restricted to the truncation masks.
    std::vector<float> cxf(cx.centroids.begin(), cx.centroids.end());
    std::vector<float> cyf(cy.centroids.begin(), cy.centroids.end());
    Ranges rxx, ryy, rxy, ryx;
    std::vector<uint8_t> mxx, myy, mxy, myx;
    auto build_masks = [&](double e) {
      if (tsw == 0) {  // no coarse information: keep everything
        mxx.assign(size_t(cx.k) * cx.k, 1);
        myy.assign(size_t(cy.k) * cy.k, 1);
        mxy.assign(size_t(cx.k) * cy.k, 1);
      } else {
        std::vector<float> Fxx, Fyx, Gyy, Gxy, gxx, gyx, gyy, gxy;
        cluster_bound(fu.a_xx, Xs, cx, cxf, d, Fxx, gxx);
        cluster_bound(fu.b_yx, Xs, cx, cxf, d, Fyx, gyx);
        cluster_bound(fu.b_yy, Ys, cy, cyf, d, Gyy, gyy);
        cluster_bound(fu.a_xy, Ys, cy, cyf, d, Gxy, gxy);
        mxx.resize(size_t(cx.k) * cx.k);
        myy.resize(size_t(cy.k) * cy.k);
        mxy.resize(size_t(cx.k) * cy.k);
        const bool sl = prm->mask_rule != 1;  // slope bound on (0, 2)
        const bool bo = prm->mask_rule == 0;  // member-box bound on (0)
        auto G = [&](std::vector<float>& v) { return sl ? v.data() : nullptr; };
        const float* bxx = bo ? cx.box.data() : nullptr;
        const float* byy = bo ? cy.box.data() : nullptr;
        truncation_mask(cx.k, cx.k, d, cxf.data(), cx.radii.data(), Fxx.data(), G(gxx), cxf.data(), cx.radii.data(), Fxx.data(), G(gxx), e, prm->theta, p, 1, mxx.data(), bxx, bxx);
        truncation_mask(cy.k, cy.k, d, cyf.data(), cy.radii.data(), Gyy.data(), G(gyy), cyf.data(), cy.radii.data(), Gyy.data(), G(gyy), e, prm->theta, p, 1, myy.data(), byy, byy);
        truncation_mask(cx.k, cy.k, d, cxf.data(), cx.radii.data(), Fyx.data(), G(gyx), cyf.data(), cy.radii.data(), Gxy.data(), G(gxy), e, prm->theta, p, 0, mxy.data(), bxx, byy);
      }
      myx.resize(size_t(cy.k) * cx.k);
      for (int64_t I = 0; I < cx.k; ++I)
        for (int64_t J = 0; J < cy.k; ++J) myx[J * cx.k + I] = mxy[I * cy.k + J];
      tile_ranges(cx.labels.data(), cx.offsets.data(), cx.k, n, cx.offsets.data(), cx.k, mxx.data(), rxx);
      tile_ranges(cy.labels.data(), cy.offsets.data(), cy.k, m, cy.offsets.data(), cy.k, myy.data(), ryy);
      tile_ranges(cx.labels.data(), cx.offsets.data(), cx.k, n, cy.offsets.data(), cy.k, mxy.data(), ryx);  // rows x, cols y
      if (prm->pair_eval) {
        // pair sets of the evaluate-once kernels (sym_self / transpose_ranges)
        rxx = sym_self(rxx, n);
        ryy = sym_self(ryy, m);
        rxy = transpose_ranges(ryx, m);  // rows y, cols x
      } else {
        tile_ranges(cy.labels.data(), cy.offsets.data(), cy.k, m, cx.offsets.data(), cx.k, myx.data(), rxy);  // rows y, cols x
      }
    };
    for (int t = tsw; t <= ns; ++t) {
      const int tt = std::min(t, ns - 1);
      const bool rebuild = (t == tsw) || (prm->retruncate > 0 && t < ns && (t - tsw) % prm->retruncate == 0);
      if (rebuild) build_masks(eps[tt]);
      const double pr = sym_update(Xs, Ys, d, fu, eps[tt], lam[tt], p, t == ns, &rxx, &ryy, &rxy, &ryx);
      if (pr < 0) return fail(MSOT_ENUMERIC, "non-finite potential at scale " + std::to_string(tt));
      S.pairs_evaluated += pr;
      S.pairs_dense += full;
      S.pairs_fine += pr;
      S.pairs_fine_dense += full;
    }
    // back to the caller's order
    auto unsort = [](const Vec& v, const std::vector<int32_t>& perm) {
      Vec o(v.size());
      for (std::size_t s = 0; s < v.size(); ++s) o[perm[s]] = v[s];
      return o;
    };
    u.a_xx = unsort(fu.a_xx, px);
    u.b_yx = unsort(fu.b_yx, px);
    u.b_yy = unsort(fu.b_yy, py);
    u.a_xy = unsort(fu.a_xy, py);
  }
  // Balanced potentials are defined up to (b_yx + c, a_xy - c); return the
  // canonical representative <a, b_yx> = <b, a_xy> (same rule as
  // csrc/loss.cu), so both implementations report the same gauge.
  if (msot_reach_is_inf(prm->reach)) {
    const Vec av(a, a + n), bv(b, b + m);
    const double c = (dot(bv, u.a_xy) - dot(av, u.b_yx)) / (msot::kahan_sum(av) + msot::kahan_sum(bv));
    for (double& v : u.b_yx) v += c;
    for (double& v : u.a_xy) v -= c;
  }
  const double loss = divergence(prm, eps[ns - 1], Vec(a, a + n), Vec(b, b + m), u);
  if (!std::isfinite(loss)) return fail(MSOT_ENUMERIC, "non-finite divergence");
  if (loss_out) *loss_out = loss;
  if (a_xx) std::copy(u.a_xx.begin(), u.a_xx.end(), a_xx);
  if (b_yy) std::copy(u.b_yy.begin(), u.b_yy.end(), b_yy);
  if (a_xy) std::copy(u.a_xy.begin(), u.a_xy.end(), a_xy);
  if (b_yx) std::copy(u.b_yx.begin(), u.b_yx.end(), b_yx);
  return MSOT_OK;
}

// grad_positions with the envelope theorem, dense plans:
//   grad_i = sum_j pi^xy_ij (x_i - y_j) - sum_k pi^xx_ik (x_i - x_k),
//   pi^xy_ij = a_i b_j exp((b_yx_i + a_xy_j - C_ij)/eps),
//   pi^xx_ik = a_i a_k exp((a_xx_i + a_xx_k - C_ik)/eps).
// sign * sum_j a_i c_j exp((f_i + g_j - C_ij)/eps) (x_i - z_j), added into out
static void plan_displacement(const double* x, const double* a, int64_t n, const double* z,
                              const double* c, int64_t m, int d, const double* f, const double* g,
                              double eps, double sign, double* out) {
  msot::parallel::for_ranges(static_cast<std::size_t>(n), [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      std::vector<double> acc(d, 0.0);
      const double* xi = x + i * d;
      for (int64_t j = 0; j < m; ++j) {
        const double* zj = z + j * d;
        const double pij = a[i] * c[j] * std::exp((f[i] + g[j] - cost(xi, zj, d, 2.0)) / eps);
        for (int k = 0; k < d; ++k) acc[k] += pij * (xi[k] - zj[k]);
      }
      for (int k = 0; k < d; ++k) out[i * d + k] += sign * acc[k];
    }
  });
}

int oracle_sinkhorn_grad(const msot_params* prm, const double* x, const double* a, int64_t n,
                         const double* y, const double* b, int64_t m, int d, double* loss_out,
                         double* grad) {
  if (prm->p != 2.0) return fail(MSOT_EUSAGE, "grad_positions needs p = 2");
  Vec axx(n), byy(m), axy(m), byx(n);
  msot_stats st{};
  const int rc = oracle_sinkhorn(prm, x, a, n, y, b, m, d, axx.data(), byy.data(), axy.data(),
                                 byx.data(), loss_out, &st);
  if (rc != MSOT_OK) return rc;
  const double eps = std::pow(prm->blur, prm->p);
  std::fill(grad, grad + n * d, 0.0);
  plan_displacement(x, a, n, y, b, m, d, byx.data(), axy.data(), eps, 1.0, grad);
  plan_displacement(x, a, n, x, a, n, d, axx.data(), axx.data(), eps, -1.0, grad);
  return MSOT_OK;
}

// transfer_labels (eq. 7): the implicit plan
// pi_ij / a_i = b_j exp((f_i + g_j - C_ij)/eps) applied to the one-hot
// label columns, dense (the exact formula; a truncation mask only drops
// terms below e^-theta).
int oracle_transfer_labels(const double* x, int64_t n, const double* y, const double* b,
                           int64_t m, int d, const double* f, const double* g, double eps,
                           const int32_t* labels, int n_classes, double* scores,
                           double* row_mass) {
  if (n_classes < 1) return fail(MSOT_EUSAGE, "transfer_labels needs at least one class");
  for (int64_t j = 0; j < m; ++j)
    if (labels[j] < 0 || labels[j] >= n_classes)
      return fail(MSOT_EDATA, "label outside [0, L)");
  msot::parallel::for_ranges(static_cast<std::size_t>(n), [&](std::size_t lo, std::size_t hi) {
    Vec acc(n_classes);
    for (std::size_t i = lo; i < hi; ++i) {
      std::fill(acc.begin(), acc.end(), 0.0);
      const double* xi = x + i * d;
      for (int64_t j = 0; j < m; ++j)
        acc[labels[j]] += b[j] * std::exp((f[i] + g[j] - cost(xi, y + j * d, d, 2.0)) / eps);
      for (int l = 0; l < n_classes; ++l) scores[i * n_classes + l] = acc[l];
      row_mass[i] = msot::pairwise_sum(acc);
    }
  });
  return MSOT_OK;
}

// plan_apply (eq. 4), dense FP64.
void oracle_plan_apply(const double* x, const double* a, int64_t n, const double* y,
                       const double* b, int64_t m, int d, const double* f, const double* g,
                       double eps, const double* v, double* out) {
  msot::parallel::for_ranges(static_cast<std::size_t>(n), [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i) {
      double s = 0.0;
      for (int64_t j = 0; j < m; ++j)
        s += b[j] * std::exp((f[i] + g[j] - cost(x + i * d, y + j * d, d, 2.0)) / eps) * v[j];
      out[i] = a[i] * s;
    }
  });
}

// Barycenter descent, same rules as msot_barycenter.
int oracle_barycenter(const msot_params* prm, const double* x0, const double* a, int64_t n, int k,
                      const double* const* ys, const double* const* bs, const int64_t* ms, int d,
                      int iters, double step, double tol, double* x_out, double* loss_traj,
                      int* steps_done) {
  if (prm->p != 2.0) return fail(MSOT_EUSAGE, "barycenter descent is defined for p = 2");
  Vec x(x0, x0 + n * d), xn(n * d), field(n * d), fieldn(n * d), g(n * d), self0(n * d);
  Vec axx0(n);
  const double eps = std::pow(prm->blur, prm->p);
  struct Reset {
    ~Reset() { g_diam_override = 0.0; }
  } reset;
  // The K solves share one eps schedule (diameter of the union of x and every
  // target) and the x-x self term of target 0's solve (its final a_xx and
  // self plan), as msot_barycenter does.
  auto evaluate = [&](const Vec& xp, Vec& fld, double& L) -> int {
    std::fill(fld.begin(), fld.end(), 0.0);
    std::vector<double> lo(d, INFINITY), hi(d, -INFINITY);
    auto extend = [&](const double* p, int64_t cnt) {
      for (int64_t i = 0; i < cnt; ++i)
        for (int q = 0; q < d; ++q) {
          lo[q] = std::min(lo[q], p[i * d + q]);
          hi[q] = std::max(hi[q], p[i * d + q]);
        }
    };
    extend(xp.data(), n);
    for (int t = 0; t < k; ++t) extend(ys[t], ms[t]);
    double d2 = 0.0;
    for (int q = 0; q < d; ++q) d2 += (hi[q] - lo[q]) * (hi[q] - lo[q]);
    g_diam_override = std::sqrt(d2);
    L = 0.0;
    for (int t = 0; t < k; ++t) {
      Vec axx(n), byy(ms[t]), axy(ms[t]), byx(n);
      msot_stats st{};
      double l = 0.0;
      const int rc = oracle_sinkhorn(prm, xp.data(), a, n, ys[t], bs[t], ms[t], d, axx.data(),
                                     byy.data(), axy.data(), byx.data(), &l, &st);
      if (rc != MSOT_OK) return rc;
      if (t == 0) {
        axx0 = axx;
        std::fill(self0.begin(), self0.end(), 0.0);
        plan_displacement(xp.data(), a, n, xp.data(), a, n, d, axx0.data(), axx0.data(), eps, 1.0,
                          self0.data());
      } else {  // S = <a, b_yx - a_xx> + <b, a_xy - b_yy>: swap in the shared a_xx
        Vec dl(n);
        for (int64_t i = 0; i < n; ++i) dl[i] = a[i] * (axx[i] - axx0[i]);
        l += msot::pairwise_sum(dl);
      }
      std::fill(g.begin(), g.end(), 0.0);
      plan_displacement(xp.data(), a, n, ys[t], bs[t], ms[t], d, byx.data(), axy.data(), eps, 1.0,
                        g.data());
      for (int64_t q = 0; q < n * d; ++q) fld[q] += (g[q] - self0[q]) / k;
      L += l;
    }
    L /= k;
    return MSOT_OK;
  };
  double L = 0.0;
  int rc = evaluate(x, field, L);
  if (rc != MSOT_OK) return rc;
  if (loss_traj) loss_traj[0] = L;
  int done = 0;
  while (done < iters) {
    // each iteration starts from the configured step; the
    // halvings of a rejected trial apply to that iteration only
    double s = step;
    bool accepted = false;
    double Ln = L;
    for (int h = 0; h <= 10; ++h) {
      for (int64_t q = 0; q < n * d; ++q) xn[q] = x[q] - s * field[q] / a[q / d];
      rc = evaluate(xn, fieldn, Ln);
      if (rc != MSOT_OK) return rc;
      if (Ln <= L) { accepted = true; break; }
      s *= 0.5;
    }
    if (!accepted) break;
    std::swap(x, xn);
    std::swap(field, fieldn);
    const double rel = (L - Ln) / std::max(std::fabs(L), 1e-300);
    L = Ln;
    ++done;
    if (loss_traj) loss_traj[done] = L;
    if (rel < tol) break;
  }
  std::copy(x.begin(), x.end(), x_out);
  if (steps_done) *steps_done = done;
  return MSOT_OK;
}

}  // extern "C"
