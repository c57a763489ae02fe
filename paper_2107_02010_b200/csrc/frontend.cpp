// frontend.cpp — the msot:: C++ API (include/msot/*.hpp) over the C ABI.
//
// Measures and their constructors follow SPEC.md:27-120 (reference
// declarations: proj/include/msot/measure.hpp); the solver operations
// forward to libmsot_b200's GPU entry points and rethrow status codes as the
// reference's exception types (proj/include/msot/common.hpp:10-19).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "../../include/msot/common.hpp"
#include "../../include/msot/measure.hpp"
#include "../../include/msot/sinkhorn.hpp"
#include "../../include/msot/labels.hpp"
#include "../../include/msot/barycenter.hpp"
#include "../../include/msot/exact.hpp"

namespace msot {

void throw_on_status(int status, const std::string& what) {
  if (status == MSOT_OK) return;
  const std::string msg = what + ": " + msot_last_error();
  if (status == MSOT_ENUMERIC) throw NumericError(msg);
  if (status == MSOT_EDATA || status == MSOT_EUSAGE) throw DataError(msg);
  throw DeviceError(msg);
}

// ------------------------------------------------------------------ measures
void CostSpec::validate() const {
  if (!(p >= 1.0 && p <= 2.0)) throw DataError("CostSpec: p must lie in [1, 2]");
}

double cost(std::span<const double> x, std::span<const double> y, const CostSpec& spec) {
  spec.validate();
  if (x.size() != y.size()) throw DataError("cost: dimension mismatch");
  double s = 0.0;
  for (std::size_t k = 0; k < x.size(); ++k) s += (x[k] - y[k]) * (x[k] - y[k]);
  if (spec.p == 2.0) return 0.5 * s;
  return std::pow(std::sqrt(s), spec.p) / spec.p;
}

DiscreteMeasure::DiscreteMeasure(std::vector<double> points, std::vector<double> weights,
                                 std::size_t dim)
    : dim_(dim) {
  if (dim == 0) throw DataError("DiscreteMeasure: dimension must be >= 1");
  if (points.size() != weights.size() * dim)
    throw DataError("DiscreteMeasure: points and weights sizes disagree");
  double mass = 0.0;
  for (std::size_t i = 0; i < weights.size(); ++i) {
    const double w = weights[i];
    if (!(w >= 0.0) || !std::isfinite(w)) throw DataError("DiscreteMeasure: weights must be >= 0");
    for (std::size_t k = 0; k < dim; ++k)
      if (!std::isfinite(points[i * dim + k])) throw DataError("DiscreteMeasure: non-finite point");
    if (w == 0.0) continue;  // zero weights dropped
    points_.insert(points_.end(), points.begin() + i * dim, points.begin() + (i + 1) * dim);
    weights_.push_back(w);
    log_weights_.push_back(std::log(w));
    mass += w;
  }
  if (weights_.empty() || !(mass > 0.0)) throw DataError("DiscreteMeasure: total mass must be > 0");
  total_mass_ = mass;
}

DiscreteMeasure DiscreteMeasure::with_points(std::vector<double> points) const {
  return DiscreteMeasure(std::move(points), weights_, dim_);
}

DiscreteMeasure DiscreteMeasure::permuted(std::span<const std::size_t> order) const {
  if (order.size() != size()) throw DataError("permuted: order has the wrong length");
  std::vector<char> seen(size(), 0);
  std::vector<double> p(points_.size()), w(size());
  for (std::size_t s = 0; s < order.size(); ++s) {
    const std::size_t i = order[s];
    if (i >= size() || seen[i]) throw DataError("permuted: not a permutation");
    seen[i] = 1;
    std::copy_n(points_.begin() + i * dim_, dim_, p.begin() + s * dim_);
    w[s] = weights_[i];
  }
  return DiscreteMeasure(std::move(p), std::move(w), dim_);
}

DiscreteMeasure encode_fibers(const FiberSet& fs) {
  const int P = fs.resample_count;
  if (P < 2) throw DataError("encode_fibers: resample_count must be >= 2");
  if (fs.fibers.empty()) throw DataError("encode_fibers: empty fiber set");
  const std::size_t n = fs.fibers.size();
  std::vector<double> pts(n * 3 * P), w(n, 1.0 / static_cast<double>(n));
  const double scale = 1.0 / std::sqrt(static_cast<double>(P));
  for (std::size_t f = 0; f < n; ++f) {
    const Polyline& line = fs.fibers[f];
    if (line.size() < 2) throw DataError("encode_fibers: fiber " + std::to_string(f) + " has < 2 points");
    std::vector<double> arc(line.size(), 0.0);
    for (std::size_t v = 1; v < line.size(); ++v) {
      double s = 0.0;
      for (int k = 0; k < 3; ++k) s += (line[v][k] - line[v - 1][k]) * (line[v][k] - line[v - 1][k]);
      arc[v] = arc[v - 1] + std::sqrt(s);
    }
    const double L = arc.back();
    if (!(L > 0.0)) throw DataError("encode_fibers: fiber " + std::to_string(f) + " is degenerate");
    std::size_t seg = 0;
    for (int q = 0; q < P; ++q) {
      const double target = L * static_cast<double>(q) / static_cast<double>(P - 1);
      while (seg + 2 < line.size() && arc[seg + 1] < target) ++seg;
      const double len = arc[seg + 1] - arc[seg];
      const double t = len > 0.0 ? std::clamp((target - arc[seg]) / len, 0.0, 1.0) : 0.0;
      for (int k = 0; k < 3; ++k)
        pts[f * 3 * P + 3 * q + k] = scale * ((1.0 - t) * line[seg][k] + t * line[seg + 1][k]);
    }
  }
  return DiscreteMeasure(std::move(pts), std::move(w), static_cast<std::size_t>(3 * P));
}

AugmentedMeasure flip_augment(const DiscreteMeasure& m, int P) {
  if (P < 1 || m.dim() != static_cast<std::size_t>(3 * P))
    throw DataError("flip_augment: atom dimension must equal 3P");
  const std::size_t n = m.size(), D = m.dim();
  std::vector<double> pts(2 * n * D), w(2 * n);
  for (std::size_t i = 0; i < n; ++i) {
    auto src = m.point(i);
    std::copy(src.begin(), src.end(), pts.begin() + i * D);
    for (int q = 0; q < P; ++q)
      for (int k = 0; k < 3; ++k) pts[(n + i) * D + 3 * q + k] = src[3 * (P - 1 - q) + k];
    w[i] = w[n + i] = 0.5 * m.weights()[i];
  }
  return {DiscreteMeasure(std::move(pts), std::move(w), D), FlipMap{n}};
}

DiscreteMeasure density_to_measure(const DensityMap& d) {
  std::vector<double> pts, w;
  double sum = 0.0, carry = 0.0;  // Kahan
  for (const DensityVoxel& v : d.voxels) {
    if (!(v.value >= 0.0) || !std::isfinite(v.value)) throw DataError("density_to_measure: negative value");
    if (v.value == 0.0) continue;
    if (v.i < 0 || v.j < 0 || v.k < 0 || v.i >= d.nx || v.j >= d.ny || v.k >= d.nz)
      throw DataError("density_to_measure: voxel index outside the grid");
    pts.push_back(d.origin[0] + (v.i + 0.5) * d.voxel_mm);
    pts.push_back(d.origin[1] + (v.j + 0.5) * d.voxel_mm);
    pts.push_back(d.origin[2] + (v.k + 0.5) * d.voxel_mm);
    w.push_back(v.value);
    const double y = v.value - carry, t = sum + y;
    carry = (t - sum) - y;
    sum = t;
  }
  if (w.empty()) throw DataError("density_to_measure: all-zero map");
  for (double& x : w) x /= sum;
  return DiscreteMeasure(std::move(pts), std::move(w), 3);
}

// -------------------------------------------------------------------- solver
msot_params SolverParams::to_c() const {
  cost.validate();
  if (!(reach > 0.0)) throw DataError("SolverParams: reach must be > 0 (or +inf)");
  msot_params p;
  msot_params_default(&p);
  p.blur = blur;
  p.reach = reach;
  p.p = cost.p;
  p.scaling = scaling;
  p.max_full_iters = max_full_iters;
  p.multiscale = multiscale ? 1 : 0;
  p.retruncate = retruncate;
  p.cluster_scale = cluster_scale;
  p.theta = theta;
  p.switch_factor = switch_factor;
  p.mask_rule = mask_rule;
  p.transfer_rule = transfer_rule;
  p.pair_eval = pair_eval;
  p.clusters = clusters;
  p.seed = seed;
  p.super_level = super_level;
  return p;
}

Device::Device(int device) { throw_on_status(msot_create(device, &ctx_), "msot_create"); }

Device::Device(int device, int rank, int world, const unsigned char nccl_id[128]) {
  throw_on_status(msot_create_dist(device, rank, world, nccl_id, &ctx_), "msot_create_dist");
}

Device::~Device() { msot_destroy(ctx_); }

Device& default_device() {
  thread_local Device dev(0);
  return dev;
}

double diameter_estimate(const DiscreteMeasure& a, const DiscreteMeasure& b, double blur) {
  if (a.dim() != b.dim()) throw DataError("diameter_estimate: dimension mismatch");
  const std::size_t D = a.dim();
  std::vector<double> lo(D, INFINITY), hi(D, -INFINITY);
  for (const DiscreteMeasure* m : {&a, &b})
    for (std::size_t i = 0; i < m->size(); ++i)
      for (std::size_t k = 0; k < D; ++k) {
        lo[k] = std::min(lo[k], m->point(i)[k]);
        hi[k] = std::max(hi[k], m->point(i)[k]);
      }
  double s = 0.0;
  for (std::size_t k = 0; k < D; ++k) s += (hi[k] - lo[k]) * (hi[k] - lo[k]);
  return std::max(std::sqrt(s), blur);
}

EpsSchedule make_schedule(double d, const SolverParams& params) {
  const msot_params p = params.to_c();
  int n = msot_schedule(d, &p, nullptr, nullptr, nullptr, 0);
  n = n < 0 ? -n : n;
  EpsSchedule s;
  s.sigma.resize(n);
  s.eps.resize(n);
  s.lambda.resize(n);
  msot_schedule(d, &p, s.sigma.data(), s.eps.data(), s.lambda.data(), n);
  return s;
}

std::vector<double> softmin(const DiscreteMeasure& rows, const DiscreteMeasure& cols,
                            const std::vector<double>& h, double eps, double lambda, Device& dev) {
  if (rows.dim() != cols.dim()) throw DataError("softmin: dimension mismatch");
  if (h.size() != cols.size()) throw DataError("softmin: potential size mismatch");
  std::vector<double> out(rows.size());
  const std::vector<double> lw(cols.log_weights().begin(), cols.log_weights().end());
  throw_on_status(msot_softmin(dev.get(), rows.points().data(), static_cast<int64_t>(rows.size()),
                               cols.points().data(), static_cast<int64_t>(cols.size()),
                               static_cast<int>(rows.dim()), lw.data(), h.data(), eps, lambda,
                               nullptr, out.data()),
                  "softmin");
  return out;
}

static DualPotentials solve(const DiscreteMeasure& a, const DiscreteMeasure& b,
                            const SolverParams& params, Device& dev, double* loss) {
  if (a.dim() != b.dim()) throw DataError("dimension mismatch between the two measures");
  const msot_params p = params.to_c();
  DualPotentials u;
  u.a_xx.resize(a.size());
  u.b_yx.resize(a.size());
  u.b_yy.resize(b.size());
  u.a_xy.resize(b.size());
  double l = 0.0;
  msot_stats st;
  throw_on_status(msot_sinkhorn(dev.get(), &p, a.points().data(), a.weights().data(),
                                static_cast<int64_t>(a.size()), b.points().data(),
                                b.weights().data(), static_cast<int64_t>(b.size()),
                                static_cast<int>(a.dim()), u.a_xx.data(), u.b_yy.data(),
                                u.a_xy.data(), u.b_yx.data(), &l, &st),
                  "sinkhorn");
  u.eps = std::pow(params.blur, params.cost.p);
  if (loss) *loss = l;
  return u;
}

DualPotentials symmetric_sinkhorn(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                  const SolverParams& params, Device& dev) {
  SolverParams q = params;
  q.multiscale = false;
  return solve(a, b, q, dev, nullptr);
}

DualPotentials multiscale_sinkhorn(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                   SolverParams params, Device& dev) {
  params.multiscale = true;
  return solve(a, b, params, dev, nullptr);
}

double divergence(const DiscreteMeasure& a, const DiscreteMeasure& b, const SolverParams& params,
                  Device& dev) {
  double loss = 0.0;
  solve(a, b, params, dev, &loss);
  return loss;
}

// ------------------------------------------------------------ implicit plan
static bool reach_inf(const SolverParams& p) {
  if (!(p.reach > 0.0)) throw DataError("SolverParams: reach must be > 0 (or +inf)");
  return std::isinf(p.reach);
}

double plan_entry(std::size_t i, std::size_t j, const DiscreteMeasure& a,
                  const DiscreteMeasure& b, const DualPotentials& duals,
                  const SolverParams& params) {
  if (i >= a.size() || j >= b.size()) throw DataError("plan_entry: index out of range");
  if (duals.b_yx.size() != a.size() || duals.a_xy.size() != b.size())
    throw DataError("plan_entry: duals do not match the measures");
  const double c = cost(a.point(i), b.point(j), params.cost);
  return a.weights()[i] * b.weights()[j] * std::exp((duals.b_yx[i] + duals.a_xy[j] - c) / duals.eps);
}

std::vector<double> plan_apply(const DiscreteMeasure& a, const DiscreteMeasure& b,
                               const DualPotentials& duals, const SolverParams& params,
                               const std::vector<double>& v, Device& dev) {
  if (a.dim() != b.dim()) throw DataError("plan_apply: dimension mismatch");
  if (v.size() != b.size()) throw DataError("plan_apply: v must be sized to b");
  if (duals.b_yx.size() != a.size() || duals.a_xy.size() != b.size())
    throw DataError("plan_apply: duals do not match the measures");
  if (params.cost.p != 2.0) throw DataError("plan_apply: the GPU path implements p = 2");
  std::vector<double> out(a.size());
  throw_on_status(msot_plan_apply(dev.get(), a.points().data(), a.weights().data(),
                                  static_cast<int64_t>(a.size()), b.points().data(),
                                  b.weights().data(), static_cast<int64_t>(b.size()),
                                  static_cast<int>(a.dim()), duals.b_yx.data(), duals.a_xy.data(),
                                  duals.eps, v.data(), out.data()),
                  "plan_apply");
  return out;
}

double ot_value(const DiscreteMeasure& a, const DiscreteMeasure& b, const DualPotentials& duals,
                const SolverParams& params, Device& dev) {
  const std::vector<double> ones(b.size(), 1.0);
  const std::vector<double> pv = plan_apply(a, b, duals, params, ones, dev);
  double mass = 0.0;
  for (double q : pv) mass += q;
  const double eps = duals.eps;
  const double ma = a.total_mass(), mb = b.total_mass();
  double s = 0.0;
  if (reach_inf(params)) {
    for (std::size_t i = 0; i < a.size(); ++i) s += a.weights()[i] * duals.b_yx[i];
    for (std::size_t j = 0; j < b.size(); ++j) s += b.weights()[j] * duals.a_xy[j];
  } else {  // PAPER.md eq. 3
    const double rho = std::pow(params.reach, params.cost.p);
    for (std::size_t i = 0; i < a.size(); ++i)
      s += rho * a.weights()[i] * (1.0 - std::exp(-duals.b_yx[i] / rho));
    for (std::size_t j = 0; j < b.size(); ++j)
      s += rho * b.weights()[j] * (1.0 - std::exp(-duals.a_xy[j] / rho));
  }
  return s + eps * (ma * mb - mass);
}

std::vector<double> grad_weights(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                 const DualPotentials& duals, const SolverParams& params) {
  if (duals.a_xx.size() != a.size() || duals.b_yx.size() != a.size())
    throw DataError("grad_weights: duals do not match the measure");
  std::vector<double> gw(a.size());
  const double eps = duals.eps;
  if (reach_inf(params)) {
    const double defect = eps * (a.total_mass() - b.total_mass());
    for (std::size_t i = 0; i < a.size(); ++i) gw[i] = duals.b_yx[i] - duals.a_xx[i] + defect;
  } else {
    const double rho = std::pow(params.reach, params.cost.p);
    for (std::size_t i = 0; i < a.size(); ++i)
      gw[i] = (rho + 0.5 * eps) * (std::exp(-duals.a_xx[i] / rho) - std::exp(-duals.b_yx[i] / rho));
  }
  return gw;
}

// ------------------------------------------------------------------ labeling
SoftLabels transfer_labels(const DiscreteMeasure& a, const DiscreteMeasure& b,
                           const LabelSet& labels, const SolverParams& params, Device& dev) {
  if (a.dim() != b.dim()) throw DataError("transfer_labels: dimension mismatch");
  if (labels.assignments.size() != b.size())
    throw DataError("transfer_labels: labels must be sized to the atlas measure");
  const msot_params p = params.to_c();
  std::vector<int32_t> lab(labels.assignments.begin(), labels.assignments.end());
  SoftLabels out;
  out.n = a.size();
  out.L = labels.L;
  out.scores.resize(a.size() * static_cast<std::size_t>(std::max(labels.L, 0)));
  out.row_mass.resize(a.size());
  double loss = 0.0;
  msot_stats st;
  throw_on_status(msot_transfer_labels(dev.get(), &p, a.points().data(), a.weights().data(),
                                       static_cast<int64_t>(a.size()), b.points().data(),
                                       b.weights().data(), static_cast<int64_t>(b.size()),
                                       static_cast<int>(a.dim()), lab.data(), labels.L,
                                       out.scores.data(), out.row_mass.data(), &loss, &st),
                  "transfer_labels");
  return out;
}

SoftLabels resolve_flips(const SoftLabels& soft, const FlipMap& map) {
  if (soft.n != 2 * map.originals) throw DataError("resolve_flips: missing flip pair");
  std::vector<int32_t> of(soft.n), ori(soft.n), chosen(map.originals);
  for (std::size_t i = 0; i < soft.n; ++i) {
    of[i] = static_cast<int32_t>(map.original_of(i));
    ori[i] = map.is_flipped(i) ? 1 : 0;
  }
  SoftLabels out;
  out.n = map.originals;
  out.L = soft.L;
  out.scores.resize(out.n * static_cast<std::size_t>(soft.L));
  out.row_mass.resize(out.n);
  throw_on_status(msot_resolve_flips(soft.scores.data(), soft.row_mass.data(),
                                     static_cast<int64_t>(soft.n), soft.L, of.data(), ori.data(),
                                     out.scores.data(), out.row_mass.data(), chosen.data()),
                  "resolve_flips");
  return out;
}

Classification classify(const SoftLabels& soft, double tau) {
  std::vector<int32_t> lab(soft.n);
  Classification c;
  c.confidence.resize(soft.n);
  throw_on_status(msot_classify(soft.scores.data(), soft.row_mass.data(),
                                static_cast<int64_t>(soft.n), soft.L, tau, lab.data(),
                                c.confidence.data()),
                  "classify");
  c.label.assign(lab.begin(), lab.end());
  return c;
}

// ------------------------------------------------------- gradients / barycenter
std::vector<double> grad_positions(const DiscreteMeasure& a, const DiscreteMeasure& b,
                                   const SolverParams& params, double* loss, Device& dev) {
  if (a.dim() != b.dim()) throw DataError("grad_positions: dimension mismatch");
  const msot_params p = params.to_c();
  std::vector<double> g(a.size() * a.dim());
  double l = 0.0;
  msot_stats st;
  throw_on_status(msot_sinkhorn_grad(dev.get(), &p, a.points().data(), a.weights().data(),
                                     static_cast<int64_t>(a.size()), b.points().data(),
                                     b.weights().data(), static_cast<int64_t>(b.size()),
                                     static_cast<int>(a.dim()), &l, g.data(), &st),
                  "grad_positions");
  if (loss) *loss = l;
  return g;
}

BarycenterResult barycenter(const std::vector<DiscreteMeasure>& targets,
                            const DiscreteMeasure& init, const SolverParams& params,
                            const BarycenterConfig& cfg, Device& dev) {
  if (targets.empty()) throw DataError("barycenter: no targets");
  const msot_params p = params.to_c();
  const int k = static_cast<int>(targets.size());
  std::vector<const double*> ys(k), bs(k);
  std::vector<int64_t> ms(k);
  for (int t = 0; t < k; ++t) {
    if (targets[t].dim() != init.dim()) throw DataError("barycenter: dimension mismatch");
    ys[t] = targets[t].points().data();
    bs[t] = targets[t].weights().data();
    ms[t] = static_cast<int64_t>(targets[t].size());
  }
  std::vector<double> x(init.size() * init.dim()), traj(cfg.iters + 1);
  int done = 0;
  msot_stats st;
  throw_on_status(msot_barycenter(dev.get(), &p, init.points().data(), init.weights().data(),
                                  static_cast<int64_t>(init.size()), k, ys.data(), bs.data(),
                                  ms.data(), static_cast<int>(init.dim()), cfg.iters, cfg.step,
                                  cfg.tol, x.data(), traj.data(), &done, &st),
                  "barycenter");
  traj.resize(done + 1);
  return {init.with_points(std::move(x)), std::move(traj)};
}

// -------------------------------------------------------------- exact oracle
DensePlan exact_ot(const DiscreteMeasure& a, const DiscreteMeasure& b, const CostSpec& spec) {
  spec.validate();
  if (a.dim() != b.dim()) throw DataError("exact_ot: dimension mismatch");
  DensePlan out;
  out.rows = a.size();
  out.cols = b.size();
  out.pi.assign(out.rows * out.cols, 0.0);
  throw_on_status(msot_exact_ot(a.points().data(), a.weights().data(),
                                static_cast<int64_t>(a.size()), b.points().data(),
                                b.weights().data(), static_cast<int64_t>(b.size()),
                                static_cast<int>(a.dim()), spec.p, out.pi.data(), &out.value),
                  "exact_ot");
  return out;
}

}  // namespace msot
