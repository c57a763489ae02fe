// C++ caller of the msot:: API (include/msot/*.hpp), as a user of the
// reference's C++ interface would write it.  Mode "cpu": host-side measure
// constructors and schedule (SPEC.md examples); mode "gpu": solves.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <atomic>
#include <numeric>

#include "msot/barycenter.hpp"
#include "msot/common.hpp"
#include "msot/exact.hpp"
#include "msot/labels.hpp"
#include "msot/measure.hpp"
#include "msot/numeric.hpp"
#include "msot/parallel.hpp"
#include "msot/sinkhorn.hpp"

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void utility_checks() {
  // the reference's utility headers (numeric.hpp:9-15, parallel.hpp:10-17)
  using namespace msot;
  std::vector<double> v(1000);
  for (std::size_t i = 0; i < v.size(); ++i) v[i] = 1.0 / static_cast<double>(i + 1);
  double serial = 0.0;
  for (double q : v) serial += q;
  CHECK(std::fabs(pairwise_sum(v) - serial) < 1e-12);
  CHECK(std::fabs(kahan_sum(v) - serial) < 1e-12);
  CHECK(pairwise_dot(v, std::vector<double>(1000, 2.0)) == 2.0 * pairwise_sum(v));
  CHECK(pairwise_sum(std::span<const double>()) == 0.0);
  for (int nt : {1, 3, 8}) {
    parallel::set_threads(nt);
    CHECK(parallel::threads() == nt);
    std::vector<int> hit(1001, 0);
    std::atomic<int> calls{0};
    parallel::for_ranges(hit.size(), [&](std::size_t b, std::size_t e) {
      ++calls;
      for (std::size_t i = b; i < e; ++i) ++hit[i];
    });
    CHECK(std::all_of(hit.begin(), hit.end(), [](int h) { return h == 1; }));
    CHECK(calls.load() == nt);  // one contiguous chunk per thread
  }
  parallel::set_threads(0);  // clamped to 1
  CHECK(parallel::threads() == 1);
}

static void cpu_checks() {
  using namespace msot;
  utility_checks();
  // cost
  const double a0[3] = {0, 0, 0}, a1[3] = {2, 0, 0};
  CHECK(cost(a0, a1, CostSpec{2.0}) == 2.0);
  const double b0[2] = {0, 0}, b1[2] = {3, 4};
  CHECK(cost(b0, b1, CostSpec{1.0}) == 5.0);
  CHECK(throws<DataError>([] { CostSpec{2.5}.validate(); }));
  // exact_ot: unit Diracs -> C(x, y), plan [[1]]; 4x4 uniform
  // -> the best of the 24 permutation matchings; unbalanced -> DataError
  {
    DensePlan d1 = exact_ot(DiscreteMeasure({0.0, 1.0}, {1.0}, 2), DiscreteMeasure({2.0, 1.0}, {1.0}, 2));
    CHECK(d1.value == 2.0 && d1(0, 0) == 1.0);
    const std::vector<double> px = {0.1, 0.9, 0.4, 0.2, 0.8, 0.5, 0.3, 0.7};
    const std::vector<double> py = {0.6, 0.1, 0.2, 0.3, 0.9, 0.8, 0.5, 0.5};
    const std::vector<double> w4(4, 0.25);
    DiscreteMeasure X(px, w4, 2), Y(py, w4, 2);
    int perm[4] = {0, 1, 2, 3};
    double best = 1e300;
    do {
      double s = 0.0;
      for (int i = 0; i < 4; ++i) s += 0.25 * cost(X.point(i), Y.point(perm[i]), CostSpec{});
      best = std::min(best, s);
    } while (std::next_permutation(perm, perm + 4));
    CHECK(std::fabs(exact_ot(X, Y).value - best) < 1e-15);
    CHECK(throws<DataError>([&] { exact_ot(X, DiscreteMeasure({0.0, 0.0}, {0.5}, 2)); }));
  }
  // zero weights dropped, invariants
  DiscreteMeasure m({0, 0, 1, 1, 2, 2}, {0.5, 0.0, 0.5}, 2);
  CHECK(m.size() == 2 && m.total_mass() == 1.0 && m.point(1)[0] == 2.0);
  CHECK(throws<DataError>([] { DiscreteMeasure({0.0}, {-1.0}, 1); }));
  CHECK(throws<DataError>([] { DiscreteMeasure({0.0, 1.0}, {0.0, 0.0}, 1); }));
  const std::size_t order[2] = {1, 0};
  CHECK(m.permuted(order).point(0)[0] == 2.0);
  // schedule
  SolverParams p;
  p.blur = 1.0;
  p.scaling = 0.5;
  auto s = make_schedule(8.0, p);
  CHECK(s.size() == 4 && s.sigma[0] == 8 && s.sigma[3] == 1 && s.eps[1] == 16 && s.lambda[2] == 1);
  p.scaling = 0.9;
  CHECK(make_schedule(10.0, p).size() == 22);
  {  // reach must be > 0 or +inf; 0 is not "balanced"
    SolverParams z;
    z.reach = 0.0;
    CHECK(throws<DataError>([&] { z.to_c(); }));
    z.reach = -1.0;
    CHECK(throws<DataError>([&] { z.to_c(); }));
  }
  CHECK(make_schedule(1.0, p).size() == 1);
  // encode_fibers
  FiberSet fs;
  fs.resample_count = 3;
  fs.fibers = {{{0, 0, 0}, {1, 0, 0}}, {{0, 0, 0}, {1, 0, 0}}};
  DiscreteMeasure f = encode_fibers(fs);
  const double r3 = 1.0 / std::sqrt(3.0);
  CHECK(f.dim() == 9 && std::fabs(f.point(0)[3] - 0.5 * r3) < 1e-15 && std::fabs(f.point(0)[6] - r3) < 1e-15);
  CHECK(f.weights()[0] == 0.5);
  FiberSet bad;
  bad.resample_count = 3;
  bad.fibers = {{{1, 1, 1}, {1, 1, 1}}};
  CHECK(throws<DataError>([&] { encode_fibers(bad); }));
  // flip_augment
  FiberSet two;
  two.resample_count = 2;
  two.fibers = {{{0, 0, 0}, {1, 0, 0}}};
  auto aug = flip_augment(encode_fibers(two), 2);
  const double r2 = 1.0 / std::sqrt(2.0);
  CHECK(aug.measure.size() == 2 && aug.map.is_flipped(1) && aug.map.original_of(1) == 0);
  CHECK(std::fabs(aug.measure.point(1)[0] - r2) < 1e-15 && aug.measure.point(1)[3] == 0.0);
  CHECK(aug.measure.total_mass() == 1.0);
  // density_to_measure
  DensityMap dm;
  dm.nx = dm.ny = dm.nz = 4;
  dm.voxels = {{0, 0, 0, 1.0}, {1, 2, 3, 3.0}, {2, 2, 2, 0.0}};
  DiscreteMeasure dmeas = density_to_measure(dm);
  CHECK(dmeas.size() == 2 && dmeas.weights()[0] == 0.25 && dmeas.point(1)[2] == 3.5);
  DensityMap empty;
  empty.nx = empty.ny = empty.nz = 1;
  empty.voxels = {{0, 0, 0, 0.0}};
  CHECK(throws<DataError>([&] { density_to_measure(empty); }));
  // resolve_flips / classify, host-only
  SoftLabels sl;
  sl.n = 4;
  sl.L = 2;
  sl.scores = {0.9, 0.0, 0.01, 0.01, 0.05, 0.0, 0.0, 0.7};
  sl.row_mass = {0.9, 0.02, 0.05, 0.7};
  SoftLabels r = resolve_flips(sl, FlipMap{2});
  CHECK(r.n == 2 && r.row_mass[0] == 0.9 && r.row_mass[1] == 0.7 && r.score(1, 1) == 0.7);
  Classification cl = classify(r, 0.5);
  CHECK(cl.label[0] == 0 && cl.label[1] == 1 && cl.confidence[0] == 1.0);
  CHECK(classify(sl, 0.5).label[1] == OUTLIER);
  CHECK(throws<DataError>([&] { resolve_flips(sl, FlipMap{3}); }));
}

static void gpu_checks() {
  using namespace msot;
  SolverParams p;
  p.blur = 0.01;
  // Dirac translation -> |t|^2/2
  DiscreteMeasure a({0, 0, 0}, {1.0}, 3), b({1.0, 0.5, 0.0}, {1.0}, 3);
  const double s = divergence(a, b, p);
  CHECK(std::fabs(s - 0.625) < 6.25e-3);
  // alpha = beta: symmetric potentials, S ~ 0
  std::vector<double> pts, w;
  for (int i = 0; i < 500; ++i) {
    pts.push_back(std::sin(1.3 * i));
    pts.push_back(std::cos(0.7 * i));
    pts.push_back(0.01 * i);
    w.push_back(1.0 + (i % 7));
  }
  DiscreteMeasure c(pts, w, 3);
  p.blur = 0.05;
  DualPotentials u = symmetric_sinkhorn(c, c, p);
  bool same = true;
  for (std::size_t i = 0; i < c.size(); ++i) same = same && u.a_xx[i] == u.b_yy[i] && u.a_xy[i] == u.b_yx[i];
  CHECK(same);
  CHECK(std::fabs(divergence(c, c, p)) < 1e-9);
  SolverParams q = p;
  q.multiscale = true;
  // multiscale fine phase evaluates each kept pair once: a_xy comes from
  // column sums and b_yx from row sums, so S(c, c) is zero up to float32
  // rounding of the potentials (1e-4 eps per unit mass; the contract allows
  // 1e-3 eps per potential)
  {
    double mass = 0.0;
    for (double v : w) mass += v;
    const double s = divergence(c, c, q);
    CHECK(std::fabs(s) < 1e-4 * 0.05 * 0.05 * mass);
  }
  // softmin of SPEC.md:170
  DiscreteMeasure x({0.0}, {1.0}, 1), y({1.5}, {1.0}, 1);
  auto f = softmin(x, y, {0.0}, 0.3);
  CHECK(std::fabs(f[0] - 1.125) < 1e-6);
  // errors surface as the reference's exception types
  SolverParams bad = p;
  bad.cost.p = 1.0;
  CHECK(throws<DataError>([&] { divergence(a, b, bad); }));
  DiscreteMeasure d2({0.0, 0.0}, {1.0}, 2);
  CHECK(throws<DataError>([&] { divergence(a, d2, p); }));
  // transfer_labels: bijective unit Diracs -> one-hot rows
  DiscreteMeasure u4({0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1}, {0.25, 0.25, 0.25, 0.25}, 3);
  DiscreteMeasure v4({0.01, 0, 0, 1.01, 0, 0, 0.01, 1, 0, 0.01, 0, 1}, {0.25, 0.25, 0.25, 0.25}, 3);
  SolverParams lp;
  lp.blur = 0.05;
  lp.scaling = 0.7;
  LabelSet ls{4, {"a", "b", "c", "d"}, {0, 1, 2, 3}};
  SoftLabels soft = transfer_labels(u4, v4, ls, lp);
  bool onehot = true;
  for (int i = 0; i < 4; ++i)
    for (int l = 0; l < 4; ++l) onehot = onehot && std::fabs(soft.score(i, l) - (i == l)) < 1e-3;
  CHECK(onehot);
  CHECK(throws<DataError>([&] { transfer_labels(u4, v4, LabelSet{4, {}, {0, 1}}, lp); }));
  // grad_positions: translated Dirac -> alpha (x - y)
  double gl = 0.0;
  auto g = grad_positions(a, b, p, &gl);
  CHECK(std::fabs(g[0] + 1.0) < 1e-2 && std::fabs(g[1] + 0.5) < 1e-2 && std::fabs(g[2]) < 1e-2);
  // barycenter of two Diracs -> their midpoint
  DiscreteMeasure t0({-1.0, 0.0, 0.0}, {1.0}, 3), t1({1.0, 0.0, 0.0}, {1.0}, 3);
  DiscreteMeasure init({0.3, 0.2, 0.0}, {1.0}, 3);
  SolverParams bp;
  bp.blur = 0.05;
  BarycenterResult br = barycenter({t0, t1}, init, bp, BarycenterConfig{20, 1.0, 0.0});
  CHECK(std::fabs(br.measure.point(0)[0]) < 1e-2 && std::fabs(br.measure.point(0)[1]) < 1e-2);
  CHECK(br.loss.back() <= br.loss.front());
  // implicit plan: unit Diracs -> plan_entry = 1, ot_value = C(x, y)
  DualPotentials du = symmetric_sinkhorn(a, b, p);
  CHECK(std::fabs(plan_entry(0, 0, a, b, du, p) - 1.0) < 1e-3);
  CHECK(std::fabs(plan_apply(a, b, du, p, {2.0})[0] - 2.0) < 2e-3);
  CHECK(std::fabs(ot_value(a, b, du, p) - 0.625) < 1e-3);
  // grad_weights: alpha = beta -> ~0
  DualPotentials uu = symmetric_sinkhorn(u4, u4, lp);
  bool zero = true;
  for (double gq : grad_weights(u4, u4, uu, lp)) zero = zero && std::fabs(gq) < 1e-6 * 0.05 * 0.05 + 1e-9;
  CHECK(zero);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_checks();
  if (mode == "gpu") gpu_checks();
  if (failures) {
    std::fprintf(stderr, "%d check(s) failed\n", failures);
    return 1;
  }
  std::printf("frontend_test %s: ok\n", mode.c_str());
  return 0;
}
