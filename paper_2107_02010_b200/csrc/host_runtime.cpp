// host_runtime.cpp — msot::kahan_sum / pairwise_sum / pairwise_dot
// (include/msot/numeric.hpp) and msot::parallel (include/msot/parallel.hpp),
// the reference's host utilities (proj/include/msot/numeric.hpp:9-15,
// parallel.hpp:10-17) re-implemented for the GPU build's front-end.
//
// Summation: the cascade tree splits a span of n > 32 terms into [0, n/2)
// and [n/2, n) and sums each leaf of <= 32 terms left to right — the
// reference's tree, so the bits agree (tests/test_abi.py checks this against
// the reference's own numeric.cpp compiled into oracle/_ref).  The tree is
// walked iteratively with an explicit stack of partial sums.
//
// Pool: persistent workers woken per call through a generation counter; the
// caller runs the last chunk itself.  Not re-entrant (as the reference,
// parallel.cpp:35-47): a for_ranges call from inside fn runs serially.
#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "msot/numeric.hpp"
#include "msot/parallel.hpp"

namespace msot {

double kahan_sum(std::span<const double> values) {
  double s = 0.0, comp = 0.0;
  for (const double v : values) {
    const double y = v - comp;
    const double t = s + y;
    comp = (t - s) - y;
    s = t;
  }
  return s;
}

namespace {

constexpr std::size_t kLeaf = 32;

// Post-order walk of the halving tree over [0, n): leaves are summed by
// `leaf(begin, end)`, inner nodes add their left and right partials.
template <class Leaf>
double cascade(std::size_t n, Leaf&& leaf) {
  struct Node {
    std::size_t b, e;
    int state;    // 0: unvisited, 1: left done
    double left;
  };
  std::vector<Node> st;
  st.reserve(64);
  st.push_back({0, n, 0, 0.0});
  double ret = 0.0;
  bool have = false;  // `ret` holds the value of the node just finished
  while (!st.empty()) {
    Node& nd = st.back();
    const std::size_t len = nd.e - nd.b;
    if (len <= kLeaf) {
      ret = leaf(nd.b, nd.e);
      have = true;
      st.pop_back();
      continue;
    }
    const std::size_t mid = nd.b + len / 2;
    if (nd.state == 0) {
      if (have) {  // returning from the left child
        nd.left = ret;
        nd.state = 1;
        have = false;
        st.push_back({mid, nd.e, 0, 0.0});
      } else {
        st.push_back({nd.b, mid, 0, 0.0});
      }
    } else {  // returning from the right child
      ret = nd.left + ret;
      have = true;
      st.pop_back();
    }
  }
  return ret;
}

}  // namespace

double pairwise_sum(std::span<const double> values) {
  const double* v = values.data();
  return cascade(values.size(), [v](std::size_t b, std::size_t e) {
    double s = 0.0;
    for (std::size_t i = b; i < e; ++i) s += v[i];
    return s;
  });
}

double pairwise_dot(std::span<const double> a, std::span<const double> b) {
  const double* x = a.data();
  const double* y = b.data();
  const std::size_t n = a.size() < b.size() ? a.size() : b.size();
  return cascade(n, [x, y](std::size_t lo, std::size_t hi) {
    double s = 0.0;
    for (std::size_t i = lo; i < hi; ++i) s += x[i] * y[i];
    return s;
  });
}

namespace parallel {
namespace {

class Workers {
 public:
  explicit Workers(int n) {
    for (int k = 0; k < n; ++k) th_.emplace_back([this, k] { loop(k); });
  }
  ~Workers() {
    {
      std::lock_guard<std::mutex> g(mu_);
      quit_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return static_cast<int>(th_.size()); }

  // task(k) for k in [0, size()] — workers take 0..size()-1, the caller size()
  void run(const std::function<void(int)>& task) {
    {
      std::lock_guard<std::mutex> g(mu_);
      task_ = &task;
      left_ = size();
      ++gen_;
    }
    cv_.notify_all();
    task(size());
    std::unique_lock<std::mutex> g(mu_);
    done_cv_.wait(g, [this] { return left_ == 0; });
    task_ = nullptr;
  }

 private:
  void loop(int k) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* t;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return quit_ || gen_ != seen; });
        if (quit_) return;
        seen = gen_;
        t = task_;
      }
      (*t)(k);
      std::lock_guard<std::mutex> g(mu_);
      if (--left_ == 0) done_cv_.notify_all();
    }
  }

  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* task_ = nullptr;
  uint64_t gen_ = 0;
  int left_ = 0;
  bool quit_ = false;
};

std::mutex g_mu;
int g_n = 0;  // 0: hardware concurrency, resolved on first use
std::unique_ptr<Workers> g_workers;
thread_local bool g_inside = false;

int resolve_locked() {
  if (g_n == 0) {
    const unsigned hc = std::thread::hardware_concurrency();
    g_n = hc ? static_cast<int>(hc) : 1;
  }
  return g_n;
}

}  // namespace

int threads() {
  std::lock_guard<std::mutex> g(g_mu);
  return resolve_locked();
}

void set_threads(int n) {
  std::lock_guard<std::mutex> g(g_mu);
  g_n = n < 1 ? 1 : n;
  g_workers.reset();
}

void for_ranges(std::size_t n, const std::function<void(std::size_t, std::size_t)>& fn) {
  if (n == 0) return;
  int nt;
  Workers* w = nullptr;
  {
    std::lock_guard<std::mutex> g(g_mu);
    nt = resolve_locked();
    if (nt > 1 && n > 1 && !g_inside) {
      if (!g_workers) g_workers = std::make_unique<Workers>(nt - 1);
      w = g_workers.get();
    }
  }
  if (!w) {
    fn(0, n);
    return;
  }
  const std::size_t chunk = (n + static_cast<std::size_t>(nt) - 1) / static_cast<std::size_t>(nt);
  w->run([&](int k) {
    const std::size_t b = static_cast<std::size_t>(k) * chunk;
    const std::size_t e = b + chunk < n ? b + chunk : n;
    if (b >= e) return;
    g_inside = true;
    fn(b, e);
    g_inside = false;
  });
}

}  // namespace parallel
}  // namespace msot
