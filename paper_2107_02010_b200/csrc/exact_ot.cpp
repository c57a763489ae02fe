// exact_ot.cpp — the exact transport oracle of SPEC.md:469-510 (module
// exact_oracle): min sum_ij pi_ij C_ij subject to
// pi 1 = a, pi^T 1 = b, pi >= 0 (§2 Eq. (1)), solved by a primal
// network simplex on the complete bipartite graph sources -> sinks.
//
// It is a small-instance ground truth (N*M <= 1e6; the acceptance fixtures
// are 32..256 atoms), single-threaded host code by specification
// — not part of the GPU path.  Design:
//   * nodes 0..n-1 sources (supply a_i), n..n+m-1 sinks (demand b_j), an
//     artificial root n+m; the starting basis is the star of artificial arcs
//     (cost A = (n+m) * (max C + 1)), oriented so that every zero-flow tree
//     arc points away from the root (a strongly feasible basis);
//   * entering arc: block pricing (most negative reduced cost in a block of
//     ~sqrt(|arcs|) arcs, wrapping around);
//   * leaving arc: the LAST blocking arc met when walking the pivot cycle in
//     its orientation from the apex (Cunningham's rule — keeps the basis
//     strongly feasible, so degenerate pivots cannot cycle);
//   * the tree is kept as parent / parent-arc / depth arrays; after a pivot
//     the cut-off subtree is re-hung from the entering arc and its
//     potentials and depths are recomputed by a walk over tree adjacency.
// The value is summed in fixed (row-major) order with pairwise summation.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/msot_gpu.h"

namespace {

struct NetworkSimplex {
  int n, m, nodes, root;
  int64_t n_real;                 // real arcs: i * m + j  (source i -> sink n + j)
  const double* cost;             // n x m
  double art_cost;
  // arcs: [0, n_real) real, then one artificial arc per non-root node
  std::vector<int> src, dst;      // artificial arcs only (real ones are implicit)
  std::vector<double> flow;       // all arcs
  std::vector<int> parent, parc, depth;
  std::vector<double> pi;
  std::vector<std::vector<int>> adj;  // tree arcs per node
  std::vector<char> in_tree;

  int tail(int64_t e) const {
    return e < n_real ? static_cast<int>(e / m) : src[e - n_real];
  }
  int head(int64_t e) const {
    return e < n_real ? n + static_cast<int>(e % m) : dst[e - n_real];
  }
  double c(int64_t e) const { return e < n_real ? cost[e] : art_cost; }
  double rc(int64_t e) const { return c(e) + pi[tail(e)] - pi[head(e)]; }

  void adj_remove(int u, int e) {
    auto& v = adj[u];
    for (size_t k = 0; k < v.size(); ++k)
      if (v[k] == e) {
        v[k] = v.back();
        v.pop_back();
        return;
      }
  }

  // Re-hang the subtree reached from `start` (new parent `par` over arc `pe`),
  // recomputing parent, depth and potentials.
  void rehang(int start, int par, int pe) {
    std::vector<int> stack{start};
    parent[start] = par;
    parc[start] = pe;
    while (!stack.empty()) {
      const int x = stack.back();
      stack.pop_back();
      const int p = parent[x];
      const int e = parc[x];
      depth[x] = depth[p] + 1;
      // tree arc rc = 0: c + pi[tail] - pi[head] = 0
      pi[x] = (tail(e) == p) ? pi[p] + c(e) : pi[p] - c(e);
      for (int f : adj[x]) {
        if (f == e) continue;
        const int y = tail(f) == x ? head(f) : tail(f);
        parent[y] = x;
        parc[y] = f;
        stack.push_back(y);
      }
    }
  }

  NetworkSimplex(int n_, int m_, const double* C, const double* a, const double* b)
      : n(n_), m(m_), nodes(n_ + m_ + 1), root(n_ + m_), n_real(int64_t(n_) * m_), cost(C) {
    double cmax = 0.0;
    for (int64_t e = 0; e < n_real; ++e) cmax = std::max(cmax, std::fabs(C[e]));
    art_cost = (cmax + 1.0) * static_cast<double>(n + m);
    const int n_art = n + m;
    src.resize(n_art);
    dst.resize(n_art);
    flow.assign(n_real + n_art, 0.0);
    parent.assign(nodes, -1);
    parc.assign(nodes, -1);
    depth.assign(nodes, 0);
    pi.assign(nodes, 0.0);
    adj.assign(nodes, {});
    in_tree.assign(n_real + n_art, 0);
    for (int v = 0; v < n + m; ++v) {
      const int e = static_cast<int>(n_real) + v;
      const double supply = v < n ? a[v] : -b[v - n];
      if (supply > 0) {  // v -> root carries the supply
        src[v] = v;
        dst[v] = root;
        flow[e] = supply;
        pi[v] = -art_cost;
      } else {  // root -> v: demand, or zero flow pointing away from the root
        src[v] = root;
        dst[v] = v;
        flow[e] = -supply;
        pi[v] = art_cost;
      }
      parent[v] = root;
      parc[v] = e;
      depth[v] = 1;
      in_tree[e] = 1;
      adj[v].push_back(e);
      adj[root].push_back(e);
    }
  }

  void pivot(int64_t ent) {
    const int u = tail(ent), v = head(ent);
    // apex
    int x = u, y = v;
    while (depth[x] > depth[y]) x = parent[x];
    while (depth[y] > depth[x]) y = parent[y];
    while (x != y) {
      x = parent[x];
      y = parent[y];
    }
    const int apex = x;
    // cycle in orientation: apex -> ... -> u, ent, v -> ... -> apex.
    // u side: walk u -> apex, collect, then visit reversed.
    std::vector<int> uside;
    for (int w = u; w != apex; w = parent[w]) uside.push_back(w);
    double delta = std::numeric_limits<double>::infinity();
    int leave_node = -1;  // child endpoint of the leaving tree arc
    bool leave_on_u = false;
    for (auto it = uside.rbegin(); it != uside.rend(); ++it) {
      const int w = *it;  // arc parent[w] -- w traversed parent -> w
      const int e = parc[w];
      if (tail(e) == w) {  // oriented w -> parent: decreases
        if (flow[e] <= delta) {
          delta = flow[e];
          leave_node = w;
          leave_on_u = true;
        }
      }
    }
    for (int w = v; w != apex; w = parent[w]) {  // traversed w -> parent
      const int e = parc[w];
      if (head(e) == w) {  // oriented parent -> w: decreases
        if (flow[e] <= delta) {
          delta = flow[e];
          leave_node = w;
          leave_on_u = false;
        }
      }
    }
    if (leave_node < 0) throw std::runtime_error("exact_ot: unbounded pivot");
    // flow update
    if (delta > 0) {
      for (int w : uside) {
        const int e = parc[w];
        flow[e] += (tail(e) == w) ? -delta : delta;
      }
      for (int w = v; w != apex; w = parent[w]) {
        const int e = parc[w];
        flow[e] += (head(e) == w) ? -delta : delta;
      }
    }
    flow[ent] = delta;
    // swap arcs in the tree
    const int le = parc[leave_node];
    const int lp = parent[leave_node];
    in_tree[le] = 0;
    adj_remove(leave_node, le);
    adj_remove(lp, le);
    in_tree[ent] = 1;
    adj[u].push_back(static_cast<int>(ent));
    adj[v].push_back(static_cast<int>(ent));
    // the entering endpoint inside the cut-off subtree is re-hung below the other
    if (leave_on_u)
      rehang(u, v, static_cast<int>(ent));
    else
      rehang(v, u, static_cast<int>(ent));
  }

  void solve(int64_t max_pivots) {
    const int64_t n_arcs = n_real;  // artificial arcs never re-enter
    const int64_t block = std::max<int64_t>(
        std::min<int64_t>(n_arcs, 10), static_cast<int64_t>(std::sqrt(double(n_arcs))));
    // potentials are sums along tree paths of magnitude up to art_cost
    const double tol = -1e-12 * art_cost;
    int64_t next = 0, pivots = 0;
    for (;;) {
      int64_t best = -1;
      double best_rc = tol;
      int64_t scanned = 0, in_block = 0;
      while (scanned < n_arcs) {
        const int64_t e = next;
        next = next + 1 == n_arcs ? 0 : next + 1;
        ++scanned;
        ++in_block;
        if (!in_tree[e]) {
          const double r = rc(e);
          if (r < best_rc) {
            best_rc = r;
            best = e;
          }
        }
        if (in_block == block) {
          if (best >= 0) break;
          in_block = 0;
        }
      }
      if (best < 0) return;
      if (++pivots > max_pivots) throw std::runtime_error("exact_ot: pivot limit exceeded");
      pivot(best);
    }
  }
};

double pairwise(const double* v, int64_t k) {
  if (k <= 8) {
    double s = 0.0;
    for (int64_t i = 0; i < k; ++i) s += v[i];
    return s;
  }
  const int64_t h = k / 2;
  return pairwise(v, h) + pairwise(v + h, k - h);
}

}  // namespace

namespace msot_host {
void set_last_error(const std::string& m);  // solver.cu
}

extern "C" int msot_exact_ot(const double* x, const double* a, int64_t n, const double* y,
                             const double* b, int64_t m, int d, double p, double* plan,
                             double* value) {
  try {
    if (!x || !a || !y || !b || !value || n < 1 || m < 1 || d < 1) {
      msot_host::set_last_error("exact_ot: invalid arguments");
      return MSOT_EUSAGE;
    }
    if (!(p >= 1.0 && p <= 2.0)) {
      msot_host::set_last_error("exact_ot: p outside [1, 2]");
      return MSOT_EDATA;
    }
    if (static_cast<double>(n) * static_cast<double>(m) > 1e6) {
      msot_host::set_last_error("exact_ot: N*M exceeds 1e6");
      return MSOT_EDATA;
    }
    double sa = 0.0, sb = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      if (!(a[i] >= 0.0) || !std::isfinite(a[i])) {
        msot_host::set_last_error("exact_ot: negative or non-finite weight");
        return MSOT_EDATA;
      }
      sa += a[i];
    }
    for (int64_t j = 0; j < m; ++j) {
      if (!(b[j] >= 0.0) || !std::isfinite(b[j])) {
        msot_host::set_last_error("exact_ot: negative or non-finite weight");
        return MSOT_EDATA;
      }
      sb += b[j];
    }
    if (std::fabs(sa - sb) > 1e-9) {
      msot_host::set_last_error("exact_ot: unbalanced masses");
      return MSOT_EDATA;
    }
    std::vector<double> C(static_cast<size_t>(n * m));
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < m; ++j) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
          const double t = x[i * d + k] - y[j * d + k];
          s += t * t;
        }
        C[i * m + j] = p == 2.0 ? 0.5 * s : std::pow(std::sqrt(s), p) / p;
      }
    NetworkSimplex ns(static_cast<int>(n), static_cast<int>(m), C.data(), a, b);
    ns.solve(int64_t(200) * (n + m) * (n + m) + 100000);
    std::vector<double> terms(static_cast<size_t>(n * m));
    for (int64_t e = 0; e < n * m; ++e) terms[e] = ns.flow[e] * C[e];
    *value = pairwise(terms.data(), n * m);
    if (plan) std::memcpy(plan, ns.flow.data(), sizeof(double) * n * m);
    return MSOT_OK;
  } catch (const std::exception& e) {
    msot_host::set_last_error(e.what());
    return MSOT_ENUMERIC;
  }
}
