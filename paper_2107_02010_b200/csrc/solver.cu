// solver.cu — host orchestration of the B200 solve and the C ABI
// (include/msot_gpu.h).
//
// One msot_ctx = one GPU (+ optional NCCL communicator; one process per GPU).
// A solve runs entirely on the device: inputs are copied once, clustered and
// sorted on the GPU, and every scale of the schedule is one launch group
//   softmin (all four updates of PAPER.md:258-290) -> finalize -> fallback
// followed, when world > 1, by an NCCL all-gather of the N+M updated
// potentials.  The host only walks the schedule scalars and
// synchronises a handful of times per solve (bounding box, cluster counts,
// mask sizes, final loss).
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/msot_gpu.h"
#include "policy.h"
#include "prims.cuh"

namespace msot_dev {
thread_local int64_t g_launches = 0;
thread_local int64_t g_host_syncs = 0;  // host waits on the device (stats.host_syncs)
}

using namespace msot_dev;

namespace {

thread_local std::string g_err;

struct Err {
  int code;
  std::string msg;
};

[[noreturn]] void raise(int code, const std::string& m) { throw Err{code, m}; }

#define CK(call)                                                                    \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess) raise(MSOT_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define NK(call)                                                                    \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess) raise(MSOT_ECUDA, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// Host waits on the device (stats.host_syncs); MSOT_DEBUG_SYNCS=1 prints the
// call sites per solve.
thread_local std::map<int, int> g_sync_sites;
cudaError_t host_sync(int line, cudaStream_t st) {
  ++g_host_syncs;
  static const bool dbg = getenv("MSOT_DEBUG_SYNCS") != nullptr;
  if (dbg) ++g_sync_sites[line];
  return cudaStreamSynchronize(st);
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return MSOT_OK;
  } catch (const Err& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MSOT_ECUDA;
  }
}

}  // namespace

// Shared with the host-only entry points of other translation units
// (exact_ot.cpp) so that msot_last_error() reports their failures too.
namespace msot_host {
void set_last_error(const std::string& m) { g_err = m; }
}  // namespace msot_host

namespace {

}  // namespace

struct msot_ctx {
  int device = 0, rank = 0, world = 1, n_sm = 148;
  cudaStream_t st = nullptr;
  // batched evaluate-once updates: consecutive colpart batches alternate
  // between two side streams so a batch's tail, row reduction and column sums
  // overlap the next batch's softmin (run_group_sym)
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_cs[2] = {nullptr, nullptr};
  ncclComm_t comm = nullptr;
  // test seam (msot_create_dist_host): host-staged collectives instead of NCCL
  msot_host_allreduce_fn host_ar = nullptr;
  msot_host_broadcast_fn host_bc = nullptr;
  void* host_user = nullptr;
  bool profiling = false;
  // barycenter (msot_barycenter): common schedule diameter (> 0: override) and
  // the x-x self term shared by every target: mode 1 = this solve records its
  // final a_xx and self-plan payload (caller order), mode 2 = this solve
  // skips the x-x problem and uses them
  double diam_override = 0.0;
  int self_mode = 0;
  float* self_axx = nullptr;    // [n] caller order
  float4* self_pay = nullptr;   // [n] caller order
  // parity seam (msot_debug_capture): the four potentials before and after
  // the update of scale `cap_scale`, in the caller's order (host buffers)
  // evaluate-once column partials: slots held per batch (0 = automatic,
  // kColpartPerAtom x (rows + cols) of the group; MSOT_COLPART_BUDGET overrides)
  int64_t colpart_budget = 0;
  int32_t force_fb = 0;  // tests: MSOT_FORCE_FALLBACK=1 sends every row to the exact path
  int64_t solve_atoms = 0;  // N + M of the running solve (automatic colpart budget)
  int cap_scale = -1;
  double* cap_in[4] = {nullptr, nullptr, nullptr, nullptr};
  double* cap_out[4] = {nullptr, nullptr, nullptr, nullptr};
  std::vector<uint8_t> cap_mask[3];     // xx, yy, xy cluster masks of that update
  int32_t cap_k[3][2] = {{0, 0}, {0, 0}, {0, 0}};
  std::vector<int32_t> cap_lab[2];      // cluster of every atom of x / y (caller order)
  std::map<std::string, std::pair<void*, size_t>> bufs;
  // pinned host staging for device -> host reads: copies of one planning
  // step land here asynchronously and are waited for with ONE sync
  // (pageable D2H copies are synchronous)
  char* pin_base = nullptr;
  size_t pin_cap = 0, pin_off = 0;
  void pin_reserve(size_t bytes) {  // call between sync points only
    pin_off = 0;
    if (bytes <= pin_cap) return;
    if (pin_base) cudaFreeHost(pin_base);
    pin_cap = std::max(bytes, size_t(1) << 20);
    if (cudaMallocHost(reinterpret_cast<void**>(&pin_base), pin_cap) != cudaSuccess) {
      pin_base = nullptr;
      pin_cap = 0;
      throw std::runtime_error("cudaMallocHost failed");
    }
  }
  template <class T>
  T* pin(size_t count) {
    const size_t a = (pin_off + 15) & ~size_t(15), b = a + std::max<size_t>(count, 1) * sizeof(T);
    if (b > pin_cap) throw std::runtime_error("pinned staging overflow (pin_reserve too small)");
    pin_off = b;
    return reinterpret_cast<T*>(pin_base + a);
  }
  std::vector<cudaEvent_t> ev;  // profiling events (pairs)
  size_t ev_used = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;

  template <class T>
  T* buf(const std::string& name, size_t count, bool headroom = true) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    auto it = bufs.find(name);
    if (it != bufs.end() && it->second.second >= bytes) return static_cast<T*>(it->second.first);
    size_t alloc = bytes;
    if (it != bufs.end()) {  // regrown buffer (sizes vary per rebuild): keep headroom
      alloc = headroom ? bytes + bytes / 2 : bytes;
      CK(host_sync(__LINE__, st));
      CK(cudaFree(it->second.first));
      bufs.erase(it);
    }
    void* p = nullptr;
    CK(cudaMalloc(&p, alloc));
    bufs[name] = {p, alloc};
    return static_cast<T*>(p);
  }
  // phase marks (profiling only): time from a mark to the next is charged to
  // the mark's phase (stats.phase_ms, see include/msot_gpu.h)
  std::vector<std::pair<int, cudaEvent_t>> marks;
  std::vector<cudaEvent_t> mark_pool;
  // NVTX ranges per phase (host timeline of nsys / ncu --nvtx; no-ops without
  // a tool attached): the open range is closed at the next mark, -1 ends
  bool nvtx_open = false;
  void mark(int phase) {
    static const char* const kNames[8] = {"msot:setup", "msot:coarse", "msot:transfer",
                                          "msot:masks", "msot:updates", "msot:loss",
                                          "msot:labels", "msot:phase7"};
    if (nvtx_open) nvtxRangePop();
    nvtx_open = phase >= 0 && phase < 8;
    if (nvtx_open) nvtxRangePushA(kNames[phase]);
    if (!profiling) return;
    if (mark_pool.size() <= marks.size()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      mark_pool.push_back(e);
    }
    cudaEvent_t e = mark_pool[marks.size()];
    CK(cudaEventRecord(e, st));
    marks.push_back({phase, e});
  }
  void ev_pair(cudaEvent_t* a, cudaEvent_t* b) {
    while (ev.size() < ev_used + 2) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      ev.push_back(e);
    }
    *a = ev[ev_used];
    *b = ev[ev_used + 1];
    ev_used += 2;
  }
};

namespace {

// Column-partial slots per row + column of an evaluate-once group (the
// bounded colpart buffer): 6 floats = 24 B per atom and per 4
// feature dimensions (the input itself is 8 D bytes per atom), plus at most
// as much again for the batches' row partials.
constexpr int64_t kColpartPerAtom = 6;

// ------------------------------------------------------------- collectives
// The two exchange steps of a sharded scale: a float64 all-reduce of
// the column sums and a broadcast of every rank's row shard.  NCCL over
// NVLink in the product; host-staged caller callbacks in the test seam.
// A communicator of one rank (msot_create_dist with world = 1) runs the NCCL
// calls too: they are no-ops on the data, but the product's NCCL path is
// exercised on a one-GPU box (tests/test_dist_gpu.py).
// float64 sum over ranks.  NCCL: ncclDouble all-reduce.  Host seam: each
// rank's vector travels through the broadcast callback as raw 32-bit words
// (bit-preserving), and every rank adds them in rank order.
void coll_allreduce64(msot_ctx* c, double* const* bufs, const int64_t* counts, int nb) {
  if (!c->comm && (c->world <= 1 || !c->host_bc)) return;
  cudaStream_t st = c->st;
  if (!c->comm) {
    for (int b = 0; b < nb; ++b) {
      const int64_t n = counts[b];
      std::vector<double> mine(n), part(n), sum(n, 0.0);
      CK(cudaMemcpyAsync(mine.data(), bufs[b], n * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(host_sync(__LINE__, st));
      for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) part = mine;
        if (n > 0 && c->host_bc(reinterpret_cast<float*>(part.data()), 2 * n, r, c->host_user) != 0)
          raise(MSOT_ECUDA, "host broadcast failed");
        for (int64_t j = 0; j < n; ++j) sum[j] += part[j];
      }
      CK(cudaMemcpyAsync(bufs[b], sum.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
      CK(host_sync(__LINE__, st));
    }
    return;
  }
  NK(ncclGroupStart());
  for (int b = 0; b < nb; ++b)
    NK(ncclAllReduce(bufs[b], bufs[b], counts[b], ncclDouble, ncclSum, c->comm, st));
  NK(ncclGroupEnd());
}

void coll_bcast_rows(msot_ctx* c, float* const* bufs, const std::vector<int64_t>* bounds, int nb) {
  if (!c->comm && (c->world <= 1 || !c->host_bc)) return;
  cudaStream_t st = c->st;
  if (!c->comm) {
    for (int b = 0; b < nb; ++b)
      for (int r = 0; r < c->world; ++r) {
        const int64_t b0 = bounds[b][r], b1 = bounds[b][r + 1];
        if (b1 <= b0) continue;
        std::vector<float> h(b1 - b0);
        CK(cudaMemcpyAsync(h.data(), bufs[b] + b0, (b1 - b0) * sizeof(float),
                           cudaMemcpyDeviceToHost, st));
        CK(host_sync(__LINE__, st));
        if (c->host_bc(h.data(), b1 - b0, r, c->host_user) != 0) raise(MSOT_ECUDA, "host broadcast failed");
        CK(cudaMemcpyAsync(bufs[b] + b0, h.data(), (b1 - b0) * sizeof(float),
                           cudaMemcpyHostToDevice, st));
        CK(host_sync(__LINE__, st));
      }
    return;
  }
  NK(ncclGroupStart());
  for (int b = 0; b < nb; ++b)
    for (int r = 0; r < c->world; ++r) {
      const int64_t b0 = bounds[b][r], b1 = bounds[b][r + 1];
      if (b1 > b0) NK(ncclBroadcast(bufs[b] + b0, bufs[b] + b0, b1 - b0, ncclFloat, r, c->comm, st));
    }
  NK(ncclGroupEnd());
}

// ---------------------------------------------------------------- measures
struct DMeasure {
  int64_t n = 0;
  int32_t k = 0;
  float4* pts = nullptr;   // sorted, centred float32 atoms
  float* lw2 = nullptr;    // log2 weights
  double* w64 = nullptr;   // float64 weights (sorted)
  int32_t* perm = nullptr; // sorted -> caller index
  int32_t* labels = nullptr;
  int32_t* offsets = nullptr;
  float4* cpts = nullptr;  // coarse measure (voxel centroids)
  float* clw2 = nullptr;
  double* cw64 = nullptr;
  float* radii = nullptr;
  float4* box_lo = nullptr;  // member boxes (truncation box bound, mask.cu)
  float4* box_hi = nullptr;
  std::vector<float> radii_h;
  std::vector<int32_t> offsets_h;  // cluster offsets (host copy, K+1)
  bool uniform = false;            // all weights equal
};

// Sort, gather and cluster several measures with two host waits in total:
// the cluster counts (and the uniform-weight flags), then the radii and
// offsets.
struct MeasureJob {
  std::string tag;
  const double* x;
  const double* w;
  int64_t n;
  DMeasure* M;
};
void prepare_measures(msot_ctx* c, const std::vector<MeasureJob>& jobs, int d, const GridSpec& g,
                      bool clusters) {
  cudaStream_t st = c->st;
  c->pin_reserve(jobs.size() * 64);
  std::vector<int32_t*> h(jobs.size());
  for (size_t q = 0; q < jobs.size(); ++q) {
    const MeasureJob& J = jobs[q];
    DMeasure& M = *J.M;
    const std::string& tag = J.tag;
    const int64_t n = J.n;
    M.n = n;
    uint32_t* keys = c->buf<uint32_t>(tag + ".keys", n);
    M.perm = c->buf<int32_t>(tag + ".perm", n);
    CK(cube_keys(J.x, n, g, keys, M.perm, st));
    void* tmp = c->buf<char>(tag + ".rstmp", radix_temp_bytes(n));
    const int bits = g.d == 1 ? MSOT_MORTON_BITS : g.d == 2 ? 2 * MSOT_MORTON_BITS : 3 * MSOT_MORTON_BITS;
    CK(radix_sort_pairs(keys, M.perm, n, bits, tmp, st));
    M.pts = c->buf<float4>(tag + ".pts", n);
    M.lw2 = c->buf<float>(tag + ".lw2", n);
    M.w64 = c->buf<double>(tag + ".w64", n);
    int32_t* nonuni = c->buf<int32_t>(tag + ".nonuni", 1);
    CK(cudaMemsetAsync(nonuni, 0, sizeof(int32_t), st));
    CK(gather_points(J.x, J.w, n, d, g, M.perm, M.pts, M.lw2, M.w64, nonuni, st));
    h[q] = c->pin<int32_t>(2);
    h[q][1] = 0;
    CK(cudaMemcpyAsync(&h[q][0], nonuni, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    if (!clusters) continue;
    uint8_t* flags = c->buf<uint8_t>(tag + ".flags", n);
    M.labels = c->buf<int32_t>(tag + ".labels", n);
    M.offsets = c->buf<int32_t>(tag + ".offsets", n + 1);
    int32_t* stmp = c->buf<int32_t>(tag + ".stmp", scan_temp_elems(n));
    int32_t* kdev = c->buf<int32_t>(tag + ".k", 1);
    CK(segment_flags(keys, n, flags, st));
    CK((scan<uint8_t, int32_t>(flags, M.labels, n, true, stmp, kdev, st)));
    CK(segment_offsets(M.labels, flags, n, M.offsets, st));
    CK(cudaMemcpyAsync(&h[q][1], kdev, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  CK(host_sync(__LINE__, st));
  for (size_t q = 0; q < jobs.size(); ++q) {
    jobs[q].M->uniform = h[q][0] == 0;
    jobs[q].M->k = h[q][1];
  }
  if (!clusters) return;
  size_t need = 0;
  for (const MeasureJob& J : jobs) need += (2 * static_cast<size_t>(J.M->k) + 1) * 4 + 64;
  c->pin_reserve(need);
  std::vector<float*> hr(jobs.size());
  std::vector<int32_t*> ho(jobs.size());
  for (size_t q = 0; q < jobs.size(); ++q) {
    DMeasure& M = *jobs[q].M;
    const std::string& tag = jobs[q].tag;
    const int32_t k = M.k;
    M.cpts = c->buf<float4>(tag + ".cpts", k);
    M.clw2 = c->buf<float>(tag + ".clw2", k);
    M.cw64 = c->buf<double>(tag + ".cw64", k);
    M.radii = c->buf<float>(tag + ".radii", k);
    M.box_lo = c->buf<float4>(tag + ".boxlo", k);
    M.box_hi = c->buf<float4>(tag + ".boxhi", k);
    CK(cluster_stats(M.pts, M.w64, M.offsets, k, d, M.cpts, M.clw2, M.cw64, M.radii, st, M.box_lo,
                     M.box_hi));
    hr[q] = c->pin<float>(k);
    ho[q] = c->pin<int32_t>(k + 1);
    CK(cudaMemcpyAsync(hr[q], M.radii, k * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(ho[q], M.offsets, (k + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  CK(host_sync(__LINE__, st));
  for (size_t q = 0; q < jobs.size(); ++q) {
    DMeasure& M = *jobs[q].M;
    M.radii_h.assign(hr[q], hr[q] + M.k);
    M.offsets_h.assign(ho[q], ho[q] + M.k + 1);
  }
}

void prepare_measure(msot_ctx* c, const std::string& tag, const double* d_x, const double* d_w,
                     int64_t n, int d, const GridSpec& g, bool clusters, DMeasure& M) {
  prepare_measures(c, {{tag, d_x, d_w, n, &M}}, d, g, clusters);
}

// Super level of the coarse phase (policy.h:msot_super_switch): consecutive
// clusters sharing a super-voxel key, with centroids / weights / radii from
// the cluster centroids weighted by the cluster masses.
struct SuperMeasure {
  int32_t k = 0;
  int32_t* labels = nullptr;  // cluster -> super cluster
  float4* cpts = nullptr;
  float* clw2 = nullptr;
};

void super_measures(msot_ctx* c, const DMeasure* const* Ms, const char* const* tags, int d,
                    SuperMeasure* const* Ss, int count) {
  cudaStream_t st = c->st;
  c->pin_reserve(64);
  int32_t* hk = c->pin<int32_t>(count);
  std::vector<int32_t*> offs(count);
  for (int q = 0; q < count; ++q) {
    const DMeasure& M = *Ms[q];
    SuperMeasure& S = *Ss[q];
    const std::string tag = tags[q];
    const int32_t k = M.k;
    uint32_t* keys = c->buf<uint32_t>(tag + ".skeys", k);
    CK(super_keys(c->buf<uint32_t>(tag + ".keys", M.n), M.offsets, k, d * MSOT_SUPER_SHIFT, keys, st));
    uint8_t* flags = c->buf<uint8_t>(tag + ".sflags", k);
    S.labels = c->buf<int32_t>(tag + ".slabels", k);
    offs[q] = c->buf<int32_t>(tag + ".soffsets", k + 1);
    int32_t* stmp = c->buf<int32_t>(tag + ".sstmp", scan_temp_elems(k));
    int32_t* kdev = c->buf<int32_t>(tag + ".sk", 1);
    CK(segment_flags(keys, k, flags, st));
    CK((scan<uint8_t, int32_t>(flags, S.labels, k, true, stmp, kdev, st)));
    CK(segment_offsets(S.labels, flags, k, offs[q], st));
    CK(cudaMemcpyAsync(&hk[q], kdev, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  CK(host_sync(__LINE__, st));
  for (int q = 0; q < count; ++q) {
    const DMeasure& M = *Ms[q];
    SuperMeasure& S = *Ss[q];
    const std::string tag = tags[q];
    S.k = hk[q];
    S.cpts = c->buf<float4>(tag + ".scpts", S.k);
    S.clw2 = c->buf<float>(tag + ".sclw2", S.k);
    double* cw = c->buf<double>(tag + ".scw64", S.k);
    float* rad = c->buf<float>(tag + ".srad", S.k);
    CK(cluster_stats(M.cpts, M.cw64, offs[q], S.k, d, S.cpts, S.clw2, cw, rad, st));
  }
}

// Occupied voxels of both clouds for a candidate edge (automatic edge rule),
// one host wait: max(k_x, k_y).
int64_t count_cells(msot_ctx* c, const double* d_x, int64_t n, const double* d_y, int64_t m,
                    const GridSpec& g) {
  cudaStream_t st = c->st;
  const int64_t nm = std::max(n, m);
  uint32_t* keys = c->buf<uint32_t>("cc.keys", nm);
  int32_t* vals = c->buf<int32_t>("cc.vals", nm);
  void* tmp = c->buf<char>("cc.rstmp", radix_temp_bytes(nm));
  uint8_t* flags = c->buf<uint8_t>("cc.flags", nm);
  int32_t* lab = c->buf<int32_t>("cc.lab", nm);
  int32_t* stmp = c->buf<int32_t>("cc.stmp", scan_temp_elems(nm));
  int32_t* kdev = c->buf<int32_t>("cc.k", 2);
  const int bits = g.d == 1 ? MSOT_MORTON_BITS : g.d == 2 ? 2 * MSOT_MORTON_BITS : 3 * MSOT_MORTON_BITS;
  const double* src[2] = {d_x, d_y};
  const int64_t len[2] = {n, m};
  for (int q = 0; q < 2; ++q) {  // same stream: the second cloud reuses the scratch
    CK(cube_keys(src[q], len[q], g, keys, vals, st));
    CK(radix_sort_pairs(keys, vals, len[q], bits, tmp, st));
    CK(segment_flags(keys, len[q], flags, st));
    CK((scan<uint8_t, int32_t>(flags, lab, len[q], true, stmp, kdev + q, st)));
  }
  c->pin_reserve(64);
  int32_t* hk = c->pin<int32_t>(2);
  CK(cudaMemcpyAsync(hk, kdev, 2 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(host_sync(__LINE__, st));
  return std::max(hk[0], hk[1]);
}

// ------------------------------------------------------------------ ranges
struct RangeSet {
  int tile_rows = kTileRows;            // rows per tile
  int64_t n_tiles = 0, n_ranges = 0;
  int32_t* tile_start = nullptr;        // device, n_tiles+1
  std::vector<int32_t> tile_start_h;
  int64_t* rptr = nullptr;
  int2* ranges = nullptr;
  int64_t* tile_cols = nullptr;
  std::vector<int64_t> tile_cols_h;
};

// Row tiles (policy.h:msot_pack_tiles): cluster-aligned when the rows carry
// cluster offsets, uniform otherwise.
void make_tiles(msot_ctx* c, const std::string& tag, int64_t rows,
                const std::vector<int32_t>* offsets, RangeSet& R) {
  const int64_t k = offsets ? static_cast<int64_t>(offsets->size()) - 1 : 0;
  std::vector<int64_t> ts(k + rows / R.tile_rows + 2);
  R.n_tiles = msot_row_tiles(offsets ? offsets->data() : nullptr, k, rows, R.tile_rows, ts.data());
  R.tile_start_h.assign(ts.begin(), ts.begin() + R.n_tiles + 1);
  R.tile_start = c->buf<int32_t>(tag + ".tstart", R.n_tiles + 1);
  // pageable host -> device: the driver stages the source before returning,
  // so the host vector may change afterwards without a wait
  CK(cudaMemcpyAsync(R.tile_start, R.tile_start_h.data(), (R.n_tiles + 1) * sizeof(int32_t),
                     cudaMemcpyHostToDevice, c->st));
}

void dense_rangeset(msot_ctx* c, const std::string& tag, int64_t rows, int64_t cols, RangeSet& R,
                    const std::vector<int32_t>* row_offsets = nullptr) {
  make_tiles(c, tag, rows, row_offsets, R);
  R.n_ranges = R.n_tiles;
  R.rptr = c->buf<int64_t>(tag + ".rptr", R.n_tiles + 1);
  R.ranges = c->buf<int2>(tag + ".ranges", R.n_tiles);
  R.tile_cols = c->buf<int64_t>(tag + ".tcols", R.n_tiles);
  CK(dense_ranges(R.n_tiles, static_cast<int32_t>(cols), R.rptr, R.ranges, R.tile_cols, c->st));
  R.tile_cols_h.assign(R.n_tiles, cols);
}

// rows with labels `rl` / cluster offsets (host) `ro`, column clusters with
// offsets `co` (ky)
void mask_rangeset(msot_ctx* c, const std::string& tag, const int32_t* rl,
                   const std::vector<int32_t>& ro, int64_t n_rows, const int32_t* co, int32_t ky,
                   const uint32_t* mask, RangeSet& R) {
  cudaStream_t st = c->st;
  if (R.tile_start_h.empty()) make_tiles(c, tag, n_rows, &ro, R);  // fixed per solve
  int64_t* nr = c->buf<int64_t>(tag + ".nr", R.n_tiles + 1);
  R.tile_cols = c->buf<int64_t>(tag + ".tcols", R.n_tiles);
  R.rptr = c->buf<int64_t>(tag + ".rptr", R.n_tiles + 1);
  int64_t* stmp = c->buf<int64_t>(tag + ".stmp", scan_temp_elems(R.n_tiles + 1));
  uint32_t* tbits = c->buf<uint32_t>(tag + ".tbits", size_t(R.n_tiles) * mask_words(ky));
  CK(tile_or(mask, ky, rl, R.tile_start, R.n_tiles, tbits, st));
  CK(tile_range_count(tbits, ky, R.n_tiles, co, nr, R.tile_cols, st));
  CK(cudaMemsetAsync(nr + R.n_tiles, 0, sizeof(int64_t), st));
  CK((scan<int64_t, int64_t>(nr, R.rptr, R.n_tiles + 1, false, stmp, nullptr, st)));
  CK(cudaMemcpyAsync(&R.n_ranges, R.rptr + R.n_tiles, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  R.tile_cols_h.resize(R.n_tiles);
  CK(cudaMemcpyAsync(R.tile_cols_h.data(), R.tile_cols, R.n_tiles * sizeof(int64_t),
                     cudaMemcpyDeviceToHost, st));
  CK(host_sync(__LINE__, st));
  R.ranges = c->buf<int2>(tag + ".ranges", R.n_ranges);
  CK(tile_range_write(tbits, ky, R.n_tiles, co, R.rptr, R.ranges, st));
}

// Pair sets of the evaluate-once softmin (mask.cu: sym_runs / sym_entries):
// the row tiles' column lists plus, per column cluster, the (tile, slot)
// entries its column sums are read from.
struct SymSet {
  RangeSet R;
  int self = 0;
  int64_t* tslot = nullptr;   // [T + 1] first colpart slot of each tile
  int64_t* ebase = nullptr;   // [K * kEntryChunks + 1]
  int64_t* eslot = nullptr;
  int32_t* etile = nullptr;
  std::vector<int64_t> tslot_h;  // host copy of tslot (batch bases)
  int64_t slots = 0, entries = 0;
  // sym_rangeset_a -> _b: device scratch and the pinned landing of the counts
  uint32_t* tbits = nullptr;
  int32_t* posword = nullptr;
  int64_t* h_tot = nullptr;   // pinned: ranges, slots, entries
  int64_t* h_tc = nullptr;    // pinned: tile_cols
  const int32_t* rl = nullptr;
  const int32_t* co = nullptr;
  int32_t ky = 0;
  bool dense = false;         // dense_symset: column sums by hd_colsum (no entries)
};

// Phase A: tile OR, per-tile range / slot / entry counts and their scans;
// the totals and per-tile column counts land in pinned memory (no wait).
void sym_rangeset_a(msot_ctx* c, const std::string& tag, const int32_t* rl,
                    const std::vector<int32_t>& ro, int64_t n_rows, const int32_t* co, int32_t ky,
                    const uint32_t* mask, int self, SymSet& S) {
  cudaStream_t st = c->st;
  RangeSet& R = S.R;
  S.self = self;
  S.rl = rl;
  S.co = co;
  S.ky = ky;
  if (R.tile_start_h.empty()) make_tiles(c, tag, n_rows, &ro, R);  // fixed per solve
  const int64_t T = R.n_tiles;
  const int32_t words = mask_words(ky);
  int64_t* nr = c->buf<int64_t>(tag + ".nr", T + 1);
  R.tile_cols = c->buf<int64_t>(tag + ".tcols", T + 1);
  R.rptr = c->buf<int64_t>(tag + ".rptr", T + 1);
  S.tslot = c->buf<int64_t>(tag + ".tslot", T + 1);
  int64_t* stmp = c->buf<int64_t>(tag + ".stmp", scan_temp_elems(T + 1));
  S.tbits = c->buf<uint32_t>(tag + ".tbits", size_t(T) * words);
  S.posword = c->buf<int32_t>(tag + ".posw", size_t(T) * words);
  CK(tile_or(mask, ky, rl, R.tile_start, T, S.tbits, st));
  CK(sym_ranges(S.tbits, ky, T, co, R.tile_start, rl, self, nr, R.tile_cols, S.posword, nullptr,
                nullptr, false, st));
  CK(cudaMemsetAsync(nr + T, 0, sizeof(int64_t), st));
  CK(cudaMemsetAsync(R.tile_cols + T, 0, sizeof(int64_t), st));
  CK((scan<int64_t, int64_t>(nr, R.rptr, T + 1, false, stmp, nullptr, st)));
  CK((scan<int64_t, int64_t>(R.tile_cols, S.tslot, T + 1, false, stmp, nullptr, st)));
  // (tile, cluster) entries, column-major
  const int64_t ne = static_cast<int64_t>(ky) * kEntryChunks;
  int32_t* ecnt = c->buf<int32_t>(tag + ".ecnt", ne + 1);
  S.ebase = c->buf<int64_t>(tag + ".ebase", ne + 1);
  int64_t* etmp = c->buf<int64_t>(tag + ".etmp", scan_temp_elems(ne + 1));
  CK(sym_entries(S.tbits, ky, T, co, R.tile_start, rl, self, S.posword, S.tslot, ecnt, nullptr,
                 nullptr, nullptr, false, st));
  CK(cudaMemsetAsync(ecnt + ne, 0, sizeof(int32_t), st));
  CK((scan<int32_t, int64_t>(ecnt, S.ebase, ne + 1, false, etmp, nullptr, st)));
  S.h_tot = c->pin<int64_t>(3);
  S.h_tc = c->pin<int64_t>(T);
  CK(cudaMemcpyAsync(&S.h_tot[0], R.rptr + T, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&S.h_tot[1], S.tslot + T, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&S.h_tot[2], S.ebase + ne, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(S.h_tc, R.tile_cols, T * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
}

// Phase B (after the caller's one sync): the ranges and the entries.
void sym_rangeset_b(msot_ctx* c, const std::string& tag, SymSet& S) {
  cudaStream_t st = c->st;
  RangeSet& R = S.R;
  const int64_t T = R.n_tiles;
  R.n_ranges = S.h_tot[0];
  S.slots = S.h_tot[1];
  S.entries = S.h_tot[2];
  R.tile_cols_h.assign(S.h_tc, S.h_tc + T);
  S.tslot_h.assign(T + 1, 0);
  for (int64_t t = 0; t < T; ++t) S.tslot_h[t + 1] = S.tslot_h[t] + R.tile_cols_h[t];
  R.ranges = c->buf<int2>(tag + ".ranges", R.n_ranges);
  CK(sym_ranges(S.tbits, S.ky, T, S.co, R.tile_start, S.rl, S.self, nullptr, nullptr, nullptr,
                R.rptr, R.ranges, true, st));
  S.eslot = c->buf<int64_t>(tag + ".eslot", S.entries);
  S.etile = c->buf<int32_t>(tag + ".etile", S.entries);
  CK(sym_entries(S.tbits, S.ky, T, S.co, R.tile_start, S.rl, S.self, S.posword, S.tslot, nullptr,
                 S.ebase, S.eslot, S.etile, true, st));
}

// The pair sets of several evaluate-once problems with one host wait.
struct SymJob {
  std::string tag;
  const int32_t* rl;
  const std::vector<int32_t>* ro;
  int64_t n_rows;
  const int32_t* co;
  int32_t ky;
  const uint32_t* mask;
  int self;
  SymSet* S;
};
void sym_rangesets(msot_ctx* c, const std::vector<SymJob>& jobs) {
  size_t need = 0;
  for (const SymJob& j : jobs) {  // tiles are fixed per solve: make them before reserving
    if (j.S->R.tile_start_h.empty()) make_tiles(c, j.tag, j.n_rows, j.ro, j.S->R);
    need += (j.S->R.n_tiles + 3) * sizeof(int64_t) + 64;
  }
  c->pin_reserve(need);
  for (const SymJob& j : jobs)
    sym_rangeset_a(c, j.tag, j.rl, *j.ro, j.n_rows, j.co, j.ky, j.mask, j.self, *j.S);
  CK(host_sync(__LINE__, c->st));
  for (const SymJob& j : jobs) sym_rangeset_b(c, j.tag, *j.S);
}

// Dense evaluate-once pair sets (high-D path): uniform 256-row tiles; self
// problems: tile t's list is [ts, n) (diagonal block, then the upper part
// whose columns also get tile t's rows); cross: [0, n_cols).
void dense_symset(msot_ctx* c, const std::string& tag, int64_t n_rows, int64_t n_cols, int self,
                  SymSet& S) {
  cudaStream_t st = c->st;
  RangeSet& R = S.R;
  S.self = self;
  S.dense = true;
  make_tiles(c, tag, n_rows, nullptr, R);
  const int64_t T = R.n_tiles;
  std::vector<int64_t> rptr(T + 1), tcols(T), tslot(T + 1, 0);
  std::vector<int2> rg(T);
  for (int64_t t = 0; t < T; ++t) {
    rptr[t] = t;
    const int32_t c0 = self ? R.tile_start_h[t] : 0;
    rg[t] = make_int2(c0, static_cast<int32_t>(n_cols));
    tcols[t] = n_cols - c0;
    tslot[t + 1] = tslot[t] + tcols[t];
  }
  rptr[T] = T;
  R.n_ranges = T;
  R.rptr = c->buf<int64_t>(tag + ".rptr", T + 1);
  R.ranges = c->buf<int2>(tag + ".ranges", T);
  R.tile_cols = c->buf<int64_t>(tag + ".tcols", T);
  S.tslot = c->buf<int64_t>(tag + ".tslot", T + 1);
  CK(cudaMemcpyAsync(R.rptr, rptr.data(), (T + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(R.ranges, rg.data(), T * sizeof(int2), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(R.tile_cols, tcols.data(), T * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(S.tslot, tslot.data(), (T + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  R.tile_cols_h = tcols;
  S.slots = tslot[T];
  S.tslot_h = tslot;  // (pageable H2D copies above are staged before they return)
}

// ------------------------------------------------------------ launch plans
struct HdOperands {  // high-dimensional path (softmin_hd.cu)
  const uint8_t* a_pack = nullptr;
  const uint8_t* b_pack = nullptr;
  const float* row_sq = nullptr;
  const float* col_sq = nullptr;
  const float* row_f = nullptr;
  const float* col_f = nullptr;
};

struct ProbSpec {
  const float4* rows;
  int64_t n_rows;
  const float4* cols;
  const float* col_lw2;
  int64_t n_cols;
  const RangeSet* rs;
  HdOperands hd{};
  const SymSet* sym = nullptr;   // evaluate-once groups
  const float* row_lw2 = nullptr;
};

struct Plan {
  int np = 0;
  bool skip_p0 = false;  // problem 0 (x-x) evaluated nowhere (shared self term)
  ProbSpec ps[kMaxProblems];
  int64_t t0[kMaxProblems], t1[kMaxProblems];
  std::vector<int64_t> row_bounds[kMaxProblems];  // world+1 row boundaries
  int32_t* ibase[kMaxProblems];
  int4* items = nullptr;
  int32_t n_items = 0;
  float* part = nullptr;
  // evaluate-once groups: the column partials (one float per (tile, column
  // list position)) are produced and reduced in batches of consecutive
  // tiles whose slots fit the context's colpart budget (memory linear in
  // N + M)
  struct Batch {
    int32_t i0 = 0, i1 = 0;                 // items [i0, i1)
    int32_t bt0[kMaxProblems] = {}, bt1[kMaxProblems] = {};  // tiles of each problem
    int64_t off[kMaxProblems] = {};         // colpart offset of each problem's first slot
  };
  std::vector<Batch> batches;
  float* colbuf = nullptr;
  int64_t batch_slots = 0, batch_items = 0;  // largest batch
  double pairs_local = 0.0, pairs_all = 0.0;
  double terms_all = 0.0;  // LSE terms summed: an evaluate-once pair feeds a row and a column
};

// Contiguous tile shards balanced on work (shared with msot_shard_tiles).
void shard_tiles(const std::vector<double>& work, int world, std::vector<int64_t>& b) {
  const int64_t nt = static_cast<int64_t>(work.size());
  b.assign(world + 1, nt);
  b[0] = 0;
  double tot = 0.0;
  for (double w : work) tot += w;
  double acc = 0.0;
  int64_t t = 0;
  for (int r = 1; r < world; ++r) {
    const double target = tot * r / world;
    while (t < nt && acc + 0.5 * work[t] < target) acc += work[t++];
    b[r] = t;
  }
}

void build_plan(msot_ctx* c, const std::string& tag, Plan& P, int waves = 32, int dim = 3) {
  cudaStream_t st = c->st;
  // per-problem shard of row tiles, weighted by evaluated pairs
  // tot_cols_all: the group's columns over every rank's tiles — item and
  // batch sizing depend on it, not on this rank's share, so the items (and
  // the row sums' additions) are the same for any number of GPUs
  int64_t tot_tiles = 0, tot_cols_all = 0;
  P.pairs_all = P.pairs_local = P.terms_all = 0.0;
  for (int p = 0; p < P.np; ++p) {
    const RangeSet& R = *P.ps[p].rs;
    std::vector<double> work(R.n_tiles);
    for (int64_t t = 0; t < R.n_tiles; ++t) {
      const int64_t rows = R.tile_start_h[t + 1] - R.tile_start_h[t];
      work[t] = static_cast<double>(rows) * static_cast<double>(R.tile_cols_h[t]) + 1.0;
      P.pairs_all += static_cast<double>(rows) * static_cast<double>(R.tile_cols_h[t]);
      const SymSet* sy = P.ps[p].sym;
      P.terms_all += static_cast<double>(rows) *
                     (sy ? 2.0 * static_cast<double>(R.tile_cols_h[t]) - (sy->self ? rows : 0)
                         : static_cast<double>(R.tile_cols_h[t]));
    }
    std::vector<int64_t> tb;
    shard_tiles(work, c->world, tb);
    if (p == 0 && P.skip_p0) tb.assign(c->world + 1, 0);
    for (int64_t t = tb[0]; t < tb[c->world]; ++t) tot_cols_all += R.tile_cols_h[t];
    P.t0[p] = tb[c->rank];
    P.t1[p] = tb[c->rank + 1];
    P.row_bounds[p].resize(c->world + 1);
    for (int r = 0; r <= c->world; ++r) P.row_bounds[p][r] = R.tile_start_h[tb[r]];
    tot_tiles += P.t1[p] - P.t0[p];
    for (int64_t t = P.t0[p]; t < P.t1[p]; ++t) {
      const int64_t rows = R.tile_start_h[t + 1] - R.tile_start_h[t];
      P.pairs_local += static_cast<double>(rows) * static_cast<double>(R.tile_cols_h[t]);
    }
  }
  // chunk size: small work items (~32 waves of resident CTAs, floor 2 column
  // tiles) keep the tail of every launch short — C3 fine phase 342 -> 314 ms
  // against ~2 waves (8: 321, 16: 315, 64: 315 ms); the high-D kernel keeps 2
  // (its CTAs walk block ranges; 32 cost config 4 ~1.5%)
  const int64_t target = static_cast<int64_t>(c->n_sm) * 12 * waves;
  int64_t chunk = std::max<int64_t>(2 * kColTile, (tot_cols_all + target - 1) / std::max<int64_t>(target, 1));
  chunk = (chunk + kColTile - 1) / kColTile * kColTile;
  if (P.ps[0].sym) {
    // colpart batches: consecutive (problem, tile) runs of at most `budget`
    // slots; each batch is cut into ~`waves` waves of items of its own
    int64_t rows_cols = 0, slots_all = tot_cols_all;  // every rank's slots
    for (int p = 0; p < P.np; ++p) rows_cols += P.ps[p].n_rows + P.ps[p].n_cols;
    // automatic budget: per atom of the group or of the whole solve, whichever
    // is larger (coarse-level groups are quadratic in the cluster count, far
    // below N + M: they keep one batch)
    const int64_t atoms = std::max<int64_t>(rows_cols, 3 * c->solve_atoms);
    const int64_t budget = c->colpart_budget > 0
                               ? c->colpart_budget
                               : std::max<int64_t>(int64_t(1) << 20,
                                                   kColpartPerAtom * atoms *
                                                       std::max(1, (dim + 3) / 4));
    // one batch when everything fits; otherwise two halves of the budget
    // (consecutive batches overlap on two streams).  The 3-D kernel's item
    // chunk does not depend on the batching (~32 waves per update; the row
    // sums then add the same partials in the same order for any budget).
    // The high-D kernel's items are coarse (~2 waves per update), so batched
    // high-D updates size their items for ~2 waves per batch instead (the
    // result then depends on the automatic budget, i.e. on N + M only).
    const int64_t lim = slots_all <= budget ? budget : std::max<int64_t>(1, budget / 2);
    if (slots_all > budget && waves <= 2) {
      chunk = std::max<int64_t>(2 * kColTile, (lim + target - 1) / std::max<int64_t>(target, 1));
      chunk = (chunk + kColTile - 1) / kColTile * kColTile;
    }
    P.batches.clear();
    Plan::Batch b;
    int64_t acc = 0, item = 0, held = 1;  // held: the largest batch (a lone tile may exceed budget)
    for (int p = 0; p < P.np; ++p) {
      b.bt0[p] = b.bt1[p] = static_cast<int32_t>(P.t0[p]);
      for (int64_t t = P.t0[p]; t < P.t1[p]; ++t) {
        const int64_t sl = P.ps[p].rs->tile_cols_h[t];
        if (acc > 0 && acc + sl > lim) {  // close the batch before tile (p, t)
          b.i1 = static_cast<int32_t>(item);
          P.batches.push_back(b);
          b = Plan::Batch{};
          b.i0 = static_cast<int32_t>(item);
          for (int q = 0; q < P.np; ++q) b.bt0[q] = b.bt1[q] = static_cast<int32_t>(q < p ? P.t1[q] : P.t0[q]);
          b.bt0[p] = b.bt1[p] = static_cast<int32_t>(t);
          acc = 0;
        }
        if (b.bt1[p] == b.bt0[p]) b.off[p] = acc;
        b.bt1[p] = static_cast<int32_t>(t + 1);
        acc += sl;
        held = std::max(held, acc);
        item += std::max<int64_t>(1, (sl + chunk - 1) / chunk);
      }
      if (p + 1 < P.np) b.bt0[p + 1] = b.bt1[p + 1] = static_cast<int32_t>(P.t0[p + 1]);
    }
    b.i1 = static_cast<int32_t>(item);
    P.batches.push_back(b);
    const size_t nbt = P.batches.size();
    // sized by the budget (not regrown per scale): 2 x lim >= 2 x held unless
    // one tile alone exceeds the half budget
    P.colbuf = c->buf<float>("sym.colpart", nbt > 1 ? std::max(budget, 2 * held) : held, false);
    P.batch_slots = held;
    P.batch_items = 0;
    for (const auto& bb : P.batches) P.batch_items = std::max<int64_t>(P.batch_items, bb.i1 - bb.i0);
  } else {
    P.batches.clear();
  }
  int32_t* cnt = c->buf<int32_t>(tag + ".icnt", tot_tiles + 1);
  int32_t* ib = c->buf<int32_t>(tag + ".ibase", tot_tiles + 1);
  int32_t* stmp = c->buf<int32_t>(tag + ".istmp", scan_temp_elems(tot_tiles + 1));
  int64_t off = 0;
  for (int p = 0; p < P.np; ++p) {
    const int64_t nt = P.t1[p] - P.t0[p];
    CK(item_counts(P.ps[p].rs->tile_cols + P.t0[p], nt, chunk, cnt + off, st));
    P.ibase[p] = ib + off - P.t0[p];
    off += nt;
  }
  CK(cudaMemsetAsync(cnt + off, 0, sizeof(int32_t), st));
  CK((scan<int32_t, int32_t>(cnt, ib, off + 1, false, stmp, nullptr, st)));
  // the item count follows from the host copy of the tile column counts
  // (item_counts_kernel's rule): no device read
  int64_t n_items = 0;
  for (int p = 0; p < P.np; ++p)
    for (int64_t t = P.t0[p]; t < P.t1[p]; ++t)
      n_items += std::max<int64_t>(1, (P.ps[p].rs->tile_cols_h[t] + chunk - 1) / chunk);
  if (n_items > 0x7fffffffLL) raise(MSOT_EUSAGE, "too many work items");
  P.n_items = static_cast<int32_t>(n_items);
  P.items = c->buf<int4>(tag + ".items", P.n_items);
  for (int p = 0; p < P.np; ++p)
    CK(item_write(P.ps[p].rs->tile_cols, P.t0[p], P.t1[p], chunk, P.ibase[p], p, P.items, st));
  if (P.batches.size() > 1)  // row partials of two in-flight batches (softmin_rowsum)
    P.part = c->buf<float>("sym.part", static_cast<size_t>(2 * P.batch_items) * kTileRows, false);
  else
    P.part = c->buf<float>(tag + ".part", static_cast<size_t>(P.n_items) * kTileRows);
}

struct ScaleArgs {
  const float* h[kMaxProblems];    // column potentials
  const float* est[kMaxProblems];  // expansion reference of the output
  float* out[kMaxProblems];
  double eps, lam, mixw;
};

struct SolveState {
  msot_stats* S;
  int d;
  int32_t* fb_count;
  int32_t* fb_total;
  int4* fb_list;
  int32_t fb_cap;
  int32_t* bad_scale = nullptr;  // device: first scale with a non-finite potential
  int scale = 0;                 // scale index of the next launch group
};

void run_group(msot_ctx* c, const Plan& P, const ScaleArgs& a, SolveState& ss) {
  cudaStream_t st = c->st;
  Group G{};
  const double ln2 = 0.69314718055994530942;
  int32_t tiles_acc = 0;
  G.tile_prefix[0] = 0;
  for (int p = 0; p < P.np; ++p) {
    Problem& Q = G.P[p];
    const ProbSpec& S = P.ps[p];
    Q.rows = S.rows;
    Q.row_est = a.est[p];
    Q.row_out = a.out[p];
    Q.cols = S.cols;
    Q.col_lw2 = S.col_lw2;
    Q.col_h = a.h[p];
    Q.a_pack = S.hd.a_pack;
    Q.b_pack = S.hd.b_pack;
    Q.row_sq = S.hd.row_sq;
    Q.col_sq = S.hd.col_sq;
    Q.row_f = S.hd.row_f;
    Q.col_f = S.hd.col_f;
    Q.tile_start = S.rs->tile_start;
    Q.tile_rptr = S.rs->rptr;
    Q.ranges = S.rs->ranges;
    Q.tile_ibase = P.ibase[p];
    Q.n_rows = static_cast<int32_t>(S.n_rows);
    Q.n_cols = static_cast<int32_t>(S.n_cols);
    Q.sc = static_cast<float>(1.0 / std::sqrt(2.0 * a.eps * ln2));
    Q.inv_eps_ln2 = static_cast<float>(1.0 / (a.eps * ln2));
    Q.inv_lam_eps_ln2 = static_cast<float>(1.0 / (a.lam * a.eps * ln2));
    Q.lam_eps = static_cast<float>(a.lam * a.eps);
    Q.mixw = static_cast<float>(a.mixw);
    G.t0[p] = static_cast<int32_t>(P.t0[p]);
    tiles_acc += static_cast<int32_t>(P.t1[p] - P.t0[p]);
    G.tile_prefix[p + 1] = tiles_acc;
  }
  G.n_problems = P.np;
  G.items = P.items;
  G.n_items = P.n_items;
  G.part = P.part;
  G.fb_count = ss.fb_count;
  G.fb_total = ss.fb_total;
  G.fb_list = ss.fb_list;
  G.fb_cap = ss.fb_cap;
  G.bad_scale = ss.bad_scale;
  G.scale = ss.scale;
  G.force_fb = c->force_fb;
  CK(cudaMemsetAsync(ss.fb_count, 0, sizeof(int32_t), st));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->profiling) {
    c->ev_pair(&e0, &e1);
    CK(cudaEventRecord(e0, st));
  }
  const bool hd = ss.d > 3;
  if (hd)
    for (int p = 0; p < P.np; ++p) {
      float* cc = c->buf<float>("hd.c" + std::to_string(p), hd_padded(G.P[p].n_cols));
      CK(hd_colconst(G.P[p], cc, nullptr, st));
      G.P[p].col_c = cc;
    }
  CK(hd ? launch_softmin_hd(G, ss.d, c->n_sm, false, st) : launch_softmin(G, ss.d, st));
  if (c->profiling) CK(cudaEventRecord(e1, st));
  CK(launch_finalize(G, st));
  CK(hd ? launch_fallback_hd(G, ss.d, c->n_sm, st) : launch_fallback(G, ss.d, c->n_sm, st));
  ss.S->softmin_launches += 1;
  ss.S->pairs_evaluated += P.pairs_all;
  ss.S->pairs_terms += P.terms_all;
  // all-gather of the updated potentials (NCCL over NVLink)
  coll_bcast_rows(c, a.out, P.row_bounds, P.np);
}

// ------------------------------------------------------------------ solve
// Evaluate-once group (softmin_sym.cu): plan problems 0 = xx, 1 = yy (self,
// rows = cols) and 2 = yx (rows x, cols y); the column side of problem 2 is
// the a_xy update, described by problem 3 (rows y over cols x) which has no
// tiles of its own.  a.{h,est,out}[3] belong to that transposed problem.
struct SymCols {
  const int32_t* labels[3];  // column clusters of problems 0..2
  const int32_t* co[3];
  float* tot[3];             // column totals (x, y, y)
  const float4* yrows;       // problem 3: rows y over cols x
  const float4* xcols;
  const float* x_lw2;
  const float* y_lw2 = nullptr;  // weights of the transposed problem's rows (zero-weight skip)
  int64_t n, m;
  bool uniform;              // both measures have uniform weights
  HdOperands hd3{};          // high-D operands of problem 3 (rows y, cols x)
  // fine phase: cluster masks (xx, yy, xy) for the neighbourhood-restricted
  // exact fallback (softmin_fallback_dense); null in dense / coarse groups
  const uint32_t* mask[3] = {nullptr, nullptr, nullptr};
  const int32_t* rlab[4] = {nullptr, nullptr, nullptr, nullptr};  // row clusters per problem
  const int32_t* fco[4] = {nullptr, nullptr, nullptr, nullptr};   // column cluster offsets
  int32_t words[4] = {0, 0, 0, 0}, kc3 = 0;
};

void fill_problem(Problem& Q, const ProbSpec& S, const float* h, const float* est, float* out,
                  double eps, double lam, double mixw) {
  const double ln2 = 0.69314718055994530942;
  Q.rows = S.rows;
  Q.row_est = est;
  Q.row_out = out;
  Q.cols = S.cols;
  Q.col_lw2 = S.col_lw2;
  Q.col_h = h;
  Q.a_pack = S.hd.a_pack;
  Q.b_pack = S.hd.b_pack;
  Q.row_sq = S.hd.row_sq;
  Q.col_sq = S.hd.col_sq;
  Q.row_f = S.hd.row_f;
  Q.col_f = S.hd.col_f;
  if (S.rs) {
    Q.tile_start = S.rs->tile_start;
    Q.tile_rptr = S.rs->rptr;
    Q.ranges = S.rs->ranges;
  }
  Q.n_rows = static_cast<int32_t>(S.n_rows);
  Q.n_cols = static_cast<int32_t>(S.n_cols);
  Q.sc = static_cast<float>(1.0 / std::sqrt(2.0 * eps * ln2));
  Q.inv_eps_ln2 = static_cast<float>(1.0 / (eps * ln2));
  Q.inv_lam_eps_ln2 = static_cast<float>(1.0 / (lam * eps * ln2));
  Q.lam_eps = static_cast<float>(lam * eps);
  Q.mixw = static_cast<float>(mixw);
  Q.ell = static_cast<float>((1.0 / lam - 1.0) / (eps * ln2));
  Q.row_lw2 = S.row_lw2;
  if (S.sym) Q.tile_slot = S.sym->tslot;
}

void run_group_sym(msot_ctx* c, const Plan& P, const ScaleArgs& a, SolveState& ss,
                   const SymCols& X) {
  cudaStream_t st = c->st;
  Group G{};
  int32_t tiles_acc = 0;
  G.tile_prefix[0] = 0;
  for (int p = 0; p < 3; ++p) {
    Problem& Q = G.P[p];
    fill_problem(Q, P.ps[p], a.h[p], a.est[p], a.out[p], a.eps, a.lam, a.mixw);
    Q.tile_ibase = P.ibase[p];
    Q.row_add = p < 2 ? X.tot[p] : nullptr;
    G.t0[p] = static_cast<int32_t>(P.t0[p]);
    tiles_acc += static_cast<int32_t>(P.t1[p] - P.t0[p]);
    G.tile_prefix[p + 1] = tiles_acc;
  }
  {
    ProbSpec T{X.yrows, X.m, X.xcols, X.x_lw2, X.n, nullptr, X.hd3};
    T.row_lw2 = X.y_lw2;
    fill_problem(G.P[3], T, a.h[3], a.est[3], a.out[3], a.eps, a.lam, a.mixw);
    G.P[3].row_add = X.tot[2];
  }
  if (X.mask[0] || X.mask[1] || X.mask[2])
    for (int p = 0; p < 4; ++p) {
      Problem& Q = G.P[p];
      Q.fb_mask = X.mask[p < 3 ? p : 2];
      Q.fb_rlab = X.rlab[p];
      Q.fb_co = X.fco[p];
      Q.fb_words = X.words[p];
      Q.fb_trans = p == 3;
      Q.fb_upper = p < 2;  // fine-phase self masks hold their upper halves
      Q.fb_kc = X.kc3;
      if (!Q.fb_rlab || !Q.fb_co) Q.fb_mask = nullptr;
    }
  G.n_problems = 3;
  G.force_fb = c->force_fb;
  G.items = P.items;
  G.n_items = P.n_items;
  G.part = P.part;
  G.fb_count = ss.fb_count;
  G.fb_total = ss.fb_total;
  G.fb_list = ss.fb_list;
  G.fb_cap = ss.fb_cap;
  G.bad_scale = ss.bad_scale;
  G.scale = ss.scale;
  CK(cudaMemsetAsync(ss.fb_count, 0, sizeof(int32_t), st));
  const bool hd = ss.d > 3;
  if (hd) {
    for (int p = 0; p < 3; ++p) {
      const size_t np = hd_padded(G.P[p].n_cols);
      float* cc = c->buf<float>("hd.c" + std::to_string(p), np);
      float* c2 = c->buf<float>("hd.cf" + std::to_string(p), np);
      CK(hd_colconst(G.P[p], cc, c2, st));
      G.P[p].col_c = cc;
      G.P[p].col_c2 = c2;
    }
  }
  // Batches of consecutive tiles (Plan::Batch): the softmin writes the
  // batch's column partials into the bounded buffer, the column-sum pass
  // folds them into float64 running totals before the next batch reuses it.
  const int nbt = static_cast<int>(P.batches.size());
  int first_b[3], last_b[3];
  for (int p = 0; p < 3; ++p) {
    first_b[p] = last_b[p] = -1;
    for (int bi = 0; bi < nbt; ++bi)
      if (P.batches[bi].bt1[p] > P.batches[bi].bt0[p]) {
        if (first_b[p] < 0) first_b[p] = bi;
        last_b[p] = bi;
      }
    if (first_b[p] < 0) first_b[p] = last_b[p] = 0;  // no local tiles: totals = 0
  }
  double* acc[3] = {nullptr, nullptr, nullptr};
  float* rsum[3] = {nullptr, nullptr, nullptr};
  const bool multi = nbt > 1;
  // several ranks: the column totals are exchanged in float64 and rounded
  // once afterwards, so they differ from a single rank's only where the
  // float64 sums (in another association) straddle a float32 rounding point
  const bool x64 = c->comm || (c->world > 1 && c->host_bc);
  // overlap consecutive batches on the two side streams; profiling keeps
  // every launch on the main stream so each softmin is timed alone
  const bool overlap = multi && !c->profiling;
  for (int p = 0; p < 3; ++p) {
    if (multi || x64) acc[p] = c->buf<double>("sym.acc" + std::to_string(p), P.ps[p].n_cols);
    if (multi) rsum[p] = c->buf<float>("sym.rsum" + std::to_string(p), P.ps[p].n_rows);
  }
  if (overlap) {
    CK(cudaEventRecord(c->ev_fork, st));
    for (int k = 0; k < 2; ++k) CK(cudaStreamWaitEvent(c->side[k], c->ev_fork, 0));
  }
  for (int bi = 0; bi < nbt; ++bi) {
    const Plan::Batch& B = P.batches[bi];
    cudaStream_t bs = overlap ? c->side[bi & 1] : st;
    float* half = P.colbuf + (multi ? (bi & 1) * P.batch_slots : 0);
    Group Gb = G;
    Gb.items = P.items + B.i0;
    Gb.n_items = B.i1 - B.i0;
    // batched: this batch's row partials in its half of the part buffer
    Gb.part = multi ? P.part + static_cast<int64_t>(bi & 1) * P.batch_items * kTileRows
                    : P.part + static_cast<int64_t>(B.i0) * kTileRows;
    const float* cp[3];
    for (int p = 0; p < 3; ++p) {
      const bool has = B.bt1[p] > B.bt0[p];
      // colpart[tile_slot[t] + pos] lands at half + off + (slot - first slot)
      cp[p] = has ? half + B.off[p] - P.ps[p].sym->tslot_h[B.bt0[p]] : half;
      Gb.P[p].colpart = const_cast<float*>(cp[p]);
      Gb.P[p].tile_slot = P.ps[p].sym->tslot;
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->profiling) {
      c->ev_pair(&e0, &e1);
      CK(cudaEventRecord(e0, bs));
    }
    if (Gb.n_items > 0) {
      if (hd) CK(launch_softmin_hd(Gb, ss.d, c->n_sm, true, bs));
      else CK(launch_softmin_sym(Gb, ss.d, X.uniform && a.lam == 1.0, bs));
    }
    if (c->profiling) CK(cudaEventRecord(e1, bs));
    if (multi) {  // reduce the batch's row partials before the half is reused
      Group Gr = Gb;
      int32_t acc_t = 0;
      Gr.tile_prefix[0] = 0;
      for (int p = 0; p < 3; ++p) {
        Gr.t0[p] = B.bt0[p];
        acc_t += B.bt1[p] - B.bt0[p];
        Gr.tile_prefix[p + 1] = acc_t;
        Gr.P[p].row_sum = rsum[p];
      }
      CK(launch_rowsum(Gr, B.i0, bs));
    }
    ColSum cs[3];
    DenseColSum ds[3];
    int ncs = 0, nds = 0;
    // column sums accumulate batch after batch: wait for the previous batch's
    if (overlap && bi > 0) CK(cudaStreamWaitEvent(bs, c->ev_cs[(bi - 1) & 1], 0));
    for (int p = 0; p < 3; ++p) {
      const bool has = B.bt1[p] > B.bt0[p];
      if (!has && bi != first_b[p]) continue;  // nothing of p in this batch
      const SymSet& S = *P.ps[p].sym;
      const int first = bi == first_b[p], last = bi == last_b[p];
      const int32_t t0 = has ? B.bt0[p] : 0, t1 = has ? B.bt1[p] : 0;
      if (S.dense) {  // dense pair sets (high-D path, coarse phase, dense solves)
        ds[nds++] = DenseColSum{cp[p], S.tslot, S.R.tile_start, x64 ? nullptr : X.tot[p], acc[p],
                                t0, t1, S.self, static_cast<int32_t>(P.ps[p].n_cols), first,
                                last};
      } else {
        cs[ncs++] = ColSum{X.labels[p], X.co[p], S.ebase, S.eslot, S.etile, S.R.tile_start, cp[p],
                           x64 ? nullptr : X.tot[p], acc[p],
                           static_cast<int32_t>(P.ps[p].n_cols), S.self, t0, t1, first, last};
      }
    }
    if (ncs > 0) CK(launch_colsum(cs, ncs, bs));
    if (nds > 0) CK(hd_colsum_group(ds, nds, bs));
    if (overlap) CK(cudaEventRecord(c->ev_cs[bi & 1], bs));
  }
  if (overlap) CK(cudaStreamWaitEvent(st, c->ev_cs[(nbt - 1) & 1], 0));
  if (multi)
    for (int p = 0; p < 3; ++p) G.P[p].row_sum = rsum[p];
  if (x64) {  // column sums of every rank's tiles (NCCL over NVLink), float64
    const int64_t cnt[3] = {P.ps[0].n_cols, P.ps[1].n_cols, P.ps[2].n_cols};
    coll_allreduce64(c, acc, cnt, 3);
    for (int p = 0; p < 3; ++p)
      CK(totals_f32(acc[p], X.tot[p], static_cast<int32_t>(P.ps[p].n_cols), st));
  }
  G.colfinal_p = 3;  // a_xy from the column totals, in the same launch
  CK(launch_finalize(G, st));
  CK(hd ? launch_fallback_hd(G, ss.d, c->n_sm, st) : launch_fallback_dense(G, ss.d, c->n_sm, st));
  ss.S->softmin_launches += nbt;
  ss.S->colpart_batches = std::max(ss.S->colpart_batches, nbt);
  ss.S->pairs_evaluated += P.pairs_all;
  ss.S->pairs_terms += P.terms_all;
  coll_bcast_rows(c, a.out, P.row_bounds, 3);  // all-gather of the row-side potentials
}



struct Potentials {
  float* v[2][4];  // [buffer][a_xx, b_yy, a_xy, b_yx]
};

void alloc_pots(msot_ctx* c, const std::string& tag, int64_t n, int64_t m, Potentials& P) {
  for (int b = 0; b < 2; ++b) {
    const std::string t = tag + std::to_string(b);
    P.v[b][0] = c->buf<float>(t + ".a_xx", n);
    P.v[b][1] = c->buf<float>(t + ".b_yy", m);
    P.v[b][2] = c->buf<float>(t + ".a_xy", m);
    P.v[b][3] = c->buf<float>(t + ".b_yx", n);
    CK(cudaMemsetAsync(P.v[b][0], 0, n * sizeof(float), c->st));
    CK(cudaMemsetAsync(P.v[b][1], 0, m * sizeof(float), c->st));
    CK(cudaMemsetAsync(P.v[b][2], 0, m * sizeof(float), c->st));
    CK(cudaMemsetAsync(P.v[b][3], 0, n * sizeof(float), c->st));
  }
}

// msot_debug_capture: copies the potentials v (a_xx, b_yy, a_xy, b_yx in
// the solver's sorted order) to the caller's host buffers in caller order.
void capture_pots(msot_ctx* c, float* const* v, const int32_t* xperm, const int32_t* yperm,
                  int64_t n, int64_t m, double* const* host) {
  const int64_t len[4] = {n, m, m, n};
  const int32_t* perm[4] = {xperm, yperm, yperm, xperm};
  double* tmp = c->buf<double>("cap.tmp", std::max(n, m));
  for (int q = 0; q < 4; ++q) {
    if (!host[q]) continue;
    CK(scatter_unsort(v[q], perm[q], len[q], nullptr, 0.0, tmp, c->st));
    CK(cudaMemcpyAsync(host[q], tmp, len[q] * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(host_sync(__LINE__, c->st));
  }
}

// msot_debug_capture: the cluster masks of the captured update (unpacked)
// and the cluster of every atom in caller order (msot_debug_mask).
void capture_masks(msot_ctx* c, const uint32_t* const* masks, const int32_t* kr,
                   const int32_t* kc, const DMeasure& X, const DMeasure& Y) {
  cudaStream_t st = c->st;
  for (int q = 0; q < 3; ++q) {
    const size_t cells = size_t(kr[q]) * kc[q];
    uint8_t* dm = c->buf<uint8_t>("cap.mask", cells);
    CK(unpack_mask(masks[q], kr[q], kc[q], dm, st));
    c->cap_mask[q].resize(cells);
    CK(cudaMemcpyAsync(c->cap_mask[q].data(), dm, cells, cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    c->cap_k[q][0] = kr[q];
    c->cap_k[q][1] = kc[q];
  }
  const DMeasure* M[2] = {&X, &Y};
  for (int s = 0; s < 2; ++s) {
    std::vector<int32_t> lab(M[s]->n), perm(M[s]->n);
    CK(cudaMemcpyAsync(lab.data(), M[s]->labels, M[s]->n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(perm.data(), M[s]->perm, M[s]->n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    c->cap_lab[s].assign(M[s]->n, -1);
    for (int64_t k = 0; k < M[s]->n; ++k) c->cap_lab[s][perm[k]] = lab[k];
  }
}

// The four symmetric problems on measures X (rows of a_xx, b_yx) and Y.
void sym_specs(Plan& P, const float4* xp, const float* xl, int64_t n, const float4* yp,
               const float* yl, int64_t m, const RangeSet* rxx, const RangeSet* ryy,
               const RangeSet* rxy, const RangeSet* ryx) {
  P.np = 4;
  P.ps[0] = {xp, n, xp, xl, n, rxx};  // a_xx: rows x, cols x
  P.ps[1] = {yp, m, yp, yl, m, ryy};  // b_yy: rows y, cols y
  P.ps[2] = {yp, m, xp, xl, n, rxy};  // a_xy: rows y, cols x
  P.ps[3] = {xp, n, yp, yl, m, ryx};  // b_yx: rows x, cols y
}

// One averaged (or final, assigned) symmetric update:
// all four read buffer `cur`, write buffer `cur ^ 1`.
void sym_step(msot_ctx* c, const Plan& P, Potentials& U, int& cur, double eps, double lam,
              bool assign, SolveState& ss) {
  float** o = U.v[cur];
  float** n = U.v[cur ^ 1];
  ScaleArgs a{};
  a.h[0] = o[0]; a.est[0] = o[0]; a.out[0] = n[0];
  a.h[1] = o[1]; a.est[1] = o[1]; a.out[1] = n[1];
  a.h[2] = o[3]; a.est[2] = o[2]; a.out[2] = n[2];
  a.h[3] = o[2]; a.est[3] = o[3]; a.out[3] = n[3];
  a.eps = eps;
  a.lam = lam;
  a.mixw = assign ? 1.0 : 0.5;
  run_group(c, P, a, ss);
  cur ^= 1;
}

// One evaluate-once symmetric update: same contract as sym_step.
void sym_step_once(msot_ctx* c, const Plan& P, Potentials& U, int& cur, double eps, double lam,
                   bool assign, SolveState& ss, const SymCols& X) {
  float** o = U.v[cur];
  float** n = U.v[cur ^ 1];
  ScaleArgs a{};
  a.h[0] = o[0]; a.est[0] = o[0]; a.out[0] = n[0];  // a_xx
  a.h[1] = o[1]; a.est[1] = o[1]; a.out[1] = n[1];  // b_yy
  a.h[2] = o[2]; a.est[2] = o[3]; a.out[2] = n[3];  // b_yx (rows x, cols y)
  a.h[3] = o[3]; a.est[3] = o[2]; a.out[3] = n[2];  // a_xy (its column side)
  a.eps = eps;
  a.lam = lam;
  a.mixw = assign ? 1.0 : 0.5;
  run_group_sym(c, P, a, ss, X);
  cur ^= 1;
}

// Implicit plan sums (plan_kernel) for problems `specs` with row potentials
// f, column potentials g and column payloads: out[p] = {m_i, u_i} per row.
// Not sharded: every rank computes all rows (the outputs are small).
void plan_group(msot_ctx* c, const std::string& tag, int np, const ProbSpec* specs,
                const float* const* f, const float* const* g, const float4* const* pay,
                float4* const* out, double eps, int d) {
  const int rank = c->rank, world = c->world;
  c->rank = 0;
  c->world = 1;
  Plan P;
  P.np = np;
  for (int p = 0; p < np; ++p) P.ps[p] = specs[p];
  try {
    build_plan(c, tag, P);
  } catch (...) {
    c->rank = rank;
    c->world = world;
    throw;
  }
  c->rank = rank;
  c->world = world;
  const double ln2 = 0.69314718055994530942;
  Group G{};
  int32_t tiles_acc = 0;
  for (int p = 0; p < np; ++p) {
    Problem& Q = G.P[p];
    const ProbSpec& S = P.ps[p];
    Q.rows = S.rows;
    Q.row_est = f[p];
    Q.row_out = nullptr;
    Q.cols = S.cols;
    Q.col_lw2 = S.col_lw2;
    Q.col_h = g[p];
    Q.tile_start = S.rs->tile_start;
    Q.tile_rptr = S.rs->rptr;
    Q.ranges = S.rs->ranges;
    Q.tile_ibase = P.ibase[p];
    Q.col_pay = pay[p];
    Q.row_plan = out[p];
    Q.n_rows = static_cast<int32_t>(S.n_rows);
    Q.n_cols = static_cast<int32_t>(S.n_cols);
    Q.sc = static_cast<float>(1.0 / std::sqrt(2.0 * eps * ln2));
    Q.inv_eps_ln2 = static_cast<float>(1.0 / (eps * ln2));
    Q.inv_lam_eps_ln2 = Q.inv_eps_ln2;  // lambda = 1: exp((f + g - C) / eps)
    Q.lam_eps = static_cast<float>(eps);
    Q.mixw = 1.f;
    G.t0[p] = 0;
    G.tile_prefix[p] = tiles_acc;
    tiles_acc += static_cast<int32_t>(S.rs->n_tiles);
  }
  G.tile_prefix[np] = tiles_acc;
  G.n_problems = np;
  G.items = P.items;
  G.n_items = P.n_items;
  G.part = c->buf<float>(tag + ".ppart", static_cast<size_t>(P.n_items) * 4 * kTileRows);
  CK(launch_plan(G, d, c->st));
}

// ---------------------------------------------------------------------------
// High-dimensional multiscale (D > 3): K-means
// coarsening (kmeans.cu) instead of the voxel grid, a dense
// evaluate-once coarse phase on the centroid measures, inheritance at the
// switch, and the block-sparse evaluate-once fine phase on the tcgen05
// kernel.  Each cluster is padded to a multiple of 128 atoms (centroid
// coordinates, weight 0) so every column range is whole 128-column blocks.
struct HdLayout {
  int K = 0;
  int64_t npad = 0;
  std::vector<int32_t> poff_h;     // padded cluster offsets (K+1)
  int32_t* poff = nullptr;         // device
  int32_t* labels = nullptr;       // cluster of every padded slot
  int32_t* src = nullptr;          // caller index, or -(I+1) for padding of cluster I
  double* centers = nullptr;       // K x d float64
  float* radii = nullptr;
  float4* box_lo = nullptr;  // member boxes (truncation box bound, mask.cu)
  float4* box_hi = nullptr;
  std::vector<float> radii_h;
  float* clw2 = nullptr;           // coarse measure
  double* cw64 = nullptr;
  uint8_t* cpack = nullptr;
  float* csq = nullptr;
  float* cf = nullptr;
  uint8_t* pack = nullptr;         // padded fine measure
  float* sq = nullptr;
  float* f = nullptr;
  float* lw2 = nullptr;
  double* w64 = nullptr;
};

void hd_layout(msot_ctx* c, const std::string& tag, const double* dx, const double* dw, int64_t n,
               int d, int K, uint64_t seed, double diam, const double* dcen, HdLayout& L) {
  cudaStream_t st = c->st;
  L.K = K;
  int32_t* perm = c->buf<int32_t>(tag + ".kperm", n);
  int32_t* off = c->buf<int32_t>(tag + ".koff", K + 1);
  uint32_t* lab = c->buf<uint32_t>(tag + ".klab", n);
  L.centers = c->buf<double>(tag + ".kcen", size_t(K) * d);
  double* cw = c->buf<double>(tag + ".kcw", K);
  L.radii = c->buf<float>(tag + ".krad", K);
  void* ws = c->buf<char>(tag + ".kws", kmeans_ws_bytes(n, d, K));
  const double tol = 1e-9 * diam;
  CK(kmeans(dx, dw, n, d, K, seed, tol * tol, MSOT_KMEANS_SOLVER_ITERS, ws, perm, off, lab,
            L.centers, cw, L.radii, nullptr, st));
  std::vector<int32_t> off_h(K + 1), perm_h(n);
  L.radii_h.resize(K);
  CK(cudaMemcpyAsync(off_h.data(), off, (K + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(perm_h.data(), perm, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(L.radii_h.data(), L.radii, K * sizeof(float), cudaMemcpyDeviceToHost, st));
  CK(host_sync(__LINE__, st));
  L.poff_h.assign(K + 1, 0);
  for (int I = 0; I < K; ++I)
    L.poff_h[I + 1] = L.poff_h[I] + (off_h[I + 1] - off_h[I] + 127) / 128 * 128;
  L.npad = L.poff_h[K];
  std::vector<int32_t> src(L.npad), labp(L.npad);
  for (int I = 0; I < K; ++I) {
    const int32_t cnt = off_h[I + 1] - off_h[I];
    for (int32_t q = 0; q < L.poff_h[I + 1] - L.poff_h[I]; ++q) {
      src[L.poff_h[I] + q] = q < cnt ? perm_h[off_h[I] + q] : -(I + 1);
      labp[L.poff_h[I] + q] = I;
    }
  }
  L.poff = c->buf<int32_t>(tag + ".poff", K + 1);
  L.labels = c->buf<int32_t>(tag + ".plab", L.npad);
  L.src = c->buf<int32_t>(tag + ".psrc", L.npad);
  CK(cudaMemcpyAsync(L.poff, L.poff_h.data(), (K + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(L.labels, labp.data(), L.npad * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(L.src, src.data(), L.npad * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  double* xp = c->buf<double>(tag + ".px64", L.npad * d);
  CK(hd_gather_padded(dx, L.centers, L.src, L.npad, d, xp, st));
  L.lw2 = c->buf<float>(tag + ".plw2", L.npad);
  L.w64 = c->buf<double>(tag + ".pw64", L.npad);
  CK(hd_padded_weights(dw, L.src, L.npad, L.lw2, L.w64, st));
  L.pack = c->buf<uint8_t>(tag + ".ppack", hd_pack_bytes(L.npad));
  L.sq = c->buf<float>(tag + ".psq", hd_padded(L.npad));
  L.f = c->buf<float>(tag + ".pf", hd_padded(L.npad) * 64);
  CK(hd_pack(xp, L.npad, d, dcen, 0, L.pack, L.sq, L.f, st));
  // the coarse measure (centroids, cluster weights)
  L.cpack = c->buf<uint8_t>(tag + ".cpack", hd_pack_bytes(K));
  L.csq = c->buf<float>(tag + ".csq", hd_padded(K));
  L.cf = c->buf<float>(tag + ".cf", hd_padded(K) * 64);
  CK(hd_pack(L.centers, K, d, dcen, 0, L.cpack, L.csq, L.cf, st));
  L.clw2 = c->buf<float>(tag + ".clw2", K);
  L.cw64 = c->buf<double>(tag + ".cw64", K);
  CK(hd_weights(cw, K, L.clw2, L.cw64, st));
  CK(host_sync(__LINE__, st));  // host vectors go out of scope
}

void hd_multiscale(msot_ctx* c, const msot_params* prm, const double* d_x, const double* d_a,
                   int64_t n, const double* d_y, const double* d_b, int64_t m, int d,
                   const double* dcen, double diam, const std::vector<double>& sig,
                   const std::vector<double>& eps, const std::vector<double>& lam, int ns,
                   Potentials& U, int& cur, DMeasure& X, DMeasure& Y, int64_t& nr, int64_t& mr,
                   uint8_t*& hd_ax, float*& hd_sqx, SolveState& ss, msot_stats* S) {
  cudaStream_t st = c->st;
  if (prm->pair_eval == 0) raise(MSOT_EUSAGE, "high-D multiscale runs the evaluate-once scheme");
  const int kx = prm->clusters > 0 ? static_cast<int>(std::min<int64_t>(prm->clusters, n))
                                   : static_cast<int>(std::ceil(std::sqrt(static_cast<double>(n))));
  const int ky = prm->clusters > 0 ? static_cast<int>(std::min<int64_t>(prm->clusters, m))
                                   : static_cast<int>(std::ceil(std::sqrt(static_cast<double>(m))));
  c->mark(0);
  HdLayout LX, LY;
  hd_layout(c, "hx", d_x, d_a, n, d, kx, static_cast<uint64_t>(prm->seed), diam, dcen, LX);
  hd_layout(c, "hy", d_y, d_b, m, d, ky, static_cast<uint64_t>(prm->seed), diam, dcen, LY);
  nr = LX.npad;
  mr = LY.npad;
  alloc_pots(c, "hpot", nr, mr, U);
  cur = 0;
  X = DMeasure{};
  Y = DMeasure{};
  X.n = nr;
  Y.n = mr;
  X.k = kx;
  Y.k = ky;
  X.lw2 = LX.lw2;
  X.w64 = LX.w64;
  X.perm = LX.src;
  X.labels = LX.labels;
  X.offsets = LX.poff;
  X.offsets_h = LX.poff_h;
  Y.lw2 = LY.lw2;
  Y.w64 = LY.w64;
  Y.perm = LY.src;
  Y.labels = LY.labels;
  Y.offsets = LY.poff;
  Y.offsets_h = LY.poff_h;
  hd_ax = LX.pack;
  hd_sqx = LX.sq;
  S->kx = kx;
  S->ky = ky;
  double rmax = 0.0;
  for (float r : LX.radii_h) rmax = std::max(rmax, double(r));
  for (float r : LY.radii_h) rmax = std::max(rmax, double(r));
  const int tsw = msot_switch_index(sig.data(), ns, rmax, prm->switch_factor);
  S->t_switch = tsw;
  S->cluster_scale = rmax;
  const double full = double(n) * n + double(m) * m + 2.0 * double(n) * m;
  // ---- coarse phase: dense evaluate-once on the centroid measures
  c->mark(1);
  float* coarse[4] = {nullptr, nullptr, nullptr, nullptr};
  if (tsw > 0) {
    Potentials Uc;
    alloc_pots(c, "hcpot", kx, ky, Uc);
    int ccur = 0;
    SymSet cxx, cyy, cyx;
    dense_symset(c, "hcs.xx", kx, kx, 1, cxx);
    dense_symset(c, "hcs.yy", ky, ky, 1, cyy);
    dense_symset(c, "hcs.yx", kx, ky, 0, cyx);
    Plan Pc;
    Pc.np = 3;
    Pc.ps[0] = {nullptr, kx, nullptr, LX.clw2, kx, &cxx.R, {LX.cpack, LX.cpack, LX.csq, LX.csq, LX.cf, LX.cf}, &cxx, LX.clw2};
    Pc.ps[1] = {nullptr, ky, nullptr, LY.clw2, ky, &cyy.R, {LY.cpack, LY.cpack, LY.csq, LY.csq, LY.cf, LY.cf}, &cyy, LY.clw2};
    Pc.ps[2] = {nullptr, kx, nullptr, LY.clw2, ky, &cyx.R, {LX.cpack, LY.cpack, LX.csq, LY.csq, LX.cf, LY.cf}, &cyx, LX.clw2};
    SymCols cc{};
    cc.tot[0] = c->buf<float>("hcs.totx", kx);
    cc.tot[1] = c->buf<float>("hcs.toty", ky);
    cc.tot[2] = c->buf<float>("hcs.totxy", ky);
    cc.x_lw2 = LX.clw2;
    cc.n = kx;
    cc.m = ky;
    cc.hd3 = {LY.cpack, LX.cpack, LY.csq, LX.csq, LY.cf, LX.cf};
    build_plan(c, "hpc", Pc, 2, d);
    const double cfull = double(kx) * kx + double(ky) * ky + 2.0 * double(kx) * ky;
    for (int t = 0; t < tsw; ++t) {
      ss.scale = t;
      sym_step_once(c, Pc, Uc, ccur, eps[t], lam[t], false, ss, cc);
      S->pairs_dense += cfull;
    }
    // coarse -> fine: inheritance (padding slots inherit
    // too), then for transfer_rule 1 one lambda-damped softmin of every fine
    // atom against the coarse measure (GeomLoss extrapolation), expanded
    // around the inherited value
    c->mark(2);
    float** co = Uc.v[ccur];
    const bool extrap = prm->transfer_rule == 1;
    float** dst = U.v[extrap ? cur ^ 1 : cur];
    CK(inherit(co[0], LX.labels, nr, dst[0], st));
    CK(inherit(co[1], LY.labels, mr, dst[1], st));
    CK(inherit(co[2], LY.labels, mr, dst[2], st));
    CK(inherit(co[3], LX.labels, nr, dst[3], st));
    for (int q = 0; q < 4; ++q) coarse[q] = co[q];
    if (extrap) {
      RangeSet exx, eyy, exy, eyx;
      dense_rangeset(c, "he.xx", nr, kx, exx);
      dense_rangeset(c, "he.yy", mr, ky, eyy);
      dense_rangeset(c, "he.xy", mr, kx, exy);
      dense_rangeset(c, "he.yx", nr, ky, eyx);
      Plan Pe;
      Pe.np = 4;
      Pe.ps[0] = {nullptr, nr, nullptr, LX.clw2, kx, &exx, {LX.pack, LX.cpack, LX.sq, LX.csq, LX.f, LX.cf}};
      Pe.ps[1] = {nullptr, mr, nullptr, LY.clw2, ky, &eyy, {LY.pack, LY.cpack, LY.sq, LY.csq, LY.f, LY.cf}};
      Pe.ps[2] = {nullptr, mr, nullptr, LX.clw2, kx, &exy, {LY.pack, LX.cpack, LY.sq, LX.csq, LY.f, LX.cf}};
      Pe.ps[3] = {nullptr, nr, nullptr, LY.clw2, ky, &eyx, {LX.pack, LY.cpack, LX.sq, LY.csq, LX.f, LY.cf}};
      build_plan(c, "hpe", Pe, 2, d);
      ScaleArgs ea{};
      ea.h[0] = co[0]; ea.est[0] = dst[0]; ea.out[0] = U.v[cur][0];
      ea.h[1] = co[1]; ea.est[1] = dst[1]; ea.out[1] = U.v[cur][1];
      ea.h[2] = co[3]; ea.est[2] = dst[2]; ea.out[2] = U.v[cur][2];
      ea.h[3] = co[2]; ea.est[3] = dst[3]; ea.out[3] = U.v[cur][3];
      ea.eps = eps[tsw - 1];
      ea.lam = lam[tsw - 1];
      ea.mixw = 1.0;
      run_group(c, Pe, ea, ss);
    }
  }
  // ---- fine phase: block-sparse evaluate-once on the padded measures
  uint32_t* mxx = c->buf<uint32_t>("hm.xx", size_t(kx) * mask_words(kx));
  uint32_t* myy = c->buf<uint32_t>("hm.yy", size_t(ky) * mask_words(ky));
  uint32_t* mxy = c->buf<uint32_t>("hm.xy", size_t(kx) * mask_words(ky));
  uint32_t* myx = c->buf<uint32_t>("hm.yx", size_t(ky) * mask_words(kx));
  float* fm[4];
  fm[0] = c->buf<float>("hm.Fxx", kx);
  fm[1] = c->buf<float>("hm.Gyy", ky);
  fm[2] = c->buf<float>("hm.Gxy", ky);
  fm[3] = c->buf<float>("hm.Fyx", kx);
  int32_t* bxr = c->buf<int32_t>("hm.bx", std::max(kx, ky));
  int32_t* byr = c->buf<int32_t>("hm.by", std::max(kx, ky));
  SymSet sxx, syy, syx;
  SymCols scol{};
  scol.labels[0] = LX.labels; scol.co[0] = LX.poff; scol.tot[0] = c->buf<float>("hs.totx", nr);
  scol.labels[1] = LY.labels; scol.co[1] = LY.poff; scol.tot[1] = c->buf<float>("hs.toty", mr);
  scol.labels[2] = LY.labels; scol.co[2] = LY.poff; scol.tot[2] = c->buf<float>("hs.totxy", mr);
  scol.x_lw2 = LX.lw2;
  scol.y_lw2 = LY.lw2;
  scol.n = nr;
  scol.m = mr;
  scol.hd3 = {LY.pack, LX.pack, LY.sq, LX.sq, LY.f, LX.f};
  Plan Pf;
  auto build_masks = [&](double e) {
    const bool info = tsw > 0;
    const double theta = info ? prm->theta : INFINITY;
    float** f = U.v[cur];
    CK(hd_cluster_fmax(f[0], LX.w64, LX.poff, kx, fm[0], st));
    CK(hd_cluster_fmax(f[1], LY.w64, LY.poff, ky, fm[1], st));
    CK(hd_cluster_fmax(f[2], LY.w64, LY.poff, ky, fm[2], st));
    CK(hd_cluster_fmax(f[3], LX.w64, LX.poff, kx, fm[3], st));
    CK(truncation_masks_hd(kx, kx, d, LX.centers, LX.radii, fm[0], LX.centers, LX.radii, fm[0], e,
                           theta, 1, mxx, nullptr, bxr, nullptr, st));
    CK(truncation_masks_hd(ky, ky, d, LY.centers, LY.radii, fm[1], LY.centers, LY.radii, fm[1], e,
                           theta, 1, myy, nullptr, byr, nullptr, st));
    CK(truncation_masks_hd(kx, ky, d, LX.centers, LX.radii, fm[3], LY.centers, LY.radii, fm[2], e,
                           theta, 0, mxy, myx, bxr, byr, st));
    sym_rangesets(c, {{"hs.xx", LX.labels, &LX.poff_h, nr, LX.poff, kx, mxx, 1, &sxx},
                      {"hs.yy", LY.labels, &LY.poff_h, mr, LY.poff, ky, myy, 1, &syy},
                      {"hs.yx", LX.labels, &LX.poff_h, nr, LY.poff, ky, mxy, 0, &syx}});
    Pf.np = 3;
    Pf.ps[0] = {nullptr, nr, nullptr, LX.lw2, nr, &sxx.R, {LX.pack, LX.pack, LX.sq, LX.sq, LX.f, LX.f}, &sxx, LX.lw2};
    Pf.ps[1] = {nullptr, mr, nullptr, LY.lw2, mr, &syy.R, {LY.pack, LY.pack, LY.sq, LY.sq, LY.f, LY.f}, &syy, LY.lw2};
    Pf.ps[2] = {nullptr, nr, nullptr, LY.lw2, mr, &syx.R, {LX.pack, LY.pack, LX.sq, LY.sq, LX.f, LY.f}, &syx, LX.lw2};
    build_plan(c, "hpf", Pf, 2, d);
  };
  for (int t = tsw; t <= ns; ++t) {
    const int tt = std::min(t, ns - 1);
    ss.scale = t;
    const bool rebuild =
        (t == tsw) || (prm->retruncate > 0 && t < ns && (t - tsw) % prm->retruncate == 0);
    if (rebuild) {
      c->mark(3);
      build_masks(eps[tt]);
    }
    c->mark(4);
    sym_step_once(c, Pf, U, cur, eps[tt], lam[tt], t == ns, ss, scol);
    S->pairs_dense += full;
    S->pairs_fine += Pf.pairs_all;
    S->pairs_fine_dense += full;
  }
  (void)coarse;
}

// transfer_labels request (K9): atlas labels in the caller's order of y.
struct LabelReq {
  const int32_t* labels;  // host, M entries in [0, L)
  int n_classes;
  double* d_scores;       // device, N x L (caller row order)
  double* d_mass;         // device, N
};

// K9 (labels.cu): scores[i][l] = sum_{label_j = l} pi_ij / a_i with
// pi_ij / a_i = b_j exp((f_i + g_j - C_ij) / eps), f = b_yx, g = a_xy.  The
// softmin kernel with est = f, h = g, lambda = 1 computes exactly these
// terms; columns are put in label order (segments padded to the high-D
// kernel's 128-column block) and work items are cut at segment boundaries.
// Dense over the columns (the exact formula of eq. 7).
void transfer_labels_dev(msot_ctx* c, const LabelReq& q, const DMeasure& X, const DMeasure& Y,
                         int64_t n, int64_t m, int d, const double* d_y, const double* hd_cen,
                         const uint8_t* hd_ax, const float* hd_sqx, const float* f_row,
                         const float* g_col, double eps) {
  cudaStream_t st = c->st;
  const int L = q.n_classes;
  const bool hd = d > 3;
  const int64_t pad = hd ? 128 : 1;
  // n: rows of the solver's layout (X.n; padded for high-D multiscale).
  // solver slot of each caller atom of y: sorted 3-D measures and padded
  // high-D multiscale layouts carry a slot -> caller permutation (-1 =
  // padding), the dense high-D layout is the caller's order
  std::vector<int32_t> solver_of(m);
  if (Y.perm) {
    std::vector<int32_t> perm(Y.n);
    CK(cudaMemcpyAsync(perm.data(), Y.perm, Y.n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    for (int64_t k = 0; k < Y.n; ++k)
      if (perm[k] >= 0) solver_of[perm[k]] = static_cast<int32_t>(k);
  } else {
    for (int64_t j = 0; j < m; ++j) solver_of[j] = static_cast<int32_t>(j);
  }
  std::vector<int64_t> cnt(L, 0), seg(L + 1, 0);
  for (int64_t j = 0; j < m; ++j) {
    const int32_t l = q.labels[j];
    if (l < 0 || l >= L) raise(MSOT_EDATA, "label outside [0, L)");
    ++cnt[l];
  }
  for (int l = 0; l < L; ++l) seg[l + 1] = seg[l] + (cnt[l] + pad - 1) / pad * pad;
  const int64_t mpad = std::max<int64_t>(seg[L], 1);
  std::vector<int32_t> src(mpad, -1), csrc(mpad, -1);  // solver slot / caller index
  std::vector<int64_t> fill(seg.begin(), seg.end() - 1);
  for (int64_t j = 0; j < m; ++j) {
    const int64_t p = fill[q.labels[j]]++;
    src[p] = solver_of[j];
    csrc[p] = static_cast<int32_t>(j);
  }
  int32_t* dsrc = c->buf<int32_t>("lab.src", mpad);
  int32_t* dcsrc = c->buf<int32_t>("lab.csrc", mpad);
  CK(cudaMemcpyAsync(dsrc, src.data(), mpad * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dcsrc, csrc.data(), mpad * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  float* lwL = c->buf<float>("lab.lw", mpad);
  float* hL = c->buf<float>("lab.h", mpad);
  float4* colsL = hd ? nullptr : c->buf<float4>("lab.cols", mpad);
  CK(gather_label_cols(hd ? nullptr : Y.pts, Y.lw2, g_col, dsrc, mpad, colsL, lwL, hL, st));
  uint8_t* bL = nullptr;
  float* sqL = nullptr;
  if (hd) {
    double* yL = c->buf<double>("lab.y64", mpad * d);
    CK(gather_rows_f64(d_y, d, dcsrc, mpad, yL, st));
    bL = c->buf<uint8_t>("lab.bpack", hd_pack_bytes(mpad));
    sqL = c->buf<float>("lab.sq", hd_padded(mpad));
    CK(hd_pack(yL, mpad, d, hd_cen, 1, bL, sqL, nullptr, st));
  }
  RangeSet R;
  dense_rangeset(c, "lab.rows", n, mpad, R);
  const int64_t T = R.n_tiles;
  // work items: (tile, label segment) cut into chunks of whole column blocks
  const int64_t target = static_cast<int64_t>(c->n_sm) * 24;
  int64_t chunk = std::max<int64_t>(2 * kColTile, (T * mpad + target - 1) / target);
  chunk = (chunk + kColTile - 1) / kColTile * kColTile;
  std::vector<int4> items;
  std::vector<int32_t> lbase(static_cast<size_t>(T) * L + 1);
  for (int64_t t = 0; t < T; ++t)
    for (int l = 0; l < L; ++l) {
      lbase[t * L + l] = static_cast<int32_t>(items.size());
      for (int64_t z = seg[l]; z < seg[l + 1]; z += chunk)
        items.push_back(make_int4(0, static_cast<int>(t), static_cast<int>(z),
                                  static_cast<int>(std::min(z + chunk, seg[l + 1]))));
    }
  lbase[T * L] = static_cast<int32_t>(items.size());
  if (items.size() > 0x7fffffffULL) raise(MSOT_EUSAGE, "too many label work items");
  int4* ditems = c->buf<int4>("lab.items", items.size());
  int32_t* dlbase = c->buf<int32_t>("lab.lbase", lbase.size());
  CK(cudaMemcpyAsync(ditems, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dlbase, lbase.data(), lbase.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  const double ln2 = 0.69314718055994530942;
  Group G{};
  Problem& Q = G.P[0];
  Q.rows = hd ? nullptr : X.pts;
  Q.row_est = f_row;
  Q.cols = colsL;
  Q.col_lw2 = lwL;
  Q.col_h = hL;
  Q.tile_start = R.tile_start;
  Q.tile_rptr = R.rptr;
  Q.ranges = R.ranges;
  Q.a_pack = hd_ax;
  Q.b_pack = bL;
  Q.row_sq = hd_sqx;
  Q.col_sq = sqL;
  Q.n_rows = static_cast<int32_t>(n);
  Q.n_cols = static_cast<int32_t>(mpad);
  Q.sc = static_cast<float>(1.0 / std::sqrt(2.0 * eps * ln2));
  Q.inv_eps_ln2 = static_cast<float>(1.0 / (eps * ln2));
  Q.inv_lam_eps_ln2 = Q.inv_eps_ln2;  // lambda = 1: exp((f + g - C) / eps)
  Q.lam_eps = static_cast<float>(eps);
  Q.mixw = 1.f;
  G.n_problems = 1;
  G.items = ditems;
  G.n_items = static_cast<int32_t>(items.size());
  G.part = c->buf<float>("lab.part", items.size() * kTileRows);
  G.tile_prefix[1] = static_cast<int32_t>(T);
  if (hd) {
    float* cc = c->buf<float>("lab.c", hd_padded(mpad));
    CK(hd_colconst(Q, cc, nullptr, st));
    Q.col_c = cc;
  }
  CK(hd ? launch_softmin_hd(G, d, c->n_sm, false, st) : launch_softmin(G, d, st));
  CK(label_finalize(G.part, dlbase, R.tile_start, T, L, X.perm, q.d_scores, q.d_mass, st));
  CK(host_sync(__LINE__, st));  // host vectors above go out of scope
}

void solve_device(msot_ctx* c, const msot_params* prm, const double* d_x, const double* d_a,
                  int64_t n, const double* d_y, const double* d_b, int64_t m, int d,
                  double* loss_out, msot_stats* S, double* h_pots[4], double* d_grad = nullptr,
                  const LabelReq* lreq = nullptr) {
  if (n < 1 || m < 1) raise(MSOT_EDATA, "empty measure");
  if (n > 0x7fffff00LL || m > 0x7fffff00LL) raise(MSOT_EDATA, "measure too large");
  if (d < 1 || d > 64) raise(MSOT_EUSAGE, "the GPU solver supports D in 1..64");
  if (!(prm->blur > 0) || !(prm->scaling > 0 && prm->scaling < 1))
    raise(MSOT_EUSAGE, "invalid blur/scaling");
  if (prm->p != 2.0) raise(MSOT_EUSAGE, "the GPU path implements p = 2");
  if (!msot_reach_valid(prm->reach)) raise(MSOT_EUSAGE, "reach must be > 0 (or +inf for balanced OT)");
  cudaStream_t st = c->st;
  const int64_t launches0 = g_launches, syncs0 = g_host_syncs;
  c->solve_atoms = n + m;
  double frame[3] = {0.0, 0.0, 0.0};  // centre of the float32 atom frame (voxel path)
  c->ev_used = 0;
  c->marks.clear();
  c->mark(0);  // phase 0: bounding box, voxel edge, clustering
  CK(cudaEventRecord(c->t0, st));

  // diameter_estimate -- exact min/max on the device
  long long* lohi = c->buf<long long>("bbox", 2 * d);
  int32_t* badw = c->buf<int32_t>("badw", 1);
  CK(cudaMemsetAsync(badw, 0, sizeof(int32_t), st));
  CK(bbox(d_x, n, d, lohi, true, st));
  CK(bbox(d_y, m, d, lohi, false, st));
  CK(count_bad_weights(d_a, n, badw, st));
  CK(count_bad_weights(d_b, m, badw, st));
  std::vector<long long> lh(2 * d);
  int32_t nbad = 0;
  CK(cudaMemcpyAsync(lh.data(), lohi, 2 * d * sizeof(long long), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&nbad, badw, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CK(host_sync(__LINE__, st));
  if (nbad) raise(MSOT_EDATA, "weights must be finite and > 0");
  std::vector<double> lov(std::max(d, 3), 0.0), hiv(std::max(d, 3), 0.0);
  double* lo = lov.data();
  double* hi = hiv.data();
  bbox_decode(lh.data(), d, lo, hi);
  for (int k = 0; k < d; ++k)
    if (!std::isfinite(lo[k]) || !std::isfinite(hi[k])) raise(MSOT_EDATA, "non-finite point");
  double diag2 = 0.0;
  for (int k = 0; k < d; ++k) diag2 += (hi[k] - lo[k]) * (hi[k] - lo[k]);
  const double diam = c->diam_override > 0 ? std::max(c->diam_override, prm->blur)
                                           : std::max(std::sqrt(diag2), prm->blur);
  S->diameter = diam;
  const int ns = msot_schedule_len(diam, prm->blur, prm->scaling);
  if (prm->max_full_iters > 0 && ns > prm->max_full_iters)
    raise(MSOT_EUSAGE, "schedule longer than max_full_iters");
  std::vector<double> sig(ns), eps(ns), lam(ns);
  msot_schedule(diam, prm, sig.data(), eps.data(), lam.data(), ns);
  S->n_scales = ns;

  const bool ms = prm->multiscale != 0;
  SolveState ss{S, d, c->buf<int32_t>("fb.count", 1), c->buf<int32_t>("fb.total", 1), nullptr, 0};
  ss.fb_cap = static_cast<int32_t>(std::min<int64_t>(2 * (n + m), 1 << 22));
  ss.fb_list = c->buf<int4>("fb.list", ss.fb_cap);
  CK(cudaMemsetAsync(ss.fb_total, 0, sizeof(int32_t), st));
  ss.bad_scale = c->buf<int32_t>("bad.scale", 1);
  CK(cudaMemsetAsync(ss.bad_scale, 0x7f, sizeof(int32_t), st));  // 0x7f7f7f7f: none

  Potentials U;
  alloc_pots(c, "pot", n, m, U);
  int cur = 0;
  int64_t nr = n, mr = m;  // rows of the internal layout (padded for high-D multiscale)
  const double full = double(n) * n + double(m) * m + 2.0 * double(n) * m;
  RangeSet fxx, fyy, fxy, fyx;  // ranges of the last update (the plan reuses them)
  DMeasure X, Y;
  double* hd_cen = nullptr;      // high-D operands kept for the label transfer
  uint8_t* hd_ax = nullptr;
  float* hd_sqx = nullptr;

  if (d > 3) {
    // ---- high feature dimension (config 4): dense eps-scaling, <x,y> on
    // the tensor cores (softmin_hd.cu); the voxel grid needs D <= 3
    if (d > 64) raise(MSOT_EUSAGE, "the high-dimensional softmin supports D <= 64");
    if (d_grad) raise(MSOT_EUSAGE, "grad_positions is implemented for D <= 3");
    std::vector<double> center(d);
    for (int k = 0; k < d; ++k) center[k] = 0.5 * (lo[k] + hi[k]);
    double* dcen = c->buf<double>("hd.center", d);
    CK(cudaMemcpyAsync(dcen, center.data(), d * sizeof(double), cudaMemcpyHostToDevice, st));
    if (ms) {
      hd_multiscale(c, prm, d_x, d_a, n, d_y, d_b, m, d, dcen, diam, sig, eps, lam, ns, U, cur,
                    X, Y, nr, mr, hd_ax, hd_sqx, ss, S);
      hd_cen = dcen;
    } else {
    // one [hi | lo] pack per measure serves as A (rows) and B (columns)
    uint8_t* ax = c->buf<uint8_t>("hd.ax", hd_pack_bytes(n));
    uint8_t* ay = c->buf<uint8_t>("hd.ay", hd_pack_bytes(m));
    uint8_t* bx = ax;
    uint8_t* by = ay;
    float* sqx = c->buf<float>("hd.sqx", n);
    float* sqy = c->buf<float>("hd.sqy", m);
    float* fx = c->buf<float>("hd.fx", hd_padded(n) * 64);
    float* fy = c->buf<float>("hd.fy", hd_padded(m) * 64);
    CK(hd_pack(d_x, n, d, dcen, 0, ax, sqx, fx, st));
    CK(hd_pack(d_y, m, d, dcen, 0, ay, sqy, fy, st));
    hd_cen = dcen;
    hd_ax = ax;
    hd_sqx = sqx;
    X.n = n;
    Y.n = m;
    X.lw2 = c->buf<float>("x.lw2", n);
    X.w64 = c->buf<double>("x.w64", n);
    Y.lw2 = c->buf<float>("y.lw2", m);
    Y.w64 = c->buf<double>("y.w64", m);
    CK(hd_weights(d_a, n, X.lw2, X.w64, st));
    CK(hd_weights(d_b, m, Y.lw2, Y.w64, st));
    c->mark(4);
    S->t_switch = 0;
    Plan P;
    SymSet hxx, hyy, hyx;
    SymCols hcol{};
    const bool once = prm->pair_eval != 0;
    if (once) {  // evaluate-once: a_xy from the column sums of the cross problem
      dense_symset(c, "h.xx", n, n, 1, hxx);
      dense_symset(c, "h.yy", m, m, 1, hyy);
      dense_symset(c, "h.yx", n, m, 0, hyx);
      P.np = 3;
      P.ps[0] = {nullptr, n, nullptr, X.lw2, n, &hxx.R, {ax, bx, sqx, sqx, fx, fx}, &hxx, X.lw2};
      P.ps[1] = {nullptr, m, nullptr, Y.lw2, m, &hyy.R, {ay, by, sqy, sqy, fy, fy}, &hyy, Y.lw2};
      P.ps[2] = {nullptr, n, nullptr, Y.lw2, m, &hyx.R, {ax, by, sqx, sqy, fx, fy}, &hyx, X.lw2};
      hcol.tot[0] = c->buf<float>("h.totx", n);
      hcol.tot[1] = c->buf<float>("h.toty", m);
      hcol.tot[2] = c->buf<float>("h.totxy", m);
      hcol.x_lw2 = X.lw2;
      hcol.n = n;
      hcol.m = m;
      hcol.hd3 = {ay, bx, sqy, sqx, fy, fx};  // a_xy: rows y, cols x
    } else {
      dense_rangeset(c, "d.xx", n, n, fxx);
      dense_rangeset(c, "d.yy", m, m, fyy);
      dense_rangeset(c, "d.xy", m, n, fxy);
      dense_rangeset(c, "d.yx", n, m, fyx);
      P.np = 4;
      P.ps[0] = {nullptr, n, nullptr, X.lw2, n, &fxx, {ax, bx, sqx, sqx, fx, fx}};  // a_xx
      P.ps[1] = {nullptr, m, nullptr, Y.lw2, m, &fyy, {ay, by, sqy, sqy, fy, fy}};  // b_yy
      P.ps[2] = {nullptr, m, nullptr, X.lw2, n, &fxy, {ay, bx, sqy, sqx, fy, fx}};  // a_xy
      P.ps[3] = {nullptr, n, nullptr, Y.lw2, m, &fyx, {ax, by, sqx, sqy, fx, fy}};  // b_yx
    }
    build_plan(c, "ph", P, 2, d);
    for (int t = 0; t <= ns; ++t) {
      const int tt = std::min(t, ns - 1);
      ss.scale = t;
      if (once)
        sym_step_once(c, P, U, cur, eps[tt], lam[tt], t == ns, ss, hcol);
      else
        sym_step(c, P, U, cur, eps[tt], lam[tt], t == ns, ss);
      S->pairs_dense += full;
    }
    }  // dense high-D
  } else {
  GridSpec g{};
  g.d = d;
  for (int k = 0; k < d; ++k) {
    g.origin[k] = lo[k];
    g.center[k] = 0.5 * (lo[k] + hi[k]);
    if (k < 3) frame[k] = g.center[k];
  }
  double cell = prm->cluster_scale > 0 ? prm->cluster_scale : msot_auto_cell(lo, hi, d, n, m);
  if (ms && prm->cluster_scale <= 0) {  // policy.h: refine on occupied voxels
    for (int it = 0; it < MSOT_AUTO_REFINE; ++it) {
      g.cell = cell;
      const int64_t kk = count_cells(c, d_x, n, d_y, m, g);
      cell = msot_refine_cell(cell, kk, n, m, d, lo, hi);
    }
  }
  g.cell = cell;
  prepare_measures(c, {{"x", d_x, d_a, n, &X}, {"y", d_y, d_b, m, &Y}}, d, g, ms);

  if (!ms) {
    // dense solves stay row-wise (4 problems per scale): the cross potentials
    // of identical measures stay bitwise symmetric, S(a, a) = 0 exactly
    c->mark(4);  // phase 4: symmetric updates
    S->t_switch = 0;
    RangeSet &rxx = fxx, &ryy = fyy, &rxy = fxy, &ryx = fyx;
    dense_rangeset(c, "d.xx", n, n, rxx);
    dense_rangeset(c, "d.yy", m, m, ryy);
    dense_rangeset(c, "d.xy", m, n, rxy);
    dense_rangeset(c, "d.yx", n, m, ryx);
    Plan P;
    sym_specs(P, X.pts, X.lw2, n, Y.pts, Y.lw2, m, &rxx, &ryy, &rxy, &ryx);
    P.skip_p0 = c->self_mode == 2;
    build_plan(c, "pd", P);
    for (int t = 0; t <= ns; ++t) {
      const int tt = std::min(t, ns - 1);
      ss.scale = t;
      const bool cap = t == c->cap_scale;
      if (cap) capture_pots(c, U.v[cur], X.perm, Y.perm, n, m, c->cap_in);
      sym_step(c, P, U, cur, eps[tt], lam[tt], t == ns, ss);
      if (cap) capture_pots(c, U.v[cur], X.perm, Y.perm, n, m, c->cap_out);
      S->pairs_dense += full;
    }
  } else {
    S->cluster_scale = cell;
    S->kx = X.k;
    S->ky = Y.k;
    double rmax = 0.0;
    for (float r : X.radii_h) rmax = std::max(rmax, double(r));
    for (float r : Y.radii_h) rmax = std::max(rmax, double(r));
    const int tsw = msot_switch_index(sig.data(), ns, rmax, prm->switch_factor);
    S->t_switch = tsw;
    c->mark(1);  // phase 1: coarse phase on the centroid measures (dense)
    float* coarse_final[4] = {nullptr, nullptr, nullptr, nullptr};
    if (tsw > 0) {
      // dense updates t in [t0, t1) of the measures (xp, xl, kx) and (yp, yl, ky)
      auto coarse_run = [&](const std::string& tg, const float4* xp, const float* xl, int32_t kx,
                            const float4* yp, const float* yl, int32_t ky, Potentials& Uq,
                            int& qcur, int t0, int t1) {
        RangeSet rxx, ryy, rxy, ryx;
        SymSet cxx, cyy, cyx;
        SymCols ccol{};
        Plan Pc;
        const bool conce = prm->pair_eval != 0;
        if (conce) {  // evaluate-once on the centroid measures (dense pair sets)
          dense_symset(c, tg + "s.xx", kx, kx, 1, cxx);
          dense_symset(c, tg + "s.yy", ky, ky, 1, cyy);
          dense_symset(c, tg + "s.yx", kx, ky, 0, cyx);
          Pc.np = 3;
          Pc.ps[0] = {xp, kx, xp, xl, kx, &cxx.R, {}, &cxx, xl};
          Pc.ps[1] = {yp, ky, yp, yl, ky, &cyy.R, {}, &cyy, yl};
          Pc.ps[2] = {xp, kx, yp, yl, ky, &cyx.R, {}, &cyx, xl};
          ccol.tot[0] = c->buf<float>(tg + "s.totx", kx);
          ccol.tot[1] = c->buf<float>(tg + "s.toty", ky);
          ccol.tot[2] = c->buf<float>(tg + "s.totxy", ky);
          ccol.yrows = yp;
          ccol.xcols = xp;
          ccol.x_lw2 = xl;
          ccol.n = kx;
          ccol.m = ky;
          ccol.uniform = false;
        } else {
          dense_rangeset(c, tg + ".xx", kx, kx, rxx);
          dense_rangeset(c, tg + ".yy", ky, ky, ryy);
          dense_rangeset(c, tg + ".xy", ky, kx, rxy);
          dense_rangeset(c, tg + ".yx", kx, ky, ryx);
          sym_specs(Pc, xp, xl, kx, yp, yl, ky, &rxx, &ryy, &rxy, &ryx);
        }
        Pc.skip_p0 = c->self_mode == 2;
        build_plan(c, "p" + tg, Pc);
        const double cfull = double(kx) * kx + double(ky) * ky + 2.0 * double(kx) * ky;
        for (int t = t0; t < t1; ++t) {
          ss.scale = t;
          if (conce)
            sym_step_once(c, Pc, Uq, qcur, eps[t], lam[t], false, ss, ccol);
          else
            sym_step(c, Pc, Uq, qcur, eps[t], lam[t], false, ss);
          S->pairs_dense += cfull;
        }
      };
      Potentials Uc;
      alloc_pots(c, "cpot", X.k, Y.k, Uc);
      int ccur = 0;
      // super level (policy.h:msot_super_switch): the first t2 scales on
      // super voxels, inherited by the clusters
      const int t2 = msot_super_switch(sig.data(), tsw, cell, d, std::max(X.k, Y.k),
                                       prm->super_level);
      if (t2 > 0) {
        SuperMeasure SX, SY;
        const DMeasure* ms2[2] = {&X, &Y};
        const char* tg2[2] = {"x", "y"};
        SuperMeasure* ss2[2] = {&SX, &SY};
        super_measures(c, ms2, tg2, d, ss2, 2);
        S->t_super = t2;
        S->k_super_x = SX.k;
        S->k_super_y = SY.k;
        Potentials U2;
        alloc_pots(c, "spot", SX.k, SY.k, U2);
        int scur = 0;
        coarse_run("u", SX.cpts, SX.clw2, SX.k, SY.cpts, SY.clw2, SY.k, U2, scur, 0, t2);
        float** so = U2.v[scur];
        float** ci = Uc.v[ccur];
        CK(inherit(so[0], SX.labels, X.k, ci[0], st));
        CK(inherit(so[1], SY.labels, Y.k, ci[1], st));
        CK(inherit(so[2], SY.labels, Y.k, ci[2], st));
        CK(inherit(so[3], SX.labels, X.k, ci[3], st));
      }
      coarse_run("c", X.cpts, X.clw2, X.k, Y.cpts, Y.clw2, Y.k, Uc, ccur, t2, tsw);
      c->mark(2);  // phase 2: coarse -> fine transfer
      // inheritance (transfer_rule 0) writes the fine
      // potentials directly; extrapolation (transfer_rule 1) is one
      // lambda-damped softmin of every fine atom against the coarse measure,
      // expanded around the inherited value.
      float** co = Uc.v[ccur];
      for (int q = 0; q < 4; ++q) coarse_final[q] = co[q];
      const bool extrap = prm->transfer_rule == 1;
      float* inh[4];
      for (int q = 0; q < 4; ++q) inh[q] = U.v[extrap ? cur ^ 1 : cur][q];
      CK(inherit(co[0], X.labels, n, inh[0], st));
      CK(inherit(co[1], Y.labels, m, inh[1], st));
      CK(inherit(co[2], Y.labels, m, inh[2], st));
      CK(inherit(co[3], X.labels, n, inh[3], st));
    }
    if (tsw > 0 && prm->transfer_rule == 1) {
      float** co = coarse_final;
      float* inh[4];
      for (int q = 0; q < 4; ++q) inh[q] = U.v[cur ^ 1][q];
      RangeSet exx, eyy, exy, eyx;
      dense_rangeset(c, "e.xx", n, X.k, exx, &X.offsets_h);
      dense_rangeset(c, "e.yy", m, Y.k, eyy, &Y.offsets_h);
      dense_rangeset(c, "e.xy", m, X.k, exy, &Y.offsets_h);
      dense_rangeset(c, "e.yx", n, Y.k, eyx, &X.offsets_h);
      Plan Pe;
      Pe.np = 4;
      Pe.ps[0] = {X.pts, n, X.cpts, X.clw2, X.k, &exx};
      Pe.ps[1] = {Y.pts, m, Y.cpts, Y.clw2, Y.k, &eyy};
      Pe.ps[2] = {Y.pts, m, X.cpts, X.clw2, X.k, &exy};
      Pe.ps[3] = {X.pts, n, Y.cpts, Y.clw2, Y.k, &eyx};
      build_plan(c, "pe", Pe);
      ScaleArgs a{};
      a.h[0] = co[0]; a.est[0] = inh[0]; a.out[0] = U.v[cur][0];
      a.h[1] = co[1]; a.est[1] = inh[1]; a.out[1] = U.v[cur][1];
      a.h[2] = co[3]; a.est[2] = inh[2]; a.out[2] = U.v[cur][2];
      a.h[3] = co[2]; a.est[3] = inh[3]; a.out[3] = U.v[cur][3];
      a.eps = eps[tsw - 1];
      a.lam = lam[tsw - 1];
      a.mixw = 1.0;
      run_group(c, Pe, a, ss);
    }
    // fine phase: block-sparse updates restricted to the truncation masks
    uint32_t* mxx = c->buf<uint32_t>("m.xx", size_t(X.k) * mask_words(X.k));
    uint32_t* myy = c->buf<uint32_t>("m.yy", size_t(Y.k) * mask_words(Y.k));
    uint32_t* mxy = c->buf<uint32_t>("m.xy", size_t(X.k) * mask_words(Y.k));
    uint32_t* myx = c->buf<uint32_t>("m.yx", size_t(Y.k) * mask_words(X.k));
    float* fmax[4];
    fmax[0] = c->buf<float>("m.Fxx", X.k);
    fmax[1] = c->buf<float>("m.Gyy", Y.k);
    fmax[2] = c->buf<float>("m.Gxy", Y.k);
    fmax[3] = c->buf<float>("m.Fyx", X.k);
    float4* grad[4];
    grad[0] = c->buf<float4>("m.gxx", X.k);
    grad[1] = c->buf<float4>("m.gyy", Y.k);
    grad[2] = c->buf<float4>("m.gxy", Y.k);
    grad[3] = c->buf<float4>("m.gyx", X.k);
    RangeSet &rxx = fxx, &ryy = fyy, &rxy = fxy, &ryx = fyx;
    Plan Pf;
    const bool once = prm->pair_eval != 0;
    double mask_terms = 0.0;  // profiling: cluster-granularity terms of the current masks
    SymSet sxx, syy, syx;
    SymCols scol{};
    if (once) {
      scol.labels[0] = X.labels; scol.co[0] = X.offsets; scol.tot[0] = c->buf<float>("s.totx", n);
      scol.labels[1] = Y.labels; scol.co[1] = Y.offsets; scol.tot[1] = c->buf<float>("s.toty", m);
      scol.labels[2] = Y.labels; scol.co[2] = Y.offsets; scol.tot[2] = c->buf<float>("s.totxy", m);
      scol.yrows = Y.pts;
      scol.xcols = X.pts;
      scol.x_lw2 = X.lw2;
      scol.n = n;
      scol.m = m;
      scol.uniform = X.uniform && Y.uniform;
      scol.mask[0] = mxx;
      scol.mask[1] = myy;
      scol.mask[2] = mxy;
      scol.rlab[0] = X.labels; scol.rlab[1] = Y.labels; scol.rlab[2] = X.labels; scol.rlab[3] = Y.labels;
      scol.fco[0] = X.offsets; scol.fco[1] = Y.offsets; scol.fco[2] = Y.offsets; scol.fco[3] = X.offsets;
      scol.words[0] = mask_words(X.k);
      scol.words[1] = scol.words[2] = scol.words[3] = mask_words(Y.k);
      scol.kc3 = X.k;
    }
    auto build_masks = [&](double e) {
      // without a coarse phase there is no information: keep every pair
      const bool info = tsw > 0;
      const double theta = info ? prm->theta : INFINITY;
      if (!info) {
        CK(cudaMemsetAsync(fmax[0], 0, X.k * sizeof(float), st));
        CK(cudaMemsetAsync(fmax[1], 0, Y.k * sizeof(float), st));
        CK(cudaMemsetAsync(fmax[2], 0, Y.k * sizeof(float), st));
        CK(cudaMemsetAsync(fmax[3], 0, X.k * sizeof(float), st));
      } else {
        float** f = U.v[cur];
        CK(cluster_bound(X.pts, X.w64, f[0], X.offsets, X.cpts, X.k, fmax[0], grad[0], st));
        CK(cluster_bound(Y.pts, Y.w64, f[1], Y.offsets, Y.cpts, Y.k, fmax[1], grad[1], st));
        CK(cluster_bound(Y.pts, Y.w64, f[2], Y.offsets, Y.cpts, Y.k, fmax[2], grad[2], st));
        CK(cluster_bound(X.pts, X.w64, f[3], X.offsets, X.cpts, X.k, fmax[3], grad[3], st));
      }
      float4* g[4];
      for (int q = 0; q < 4; ++q) g[q] = (info && prm->mask_rule != 1) ? grad[q] : nullptr;
      // member boxes (mask.cu: B_c) with the slope bound, mask_rule 0
      const float4* bxy[4] = {X.box_lo, X.box_hi, Y.box_lo, Y.box_hi};
      const float4* bxx[4] = {X.box_lo, X.box_hi, X.box_lo, X.box_hi};
      const float4* byy[4] = {Y.box_lo, Y.box_hi, Y.box_lo, Y.box_hi};
      const bool use_box = info && prm->mask_rule == 0;
      const float4* const* Bxy = use_box ? bxy : nullptr;
      const float4* const* Bxx = use_box ? bxx : nullptr;
      const float4* const* Byy = use_box ? byy : nullptr;
      int32_t* bxr = c->buf<int32_t>("m.bx", std::max(X.k, Y.k));
      int32_t* byr = c->buf<int32_t>("m.by", std::max(X.k, Y.k));
      void* bws = c->buf<char>("m.blk", mask_block_ws_bytes(std::max(X.k, Y.k), std::max(X.k, Y.k)));
      if (once) {
        // row-sharded: each rank computes 1/world of the mask rows, the row
        // blocks are exchanged (grouped broadcasts), then the column bests
        // of the cross mask are set from the whole mask on every rank
        const int rk = c->rank, wd = c->world;
        auto cut = [&](int32_t k, int r) { return static_cast<int32_t>(int64_t(k) * r / wd); };
        if (c->self_mode == 2)  // shared self term: the x-x problem is not evaluated
          CK(cudaMemsetAsync(mxx, 0, size_t(X.k) * mask_words(X.k) * sizeof(uint32_t), st));
        else
          CK(truncation_masks_rows(X.k, X.k, d, X.cpts, X.radii, fmax[0], g[0], X.cpts, X.radii,
                                   fmax[0], g[0], e, theta, 1, cut(X.k, rk), cut(X.k, rk + 1),
                                   mxx, bxr, bws, st, Bxx));
        CK(truncation_masks_rows(Y.k, Y.k, d, Y.cpts, Y.radii, fmax[1], g[1], Y.cpts, Y.radii,
                                 fmax[1], g[1], e, theta, 1, cut(Y.k, rk), cut(Y.k, rk + 1), myy,
                                 byr, bws, st, Byy));
        CK(truncation_masks_rows(X.k, Y.k, d, X.cpts, X.radii, fmax[3], g[3], Y.cpts, Y.radii,
                                 fmax[2], g[2], e, theta, 0, cut(X.k, rk), cut(X.k, rk + 1), mxy,
                                 bxr, bws, st, Bxy));
        if (wd > 1 || c->comm) {
          std::vector<int64_t> bnd[3];
          const int32_t kr[3] = {X.k, Y.k, X.k}, kc[3] = {X.k, Y.k, Y.k};
          for (int q = 0; q < 3; ++q) {
            bnd[q].resize(wd + 1);
            for (int r = 0; r <= wd; ++r) bnd[q][r] = int64_t(cut(kr[q], r)) * mask_words(kc[q]);
          }
          float* mb[3] = {reinterpret_cast<float*>(mxx), reinterpret_cast<float*>(myy),
                          reinterpret_cast<float*>(mxy)};  // 32-bit words, moved as bytes
          coll_bcast_rows(c, mb, bnd, 3);
        }
        CK(truncation_masks_cols(X.k, Y.k, d, X.cpts, X.radii, fmax[3], g[3], Y.cpts, Y.radii,
                                 fmax[2], g[2], mxy, byr, bws, st, Bxy));
      } else {
        CK(truncation_masks(X.k, X.k, d, X.cpts, X.radii, fmax[0], g[0], X.cpts, X.radii, fmax[0],
                            g[0], e, theta, 1, mxx, nullptr, bxr, nullptr, bws, st, Bxx));
        CK(truncation_masks(Y.k, Y.k, d, Y.cpts, Y.radii, fmax[1], g[1], Y.cpts, Y.radii, fmax[1],
                            g[1], e, theta, 1, myy, nullptr, byr, nullptr, bws, st, Byy));
        // cross pair: (F, G) = (max b_yx, max a_xy); the slack is symmetric, so
        // the yx mask (rows y) is the exact transpose of the xy mask (rows x)
        CK(truncation_masks(X.k, Y.k, d, X.cpts, X.radii, fmax[3], g[3], Y.cpts, Y.radii, fmax[2],
                            g[2], e, theta, 0, mxy, myx, bxr, byr, bws, st, Bxy));
      }
      if (once && (c->profiling || c->cap_scale >= tsw)) {
        // whole self masks for the pair count and the debug capture
        CK(mask_mirror(mxx, X.k, st));
        CK(mask_mirror(myy, Y.k, st));
      }
      if (c->profiling) {  // cluster-granularity pair count of the four masks
        double* cnt = c->buf<double>("m.cnt", 1);
        CK(cudaMemsetAsync(cnt, 0, sizeof(double), st));
        CK(mask_pair_count(mxx, X.k, X.k, X.offsets, X.offsets, cnt, st));
        CK(mask_pair_count(myy, Y.k, Y.k, Y.offsets, Y.offsets, cnt, st));
        CK(mask_pair_count(mxy, X.k, Y.k, X.offsets, Y.offsets, cnt, st));
        if (once)  // myx is not built: the transpose has the same count
          CK(mask_pair_count(mxy, X.k, Y.k, X.offsets, Y.offsets, cnt, st));
        else
          CK(mask_pair_count(myx, Y.k, X.k, Y.offsets, X.offsets, cnt, st));
        double h = 0.0;
        CK(cudaMemcpyAsync(&h, cnt, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(host_sync(__LINE__, st));
        mask_terms = h;
      }
      if (once) {  // evaluate-once pair sets (oracle.cpp: sym_self, transpose_ranges)
        sym_rangesets(c, {{"s.xx", X.labels, &X.offsets_h, n, X.offsets, X.k, mxx, 1, &sxx},
                          {"s.yy", Y.labels, &Y.offsets_h, m, Y.offsets, Y.k, myy, 1, &syy},
                          {"s.yx", X.labels, &X.offsets_h, n, Y.offsets, Y.k, mxy, 0, &syx}});
        Pf.np = 3;
        Pf.ps[0] = {X.pts, n, X.pts, X.lw2, n, &sxx.R, {}, &sxx, X.lw2};
        Pf.ps[1] = {Y.pts, m, Y.pts, Y.lw2, m, &syy.R, {}, &syy, Y.lw2};
        Pf.ps[2] = {X.pts, n, Y.pts, Y.lw2, m, &syx.R, {}, &syx, X.lw2};
      } else {
        mask_rangeset(c, "f.xx", X.labels, X.offsets_h, n, X.offsets, X.k, mxx, rxx);
        mask_rangeset(c, "f.yy", Y.labels, Y.offsets_h, m, Y.offsets, Y.k, myy, ryy);
        mask_rangeset(c, "f.yx", X.labels, X.offsets_h, n, Y.offsets, Y.k, mxy, ryx);  // rows x, cols y
        mask_rangeset(c, "f.xy", Y.labels, Y.offsets_h, m, X.offsets, X.k, myx, rxy);  // rows y, cols x
        sym_specs(Pf, X.pts, X.lw2, n, Y.pts, Y.lw2, m, &rxx, &ryy, &rxy, &ryx);
      }
      Pf.skip_p0 = c->self_mode == 2;
      build_plan(c, "pf", Pf);
    };
    for (int t = tsw; t <= ns; ++t) {
      const int tt = std::min(t, ns - 1);
      ss.scale = t;
      const bool rebuild =
          (t == tsw) || (prm->retruncate > 0 && t < ns && (t - tsw) % prm->retruncate == 0);
      if (rebuild) {
        c->mark(3);  // phase 3: truncation masks, ranges, work items
        build_masks(eps[tt]);
      }
      c->mark(4);
      const bool cap = t == c->cap_scale;
      if (cap) capture_pots(c, U.v[cur], X.perm, Y.perm, n, m, c->cap_in);
      if (once)
        sym_step_once(c, Pf, U, cur, eps[tt], lam[tt], t == ns, ss, scol);
      else
        sym_step(c, Pf, U, cur, eps[tt], lam[tt], t == ns, ss);
      if (cap) {
        capture_pots(c, U.v[cur], X.perm, Y.perm, n, m, c->cap_out);
        const uint32_t* mk[3] = {mxx, myy, mxy};
        const int32_t kr[3] = {X.k, Y.k, X.k}, kc[3] = {X.k, Y.k, Y.k};
        capture_masks(c, mk, kr, kc, X, Y);
      }
      S->pairs_dense += full;
      S->pairs_fine += Pf.pairs_all;
      S->pairs_fine_dense += full;
      S->pairs_mask_terms += mask_terms;
    }
    if (once && d_grad) {  // the plans of grad_positions read per-row ranges
      CK(mask_mirror(mxx, X.k, st));
      mask_rangeset(c, "f.xx", X.labels, X.offsets_h, n, X.offsets, X.k, mxx, fxx);
      mask_rangeset(c, "f.yx", X.labels, X.offsets_h, n, Y.offsets, Y.k, mxy, fyx);
    }
  }
  }  // d <= 3

  // grad_positions from the final potentials, on the pair
  // sets of the last update: cross plan (rows x, cols y) and self plan
  // shared self term (msot_barycenter): this solve skipped the x-x problem,
  // its final a_xx is the recorded one (caller order -> this solve's order)
  if (c->self_mode == 2) CK(inherit(c->self_axx, X.perm, n, U.v[cur][0], st));
  if (d_grad) {
    c->mark(5);
    float** f = U.v[cur];
    const ProbSpec specs[2] = {{X.pts, n, Y.pts, Y.lw2, m, &fyx}, {X.pts, n, X.pts, X.lw2, n, &fxx}};
    const float* fr[2] = {f[3], f[0]};  // b_yx, a_xx
    const float* gc[2] = {f[2], f[0]};  // a_xy, a_xx
    const float4* pay[2] = {Y.pts, X.pts};
    float4* outp[2] = {c->buf<float4>("grad.pxy", n), c->buf<float4>("grad.pxx", n)};
    // the recorded payload {mass, sum pi x} is kept in absolute coordinates
    // (each solve centres its float32 atoms on its own bounding box)
    if (c->self_mode == 2) {  // cross plan only; the self plan's payload is recorded
      plan_group(c, "pg", 1, specs, fr, gc, pay, outp, eps[ns - 1], d);
      CK(gather_f4(c->self_pay, X.perm, n, outp[1], st));
      CK(shift_payload(outp[1], n, -frame[0], -frame[1], -frame[2], st));
    } else {
      plan_group(c, "pg", 2, specs, fr, gc, pay, outp, eps[ns - 1], d);
    }
    if (c->self_mode == 1) {
      CK(scatter_f4(outp[1], X.perm, n, c->self_pay, st));
      CK(shift_payload(c->self_pay, n, frame[0], frame[1], frame[2], st));
      CK(scatter_f32(f[0], X.perm, n, c->self_axx, st));
    }
    CK(grad_positions(X.pts, X.w64, outp[0], outp[1], X.perm, n, d, d_grad, st));
  } else if (c->self_mode == 1) {
    CK(scatter_f32(U.v[cur][0], X.perm, n, c->self_axx, st));
  }

  // transfer_labels (K9) from the final cross potentials
  if (lreq) {
    c->mark(6);
    float** f = U.v[cur];
    transfer_labels_dev(c, *lreq, X, Y, nr, m, d, d_y, hd_cen, hd_ax, hd_sqx, f[3], f[2],
                        eps[ns - 1]);
  }

  // divergence (eq. 5-6), fixed-order float64
  const double rho = msot_reach_is_inf(prm->reach) ? 0.0 : std::pow(prm->reach, prm->p);
  c->mark(5);
  const int nb = 256;
  double* partials = c->buf<double>("loss.part", 5 * nb);
  double* lout = c->buf<double>("loss.out", 4);
  float** f = U.v[cur];
  CK(divergence_partial(X.w64, Y.w64, nr, mr, f[0], f[1], f[2], f[3], rho, partials, nb, st));
  CK(divergence_final(partials, nb, eps[ns - 1], rho, lout, st));
  double res[4];
  int32_t fbt = 0;
  CK(cudaMemcpyAsync(res, lout, sizeof(res), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&fbt, ss.fb_total, sizeof(fbt), cudaMemcpyDeviceToHost, st));
  int32_t bad = 0x7f7f7f7f;
  CK(cudaMemcpyAsync(&bad, ss.bad_scale, sizeof(bad), cudaMemcpyDeviceToHost, st));
  if (h_pots) {
    double* tmp = c->buf<double>("unsort", std::max(n, m));
    const int64_t len[4] = {nr, mr, mr, nr};   // internal rows (padding skipped by perm < 0)
    const int64_t outn[4] = {n, m, m, n};
    const int32_t* perm[4] = {X.perm, Y.perm, Y.perm, X.perm};
    // canonical gauge of the balanced cross pair (loss.cu): a_xy - c, b_yx + c
    const double sign[4] = {0.0, 0.0, -1.0, 1.0};
    for (int q = 0; q < 4; ++q) {
      if (!h_pots[q]) continue;
      CK(scatter_unsort(f[q], perm[q], len[q], lout + 3, sign[q], tmp, st));
      CK(cudaMemcpyAsync(h_pots[q], tmp, outn[q] * sizeof(double), cudaMemcpyDeviceToHost, st));
      CK(host_sync(__LINE__, st));
      S->d2h_bytes += outn[q] * sizeof(double);
    }
  }
  c->mark(-1);
  CK(cudaEventRecord(c->t1, st));
  CK(host_sync(__LINE__, st));
  float ms_total = 0.f;
  CK(cudaEventElapsedTime(&ms_total, c->t0, c->t1));
  S->total_ms = ms_total;
  if (c->profiling) {
    double acc = 0.0;
    for (size_t k = 0; k + 1 < c->ev_used; k += 2) {
      float e = 0.f;
      CK(cudaEventElapsedTime(&e, c->ev[k], c->ev[k + 1]));
      acc += e;
    }
    S->softmin_ms = acc;
    for (size_t k = 0; k + 1 < c->marks.size(); ++k) {
      float e = 0.f;
      CK(cudaEventElapsedTime(&e, c->marks[k].second, c->marks[k + 1].second));
      const int ph = c->marks[k].first;
      if (ph >= 0 && ph < 8) S->phase_ms[ph] += e;
    }
  }
  S->fallback_rows = fbt;
  S->gpu_launches = g_launches - launches0;
  S->host_syncs = g_host_syncs - syncs0;
  if (getenv("MSOT_DEBUG_SYNCS")) {
    for (const auto& kv : g_sync_sites) fprintf(stderr, "[msot] sync at solver.cu:%d x%d\n", kv.first, kv.second);
    g_sync_sites.clear();
  }
  S->device_bytes = 0.0;
  for (const auto& kv : c->bufs) S->device_bytes += static_cast<double>(kv.second.second);
  S->d2h_bytes += sizeof(res);
  if (bad != 0x7f7f7f7f) {  // NumericError naming the scale
    const int t = std::min(bad, ns - 1);
    raise(MSOT_ENUMERIC, "non-finite potential at scale " + std::to_string(bad) + " of " +
                             std::to_string(ns) + (bad >= ns ? " (final update" : " (") +
                             ", sigma = " + std::to_string(sig[t]) + ")");
  }
  if (!std::isfinite(res[0])) raise(MSOT_ENUMERIC, "non-finite divergence");
  *loss_out = res[0];
}

}  // namespace

// =================================================================== C ABI
extern "C" {

const char* msot_last_error(void) { return g_err.c_str(); }

void msot_params_default(msot_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->blur = 0.05;
  p->reach = INFINITY;
  p->p = 2.0;
  p->scaling = 0.9;
  p->multiscale = 0;
  p->retruncate = 0;
  p->cluster_scale = 0.0;
  p->theta = 20.0;
  p->switch_factor = 2.0;
  p->max_full_iters = 10000;
  p->pair_eval = 1;
  p->super_level = -1;
}

int msot_schedule(double diameter, const msot_params* p, double* sigma, double* eps, double* lam,
                  int cap) {
  if (!msot_reach_valid(p->reach)) {  // 0 = invalid parameters (n >= 1 otherwise)
    g_err = "reach must be > 0 (or +inf for balanced OT)";
    return 0;
  }
  const int n = msot_schedule_len(diameter, p->blur, p->scaling);
  if (n > cap) return -n;
  for (int t = 0; t < n; ++t) {
    sigma[t] = msot_schedule_sigma(diameter, p->blur, p->scaling, n, t);
    eps[t] = std::pow(sigma[t], p->p);
    lam[t] = msot_lambda(eps[t], p);
  }
  return n;
}

int msot_shard_tiles(const double* work, int64_t n_tiles, int world, int64_t* bounds) {
  if (world < 1 || n_tiles < 0) {
    g_err = "invalid shard request";
    return MSOT_EUSAGE;
  }
  std::vector<double> w(work, work + n_tiles);
  std::vector<int64_t> b;
  shard_tiles(w, world, b);
  std::copy(b.begin(), b.end(), bounds);
  return MSOT_OK;
}

static int create_common(int device, msot_ctx** out, msot_ctx* c) {
  if (const char* e = getenv("MSOT_COLPART_BUDGET")) c->colpart_budget = atoll(e);
  if (const char* e = getenv("MSOT_FORCE_FALLBACK")) c->force_fb = atoi(e) != 0;
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking));
  for (int k = 0; k < 2; ++k) {
    CK(cudaStreamCreateWithFlags(&c->side[k], cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_cs[k], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreate(&c->t0));
  CK(cudaEventCreate(&c->t1));
  CK(cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device));
  c->device = device;
  *out = c;
  return MSOT_OK;
}

int msot_create(int device, msot_ctx** out) {
  return guard([&] {
    auto* c = new msot_ctx();
    try {
      create_common(device, out, c);
    } catch (...) {
      delete c;
      throw;
    }
  });
}

int msot_nccl_unique_id(unsigned char out[128]) {
  return guard([&] {
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out, &id, 128);
  });
}

int msot_create_dist(int device, int rank, int world, const unsigned char nccl_id[128],
                     msot_ctx** out) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) raise(MSOT_EUSAGE, "invalid rank/world");
    auto* c = new msot_ctx();
    try {
      create_common(device, out, c);
      c->rank = rank;
      c->world = world;
      {  // world 1 too: a one-rank communicator (see coll_allreduce)
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, 128);
        NK(ncclCommInitRank(&c->comm, world, id, rank));
      }
    } catch (...) {
      delete c;
      *out = nullptr;
      throw;
    }
  });
}

int msot_debug_capture(msot_ctx* c, int scale, double* const in[4], double* const out[4]) {
  return guard([&] {
    if (!c) raise(MSOT_EUSAGE, "null context");
    c->cap_scale = scale;
    for (int q = 0; q < 4; ++q) {
      c->cap_in[q] = scale >= 0 && in ? in[q] : nullptr;
      c->cap_out[q] = scale >= 0 && out ? out[q] : nullptr;
    }
  });
}

int msot_debug_mask(const msot_ctx* c, int which, int32_t* k_rows, int32_t* k_cols,
                    uint8_t* mask, int32_t* row_cluster, int32_t* col_cluster) {
  return guard([&] {
    if (!c || which < 0 || which > 2) raise(MSOT_EUSAGE, "invalid mask request");
    if (c->cap_mask[which].empty()) raise(MSOT_EUSAGE, "no mask captured");
    if (k_rows) *k_rows = c->cap_k[which][0];
    if (k_cols) *k_cols = c->cap_k[which][1];
    if (mask) std::memcpy(mask, c->cap_mask[which].data(), c->cap_mask[which].size());
    const std::vector<int32_t>& rl = c->cap_lab[which == 1 ? 1 : 0];
    const std::vector<int32_t>& cl = c->cap_lab[which == 0 ? 0 : 1];
    if (row_cluster) std::copy(rl.begin(), rl.end(), row_cluster);
    if (col_cluster) std::copy(cl.begin(), cl.end(), col_cluster);
  });
}

int msot_world_info(const msot_ctx* c, int* rank, int* world, int* comm_ranks) {
  return guard([&] {
    if (!c) raise(MSOT_EUSAGE, "null context");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
    if (comm_ranks) {
      int n = c->world > 1 ? 0 : 1;  // msot_create: no communicator at world 1
      if (c->comm) NK(ncclCommCount(c->comm, &n));
      else if (c->host_ar) n = c->world;  // host-collective test seam
      *comm_ranks = n;
    }
  });
}

int msot_create_dist_host(int device, int rank, int world, msot_host_allreduce_fn allreduce,
                          msot_host_broadcast_fn broadcast, void* user, msot_ctx** out) {
  return guard([&] {
    if (world < 1 || rank < 0 || rank >= world) raise(MSOT_EUSAGE, "invalid rank/world");
    if (!allreduce || !broadcast) raise(MSOT_EUSAGE, "both host collectives are required");
    auto* c = new msot_ctx();
    try {
      create_common(device, out, c);
      c->rank = rank;
      c->world = world;
      c->host_ar = allreduce;
      c->host_bc = broadcast;
      c->host_user = user;
    } catch (...) {
      delete c;
      *out = nullptr;
      throw;
    }
  });
}

void msot_destroy(msot_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  if (getenv("MSOT_DEBUG_BUFS")) {  // dev: the buffer table, largest first
    std::vector<std::pair<size_t, std::string>> v;
    for (auto& kv : c->bufs) v.push_back({kv.second.second, kv.first});
    std::sort(v.rbegin(), v.rend());
    size_t tot = 0;
    for (auto& e : v) tot += e.first;
    fprintf(stderr, "[msot] %zu buffers, %.1f MB\n", v.size(), tot / 1e6);
    for (size_t k = 0; k < v.size() && k < 40; ++k)
      fprintf(stderr, "[msot]   %10.3f MB  %s\n", v[k].first / 1e6, v[k].second.c_str());
  }
  for (auto& kv : c->bufs) cudaFree(kv.second.first);
  for (auto e : c->ev) cudaEventDestroy(e);
  for (auto e : c->mark_pool) cudaEventDestroy(e);
  if (c->t0) cudaEventDestroy(c->t0);
  if (c->t1) cudaEventDestroy(c->t1);
  if (c->comm) ncclCommDestroy(c->comm);
  for (int k = 0; k < 2; ++k) {
    if (c->side[k]) cudaStreamDestroy(c->side[k]);
    if (c->ev_cs[k]) cudaEventDestroy(c->ev_cs[k]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->pin_base) cudaFreeHost(c->pin_base);
  if (c->st) cudaStreamDestroy(c->st);
  delete c;
}

int msot_set_profiling(msot_ctx* c, int on) {
  if (!c) return MSOT_EUSAGE;
  c->profiling = on != 0;
  return MSOT_OK;
}

int msot_set_colpart_budget(msot_ctx* c, int64_t slots) {
  if (!c || slots < 0) return MSOT_EUSAGE;
  c->colpart_budget = slots;
  return MSOT_OK;
}

int msot_probe_ex2(msot_ctx* c, double* ex2_per_s) {
  return guard([&] {
    if (!c || !ex2_per_s) raise(MSOT_EUSAGE, "null argument");
    CK(cudaSetDevice(c->device));
    float* sink = c->buf<float>("probe.sink", 256);
    double per = 0.0;
    int blocks = 0;
    const int iters = 4096;
    CK(ex2_probe(c->n_sm, iters, sink, &per, &blocks, c->st));  // warm-up
    CK(cudaEventRecord(c->t0, c->st));
    for (int r = 0; r < 5; ++r) CK(ex2_probe(c->n_sm, iters, sink, &per, &blocks, c->st));
    CK(cudaEventRecord(c->t1, c->st));
    CK(host_sync(__LINE__, c->st));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->t0, c->t1));
    *ex2_per_s = 5.0 * per / (ms * 1e-3);
  });
}

static void check_weights(const double* w, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!(w[i] > 0) || !std::isfinite(w[i])) raise(MSOT_EDATA, "weights must be finite and > 0");
}

int msot_sinkhorn(msot_ctx* c, const msot_params* prm, const double* x, const double* a, int64_t n,
                  const double* y, const double* b, int64_t m, int d, double* a_xx, double* b_yy,
                  double* a_xy, double* b_yx, double* loss_out, msot_stats* stats) {
  return guard([&] {
    if (!c || !prm || !x || !a || !y || !b || !loss_out) raise(MSOT_EUSAGE, "null argument");
    if (n < 1 || m < 1) raise(MSOT_EDATA, "empty measure");
    // weights and points are validated on the device (solve_device)
    CK(cudaSetDevice(c->device));
    msot_stats local{};
    msot_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    S->rank = c->rank;
    S->world = c->world;
    double* dx = c->buf<double>("in.x", n * d);
    double* da = c->buf<double>("in.a", n);
    double* dy = c->buf<double>("in.y", m * d);
    double* db = c->buf<double>("in.b", m);
    CK(cudaMemcpyAsync(dx, x, n * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(da, a, n * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(dy, y, m * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(db, b, m * sizeof(double), cudaMemcpyHostToDevice, c->st));
    S->h2d_bytes = double((n + m) * (d + 1)) * sizeof(double);
    double* hp[4] = {a_xx, b_yy, a_xy, b_yx};
    solve_device(c, prm, dx, da, n, dy, db, m, d, loss_out, S, hp);
  });
}

int msot_sinkhorn_device(msot_ctx* c, const msot_params* prm, const double* d_x, const double* d_a,
                         int64_t n, const double* d_y, const double* d_b, int64_t m, int d,
                         double* loss_out, msot_stats* stats) {
  return guard([&] {
    if (!c || !prm || !d_x || !d_a || !d_y || !d_b || !loss_out) raise(MSOT_EUSAGE, "null argument");
    CK(cudaSetDevice(c->device));
    msot_stats local{};
    msot_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    S->rank = c->rank;
    S->world = c->world;
    solve_device(c, prm, d_x, d_a, n, d_y, d_b, m, d, loss_out, S, nullptr);
  });
}

int msot_sinkhorn_grad(msot_ctx* c, const msot_params* prm, const double* x, const double* a,
                       int64_t n, const double* y, const double* b, int64_t m, int d,
                       double* loss_out, double* grad_x, msot_stats* stats) {
  return guard([&] {
    if (!c || !prm || !x || !a || !y || !b || !loss_out || !grad_x) raise(MSOT_EUSAGE, "null argument");
    if (n < 1 || m < 1) raise(MSOT_EDATA, "empty measure");
    if (prm->p != 2.0) raise(MSOT_EUSAGE, "grad_positions is defined for p = 2 (SPEC.md:348)");
    check_weights(a, n);
    check_weights(b, m);
    CK(cudaSetDevice(c->device));
    msot_stats local{};
    msot_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    S->rank = c->rank;
    S->world = c->world;
    double* dx = c->buf<double>("in.x", n * d);
    double* da = c->buf<double>("in.a", n);
    double* dy = c->buf<double>("in.y", m * d);
    double* db = c->buf<double>("in.b", m);
    double* dg = c->buf<double>("in.grad", n * d);
    CK(cudaMemcpyAsync(dx, x, n * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(da, a, n * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(dy, y, m * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(db, b, m * sizeof(double), cudaMemcpyHostToDevice, c->st));
    solve_device(c, prm, dx, da, n, dy, db, m, d, loss_out, S, nullptr, dg);
    CK(cudaMemcpyAsync(grad_x, dg, n * d * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(host_sync(__LINE__, c->st));
  });
}

int msot_resolve_flips(const double* scores, const double* row_mass, int64_t n, int n_classes,
                       const int32_t* flip_of, const int32_t* orientation, double* scores_out,
                       double* row_mass_out, int32_t* chosen) {
  return guard([&] {
    if (!scores || !row_mass || !flip_of || !orientation || !scores_out || !row_mass_out || !chosen)
      raise(MSOT_EUSAGE, "null argument");
    if (n < 0 || n % 2 != 0 || n_classes < 1) raise(MSOT_EDATA, "need an even number of rows");
    const int64_t no = n / 2;
    std::vector<int64_t> row(2 * no, -1);  // [original][orientation] -> augmented row
    for (int64_t i = 0; i < n; ++i) {
      const int64_t o = flip_of[i];
      const int32_t r = orientation[i];
      if (o < 0 || o >= no || (r != 0 && r != 1)) raise(MSOT_EDATA, "flip map out of range");
      if (row[2 * o + r] >= 0) raise(MSOT_EDATA, "duplicate entry in the flip map");
      row[2 * o + r] = i;
    }
    for (int64_t o = 0; o < no; ++o) {
      if (row[2 * o] < 0 || row[2 * o + 1] < 0) raise(MSOT_EDATA, "missing flip pair");
      const int64_t a = row[2 * o], b = row[2 * o + 1];
      const int64_t k = row_mass[b] > row_mass[a] ? b : a;  // ties -> original
      chosen[o] = static_cast<int32_t>(k);
      row_mass_out[o] = row_mass[k];
      std::memcpy(scores_out + o * n_classes, scores + k * n_classes, n_classes * sizeof(double));
    }
  });
}

int msot_classify(const double* scores, const double* row_mass, int64_t n, int n_classes,
                  double tau, int32_t* label, double* confidence) {
  return guard([&] {
    if (!scores || !row_mass || !label || !confidence) raise(MSOT_EUSAGE, "null argument");
    if (n_classes < 1) raise(MSOT_EUSAGE, "classify needs at least one class");
    for (int64_t i = 0; i < n; ++i) {
      const double* s = scores + i * n_classes;
      int best = 0;
      for (int l = 1; l < n_classes; ++l)
        if (s[l] > s[best]) best = l;
      const bool out = row_mass[i] < tau;
      label[i] = out ? -1 : best;
      confidence[i] = row_mass[i] > 0 ? s[best] / row_mass[i] : 0.0;
    }
  });
}

int msot_transfer_labels(msot_ctx* c, const msot_params* prm, const double* x, const double* a,
                         int64_t n, const double* y, const double* b, int64_t m, int d,
                         const int32_t* labels, int n_classes, double* scores, double* row_mass,
                         double* loss_out, msot_stats* stats) {
  return guard([&] {
    if (!c || !prm || !x || !a || !y || !b || !labels || !scores || !row_mass || !loss_out)
      raise(MSOT_EUSAGE, "null argument");
    if (n < 1 || m < 1) raise(MSOT_EDATA, "empty measure");
    if (n_classes < 1) raise(MSOT_EUSAGE, "transfer_labels needs at least one class");
    for (int64_t j = 0; j < m; ++j)
      if (labels[j] < 0 || labels[j] >= n_classes) raise(MSOT_EDATA, "label outside [0, L)");
    check_weights(a, n);
    check_weights(b, m);
    CK(cudaSetDevice(c->device));
    msot_stats local{};
    msot_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    S->rank = c->rank;
    S->world = c->world;
    double* dx = c->buf<double>("in.x", n * d);
    double* da = c->buf<double>("in.a", n);
    double* dy = c->buf<double>("in.y", m * d);
    double* db = c->buf<double>("in.b", m);
    CK(cudaMemcpyAsync(dx, x, n * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(da, a, n * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(dy, y, m * d * sizeof(double), cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(db, b, m * sizeof(double), cudaMemcpyHostToDevice, c->st));
    LabelReq q{labels, n_classes, c->buf<double>("lab.scores", size_t(n) * n_classes),
               c->buf<double>("lab.mass", n)};
    solve_device(c, prm, dx, da, n, dy, db, m, d, loss_out, S, nullptr, nullptr, &q);
    CK(cudaMemcpyAsync(scores, q.d_scores, size_t(n) * n_classes * sizeof(double),
                       cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(row_mass, q.d_mass, n * sizeof(double), cudaMemcpyDeviceToHost, c->st));
    CK(host_sync(__LINE__, c->st));
  });
}

// Wasserstein barycenter by descent on the atom positions (SPEC.md:356-364,
// PAPER.md:374-386): minimise (1/K) sum_k S(alpha, beta_k) over x with frozen
// weights; field = mean_k grad_k / a_i; x <- x - step * field, the step
// halved (up to 10 times) until the loss does not increase; stops after
// `iters` accepted steps or when the relative decrease falls below `tol`.
int msot_barycenter(msot_ctx* c, const msot_params* prm, const double* x0, const double* a,
                    int64_t n, int k, const double* const* ys, const double* const* bs,
                    const int64_t* ms, int d, int iters, double step, double tol, double* x_out,
                    double* loss_traj, int* steps_done, msot_stats* stats) {
  return guard([&] {
    if (!c || !prm || !x0 || !a || !ys || !bs || !ms || !x_out || k < 1 || iters < 0)
      raise(MSOT_EUSAGE, "invalid barycenter arguments");
    if (prm->p != 2.0) raise(MSOT_EUSAGE, "barycenter descent is defined for p = 2");
    if (!msot_reach_is_inf(prm->reach)) raise(MSOT_EUSAGE, "barycenter requires reach = inf (SPEC.md:332)");
    if (!(step > 0)) raise(MSOT_EUSAGE, "step must be > 0");
    check_weights(a, n);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    msot_stats local{};
    msot_stats* S = stats ? stats : &local;
    std::memset(S, 0, sizeof(*S));
    S->rank = c->rank;
    S->world = c->world;
    double* dx = c->buf<double>("bc.x", n * d);
    double* dxn = c->buf<double>("bc.xnew", n * d);
    double* da = c->buf<double>("bc.a", n);
    double* field = c->buf<double>("bc.field", n * d);
    double* fieldn = c->buf<double>("bc.fieldnew", n * d);
    double* grad = c->buf<double>("bc.grad", n * d);
    std::vector<double*> dy(k), db(k);
    for (int t = 0; t < k; ++t) {
      if (ms[t] < 1) raise(MSOT_EDATA, "empty target measure");
      check_weights(bs[t], ms[t]);
      dy[t] = c->buf<double>("bc.y" + std::to_string(t), ms[t] * d);
      db[t] = c->buf<double>("bc.b" + std::to_string(t), ms[t]);
      CK(cudaMemcpyAsync(dy[t], ys[t], ms[t] * d * sizeof(double), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(db[t], bs[t], ms[t] * sizeof(double), cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(dx, x0, n * d * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(da, a, n * sizeof(double), cudaMemcpyHostToDevice, st));
    // The K solves of one evaluation share one eps schedule (diameter of the
    // union of the barycenter and every target) and therefore one x-x self
    // term: target 0's solve records its final a_xx and self-plan payload,
    // the others skip the x-x problem (its work is ~N/M times the cross
    // problem's) and use them (the test oracle's barycenter does the same).
    struct SelfScope {
      msot_ctx* c;
      ~SelfScope() {
        c->self_mode = 0;
        c->diam_override = 0.0;
      }
    } scope{c};
    c->self_axx = c->buf<float>("bc.saxx", n);
    c->self_pay = c->buf<float4>("bc.spay", n);
    long long* lohi = c->buf<long long>("bc.bbox", 2 * d);
    auto union_diameter = [&](const double* xp) {
      CK(bbox(xp, n, d, lohi, true, st));
      for (int t = 0; t < k; ++t) CK(bbox(dy[t], ms[t], d, lohi, false, st));
      std::vector<long long> lh(2 * d);
      CK(cudaMemcpyAsync(lh.data(), lohi, 2 * d * sizeof(long long), cudaMemcpyDeviceToHost, st));
      CK(host_sync(__LINE__, st));
      std::vector<double> lo(d), hi(d);
      bbox_decode(lh.data(), d, lo.data(), hi.data());
      double d2 = 0.0;
      for (int q = 0; q < d; ++q) d2 += (hi[q] - lo[q]) * (hi[q] - lo[q]);
      return std::sqrt(d2);
    };
    // loss and mean gradient at positions xp (into fld)
    auto evaluate = [&](const double* xp, double* fld) {
      CK(cudaMemsetAsync(fld, 0, n * d * sizeof(double), st));
      double tot = 0.0;
      c->diam_override = union_diameter(xp);
      for (int t = 0; t < k; ++t) {
        msot_stats s1{};
        double l = 0.0;
        c->self_mode = t == 0 ? 1 : 2;
        solve_device(c, prm, xp, da, n, dy[t], db[t], ms[t], d, &l, &s1, nullptr, grad);
        CK(field_accumulate(fld, grad, 1.0 / k, n * d, st));
        tot += l;
        S->pairs_evaluated += s1.pairs_evaluated;
        S->pairs_dense += s1.pairs_dense;
        S->softmin_launches += s1.softmin_launches;
        S->gpu_launches += s1.gpu_launches;
        S->total_ms += s1.total_ms;
        S->fallback_rows += s1.fallback_rows;
      }
      return tot / k;
    };
    double L = evaluate(dx, field);
    if (!std::isfinite(L)) raise(MSOT_ENUMERIC, "non-finite barycenter loss at iteration 0");
    if (loss_traj) loss_traj[0] = L;
    int done = 0;
    while (done < iters) {
      // each iteration starts from the configured step; the
      // halvings of a rejected trial apply to that iteration only
      double s = step;
      bool accepted = false;
      double Ln = L;
      for (int h = 0; h <= 10; ++h) {
        CK(bary_step(dxn, dx, field, da, s, n, d, st));
        Ln = evaluate(dxn, fieldn);
        if (!std::isfinite(Ln))
          raise(MSOT_ENUMERIC, "non-finite barycenter loss at iteration " + std::to_string(done + 1));
        if (Ln <= L) {
          accepted = true;
          break;
        }
        s *= 0.5;
      }
      if (!accepted) break;
      std::swap(dx, dxn);
      std::swap(field, fieldn);
      const double rel = (L - Ln) / std::max(std::fabs(L), 1e-300);
      L = Ln;
      ++done;
      if (loss_traj) loss_traj[done] = L;
      if (rel < tol) break;
    }
    CK(cudaMemcpyAsync(x_out, dx, n * d * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    if (steps_done) *steps_done = done;
  });
}

// One dense softmin through the production kernel (rows in caller order).
int msot_softmin(msot_ctx* c, const double* x, int64_t n, const double* y, int64_t m, int d,
                 const double* logw_y, const double* h, double eps, double lambda,
                 const double* f_est, double* f_out) {
  return guard([&] {
    if (!c || !x || !y || !logw_y || !h || !f_out) raise(MSOT_EUSAGE, "null argument");
    if (n < 1 || m < 1) raise(MSOT_EDATA, "empty input");
    if (d < 1 || d > 3) raise(MSOT_EUSAGE, "the GPU softmin supports D in 1..3");
    if (!(eps > 0) || !(lambda > 0)) raise(MSOT_EUSAGE, "eps and lambda must be > 0");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    // centre on the joint bounding box, as the solver does
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < d; ++k) lo[k] = std::min(lo[k], x[i * d + k]), hi[k] = std::max(hi[k], x[i * d + k]);
    for (int64_t j = 0; j < m; ++j)
      for (int k = 0; k < d; ++k) lo[k] = std::min(lo[k], y[j * d + k]), hi[k] = std::max(hi[k], y[j * d + k]);
    // rows: sorted by Morton cube id on the device (compact 256-row tiles),
    // exactly as the solver prepares its measures
    GridSpec g{};
    g.d = d;
    for (int k = 0; k < d; ++k) {
      g.origin[k] = lo[k];
      g.center[k] = 0.5 * (lo[k] + hi[k]);
    }
    g.cell = msot_auto_cell(lo, hi, d, n, m);
    double* dx64 = c->buf<double>("sm.x64", n * d);
    double* dw64 = c->buf<double>("sm.w64", n);
    CK(cudaMemcpyAsync(dx64, x, n * d * sizeof(double), cudaMemcpyHostToDevice, st));
    std::vector<double> ones(n, 1.0);
    CK(cudaMemcpyAsync(dw64, ones.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    DMeasure MX;
    prepare_measure(c, "sm", dx64, dw64, n, d, g, false, MX);
    std::vector<int32_t> perm(n);
    CK(cudaMemcpyAsync(perm.data(), MX.perm, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    std::vector<float4> yp(m);
    std::vector<float> yl(m), hh(m), fe(n, 0.f);
    if (f_est)
      for (int64_t s = 0; s < n; ++s) fe[s] = static_cast<float>(f_est[perm[s]]);
    for (int64_t j = 0; j < m; ++j) {
      float v[3] = {0, 0, 0};
      for (int k = 0; k < d; ++k) v[k] = static_cast<float>(y[j * d + k] - 0.5 * (lo[k] + hi[k]));
      yp[j] = make_float4(v[0], v[1], v[2], 0.f);
      yl[j] = static_cast<float>(logw_y[j] / 0.69314718055994530942);
      hh[j] = static_cast<float>(h[j]);
    }
    float4* dxp = MX.pts;
    float4* dyp = c->buf<float4>("sm.y", m);
    float* dyl = c->buf<float>("sm.yl", m);
    float* dh = c->buf<float>("sm.h", m);
    float* dfe = c->buf<float>("sm.fe", n);
    float* dfo = c->buf<float>("sm.fo", n);
    CK(cudaMemcpyAsync(dyp, yp.data(), m * sizeof(float4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dyl, yl.data(), m * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dh, hh.data(), m * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dfe, fe.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
    RangeSet R;
    dense_rangeset(c, "sm.r", n, m, R);
    Plan P;
    P.np = 1;
    P.ps[0] = {dxp, n, dyp, dyl, m, &R};
    const int rank = c->rank, world = c->world;
    c->rank = 0;
    c->world = 1;  // a single softmin is not sharded
    msot_stats S{};
    SolveState ss{&S, d, c->buf<int32_t>("fb.count", 1), c->buf<int32_t>("fb.total", 1), nullptr, 0};
    ss.fb_cap = static_cast<int32_t>(std::min<int64_t>(n, 1 << 22));
    ss.fb_list = c->buf<int4>("fb.list", std::max<int64_t>(ss.fb_cap, 2 * 1));
    try {
      build_plan(c, "psm", P);
      ScaleArgs a{};
      a.h[0] = dh;
      a.est[0] = dfe;
      a.out[0] = dfo;
      a.eps = eps;
      a.lam = lambda;
      a.mixw = 1.0;
      run_group(c, P, a, ss);
    } catch (...) {
      c->rank = rank;
      c->world = world;
      throw;
    }
    c->rank = rank;
    c->world = world;
    std::vector<float> fo(n);
    CK(cudaMemcpyAsync(fo.data(), dfo, n * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    for (int64_t s = 0; s < n; ++s) f_out[perm[s]] = fo[s];
  });
}

int msot_plan_apply(msot_ctx* c, const double* x, const double* a, int64_t n, const double* y,
                    const double* b, int64_t m, int d, const double* f, const double* g,
                    double eps, const double* v, double* out) {
  return guard([&] {
    if (!c || !x || !a || !y || !b || !f || !g || !v || !out) raise(MSOT_EUSAGE, "null argument");
    if (n < 1 || m < 1) raise(MSOT_EDATA, "empty input");
    if (d < 1 || d > 3) raise(MSOT_EUSAGE, "the GPU plan_apply supports D in 1..3");
    if (!(eps > 0)) raise(MSOT_EUSAGE, "eps must be > 0");
    check_weights(a, n);
    check_weights(b, m);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < d; ++k) lo[k] = std::min(lo[k], x[i * d + k]), hi[k] = std::max(hi[k], x[i * d + k]);
    for (int64_t j = 0; j < m; ++j)
      for (int k = 0; k < d; ++k) lo[k] = std::min(lo[k], y[j * d + k]), hi[k] = std::max(hi[k], y[j * d + k]);
    GridSpec gs{};
    gs.d = d;
    for (int k = 0; k < d; ++k) {
      gs.origin[k] = lo[k];
      gs.center[k] = 0.5 * (lo[k] + hi[k]);
    }
    gs.cell = msot_auto_cell(lo, hi, d, n, m);
    // rows sorted by Morton cube id (compact tiles), as in the solver
    double* dx64 = c->buf<double>("pa.x64", n * d);
    double* da64 = c->buf<double>("pa.a64", n);
    CK(cudaMemcpyAsync(dx64, x, n * d * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(da64, a, n * sizeof(double), cudaMemcpyHostToDevice, st));
    DMeasure MX;
    prepare_measure(c, "pa", dx64, da64, n, d, gs, false, MX);
    std::vector<int32_t> perm(n);
    CK(cudaMemcpyAsync(perm.data(), MX.perm, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    std::vector<float4> yp(m), pay(m);
    std::vector<float> yl(m), gg(m), ff(n);
    for (int64_t s = 0; s < n; ++s) ff[s] = static_cast<float>(f[perm[s]]);
    for (int64_t j = 0; j < m; ++j) {
      float q[3] = {0, 0, 0};
      for (int k = 0; k < d; ++k) q[k] = static_cast<float>(y[j * d + k] - gs.center[k]);
      yp[j] = make_float4(q[0], q[1], q[2], 0.f);
      yl[j] = static_cast<float>(std::log2(b[j]));
      gg[j] = static_cast<float>(g[j]);
      pay[j] = make_float4(static_cast<float>(v[j]), 0.f, 0.f, 0.f);
    }
    float4* dyp = c->buf<float4>("pa.y", m);
    float4* dpay = c->buf<float4>("pa.v", m);
    float* dyl = c->buf<float>("pa.yl", m);
    float* dg = c->buf<float>("pa.g", m);
    float* df = c->buf<float>("pa.f", n);
    float4* dout = c->buf<float4>("pa.out", n);
    CK(cudaMemcpyAsync(dyp, yp.data(), m * sizeof(float4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dpay, pay.data(), m * sizeof(float4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dyl, yl.data(), m * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dg, gg.data(), m * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(df, ff.data(), n * sizeof(float), cudaMemcpyHostToDevice, st));
    RangeSet R;
    dense_rangeset(c, "pa.r", n, m, R);
    const ProbSpec spec{MX.pts, n, dyp, dyl, m, &R};
    const float* fr[1] = {df};
    const float* gc[1] = {dg};
    const float4* py[1] = {dpay};
    float4* po[1] = {dout};
    plan_group(c, "ppa", 1, &spec, fr, gc, py, po, eps, d);
    std::vector<float4> o(n);
    CK(cudaMemcpyAsync(o.data(), dout, n * sizeof(float4), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    // row_plan = {sum_j pi_ij / a_i, sum_j pi_ij v_j / a_i, ...}
    for (int64_t s = 0; s < n; ++s) out[perm[s]] = a[perm[s]] * static_cast<double>(o[s].y);
  });
}

int msot_kmeans(msot_ctx* c, const double* x, const double* w, int64_t n, int d, int k,
                uint64_t seed, int32_t* perm, int32_t* offsets, int32_t* labels, double* centroids,
                double* cweights, float* radii, int* iters) {
  return guard([&] {
    if (!c || !x || !w || !perm || !offsets || !labels || !centroids || !cweights || !radii)
      raise(MSOT_EUSAGE, "null argument");
    if (n < 1) raise(MSOT_EDATA, "empty measure");
    if (k < 1 || k > n) raise(MSOT_EDATA, "K must lie in [1, N] (SPEC.md:263)");
    if (d < 1 || d > 64) raise(MSOT_EUSAGE, "K-means supports D in 1..64");
    check_weights(w, n);
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    double* dx = c->buf<double>("km.x", n * d);
    double* dw = c->buf<double>("km.w", n);
    CK(cudaMemcpyAsync(dx, x, n * d * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dw, w, n * sizeof(double), cudaMemcpyHostToDevice, st));
    // tolerance 1e-9 d on the centre moves, d = bbox diagonal
    std::vector<double> lo(d, INFINITY), hi(d, -INFINITY);
    for (int64_t i = 0; i < n; ++i)
      for (int q = 0; q < d; ++q) lo[q] = std::min(lo[q], x[i * d + q]), hi[q] = std::max(hi[q], x[i * d + q]);
    double diag2 = 0.0;
    for (int q = 0; q < d; ++q) diag2 += (hi[q] - lo[q]) * (hi[q] - lo[q]);
    const double tol = 1e-9 * std::sqrt(diag2);
    int32_t* dperm = c->buf<int32_t>("km.perm", n);
    int32_t* doff = c->buf<int32_t>("km.off", k + 1);
    uint32_t* dlab = c->buf<uint32_t>("km.lab", n);
    double* dcen = c->buf<double>("km.cen", size_t(k) * d);
    double* dcw = c->buf<double>("km.cw", k);
    float* drad = c->buf<float>("km.rad", k);
    void* ws = c->buf<char>("km.ws", kmeans_ws_bytes(n, d, k));
    int it = 0;
    CK(kmeans(dx, dw, n, d, k, seed, tol * tol, 100, ws, dperm, doff, dlab, dcen, dcw, drad, &it,
              st));
    CK(cudaMemcpyAsync(perm, dperm, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(offsets, doff, (k + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(labels, dlab, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(centroids, dcen, size_t(k) * d * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(cweights, dcw, k * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(radii, drad, k * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    if (iters) *iters = it;
  });
}

int msot_grid_cluster(msot_ctx* c, const double* x, const double* w, int64_t n, int d,
                      const double* origin, double cell, int32_t* perm, int32_t* labels,
                      int32_t* offsets, int32_t* k_out, double* centroids, double* cweights,
                      float* radii) {
  return guard([&] {
    if (!c || !x || !w || !origin || !perm || !labels || !offsets || !k_out) raise(MSOT_EUSAGE, "null argument");
    if (d < 1 || d > 3) raise(MSOT_EUSAGE, "grid clustering supports D in 1..3");
    if (n < 1) raise(MSOT_EDATA, "empty measure");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    double* dx = c->buf<double>("gc.x", n * d);
    double* dw = c->buf<double>("gc.w", n);
    CK(cudaMemcpyAsync(dx, x, n * d * sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dw, w, n * sizeof(double), cudaMemcpyHostToDevice, st));
    GridSpec g{};
    g.d = d;
    g.cell = cell;
    for (int k = 0; k < d; ++k) g.origin[k] = origin[k];  // center = 0: raw coordinates
    DMeasure M;
    prepare_measure(c, "gc", dx, dw, n, d, g, true, M);
    CK(cudaMemcpyAsync(perm, M.perm, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(labels, M.labels, n * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(offsets, M.offsets, (M.k + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    std::vector<float4> cp(M.k);
    CK(cudaMemcpyAsync(cp.data(), M.cpts, M.k * sizeof(float4), cudaMemcpyDeviceToHost, st));
    if (cweights) CK(cudaMemcpyAsync(cweights, M.cw64, M.k * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (radii) CK(cudaMemcpyAsync(radii, M.radii, M.k * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
    *k_out = M.k;
    if (centroids)
      for (int32_t I = 0; I < M.k; ++I) {
        const float v[3] = {cp[I].x, cp[I].y, cp[I].z};
        for (int k = 0; k < d; ++k) centroids[int64_t(I) * d + k] = v[k];
      }
  });
}

int msot_truncation_mask(msot_ctx* c, int64_t kx, int64_t ky, int d, const float* cx,
                         const float* rx, const float* fx, const float* gx, const float* cy,
                         const float* ry, const float* gy, const float* hy, double eps,
                         double theta, double p, int self, uint8_t* mask_out) {
  return msot_truncation_mask_box(c, kx, ky, d, cx, rx, fx, gx, nullptr, cy, ry, gy, hy, nullptr,
                                  eps, theta, p, self, mask_out);
}

int msot_truncation_mask_box(msot_ctx* c, int64_t kx, int64_t ky, int d, const float* cx,
                             const float* rx, const float* fx, const float* gx, const float* bx,
                             const float* cy, const float* ry, const float* gy, const float* hy,
                             const float* by, double eps, double theta, double p, int self,
                             uint8_t* mask_out) {
  return guard([&] {
    if (!c || !cx || !rx || !fx || !cy || !ry || !gy || !mask_out) raise(MSOT_EUSAGE, "null argument");
    if ((gx == nullptr) != (hy == nullptr)) raise(MSOT_EUSAGE, "slopes: both sides or neither");
    if ((bx == nullptr) != (by == nullptr)) raise(MSOT_EUSAGE, "boxes: both sides or neither");
    if (bx && !gx) raise(MSOT_EUSAGE, "the box bound needs the slope inputs");
    if (p != 2.0) raise(MSOT_EUSAGE, "the GPU path implements p = 2");
    if (d < 1 || d > 3) raise(MSOT_EUSAGE, "D in 1..3");
    if (kx < 1 || ky < 1) raise(MSOT_EDATA, "empty cluster set");
    CK(cudaSetDevice(c->device));
    cudaStream_t st = c->st;
    std::vector<float4> hcx(kx), hcy(ky);
    for (int64_t I = 0; I < kx; ++I) {
      float v[3] = {0, 0, 0};
      for (int k = 0; k < d; ++k) v[k] = cx[I * d + k];
      hcx[I] = make_float4(v[0], v[1], v[2], 0.f);
    }
    for (int64_t J = 0; J < ky; ++J) {
      float v[3] = {0, 0, 0};
      for (int k = 0; k < d; ++k) v[k] = cy[J * d + k];
      hcy[J] = make_float4(v[0], v[1], v[2], 0.f);
    }
    float4* dcx = c->buf<float4>("tm.cx", kx);
    float4* dcy = c->buf<float4>("tm.cy", ky);
    float* drx = c->buf<float>("tm.rx", kx);
    float* dfx = c->buf<float>("tm.fx", kx);
    float* dry = c->buf<float>("tm.ry", ky);
    float* dgy = c->buf<float>("tm.gy", ky);
    uint32_t* dbits = c->buf<uint32_t>("tm.bits", kx * mask_words(static_cast<int32_t>(ky)));
    int32_t* dbr = c->buf<int32_t>("tm.br", kx);
    int32_t* dbc = c->buf<int32_t>("tm.bc", ky);
    uint8_t* dm = c->buf<uint8_t>("tm.m", kx * ky);
    CK(cudaMemcpyAsync(dcx, hcx.data(), kx * sizeof(float4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dcy, hcy.data(), ky * sizeof(float4), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(drx, rx, kx * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dfx, fx, kx * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dry, ry, ky * sizeof(float), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(dgy, gy, ky * sizeof(float), cudaMemcpyHostToDevice, st));
    float4 *dgx = nullptr, *dhy = nullptr;
    if (gx) {
      dgx = c->buf<float4>("tm.gx", kx);
      dhy = c->buf<float4>("tm.hy", ky);
      CK(cudaMemcpyAsync(dgx, gx, kx * sizeof(float4), cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(dhy, hy, ky * sizeof(float4), cudaMemcpyHostToDevice, st));
    }
    const float4* box[4] = {nullptr, nullptr, nullptr, nullptr};
    if (bx) {  // {lo[3], hi[3]} per cluster -> float4 lo / hi
      std::vector<float4> h(2 * (kx + ky));
      auto unpack = [&](const float* b, int64_t k, float4* lo, float4* hi) {
        for (int64_t I = 0; I < k; ++I) {
          float l[3] = {0, 0, 0}, u[3] = {0, 0, 0};
          for (int q = 0; q < d; ++q) { l[q] = b[I * 6 + q]; u[q] = b[I * 6 + 3 + q]; }
          lo[I] = make_float4(l[0], l[1], l[2], 0.f);
          hi[I] = make_float4(u[0], u[1], u[2], 0.f);
        }
      };
      unpack(bx, kx, h.data(), h.data() + kx);
      unpack(by, ky, h.data() + 2 * kx, h.data() + 2 * kx + ky);
      float4* db = c->buf<float4>("tm.box", h.size());
      CK(cudaMemcpyAsync(db, h.data(), h.size() * sizeof(float4), cudaMemcpyHostToDevice, st));
      CK(host_sync(__LINE__, st));  // h is a local vector
      box[0] = db; box[1] = db + kx; box[2] = db + 2 * kx; box[3] = db + 2 * kx + ky;
    }
    if (self && kx != ky) raise(MSOT_EUSAGE, "a self mask is square");
    void* bws = c->buf<char>("tm.blk", mask_block_ws_bytes(static_cast<int32_t>(kx),
                                                          static_cast<int32_t>(ky)));
    CK(truncation_masks(static_cast<int32_t>(kx), static_cast<int32_t>(ky), d, dcx, drx, dfx, dgx,
                        dcy, dry, dgy, dhy, eps, theta, self, dbits, nullptr, dbr, dbc, bws, st,
                        bx ? box : nullptr));
    CK(unpack_mask(dbits, static_cast<int32_t>(kx), static_cast<int32_t>(ky), dm, st));
    CK(cudaMemcpyAsync(mask_out, dm, kx * ky, cudaMemcpyDeviceToHost, st));
    CK(host_sync(__LINE__, st));
  });
}

}  // extern "C"
