// prims.cuh — declarations of the device primitives and kernel launchers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace msot_dev {

// scans (prims.cu)
size_t scan_temp_elems(int64_t n);
template <typename TI, typename TO>
cudaError_t scan(const TI* in, TO* out, int64_t n, bool inclusive, TO* tmp, TO* total,
                 cudaStream_t st);

// bounding box (prims.cu); lohi holds ordered-int64 keys of min/max per dim
cudaError_t bbox(const double* x, int64_t n, int d, long long* lohi_dev, bool init,
                 cudaStream_t st);
void bbox_decode(const long long* lohi_host, int d, double* lo, double* hi);
cudaError_t count_bad_weights(const double* w, int64_t n, int32_t* bad, cudaStream_t st);

// stable LSD radix sort of (key, value) by the low `key_bits` bits
size_t radix_temp_bytes(int64_t n);
cudaError_t radix_sort_pairs(uint32_t* keys, int32_t* vals, int64_t n, int key_bits, void* temp,
                             cudaStream_t st);

// softmin (softmin.cu)
cudaError_t launch_softmin(const Group& g, int d, cudaStream_t st);
cudaError_t launch_finalize(const Group& g, cudaStream_t st);
cudaError_t launch_rowsum(const Group& g, int32_t i0, cudaStream_t st);  // batched row partials
cudaError_t launch_fallback(const Group& g, int d, int n_sm, cudaStream_t st);
cudaError_t launch_plan(const Group& g, int d, cudaStream_t st);  // plan_kernel + plan_finalize

// evaluate-once block-sparse softmin (softmin_sym.cu) and its pair sets (mask.cu)
constexpr int kEntryChunks = 32;  // tile chunks of the column-major entry pass
struct ColSum {
  const int32_t* labels;     // column -> cluster
  const int32_t* co;         // cluster offsets of the columns
  const int64_t* eptr;       // [K * kEntryChunks + 1]: entries of cluster J at [J*C, (J+1)*C)
  const int64_t* eslot;
  const int32_t* etile;
  const int32_t* tile_start;
  const float* colpart;       // base such that colpart[eslot] is the slot (batch-shifted)
  float* tot;                 // null: the float64 total stays in acc (multi-rank exchange)
  double* acc;                // running float64 totals across batches (nullable: one batch)
  int32_t n_cols, self, t0, t1;
  int32_t first, last;        // first / last batch of this problem
};
struct ColSumGroup {
  ColSum c[3];
  int n;
};
// uniform: every row weight equal and lambda = 1 (column sums need no row factor)
cudaError_t launch_softmin_sym(const Group& g, int d, bool uniform, cudaStream_t st);
cudaError_t launch_colsum(const ColSum* c, int n, cudaStream_t st);
cudaError_t totals_f32(const double* acc, float* tot, int32_t n, cudaStream_t st);
cudaError_t launch_fallback_dense(const Group& g, int d, int n_sm, cudaStream_t st);
cudaError_t sym_ranges(const uint32_t* tbits, int32_t k, int64_t nt, const int32_t* co,
                       const int32_t* ts, const int32_t* rl, int self, int64_t* n_ranges,
                       int64_t* n_cols, int32_t* posword, const int64_t* rptr, int2* ranges,
                       bool write, cudaStream_t st);
cudaError_t sym_entries(const uint32_t* tbits, int32_t k, int64_t nt, const int32_t* co,
                        const int32_t* ts, const int32_t* rl, int self, const int32_t* posword,
                        const int64_t* tslot, int32_t* cnt, const int64_t* ebase, int64_t* eslot,
                        int32_t* etile, bool fill, cudaStream_t st);

// high-dimensional softmin (softmin_hd.cu): tcgen05 split-f16 <x,y>
int64_t hd_padded(int64_t n);
size_t hd_pack_bytes(int64_t n);
cudaError_t hd_pack(const double* x, int64_t n, int d, const double* center, int role,
                    uint8_t* pack, float* sq, float* xf, cudaStream_t st);
cudaError_t hd_weights(const double* w, int64_t n, float* lw2, double* w64, cudaStream_t st);
// sym: evaluate-once (column partials into P.colpart)
cudaError_t launch_softmin_hd(const Group& g, int d, int n_sm, bool sym, cudaStream_t st);
// per-scale column constants of a high-D problem into `out` (hd_padded(n_cols));
// out2 (nullable): column factor exponents of evaluate-once groups
cudaError_t hd_colconst(const Problem& P, float* out, float* out2, cudaStream_t st);
// the dense column sums of up to three problems in one launch
struct DenseColSum {
  const float* colpart;
  const int64_t* tslot;
  const int32_t* ts;
  float* tot;                 // null: keep the float64 total in acc (multi-rank exchange)
  double* acc;
  int32_t t0, t1, self, n_cols, first, last;
};
struct DenseColSumGroup {
  DenseColSum c[3];
  int n;
};
cudaError_t hd_colsum_group(const DenseColSum* c, int n, cudaStream_t st);
cudaError_t launch_fallback_hd(const Group& g, int d, int n_sm, cudaStream_t st);

// label transfer (labels.cu, K9)
cudaError_t gather_label_cols(const float4* pts, const float* lw2, const float* h,
                              const int32_t* src, int64_t mpad, float4* cols, float* lw_out,
                              float* h_out, cudaStream_t st);
cudaError_t gather_rows_f64(const double* x, int d, const int32_t* src, int64_t mpad, double* out,
                            cudaStream_t st);
cudaError_t label_finalize(const float* part, const int32_t* lbase, const int32_t* tile_start,
                           int64_t n_tiles, int n_classes, const int32_t* perm, double* scores,
                           double* mass, cudaStream_t st);

// positions gradient of S (loss.cu): rows of x, sorted order ->
// grad[perm[s]] = a_s ((m_xy - m_xx) x_s - (u_xy - u_xx)) (float64, caller order;
// frame-invariant, so the centred coordinates are used as they are)
cudaError_t grad_positions(const float4* pts, const double* w64, const float4* plan_xy,
                           const float4* plan_xx, const int32_t* perm, int64_t n, int d,
                           double* grad, cudaStream_t st);
// barycenter descent helpers (loss.cu)
cudaError_t field_accumulate(double* field, const double* grad, double scale, int64_t len,
                             cudaStream_t st);
cudaError_t bary_step(double* x_new, const double* x, const double* field, const double* a,
                      double step, int64_t n, int d, cudaStream_t st);

// clustering (cluster.cu)
struct GridSpec {
  double origin[3];
  double center[3];
  double cell;
  int d;
};
cudaError_t cube_keys(const double* x, int64_t n, GridSpec g, uint32_t* keys, int32_t* iota,
                      cudaStream_t st);
// nonuniform (nullable): set to 1 when the weights are not all equal
cudaError_t gather_points(const double* x, const double* w, int64_t n, int d, GridSpec g,
                          const int32_t* perm, float4* pts, float* lw2, double* w64,
                          int32_t* nonuniform, cudaStream_t st);
cudaError_t segment_flags(const uint32_t* sorted_keys, int64_t n, uint8_t* flags,
                          cudaStream_t st);
cudaError_t segment_offsets(const int32_t* labels, const uint8_t* flags, int64_t n,
                            int32_t* offsets, cudaStream_t st);
// box_lo / box_hi (nullable): the members' offsets from the float centroid,
// per axis min / max rounded outward to float (the truncation box bound)
cudaError_t cluster_stats(const float4* pts, const double* w64, const int32_t* offsets, int32_t k,
                          int d, float4* cen, float* clw2, double* cw64, float* radii,
                          cudaStream_t st, float4* box_lo = nullptr, float4* box_hi = nullptr);
cudaError_t cluster_bound(const float4* pts, const double* w64, const float* f,
                          const int32_t* offsets, const float4* cen, int32_t k, float* fmax,
                          float4* grad, cudaStream_t st);
cudaError_t inherit(const float* coarse, const int32_t* labels, int64_t n, float* fine,
                    cudaStream_t st);
cudaError_t gather_f4(const float4* src, const int32_t* idx, int64_t n, float4* dst, cudaStream_t st);
cudaError_t scatter_f4(const float4* src, const int32_t* idx, int64_t n, float4* dst, cudaStream_t st);
cudaError_t scatter_f32(const float* src, const int32_t* idx, int64_t n, float* dst, cudaStream_t st);
cudaError_t shift_payload(float4* p, int64_t n, double cx, double cy, double cz, cudaStream_t st);
cudaError_t super_keys(const uint32_t* sorted_keys, const int32_t* offsets, int32_t k, int bits,
                       uint32_t* out, cudaStream_t st);

// K-means coarsening (kmeans.cu), float64, bit-identical to the oracle.
// perm: atoms grouped by cluster (index order inside), off[K+1], labels per
// atom (caller order), centers K x d, cw cluster weights, radii (rounded up).
size_t kmeans_ws_bytes(int64_t n, int d, int K);
cudaError_t kmeans(const double* x, const double* w, int64_t n, int d, int K, uint64_t seed,
                   double tol2, int max_iter, void* ws, int32_t* perm, int32_t* off,
                   uint32_t* labels, double* centers, double* cw, float* radii, int* iters,
                   cudaStream_t st);

// padded cluster layout of the high-D multiscale solver (kmeans.cu)
cudaError_t hd_gather_padded(const double* x, const double* centers, const int32_t* src,
                             int64_t npad, int d, double* out, cudaStream_t st);
cudaError_t hd_padded_weights(const double* w, const int32_t* src, int64_t npad, float* lw2,
                              double* w64, cudaStream_t st);
cudaError_t hd_cluster_fmax(const float* f, const double* w64, const int32_t* off, int K,
                            float* fmax, cudaStream_t st);
// high-D truncation masks (mask.cu): the centroid/radius bound B_a with float64
// centroids (D <= 64), best pairs, self diagonal; maskT = exact transpose
cudaError_t truncation_masks_hd(int32_t kx, int32_t ky, int d, const double* cx, const float* rx,
                                const float* fx, const double* cy, const float* ry,
                                const float* gy, double eps, double theta, int self,
                                uint32_t* mask, uint32_t* maskT, int32_t* best_r, int32_t* best_c,
                                cudaStream_t st);

// truncation mask + ranges (mask.cu)
__host__ __device__ inline int32_t mask_words(int32_t ky) { return (ky + 31) / 32; }
// bit-packed mask: Kx rows of mask_words(Ky) uint32 words
// gx / hy (nullable): {slope G, F'} per cluster for the gradient bound
// Keep bits + best pairs of one truncation test.  self: kx == ky, one
// symmetric mask (maskT, best_c unused).  Otherwise mask (kx rows over ky)
// and maskT (ky rows over kx, its exact transpose), both with the row and
// column best pairs; best_r (kx) / best_c (ky) are workspaces, blkws holds
// the column-block bounds (mask_block_ws_bytes).  box (nullable, only with
// the slope inputs gx/hy): {lo_x, hi_x, lo_y, hi_y} member boxes per cluster
// (cluster_stats), adding the box bound B_c (mask.cu header).
cudaError_t truncation_masks(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                             const float* fx, const float4* gx, const float4* cy, const float* ry,
                             const float* gy, const float4* hy, double eps, double theta, int self,
                             uint32_t* mask, uint32_t* maskT, int32_t* best_r, int32_t* best_c,
                             void* blkws, cudaStream_t st, const float4* const* box = nullptr);
// Self masks: lower half from the upper half (bitwise transpose of the
// blocks below the diagonal).  truncation_masks_rows(self) computes the
// upper half only (row I: words from I / 32 on, the words below zero) — all
// the evaluate-once pair sets read — and leaves the mirror to the callers
// that need whole rows.
cudaError_t mask_mirror(uint32_t* mask, int32_t k, cudaStream_t st);
cudaError_t truncation_masks_rows(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                                  const float* fx, const float4* gx, const float4* cy,
                                  const float* ry, const float* gy, const float4* hy, double eps,
                                  double theta, int self, int32_t r0, int32_t r1, uint32_t* mask,
                                  int32_t* best_r, void* blkws, cudaStream_t st,
                                  const float4* const* box = nullptr);
cudaError_t truncation_masks_cols(int32_t kx, int32_t ky, int d, const float4* cx, const float* rx,
                                  const float* fx, const float4* gx, const float4* cy,
                                  const float* ry, const float* gy, const float4* hy, uint32_t* mask,
                                  int32_t* best_c, void* blkws, cudaStream_t st,
                                  const float4* const* box = nullptr);
inline size_t mask_block_ws_bytes(int32_t kx, int32_t ky) {
  return static_cast<size_t>(mask_words(kx) + mask_words(ky)) * (sizeof(float4) + sizeof(float)) +
         static_cast<size_t>(mask_words(ky)) * sizeof(uint32_t);
}
cudaError_t mask_pair_count(const uint32_t* mask, int32_t kx, int32_t ky, const int32_t* ro,
                            const int32_t* co, double* out, cudaStream_t st);
cudaError_t unpack_mask(const uint32_t* mask, int32_t kx, int32_t ky, uint8_t* out,
                        cudaStream_t st);
// per tile: OR of its clusters' mask rows, then count / write column ranges
cudaError_t tile_or(const uint32_t* mask, int32_t ky, const int32_t* row_labels,
                    const int32_t* tile_start, int64_t nt, uint32_t* tbits, cudaStream_t st);
cudaError_t tile_range_count(const uint32_t* tbits, int32_t ky, int64_t nt,
                             const int32_t* col_offsets, int64_t* n_ranges, int64_t* n_cols,
                             cudaStream_t st);
cudaError_t tile_range_write(const uint32_t* tbits, int32_t ky, int64_t nt,
                             const int32_t* col_offsets, const int64_t* rptr, int2* ranges,
                             cudaStream_t st);
cudaError_t dense_ranges(int64_t n_tiles, int32_t n_cols, int64_t* rptr, int2* ranges,
                         int64_t* tile_cols, cudaStream_t st);
// work items: per tile ceil(cols/chunk) items
cudaError_t item_counts(const int64_t* tile_cols, int64_t n_tiles, int64_t chunk, int32_t* cnt,
                        cudaStream_t st);
cudaError_t item_write(const int64_t* tile_cols, int64_t t0, int64_t t1, int64_t chunk,
                       const int32_t* ibase, int problem, int4* items, cudaStream_t st);

// loss (loss.cu)
cudaError_t divergence_partial(const double* a, const double* b, int64_t n, int64_t m,
                               const float* a_xx, const float* b_yy, const float* a_xy,
                               const float* b_yx, double rho /* <=0: balanced */,
                               double* partials, int nblocks, cudaStream_t st);
cudaError_t divergence_final(const double* partials, int nblocks, double eps, double rho,
                             double* out, cudaStream_t st);
cudaError_t scatter_unsort(const float* v, const int32_t* perm, int64_t n, const double* shift,
                           double sign, double* out, cudaStream_t st);

// MUFU.EX2 throughput probe (probe.cu)
cudaError_t ex2_probe(int n_sm, int iters, float* sink, double* ex2_per_launch, int* blocks,
                      cudaStream_t st);

}  // namespace msot_dev
