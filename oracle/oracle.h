/* oracle.h — FP64 CPU restatement of the reference's Sinkhorn hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library,
 * and only as the checker / the timed CPU baseline — never as the product.
 *
 * The reference ships no Sinkhorn code: the algorithm is
 * restated from PAPER.md:235-326 (Algorithm), PAPER.md:146-207 (Eqs. 2-6)
 * and SPEC.md:122-467.  It runs on the reference's own CPU executor and
 * summation (proj/src/parallel.cpp, proj/src/numeric.cpp) built unmodified
 * into oracle/_ref/.  Parity pins: the SPEC closed-form known answers
 * (tests/test_oracle.py) — GeomLoss/KeOps, the paper's arithmetic, are not
 * vendored and no version is pinned, so equivalence with them is unpinned.
 */
#ifndef MSOT_ORACLE_H
#define MSOT_ORACLE_H

#include <stdint.h>

#include "../include/msot_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

void oracle_set_threads(int n);   /* msot::parallel::set_threads (parallel.hpp:11) */
int oracle_threads(void);

int oracle_schedule(double diameter, const msot_params* p, double* sigma, double* eps,
                    double* lam, int cap);

/* Dense softmin, rows x over columns y. */
void oracle_softmin(const double* x, int64_t n, const double* y, int64_t m, int d,
                    const double* logw_y, const double* h, double eps, double lambda,
                    double p, double* f_out);

/* Voxel-grid clustering: same contract as msot_grid_cluster. */
int oracle_grid_cluster(const double* x, const double* w, int64_t n, int d,
                        const double* origin, double cell, int32_t* perm, int32_t* labels,
                        int32_t* offsets, int32_t* k_out, double* centroids,
                        double* cweights, float* radii);

/* K-means coarsening: same contract as msot_kmeans. */
int oracle_kmeans(const double* x, const double* w, int64_t n, int d, int k, uint64_t seed,
                  int32_t* perm, int32_t* offsets, int32_t* labels, double* centroids,
                  double* cweights, float* radii, int* iters);

/* Truncation mask: same contract as msot_truncation_mask. */
void oracle_truncation_mask(int64_t kx, int64_t ky, int d, const float* cx, const float* rx,
                            const float* fx, const float* gx, const float* cy, const float* ry,
                            const float* gy, const float* hy, double eps, double theta, double p,
                            int self, uint8_t* mask_out);
/* With member boxes {lo[3], hi[3]} per cluster (msot_truncation_mask_box). */
void oracle_truncation_mask_box(int64_t kx, int64_t ky, int d, const float* cx, const float* rx,
                                const float* fx, const float* gx, const float* bx, const float* cy,
                                const float* ry, const float* gy, const float* hy, const float* by,
                                double eps, double theta, double p, int self, uint8_t* mask_out);

/* Cluster-aligned row tiles (policy.h:msot_pack_tiles) and the column
 * ranges of each tile from a cluster mask.  Returns the number of ranges
 * (ranges written only when cap is large enough; call with cap=0 to size).
 * tile_start/tile_ptr need kx + n_rows/256 + 2 entries. */
int64_t oracle_tile_ranges(const int32_t* row_labels, const int32_t* row_offsets,
                           int64_t n_rows, int64_t kx, const int32_t* col_offsets, int64_t ky,
                           const uint8_t* mask, int64_t* n_tiles, int64_t* tile_start,
                           int64_t* tile_ptr, int32_t* ranges, int64_t cap);

/* Full solve: dense or multiscale per prm->multiscale.  Potentials are in
 * the caller's atom order (nullable).  Returns a status. */
int oracle_sinkhorn(const msot_params* prm, const double* x, const double* a, int64_t n,
                    const double* y, const double* b, int64_t m, int d, double* a_xx,
                    double* b_yy, double* a_xy, double* b_yx, double* loss_out,
                    msot_stats* stats);

/* Divergence from given potentials (eq. 5-6). */
double oracle_divergence_from_potentials(const msot_params* prm, double eps, const double* a,
                                         int64_t n, const double* b, int64_t m,
                                         const double* a_xx, const double* b_yy,
                                         const double* a_xy, const double* b_yx);

/* grad_positions (dense plans) and the barycenter descent
 * (SPEC.md:356-364): same contracts as msot_sinkhorn_grad / msot_barycenter. */
int oracle_sinkhorn_grad(const msot_params* prm, const double* x, const double* a, int64_t n,
                         const double* y, const double* b, int64_t m, int d, double* loss_out,
                         double* grad);
int oracle_barycenter(const msot_params* prm, const double* x0, const double* a, int64_t n, int k,
                      const double* const* ys, const double* const* bs, const int64_t* ms, int d,
                      int iters, double step, double tol, double* x_out, double* loss_traj,
                      int* steps_done);

/* transfer_labels (eq. 7), dense, given duals f
 * (on x, = b_yx) and g (on y, = a_xy):
 *   scores[i][l] = sum_{j: labels_j = l} b_j exp((f_i + g_j - C_ij)/eps),
 *   row_mass[i]  = sum_l scores[i][l]  (pairwise_sum order over l).  */
int oracle_transfer_labels(const double* x, int64_t n, const double* y, const double* b,
                           int64_t m, int d, const double* f, const double* g, double eps,
                           const int32_t* labels, int n_classes, double* scores,
                           double* row_mass);

/* plan_apply, dense FP64:
 *   out_i = sum_j a_i b_j exp((f_i + g_j - C_ij)/eps) v_j. */
void oracle_plan_apply(const double* x, const double* a, int64_t n, const double* y,
                       const double* b, int64_t m, int d, const double* f, const double* g,
                       double eps, const double* v, double* out);

const char* oracle_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
