/* msot_gpu.h — C ABI of the B200-native multiscale Sinkhorn solver.
 *
 * This is the drop-in boundary for the reference's Sinkhorn hot path.  The
 * reference (`/root/reference/proj`) specifies the solver as C++ operations
 * of the `msot::` namespace
 * over `msot::DiscreteMeasure` (measure.hpp:20-51) and reports failures as
 * `msot::DataError` / `msot::NumericError` (common.hpp:10-19).  Every entry
 * point below replaces one of those operations; the C++ front-end in
 * the headers under include/msot/ re-expose them under the reference names and rethrows
 * the status codes as the reference's exception types.
 *
 * Conventions
 *   - Host buffers belong to the caller; they are read/written synchronously.
 *   - Points are row-major N x D float64 (measure.hpp:24, :46).
 *   - Status: MSOT_OK, MSOT_EUSAGE (2), MSOT_EDATA (3), MSOT_ENUMERIC (4),
 *     MSOT_ECUDA (5) — the CLI exit-code convention of SPEC.md:566 plus 5.
 *   - One host thread per context.  No CPU fallback: every compute entry
 *     point runs on the GPU or fails with MSOT_ECUDA.
 */
#ifndef MSOT_GPU_H
#define MSOT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MSOT_OK = 0,
  MSOT_EUSAGE = 2,
  MSOT_EDATA = 3,
  MSOT_ENUMERIC = 4,
  MSOT_ECUDA = 5
};

/* Solver parameters.  Fields blur/reach/p/scaling are SolverParams of
 * SPEC.md:127-130 (+ CostSpec.p, measure.hpp:11-16); the multiscale fields
 * are the knobs of SPEC.md:306-309 (switch scale, theta) with the voxel-grid
 * coarsening of the north star replacing K-means. */
typedef struct msot_params {
  double blur;           /* > 0: final sigma; eps_final = blur^p                 */
  double reach;          /* > 0, or +inf (any value <= 0 is also read as +inf)   */
  double p;              /* cost exponent; the GPU path implements p = 2         */
  double scaling;        /* q in (0,1): sigma_{t+1} = q sigma_t                  */
  int32_t multiscale;    /* 0 = dense eps-scaling, 1 = voxel-grid coarse-to-fine */
  int32_t retruncate;    /* 0 = mask built once at the switch;
                            k > 0 = rebuild the mask every k fine scales        */
  double cluster_scale;  /* voxel edge; <= 0 selects the automatic rule          */
  double theta;          /* truncation slack in units of eps       */
  double switch_factor;  /* switch at first sigma < switch_factor * r_max (:306) */
  int32_t max_full_iters;/* safety cap on schedule length          */
  int32_t mask_rule;     /* 0 = min(centroid/radius, slope, member-box bound) (default),
                            1 = centroid/radius bound only (msot_truncation_mask),
                            2 = min(centroid/radius, slope bound) (round 1)        */
  int32_t transfer_rule; /* coarse -> fine potentials at the switch:
                            0 = inheritance (default),
                            1 = extrapolation: one lambda-damped softmin of the
                                fine atoms against the coarse measure (GeomLoss) */
  int32_t pair_eval;     /* fine phase: 1 = evaluate each kept pair once for its
                            row and its column (default; PAPER.md:258-290's
                            cross kernel is shared by a_xy / b_yx and the
                            self kernels are symmetric), 0 = one row-wise
                            problem per potential (4 per scale)              */
  int32_t clusters;      /* D > 3 multiscale: K-means clusters per measure, 0 =
                            ceil(sqrt(N))                       */
  int32_t seed;          /* K-means seeding: first centre = atom (seed mod N)  */
  int32_t super_level;   /* voxel multiscale: a super-voxel level before the
                            cluster-level coarse phase (policy.h:
                            msot_super_switch): -1 = automatic (when either
                            measure has >= MSOT_SUPER_MIN_CLUSTERS clusters,
                            default), 0 = off, 1 = on                         */
} msot_params;

/* Defaults of SPEC.md:128 (q=0.9), :306 (switch 2x radius), :308 (theta=20). */
void msot_params_default(msot_params* p);

/* Counters of one solve (what SPEC.md:526/:556 asks the CLI to report, plus
 * the roofline evidence of SURVEY.md §8d). */
typedef struct msot_stats {
  int32_t n_scales;         /* schedule length n (final update not counted)      */
  int32_t t_switch;         /* first fine scale index (n if never; 0 if dense)   */
  int32_t kx, ky;           /* voxel clusters of x and y (0 in dense mode)       */
  double  diameter;         /* bounding-box diagonal used for the schedule       */
  double  cluster_scale;    /* voxel edge used                                   */
  double  pairs_dense;      /* pairs a dense solve would evaluate (all updates)  */
  double  pairs_evaluated;  /* pairs actually evaluated by softmin launches      */
  double  pairs_fine;       /* evaluated in the fine (block-sparse) phase         */
  double  pairs_fine_dense; /* what the fine phase would evaluate densely         */
  double  softmin_ms;       /* summed CUDA-event time of softmin launches        */
  int64_t softmin_launches; /* number of softmin kernel launches                 */
  double  total_ms;         /* device time of the whole solve (event-timed)      */
  int64_t fallback_rows;    /* rows recomputed by the exact online-max path       */
  int64_t gpu_launches;     /* all kernels launched by this solve                 */
  double  h2d_bytes, d2h_bytes;
  int32_t rank, world;
  /* device time per phase when profiling (ms): 0 setup (bounding box,
   * clustering), 1 coarse phase, 2 extrapolation, 3 masks/ranges/work
   * items, 4 symmetric updates at full resolution, 5 loss and outputs,
   * 6 label transfer */
  double  phase_ms[8];
  double  pairs_terms;      /* LSE terms summed over all potentials: a pair evaluated
                               once for its row and its column counts twice (what a
                               row-wise CPU solver evaluates for the same solve)  */
  double  pairs_mask_terms; /* profiling: fine-phase LSE terms at cluster granularity
                               (the masks without the 256-row tile union)          */
  int32_t t_super;          /* voxel multiscale: first cluster-level scale after the
                               super-voxel level (0: no super level)              */
  int32_t k_super_x, k_super_y;  /* super clusters                                */
  int32_t colpart_batches;  /* most column-partial batches of one fine update       */
  double  device_bytes;     /* device memory the context holds after the solve     */
  int64_t host_syncs;       /* host waits on the device during the solve           */
} msot_stats;

typedef struct msot_ctx msot_ctx;

/* Thread-local message describing the last failure. */
const char* msot_last_error(void);

/* Single-GPU context on CUDA device `device`. */
int msot_create(int device, msot_ctx** out);
/* One process per GPU: rank `rank` of `world`, NCCL communicator from a
 * unique id produced by msot_nccl_unique_id on rank 0 (128 bytes). */
int msot_nccl_unique_id(unsigned char out[128]);
int msot_create_dist(int device, int rank, int world, const unsigned char nccl_id[128],
                     msot_ctx** out);

/* Parity seam (tests): for the next solves on this context, copy the four
 * potentials (a_xx[n], b_yy[m], a_xy[m], b_yx[n], caller order, raw gauge)
 * before and after the update of schedule index `scale` (0..n_scales; the
 * final assignment is n_scales) into the given host buffers (entries may be
 * NULL).  Captured on fine-phase and dense 3-D updates; scale < 0 disables. */
int msot_debug_capture(msot_ctx* ctx, int scale, double* const in[4], double* const out[4]);

/* Parity seam (tests): the cluster mask of the captured multiscale update
 * (which: 0 = x-x, 1 = y-y, 2 = x-y; unpacked k_rows x k_cols bytes, 1 =
 * kept) and the cluster of every row / column atom in caller order.  Call
 * with NULL buffers to read the sizes. */
int msot_debug_mask(const msot_ctx* ctx, int which, int32_t* k_rows, int32_t* k_cols,
                    uint8_t* mask, int32_t* row_cluster, int32_t* col_cluster);

/* Rank, world size and the rank count of the context's communicator as NCCL
 * reports it (ncclCommCount; 1 without one, world for the host seam). */
int msot_world_info(const msot_ctx* ctx, int* rank, int* world, int* comm_ranks);
/* Test seam: the same sharded solve with host-staged collectives supplied by
 * the caller (e.g. torch.distributed gloo) in place of NCCL, so the
 * multi-rank logic runs with several processes on one GPU.  allreduce sums
 * `count` floats in place across ranks; broadcast copies root's `count`
 * 32-bit words to every rank bit for bit (the solver also moves its float64
 * column totals through it, all-gather style).  Both return 0 on success.
 * (The current solver exchanges everything through broadcast; allreduce is
 * kept for the signature and must still be supplied.) */
typedef int (*msot_host_allreduce_fn)(float* data, int64_t count, void* user);
typedef int (*msot_host_broadcast_fn)(float* data, int64_t count, int root, void* user);
int msot_create_dist_host(int device, int rank, int world, msot_host_allreduce_fn allreduce,
                          msot_host_broadcast_fn broadcast, void* user, msot_ctx** out);
void msot_destroy(msot_ctx* ctx);
/* 1 = time every softmin launch with CUDA events (stats.softmin_ms). */
int msot_set_profiling(msot_ctx* ctx, int on);
/* Column-partial slots an evaluate-once update may hold at once (0 =
 * automatic: 6 per row + column of the group).  Larger values
 * mean fewer, larger batches; results do not depend on it (bitwise). */
int msot_set_colpart_budget(msot_ctx* ctx, int64_t slots);

/* Measures the GPU's MUFU.EX2 rate (ex2 per second, all SMs) with the
 * ex2.approx.ftz.f32 instruction the softmin issues: the measured roofline
 * denominator of the softmin (pairs/s <= ex2/s). */
int msot_probe_ex2(msot_ctx* ctx, double* ex2_per_s);

/* --- host-side helpers shared with the oracle (no GPU work) ------------- */

/* make_schedule: writes n sigmas/eps/lambdas, returns n
 * (-n when cap < n; 0 for invalid parameters: reach must be > 0 or +inf).  n = floor(log(d/blur)/log(1/q)) + 1, sigma_t =
 * d q^t for t < n-1 and sigma_{n-1} = blur. */
int msot_schedule(double diameter, const msot_params* p, double* sigma, double* eps,
                  double* lam, int cap);

/* Contiguous, tile-aligned split of `n_tiles` row tiles with per-tile cost
 * `work` into `world` shards: writes world+1 tile boundaries. */
int msot_shard_tiles(const double* work, int64_t n_tiles, int world, int64_t* bounds);

/* resolve_flips, host only: soft labels of a
 * flip-augmented subject (n rows = 2 x originals, L classes) -> one row per
 * original fibre.  flip_of[i] = original index of row i, orientation[i] = 0
 * (original) / 1 (flipped); every original must appear once per orientation
 * (MSOT_EDATA otherwise).  The orientation with the larger row mass is kept,
 * ties to the original.  chosen[o] = the augmented row kept for original o. */
int msot_resolve_flips(const double* scores, const double* row_mass, int64_t n, int n_classes,
                       const int32_t* flip_of, const int32_t* orientation, double* scores_out,
                       double* row_mass_out, int32_t* chosen);

/* classify, host only: label[i] = -1 (OUTLIER) iff
 * row_mass[i] < tau, else the argmax class (ties to the lowest index);
 * confidence[i] = max score / row_mass (0 for outliers with zero mass). */
int msot_classify(const double* scores, const double* row_mass, int64_t n, int n_classes,
                  double tau, int32_t* label, double* confidence);

/* --- device operations (host buffers) ----------------------------------- */

/* One dense softmin, rows x (N x D)
 * over columns y (M x D):
 *   f_i = -lambda eps log sum_j exp(logw_j + (h_j - |x_i - y_j|^2 / 2) / eps)
 * f_est (nullable) is the reference value the kernel expands around. */
int msot_softmin(msot_ctx* ctx, const double* x, int64_t n, const double* y, int64_t m,
                 int d, const double* logw_y, const double* h, double eps, double lambda,
                 const double* f_est, double* f_out);

/* plan_apply (eq. 4): the implicit transport plan
 * of the given duals applied to an M-vector, without materialising it,
 *   out_i = sum_j a_i b_j exp((f_i + g_j - |x_i - y_j|^2 / 2) / eps) v_j,
 * dense over the columns, D in 1..3 (f = b_yx on x, g = a_xy on y). */
int msot_plan_apply(msot_ctx* ctx, const double* x, const double* a, int64_t n, const double* y,
                    const double* b, int64_t m, int d, const double* f, const double* g,
                    double eps, const double* v, double* out);

/* Voxel-grid clustering (north star; replaces kmeans_coarsen SPEC.md:260):
 * cube ids floor((x - origin)/cell) in float64, Morton-interleaved, stable
 * LSD radix sort.  perm[k] = original index of the k-th sorted atom;
 * labels[k] = cluster of sorted atom k; offsets[0..K]; centroids K x D,
 * cweights K, radii K (max distance to the centroid, rounded up). */
int msot_grid_cluster(msot_ctx* ctx, const double* x, const double* w, int64_t n, int d,
                      const double* origin, double cell, int32_t* perm, int32_t* labels,
                      int32_t* offsets, int32_t* k_out, double* centroids,
                      double* cweights, float* radii);

/* K-means coarsening (kmeans_coarsen): farthest-point
 * seeding from atom (seed mod N), Lloyd iterations with mass-weighted
 * centroids until the largest centre move is < 1e-9 d (d = bounding-box
 * diagonal) or 100 iterations; float64, ties to the lowest index.
 * labels[i] = cluster of atom i (caller order); perm[k] = caller index of the
 * k-th atom grouped by cluster (index order inside); offsets[0..K];
 * centroids K x D; cweights K; radii K (max distance, rounded up); iters
 * (nullable) = Lloyd iterations run. */
int msot_kmeans(msot_ctx* ctx, const double* x, const double* w, int64_t n, int d, int k,
                uint64_t seed, int32_t* perm, int32_t* offsets, int32_t* labels,
                double* centroids, double* cweights, float* radii, int* iters);

/* Exact optimal transport (module exact_oracle; the
 * reference names exact_ot(a, b, spec) -> DensePlan without a header):
 * min sum pi_ij C_ij over pi >= 0 with row sums a and column sums b, C the
 * (1/p)|x - y|^p cost of the n x d and m x d row-major points.  Host-only,
 * single-threaded network simplex (a test / `msot verify` ground truth, not
 * the GPU path; no context).  Requires sum a = sum b within 1e-9 and
 * n * m <= 1e6 (MSOT_EDATA otherwise).  plan (nullable): n x m row-major
 * optimal vertex; value: sum pi_ij C_ij in fixed pairwise order. */
int msot_exact_ot(const double* x, const double* a, int64_t n, const double* y, const double* b,
                  int64_t m, int d, double p, double* plan, double* value);

/* Truncation mask: keep (I,J) iff
 *   min(B_a, B_b) >= -theta * eps,  D = X_I - Y_J,
 *   B_a = F_I + G_J - (1/2) max(0, |D| - (r_I + r_J))^2
 *   B_b = F'_I + G'_J + r_I |S_I - D| + r_J |T_J + D| - |D|^2 / 2
 * (B_b only when the slope arrays gx = {S_I, F'_I}, hy = {T_J, G'_J}, 4
 * floats per cluster, are given — both or neither), evaluated in float64
 * without FMA on float32 inputs, plus each row's and each column's best
 * pair (ties to the lowest index) and, when `self` is set, the diagonal.
 * mask_out is Kx x Ky bytes. */
int msot_truncation_mask(msot_ctx* ctx, int64_t kx, int64_t ky, int d, const float* cx,
                         const float* rx, const float* fx, const float* gx, const float* cy,
                         const float* ry, const float* gy, const float* hy, double eps,
                         double theta, double p, int self, uint8_t* mask_out);
/* The same with the member boxes of the clusters, bx (kx x 6) / by (ky x 6):
 * {lo[0..2], hi[0..2]} = the min / max of the members' offsets from the
 * centroid per axis (the solver's cluster_stats rounds them outward).  Adds
 * the box bound B_c (mask.cu header) to min(B_a, B_b); needs gx / hy. */
int msot_truncation_mask_box(msot_ctx* ctx, int64_t kx, int64_t ky, int d, const float* cx,
                             const float* rx, const float* fx, const float* gx, const float* bx,
                             const float* cy, const float* ry, const float* gy, const float* hy,
                             const float* by, double eps, double theta, double p, int self,
                             uint8_t* mask_out);

/* The symmetric eps-scaling Sinkhorn solve + debiased divergence
 * (PAPER.md:235-326).  Potential outputs are
 * nullable (in the caller's atom order).  loss_out receives S_eps,rho. */
int msot_sinkhorn(msot_ctx* ctx, const msot_params* prm, const double* x, const double* a,
                  int64_t n, const double* y, const double* b, int64_t m, int d,
                  double* a_xx, double* b_yy, double* a_xy, double* b_yx, double* loss_out,
                  msot_stats* stats);

/* The solve plus grad_positions: envelope-theorem
 * gradient of S with respect to the atoms of alpha (p = 2),
 *   grad_i = sum_j pi^xy_ij (x_i - y_j) - sum_k pi^xx_ik (x_i - x_k),
 * pi from the final potentials on the pair set of the last update.
 * grad_x is N x D (caller order). */
int msot_sinkhorn_grad(msot_ctx* ctx, const msot_params* prm, const double* x, const double* a,
                       int64_t n, const double* y, const double* b, int64_t m, int d,
                       double* loss_out, double* grad_x, msot_stats* stats);

/* transfer_labels (eq. 7, config 4): solves the
 * divergence of (alpha, beta) like msot_sinkhorn, then applies the implicit
 * plan of the final cross potentials f = b_yx, g = a_xy to the one-hot atlas
 * labels without materialising it:
 *   scores[i][l] = sum_{j : labels[j] = l} b_j exp((f_i + g_j - C_ij)/eps),
 *   row_mass[i]  = sum_l scores[i][l]
 * (eps = blur^p).  labels: M class indices in [0, n_classes) (caller order
 * of y); scores: N x n_classes row-major, caller order of x. */
int msot_transfer_labels(msot_ctx* ctx, const msot_params* prm, const double* x, const double* a,
                         int64_t n, const double* y, const double* b, int64_t m, int d,
                         const int32_t* labels, int n_classes, double* scores, double* row_mass,
                         double* loss_out, msot_stats* stats);

/* Wasserstein barycenter of K target measures (PAPER.md
 * :374-386, config 5): descent on the positions of alpha (weights frozen),
 * x <- x - step * mean_k(grad_k) / a, the step halved (<= 10 times) until the
 * mean divergence does not increase; stops after `iters` accepted steps or a
 * relative decrease below `tol`.  reach must be infinite, p = 2.
 * loss_traj (nullable) receives iters+1 values; x_out is N x D. */
int msot_barycenter(msot_ctx* ctx, const msot_params* prm, const double* x0, const double* a,
                    int64_t n, int k, const double* const* ys, const double* const* bs,
                    const int64_t* ms, int d, int iters, double step, double tol,
                    double* x_out, double* loss_traj, int* steps_done, msot_stats* stats);

/* Same, inputs already resident on the device (float64 device pointers). */
int msot_sinkhorn_device(msot_ctx* ctx, const msot_params* prm, const double* d_x,
                         const double* d_a, int64_t n, const double* d_y, const double* d_b,
                         int64_t m, int d, double* loss_out, msot_stats* stats);

#ifdef __cplusplus
}
#endif
#endif /* MSOT_GPU_H */
