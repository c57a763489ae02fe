/* policy.h — host-side parameter rules shared verbatim by the GPU front-end
 * and the FP64 oracle, so both run the *same* algorithm:
 *   - the eps-schedule,
 *   - the automatic voxel edge and the cube-id / Morton key (north star),
 *   - the coarse->fine switch index,
 *   - the row-tile size that defines the block-sparse pair set.
 * Pure C99 + libm; header-only (static inline).
 */
#ifndef MSOT_POLICY_H
#define MSOT_POLICY_H

#include <math.h>
#include <stdint.h>

#include "../../include/msot_gpu.h"

#ifdef __CUDACC__
#define MSOT_HD __host__ __device__
#else
#define MSOT_HD
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Rows per block-sparse tile: the truncation mask is expanded to column
 * ranges per tile of MSOT_TILE_ROWS consecutive (cluster-sorted) rows. */
#define MSOT_TILE_ROWS 256
/* Target atoms per occupied voxel for the automatic cluster_scale rule.
 * Measured on C3 (1M Gaussian mixtures, blur 0.01, profiles/r1_cell_sweep.jsonl)
 * with the evaluate-once fine phase: 48 -> 0.74 s, S within 4.1e-4 of the
 * dense solve; 28 -> 0.50 s, within 7.4e-5; below ~25 the switch (sigma <
 * r_max) leaves too few fine scales (16 atoms: +2.9e-3). */
#define MSOT_AUTO_ATOMS_PER_CELL 28.0
/* Lloyd iterations of the K-means coarsening inside the multiscale solver
 * (the stand-alone kmeans_coarsen op keeps SPEC.md:265's cap of 100): the
 * clusters only steer efficiency (truncation), never the result, and the
 * float64 assignment of 400k x 633 x 60 costs ~5 ms per iteration.  Config 4,
 * 20 -> 8 iterations: setup 353 -> 199 ms, total 2.03 -> 1.73 s, S 3.9e-4 ->
 * 1.9e-4 from dense (the cluster radii move the switch one scale later). */
#define MSOT_KMEANS_SOLVER_ITERS 8
/* Cube ids are Morton-interleaved with this many bits per axis (D <= 3). */
#define MSOT_MORTON_BITS 10

/* reach = +inf is the only encoding of balanced OT; callers validate with
 * msot_reach_valid first (reach > 0 or inf). */
static inline int msot_reach_valid(double reach) { return reach > 0.0; }
static inline int msot_reach_is_inf(double reach) { return isinf(reach) && reach > 0.0; }

/* lambda = 1 / (1 + eps/rho), rho = reach^p. */
static inline double msot_lambda(double eps, const msot_params* p) {
  if (msot_reach_is_inf(p->reach)) return 1.0;
  return 1.0 / (1.0 + eps / pow(p->reach, p->p));
}

/* Schedule length: n = floor(log(d/blur) / log(1/q)) + 1; a ratio within
 * 1e-9 below an integer counts as that integer (so d=8, blur=1, q=1/2 gives
 * [8,4,2,1] as SPEC.md:160 requires). */
static inline int msot_schedule_len(double d, double blur, double q) {
  if (!(d > blur)) return 1;
  double r = log(d / blur) / log(1.0 / q);
  double k = floor(r);
  if (r - k > 1.0 - 1e-9) k += 1.0;
  return (int)k + 1;
}

static inline double msot_schedule_sigma(double d, double blur, double q, int n, int t) {
  if (t >= n - 1) return blur;
  return d * pow(q, (double)t);
}

/* Automatic voxel edge: a grid over the joint bounding box with about
 * MSOT_AUTO_ATOMS_PER_CELL atoms per cell for the larger cloud, never more
 * than 2^MSOT_MORTON_BITS - 1 cells along an axis. */
static inline double msot_auto_cell(const double* lo, const double* hi, int d, int64_t n,
                                    int64_t m) {
  double nmax = (double)(n > m ? n : m);
  double cells = nmax / MSOT_AUTO_ATOMS_PER_CELL;
  if (cells < 1.0) cells = 1.0;
  double vol = 1.0, ext_max = 0.0;
  int nd = 0;
  for (int k = 0; k < d; ++k) {
    double e = hi[k] - lo[k];
    if (e > ext_max) ext_max = e;
  }
  if (ext_max <= 0.0) return 1.0;
  for (int k = 0; k < d; ++k) {
    double e = hi[k] - lo[k];
    if (e > 1e-6 * ext_max) { vol *= e; ++nd; }
  }
  double s = pow(vol / cells, 1.0 / (double)(nd > 0 ? nd : 1));
  double smin = ext_max / (double)((1 << MSOT_MORTON_BITS) - 2);
  if (s < smin) s = smin;
  return s;
}

/* Refinement of the automatic edge for clustered data (the first guess
 * assumes the bounding box is uniformly filled): rescale so the number of
 * occupied voxels k approaches max(n,m)/MSOT_AUTO_ATOMS_PER_CELL.  The
 * solver applies it MSOT_AUTO_REFINE times, recounting occupied voxels of
 * both clouds (max) in between. */
#define MSOT_AUTO_REFINE 2
static inline double msot_refine_cell(double cell, int64_t k_occupied, int64_t n, int64_t m,
                                      int d, const double* lo, const double* hi) {
  double target = (double)(n > m ? n : m) / MSOT_AUTO_ATOMS_PER_CELL;
  if (target < 1.0) target = 1.0;
  if (k_occupied < 1) k_occupied = 1;
  double s = cell * pow((double)k_occupied / target, 1.0 / (double)d);
  double ext_max = 0.0;
  for (int k = 0; k < d; ++k)
    if (hi[k] - lo[k] > ext_max) ext_max = hi[k] - lo[k];
  double smin = ext_max / (double)((1 << MSOT_MORTON_BITS) - 2);
  if (s < smin) s = smin;
  if (ext_max > 0.0 && s > 2.0 * ext_max) s = 2.0 * ext_max;
  return s;
}

/* Voxel coordinate along one axis: floor((x - origin) / cell) in float64
 * (one correctly rounded subtraction, one correctly rounded division). */
MSOT_HD static inline uint32_t msot_cube_coord(double x, double origin, double cell) {
  double q = floor((x - origin) / cell);
  if (q < 0.0) q = 0.0;
  double qmax = (double)((1u << MSOT_MORTON_BITS) - 1u);
  if (q > qmax) q = qmax;
  return (uint32_t)q;
}

MSOT_HD static inline uint32_t msot_spread3(uint32_t v) { /* 10 bits -> every 3rd bit */
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000ffu;
  v = (v | (v << 8)) & 0x0300f00fu;
  v = (v | (v << 4)) & 0x030c30c3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
MSOT_HD static inline uint32_t msot_spread2(uint32_t v) { /* 10 bits -> every 2nd bit */
  v &= 0x3ffu;
  v = (v | (v << 8)) & 0x00ff00ffu;
  v = (v | (v << 4)) & 0x0f0f0f0fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

/* Morton cube id of one atom (D in 1..3). */
MSOT_HD static inline uint32_t msot_cube_key(const double* x, int d, const double* origin,
                                     double cell) {
  if (d == 1) return msot_cube_coord(x[0], origin[0], cell);
  if (d == 2)
    return msot_spread2(msot_cube_coord(x[0], origin[0], cell)) |
           (msot_spread2(msot_cube_coord(x[1], origin[1], cell)) << 1);
  return msot_spread3(msot_cube_coord(x[0], origin[0], cell)) |
         (msot_spread3(msot_cube_coord(x[1], origin[1], cell)) << 1) |
         (msot_spread3(msot_cube_coord(x[2], origin[2], cell)) << 2);
}

/* Row tiles of the block-sparse reduction.  With clusters (offsets != NULL)
 * tiles are cluster-aligned: consecutive whole clusters are packed greedily
 * while they fit in `cap` rows, and a cluster larger than `cap` is split into
 * ceil(len/cap) near-equal tiles.  Without clusters: uniform tiles of `cap`.
 * Writes tile_start[0..T] (T+1 entries, tile_start[T] = n), returns T.
 * Capacity needed: k + n/cap + 2 entries. */
static inline int64_t msot_pack_tiles(const int32_t* offsets, int64_t k, int64_t n, int64_t cap,
                                      int64_t* tile_start) {
  int64_t t = 0;
  if (!offsets) {
    for (int64_t s = 0; s < n; s += cap) tile_start[t++] = s;
    tile_start[t] = n;
    return t;
  }
  int64_t cur = -1; /* start of the open tile, -1 = none */
  for (int64_t I = 0; I < k; ++I) {
    const int64_t b = offsets[I], e = offsets[I + 1], len = e - b;
    if (len > cap) {
      if (cur >= 0) { tile_start[t++] = cur; cur = -1; }
      const int64_t parts = (len + cap - 1) / cap;
      for (int64_t q = 0; q < parts; ++q) tile_start[t++] = b + q * len / parts;
    } else if (cur >= 0 && e - cur > cap) {
      tile_start[t++] = cur;
      cur = b;
    } else if (cur < 0) {
      cur = b;
    }
  }
  if (cur >= 0) tile_start[t++] = cur;
  tile_start[t] = n;
  return t;
}

/* The row tiling the block-sparse phase uses.  With ~48 atoms per voxel a
 * 256-row tile of Morton-sorted atoms spans ~5 neighbouring voxels whichever
 * way it is cut, so uniform tiles (100% thread fill) are used; the
 * cluster-aligned packing above stays available for coarse voxels. */
#define MSOT_CLUSTER_ALIGNED_TILES 0
static inline int64_t msot_row_tiles(const int32_t* offsets, int64_t k, int64_t n,
                                     int64_t tile_rows, int64_t* tile_start) {
  return msot_pack_tiles(MSOT_CLUSTER_ALIGNED_TILES ? offsets : 0, k, n, tile_rows, tile_start);
}

/* First fine scale: the first t with sigma_t < factor * r_max;
 * n when no scale qualifies (then only the final update runs fine). */
static inline int msot_switch_index(const double* sigma, int n, double r_max, double factor) {
  for (int t = 0; t < n; ++t)
    if (sigma[t] < factor * r_max) return t;
  return n;
}

/* Super level of the coarse phase (voxel path): super voxels of 2^MSOT_SUPER_SHIFT
 * voxels per axis group consecutive clusters (Morton order: the super key is
 * the voxel key >> d * MSOT_SUPER_SHIFT).  The super measure runs the scales
 * with sigma_t >= MSOT_SUPER_SWITCH * (half-diagonal of a super voxel) and
 * hands its duals to the clusters by inheritance, which
 * continue to the fine switch.  Returns the first cluster-level scale t2 (0:
 * no super level — it must take at least MSOT_SUPER_MIN_SCALES scales off the
 * cluster level). */
#define MSOT_SUPER_SHIFT 1
#define MSOT_SUPER_SWITCH 2.0  /* C3: S within 8.6e-5 of dense (1.0: 7.3e-4; none: 9.0e-5) */
#define MSOT_SUPER_MIN_SCALES 4
/* automatic mode: only where the cluster-level coarse phase costs something
 * (C3, 34k clusters: 32 -> 11 ms; config 2, 3k clusters: no gain, S 4.5e-4 ->
 * 7.4e-4 from dense) */
#define MSOT_SUPER_MIN_CLUSTERS 16384
static inline int msot_super_switch(const double* sigma, int tsw, double cell, int d,
                                    int64_t kmax, int mode) {
  if (mode == 0 || (mode < 0 && kmax < MSOT_SUPER_MIN_CLUSTERS)) return 0;
  const double r = 0.5 * sqrt((double)d) * cell * (double)(1 << MSOT_SUPER_SHIFT);
  const int t2 = msot_switch_index(sigma, tsw, r, MSOT_SUPER_SWITCH);
  return (tsw - t2 >= MSOT_SUPER_MIN_SCALES) ? t2 : 0;
}

#ifdef __cplusplus
}
#endif
#endif /* MSOT_POLICY_H */
