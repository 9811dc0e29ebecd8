/*
 * vmi.h -- C ABI of the B200 batched MI pose-evaluation library (libvmi.so).
 *
 * The reference (`voxmi`, pure Python/numpy) has no FFI; its "operator API" for
 * the hot path is the Python objective contract
 *     mi_objective(feat_a, cloud_b, pose, grid, spec, include_phi, n_jobs) -> float
 * (reference pkg/src/voxmi/mi.py:194-219), fed by _prepare's scan-A feature map
 * (align.py:114-119) and driven by align's objective closure (align.py:134-136)
 * and sweep_axis's loop (align.py:191-197).  Each entry point below replaces one
 * piece of that contract; the Python package paper_1709_06948_b200 binds them
 * with ctypes (see INTEGRATION.md for the binding a voxmi maintainer would add).
 *
 * Conventions
 *   - Return codes: 0 = OK, negative = error; vmi_last_error(ctx) has the text.
 *   - Per-pose status (vmi_eval*): VMI_OK, VMI_EMPTY_REGION, VMI_KEY_RANGE,
 *     VMI_PHI_OFF_EMPTY.  Any non-OK status comes with mi = VMI_SENTINEL
 *     (-1e300), the reference's NO_OVERLAP_SENTINEL (mi.py:34, :206-219).
 *   - A context is bound to one CUDA device, single-threaded and stream-ordered.
 *     Host inputs are copied; the context owns every device buffer it allocates.
 *   - There is no CPU fallback: without a usable CUDA device vmi_create fails.
 */
#ifndef VMI_H_
#define VMI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vmi_ctx vmi_ctx;

#define VMI_SENTINEL (-1e300)

enum vmi_status {
  VMI_OK = 0,
  VMI_EMPTY_REGION = 1,  /* compute_overlap empty (mi.py:211-213) */
  VMI_KEY_RANGE = 2,     /* OutOfBoundsError from voxel_indices (mi.py:206-209) */
  VMI_PHI_OFF_EMPTY = 3  /* include_phi=False, no co-occupied voxel (mi.py:215-219) */
};

enum vmi_kind { VMI_VARZ = 0, VMI_COUNT = 1 }; /* FeatureKind (voxel.py:33-46) */

enum vmi_error {
  VMI_ERR_ARG = -1,
  VMI_ERR_CUDA = -2,
  VMI_ERR_ALLOC = -3,
  VMI_ERR_STATE = -4,
  VMI_ERR_RANGE = -5,       /* scan A leaves the voxel key range (voxel.py:200-206) */
  VMI_ERR_UNSUPPORTED = -6  /* e.g. bins > 64, a pair set whose scan A needs the sparse reference */
};

/* Context lifetime.  device = CUDA ordinal.  Replaces nothing in the reference
   (it holds the state _prepare/mi_objective recompute per call). */
int vmi_create(int device, vmi_ctx** out);
int vmi_destroy(vmi_ctx* ctx);
const char* vmi_last_error(const vmi_ctx* ctx);
/* Library/build identification string (static storage). */
const char* vmi_version(void);

/* GridSpec (voxel.py:49-62) + BinningSpec (mi.py:40-59) + include_phi
   (mi.py:177-191).  kind: vmi_kind.  Must precede vmi_set_reference_*.
   bins in [2, 64]; clamp > 0. */
int vmi_set_params(vmi_ctx* ctx, const double origin[3], double resolution, int kind, int bins,
                   double clamp, int include_phi);

/* Scan A from raw points: voxelize + compute_feature_map on the GPU
   (_prepare, align.py:114-119; voxel.py:210-222, :267-295), bit-exact including
   VARZ.  xyz: host (n, 3) float64, row-major.  Returns VMI_ERR_RANGE when a
   point leaves the key range (the reference raises OutOfBoundsError). */
int vmi_set_reference_points(vmi_ctx* ctx, const double* xyz, int64_t n);

/* Scan A as KITTI .bin records (x, y, z, intensity float32; scan_io.py:57-75),
   uploaded as they are (16 B/point; no float64 upcast on the host) and widened
   exactly on the GPU -- the reference loads them as PointCloud(data[:, :3]
   .astype(float64)) (scan_io.py:74).  Same results as vmi_set_reference_points
   on the widened coordinates. */
int vmi_set_reference_records_f32(vmi_ctx* ctx, const float* xyzi, int64_t n);

/* Scan A from an existing FeatureMap (voxel.py:129-164): packed keys
   (pack_keys, voxel.py:65-73) sorted ascending, values >= 0, bounds =
   [xmin, ymin, zmin, xmax, ymax, zmax].  The injection point the reference's
   tests use (test_mi.py:37-50). */
int vmi_set_reference_features(vmi_ctx* ctx, const int64_t* keys, const double* values, int64_t n,
                               const int64_t bounds[6]);

/* Export the GPU-built scan-A FeatureMap (keys, values, bounds).  With keys ==
   NULL only *n_out is written.  cap = capacity of keys/values. */
int vmi_get_reference_features(vmi_ctx* ctx, int64_t* keys, double* values, int64_t cap,
                               int64_t* n_out, int64_t bounds[6]);

/* Scan B (PointCloud, geometry.py:36-65): host (n, 3) float64.  Stored as
   float4 when every coordinate is float32-exact (KITTI input), else double.
   Point order never changes a result; the fused kernel aggregates runs of
   consecutive points in one voxel, so ring-ordered (or, for COUNT,
   voxel-grouped) scans run fastest. */
int vmi_set_query_points(vmi_ctx* ctx, const double* xyz, int64_t n);
/* Scan B as KITTI .bin records (x, y, z, intensity float32; scan_io.py:57-75). */
int vmi_set_query_records_f32(vmi_ctx* ctx, const float* xyzi, int64_t n);

/* Optional, after vmi_set_query_*: a superset of scan B's convex-hull vertices
   ((n, 3) float64, the scan's own coordinates; qhull's vertices qualify).  The
   fast kernel then takes each pose's voxel bounds (voxel.py:220) from these
   instead of from every point; a pose whose extreme lies within 1e-6 voxel of
   an integer is re-run on the exact path.  n = 0 removes it.  Passing points
   that do NOT cover the hull gives wrong bounds. */
int vmi_set_query_hull(vmi_ctx* ctx, const double* xyz, int64_t n);

/* euler_to_transform (geometry.py:126-138) for P poses (tx,ty,tz,rx,ry,rz):
   12 float64 per pose, R row-major then t, bit-identical to the reference
   (glibc sin/cos, no FP contraction).  Host only; threads <= 0 = all cores. */
int vmi_poses_to_mats(const double* poses, int64_t n, double* mats, int threads);

/* Batched mi_objective (mi.py:194-219) over P pose matrices, host buffers,
   synchronous.  mi_out[P], status_out[P] required; hist_out (P*(bins+1)^2
   int64, JointHistogram.counts, mi.py:82-98) and total_out (P int64,
   JointHistogram.total) may be NULL. */
int vmi_eval(vmi_ctx* ctx, const double* mats, int64_t P, double* mi_out, int32_t* status_out,
             int64_t* hist_out, int64_t* total_out);

/* vmi_eval from poses: P x 6 float64 (tx, ty, tz, roll, pitch, yaw), the
   reference's EulerPose fields (geometry.py:68-102).  The pose -> matrix step
   (euler_to_transform, geometry.py:126-138, glibc sin/cos) runs on the host
   and is overlapped with the GPU: the first poses are launched while the rest
   are converted and uploaded (pinned staging, second stream).  Results are
   identical to vmi_poses_to_mats + vmi_eval.  Synchronous. */
int vmi_eval_poses(vmi_ctx* ctx, const double* poses, int64_t P, double* mi_out,
                   int32_t* status_out, int64_t* hist_out, int64_t* total_out);

/* Same with device pointers on a caller stream (cudaStream_t as void*);
   asynchronous: no host sync, no fix-up pass (see vmi_eval_fixups). */
int vmi_eval_device(vmi_ctx* ctx, const double* mats_dev, int64_t P, double* mi_dev,
                    int32_t* status_dev, int64_t* hist_dev, int64_t* total_dev, void* stream);

/* After vmi_eval_device: re-evaluate, through the exact sort-based path, the
   poses whose fast-path status carries VMI_FLAG_RECHECK (table overflow or a
   VARZ value within rounding of a bin edge).  Synchronous. Returns count. */
int vmi_eval_fixups(vmi_ctx* ctx, const double* mats_dev, int64_t P, double* mi_dev,
                    int32_t* status_dev, int64_t* hist_dev, int64_t* total_dev, void* stream,
                    int64_t* n_fixed);
#define VMI_FLAG_RECHECK 0x100

/* Pose grids (rotations repeat): rotation-major evaluation.  Scan B is rotated
   once per distinct rotation (R copies; rots12_dev: R x 12 matrices, rows 0-2
   used) and the point loop reads the copy of rotation rot_idx_dev[q] for the
   pose in slot q (mats_dev: P x 12, slots in rotation-major order so CTAs
   share a copy in L2).  Fix-ups included (synchronous); results are written
   at perm_dev[q] (the slot's pose in the caller's order), bit-identical to
   vmi_eval_device + vmi_eval_fixups on the unpermuted batch.  Replaces the
   per-pose transform of the reference's grid consumers (sweep_axis,
   align.py:191-197; cli.py:202's grid argmax) for repeated rotations.
   VMI_ERR_UNSUPPORTED: too many rotations for the memory budget (VMI_ROT_MB,
   default 4096) or a table that needs the multi-pass layout.  With VMI_ROT=1,
   vmi_eval_poses takes this path by itself for grid batches (>= 4096 poses,
   distinct rotations <= P/16, no histograms).  Measured slower than the
   per-pose path on B200 (the 32-byte rotated records double the point loop's
   L2 traffic), hence opt-in. */
int vmi_eval_rot_device(vmi_ctx* ctx, const double* rots12_dev, int64_t R, const double* mats_dev,
                        const int32_t* rot_idx_dev, const int64_t* perm_dev, int64_t P,
                        double* mi_dev, int32_t* status_dev, int64_t* total_dev, void* stream);

/* Exact (sort-based, reference-order) evaluation of P poses: the slow
   cross-check path, bit-exact features by construction. */
int vmi_eval_exact(vmi_ctx* ctx, const double* mats, int64_t P, double* mi_out,
                   int32_t* status_out, int64_t* hist_out, int64_t* total_out);

/* Debug / parity: B's feature map at one pose (voxelize + compute_feature_map
   of the transformed scan), via the exact path.  keys/values capacity cap. */
int vmi_query_features(vmi_ctx* ctx, const double mat[12], int64_t* keys, double* values,
                       int64_t cap, int64_t* n_out, int64_t bounds[6], int32_t* status);

/* Debug / parity: B's per-voxel features at one pose as the FAST path computed
   them (voxels inside scan A's AABB only; VARZ from the pivot-shifted sums),
   unsorted.  *n_out = number of voxels (may exceed cap: then nothing copied). */
int vmi_fast_features(vmi_ctx* ctx, const double mat[12], int64_t* keys, double* values,
                      int64_t cap, int64_t* n_out, int32_t* status);

/* Device-side argmax over mi (first index of the max, np.argmax semantics,
   cli.py:202).  Writes best value and index to host. */
int vmi_argmax_device(vmi_ctx* ctx, const double* mi_dev, int64_t P, double* best_mi,
                      int64_t* best_idx, void* stream);

/* Device-side top-K over mi: the min(K, P) largest values in descending
   order with their candidate indices; equal values keep ascending index order,
   so entry 0 is np.argmax's first maximum (cli.py:202).  The per-rank
   exchange unit of a sharded search (top-K (mi, idx) per GPU,
   then one all-gather).  Writes K doubles and K indices to host. */
int vmi_topk_device(vmi_ctx* ctx, const double* mi_dev, int64_t P, int64_t K, double* top_mi,
                    int64_t* top_idx, void* stream);

/* ---- Lockstep Nelder-Mead over many runs (nm_lockstep.cpp) -------------------
   K independent nelder_mead_maximize runs (optim.py:62-175) advanced together:
   each step hands ALL runs' pending probes to one evaluator call.  Decisions are
   the reference's, in its order; a comparison between values closer than the
   backend's error bound (and not from the same joint histogram) marks the run
   `uncertain` -- the caller must redo it on exact values.  termination:
   VMI_NM_CONVERGED_F / _X / VMI_NM_MAX_ITER.  trace: -values[0] after every sort
   (OptimResult.trace), trace_cap doubles per run, trace_len = its length. */
#define VMI_NM_CONVERGED_F 0
#define VMI_NM_CONVERGED_X 1
#define VMI_NM_MAX_ITER 2
/* evaluator: n poses (n x 6) with their run index -> g[i] = -objective and an
   identity h[i] of the value's source (equal identities must mean equal values) */
typedef int (*vmi_nm_eval_fn)(void* user, const double* poses, const int32_t* run, int64_t n,
                              double* g, uint64_t* h);
/* spec_budget: probes per step up to which an iteration evaluates its four
   candidates at once (< 0: always); above it, the reflection first and then the
   one follow-up the reference needs (same decisions, fewer probes). */
int vmi_nm_run(int64_t K, const double* x0, const double steps[6], int max_iterations,
               double f_tol, double x_tol, int restarts, int64_t spec_budget, vmi_nm_eval_fn fn,
               void* user,
               double* best_x, double* best_value, int32_t* iterations, int32_t* termination,
               int32_t* n_evaluations, int32_t* uncertain, double* trace, int32_t* trace_len,
               int64_t trace_cap);

/* ---- Many resident scan pairs (C5: a drive's consecutive pairs) ---------------
   vmi_set_pairs builds npairs (scan A, scan B) pairs on the device at once --
   each scan A voxelized + featurized (_prepare, align.py:114-119) into its own
   dense bin grid, each scan B in its own span layout -- replacing any previous
   set.  a[i] / b[i]: host points, (n, 4) float32 KITTI records (is_rec = 1) or
   (n, 3) float64 (is_rec = 0).  Independent of the single pair set by
   vmi_set_reference_* / vmi_set_query_*. */
int vmi_set_pairs(vmi_ctx* ctx, int64_t npairs, const void* const* a, const int64_t* na,
                  const void* const* b, const int64_t* nb, int is_rec);

/* mi_objective (mi.py:194-219) for P poses, pose p against pair pair[p] of the
   set, in ONE multi-pair kernel launch; host buffers, synchronous.  hash_out
   (nullable): a 64-bit identity of each pose's joint histogram (equal identity
   => equal histogram, up to 2^-64 collisions; 0 for sentinel poses); hist_out
   (nullable) as vmi_eval. */
int vmi_eval_pairs(vmi_ctx* ctx, const double* poses, const int32_t* pair, int64_t P,
                   double* mi_out, int32_t* status_out, uint64_t* hash_out, int64_t* hist_out);

/* align()'s optimiser (optim.py:62-175, align.py:122-159) for every pair of the
   set at once: vmi_nm_run with the multi-pair kernel as the objective (one
   launch per lockstep step across all pairs).  x0: one start pose (6) per pair.
   Outputs as vmi_nm_run; a run flagged `uncertain` met a comparison the GPU's
   MI cannot decide exactly and must be redone on exact values. */
int vmi_align_pairs(vmi_ctx* ctx, int64_t K, const double* x0, const double steps[6],
                    int max_iterations, double f_tol, double x_tol, int restarts, double* best_x,
                    double* best_value, int32_t* iterations, int32_t* termination,
                    int32_t* n_evaluations, int32_t* uncertain, double* trace, int32_t* trace_len,
                    int64_t trace_cap);

/* Number of kernel launches issued by this context so far (bench accounting). */
int64_t vmi_launch_count(const vmi_ctx* ctx);
/* Counters: [0] kernel launches, [1] table re-plans (an under-estimated scan-B
   occupancy grown after > 1% of a launch overflowed), [2] poses re-run on the
   exact path, [3] the current pair's scan-B occupancy estimate, [4] lockstep
   Nelder-Mead steps, [5] poses they scored (vmi_align_pairs, cumulative). */
int vmi_get_counters(const vmi_ctx* ctx, int64_t out[6]);

/* Fast-path configuration knobs (tests/bench): table capacity (0 = sized from
   scan B's occupancy; larger than fits shared memory = clamped) and CUDA threads per CTA (0 = default = 512, one scan-B span per
   thread). */
int vmi_set_tuning(vmi_ctx* ctx, int table_cap, int threads);

/* Voxel-space hash partitions per pose (0 = automatic: enough passes that each
   pass's share of scan B's voxels fills about half the shared-memory table;
   large grids such as 0.2 m voxels over 100 m need several). */
int vmi_set_passes(vmi_ctx* ctx, int npass);

#ifdef __cplusplus
}
#endif
#endif /* VMI_H_ */
