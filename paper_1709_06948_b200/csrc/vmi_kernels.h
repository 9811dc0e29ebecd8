// vmi_kernels.h -- host-side launchers for the device kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "vmi_types.h"

namespace vmi {

// ---- K1 fast path (k_fast.cu) ---------------------------------------------
struct FeatureDump {
  unsigned long long* keys = nullptr;  // packed reference keys (pack_keys)
  double* values = nullptr;            // VARZ / COUNT as the fast path computed it
  int* n = nullptr;                    // device counter
  int cap = 0;
};
struct FastLaunch {
  GridParams g;
  RefView A;
  QueryView B;
  const double* mats;
  int64_t P;
  int cap;
  int grid;
  double* mi;
  int32_t* status;
  long long* hist;
  long long* total;
  FeatureDump dump;  // debug: B's per-voxel features from the fast path (P == 1)
  int streams = 1;   // spans per thread: 1 (CTA = B.threads) or 2 (CTA = B.threads / 2)
  double2* sums = nullptr;  // VARZ: grid * cap (S1, S2) scratch, L2-resident
  int npass = 1;            // hash partitions of the voxel space (table capacity)
  int multi = 0;            // multi-pass layout (4-byte slots, counts in L2), any npass
  // multi-pair launches (vmi_eval_pairs): pose p scores pair pose_pair[p] of pairs[]
  const PairDesc* pairs = nullptr;
  const int32_t* pose_pair = nullptr;
  unsigned long long* hash = nullptr;  // per-pose 64-bit identity of the joint histogram
  unsigned int* sched = nullptr;  // dynamic pose scheduling: a ticket counter (zeroed per launch)
  // rotation-major grids: B.pts = k_rotate's output, pose p reads rotation
  // rot_idx[p]'s records (rot_stride records apart); B.is_f32 must be 0
  const int32_t* rot_idx = nullptr;
  int64_t rot_stride = 0;
};
// Scan B's fast layout (span layout, float4 split or double4 records) rotated
// by each of R matrices (rows 0-2 of mats12[r*12..]): out[r*stride + i] =
// double4((R p_i)_x, (R p_i)_y, (R p_i)_z, 0) with the kernel's FMA chains
// (bit-identical to what the point loop computes); stride = rows * threads.
cudaError_t launch_rotate(const void* pts, int is_f32, int64_t rows, int threads,
                          const double* rots12, int64_t R, void* out, cudaStream_t st);
size_t fast_smem_bytes(int kind, int cap, int bins, int threads, int f32, int ns, int multi);
int fast_slot_bytes(int kind, int multi);  // shared-memory bytes per table slot
cudaError_t launch_fast(const FastLaunch& fl, cudaStream_t st);

// ---- exact sort-based path (k_exact.cu) -------------------------------------
// Scratch for voxelizing up to `cap_n` points at once.
struct ExactScratch {
  int64_t cap_n = 0;
  unsigned long long* keys = nullptr;
  unsigned long long* keys_sorted = nullptr;
  int* idx = nullptr;
  int* idx_sorted = nullptr;
  double* z = nullptr;
  double* zs = nullptr;
  unsigned long long* ukeys = nullptr;
  int* counts = nullptr;
  int* offsets = nullptr;
  double* values = nullptr;
  int* nruns = nullptr;   // device scalar
  int* bounds = nullptr;  // device [6] + [6]=bad flag
  unsigned int* ghist = nullptr;  // (65*65)
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
};
cudaError_t exact_alloc(ExactScratch& s, int64_t n);
void exact_free(ExactScratch& s);

// Point sources for the exact path.
struct PointSource {
  const float4* rec = nullptr;  // contiguous KITTI (x, y, z, i) float32 records, or
  const double* xyz;  // contiguous (n, 3) doubles, or nullptr (both) to use B
  QueryView B;
  int64_t n;
};

// voxelize + compute_feature_map of `src` under `mat` (device ptr, 12 f64;
// nullptr = raw points, as _prepare does for scan A).  Asynchronous; on
// return the device holds: s.ukeys[0..V), s.values[0..V), *s.nruns = V,
// s.bounds[0..5], s.bounds[6] = key-range flag.  Launch count added to *launches.
cudaError_t exact_voxelize(ExactScratch& s, const PointSource& src, const double* mat,
                           const GridParams& g, cudaStream_t st, int64_t* launches);

// Scan A of a pair set whose voxel box [amin, amin + ext) is known exactly
// (host AABB): voxelize + compute_feature_map with 32-bit box indices as keys
// (same order, fewer radix passes).  Leaves box indices in s.ukeys (as u32),
// features in s.values, *s.nruns = V, s.bounds[6] = 1 if a point left the box.
cudaError_t box_voxelize(ExactScratch& s, const PointSource& src, const GridParams& g,
                         const int amin[3], const uint32_t ext[3], cudaStream_t st,
                         int64_t* launches);
// A's grid + voxel list from box_voxelize's output (V = *s.nruns <= Vmax)
cudaError_t build_reference_box(const ExactScratch& s, int Vmax, const GridParams& g,
                                const uint32_t ext[3], uint8_t* grid, int4* tmp, int4* avox,
                                uint32_t* bin_total, int* cursor, cudaStream_t st,
                                int64_t* launches);

// Sparse reference table being built (RefView.hkeys/hbins/hmask): keys
// pre-filled with ~0, mask + 1 a power of two >= 2x the voxel count.
struct SparseRef {
  unsigned long long* keys;
  uint8_t* bins;
  uint32_t mask;
};

// Build A's bin grid and sorted voxel list from V feature-map entries (keys +
// values on device; with Vdev the count is *Vdev and V only an upper bound).
// grid (zeroed, ext-sized) or, with grid null, the sparse table sp; tmp and
// avox hold V entries each.
cudaError_t build_reference(const unsigned long long* keys, const double* values, int V,
                            const int* Vdev, const GridParams& g, const int amin[3],
                            const uint32_t ext[3], uint8_t* grid, int4* tmp, int4* avox,
                            uint32_t* bin_total, int* cursor, cudaStream_t st, int64_t* launches,
                            SparseRef sp = SparseRef{});

// Histogram + finalisation + MI for pose p from an exact voxelization held in
// s (after exact_voxelize).  Writes mi[p], status[p], hist[p], total[p].
cudaError_t exact_score(ExactScratch& s, const GridParams& g, const RefView& A, int64_t p,
                        double* mi, int32_t* status, long long* hist, long long* total,
                        cudaStream_t st, int64_t* launches, unsigned long long* hash = nullptr);

// First-max argmax (np.argmax) over P doubles -> out[0] = value, out_idx[0] = index.
cudaError_t launch_argmax(const double* v, int64_t P, double* out_val, long long* out_idx,
                          cudaStream_t st);

// Stable descending sort of P MI values with their indices (tmp == nullptr:
// *tmp_bytes receives the scratch size).  Two launches (iota + CUB sort).
cudaError_t topk_sort(const double* mi, int P, double* keys_out, int* idx_in, int* idx_out,
                      void* tmp, size_t* tmp_bytes, cudaStream_t st);

// After exact_voxelize of n contiguous points (identity pose): *changes =
// number of voxel changes between consecutive points (runs - 1), and, with
// dst, the points (rec = 16: float4 records, 24: float64 xyz) in the sort's
// voxel-grouped order (dst[i] = src[s.idx_sorted[i]]).
cudaError_t voxel_order(const ExactScratch& s, const void* src, int rec, int64_t n, int* changes,
                        void* dst, cudaStream_t st);

// One pair of a pair-set group (vmi_set_pairs): inputs (raw uploaded scans)
// and outputs (A's grid / voxel list / bin totals, B's span layout).
struct GroupPair {
  const void* raw_a;
  const void* raw_b;
  int64_t n;    // scan A's points
  int64_t off;  // their offset in the group's key array
  int64_t nb;   // scan B's points
  int3 amin;
  uint3 ext;
  uint8_t* grid;
  size_t grid_bytes;
  int4* avox;
  uint32_t* bin_total;
  void* pts;    // scan B's span layout
  int span, rem, b_split;
};
// Build G pairs at once (scan A: keys (pair << nbits) | box index, one sort /
// encode / scan / features / grid / scatter launch each; scan B: one layout
// launch).  vcount[g] = pair g's voxel count; bad[g] set if a point left its
// host-computed box (cannot happen).  G <= 2^(32 - nbits).
cudaError_t build_pair_group(ExactScratch& s, const GroupPair* gp_dev, int G, int64_t n_total,
                             int max_na, int max_nb_rows, size_t max_grid, int nbits,
                             const GridParams& g, int in_f32, int threads, int4* avox_tmp,
                             int* cursor, int* vcount, int* bad, cudaStream_t st,
                             int64_t* launches);

// Summed-volume tables of A's n voxels (avox) for nb bins: bin_slot_dev[bin]
// = table index or -1; sat holds nb * (ext+1)^3-shaped u32 tables.
cudaError_t build_sat(const int4* avox, int n, const int* bin_slot_dev, int nb,
                      const uint32_t ext[3], uint32_t* sat, cudaStream_t st);

// dst[r] = src[idx[r]] (rows of w elements), or the reverse with scatter.
template <typename T>
cudaError_t gather_rows(const T* src, const int64_t* idx, int64_t n, int w, T* dst, bool scatter,
                        cudaStream_t st);

// Reorder contiguous points into the fast path's span layout.
cudaError_t launch_span_layout(const void* src, int in_f32, int out_split, int64_t n, int span,
                               int rem, int threads, void* dst, cudaStream_t st);

}  // namespace vmi
