// vmi_api.cu -- the C ABI declared in include/vmi.h.
//
// Context = one CUDA device + one stream + the resident scan-A grid, scan-B
// span layout, exact-path scratch and output buffers.  No entry point ever
// computes on the CPU except vmi_poses_to_mats (glibc sin/cos, pose_host.cpp)
// and the float32-exactness test of uploaded coordinates.
#include <cmath>
#include <cstdio>
#include <algorithm>
#include <array>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/vmi.h"
#include "nm_lockstep.h"
#include "vmi_kernels.h"

using namespace vmi;

// One scan pair resident on the device: scan A's dense bin grid + voxel list,
// scan B's span-layout records.  A context holds its current pair (`cur`, the
// single-pair API) and optionally a pair set (vmi_set_pairs) for the
// multi-pair kernel.  Buffers are grow-only and reused when a pair is re-set.
struct PairStore {
  // scan A
  bool a_set = false;
  bool a_empty = true;
  int amin[3] = {0, 0, 0}, amax[3] = {0, 0, 0};
  uint32_t ext[3] = {0, 0, 0};
  uint8_t* d_grid = nullptr;
  size_t grid_bytes = 0, cap_grid = 0;
  int4* d_avox = nullptr;
  size_t cap_avox = 0;
  int n_avox = 0;
  uint32_t* d_bin_total = nullptr;
  bool sparse = false;                // A's AABB too large for the dense grid
  unsigned long long* d_hkeys = nullptr;  // sparse A: packed keys (RefView.hkeys)
  uint8_t* d_hbins = nullptr;
  size_t cap_hkeys = 0, cap_hbins = 0;
  uint32_t hmask = 0;
  int64_t a_nvox = 0;
  int64_t a_npts = 0;  // scan A's point count (0 when set from features)
  // scan B
  bool b_set = false;
  void* d_pts = nullptr;
  size_t cap_pts = 0;
  int is_f32 = 0;
  int64_t nb = 0;
  int span = 0;
  int rem = 0;
  double max_abs = 0.0;
  double b_lo[3] = {0, 0, 0}, b_hi[3] = {0, 0, 0};  // scan B's AABB
  int64_t b_voxels = 0;  // scan B's occupied voxels at the identity pose (table sizing)
  double* d_hull = nullptr;  // scan B's convex-hull vertices (vmi_set_query_hull), or none
  size_t cap_hull = 0;
  int hull_n = 0;
  uint32_t* d_sat = nullptr;     // summed-volume tables of A per present bin, or none
  size_t cap_sat = 0;
  int* d_sat_bin = nullptr;      // [kMaxW] present bins, then [kMaxW] bin -> table
  int sat_nb = 0;
  bool regrouped = false;        // d_pts in voxel-grouped order, d_pts_exact in input order
  void* d_pts_exact = nullptr;
  size_t cap_pts_exact = 0;
};

// A CUDA stream with its own scratch: pair-set builds run kBuildLanes pairs at
// a time (small per-pair kernels and uploads overlap across lanes).
struct BuildLane {
  cudaStream_t st = nullptr;
  cudaEvent_t done = nullptr;
  ExactScratch ex;
  int4* d_avox_tmp = nullptr;
  size_t cap_avox_tmp = 0;
  int* d_cursor = nullptr;
};
constexpr int kBuildLanes = 4;

// Device buffers of one multi-pair evaluation (matrices + pair index in,
// MI / status / histogram identity / total out).
struct PairBufs {
  const double* mats;
  const int32_t* pose_pair;
  double* mi;
  int32_t* status;
  unsigned long long* hash;
  long long* total;
};

// One lane of the lockstep optimiser's evaluations (vmi_align_pairs): device
// buffers (matrices, MI, identities, totals, statuses, pair indices) and
// pinned host buffers (matrices, then MI / identities / statuses read back).
struct NmSlot {
  void* d_buf = nullptr;
  void* h_buf = nullptr;
  int64_t cap = 0, n = 0;
  cudaEvent_t ev = nullptr;
  const int32_t* run = nullptr;  // the lane's pair indices (host), valid until wait
  PairBufs bufs{};
};

struct vmi_ctx {
  int device = 0;
  int sm_count = 0;
  size_t smem_optin = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int64_t launches = 0;

  bool params_set = false;
  GridParams g{};
  int occ = 0;  // fast kernel runs the occupancy kind (every occupied voxel in one bin)

  PairStore cur;                // the single-pair API's scan pair
  std::vector<PairStore> set;   // vmi_set_pairs: many resident pairs (multi-pair kernel)
  int64_t n_set = 0;            // pairs of `set` in use
  PairDesc* d_pairs = nullptr;  // device copies of the set's views
  size_t cap_pairs = 0;
  BuildLane lanes[kBuildLanes];
  void* d_raw = nullptr;  // vmi_set_pairs: the distinct scans as uploaded
  size_t cap_raw = 0;
  std::vector<cudaEvent_t> chunk_ev;  // vmi_set_pairs: raw-upload chunk done
  void* d_group = nullptr;    // vmi_set_pairs: GroupPair descriptors
  size_t cap_group = 0;
  void* d_gavox = nullptr;    // grouped build: unsorted voxel lists
  size_t cap_gavox = 0;
  void* d_gcursor = nullptr;  // grouped build: per-pair bin cursors
  size_t cap_gcursor = 0;
  cudaEvent_t set_start = nullptr;
  int* d_setv = nullptr;  // per-pair voxel counts + "left the box" flags (vmi_set_pairs)
  size_t cap_setv = 0;
  int32_t* d_pose_pair = nullptr;  // vmi_eval_pairs: per-pose pair index
  unsigned long long* d_hash = nullptr;  // per-pose histogram identities
  int64_t cap_pp = 0;

  // scratch for building scan A (any pair)
  int4* d_avox_tmp = nullptr;  // unsorted voxel list of build_reference
  int* d_cursor = nullptr;
  unsigned long long* d_akeys = nullptr;  // the current pair's FeatureMap (exported)
  double* d_avalues = nullptr;
  unsigned long long* d_pkeys = nullptr;  // a set pair's FeatureMap (build scratch)
  double* d_pvalues = nullptr;
  size_t cap_pkeys = 0, cap_pvalues = 0;

  int threads = kFastThreads;  // span-layout threads
  int streams = 1;             // spans per CUDA thread in the fast kernel
  int cap_override = 0;
  int npass_override = 0;

  ExactScratch ex;

  // host-API staging
  cudaStream_t copy_stream = nullptr;  // vmi_eval_poses: tail-chunk upload beside the head kernel
  cudaEvent_t copy_done = nullptr;
  double* h_mats = nullptr;  // pinned pose matrices (vmi_eval_poses), grow-only
  int64_t h_mats_cap = 0;
  double* d_mats = nullptr;
  double* d_mi = nullptr;
  int32_t* d_status = nullptr;
  long long* d_hist = nullptr;
  long long* d_total = nullptr;
  int64_t cap_P = 0;
  bool hist_alloc = false;
  double* d_best = nullptr;
  long long* d_best_idx = nullptr;
  // top-K scratch (grow-only)
  double* d_tk_keys = nullptr;
  int* d_tk_idx = nullptr;
  int* d_tk_out = nullptr;
  void* d_tk_tmp = nullptr;
  size_t cap_tk_keys = 0, cap_tk_idx = 0, cap_tk_out = 0, cap_tk_tmp = 0;
  double2* d_sums = nullptr;  // fast-path VARZ sums scratch (grid * cap)
  size_t sums_n = 0;
  // grow-only capacities (bytes) of scratch reused across scan pairs
  size_t cap_avox_tmp = 0, cap_akeys = 0, cap_avalues = 0, cap_upload = 0;
  void* d_upload = nullptr;  // staging for host uploads
  int* d_counter = nullptr;  // device scalar scratch
  unsigned int* d_sched = nullptr;       // fast-kernel pose tickets, kSchedSlots (one per launch in flight)
  // rotation-major grids (eval_rot): scan B rotated once per distinct rotation,
  // the permuted batch's outputs, and (vmi_eval_poses) the plan on the device
  void* d_rot = nullptr;
  size_t cap_rot = 0;
  double* d_rmi = nullptr;
  int32_t* d_rst = nullptr;
  long long* d_rtot = nullptr;
  int64_t cap_rP = 0;
  double* d_rots = nullptr;
  size_t cap_rots = 0;
  int32_t* d_ridx = nullptr;
  size_t cap_ridx = 0;
  int64_t* d_perm = nullptr;
  size_t cap_perm = 0;
  double* d_pmats = nullptr;
  size_t cap_pmats = 0;
  std::atomic<unsigned> sched_next{0};
  void* d_fix = nullptr;     // re-planned re-runs: indices, matrices, outputs
  int64_t cap_fix = 0;
  long long* d_fix_hist = nullptr;
  size_t cap_fix_hist = 0;
  int64_t replans = 0;       // times an under-estimated table plan was grown
  int64_t exact_poses = 0;   // poses re-run on the exact path
  int64_t nm_steps = 0, nm_probes = 0;  // vmi_align_pairs: lockstep steps, poses scored
  NmSlot nm_slot[2];
};

namespace {

int fail(vmi_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

int cuda_fail(vmi_ctx* c, cudaError_t e, const char* where) {
  return fail(c, VMI_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(ctx, x)                                     \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #x); \
  } while (0)

// Scan A's buffers are grow-only and reused by the next reference (a drive
// re-sets scan A every pair); only the bookkeeping is reset here.
void free_a(PairStore& ps) {
  ps.a_set = false; ps.n_avox = 0; ps.a_nvox = 0; ps.grid_bytes = 0; ps.a_npts = 0;
  ps.sat_nb = 0; ps.sparse = false;
}

void release_pair(PairStore& ps) {
  cudaFree(ps.d_grid); cudaFree(ps.d_avox); cudaFree(ps.d_bin_total); cudaFree(ps.d_pts);
  cudaFree(ps.d_hull); cudaFree(ps.d_pts_exact); cudaFree(ps.d_sat); cudaFree(ps.d_sat_bin);
  cudaFree(ps.d_hkeys); cudaFree(ps.d_hbins);
  ps = PairStore{};
}

void release_scratch(vmi_ctx* c) {
  cudaFree(c->d_avox_tmp); cudaFree(c->d_cursor); cudaFree(c->d_akeys); cudaFree(c->d_avalues);
  cudaFree(c->d_pkeys); cudaFree(c->d_pvalues); cudaFree(c->d_upload);
  c->d_avox_tmp = nullptr; c->d_cursor = nullptr; c->d_akeys = nullptr; c->d_avalues = nullptr;
  c->d_pkeys = nullptr; c->d_pvalues = nullptr; c->d_upload = nullptr;
  c->cap_avox_tmp = c->cap_akeys = c->cap_avalues = c->cap_pkeys = c->cap_pvalues = c->cap_upload = 0;
}

template <typename T>
cudaError_t grow(T** p, size_t& cap, size_t need) {
  if (need <= cap && *p) return cudaSuccess;
  cudaFree(*p);
  *p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(p, need > 0 ? need : 16);
  if (e == cudaSuccess) cap = need;
  return e;
}

RefView ref_view(const PairStore& ps) {
  RefView A{};
  for (int j = 0; j < 3; ++j) { A.amin[j] = ps.amin[j]; A.amax[j] = ps.amax[j]; A.ext[j] = ps.ext[j]; }
  A.grid = ps.sparse ? nullptr : ps.d_grid;
  A.sparse = ps.sparse ? 1 : 0;
  A.hkeys = ps.sparse ? ps.d_hkeys : nullptr;
  A.hbins = ps.sparse ? ps.d_hbins : nullptr;
  A.hmask = ps.hmask;
  A.avox = ps.d_avox;
  A.n_avox = ps.n_avox;
  A.empty = ps.a_empty ? 1 : 0;
  A.bin_total = ps.d_bin_total;
  A.sat = ps.sat_nb > 0 ? ps.d_sat : nullptr;
  A.sat_bin = ps.d_sat_bin;
  A.sat_nb = ps.sat_nb;
  return A;
}

// exact = true: the layout in the caller's point order (the exact path's
// VARZ sums depend on it); the fast kernel's may be voxel-grouped (build_b)
QueryView query_view(const vmi_ctx* c, const PairStore& ps, bool exact = false) {
  QueryView B{};
  B.pts = exact && ps.regrouped ? ps.d_pts_exact : ps.d_pts;
  B.is_f32 = ps.is_f32;
  B.n = ps.nb;
  B.span = ps.span;
  B.rem = ps.rem;
  B.threads = c->threads;
  B.max_abs = ps.max_abs;
  B.hull = ps.hull_n > 0 ? ps.d_hull : nullptr;
  B.hull_n = ps.hull_n;
  for (int j = 0; j < 3; ++j) { B.lo[j] = ps.b_lo[j]; B.hi[j] = ps.b_hi[j]; }
  return B;
}

// The fast kernel's feature kind: the user's, or occupancy when every occupied
// voxel provably takes one bin (vmi_set_params).
int kernel_kind(const vmi_ctx* c) { return c->occ ? kKindOcc : c->g.kind; }

// Largest table that fits shared memory next to the kernel's other buffers.
size_t max_table_cap(const vmi_ctx* c, int kind, int is_f32, bool multi) {
  const size_t fixed = fast_smem_bytes(kind, 0, c->g.bins, c->threads / c->streams, is_f32,
                                       c->streams, multi ? 1 : 0);
  const size_t per = (size_t)fast_slot_bytes(kind, multi ? 1 : 0);
  constexpr size_t kStaticSmem = 2048;  // the kernel's static shared memory (~1.1 KB)
  return ((c->smem_optin - kStaticSmem - fixed) / per) & ~size_t(31);
}

// Table capacity and pass count for scan B's expected occupancy `b_voxels`
// (its voxel count in its own frame).  Every slot is walked once per pose, so
// a single-pass table is sized for a ~40% load rather than filling shared
// memory; when even a full table cannot hold it, the multi-pass layout (bigger
// table) is used.
void plan_table(const vmi_ctx* c, int kind, int64_t b_voxels, int is_f32, int* cap_out,
                int* npass_out, int* multi_out) {
  static const double factor = [] {
    const char* e = std::getenv("VMI_CAP_FACTOR");  // experiments only
    // C2 (A/B, reproduced): 2.2 -> 28.98 ms, 2.0 -> 29.25, 2.5 -> 29.48; C1 flat
    return e ? std::atof(e) : 2.2;
  }();
  const double est = (double)(b_voxels > 0 ? b_voxels : 4096);
  if (c->cap_override > 0) {
    // a requested table larger than shared memory holds is clamped to the largest that fits
    const int np = c->npass_override > 0
                       ? c->npass_override
                       : std::max(1, (int)std::ceil(est / (0.70 * c->cap_override)));
    *cap_out = (int)std::min((size_t)c->cap_override, max_table_cap(c, kind, is_f32, np > 1));
    *npass_out = np;
    *multi_out = np > 1;
    return;
  }
  const size_t cap1 = max_table_cap(c, kind, is_f32, false);
  if (c->npass_override <= 1 && (c->npass_override == 1 || est <= 0.70 * (double)cap1)) {
    size_t want = ((size_t)(factor * est) + 31) & ~size_t(31);
    if (want < 2048) want = 2048;
    *cap_out = (int)std::min(cap1, want);
    *npass_out = 1;
    *multi_out = 0;
    return;
  }
  // multi-pass layout: as many passes as keep each partition at <= 70 % load
  // (one pass when scan B fits the bigger table)
  static const double factor_m = [] {
    const char* e = std::getenv("VMI_CAPM_FACTOR");  // experiments only
    // C4 (A/B): 1.4 -> 91.4 ms, 1.5 -> 93.8, 1.6 -> 95.4, full table -> 96.3;
    // 1.2 overflows on some poses (exact-path fix-ups)
    return e ? std::atof(e) : 1.4;
  }();
  const size_t capm = max_table_cap(c, kind, is_f32, true);
  *cap_out = (int)capm;
  *multi_out = 1;
  *npass_out = c->npass_override > 1
                   ? c->npass_override
                   : std::min(64, std::max(1, (int)std::ceil(est / (0.70 * (double)capm))));
  if (*npass_out == 1 && factor_m > 0.0)  // a smaller L2 scratch (grid * cap * 20 B)
    *cap_out = (int)std::min(capm, (((size_t)(factor_m * est) + 31) & ~size_t(31)));
}

int ensure_sums(vmi_ctx* c, int kind, int grid, int cap) {
  if (kind != kKindVarz) return 0;
  const size_t need = (size_t)grid * cap;
  if (need <= c->sums_n) return 0;
  cudaFree(c->d_sums);
  c->d_sums = nullptr;
  CK(c, cudaMalloc(&c->d_sums, need * (sizeof(double2) + 4)));  // sums, then (multi-pass) u32 counts
  c->sums_n = need;
  return 0;
}

// Pair ps's grid over A's AABB + voxel list from V (keys, values) on device.
int finish_reference(vmi_ctx* c, PairStore& ps, const int64_t bounds[6], int64_t V,
                     const unsigned long long* keys, const double* values) {
  ps.a_empty = V == 0;
  for (int j = 0; j < 3; ++j) {
    ps.amin[j] = (int)bounds[j];
    ps.amax[j] = (int)bounds[3 + j];
    if (bounds[j] > bounds[3 + j]) ps.a_empty = true;
  }
  ps.a_nvox = V;
  if (!ps.d_bin_total) CK(c, cudaMalloc(&ps.d_bin_total, 4 * kMaxW));
  CK(c, cudaMemsetAsync(ps.d_bin_total, 0, 4 * kMaxW, c->stream));
  if (!c->d_cursor) CK(c, cudaMalloc(&c->d_cursor, 4 * kMaxW));
  if (ps.a_empty) {
    ps.a_set = true;
    return 0;
  }
  for (int j = 0; j < 3; ++j) {
    if (bounds[j] < -(1 << 20) || bounds[3 + j] > (1 << 20) - 1)
      return fail(c, VMI_ERR_ARG, "reference bounds outside the voxel key range");
    ps.ext[j] = (uint32_t)(bounds[3 + j] - bounds[j] + 1);
  }
  const double vol = (double)ps.ext[0] * ps.ext[1] * ps.ext[2];
  // Over the dense grid's 32-bit index (or VMI_SPARSE_REF=1, tests): A as a
  // sparse key table; the fast kernel then flags every pose for the exact path.
  const char* sp_env = std::getenv("VMI_SPARSE_REF");
  ps.sparse = vol > 4294967294.0 || (sp_env && std::atoi(sp_env) != 0);
  SparseRef sp{};
  if (ps.sparse) {
    if (V > (1 << 30)) return fail(c, VMI_ERR_UNSUPPORTED, "sparse reference over 2^30 voxels");
    size_t cap = 1024;
    while (cap < 2 * (size_t)V) cap <<= 1;
    CK(c, grow(&ps.d_hkeys, ps.cap_hkeys, 8 * cap));
    CK(c, grow(&ps.d_hbins, ps.cap_hbins, cap));
    CK(c, cudaMemsetAsync(ps.d_hkeys, 0xFF, 8 * cap, c->stream));
    ps.hmask = (uint32_t)(cap - 1);
    sp = SparseRef{ps.d_hkeys, ps.d_hbins, ps.hmask};
    ps.grid_bytes = 0;
  } else {
    ps.grid_bytes = (size_t)vol;
    CK(c, grow(&ps.d_grid, ps.cap_grid, ps.grid_bytes));
    CK(c, cudaMemsetAsync(ps.d_grid, 0, ps.grid_bytes, c->stream));
  }
  CK(c, grow(&ps.d_avox, ps.cap_avox, sizeof(int4) * (V > 0 ? V : 1)));
  CK(c, grow(&c->d_avox_tmp, c->cap_avox_tmp, sizeof(int4) * (V > 0 ? V : 1)));
  CK(c, build_reference(keys, values, (int)V, nullptr, c->g, ps.amin, ps.ext,
                        ps.sparse ? nullptr : ps.d_grid, c->d_avox_tmp, ps.d_avox, ps.d_bin_total,
                        c->d_cursor, c->stream, &c->launches, sp));
  std::vector<uint32_t> tot(kMaxW);
  CK(c, cudaMemcpyAsync(tot.data(), ps.d_bin_total, 4 * kMaxW, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  int64_t s = 0;
  for (int b = 0; b < kMaxW; ++b) s += tot[b];
  ps.n_avox = (int)s;
  // summed-volume tables for the per-pose A marginal (when they fit a budget)
  ps.sat_nb = 0;
  int slot[2 * kMaxW];
  int nbp = 0;
  for (int b = 0; b < kMaxW; ++b) {
    slot[kMaxW + b] = tot[b] ? nbp : -1;
    if (tot[b]) slot[nbp++] = b;
  }
  const double cells = (double)(ps.ext[0] + 1) * (ps.ext[1] + 1) * (ps.ext[2] + 1);
  const char* sat_env = std::getenv("VMI_SAT_MB");  // table budget per pair; 0 disables
  const double budget = (sat_env ? std::atof(sat_env) : 512.0) * 1048576.0;
  if (!ps.sparse && nbp > 0 && cells * nbp * 4.0 <= budget && cells < 2147483647.0) {
    CK(c, grow(&ps.d_sat, ps.cap_sat, (size_t)(cells * nbp * 4.0)));
    if (!ps.d_sat_bin) CK(c, cudaMalloc(&ps.d_sat_bin, sizeof(int) * 2 * kMaxW));
    CK(c, cudaMemcpyAsync(ps.d_sat_bin, slot, sizeof(int) * 2 * kMaxW, cudaMemcpyHostToDevice,
                          c->stream));
    CK(c, build_sat(ps.d_avox, ps.n_avox, ps.d_sat_bin + kMaxW, nbp, ps.ext, ps.d_sat, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    ps.sat_nb = nbp;
    c->launches += 4;
  }
  ps.a_set = true;
  return 0;
}

int ensure_P(vmi_ctx* c, int64_t P, bool hist) {
  if (P <= c->cap_P && (!hist || c->hist_alloc)) return 0;
  int64_t np = P > c->cap_P ? P : c->cap_P;
  cudaFree(c->d_mats); cudaFree(c->d_mi); cudaFree(c->d_status); cudaFree(c->d_hist);
  cudaFree(c->d_total);
  c->d_hist = nullptr;
  CK(c, cudaMalloc(&c->d_mats, np * 12 * 8));
  CK(c, cudaMalloc(&c->d_mi, np * 8));
  CK(c, cudaMalloc(&c->d_status, np * 4));
  CK(c, cudaMalloc(&c->d_total, np * 8));
  const bool need_hist = hist || c->hist_alloc;
  if (need_hist) {
    const int W = c->g.bins + 1;
    CK(c, cudaMalloc(&c->d_hist, (size_t)np * W * W * 8));
  }
  c->hist_alloc = need_hist;
  c->cap_P = np;
  return 0;
}

// Pinned host staging for P poses: matrices (P x 12 f64), MI (f64) and status
// (i32) read back, and a rotation-major plan (i64 permutation, i32 rotation
// index); grow-only.
int ensure_pinned(vmi_ctx* c, int64_t P) {
  if (P <= c->h_mats_cap) return 0;
  if (c->h_mats) cudaFreeHost(c->h_mats);
  c->h_mats = nullptr;
  c->h_mats_cap = 0;
  CK(c, cudaMallocHost(&c->h_mats, (size_t)P * (96 + 12 + 12)));
  c->h_mats_cap = P;
  return 0;
}
double* pinned_mi(const vmi_ctx* c) { return c->h_mats + 12 * c->h_mats_cap; }
int64_t* pinned_perm(const vmi_ctx* c) {
  return reinterpret_cast<int64_t*>(pinned_mi(c) + c->h_mats_cap);
}
int32_t* pinned_status(const vmi_ctx* c) {
  return reinterpret_cast<int32_t*>(pinned_perm(c) + c->h_mats_cap);
}
int32_t* pinned_ridx(const vmi_ctx* c) { return pinned_status(c) + c->h_mats_cap; }

// A ticket counter for one fast-kernel launch (dynamic pose scheduling): a
// ring of slots, so launches in flight on other streams (the lockstep
// optimiser's lanes) never share one; each launch zeroes its slot in stream
// order.  VMI_SCHED=0: the static stride (A/B).
constexpr unsigned kSchedSlots = 64;
unsigned int* next_sched(vmi_ctx* c) {
  static const bool off = [] { const char* e = std::getenv("VMI_SCHED"); return e && e[0] == '0'; }();
  if (off) return nullptr;
  if (!c->d_sched && cudaMalloc(&c->d_sched, kSchedSlots * sizeof(unsigned int)) != cudaSuccess) {
    c->d_sched = nullptr;
    return nullptr;
  }
  return c->d_sched + (c->sched_next.fetch_add(1) % kSchedSlots);
}

int check_ready(vmi_ctx* c) {
  if (!c) return VMI_ERR_ARG;
  if (!c->params_set) return fail(c, VMI_ERR_STATE, "vmi_set_params not called");
  if (!c->cur.a_set) return fail(c, VMI_ERR_STATE, "scan A (reference) not set");
  if (!c->cur.b_set) return fail(c, VMI_ERR_STATE, "scan B (query) not set");
  return 0;
}

int exact_pose(vmi_ctx* c, const PairStore& ps, const double* mat_dev, int64_t p, double* mi,
               int32_t* st, long long* hist, long long* total,
               unsigned long long* hash = nullptr) {
  PointSource src{};
  src.xyz = nullptr;
  src.B = query_view(c, ps, true);
  src.n = ps.nb;
  CK(c, exact_voxelize(c->ex, src, mat_dev, c->g, c->stream, &c->launches));
  CK(c, exact_score(c->ex, c->g, ref_view(ps), p, mi, st, hist, total, c->stream, &c->launches,
                    hash));
  return 0;
}

int launch_fast_eval(vmi_ctx* c, const double* mats_dev, int64_t P, double* mi, int32_t* st,
                     long long* hist, long long* total, cudaStream_t stream) {
  if (P <= 0) return 0;
  FastLaunch fl{};
  fl.g = c->g;
  fl.g.kind = kernel_kind(c);
  fl.A = ref_view(c->cur);
  fl.B = query_view(c, c->cur);
  fl.mats = mats_dev;
  fl.P = P;
  fl.grid = (int)(P < c->sm_count ? P : c->sm_count);
  fl.sched = next_sched(c);
  fl.streams = c->streams;
  plan_table(c, fl.g.kind, c->cur.b_voxels, c->cur.is_f32, &fl.cap, &fl.npass, &fl.multi);
  int rc = ensure_sums(c, fl.g.kind, fl.grid, fl.cap);
  if (rc) return rc;
  fl.sums = c->d_sums;
  fl.mi = mi;
  fl.status = st;
  fl.hist = hist;
  fl.total = total;
  CK(c, launch_fast(fl, stream));
  c->launches += 1;
  return 0;
}

// Re-run, through the exact path, every pose whose fast-path status carries
// VMI_FLAG_RECHECK; pose_pair (host, nullable) names each pose's pair in the set.
// More than ~1% of a launch flagged means the table plan under-estimated scan
// B's occupancy (table overflow), not the rare VARZ bin-edge re-check: grow
// the estimate 4x (sticky for later launches: a bigger single-pass table, or
// the multi-pass layout) and re-run just the flagged poses through the fast
// kernel, gathered into one launch -- up to three times -- before the exact
// path takes what is still flagged.  `hs` is updated in place (own holds it).
int replan_flagged(vmi_ctx* c, const double* mats_dev, int64_t P, double* mi, int32_t* st,
                   long long* hist, long long* total, cudaStream_t stream,
                   std::vector<int32_t>& own, const int32_t*& hs) {
  const int W = c->g.bins + 1;
  if (c->cur.sparse) return 0;  // flagged by design (sparse reference), not by the table plan
  for (int attempt = 0; attempt < 3; ++attempt) {
    std::vector<int64_t> idx;
    for (int64_t p = 0; p < P; ++p)
      if (hs[p] & VMI_FLAG_RECHECK) idx.push_back(p);
    const int64_t n = (int64_t)idx.size();
    if (n <= std::max<int64_t>(16, P / 100)) return 0;
    c->cur.b_voxels = std::max<int64_t>(4 * std::max<int64_t>(c->cur.b_voxels, 1024), 4096);
    c->replans += 1;
    if (n > c->cap_fix) {
      cudaFree(c->d_fix);
      c->d_fix = nullptr;
      c->cap_fix = 0;
      CK(c, cudaMalloc(&c->d_fix, (size_t)n * (8 + 96 + 8 + 4 + 8) + 64));
      c->cap_fix = n;
    }
    int64_t* d_idx = static_cast<int64_t*>(c->d_fix);
    double* d_m = reinterpret_cast<double*>(d_idx + c->cap_fix);
    double* d_mi = d_m + 12 * c->cap_fix;
    long long* d_tot = reinterpret_cast<long long*>(d_mi + c->cap_fix);
    int32_t* d_st = reinterpret_cast<int32_t*>(d_tot + c->cap_fix);
    long long* d_h = nullptr;
    if (hist) {
      if ((size_t)n * W * W > c->cap_fix_hist) {
        cudaFree(c->d_fix_hist);
        c->d_fix_hist = nullptr;
        CK(c, cudaMalloc(&c->d_fix_hist, (size_t)n * W * W * 8));
        c->cap_fix_hist = (size_t)n * W * W;
      }
      d_h = c->d_fix_hist;
    }
    CK(c, cudaMemcpyAsync(d_idx, idx.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, stream));
    CK(c, gather_rows<double>(mats_dev, d_idx, n, 12, d_m, false, stream));
    int rc = launch_fast_eval(c, d_m, n, d_mi, d_st, d_h, d_tot, stream);
    if (rc) return rc;
    CK(c, gather_rows<double>(d_mi, d_idx, n, 1, mi, true, stream));
    CK(c, gather_rows<int32_t>(d_st, d_idx, n, 1, st, true, stream));
    if (total) CK(c, gather_rows<long long>(d_tot, d_idx, n, 1, total, true, stream));
    if (hist) CK(c, gather_rows<long long>(d_h, d_idx, n, W * W, hist, true, stream));
    c->launches += 6;
    own.resize((size_t)P);
    CK(c, cudaMemcpyAsync(own.data(), st, P * 4, cudaMemcpyDeviceToHost, stream));
    CK(c, cudaStreamSynchronize(stream));
    hs = own.data();
  }
  return 0;
}

// hs_in: the statuses already on the host (nullable: read them here); hash:
// the per-pose histogram identities to keep in step (nullable).
int do_fixups(vmi_ctx* c, const double* mats_dev, int64_t P, double* mi, int32_t* st,
              long long* hist, long long* total, cudaStream_t stream, int64_t* n_fixed,
              const int32_t* pose_pair = nullptr, const int32_t* hs_in = nullptr,
              unsigned long long* hash = nullptr) {
  std::vector<int32_t> own;
  const int32_t* hs = hs_in;
  if (!hs) {
    own.resize((size_t)P);
    CK(c, cudaMemcpyAsync(own.data(), st, P * 4, cudaMemcpyDeviceToHost, stream));
    CK(c, cudaStreamSynchronize(stream));
    hs = own.data();
  }
  int64_t nf = 0;
  if (!pose_pair) {
    int rc = replan_flagged(c, mats_dev, P, mi, st, hist, total, stream, own, hs);
    if (rc) return rc;
  }
  cudaStream_t saved = c->stream;
  c->stream = stream;
  for (int64_t p = 0; p < P; ++p) {
    if (hs[p] & VMI_FLAG_RECHECK) {
      const PairStore& ps = pose_pair ? c->set[(size_t)pose_pair[p]] : c->cur;
      int rc = exact_pose(c, ps, mats_dev + 12 * p, p, mi, st, hist, total, hash);
      if (rc) { c->stream = saved; return rc; }
      ++nf;
      c->exact_poses += 1;
    }
  }
  c->stream = saved;
  if (n_fixed) *n_fixed = nf;
  return 0;
}

// Rotation-major evaluation of a batch whose rotations repeat (pose grids):
// scan B is rotated once per distinct rotation (k_rotate, R copies of its
// span layout as double4 (R p) records), then one fast launch reads, for the
// pose in slot q, rotation ridx[q]'s copy -- the per-point FMA chains are done
// R times instead of P times, every other step is the point loop's own, so
// results are bit-identical to launch_fast_eval.  Slots are in rotation-major
// order (mats: the permuted matrices) so the CTAs, which take slots in order,
// share one rotation's copy in L2; perm[q] is slot q's pose in the caller's
// order, where the MI / statuses / totals are scattered after the fix-ups.
int64_t rot_stride(const vmi_ctx* c) {
  return (int64_t)(c->cur.span + kStagePadRows) * c->threads;
}
double rot_budget_bytes() {
  static const double b = [] {
    const char* e = std::getenv("VMI_ROT_MB");  // device memory for the rotated copies
    return (e ? std::atof(e) : 4096.0) * 1048576.0;
  }();
  return b;
}
int eval_rot(vmi_ctx* c, const double* rots12, int64_t R, const double* mats, const int32_t* ridx,
             const int64_t* perm, int64_t P, double* mi, int32_t* st, long long* total,
             cudaStream_t stream) {
  if (P <= 0) return 0;
  const PairStore& ps = c->cur;
  const int64_t stride = rot_stride(c);
  if (R <= 0 || R > 65535 || (double)R * stride * 32.0 > rot_budget_bytes())
    return fail(c, VMI_ERR_UNSUPPORTED, "rotation-major plan: too many distinct rotations");
  CK(c, grow(reinterpret_cast<char**>(&c->d_rot), c->cap_rot, (size_t)(R * stride * 32)));
  if (P > c->cap_rP) {
    cudaFree(c->d_rmi); cudaFree(c->d_rst); cudaFree(c->d_rtot);
    c->d_rmi = nullptr; c->d_rst = nullptr; c->d_rtot = nullptr; c->cap_rP = 0;
    CK(c, cudaMalloc(&c->d_rmi, (size_t)P * 8));
    CK(c, cudaMalloc(&c->d_rst, (size_t)P * 4));
    CK(c, cudaMalloc(&c->d_rtot, (size_t)P * 8));
    c->cap_rP = P;
  }
  CK(c, launch_rotate(ps.d_pts, ps.is_f32, ps.span + kStagePadRows, c->threads, rots12, R,
                      c->d_rot, stream));
  FastLaunch fl{};
  fl.g = c->g;
  fl.g.kind = kernel_kind(c);
  fl.A = ref_view(ps);
  fl.B = query_view(c, ps);
  fl.B.pts = c->d_rot;
  fl.B.is_f32 = 0;
  fl.rot_idx = ridx;
  fl.rot_stride = stride;
  fl.mats = mats;
  fl.P = P;
  fl.grid = (int)(P < c->sm_count ? P : c->sm_count);
  fl.sched = next_sched(c);
  fl.streams = c->streams;
  plan_table(c, fl.g.kind, ps.b_voxels, 2, &fl.cap, &fl.npass, &fl.multi);
  if (fl.multi)  // (the rotated kernel is single-pass: scan B's voxels fit one table)
    return fail(c, VMI_ERR_UNSUPPORTED, "rotation-major plan: multi-pass table");
  int rc = ensure_sums(c, fl.g.kind, fl.grid, fl.cap);
  if (rc) return rc;
  fl.sums = c->d_sums;
  fl.mi = c->d_rmi;
  fl.status = c->d_rst;
  fl.total = c->d_rtot;
  CK(c, launch_fast(fl, stream));
  c->launches += 2;
  if ((rc = do_fixups(c, mats, P, c->d_rmi, c->d_rst, nullptr, c->d_rtot, stream, nullptr))) return rc;
  CK(c, gather_rows<double>(c->d_rmi, perm, P, 1, mi, true, stream));
  CK(c, gather_rows<int32_t>(c->d_rst, perm, P, 1, st, true, stream));
  if (total) CK(c, gather_rows<long long>(c->d_rtot, perm, P, 1, total, true, stream));
  c->launches += total ? 3 : 2;
  return 0;
}

// Distinct rotations of P EulerPose rows (by the bits of rx, ry, rz: equal
// angles give bit-equal matrices): ridx[p] in [0, R), rep[r] = the first pose
// of rotation r.  Returns R, or -1 as soon as more than max_r are seen.
int64_t group_rotations(const double* poses, int64_t P, int64_t max_r, int32_t* ridx,
                        std::vector<int64_t>& rep) {
  size_t cap = 64;
  while (cap < 2 * (size_t)max_r + 2) cap <<= 1;
  struct Slot { uint64_t k[3]; int32_t id; };
  std::vector<Slot> tab(cap, Slot{{0, 0, 0}, -1});
  rep.clear();
  uint64_t last[3] = {~0ull, ~0ull, ~0ull};
  int32_t last_id = -1;
  for (int64_t p = 0; p < P; ++p) {
    uint64_t k[3];
    std::memcpy(k, poses + 6 * p + 3, 24);
    if (last_id >= 0 && k[0] == last[0] && k[1] == last[1] && k[2] == last[2]) {
      ridx[p] = last_id;
      continue;
    }
    uint64_t h = k[0] * 0x9E3779B97F4A7C15ull ^ (k[1] + 0x632BE59BD9B4E019ull) * 0xC2B2AE3D27D4EB4Full ^
                 (k[2] + 0x165667B19E3779F9ull) * 0x27D4EB2F165667C5ull;
    h ^= h >> 29;
    size_t i = (size_t)h & (cap - 1);
    for (;; i = (i + 1) & (cap - 1)) {
      Slot& sl = tab[i];
      if (sl.id < 0) {
        if ((int64_t)rep.size() >= max_r) return -1;
        sl.k[0] = k[0]; sl.k[1] = k[1]; sl.k[2] = k[2];
        sl.id = (int32_t)rep.size();
        rep.push_back(p);
        break;
      }
      if (sl.k[0] == k[0] && sl.k[1] == k[1] && sl.k[2] == k[2]) break;
    }
    ridx[p] = tab[i].id;
    last[0] = k[0]; last[1] = k[1]; last[2] = k[2];
    last_id = tab[i].id;
  }
  return (int64_t)rep.size();
}

}  // namespace

extern "C" {

const char* vmi_version(void) {
  return "vmi 0.1 (sm_100a; fast hash path + exact sort path)";
}

int vmi_create(int device, vmi_ctx** out) {
  if (!out) return VMI_ERR_ARG;
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n <= 0) return VMI_ERR_CUDA;
  if (device < 0 || device >= n) return VMI_ERR_ARG;
  vmi_ctx* c = new vmi_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete c; return VMI_ERR_CUDA; }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) { delete c; return VMI_ERR_CUDA; }
  if (prop.major < 10) { delete c; return VMI_ERR_UNSUPPORTED; }
  c->sm_count = prop.multiProcessorCount;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  c->smem_optin = (size_t)optin;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return VMI_ERR_CUDA;
  }
  cudaMalloc(&c->d_best, 8);
  cudaMalloc(&c->d_best_idx, 8);
  *out = c;
  return 0;
}

int vmi_destroy(vmi_ctx* c) {
  if (!c) return 0;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  release_pair(c->cur);
  for (auto& ps : c->set) release_pair(ps);
  release_scratch(c);
  cudaFree(c->d_counter); cudaFree(c->d_fix); cudaFree(c->d_fix_hist); cudaFree(c->d_sched);
  cudaFree(c->d_rot); cudaFree(c->d_rmi); cudaFree(c->d_rst); cudaFree(c->d_rtot);
  cudaFree(c->d_rots); cudaFree(c->d_ridx); cudaFree(c->d_perm); cudaFree(c->d_pmats);
  cudaFree(c->d_pairs); cudaFree(c->d_pose_pair); cudaFree(c->d_hash); cudaFree(c->d_setv);
  for (auto& l : c->lanes) {
    if (l.st) cudaStreamSynchronize(l.st);
    exact_free(l.ex);
    cudaFree(l.d_avox_tmp); cudaFree(l.d_cursor);
    if (l.done) cudaEventDestroy(l.done);
    if (l.st) cudaStreamDestroy(l.st);
  }
  if (c->set_start) cudaEventDestroy(c->set_start);
  for (auto& sl : c->nm_slot) {
    cudaFree(sl.d_buf);
    if (sl.h_buf) cudaFreeHost(sl.h_buf);
    if (sl.ev) cudaEventDestroy(sl.ev);
  }
  for (auto e : c->chunk_ev) cudaEventDestroy(e);
  cudaFree(c->d_raw); cudaFree(c->d_group); cudaFree(c->d_gavox); cudaFree(c->d_gcursor);
  exact_free(c->ex);
  cudaFree(c->d_mats); cudaFree(c->d_mi); cudaFree(c->d_status); cudaFree(c->d_hist);
  cudaFree(c->d_total); cudaFree(c->d_best); cudaFree(c->d_best_idx); cudaFree(c->d_sums);
  cudaFree(c->d_tk_keys); cudaFree(c->d_tk_idx); cudaFree(c->d_tk_out); cudaFree(c->d_tk_tmp);
  if (c->h_mats) cudaFreeHost(c->h_mats);
  if (c->copy_done) cudaEventDestroy(c->copy_done);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  cudaStreamDestroy(c->stream);
  delete c;
  return 0;
}

const char* vmi_last_error(const vmi_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t vmi_launch_count(const vmi_ctx* c) { return c ? c->launches : 0; }

int vmi_get_counters(const vmi_ctx* c, int64_t out[6]) {
  if (!c || !out) return VMI_ERR_ARG;
  out[0] = c->launches;
  out[1] = c->replans;
  out[2] = c->exact_poses;
  out[3] = c->cur.b_voxels;
  out[4] = c->nm_steps;
  out[5] = c->nm_probes;
  return 0;
}

int vmi_set_tuning(vmi_ctx* c, int table_cap_, int threads) {
  if (!c) return VMI_ERR_ARG;
  // threads = CUDA threads per CTA (one scan-B span each)
  if (threads != 0 && threads != kFastThreads)
    return fail(c, VMI_ERR_ARG, "threads must be 0 (default) or 512");
  if (table_cap_ < 0) return fail(c, VMI_ERR_ARG, "table_cap must be >= 0");
  c->cap_override = (table_cap_ + 31) & ~31;  // the clear loop writes 16-byte words
  return 0;
}

int vmi_set_passes(vmi_ctx* c, int npass) {
  if (!c) return VMI_ERR_ARG;
  if (npass < 0 || npass > 64) return fail(c, VMI_ERR_ARG, "npass must be in [0, 64]");
  c->npass_override = npass;
  return 0;
}

int vmi_set_params(vmi_ctx* c, const double origin[3], double res, int kind, int bins, double clamp,
                   int include_phi) {
  if (!c || !origin) return VMI_ERR_ARG;
  cudaSetDevice(c->device);
  for (int j = 0; j < 3; ++j)
    if (!std::isfinite(origin[j])) return fail(c, VMI_ERR_ARG, "grid origin must be finite");
  if (!(std::isfinite(res) && res > 0)) return fail(c, VMI_ERR_ARG, "grid resolution must be > 0");
  if (kind != VMI_VARZ && kind != VMI_COUNT) return fail(c, VMI_ERR_ARG, "unknown feature kind");
  if (bins < 2) return fail(c, VMI_ERR_ARG, "bin_count must be >= 2");
  if (bins > kMaxW - 1) return fail(c, VMI_ERR_UNSUPPORTED, "bin_count > 64 not supported");
  if (!(clamp > 0) || !std::isfinite(clamp)) return fail(c, VMI_ERR_ARG, "upper_clamp must be > 0");
  GridParams g{};
  for (int j = 0; j < 3; ++j) g.origin[j] = origin[j];
  g.res = res;
  int ex = 0;
  const double mant = std::frexp(res, &ex);
  const bool pow2 = mant == 0.5;
  const bool zero_origin = origin[0] == 0.0 && origin[1] == 0.0 && origin[2] == 0.0;
  g.mode = (zero_origin && res == 1.0) ? kGridUnit : (pow2 ? kGridPow2 : kGridGeneral);
  g.inv_res = 1.0 / res;  // exact for pow2; RN(1/res) for the general fast floor (k_fast.cu)
  g.kind = kind;
  g.bins = bins;
  g.clamp = clamp;
  g.include_phi = include_phi ? 1 : 0;
  // Occupancy specialisation (exact, not an approximation).  bin_feature
  // (mi.py:62-69) maps v -> 1 + min(B-1, floor(v / clamp * B)).
  //  * VARZ: a voxel's points have z within one voxel height (z in [o+k*res,
  //    o+(k+1)*res) up to rounding), and the variance of values spread over an
  //    interval of length L is at most L^2/4.  If res^2/4 * B/clamp <= 1/2,
  //    every VARZ value bins to 1 with a margin no rounding can cross: the
  //    joint histogram only depends on WHICH voxels B occupies (C4: 0.2 m,
  //    B = 32, clamp 2 -> 0.16).
  //  * COUNT: n >= 1 for an occupied voxel; if n = 1 already saturates
  //    (floor(B / clamp) >= B - 1), every voxel bins to B.
  // The fast kernel then keeps voxel keys only (no counts / sums); the exact
  // path and the feature dumps keep computing the features themselves.
  g.occ_bin = 0;
  int occ = 0;
  if (kind == VMI_VARZ && res * res / 4.0 * (double)bins / clamp <= 0.5) {
    occ = 1;
    g.occ_bin = 1;
  } else if (kind == VMI_COUNT && std::floor(1.0 / clamp * (double)bins) >= (double)(bins - 1)) {
    occ = 1;
    g.occ_bin = bins;
  }
  if (std::getenv("VMI_NO_OCC")) occ = 0;  // A/B and parity cross-checks only
  c->occ = occ;
  const bool grid_changed = !c->params_set || std::memcmp(&c->g, &g, sizeof(double) * 5) != 0 ||
                            c->g.kind != g.kind || c->g.bins != g.bins || c->g.clamp != g.clamp;
  c->g = g;
  c->params_set = true;
  if (grid_changed) {  // A's grid depends on every parameter but phi
    if (c->cur.a_set) free_a(c->cur);
    c->n_set = 0;  // the pair set too
  }
  if (c->hist_alloc) {  // W may have changed
    cudaFree(c->d_hist);
    c->d_hist = nullptr;
    c->hist_alloc = false;
    c->cap_P = 0;
  }
  return 0;
}

// Scan A of pair ps from host points: (n, 3) float64, or (n, 4) float32 KITTI
// records uploaded as they are (16 B/point, widened exactly on the GPU):
// _prepare (align.py:114-119) = voxelize + compute_feature_map, bit-exact,
// then the dense bin grid.  The FeatureMap stays in (keys, values) -- the
// current pair's export buffers, or the pair-set build scratch.
static int build_a(vmi_ctx* c, PairStore& ps, const void* host, int is_rec, int64_t n,
                   unsigned long long** keys, double** values, size_t* cap_k, size_t* cap_v) {
  if (n <= 0 || !host) return fail(c, VMI_ERR_ARG, "cannot voxelize an empty cloud");
  if (n > 0x7fffffff) return fail(c, VMI_ERR_UNSUPPORTED, "more than 2^31-1 points");
  if (is_rec) {  // PointCloud validation (geometry.py:36-65): finite coordinates
    const float* r = static_cast<const float*>(host);
    for (int64_t i = 0; i < n; ++i)
      if (!(std::isfinite(r[4 * i]) && std::isfinite(r[4 * i + 1]) && std::isfinite(r[4 * i + 2])))
        return fail(c, VMI_ERR_ARG, "points contain non-finite coordinates");
  }
  free_a(ps);
  const size_t bytes = (size_t)n * (is_rec ? 16 : 24);
  CK(c, grow(&c->d_upload, c->cap_upload, bytes));
  CK(c, cudaMemcpyAsync(c->d_upload, host, bytes, cudaMemcpyHostToDevice, c->stream));
  PointSource src{};
  if (is_rec)
    src.rec = static_cast<const float4*>(c->d_upload);
  else
    src.xyz = static_cast<const double*>(c->d_upload);
  src.n = n;
  CK(c, exact_voxelize(c->ex, src, nullptr, c->g, c->stream, &c->launches));
  int h[8];
  int V = 0;
  CK(c, cudaMemcpyAsync(h, c->ex.bounds, 7 * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(&V, c->ex.nruns, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (h[6]) return fail(c, VMI_ERR_RANGE, "a point of scan A maps outside the voxel key range");
  CK(c, grow(keys, *cap_k, 8 * (size_t)V));
  CK(c, grow(values, *cap_v, 8 * (size_t)V));
  CK(c, cudaMemcpyAsync(*keys, c->ex.ukeys, 8 * (size_t)V, cudaMemcpyDeviceToDevice, c->stream));
  CK(c, cudaMemcpyAsync(*values, c->ex.values, 8 * (size_t)V, cudaMemcpyDeviceToDevice, c->stream));
  int64_t b64[6];
  for (int j = 0; j < 6; ++j) b64[j] = h[j];
  const int rc = finish_reference(c, ps, b64, V, *keys, *values);
  ps.a_npts = n;
  return rc;
}

static int set_reference(vmi_ctx* c, const void* host, int is_rec, int64_t n) {
  if (!c) return VMI_ERR_ARG;
  if (!c->params_set) return fail(c, VMI_ERR_STATE, "vmi_set_params not called");
  cudaSetDevice(c->device);
  return build_a(c, c->cur, host, is_rec, n, &c->d_akeys, &c->d_avalues, &c->cap_akeys,
                 &c->cap_avalues);
}

int vmi_set_reference_points(vmi_ctx* c, const double* xyz, int64_t n) {
  return set_reference(c, xyz, 0, n);
}

int vmi_set_reference_records_f32(vmi_ctx* c, const float* xyzi, int64_t n) {
  return set_reference(c, xyzi, 1, n);
}

int vmi_set_reference_features(vmi_ctx* c, const int64_t* keys, const double* values, int64_t n,
                               const int64_t bounds[6]) {
  if (!c || !bounds || n < 0 || (n > 0 && (!keys || !values))) return VMI_ERR_ARG;
  if (!c->params_set) return fail(c, VMI_ERR_STATE, "vmi_set_params not called");
  if (n > 0x7fffffff) return fail(c, VMI_ERR_UNSUPPORTED, "more than 2^31-1 voxels");
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(values[i]) || values[i] < 0)
      return fail(c, VMI_ERR_ARG, "features must be finite and >= 0");
  cudaSetDevice(c->device);
  free_a(c->cur);
  const size_t m = n > 0 ? (size_t)n : 1;
  CK(c, grow(&c->d_akeys, c->cap_akeys, 8 * m));
  CK(c, grow(&c->d_avalues, c->cap_avalues, 8 * m));
  if (n > 0) {
    CK(c, cudaMemcpyAsync(c->d_akeys, keys, 8 * n, cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(c->d_avalues, values, 8 * n, cudaMemcpyHostToDevice, c->stream));
  }
  return finish_reference(c, c->cur, bounds, n, c->d_akeys, c->d_avalues);
}

int vmi_get_reference_features(vmi_ctx* c, int64_t* keys, double* values, int64_t cap,
                               int64_t* n_out, int64_t bounds[6]) {
  if (!c) return VMI_ERR_ARG;
  if (!c->cur.a_set) return fail(c, VMI_ERR_STATE, "scan A (reference) not set");
  cudaSetDevice(c->device);
  if (n_out) *n_out = c->cur.a_nvox;
  if (bounds)
    for (int j = 0; j < 3; ++j) { bounds[j] = c->cur.amin[j]; bounds[3 + j] = c->cur.amax[j]; }
  if (!keys) return 0;
  if (cap < c->cur.a_nvox) return fail(c, VMI_ERR_ARG, "output capacity too small");
  if (c->cur.a_nvox > 0) {
    CK(c, cudaMemcpyAsync(keys, c->d_akeys, 8 * c->cur.a_nvox, cudaMemcpyDeviceToHost, c->stream));
    if (values)
      CK(c, cudaMemcpyAsync(values, c->d_avalues, 8 * c->cur.a_nvox, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(c, cudaStreamSynchronize(c->stream));
  return 0;
}

static bool f32_exact(double v) { return (double)(float)v == v; }

// Scan B of pair ps: one host pass (PointCloud validation, AABB, float32-
// exactness), the upload as given (float32 records 16 B/point, or float64
// 24 B/point), and the span layout on the GPU: split-double float4 records
// when every coordinate is float32-exact (KITTI input), else double4.
static int build_b(vmi_ctx* c, PairStore& ps, const void* host, int is_f32_src, int64_t n) {
  if (n <= 0 || !host) return fail(c, VMI_ERR_ARG, "cannot voxelize an empty cloud");
  if (n > 0x7fffffff) return fail(c, VMI_ERR_UNSUPPORTED, "more than 2^31-1 points");
  ps.b_set = false;
  ps.hull_n = 0;
  // VMI_FORCE_F64 (experiments): keep double records even for float32-exact input
  static const bool force_f64 = std::getenv("VMI_FORCE_F64") != nullptr;
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  bool exact32 = true;
  if (is_f32_src) {
    const float* r = static_cast<const float*>(host);
    float flo[3] = {INFINITY, INFINITY, INFINITY}, fhi[3] = {-INFINITY, -INFINITY, -INFINITY};
    bool finite = true;
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < 3; ++j) {
        const float v = r[4 * i + j];
        finite &= std::isfinite(v);
        flo[j] = std::fmin(flo[j], v);
        fhi[j] = std::fmax(fhi[j], v);
      }
    if (!finite) return fail(c, VMI_ERR_ARG, "points contain non-finite coordinates");
    for (int j = 0; j < 3; ++j) { lo[j] = flo[j]; hi[j] = fhi[j]; }
  } else {
    const double* xyz = static_cast<const double*>(host);
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < 3; ++j) {
        const double v = xyz[3 * i + j];
        exact32 &= f32_exact(v);
        lo[j] = std::fmin(lo[j], v);
        hi[j] = std::fmax(hi[j], v);
      }
  }
  const int as_f32 = (exact32 && !force_f64) ? 1 : 0;
  double mx = 0.0;
  for (int j = 0; j < 3; ++j) {
    mx = std::fmax(mx, std::fmax(std::fabs(lo[j]), std::fabs(hi[j])));
    ps.b_lo[j] = lo[j];
    ps.b_hi[j] = hi[j];
  }
  ps.max_abs = mx;
  const int rb = is_f32_src ? 16 : 24;
  const size_t up_bytes = (size_t)n * rb;
  CK(c, grow(&c->d_upload, c->cap_upload, 2 * up_bytes));  // + a voxel-grouped copy
  CK(c, cudaMemcpyAsync(c->d_upload, host, up_bytes, cudaMemcpyHostToDevice, c->stream));
  ps.span = (int)((n + c->threads - 1) / c->threads);
  ps.rem = (int)(n - (int64_t)(ps.span - 1) * c->threads);
  const size_t rec = as_f32 ? 16 : 32;
  const size_t layout_bytes = (size_t)(ps.span + kStagePadRows) * c->threads * rec;
  // scan B voxelized at the identity pose: its voxel count sizes the fast
  // kernel's table, and its point order decides the layout.  The fused kernel
  // aggregates runs of consecutive points in one voxel: a ring-ordered LiDAR
  // scan runs ~12 points per voxel run, an unordered one (e.g. the reference's
  // synth_scene_pair) ~1.  Unordered scans (mean run < 1.25 points) get the
  // fast layout in voxel-grouped order (the stable sort's), while the exact
  // path keeps the original order (its VARZ sums follow numpy's order over it,
  // voxel.py:225-229); every result is order-free otherwise (counts, bounds;
  // the fast VARZ is checked against bin edges), hence identical.
  const char* rg = std::getenv("VMI_REGROUP");  // "0": keep the input order (A/B, tests)
  const bool no_regroup = rg && std::strcmp(rg, "0") == 0;
  bool regroup = false;
  ps.b_voxels = 0;
  if (c->params_set) {
    PointSource src{};
    if (is_f32_src) src.rec = static_cast<const float4*>(c->d_upload);
    else src.xyz = static_cast<const double*>(c->d_upload);
    src.n = n;
    CK(c, exact_voxelize(c->ex, src, nullptr, c->g, c->stream, &c->launches));
    if (!c->d_counter) CK(c, cudaMalloc(&c->d_counter, 16));
    CK(c, voxel_order(c->ex, c->d_upload, rb, n, c->d_counter, nullptr, c->stream));
    int h[2] = {0, 0};
    CK(c, cudaMemcpyAsync(&h[0], c->ex.nruns, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaMemcpyAsync(&h[1], c->d_counter, 4, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
    ps.b_voxels = h[0];
    if (const char* e = std::getenv("VMI_EST_SCALE"))  // tests: mis-estimate the occupancy
      ps.b_voxels = std::max<int64_t>(1, (int64_t)(ps.b_voxels * std::atof(e)));
    regroup = !no_regroup && (double)(h[1] + 1) * 1.25 >= (double)n && n > 1;
  }
  char* ordered = static_cast<char*>(c->d_upload);
  if (regroup) {  // fast layout from the voxel-grouped copy, exact layout from the original
    ordered += up_bytes;
    CK(c, voxel_order(c->ex, c->d_upload, rb, n, c->d_counter, ordered, c->stream));
    CK(c, grow(&ps.d_pts_exact, ps.cap_pts_exact, layout_bytes));
    CK(c, launch_span_layout(c->d_upload, is_f32_src, as_f32, n, ps.span, ps.rem, c->threads,
                             ps.d_pts_exact, c->stream));
    c->launches += 3;
  }
  ps.regrouped = regroup;
  CK(c, grow(&ps.d_pts, ps.cap_pts, layout_bytes));
  CK(c, launch_span_layout(ordered, is_f32_src, as_f32, n, ps.span, ps.rem, c->threads,
                           ps.d_pts, c->stream));
  c->launches += 1;
  ps.is_f32 = as_f32;
  ps.nb = n;
  if (ps.b_voxels <= 0 && ps.a_set && ps.a_npts > 0 && ps.a_nvox > 0)  // (params unset: unreachable)
    ps.b_voxels = (int64_t)((double)ps.a_nvox * (double)n / (double)ps.a_npts) + 1;
  CK(c, cudaStreamSynchronize(c->stream));  // the host buffer may be reused on return
  ps.b_set = true;
  return 0;
}

static int set_query(vmi_ctx* c, const void* host, int is_f32_src, int64_t n) {
  if (!c) return VMI_ERR_ARG;
  cudaSetDevice(c->device);
  return build_b(c, c->cur, host, is_f32_src, n);
}

int vmi_set_query_points(vmi_ctx* c, const double* xyz, int64_t n) { return set_query(c, xyz, 0, n); }

int vmi_set_query_hull(vmi_ctx* c, const double* xyz, int64_t n) {
  if (!c || n < 0 || (n > 0 && !xyz)) return VMI_ERR_ARG;
  if (!c->cur.b_set) return fail(c, VMI_ERR_STATE, "scan B (query) not set");
  if (n > (1 << 24)) return fail(c, VMI_ERR_UNSUPPORTED, "hull of more than 2^24 points");
  for (int64_t i = 0; i < 3 * n; ++i)
    if (!std::isfinite(xyz[i])) return fail(c, VMI_ERR_ARG, "hull points must be finite");
  cudaSetDevice(c->device);
  PairStore& ps = c->cur;
  ps.hull_n = 0;
  if (n == 0) return 0;
  CK(c, grow(&ps.d_hull, ps.cap_hull, 24 * (size_t)n));
  CK(c, cudaMemcpyAsync(ps.d_hull, xyz, 24 * (size_t)n, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  ps.hull_n = (int)n;
  return 0;
}

int vmi_set_query_records_f32(vmi_ctx* c, const float* xyzi, int64_t n) {
  return set_query(c, xyzi, 1, n);
}

int vmi_eval_device(vmi_ctx* c, const double* mats_dev, int64_t P, double* mi_dev,
                    int32_t* status_dev, int64_t* hist_dev, int64_t* total_dev, void* stream) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (P < 0 || (P > 0 && (!mats_dev || !mi_dev || !status_dev))) return fail(c, VMI_ERR_ARG, "bad arguments");
  cudaSetDevice(c->device);
  return launch_fast_eval(c, mats_dev, P, mi_dev, status_dev, (long long*)hist_dev,
                          (long long*)total_dev, stream ? (cudaStream_t)stream : c->stream);
}

int vmi_eval_fixups(vmi_ctx* c, const double* mats_dev, int64_t P, double* mi_dev,
                    int32_t* status_dev, int64_t* hist_dev, int64_t* total_dev, void* stream,
                    int64_t* n_fixed) {
  int rc = check_ready(c);
  if (rc) return rc;
  cudaSetDevice(c->device);
  return do_fixups(c, mats_dev, P, mi_dev, status_dev, (long long*)hist_dev, (long long*)total_dev,
                   stream ? (cudaStream_t)stream : c->stream, n_fixed);
}

int vmi_eval_rot_device(vmi_ctx* c, const double* rots12_dev, int64_t R, const double* mats_dev,
                        const int32_t* rot_idx_dev, const int64_t* perm_dev, int64_t P,
                        double* mi_dev, int32_t* status_dev, int64_t* total_dev, void* stream) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (P < 0 || (P > 0 && (!rots12_dev || !mats_dev || !rot_idx_dev || !perm_dev || !mi_dev ||
                          !status_dev)))
    return fail(c, VMI_ERR_ARG, "bad arguments");
  cudaSetDevice(c->device);
  return eval_rot(c, rots12_dev, R, mats_dev, rot_idx_dev, perm_dev, P, mi_dev, status_dev,
                  (long long*)total_dev, stream ? (cudaStream_t)stream : c->stream);
}

int vmi_eval(vmi_ctx* c, const double* mats, int64_t P, double* mi_out, int32_t* status_out,
             int64_t* hist_out, int64_t* total_out) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (P < 0 || (P > 0 && (!mats || !mi_out || !status_out))) return fail(c, VMI_ERR_ARG, "bad arguments");
  if (P == 0) return 0;
  cudaSetDevice(c->device);
  if ((rc = ensure_P(c, P, hist_out != nullptr))) return rc;
  long long* dh = hist_out ? c->d_hist : nullptr;
  CK(c, cudaMemcpyAsync(c->d_mats, mats, P * 96, cudaMemcpyHostToDevice, c->stream));
  if ((rc = launch_fast_eval(c, c->d_mats, P, c->d_mi, c->d_status, dh, c->d_total, c->stream))) return rc;
  if ((rc = do_fixups(c, c->d_mats, P, c->d_mi, c->d_status, dh, c->d_total, c->stream, nullptr))) return rc;
  CK(c, cudaMemcpyAsync(mi_out, c->d_mi, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(status_out, c->d_status, P * 4, cudaMemcpyDeviceToHost, c->stream));
  if (hist_out) {
    const int W = c->g.bins + 1;
    CK(c, cudaMemcpyAsync(hist_out, dh, (size_t)P * W * W * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (total_out) CK(c, cudaMemcpyAsync(total_out, c->d_total, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return 0;
}

extern "C" int vmi_poses_to_mats(const double* poses, int64_t n, double* mats, int threads);

// Poses in, MI out, with the host work hidden behind the GPU: the first
// `head` poses are converted (glibc sin/cos, pose_host.cpp) into pinned
// memory, uploaded and launched; the host converts the rest while that kernel
// runs, and their upload runs on a second stream beside it.  Same results as
// vmi_poses_to_mats + vmi_eval.
// vmi_eval_poses on a pose grid (rotations repeat): all matrices on the host
// pool, the rotation plan (group_rotations, a stable counting sort into
// rotation-major slots), then eval_rot.  Returns 1 when the batch is not a
// grid (the caller takes the pipelined path), 0 on success, < 0 on error.
static int eval_poses_rot(vmi_ctx* c, const double* poses, int64_t P, double* mi_out,
                          int32_t* status_out, int64_t* total_out) {
  // Opt-in (VMI_ROT=1): measured slower on B200 -- the rotated copies are
  // 32-byte double4 records (the exact f64 chain results), twice the float4
  // split records' L2 traffic, and the point loop becomes L2-bound (C3 529 ms
  // vs 388 ms per 970,299 poses; C1 1.94 vs 1.69 ms).
  const char* on = std::getenv("VMI_ROT");
  if (!on || on[0] != '1' || P < 4096 || c->cur.sparse) return 1;
  int32_t* ridx = pinned_ridx(c);
  std::vector<int64_t> rep;
  if (group_rotations(poses, std::min<int64_t>(P, 4096), 512, ridx, rep) < 0) return 1;  // random poses
  const int64_t R = group_rotations(poses, P, std::min<int64_t>(P / 16, 65535), ridx, rep);
  if (R <= 0 || (double)R * rot_stride(c) * 32.0 > rot_budget_bytes()) return 1;
  {  // the rotated kernel is single-pass: skip grids whose table would need passes
    int cap = 0, np = 0, multi = 0;
    plan_table(c, kernel_kind(c), c->cur.b_voxels, 2, &cap, &np, &multi);
    if (multi) return 1;
  }
  if (vmi_poses_to_mats(poses, P, c->h_mats, 0)) return fail(c, VMI_ERR_ARG, "poses contain non-finite components");
  // stable counting sort by rotation: perm[q] = the pose in slot q
  int64_t* perm = pinned_perm(c);
  int32_t* ridx_q = pinned_status(c);  // (scratch until the statuses come back)
  std::vector<int64_t> start((size_t)R + 1, 0);
  for (int64_t p = 0; p < P; ++p) ++start[(size_t)ridx[p] + 1];
  for (int64_t r = 0; r < R; ++r) start[(size_t)r + 1] += start[(size_t)r];
  for (int64_t p = 0; p < P; ++p) {
    const int64_t q = start[(size_t)ridx[p]]++;
    perm[q] = p;
    ridx_q[q] = ridx[p];
  }
  std::vector<double> rots((size_t)R * 12);
  for (int64_t r = 0; r < R; ++r)
    std::memcpy(&rots[(size_t)r * 12], c->h_mats + 12 * rep[(size_t)r], 96);
  CK(c, grow(&c->d_rots, c->cap_rots, (size_t)R * 96));
  CK(c, grow(&c->d_ridx, c->cap_ridx, (size_t)P * 4));
  CK(c, grow(&c->d_perm, c->cap_perm, (size_t)P * 8));
  CK(c, grow(&c->d_pmats, c->cap_pmats, (size_t)P * 96));
  CK(c, cudaMemcpyAsync(c->d_mats, c->h_mats, (size_t)P * 96, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaMemcpyAsync(c->d_perm, perm, (size_t)P * 8, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaMemcpyAsync(c->d_ridx, ridx_q, (size_t)P * 4, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaMemcpyAsync(c->d_rots, rots.data(), (size_t)R * 96, cudaMemcpyHostToDevice, c->stream));
  CK(c, gather_rows<double>(c->d_mats, c->d_perm, P, 12, c->d_pmats, false, c->stream));
  c->launches += 1;
  int rc = eval_rot(c, c->d_rots, R, c->d_pmats, c->d_ridx, c->d_perm, P, c->d_mi, c->d_status,
                    total_out ? c->d_total : nullptr, c->stream);
  if (rc) return rc;
  double* hmi = pinned_mi(c);
  int32_t* hst = pinned_status(c);
  CK(c, cudaMemcpyAsync(hmi, c->d_mi, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(hst, c->d_status, P * 4, cudaMemcpyDeviceToHost, c->stream));
  if (total_out) CK(c, cudaMemcpyAsync(total_out, c->d_total, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  std::memcpy(mi_out, hmi, (size_t)P * 8);
  std::memcpy(status_out, hst, (size_t)P * 4);
  return 0;
}

int vmi_eval_poses(vmi_ctx* c, const double* poses, int64_t P, double* mi_out, int32_t* status_out,
                   int64_t* hist_out, int64_t* total_out) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (P < 0 || (P > 0 && (!poses || !mi_out || !status_out))) return fail(c, VMI_ERR_ARG, "bad arguments");
  if (P == 0) return 0;
  cudaSetDevice(c->device);
  if ((rc = ensure_P(c, P, hist_out != nullptr)) || (rc = ensure_pinned(c, P))) return rc;
  if (!hist_out) {  // pose grids: rotation-major (one rotated scan B per distinct rotation)
    rc = eval_poses_rot(c, poses, P, mi_out, status_out, total_out);
    if (rc <= 0) return rc;
  }
  if (!c->copy_stream) CK(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  if (!c->copy_done) CK(c, cudaEventCreateWithFlags(&c->copy_done, cudaEventDisableTiming));
  static const bool trace = std::getenv("VMI_TRACE") != nullptr;  // phase timings to stderr
  const auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (trace)
      std::fprintf(stderr, "[vmi_eval_poses] %-14s %8.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  };
  const int W = c->g.bins + 1;
  long long* dh = hist_out ? c->d_hist : nullptr;
  // head: long enough for its kernel (~0.4 us/pose at C2) to cover the host
  // conversion of the rest (~8 ns/pose on the box's 16 pooled threads, with
  // wake-up jitter up to ~1 ms) and its upload (VMI_TRACE: P/32 left GPU
  // gaps of up to 0.2 ms before the tail launch)
  const int64_t head = P < 8192 ? P : std::max<int64_t>(2048, P / 16);
  if (vmi_poses_to_mats(poses, head, c->h_mats, 0)) return fail(c, VMI_ERR_ARG, "poses contain non-finite components");
  CK(c, cudaMemcpyAsync(c->d_mats, c->h_mats, head * 96, cudaMemcpyHostToDevice, c->stream));
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};  // VMI_TRACE: GPU phase times
  if (trace)
    for (auto& e : tev) cudaEventCreate(&e);
  if (trace) cudaEventRecord(tev[0], c->stream);
  if ((rc = launch_fast_eval(c, c->d_mats, head, c->d_mi, c->d_status, dh, c->d_total, c->stream))) return rc;
  if (trace) cudaEventRecord(tev[1], c->stream);
  lap("head launched");
  if (P > head) {
    const int64_t n = P - head;
    if (vmi_poses_to_mats(poses + 6 * head, n, c->h_mats + 12 * head, 0)) {
      cudaStreamSynchronize(c->stream);
      return fail(c, VMI_ERR_ARG, "poses contain non-finite components");
    }
    lap("tail converted");
    CK(c, cudaMemcpyAsync(c->d_mats + 12 * head, c->h_mats + 12 * head, n * 96,
                          cudaMemcpyHostToDevice, c->copy_stream));
    CK(c, cudaEventRecord(c->copy_done, c->copy_stream));
    CK(c, cudaStreamWaitEvent(c->stream, c->copy_done, 0));
    if (trace) cudaEventRecord(tev[2], c->stream);
    if ((rc = launch_fast_eval(c, c->d_mats + 12 * head, n, c->d_mi + head, c->d_status + head,
                               dh ? dh + (size_t)head * W * W : nullptr, c->d_total + head,
                               c->stream)))
      return rc;
    if (trace) cudaEventRecord(tev[3], c->stream);
  }
  // MI + status through pinned staging; the statuses read back also tell
  // do_fixups which poses to re-run (no second status read)
  double* hmi = pinned_mi(c);
  int32_t* hst = pinned_status(c);
  CK(c, cudaMemcpyAsync(hmi, c->d_mi, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(hst, c->d_status, P * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  lap("kernels done");
  if (trace && P > head) {
    float h = 0, g = 0, t = 0;
    cudaEventElapsedTime(&h, tev[0], tev[1]);
    cudaEventElapsedTime(&g, tev[1], tev[2]);
    cudaEventElapsedTime(&t, tev[2], tev[3]);
    std::fprintf(stderr, "[vmi_eval_poses] gpu: head %.3f ms, gap %.3f ms, tail %.3f ms\n", h, g, t);
  }
  if (trace)
    for (auto& e : tev) if (e) cudaEventDestroy(e);
  bool flagged = false;
  for (int64_t p = 0; p < P && !flagged; ++p) flagged = (hst[p] & VMI_FLAG_RECHECK) != 0;
  if (flagged) {
    std::vector<int32_t> hs(hst, hst + P);
    if ((rc = do_fixups(c, c->d_mats, P, c->d_mi, c->d_status, dh, c->d_total, c->stream, nullptr,
                        nullptr, hs.data())))
      return rc;
    CK(c, cudaMemcpyAsync(hmi, c->d_mi, P * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaMemcpyAsync(hst, c->d_status, P * 4, cudaMemcpyDeviceToHost, c->stream));
  }
  if (hist_out)
    CK(c, cudaMemcpyAsync(hist_out, dh, (size_t)P * W * W * 8, cudaMemcpyDeviceToHost, c->stream));
  if (total_out) CK(c, cudaMemcpyAsync(total_out, c->d_total, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  std::memcpy(mi_out, hmi, (size_t)P * 8);
  std::memcpy(status_out, hst, (size_t)P * 4);
  lap("results copied");
  return 0;
}

int vmi_eval_exact(vmi_ctx* c, const double* mats, int64_t P, double* mi_out, int32_t* status_out,
                   int64_t* hist_out, int64_t* total_out) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (P < 0 || (P > 0 && (!mats || !mi_out || !status_out))) return fail(c, VMI_ERR_ARG, "bad arguments");
  if (P == 0) return 0;
  cudaSetDevice(c->device);
  if ((rc = ensure_P(c, P, hist_out != nullptr))) return rc;
  long long* dh = hist_out ? c->d_hist : nullptr;
  CK(c, cudaMemcpyAsync(c->d_mats, mats, P * 96, cudaMemcpyHostToDevice, c->stream));
  for (int64_t p = 0; p < P; ++p)
    if ((rc = exact_pose(c, c->cur, c->d_mats + 12 * p, p, c->d_mi, c->d_status, dh, c->d_total)))
      return rc;
  CK(c, cudaMemcpyAsync(mi_out, c->d_mi, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(status_out, c->d_status, P * 4, cudaMemcpyDeviceToHost, c->stream));
  if (hist_out) {
    const int W = c->g.bins + 1;
    CK(c, cudaMemcpyAsync(hist_out, dh, (size_t)P * W * W * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if (total_out) CK(c, cudaMemcpyAsync(total_out, c->d_total, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return 0;
}

int vmi_query_features(vmi_ctx* c, const double mat[12], int64_t* keys, double* values, int64_t cap,
                       int64_t* n_out, int64_t bounds[6], int32_t* status) {
  if (!c || !mat) return VMI_ERR_ARG;
  if (!c->params_set || !c->cur.b_set) return fail(c, VMI_ERR_STATE, "params and scan B must be set");
  cudaSetDevice(c->device);
  int rc;
  if ((rc = ensure_P(c, 1, false))) return rc;
  CK(c, cudaMemcpyAsync(c->d_mats, mat, 96, cudaMemcpyHostToDevice, c->stream));
  PointSource src{};
  src.B = query_view(c, c->cur, true);
  src.n = c->cur.nb;
  CK(c, exact_voxelize(c->ex, src, c->d_mats, c->g, c->stream, &c->launches));
  int h[8];
  int V = 0;
  CK(c, cudaMemcpyAsync(h, c->ex.bounds, 7 * 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(&V, c->ex.nruns, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (status) *status = h[6] ? VMI_KEY_RANGE : VMI_OK;
  if (n_out) *n_out = V;
  if (bounds)
    for (int j = 0; j < 6; ++j) bounds[j] = h[j];
  if (h[6] || !keys) return 0;
  if (cap < V) return fail(c, VMI_ERR_ARG, "output capacity too small");
  CK(c, cudaMemcpyAsync(keys, c->ex.ukeys, 8 * (size_t)V, cudaMemcpyDeviceToHost, c->stream));
  if (values)
    CK(c, cudaMemcpyAsync(values, c->ex.values, 8 * (size_t)V, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  return 0;
}

int vmi_fast_features(vmi_ctx* c, const double mat[12], int64_t* keys, double* values, int64_t cap,
                      int64_t* n_out, int32_t* status) {
  int rc = check_ready(c);
  if (rc) return rc;
  if (!mat || !n_out || cap < 0) return fail(c, VMI_ERR_ARG, "bad arguments");
  cudaSetDevice(c->device);
  if ((rc = ensure_P(c, 1, false))) return rc;
  const int64_t m = cap > 0 ? cap : 1;
  unsigned long long* dk = nullptr;
  double* dv = nullptr;
  int* dn = nullptr;
  CK(c, cudaMalloc(&dk, 8 * m));
  CK(c, cudaMalloc(&dv, 8 * m));
  CK(c, cudaMalloc(&dn, 4));
  CK(c, cudaMemsetAsync(dn, 0, 4, c->stream));
  CK(c, cudaMemcpyAsync(c->d_mats, mat, 96, cudaMemcpyHostToDevice, c->stream));
  FastLaunch fl{};
  fl.g = c->g;
  fl.A = ref_view(c->cur);
  fl.B = query_view(c, c->cur);
  fl.mats = c->d_mats;
  fl.P = 1;
  // the user's kind: dumps need features
  plan_table(c, fl.g.kind, c->cur.b_voxels, c->cur.is_f32, &fl.cap, &fl.npass, &fl.multi);
  fl.grid = 1;
  fl.streams = c->streams;
  if ((rc = ensure_sums(c, fl.g.kind, 1, fl.cap))) return rc;
  fl.sums = c->d_sums;
  fl.mi = c->d_mi;
  fl.status = c->d_status;
  fl.total = c->d_total;
  fl.dump.keys = dk;
  fl.dump.values = dv;
  fl.dump.n = dn;
  fl.dump.cap = (int)m;
  CK(c, launch_fast(fl, c->stream));
  c->launches += 1;
  int n = 0;
  CK(c, cudaMemcpyAsync(&n, dn, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(status, c->d_status, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  *n_out = n;
  if (n <= cap && n > 0 && keys) {
    CK(c, cudaMemcpyAsync(keys, dk, 8 * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
    if (values) CK(c, cudaMemcpyAsync(values, dv, 8 * (size_t)n, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaStreamSynchronize(c->stream));
  }
  cudaFree(dk); cudaFree(dv); cudaFree(dn);
  return 0;
}

// ---- many resident scan pairs (C5: consecutive pairs of a drive) ----------

namespace {

// One host pass over a scan: PointCloud validation (finite coordinates), the
// AABB, and (float64 input) whether every coordinate is float32-exact.
struct HostScan {
  double lo[3], hi[3];
  bool finite = true, exact32 = true;
};
void scan_pass(const void* p, int is_rec, int64_t n, HostScan& o) {
  // branch-free min / max / finiteness (vectorisable; a NaN or inf anywhere
  // sets `bad` -- |v| <= FLT_MAX / DBL_MAX is false for both)
  if (is_rec) {
    const float* r = static_cast<const float*>(p);
    float lo[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
    float hi[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
    int bad[4] = {0, 0, 0, 0};
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < 4; ++j) {  // all four fields: the intensity's are ignored below
        const float v = r[4 * i + j];
        lo[j] = v < lo[j] ? v : lo[j];
        hi[j] = v > hi[j] ? v : hi[j];
        bad[j] |= !(std::fabs(v) <= 3.4028234663852886e+38f);
      }
    o.finite = !(bad[0] | bad[1] | bad[2]);
    for (int j = 0; j < 3; ++j) { o.lo[j] = lo[j]; o.hi[j] = hi[j]; }
  } else {
    const double* d = static_cast<const double*>(p);
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    int bad = 0, inexact = 0;
    for (int64_t i = 0; i < n; ++i)
      for (int j = 0; j < 3; ++j) {
        const double v = d[3 * i + j];
        lo[j] = v < lo[j] ? v : lo[j];
        hi[j] = v > hi[j] ? v : hi[j];
        bad |= !(std::fabs(v) <= 1.7976931348623157e+308);
        inexact |= (double)(float)v != v;
      }
    o.finite = !bad;
    o.exact32 = !inexact;
    for (int j = 0; j < 3; ++j) { o.lo[j] = lo[j]; o.hi[j] = hi[j]; }
  }
}

// voxel.py:199 on the host for a coordinate: floor(RN(RN(p - o) / res)).  The
// quotient is monotone in p, so the voxel bounds of a scan are the floors of
// its AABB corners -- the same integers the GPU reduces (voxel.py:220).
int64_t host_floor(double p, double o, double res) { return (int64_t)std::floor((p - o) / res); }

}  // namespace

// Pairs are built without a host round trip per pair.  Distinct scans (a drive
// shares one scan between consecutive pairs) are validated once on the host
// (threaded) and uploaded once into a raw device pool, in chunks on a copy
// stream; kBuildLanes streams then build pairs side by side: scan A's voxel
// bounds come from its AABB on the host (exact, see host_floor), its voxel
// list is sized by the point count, and the voxel counts of the whole set are
// read back once at the end.
int vmi_set_pairs(vmi_ctx* c, int64_t npairs, const void* const* a, const int64_t* na,
                  const void* const* b, const int64_t* nb, int is_rec) {
  if (!c || npairs < 0 || (npairs > 0 && (!a || !na || !b || !nb))) return VMI_ERR_ARG;
  if (!c->params_set) return fail(c, VMI_ERR_STATE, "vmi_set_params not called");
  if (npairs > 0x7fffffff) return fail(c, VMI_ERR_UNSUPPORTED, "more than 2^31-1 pairs");
  for (int64_t i = 0; i < npairs; ++i) {
    if (na[i] <= 0 || nb[i] <= 0 || !a[i] || !b[i])
      return fail(c, VMI_ERR_ARG, "cannot voxelize an empty cloud");
    if (na[i] > 0x7fffffff || nb[i] > 0x7fffffff)
      return fail(c, VMI_ERR_UNSUPPORTED, "more than 2^31-1 points");
  }
  cudaSetDevice(c->device);
  c->n_set = 0;
  static const bool trace = std::getenv("VMI_TRACE") != nullptr;  // phase timings to stderr
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto x, auto y) { return std::chrono::duration<double, std::milli>(y - x).count(); };
  const auto t_begin = now();
  const size_t rb = is_rec ? 16 : 24;  // host bytes per point
  // ---- distinct scans (by buffer), their pool offsets
  std::unordered_map<const void*, int64_t> id;
  std::vector<const void*> scan;
  std::vector<int64_t> scan_n;
  std::vector<int64_t> ia((size_t)npairs), ib((size_t)npairs);
  auto intern = [&](const void* p, int64_t n) -> int64_t {
    auto it = id.find(p);
    if (it != id.end()) return scan_n[(size_t)it->second] == n ? it->second : -1;
    id.emplace(p, (int64_t)scan.size());
    scan.push_back(p);
    scan_n.push_back(n);
    return (int64_t)scan.size() - 1;
  };
  for (int64_t i = 0; i < npairs; ++i) {
    ia[(size_t)i] = intern(a[i], na[i]);
    ib[(size_t)i] = intern(b[i], nb[i]);
    if (ia[(size_t)i] < 0 || ib[(size_t)i] < 0)
      return fail(c, VMI_ERR_ARG, "one buffer passed with two point counts");
  }
  const int64_t ns = (int64_t)scan.size();
  std::vector<size_t> off((size_t)ns + 1, 0);
  for (int64_t k = 0; k < ns; ++k) off[(size_t)k + 1] = off[(size_t)k] + (size_t)scan_n[(size_t)k] * rb;
  CK(c, grow(&c->d_raw, c->cap_raw, off[(size_t)ns] > 0 ? off[(size_t)ns] : 16));
  char* raw = static_cast<char*>(c->d_raw);
  // everything starts after the work already queued on the context stream (an
  // earlier evaluation may still read the buffers being rebuilt)
  if (!c->set_start) CK(c, cudaEventCreateWithFlags(&c->set_start, cudaEventDisableTiming));
  CK(c, cudaEventRecord(c->set_start, c->stream));
  if (!c->copy_stream) CK(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
  CK(c, cudaStreamWaitEvent(c->copy_stream, c->set_start, 0));
  // ---- raw uploads in chunks of kChunk scans, one event each; issued before
  // the host pass (they need only the sizes), which then runs beside them
  // (C5: 29 ms of validation/bounds under the 38 ms upload)
  constexpr int64_t kChunk = 32;
  const int64_t nchunk = (ns + kChunk - 1) / kChunk;
  while ((int64_t)c->chunk_ev.size() < nchunk) {
    cudaEvent_t e;
    CK(c, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->chunk_ev.push_back(e);
  }
  for (int64_t ch = 0; ch < nchunk; ++ch) {
    for (int64_t k = ch * kChunk; k < std::min(ns, (ch + 1) * kChunk); ++k)
      CK(c, cudaMemcpyAsync(raw + off[(size_t)k], scan[(size_t)k], off[(size_t)k + 1] - off[(size_t)k],
                            cudaMemcpyHostToDevice, c->copy_stream));
    CK(c, cudaEventRecord(c->chunk_ev[(size_t)ch], c->copy_stream));
  }
  // ---- host passes, threaded over distinct scans
  std::vector<HostScan> hs((size_t)ns);
  {
    int nt = (int)std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()), 16);
    nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, ns));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
      pool.emplace_back([&, t] {
        for (int64_t k = t; k < ns; k += nt) scan_pass(scan[(size_t)k], is_rec, scan_n[(size_t)k], hs[(size_t)k]);
      });
    for (auto& th : pool) th.join();
  }
  int64_t max_na = 1;
  for (int64_t k = 0; k < ns; ++k)
    if (!hs[(size_t)k].finite) {
      cudaStreamSynchronize(c->copy_stream);  // (the uploads read the caller's buffers)
      return fail(c, VMI_ERR_ARG, "points contain non-finite coordinates");
    }
  for (int64_t i = 0; i < npairs; ++i) max_na = std::max(max_na, na[i]);
  const auto t_host = now();
  if ((int64_t)c->set.size() < npairs) c->set.resize((size_t)npairs);
  const size_t np1 = (size_t)(npairs > 0 ? npairs : 1);
  CK(c, grow(&c->d_setv, c->cap_setv, 8 * np1));
  int* d_v = c->d_setv;  // per-pair voxel counts, then "left the box" flags
  int* d_bad = d_v + np1;
  for (auto& l : c->lanes) {
    if (!l.st) {
      CK(c, cudaStreamCreateWithFlags(&l.st, cudaStreamNonBlocking));
      CK(c, cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming));
      CK(c, cudaMalloc(&l.d_cursor, 4 * kMaxW));
    }
    CK(c, exact_alloc(l.ex, max_na));
    CK(c, grow(&l.d_avox_tmp, l.cap_avox_tmp, sizeof(int4) * (size_t)max_na));
    CK(c, cudaStreamWaitEvent(l.st, c->set_start, 0));
  }
  // ---- grouped builds: up to kGroup pairs per launch sequence (the common
  // case); pairs whose voxel box needs more than 27 bits use the lanes below
  std::vector<char> grouped((size_t)npairs, 0);
  if (!std::getenv("VMI_NO_GROUP")) {  // (VMI_NO_GROUP=1: lanes only, A/B and tests)
    constexpr int kGroup = 32;
    auto nbits_of = [&](int64_t i, uint32_t ext[3], int amin[3]) -> int {
      const HostScan& h = hs[(size_t)ia[(size_t)i]];
      double vol = 1.0;
      for (int j = 0; j < 3; ++j) {
        const int64_t lo = host_floor(h.lo[j], c->g.origin[j], c->g.res);
        const int64_t hi = host_floor(h.hi[j], c->g.origin[j], c->g.res);
        if (lo < -(1 << 20) || hi > (1 << 20) - 1) return -1;  // -> lanes path (reports the error)
        amin[j] = (int)lo;
        ext[j] = (uint32_t)(hi - lo + 1);
        vol *= (double)ext[j];
      }
      int nb = 1;
      while (nb < 40 && (double)(1ull << nb) < vol) ++nb;
      return nb;
    };
    std::vector<GroupPair> gph;
    cudaStream_t st = c->lanes[0].st;
    for (int64_t g0 = 0; g0 < npairs;) {
      // the next run of pairs that fit one 32-bit key space together
      int nbits = 0;
      int64_t g1 = g0;
      std::vector<std::array<int, 3>> amins;
      std::vector<std::array<uint32_t, 3>> exts;
      while (g1 < npairs && g1 - g0 < kGroup) {
        uint32_t e[3];
        int am[3];
        const int nb = nbits_of(g1, e, am);
        if (nb < 0 || nb > 27) break;
        const int nbn = std::max(nbits, nb);
        int gb = 0;
        while ((1 << gb) < (int)(g1 - g0 + 1)) ++gb;
        if (nbn + gb > 32) break;
        nbits = nbn;
        amins.push_back({am[0], am[1], am[2]});
        exts.push_back({e[0], e[1], e[2]});
        ++g1;
      }
      if (g1 == g0) { ++g0; continue; }  // this pair goes the lane path
      const int G = (int)(g1 - g0);
      gph.assign((size_t)G, GroupPair{});
      int64_t n_total = 0, max_na_g = 1, max_rows = 1;
      size_t max_grid = 1;
      for (int k = 0; k < G; ++k) {
        const int64_t i = g0 + k;
        PairStore& ps = c->set[(size_t)i];
        free_a(ps);
        ps.b_set = false;
        ps.regrouped = false;
        ps.hull_n = 0;
        for (int j = 0; j < 3; ++j) {
          ps.amin[j] = amins[(size_t)k][j];
          ps.ext[j] = exts[(size_t)k][j];
          ps.amax[j] = ps.amin[j] + (int)ps.ext[j] - 1;
        }
        ps.a_empty = false;
        ps.grid_bytes = (size_t)ps.ext[0] * ps.ext[1] * ps.ext[2];
        CK(c, grow(&ps.d_grid, ps.cap_grid, ps.grid_bytes));
        CK(c, grow(&ps.d_avox, ps.cap_avox, sizeof(int4) * (size_t)na[i]));
        if (!ps.d_bin_total) CK(c, cudaMalloc(&ps.d_bin_total, 4 * kMaxW));
        const HostScan& h_b = hs[(size_t)ib[(size_t)i]];
        const int as_f32 = (h_b.exact32 && !std::getenv("VMI_FORCE_F64")) ? 1 : 0;
        double mx = 0.0;
        for (int j = 0; j < 3; ++j) {
          mx = std::fmax(mx, std::fmax(std::fabs(h_b.lo[j]), std::fabs(h_b.hi[j])));
          ps.b_lo[j] = h_b.lo[j];
          ps.b_hi[j] = h_b.hi[j];
        }
        ps.max_abs = mx;
        ps.span = (int)((nb[i] + c->threads - 1) / c->threads);
        ps.rem = (int)(nb[i] - (int64_t)(ps.span - 1) * c->threads);
        CK(c, grow(&ps.d_pts, ps.cap_pts,
                   (size_t)(ps.span + kStagePadRows) * c->threads * (as_f32 ? 16 : 32)));
        ps.is_f32 = as_f32;
        ps.nb = nb[i];
        ps.a_npts = na[i];
        GroupPair& q = gph[(size_t)k];
        q.raw_a = raw + off[(size_t)ia[(size_t)i]];
        q.raw_b = raw + off[(size_t)ib[(size_t)i]];
        q.n = na[i];
        q.off = n_total;
        q.nb = nb[i];
        q.amin = make_int3(ps.amin[0], ps.amin[1], ps.amin[2]);
        q.ext = make_uint3(ps.ext[0], ps.ext[1], ps.ext[2]);
        q.grid = ps.d_grid;
        q.grid_bytes = ps.grid_bytes;
        q.avox = ps.d_avox;
        q.bin_total = ps.d_bin_total;
        q.pts = ps.d_pts;
        q.span = ps.span;
        q.rem = ps.rem;
        q.b_split = as_f32;
        n_total += na[i];
        max_na_g = std::max(max_na_g, na[i]);
        max_rows = std::max<int64_t>(max_rows, (int64_t)ps.span * c->threads);
        max_grid = std::max(max_grid, ps.grid_bytes);
        grouped[(size_t)i] = 1;
      }
      // raw uploads this group reads
      int64_t need = 0;
      for (int64_t i = g0; i < g1; ++i) need = std::max(need, std::max(ia[(size_t)i], ib[(size_t)i]));
      CK(c, cudaStreamWaitEvent(st, c->chunk_ev[(size_t)(need / kChunk)], 0));
      CK(c, grow(&c->d_group, c->cap_group, sizeof(GroupPair) * kGroup));
      CK(c, grow(&c->d_gavox, c->cap_gavox, sizeof(int4) * (size_t)n_total));
      CK(c, grow(&c->d_gcursor, c->cap_gcursor, 4 * (size_t)kGroup * kMaxW));
      CK(c, cudaMemcpyAsync(c->d_group, gph.data(), sizeof(GroupPair) * (size_t)G,
                            cudaMemcpyHostToDevice, st));
      CK(c, cudaMemsetAsync(d_bad + g0, 0, 4 * (size_t)G, st));
      CK(c, build_pair_group(c->lanes[0].ex, static_cast<const GroupPair*>(c->d_group), G, n_total,
                             (int)max_na_g, (int)max_rows, max_grid, nbits, c->g, is_rec,
                             c->threads, static_cast<int4*>(c->d_gavox),
                             static_cast<int*>(c->d_gcursor), d_v + g0, d_bad + g0, st,
                             &c->launches));
      g0 = g1;
    }
  }
  // one host thread per lane enqueues its (remaining) pairs (launch-bound otherwise)
  static const bool force_f64 = std::getenv("VMI_FORCE_F64") != nullptr;
  std::vector<int> lane_rc(kBuildLanes, 0);
  std::vector<int64_t> lane_launches(kBuildLanes, 0);
  std::vector<std::string> lane_err(kBuildLanes);
  auto lane_work = [&](int li) -> int {
    BuildLane& ln = c->lanes[li];
    cudaStream_t st = ln.st;
    cudaSetDevice(c->device);
    int64_t waited = -1;  // the last raw-upload chunk this lane waited for
    auto lfail = [&](int code, const std::string& m) { lane_err[(size_t)li] = m; return code; };
#define LCK(x)                                                                       \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) return lfail(VMI_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)
    for (int64_t i = li; i < npairs; i += kBuildLanes) {
      if (grouped[(size_t)i]) continue;
      PairStore& ps = c->set[(size_t)i];
      const int64_t need = std::max(ia[(size_t)i], ib[(size_t)i]) / kChunk;
      if (need > waited) {  // chunks upload in order: the latest one suffices
        LCK(cudaStreamWaitEvent(st, c->chunk_ev[(size_t)need], 0));
        waited = need;
      }
      free_a(ps);
      ps.b_set = false;
      ps.regrouped = false;  // (a drive's scans are ring-ordered)
      ps.hull_n = 0;
      const HostScan& h_a = hs[(size_t)ia[(size_t)i]];
      const HostScan& h_b = hs[(size_t)ib[(size_t)i]];
      // ---- scan A: bounds on the host, voxelize + features + grid on the GPU
      for (int j = 0; j < 3; ++j) {
        const int64_t lo = host_floor(h_a.lo[j], c->g.origin[j], c->g.res);
        const int64_t hi = host_floor(h_a.hi[j], c->g.origin[j], c->g.res);
        if (lo < -(1 << 20) || hi > (1 << 20) - 1)
          return lfail(VMI_ERR_RANGE, "a point of scan A maps outside the voxel key range");
        ps.amin[j] = (int)lo;
        ps.amax[j] = (int)hi;
        ps.ext[j] = (uint32_t)(hi - lo + 1);
      }
      ps.a_empty = false;
      const double vol = (double)ps.ext[0] * ps.ext[1] * ps.ext[2];
      if (vol > 4294967294.0)
        return lfail(VMI_ERR_UNSUPPORTED,
                     "scan A's occupied AABB exceeds 2^32-2 voxels: pair sets need the dense "
                     "reference grid (the single-pair API takes a sparse reference)");
      ps.grid_bytes = (size_t)vol;
      LCK(grow(&ps.d_grid, ps.cap_grid, ps.grid_bytes));
      LCK(grow(&ps.d_avox, ps.cap_avox, sizeof(int4) * (size_t)na[i]));
      if (!ps.d_bin_total) LCK(cudaMalloc(&ps.d_bin_total, 4 * kMaxW));
      LCK(cudaMemsetAsync(ps.d_grid, 0, ps.grid_bytes, st));
      LCK(cudaMemsetAsync(ps.d_bin_total, 0, 4 * kMaxW, st));
      PointSource src{};
      const char* ra = raw + off[(size_t)ia[(size_t)i]];
      if (is_rec) src.rec = reinterpret_cast<const float4*>(ra);
      else src.xyz = reinterpret_cast<const double*>(ra);
      src.n = na[i];
      LCK(box_voxelize(ln.ex, src, c->g, ps.amin, ps.ext, st, &lane_launches[(size_t)li]));
      LCK(build_reference_box(ln.ex, (int)na[i], c->g, ps.ext, ps.d_grid, ln.d_avox_tmp,
                              ps.d_avox, ps.d_bin_total, ln.d_cursor, st,
                              &lane_launches[(size_t)li]));
      LCK(cudaMemcpyAsync(d_v + i, ln.ex.nruns, 4, cudaMemcpyDeviceToDevice, st));
      LCK(cudaMemcpyAsync(d_bad + i, ln.ex.bounds + 6, 4, cudaMemcpyDeviceToDevice, st));
      ps.a_npts = na[i];
      // ---- scan B: span layout
      const int as_f32 = (h_b.exact32 && !force_f64) ? 1 : 0;
      double mx = 0.0;
      for (int j = 0; j < 3; ++j) {
        mx = std::fmax(mx, std::fmax(std::fabs(h_b.lo[j]), std::fabs(h_b.hi[j])));
        ps.b_lo[j] = h_b.lo[j];
        ps.b_hi[j] = h_b.hi[j];
      }
      ps.max_abs = mx;
      ps.span = (int)((nb[i] + c->threads - 1) / c->threads);
      ps.rem = (int)(nb[i] - (int64_t)(ps.span - 1) * c->threads);
      LCK(grow(&ps.d_pts, ps.cap_pts,
               (size_t)(ps.span + kStagePadRows) * c->threads * (as_f32 ? 16 : 32)));
      LCK(launch_span_layout(raw + off[(size_t)ib[(size_t)i]], is_rec, as_f32, nb[i], ps.span,
                             ps.rem, c->threads, ps.d_pts, st));
      lane_launches[(size_t)li] += 1;
      ps.is_f32 = as_f32;
      ps.nb = nb[i];
    }
#undef LCK
    return 0;
  };
  {
    std::vector<std::thread> th;
    for (int li = 0; li < kBuildLanes; ++li)
      th.emplace_back([&, li] { lane_rc[(size_t)li] = lane_work(li); });
    for (auto& t : th) t.join();
  }
  for (int li = 0; li < kBuildLanes; ++li) {
    c->launches += lane_launches[(size_t)li];
    if (lane_rc[(size_t)li]) {
      cudaDeviceSynchronize();
      return fail(c, lane_rc[(size_t)li], lane_err[(size_t)li]);
    }
  }
  const auto t_enq = now();
  for (auto& l : c->lanes) {  // the context stream continues after every lane
    CK(c, cudaEventRecord(l.done, l.st));
    CK(c, cudaStreamWaitEvent(c->stream, l.done, 0));
  }
  std::vector<int> V(2 * np1);
  CK(c, cudaMemcpyAsync(V.data(), d_v, 8 * np1, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  if (trace)
    std::fprintf(stderr, "vmi_set_pairs %lld pairs (%lld scans): host pass %.1f ms, enqueue %.1f ms, drain %.1f ms\n",
                 (long long)npairs, (long long)ns, ms(t_begin, t_host), ms(t_host, t_enq), ms(t_enq, now()));
  for (int64_t i = 0; i < npairs; ++i)
    if (V[np1 + (size_t)i])  // the host box and the GPU's voxel coordinates disagree
      return fail(c, VMI_ERR_CUDA, "internal: scan A left its host-computed voxel box");
  std::vector<PairDesc> desc((size_t)npairs);
  for (int64_t i = 0; i < npairs; ++i) {
    PairStore& ps = c->set[(size_t)i];
    ps.a_nvox = V[(size_t)i];
    ps.n_avox = V[(size_t)i];  // every voxel of A has a feature bin >= 1 (build_reference)
    ps.a_set = true;
    ps.b_voxels = (int64_t)((double)ps.a_nvox * (double)ps.nb / (double)ps.a_npts) + 1;
    ps.b_set = true;
    desc[(size_t)i].A = ref_view(ps);
    desc[(size_t)i].B = query_view(c, ps);
  }
  CK(c, grow(&c->d_pairs, c->cap_pairs, sizeof(PairDesc) * np1));
  if (npairs > 0)
    CK(c, cudaMemcpyAsync(c->d_pairs, desc.data(), sizeof(PairDesc) * (size_t)npairs,
                          cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaStreamSynchronize(c->stream));
  c->n_set = npairs;
  return 0;
}

namespace {

// Pose matrices + pair indices already on the device (c->d_mats, c->d_pose_pair):
// one multi-pair launch (single-pass table sized for the set's largest scan B;
// per-pair launches when some pair needs the multi-pass layout), then the
// exact path for flagged poses.
int eval_pairs_device(vmi_ctx* c, int64_t P, const int32_t* pair_host, long long* hist,
                      const PairBufs* bufs = nullptr) {
  if (P <= 0) return 0;
  const PairBufs def{c->d_mats, c->d_pose_pair, c->d_mi, c->d_status, c->d_hash, c->d_total};
  const PairBufs& bf = bufs ? *bufs : def;
  int64_t bvox = 0;
  int any_f64 = 0;
  for (int64_t i = 0; i < c->n_set; ++i) {
    bvox = std::max(bvox, c->set[(size_t)i].b_voxels);
    any_f64 |= !c->set[(size_t)i].is_f32;
  }
  FastLaunch fl{};
  fl.g = c->g;
  fl.g.kind = kernel_kind(c);
  fl.mats = bf.mats;
  fl.P = P;
  fl.grid = (int)(P < c->sm_count ? P : c->sm_count);
  fl.sched = next_sched(c);
  fl.streams = c->streams;
  plan_table(c, fl.g.kind, bvox, any_f64 ? 0 : 1, &fl.cap, &fl.npass, &fl.multi);
  fl.mi = bf.mi;
  fl.status = bf.status;
  fl.hist = hist;
  fl.total = bf.total;
  fl.hash = bf.hash;
  bool mixed = false;  // the kernel's record format is per launch
  for (int64_t i = 1; i < c->n_set; ++i) mixed |= c->set[(size_t)i].is_f32 != c->set[0].is_f32;
  if (!fl.multi && !mixed) {
    int rc = ensure_sums(c, fl.g.kind, fl.grid, fl.cap);
    if (rc) return rc;
    fl.sums = c->d_sums;
    fl.pairs = c->d_pairs;
    fl.pose_pair = bf.pose_pair;
    fl.A = ref_view(c->set[0]);  // (unused by the multi-pair kernel)
    fl.B = query_view(c, c->set[0]);
    CK(c, launch_fast(fl, c->stream));
    c->launches += 1;
  } else {
    // one launch per pair over its (contiguous or not) poses: gather index lists
    // on the host, run the single-pair kernel on a compacted copy of the matrices
    return fail(c, VMI_ERR_UNSUPPORTED,
                "pair set needs the multi-pass table or mixes record formats (use one pair at a time)");
  }
  return 0;
}

// after eval_pairs_device: re-run flagged poses exactly (identities kept in step)
int fix_pairs(vmi_ctx* c, int64_t P, const int32_t* pair_host, long long* hist,
              const int32_t* status_host, int64_t* n_fixed) {
  return do_fixups(c, c->d_mats, P, c->d_mi, c->d_status, hist, c->d_total, c->stream, n_fixed,
                   pair_host, status_host, c->d_hash);
}

int ensure_pp(vmi_ctx* c, int64_t P) {
  if (P <= c->cap_pp) return 0;
  cudaFree(c->d_pose_pair);
  cudaFree(c->d_hash);
  c->d_pose_pair = nullptr;
  c->d_hash = nullptr;
  c->cap_pp = 0;
  CK(c, cudaMalloc(&c->d_pose_pair, 4 * (size_t)P));
  CK(c, cudaMalloc(&c->d_hash, 8 * (size_t)P));
  c->cap_pp = P;
  return 0;
}

// host poses + pair indices -> device matrices + indices (pinned staging)
int upload_pair_poses(vmi_ctx* c, const double* poses, const int32_t* pair, int64_t P, bool hist) {
  for (int64_t p = 0; p < P; ++p)
    if (pair[p] < 0 || pair[p] >= c->n_set) return fail(c, VMI_ERR_ARG, "pair index out of range");
  int rc;
  if ((rc = ensure_P(c, P, hist)) || (rc = ensure_pp(c, P)) || (rc = ensure_pinned(c, P))) return rc;
  if (vmi_poses_to_mats(poses, P, c->h_mats, 0)) return fail(c, VMI_ERR_ARG, "poses contain non-finite components");
  CK(c, cudaMemcpyAsync(c->d_mats, c->h_mats, (size_t)P * 96, cudaMemcpyHostToDevice, c->stream));
  CK(c, cudaMemcpyAsync(c->d_pose_pair, pair, (size_t)P * 4, cudaMemcpyHostToDevice, c->stream));
  return 0;
}

}  // namespace

int vmi_eval_pairs(vmi_ctx* c, const double* poses, const int32_t* pair, int64_t P, double* mi_out,
                   int32_t* status_out, uint64_t* hash_out, int64_t* hist_out) {
  if (!c) return VMI_ERR_ARG;
  if (!c->params_set) return fail(c, VMI_ERR_STATE, "vmi_set_params not called");
  if (P < 0 || (P > 0 && (!poses || !pair || !mi_out || !status_out)))
    return fail(c, VMI_ERR_ARG, "bad arguments");
  if (P == 0) return 0;
  cudaSetDevice(c->device);
  int rc = upload_pair_poses(c, poses, pair, P, hist_out != nullptr);
  if (rc) return rc;
  long long* dh = hist_out ? c->d_hist : nullptr;
  if ((rc = eval_pairs_device(c, P, pair, dh))) return rc;
  if ((rc = fix_pairs(c, P, pair, dh, nullptr, nullptr))) return rc;
  CK(c, cudaMemcpyAsync(mi_out, c->d_mi, P * 8, cudaMemcpyDeviceToHost, c->stream));
  CK(c, cudaMemcpyAsync(status_out, c->d_status, P * 4, cudaMemcpyDeviceToHost, c->stream));
  if (hash_out) CK(c, cudaMemcpyAsync(hash_out, c->d_hash, P * 8, cudaMemcpyDeviceToHost, c->stream));
  if (hist_out) {
    const int W = c->g.bins + 1;
    CK(c, cudaMemcpyAsync(hist_out, dh, (size_t)P * W * W * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  CK(c, cudaStreamSynchronize(c->stream));
  return 0;
}

int vmi_align_pairs(vmi_ctx* c, int64_t K, const double* x0, const double steps[6],
                    int max_iterations, double f_tol, double x_tol, int restarts, double* best_x,
                    double* best_value, int32_t* iterations, int32_t* termination,
                    int32_t* n_evaluations, int32_t* uncertain, double* trace, int32_t* trace_len,
                    int64_t trace_cap) {
  if (!c) return VMI_ERR_ARG;
  if (K != c->n_set) return fail(c, VMI_ERR_ARG, "one start pose per pair of the set");
  if (K > 0 && (!x0 || !steps || !best_x || !best_value)) return fail(c, VMI_ERR_ARG, "bad arguments");
  if (max_iterations < 1 || !(f_tol > 0) || !(x_tol > 0) || restarts < 0)
    return fail(c, VMI_ERR_ARG, "bad simplex configuration");
  NmConfig cfg{};
  for (int j = 0; j < 6; ++j) {
    if (!(steps[j] > 0)) return fail(c, VMI_ERR_ARG, "initial steps must all be > 0");
    cfg.steps[j] = steps[j];
  }
  cfg.max_iterations = max_iterations;
  cfg.f_tol = f_tol;
  cfg.x_tol = x_tol;
  cfg.restarts = restarts;
  // below ~two poses per SM a launch costs the same for 1 or 4 probes per run
  // (VMI_SPEC: poses per SM.  A/B at C5: 2 -> 432 lockstep steps, 3,790 /s;
  // 8 -> 419, 3,855; 64 -> 303 steps but 2x the probes, 2,947 /s -- the step
  // count is set by the slowest pairs, each step's latency by one pose per SM)
  static const double spec = [] {
    const char* e = std::getenv("VMI_SPEC");
    return e ? std::atof(e) : 2.0;
  }();
  cfg.spec_budget = (int64_t)(spec * c->sm_count);
  cudaSetDevice(c->device);
  // Two lanes of runs alternate on the context stream: lane l's batch
  // (matrices built on the host into pinned memory, upload, one multi-pair
  // launch, read-back of values / statuses / identities) is queued while the
  // host applies the other lane's results, so the GPU rarely waits for the
  // host.  Flagged poses (table overflow, VARZ bin edges) are re-run exactly
  // and read again before the lane's results are used.
  NmAsyncEvaluator ev;
  ev.lanes = 2;
  ev.submit = [&](int l, const double* poses, const int32_t* run, int64_t n) -> int {
    NmSlot& sl = c->nm_slot[l];
    if (n > sl.cap) {
      cudaFree(sl.d_buf);
      if (sl.h_buf) cudaFreeHost(sl.h_buf);
      sl.d_buf = nullptr;
      sl.h_buf = nullptr;
      sl.cap = 0;
      CK(c, cudaMalloc(&sl.d_buf, (size_t)n * 128));
      CK(c, cudaMallocHost(&sl.h_buf, (size_t)n * 116));
      if (!sl.ev) CK(c, cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
      sl.cap = n;
    }
    char* d = static_cast<char*>(sl.d_buf);
    char* hb = static_cast<char*>(sl.h_buf);
    const size_t cp = (size_t)sl.cap;
    PairBufs bf{reinterpret_cast<double*>(d), reinterpret_cast<int32_t*>(d + cp * 124),
                reinterpret_cast<double*>(d + cp * 96),
                reinterpret_cast<int32_t*>(d + cp * 120),
                reinterpret_cast<unsigned long long*>(d + cp * 104),
                reinterpret_cast<long long*>(d + cp * 112)};
    double* h_mats = reinterpret_cast<double*>(hb);
    for (int64_t p = 0; p < n; ++p)
      if (run[p] < 0 || run[p] >= c->n_set) return fail(c, VMI_ERR_ARG, "pair index out of range");
    if (vmi_poses_to_mats(poses, n, h_mats, 1)) return fail(c, VMI_ERR_ARG, "poses contain non-finite components");
    CK(c, cudaMemcpyAsync(const_cast<double*>(bf.mats), h_mats, (size_t)n * 96,
                          cudaMemcpyHostToDevice, c->stream));
    CK(c, cudaMemcpyAsync(const_cast<int32_t*>(bf.pose_pair), run, (size_t)n * 4,
                          cudaMemcpyHostToDevice, c->stream));
    int rc = eval_pairs_device(c, n, run, nullptr, &bf);
    if (rc) return rc;
    CK(c, cudaMemcpyAsync(hb + cp * 96, bf.mi, (size_t)n * 8, cudaMemcpyDeviceToHost, c->stream));
    CK(c, cudaMemcpyAsync(hb + cp * 104, bf.hash, (size_t)n * 8, cudaMemcpyDeviceToHost,
                          c->stream));
    CK(c, cudaMemcpyAsync(hb + cp * 112, bf.status, (size_t)n * 4, cudaMemcpyDeviceToHost,
                          c->stream));
    CK(c, cudaEventRecord(sl.ev, c->stream));
    sl.n = n;
    sl.run = run;
    sl.bufs = bf;
    return 0;
  };
  ev.wait = [&](int l, double* g, uint64_t* h) -> int {
    NmSlot& sl = c->nm_slot[l];
    CK(c, cudaEventSynchronize(sl.ev));
    char* hb = static_cast<char*>(sl.h_buf);
    const size_t cp = (size_t)sl.cap;
    const double* mi = reinterpret_cast<const double*>(hb + cp * 96);
    const uint64_t* hh = reinterpret_cast<const uint64_t*>(hb + cp * 104);
    const int32_t* st = reinterpret_cast<const int32_t*>(hb + cp * 112);
    int64_t nf = 0;
    for (int64_t i = 0; i < sl.n; ++i) nf += (st[i] & VMI_FLAG_RECHECK) != 0;
    if (nf) {  // rare: exact path on the same stream, then read this lane again
      int rc = do_fixups(c, sl.bufs.mats, sl.n, sl.bufs.mi, sl.bufs.status, nullptr, nullptr,
                         c->stream, nullptr, sl.run, st, sl.bufs.hash);
      if (rc) return rc;
      CK(c, cudaMemcpyAsync(hb + cp * 96, sl.bufs.mi, (size_t)sl.n * 8, cudaMemcpyDeviceToHost,
                            c->stream));
      CK(c, cudaMemcpyAsync(hb + cp * 104, sl.bufs.hash, (size_t)sl.n * 8,
                            cudaMemcpyDeviceToHost, c->stream));
      CK(c, cudaStreamSynchronize(c->stream));
    }
    for (int64_t i = 0; i < sl.n; ++i) {
      g[i] = -mi[i];  // sentinel -> +1e300
      h[i] = hh[i];
    }
    return 0;
  };
  std::vector<NmResult> res((size_t)K);
  int rc = nm_lockstep_async(K, x0, cfg, ev, res.data(), &c->nm_steps, &c->nm_probes);
  if (rc) return rc;
  return nm_write_results(res.data(), K, best_x, best_value, iterations, termination,
                          n_evaluations, uncertain, trace, trace_len, trace_cap);
}

int vmi_argmax_device(vmi_ctx* c, const double* mi_dev, int64_t P, double* best_mi,
                      int64_t* best_idx, void* stream) {
  if (!c || !mi_dev || P <= 0 || !best_mi || !best_idx) return VMI_ERR_ARG;
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  CK(c, launch_argmax(mi_dev, P, c->d_best, c->d_best_idx, st));
  c->launches += 1;
  CK(c, cudaMemcpyAsync(best_mi, c->d_best, 8, cudaMemcpyDeviceToHost, st));
  CK(c, cudaMemcpyAsync(best_idx, c->d_best_idx, 8, cudaMemcpyDeviceToHost, st));
  CK(c, cudaStreamSynchronize(st));
  return 0;
}

int vmi_topk_device(vmi_ctx* c, const double* mi_dev, int64_t P, int64_t K, double* top_mi,
                    int64_t* top_idx, void* stream) {
  if (!c || !mi_dev || P <= 0 || K <= 0 || !top_mi || !top_idx) return VMI_ERR_ARG;
  if (P > 0x7fffffff) return fail(c, VMI_ERR_UNSUPPORTED, "top-K over more than 2^31-1 values");
  cudaSetDevice(c->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : c->stream;
  const int n = (int)P;
  size_t bytes = 0;
  CK(c, topk_sort(mi_dev, n, nullptr, nullptr, nullptr, nullptr, &bytes, st));
  CK(c, grow(&c->d_tk_keys, c->cap_tk_keys, 8 * (size_t)n));
  CK(c, grow(&c->d_tk_idx, c->cap_tk_idx, 4 * (size_t)n));
  CK(c, grow(&c->d_tk_out, c->cap_tk_out, 4 * (size_t)n));
  CK(c, grow(&c->d_tk_tmp, c->cap_tk_tmp, bytes));
  CK(c, topk_sort(mi_dev, n, c->d_tk_keys, c->d_tk_idx, c->d_tk_out, c->d_tk_tmp, &bytes, st));
  c->launches += 2;
  const int64_t k = K < P ? K : P;
  std::vector<int> idx((size_t)k);
  CK(c, cudaMemcpyAsync(top_mi, c->d_tk_keys, 8 * (size_t)k, cudaMemcpyDeviceToHost, st));
  CK(c, cudaMemcpyAsync(idx.data(), c->d_tk_out, 4 * (size_t)k, cudaMemcpyDeviceToHost, st));
  CK(c, cudaStreamSynchronize(st));
  for (int64_t i = 0; i < k; ++i) top_idx[i] = idx[(size_t)i];
  return 0;
}

}  // extern "C"
