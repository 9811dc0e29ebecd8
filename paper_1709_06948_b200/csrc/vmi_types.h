// vmi_types.h -- plain structs shared by host code and kernels.
#pragma once
#include <cstdint>

namespace vmi {

constexpr int kMaxW = 65;  // histogram width limit: bin_count <= 64

// How voxel_indices' `(p - origin) / resolution` is evaluated (voxel.py:199).
enum GridMode : int {
  kGridUnit = 0,     // origin == 0 and resolution == 1: q = p exactly
  kGridPow2 = 1,     // resolution a power of two: q = (p - o) * (1/res), exact
  kGridGeneral = 2,  // IEEE division
};

// Fast-kernel feature kinds.  kKindOcc is internal: chosen by the host when
// every occupied voxel provably lands in one feature bin (see vmi_set_params),
// so the histogram needs only which voxels are occupied, not their features.
constexpr int kKindVarz = 0, kKindCount = 1, kKindOcc = 2;

struct GridParams {
  double origin[3];
  double res;
  double inv_res;
  int mode;
  int kind;  // 0 varz, 1 count (exact path / user); fast kernel: + 2 occupancy
  int bins;
  int include_phi;
  double clamp;
  int occ_bin;  // kKindOcc: the one B-side bin every occupied voxel takes
};

// Scan A as the kernels see it: a dense u8 bin grid over A's occupied AABB
// (0 = no feature), and the occupied voxels sorted by bin for the per-pose
// A marginal over the overlap region.
struct RefView {
  int amin[3];
  int amax[3];
  uint32_t ext[3];            // amax - amin + 1
  const uint8_t* grid;        // ext[0]*ext[1]*ext[2], x-major
  const int4* avox;           // (rx, ry, rz, bin), sorted by bin
  int n_avox;
  int empty;                  // FeatureMap with no voxels / empty bounds
  const uint32_t* bin_total;  // per-bin count of all A voxels (full-cover shortcut)
  // Summed-volume tables of A's voxels, one per bin present in A (or none):
  // sat[k][x][y][z] = # voxels with bin sat_bin[k] in [0,x)x[0,y)x[0,z) of the
  // box, (ext+1)-strided -- a region's marginal is 8 lookups per bin.
  const uint32_t* sat;
  const int* sat_bin;
  int sat_nb;
  // Sparse reference: when A's AABB exceeds the dense grid's 32-bit index
  // (> 2^32-2 voxels, e.g. a map-scale scan A at fine resolution) `grid` is
  // null and A is an open-addressing table of its packed voxel keys
  // (voxel.py:65-73's int64 packing; empty slot = ~0) with a parallel bin
  // array -- the reference's own sparse representation.  The fast kernel
  // flags such poses; the exact path looks bins up here.
  const unsigned long long* hkeys;
  const uint8_t* hbins;
  uint32_t hmask;
  int sparse;
};

// Scan B in the fast path's "span layout".  The ring-ordered scan is cut into
// T contiguous spans: the first `rem` spans hold `span` points, the others
// `span - 1` (n = T*(span-1) + rem, 0 < rem <= T).  Span s is walked by thread
// t = (s % NW)*32 + s / NW (NW = T/32 warps), so each warp's 32 lanes sample
// the whole scan and every warp gets a similar share of voxel-run records
// (far rings produce many more than near ones).  Element r of thread t's
// span is stored at r*T + t: every warp load is 32 consecutive records.
#ifndef VMI_FAST_THREADS
#define VMI_FAST_THREADS 512
#endif
constexpr int kFastThreads = VMI_FAST_THREADS;  // spans per CTA (span layout "threads")

// Extra rows allocated after the span layout: the fast kernel's staging ring
// streams up to this many rows past the span without bounds checks.
constexpr int kStagePadRows = 16;

struct QueryView {
  const void* pts;  // float4 (x, y, z, i) or double4 (x, y, z, pad)
  int is_f32;
  int64_t n;
  int span;
  int rem;
  int threads;
  double max_abs;  // max |coordinate| of scan B (pose safety bound)
  const double* hull;  // (hull_n, 3): a superset of scan B's convex-hull vertices, or none
  int hull_n;          // > 0: per-pose voxel bounds from the hull instead of every point
  double lo[3];    // scan B's AABB in its own frame (per-pose key box, k_fast.cu)
  double hi[3];
};

// One resident scan pair as the multi-pair kernel sees it (vmi_set_pairs):
// loaded into shared memory at the start of every pose.
struct PairDesc {
  RefView A;
  QueryView B;
};

__host__ __device__ inline int span_of_thread(int t, int threads) {
  return (t & 31) * (threads >> 5) + (t >> 5);
}

__host__ __device__ inline int thread_of_span(int s, int threads) {
  const int nw = threads >> 5;
  return (s % nw) * 32 + s / nw;
}

// Layout slot of original point i (inverse of the ownership rule above).
__host__ __device__ inline int64_t span_slot(int64_t i, int span, int rem, int threads) {
  int64_t s, r;
  const int64_t head = (int64_t)rem * span;
  if (i < head) {
    s = i / span;
    r = i - s * span;
  } else {
    const int64_t j = i - head;
    s = rem + j / (span - 1);
    r = j - (s - rem) * (span - 1);
  }
  return r * threads + thread_of_span((int)s, threads);
}

}  // namespace vmi
