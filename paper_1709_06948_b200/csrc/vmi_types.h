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

struct GridParams {
  double origin[3];
  double res;
  double inv_res;
  int mode;
  int kind;  // 0 varz, 1 count
  int bins;
  int include_phi;
  double clamp;
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
};

// Scan B in the fast path's "span layout": thread t of a CTA with T threads
// owns original points [t*span, (t+1)*span); element r of that span is stored
// at r*T + t so every warp load is 32 consecutive records.
struct QueryView {
  const void* pts;  // float4 (x, y, z, i) or double4 (x, y, z, pad)
  int is_f32;
  int64_t n;
  int64_t span;
  int threads;
};

}  // namespace vmi
