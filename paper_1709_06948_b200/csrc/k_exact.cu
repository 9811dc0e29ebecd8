// k_exact.cu -- exact, reference-order voxelization on the GPU.
//
// This is the bit-exact counterpart of voxelize + compute_feature_map
// (reference pkg/src/voxmi/voxel.py:210-222, :267-295):
//   keys    : pack_keys of floor((p - origin)/res)           (voxel.py:65-73, :199)
//   order   : stable radix sort of the packed keys            (voxel.py:216, kind="stable")
//   CSR     : run-length encode -> unique keys + offsets      (voxel.py:217-219)
//   bounds  : min/max of ijk over ALL points                  (voxel.py:220)
//   VARZ    : reduceat sums in numpy's pairwise order, mean, reduceat of squared
//             deviations, max(ssd, 0)/n                       (voxel.py:285-293)
// It builds scan A's reference grid once per scan pair (_prepare,
// align.py:114-119) and re-evaluates, exactly, the rare poses the fast path
// flags (VMI_FLAG_RECHECK).  Sorting uses CUB (CUDA toolkit library code).
#include <algorithm>
#include <cstdint>
#include <climits>
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "vmi_device.cuh"
#include "vmi_kernels.h"

namespace vmi {

#define VMI_TRY(x)                           \
  do {                                       \
    cudaError_t e_ = (x);                    \
    if (e_ != cudaSuccess) return e_;        \
  } while (0)

__device__ __forceinline__ void point_at(const PointSource& src, int64_t i, double& x, double& y,
                                         double& z) {
  if (src.rec) {  // float32 records widen exactly (the reference's astype(float64))
    const float4 v = src.rec[i];
    x = v.x; y = v.y; z = v.z;
    return;
  }
  if (src.xyz) {
    x = src.xyz[3 * i]; y = src.xyz[3 * i + 1]; z = src.xyz[3 * i + 2];
    return;
  }
  const int64_t li = span_slot(i, src.B.span, src.B.rem, src.B.threads);
  if (src.B.is_f32) {
#if VMI_SPLITREC
    split_decode(reinterpret_cast<const uint4*>(src.B.pts)[li], x, y, z);
#else
    float4 v = reinterpret_cast<const float4*>(src.B.pts)[li];
    x = v.x; y = v.y; z = v.z;
#endif
  } else {
    const double* d = reinterpret_cast<const double*>(src.B.pts) + 4 * li;
    x = d[0]; y = d[1]; z = d[2];
  }
}

__global__ void k_exact_keys(PointSource src, const double* __restrict__ mat, GridParams g,
                             unsigned long long* keys, int* idx, double* zout, int* bounds) {
  __shared__ int sb[7];
  if (threadIdx.x < 3) { sb[threadIdx.x] = INT_MAX; sb[3 + threadIdx.x] = INT_MIN; }
  if (threadIdx.x == 6) sb[6] = 0;
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int ix = INT_MAX, iy = INT_MAX, iz = INT_MAX, ax = INT_MIN, ay = INT_MIN, az = INT_MIN;
  bool bad = false;
  if (i < src.n) {
    double x, y, z;
    point_at(src, i, x, y, z);
    double X = x, Y = y, Z = z;
    if (mat) {
      X = xform_row(x, y, z, mat[0], mat[1], mat[2], mat[9]);
      Y = xform_row(x, y, z, mat[3], mat[4], mat[5], mat[10]);
      Z = xform_row(x, y, z, mat[6], mat[7], mat[8], mat[11]);
    }
    int a, b, c;
    bool ok = voxel_coord(X, g.origin[0], g.res, g.inv_res, g.mode, a);
    ok &= voxel_coord(Y, g.origin[1], g.res, g.inv_res, g.mode, b);
    ok &= voxel_coord(Z, g.origin[2], g.res, g.inv_res, g.mode, c);
    bad = !ok;
    ix = ax = a; iy = ay = b; iz = az = c;
    const unsigned long long off = 1ull << 20;
    keys[i] = (((unsigned long long)(long long)a + off) << 42) |
              (((unsigned long long)(long long)b + off) << 21) |
              ((unsigned long long)(long long)c + off);
    idx[i] = (int)i;
    zout[i] = Z;
  }
  ix = __reduce_min_sync(0xffffffffu, ix); iy = __reduce_min_sync(0xffffffffu, iy);
  iz = __reduce_min_sync(0xffffffffu, iz); ax = __reduce_max_sync(0xffffffffu, ax);
  ay = __reduce_max_sync(0xffffffffu, ay); az = __reduce_max_sync(0xffffffffu, az);
  const bool anybad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&sb[0], ix); atomicMin(&sb[1], iy); atomicMin(&sb[2], iz);
    atomicMax(&sb[3], ax); atomicMax(&sb[4], ay); atomicMax(&sb[5], az);
    if (anybad) sb[6] = 1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicMin(&bounds[0], sb[0]); atomicMin(&bounds[1], sb[1]); atomicMin(&bounds[2], sb[2]);
    atomicMax(&bounds[3], sb[3]); atomicMax(&bounds[4], sb[4]); atomicMax(&bounds[5], sb[5]);
    if (sb[6]) atomicOr(&bounds[6], 1);
  }
}

__global__ void k_init_bounds(int* b) {
  if (threadIdx.x < 3) { b[threadIdx.x] = INT_MAX; b[3 + threadIdx.x] = INT_MIN; }
  if (threadIdx.x == 6) b[6] = 0;
}

__global__ void k_gather(const double* z, const int* idx, int64_t n, double* zs) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) zs[i] = z[idx[i]];
}

struct ZAt {
  const double* z;
  __device__ double operator()(int64_t i) const { return z[i]; }
};
struct SqDevAt {
  const double* z;
  double mean;
  __device__ double operator()(int64_t i) const {
    const double d = __dsub_rn(z[i], mean);
    return __dmul_rn(d, d);
  }
};

__global__ void k_features(const int* counts, const int* offsets, const int* nruns, const double* zs,
                           int kind, double* values) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= *nruns) return;
  const int64_t lo = offsets[v], hi = lo + counts[v];
  const double cnt = (double)counts[v];
  if (kind == 1) {
    values[v] = cnt;
    return;
  }
  const double mean = __ddiv_rn(segment_sum(ZAt{zs}, lo, hi), cnt);
  const double ssd = segment_sum(SqDevAt{zs, mean}, lo, hi);
  values[v] = __ddiv_rn(ssd > 0.0 ? ssd : 0.0, cnt);
}

cudaError_t exact_alloc(ExactScratch& s, int64_t n) {
  if (n <= s.cap_n) return cudaSuccess;
  exact_free(s);
  const int64_t m = n < 1 ? 1 : n;
  VMI_TRY(cudaMalloc(&s.keys, m * 8));
  VMI_TRY(cudaMalloc(&s.keys_sorted, m * 8));
  VMI_TRY(cudaMalloc(&s.idx, m * 4));
  VMI_TRY(cudaMalloc(&s.idx_sorted, m * 4));
  VMI_TRY(cudaMalloc(&s.z, m * 8));
  VMI_TRY(cudaMalloc(&s.zs, m * 8));
  VMI_TRY(cudaMalloc(&s.ukeys, m * 8));
  VMI_TRY(cudaMalloc(&s.counts, m * 4));
  VMI_TRY(cudaMalloc(&s.offsets, m * 4));
  VMI_TRY(cudaMalloc(&s.values, m * 8));
  VMI_TRY(cudaMalloc(&s.nruns, 16));
  VMI_TRY(cudaMalloc(&s.bounds, 16 * 4));
  VMI_TRY(cudaMalloc(&s.ghist, kMaxW * kMaxW * 4));
  size_t b1 = 0, b2 = 0, b3 = 0;
  VMI_TRY(cub::DeviceRadixSort::SortPairs(nullptr, b1, s.keys, s.keys_sorted, s.idx, s.idx_sorted,
                                          (int)m, 0, 63));
  VMI_TRY(cub::DeviceRunLengthEncode::Encode(nullptr, b2, s.keys_sorted, s.ukeys, s.counts,
                                             s.nruns, (int)m));
  VMI_TRY(cub::DeviceScan::ExclusiveSum(nullptr, b3, s.counts, s.offsets, (int)m));
  s.cub_bytes = b1 > b2 ? b1 : b2;
  if (b3 > s.cub_bytes) s.cub_bytes = b3;
  {  // the box path (box_voxelize) sorts / encodes 32-bit keys in the same buffers
    uint32_t* k32 = reinterpret_cast<uint32_t*>(s.keys);
    uint32_t* k32s = reinterpret_cast<uint32_t*>(s.keys_sorted);
    size_t c1 = 0, c2 = 0;
    VMI_TRY(cub::DeviceRadixSort::SortPairs(nullptr, c1, k32, k32s, s.idx, s.idx_sorted, (int)m, 0,
                                            32));
    VMI_TRY(cub::DeviceRunLengthEncode::Encode(nullptr, c2, k32s,
                                               reinterpret_cast<uint32_t*>(s.ukeys), s.counts,
                                               s.nruns, (int)m));
    if (c1 > s.cub_bytes) s.cub_bytes = c1;
    if (c2 > s.cub_bytes) s.cub_bytes = c2;
  }
  VMI_TRY(cudaMalloc(&s.cub_tmp, s.cub_bytes));
  s.cap_n = m;
  return cudaSuccess;
}

void exact_free(ExactScratch& s) {
  void* ptrs[] = {s.keys, s.keys_sorted, s.idx, s.idx_sorted, s.z, s.zs, s.ukeys, s.counts,
                  s.offsets, s.values, s.nruns, s.bounds, s.ghist, s.cub_tmp};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  s = ExactScratch();
}

cudaError_t exact_voxelize(ExactScratch& s, const PointSource& src, const double* mat,
                           const GridParams& g, cudaStream_t st, int64_t* launches) {
  const int64_t n = src.n;
  VMI_TRY(exact_alloc(s, n));
  const int T = 256;
  const int blocks = (int)((n + T - 1) / T);
  k_init_bounds<<<1, 32, 0, st>>>(s.bounds);
  k_exact_keys<<<blocks, T, 0, st>>>(src, mat, g, s.keys, s.idx, s.z, s.bounds);
  size_t bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceRadixSort::SortPairs(s.cub_tmp, bytes, s.keys, s.keys_sorted, s.idx,
                                          s.idx_sorted, (int)n, 0, 63, st));
  bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceRunLengthEncode::Encode(s.cub_tmp, bytes, s.keys_sorted, s.ukeys, s.counts,
                                             s.nruns, (int)n, st));
  // counts past the run count are stale; the scan over n entries only needs
  // the first V offsets to be right
  bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceScan::ExclusiveSum(s.cub_tmp, bytes, s.counts, s.offsets, (int)n, st));
  k_gather<<<blocks, T, 0, st>>>(s.z, s.idx_sorted, n, s.zs);
  k_features<<<blocks, T, 0, st>>>(s.counts, s.offsets, s.nruns, s.zs, g.kind, s.values);
  if (launches) *launches += 5;  // own kernels (CUB launches not counted)
  return cudaGetLastError();
}

// ---- scan A inside a known box (pair sets: bounds from the host AABB) --------
// The packed key's x-major lexicographic order (voxel.py:65-73) is the order of
// the linear index inside scan A's voxel box, so a stable sort of 32-bit box
// indices over ceil(log2(volume)) bits gives voxelize's exact order (stable
// within a voxel: numpy's reduceat order for VARZ) in a few radix passes
// instead of eight 64-bit ones.
__global__ void k_box_keys(PointSource src, GridParams g, int3 amin, uint3 ext, uint32_t* keys,
                           int* idx, double* zout, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= src.n) return;
  double x, y, z;
  point_at(src, i, x, y, z);
  int a, b, c;
  bool ok = voxel_coord(x, g.origin[0], g.res, g.inv_res, g.mode, a);
  ok &= voxel_coord(y, g.origin[1], g.res, g.inv_res, g.mode, b);
  ok &= voxel_coord(z, g.origin[2], g.res, g.inv_res, g.mode, c);
  const uint32_t rx = (uint32_t)(a - amin.x), ry = (uint32_t)(b - amin.y), rz = (uint32_t)(c - amin.z);
  if (!ok || rx >= ext.x || ry >= ext.y || rz >= ext.z) {  // cannot happen: the box is exact
    *bad = 1;
    keys[i] = 0;
  } else {
    keys[i] = (rx * ext.y + ry) * ext.z + rz;
  }
  idx[i] = (int)i;
  zout[i] = z;
}

cudaError_t box_voxelize(ExactScratch& s, const PointSource& src, const GridParams& g,
                         const int amin[3], const uint32_t ext[3], cudaStream_t st,
                         int64_t* launches) {
  const int64_t n = src.n;
  VMI_TRY(exact_alloc(s, n));
  const uint64_t vol = (uint64_t)ext[0] * ext[1] * ext[2];
  int nbits = 1;
  while (nbits < 32 && (1ull << nbits) < vol) ++nbits;
  const int T = 256;
  const int blocks = (int)((n + T - 1) / T);
  uint32_t* k32 = reinterpret_cast<uint32_t*>(s.keys);
  uint32_t* k32s = reinterpret_cast<uint32_t*>(s.keys_sorted);
  uint32_t* u32 = reinterpret_cast<uint32_t*>(s.ukeys);
  VMI_TRY(cudaMemsetAsync(s.bounds + 6, 0, 4, st));
  k_box_keys<<<blocks, T, 0, st>>>(src, g, make_int3(amin[0], amin[1], amin[2]),
                                   make_uint3(ext[0], ext[1], ext[2]), k32, s.idx, s.z,
                                   s.bounds + 6);
  size_t bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceRadixSort::SortPairs(s.cub_tmp, bytes, k32, k32s, s.idx, s.idx_sorted, (int)n,
                                          0, nbits, st));
  bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceRunLengthEncode::Encode(s.cub_tmp, bytes, k32s, u32, s.counts, s.nruns,
                                             (int)n, st));
  bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceScan::ExclusiveSum(s.cub_tmp, bytes, s.counts, s.offsets, (int)n, st));
  k_gather<<<blocks, T, 0, st>>>(s.z, s.idx_sorted, n, s.zs);
  k_features<<<blocks, T, 0, st>>>(s.counts, s.offsets, s.nruns, s.zs, g.kind, s.values);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

__global__ void k_build_grid_box(const uint32_t* lin, const double* values, const int* Vdev,
                                 GridParams g, uint3 ext, uint8_t* grid, int4* avox_tmp,
                                 uint32_t* bin_total) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= *Vdev) return;
  const uint32_t l = lin[v];
  const uint32_t rz = l % ext.z, rxy = l / ext.z;
  const uint32_t ry = rxy % ext.y, rx = rxy / ext.y;
  const int bin = feature_bin(values[v], g.clamp, g.bins);
  grid[l] = (uint8_t)bin;
  avox_tmp[v] = make_int4((int)rx, (int)ry, (int)rz, bin);
  atomicAdd(&bin_total[bin], 1u);
}

// ---- scan A's reference grid -------------------------------------------------
__global__ void k_build_grid(const unsigned long long* keys, const double* values, int V,
                             const int* Vdev, GridParams g, int3 amin, uint3 ext, uint8_t* grid,
                             int4* avox_tmp, uint32_t* bin_total, SparseRef sp) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (Vdev ? *Vdev : V)) return;
  const unsigned long long k = keys[v];
  const int x = (int)((k >> 42) & 0x1FFFFF) - (1 << 20);
  const int y = (int)((k >> 21) & 0x1FFFFF) - (1 << 20);
  const int z = (int)(k & 0x1FFFFF) - (1 << 20);
  const uint32_t rx = x - amin.x, ry = y - amin.y, rz = z - amin.z;
  const int bin = feature_bin(values[v], g.clamp, g.bins);
  // keys outside the declared bounds can never fall in an overlap region
  // (mi.py:139-142 masks them away); drop them from the voxel list too
  if (!(rx < ext.x && ry < ext.y && rz < ext.z)) {
    avox_tmp[v] = make_int4(0, 0, 0, -1);
    return;
  }
  if (grid) {
    grid[((size_t)rx * ext.y + ry) * ext.z + rz] = (uint8_t)bin;
  } else {  // sparse reference: insert k (a repeated key keeps one slot, last bin wins)
    for (uint32_t h = ref_slot(k, sp.mask);; h = (h + 1) & sp.mask) {
      const unsigned long long prev = atomicCAS(&sp.keys[h], ~0ull, k);
      if (prev == ~0ull || prev == k) { sp.bins[h] = (uint8_t)bin; break; }
    }
  }
  avox_tmp[v] = make_int4((int)rx, (int)ry, (int)rz, bin);
  atomicAdd(&bin_total[bin], 1u);
}

__global__ void k_bin_offsets(const uint32_t* bin_total, int W, int* cursor) {
  if (threadIdx.x == 0) {
    int s = 0;
    for (int b = 0; b < W; ++b) { cursor[b] = s; s += (int)bin_total[b]; }
  }
}

__global__ void k_scatter_by_bin(const int4* avox_tmp, int V, const int* Vdev, int* cursor,
                                 int4* avox) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= (Vdev ? *Vdev : V)) return;
  const int4 a = avox_tmp[v];
  if (a.w >= 0) avox[atomicAdd(&cursor[a.w], 1)] = a;
}

cudaError_t build_reference_box(const ExactScratch& s, int Vmax, const GridParams& g,
                                const uint32_t ext[3], uint8_t* grid, int4* tmp, int4* avox,
                                uint32_t* bin_total, int* cursor, cudaStream_t st,
                                int64_t* launches) {
  if (Vmax <= 0) return cudaSuccess;
  const int T = 256, blocks = (Vmax + T - 1) / T;
  k_build_grid_box<<<blocks, T, 0, st>>>(reinterpret_cast<const uint32_t*>(s.ukeys), s.values,
                                         s.nruns, g, make_uint3(ext[0], ext[1], ext[2]), grid, tmp,
                                         bin_total);
  k_bin_offsets<<<1, 32, 0, st>>>(bin_total, g.bins + 1, cursor);
  k_scatter_by_bin<<<blocks, T, 0, st>>>(tmp, Vmax, s.nruns, cursor, avox);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

cudaError_t build_reference(const unsigned long long* keys, const double* values, int V,
                            const int* Vdev, const GridParams& g, const int amin[3],
                            const uint32_t ext[3], uint8_t* grid, int4* tmp, int4* avox,
                            uint32_t* bin_total, int* cursor, cudaStream_t st, int64_t* launches,
                            SparseRef sp) {
  if (V <= 0) return cudaSuccess;
  const int T = 256, blocks = (V + T - 1) / T;
  k_build_grid<<<blocks, T, 0, st>>>(keys, values, V, Vdev, g,
                                     make_int3(amin[0], amin[1], amin[2]),
                                     make_uint3(ext[0], ext[1], ext[2]), grid, tmp, bin_total, sp);
  k_bin_offsets<<<1, 32, 0, st>>>(bin_total, g.bins + 1, cursor);
  k_scatter_by_bin<<<blocks, T, 0, st>>>(tmp, V, Vdev, cursor, avox);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

// ---- exact histogram + score for one pose ----------------------------------
__global__ void k_exact_hist(const unsigned long long* keys, const double* values,
                             const int* nruns, GridParams g, RefView A, unsigned int* ghist) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= *nruns) return;
  const unsigned long long k = keys[v];
  const int x = (int)((k >> 42) & 0x1FFFFF) - (1 << 20);
  const int y = (int)((k >> 21) & 0x1FFFFF) - (1 << 20);
  const int z = (int)(k & 0x1FFFFF) - (1 << 20);
  const uint32_t rx = x - A.amin[0], ry = y - A.amin[1], rz = z - A.amin[2];
  if (A.empty || !(rx < A.ext[0] && ry < A.ext[1] && rz < A.ext[2])) return;
  const int W = g.bins + 1;
  const int ba = A.sparse ? ref_sparse_bin(A, k) : A.grid[((size_t)rx * A.ext[1] + ry) * A.ext[2] + rz];
  const int bb = feature_bin(values[v], g.clamp, g.bins);
  atomicAdd(&ghist[ba * W + bb], 1u);
}

constexpr int kScoreThreads = 512;

__global__ void __launch_bounds__(kScoreThreads)
    k_exact_finalize(const int* bounds, const unsigned int* ghist, GridParams g, RefView A,
                     int64_t p, double* mi_out, int32_t* status_out, long long* hist_out,
                     long long* total_out, unsigned long long* hash_out) {
  __shared__ uint32_t hist[kMaxW * kMaxW];
  __shared__ uint32_t marg[kMaxW];
  __shared__ double red[3 * kScoreThreads / 32];
  __shared__ long long rows[kMaxW], cols[kMaxW], h00;
  const int W = g.bins + 1;
  const int tid = threadIdx.x;
  int status = 0;
  int rlo[3], rhi[3];
  long long n_region = 0;
  if (bounds[6]) status = 2;
  else if (A.empty) status = 1;
  else {
    n_region = 1;
    for (int j = 0; j < 3; ++j) {
      rlo[j] = max(A.amin[j], bounds[j]);
      rhi[j] = min(A.amax[j], bounds[3 + j]);
      if (rlo[j] > rhi[j]) status = 1;
      n_region *= (long long)(rhi[j] - rlo[j] + 1);
    }
  }
  if (status != 0) {
    if (tid == 0) {
      mi_out[p] = -1e300;
      status_out[p] = status;
      if (total_out) total_out[p] = 0;
      if (hash_out) hash_out[p] = 0;
    }
    if (hist_out)
      for (int i = tid; i < W * W; i += kScoreThreads) hist_out[p * W * W + i] = 0;
    return;
  }
  for (int i = tid; i < W * W; i += kScoreThreads) hist[i] = ghist[i];
  for (int i = tid; i < W; i += kScoreThreads) marg[i] = 0;
  __syncthreads();
  for (int j = tid; j < A.n_avox; j += kScoreThreads) {
    const int4 v = A.avox[j];
    const int x = v.x + A.amin[0], y = v.y + A.amin[1], z = v.z + A.amin[2];
    if (x >= rlo[0] && x <= rhi[0] && y >= rlo[1] && y <= rhi[1] && z >= rlo[2] && z <= rhi[2])
      atomicAdd(&marg[v.w], 1u);
  }
  __syncthreads();
  MIOut r = finalize_mi<kScoreThreads>(hist, marg, W, n_region, g.include_phi, red, rows, cols, &h00);
  if (tid == 0) {
    mi_out[p] = r.status == 0 ? r.mi : -1e300;
    status_out[p] = r.status;
    if (total_out) total_out[p] = n_region;
  }
  if (hist_out)
    for (int i = tid; i < W * W; i += kScoreThreads)
      hist_out[p * W * W + i] = i == 0 ? r.h00 : (long long)hist[i];
  if (hash_out) {  // the fast kernel's histogram identity (vmi_device.cuh)
    __shared__ unsigned long long hred[kScoreThreads / 32];
    const unsigned long long h = block_hist_hash<kScoreThreads>(hist, r.h00, W, hred);
    if (tid == 0) hash_out[p] = r.status == 0 ? h : 0ull;
  }
}

cudaError_t exact_score(ExactScratch& s, const GridParams& g, const RefView& A, int64_t p,
                        double* mi, int32_t* status, long long* hist, long long* total,
                        cudaStream_t st, int64_t* launches, unsigned long long* hash) {
  const int W = g.bins + 1;
  VMI_TRY(cudaMemsetAsync(s.ghist, 0, (size_t)W * W * 4, st));
  const int T = 256;
  const int blocks = (int)((s.cap_n + T - 1) / T);
  k_exact_hist<<<blocks, T, 0, st>>>(s.ukeys, s.values, s.nruns, g, A, s.ghist);
  k_exact_finalize<<<1, kScoreThreads, 0, st>>>(s.bounds, s.ghist, g, A, p, mi, status, hist, total,
                                                hash);
  if (launches) *launches += 2;
  return cudaGetLastError();
}

// ---- argmax (np.argmax: first index of the maximum) ---------------------------
__global__ void k_argmax(const double* v, int64_t P, double* out_val, long long* out_idx) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  double best = -INFINITY;
  long long bi = LLONG_MAX;
  for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
    const double x = v[i];
    if (x > best) { best = x; bi = i; }  // strided: first hit per thread is its lowest index
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sv[threadIdx.x >> 5] = best; si[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sv[w] > best || (sv[w] == best && si[w] < bi)) { best = sv[w]; bi = si[w]; }
    *out_val = best;
    *out_idx = bi;
  }
}

cudaError_t launch_argmax(const double* v, int64_t P, double* out_val, long long* out_idx,
                          cudaStream_t st) {
  k_argmax<<<1, 1024, 0, st>>>(v, P, out_val, out_idx);
  return cudaGetLastError();
}

// ---- top-K: stable descending radix sort of (mi, index) -----------------------
__global__ void k_iota(int* a, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}

cudaError_t topk_sort(const double* mi, int P, double* keys_out, int* idx_in, int* idx_out,
                      void* tmp, size_t* tmp_bytes, cudaStream_t st) {
  if (!tmp)  // size query
    return cub::DeviceRadixSort::SortPairsDescending(nullptr, *tmp_bytes, mi, keys_out, idx_in,
                                                     idx_out, P, 0, 64, st);
  k_iota<<<(P + 255) / 256, 256, 0, st>>>(idx_in, P);
  // CUB's radix sort is stable: equal MI keep ascending candidate order, so
  // the first entry is np.argmax's first maximum
  return cub::DeviceRadixSort::SortPairsDescending(tmp, *tmp_bytes, mi, keys_out, idx_in, idx_out,
                                                   P, 0, 64, st);
}

// ---- span layout (see QueryView) ------------------------------------------------
// ---- scan B's voxel-grouped order (unordered scans) ---------------------------
// Keys are exact_voxelize's packed voxel keys in ORIGINAL point order (s.keys):
// count the places where consecutive points change voxel (runs - 1).
__global__ void k_count_changes(const unsigned long long* keys, int64_t n, int* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool ch = i >= 1 && i < n && keys[i] != keys[i - 1];
  const unsigned m = __ballot_sync(0xffffffffu, ch);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(out, __popc(m));
}

// dst[i] = src[perm[i]] for 16- or 24-byte point records
__global__ void k_gather_points(const void* src, int rec, const int* perm, int64_t n, void* dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = perm[i];
  if (rec == 16) {
    reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[j];
  } else {
    const double* s = reinterpret_cast<const double*>(src) + 3 * j;
    double* d = reinterpret_cast<double*>(dst) + 3 * i;
    d[0] = s[0]; d[1] = s[1]; d[2] = s[2];
  }
}

cudaError_t voxel_order(const ExactScratch& s, const void* src, int rec, int64_t n, int* changes,
                        void* dst, cudaStream_t st) {
  const int T = 256;
  const int blocks = (int)((n + T - 1) / T);
  VMI_TRY(cudaMemsetAsync(changes, 0, 4, st));
  k_count_changes<<<blocks, T, 0, st>>>(s.keys, n, changes);
  if (dst) k_gather_points<<<blocks, T, 0, st>>>(src, rec, s.idx_sorted, n, dst);
  return cudaGetLastError();
}

// ---- summed-volume tables of scan A per present bin (RefView.sat) -------------
__global__ void k_sat_fill(const int4* avox, int n, const int* bin_slot, uint3 ext, uint32_t* sat) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const int4 a = avox[v];
  const int k = bin_slot[a.w];
  if (k < 0) return;
  const size_t sy = ext.z + 1, sx = (size_t)(ext.y + 1) * sy, vol = sx * (ext.x + 1);
  sat[(size_t)k * vol + (a.x + 1) * sx + (a.y + 1) * sy + (a.z + 1)] = 1u;
}
// inclusive prefix along one axis: lines = every (k, other two coordinates)
__global__ void k_sat_scan(uint32_t* sat, int nb, uint3 ext, int axis) {
  const size_t sy = ext.z + 1, sx = (size_t)(ext.y + 1) * sy, vol = sx * (ext.x + 1);
  const size_t n1 = ext.x + 1, n2 = ext.y + 1, n3 = ext.z + 1;
  const size_t len = axis == 0 ? n1 : axis == 1 ? n2 : n3;
  const size_t stride = axis == 0 ? sx : axis == 1 ? sy : 1;
  const size_t lines_per = vol / len;
  const size_t line = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (line >= lines_per * (size_t)nb) return;
  const size_t k = line / lines_per, r = line - k * lines_per;
  size_t base;
  if (axis == 2) base = r * n3;                           // r = x * n2 + y
  else if (axis == 1) base = (r / n3) * sx + (r % n3);    // r = x * n3 + z
  else base = r;                                          // r = y * n3 + z
  uint32_t* t = sat + k * vol + base;
  uint32_t acc = 0;
  for (size_t i = 0; i < len; ++i) {
    acc += t[i * stride];
    t[i * stride] = acc;
  }
}
cudaError_t build_sat(const int4* avox, int n, const int* bin_slot_dev, int nb, const uint32_t ext[3],
                      uint32_t* sat, cudaStream_t st) {
  const uint3 e = make_uint3(ext[0], ext[1], ext[2]);
  const size_t vol = (size_t)(e.x + 1) * (e.y + 1) * (e.z + 1);
  VMI_TRY(cudaMemsetAsync(sat, 0, vol * nb * 4, st));
  const int T = 256;
  if (n > 0) k_sat_fill<<<(n + T - 1) / T, T, 0, st>>>(avox, n, bin_slot_dev, e, sat);
  const size_t lens[3] = {e.x + 1, e.y + 1, e.z + 1};
  for (int axis = 2; axis >= 0; --axis) {
    const size_t lines = vol / lens[axis] * nb;
    k_sat_scan<<<(unsigned)((lines + T - 1) / T), T, 0, st>>>(sat, nb, e, axis);
  }
  return cudaGetLastError();
}

// ---- re-planned re-runs of flagged poses (vmi_api.cu do_fixups) ----------------
template <typename T>
__global__ void k_gather_rows(const T* src, const int64_t* idx, int64_t n, int w, T* dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * w) return;
  const int64_t r = i / w, k = i - r * w;
  dst[i] = src[idx[r] * w + k];
}
template <typename T>
__global__ void k_scatter_rows(const T* src, const int64_t* idx, int64_t n, int w, T* dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * w) return;
  const int64_t r = i / w, k = i - r * w;
  dst[idx[r] * w + k] = src[i];
}
template <typename T>
cudaError_t gather_rows(const T* src, const int64_t* idx, int64_t n, int w, T* dst, bool scatter,
                        cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int T_ = 256;
  const unsigned blocks = (unsigned)((n * w + T_ - 1) / T_);
  if (scatter) k_scatter_rows<T><<<blocks, T_, 0, st>>>(src, idx, n, w, dst);
  else k_gather_rows<T><<<blocks, T_, 0, st>>>(src, idx, n, w, dst);
  return cudaGetLastError();
}
template cudaError_t gather_rows<double>(const double*, const int64_t*, int64_t, int, double*, bool,
                                         cudaStream_t);
template cudaError_t gather_rows<int32_t>(const int32_t*, const int64_t*, int64_t, int, int32_t*,
                                          bool, cudaStream_t);
template cudaError_t gather_rows<long long>(const long long*, const int64_t*, int64_t, int,
                                            long long*, bool, cudaStream_t);

// Contiguous host-order points -> the fast kernel's span layout: split-double
// float4 records (out_split; every coordinate float32-exact), else double4.
// src is float32 (x, y, z, i) records (in_f32) or (n, 3) doubles.
__device__ __forceinline__ void span_layout_one(const void* src, int in_f32, int out_split,
                                                int64_t n, int span, int rem, int threads,
                                                void* dst, int64_t i) {
  double x = 0.0, y = 0.0, z = 0.0;
  int64_t li;
  if (i >= n) {  // padding slots: the (threads - rem) unused last-iteration entries
    li = (int64_t)(span - 1) * threads + thread_of_span(rem + (int)(i - n), threads);
  } else {
    li = span_slot(i, span, rem, threads);
    if (in_f32) {
      const float4 v = reinterpret_cast<const float4*>(src)[i];
      x = v.x; y = v.y; z = v.z;
    } else {
      const double* s = reinterpret_cast<const double*>(src);
      x = s[3 * i]; y = s[3 * i + 1]; z = s[3 * i + 2];
    }
  }
  if (out_split) {  // (the intensity is unused)
#if VMI_SPLITREC
    reinterpret_cast<uint4*>(dst)[li] = split_encode((float)x, (float)y, (float)z);
#else
    reinterpret_cast<float4*>(dst)[li] = make_float4((float)x, (float)y, (float)z, 0.f);
#endif
  } else {
    reinterpret_cast<double4*>(dst)[li] = make_double4(x, y, z, 0.0);
  }
}

__global__ void k_span_layout(const void* src, int in_f32, int out_split, int64_t n, int span,
                              int rem, int threads, void* dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // original index
  if (i >= (int64_t)span * threads) return;
  span_layout_one(src, in_f32, out_split, n, span, rem, threads, dst, i);
}

// ---- a group of pair-set pairs built together (vmi_set_pairs) -----------------
// One launch per stage for G pairs: scan A's 32-bit keys are (pair << nbits) |
// box index, so ONE stable radix sort over the group orders every pair's
// points exactly as its own voxelize would (pair-major, then x-major, then
// input order), and run-length encoding, the features and the grids follow in
// single launches too.
__global__ void k_group_zero(const GroupPair* gp, int* vcount) {
  const GroupPair& q = gp[blockIdx.y];
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < q.grid_bytes;
       i += (size_t)gridDim.x * blockDim.x)
    q.grid[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < kMaxW) q.bin_total[threadIdx.x] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) vcount[blockIdx.y] = 0;
}

__global__ void k_group_keys(const GroupPair* gp, GridParams g, int in_f32, int nbits,
                             uint32_t* keys, int* idx, double* zout, int* bad) {
  const GroupPair& q = gp[blockIdx.y];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= q.n) return;
  PointSource src{};
  if (in_f32) src.rec = static_cast<const float4*>(q.raw_a);
  else src.xyz = static_cast<const double*>(q.raw_a);
  src.n = q.n;
  double x, y, z;
  point_at(src, j, x, y, z);
  int a, b, c;
  bool ok = voxel_coord(x, g.origin[0], g.res, g.inv_res, g.mode, a);
  ok &= voxel_coord(y, g.origin[1], g.res, g.inv_res, g.mode, b);
  ok &= voxel_coord(z, g.origin[2], g.res, g.inv_res, g.mode, c);
  const uint32_t rx = (uint32_t)(a - q.amin.x), ry = (uint32_t)(b - q.amin.y),
                 rz = (uint32_t)(c - q.amin.z);
  const int64_t o = q.off + j;
  if (!ok || rx >= q.ext.x || ry >= q.ext.y || rz >= q.ext.z) {  // cannot happen: exact box
    bad[blockIdx.y] = 1;
    keys[o] = (uint32_t)blockIdx.y << nbits;
  } else {
    keys[o] = ((uint32_t)blockIdx.y << nbits) | ((rx * q.ext.y + ry) * q.ext.z + rz);
  }
  idx[o] = (int)o;
  zout[o] = z;
}

__global__ void k_group_grid(const GroupPair* gp, const uint32_t* ukeys, const double* values,
                             const int* nruns, GridParams g, int nbits, int4* avox_tmp,
                             int* vcount) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= *nruns) return;
  const uint32_t k = ukeys[v];
  const int pr = (int)(k >> nbits);
  const uint32_t l = k & ((1u << nbits) - 1u);
  const GroupPair& q = gp[pr];
  const uint32_t rz = l % q.ext.z, rxy = l / q.ext.z;
  const uint32_t ry = rxy % q.ext.y, rx = rxy / q.ext.y;
  const int bin = feature_bin(values[v], g.clamp, g.bins);
  q.grid[l] = (uint8_t)bin;
  avox_tmp[v] = make_int4((int)rx, (int)ry, (int)rz, bin | (pr << 16));
  atomicAdd(&q.bin_total[bin], 1u);
  atomicAdd(&vcount[pr], 1);
}

__global__ void k_group_cursors(const GroupPair* gp, int W, int* cursor) {
  if (threadIdx.x == 0) {
    const GroupPair& q = gp[blockIdx.x];
    int s = 0;
    for (int b = 0; b < W; ++b) { cursor[blockIdx.x * kMaxW + b] = s; s += (int)q.bin_total[b]; }
  }
}

__global__ void k_group_scatter(const GroupPair* gp, const int4* avox_tmp, const int* nruns,
                                int* cursor) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= *nruns) return;
  int4 a = avox_tmp[v];
  const int pr = a.w >> 16;
  a.w &= 0xFFFF;
  gp[pr].avox[atomicAdd(&cursor[pr * kMaxW + a.w], 1)] = a;
}

__global__ void k_group_layout(const GroupPair* gp, int in_f32, int threads) {
  const GroupPair& q = gp[blockIdx.y];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)q.span * threads) return;
  span_layout_one(q.raw_b, in_f32, q.b_split, q.nb, q.span, q.rem, threads, q.pts, i);
}

cudaError_t build_pair_group(ExactScratch& s, const GroupPair* gp_dev, int G, int64_t n_total,
                             int max_na, int max_nb_rows, size_t max_grid, int nbits,
                             const GridParams& g, int in_f32, int threads, int4* avox_tmp,
                             int* cursor, int* vcount, int* bad, cudaStream_t st,
                             int64_t* launches) {
  VMI_TRY(exact_alloc(s, n_total));
  const int T = 256;
  const int zb = (int)std::min<size_t>(1024, (max_grid + T * 4 - 1) / (T * 4));
  k_group_zero<<<dim3(zb > 0 ? zb : 1, G), T, 0, st>>>(gp_dev, vcount);
  uint32_t* k32 = reinterpret_cast<uint32_t*>(s.keys);
  uint32_t* k32s = reinterpret_cast<uint32_t*>(s.keys_sorted);
  uint32_t* u32 = reinterpret_cast<uint32_t*>(s.ukeys);
  k_group_keys<<<dim3((max_na + T - 1) / T, G), T, 0, st>>>(gp_dev, g, in_f32, nbits, k32, s.idx,
                                                            s.z, bad);
  int gbits = 0;
  while ((1 << gbits) < G) ++gbits;
  size_t bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceRadixSort::SortPairs(s.cub_tmp, bytes, k32, k32s, s.idx, s.idx_sorted,
                                          (int)n_total, 0, nbits + gbits, st));
  bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceRunLengthEncode::Encode(s.cub_tmp, bytes, k32s, u32, s.counts, s.nruns,
                                             (int)n_total, st));
  bytes = s.cub_bytes;
  VMI_TRY(cub::DeviceScan::ExclusiveSum(s.cub_tmp, bytes, s.counts, s.offsets, (int)n_total, st));
  const int blocks = (int)((n_total + T - 1) / T);
  k_gather<<<blocks, T, 0, st>>>(s.z, s.idx_sorted, n_total, s.zs);
  k_features<<<blocks, T, 0, st>>>(s.counts, s.offsets, s.nruns, s.zs, g.kind, s.values);
  k_group_grid<<<blocks, T, 0, st>>>(gp_dev, u32, s.values, s.nruns, g, nbits, avox_tmp, vcount);
  k_group_cursors<<<G, 32, 0, st>>>(gp_dev, g.bins + 1, cursor);
  k_group_scatter<<<blocks, T, 0, st>>>(gp_dev, avox_tmp, s.nruns, cursor);
  k_group_layout<<<dim3((max_nb_rows + T - 1) / T, G), T, 0, st>>>(gp_dev, in_f32, threads);
  if (launches) *launches += 9;
  return cudaGetLastError();
}

cudaError_t launch_span_layout(const void* src, int in_f32, int out_split, int64_t n, int span,
                               int rem, int threads, void* dst, cudaStream_t st) {
  const int64_t total = (int64_t)span * threads;
  const int T = 256;
  k_span_layout<<<(unsigned)((total + T - 1) / T), T, 0, st>>>(src, in_f32, out_split, n, span,
                                                               rem, threads, dst);
  return cudaGetLastError();
}

}  // namespace vmi
