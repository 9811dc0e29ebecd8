// vmi_device.cuh -- device-side building blocks shared by the fast (hash) and
// exact (sort) pose-evaluation paths.  Every floating-point step that the
// reference's bit pattern depends on is written with explicit-rounding
// intrinsics so nvcc's FMA contraction can never change it.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "vmi_types.h"

namespace vmi {

constexpr uint32_t kNoVoxel = 0xFFFFFFFFu;
constexpr int kKeyMin = -(1 << 20);
constexpr int kKeyMax = (1 << 20) - 1;

// ---- float32 scan-B records, stored pre-widened ("split doubles") -----------
// (double)f of a float has a 24-bit significand: the double's low word holds
// only its top 3 bits.  Words 0-2 of a record are the high words of (double)x,
// (double)y, (double)z; word 3 packs the three low words' top bits (x in bits
// 31..29, y in 28..26, z in 25..23).  Decoding is 4 integer ops instead of 3
// F2F.F64.F32 conversions (XU pipe, variable latency) per point.
#ifndef VMI_SPLITREC
#define VMI_SPLITREC 1
#endif
__device__ __forceinline__ uint4 split_encode(float x, float y, float z) {
  const double d[3] = {(double)x, (double)y, (double)z};
  uint4 r;
  r.x = (uint32_t)__double2hiint(d[0]);
  r.y = (uint32_t)__double2hiint(d[1]);
  r.z = (uint32_t)__double2hiint(d[2]);
  r.w = ((uint32_t)__double2loint(d[0]) & 0xE0000000u) |
        (((uint32_t)__double2loint(d[1]) & 0xE0000000u) >> 3) |
        (((uint32_t)__double2loint(d[2]) & 0xE0000000u) >> 6);
  return r;
}
__device__ __forceinline__ void split_decode(uint4 v, double& x, double& y, double& z) {
  x = __hiloint2double((int)v.x, (int)(v.w & 0xE0000000u));
  y = __hiloint2double((int)v.y, (int)((v.w << 3) & 0xE0000000u));
  z = __hiloint2double((int)v.z, (int)(v.w << 6));
}


// ---- geometry.py:162-166: numpy `points @ R.T + t` through OpenBLAS dgemm is,
// bit for bit, fma(z, R[j][2], fma(y, R[j][1], x * R[j][0])) + t[j].
// the same chain before + t[j] (R p alone)
__device__ __forceinline__ double rot_row(double x, double y, double z, double r0, double r1,
                                          double r2) {
  return __fma_rn(z, r2, __fma_rn(y, r1, __dmul_rn(x, r0)));
}
__device__ __forceinline__ double xform_row(double x, double y, double z, double r0, double r1,
                                            double r2, double t) {
  return __dadd_rn(__fma_rn(z, r2, __fma_rn(y, r1, __dmul_rn(x, r0))), t);
}

// ---- voxel.py:199: floor((p - origin) / resolution) -> int64, then the
// key-range test of voxel.py:200.  The floor is DADD.RM against 1.5*2^52: the
// result's bit pattern minus the magic's is floor(q) for |q| < 2^51, and lands
// far outside the key range otherwise (incl. inf/nan), so one compare covers
// OutOfBoundsError.  Returns false when out of the key range.
__device__ __forceinline__ bool voxel_coord(double p, double origin, double res, double inv_res,
                                            int mode, int& out) {
  double v = (mode == kGridUnit) ? p : __dsub_rn(p, origin);
  double q;
  if (mode == kGridUnit) q = v;
  else if (mode == kGridPow2) q = __dmul_rn(v, inv_res);  // exact: same real number as v/res
  else q = __ddiv_rn(v, res);
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  double r = __dadd_rd(q, magic);
  long long k = __double_as_longlong(r) - __double_as_longlong(magic);
  out = (int)k;
  return (unsigned long long)(k - kKeyMin) <= (unsigned long long)(kKeyMax - kKeyMin);
}

// Compile-time-specialised q = (p - origin) / resolution (voxel.py:199).
template <int MODE>
__device__ __forceinline__ double grid_q(double p, double origin, double res, double inv_res) {
  if (MODE == kGridUnit) return p;
  const double v = __dsub_rn(p, origin);
  if (MODE == kGridPow2) return __dmul_rn(v, inv_res);  // exact: same real number as v/res
  return __ddiv_rn(v, res);
}

// floor(q) as int32 via DADD.RM against 1.5*2^52: bits(r) = bits(magic) + floor(q),
// so the low word is floor(q) whenever |q| < 2^31 (callers guarantee |q| < 2^30).
__device__ __forceinline__ int floor_i32(double q) {
  return __double2loint(__dadd_rd(q, 6755399441055744.0));
}

// ---- mi.py:72-79 bin_features: 1 + min(B-1, floor(v / clamp * B))
__device__ __forceinline__ int feature_bin(double v, double clamp, int bins) {
  double x = __dmul_rn(__ddiv_rn(v, clamp), (double)bins);
  double f = floor(x);
  int raw = f >= (double)(bins - 1) ? bins - 1 : (int)f;
  return 1 + raw;
}

// ---- sparse reference table (RefView.sparse) ----------------------------------
// Slot of packed key k: multiplicative hash, linear probing, ~0 = empty.
__device__ __forceinline__ uint32_t ref_slot(unsigned long long k, uint32_t mask) {
  return (uint32_t)((k * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}

// Scan A's bin of packed key k (0 = not occupied).
__device__ __forceinline__ int ref_sparse_bin(const RefView& A, unsigned long long k) {
  for (uint32_t h = ref_slot(k, A.hmask);; h = (h + 1) & A.hmask) {
    const unsigned long long s = __ldg(&A.hkeys[h]);
    if (s == k) return __ldg(&A.hbins[h]);
    if (s == ~0ull) return 0;
  }
}

// numpy pairwise_sum (loops_utils.h.src) over f(lo .. lo+n-1); F(i) -> double.
template <typename F>
__device__ double pairwise_sum(const F& f, int64_t lo, int64_t n) {
  // The reference recursion (split at n2 = n/2 - (n/2)%8, left + right) run
  // post-order on an explicit stack; depth <= 26 for n < 2^32.
  struct Frame { int64_t lo, n; int state; double left; };
  Frame fr[32];
  int sp = 0;
  fr[0] = {lo, n, 0, 0.0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& cur = fr[sp];
    if (cur.n > 128) {  // split: evaluate the left half first
      int64_t n2 = cur.n / 2;
      n2 -= n2 % 8;
      cur.state = 1;
      fr[sp + 1] = {cur.lo, n2, 0, 0.0};
      ++sp;
      continue;
    }
    if (cur.n < 8) {
      ret = 0.0;
      for (int64_t i = 0; i < cur.n; ++i) ret = __dadd_rn(ret, f(cur.lo + i));
    } else {
      double r[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = f(cur.lo + j);
      int64_t i = 8;
      for (; i < cur.n - (cur.n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], f(cur.lo + i + j));
      }
      ret = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                      __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
      for (; i < cur.n; ++i) ret = __dadd_rn(ret, f(cur.lo + i));
    }
    --sp;
    while (sp >= 0) {  // hand the finished block to its parent
      Frame& par = fr[sp];
      if (par.state == 1) {
        par.left = ret;
        par.state = 2;
        int64_t n2 = par.n / 2;
        n2 -= n2 % 8;
        fr[sp + 1] = {par.lo + n2, par.n - n2, 0, 0.0};
        ++sp;
        break;
      }
      ret = __dadd_rn(par.left, ret);
      --sp;
    }
  }
  return ret;
}

// np.add.reduceat segment: a[lo] + pairwise(a[lo+1 : hi])  (voxel.py:225-229)
template <typename F>
__device__ __forceinline__ double segment_sum(const F& f, int64_t lo, int64_t hi) {
  if (hi - lo == 1) return f(lo);
  return __dadd_rn(f(lo), pairwise_sum(f, lo + 1, hi - lo - 1));
}

// ---- block-wide helpers -------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- 64-bit identity of a joint histogram: sum of cell * mix(cell index)
// mod 2^64 (order-free, so any reduction order gives the same value; the
// splitmix64 mixer).  Equal identities <=> equal histograms up to 2^-64.
__device__ __forceinline__ unsigned long long cell_mix(unsigned long long i) {
  i += 0x9E3779B97F4A7C15ull;
  i = (i ^ (i >> 30)) * 0xBF58476D1CE4E5B9ull;
  i = (i ^ (i >> 27)) * 0x94D049BB133111EBull;
  return i ^ (i >> 31);
}
// block-wide: hist (W x W, cell (0,0) = h00) -> identity; red >= THREADS/32
// entries of shared memory; result valid in thread 0; all threads must call
template <int THREADS>
__device__ unsigned long long block_hist_hash(const uint32_t* hist, long long h00, int W,
                                              unsigned long long* red) {
  unsigned long long h = 0;
  for (int i = threadIdx.x; i < W * W; i += THREADS)
    h += (unsigned long long)(i == 0 ? h00 : (long long)hist[i]) * cell_mix((unsigned long long)i);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = h;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < THREADS / 32; ++w) t += red[w];
  return t;
}

// ---- Histogram finalisation + MI (mi.py:124-160 analytic cells, :163-191).
// hist: (W x W) u32 in shared memory holding the enumerated cells (every B
// voxel inside the region, binned against A's grid); marg: per-A-bin count of
// A voxels inside the region.  Fills column 0 of rows >= 1 and cell (0,0),
// then computes entropies.  Must be called by all threads of the block.
struct MIOut {
  double mi, hx, hy, hxy;
  int status;
  long long h00;
};

template <int THREADS>
__device__ MIOut finalize_mi(uint32_t* hist, const uint32_t* marg, int W, long long n_region,
                             int include_phi, double* red /* >= 3*THREADS/32 doubles */,
                             long long* rows /* W */, long long* cols /* W */,
                             long long* h00_s /* 1 */) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = THREADS / 32;
  // (1) rows a >= 1: A-only voxels pair with the phi column (mi.py:146-156);
  //     one warp per row, two cells per lane (W <= 65)
  for (int a = 1 + wid; a < W; a += NW) {
    uint32_t v = 0;
    if (lane + 1 < W) v += hist[a * W + lane + 1];
    if (lane + 33 < W) v += hist[a * W + lane + 33];
    v = __reduce_add_sync(0xffffffffu, v);
    if (lane == 0) hist[a * W] = marg[a] - v;
  }
  // (2) (phi, phi) = region - |A in region| - |B-only in region|  (mi.py:158-159)
  if (wid == NW - 1) {
    uint32_t v = 0;
    for (int i = 1 + lane; i < W; i += 32) v += marg[i] + hist[i];
    v = __reduce_add_sync(0xffffffffu, v);
    if (lane == 0) *h00_s = n_region - (long long)v;
  }
  __syncthreads();
  const long long h00 = *h00_s;
  const int o = include_phi ? 0 : 1;
  const int m = W - o;
  auto cell = [&](int a, int b) -> long long {
    return (a == 0 && b == 0) ? h00 : (long long)hist[a * W + b];
  };
  // (3) exact int64 marginals m.sum(axis=1) / m.sum(axis=0): one warp per line
  for (int j = wid; j < 2 * m; j += NW) {
    const bool is_row = j < m;
    const int x = (is_row ? j : j - m) + o;
    long long v = 0;
    for (int y = o + lane; y < W; y += 32) v += is_row ? cell(x, y) : cell(y, x);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) (is_row ? rows : cols)[x - o] = v;
  }
  __syncthreads();
  // total = sum of the row marginals: every warp reduces the (<= 65) rows
  // itself (two per lane, one shuffle tree) instead of a 33-deep serial chain
  long long total = (lane < m ? rows[lane] : 0LL) + (lane + 32 < m ? rows[lane + 32] : 0LL) +
                    (lane + 64 < m ? rows[lane + 64] : 0LL);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) total += __shfl_xor_sync(0xffffffffu, total, off);
  MIOut out;
  out.h00 = h00;
  if (total <= 0) {  // entropy of an all-zero block raises -> sentinel (mi.py:215-219)
    out.status = 3;
    out.mi = out.hx = out.hy = out.hxy = 0.0;
    return out;
  }
  // (4) -sum p log p, fixed-order block reduction (deterministic)
  const double inv_tot = 1.0 / (double)total;
  double sx = 0.0, sy = 0.0, sxy = 0.0;
  for (int i = tid; i < m * m; i += THREADS) {
    const long long c = cell(i / m + o, i % m + o);
    if (c > 0) {
      const double p = (double)c * inv_tot;
      sxy += p * log(p);
    }
  }
  for (int i = tid; i < m; i += THREADS) {
    if (rows[i] > 0) { const double p = (double)rows[i] * inv_tot; sx += p * log(p); }
    if (cols[i] > 0) { const double p = (double)cols[i] * inv_tot; sy += p * log(p); }
  }
  sx = warp_sum(sx);
  sy = warp_sum(sy);
  sxy = warp_sum(sxy);
  if (lane == 0) { red[wid] = sx; red[NW + wid] = sy; red[2 * NW + wid] = sxy; }
  __syncthreads();
  // per-warp partials -> totals by one fixed-order shuffle tree (deterministic)
  static_assert(NW <= 32, "one partial per lane");
  double hx = lane < NW ? red[lane] : 0.0, hy = lane < NW ? red[NW + lane] : 0.0,
         hxy = lane < NW ? red[2 * NW + lane] : 0.0;
  hx = warp_sum(hx);
  hy = warp_sum(hy);
  hxy = warp_sum(hxy);
  hx = -hx; hy = -hy; hxy = -hxy;
  double mi = hx + hy - hxy;
  if (mi >= -1e-12 && mi < 0.0) mi = 0.0;  // mi.py:189-190
  out.status = 0;
  out.mi = mi; out.hx = hx; out.hy = hy; out.hxy = hxy;
  return out;
}

}  // namespace vmi
