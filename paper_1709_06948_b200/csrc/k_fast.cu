// k_fast.cu -- K1: fused candidate-pose evaluation (the hot path).
//
// One persistent CTA per SM walks poses p = blockIdx.x, +gridDim.x, ...  For
// each pose it replaces the whole body of mi_objective (reference
// pkg/src/voxmi/mi.py:194-219):
//
//   apply_transform (geometry.py:162-166)   fp64 FMA chain, bit-exact
//   voxel_indices   (voxel.py:192-207)      DADD.RM floor + key-range check
//   voxelize bounds (voxel.py:220)          per-thread int min/max, block reduce
//   compute_feature_map (voxel.py:267-295)  per-thread run aggregation over the
//                                           ring-ordered span, flushed into a
//                                           shared-memory open-addressing table
//                                           keyed by the voxel's index inside
//                                           A's AABB (only those voxels can be
//                                           in the overlap region)
//   compute_overlap (voxel.py:298-318)      from the reduced bounds
//   build_joint_histogram (mi.py:124-160)   table walk -> A-grid lookup ->
//                                           shared u32 histogram; A marginal
//                                           over the region from A's voxel list;
//                                           phi cells analytically
//   mutual_information (mi.py:163-191)      fused epilogue (finalize_mi)
//
// VARZ is accumulated as (n, S1 = sum(z-K), S2 = sum((z-K)^2)) around a pivot K
// that is (the float32 rounding of) the z of the first run to reach the slot:
// within ~1e-14 relative of the reference's two-pass value.  A VARZ value that
// falls within rounding distance of a bin edge, or a table overflow, marks the
// pose VMI_FLAG_RECHECK and the host re-evaluates it through the exact
// sort-based path (k_exact.cu), so histograms stay bit-exact.
#include <cstdint>
#include <climits>
#include <type_traits>
#include <cuda_runtime.h>

#include "vmi_device.cuh"
#include "vmi_kernels.h"

namespace vmi {

constexpr unsigned long long kEmpty64 = ~0ull;
constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t slot_of(uint32_t lin, uint32_t cap) {
  return __umulhi(lin * 0x9E3779B1u, cap);
}

// ---- cp.async staging of scan-B records (LDGSTS, L1 bypass) ---------------
#ifndef VMI_UNROLL
#define VMI_UNROLL 4
#endif
#ifndef VMI_STAGES
#ifndef VMI_TMA
#define VMI_STAGES 6  // cp.async ring: 6 records in flight per thread (2 push groups)
#else
#define VMI_STAGES 8  // TMA: two groups of four records in flight per warp
#endif
#endif
#if !defined(VMI_TMA) && defined(VMI_SINGLE_PUSH)
constexpr int kUnroll = VMI_UNROLL;  // main point loop unroll (A/B tunable)
#endif
// Pipeline shape per instantiation.  Single-pass poses: kPG points per queue
// push with an S-record cp.async ring (two push groups in flight).  Multi-pass
// (large grids): shared memory goes to the table instead (more capacity =
// fewer passes), so one point per push and a 4-record ring.
#ifndef VMI_STAGES64
#define VMI_STAGES64 2  // double records: a small ring leaves room for the table (A/B: C1)
#endif
template <bool F32, bool MULTI = false>
__host__ __device__ constexpr int kStages() {
  return MULTI ? 4 : (F32 ? VMI_STAGES : VMI_STAGES64);
}
template <typename Rec>
__device__ __forceinline__ void cp_async_rec(uint32_t dst, const Rec* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  if (sizeof(Rec) == 32)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16),
                 "l"(reinterpret_cast<const char*>(src) + 16)
                 : "memory");
}
// ---- TMA bulk staging (cp.async.bulk + mbarrier) ------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
template <typename Rec>
__device__ __forceinline__ Rec lds_rec(uint32_t a);
template <>
__device__ __forceinline__ float4 lds_rec<float4>(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
template <>
__device__ __forceinline__ double4 lds_rec<double4>(uint32_t a) {
  double4 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.z), "=d"(v.w) : "r"(a + 16) : "memory");
  return v;
}
// VARZ table: keys and counts in shared memory; the per-slot pivot-shifted
// sums (S1, S2) in a per-CTA, L2-resident global array updated with native
// fire-and-forget f64 reductions (RED.ADD.F64) -- a shared-memory f64
// atomicAdd is a CAS loop on sm_100 and was ~30% of the kernel's stalls.
// VARZ slot counts live in shared memory (12-byte slots) for single-pass
// poses, but in the L2 scratch next to the sums (8-byte slots: ~50 % more
// capacity, hence fewer passes) for the multi-pass large-grid mode.  A/B:
// C2 33.4 vs 35.3 ms (global counts slower), C4 314k vs 383k pose-evals/s.
template <bool MULTI>
__host__ __device__ constexpr bool kGlobalCounts() {
#ifdef VMI_GCNT
  return true;
#else
  return MULTI;
#endif
}
__host__ __device__ inline int slot_bytes(int kind, int multi) {
  if (kind != 0) return 4 + 4;
  return (multi ? kGlobalCounts<true>() : kGlobalCounts<false>()) ? 8 : 8 + 4;
}

struct VarzTable {
  unsigned long long* key;  // (lin << 32) | float32 bits of the slot pivot
  uint32_t* cnt;            // shared memory, or (VMI_GCNT) the per-CTA global scratch
  double2* sums;            // global: this CTA's [cap] (S1, S2)
};

__device__ __forceinline__ void flush_varz(const VarzTable& T, uint32_t cap, uint32_t lin, int n,
                                           double K, double a1, double a2, int* overflow) {
  uint32_t s = slot_of(lin, cap);
  const unsigned long long mine =
      ((unsigned long long)lin << 32) | __float_as_uint(__double2float_rn(K));
  unsigned long long w;
  uint32_t probes = 0;
  while (true) {
    w = ((volatile unsigned long long*)T.key)[s];
    if ((uint32_t)(w >> 32) == lin) break;
    if (w == kEmpty64) {
      unsigned long long old = atomicCAS(&T.key[s], kEmpty64, mine);
      if (old == kEmpty64) { w = mine; break; }
      if ((uint32_t)(old >> 32) == lin) { w = old; break; }
    }
    if (++s == cap) s = 0;
    if (++probes >= cap) { *overflow = 1; return; }
  }
  const double kp = (double)__uint_as_float((uint32_t)w);
  const double dl = K - kp;
  const double nd = (double)n;
  atomicAdd(&T.cnt[s], (uint32_t)n);
  atomicAdd(&T.sums[s].x, a1 + nd * dl);
  atomicAdd(&T.sums[s].y, a2 + dl * (2.0 * a1 + nd * dl));
}

__device__ __forceinline__ void flush_count(uint32_t* key, uint32_t* cnt, uint32_t cap,
                                            uint32_t lin, int n, int* overflow) {
  uint32_t s = slot_of(lin, cap);
  uint32_t probes = 0;
  while (true) {
    uint32_t w = ((volatile uint32_t*)key)[s];
    if (w == lin) break;
    if (w == kEmpty32) {
      uint32_t old = atomicCAS(&key[s], kEmpty32, lin);
      if (old == kEmpty32 || old == lin) break;
    }
    if (++s == cap) s = 0;
    if (++probes >= cap) { *overflow = 1; return; }
  }
  atomicAdd(&cnt[s], (uint32_t)n);
}

// Warp-private flush queue: run records pushed by any lane, drained 32 at a
// time by the whole warp so the hash/atomic path always runs converged.
constexpr int kQueueMax = 128;  // >= 32 * kPG (a group's pushes; the pending partial round is flushed first when needed)
#ifndef VMI_SINGLE_PUSH
constexpr bool kPairPush = true;   // one queue push per group of kPG points
#else
constexpr bool kPairPush = false;
#endif
#ifndef VMI_PG
#define VMI_PG 3  // A/B (C2): 3 > 4 (which needs a queue-overrun guard) > 2
#endif
#ifndef VMI_PG64
#define VMI_PG64 1
#endif
template <bool F32, bool MULTI>
__host__ __device__ constexpr int kPGt() {  // points per queue push
  return (MULTI || !kPairPush) ? 1 : (F32 ? VMI_PG : VMI_PG64);
}
template <bool F32, bool MULTI>
__host__ __device__ constexpr int kQueueT() {  // warp queue entries: >= 32*max(kPG, 2), pow2
  return kPGt<F32, MULTI>() == 1 ? 64 : 128;
}
#ifndef VMI_GROUP_UNROLL
#define VMI_GROUP_UNROLL 2
#endif
constexpr int kGroupUnroll = VMI_GROUP_UNROLL;  // entries per warp: a step pushes <= 32*NS, drained at 32

// Shared-memory layout helper (bytes), mirrored by fast_smem_bytes() on the host.
constexpr int kCountLut = 1024;  // COUNT bins precomputed for n < kCountLut

struct FastSmem {
  size_t stage, bars, table, queue, hist, marg, red, rows, cols, misc, lut, total;
};
__host__ __device__ inline FastSmem fast_layout(int kind, int cap, int W, int threads, int f32,
                                                int ns, int multi) {
  FastSmem L;
  size_t off = 0;
  L.stage = off;
  const int stages = multi ? kStages<true, true>() : (f32 ? kStages<true>() : kStages<false>());
  off += (size_t)threads * ns * (f32 ? 16 : 32) * stages;
  L.bars = off;  // two mbarriers per warp (TMA bulk staging)
  off += (size_t)(threads / 32) * 16;
  L.table = off;
  off += (size_t)cap * slot_bytes(kind, multi);
  off = (off + 15) & ~size_t(15);
  L.queue = off;
  const int queue = ns != 1 ? kQueueMax
                    : (multi ? kQueueT<true, true>() : (f32 ? kQueueT<true, false>() : kQueueT<false, false>()));
  off += (size_t)(threads / 32) * queue * (kind == 0 ? (4 + 4 + 8 + 8 + 8) : (4 + 4));
  off = (off + 15) & ~size_t(15);
  L.hist = off; off += (size_t)W * W * 4; off = (off + 15) & ~size_t(15);
  L.marg = off; off += (size_t)W * 4; off = (off + 15) & ~size_t(15);
  L.red = off; off += (size_t)3 * (threads / 32) * 8; off = (off + 15) & ~size_t(15);
  L.rows = off; off += (size_t)W * 8;
  L.cols = off; off += (size_t)W * 8;
  L.misc = off; off += 128;
  L.lut = off; off += kind == 1 ? kCountLut : 0;
  off = (off + 15) & ~size_t(15);
  L.total = off;
  return L;
}

size_t fast_smem_bytes(int kind, int cap, int bins, int threads, int f32, int ns, int multi) {
  return fast_layout(kind, cap, bins + 1, threads, f32, ns, multi).total;
}

int fast_slot_bytes(int kind, int multi) { return slot_bytes(kind, multi); }

__device__ __forceinline__ void st_shared_v4(uint32_t a, uint32_t x, uint32_t y, uint32_t z,
                                             uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}
__device__ __forceinline__ void st_shared_v2(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void st_shared_f64(uint32_t a, double x) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(x) : "memory");
}
// predicated queue-record stores (no divergent branch around them)
__device__ __forceinline__ void st_rec32_if(bool p, uint32_t a, uint32_t l, uint32_t n, double K,
                                            double s1, double s2) {
#ifndef VMI_SEQ_STS128  // 64-bit stores straight from the run registers: no moves into
                         // aligned quads (A/B: -1.5 % vs two st.shared.v4)
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n"
      " @q st.shared.v2.u32 [%1], {%2, %3};\n"
      " @q st.shared.f64 [%1+8], %4;\n"
      " @q st.shared.f64 [%1+16], %5;\n"
      " @q st.shared.f64 [%1+24], %6;\n}" ::"r"((int)p),
      "r"(a), "r"(l), "r"(n), "d"(K), "d"(s1), "d"(s2)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n"
      " @q st.shared.v4.u32 [%1], {%2, %3, %4, %5};\n"
      " @q st.shared.v4.u32 [%1+16], {%6, %7, %8, %9};\n}" ::"r"((int)p),
      "r"(a), "r"(l), "r"(n), "r"(__double2loint(K)), "r"(__double2hiint(K)),
      "r"(__double2loint(s1)), "r"(__double2hiint(s1)), "r"(__double2loint(s2)),
      "r"(__double2hiint(s2))
      : "memory");
}
__device__ __forceinline__ void st_rec8_if(bool p, uint32_t a, uint32_t l, uint32_t n) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.v2.u32 [%1], {%2, %3};\n}" ::"r"(
          (int)p),
      "r"(a), "r"(l), "r"(n)
      : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld_shared_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ int pin_reg(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ uint32_t pin_reg(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ double pin_reg(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}
__device__ __forceinline__ uint32_t dlo(double d) { return (uint32_t)__double2loint(d); }
__device__ __forceinline__ uint32_t dhi(double d) { return (uint32_t)__double2hiint(d); }
__device__ __forceinline__ double mkd(uint32_t lo, uint32_t hi) {
  return __hiloint2double((int)hi, (int)lo);
}

template <int THREADS, int NS, int KIND, bool F32, int MODE, bool MULTI>
__global__ void __launch_bounds__(THREADS, 1)
    k_pose_fast(GridParams g, RefView A, QueryView B, const double* __restrict__ mats, int64_t P,
                int cap, double* __restrict__ mi_out, int32_t* __restrict__ status_out,
                long long* __restrict__ hist_out, long long* __restrict__ total_out,
                FeatureDump dump, double2* __restrict__ gsums, int npass) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = g.bins + 1;
  const FastSmem L = fast_layout(KIND, cap, W, THREADS, F32 ? 1 : 0, NS, MULTI ? 1 : 0);
  constexpr int kPG = kPGt<F32, MULTI>();
  const uint32_t stage_base = (uint32_t)__cvta_generic_to_shared(smem + L.stage);
  uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L.hist);
  uint32_t* marg = reinterpret_cast<uint32_t*>(smem + L.marg);
  double* red = reinterpret_cast<double*>(smem + L.red);
  long long* rows = reinterpret_cast<long long*>(smem + L.rows);
  long long* cols = reinterpret_cast<long long*>(smem + L.cols);
  int* misc = reinterpret_cast<int*>(smem + L.misc);  // [0..5] bounds, [6] bad, [7] overflow, [8] recheck
  long long* h00_s = reinterpret_cast<long long*>(smem + L.misc + 64);
  double* mat_s = reinterpret_cast<double*>(smem + L.red);  // aliases red before the epilogue

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int wid = tid >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const uint32_t ucap = (uint32_t)cap;

  VarzTable VT;
  uint32_t* ckey = nullptr;
  uint32_t* ccnt = nullptr;
  // warp queue: AoS records, VARZ 32 B {lin, n, K, S1, S2}, COUNT 8 B {lin, n}
  constexpr uint32_t kRec = KIND == 0 ? 32u : 8u;
  constexpr int kQueue = NS == 1 ? kQueueT<F32, MULTI>() : kQueueMax;
  const uint32_t qbase = (uint32_t)__cvta_generic_to_shared(smem + L.queue) + wid * kQueue * kRec;
  if (KIND == 0) {
    VT.key = reinterpret_cast<unsigned long long*>(smem + L.table);
    if (kGlobalCounts<MULTI>())  // counts next to the sums in L2 (native RED.ADD.U32)
      VT.cnt = reinterpret_cast<uint32_t*>(gsums + (size_t)gridDim.x * cap) + (size_t)blockIdx.x * cap;
    else
      VT.cnt = reinterpret_cast<uint32_t*>(smem + L.table + (size_t)cap * 8);
    VT.sums = gsums + (size_t)blockIdx.x * cap;
  } else {
    ckey = reinterpret_cast<uint32_t*>(smem + L.table);
    ccnt = reinterpret_cast<uint32_t*>(smem + L.table + (size_t)cap * 4);
  }

#ifdef VMI_TMA
  static_assert(NS == 1, "TMA staging assumes one span per thread");
  using RecT = typename std::conditional<F32, float4, double4>::type;
  constexpr int G = F32 ? 4 : 2;                              // iterations per group
  constexpr uint32_t kChunk = 32u * (uint32_t)sizeof(RecT);  // one warp, one iteration
  const uint32_t wstage = stage_base + (uint32_t)wid * 2u * G * kChunk;
  const uint32_t wbar = (uint32_t)__cvta_generic_to_shared(smem + L.bars) + (uint32_t)wid * 16u;
  const char* wsrc = reinterpret_cast<const char*>(B.pts) + (size_t)wid * kChunk;
  const int full_it = B.span - 1;
  const int ng = (full_it + G - 1) / G;  // groups per pass over the span
  uint32_t gp = 0, gq = 0;               // groups produced / consumed (warp-uniform)
  auto produce = [&]() {
    if (ng == 0) return;
    const int r0 = (int)(gp % (uint32_t)ng) * G;
    const int cnt = min(G, full_it - r0);
    const uint32_t slot = gp & 1u;
    if (lane == 0) {
      fence_proxy_async();  // prior generic reads of this buffer before the async write
      mbar_arrive_expect_tx(wbar + slot * 8u, (uint32_t)cnt * kChunk);
      for (int u = 0; u < cnt; ++u)
        bulk_g2s(wstage + (slot * G + u) * kChunk,
                 wsrc + (size_t)(r0 + u) * (size_t)THREADS * sizeof(RecT), kChunk, wbar + slot * 8u);
    }
    ++gp;
  };
  if (lane == 0) {
    mbar_init(wbar, 1);
    mbar_init(wbar + 8, 1);
    fence_mbar_init();
  }
  __syncwarp();
  produce();
  produce();
#endif

  // The table is cleared once here; afterwards the per-pose table walk resets
  // every slot it reads, so each pose starts from an empty table.
  auto clear_table = [&]() {
    uint4* t4 = reinterpret_cast<uint4*>(smem + L.table);
    const int key_words = KIND == 0 ? cap / 2 : cap / 4;  // uint4s holding keys
    const int all_words = (int)((L.queue - L.table) / 16);
    const uint4 ones = make_uint4(~0u, ~0u, ~0u, ~0u), zero = make_uint4(0u, 0u, 0u, 0u);
    for (int i = tid; i < all_words; i += THREADS) t4[i] = i < key_words ? ones : zero;
    if (KIND == 0)
      for (int i = tid; i < cap; i += THREADS) VT.sums[i] = make_double2(0.0, 0.0);
    if (KIND == 0 && kGlobalCounts<MULTI>())
      for (int i = tid; i < cap; i += THREADS) VT.cnt[i] = 0u;
  };
  clear_table();
  // COUNT features are small integers: their bins (mi.py:72-79) come from a LUT
  uint8_t* count_lut = reinterpret_cast<uint8_t*>(smem + L.lut);
  if (KIND == 1)
    for (int n = tid; n < kCountLut; n += THREADS)
      count_lut[n] = (uint8_t)feature_bin((double)n, g.clamp, g.bins);
  const double bin_scale = (double)g.bins / g.clamp;

  for (int64_t p = blockIdx.x; p < P; p += gridDim.x) {
    for (int i = tid; i < W * W; i += THREADS) hist[i] = 0u;
    for (int i = tid; i < W; i += THREADS) marg[i] = 0u;
    if (tid < 3) { misc[tid] = INT_MAX; misc[3 + tid] = INT_MIN; }
    if (tid >= 6 && tid < 9) misc[tid] = 0;
    if (tid < 12) mat_s[tid] = mats[p * 12 + tid];
    __syncthreads();
    const double m0 = mat_s[0], m1 = mat_s[1], m2 = mat_s[2], m3 = mat_s[3], m4 = mat_s[4],
                 m5 = mat_s[5], m6 = mat_s[6], m7 = mat_s[7], m8 = mat_s[8], t0 = mat_s[9],
                 t1 = mat_s[10], t2 = mat_s[11];
    // Every |q| < 2^30 here (rotation rows bound |R p| by sum|R_jk| * max|p|), so
    // floor(q) fits int32 without a per-point check; the +-2^20 key range is
    // checked exactly on the reduced bounds.  Poses beyond that (translations
    // of ~1e9 voxels) go to the exact path, which reports KEY_RANGE.
    {
      const double lim = 1073741824.0 * g.res;
      const double mx = B.max_abs;
      const bool unsafe =
          fabs(t0 - g.origin[0]) + (fabs(m0) + fabs(m1) + fabs(m2)) * mx >= lim ||
          fabs(t1 - g.origin[1]) + (fabs(m3) + fabs(m4) + fabs(m5)) * mx >= lim ||
          fabs(t2 - g.origin[2]) + (fabs(m6) + fabs(m7) + fabs(m8)) * mx >= lim;
      if (unsafe) {
        if (tid == 0) {
          mi_out[p] = -1e300;
          status_out[p] = 0x100;
          if (total_out) total_out[p] = 0;
        }
        __syncthreads();
        continue;
      }
    }

    // ---- overlap region (voxel.py:298-318) -------------------------------
    int status = 0;
    int rlo[3], rhi[3];
    long long n_region = 0;
    const double bins_d = (double)g.bins;
    bool recheck = false;
    // npass > 1 only when scan B's voxels outgrow the table: pass k aggregates
    // the voxels of hash partition k, so every voxel is complete in one pass.
    if (!MULTI) npass = 1;  // single-pass instantiation: the pass loop folds away
    for (int pass = 0; pass < npass; ++pass) {
      // ---- pass over this thread's span(s) of scan B ------------------------
      // Each thread walks NS spans ("virtual threads" tid + k*THREADS of the
      // span layout) in lock step: NS independent dependency chains per thread.
      constexpr int VTH = THREADS * NS;  // virtual threads = spans per CTA
      int bmin0 = INT_MAX, bmin1 = INT_MAX, bmin2 = INT_MAX;
      int bmax0 = INT_MIN, bmax1 = INT_MIN, bmax2 = INT_MIN;
      uint32_t cur[NS];
      int cn[NS];
      double cK[NS], cs1[NS], cs2[NS];
  #pragma unroll
      for (int k = 0; k < NS; ++k) { cur[k] = kNoVoxel; cn[k] = 0; cK[k] = cs1[k] = cs2[k] = 0.0; }
      uint32_t qh = 0, qt = 0;  // warp-uniform queue head / tail

      auto flush_rec = [&](uint32_t idx) {  // one queued record -> table
        const uint32_t a = qbase + (idx & (kQueue - 1)) * kRec;
        if (KIND == 0) {
          const uint4 r0 = ld_shared_v4(a), r1 = ld_shared_v4(a + 16);
          flush_varz(VT, ucap, r0.x, (int)r0.y, mkd(r0.z, r0.w), mkd(r1.x, r1.y), mkd(r1.z, r1.w),
                     &misc[7]);
        } else {
          const uint2 r0 = ld_shared_v2(a);
          flush_count(ckey, ccnt, ucap, r0.x, (int)r0.y, &misc[7]);
        }
      };
      auto store_rec = [&](uint32_t pos, int k) {
        const uint32_t a = qbase + (pos & (kQueue - 1)) * kRec;
        if (KIND == 0) {
#ifndef VMI_SCALAR_STORES
          st_shared_v4(a, cur[k], (uint32_t)cn[k], dlo(cK[k]), dhi(cK[k]));
          st_shared_v4(a + 16, dlo(cs1[k]), dhi(cs1[k]), dlo(cs2[k]), dhi(cs2[k]));
#else  // scalar stores: no register shuffling into vector quads
          st_shared_v2(a, cur[k], (uint32_t)cn[k]);
          st_shared_f64(a + 8, cK[k]);
          st_shared_f64(a + 16, cs1[k]);
          st_shared_f64(a + 24, cs2[k]);
#endif
        } else {
          st_shared_v2(a, cur[k], (uint32_t)cn[k]);
        }
      };
      // whole warp: enqueue the finished runs, drain 32 at a time (converged)
      auto push = [&](const bool* do_push) {
        unsigned m[NS];
        unsigned any = 0u;
  #pragma unroll
        for (int k = 0; k < NS; ++k) { m[k] = __ballot_sync(0xffffffffu, do_push[k]); any |= m[k]; }
        if (any == 0u) return;
        uint32_t base = qt;
  #pragma unroll
        for (int k = 0; k < NS; ++k) {
          if (do_push[k]) store_rec(base + __popc(m[k] & lt_mask), k);
          base += __popc(m[k]);
        }
        qt = base;
        while (qt - qh >= 32) {
          __syncwarp();
          flush_rec(qh + lane);
          qh += 32;
          __syncwarp();
        }
      };
      // transform, voxel index, bounds, voxel inside A's AABB (pure per point)
#ifdef VMI_PIN_CONSTS
      // opaque copies: kept in registers instead of re-loaded from the
      // constant bank on every point
      const int am0 = pin_reg(A.amin[0]), am1 = pin_reg(A.amin[1]), am2 = pin_reg(A.amin[2]);
      const uint32_t ex0 = pin_reg(A.ext[0]), ex1 = pin_reg(A.ext[1]), ex2 = pin_reg(A.ext[2]);
#else
      const int am0 = A.amin[0], am1 = A.amin[1], am2 = A.amin[2];
      const uint32_t ex0 = A.ext[0], ex1 = A.ext[1], ex2 = A.ext[2];
#endif
      // floor(q) - amin straight from DADD.RM against 1.5*2^52 - amin (an
      // integer in [2^52, 2^53), so the sum rounds down to kc + floor(q) and
      // its low word is floor(q) - amin); bounds are tracked relative to amin
      // (opaque copies: otherwise they are recomputed from amin on every step)
      const double kc0 = pin_reg(6755399441055744.0 - (double)am0);
      const double kc1 = pin_reg(6755399441055744.0 - (double)am1);
      const double kc2 = pin_reg(6755399441055744.0 - (double)am2);
      auto locate = [&](double x, double y, double z, bool valid, uint32_t& lin, double& Z) {
        const double X = xform_row(x, y, z, m0, m1, m2, t0);
        const double Y = xform_row(x, y, z, m3, m4, m5, t1);
        Z = xform_row(x, y, z, m6, m7, m8, t2);
        const int ix = __double2loint(__dadd_rd(grid_q<MODE>(X, g.origin[0], g.res, g.inv_res), kc0));
        const int iy = __double2loint(__dadd_rd(grid_q<MODE>(Y, g.origin[1], g.res, g.inv_res), kc1));
        const int iz = __double2loint(__dadd_rd(grid_q<MODE>(Z, g.origin[2], g.res, g.inv_res), kc2));
        lin = kNoVoxel;
        if (valid) {
          bmin0 = min(bmin0, ix); bmax0 = max(bmax0, ix);
          bmin1 = min(bmin1, iy); bmax1 = max(bmax1, iy);
          bmin2 = min(bmin2, iz); bmax2 = max(bmax2, iz);
          const uint32_t rx = (uint32_t)ix;
          const uint32_t ry = (uint32_t)iy;
          const uint32_t rz = (uint32_t)iz;
          const bool inside = (rx < ex0) & (ry < ex1) & (rz < ex2);
          lin = inside ? (rx * ex1 + ry) * ex2 + rz : kNoVoxel;
        if (npass > 1 && lin != kNoVoxel && __umulhi(lin * 0x85EBCA6Bu, (uint32_t)npass) != (uint32_t)pass)
          lin = kNoVoxel;  // another pass's partition
        }
      };
      // run aggregation for one point of every stream
      auto advance = [&](const uint32_t* lin, const double* Z) {
        bool ends[NS], pushes[NS];
  #pragma unroll
        for (int k = 0; k < NS; ++k) {
          ends[k] = lin[k] != cur[k];
          pushes[k] = ends[k] && cur[k] != kNoVoxel;
        }
        push(pushes);
  #pragma unroll
        for (int k = 0; k < NS; ++k) {
          if (ends[k]) {
            cur[k] = lin[k]; cn[k] = 1; cK[k] = Z[k]; cs1[k] = 0.0; cs2[k] = 0.0;
          } else {
            const double d = Z[k] - cK[k];
            ++cn[k]; cs1[k] += d; cs2[k] = fma(d, d, cs2[k]);
          }
        }
      };

      using Rec = typename std::conditional<F32, float4, double4>::type;
      const Rec* pts = reinterpret_cast<const Rec*>(B.pts) + tid;
      const int full = B.span - 1;  // iterations every span owns
#ifndef VMI_TMA
      // Scan-B records are staged through shared memory with cp.async: each
      // virtual thread streams its own span kStages-1 records ahead into a
      // private ring slot (no cross-thread dependency, so no barrier), then reads
      // the record back with one LDS when it is its turn.  Keeping the prefetch
      // out of the register file stops the compiler from hoisting conversions of
      // in-flight data (which turned a register prefetch into stalls).
      constexpr int S = kStages<F32, MULTI>();
      const uint32_t my_stage = stage_base + (uint32_t)tid * (uint32_t)sizeof(Rec);
      constexpr uint32_t kStageStride = (uint32_t)(VTH * sizeof(Rec));
      constexpr uint32_t kStreamOff = (uint32_t)(THREADS * sizeof(Rec));
      auto issue = [&](int r) {
        if (r < full) {
  #pragma unroll
          for (int k = 0; k < NS; ++k)
            cp_async_rec<Rec>(my_stage + (uint32_t)(r % S) * kStageStride + k * kStreamOff,
                              pts + r * VTH + k * THREADS);
        }
        cp_async_commit();
      };
#if defined(VMI_SINGLE_PUSH)
  #pragma unroll
      for (int r = 0; r < S - 1; ++r) issue(r);
#endif
      // body for record r held in ring slot `slot` (a compile-time constant in
      // the unrolled main loop, so every shared address is base + immediate)
      auto body = [&](int r, int slot) {
        issue(r + S - 1);
        cp_async_wait<S - 1>();
        uint32_t lin[NS];
        double Z[NS];
  #pragma unroll
        for (int k = 0; k < NS; ++k) {
          const Rec v = lds_rec<Rec>(my_stage + (uint32_t)slot * kStageStride + k * kStreamOff);
          locate((double)v.x, (double)v.y, (double)v.z, true, lin[k], Z[k]);
        }
        advance(lin, Z);
      };
#if !defined(VMI_SINGLE_PUSH)
      // two points per step: both located first (independent fp64 chains),
      // then both run updates, then ONE warp-wide queue push for the up to
      // two runs each lane finished
      auto store_state = [&](uint32_t pos, uint32_t l, uint32_t n, double K, double a1, double a2) {
        const uint32_t a = qbase + (pos & (kQueue - 1)) * kRec;
        if (KIND == 0) {
#ifdef VMI_STS64
          st_shared_v2(a, l, n);
          st_shared_f64(a + 8, K);
          st_shared_f64(a + 16, a1);
          st_shared_f64(a + 24, a2);
#else
          st_shared_v4(a, l, n, dlo(K), dhi(K));
          st_shared_v4(a + 16, dlo(a1), dhi(a1), dlo(a2), dhi(a2));
#endif
        } else {
          st_shared_v2(a, l, n);
        }
      };
      auto step1 = [&](uint32_t lin, double Z, bool& pend, uint32_t& pl, uint32_t& pn, double& pK,
                       double& p1, double& p2) {
        const bool e = lin != cur[0];
        pend = e && cur[0] != kNoVoxel;
        pl = cur[0]; pn = (uint32_t)cn[0]; pK = cK[0]; p1 = cs1[0]; p2 = cs2[0];
#ifdef VMI_BRANCHLESS_STEP
        // reset folds into the update: on a new run cK = Z makes d = 0 and the
        // 0/1 factor clears the sums (DP pipe has headroom; no branches/moves)
        cur[0] = lin;  // equal to the old value when the run continues
        cK[0] = e ? Z : cK[0];
        cn[0] = e ? 1 : cn[0] + 1;
        const double keep = e ? 0.0 : 1.0;
        const double d = Z - cK[0];
        cs1[0] = fma(cs1[0], keep, d);
        cs2[0] = fma(d, d, cs2[0] * keep);
#else
        if (e) {
          cur[0] = lin; cn[0] = 1; cK[0] = Z; cs1[0] = 0.0; cs2[0] = 0.0;
        } else {
          const double d = Z - cK[0];
          ++cn[0]; cs1[0] += d; cs2[0] = fma(d, d, cs2[0]);
        }
#endif
      };
      // Group staging: rows are issued kPG at a time as one commit group from a
      // running pointer.  The span layout is padded with kStagePadRows rows, so
      // rows past the span are issued unconditionally (and never read back).
      static_assert(S % kPG == 0, "ring holds whole groups");
      static_assert(S <= kStagePadRows, "span layout padding covers the ring");
      constexpr int kGroups = S / kPG;  // commit groups in flight
      constexpr size_t kRowBytes = (size_t)VTH * sizeof(Rec);
      const char* src = reinterpret_cast<const char*>(pts);
      auto issue_group = [&](int slot0) {
#pragma unroll
        for (int u = 0; u < kPG; ++u)
          cp_async_rec<Rec>(my_stage + (uint32_t)(slot0 + u) * kStageStride,
                            reinterpret_cast<const Rec*>(src + u * kRowBytes));
        src += kPG * kRowBytes;
        cp_async_commit();
      };
      auto group_body = [&](int r) {
        cp_async_wait<kGroups - 1>();  // rows r .. r+kPG-1 have landed
        uint32_t l[kPG];
        double Z[kPG];
#pragma unroll
        for (int u = 0; u < kPG; ++u) {
          const Rec v = lds_rec<Rec>(my_stage + (uint32_t)((r + u) % S) * kStageStride);
          locate((double)v.x, (double)v.y, (double)v.z, true, l[u], Z[u]);
        }
        issue_group(r % S);  // refill the slots just consumed with rows r+S ..
#ifndef VMI_BATCH_PUSH  // (batched ballots + branchy stores: A/B measured 0.8% slower)
        // per point: ballot, predicated store of the finished run straight from
        // the run registers, then the run update (no pending copies, no branches).
        // A group adds <= 32*kPG records to < 32 unflushed ones.
        static_assert(32 * kPG + 31 <= kQueue, "a push group must fit the run queue");
#pragma unroll
        for (int u = 0; u < kPG; ++u) {
          const bool e = l[u] != cur[0];
          const bool pdu = e && cur[0] != kNoVoxel;
          const unsigned mu = __ballot_sync(0xffffffffu, pdu);
          const uint32_t a = qbase + ((qt + __popc(mu & lt_mask)) & (kQueue - 1)) * kRec;
          if (KIND == 0)
            st_rec32_if(pdu, a, cur[0], (uint32_t)cn[0], cK[0], cs1[0], cs2[0]);
          else
            st_rec8_if(pdu, a, cur[0], (uint32_t)cn[0]);
          qt += __popc(mu);
#ifdef VMI_SEQ_BRANCHLESS  // experiment: fewer instructions, longer dependency chain (A/B: +0.6 % time)
          // reset folded into the update: a new run takes cK = Z, so d = 0 and
          // the 0/1 factor clears the sums (fma(x, 1, d) == x + d exactly)
          cur[0] = l[u];
          cK[0] = e ? Z[u] : cK[0];
          const double keep = e ? 0.0 : 1.0;
          const double d = Z[u] - cK[0];
          cn[0] = e ? 1 : cn[0] + 1;
          cs1[0] = fma(cs1[0], keep, d);
          cs2[0] = fma(d, d, cs2[0] * keep);
#else
          if (e) {
            cur[0] = l[u]; cn[0] = 1; cK[0] = Z[u]; cs1[0] = 0.0; cs2[0] = 0.0;
          } else {
            const double d = Z[u] - cK[0];
            ++cn[0]; cs1[0] += d; cs2[0] = fma(d, d, cs2[0]);
          }
#endif
        }
        while (qt - qh >= 32) {
          __syncwarp();
          flush_rec(qh + lane);
          qh += 32;
          __syncwarp();
        }
#else
        bool pd[kPG];
        uint32_t pl[kPG], pn[kPG];
        double pK[kPG], p1[kPG], p2[kPG];
#pragma unroll
        for (int u = 0; u < kPG; ++u) step1(l[u], Z[u], pd[u], pl[u], pn[u], pK[u], p1[u], p2[u]);
        unsigned m[kPG];
        unsigned any = 0u;
#pragma unroll
        for (int u = 0; u < kPG; ++u) { m[u] = __ballot_sync(0xffffffffu, pd[u]); any |= m[u]; }
        if (any != 0u) {
          // A group can push up to 32*kPG records on top of < 32 unflushed ones:
          // when that would overrun the ring, flush the partial round first.
          uint32_t n = 0;
#pragma unroll
          for (int u = 0; u < kPG; ++u) n += __popc(m[u]);
#ifndef VMI_NO_QUEUE_GUARD  // A/B timing experiment only (unsafe for dense pushes)
          if (32 * kPG + 31 > kQueue && qt - qh + n > (uint32_t)kQueue) {
            __syncwarp();
            if ((uint32_t)lane < qt - qh) flush_rec(qh + lane);
            qh = qt;
            __syncwarp();
          }
#endif
          uint32_t base = qt;
#pragma unroll
          for (int u = 0; u < kPG; ++u) {
            if (pd[u]) store_state(base + __popc(m[u] & lt_mask), pl[u], pn[u], pK[u], p1[u], p2[u]);
            base += __popc(m[u]);
          }
          qt = base;
          while (qt - qh >= 32) {
            __syncwarp();
            flush_rec(qh + lane);
            qh += 32;
            __syncwarp();
          }
        }
#endif
      };
      static_assert(S >= kPG, "ring must hold a full group");
#pragma unroll
      for (int gi = 0; gi < kGroups; ++gi) issue_group(gi * kPG);  // rows 0 .. S-1 in flight
      int rr = 0;
#pragma unroll kGroupUnroll
      for (; rr + kPG <= full; rr += kPG) group_body(rr);
      for (; rr < full; ++rr) {  // leftover (< kPG) points
        cp_async_wait<0>();
        uint32_t lin[NS];
        double Zs[NS];
        const Rec v = lds_rec<Rec>(my_stage + (uint32_t)(rr % S) * kStageStride);
        locate((double)v.x, (double)v.y, (double)v.z, true, lin[0], Zs[0]);
        advance(lin, Zs);
      }
#elif !defined(VMI_STATIC_SLOT)
      #pragma unroll kUnroll
      for (int r = 0; r < full; ++r) body(r, r % S);
#else
      int r0 = 0;
      for (; r0 + S <= full; r0 += S) {
  #pragma unroll
        for (int u = 0; u < S; ++u) body(r0 + u, u);
      }
      for (int r = r0; r < full; ++r) body(r, r % S);
#endif
      cp_async_wait<0>();
#else
      // Scan-B records are staged through shared memory by TMA bulk copies:
      // in the span layout a warp's 32 records of one iteration are one
      // contiguous 32*sizeof(Rec)-byte chunk, so lane 0 streams groups of G
      // iterations (two groups in flight, one mbarrier each) and every lane
      // reads its record back with one LDS.  The stream runs continuously
      // across passes and poses (scan B is the same for every pose).
      for (int q = 0; q < ng; ++q) {
        const uint32_t slot = gq & 1u;
        while (!mbar_try_wait(wbar + slot * 8u, (gq >> 1) & 1u)) {
        }
        const int r0 = q * G;
#pragma unroll
        for (int u = 0; u < G; ++u) {
          if (r0 + u < full) {  // warp-uniform
            uint32_t lin[NS];
            double Z[NS];
            const Rec v = lds_rec<Rec>(wstage + (slot * G + u) * kChunk + (uint32_t)lane * sizeof(Rec));
            locate((double)v.x, (double)v.y, (double)v.z, true, lin[0], Z[0]);
            advance(lin, Z);
          }
        }
        __syncwarp();  // every lane has read this buffer: it may be refilled
        ++gq;
        produce();
      }
#endif
      {  // the ragged last iteration
        uint32_t lin[NS];
        double Z[NS];
  #pragma unroll
        for (int k = 0; k < NS; ++k) {
          const Rec v = pts[full * VTH + k * THREADS];
          const bool has_last = span_of_thread(tid + k * THREADS, VTH) < B.rem;
          locate((double)v.x, (double)v.y, (double)v.z, has_last, lin[k], Z[k]);
        }
        advance(lin, Z);
      }
      {
        bool fin[NS];
  #pragma unroll
        for (int k = 0; k < NS; ++k) fin[k] = cur[k] != kNoVoxel;
        push(fin);
      }
      while (qh != qt) {  // drain the tail (partial round)
        __syncwarp();
        if ((uint32_t)lane < qt - qh) flush_rec(qh + lane);
        qh = (qt - qh > 32u) ? qh + 32 : qt;
        __syncwarp();
      }
      if (pass == 0) {
        // ---- reduce bounds / key-range flag ----------------------------------
        bmin0 = __reduce_min_sync(0xffffffffu, bmin0);
        bmin1 = __reduce_min_sync(0xffffffffu, bmin1);
        bmin2 = __reduce_min_sync(0xffffffffu, bmin2);
        bmax0 = __reduce_max_sync(0xffffffffu, bmax0);
        bmax1 = __reduce_max_sync(0xffffffffu, bmax1);
        bmax2 = __reduce_max_sync(0xffffffffu, bmax2);
        if (lane == 0 && bmin0 != INT_MAX) {  // relative to amin (locate); a warp may have no points
          atomicMin(&misc[0], bmin0 + am0); atomicMin(&misc[1], bmin1 + am1);
          atomicMin(&misc[2], bmin2 + am2);
          atomicMax(&misc[3], bmax0 + am0); atomicMax(&misc[4], bmax1 + am1);
          atomicMax(&misc[5], bmax2 + am2);
        }
        __syncthreads();
        // voxel.py:200-206: any index outside [-2^20, 2^20-1] -> OutOfBoundsError
        if (tid == 0 && (misc[0] < kKeyMin || misc[1] < kKeyMin || misc[2] < kKeyMin ||
                         misc[3] > kKeyMax || misc[4] > kKeyMax || misc[5] > kKeyMax))
          misc[6] = 1;
        __syncthreads();

        if (misc[6]) {
          status = 2;  // KEY_RANGE
        } else if (A.empty) {
          status = 1;
        } else {
          n_region = 1;
          for (int j = 0; j < 3; ++j) {
            rlo[j] = max(A.amin[j], misc[j]);
            rhi[j] = min(A.amax[j], misc[3 + j]);
            if (rlo[j] > rhi[j]) status = 1;
            n_region *= (long long)(rhi[j] - rlo[j] + 1);
          }
        }
        if (status != 0) break;  // block-uniform
      } else {
        __syncthreads();  // every flush of this pass has landed
      }
      // ---- enumerate B voxels (all inside A's AABB, hence in the region) ---
      // Every slot read is reset for the next pose.  VARZ bins use
      // var * (B / clamp): our VARZ is itself within ~1e-14 of the reference's,
      // and any value within rounding distance of a bin edge marks the pose for
      // the exact path.
      auto finish_slot = [&](int s, uint32_t lin, int ba, double2 sum) {
        int bb;
        double dump_feat = 0.0;
        if (KIND == 0) {
          const double nd = (double)(kGlobalCounts<MULTI>() ? __ldcg(&VT.cnt[s]) : VT.cnt[s]);
          const double S1 = sum.x, S2 = sum.y;
          VT.key[s] = kEmpty64; VT.cnt[s] = 0u;
          VT.sums[s] = make_double2(0.0, 0.0);
          const double rn = __drcp_rn(nd);
          const double c1 = S1 * S1 * rn;
          const double ssd = S2 - c1;
          const double feat = (ssd > 0.0 ? ssd : 0.0) * rn;
          const double x = feat * bin_scale;
          const double k = rint(x);
          if (k >= 1.0 && k <= bins_d - 1.0) {
            const double tol = ((nd + 8.0) * 4.440892098500626e-16 * (S2 + c1) * rn +
                                feat * 9.094947017729282e-13) * bin_scale + 1e-300;
            if (fabs(x - k) <= tol) recheck = true;
          }
          const double f = floor(x);
          bb = 1 + (f >= bins_d - 1.0 ? g.bins - 1 : (int)f);
          dump_feat = feat;
        } else {
          const uint32_t n = ccnt[s];
          ckey[s] = kEmpty32; ccnt[s] = 0u;
          bb = n < (uint32_t)kCountLut ? (int)count_lut[n] : feature_bin((double)n, g.clamp, g.bins);
          dump_feat = (double)n;
        }
        atomicAdd(&hist[ba * W + bb], 1u);
        if (dump.keys) {  // debug export (vmi_fast_features): lin -> packed key, feature
          const int j = atomicAdd(dump.n, 1);
          if (j < dump.cap) {
            const uint32_t rz = lin % A.ext[2], rxy = lin / A.ext[2];
            const uint32_t ry = rxy % A.ext[1], rx = rxy / A.ext[1];
            const unsigned long long off = 1ull << 20;
            dump.keys[j] = ((unsigned long long)(long long)((int)rx + A.amin[0]) + off) << 42 |
                           ((unsigned long long)(long long)((int)ry + A.amin[1]) + off) << 21 |
                           ((unsigned long long)(long long)((int)rz + A.amin[2]) + off);
            dump.values[j] = dump_feat;
          }
        }
      };
      if constexpr (KIND == 0) {
        // VARZ: each warp owns a contiguous slice of the table; it compacts the
        // occupied slots (ballot) into a ring in its share of the (idle)
        // staging buffer, then takes them four per lane, so a lane's A-grid and
        // L2 sums loads are in flight together and only occupied slots cost a
        // load round (the whole CTA is in this phase at once: nothing else
        // hides the latency).  A/B: -3 % kernel time at C2.
        constexpr int NW = THREADS / 32;
        constexpr int kWR = 256;  // ring entries; kWU ballots per scan step / entries per lane
        constexpr int kWU = kWR / 64;
#ifndef VMI_TMA
        static_assert(kStages<F32, MULTI>() * NS * (F32 ? 16 : 32) * 32 >= kWR * 4,
                      "walk ring fits the warp's staging slice");
        uint32_t* wl = reinterpret_cast<uint32_t*>(
            smem + L.stage + (size_t)wid * 32 * NS * (F32 ? 16 : 32) * kStages<F32, MULTI>());
#else
        static_assert(kQueue * kRec >= kWR * 4, "walk ring fits the run queue");
        uint32_t* wl = reinterpret_cast<uint32_t*>(smem + L.queue + (size_t)wid * kQueue * kRec);
#endif
        const int per = ((cap + NW - 1) / NW + 31) & ~31;
        const int se = min(cap, wid * per + per);
        int scan = wid * per;
        uint32_t wh = 0, wt = 0;  // ring head / tail (warp-uniform)
        while (scan < se || wt != wh) {  // warp-uniform
          while (scan < se && wt - wh < (uint32_t)(32 * kWU)) {
            bool occ[kWU];
            unsigned m[kWU];
#pragma unroll
            for (int u = 0; u < kWU; ++u) {
              const int s = scan + u * 32 + lane;
              occ[u] = s < se && VT.key[s] != kEmpty64;
              m[u] = __ballot_sync(0xffffffffu, occ[u]);
            }
#pragma unroll
            for (int u = 0; u < kWU; ++u) {
              if (occ[u]) wl[(wt + __popc(m[u] & lt_mask)) & (kWR - 1)] = (uint32_t)(scan + u * 32 + lane);
              wt += __popc(m[u]);
            }
            scan += 32 * kWU;
          }
          __syncwarp();
          const uint32_t take = min(wt - wh, (uint32_t)(32 * kWU));
          int sl[kWU];
          uint32_t lin[kWU];
          int ba[kWU];
          double2 sum[kWU];
#pragma unroll
          for (int u = 0; u < kWU; ++u) {
            const uint32_t i = (uint32_t)(u * 32 + lane);
            sl[u] = i < take ? (int)wl[(wh + i) & (kWR - 1)] : -1;
            lin[u] = sl[u] >= 0 ? (uint32_t)(VT.key[sl[u]] >> 32) : kNoVoxel;
            ba[u] = lin[u] != kNoVoxel ? (int)__ldg(&A.grid[lin[u]]) : 0;
            // L2 copy (the reductions happen in L2; never trust a stale L1 line)
            sum[u] = lin[u] != kNoVoxel ? __ldcg(&VT.sums[sl[u]]) : make_double2(0.0, 0.0);
          }
          wh += take;
          __syncwarp();  // entries read: the ring may be refilled
#pragma unroll
          for (int u = 0; u < kWU; ++u)
            if (lin[u] != kNoVoxel) finish_slot(sl[u], lin[u], ba[u], sum[u]);
        }
      } else {
        // COUNT: four slots per thread per step, four A-grid loads in flight
        // (no L2 sums to fetch: compaction measured slower here)
        for (int s0 = tid; s0 < cap; s0 += 4 * THREADS) {
          uint32_t lin[4];
          int ba[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int s = s0 + u * THREADS;
            lin[u] = kNoVoxel;
            if (s < cap) {
              const uint32_t w = ckey[s];
              if (w != kEmpty32) lin[u] = w;
            }
            ba[u] = lin[u] != kNoVoxel ? (int)__ldg(&A.grid[lin[u]]) : 0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (lin[u] != kNoVoxel) finish_slot(s0 + u * THREADS, lin[u], ba[u], make_double2(0.0, 0.0));
        }
      }
      __syncthreads();  // walk done (slots reset) before the next pass refills
    }
    if (status != 0) {
      if (tid == 0) {
        mi_out[p] = -1e300;
        status_out[p] = status;
        if (total_out) total_out[p] = 0;
      }
      if (hist_out)
        for (int i = tid; i < W * W; i += THREADS) hist_out[p * W * W + i] = 0;
      clear_table();  // the walk below (which resets slots) is skipped
      __syncthreads();
      continue;
    }
    if (recheck) misc[8] = 1;

    // ---- A marginal over the region --------------------------------------
#ifdef VMI_TIMING_SKIP_MARG  // timing experiment only (wrong marginals)
    const bool cover_all = true;
#else
    const bool cover_all = rlo[0] == A.amin[0] && rlo[1] == A.amin[1] && rlo[2] == A.amin[2] &&
                      rhi[0] == A.amax[0] && rhi[1] == A.amax[1] && rhi[2] == A.amax[2];
#endif
    if (cover_all) {
      for (int i = tid; i < W; i += THREADS) marg[i] = A.bin_total[i];
    } else {
      const int lo0 = rlo[0] - A.amin[0], lo1 = rlo[1] - A.amin[1], lo2 = rlo[2] - A.amin[2];
      const int hi0 = rhi[0] - A.amin[0], hi1 = rhi[1] - A.amin[1], hi2 = rhi[2] - A.amin[2];
      for (int j0 = wid * 32; j0 < A.n_avox; j0 += 2 * THREADS) {
        int4 v[2];
        bool in[2];
        int bin[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int j = j0 + u * THREADS + lane;
          v[u] = j < A.n_avox ? __ldg(&A.avox[j]) : make_int4(-1, -1, -1, -1);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          bin[u] = v[u].w;
          in[u] = bin[u] >= 0 && v[u].x >= lo0 && v[u].x <= hi0 && v[u].y >= lo1 &&
                  v[u].y <= hi1 && v[u].z >= lo2 && v[u].z <= hi2;
          const unsigned grp =
              __match_any_sync(0xffffffffu, bin[u]) & __ballot_sync(0xffffffffu, in[u]);
          if (in[u] && lane == __ffs(grp) - 1) atomicAdd(&marg[bin[u]], (uint32_t)__popc(grp));
        }
      }
    }
    __syncthreads();

    // ---- analytic phi cells + MI (fused K2) -------------------------------
#ifdef VMI_TIMING_SKIP_FINAL  // timing experiment only (no MI)
    MIOut r{};
#else
    MIOut r = finalize_mi<THREADS>(hist, marg, W, n_region, g.include_phi, red, rows, cols, h00_s);
#endif
    const bool flag = misc[7] || misc[8];
    if (tid == 0) {
      mi_out[p] = r.status == 0 ? r.mi : -1e300;
      status_out[p] = r.status | (flag ? 0x100 : 0);
      if (total_out) total_out[p] = n_region;
    }
    if (hist_out) {
      for (int i = tid; i < W * W; i += THREADS)
        hist_out[p * W * W + i] = i == 0 ? r.h00 : (long long)hist[i];
    }
    __syncthreads();
  }
#ifdef VMI_TMA
  // retire the two groups still in flight (no bulk copy may outlive the CTA)
  for (int i = 0; i < 2 && ng > 0; ++i) {
    while (!mbar_try_wait(wbar + (gq & 1u) * 8u, (gq >> 1) & 1u)) {
    }
    ++gq;
  }
#endif
}

template <int THREADS, int NS, int KIND, bool F32, int MODE, bool MULTI>
static cudaError_t launch_fast_t(const FastLaunch& fl, cudaStream_t st) {
  auto k = k_pose_fast<THREADS, NS, KIND, F32, MODE, MULTI>;
  size_t smem = fast_smem_bytes(KIND, fl.cap, fl.g.bins, THREADS, F32 ? 1 : 0, NS, MULTI ? 1 : 0);
  // The opt-in is set to the device maximum, never to this launch's size:
  // contexts on other host threads launch the same instantiation with other
  // table sizes, and a smaller per-launch value could land between another
  // thread's attribute call and its launch.
  static const int optin = [k] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k) == cudaSuccess) v -= (int)fa.sharedSizeBytes;
    return v;
  }();
  if ((int)smem > optin) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  if (e != cudaSuccess) return e;
  k<<<fl.grid, THREADS, smem, st>>>(fl.g, fl.A, fl.B, fl.mats, fl.P, fl.cap, fl.mi, fl.status,
                                    fl.hist, fl.total, fl.dump, fl.sums, fl.npass);
  return cudaGetLastError();
}

template <int T, int NS, int KIND, bool F32, bool MULTI>
static cudaError_t launch_grid(const FastLaunch& fl, cudaStream_t st) {
  switch (fl.g.mode) {
    case kGridUnit: return launch_fast_t<T, NS, KIND, F32, kGridUnit, MULTI>(fl, st);
    case kGridPow2: return launch_fast_t<T, NS, KIND, F32, kGridPow2, MULTI>(fl, st);
    default: return launch_fast_t<T, NS, KIND, F32, kGridGeneral, MULTI>(fl, st);
  }
}

// The multi-pass loop costs ~8% even at npass == 1 (measured), so single- and
// multi-pass are separate instantiations.
template <int T, int NS, int KIND, bool F32>
static cudaError_t launch_mode(const FastLaunch& fl, cudaStream_t st) {
  return fl.npass > 1 ? launch_grid<T, NS, KIND, F32, true>(fl, st)
                      : launch_grid<T, NS, KIND, F32, false>(fl, st);
}

template <int T, int NS>
static cudaError_t launch_threads(const FastLaunch& fl, cudaStream_t st) {
  const bool f32 = fl.B.is_f32 != 0;
  if (fl.g.kind == 0)
    return f32 ? launch_mode<T, NS, 0, true>(fl, st) : launch_mode<T, NS, 0, false>(fl, st);
  return f32 ? launch_mode<T, NS, 1, true>(fl, st) : launch_mode<T, NS, 1, false>(fl, st);
}

// NS = 2 (two spans per thread at 256 threads) compiles and is exact, but was
// measured slower on B200 (IPC 1.5 with 8 warps/SM vs 2.2 with 16): only the
// one-span-per-thread configuration is instantiated.
cudaError_t launch_fast(const FastLaunch& fl, cudaStream_t st) {
  if (fl.B.threads != kFastThreads || fl.streams != 1) return cudaErrorInvalidValue;
  return launch_threads<kFastThreads, 1>(fl, st);
}

}  // namespace vmi
