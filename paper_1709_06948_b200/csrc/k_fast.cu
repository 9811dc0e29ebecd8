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
// that is the z of the voxel's lower face (|z - K| < resolution): within
// ~1e-12 relative of the reference's two-pass value.  A VARZ value that
// falls within rounding distance of a bin edge, or a table overflow, marks the
// pose VMI_FLAG_RECHECK and the host re-evaluates it through the exact
// sort-based path (k_exact.cu), so histograms stay bit-exact.
#include <cstdint>
#include <climits>
#include <cstdio>
#include <type_traits>
#include <cuda_runtime.h>

#include "vmi_device.cuh"
#include "vmi_kernels.h"

namespace vmi {

constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t slot_of(uint32_t lin, uint32_t cap) {
  return __umulhi(lin * 0x9E3779B1u, cap);
}

// ---- cp.async staging of scan-B records (LDGSTS, L1 bypass) ---------------
// Pipeline shape per instantiation.  Single-pass poses: kPG points per queue
// push with an S-record cp.async ring (two push groups in flight).  Multi-pass
// (large grids): shared memory goes to the table instead (more capacity =
// fewer passes), so one point per push and a 4-record ring.
// VARZ walk: compaction ring entries (loads in flight per lane = ring / 64).
// A/B (round 1): single-pass C2 512 -> 28.87 ms, 256 -> 28.97, 128 -> 29.34; multi-layout
// C4 128 -> 87.3 ms, 256 -> 91.9, 512 -> 97.2.
#ifndef VMI_WALK_RING
#define VMI_WALK_RING 256  // round 2 A/B (C2): 256 -> 27.80 ms, 512 -> 28.56 (was best in round 1)
#endif
#ifndef VMI_WALK_RING_M
#define VMI_WALK_RING_M 128
#endif
#ifndef VMI_MAT_PREFETCH  // A/B switch: pose matrices loaded one pose ahead
#define VMI_MAT_PREFETCH 1
#endif
// VARZ sums are taken of s_z = the z row's FMA chain before + t_z (= Z - t_z
// up to one rounding of Z), not of z relative to the voxel's lower face: no
// per-point pivot arithmetic.  The per-point offset r (|r| <= 2^-53 |Z|) moves
// a voxel's variance by at most res |r|max + r^2 (var_shift), and the sums'
// own rounding is bounded through S2 + S1^2/n whatever the pivot.
// A/B (r02): C2 26.56 -> 26.04 ms, C4 32.98 -> 32.30, C1 1.68 -> 1.665
#ifndef VMI_HULL_SPLIT  // the point loop compiled twice: with / without per-point bounds
#define VMI_HULL_SPLIT 1
#endif
#ifndef VMI_PROBE4  // VARZ / COUNT collisions: linear probing four slots per LDS.128
#define VMI_PROBE4 1
#endif
#ifndef VMI_OCC_BFREE
#define VMI_OCC_BFREE 1
#endif
#ifndef VMI_OCC_BUCKET  // occupancy kind: 4-slot buckets (see flush_rec)
#define VMI_OCC_BUCKET 1
#endif
#ifndef VMI_PIN_CONST  // general resolutions: AABB extents / 1/res in registers in the point loop
#define VMI_PIN_CONST 1
#endif
#ifndef VMI_REC_V2  // the run record's two sums in one 16-byte store
#define VMI_REC_V2 1
#endif
#ifndef VMI_PIVOT_SZ
#define VMI_PIVOT_SZ 1
#endif
#ifndef VMI_NEAR_FIX  // 0: teeth check of the near-integer test only (wrong floors)
#define VMI_NEAR_FIX 1
#endif
#ifndef VMI_STAGES
#define VMI_STAGES 6  // cp.async ring: 6 records in flight per thread (2 push groups)
#endif
// multi-pass layout: ring depth / points per push.  A/B (C4, 1 point per
// push): 2 stages 80.4 ms, 3 stages 90.2, 4 stages 87.7; 2 points per push
// (4 stages) 107.3, 3 points (6 stages) 109.1.
#ifndef VMI_STAGESM
#define VMI_STAGESM 2
#endif
#ifndef VMI_PGM
#define VMI_PGM 1
#endif
#ifndef VMI_STAGES64
#define VMI_STAGES64 2  // double records: a small ring leaves room for the table (A/B: C1)
#endif
// occupancy kind (4-byte keys, no counts / sums): a 3-deep ring (one push group
// in flight) -- the shared memory goes to a bigger key table (fewer probes).
// A/B (C4): 3 stages 45.8 ms, 6 stages 49.3; C2 (VARZ) keeps 6: 27.8 vs 28.2.
#ifndef VMI_STAGES_OCC
#define VMI_STAGES_OCC 3
#endif
// pre-rotated double4 records (ROT): a 3-deep ring of 32-byte records takes
// the shared memory of the float4 path's 6-deep one
#ifndef VMI_STAGES_ROT
#define VMI_STAGES_ROT 3
#endif
template <bool F32, bool MULTI = false, int KIND = 0, bool ROT = false>
__host__ __device__ constexpr int kStages() {
  return ROT ? VMI_STAGES_ROT
             : MULTI ? VMI_STAGESM : (F32 ? (KIND == 2 ? VMI_STAGES_OCC : VMI_STAGES) : VMI_STAGES64);
}
template <typename Rec>
__device__ __forceinline__ void cp_async_rec(uint32_t dst, const Rec* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
  if (sizeof(Rec) == 32)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + 16),
                 "l"(reinterpret_cast<const char*>(src) + 16)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// a staged record's coordinates as doubles (float4 records are split doubles,
// vmi_device.cuh, unless VMI_SPLITREC=0)
__device__ __forceinline__ void rec_xyz(const float4& v, double& x, double& y, double& z) {
#if VMI_SPLITREC
  split_decode(make_uint4(__float_as_uint(v.x), __float_as_uint(v.y), __float_as_uint(v.z),
                          __float_as_uint(v.w)),
               x, y, z);
#else
  x = v.x; y = v.y; z = v.z;
#endif
}
__device__ __forceinline__ void rec_xyz(const double4& v, double& x, double& y, double& z) {
  x = v.x; y = v.y; z = v.z;
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
// VARZ is accumulated as (n, S1 = sum(z - K), S2 = sum((z - K)^2)) around the
// pivot K = the z of the voxel's lower face (a deterministic function of the
// voxel index, so every run of a voxel shares it: runs merge by plain addition
// and the table key is the voxel alone).  Keys (32-bit voxel index) and counts
// live in shared memory; (S1, S2) in a per-CTA, L2-resident global array
// updated with native fire-and-forget f64 reductions (RED.ADD.F64) -- a
// shared-memory f64 atomicAdd is a CAS loop on sm_100 and was ~30% of the
// kernel's stalls.  The multi-pass large-grid mode also keeps the counts in the
// L2 scratch (4-byte slots: more capacity, hence fewer passes).
template <bool MULTI>
__host__ __device__ constexpr bool kGlobalCounts() {
  return MULTI;
}
// (A/B: a per-run pivot -- the run's first z, re-pivoted on merge into a
// 64-bit key+pivot slot -- was 7 % slower at C2.)
using VKey = uint32_t;
constexpr VKey kEmptyKey = kEmpty32;
__host__ __device__ inline int slot_bytes(int kind, int multi) {
  if (kind == kKindOcc) return 4;  // key only
  if (kind != 0) return 4 + 4;
  return (int)sizeof(VKey) + (multi ? 0 : 4);
}
// queued run record: VARZ {lin, n, -, -, S1, S2}, COUNT {lin, n}, occupancy {lin}
__host__ __device__ constexpr int rec_bytes(int kind) { return kind == 0 ? 32 : kind == 1 ? 8 : 4; }

struct VarzTable {
  VKey* key;      // voxel index inside A's AABB (kEmptyKey = free)
  uint32_t* cnt;  // shared memory, or (multi-pass) the per-CTA global scratch
  double2* sums;  // global: this CTA's [cap] (S1, S2)
};

// Warp-private flush queue: run records pushed by any lane, drained 32 at a
// time by the whole warp so the hash/atomic path always runs converged.
#ifndef VMI_PG
#define VMI_PG 3  // A/B (C2): 3 > 4 (which needs a queue-overrun guard) > 2
#endif
#ifndef VMI_PG64
#define VMI_PG64 1
#endif
template <bool F32, bool MULTI, bool ROT = false>
__host__ __device__ constexpr int kPGt() {  // points per queue push
  return ROT ? VMI_PG : MULTI ? VMI_PGM : (F32 ? VMI_PG : VMI_PG64);
}
template <bool F32, bool MULTI, bool ROT = false>
__host__ __device__ constexpr int kQueueT() {  // warp queue entries: > 32*kPG + 31, pow2
  return kPGt<F32, MULTI, ROT>() == 1 ? 64 : 128;
}

// Shared-memory layout helper (bytes), mirrored by fast_smem_bytes() on the host.
constexpr int kCountLut = 1024;  // COUNT bins precomputed for n < kCountLut

struct FastSmem {
  size_t stage, table, queue, hist, marg, red, rows, cols, misc, lut, total;
};
__host__ __device__ inline FastSmem fast_layout(int kind, int cap, int W, int threads, int f32,
                                                int ns, int multi) {
  FastSmem L;
  size_t off = 0;
  L.stage = off;
  // f32: record kind -- 0 double4 input, 1 float4 split, 2 pre-rotated double4
  const int stages = multi ? kStages<true, true>()
                           : f32 == 2 ? kStages<false, false, 0, true>()
                           : (f32 ? (kind == 2 ? kStages<true, false, 2>() : kStages<true>())
                                  : kStages<false>());
  off += (size_t)threads * ns * (f32 == 1 ? 16 : 32) * stages;
  L.table = off;
  off += (size_t)cap * slot_bytes(kind, multi);
  off = (off + 15) & ~size_t(15);
  L.queue = off;
  const int queue = multi ? kQueueT<true, true>()
                  : f32 == 2 ? kQueueT<false, false, true>()
                  : (f32 ? kQueueT<true, false>() : kQueueT<false, false>());
  // + one warp queue of slack: the kernel aligns the queues to their size
  off += (size_t)(threads / 32 + 1) * queue * rec_bytes(kind);
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

__device__ __forceinline__ uint4 ld_shared_v4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ uint32_t atom_cas_shared(uint32_t a, uint32_t cmp, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(v)
               : "memory");
  return old;
}
__device__ __forceinline__ void red_add_shared(uint32_t a, uint32_t v) {
  asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld_shared_v2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
// predicated run-record stores straight from the run registers (no branch, no
// moves into aligned register quads): VARZ {lin, n, -, -, S1, S2} (32 B),
// COUNT {lin, n} (8 B)
__device__ __forceinline__ void st_rec32_if(bool p, uint32_t a, uint32_t l, uint32_t n, double s1,
                                            double s2) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n"
      " @q st.shared.v2.u32 [%1], {%2, %3};\n"
#if VMI_REC_V2
      " @q st.shared.v2.f64 [%1+16], {%4, %5};\n}" ::"r"((int)p),
#else
      " @q st.shared.f64 [%1+16], %4;\n"
      " @q st.shared.f64 [%1+24], %5;\n}" ::"r"((int)p),
#endif
      "r"(a), "r"(l), "r"(n), "d"(s1), "d"(s2)
      : "memory");
}
__device__ __forceinline__ void st_rec4_if(bool p, uint32_t a, uint32_t l) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.u32 [%1], %2;\n}" ::"r"((int)p),
               "r"(a), "r"(l)
               : "memory");
}
__device__ __forceinline__ void st_rec8_if(bool p, uint32_t a, uint32_t l, uint32_t n) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %0, 0;\n @q st.shared.v2.u32 [%1], {%2, %3};\n}" ::"r"(
          (int)p),
      "r"(a), "r"(l), "r"(n)
      : "memory");
}
// a new run starts: zero the run registers in place (predicated; no selects)
__device__ __forceinline__ void run_reset_if(bool p, uint32_t& n, double& s1, double& s2) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %3, 0;\n"
      " @q mov.b32 %0, 0;\n @q mov.b64 %1, 0;\n @q mov.b64 %2, 0;\n}"
      : "+r"(n), "+d"(s1), "+d"(s2)
      : "r"((int)p));
}
// lin if (rx, ry, rz) lies inside A's AABB, else kNoVoxel (one predicate chain)
__device__ __forceinline__ uint32_t inside_lin(uint32_t rx, uint32_t ry, uint32_t rz, uint32_t ex0,
                                               uint32_t ex1, uint32_t ex2) {
  const uint32_t lin = (rx * ex1 + ry) * ex2 + rz;
  uint32_t r;
  asm("{\n .reg .pred q;\n setp.lt.u32 q, %1, %4;\n setp.lt.and.u32 q, %2, %5, q;\n"
      " setp.lt.and.u32 q, %3, %6, q;\n selp.b32 %0, %7, -1, q;\n}"
      : "=r"(r)
      : "r"(rx), "r"(ry), "r"(rz), "r"(ex0), "r"(ex1), "r"(ex2), "r"(lin));
  return r;
}
__device__ __forceinline__ double mkd(uint32_t lo, uint32_t hi) {
  return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ uint32_t pin_u32(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
__device__ __forceinline__ double pin_reg(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}

#ifdef VMI_WATCHDOG  // debug builds: trap a runaway loop with its location
#define VMI_WD(id, cnt, a, b)                                                              \
  if (++cnt > (1u << 24)) {                                                                \
    printf("vmi watchdog %d block %d tid %d: %u %u\n", id, blockIdx.x, threadIdx.x,         \
           (unsigned)(a), (unsigned)(b));                                                  \
    __trap();                                                                              \
  }
#define VMI_TR(msg, a)                                                                    \
  if (threadIdx.x % 32 == 0 && blockIdx.x == 0) printf("tr %s warp %d: %d\n", msg, threadIdx.x / 32, (int)(a));
#else
#define VMI_WD(id, cnt, a, b)
#define VMI_TR(msg, a)
#endif

// MP (multi-pair): pose p scores pair pose_pair[p] of pairs[] (descriptor
// copied to shared memory per pose); otherwise the kernel parameters A0/B0.
// ROT (rotation-major grids): scan B's records are already rotated -- pose p
// reads the double4 (R p)_xyz records of rotation rot_idx[p] (k_rotate), so
// the per-point FMA chains are skipped; X = RN((R p)_x + t_x) as always.
template <int THREADS, int NS, int KIND, bool F32, int MODE, bool MULTI, bool MP, bool ROT = false>
__global__ void __launch_bounds__(THREADS, 1)
    k_pose_fast(GridParams g, const __grid_constant__ RefView A0,
                const __grid_constant__ QueryView B0, const double* __restrict__ mats, int64_t P,
                int cap, double* __restrict__ mi_out, int32_t* __restrict__ status_out,
                long long* __restrict__ hist_out, long long* __restrict__ total_out,
                FeatureDump dump, double2* __restrict__ gsums, int npass,
                const PairDesc* __restrict__ pairs, const int32_t* __restrict__ pose_pair,
                unsigned long long* __restrict__ hash_out, unsigned int* __restrict__ sched,
                const int32_t* __restrict__ rot_idx, int64_t rot_stride) {
  static_assert(!ROT || (!F32 && !MULTI && !MP), "pre-rotated records: double4, single pass, one pair");
  static_assert(NS == 1, "one span per thread");
  static_assert(sizeof(PairDesc) % 4 == 0 && sizeof(PairDesc) / 4 <= THREADS, "descriptor copy");
  __shared__ __align__(16) PairDesc desc_s;
  __shared__ double hull_s[6][THREADS / 32];
  __shared__ unsigned long long hash_s[THREADS / 32];
  __shared__ __align__(16) uint32_t cst_s[6];  // A's extents (single pair), 1/res (lo, hi)
  __shared__ long long nxt_s;                   // the CTA's next pose
  extern __shared__ __align__(16) unsigned char smem[];
  const int W = g.bins + 1;
  const FastSmem L = fast_layout(KIND, cap, W, THREADS, ROT ? 2 : (F32 ? 1 : 0), NS, MULTI ? 1 : 0);
  constexpr int kPG = kPGt<F32, MULTI, ROT>();
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
  // warp queue: AoS records, VARZ 32 B {lin, n, -, -, S1, S2}, COUNT 8 B {lin, n},
  // occupancy 4 B {lin}
  constexpr uint32_t kRec = (uint32_t)rec_bytes(KIND);
  constexpr int kQueue = kQueueT<F32, MULTI, ROT>();
  // Each warp's queue is aligned to its size QB, so a record address is
  // qbase | (byte offset mod QB): one LOP3 per push.
  constexpr uint32_t QB = (uint32_t)kQueue * kRec;
  // (an opaque copy: otherwise it is rematerialised from the shared window
  // base inside the point loop)
  const uint32_t qbase = pin_u32(
      (((uint32_t)__cvta_generic_to_shared(smem + L.queue) + QB - 1) & ~(QB - 1)) + wid * QB);
  if (KIND == 0) {
    VT.key = reinterpret_cast<VKey*>(smem + L.table);
    if (kGlobalCounts<MULTI>())  // counts next to the sums in L2 (native RED.ADD.U32)
      VT.cnt = reinterpret_cast<uint32_t*>(gsums + (size_t)gridDim.x * cap) + (size_t)blockIdx.x * cap;
    else
      VT.cnt = reinterpret_cast<uint32_t*>(smem + L.table + (size_t)cap * sizeof(VKey));
    VT.sums = gsums + (size_t)blockIdx.x * cap;
  } else {
    ckey = reinterpret_cast<uint32_t*>(smem + L.table);
    if (KIND == kKindCount) ccnt = reinterpret_cast<uint32_t*>(smem + L.table + (size_t)cap * 4);
  }

  // shared-window addresses of the table's keys / counts (pinned: see my_stage)
  const uint32_t key_sa = pin_u32((uint32_t)__cvta_generic_to_shared(smem + L.table));
  const uint32_t cnt_sa = pin_u32(key_sa + (uint32_t)cap * 4u);  // counts follow the keys
  // The table is cleared once here; afterwards the per-pose table walk resets
  // every slot it reads, so each pose starts from an empty table.
  auto clear_table = [&]() {
    uint4* t4 = reinterpret_cast<uint4*>(smem + L.table);
    const int key_words = KIND == 0 ? cap * (int)sizeof(VKey) / 16 : cap / 4;  // uint4s holding keys
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
  if (tid == 0) {  // (the first pose's barriers order these before any read)
    cst_s[0] = A0.ext[0]; cst_s[1] = A0.ext[1]; cst_s[2] = A0.ext[2]; cst_s[3] = 0u;
    cst_s[4] = (uint32_t)__double2loint(g.inv_res); cst_s[5] = (uint32_t)__double2hiint(g.inv_res);
  }

  // Poses after each CTA's first are claimed from a launch-wide ticket
  // counter (sched, zeroed by the host), one pose ahead: a CTA that drew
  // cheap poses takes more, so the launch ends within ~one pose time on every
  // SM instead of waiting for the slowest CTA's fixed share.  Without sched:
  // the static stride.  The next pose's matrix is loaded one pose ahead (its
  // L2 latency hides behind the current pose).
  auto claim = [&](long long cur) -> long long {
    return sched ? (long long)gridDim.x + (long long)atomicAdd(sched, 1u) : cur + gridDim.x;
  };
  if (tid == 0) nxt_s = claim(blockIdx.x);
  __syncthreads();
  double mat_next = (tid < 12 && blockIdx.x < P) ? mats[(int64_t)blockIdx.x * 12 + tid] : 0.0;
  for (int64_t p = blockIdx.x, nx = 0; p < P; p = nx) {
    nx = nxt_s;  // (read by every thread before the barrier below; re-claimed after it)
    if (MP && tid < (int)(sizeof(PairDesc) / 4))
      reinterpret_cast<uint32_t*>(&desc_s)[tid] =
          reinterpret_cast<const uint32_t*>(pairs + pose_pair[p])[tid];
    for (int i = tid; i < W * W; i += THREADS) hist[i] = 0u;
    for (int i = tid; i < W; i += THREADS) marg[i] = 0u;
    if (tid < 3) { misc[tid] = INT_MAX; misc[3 + tid] = INT_MIN; }
    if (tid >= 6 && tid < 9) misc[tid] = 0;
    if (tid < 12) {
#if VMI_MAT_PREFETCH
      mat_s[tid] = mat_next;
      if (nx < P) mat_next = mats[nx * 12 + tid];
#else
      mat_s[tid] = mats[p * 12 + tid];
      (void)mat_next;
#endif
    }
    __syncthreads();
    if (tid == 0) nxt_s = claim(nx);
    const RefView& A = MP ? desc_s.A : A0;
    const QueryView& B = MP ? desc_s.B : B0;
    const double m0 = mat_s[0], m1 = mat_s[1], m2 = mat_s[2], m3 = mat_s[3], m4 = mat_s[4],
                 m5 = mat_s[5], m6 = mat_s[6], m7 = mat_s[7], m8 = mat_s[8], t0 = mat_s[9],
                 t1 = mat_s[10], t2 = mat_s[11];
    // Every |q| < 2^30 here (rotation rows bound |R p| by sum|R_jk| * max|p|), so
    // floor(q) fits int32 without a per-point check; the +-2^20 key range is
    // checked exactly on the reduced bounds.  Poses beyond that (translations
    // of ~1e9 voxels) go to the exact path, which reports KEY_RANGE.
    {
      // kGridGeneral's fast floor needs |q - amin| < 2^22 (locate): 2^21 - max|amin|
      const int amx = max(max(abs(A.amin[0]), abs(A.amin[1])), abs(A.amin[2]));
      const double lim = (MODE == kGridGeneral ? 2097152.0 - (double)amx : 1073741824.0) * g.res;
      const double mx = B.max_abs;
      const double r0 = (fabs(m0) + fabs(m1) + fabs(m2)) * mx, r1 = (fabs(m3) + fabs(m4) + fabs(m5)) * mx,
                   r2 = (fabs(m6) + fabs(m7) + fabs(m8)) * mx;
      bool unsafe = fabs(t0 - g.origin[0]) + r0 >= lim || fabs(t1 - g.origin[1]) + r1 >= lim ||
                    fabs(t2 - g.origin[2]) + r2 >= lim;
      if (MODE == kGridGeneral) {  // the fast floor's |s + t| term (locate)
        const double lim2 = 16777216.0 * g.res;
        unsafe |= fabs(t0) + r0 >= lim2 || fabs(t1) + r1 >= lim2 || fabs(t2) + r2 >= lim2;
      }
      unsafe |= A.sparse != 0;  // no dense grid: the exact path looks A up (RefView.sparse)
      if (unsafe) {
        if (tid == 0) {
          mi_out[p] = -1e300;
          status_out[p] = 0x100;
          if (total_out) total_out[p] = 0;
          if (hash_out) hash_out[p] = 0;
        }
        __syncthreads();
        continue;
      }
    }

    // general resolutions: u = RN(t - o) for the fast floor (locate).  The
    // per-point error E of d against the reference's Z up to a per-pose
    // constant (d = s_z: one rounding of Z, <= 2^-53 |Z|; general mode's
    // pivot-relative d: <= 2^-52 (|t| + |o| + |R p|)) moves a voxel's VARZ by
    // <= res E + E^2 (its z spread is below res): var_shift covers both.
    const double u0 = __dsub_rn(t0, g.origin[0]), u1 = __dsub_rn(t1, g.origin[1]),
                 u2 = __dsub_rn(t2, g.origin[2]);
    const double cq0 = __dmul_rn(u0, g.inv_res), cq1 = __dmul_rn(u1, g.inv_res),
                 cq2 = __dmul_rn(u2, g.inv_res);
    const double var_shift =
        (MODE == kGridGeneral || VMI_PIVOT_SZ)
            ? 2.0 * g.res * 2.220446049250313e-16 *
                  (fabs(t2) + fabs(g.origin[2]) + (fabs(m6) + fabs(m7) + fabs(m8)) * B.max_abs + g.res)
            : 0.0;

    // ---- scan B's voxel bounds (voxel.py:220) from its convex hull ----------
    // For every direction the extreme of a point set is attained at a hull
    // vertex, so min/max of each transformed coordinate over ALL points equal
    // those over the hull -- up to rounding (~1e-13) and qhull's precision
    // (~1e-11 m) for points on or next to a face.  The floors are therefore
    // exact unless an extreme q lies within kHullEps of an integer; such a
    // pose (a few in 10^6) is re-run on the exact path.  The point loop then
    // skips its per-point min/max.
    const bool hull_bounds = B.hull_n > 0;
    if (hull_bounds) {
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (int i = tid; i < B.hull_n; i += THREADS) {
        const double x = B.hull[3 * i], y = B.hull[3 * i + 1], z = B.hull[3 * i + 2];
        const double q[3] = {grid_q<MODE>(xform_row(x, y, z, m0, m1, m2, t0), g.origin[0], g.res, g.inv_res),
                             grid_q<MODE>(xform_row(x, y, z, m3, m4, m5, t1), g.origin[1], g.res, g.inv_res),
                             grid_q<MODE>(xform_row(x, y, z, m6, m7, m8, t2), g.origin[2], g.res, g.inv_res)};
#pragma unroll
        for (int j = 0; j < 3; ++j) { lo[j] = fmin(lo[j], q[j]); hi[j] = fmax(hi[j], q[j]); }
      }
#pragma unroll
      for (int j = 0; j < 3; ++j) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo[j] = fmin(lo[j], __shfl_xor_sync(0xffffffffu, lo[j], o));
          hi[j] = fmax(hi[j], __shfl_xor_sync(0xffffffffu, hi[j], o));
        }
        if (lane == 0) { hull_s[j][wid] = lo[j]; hull_s[3 + j][wid] = hi[j]; }
      }
      __syncthreads();
      if (tid == 0) {
        bool amb = false;
        for (int j = 0; j < 3; ++j) {
          double a = INFINITY, b = -INFINITY;
          for (int w = 0; w < THREADS / 32; ++w) { a = fmin(a, hull_s[j][w]); b = fmax(b, hull_s[3 + j][w]); }
          const double fa = floor(a), fb = floor(b);
          constexpr double kHullEps = 1e-6;  // voxel units
          amb |= a - fa <= kHullEps + fabs(a) * 1e-12;           // the true min may be below fa
          amb |= fb + 1.0 - b <= kHullEps + fabs(b) * 1e-12;     // the true max may reach fb + 1
          misc[j] = (int)fa;
          misc[3 + j] = (int)fb;
        }
        if (amb) misc[8] = 1;  // exact path
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
      // ---- pass over this thread's span of scan B ---------------------------
      int bmin0 = INT_MAX, bmin1 = INT_MAX, bmin2 = INT_MAX;
      int bmax0 = INT_MIN, bmax1 = INT_MIN, bmax2 = INT_MIN;
      // the open run: voxel, point count, S1, S2 (pivot: the voxel's lower z face)
      uint32_t cur = kNoVoxel, cn = 0u;
      double cs1 = 0.0, cs2 = 0.0;
      uint32_t qh = 0, qt = 0;  // warp-uniform queue head / tail, in bytes
      // occupancy kind: cells counted at insert time (no table walk) unless a
      // feature dump wants the walk
      const bool occ_insert = KIND == kKindOcc && !dump.keys;
      uint32_t occ_miss = 0, occ_hit = 0;

      // one queued record per lane -> table.  The first probe (a hit, or the
      // insert into an empty home slot: most records) is one straight-line CAS,
      // so those lanes issue the count/sum atomics together once; only
      // collisions take the divergent probe loop.  (A probe loop that lanes
      // leave one by one re-issued the atomics ~3.4 times per drain.)
      auto flush_rec = [&](uint32_t idx, bool has) {
        const uint32_t a = qbase | (idx & (QB - 1));
        uint2 r0 = make_uint2(kNoVoxel, 0u);
        if (KIND == kKindOcc) {
          if (has) r0.x = ld_shared_u32(a);
        } else if (has) {
          r0 = ld_shared_v2(a);
        }
        uint32_t sl = slot_of(r0.x, ucap);
        // occupancy: A's bin at this voxel, loaded ahead (its latency overlaps
        // the CAS); a voxel's cell is counted when its key is first inserted
        const int ba_occ = (KIND == kKindOcc && occ_insert && has) ? (int)__ldg(&A.grid[r0.x]) : 0;
        auto count_new = [&]() {
          if (KIND == kKindOcc && occ_insert) {
            if (ba_occ == 0) ++occ_miss;
            else if (ba_occ == g.occ_bin) ++occ_hit;
            else atomicAdd(&hist[ba_occ * W + g.occ_bin], 1u);  // (injected A features)
          }
        };
        if constexpr (KIND == kKindOcc && VMI_OCC_BUCKET) {
          // Occupancy keys in 16-byte buckets of four slots: one LDS.128 finds
          // the key or the bucket's first free slot (a CAS there), so nearly
          // every lane is done in one round -- linear probing one slot at a
          // time kept a few lanes (and the warp) in the probe loop on most
          // drains.  Keys are never removed during a pose, so every lane with
          // a given key walks the same buckets to the same first free slot.
          // A/B: C4 40.5 -> 35.2 ms; the VARZ / COUNT tables (loads ~0.4, a
          // record carrying counts / sums) are faster with the blind first CAS
          // below (C2 26.56 vs 27.43 ms, C1 1.69 vs 1.73 with buckets).
          if (!has) return;
          const uint32_t nb = ucap >> 2;
          uint32_t b = slot_of(r0.x, nb);
          for (uint32_t probes = 0;;) {
            const uint32_t ba = key_sa + 16u * b;
            const uint4 w = ld_shared_v4(ba);
#if VMI_OCC_BFREE  // branch-free bucket scan: masks, then the first free slot by FFS
            const bool present = (w.x == r0.x) | (w.y == r0.x) | (w.z == r0.x) | (w.w == r0.x);
            if (present) break;
            const uint32_t em = (uint32_t)(w.x == kEmpty32) | ((uint32_t)(w.y == kEmpty32) << 1) |
                                ((uint32_t)(w.z == kEmpty32) << 2) | ((uint32_t)(w.w == kEmpty32) << 3);
            const uint32_t j = em ? (uint32_t)__ffs((int)em) - 1u : 4u;
#else
            if (w.x == r0.x || w.y == r0.x || w.z == r0.x || w.w == r0.x) break;  // present
            const uint32_t j = w.x == kEmpty32 ? 0u : w.y == kEmpty32 ? 1u
                             : w.z == kEmpty32 ? 2u : w.w == kEmpty32 ? 3u : 4u;
#endif
            if (j == 4u) {  // full: the next bucket
              if (++b == nb) b = 0;
              if (++probes >= nb) { misc[7] = 1; break; }  // table full -> exact path
              continue;
            }
            const uint32_t old = atom_cas_shared(ba + 4u * j, kEmpty32, r0.x);
            if (old == kEmpty32) { count_new(); break; }
            if (old == r0.x) break;
            // another key took that slot: read the bucket again
          }
          return;
        }
        // first probe = one CAS (hit or insert), no branch before the atomics;
        // shared-window addresses (key_sa / cnt_sa) avoid generic -> shared
        // conversions in this loop
        const uint32_t old0 = has ? atom_cas_shared(key_sa + 4u * sl, kEmpty32, r0.x) : 0u;
        const bool done = has && (old0 == kEmpty32 || old0 == r0.x);
        if (KIND == kKindOcc && has && old0 == kEmpty32) count_new();
        auto add = [&](uint32_t slot) {
          if (KIND == 0) {
            const uint4 r1 = ld_shared_v4(a + 16);
            if (kGlobalCounts<MULTI>()) atomicAdd(&VT.cnt[slot], r0.y);
            else red_add_shared(cnt_sa + 4u * slot, r0.y);
            atomicAdd(&VT.sums[slot].x, mkd(r1.x, r1.y));
            atomicAdd(&VT.sums[slot].y, mkd(r1.z, r1.w));
          } else if (KIND == kKindCount) {
            red_add_shared(cnt_sa + 4u * slot, r0.y);
          }  // occupancy: the key is all there is
        };
        if (done) {
          add(sl);
        } else if (has) {  // collision: linear probing from the next slot
#if VMI_PROBE4
          // the same slot order, four slots per LDS.128: the first slot at or
          // after pos holding the key or free decides (masks + FFS, no
          // per-slot branches).  A/B: C1v 2.87 -> 2.69 ms, C1 1.69 -> 1.68;
          // the unit-resolution instantiation (C2, C3, C5) measured slower
          // with it (26.57 -> 26.85 ms) and keeps the one-slot loop below.
          if constexpr (MODE != kGridUnit) {
          uint32_t pos = sl + 1 == ucap ? 0u : sl + 1;
          for (uint32_t probes = 1;;) {
            const uint32_t g4 = pos & ~3u, off = pos & 3u;
            const uint4 w = ld_shared_v4(key_sa + 4u * g4);
            uint32_t valid = (0xFu << off) & 0xFu;
            if (ucap - g4 < 4u) valid &= (1u << (ucap - g4)) - 1u;
            const uint32_t eq = ((uint32_t)(w.x == r0.x) | ((uint32_t)(w.y == r0.x) << 1) |
                                 ((uint32_t)(w.z == r0.x) << 2) | ((uint32_t)(w.w == r0.x) << 3)) & valid;
            const uint32_t em = ((uint32_t)(w.x == kEmpty32) | ((uint32_t)(w.y == kEmpty32) << 1) |
                                 ((uint32_t)(w.z == kEmpty32) << 2) | ((uint32_t)(w.w == kEmpty32) << 3)) & valid;
            const uint32_t dec = eq | em;
            if (dec) {
              const uint32_t j = (uint32_t)__ffs((int)dec) - 1u;
              if ((eq >> j) & 1u) { add(g4 + j); break; }
              const uint32_t old = atom_cas_shared(key_sa + 4u * (g4 + j), kEmpty32, r0.x);
              if (old == kEmpty32) count_new();
              if (old == kEmpty32 || old == r0.x) { add(g4 + j); break; }
              pos = g4 + j + 1u;  // another key took it: probe on past it
            } else {
              probes += __popc(valid);
              pos = g4 + 4u;
            }
            if (pos >= ucap) pos = 0;
            if (probes >= ucap) { misc[7] = 1; break; }  // table full -> exact path
          }
          return;
          }
#endif
          uint32_t probes = 1;
          while (true) {
            if (++sl == ucap) sl = 0;
            if (probes++ >= ucap) { misc[7] = 1; break; }  // table full -> exact path
            const uint32_t w = ld_shared_u32(key_sa + 4u * sl);
            if (w == r0.x) { add(sl); break; }
            if (w == kEmpty32) {
              const uint32_t old = atom_cas_shared(key_sa + 4u * sl, kEmpty32, r0.x);
              if (old == kEmpty32) count_new();
              if (old == kEmpty32 || old == r0.x) { add(sl); break; }
            }
          }
        }
      };
      auto drain_full = [&]() {  // whole warp, converged: 32 records at a time
        uint32_t wd = 0; (void)wd;
        while (qt - qh >= 32 * kRec) {
          VMI_WD(1, wd, qt, qh)
          __syncwarp();
          flush_rec(qh + lane * kRec, true);
          qh += 32 * kRec;
          __syncwarp();
        }
      };
      // per point: ballot the runs that just ended, predicated store of the
      // finished run straight from the run registers, then the run update
      auto run_step = [&](uint32_t lin, double d) {  // d: z - pivot
        const bool e = lin != cur;
        const bool pdu = e && cur != kNoVoxel;
        const unsigned mu = __ballot_sync(0xffffffffu, pdu);
        const uint32_t a = qbase | ((qt + __popc(mu & lt_mask) * kRec) & (QB - 1));
        if (KIND == 0)
          st_rec32_if(pdu, a, cur, cn, cs1, cs2);
        else if (KIND == kKindCount)
          st_rec8_if(pdu, a, cur, cn);
        else
          st_rec4_if(pdu, a, cur);
        qt += __popc(mu) * kRec;
#ifdef VMI_PRED_RESET
        run_reset_if(e, cn, cs1, cs2);
        ++cn;
        cs1 = __dadd_rn(cs1, d);
        cs2 = __fma_rn(d, d, cs2);
#else
        // a new run restarts the sums through a 0/1 factor (fma(x, 0, d) == d,
        // fma(x, 1, d) == x + d): one select instead of four 32-bit ones
        const double keep = e ? 0.0 : 1.0;
        cn = e ? 1u : cn + 1u;
        cs1 = __fma_rn(cs1, keep, d);
        cs2 = __fma_rn(cs2, keep, __dmul_rn(d, d));
#endif
        cur = lin;
      };
      const int am0 = A.amin[0], am1 = A.amin[1], am2 = A.amin[2];
      // General resolutions: A's extents and 1/res held in registers, read
      // from shared memory (opaque to ptxas, which rematerialises any copy of
      // a kernel parameter from the constant bank on every point).  A/B: C4
      // -0.2 %; the unit / power-of-two loops (C2, C1v) are 1.7 % faster with
      // the constant-bank operands (fewer live registers).
      uint32_t ex0 = A.ext[0], ex1 = A.ext[1], ex2 = A.ext[2];
      double inv_res_r = g.inv_res;
      if constexpr (MODE == kGridGeneral && VMI_PIN_CONST) {
        const uint32_t ext_sa = (uint32_t)__cvta_generic_to_shared(
            MP ? (const void*)&desc_s.A.ext[0] : (const void*)cst_s);
        const uint32_t cst_sa = (uint32_t)__cvta_generic_to_shared(cst_s);
        ex0 = ld_shared_u32(ext_sa); ex1 = ld_shared_u32(ext_sa + 4u); ex2 = ld_shared_u32(ext_sa + 8u);
        inv_res_r = mkd(ld_shared_u32(cst_sa + 16u), ld_shared_u32(cst_sa + 20u));
      }
      // floor(q) - amin straight from DADD.RM against 1.5*2^52 - amin (an
      // integer in [2^52, 2^53), so the sum rounds down to kc + floor(q) and
      // its low word is floor(q) - amin); bounds are tracked relative to amin
      // (opaque copies: otherwise they are recomputed from amin on every step)
      const double kc0 = pin_reg(6755399441055744.0 - (double)am0);
      const double kc1 = pin_reg(6755399441055744.0 - (double)am1);
      const double kc2 = pin_reg(6755399441055744.0 - (double)am2);
      // General resolutions (kGridGeneral): q' = (p - o) * RN(1/res) is within
      // |q'| * 2^-51 of numpy's RN((p - o) / res), i.e. < 2^-30 voxel for the
      // |q'| < 2^21 this pose is guaranteed (see `unsafe` above).  q' is
      // floored on a 2^-29 grid by DADD.RM against 1.5*2^23 - amin: the
      // mantissa >> 29 is 2^22 + floor(q') - amin and the low 29 bits are the
      // fraction.  Only a fraction within 4 grid steps of an integer can floor
      // differently from the reference; such a point (about 1 in 10^8) takes
      // the IEEE division.
      const double kf0 = pin_reg(12582912.0 - (double)am0);
      const double kf1 = pin_reg(12582912.0 - (double)am1);
      const double kf2 = pin_reg(12582912.0 - (double)am2);
      // transform (geometry.py:162-166), voxel index (voxel.py:192-207), lin
      // inside A's AABB, and d = z - (the voxel's lower z face): pure per point
      auto locate = [&](double x, double y, double z, uint32_t& lin, double& d, int& ix, int& iy,
                        int& iz) {
        if constexpr (MODE == kGridGeneral) {
          // Fast floor of q = (X - o) / res: q' = RN(RN(s + u) * RN(1/res)) with
          // s = the rows' FMA chains (xform_row before + t) and u = RN(t - o)
          // per pose.  |q' - numpy's RN(RN(X - o) / res)| <= (|t - o| + |X - o|
          // + |s + t|) / res * 2^-53 + |q| * 2^-52 < 2^-27.5 voxel under the
          // pose bounds of `unsafe` (|t - o| + |R p| < 2^21 res, |t| + |R p| <
          // 2^24 res).  q' is floored on a 2^-29 grid by DADD.RM against
          // 1.5*2^23 - amin (mantissa >> 29 = 2^22 + floor(q') - amin, low 29
          // bits = the fraction); only a fraction within 4 grid steps (2^-27) of
          // an integer can floor differently from the reference, and such a
          // point (about 1 in 10^8) takes the reference's own X = RN(s + t) and
          // IEEE quotient.
          const double sx = ROT ? x : rot_row(x, y, z, m0, m1, m2);
          const double sy = ROT ? y : rot_row(x, y, z, m3, m4, m5);
          const double sz = ROT ? z : rot_row(x, y, z, m6, m7, m8);
          // q' = RN(s * RN(1/res) + RN(u * RN(1/res))) in one FMA: besides the
          // rounding of c = u * RN(1/res) (|u / res| 2^-53 < 2^-32), the same
          // bound as RN(RN(s + u) * RN(1/res)).  VARZ keeps Zp = RN(s + u) for
          // its pivot-relative z.
          const double Zp = __dadd_rn(sz, u2);  // ~ Z - o_z
          const double qx = __fma_rn(sx, inv_res_r, cq0);
          const double qy = __fma_rn(sy, inv_res_r, cq1);
          const double qz = KIND == kKindOcc ? __fma_rn(sz, inv_res_r, cq2) : __dmul_rn(Zp, inv_res_r);
          const double rx = __dadd_rd(qx, kf0), ry = __dadd_rd(qy, kf1), rz = __dadd_rd(qz, kf2);
          const uint32_t lx = (uint32_t)__double2loint(rx), ly = (uint32_t)__double2loint(ry),
                         lz = (uint32_t)__double2loint(rz);
          constexpr uint32_t kFB = 0x0B400000u;  // (hi(2^23) << 3) + 2^22
          ix = (int)(__funnelshift_r(lx, (uint32_t)__double2hiint(rx), 29) - kFB);
          iy = (int)(__funnelshift_r(ly, (uint32_t)__double2hiint(ry), 29) - kFB);
          iz = (int)(__funnelshift_r(lz, (uint32_t)__double2hiint(rz), 29) - kFB);
          // fraction within 4 steps of an integer: ((l + 4) << 3) < 64, all three at once
          const bool near = __vimin3_u32(lx * 8u + 32u, ly * 8u + 32u, lz * 8u + 32u) < 64u;
          // floor(q_z) as a double: rz with its 29 fraction bits cleared, minus kf2
          double qf = __dsub_rn(__hiloint2double(__double2hiint(rz), (int)(lz & 0xE0000000u)), kf2);
          if (VMI_NEAR_FIX && __builtin_expect(near, 0)) {  // the reference's X and IEEE quotient
            const double X = __dadd_rn(sx, t0), Y = __dadd_rn(sy, t1), Z = __dadd_rn(sz, t2);
            ix = __double2loint(__dadd_rd(grid_q<MODE>(X, g.origin[0], g.res, g.inv_res), kc0));
            iy = __double2loint(__dadd_rd(grid_q<MODE>(Y, g.origin[1], g.res, g.inv_res), kc1));
            const double fz = __dadd_rd(grid_q<MODE>(Z, g.origin[2], g.res, g.inv_res), kc2);
            iz = __double2loint(fz);
            qf = __dsub_rn(fz, kc2);
          }
          // pivot: the voxel's lower face relative to o_z (a function of the voxel)
          d = VMI_PIVOT_SZ ? sz : __fma_rn(-qf, g.res, Zp);
          lin = inside_lin((uint32_t)ix, (uint32_t)iy, (uint32_t)iz, ex0, ex1, ex2);
          if (MULTI && npass > 1 && lin != kNoVoxel &&
              __umulhi(lin * 0x85EBCA6Bu, (uint32_t)npass) != (uint32_t)pass)
            lin = kNoVoxel;  // another pass's partition
          return;
        }
        const double X = ROT ? __dadd_rn(x, t0) : xform_row(x, y, z, m0, m1, m2, t0);
        const double Y = ROT ? __dadd_rn(y, t1) : xform_row(x, y, z, m3, m4, m5, t1);
        const double sz = ROT ? z : rot_row(x, y, z, m6, m7, m8);
        const double Z = __dadd_rn(sz, t2);  // = xform_row
        const double fx = __dadd_rd(grid_q<MODE>(X, g.origin[0], g.res, g.inv_res), kc0);
        const double fy = __dadd_rd(grid_q<MODE>(Y, g.origin[1], g.res, g.inv_res), kc1);
        const double fz = __dadd_rd(grid_q<MODE>(Z, g.origin[2], g.res, g.inv_res), kc2);
        ix = __double2loint(fx);
        iy = __double2loint(fy);
        iz = __double2loint(fz);
        // fz - kc2 == floor(q_z) exactly (both integers below 2^53)
        if (VMI_PIVOT_SZ) {
          d = sz;
        } else {
          const double qf = __dsub_rn(fz, kc2);
          d = __dsub_rn(Z, MODE == kGridUnit ? qf : __fma_rn(qf, g.res, g.origin[2]));
        }
        lin = inside_lin((uint32_t)ix, (uint32_t)iy, (uint32_t)iz, ex0, ex1, ex2);
        if (MULTI && npass > 1 && lin != kNoVoxel &&
            __umulhi(lin * 0x85EBCA6Bu, (uint32_t)npass) != (uint32_t)pass)
          lin = kNoVoxel;  // another pass's partition
      };

      using Rec = typename std::conditional<F32, float4, double4>::type;
      const Rec* pts = reinterpret_cast<const Rec*>(B.pts) +
                       (ROT ? (size_t)rot_idx[p] * (size_t)rot_stride : (size_t)0) + tid;
      const int full = B.span - 1;  // iterations every span owns
      // Scan-B records are staged through shared memory with cp.async: each
      // thread streams its own span S-1 records ahead into a private ring slot
      // (no cross-thread dependency, so no barrier), then reads the record back
      // with one LDS when it is its turn.  Rows are issued kPG at a time as one
      // commit group from a running pointer; the span layout is padded with
      // kStagePadRows rows, so rows past the span are issued unconditionally
      // (and never read back).
      constexpr int S = kStages<F32, MULTI, KIND, ROT>();
      // (opaque: otherwise rebuilt from the CTA's shared window base, an
      // S2UR SR_CgaCtaId round trip, before every group)
      const uint32_t my_stage = pin_u32(stage_base + (uint32_t)tid * (uint32_t)sizeof(Rec));
      constexpr uint32_t kStageStride = (uint32_t)(THREADS * sizeof(Rec));
      static_assert(S % kPG == 0, "ring holds whole groups");
      static_assert(S <= kStagePadRows, "span layout padding covers the ring");
      static_assert(32 * kPG + 31 <= kQueue, "a push group must fit the run queue");
      constexpr int kGroups = S / kPG;  // commit groups in flight
      constexpr size_t kRowBytes = (size_t)THREADS * sizeof(Rec);
      const char* src = reinterpret_cast<const char*>(pts);
      auto issue_group = [&](int slot0) {
#pragma unroll
        for (int u = 0; u < kPG; ++u)
          cp_async_rec<Rec>(my_stage + (uint32_t)(slot0 + u) * kStageStride,
                            reinterpret_cast<const Rec*>(src + u * kRowBytes));
        src += kPG * kRowBytes;
        cp_async_commit();
      };
      // hb: the hull supplies the bounds (compile-time in the main loop when
      // VMI_HULL_SPLIT: two copies of it, no per-group branch)
      auto group_body = [&](int slot0, auto hb) {  // the group starts in ring slot slot0
        constexpr bool kHB = decltype(hb)::value;
        cp_async_wait<kGroups - 1>();  // rows r .. r+kPG-1 have landed
        uint32_t l[kPG];
        double D[kPG];
        int ix[kPG], iy[kPG], iz[kPG];
#pragma unroll
        for (int u = 0; u < kPG; ++u) {
          const Rec v = lds_rec<Rec>(my_stage + (uint32_t)(slot0 + u) * kStageStride);
          double x, y, z;
          rec_xyz(v, x, y, z);
          locate(x, y, z, l[u], D[u], ix[u], iy[u], iz[u]);
        }
        issue_group(slot0);  // refill the slots just consumed with rows r+S ..
        if (VMI_HULL_SPLIT ? !kHB : !hull_bounds) {  // bounds: one min/max tree per group
          int n0 = ix[0], n1 = iy[0], n2 = iz[0], x0 = ix[0], x1 = iy[0], x2 = iz[0];
#pragma unroll
          for (int u = 1; u < kPG; ++u) {
            n0 = min(n0, ix[u]); n1 = min(n1, iy[u]); n2 = min(n2, iz[u]);
            x0 = max(x0, ix[u]); x1 = max(x1, iy[u]); x2 = max(x2, iz[u]);
          }
          bmin0 = min(bmin0, n0); bmin1 = min(bmin1, n1); bmin2 = min(bmin2, n2);
          bmax0 = max(bmax0, x0); bmax1 = max(bmax1, x1); bmax2 = max(bmax2, x2);
        }
        // a group adds <= 32*kPG records to < 32 unflushed ones
#pragma unroll
        for (int u = 0; u < kPG; ++u) run_step(l[u], D[u]);
        drain_full();
      };
#pragma unroll
      for (int gi = 0; gi < kGroups; ++gi) issue_group(gi * kPG);  // rows 0 .. S-1 in flight
      int rr = 0;
      // one trip = one lap of the ring (compile-time slots), then the last groups
      auto main_loop = [&](auto hb) {
        for (; rr + S <= full; rr += S) {
#pragma unroll
          for (int gi = 0; gi < kGroups; ++gi) group_body(gi * kPG, hb);
        }
        for (; rr + kPG <= full; rr += kPG) group_body(rr % S, hb);
      };
      if (VMI_HULL_SPLIT && hull_bounds)
        main_loop(std::true_type{});
      else
        main_loop(std::false_type{});
      cp_async_wait<0>();
      VMI_TR("main loop done", rr)
      for (; rr <= full; ++rr) {  // leftover (< kPG) points and the ragged last row
        const bool has = rr < full || span_of_thread(tid, THREADS) < B.rem;
        const Rec v = rr < full ? lds_rec<Rec>(my_stage + (uint32_t)(rr % S) * kStageStride)
                                : pts[(size_t)full * THREADS];
        uint32_t lin;
        double d;
        int ix, iy, iz;
        double x, y, z;
        rec_xyz(v, x, y, z);
        locate(x, y, z, lin, d, ix, iy, iz);
        if (has) {
          bmin0 = min(bmin0, ix); bmin1 = min(bmin1, iy); bmin2 = min(bmin2, iz);
          bmax0 = max(bmax0, ix); bmax1 = max(bmax1, iy); bmax2 = max(bmax2, iz);
        } else {
          lin = kNoVoxel;
        }
        run_step(lin, d);
        drain_full();
      }
      VMI_TR("leftover done", rr)
      run_step(kNoVoxel, 0.0);  // close the open run
      uint32_t wd2 = 0; (void)wd2;
      while (qh != qt) {  // drain the tail (partial round)
        VMI_WD(2, wd2, qt, qh)
        __syncwarp();
        if ((uint32_t)lane * kRec < qt - qh) flush_rec(qh + lane * kRec, true);
        qh = (qt - qh > 32u * kRec) ? qh + 32 * kRec : qt;
        __syncwarp();
      }
      VMI_TR("tail drained", qt)
      if (pass == 0) {
        // ---- reduce bounds / key-range flag ----------------------------------
        bmin0 = __reduce_min_sync(0xffffffffu, bmin0);
        bmin1 = __reduce_min_sync(0xffffffffu, bmin1);
        bmin2 = __reduce_min_sync(0xffffffffu, bmin2);
        bmax0 = __reduce_max_sync(0xffffffffu, bmax0);
        bmax1 = __reduce_max_sync(0xffffffffu, bmax1);
        bmax2 = __reduce_max_sync(0xffffffffu, bmax2);
        if (!hull_bounds && lane == 0 && bmin0 != INT_MAX) {  // relative to amin (locate); a warp may have no points
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
      auto finish_slot = [&](int s, uint32_t lin, int ba, double2 sum, uint32_t cnt) {
        int bb;
        double dump_feat = 0.0;
        if (KIND == 0) {
          const double nd = (double)cnt;
          const double S1 = sum.x, S2 = sum.y;
          VT.key[s] = kEmptyKey; VT.cnt[s] = 0u;
          VT.sums[s] = make_double2(0.0, 0.0);
          const double rn = __drcp_rn(nd);
          const double c1 = S1 * S1 * rn;
          const double ssd = S2 - c1;
          const double feat = (ssd > 0.0 ? ssd : 0.0) * rn;
          const double x = feat * bin_scale;
          const double k = rint(x);
          if (k >= 1.0 && k <= bins_d - 1.0) {
            const double tol = ((nd + 8.0) * 4.440892098500626e-16 * (S2 + c1) * rn +
                                feat * 9.094947017729282e-13 + var_shift) * bin_scale + 1e-300;
            if (fabs(x - k) <= tol) recheck = true;
          }
          const double f = floor(x);
          bb = 1 + (f >= bins_d - 1.0 ? g.bins - 1 : (int)f);
          dump_feat = feat;
        } else if (KIND == kKindCount) {
          const uint32_t n = ccnt[s];
          ckey[s] = kEmpty32; ccnt[s] = 0u;
          bb = n < (uint32_t)kCountLut ? (int)count_lut[n] : feature_bin((double)n, g.clamp, g.bins);
          dump_feat = (double)n;
        } else {  // occupancy: every occupied voxel has the same bin
          ckey[s] = kEmpty32;
          bb = g.occ_bin;
          dump_feat = __longlong_as_double(0x7ff8000000000000LL);  // no feature value (NaN)
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
      VMI_TR("walk start", status)
      if (KIND == kKindOcc && occ_insert) {
        // the cells were counted at insert time: add them up and reset the keys
        occ_miss = __reduce_add_sync(0xffffffffu, occ_miss);
        occ_hit = __reduce_add_sync(0xffffffffu, occ_hit);
        if (lane == 0) {
          if (occ_miss) atomicAdd(&hist[g.occ_bin], occ_miss);
          if (occ_hit) atomicAdd(&hist[g.occ_bin * W + g.occ_bin], occ_hit);
        }
        uint4* t4 = reinterpret_cast<uint4*>(smem + L.table);
        const uint4 ones = make_uint4(~0u, ~0u, ~0u, ~0u);
        for (int i = tid; i < cap / 4; i += THREADS) t4[i] = ones;
      } else if constexpr (KIND == 0) {
        // VARZ: each warp owns a contiguous slice of the table; it compacts the
        // occupied slots (ballot) into a ring in its share of the (idle)
        // staging buffer, then takes them four per lane, so a lane's A-grid and
        // L2 sums loads are in flight together and only occupied slots cost a
        // load round (the whole CTA is in this phase at once: nothing else
        // hides the latency).  A/B: -3 % kernel time at C2.
        constexpr int NW = THREADS / 32;
        constexpr int kWR = MULTI ? VMI_WALK_RING_M : VMI_WALK_RING;  // ring entries; kWU ballots per scan step / entries per lane
        constexpr int kWU = kWR / 64;
        static_assert(kStages<F32, MULTI, KIND, ROT>() * NS * (F32 ? 16 : 32) * 32 >= kWR * 4,
                      "walk ring fits the warp's staging slice");
        uint32_t* wl = reinterpret_cast<uint32_t*>(
            smem + L.stage + (size_t)wid * 32 * NS * (F32 ? 16 : 32) * kStages<F32, MULTI, KIND, ROT>());
        const int per = ((cap + NW - 1) / NW + 31) & ~31;
        const int se = min(cap, wid * per + per);
        int scan = wid * per;
        uint32_t wh = 0, wt = 0;  // ring head / tail (warp-uniform)
        uint32_t wd3 = 0; (void)wd3;
        while (scan < se || wt != wh) {  // warp-uniform
          VMI_WD(3, wd3, scan, wt - wh)
          while (scan < se && wt - wh < (uint32_t)(32 * kWU)) {
            bool occ[kWU];
            unsigned m[kWU];
#pragma unroll
            for (int u = 0; u < kWU; ++u) {
              const int s = scan + u * 32 + lane;
              occ[u] = s < se && VT.key[s] != kEmptyKey;
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
          uint32_t cnt[kWU];
#pragma unroll
          for (int u = 0; u < kWU; ++u) {
            const uint32_t i = (uint32_t)(u * 32 + lane);
            sl[u] = i < take ? (int)wl[(wh + i) & (kWR - 1)] : -1;
            lin[u] = sl[u] >= 0 ? VT.key[sl[u]] : kNoVoxel;
            ba[u] = lin[u] != kNoVoxel ? (int)__ldg(&A.grid[lin[u]]) : 0;
            // L2 copy (the reductions happen in L2; never trust a stale L1 line)
            sum[u] = lin[u] != kNoVoxel ? __ldcg(&VT.sums[sl[u]]) : make_double2(0.0, 0.0);
            // (multi-pass: the counts live in L2 too; load them with the sums)
            cnt[u] = lin[u] == kNoVoxel ? 0u : kGlobalCounts<MULTI>() ? __ldcg(&VT.cnt[sl[u]]) : VT.cnt[sl[u]];
          }
          wh += take;
          __syncwarp();  // entries read: the ring may be refilled
#pragma unroll
          for (int u = 0; u < kWU; ++u)
            if (lin[u] != kNoVoxel) finish_slot(sl[u], lin[u], ba[u], sum[u], cnt[u]);
        }
      } else {
        // COUNT / occupancy: four slots per thread per step, four A-grid loads
        // in flight (no L2 sums to fetch: compaction measured slower here)
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
          for (int u = 0; u < 4; ++u) {
            if (lin[u] == kNoVoxel) continue;
            if (KIND == kKindOcc && !dump.keys && (ba[u] == 0 || ba[u] == g.occ_bin)) {
              // occupancy: A's occupied voxels share the one bin too, so nearly
              // every cell update lands on (0, occ) or (occ, occ): count them
              // in registers (one atomic per warp below, not one per voxel)
              ckey[s0 + u * THREADS] = kEmpty32;
              if (ba[u] == 0) ++occ_miss; else ++occ_hit;
            } else {
              finish_slot(s0 + u * THREADS, lin[u], ba[u], make_double2(0.0, 0.0), 0u);
            }
          }
        }
        if (KIND == kKindOcc) {
          occ_miss = __reduce_add_sync(0xffffffffu, occ_miss);
          occ_hit = __reduce_add_sync(0xffffffffu, occ_hit);
          if (lane == 0) {
            if (occ_miss) atomicAdd(&hist[g.occ_bin], occ_miss);
            if (occ_hit) atomicAdd(&hist[g.occ_bin * W + g.occ_bin], occ_hit);
          }
        }
      }
      VMI_TR("walk done", 0)
      __syncthreads();  // walk done (slots reset) before the next pass refills
    }
    if (status != 0) {
      if (tid == 0) {
        mi_out[p] = -1e300;
        status_out[p] = status;
        if (total_out) total_out[p] = 0;
        if (hash_out) hash_out[p] = 0;
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
    } else if (A.sat) {
      // inclusion-exclusion on the summed-volume table of each present bin
      const uint32_t x0 = rlo[0] - A.amin[0], y0 = rlo[1] - A.amin[1], z0 = rlo[2] - A.amin[2];
      const uint32_t x1 = rhi[0] - A.amin[0] + 1, y1 = rhi[1] - A.amin[1] + 1,
                     z1 = rhi[2] - A.amin[2] + 1;
      const size_t sy = A.ext[2] + 1, sx = (size_t)(A.ext[1] + 1) * sy;
      const size_t vol = sx * (A.ext[0] + 1);
      for (int k = tid; k < A.sat_nb; k += THREADS) {
        const uint32_t* t = A.sat + (size_t)k * vol;
        auto at = [&](uint32_t x, uint32_t y, uint32_t z) { return __ldg(&t[x * sx + y * sy + z]); };
        const uint32_t c = at(x1, y1, z1) - at(x0, y1, z1) - at(x1, y0, z1) - at(x1, y1, z0) +
                           at(x0, y0, z1) + at(x0, y1, z0) + at(x1, y0, z0) - at(x0, y0, z0);
        marg[A.sat_bin[k]] = c;
      }
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
    if (hash_out) {  // block-uniform
      const unsigned long long h = block_hist_hash<THREADS>(hist, r.h00, W, hash_s);
      if (tid == 0) hash_out[p] = r.status == 0 ? h : 0ull;
    }
    __syncthreads();
  }
}

template <int THREADS, int NS, int KIND, bool F32, int MODE, bool MULTI, bool MP, bool ROT = false>
static cudaError_t launch_fast_t(const FastLaunch& fl, cudaStream_t st) {
  auto k = k_pose_fast<THREADS, NS, KIND, F32, MODE, MULTI, MP, ROT>;
  size_t smem = fast_smem_bytes(KIND, fl.cap, fl.g.bins, THREADS, ROT ? 2 : (F32 ? 1 : 0), NS,
                                MULTI ? 1 : 0);
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
  if (fl.sched) {
    cudaError_t z = cudaMemsetAsync(fl.sched, 0, sizeof(unsigned int), st);
    if (z != cudaSuccess) return z;
  }
  k<<<fl.grid, THREADS, smem, st>>>(fl.g, fl.A, fl.B, fl.mats, fl.P, fl.cap, fl.mi, fl.status,
                                    fl.hist, fl.total, fl.dump, fl.sums, fl.npass, fl.pairs,
                                    fl.pose_pair, fl.hash, fl.sched, fl.rot_idx, fl.rot_stride);
  return cudaGetLastError();
}

template <int T, int NS, int KIND, bool F32, bool MULTI, bool MP>
static cudaError_t launch_grid(const FastLaunch& fl, cudaStream_t st) {
  switch (fl.g.mode) {
    case kGridUnit: return launch_fast_t<T, NS, KIND, F32, kGridUnit, MULTI, MP>(fl, st);
    case kGridPow2: return launch_fast_t<T, NS, KIND, F32, kGridPow2, MULTI, MP>(fl, st);
    default: return launch_fast_t<T, NS, KIND, F32, kGridGeneral, MULTI, MP>(fl, st);
  }
}

// The multi-pass loop costs ~8% even at npass == 1 (measured), so single- and
// multi-pass are separate instantiations; the multi-pass layout (a ~3x bigger
// table) also runs single-pass when scan B's voxels fit it but not the
// single-pass table.
// Multi-pair launches are single-pass only (the host plans them so).
template <int T, int NS, int KIND>
static cudaError_t launch_rot(const FastLaunch& fl, cudaStream_t st) {
  if (fl.multi || fl.pairs || fl.B.is_f32) return cudaErrorInvalidValue;
  switch (fl.g.mode) {
    case kGridUnit: return launch_fast_t<T, NS, KIND, false, kGridUnit, false, false, true>(fl, st);
    case kGridPow2: return launch_fast_t<T, NS, KIND, false, kGridPow2, false, false, true>(fl, st);
    default: return launch_fast_t<T, NS, KIND, false, kGridGeneral, false, false, true>(fl, st);
  }
}

template <int T, int NS, int KIND, bool F32>
static cudaError_t launch_mode(const FastLaunch& fl, cudaStream_t st) {
  if (fl.rot_idx) return launch_rot<T, NS, KIND>(fl, st);
  if (fl.pairs) {
    if (fl.multi) return cudaErrorInvalidValue;
    return launch_grid<T, NS, KIND, F32, false, true>(fl, st);
  }
  return fl.multi ? launch_grid<T, NS, KIND, F32, true, false>(fl, st)
                  : launch_grid<T, NS, KIND, F32, false, false>(fl, st);
}

template <int T, int NS>
static cudaError_t launch_threads(const FastLaunch& fl, cudaStream_t st) {
  const bool f32 = fl.B.is_f32 != 0;
  if (fl.g.kind == kKindVarz)
    return f32 ? launch_mode<T, NS, 0, true>(fl, st) : launch_mode<T, NS, 0, false>(fl, st);
  if (fl.g.kind == kKindCount)
    return f32 ? launch_mode<T, NS, 1, true>(fl, st) : launch_mode<T, NS, 1, false>(fl, st);
  return f32 ? launch_mode<T, NS, 2, true>(fl, st) : launch_mode<T, NS, 2, false>(fl, st);
}

// ---- rotation-major grids: scan B pre-rotated once per distinct rotation ----
__global__ void k_rotate(const void* __restrict__ pts, int is_f32, int64_t n_rec,
                         const double* __restrict__ rots12, double4* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_rec) return;
  const double* m = rots12 + 12 * (int64_t)blockIdx.y;
  double x, y, z;
  if (is_f32)
    rec_xyz(reinterpret_cast<const float4*>(pts)[i], x, y, z);
  else
    rec_xyz(reinterpret_cast<const double4*>(pts)[i], x, y, z);
  out[(int64_t)blockIdx.y * n_rec + i] =
      make_double4(rot_row(x, y, z, m[0], m[1], m[2]), rot_row(x, y, z, m[3], m[4], m[5]),
                   rot_row(x, y, z, m[6], m[7], m[8]), 0.0);
}

cudaError_t launch_rotate(const void* pts, int is_f32, int64_t rows, int threads,
                          const double* rots12, int64_t R, void* out, cudaStream_t st) {
  if (R <= 0) return cudaSuccess;
  if (R > 65535) return cudaErrorInvalidValue;
  const int64_t n = rows * threads;
  const int T = 256;
  k_rotate<<<dim3((unsigned)((n + T - 1) / T), (unsigned)R), T, 0, st>>>(
      pts, is_f32, n, rots12, reinterpret_cast<double4*>(out));
  return cudaGetLastError();
}

// NS = 2 (two spans per thread at 256 threads) compiles and is exact, but was
// measured slower on B200 (IPC 1.5 with 8 warps/SM vs 2.2 with 16): only the
// one-span-per-thread configuration is instantiated.
cudaError_t launch_fast(const FastLaunch& fl, cudaStream_t st) {
  if (fl.B.threads != kFastThreads || fl.streams != 1) return cudaErrorInvalidValue;
  return launch_threads<kFastThreads, 1>(fl, st);
}

}  // namespace vmi
