/*
 * voxmi_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity CHECKER for the B200 path, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  It restates, in plain C, the numpy algorithm of the
 * reference package `voxmi` (/root/reference/pkg/src/voxmi, numpy >= 1.24,
 * here numpy 2.3.5 with OpenBLAS 0.3.30 `SkylakeX`), one function per reference
 * symbol, with the numpy library behaviour that fixes the bit pattern spelled
 * out where it matters:
 *
 *   geometry.py:126-138  euler_to_transform  -> orc_poses_to_mats
 *       math.sin/math.cos are glibc; products left to right; built with
 *       -ffp-contract=off so no FMA is formed.
 *   geometry.py:162-166  apply_transform     -> orc_transform
 *       `points @ R.T + t` through OpenBLAS dgemm is, bit for bit (N >= 7),
 *       fma(z, R[j][2], fma(y, R[j][1], x * R[j][0])) + t[j].
 *   voxel.py:192-207     voxel_indices       -> orc_voxel_indices
 *   voxel.py:65-73       pack_keys           -> orc_pack_key
 *   voxel.py:210-222     voxelize            -> orc_voxelize_features (stable sort)
 *   voxel.py:225-229     _segment_sums       -> seg_sum (np.add.reduceat:
 *       a[lo] + pairwise(a[lo+1:hi]) with numpy's 8-way pairwise_sum)
 *   voxel.py:267-295     compute_feature_map -> orc_voxelize_features
 *   voxel.py:298-318     compute_overlap / overlap_voxel_count
 *   mi.py:72-79          bin_features        -> orc_bin
 *   mi.py:124-160        build_joint_histogram -> orc_joint_histogram
 *   mi.py:163-174        entropy             -> orc_entropy (np.sort then
 *       pairwise np.sum; glibc log differs from numpy's SIMD log by <= 1 ulp
 *       on ~0.3% of inputs, so MI agrees to ~1e-15, not bitwise)
 *   mi.py:177-191        mutual_information  -> orc_mutual_information
 *   mi.py:194-219        mi_objective        -> orc_mi_objective(_batch)
 *
 * Pinned against golden vectors produced by the real reference
 * (tests/golden/make_golden.py) in tests/test_oracle.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define KEY_INDEX_MIN (-(1LL << 20))
#define KEY_INDEX_MAX ((1LL << 20) - 1)
#define NO_OVERLAP_SENTINEL (-1e300)

enum { ORC_OK = 0, ORC_EMPTY_REGION = 1, ORC_KEY_RANGE = 2, ORC_PHI_OFF_EMPTY = 3 };
enum { KIND_VARZ = 0, KIND_COUNT = 1 };

/* ---- geometry.py:126-138 ---------------------------------------------- */
void orc_poses_to_mats(const double* poses, int64_t n, double* mats) {
  for (int64_t p = 0; p < n; ++p) {
    const double* v = poses + 6 * p;
    double* m = mats + 12 * p;
    double sr = sin(v[3]), cr = cos(v[3]);
    double sp = sin(v[4]), cp = cos(v[4]);
    double sy = sin(v[5]), cy = cos(v[5]);
    m[0] = cy * cp;
    m[1] = cy * sp * sr - sy * cr;
    m[2] = cy * sp * cr + sy * sr;
    m[3] = sy * cp;
    m[4] = sy * sp * sr + cy * cr;
    m[5] = sy * sp * cr - cy * sr;
    m[6] = -sp;
    m[7] = cp * sr;
    m[8] = cp * cr;
    m[9] = v[0];
    m[10] = v[1];
    m[11] = v[2];
  }
}

/* ---- geometry.py:162-166 (numpy/OpenBLAS dgemm bit pattern) ------------ */
void orc_transform(const double* pts, int64_t n, const double* m, double* out) {
  for (int64_t i = 0; i < n; ++i) {
    double x = pts[3 * i], y = pts[3 * i + 1], z = pts[3 * i + 2];
    for (int j = 0; j < 3; ++j) {
      double s = fma(z, m[3 * j + 2], fma(y, m[3 * j + 1], x * m[3 * j]));
      out[3 * i + j] = s + m[9 + j];
    }
  }
}

/* ---- voxel.py:192-207; returns index of first offending point or -1 ---- */
int64_t orc_voxel_indices(const double* pts, int64_t n, const double* origin, double res,
                          int64_t* ijk) {
  int64_t bad = -1;
  for (int64_t i = 0; i < n; ++i) {
    for (int j = 0; j < 3; ++j) {
      double q = floor((pts[3 * i + j] - origin[j]) / res);
      /* numpy astype(int64) of an out-of-range float is undefined; anything
         outside the key range is an error either way */
      int64_t k = (q < -9.2e18 || q > 9.2e18) ? INT64_MIN : (int64_t)q;
      ijk[3 * i + j] = k;
      if ((k < KEY_INDEX_MIN || k > KEY_INDEX_MAX) && bad < 0) bad = i;
    }
  }
  return bad;
}

/* ---- voxel.py:65-73 ------------------------------------------------------ */
static inline int64_t orc_pack_key(const int64_t* ijk) {
  return ((ijk[0] + (1LL << 20)) << 42) | ((ijk[1] + (1LL << 20)) << 21) | (ijk[2] + (1LL << 20));
}

/* numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), unit stride */
static double pairwise(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise(a, n2) + pairwise(a + n2, n - n2);
  }
}

/* np.add.reduceat segment: a[lo] + pairwise(a[lo+1:hi]) (voxel.py:225-229) */
static double seg_sum(const double* a, int64_t lo, int64_t hi) {
  if (hi - lo == 1) return a[lo];
  return a[lo] + pairwise(a + lo + 1, hi - lo - 1);
}

typedef struct { int64_t key; int64_t idx; } kv_t;
static int kv_cmp(const void* x, const void* y) {
  const kv_t* a = (const kv_t*)x;
  const kv_t* b = (const kv_t*)y;
  if (a->key != b->key) return a->key < b->key ? -1 : 1;
  return a->idx < b->idx ? -1 : (a->idx > b->idx);
}

/*
 * voxelize + compute_feature_map (voxel.py:210-222, 267-295).
 * keys/values must hold n entries; returns V (occupied voxels), or
 * -(1 + first bad point) when a voxel index leaves the key range.
 * bounds = [min x,y,z, max x,y,z] over all points.
 */
int64_t orc_voxelize_features(const double* pts, int64_t n, const double* origin, double res,
                              int kind, int64_t* keys, double* values, int64_t* bounds) {
  int64_t* ijk = (int64_t*)malloc(sizeof(int64_t) * 3 * (n ? n : 1));
  int64_t bad = orc_voxel_indices(pts, n, origin, res, ijk);
  if (bad >= 0) { free(ijk); return -(1 + bad); }
  kv_t* kv = (kv_t*)malloc(sizeof(kv_t) * (n ? n : 1));
  for (int j = 0; j < 3; ++j) { bounds[j] = INT64_MAX; bounds[3 + j] = INT64_MIN; }
  for (int64_t i = 0; i < n; ++i) {
    kv[i].key = orc_pack_key(ijk + 3 * i);
    kv[i].idx = i;
    for (int j = 0; j < 3; ++j) {
      if (ijk[3 * i + j] < bounds[j]) bounds[j] = ijk[3 * i + j];
      if (ijk[3 * i + j] > bounds[3 + j]) bounds[3 + j] = ijk[3 * i + j];
    }
  }
  free(ijk);
  qsort(kv, n, sizeof(kv_t), kv_cmp); /* (key, idx) order == stable argsort */
  double* z = (double*)malloc(sizeof(double) * (n ? n : 1));
  double* sq = (double*)malloc(sizeof(double) * (n ? n : 1));
  for (int64_t i = 0; i < n; ++i) z[i] = pts[3 * kv[i].idx + 2];
  int64_t v = 0, lo = 0;
  while (lo < n) {
    int64_t hi = lo + 1;
    while (hi < n && kv[hi].key == kv[lo].key) ++hi;
    keys[v] = kv[lo].key;
    double cnt = (double)(hi - lo);
    if (kind == KIND_COUNT) {
      values[v] = cnt;
    } else {
      double mean = seg_sum(z, lo, hi) / cnt;
      for (int64_t i = lo; i < hi; ++i) { double d = z[i] - mean; sq[i] = d * d; }
      double ssd = seg_sum(sq, lo, hi);
      values[v] = (ssd > 0.0 ? ssd : 0.0) / cnt;
    }
    ++v;
    lo = hi;
  }
  free(kv); free(z); free(sq);
  return v;
}

/* ---- mi.py:72-79 ---------------------------------------------------------- */
static inline int64_t orc_bin(double v, int bins, double clamp) {
  int64_t raw = (int64_t)floor(v / clamp * bins);
  return 1 + (raw < bins - 1 ? raw : bins - 1);
}

void orc_bin_features(const double* v, int64_t n, int bins, double clamp, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_bin(v[i], bins, clamp);
}

static inline int in_region(int64_t key, const int64_t* reg /* xmin,ymin,zmin,xmax,ymax,zmax */) {
  int64_t x = ((key >> 42) & 0x1FFFFF) - (1LL << 20);
  int64_t y = ((key >> 21) & 0x1FFFFF) - (1LL << 20);
  int64_t z = (key & 0x1FFFFF) - (1LL << 20);
  return x >= reg[0] && x <= reg[3] && y >= reg[1] && y <= reg[4] && z >= reg[2] && z <= reg[5];
}

/* compute_overlap (voxel.py:298-307): returns 1 if empty */
int orc_overlap(const int64_t* ba, const int64_t* bb, int64_t* reg) {
  for (int j = 0; j < 3; ++j) {
    reg[j] = ba[j] > bb[j] ? ba[j] : bb[j];
    reg[3 + j] = ba[3 + j] < bb[3 + j] ? ba[3 + j] : bb[3 + j];
  }
  return reg[0] > reg[3] || reg[1] > reg[4] || reg[2] > reg[5];
}

/*
 * build_joint_histogram (mi.py:124-160) over sorted A/B keys.  counts must be
 * (bins+1)^2 int64, zeroed here.  Returns n_region (the histogram total).
 */
int64_t orc_joint_histogram(const int64_t* ka, const double* va, int64_t na,
                            const int64_t* kb, const double* vb, int64_t nb,
                            const int64_t* reg, int bins, double clamp, int64_t* counts) {
  int w = bins + 1;
  memset(counts, 0, sizeof(int64_t) * w * w);
  int64_t n_region = (reg[3] - reg[0] + 1) * (reg[4] - reg[1] + 1) * (reg[5] - reg[2] + 1);
  int64_t i = 0, j = 0, n_a = 0, n_b = 0, n_common = 0;
  /* merge-walk of the two sorted key lists restricted to the region */
  while (i < na || j < nb) {
    int take_a = j >= nb || (i < na && ka[i] <= kb[j]);
    int take_b = i >= na || (j < nb && kb[j] <= ka[i]);
    if (take_a && take_b) { /* common key */
      int ia = in_region(ka[i], reg);
      if (ia) {
        counts[orc_bin(va[i], bins, clamp) * w + orc_bin(vb[j], bins, clamp)]++;
        ++n_a; ++n_b; ++n_common;
      }
      ++i; ++j;
    } else if (take_a) {
      if (in_region(ka[i], reg)) { counts[orc_bin(va[i], bins, clamp) * w]++; ++n_a; }
      ++i;
    } else {
      if (in_region(kb[j], reg)) { counts[orc_bin(vb[j], bins, clamp)]++; ++n_b; }
      ++j;
    }
  }
  counts[0] += n_region - (n_a + n_b - n_common);
  return n_region;
}

static int dcmp(const void* x, const void* y) {
  double a = *(const double*)x, b = *(const double*)y;
  return (a > b) - (a < b);
}

/* entropy (mi.py:163-174); returns NAN for an all-zero distribution */
double orc_entropy(const double* c, int64_t n) {
  double total = pairwise(c, n);
  if (!(total > 0)) return NAN;
  double* t = (double*)malloc(sizeof(double) * (n ? n : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (c[i] > 0) { double p = c[i] / total; t[m++] = p * log(p); }
  qsort(t, m, sizeof(double), dcmp);
  double s = pairwise(t, m);
  free(t);
  return -s;
}

/* mutual_information (mi.py:177-191); out = mi, h_x, h_y, h_xy.
   returns 0, or 1 when an entropy is undefined (all-zero block). */
int orc_mutual_information(const int64_t* counts, int w, int include_phi, double* out) {
  int o = include_phi ? 0 : 1, m = w - o;
  double* cells = (double*)malloc(sizeof(double) * m * m);
  double* rows = (double*)malloc(sizeof(double) * m);
  double* cols = (double*)malloc(sizeof(double) * m);
  double* tmp = (double*)malloc(sizeof(double) * m);
  for (int a = 0; a < m; ++a)
    for (int b = 0; b < m; ++b) cells[a * m + b] = (double)counts[(a + o) * w + (b + o)];
  /* m.sum(axis=1) / m.sum(axis=0) on an int64 array: exact integer sums */
  for (int a = 0; a < m; ++a) {
    int64_t rs = 0, cs = 0;
    for (int b = 0; b < m; ++b) { rs += counts[(a + o) * w + (b + o)]; cs += counts[(b + o) * w + (a + o)]; }
    rows[a] = (double)rs; cols[a] = (double)cs;
  }
  (void)tmp;
  double hx = orc_entropy(rows, m), hy = orc_entropy(cols, m), hxy = orc_entropy(cells, (int64_t)m * m);
  free(cells); free(rows); free(cols); free(tmp);
  if (isnan(hx) || isnan(hy) || isnan(hxy)) return 1;
  double mi = hx + hy - hxy;
  if (mi >= -1e-12 && mi < 0.0) mi = 0.0;
  out[0] = mi; out[1] = hx; out[2] = hy; out[3] = hxy;
  return 0;
}

/*
 * mi_objective (mi.py:194-219) for one pose matrix against a prebuilt A map.
 * status: 0 ok, 1 empty region, 2 key range, 3 phi-off empty.  Optional
 * counts ((bins+1)^2) and region_total outputs (NULL to skip).
 */
double orc_mi_objective(const int64_t* ka, const double* va, int64_t na, const int64_t* bounds_a,
                        const double* pts_b, int64_t nb, const double* mat, const double* origin,
                        double res, int kind, int bins, double clamp, int include_phi,
                        int32_t* status, int64_t* counts_out, int64_t* total_out) {
  double* moved = (double*)malloc(sizeof(double) * 3 * nb);
  orc_transform(pts_b, nb, mat, moved);
  int64_t* kb = (int64_t*)malloc(sizeof(int64_t) * nb);
  double* vb = (double*)malloc(sizeof(double) * nb);
  int64_t bb[6], reg[6];
  int64_t v = orc_voxelize_features(moved, nb, origin, res, kind, kb, vb, bb);
  free(moved);
  double result = NO_OVERLAP_SENTINEL;
  int32_t st = ORC_OK;
  int w = bins + 1;
  int64_t local[64 * 64];
  int64_t* counts = counts_out ? counts_out : local;
  if (v < 0) {
    st = ORC_KEY_RANGE;
  } else if (orc_overlap(bounds_a, bb, reg)) {
    st = ORC_EMPTY_REGION;
  } else {
    int64_t total = orc_joint_histogram(ka, va, na, kb, vb, v, reg, bins, clamp, counts);
    if (total_out) *total_out = total;
    double mi[4];
    if (orc_mutual_information(counts, w, include_phi, mi)) st = ORC_PHI_OFF_EMPTY;
    else result = mi[0];
  }
  free(kb); free(vb);
  if (status) *status = st;
  return result;
}

/* Batch driver over P pose matrices; nthreads <= 0 means every host CPU
   (OpenMP; omp_get_num_procs, so torchrun's OMP_NUM_THREADS=1 does not
   silently serialise the CPU baseline). */
void orc_mi_objective_batch(const int64_t* ka, const double* va, int64_t na, const int64_t* bounds_a,
                            const double* pts_b, int64_t nb, const double* mats, int64_t P,
                            const double* origin, double res, int kind, int bins, double clamp,
                            int include_phi, int nthreads, double* mi_out, int32_t* status_out) {
#ifdef _OPENMP
  if (nthreads <= 0) nthreads = omp_get_num_procs();
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads)
#endif
  for (int64_t p = 0; p < P; ++p)
    mi_out[p] = orc_mi_objective(ka, va, na, bounds_a, pts_b, nb, mats + 12 * p, origin, res, kind,
                                 bins, clamp, include_phi, status_out + p, NULL, NULL);
}

int orc_max_threads(void) {
#ifdef _OPENMP
  return omp_get_num_procs();
#else
  return 1;
#endif
}
