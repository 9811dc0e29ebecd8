// nm_lockstep.cpp -- Nelder-Mead for many scan pairs at once, on the host.
//
// The reference aligns one pair at a time: align() (pkg/src/voxmi/align.py:
// 122-159) runs nelder_mead_maximize (optim.py:62-175) with one objective call
// per probe.  Here K independent runs advance in lockstep: every step gathers
// each active run's pending probes -- the initial simplex, a restart simplex,
// a shrink, or the speculative {reflection, expansion, outside contraction,
// inside contraction} of an iteration (all four depend only on the centroid
// and the worst vertex) -- into ONE batch for the evaluator (the multi-pair GPU
// kernel: thousands of poses per launch), then replays each run's decision
// rules on the returned values.  Only the probes the reference would have
// evaluated are committed (best-ever tracking, evaluation count), in the
// reference's order, so with the reference's objective values every run is
// decision-for-decision the reference's (paper_1709_06948_b200/optim.py is the
// same schedule for one run, pinned by tests/test_optim.py).
//
// Objective values come from the GPU (<= ~1e-13 from the reference's numpy
// formula, tests/test_gpu_headline_parity.py), so a comparison whose operands
// are within kRel/kAbs of each other -- and do not come from the same joint
// histogram (64-bit histogram hash from the kernel) -- cannot be decided
// exactly here: the run is marked `uncertain` and the caller re-runs that pair
// on exact values (align(), host re-score of bit-exact histograms).  Pose
// arithmetic restates numpy bit for bit (this file is compiled with
// -ffp-contract=off): mean over the first n vertices = sequential sum / n,
// vertex norms = sequential sum of squares (tests/test_nm_lockstep.py pins
// both against numpy).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <vector>

#include "nm_lockstep.h"

namespace vmi {

namespace {

constexpr int N = kNmDim;      // pose dimension (tx, ty, tz, rx, ry, rz)
constexpr int V = kNmDim + 1;  // simplex vertices
constexpr double kRefl = 1.0, kExp = 2.0, kContr = 0.5, kShrink = 0.5;  // optim.py:19-22
constexpr double kRel = 1e-11, kAbs = 1e-13;  // "cannot be told apart" bound on -MI values

// kIter: the four speculative candidates pending; kIterR: the reflection
// alone; kIterE / kIterCO / kIterCI: the one follow-up it asked for
enum Phase { kInit, kIter, kIterR, kIterE, kIterCO, kIterCI, kShrinkPh, kRestart, kDone };

struct Run {
  double simplex[V][N];
  double values[V];
  uint64_t hashes[V];
  double steps[N];
  int iteration = 0, restarts_left = 0;
  Phase phase = kInit;
  double pend[V][N];
  int npend = 0;
  double refl[N], expd[N], cout_[N], cin_[N];
  double best_x[N];
  double best_g = INFINITY;
  uint64_t best_h = ~0ull;  // matches no histogram hash
  int n_eval = 0, n_batches = 0, n_spec = 0;
  std::vector<double> trace, spread;
  int termination = kNmMaxIter;
  bool uncertain = false;
  double g_r = 0.0;  // two-phase iterations: the reflection's value
  uint64_t h_r = 0;
};

// Could a and b (each within the backend's error of the reference's value)
// compare differently on the reference's values?  Not when they come from the
// same joint histogram (equal hashes: equal values on every backend), nor when
// one is the +inf "nothing yet" of the best-ever tracker.
bool close(double a, uint64_t ha, double b, uint64_t hb) {
  if (ha == hb || std::isinf(a) || std::isinf(b)) return false;
  return std::fabs(a - b) <= kRel * std::max(std::fabs(a), std::fabs(b)) + kAbs;
}
// a < b / a <= b on -MI values, flagging the run when the order is not certain
bool lt(Run& r, double a, uint64_t ha, double b, uint64_t hb) {
  if (close(a, ha, b, hb)) r.uncertain = true;
  return a < b;
}
bool le(Run& r, double a, uint64_t ha, double b, uint64_t hb) {
  if (close(a, ha, b, hb)) r.uncertain = true;
  return a <= b;
}

void initial_simplex(double out[V][N], const double center[N], const double steps[N]) {
  for (int v = 0; v < V; ++v)
    for (int j = 0; j < N; ++j) out[v][j] = center[j];
  for (int i = 0; i < N; ++i) out[i + 1][i] += steps[i];
}

// the reference's g(): count the evaluation, keep the best point ever seen
// (optim.py:85-91: strictly smaller replaces)
void commit(Run& r, const double x[N], double g, uint64_t h) {
  r.n_eval += 1;
  if (lt(r, g, h, r.best_g, r.best_h)) {
    r.best_g = g;
    r.best_h = h;
    std::memcpy(r.best_x, x, sizeof(double) * N);
  }
}

// the sort / convergence / next-probe block at the top of the reference loop
// (optim.py:110-160); leaves the run with its next pending batch, or done
void check(Run& r, const NmConfig& cfg, bool speculate) {
  {
    int order[V];
    for (int v = 0; v < V; ++v) order[v] = v;
    std::stable_sort(order, order + V, [&](int a, int b) { return r.values[a] < r.values[b]; });
    double s2[V][N], v2[V];
    uint64_t h2[V];
    for (int v = 0; v < V; ++v) {
      std::memcpy(s2[v], r.simplex[order[v]], sizeof(double) * N);
      v2[v] = r.values[order[v]];
      h2[v] = r.hashes[order[v]];
    }
    std::memcpy(r.simplex, s2, sizeof(s2));
    std::memcpy(r.values, v2, sizeof(v2));
    std::memcpy(r.hashes, h2, sizeof(h2));
    // an order that near-equal values of different histograms could flip
    for (int a = 0; a < V; ++a)
      for (int b = a + 1; b < V; ++b)
        if (close(r.values[a], r.hashes[a], r.values[b], r.hashes[b])) r.uncertain = true;
    const double f_spread = r.values[V - 1] - r.values[0];
    double x_spread = 0.0;
    for (int v = 0; v < V; ++v) {
      double s = 0.0;
      for (int j = 0; j < N; ++j) {
        const double d = r.simplex[v][j] - r.simplex[0][j];
        s = s + d * d;
      }
      const double nv = std::sqrt(s);
      if (nv > x_spread) x_spread = nv;
    }
    r.trace.push_back(-r.values[0]);
    r.spread.push_back(f_spread);
    int converged = -1;
    // f_spread carries the error of two values
    if (r.hashes[V - 1] != r.hashes[0] &&
        std::fabs(f_spread - cfg.f_tol) <=
            2.0 * (kRel * std::max(std::fabs(r.values[0]), std::fabs(r.values[V - 1])) + kAbs))
      r.uncertain = true;
    if (std::fabs(x_spread - cfg.x_tol) <= 1e-12 * cfg.x_tol) r.uncertain = true;
    if (f_spread < cfg.f_tol) converged = kNmConvergedF;
    else if (x_spread < cfg.x_tol) converged = kNmConvergedX;
    if (converged >= 0) {
      if (r.restarts_left > 0 && r.iteration < cfg.max_iterations) {
        r.restarts_left -= 1;
        for (int j = 0; j < N; ++j) r.steps[j] = r.steps[j] * 0.5;
        double c[N];
        std::memcpy(c, r.simplex[0], sizeof(c));
        initial_simplex(r.simplex, c, r.steps);
        for (int v = 1; v < V; ++v) std::memcpy(r.pend[v - 1], r.simplex[v], sizeof(double) * N);
        r.npend = N;
        r.phase = kRestart;
        return;
      }
      r.termination = converged;
      r.phase = kDone;
      return;
    }
    if (r.iteration >= cfg.max_iterations) {
      r.termination = kNmMaxIter;
      r.phase = kDone;
      return;
    }
    r.iteration += 1;
    double c[N];
    for (int j = 0; j < N; ++j) {  // simplex[:-1].mean(axis=0): sequential sum, then / n
      double s = r.simplex[0][j];
      for (int v = 1; v < N; ++v) s = s + r.simplex[v][j];
      c[j] = s / (double)N;
    }
    const double* w = r.simplex[V - 1];
    for (int j = 0; j < N; ++j) {
      r.refl[j] = c[j] + kRefl * (c[j] - w[j]);
      r.expd[j] = c[j] + kExp * (c[j] - w[j]);
    }
    for (int j = 0; j < N; ++j) {
      r.cout_[j] = c[j] + kContr * (r.refl[j] - c[j]);
      r.cin_[j] = c[j] - kContr * (c[j] - w[j]);
    }
    std::memcpy(r.pend[0], r.refl, sizeof(r.refl));
    if (!speculate) {
      r.npend = 1;
      r.phase = kIterR;
      return;
    }
    std::memcpy(r.pend[1], r.expd, sizeof(r.expd));
    std::memcpy(r.pend[2], r.cout_, sizeof(r.cout_));
    std::memcpy(r.pend[3], r.cin_, sizeof(r.cin_));
    r.npend = 4;
    r.phase = kIter;
    return;
  }
}

void shrink(Run& r) {
  for (int v = 1; v < V; ++v)
    for (int j = 0; j < N; ++j)
      r.simplex[v][j] = r.simplex[0][j] + kShrink * (r.simplex[v][j] - r.simplex[0][j]);
  for (int v = 1; v < V; ++v) std::memcpy(r.pend[v - 1], r.simplex[v], sizeof(double) * N);
  r.npend = N;
  r.phase = kShrinkPh;
}

void replace_worst(Run& r, const double x[N], double g, uint64_t h) {
  std::memcpy(r.simplex[V - 1], x, sizeof(double) * N);
  r.values[V - 1] = g;
  r.hashes[V - 1] = h;
}

void pend_one(Run& r, const double x[N], Phase ph) {
  std::memcpy(r.pend[0], x, sizeof(double) * N);
  r.npend = 1;
  r.phase = ph;
}

// the run's pending probes came back: apply the reference's rules (optim.py:135-175)
void apply(Run& r, const NmConfig& cfg, const double* g, const uint64_t* h, bool speculate) {
  r.n_batches += 1;
  r.n_spec += r.npend;
  switch (r.phase) {
    case kInit:
      for (int v = 0; v < V; ++v) {
        commit(r, r.simplex[v], g[v], h[v]);
        r.values[v] = g[v];
        r.hashes[v] = h[v];
      }
      break;
    case kRestart:
    case kShrinkPh:
      for (int v = 1; v < V; ++v) {
        commit(r, r.simplex[v], g[v - 1], h[v - 1]);
        r.values[v] = g[v - 1];
        r.hashes[v] = h[v - 1];
      }
      break;
    case kIter: {
      const double g_r = g[0], g_e = g[1], g_co = g[2], g_ci = g[3];
      const uint64_t h_r = h[0], h_e = h[1], h_co = h[2], h_ci = h[3];
      commit(r, r.refl, g_r, h_r);
      if (lt(r, g_r, h_r, r.values[0], r.hashes[0])) {
        commit(r, r.expd, g_e, h_e);
        if (lt(r, g_e, h_e, g_r, h_r)) replace_worst(r, r.expd, g_e, h_e);
        else replace_worst(r, r.refl, g_r, h_r);
        break;
      }
      if (lt(r, g_r, h_r, r.values[V - 2], r.hashes[V - 2])) {
        replace_worst(r, r.refl, g_r, h_r);
        break;
      }
      if (lt(r, g_r, h_r, r.values[V - 1], r.hashes[V - 1])) {
        commit(r, r.cout_, g_co, h_co);
        if (le(r, g_co, h_co, g_r, h_r)) {
          replace_worst(r, r.cout_, g_co, h_co);
          break;
        }
      } else {
        commit(r, r.cin_, g_ci, h_ci);
        if (lt(r, g_ci, h_ci, r.values[V - 1], r.hashes[V - 1])) {
          replace_worst(r, r.cin_, g_ci, h_ci);
          break;
        }
      }
      shrink(r);
      return;  // wait for the shrunk vertices
    }
    case kIterR: {  // the same rules, one probe at a time (the reference's order)
      r.g_r = g[0];
      r.h_r = h[0];
      commit(r, r.refl, r.g_r, r.h_r);
      if (lt(r, r.g_r, r.h_r, r.values[0], r.hashes[0])) {
        pend_one(r, r.expd, kIterE);
        return;
      }
      if (lt(r, r.g_r, r.h_r, r.values[V - 2], r.hashes[V - 2])) {
        replace_worst(r, r.refl, r.g_r, r.h_r);
        break;
      }
      if (lt(r, r.g_r, r.h_r, r.values[V - 1], r.hashes[V - 1])) pend_one(r, r.cout_, kIterCO);
      else pend_one(r, r.cin_, kIterCI);
      return;
    }
    case kIterE:
      commit(r, r.expd, g[0], h[0]);
      if (lt(r, g[0], h[0], r.g_r, r.h_r)) replace_worst(r, r.expd, g[0], h[0]);
      else replace_worst(r, r.refl, r.g_r, r.h_r);
      break;
    case kIterCO:
      commit(r, r.cout_, g[0], h[0]);
      if (le(r, g[0], h[0], r.g_r, r.h_r)) {
        replace_worst(r, r.cout_, g[0], h[0]);
        break;
      }
      shrink(r);
      return;
    case kIterCI:
      commit(r, r.cin_, g[0], h[0]);
      if (lt(r, g[0], h[0], r.values[V - 1], r.hashes[V - 1])) {
        replace_worst(r, r.cin_, g[0], h[0]);
        break;
      }
      shrink(r);
      return;
    default:
      return;
  }
  check(r, cfg, speculate);
}

}  // namespace

int nm_lockstep_async(int64_t K, const double* x0, const NmConfig& cfg,
                      const NmAsyncEvaluator& ev, NmResult* out, int64_t* steps_out,
                      int64_t* probes_out) {
  std::vector<Run> runs((size_t)K);
  for (int64_t k = 0; k < K; ++k) {
    Run& r = runs[(size_t)k];
    for (int j = 0; j < N; ++j)
      if (!std::isfinite(x0[N * k + j])) return -1;
    std::memcpy(r.steps, cfg.steps, sizeof(r.steps));
    r.restarts_left = cfg.restarts;
    initial_simplex(r.simplex, x0 + N * k, r.steps);
    for (int v = 0; v < V; ++v) std::memcpy(r.pend[v], r.simplex[v], sizeof(double) * N);
    r.npend = V;
    r.phase = kInit;
  }
  // runs k with k % L == l form lane l; a lane's batch is in flight while the
  // host applies the other lanes' results (the evaluator overlaps them)
  const int L = std::max(1, ev.lanes);
  struct Lane {
    std::vector<double> poses;
    std::vector<int32_t> pair;
    std::vector<int64_t> run, first;
    std::vector<double> g;
    std::vector<uint64_t> h;
    bool pending = false;
    bool speculate = true;
  };
  std::vector<Lane> lane((size_t)L);
  int64_t active = K, steps = 0;
  auto submit = [&](int l) -> int {
    Lane& ln = lane[(size_t)l];
    ln.poses.clear();
    ln.pair.clear();
    ln.run.clear();
    ln.first.clear();
    ln.speculate = 4 * active <= cfg.spec_budget;
    for (int64_t k = l; k < K; k += L) {
      Run& r = runs[(size_t)k];
      if (r.phase == kDone) continue;
      ln.run.push_back(k);
      ln.first.push_back((int64_t)ln.pair.size());
      for (int i = 0; i < r.npend; ++i) {
        ln.poses.insert(ln.poses.end(), r.pend[i], r.pend[i] + N);
        ln.pair.push_back((int32_t)k);
      }
    }
    const int64_t P = (int64_t)ln.pair.size();
    ln.pending = P > 0;
    if (!ln.pending) return 0;
    ++steps;
    if (probes_out) *probes_out += P;
    ln.g.assign((size_t)P, 0.0);
    ln.h.assign((size_t)P, 0);
    return ev.submit(l, ln.poses.data(), ln.pair.data(), P);
  };
  for (int l = 0; l < L; ++l) {
    const int rc = submit(l);
    if (rc) return rc;
  }
  bool any = true;
  while (any) {
    any = false;
    for (int l = 0; l < L; ++l) {
      Lane& ln = lane[(size_t)l];
      if (!ln.pending) continue;
      int rc = ev.wait(l, ln.g.data(), ln.h.data());
      if (rc) return rc;
      for (size_t q = 0; q < ln.run.size(); ++q) {
        Run& r = runs[(size_t)ln.run[q]];
        const size_t f = (size_t)ln.first[q];
        apply(r, cfg, ln.g.data() + f, ln.h.data() + f, ln.speculate);
        if (r.phase == kDone) --active;
      }
      if ((rc = submit(l))) return rc;
      any |= ln.pending;
    }
  }
  for (int64_t k = 0; k < K; ++k) {
    const Run& r = runs[(size_t)k];
    NmResult& o = out[k];
    std::memcpy(o.best_x, r.best_x, sizeof(o.best_x));
    o.best_value = -r.best_g;
    o.iterations = r.iteration;
    o.termination = r.termination;
    o.n_evaluations = r.n_eval;
    o.n_batches = r.n_batches;
    o.n_speculative = r.n_spec;
    o.uncertain = r.uncertain ? 1 : 0;
    o.trace = r.trace;
    o.trace_spread = r.spread;
  }
  if (steps_out) *steps_out += steps;
  return 0;
}

int nm_lockstep(int64_t K, const double* x0, const NmConfig& cfg, const NmEvaluator& eval,
                NmResult* out, int64_t* steps_out, int64_t* probes_out) {
  // one lane, evaluated on wait()
  const double* sp = nullptr;
  const int32_t* sr = nullptr;
  int64_t sn = 0;
  NmAsyncEvaluator ev;
  ev.lanes = 1;
  ev.submit = [&](int, const double* p, const int32_t* r, int64_t n) {
    sp = p;
    sr = r;
    sn = n;
    return 0;
  };
  ev.wait = [&](int, double* g, uint64_t* h) { return eval(sp, sr, sn, g, h); };
  return nm_lockstep_async(K, x0, cfg, ev, out, steps_out, probes_out);
}

}  // namespace vmi

// ---- C ABI: the driver with a caller-supplied objective (tests, other backends)
extern "C" int vmi_nm_run(int64_t K, const double* x0, const double steps[6], int max_iterations,
                          double f_tol, double x_tol, int restarts, int64_t spec_budget,
                          vmi_nm_eval_fn fn, void* user,
                          double* best_x, double* best_value, int32_t* iterations,
                          int32_t* termination, int32_t* n_evaluations, int32_t* uncertain,
                          double* trace, int32_t* trace_len, int64_t trace_cap) {
  if (K < 0 || (K > 0 && (!x0 || !steps || !fn || !best_x || !best_value))) return -1;
  if (max_iterations < 1 || !(f_tol > 0) || !(x_tol > 0) || restarts < 0) return -1;
  vmi::NmConfig cfg{};
  std::memcpy(cfg.steps, steps, sizeof(cfg.steps));
  for (int j = 0; j < 6; ++j)
    if (!(cfg.steps[j] > 0)) return -1;
  cfg.max_iterations = max_iterations;
  cfg.f_tol = f_tol;
  cfg.x_tol = x_tol;
  cfg.restarts = restarts;
  cfg.spec_budget = spec_budget < 0 ? INT64_MAX : spec_budget;
  std::vector<vmi::NmResult> res((size_t)K);
  // VMI_NM_LANES (tests): deal the runs to that many lanes, as the GPU driver
  // does (vmi_align_pairs); the callback runs when a lane is waited for
  const char* le = std::getenv("VMI_NM_LANES");
  const int lanes = le ? std::max(1, std::atoi(le)) : 1;
  struct Pend {
    const double* p = nullptr;
    const int32_t* r = nullptr;
    int64_t n = 0;
  };
  std::vector<Pend> pend((size_t)lanes);
  vmi::NmAsyncEvaluator ev;
  ev.lanes = lanes;
  ev.submit = [&](int l, const double* p, const int32_t* r, int64_t n) {
    pend[(size_t)l] = {p, r, n};
    return 0;
  };
  ev.wait = [&](int l, double* g, uint64_t* h) {
    const Pend& q = pend[(size_t)l];
    return fn(user, q.p, q.r, q.n, g, h);
  };
  int rc = vmi::nm_lockstep_async(K, x0, cfg, ev, res.data());
  if (rc) return rc;
  return vmi::nm_write_results(res.data(), K, best_x, best_value, iterations, termination,
                               n_evaluations, uncertain, trace, trace_len, trace_cap);
}

int vmi::nm_write_results(const NmResult* res, int64_t K, double* best_x, double* best_value,
                          int32_t* iterations, int32_t* termination, int32_t* n_evaluations,
                          int32_t* uncertain, double* trace, int32_t* trace_len,
                          int64_t trace_cap) {
  for (int64_t k = 0; k < K; ++k) {
    const NmResult& o = res[k];
    std::memcpy(best_x + 6 * k, o.best_x, sizeof(double) * 6);
    best_value[k] = o.best_value;
    if (iterations) iterations[k] = o.iterations;
    if (termination) termination[k] = o.termination;
    if (n_evaluations) n_evaluations[k] = o.n_evaluations;
    if (uncertain) uncertain[k] = o.uncertain;
    if (trace && trace_len) {
      const int64_t n = std::min<int64_t>((int64_t)o.trace.size(), trace_cap);
      for (int64_t i = 0; i < n; ++i) trace[k * trace_cap + i] = o.trace[(size_t)i];
      trace_len[k] = (int32_t)o.trace.size();
    }
  }
  return 0;
}
