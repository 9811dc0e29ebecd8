// nm_lockstep.h -- lockstep Nelder-Mead over many scan pairs (nm_lockstep.cpp).
#pragma once
#include <cstdint>
#include <climits>
#include <functional>
#include <vector>

#include "../../include/vmi.h"

namespace vmi {

constexpr int kNmDim = 6;
// OptimResult.termination (optim.py:49-59)
constexpr int kNmConvergedF = VMI_NM_CONVERGED_F, kNmConvergedX = VMI_NM_CONVERGED_X,
              kNmMaxIter = VMI_NM_MAX_ITER;

struct NmConfig {  // SimplexConfig (optim.py:26-46)
  double steps[kNmDim];
  int max_iterations;
  double f_tol, x_tol;
  int restarts;
  // Probes per step up to which an iteration evaluates all four candidates
  // (reflection, expansion, both contractions) at once; above it, the
  // reflection first and then only the one follow-up the reference needs (two
  // steps, ~2.5x fewer probes: the evaluator is throughput-bound there).
  int64_t spec_budget = INT64_MAX;
};

struct NmResult {
  double best_x[kNmDim];
  double best_value;  // MI (the maximised objective)
  int iterations, termination, n_evaluations, n_batches, n_speculative, uncertain;
  std::vector<double> trace, trace_spread;
};

// n poses (n x 6) with their run index -> g = -objective and a 64-bit identity
// of the value's source (equal identities = equal values on every backend)
using NmEvaluator =
    std::function<int(const double* poses, const int32_t* run, int64_t n, double* g, uint64_t* h)>;

// The same evaluator split in two so batches can be in flight while the host
// works: runs are dealt to `lanes` lanes (run k -> lane k % lanes); submit(l,
// ...) starts lane l's batch, wait(l, g, h) finishes it (g, h sized as that
// batch).  Decisions are unchanged: every run only ever sees its own values.
struct NmAsyncEvaluator {
  int lanes = 1;
  std::function<int(int lane, const double* poses, const int32_t* run, int64_t n)> submit;
  std::function<int(int lane, double* g, uint64_t* h)> wait;
};
int nm_lockstep_async(int64_t K, const double* x0, const NmConfig& cfg,
                      const NmAsyncEvaluator& ev, NmResult* out, int64_t* steps = nullptr,
                      int64_t* probes = nullptr);

// steps / probes (nullable): evaluator calls and poses evaluated
int nm_lockstep(int64_t K, const double* x0, const NmConfig& cfg, const NmEvaluator& eval,
                NmResult* out, int64_t* steps = nullptr, int64_t* probes = nullptr);

int nm_write_results(const NmResult* res, int64_t K, double* best_x, double* best_value,
                     int32_t* iterations, int32_t* termination, int32_t* n_evaluations,
                     int32_t* uncertain, double* trace, int32_t* trace_len, int64_t trace_cap);

}  // namespace vmi
