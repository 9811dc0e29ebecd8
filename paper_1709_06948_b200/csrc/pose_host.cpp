// pose_host.cpp -- euler_to_transform for pose batches, on the host.
//
// Reference: pkg/src/voxmi/geometry.py:126-138.  The reference evaluates
// math.sin / math.cos (glibc) and Python float products left to right, each
// rounded separately.  This translation unit is compiled by g++ with
// -ffp-contract=off (see build.py) and calls glibc's sin/cos, so every entry
// is bit-identical; CUDA's device sin/cos carry no such guarantee, which is
// why this O(P) step stays on the host.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdint>
#include <thread>
#include <vector>

extern "C" int vmi_poses_to_mats(const double* poses, int64_t n, double* mats, int threads) {
  if (n < 0 || (n > 0 && (!poses || !mats))) return -1;
  auto work = [&](int64_t lo, int64_t hi) {
    for (int64_t p = lo; p < hi; ++p) {
      const double* v = poses + 6 * p;
      double* m = mats + 12 * p;
      const double sr = std::sin(v[3]), cr = std::cos(v[3]);
      const double sp = std::sin(v[4]), cp = std::cos(v[4]);
      const double sy = std::sin(v[5]), cy = std::cos(v[5]);
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
  };
  int hw = (int)std::thread::hardware_concurrency();
  if (threads <= 0) {
    // one process per GPU (torchrun): share the host cores between the local ranks
    const char* lws = std::getenv("LOCAL_WORLD_SIZE");
    const int ranks = lws ? std::max(1, std::atoi(lws)) : 1;
    threads = hw > 0 ? std::max(1, hw / ranks) : 1;
  }
  if (n < 4096 || threads == 1) {
    work(0, n);
    return 0;
  }
  if (threads > 64) threads = 64;
  std::vector<std::thread> pool;
  const int64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const int64_t lo = t * chunk, hi = lo + chunk < n ? lo + chunk : n;
    if (lo >= hi) break;
    pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
  return 0;
}
