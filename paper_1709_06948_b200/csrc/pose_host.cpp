// pose_host.cpp -- euler_to_transform for pose batches, on the host.
//
// Reference: pkg/src/voxmi/geometry.py:126-138.  The reference evaluates
// math.sin / math.cos (glibc) and Python float products left to right, each
// rounded separately.  This translation unit is compiled by g++ with
// -ffp-contract=off (see build.py) and calls glibc's sin/cos, so every entry
// is bit-identical; CUDA's device sin/cos carry no such guarantee, which is
// why this O(P) step stays on the host.
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace {

// Persistent workers: a conversion on the critical path of vmi_eval_poses
// (the first chunk, before its kernel can start) must not pay ~20 us per
// thread creation.  Chunks are claimed from an atomic counter; the calling
// thread works too.
class Pool {
 public:
  void run(int workers, int64_t nchunks, const std::function<void(int64_t)>& fn) {
    std::lock_guard<std::mutex> one(run_m_);  // one job at a time (calls from several host threads)
    std::unique_lock<std::mutex> lk(m_);
    ensure(workers);
    fn_ = &fn;
    nchunks_ = nchunks;
    next_.store(0);
    active_ = (int)th_;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    drain();
    lk.lock();
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  void ensure(int workers) {  // (m_ held)
    while ((int)th_ < workers) {  // a new worker joins the job about to be posted
      const uint64_t seen = gen_;
      std::thread([this, seen] { loop(seen); }).detach();
      ++th_;
    }
  }
  void drain() {
    for (int64_t k; (k = next_.fetch_add(1)) < nchunks_;) (*fn_)(k);
  }
  void loop(uint64_t seen) {
    for (;;) {
      std::unique_lock<std::mutex> lk(m_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      lk.unlock();
      drain();
      lk.lock();
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::mutex run_m_, m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int64_t)>* fn_ = nullptr;
  std::atomic<int64_t> next_{0};
  int64_t nchunks_ = 0;
  int active_ = 0;
  uint64_t gen_ = 0;
  size_t th_ = 0;
};

Pool& pool() {
  // never destroyed: detached workers may still wait on it at exit.  A forked
  // child gets a fresh pool (its copy's workers and lock state are not usable).
  static std::atomic<Pool*> p{nullptr};
  static std::atomic<pid_t> owner{0};
  static std::mutex init_m;  // (held for a moment; first use from several threads)
  Pool* q = p.load();
  if (!q || owner.load() != getpid()) {
    std::lock_guard<std::mutex> g(init_m);
    q = p.load();
    if (!q || owner.load() != getpid()) {
      q = new Pool;
      p.store(q);
      owner.store(getpid());
    }
  }
  return *q;
}

}  // namespace

extern "C" int vmi_poses_to_mats(const double* poses, int64_t n, double* mats, int threads) {
  if (n < 0 || (n > 0 && (!poses || !mats))) return -1;
  std::atomic<bool> bad{false};  // a non-finite component: -2 (EulerPose validation, geometry.py:68-102)
  auto work = [&](int64_t lo, int64_t hi) {
    bool nf = false;
    for (int64_t p = lo; p < hi; ++p) {
      const double* v = poses + 6 * p;
      double* m = mats + 12 * p;
      nf |= !(std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]) &&
              std::isfinite(v[3]) && std::isfinite(v[4]) && std::isfinite(v[5]));
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
    if (nf) bad.store(true);
  };
  int hw = (int)std::thread::hardware_concurrency();
  if (threads <= 0) {
    // one process per GPU (torchrun): share the host cores between the local ranks
    const char* lws = std::getenv("LOCAL_WORLD_SIZE");
    const int ranks = lws ? std::max(1, std::atoi(lws)) : 1;
    threads = hw > 0 ? std::max(1, hw / ranks) : 1;
  }
  if (n < 512 || threads == 1) {
    work(0, n);
    return bad.load() ? -2 : 0;
  }
  if (threads > 64) threads = 64;
  const int64_t chunk = std::max<int64_t>(256, (n + 4 * threads - 1) / (4 * threads));
  const int64_t nchunks = (n + chunk - 1) / chunk;
  const std::function<void(int64_t)> fn = [&](int64_t k) {
    work(k * chunk, std::min(n, (k + 1) * chunk));
  };
  pool().run(threads - 1, nchunks, fn);
  return bad.load() ? -2 : 0;
}
