// Minimal persistent host thread pool for the lockstep search: the GA steps
// of independent arms (candidate generation, population bookkeeping) and the
// packing of a wave run in parallel between GPU waves.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace hpg {

class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }

  // Runs fn(i) for i in [0, n); the caller participates. Blocks until done.
  // Callers from different threads (separate engine contexts) take turns.
  void run(int n, const std::function<void(int)>& fn) {
    if (workers_.empty() || n <= 1) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    std::lock_guard<std::mutex> call_lock(call_m_);
    {
      std::lock_guard<std::mutex> lk(m_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      pending_ = static_cast<int>(workers_.size());
      ++gen_;
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  HostPool() {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int n = static_cast<int>(std::min(16u, hw)) - 1;
    for (int i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }

  void drain() {
    for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*fn_)(i);
  }

  void loop() {
    long seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
      }
      drain();
      {
        std::lock_guard<std::mutex> lk(m_);
        if (--pending_ == 0) done_cv_.notify_one();
      }
    }
  }

  std::vector<std::thread> workers_;
  std::mutex m_, call_m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0};
  int pending_ = 0;
  long gen_ = 0;
  bool stop_ = false;
};

template <typename F>
inline void host_parallel_for(int n, bool parallel, F&& f) {
  if (!parallel) {
    for (int i = 0; i < n; ++i) f(i);
    return;
  }
  const std::function<void(int)> fn = f;
  HostPool::get().run(n, fn);
}

}  // namespace hpg
