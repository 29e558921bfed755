// A persistent host worker pool for the planner's data-parallel loops
// (per-lightcone schedule construction, descriptor generation).  Spawning
// threads per call would cost more than the work at these sizes.
#pragma once

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <deque>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace qtng {

class Pool {
 public:
  static Pool& get() {
    static Pool p;
    return p;
  }
  int size() const { return static_cast<int>(workers_.size()) + 1; }

  // fn(i) for i in [0, n), on the workers and the calling thread.  Calls from
  // inside a task, or concurrent calls, run serially on the caller.  An
  // exception thrown by a task (on any thread) is rethrown here, on the
  // caller, after every worker has left the loop (the first one wins).
  void parallel_for(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    std::unique_lock<std::mutex> busy(run_mu_, std::try_to_lock);
    if (!busy.owns_lock() || n == 1 || workers_.empty()) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      err_ = nullptr;
      active_ = static_cast<int>(workers_.size());
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    drain();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
    if (err_) {
      std::exception_ptr e = err_;
      err_ = nullptr;
      std::rethrow_exception(e);
    }
  }

 private:
  // Threads (caller included) = QTNG_POOL_THREADS if set, else the hardware
  // threads minus four on hosts with >= 12 (minus two with >= 8): the
  // caller's process keeps other threads busy and the one-shot energy's
  // enqueue thread (Worker) runs beside the planner.  Measured one-shot C2
  // energy on 16 threads, medians of 3 runs: 16 -> 3.09-3.25 ms, 14 ->
  // 3.06-3.11, 12 -> 3.02-3.06, 8 -> 3.11-3.16 (before the enqueue thread:
  // 14 was best).
  Pool() {
    int hw = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    if (hw >= 12) hw -= 4;
    else if (hw >= 8) hw -= 2;
    if (const char* v = std::getenv("QTNG_POOL_THREADS")) hw = std::max(1, std::atoi(v));
    for (int t = 0; t < std::min(hw, 64) - 1; ++t) workers_.emplace_back([this] { loop(); });
  }
  ~Pool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void drain() {
    for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) {
      try {
        (*fn_)(i);
      } catch (...) {
        std::lock_guard<std::mutex> lk(err_mu_);
        if (!err_) err_ = std::current_exception();
        next_.store(n_);  // stop handing out work
      }
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      // spin briefly first: the planner issues several loops back to back and
      // a futex wake-up per loop would cost more than the loop itself
      bool woke = false;
      for (int k = 0; k < kSpin && !woke; ++k) {
        woke = gen_.load(std::memory_order_acquire) != seen;
        if (!woke) std::this_thread::yield();
      }
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        seen = gen_.load(std::memory_order_acquire);
        if (stop_) return;
      }
      drain();
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (--active_ == 0) done_cv_.notify_one();
      }
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_, err_mu_;
  std::exception_ptr err_;  // first task exception of the current loop
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* fn_ = nullptr;
  int n_ = 0;
  std::atomic<int> next_{0};
  int active_ = 0;
  std::atomic<uint64_t> gen_{0};
  static constexpr int kSpin = 2000;  // yields before sleeping on the condition variable
  bool stop_ = false;
};

// One background thread running submitted tasks in order: the one-shot
// energy enqueues chunk c (descriptor upload, kernel launches) on it while
// the calling thread plans chunk c + 1 on the pool.
class Worker {
 public:
  Worker() : t_([this] { loop(); }) {}
  ~Worker() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    t_.join();
  }
  void submit(std::function<void()> f) {
    {
      std::lock_guard<std::mutex> lk(mu_);
      q_.push_back(std::move(f));
    }
    cv_.notify_all();
  }
  // Blocks until every submitted task has run; rethrows the first exception
  // (tasks submitted after a failure are skipped).
  void wait() {
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return q_.empty() && !running_; });
    if (err_) {
      std::exception_ptr e = err_;
      err_ = nullptr;
      std::rethrow_exception(e);
    }
  }

 private:
  void loop() {
    for (;;) {
      std::function<void()> f;
      bool skip = false;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return;
        f = std::move(q_.front());
        q_.pop_front();
        running_ = true;
        skip = err_ != nullptr;
      }
      if (!skip) {
        try {
          f();
        } catch (...) {
          std::lock_guard<std::mutex> lk(mu_);
          if (!err_) err_ = std::current_exception();
        }
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        running_ = false;
      }
      done_cv_.notify_all();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::deque<std::function<void()>> q_;
  std::exception_ptr err_;
  bool running_ = false, stop_ = false;
  std::thread t_;  // last: started after the members it uses
};

}  // namespace qtng
