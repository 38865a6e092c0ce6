// host_pool.h — a small persistent host thread pool per context, used to
// stage pageable caller buffers through the context's pinned buffers: worker
// threads copy 1 MiB chunks into pinned memory and enqueue each chunk's DMA
// right behind it, so the host copy of chunk k + 1 overlaps the DMA of chunk
// k (a pageable cudaMemcpyAsync would run both serially on the caller's
// thread), and downloaded row bands are copied out as their DMAs complete.
#pragma once

#include <atomic>
#include <condition_variable>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

namespace mfb {

class HostPool {
 public:
  explicit HostPool(int workers) {
    for (int i = 0; i < workers; ++i) threads_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : threads_) t.join();
  }
  int size() const { return static_cast<int>(threads_.size()); }

  // Starts fn(0..n-1) on the workers (indices handed out in increasing
  // order) and returns at once; wait() blocks until every index has run and
  // rethrows the first exception raised by fn. One job at a time per pool.
  void start(int n, std::function<void(int)> fn) {
    auto j = std::make_shared<Job>();
    j->fn = std::move(fn);
    j->n = n;
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = j;
      ++gen_;
    }
    cv_.notify_all();
  }
  void wait() {
    std::shared_ptr<Job> j;
    {
      std::unique_lock<std::mutex> lk(mu_);
      j = job_;
      if (!j) return;
      done_cv_.wait(lk, [&] { return j->done >= j->n; });
      job_.reset();
    }
    if (j->err) std::rethrow_exception(j->err);
  }
  void run(int n, std::function<void(int)> fn) {
    start(n, std::move(fn));
    wait();
  }

 private:
  struct Job {
    std::function<void(int)> fn;
    int n = 0;
    int done = 0;  // guarded by the pool mutex
    std::atomic<int> next{0};
    std::exception_ptr err;
  };

  void loop() {
    uint64_t seen = 0;
    for (;;) {
      std::shared_ptr<Job> j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_); });
        if (stop_) return;
        seen = gen_;
        j = job_;
      }
      int ran = 0;
      std::exception_ptr err;
      for (int i = j->next.fetch_add(1); i < j->n; i = j->next.fetch_add(1)) {
        try {
          j->fn(i);
        } catch (...) {
          if (!err) err = std::current_exception();
        }
        ++ran;
      }
      if (ran) {
        std::lock_guard<std::mutex> lk(mu_);
        if (err && !j->err) j->err = err;
        j->done += ran;
        if (j->done >= j->n) done_cv_.notify_all();
      }
    }
  }

  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::shared_ptr<Job> job_;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

}  // namespace mfb
