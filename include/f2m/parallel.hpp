// f2m/parallel.hpp — the reference's data-parallel helpers (parallel.hpp / parallel.cpp:5-106) for
// code that still calls the pooled internal entry points (dual.hpp:83-87).
//
// On the B200 the sweeps, the dual objective and the extraction run on the GPU grid, so the pool
// never does solver work: the pooled overloads of jacobi_sweep / dual_objective_pooled accept it
// and ignore it. ThreadPool itself is a small, complete host pool (chunked index ranges, calling
// thread participates, exceptions rethrown on the caller) so that caller code using it for its own
// loops keeps working. Chunk boundaries depend only on the item count (kNodeChunk / kEdgeChunk),
// as in the reference.
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

namespace f2m {
inline namespace b200 {

inline constexpr std::int64_t kNodeChunk = 2048;
inline constexpr std::int64_t kEdgeChunk = 8192;

inline int default_thread_count() {
  const unsigned hw = std::thread::hardware_concurrency();
  return hw ? static_cast<int>(hw) : 1;
}

inline std::int64_t chunk_count(std::int64_t items, std::int64_t chunk) {
  return items > 0 ? (items + chunk - 1) / chunk : 0;
}

class ThreadPool {
 public:
  explicit ThreadPool(int threads) {
    const int extra = threads > 1 ? threads - 1 : 0;
    for (int i = 0; i < extra; ++i) threads_.emplace_back([this] { serve(); });
  }
  ~ThreadPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      quit_ = true;
      ++epoch_;
    }
    cv_work_.notify_all();
    for (std::thread& t : threads_) t.join();
  }
  ThreadPool(const ThreadPool&) = delete;
  ThreadPool& operator=(const ThreadPool&) = delete;

  int thread_count() const { return static_cast<int>(threads_.size()) + 1; }

  // body(chunk_index, begin, end) for every chunk of [0, items); returns when all are done
  void for_chunks(std::int64_t items, std::int64_t chunk,
                  const std::function<void(std::int64_t, std::int64_t, std::int64_t)>& body) {
    if (items <= 0) return;
    if (chunk < 1) chunk = 1;
    const std::int64_t chunks = chunk_count(items, chunk);
    if (threads_.empty() || chunks == 1) {
      for (std::int64_t c = 0; c < chunks; ++c) body(c, c * chunk, std::min(items, (c + 1) * chunk));
      return;
    }
    Job job{&body, items, chunk, chunks};
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &job;
      ++epoch_;
    }
    cv_work_.notify_all();
    work(job);
    std::unique_lock<std::mutex> lk(mu_);
    cv_done_.wait(lk, [&] { return job.finished.load() == chunks && busy_ == 0; });
    job_ = nullptr;
    if (job.error) std::rethrow_exception(job.error);
  }

 private:
  struct Job {
    const std::function<void(std::int64_t, std::int64_t, std::int64_t)>* body;
    std::int64_t items, chunk, chunks;
    std::atomic<std::int64_t> next{0};
    std::atomic<std::int64_t> finished{0};
    std::exception_ptr error;
    std::mutex error_mu;
  };

  static void work(Job& job) {
    for (std::int64_t c; (c = job.next.fetch_add(1)) < job.chunks;) {
      try {
        (*job.body)(c, c * job.chunk, std::min(job.items, (c + 1) * job.chunk));
      } catch (...) {
        std::lock_guard<std::mutex> lk(job.error_mu);
        if (!job.error) job.error = std::current_exception();
      }
      job.finished.fetch_add(1);
    }
  }

  void serve() {
    std::uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_work_.wait(lk, [&] { return epoch_ != seen; });
      seen = epoch_;
      if (quit_) return;
      Job* job = job_;
      if (!job) continue;
      ++busy_;
      lk.unlock();
      work(*job);
      lk.lock();
      --busy_;
      cv_done_.notify_all();
    }
  }

  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable cv_work_, cv_done_;
  Job* job_ = nullptr;
  std::uint64_t epoch_ = 0;
  int busy_ = 0;
  bool quit_ = false;
};

// partials combined in ascending chunk order (one left-to-right fp64 chain)
inline double combine_partials(const std::vector<double>& partials) {
  double total = 0.0;
  for (const double p : partials) total += p;
  return total;
}

}  // namespace b200
}  // namespace f2m
