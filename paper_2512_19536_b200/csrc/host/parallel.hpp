// Host thread pool for one-time setup loops (assembly, factorisation).
// Disjoint-write contract as in /root/reference/proj/include/polydg/parallel.hpp:14-16,
// so results are independent of the schedule.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <exception>
#include <mutex>
#include <thread>
#include <vector>

namespace pdg {

inline int setup_threads() {
  int n = static_cast<int>(std::thread::hardware_concurrency());
  if (n < 1) n = 1;
  if (const char* env = std::getenv("POLYDG_THREADS")) {
    const int cap = std::atoi(env);
    if (cap >= 1) n = std::min(n, cap);
  }
  return std::min(n, 64);
}

// fn(i) for i in [0, n), dynamic chunks; rethrows the first exception.
template <class F>
void parallel_for(int n, F&& fn, int grain = 1) {
  const int workers = std::min(setup_threads(), std::max(1, n / std::max(grain, 1)));
  if (workers <= 1) {
    for (int i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<int> next{0};
  std::exception_ptr err;
  std::mutex mu;
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w)
    pool.emplace_back([&] {
      try {
        for (;;) {
          const int i = next.fetch_add(grain);
          if (i >= n) break;
          for (int k = i; k < std::min(n, i + grain); ++k) fn(k);
        }
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!err) err = std::current_exception();
        next.store(n);
      }
    });
  for (auto& t : pool) t.join();
  if (err) std::rethrow_exception(err);
}

}  // namespace pdg
