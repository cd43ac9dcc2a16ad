// launch_worker.hpp — host threads that submit one device's share of a collective call
// (comm.cpp). Header-only so the hand-off protocol is unit-tested on the CPU
// (tests/test_launch_worker.py).
#pragma once

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>

// One host thread per extra device of a one-process communicator. An eager call submits to
// every device (a cooperative launch costs ~4 us of host time, tools/capi_latency.cpp); the
// workers submit to their devices while the calling thread does the first, so a call costs one
// launch instead of one per device. A worker sleeps on a condition variable between jobs (it can
// be made to spin a while first, PAT_WORKER_SPIN_US).
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
  __builtin_ia32_pause();
#elif defined(__aarch64__)
  asm volatile("yield" ::: "memory");
#endif
}

struct LaunchWorker {
  std::thread th;
  std::atomic<uint32_t> posted{0}, finished{0};
  std::atomic<bool> stop{false}, sleeping{false};
  std::mutex m;
  std::condition_variable cv;
  // busy-wait after a job before sleeping (PAT_WORKER_SPIN_US, comm.cpp). Default 0: a spinning
  // worker cut a one-process job's host-side copies (bench e2e) to a third (2 GPUs: 12 vs 29 GB/s)
  // while saving ~4 us only on isolated eager calls (profiles/r02_worker_spin_*)
  int64_t spin_us = 0;
  const std::function<int()>* job = nullptr;  // valid while posted != finished
  int result = 0;

  void run() {
    uint32_t seen = 0;
    for (;;) {
      auto t0 = std::chrono::steady_clock::now();
      uint32_t spins = 0;
      while (posted.load(std::memory_order_acquire) == seen && !stop.load(std::memory_order_relaxed)) {
        cpu_relax();  // an SMT sibling (e.g. the thread copying a step's inputs) keeps its issue slots
        if ((++spins & 255u) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(spin_us)) {
          std::unique_lock<std::mutex> lk(m);
          // store-buffering pair with post(): sleeping.store / posted.load here against
          // posted.fetch_add / sleeping.load there. Both loads must be seq_cst, or each side may
          // read the other's stale value (an acquire load may be LDAPR on armv8.3+) and the
          // worker sleeps through a post.
          sleeping.store(true, std::memory_order_seq_cst);
          cv.wait(lk, [&] { return posted.load(std::memory_order_seq_cst) != seen || stop.load(); });
          sleeping.store(false, std::memory_order_relaxed);
          t0 = std::chrono::steady_clock::now();
        }
      }
      if (stop.load()) return;
      seen = posted.load(std::memory_order_acquire);
      result = (*job)();
      finished.store(seen, std::memory_order_release);
    }
  }
  void post(const std::function<int()>* j) {
    job = j;
    posted.fetch_add(1, std::memory_order_seq_cst);
    if (sleeping.load(std::memory_order_seq_cst)) {
      std::lock_guard<std::mutex> lk(m);
      cv.notify_one();
    }
  }
  int wait() {
    const uint32_t want = posted.load(std::memory_order_relaxed);
    while (finished.load(std::memory_order_acquire) != want) std::this_thread::yield();
    return result;
  }
  void shutdown() {
    {
      std::lock_guard<std::mutex> lk(m);
      stop.store(true);
    }
    cv.notify_one();
    if (th.joinable()) th.join();
  }
};
