// Sense-reversing spin barrier for small teams of host threads that step through microsecond-
// scale phases together (the reflectors of the dense Householder reduction, the row scans of
// the dense-block search): far cheaper than a condition variable at that grain.  Members that
// wait long yield the core.
#pragma once

#include <atomic>
#include <thread>

namespace flz {

class SpinBarrier {
 public:
  explicit SpinBarrier(unsigned count) : count_(count) {}
  void wait() {
    const unsigned gen = generation_.load(std::memory_order_acquire);
    if (arrived_.fetch_add(1, std::memory_order_acq_rel) + 1 == count_) {
      arrived_.store(0, std::memory_order_relaxed);
      generation_.store(gen + 1, std::memory_order_release);
    } else {
      unsigned spins = 0;
      while (generation_.load(std::memory_order_acquire) == gen)
        if (++spins > 4096) std::this_thread::yield();
    }
  }

 private:
  const unsigned count_;
  std::atomic<unsigned> arrived_{0}, generation_{0};
};

}  // namespace flz
