// prefault.hpp -- first touch of large host vectors on all threads.
//
// The drop-in's O(n) host arrays at BASELINE C5 (n = 1e8: the 2.4 GB shade
// CSR, the 800 MB accumulators, the 400 MB flagged list) are sized with
// std::vector::assign / resize, which zero-fill on ONE thread and take one
// page fault per 4 KB page on the way: ~0.4 s per GB.  reserve_prefaulted
// reserves the capacity and has the kernel populate the pages writable
// (madvise MADV_POPULATE_WRITE, Linux >= 5.14) on all OpenMP threads first;
// the following assign / resize then runs at memset speed.  No element is
// written here, and where the advice is not supported nothing changes.
#pragma once
#include <sys/mman.h>
#include <unistd.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#ifndef MADV_POPULATE_WRITE
#define MADV_POPULATE_WRITE 23
#endif

namespace tsieve::detail {

template <typename T>
void reserve_prefaulted(std::vector<T>& v, std::size_t n) {
  v.reserve(n);
  const std::size_t bytes = n * sizeof(T);
  if (bytes < (std::size_t{64} << 20)) return;
  const std::uintptr_t page = static_cast<std::uintptr_t>(::sysconf(_SC_PAGESIZE));
  const std::uintptr_t lo = (reinterpret_cast<std::uintptr_t>(v.data()) + page - 1) & ~(page - 1);
  const std::uintptr_t hi = (reinterpret_cast<std::uintptr_t>(v.data()) + bytes) & ~(page - 1);
  if (hi <= lo) return;
  const std::int64_t chunk = std::int64_t{32} << 20;
  const std::int64_t parts = static_cast<std::int64_t>((hi - lo + chunk - 1) / chunk);
#pragma omp parallel for schedule(dynamic, 1)
  for (std::int64_t i = 0; i < parts; ++i) {
    const std::uintptr_t a = lo + static_cast<std::uintptr_t>(i * chunk);
    const std::uintptr_t b = a + chunk < hi ? a + chunk : hi;
    (void)::madvise(reinterpret_cast<void*>(a), b - a, MADV_POPULATE_WRITE);
  }
}

}  // namespace tsieve::detail
