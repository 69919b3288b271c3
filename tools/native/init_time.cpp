// Times the first engine call of a process (CUDA context + module load) and
// a second one, to separate start-up cost from work in CLI timings.
#include <chrono>
#include <cstdio>
#include <cstdint>
#include "tsv.h"
int main() {
  using C = std::chrono::steady_clock;
  uint64_t a = 3, b = 5, out = 0;
  auto t0 = C::now();
  int rc = tsv_gf_mul_device(0, 1, &a, &b, &out);
  auto t1 = C::now();
  rc |= tsv_gf_mul_device(0, 1, &a, &b, &out);
  auto t2 = C::now();
  std::printf("rc=%d first call %.1f ms, second %.3f ms\n", rc,
              std::chrono::duration<double, std::milli>(t1 - t0).count(),
              std::chrono::duration<double, std::milli>(t2 - t1).count());
  return rc;
}
