// Host build of csrc/fastmath.cuh for tests/test_fastmath.py (the same
// arithmetic the device runs, minus the hardware reciprocal seed).
#include <cstdint>

#include "fastmath.cuh"

extern "C" void fm_eval_host(int kind, const double* x, double* y, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    const double v = x[i];
    y[i] = kind == 0 ? hpac::fm::exp(v)
         : kind == 1 ? hpac::fm::log(v)
         : kind == 2 ? hpac::fm::erfc(v)
                     : hpac::fm::div(1.0, v);
  }
}
