// Prints binary16 bits of dmath_b200::detail::half_from_double for doubles read
// from stdin (one per line, as hex bit patterns); tests/test_cpp_api.py compares
// them with numpy's round-to-nearest-even float64 -> float16 conversion.
#include <cinttypes>
#include <cstdio>
#include <cstring>

#include "dmath_b200.hpp"

int main() {
  unsigned long long bits;
  while (std::scanf("%llx", &bits) == 1) {
    double v;
    std::memcpy(&v, &bits, 8);
    std::printf("%04x\n", static_cast<unsigned>(dmath_b200::detail::half_from_double(v)));
  }
  return 0;
}
