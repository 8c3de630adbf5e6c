// Test infrastructure: the reference's read_points (geometry.cpp:194-226)
// as a standalone tool -- prints n, then one line of five %.17g values per
// point, or "error: <what>" and exit 2.  (Its iostream CSV parsing crashes
// when the reference is loaded into the Python process through ctypes, so
// tests/test_harness_cpu.py runs it out of process.)
#include <cstdio>
#include <exception>

#include "ifgf/geometry.hpp"

int main(int argc, char** argv) {
  if (argc != 2) return 1;
  try {
    const ifgf::PointCloud pc = ifgf::read_points(argv[1]);
    std::printf("%zu\n", pc.size());
    for (std::size_t i = 0; i < pc.size(); ++i)
      std::printf("%.17g %.17g %.17g %.17g %.17g\n", pc.x1[i], pc.x2[i], pc.x3[i], pc.a_re[i],
                  pc.a_im[i]);
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 2;
  }
  return 0;
}
