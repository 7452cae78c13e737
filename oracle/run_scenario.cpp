// Runs the UNMODIFIED reference DES driver (moesim::run_scenario,
// proj/core/include/moesim/driver.hpp:20-21) on a scenario JSON: test
// infrastructure for tests/test_des_b200.py, which feeds it the cost model
// measured on the B200 (profiles/r01_cost_model.json).  A separate process
// rather than a call through libmoesim_ref.so: the driver's std::async /
// std::filesystem code needs the libstdc++ it was built with, not the one a
// Python process has already loaded.
#include <cstdio>

#include "moesim/driver.hpp"

int main(int argc, char** argv) {
  if (argc != 3) {
    std::fprintf(stderr, "usage: run_scenario <scenario.json> <output_dir>\n");
    return 2;
  }
  moesim::RunOverrides o;
  o.quiet = true;
  const int failed = moesim::run_scenario(argv[1], argv[2], o);
  std::printf("failed %d\n", failed);
  return failed == 0 ? 0 : 1;
}
