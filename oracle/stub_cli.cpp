// TEST INFRASTRUCTURE ONLY. pars::run_cli (proj/include/pars/cli.hpp:9)
// stand-in for the acceptance binary: the reference's cli.cpp needs CLI11,
// which is absent here, and the CLI is out of scope. Only
// acceptance check 12 (byte-identical CLI reruns, acceptance_main.cpp:683-753)
// calls it; it reports failure so that check fails loudly instead of passing.
#include <cstdio>

#include "pars/cli.hpp"

namespace pars {
int run_cli(int, const char* const*) {
  std::fprintf(stderr, "run_cli: the CLI is not built in this harness (CLI11 absent)\n");
  return 2;
}
}  // namespace pars
