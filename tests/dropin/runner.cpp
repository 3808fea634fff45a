// Runs every registered case (see doctest.h); exit code = failing cases.
#include <cstdio>
#include <cstring>
#include <exception>

#include "doctest.h"

// argv: substrings of case names to skip (cases outside the drop-in's scope)
int main(int argc, char** argv) {
  int bad = 0, skipped = 0;
  for (const auto& c : doctest::registry()) {
    bool skip = false;
    for (int i = 1; i < argc; ++i) skip = skip || std::strstr(c.name, argv[i]) != nullptr;
    if (skip) {
      std::printf("SKIP %s\n", c.name);
      ++skipped;
      continue;
    }
    const int before = doctest::failures();
    bool threw = false;
    try {
      c.fn();
    } catch (const doctest::Failed&) {
    } catch (const std::exception& e) {
      std::printf("    exception: %s\n", e.what());
      threw = true;
    }
    const bool ok = !threw && doctest::failures() == before;
    bad += !ok;
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", c.name);
  }
  std::printf("%d cases, %d skipped, %d failed\n", int(doctest::registry().size()), skipped, bad);
  return bad;
}
