// Drop-in check: runs reference run specs (proj/corpus/*.json style) through
// the reference's own load_run_config + materialize, then through
// execute_mode("oracle") and the added execute_mode("b200"), and verifies
// them the way cmd_run --verify does (verify_against_oracle, driver.cpp:269:
// int64 bit-equal; real within the device tolerance). Prints one JSON line
// per spec and exits 5 (kExitVerifyMismatch) on any mismatch.
#include <cstdio>
#include <exception>
#include <iostream>

#include "ixsum_b200_mode.hpp"

int main(int argc, char** argv) {
  int rc = 0;
  for (int a = 1; a < argc; ++a) {
    try {
      ixsum::RunConfig cfg = ixsum::load_run_config(argv[a]);
      ixsum::BoundProblem prob = ixsum::materialize(cfg);
      ixsum::ModeResult ref = ixsum::b200::execute_mode("oracle", prob);
      ixsum::ModeResult dev = ixsum::b200::execute_mode("b200", prob);
      bool ok;
      double err = 0.0;
      if (ref.result.is_int()) {
        ok = ref.result.bit_equal(dev.result);
      } else {
        err = ixsum::max_rel_error(ref.result, dev.result);
        ok = err <= 1e-2;
      }
      std::printf("{\"spec\": \"%s\", \"ok\": %s, \"rel_err\": %.3g, \"b200_ms\": %.3f, "
                  "\"oracle_ms\": %.3f, \"gathers\": %lld, \"scatters\": %lld}\n",
                  argv[a], ok ? "true" : "false", err, dev.wall_ms, ref.wall_ms,
                  static_cast<long long>(dev.counters.gathers),
                  static_cast<long long>(dev.counters.scatters));
      if (!ok) rc = ixsum::kExitVerifyMismatch;
    } catch (const std::exception& e) {
      rc = ixsum::report_error(std::cerr, e);
    }
  }
  return rc;
}
