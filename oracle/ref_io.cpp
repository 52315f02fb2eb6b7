// TEST INFRASTRUCTURE ONLY: file-format entry points of the unmodified
// reference library, one process per call (C++ exceptions thrown inside the
// reference crash a Python process that has numpy's bundled runtime loaded,
// so the ctypes bridge cannot exercise these error paths).
//   ref_io mtx <path>        -> JSON of load_matrix_market (or {"error": what})
//   ref_io convert <input> <out_dir> <format> <g> <group_dim> [bM bK] [prefix]
//                            -> cmd_convert (the reference CLI needs the absent CLI11)
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <string>
#include <variant>

#include "ixsum/driver.hpp"
#include "ixsum/matrix_market.hpp"

namespace {

void print_values(const ixsum::Tensor& t) {
  std::printf("[");
  const int64_t n = t.numel();
  for (int64_t i = 0; i < n; ++i) {
    if (t.is_int()) std::printf("%s%lld", i ? "," : "", static_cast<long long>(t.ints()[i]));
    else std::printf("%s%.17g", i ? "," : "", t.reals()[i]);
  }
  std::printf("]");
}

void print_ints(const std::vector<int64_t>& v) {
  std::printf("[");
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%lld", i ? "," : "", static_cast<long long>(v[i]));
  std::printf("]");
}

std::string json_escape(const std::string& s) {
  std::string o;
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 3 && std::string(argv[1]) == "mtx") {
    try {
      ixsum::MatrixMarketData d = ixsum::load_matrix_market(argv[2]);
      if (std::holds_alternative<ixsum::Tensor>(d)) {
        const ixsum::Tensor& t = std::get<ixsum::Tensor>(d);
        std::printf("{\"kind\":%d,\"shape\":[%lld,%lld],\"dense\":", t.is_int() ? 1 : 0,
                    static_cast<long long>(t.dim(0)), static_cast<long long>(t.dim(1)));
        print_values(t);
        std::printf("}\n");
      } else {
        const ixsum::CooMatrix& c = std::get<ixsum::CooMatrix>(d);
        std::printf("{\"kind\":%d,\"rows\":%lld,\"cols\":%lld,\"row\":", c.values.is_int() ? 1 : 0,
                    static_cast<long long>(c.rows), static_cast<long long>(c.cols));
        print_ints(c.row_coord);
        std::printf(",\"col\":");
        print_ints(c.col_coord);
        std::printf(",\"values\":");
        print_values(c.values);
        std::printf("}\n");
      }
    } catch (const std::exception& e) {
      std::printf("{\"error\":\"%s\"}\n", json_escape(e.what()).c_str());
    }
    return 0;
  }
  if (argc >= 7 && std::string(argv[1]) == "convert") {
    ixsum::ConvertConfig cfg;
    cfg.input = argv[2];
    cfg.out_dir = argv[3];
    cfg.format = argv[4];
    cfg.g = std::atoll(argv[5]);
    cfg.group_dim = std::atoi(argv[6]);
    if (argc >= 9 && std::atoll(argv[7]) > 0) cfg.block = {std::atoll(argv[7]), std::atoll(argv[8])};
    if (argc >= 10) cfg.prefix = argv[9];
    if (const char* m = std::getenv("IXR_MEASURE")) cfg.measure = std::atoi(m) != 0;  // --measure
    try {
      return ixsum::cmd_convert(cfg, std::cout, std::cerr);
    } catch (const std::exception& e) {
      return ixsum::report_error(std::cerr, e);
    }
  }
  std::cerr << "usage: ref_io mtx <path> | ref_io convert input out_dir format g group_dim [bM bK] [prefix]\n";
  return 1;
}
