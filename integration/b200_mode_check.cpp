// Drop-in check, linked against the reference library compiled in place
// (oracle/_ref) and libixb.so; run on the GPU box by
// tests/test_gpu_integration.py.
//
//   b200_mode_check spec.json ...   For each reference run spec: the
//       reference's load_run_config, then ixsum::materialize (host builders)
//       and ixsum::b200::materialize (device builders) — every bound operand,
//       format byte count and tuner report must be identical — then
//       execute_mode("oracle") on the reference problem against the added
//       execute_mode("b200") on the device-built one, verified like
//       cmd_run --verify (driver.cpp:269: int64 bit-equal; real within
//       b200::device_tolerance: 1e-5 fp32 SpMM, 1e-2 bf16 operands).
//   b200_mode_check --builders      The drop-in builders against the
//       reference builders at BASELINE scale: cfg1's 4096^2 1 % matrix
//       (dense_to_coo, tuner report, coo_to_groupcoo on both dims,
//       canonicalize of a shuffled copy), cfg2's 8192^2 16x16-block matrix
//       (dense_to_blockgroupcoo on both dims) and rank-3/4 COO tensors
//       (group_coo_tensor on every dim), real and int64 values.
// Prints one JSON line per check and exits 5 (kExitVerifyMismatch) on any
// mismatch.
#include <algorithm>
#include <cstdio>
#include <exception>
#include <iostream>
#include <random>
#include <string>

#include "ixsum/synth.hpp"
#include "ixsum_b200_formats.hpp"
#include "ixsum_b200_mode.hpp"

namespace {

using namespace ixsum;

bool same_report(const TuneReport& a, const TuneReport& b) {
  return a.chosen == b.chosen && a.gstar == b.gstar && a.candidates == b.candidates &&
         a.brute_optimal == b.brute_optimal;
}

// Every operand, the output buffer, format bytes and tuner reports.
bool same_problem(const BoundProblem& a, const BoundProblem& b, std::string& why) {
  if (a.tensors.size() != b.tensors.size()) {
    why = "operand sets differ";
    return false;
  }
  for (const auto& [name, t] : a.tensors) {
    auto it = b.tensors.find(name);
    if (it == b.tensors.end()) {
      why = "missing operand " + name;
      return false;
    }
    if (!t.same_shape(it->second) || t.kind() != it->second.kind() || !t.bit_equal(it->second)) {
      why = "operand " + name + " differs";
      return false;
    }
  }
  if (!a.out.bit_equal(b.out)) {
    why = "output buffer differs";
    return false;
  }
  if (a.format_bytes != b.format_bytes) {
    why = "format bytes differ";
    return false;
  }
  if (a.tuner_reports.size() != b.tuner_reports.size()) {
    why = "tuner report sets differ";
    return false;
  }
  for (const auto& [name, r] : a.tuner_reports) {
    auto it = b.tuner_reports.find(name);
    if (it == b.tuner_reports.end() || !same_report(r, it->second)) {
      why = "tuner report " + name + " differs";
      return false;
    }
  }
  if (!(a.stmt == b.stmt)) {
    why = "statement differs";
    return false;
  }
  return true;
}

bool same(const GroupCooMatrix& a, const GroupCooMatrix& b) {
  return a.rows == b.rows && a.cols == b.cols && a.group_dim == b.group_dim &&
         a.group_size == b.group_size && a.group_coord == b.group_coord &&
         a.member_coord == b.member_coord && a.values.same_shape(b.values) &&
         a.values.bit_equal(b.values) && a.pad_mask == b.pad_mask;
}

bool same(const BlockGroupCooMatrix& a, const BlockGroupCooMatrix& b) {
  return a.rows == b.rows && a.cols == b.cols && a.block_rows == b.block_rows &&
         a.block_cols == b.block_cols && a.group_dim == b.group_dim &&
         a.group_size == b.group_size && a.group_coord == b.group_coord &&
         a.member_coord == b.member_coord && a.values.same_shape(b.values) &&
         a.values.bit_equal(b.values) && a.pad_mask == b.pad_mask;
}

bool same(const GroupCooTensor& a, const GroupCooTensor& b) {
  return a.shape == b.shape && a.group_dim == b.group_dim && a.group_size == b.group_size &&
         a.group_coord == b.group_coord && a.member_coords == b.member_coords &&
         a.member_dims == b.member_dims && a.values.same_shape(b.values) &&
         a.values.bit_equal(b.values) && a.pad_mask == b.pad_mask;
}

int report(const char* what, bool ok, const std::string& extra = "") {
  std::printf("{\"check\": \"%s\", \"ok\": %s%s}\n", what, ok ? "true" : "false", extra.c_str());
  std::fflush(stdout);
  return ok ? 0 : kExitVerifyMismatch;
}

int check_builders() {
  int rc = 0;
  for (ElemKind kind : {ElemKind::Real64, ElemKind::Int64}) {
    const std::string k = kind == ElemKind::Int64 ? "int" : "real";
    // cfg1: materialize order (driver.cpp:169-186): dense B first, then A
    Rng rng(1);
    synth_dense({4096, 128}, kind, rng);
    Tensor A = synth_sparse_matrix(4096, 4096, 0.01, kind, rng);
    CooMatrix ref_coo = dense_to_coo(A);
    CooMatrix dev_coo = b200::dense_to_coo(A);
    rc |= report(("cfg1 dense_to_coo " + k).c_str(), structurally_equal(ref_coo, dev_coo) &&
                                                       dev_coo.canonical,
                 ", \"nnz\": " + std::to_string(dev_coo.nnz()));
    for (int dim : {0, 1}) {
      TuneReport rr = select(OccProfile::from_coo(ref_coo, dim));
      TuneReport dr = b200::tune(dev_coo, dim);
      rc |= report(("cfg1 tuner dim" + std::to_string(dim) + " " + k).c_str(),
                   same_report(rr, dr), ", \"g\": " + std::to_string(dr.chosen));
      GroupCooMatrix rg = coo_to_groupcoo(ref_coo, dim, rr.chosen);
      GroupCooMatrix dg = b200::coo_to_groupcoo(dev_coo, dim, dr.chosen);
      rc |= report(("cfg1 coo_to_groupcoo dim" + std::to_string(dim) + " " + k).c_str(),
                   same(rg, dg), ", \"G\": " + std::to_string(dg.num_groups()));
      // the helpers around the format (formats.cpp:105-113, 176-208)
      rc |= report(("cfg1 real/pad_count, is_ell, groupcoo_to_coo dim" + std::to_string(dim) +
                    " " + k).c_str(),
                   rg.real_count() == b200::real_count(dg) &&
                       rg.pad_count() == b200::pad_count(dg) && is_ell(rg) == b200::is_ell(dg) &&
                       structurally_equal(groupcoo_to_coo(rg), b200::groupcoo_to_coo(dg)));
      GroupCooMatrix re = ell_view(ref_coo, dim), de = b200::ell_view(dev_coo, dim);
      rc |= report(("cfg1 ell_view dim" + std::to_string(dim) + " " + k).c_str(),
                   same(re, de) && is_ell(re) == b200::is_ell(de),
                   ", \"g\": " + std::to_string(de.group_size));
    }
    // canonicalize + grouping of an unsorted (shuffled) COO
    CooMatrix shuf = ref_coo;
    std::vector<int64_t> perm(static_cast<size_t>(shuf.nnz()));
    for (size_t i = 0; i < perm.size(); ++i) perm[i] = static_cast<int64_t>(i);
    std::shuffle(perm.begin(), perm.end(), std::mt19937_64(7));
    for (size_t i = 0; i < perm.size(); ++i) {
      shuf.row_coord[i] = ref_coo.row_coord[static_cast<size_t>(perm[i])];
      shuf.col_coord[i] = ref_coo.col_coord[static_cast<size_t>(perm[i])];
      shuf.values.copy_elem_from(static_cast<int64_t>(i), ref_coo.values, perm[i]);
    }
    shuf.canonical = false;
    rc |= report(("cfg1 canonicalize shuffled " + k).c_str(),
                 structurally_equal(canonicalize(shuf), b200::canonicalize(shuf)));
    rc |= report(("cfg1 coo_to_groupcoo shuffled g=5 " + k).c_str(),
                 same(coo_to_groupcoo(shuf, 0, 5), b200::coo_to_groupcoo(shuf, 0, 5)));
    // cfg2: 8192^2, 16x16 blocks at 10 %, g = 8 (the tuner's choice)
    Rng rng2(1);
    synth_dense({512, 16, 512}, kind, rng2);
    Tensor A2 = synth_block_sparse_matrix(8192, 8192, 16, 16, 0.10, kind, rng2);
    for (int dim : {0, 1}) {
      BlockGroupCooMatrix rb = dense_to_blockgroupcoo(A2, 16, 16, 8, dim);
      BlockGroupCooMatrix db = b200::dense_to_blockgroupcoo(A2, 16, 16, 8, dim);
      rc |= report(("cfg2 dense_to_blockgroupcoo dim" + std::to_string(dim) + " " + k).c_str(),
                   same(rb, db), ", \"G\": " + std::to_string(db.num_groups()));
    }
    // ragged blocks (5x6 with 4x4 blocks, test_formats.cpp:197-205 shape)
    Rng rng3(3);
    Tensor A3 = synth_sparse_matrix(37, 53, 0.2, kind, rng3);
    rc |= report(("ragged dense_to_blockgroupcoo " + k).c_str(),
                 same(dense_to_blockgroupcoo(A3, 4, 4, 3, 0),
                      b200::dense_to_blockgroupcoo(A3, 4, 4, 3, 0)));
    // rank-3 and rank-4 COO tensors (conv map / CG shapes), every group dim
    Rng rng4(5);
    CooTensor c3 = synth_coo_tensor({300, 300, 27}, 20000, kind, rng4);
    CooTensor c4 = synth_coo_tensor({16, 16, 16, 23}, 353, kind, rng4);
    bool all_ok = true;
    for (const CooTensor* c : {&c3, &c4}) {
      for (int d = 0; d < c->rank(); ++d) {
        for (int64_t g : {1, 4, 16}) {
          if (!same(group_coo_tensor(*c, d, g), b200::group_coo_tensor(*c, d, g))) {
            all_ok = false;
            report(("group_coo_tensor rank" + std::to_string(c->rank()) + " dim" +
                    std::to_string(d) + " g" + std::to_string(g) + " " + k)
                       .c_str(),
                   false);
          }
        }
      }
    }
    rc |= report(("group_coo_tensor rank 3/4, every dim, g 1/4/16 " + k).c_str(), all_ok);
  }
  // errors: the reference's exception types and messages
  Tensor r3 = Tensor::zeros(ElemKind::Real64, {2, 2, 2});
  auto msg = [](auto&& f) -> std::string {
    try {
      f();
    } catch (const std::exception& e) {
      return e.what();
    }
    return "<no error>";
  };
  const bool same_err =
      msg([&] { dense_to_coo(r3); }) == msg([&] { b200::dense_to_coo(r3); }) &&
      msg([&] { coo_to_groupcoo(CooMatrix{}, 0, 0); }) ==
          msg([&] { b200::coo_to_groupcoo(CooMatrix{}, 0, 0); }) &&
      msg([&] { coo_to_groupcoo(CooMatrix{}, 2, 1); }) ==
          msg([&] { b200::coo_to_groupcoo(CooMatrix{}, 2, 1); }) &&
      msg([&] { dense_to_blockgroupcoo(r3, 2, 2, 1); }) ==
          msg([&] { b200::dense_to_blockgroupcoo(r3, 2, 2, 1); });
  rc |= report("builder errors (types and messages)", same_err);
  return rc;
}

}  // namespace

int main(int argc, char** argv) {
  int rc = 0;
  for (int a = 1; a < argc; ++a) {
    const std::string arg = argv[a];
    if (arg == "--builders") {
      try {
        rc |= check_builders();
      } catch (const std::exception& e) {
        rc = ixsum::report_error(std::cerr, e);
      }
      continue;
    }
    try {
      ixsum::RunConfig cfg = ixsum::load_run_config(arg);
      ixsum::BoundProblem ref_prob = ixsum::materialize(cfg);
      ixsum::BoundProblem dev_prob = ixsum::b200::materialize(cfg);
      std::string why;
      const bool formats_ok = same_problem(ref_prob, dev_prob, why);
      ixsum::ModeResult ref = ixsum::b200::execute_mode("oracle", ref_prob);
      ixsum::ModeResult dev = ixsum::b200::execute_mode("b200", dev_prob);
      bool ok;
      double err = 0.0;
      const double tol = ixsum::b200::device_tolerance(dev_prob.stmt);
      if (ref.result.is_int()) {
        ok = ref.result.bit_equal(dev.result);
      } else {
        err = ixsum::max_rel_error(ref.result, dev.result);
        ok = err <= tol;
      }
      std::printf("{\"spec\": \"%s\", \"ok\": %s, \"formats_identical\": %s, \"why\": \"%s\", "
                  "\"rel_err\": %.3g, \"tol\": %g, \"b200_ms\": %.3f, \"oracle_ms\": %.3f, "
                  "\"gathers\": %lld, \"scatters\": %lld}\n",
                  arg.c_str(), ok && formats_ok ? "true" : "false",
                  formats_ok ? "true" : "false", why.c_str(), err, tol, dev.wall_ms,
                  ref.wall_ms, static_cast<long long>(dev.counters.gathers),
                  static_cast<long long>(dev.counters.scatters));
      if (!ok || !formats_ok) rc = ixsum::kExitVerifyMismatch;
    } catch (const std::exception& e) {
      rc = ixsum::report_error(std::cerr, e);
    }
  }
  return rc;
}
