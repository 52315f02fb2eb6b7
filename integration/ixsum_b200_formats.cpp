// Drop-in format builders (see ixsum_b200_formats.hpp): the reference's
// builder signatures over the device builders of libixb.so. Each call moves
// the reference's host data to the device once (coordinates narrowed to the
// device's int32, values kept as their 8-byte fp64/int64 payload so the output
// arrays are byte-identical), runs the two-phase *_plan / *_pack builder and
// returns the reference struct.
#include "ixsum_b200_formats.hpp"

#include <memory>
#include <string>
#include <vector>

#include "b200_util.hpp"
#include "ixsum/matrix_market.hpp"
#include "ixsum/synth.hpp"

namespace ixsum::b200 {

using detail::check;
using detail::DevBuf;

namespace {

struct Pack {
  ixb_pack* p = nullptr;
  ~Pack() { ixb_pack_free(p); }
};

void sync() { detail::cuda_ok(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

}  // namespace

CooMatrix dense_to_coo(const Tensor& t) {
  if (t.rank() != 2) {
    throw ShapeError("dense_to_coo expects a rank-2 tensor, got rank " +
                     std::to_string(t.rank()));
  }
  CooMatrix c;
  c.rows = t.dim(0);
  c.cols = t.dim(1);
  c.canonical = true;
  auto dense = detail::upload_values(t);
  Pack pk;
  int64_t nnz = 0;
  check(ixb_dense_to_coo_plan(dense->p, detail::value_dtype(t), c.rows, c.cols, nullptr, &pk.p,
                              &nnz));
  DevBuf r(static_cast<size_t>(nnz) * 4), k(static_cast<size_t>(nnz) * 4),
      v(static_cast<size_t>(nnz) * 8);
  check(ixb_dense_to_coo_pack(pk.p, r.as<int32_t>(), k.as<int32_t>(), v.p, nullptr));
  sync();
  c.row_coord = detail::download_coords(r, nnz);
  c.col_coord = detail::download_coords(k, nnz);
  c.values = detail::download_values(v, t.kind(), {nnz});
  return c;
}

GroupCooMatrix coo_to_groupcoo(const CooMatrix& c, int group_dim, int64_t g) {
  // the reference's validation order and messages (formats.cpp:116-117)
  if (g < 1) throw ShapeError("group size must be >= 1, got " + std::to_string(g));
  if (group_dim != 0 && group_dim != 1) throw ShapeError("group_dim must be 0 or 1");
  GroupCooMatrix gc;
  gc.rows = c.rows;
  gc.cols = c.cols;
  gc.group_dim = group_dim;
  gc.group_size = g;
  const int64_t nnz = c.nnz();
  auto r = detail::upload_coords(c.row_coord, "row");
  auto k = detail::upload_coords(c.col_coord, "col");
  auto v = detail::upload_values(c.values);
  Pack pk;
  int64_t G = 0, g_used = 0;
  check(ixb_groupcoo_plan(r->as<int32_t>(), k->as<int32_t>(), nnz, c.rows, c.cols,
                          c.canonical ? 1 : 0, group_dim, g, nullptr, &pk.p, &G, &g_used));
  const size_t slots = static_cast<size_t>(G * g);
  DevBuf AM(static_cast<size_t>(G) * 4), AK(slots * 4), AV(slots * 8), mask(slots);
  check(ixb_groupcoo_pack(pk.p, v->p, detail::value_dtype(c.values), AM.as<int32_t>(),
                          AK.as<int32_t>(), AV.p, mask.as<uint8_t>(), nullptr));
  sync();
  gc.group_coord = detail::download_coords(AM, G);
  gc.member_coord = detail::download_coords(AK, G * g);
  gc.values = detail::download_values(AV, c.values.kind(), {G, g});
  gc.pad_mask = detail::download_mask(mask, G * g);
  return gc;
}

CooMatrix canonicalize(const CooMatrix& c) {
  // canonical COO == GroupCOO with g = 1 along rows (formats.cpp:68-89 order)
  CooMatrix in = c;
  in.canonical = false;
  GroupCooMatrix gc = b200::coo_to_groupcoo(in, 0, 1);
  CooMatrix out;
  out.rows = c.rows;
  out.cols = c.cols;
  out.row_coord = std::move(gc.group_coord);
  out.col_coord = std::move(gc.member_coord);
  out.values = gc.values.reshape({c.nnz()});
  out.canonical = true;
  return out;
}

int64_t real_count(const GroupCooMatrix& gc) {
  DevBuf mask(gc.pad_mask.size());
  detail::cuda_ok(cudaMemcpy(mask.p, gc.pad_mask.data(), gc.pad_mask.size(),
                             cudaMemcpyHostToDevice),
                  "cudaMemcpy H2D");
  int64_t n = 0;
  check(ixb_mask_real_count(mask.as<uint8_t>(), static_cast<int64_t>(gc.pad_mask.size()), nullptr,
                            &n));
  return n;
}

int64_t pad_count(const GroupCooMatrix& gc) {
  return static_cast<int64_t>(gc.pad_mask.size()) - b200::real_count(gc);
}

CooMatrix groupcoo_to_coo(const GroupCooMatrix& gc) {
  const int64_t G = gc.num_groups(), g = gc.group_size, slots = G * g;
  auto am = detail::upload_coords(gc.group_coord, "group");
  auto ak = detail::upload_coords(gc.member_coord, "member");
  auto av = detail::upload_values(gc.values);
  DevBuf mask(static_cast<size_t>(slots));
  detail::cuda_ok(cudaMemcpy(mask.p, gc.pad_mask.data(), static_cast<size_t>(slots),
                             cudaMemcpyHostToDevice),
                  "cudaMemcpy H2D");
  int64_t nnz = 0;
  check(ixb_mask_real_count(mask.as<uint8_t>(), slots, nullptr, &nnz));
  DevBuf r(static_cast<size_t>(nnz) * 4), k(static_cast<size_t>(nnz) * 4),
      v(static_cast<size_t>(nnz) * 8);
  check(ixb_groupcoo_to_coo(am->as<int32_t>(), ak->as<int32_t>(), av->p,
                            detail::value_dtype(gc.values), mask.as<uint8_t>(), G, g,
                            gc.group_dim, r.as<int32_t>(), k.as<int32_t>(), v.p, nullptr));
  sync();
  CooMatrix c;
  c.rows = gc.rows;
  c.cols = gc.cols;
  c.row_coord = detail::download_coords(r, nnz);
  c.col_coord = detail::download_coords(k, nnz);
  c.values = detail::download_values(v, gc.values.kind(), {nnz});
  return b200::canonicalize(c);  // formats.cpp:193
}

GroupCooMatrix ell_view(const CooMatrix& c, int group_dim) {
  if (group_dim != 0 && group_dim != 1) throw ShapeError("occupancy: dim must be 0 or 1");
  const auto& coord = group_dim == 0 ? c.row_coord : c.col_coord;
  auto d = detail::upload_coords(coord, group_dim == 0 ? "row" : "col");
  int64_t m = 0;
  check(ixb_max_occupancy(d->as<int32_t>(), c.nnz(), group_dim == 0 ? c.rows : c.cols, nullptr,
                          &m));
  return b200::coo_to_groupcoo(c, group_dim, m > 1 ? m : 1);
}

bool is_ell(const GroupCooMatrix& gc) {
  auto am = detail::upload_coords(gc.group_coord, "group");
  int f = 1;
  check(ixb_is_ell(am->as<int32_t>(), gc.num_groups(), nullptr, &f));
  return f != 0;
}

BlockGroupCooMatrix dense_to_blockgroupcoo(const Tensor& t, int64_t block_rows,
                                           int64_t block_cols, int64_t g, int group_dim) {
  // formats.cpp:226-228, then group_dim through coo_to_groupcoo (:265)
  if (t.rank() != 2) throw ShapeError("dense_to_blockgroupcoo expects a rank-2 tensor");
  if (block_rows < 1 || block_cols < 1) throw ShapeError("block dims must be >= 1");
  if (g < 1) throw ShapeError("group size must be >= 1");
  if (group_dim != 0 && group_dim != 1) throw ShapeError("group_dim must be 0 or 1");
  BlockGroupCooMatrix b;
  b.rows = t.dim(0);
  b.cols = t.dim(1);
  b.block_rows = block_rows;
  b.block_cols = block_cols;
  b.group_dim = group_dim;
  b.group_size = g;
  auto dense = detail::upload_values(t);
  Pack pk;
  int64_t G = 0, g_used = 0, nblocks = 0;
  check(ixb_blockgroupcoo_plan(dense->p, detail::value_dtype(t), b.rows, b.cols, block_rows,
                               block_cols, g, group_dim, nullptr, &pk.p, &G, &g_used, &nblocks));
  const size_t slots = static_cast<size_t>(G * g);
  DevBuf AM(static_cast<size_t>(G) * 4), AK(slots * 4),
      AV(slots * static_cast<size_t>(block_rows * block_cols) * 8), mask(slots);
  check(ixb_blockgroupcoo_pack(pk.p, AM.as<int32_t>(), AK.as<int32_t>(), AV.p,
                               mask.as<uint8_t>(), nullptr));
  sync();
  b.group_coord = detail::download_coords(AM, G);
  b.member_coord = detail::download_coords(AK, G * g);
  b.values = detail::download_values(AV, t.kind(), {G, g, block_rows, block_cols});
  b.pad_mask = detail::download_mask(mask, G * g);
  return b;
}

GroupCooTensor group_coo_tensor(const CooTensor& c, int group_dim, int64_t g) {
  // formats.cpp:418-419
  if (g < 1) throw ShapeError("group size must be >= 1");
  if (group_dim < 0 || group_dim >= c.rank()) throw ShapeError("group_dim out of range");
  GroupCooTensor out;
  out.shape = c.shape;
  out.group_dim = group_dim;
  out.group_size = g;
  for (int d = 0; d < c.rank(); ++d)
    if (d != group_dim) out.member_dims.push_back(d);
  const int64_t nnz = c.nnz();
  std::vector<std::unique_ptr<DevBuf>> dc;
  std::vector<const int32_t*> cptr;
  for (int d = 0; d < c.rank(); ++d) {
    dc.push_back(detail::upload_coords(c.coords[static_cast<size_t>(d)], "COO tensor"));
    cptr.push_back(dc.back()->as<int32_t>());
  }
  auto v = detail::upload_values(c.values);
  Pack pk;
  int64_t G = 0;
  check(ixb_group_coo_tensor_plan(c.rank(), c.shape.data(), cptr.data(), nnz, group_dim, g, 0,
                                  nullptr, &pk.p, &G));
  const size_t slots = static_cast<size_t>(G * g);
  DevBuf gcoord(static_cast<size_t>(G) * 4), vals(slots * 8), mask(slots);
  std::vector<std::unique_ptr<DevBuf>> mc;
  std::vector<int32_t*> mptr;
  for (size_t m = 0; m < out.member_dims.size(); ++m) {
    mc.push_back(std::make_unique<DevBuf>(slots * 4));
    mptr.push_back(mc.back()->as<int32_t>());
  }
  check(ixb_group_coo_tensor_pack(pk.p, v->p, detail::value_dtype(c.values), gcoord.as<int32_t>(),
                                  mptr.data(), vals.p, mask.as<uint8_t>(), nullptr));
  sync();
  out.group_coord = detail::download_coords(gcoord, G);
  for (auto& m : mc) out.member_coords.push_back(detail::download_coords(*m, G * g));
  out.values = detail::download_values(vals, c.values.kind(), {G, g});
  out.pad_mask = detail::download_mask(mask, G * g);
  return out;
}

TuneReport tune(const CooMatrix& c, int dim, bool count_empty_rows) {
  if (dim != 0 && dim != 1) throw ShapeError("occupancy: dim must be 0 or 1");
  const auto& coord = dim == 0 ? c.row_coord : c.col_coord;
  const int64_t extent = dim == 0 ? c.rows : c.cols;
  auto d = detail::upload_coords(coord, dim == 0 ? "row" : "col");
  TuneReport rep;
  int64_t chosen = 1, cand_g[2] = {1, 1};
  double gstar = 1.0, cand_score[2] = {0, 0};
  int ncand = 0;
  check(ixb_tune_report(d->as<int32_t>(), c.nnz(), extent, count_empty_rows ? 1 : 0, nullptr,
                        &chosen, &gstar, cand_g, cand_score, &ncand));
  rep.gstar = gstar;
  rep.chosen = chosen;
  for (int i = 0; i < ncand; ++i) rep.candidates.emplace_back(cand_g[i], cand_score[i]);
  int64_t bg = 0, bf = 0;
  check(ixb_tune_brute(d->as<int32_t>(), c.nnz(), extent, nullptr, &bg, &bf));
  if (bg > 0) rep.brute_optimal = std::make_pair(bg, bf);
  return rep;
}

namespace {

std::vector<std::string> default_suffixes(size_t rank) {
  // driver.cpp:33-39: matrix convention first (AM/AK), then block coordinates
  if (rank == 2) return {"M", "K"};
  std::vector<std::string> s;
  for (size_t i = 0; i < rank; ++i) s.push_back(std::string(1, static_cast<char>('I' + i)));
  return s;
}

// bind_matrix_format (driver.cpp:98-136) over the device builders
void bind_matrix_format(const SparseSpec& spec, const Tensor& dense, BoundProblem& problem,
                        bool count_empty_rows) {
  const auto suffixes = spec.suffixes.empty() ? default_suffixes(2) : spec.suffixes;
  std::map<std::string, Tensor> ops;
  if (spec.format == "coo") {
    CooMatrix coo = b200::dense_to_coo(dense);
    ops = emit_operands(coo, spec.name, suffixes[0], suffixes[1]);
    problem.format_bytes[spec.name] = format_nbytes(coo);
  } else if (spec.format == "groupcoo" || spec.format == "auto") {
    CooMatrix coo = b200::dense_to_coo(dense);
    int64_t g = spec.g;
    if (spec.format == "auto") {
      TuneReport report = b200::tune(coo, spec.group_dim, count_empty_rows);
      g = report.chosen;
      problem.tuner_reports[spec.name] = std::move(report);
    }
    GroupCooMatrix gc = b200::coo_to_groupcoo(coo, spec.group_dim, g);
    ops = emit_operands(gc, spec.name, suffixes[0], suffixes[1]);
    problem.format_bytes[spec.name] = format_nbytes(gc);
  } else if (spec.format == "blockgroupcoo") {
    if (spec.format_block.size() != 2) {
      throw std::invalid_argument("blockgroupcoo needs formatBlock [bM, bK] for " + spec.name);
    }
    BlockGroupCooMatrix b = b200::dense_to_blockgroupcoo(dense, spec.format_block[0],
                                                   spec.format_block[1], spec.g, spec.group_dim);
    ops = emit_operands(b, spec.name, suffixes[0], suffixes[1]);
    problem.format_bytes[spec.name] = format_nbytes(b);
  } else {
    throw std::invalid_argument("unknown format directive: " + spec.format);
  }
  for (auto& [name, tensor] : ops) problem.tensors[name] = std::move(tensor);
}

// bind_tensor_format (driver.cpp:138-161) over the device grouping
void bind_tensor_format(const SparseSpec& spec, const CooTensor& coo, BoundProblem& problem) {
  const auto suffixes = spec.suffixes.empty() ? default_suffixes(coo.shape.size())
                                              : spec.suffixes;
  if (suffixes.size() != coo.shape.size()) {
    throw std::invalid_argument("suffix count does not match rank for " + spec.name);
  }
  if (spec.format == "coo") {
    for (size_t d = 0; d < coo.coords.size(); ++d) {
      problem.tensors[spec.name + suffixes[d]] = Tensor::from_int({coo.nnz()}, coo.coords[d]);
    }
    problem.tensors[spec.name + "V"] = coo.values;
    problem.format_bytes[spec.name] =
        8 * (static_cast<int64_t>(coo.coords.size()) * coo.nnz() + coo.nnz());
  } else if (spec.format == "groupcoo") {
    GroupCooTensor gc = b200::group_coo_tensor(coo, spec.group_dim, spec.g);
    problem.tensors[spec.name + suffixes[static_cast<size_t>(spec.group_dim)]] =
        Tensor::from_int({gc.num_groups()}, gc.group_coord);
    for (size_t m = 0; m < gc.member_coords.size(); ++m) {
      problem.tensors[spec.name + suffixes[static_cast<size_t>(gc.member_dims[m])]] =
          Tensor::from_int({gc.num_groups(), gc.group_size}, gc.member_coords[m]);
    }
    problem.tensors[spec.name + "V"] = gc.values;
    const int64_t slots = gc.num_groups() * gc.group_size;
    problem.format_bytes[spec.name] =
        8 * (gc.num_groups() + static_cast<int64_t>(gc.member_coords.size()) * slots + slots);
  } else {
    throw std::invalid_argument("rank-" + std::to_string(coo.shape.size()) +
                                " sparse operand " + spec.name + " supports coo or groupcoo");
  }
}

}  // namespace

BoundProblem materialize(const RunConfig& cfg) {
  // driver.cpp:165-233: the same synth call order (the RNG stream is part of
  // the contract), the format directives on the device
  BoundProblem problem;
  Rng rng(cfg.seed);
  for (const auto& spec : cfg.dense) {
    problem.tensors[spec.name] = synth_dense(spec.shape, cfg.elem, rng);
  }
  for (const auto& spec : cfg.index) {
    Tensor t = Tensor::zeros(ElemKind::Int64, spec.shape);
    std::uniform_int_distribution<int64_t> dist(0, std::max<int64_t>(spec.bound - 1, 0));
    for (int64_t i = 0; i < t.numel(); ++i) t.int_at(i) = dist(rng);
    problem.tensors[spec.name] = std::move(t);
  }
  for (const auto& spec : cfg.sparse) {
    if (spec.shape.size() == 2) {
      Tensor dense = spec.gen_block.empty()
                         ? synth_sparse_matrix(spec.shape[0], spec.shape[1], spec.density,
                                               cfg.elem, rng)
                         : synth_block_sparse_matrix(spec.shape[0], spec.shape[1],
                                                     spec.gen_block[0], spec.gen_block[1],
                                                     spec.block_density, cfg.elem, rng);
      bind_matrix_format(spec, dense, problem, cfg.tuner_count_empty_rows);
    } else {
      int64_t nnz = spec.nnz;
      if (nnz < 0) {
        int64_t capacity = 1;
        for (int64_t d : spec.shape) capacity *= d;
        nnz = std::max<int64_t>(1, static_cast<int64_t>(spec.density * capacity));
      }
      CooTensor coo = synth_coo_tensor(spec.shape, nnz, cfg.elem, rng);
      bind_tensor_format(spec, coo, problem);
    }
  }
  for (const auto& [name, path] : cfg.bindings) {
    if (path.size() > 4 && path.substr(path.size() - 4) == ".mtx") {
      MatrixMarketData data = load_matrix_market(path);
      if (std::holds_alternative<Tensor>(data)) {
        problem.tensors[name] = std::get<Tensor>(data);
      } else {
        // coordinate files bind their arrays under the standard suffixes
        CooMatrix coo = b200::canonicalize(std::get<CooMatrix>(data));
        for (auto& [n, t] : emit_operands(coo, name)) problem.tensors[n] = std::move(t);
        problem.format_bytes[name] = format_nbytes(coo);
      }
    } else {
      problem.tensors[name] = load_tensor(path);
    }
  }
  if (cfg.output_name.empty()) throw BindError("no output tensor configured");
  // a file-bound output primes the accumulation buffer for `+=` statements
  auto bound_out = problem.tensors.find(cfg.output_name);
  if (bound_out != problem.tensors.end()) {
    if (!cfg.output_shape.empty() && bound_out->second.shape() != cfg.output_shape) {
      throw BindError("bound output " + cfg.output_name +
                      " does not match the configured output shape");
    }
    problem.out = bound_out->second;
    problem.tensors.erase(bound_out);
  } else {
    problem.out = Tensor::zeros(cfg.elem, cfg.output_shape);
  }
  ShapeMap shapes;
  for (const auto& [name, t] : problem.tensors) shapes[name] = t.shape();
  shapes[cfg.output_name] = problem.out.shape();
  problem.stmt = infer_extents(parse(cfg.expression), shapes);
  return problem;
}

}  // namespace ixsum::b200
