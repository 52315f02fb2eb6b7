// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// ctypes bridge over the *unmodified* reference library (`ixsum`, compiled in
// place from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// It lets the Python tests and bench.py's `--impl reference` arm call the
// reference's own synth / builders / tuner / executors and read the results.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
// legs may load it.
//
// Everything crosses the boundary as a "bag": a named map of reference
// `ixsum::Tensor`s (fp64 or int64) plus named scalars.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "ixsum/driver.hpp"
#include "ixsum/formats.hpp"
#include "ixsum/kernel.hpp"
#include "ixsum/matrix_market.hpp"
#include "ixsum/plan.hpp"
#include "ixsum/synth.hpp"
#include "ixsum/tensor.hpp"
#include "ixsum/tuner.hpp"

using namespace ixsum;

namespace {

struct Bag {
  std::map<std::string, Tensor> t;
  std::map<std::string, double> s;
  std::string text;
  // Set for bags made by ixr_problem_from_spec.
  std::unique_ptr<BoundProblem> problem;
};

thread_local std::string g_err;
thread_local int g_code = 0;

// Same classification as report_error (driver.cpp:571-580).
int classify(const std::exception& e) {
  if (dynamic_cast<const ParseError*>(&e)) return kExitParseError;
  if (dynamic_cast<const BindError*>(&e)) return kExitUnboundTensor;
  if (dynamic_cast<const IndexRangeError*>(&e)) return kExitIndexRange;
  if (dynamic_cast<const InferenceError*>(&e) || dynamic_cast<const ShapeError*>(&e)) {
    return kExitShapeError;
  }
  return kFailure;
}

template <typename F>
auto guard(F&& f, decltype(f()) fail) -> decltype(f()) {
  try {
    g_code = 0;
    g_err.clear();
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    g_code = classify(e);
    return fail;
  }
}

Tensor make_tensor(int kind, int rank, const int64_t* shape, const void* data) {
  std::vector<int64_t> sh(shape, shape + rank);
  int64_t n = 1;
  for (int64_t d : sh) n *= d;
  if (kind == 0) {
    const double* p = static_cast<const double*>(data);
    return Tensor::from_real(sh, std::vector<double>(p, p + n));
  }
  const int64_t* p = static_cast<const int64_t*>(data);
  return Tensor::from_int(sh, std::vector<int64_t>(p, p + n));
}

std::vector<int64_t> u8_to_i64(const std::vector<uint8_t>& v) {
  return std::vector<int64_t>(v.begin(), v.end());
}

ElemKind kind_of(int k) { return k == 0 ? ElemKind::Real64 : ElemKind::Int64; }

}  // namespace

extern "C" {

const char* ixr_last_error() { return g_err.c_str(); }
int ixr_last_code() { return g_code; }

void ixr_free(void* bag) { delete static_cast<Bag*>(bag); }

// ---- bag access --------------------------------------------------------
int ixr_bag_count(void* h) { return static_cast<int>(static_cast<Bag*>(h)->t.size()); }

const char* ixr_bag_name(void* h, int i) {
  auto* b = static_cast<Bag*>(h);
  auto it = b->t.begin();
  std::advance(it, i);
  return it->first.c_str();
}

// kind: 0 real64, 1 int64. Returns rank, or -1 if absent.
int ixr_bag_info(void* h, const char* name, int* kind, int64_t* shape16) {
  auto* b = static_cast<Bag*>(h);
  auto it = b->t.find(name);
  if (it == b->t.end()) return -1;
  *kind = it->second.is_int() ? 1 : 0;
  for (int i = 0; i < it->second.rank(); ++i) shape16[i] = it->second.dim(i);
  return it->second.rank();
}

int ixr_bag_read(void* h, const char* name, void* dst) {
  auto* b = static_cast<Bag*>(h);
  auto it = b->t.find(name);
  if (it == b->t.end()) return -1;
  const Tensor& t = it->second;
  if (t.is_int()) {
    std::memcpy(dst, t.ints().data(), t.ints().size() * 8);
  } else {
    std::memcpy(dst, t.reals().data(), t.reals().size() * 8);
  }
  return 0;
}

void ixr_bag_set(void* h, const char* name, int kind, int rank, const int64_t* shape,
                 const void* data) {
  static_cast<Bag*>(h)->t[name] = make_tensor(kind, rank, shape, data);
}

void* ixr_bag_new() { return new Bag(); }

double ixr_bag_scalar(void* h, const char* name) {
  auto* b = static_cast<Bag*>(h);
  auto it = b->s.find(name);
  return it == b->s.end() ? -1.0 : it->second;
}

const char* ixr_bag_text(void* h) { return static_cast<Bag*>(h)->text.c_str(); }

// ---- synth (synth.hpp:17-29) -------------------------------------------
void* ixr_rng_new(uint64_t seed) { return new Rng(seed); }
void ixr_rng_free(void* r) { delete static_cast<Rng*>(r); }

void* ixr_synth_dense(void* rng, int kind, int rank, const int64_t* shape) {
  return guard([&]() -> void* {
    auto* b = new Bag();
    b->t["t"] = synth_dense(std::vector<int64_t>(shape, shape + rank), kind_of(kind),
                            *static_cast<Rng*>(rng));
    return b;
  }, nullptr);
}

void* ixr_synth_sparse_matrix(void* rng, int kind, int64_t rows, int64_t cols, double density) {
  return guard([&]() -> void* {
    auto* b = new Bag();
    b->t["t"] = synth_sparse_matrix(rows, cols, density, kind_of(kind), *static_cast<Rng*>(rng));
    return b;
  }, nullptr);
}

void* ixr_synth_block_sparse_matrix(void* rng, int kind, int64_t rows, int64_t cols,
                                    int64_t br, int64_t bc, double bdens) {
  return guard([&]() -> void* {
    auto* b = new Bag();
    b->t["t"] = synth_block_sparse_matrix(rows, cols, br, bc, bdens, kind_of(kind),
                                          *static_cast<Rng*>(rng));
    return b;
  }, nullptr);
}

void* ixr_synth_coo_tensor(void* rng, int kind, int rank, const int64_t* shape, int64_t nnz) {
  return guard([&]() -> void* {
    auto* b = new Bag();
    CooTensor c = synth_coo_tensor(std::vector<int64_t>(shape, shape + rank), nnz,
                                   kind_of(kind), *static_cast<Rng*>(rng));
    int64_t n = c.nnz();
    std::vector<int64_t> flat;
    for (const auto& v : c.coords) flat.insert(flat.end(), v.begin(), v.end());
    b->t["coords"] = Tensor::from_int({static_cast<int64_t>(c.coords.size()), n}, flat);
    b->t["values"] = c.values;
    return b;
  }, nullptr);
}

uint64_t ixr_rng_next(void* rng) { return (*static_cast<Rng*>(rng))(); }

int64_t ixr_uniform_int(void* rng, int64_t lo, int64_t hi) {
  std::uniform_int_distribution<int64_t> d(lo, hi);
  return d(*static_cast<Rng*>(rng));
}

// ---- builders (formats.hpp) -------------------------------------------
// Dense → COO (formats.cpp:24-46). Bag: row_coord, col_coord, values.
void* ixr_dense_to_coo(int kind, int64_t rows, int64_t cols, const void* data) {
  return guard([&]() -> void* {
    int64_t sh[2] = {rows, cols};
    CooMatrix c = dense_to_coo(make_tensor(kind, 2, sh, data));
    auto* b = new Bag();
    b->t["row_coord"] = Tensor::from_int({c.nnz()}, c.row_coord);
    b->t["col_coord"] = Tensor::from_int({c.nnz()}, c.col_coord);
    b->t["values"] = c.values;
    b->s["nbytes"] = static_cast<double>(format_nbytes(c));
    return b;
  }, nullptr);
}

static CooMatrix coo_from(int64_t rows, int64_t cols, const int64_t* r, const int64_t* c,
                          int kind, const void* vals, int64_t nnz, int canonical) {
  CooMatrix m;
  m.rows = rows;
  m.cols = cols;
  m.row_coord.assign(r, r + nnz);
  m.col_coord.assign(c, c + nnz);
  int64_t sh[1] = {nnz};
  m.values = make_tensor(kind, 1, sh, vals);
  m.canonical = canonical != 0;
  return m;
}

// coo_to_groupcoo (formats.cpp:115-174). Bag: AM, AK, AV, mask (+ G, nbytes, maskbytes).
void* ixr_coo_to_groupcoo(int64_t rows, int64_t cols, const int64_t* r, const int64_t* c,
                          int kind, const void* vals, int64_t nnz, int canonical,
                          int group_dim, int64_t g) {
  return guard([&]() -> void* {
    GroupCooMatrix gc =
        coo_to_groupcoo(coo_from(rows, cols, r, c, kind, vals, nnz, canonical), group_dim, g);
    auto* b = new Bag();
    b->t["AM"] = Tensor::from_int({gc.num_groups()}, gc.group_coord);
    b->t["AK"] = Tensor::from_int({gc.num_groups(), g}, gc.member_coord);
    b->t["AV"] = gc.values;
    b->t["mask"] = Tensor::from_int({gc.num_groups(), g}, u8_to_i64(gc.pad_mask));
    b->s["G"] = static_cast<double>(gc.num_groups());
    b->s["nbytes"] = static_cast<double>(format_nbytes(gc));
    b->s["maskbytes"] = static_cast<double>(mask_nbytes(gc));
    b->s["is_ell"] = is_ell(gc) ? 1.0 : 0.0;
    return b;
  }, nullptr);
}

// dense_to_blockgroupcoo (formats.cpp:224-292).
void* ixr_dense_to_blockgroupcoo(int kind, int64_t rows, int64_t cols, const void* data,
                                 int64_t bm, int64_t bk, int64_t g, int group_dim) {
  return guard([&]() -> void* {
    int64_t sh[2] = {rows, cols};
    BlockGroupCooMatrix m =
        dense_to_blockgroupcoo(make_tensor(kind, 2, sh, data), bm, bk, g, group_dim);
    auto* b = new Bag();
    b->t["AM"] = Tensor::from_int({m.num_groups()}, m.group_coord);
    b->t["AK"] = Tensor::from_int({m.num_groups(), g}, m.member_coord);
    b->t["AV"] = m.values;
    b->t["mask"] = Tensor::from_int({m.num_groups(), g}, u8_to_i64(m.pad_mask));
    b->t["dense_back"] = blockgroupcoo_to_dense(m);
    b->s["G"] = static_cast<double>(m.num_groups());
    b->s["nbytes"] = static_cast<double>(format_nbytes(m));
    return b;
  }, nullptr);
}

// group_coo_tensor (formats.cpp:417-479). coords is [rank, nnz] row-major.
void* ixr_group_coo_tensor(int rank, const int64_t* shape, const int64_t* coords, int kind,
                           const void* vals, int64_t nnz, int group_dim, int64_t g) {
  return guard([&]() -> void* {
    CooTensor c;
    c.shape.assign(shape, shape + rank);
    c.coords.resize(static_cast<size_t>(rank));
    for (int d = 0; d < rank; ++d) c.coords[d].assign(coords + d * nnz, coords + (d + 1) * nnz);
    int64_t sh[1] = {nnz};
    c.values = make_tensor(kind, 1, sh, vals);
    GroupCooTensor gt = group_coo_tensor(c, group_dim, g);
    auto* b = new Bag();
    int64_t G = gt.num_groups();
    b->t["group_coord"] = Tensor::from_int({G}, gt.group_coord);
    std::vector<int64_t> flat;
    for (const auto& v : gt.member_coords) flat.insert(flat.end(), v.begin(), v.end());
    b->t["member_coords"] =
        Tensor::from_int({static_cast<int64_t>(gt.member_coords.size()), G, g}, flat);
    b->t["values"] = gt.values;
    b->t["mask"] = Tensor::from_int({G, g}, u8_to_i64(gt.pad_mask));
    b->s["G"] = static_cast<double>(G);
    return b;
  }, nullptr);
}

// ---- tuner (tuner.cpp:100-118) -----------------------------------------
// out6: gstar, chosen, brute_g, brute_f, ncand, cost_exact(chosen); cands: up to 2 (g, score)
int ixr_tune(const int64_t* occ, int64_t n, int count_empty_rows, double* out6, double* cands) {
  return guard([&]() -> int {
    OccProfile p{std::vector<int64_t>(occ, occ + n)};
    TuneReport r = select(p, {}, count_empty_rows != 0);
    out6[0] = r.gstar;
    out6[1] = static_cast<double>(r.chosen);
    out6[2] = r.brute_optimal ? static_cast<double>(r.brute_optimal->first) : -1;
    out6[3] = r.brute_optimal ? static_cast<double>(r.brute_optimal->second) : -1;
    out6[4] = static_cast<double>(r.candidates.size());
    out6[5] = static_cast<double>(cost_exact(p, r.chosen));
    for (size_t i = 0; i < r.candidates.size() && i < 2; ++i) {
      cands[2 * i] = static_cast<double>(r.candidates[i].first);
      cands[2 * i + 1] = r.candidates[i].second;
    }
    return 0;
  }, -1);
}

int64_t ixr_cost_exact(const int64_t* occ, int64_t n, int64_t g) {
  return guard([&]() -> int64_t {
    return cost_exact(OccProfile{std::vector<int64_t>(occ, occ + n)}, g);
  }, -1);
}

double ixr_cost_relaxed(const int64_t* occ, int64_t n, double g, int count_empty) {
  return guard([&]() -> double {
    return cost_relaxed(OccProfile{std::vector<int64_t>(occ, occ + n)}, g, count_empty != 0);
  }, -1.0);
}

// ---- problems from run specs (driver.cpp:43-233) -----------------------
void* ixr_problem_from_spec(const char* path) {
  return guard([&]() -> void* {
    RunConfig cfg = load_run_config(path);
    auto* b = new Bag();
    b->problem = std::make_unique<BoundProblem>(materialize(cfg));
    for (const auto& [n, t] : b->problem->tensors) b->t[n] = t;
    b->t["__out__"] = b->problem->out;
    b->text = to_string(b->problem->stmt);
    for (const auto& [n, rep] : b->problem->tuner_reports) {
      b->s["g." + n] = static_cast<double>(rep.chosen);
      b->s["gstar." + n] = rep.gstar;
    }
    for (const auto& [n, by] : b->problem->format_bytes) {
      b->s["bytes." + n] = static_cast<double>(by);
    }
    return b;
  }, nullptr);
}

// Runs `expr` over the tensors of `bag` (output buffer = tensor `out_name`,
// its contents prime `+=`) in one of the reference modes of execute_mode
// (driver.cpp:235-265): oracle | plan | fused-eager | fused-lazy.
// Result bag: "result" + scalars wall_ms, gathers, scatters, atomic_updates.
void* ixr_run(void* h, const char* expr, const char* out_name, const char* mode, int threads) {
  return guard([&]() -> void* {
    auto* b = static_cast<Bag*>(h);
    BoundProblem prob;
    for (const auto& [n, t] : b->t) {
      if (n != out_name) prob.tensors[n] = t;
    }
    prob.out = b->t.at(out_name);
    ShapeMap shapes;
    for (const auto& [n, t] : prob.tensors) shapes[n] = t.shape();
    shapes[out_name] = prob.out.shape();
    prob.stmt = infer_extents(parse(expr), shapes);
    ModeResult mo = execute_mode(mode, prob, threads, {});
    auto* r = new Bag();
    r->t["result"] = std::move(mo.result);
    r->s["wall_ms"] = mo.wall_ms;
    r->s["gathers"] = static_cast<double>(mo.counters.gathers);
    r->s["scatters"] = static_cast<double>(mo.counters.scatters);
    r->s["atomic_updates"] = static_cast<double>(mo.counters.atomic_updates);
    r->s["kernel_count"] = static_cast<double>(mo.kernel_count);
    r->s["hash"] = static_cast<double>(tensor_hash(r->t["result"]) >> 11);
    r->text = to_string(prob.stmt);
    return r;
  }, nullptr);
}

// GroupCOO access-count model (plan.cpp:607-631) for expr over bag (AM/AK/...).
int ixr_count_model(int64_t G, int64_t g, void* h, const char* expr, const char* out_name,
                    int64_t* out3) {
  return guard([&]() -> int {
    auto* b = static_cast<Bag*>(h);
    ShapeMap shapes;
    for (const auto& [n, t] : b->t) shapes[n] = t.shape();
    EinsumStmt stmt = infer_extents(parse(expr), shapes);
    GroupCooMatrix gc;
    gc.group_size = g;
    gc.group_coord.assign(static_cast<size_t>(G), 0);
    AccessCounters c = count_accesses_model(gc, stmt);
    out3[0] = c.gathers;
    out3[1] = c.scatters;
    out3[2] = c.atomic_updates;
    (void)out_name;
    return 0;
  }, -1);
}

double ixr_max_rel_error(int kind, int64_t n, const void* a, const void* bb) {
  int64_t sh[1] = {n};
  return max_rel_error(make_tensor(kind, 1, sh, a), make_tensor(kind, 1, sh, bb));
}

uint64_t ixr_tensor_hash(int kind, int rank, const int64_t* shape, const void* data) {
  return tensor_hash(make_tensor(kind, rank, shape, data));
}

// ---- .ixt files (tensor.cpp:158-225)
void* ixr_load_tensor(const char* path) {
  return guard(
      [&]() -> void* {
        auto* b = new Bag();
        b->t["t"] = load_tensor(path);
        return b;
      },
      nullptr);
}

int ixr_save_tensor(const char* path, int kind, int rank, const int64_t* shape, const void* data) {
  return guard(
      [&]() -> int {
        save_tensor(path, make_tensor(kind, rank, shape, data));
        return 0;
      },
      -1);
}

}  // extern "C"
