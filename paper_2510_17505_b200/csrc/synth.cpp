// Seeded synthetic inputs on the host (the reference's parity contract,
// synth.hpp:13-29): std::mt19937_64 with libstdc++'s distributions, consumed
// in the same order as synth.cpp:10-106, written straight into the device
// value type (fp32 / bf16 rounding of the reference's fp64 values, or exact
// int64 / fp64). One Rng is shared by every operand in materialize order
// (driver.cpp:167-197).
#include <algorithm>
#include <cstring>
#include <random>
#include <set>
#include <vector>

#include <cuda_bf16.h>

#include "ixb_internal.h"

struct ixb_rng {
  std::mt19937_64 g;
};

namespace {

enum { OUT_F32 = 0, OUT_BF16 = 1, OUT_F64 = 2, OUT_I64 = 3 };

int64_t nonzero_int(std::mt19937_64& r) {  // synth.cpp:10-15
  std::uniform_int_distribution<int64_t> dist(1, 4);
  std::bernoulli_distribution sign(0.5);
  int64_t v = dist(r);
  return sign(r) ? v : -v;
}

double nonzero_real(std::mt19937_64& r) {  // synth.cpp:17-22
  std::uniform_real_distribution<double> dist(0.125, 1.0);
  std::bernoulli_distribution sign(0.5);
  double v = dist(r);
  return sign(r) ? v : -v;
}

// kind: 0 real (fp64 stream), 1 int (int64 stream); written as `out` type.
void put(std::mt19937_64& r, int kind, int out, void* dst, int64_t i) {
  if (kind == 1) {
    int64_t v = nonzero_int(r);
    switch (out) {
      case OUT_F32: static_cast<float*>(dst)[i] = static_cast<float>(v); break;
      case OUT_BF16: static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16(static_cast<float>(v)); break;
      case OUT_F64: static_cast<double*>(dst)[i] = static_cast<double>(v); break;
      default: static_cast<int64_t*>(dst)[i] = v;
    }
  } else {
    double v = nonzero_real(r);
    switch (out) {
      case OUT_F32: static_cast<float*>(dst)[i] = static_cast<float>(v); break;
      case OUT_BF16: static_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(static_cast<float>(v)); break;
      case OUT_F64: static_cast<double*>(dst)[i] = v; break;
      default: ixb::fail(IXB_FAILURE, "real synth cannot be written as int64");
    }
  }
}

size_t elem_bytes(int out) { return out == OUT_BF16 ? 2 : (out == OUT_F32 ? 4 : 8); }

}  // namespace

extern "C" {

ixb_rng* ixb_rng_new(uint64_t seed) { return new ixb_rng{std::mt19937_64(seed)}; }
void ixb_rng_free(ixb_rng* r) { delete r; }
uint64_t ixb_rng_next(ixb_rng* r) { return r->g(); }

int ixb_synth_dense(ixb_rng* r, int kind, int64_t numel, int out, void* dst) {
  return ixb_guard([&] {  // synth.cpp:36-40
    for (int64_t i = 0; i < numel; ++i) put(r->g, kind, out, dst, i);
  });
}

int ixb_synth_sparse_matrix(ixb_rng* r, int kind, int64_t rows, int64_t cols, double density,
                            int out, void* dst) {
  return ixb_guard([&] {  // synth.cpp:42-54
    std::memset(dst, 0, static_cast<size_t>(rows * cols) * elem_bytes(out));
    std::bernoulli_distribution keep(density);
    for (int64_t i = 0; i < rows * cols; ++i) {
      if (!keep(r->g)) continue;
      put(r->g, kind, out, dst, i);
    }
  });
}

int ixb_synth_block_sparse_matrix(ixb_rng* r, int kind, int64_t rows, int64_t cols, int64_t br,
                                  int64_t bc, double bdens, int out, void* dst) {
  return ixb_guard([&] {  // synth.cpp:56-78
    std::memset(dst, 0, static_cast<size_t>(rows * cols) * elem_bytes(out));
    std::bernoulli_distribution keep(bdens);
    const int64_t gr = (rows + br - 1) / br, gc = (cols + bc - 1) / bc;
    for (int64_t bi = 0; bi < gr; ++bi) {
      for (int64_t bj = 0; bj < gc; ++bj) {
        if (!keep(r->g)) continue;
        for (int64_t i = bi * br; i < std::min((bi + 1) * br, rows); ++i) {
          for (int64_t j = bj * bc; j < std::min((bj + 1) * bc, cols); ++j) {
            put(r->g, kind, out, dst, i * cols + j);
          }
        }
      }
    }
  });
}

// Voxelised sphere shells (no reference counterpart; the cfg5 point cloud of
// BASELINE.json): voxels with R-1/2 <= |v - c| < R+1/2 for R = 282, shells
// centred 1000 apart along x until n_target voxels, emitted in (x, y, z)
// order (unique, sorted) and truncated to n_target. Deterministic, no RNG.
int ixb_synth_voxel_shells(int64_t n_target, int32_t* coords, int64_t* n_out) {
  return ixb_guard([&] {
    const int R = 282;
    const double lo = (R - 0.5) * (R - 0.5), hi = (R + 0.5) * (R + 0.5);
    int64_t n = 0;
    for (int shell = 0; n < n_target; ++shell) {
      const int cx = shell * 1000;
      for (int x = -R - 1; x <= R + 1 && n < n_target; ++x) {
        for (int y = -R - 1; y <= R + 1 && n < n_target; ++y) {
          for (int z = -R - 1; z <= R + 1 && n < n_target; ++z) {
            const double d = static_cast<double>(x) * x + static_cast<double>(y) * y +
                             static_cast<double>(z) * z;
            if (d < lo || d >= hi) continue;
            if (coords) {
              coords[3 * n] = cx + x;
              coords[3 * n + 1] = y;
              coords[3 * n + 2] = z;
            }
            ++n;
          }
        }
      }
    }
    *n_out = n;
  });
}

// synth_coo_tensor (synth.cpp:80-106): coords [rank, nnz_realised] int32.
int ixb_synth_coo_tensor(ixb_rng* r, int kind, int rank, const int64_t* shape, int64_t nnz,
                         int out, int32_t* coords, void* vals, int64_t* nnz_out) {
  return ixb_guard([&] {
    int64_t cap = 1;
    for (int d = 0; d < rank; ++d) cap *= shape[d];
    nnz = std::min(nnz, cap);
    std::set<std::vector<int64_t>> seen;
    std::vector<std::vector<int64_t>> picked;
    while (static_cast<int64_t>(picked.size()) < nnz) {
      std::vector<int64_t> c(static_cast<size_t>(rank));
      for (int d = 0; d < rank; ++d) {
        std::uniform_int_distribution<int64_t> dist(0, shape[d] - 1);
        c[static_cast<size_t>(d)] = dist(r->g);
      }
      if (seen.insert(c).second) picked.push_back(std::move(c));
    }
    std::sort(picked.begin(), picked.end());
    const int64_t n = static_cast<int64_t>(picked.size());
    for (int64_t p = 0; p < n; ++p) {
      for (int d = 0; d < rank; ++d) coords[d * n + p] = static_cast<int32_t>(picked[p][d]);
    }
    for (int64_t p = 0; p < n; ++p) put(r->g, kind, out, vals, p);
    *nnz_out = n;
  });
}

}  // extern "C"
