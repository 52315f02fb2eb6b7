// On-disk formats straight to and from device memory:
//   .ixt tensor files   (tensor.hpp:65-73, tensor.cpp:158-225, docs/file-formats.md)
//   MatrixMarket (.mtx) (matrix_market.hpp:16, matrix_market.cpp:30-159)
// File parsing is host work, as in the reference. The payload moves through
// two pinned staging buffers (the read of chunk i+1 overlaps the H2D copy of
// chunk i), and one device kernel converts between the file's 8-byte element
// kinds (real64 / int64) and the device dtypes the evaluators consume
// (int32 indices with a range check, fp32 / bf16 / fp64 values). Saving is
// the mirror image, bitwise-compatible with the reference's save_tensor.
#include <cuda_bf16.h>

#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "common.cuh"

namespace ixb {
namespace {

constexpr uint32_t kIxtMagic = 0x4E545849;  // "IXTN" little-endian
constexpr uint32_t kIxtVersion = 1;
constexpr int64_t kChunkElems = 1 << 22;  // 32 MiB of 8-byte elements per staging buffer

int dtype_bytes(int dtype) {
  switch (dtype) {
    case IXB_F32:
    case IXB_I32:
      return 4;
    case IXB_BF16:
      return 2;
    case IXB_F64:
    case IXB_I64:
      return 8;
    case IXB_U8:
      return 1;
  }
  fail(IXB_FAILURE, "unsupported dtype");
}
bool dtype_is_int(int dtype) { return dtype == IXB_I32 || dtype == IXB_I64 || dtype == IXB_U8; }

// ------------------------------------------------------------ conversions
// file element (kind 0 real64, 1 int64) -> device dtype; int64 -> int32 out of
// range is recorded (first offender) instead of silently wrapping.
__global__ void from_file_kernel(const void* src, int kind, int64_t n, void* dst, int dtype,
                                 int64_t base, unsigned long long* bad) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double r = kind == 0 ? static_cast<const double*>(src)[i] : 0.0;
    const long long v = kind == 1 ? static_cast<const long long*>(src)[i] : 0;
    switch (dtype) {
      case IXB_F32:
        static_cast<float*>(dst)[i] = kind == 0 ? static_cast<float>(r) : static_cast<float>(v);
        break;
      case IXB_BF16:
        static_cast<__nv_bfloat16*>(dst)[i] =
            kind == 0 ? __double2bfloat16(r) : __double2bfloat16(static_cast<double>(v));
        break;
      case IXB_F64:
        static_cast<double*>(dst)[i] = kind == 0 ? r : static_cast<double>(v);
        break;
      case IXB_I32:
        if (v < INT32_MIN || v > INT32_MAX) atomicMin(bad, static_cast<unsigned long long>(base + i));
        static_cast<int32_t*>(dst)[i] = static_cast<int32_t>(v);
        break;
      case IXB_I64:
        static_cast<long long*>(dst)[i] = v;
        break;
      case IXB_U8:
        static_cast<uint8_t*>(dst)[i] = static_cast<uint8_t>(v);
        break;
    }
  }
}

// device dtype -> file element (real64 for float dtypes, int64 for int dtypes)
__global__ void to_file_kernel(const void* src, int dtype, int64_t n, void* dst) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    switch (dtype) {
      case IXB_F32:
        static_cast<double*>(dst)[i] = static_cast<const float*>(src)[i];
        break;
      case IXB_BF16:
        static_cast<double*>(dst)[i] = __bfloat162float(static_cast<const __nv_bfloat16*>(src)[i]);
        break;
      case IXB_F64:
        static_cast<double*>(dst)[i] = static_cast<const double*>(src)[i];
        break;
      case IXB_I32:
        static_cast<long long*>(dst)[i] = static_cast<const int32_t*>(src)[i];
        break;
      case IXB_I64:
        static_cast<long long*>(dst)[i] = static_cast<const long long*>(src)[i];
        break;
      case IXB_U8:
        static_cast<long long*>(dst)[i] = static_cast<const uint8_t*>(src)[i];
        break;
    }
  }
}

int64_t grid_for(int64_t n) {
  int64_t g = ceil_div(n, 256);
  const int64_t cap = 8 * static_cast<int64_t>(sm_count());
  return g < 1 ? 1 : (g > cap ? cap : g);
}

// Pinned double-buffered staging (host <-> device) of 8-byte elements.
struct Staging {
  void* host[2] = {nullptr, nullptr};
  Scratch<long long> dev[2];
  cudaEvent_t done[2] = {nullptr, nullptr};
  explicit Staging(cudaStream_t s) {
    for (int b = 0; b < 2; ++b) {
      IXB_CUDA_CHECK(cudaHostAlloc(&host[b], kChunkElems * 8, cudaHostAllocDefault));
      dev[b] = Scratch<long long>(kChunkElems, s);
      IXB_CUDA_CHECK(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    }
  }
  ~Staging() {
    for (int b = 0; b < 2; ++b) {
      if (done[b]) cudaEventSynchronize(done[b]), cudaEventDestroy(done[b]);
      if (host[b]) cudaFreeHost(host[b]);
    }
  }
};

struct File {
  FILE* f = nullptr;
  File(const std::string& path, const char* mode) : f(std::fopen(path.c_str(), mode)) {}
  ~File() {
    if (f) std::fclose(f);
  }
};

struct IxtHeader {
  uint32_t kind = 0, rank = 0;
  int64_t dims[16] = {};
  int64_t numel = 1;
};

// load_tensor's header checks and messages (tensor.cpp:198-214)
IxtHeader read_header(FILE* f, const std::string& path) {
  auto rd = [&](void* p, size_t n) {
    if (std::fread(p, 1, n, f) != n) fail(IXB_IO, "truncated tensor file: " + path);
  };
  uint32_t magic, version;
  IxtHeader h;
  rd(&magic, 4);
  if (magic != kIxtMagic) fail(IXB_IO, "bad magic in " + path);
  rd(&version, 4);
  if (version != kIxtVersion) fail(IXB_IO, "unsupported version in " + path);
  rd(&h.kind, 4);
  if (h.kind > 1) fail(IXB_IO, "bad element kind in " + path);
  rd(&h.rank, 4);
  if (h.rank == 0 || h.rank > 16) fail(IXB_IO, "bad rank in " + path);
  for (uint32_t i = 0; i < h.rank; ++i) {
    rd(&h.dims[i], 8);
    if (h.dims[i] < 0) fail(IXB_IO, "negative dimension in " + path);
    h.numel *= h.dims[i];
  }
  return h;
}

// ------------------------------------------------------------ MatrixMarket
// Restatement of load_matrix_market (matrix_market.cpp:30-159): same header
// rules, same messages, same istream-style token semantics (a token ends
// where the number's grammar ends, so "3.5" read as an integer is 3).
struct Cursor {
  const char* p;
  const char* end;
  bool ws() {
    while (p < end && (*p == ' ' || *p == '\t' || *p == '\r' || *p == '\v' || *p == '\f')) ++p;
    return p < end;
  }
  bool i64(int64_t& v) {
    if (!ws()) return false;
    const char* q = p;
    if (*q == '+' || *q == '-') ++q;
    if (q >= end || *q < '0' || *q > '9') return false;
    char* stop;
    errno = 0;
    long long x = std::strtoll(p, &stop, 10);
    if (errno == ERANGE || stop > end) return false;
    v = x;
    p = stop;
    return true;
  }
  bool f64(double& v) {
    if (!ws()) return false;
    // [sign] digits [. digits] [(e|E) [sign] digits] -- the num_get grammar
    const char* q = p;
    if (q < end && (*q == '+' || *q == '-')) ++q;
    const char* d0 = q;
    while (q < end && *q >= '0' && *q <= '9') ++q;
    bool digits = q > d0;
    if (q < end && *q == '.') {
      ++q;
      const char* d1 = q;
      while (q < end && *q >= '0' && *q <= '9') ++q;
      digits = digits || q > d1;
    }
    if (!digits) return false;
    if (q < end && (*q == 'e' || *q == 'E')) {
      const char* e = q + 1;
      if (e < end && (*e == '+' || *e == '-')) ++e;
      const char* e0 = e;
      while (e < end && *e >= '0' && *e <= '9') ++e;
      if (e > e0) q = e;
    }
    std::string tok(p, q);
    v = std::strtod(tok.c_str(), nullptr);
    p = q;
    return true;
  }
};

std::string lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

}  // namespace
}  // namespace ixb

struct ixb_mtx {
  bool dense = false;
  int kind = 0;  // 0 real64, 1 int64
  int64_t rows = 0, cols = 0;
  std::vector<int64_t> r, c;  // coordinate: zero-based, duplicates and mirror entries kept
  std::vector<double> rv;     // real values (coordinate) or dense row-major
  std::vector<int64_t> iv;    // integer values
};

using namespace ixb;

namespace {

ixb_mtx* parse_mtx(const std::string& path) {
  File fh(path, "rb");
  if (!fh.f) fail(IXB_IO, "cannot open: " + path);
  std::string text;
  {
    char buf[1 << 16];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, fh.f)) > 0) text.append(buf, n);
  }
  size_t pos = 0;
  auto getline = [&](std::string_view& line) {
    if (pos >= text.size()) return false;
    size_t e = text.find('\n', pos);
    if (e == std::string::npos) e = text.size();
    line = std::string_view(text.data() + pos, e - pos);
    pos = e + 1;
    return true;
  };
  auto next_data_line = [&](std::string_view& line) {
    while (getline(line)) {
      size_t f = line.find_first_not_of(" \t\r\n");
      if (f == std::string_view::npos) continue;
      if (line[f] == '%') continue;
      return true;
    }
    return false;
  };
  std::string_view header;
  if (!getline(header)) fail(IXB_IO, "empty MatrixMarket file: " + path);
  std::vector<std::string> w;
  {
    size_t i = 0;
    while (i < header.size() && w.size() < 5) {
      while (i < header.size() && std::isspace(static_cast<unsigned char>(header[i]))) ++i;
      size_t j = i;
      while (j < header.size() && !std::isspace(static_cast<unsigned char>(header[j]))) ++j;
      if (j > i) w.emplace_back(header.substr(i, j - i));
      i = j;
    }
    w.resize(5);
  }
  if (lower(w[0]) != "%%matrixmarket" || lower(w[1]) != "matrix")
    fail(IXB_IO, "malformed MatrixMarket header in " + path);
  const std::string format = lower(w[2]), field = lower(w[3]), symmetry = lower(w[4]);
  if (format != "coordinate" && format != "array")
    fail(IXB_IO, "unsupported MatrixMarket format '" + format + "' in " + path);
  if (field != "real" && field != "integer" && field != "pattern" && field != "double")
    fail(IXB_IO, "unsupported MatrixMarket field '" + field + "' in " + path);
  if (symmetry != "general" && symmetry != "symmetric" && symmetry != "skew-symmetric")
    fail(IXB_IO, "unsupported MatrixMarket symmetry '" + symmetry + "' in " + path);
  const bool pattern = field == "pattern";
  auto m = std::make_unique<ixb_mtx>();
  m->kind = field == "integer" ? 1 : 0;
  std::string_view line;
  if (!next_data_line(line)) fail(IXB_IO, "missing size line in " + path);
  Cursor sz{line.data(), line.data() + line.size()};

  if (format == "array") {
    if (pattern) fail(IXB_IO, "pattern field is invalid for array format in " + path);
    int64_t rows = 0, cols = 0;
    if (!sz.i64(rows) || !sz.i64(cols) || rows < 0 || cols < 0)
      fail(IXB_IO, "malformed array size line in " + path);
    m->dense = true;
    m->rows = rows, m->cols = cols;
    if (m->kind) m->iv.assign(rows * cols, 0);
    else m->rv.assign(rows * cols, 0.0);
    auto read_value = [&](int64_t i, int64_t j) {
      if (!next_data_line(line)) fail(IXB_IO, "truncated array data in " + path);
      Cursor vs{line.data(), line.data() + line.size()};
      const int64_t flat = i * cols + j;
      if (m->kind) {
        int64_t v;
        if (!vs.i64(v)) fail(IXB_IO, "bad integer value in " + path);
        m->iv[flat] = v;
      } else {
        double v;
        if (!vs.f64(v)) fail(IXB_IO, "bad real value in " + path);
        m->rv[flat] = v;
      }
    };
    if (symmetry == "general") {
      for (int64_t j = 0; j < cols; ++j)
        for (int64_t i = 0; i < rows; ++i) read_value(i, j);
    } else {
      if (rows != cols) fail(IXB_IO, "symmetric array must be square in " + path);
      const bool skew = symmetry == "skew-symmetric";
      for (int64_t j = 0; j < cols; ++j) {
        for (int64_t i = j; i < rows; ++i) {
          read_value(i, j);
          if (i == j) continue;
          if (m->kind) m->iv[j * cols + i] = (skew ? -1 : 1) * m->iv[i * cols + j];
          else m->rv[j * cols + i] = (skew ? -1.0 : 1.0) * m->rv[i * cols + j];
        }
      }
    }
    return m.release();
  }

  int64_t rows = 0, cols = 0, nnz = 0;
  if (!sz.i64(rows) || !sz.i64(cols) || !sz.i64(nnz) || rows < 0 || cols < 0 || nnz < 0)
    fail(IXB_IO, "malformed coordinate size line in " + path);
  m->rows = rows, m->cols = cols;
  const bool sym = symmetry != "general", skew = symmetry == "skew-symmetric";
  m->r.reserve(nnz), m->c.reserve(nnz);
  for (int64_t e = 0; e < nnz; ++e) {
    if (!next_data_line(line)) fail(IXB_IO, "truncated coordinate data in " + path);
    Cursor es{line.data(), line.data() + line.size()};
    int64_t i = 0, j = 0;
    if (!es.i64(i) || !es.i64(j)) fail(IXB_IO, "bad coordinate entry in " + path);
    if (i < 1 || i > rows || j < 1 || j > cols)
      fail(IXB_IO, "coordinate (" + std::to_string(i) + "," + std::to_string(j) +
                       ") out of declared bounds in " + path);
    double rv = 1.0;
    int64_t iv = 1;
    if (!pattern) {
      if (m->kind) {
        if (!es.i64(iv)) fail(IXB_IO, "bad integer value in " + path);
      } else {
        if (!es.f64(rv)) fail(IXB_IO, "bad real value in " + path);
      }
    }
    auto push = [&](int64_t r0, int64_t c0, double rvv, int64_t ivv) {
      m->r.push_back(r0);
      m->c.push_back(c0);
      if (m->kind) m->iv.push_back(ivv);
      else m->rv.push_back(rvv);
    };
    push(i - 1, j - 1, rv, iv);
    if (sym && i != j) push(j - 1, i - 1, skew ? -rv : rv, skew ? -iv : iv);
  }
  return m.release();
}

// Host 8-byte payload -> device dtype, chunked through the pinned staging.
void upload8(const void* src, int kind, int64_t n, void* dst, int dtype, cudaStream_t s,
             const std::string& what) {
  if (n == 0) return;
  if ((dtype == IXB_F64 && kind == 0) || (dtype == IXB_I64 && kind == 1)) {
    IXB_CUDA_CHECK(cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyHostToDevice, s));
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));  // pageable source: keep it alive
    return;
  }
  Staging st(s);
  Scratch<unsigned long long> bad(1, s);
  IXB_CUDA_CHECK(cudaMemsetAsync(bad.p, 0xFF, 8, s));
  const int eb = dtype_bytes(dtype);
  for (int64_t c0 = 0, k = 0; c0 < n; c0 += kChunkElems, ++k) {
    const int b = static_cast<int>(k & 1);
    const int64_t cn = n - c0 < kChunkElems ? n - c0 : kChunkElems;
    IXB_CUDA_CHECK(cudaEventSynchronize(st.done[b]));
    std::memcpy(st.host[b], static_cast<const char*>(src) + c0 * 8, cn * 8);
    IXB_CUDA_CHECK(cudaMemcpyAsync(st.dev[b].p, st.host[b], cn * 8, cudaMemcpyHostToDevice, s));
    from_file_kernel<<<grid_for(cn), 256, 0, s>>>(st.dev[b].p, kind, cn,
                                                  static_cast<char*>(dst) + c0 * eb, dtype, c0,
                                                  bad.p);
    IXB_LAUNCH_CHECK("from_file_kernel");
    IXB_CUDA_CHECK(cudaEventRecord(st.done[b], s));
  }
  unsigned long long h = 0;
  IXB_CUDA_CHECK(cudaMemcpyAsync(&h, bad.p, 8, cudaMemcpyDeviceToHost, s));
  IXB_CUDA_CHECK(cudaStreamSynchronize(s));
  if (h != ~0ull)
    fail(IXB_SHAPE, what + ": value at position [" + std::to_string(h) +
                        "] does not fit the int32 device index type");
}

}  // namespace

extern "C" {

int ixb_ixt_info(const char* path, int* kind, int* rank, int64_t* dims16) {
  return ixb_guard([&] {
    File fh(path, "rb");
    if (!fh.f) fail(IXB_IO, std::string("cannot open: ") + path);
    const IxtHeader h = read_header(fh.f, path);
    if (kind) *kind = static_cast<int>(h.kind);
    if (rank) *rank = static_cast<int>(h.rank);
    if (dims16)
      for (uint32_t i = 0; i < h.rank; ++i) dims16[i] = h.dims[i];
  });
}

int ixb_ixt_load(const char* path, void* dst, int dtype, ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    File fh(path, "rb");
    if (!fh.f) fail(IXB_IO, std::string("cannot open: ") + path);
    const IxtHeader h = read_header(fh.f, path);
    const int eb = dtype_bytes(dtype);
    if (h.kind == 0 && dtype_is_int(dtype))
      fail(IXB_FAILURE, std::string("real64 tensor cannot be loaded as an integer dtype: ") + path);
    const int64_t n = h.numel;
    if (n == 0) return;
    Staging st(s);
    Scratch<unsigned long long> bad(1, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(bad.p, 0xFF, 8, s));
    const bool raw = (dtype == IXB_F64 && h.kind == 0) || (dtype == IXB_I64 && h.kind == 1);
    for (int64_t c0 = 0, k = 0; c0 < n; c0 += kChunkElems, ++k) {
      const int b = static_cast<int>(k & 1);
      const int64_t cn = n - c0 < kChunkElems ? n - c0 : kChunkElems;
      IXB_CUDA_CHECK(cudaEventSynchronize(st.done[b]));  // buffer b's previous copy retired
      if (std::fread(st.host[b], 8, cn, fh.f) != static_cast<size_t>(cn))
        fail(IXB_IO, std::string("truncated payload in ") + path);
      void* out = static_cast<char*>(dst) + c0 * eb;
      if (raw) {
        IXB_CUDA_CHECK(cudaMemcpyAsync(out, st.host[b], cn * 8, cudaMemcpyHostToDevice, s));
      } else {
        IXB_CUDA_CHECK(
            cudaMemcpyAsync(st.dev[b].p, st.host[b], cn * 8, cudaMemcpyHostToDevice, s));
        from_file_kernel<<<grid_for(cn), 256, 0, s>>>(st.dev[b].p, static_cast<int>(h.kind), cn,
                                                      out, dtype, c0, bad.p);
        IXB_LAUNCH_CHECK("from_file_kernel");
      }
      IXB_CUDA_CHECK(cudaEventRecord(st.done[b], s));
    }
    unsigned long long hb = 0;
    IXB_CUDA_CHECK(cudaMemcpyAsync(&hb, bad.p, 8, cudaMemcpyDeviceToHost, s));
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));
    if (hb != ~0ull)
      fail(IXB_SHAPE, std::string(path) + ": value at position [" + std::to_string(hb) +
                          "] does not fit the int32 device index type");
  });
}

int ixb_ixt_save(const char* path, const void* src, int dtype, int rank, const int64_t* dims,
                 ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    // save_tensor (tensor.cpp:176-195): rank-0 refused; float dtypes are
    // stored as real64, integer dtypes as int64
    if (rank == 0) fail(IXB_IO, std::string("refusing to save rank-0 tensor to ") + path);
    if (rank < 0 || rank > 16) fail(IXB_SHAPE, "ixb_ixt_save: bad rank");
    const int eb = dtype_bytes(dtype);
    int64_t n = 1;
    for (int i = 0; i < rank; ++i) {
      if (dims[i] < 0) fail(IXB_SHAPE, "ixb_ixt_save: negative dimension");
      n *= dims[i];
    }
    File fh(path, "wb");
    if (!fh.f) fail(IXB_IO, std::string("cannot open for writing: ") + path);
    const uint32_t kind = dtype_is_int(dtype) ? 1 : 0, r = static_cast<uint32_t>(rank);
    bool ok = std::fwrite(&kIxtMagic, 4, 1, fh.f) == 1 && std::fwrite(&kIxtVersion, 4, 1, fh.f) == 1 &&
              std::fwrite(&kind, 4, 1, fh.f) == 1 && std::fwrite(&r, 4, 1, fh.f) == 1 &&
              std::fwrite(dims, 8, rank, fh.f) == static_cast<size_t>(rank);
    if (n > 0) {
      Staging st(s);
      std::vector<int64_t> lens;
      for (int64_t c0 = 0, k = 0; c0 < n; c0 += kChunkElems, ++k) {
        const int b = static_cast<int>(k & 1);
        const int64_t cn = n - c0 < kChunkElems ? n - c0 : kChunkElems;
        const void* in = static_cast<const char*>(src) + c0 * eb;
        if (eb == 8) {
          IXB_CUDA_CHECK(cudaMemcpyAsync(st.host[b], in, cn * 8, cudaMemcpyDeviceToHost, s));
        } else {
          to_file_kernel<<<grid_for(cn), 256, 0, s>>>(in, dtype, cn, st.dev[b].p);
          IXB_LAUNCH_CHECK("to_file_kernel");
          IXB_CUDA_CHECK(
              cudaMemcpyAsync(st.host[b], st.dev[b].p, cn * 8, cudaMemcpyDeviceToHost, s));
        }
        IXB_CUDA_CHECK(cudaEventRecord(st.done[b], s));
        // write the previous chunk while this one is in flight
        if (k > 0) {
          const int pb = 1 - b;
          IXB_CUDA_CHECK(cudaEventSynchronize(st.done[pb]));
          ok = ok && std::fwrite(st.host[pb], 8, lens.back(), fh.f) ==
                         static_cast<size_t>(lens.back());
        }
        lens.push_back(cn);
      }
      const int lb = static_cast<int>((lens.size() - 1) & 1);
      IXB_CUDA_CHECK(cudaEventSynchronize(st.done[lb]));
      ok = ok && std::fwrite(st.host[lb], 8, lens.back(), fh.f) == static_cast<size_t>(lens.back());
    }
    if (!ok || std::fflush(fh.f) != 0) fail(IXB_IO, std::string("write failed: ") + path);
  });
}

int ixb_mtx_read(const char* path, ixb_mtx** out, int* is_dense, int* kind, int64_t* rows,
                 int64_t* cols, int64_t* nnz) {
  return ixb_guard([&] {
    if (!out) fail(IXB_SHAPE, "ixb_mtx_read: null handle pointer");
    *out = nullptr;
    ixb_mtx* m = parse_mtx(path);
    *out = m;
    if (is_dense) *is_dense = m->dense ? 1 : 0;
    if (kind) *kind = m->kind;
    if (rows) *rows = m->rows;
    if (cols) *cols = m->cols;
    if (nnz) *nnz = m->dense ? m->rows * m->cols : static_cast<int64_t>(m->r.size());
  });
}

int ixb_mtx_to_host(const ixb_mtx* m, int64_t* row, int64_t* col, void* values) {
  return ixb_guard([&] {
    if (!m) fail(IXB_SHAPE, "ixb_mtx_to_host: null handle");
    const size_t n = m->dense ? static_cast<size_t>(m->rows * m->cols) : m->r.size();
    if (!m->dense) {
      if (row) std::memcpy(row, m->r.data(), n * 8);
      if (col) std::memcpy(col, m->c.data(), n * 8);
    }
    if (values) std::memcpy(values, m->kind ? static_cast<const void*>(m->iv.data())
                                            : static_cast<const void*>(m->rv.data()),
                            n * 8);
  });
}

int ixb_mtx_to_device(const ixb_mtx* m, int32_t* row, int32_t* col, void* values, int dtype,
                      ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!m) fail(IXB_SHAPE, "ixb_mtx_to_device: null handle");
    if (m->rows > INT32_MAX || m->cols > INT32_MAX)
      fail(IXB_SHAPE, "matrix extents exceed the int32 device index type");
    const int64_t n = m->dense ? m->rows * m->cols : static_cast<int64_t>(m->r.size());
    if (!m->dense) {
      if (row) upload8(m->r.data(), 1, n, row, IXB_I32, s, "row coordinates");
      if (col) upload8(m->c.data(), 1, n, col, IXB_I32, s, "column coordinates");
    }
    if (values) {
      if (m->kind == 0 && dtype_is_int(dtype))
        fail(IXB_FAILURE, "real MatrixMarket values cannot be loaded as an integer dtype");
      upload8(m->kind ? static_cast<const void*>(m->iv.data())
                      : static_cast<const void*>(m->rv.data()),
              m->kind, n, values, dtype, s, "values");
    }
  });
}

void ixb_mtx_free(ixb_mtx* m) { delete m; }

}  // extern "C"
