// Shared plumbing of the drop-in (integration/): device buffers, host<->device
// moves of reference Tensors and coordinate vectors, and the mapping of ixb
// status codes back onto the reference's exception types (driver.hpp:19-27).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "ixb.h"
#include "ixsum/driver.hpp"

namespace ixsum::b200::detail {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  explicit DevBuf(size_t n) : bytes(n) {
    if (cudaMalloc(&p, n ? n : 16) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

inline void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

/// ixb status -> the reference exception class with the library's message.
inline void check(int code) {
  if (code == IXB_OK) return;
  const std::string msg = ixb_last_error();
  switch (code) {
    case IXB_PARSE: throw ParseError(msg, 0);
    case IXB_BIND: throw BindError(msg);
    case IXB_SHAPE: throw ShapeError(msg);
    case IXB_INDEX_RANGE: throw IndexRangeError(msg);
    case IXB_IO: throw IoError(msg);
    default: throw std::runtime_error(msg);
  }
}

/// The reference stores fp64 or int64; the builders move 8-byte values unchanged.
inline int value_dtype(const Tensor& t) { return t.is_int() ? IXB_I64 : IXB_F64; }

inline std::unique_ptr<DevBuf> upload_values(const Tensor& t) {
  auto d = std::make_unique<DevBuf>(static_cast<size_t>(t.numel()) * 8);
  const void* src = t.is_int() ? static_cast<const void*>(t.ints().data())
                               : static_cast<const void*>(t.reals().data());
  cuda_ok(cudaMemcpy(d->p, src, d->bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  return d;
}

inline Tensor download_values(const DevBuf& d, ElemKind kind, std::vector<int64_t> shape) {
  Tensor t = Tensor::zeros(kind, std::move(shape));
  void* dst = t.is_int() ? static_cast<void*>(t.ints().data())
                         : static_cast<void*>(t.reals().data());
  cuda_ok(cudaMemcpy(dst, d.p, static_cast<size_t>(t.numel()) * 8, cudaMemcpyDeviceToHost),
          "cudaMemcpy D2H");
  return t;
}

/// int64 coordinates -> device int32. Device coordinates are int32 (every
/// extent the device formats address is below 2^31); a coordinate outside
/// that range cannot be represented and is rejected, never wrapped.
inline std::unique_ptr<DevBuf> upload_coords(const std::vector<int64_t>& v, const char* what) {
  std::vector<int32_t> h(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i] < INT32_MIN || v[i] > INT32_MAX) {
      throw ShapeError(std::string(what) + " coordinate " + std::to_string(v[i]) +
                       " at position [" + std::to_string(i) +
                       "] exceeds the device's int32 range");
    }
    h[i] = static_cast<int32_t>(v[i]);
  }
  auto d = std::make_unique<DevBuf>(h.size() * 4);
  cuda_ok(cudaMemcpy(d->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
  return d;
}

inline std::vector<int64_t> download_coords(const DevBuf& d, int64_t n) {
  std::vector<int32_t> h(static_cast<size_t>(n));
  cuda_ok(cudaMemcpy(h.data(), d.p, h.size() * 4, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  return std::vector<int64_t>(h.begin(), h.end());
}

inline std::vector<uint8_t> download_mask(const DevBuf& d, int64_t n) {
  std::vector<uint8_t> h(static_cast<size_t>(n));
  cuda_ok(cudaMemcpy(h.data(), d.p, h.size(), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
  return h;
}

}  // namespace ixsum::b200::detail
