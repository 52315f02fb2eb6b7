// Internal host/device definitions shared by the ixb translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/ixb.h"

namespace ixb {

// Device-side record of the first index-range offender (see common.cuh).
struct ErrorRecord {
  unsigned long long key;  // (operand << 56) | flat position; ~0 = none
  long long value[8];
};

constexpr unsigned long long kNoError = ~0ull;

// Host exception carrying an ixb_status; converted at the C-ABI boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);
#define IXB_CUDA_CHECK(x) ::ixb::cuda_check((x), #x)
#define IXB_LAUNCH_CHECK(name) \
  do {                         \
    ::ixb::note_launch();      \
    ::ixb::cuda_check(cudaGetLastError(), name); \
  } while (0)

void note_launch(int n = 1);
int sm_count();
// Opts `func` in to `bytes` of dynamic shared memory on the CURRENT device.
// The attribute is per device/context, so the opt-in is tracked per
// (device, function) and repeated on every device the process drives.
void set_max_dynamic_smem(const void* func, int bytes, const char* name);

// Per-device error record (lazily allocated, reset after each check).
ErrorRecord* device_error_record();
// n arrival counters for a kernel launched on `stream` (one region per
// stream, so concurrent launches never share one): zero on entry, and every
// kernel using them leaves them zero again.
unsigned* work_counters(cudaStream_t stream, size_t n);
// A persistent device buffer of at least `bytes` owned by `stream` (grown on
// demand, never shrunk): kernel scratch that must not add allocation nodes
// to a captured CUDA graph. Contents are undefined on entry. Returns null
// when the buffer would have to grow while `stream` is being captured.
// `tag` keeps the buffers of different kernels apart.
enum { kBufK4Partials = 0, kBufK3Split = 1 };
void* stream_buffer(cudaStream_t stream, size_t bytes, int tag);
// Resets the record on `stream` before a checked launch.
void reset_error_record(cudaStream_t stream);
// Syncs `stream`, reads the record; on an offender throws IXB_INDEX_RANGE with
// the reference message (plan.cpp:253-256). names/index arrays/extents are
// per operand; idx_arrays are the device index arrays the operand id refers to.
struct OperandInfo {
  const char* index_name;   // e.g. "AK"
  const char* target_name;  // e.g. "B"
  int target_dim;           // dim of the target indexed
  int64_t extent;           // its extent
  const int32_t* device_array;
  int64_t numel;
};
void check_error_record(cudaStream_t stream, const OperandInfo* ops, int nops);

// Small device->host reads of a plan phase through one pinned staging
// buffer per host thread: every add() is queued on `stream`, wait() syncs
// once and copies the values out (a pageable destination would make each
// read its own staged, host-blocking round trip). Reads past the buffer's
// 4 KB go straight to their destination.
class HostReads {
 public:
  explicit HostReads(cudaStream_t stream) : s_(stream) {}
  void add(void* dst, const void* src, size_t bytes);
  void wait();

 private:
  cudaStream_t s_;
  size_t used_ = 0;
  struct Item { void* dst; size_t off, bytes; };
  Item items_[16];
  int n_ = 0;
};

// Stream-ordered scratch allocation (cudaMallocAsync pool).
void* scratch_alloc(size_t bytes, cudaStream_t stream);
void scratch_free(void* p, cudaStream_t stream);

template <typename T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  Scratch() = default;
  Scratch(size_t n, cudaStream_t st) : s(st) {
    p = static_cast<T*>(scratch_alloc(n * sizeof(T) + 16, st));
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  Scratch(Scratch&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
  Scratch& operator=(Scratch&& o) noexcept {
    reset();
    p = o.p;
    s = o.s;
    o.p = nullptr;
    return *this;
  }
  void reset() {
    if (p) scratch_free(p, s);
    p = nullptr;
  }
  ~Scratch() { reset(); }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// K8 — index range validation (checked_index, plan.cpp:249-259): records the
// first position of `idx` outside [0, extent) as `operand` in the error record.
void validate_range(const int32_t* idx, int64_t n, int64_t extent, int operand, cudaStream_t s);
// Whether a group-coordinate array is non-decreasing (one pass + sync).
bool groups_sorted(const int32_t* AM, int64_t G, cudaStream_t s);
// Stable permutation of groups by group coordinate (CUB radix sort).
void sort_groups(const int32_t* AM, int64_t G, cudaStream_t s, Scratch<int32_t>& am_sorted,
                 Scratch<int32_t>& perm);
// dst[i, :] = src[perm[i], :] for rows of `row_bytes` bytes (multiple of 4).
void gather_rows(const int32_t* perm, const void* src, void* dst, int64_t rows, int64_t row_bytes,
                 cudaStream_t s);

// Conv plan helpers for the sharded entry (shard.cpp): output rows of the
// plan, and `=` evaluation of rows [r0, r1) (r0 a multiple of 128; the unit
// tensor-core path, or the whole plan with r0 == 0 and r1 == rows).
int64_t conv_plan_rows(const ixb_conv_plan* plan);
void conv_plan_run_rows(ixb_conv_plan* plan, const void* In, int64_t Cin, const void* Weight,
                        int64_t Cout, float* Out, int64_t r0, int64_t r1, cudaStream_t s);

}  // namespace ixb

// ABI guard: converts exceptions into status codes + thread-local message.
int ixb_guard_set(int code, const char* msg);
template <typename F>
int ixb_guard(F&& f) {
  try {
    f();
    return ixb_guard_set(IXB_OK, "");
  } catch (const ixb::Error& e) {
    return ixb_guard_set(e.code, e.what());
  } catch (const std::exception& e) {
    return ixb_guard_set(IXB_FAILURE, e.what());
  }
}
