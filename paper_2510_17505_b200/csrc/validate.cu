// K8 — index range validation and group-order utilities shared by the
// evaluators (checked_index semantics, plan.cpp:249-259).
#include "common.cuh"

namespace ixb {
namespace {

__global__ void validate_range_kernel(const int32_t* idx, int64_t n, int64_t extent, int operand,
                                      ErrorRecord* err) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = idx[i];
    if (v < 0 || static_cast<int64_t>(v) >= extent) report_index_error(err, operand, i, v);
  }
}

__global__ void gather_rows_kernel(const int32_t* perm, const uint32_t* src, uint32_t* dst,
                                   int64_t rows, int64_t words) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows * words;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / words;
    dst[i] = src[static_cast<int64_t>(perm[r]) * words + i % words];
  }
}

}  // namespace

void validate_range(const int32_t* idx, int64_t n, int64_t extent, int operand, cudaStream_t s) {
  if (n <= 0) return;
  int64_t grid = ceil_div(n, 256);
  if (grid > 8 * sm_count()) grid = 8 * sm_count();
  validate_range_kernel<<<grid, 256, 0, s>>>(idx, n, extent, operand, device_error_record());
  IXB_LAUNCH_CHECK("validate_range_kernel");
}

void gather_rows(const int32_t* perm, const void* src, void* dst, int64_t rows, int64_t row_bytes,
                 cudaStream_t s) {
  if (rows <= 0) return;
  const int64_t words = row_bytes / 4;
  int64_t grid = ceil_div(rows * words, 256);
  if (grid > 16 * sm_count()) grid = 16 * sm_count();
  gather_rows_kernel<<<grid, 256, 0, s>>>(perm, static_cast<const uint32_t*>(src),
                                          static_cast<uint32_t*>(dst), rows, words);
  IXB_LAUNCH_CHECK("gather_rows_kernel");
}

}  // namespace ixb
