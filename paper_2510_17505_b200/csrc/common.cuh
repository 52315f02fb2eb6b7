// Shared device helpers for the sm_100a kernels of the Insum executor.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ixb_internal.h"

namespace ixb {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// In-kernel index validation (reference semantics: checked_index,
// plan.cpp:249-259). The first offender — in the order the reference's plan
// executor meets them: gathers (inputs) before scatters (outputs), then by
// flat position — wins through one 64-bit atomicMin on a packed key.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void report_index_error(ErrorRecord* rec, int operand, int64_t pos,
                                                   int64_t value) {
  unsigned long long key =
      (static_cast<unsigned long long>(operand) << 56) | static_cast<unsigned long long>(pos);
  unsigned long long old = atomicMin(&rec->key, key);
  if (key < old) {
    // Racy but benign: a later smaller key overwrites; host re-reads after sync.
    rec->value[operand] = value;
  }
}

// ---------------------------------------------------------------------------
// Cache-hinted global loads.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Read-only 128-bit load that keeps the line in L2 (dense operand reused
// across groups) and skips L1 allocation.
__device__ __forceinline__ float4 ldg_f4_keep(const float* p, uint64_t pol) {
  float4 v;
  asm volatile(
      "ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldg_f_keep(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v)
               : "l"(p), "l"(pol));
  return v;
}
// Streaming loads for format metadata (read once).
__device__ __forceinline__ int ldg_i_stream(const int* p, uint64_t pol) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ldg_f_stream(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(v)
               : "l"(p), "l"(pol));
  return v;
}

// 16-byte read-only load that skips L1 allocation (gathered rows).
__device__ __forceinline__ uint4 ldg_nc_v4(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

}  // namespace ixb
