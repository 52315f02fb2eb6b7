// TMA tensor-map helpers (bf16 tensors).
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace ixb {

CUtensorMap make_tmap_2d(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                         uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw);
// 2-D fp32 tensor (e.g. an output tile written back by TMA store).
CUtensorMap make_tmap_2d_f32(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                             uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw);
// 2-D int32 tensor (no swizzle), e.g. index tables staged by TMA.
CUtensorMap make_tmap_2d_i32(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                             uint32_t box_inner, uint32_t box_outer);
// 3-D bf16 tensor (fp32 with f32 = true).
CUtensorMap make_tmap_3d(const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1,
                         uint64_t s2, uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle sw,
                         bool f32 = false);

}  // namespace ixb
