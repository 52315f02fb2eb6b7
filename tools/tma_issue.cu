// Microbenchmark: how fast can one CTA move K4-shaped gathers (perf experiment
// backing DESIGN.md §K4, not part of the library)?
//   tma  : W warps each run their own STAGES-deep ring of BOXES TMA boxes per
//          stage (4 KB {64,16,2} B tiles or 512 B {16,16} AV blocks), one
//          issuing lane per warp; a consumer lane per warp releases stages.
//   cpa  : W warps gather 4 KB tiles with cp.async (16 B per lane, 8
//          instructions per tile), completion via cp.async.mbarrier.arrive.noinc.
// Reports GB/s over the whole GPU for 1 and 2 CTAs per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I ../paper_2510_17505_b200/csrc tma_issue.cu -o tma_issue -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace ixb::sm100;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352d;
  x ^= x >> 15;
  x *= 0x846ca68b;
  x ^= x >> 16;
  return x;
}

constexpr int STAGES = 4;

// mode 0: 3-D 4 KB boxes; mode 1: 2-D 512 B boxes; mode 2: cp.async 4 KB tiles
__global__ void issue_kernel(const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmA, const uint8_t* gB,
                             int mode, int iters, int boxes, uint32_t region) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  __shared__ uint64_t full[16][STAGES], empty[16][STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int w = 0; w < nw; ++w)
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[w][s], mode == 2 ? 32 : 1);
        mbar_init(&empty[w][s], 1);
      }
    fence_barrier_init();
  }
  __syncthreads();
  const uint32_t box = mode == 1 ? 512 : 4096;
  uint8_t* mine = smem + warp * region;
  const uint64_t keep = l2_evict_last();
  // the issuing warp consumes its own ring: before reusing stage s it waits
  // for the previous fill of s to land
  for (int it = 0; it < iters; ++it) {
    const int stage = it % STAGES;
    if (it >= STAGES && (lane == 0 || mode == 2))
      mbar_wait(&full[warp][stage], ((it / STAGES) - 1) & 1);
    __syncwarp();
    uint8_t* st = mine + stage * boxes * box;
    if (mode == 2) {
      for (int b = 0; b < boxes; ++b) {
        const uint32_t kb = hash32(blockIdx.x * 7919u + warp * 104729u + it * 16 + b) % 512;
        const uint8_t* src = gB + static_cast<size_t>(kb) * 16 * 1024;  // 16 rows x 256 B
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int idx = c * 32 + lane;  // 16 B chunk of the 4 KB tile
          const int row = idx >> 4, col = idx & 15;
          cp_async_16(smem_u32(st + b * box + idx * 16), src + row * 1024 + col * 16, 16);
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                       smem_u32(&full[warp][stage]))
                   : "memory");
    } else if (lane == 0) {
      mbar_arrive_expect_tx(&full[warp][stage], boxes * box);
      for (int b = 0; b < boxes; ++b) {
        const uint32_t h = hash32(blockIdx.x * 7919u + warp * 104729u + it * 16 + b);
        if (mode == 0)
          tma_load_3d(st + b * box, &tmB, &full[warp][stage], 0, (h % 512) * 16, 0, keep);
        else
          tma_load_2d(st + b * box, &tmA, &full[warp][stage], 0, (h % 28000) * 16, keep);
      }
    }
  }
  for (int it = iters; it < iters + STAGES; ++it) {
    const int stage = it % STAGES;
    if (it >= STAGES && (lane == 0 || mode == 2))
      mbar_wait(&full[warp][stage], ((it / STAGES) - 1) & 1);
  }
  __syncwarp();
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void *bufB, *bufA;
  cudaMalloc(&bufB, 8u << 20);   // B [8192 rows x 512] bf16
  cudaMalloc(&bufA, 15u << 20);  // AV [28000 x 16 x 16] bf16
  cudaMemset(bufB, 1, 8u << 20);
  cudaMemset(bufA, 1, 15u << 20);
  auto enc = encode();
  CUtensorMap tmB, tmA;
  {
    cuuint64_t dims[3] = {64, 8192, 8};
    cuuint64_t strides[2] = {1024, 128};
    cuuint32_t boxd[3] = {64, 16, 2};
    cuuint32_t es[3] = {1, 1, 1};
    enc(&tmB, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, bufB, dims, strides, boxd, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[2] = {16, 28000 * 16};
    cuuint64_t strides[1] = {32};
    cuuint32_t boxd[2] = {16, 16};
    cuuint32_t es[2] = {1, 1};
    enc(&tmA, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, bufA, dims, strides, boxd, es,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"tma_4KB", "tma_512B", "cpasync_4KB"};
  printf("[");
  bool first = true;
  for (int mode = 0; mode < 3; ++mode) {
    for (int cps : {1, 2}) {
      for (int warps : {1, 2, 4, 8}) {
        for (int boxes : {1, 4}) {
          const uint32_t box = mode == 1 ? 512 : 4096;
          const uint32_t region = STAGES * boxes * box;
          const size_t smem = size_t(region) * warps + 1024;
          if (smem > 200 * 1024 / cps) continue;
          cudaFuncSetAttribute(issue_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(smem));
          const int iters = 512 / boxes;
          const int grid = sms * cps;
          issue_kernel<<<grid, warps * 32, smem>>>(tmB, tmA, static_cast<uint8_t*>(bufB), mode,
                                                  8, boxes, region);
          cudaEventRecord(e0);
          issue_kernel<<<grid, warps * 32, smem>>>(tmB, tmA, static_cast<uint8_t*>(bufB), mode,
                                                  iters, boxes, region);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          const double nbox = double(grid) * warps * iters * boxes;
          printf("%s{\"mode\": \"%s\", \"ctas_per_sm\": %d, \"warps\": %d, \"boxes_per_stage\": %d, "
                 "\"GBps\": %.1f, \"cycles_per_box_per_sm\": %.1f, \"err\": %d}\n",
                 first ? "" : ",", names[mode], cps, warps, boxes, nbox * box / ms / 1e6,
                 ms * 1e-3 * 1.965e9 / (nbox / sms), int(cudaGetLastError()));
          first = false;
        }
      }
    }
  }
  printf("]\n");
  return 0;
}
