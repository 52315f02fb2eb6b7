// Microbenchmark: L2 -> SM read throughput on B200 (the denominator of the
// L2 fraction bench.py reports for the gather paths) and the TMA gather rate
// of K4-shaped B tiles. Not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I ../paper_2510_17505_b200/csrc l2_rate.cu -o l2_rate -lcuda
//
// mode ldg: every warp reads random 4 KB chunks of an L2-resident buffer with
//   16-byte ld.global.nc (8 independent loads in flight per lane).
// mode tma: one producer thread per CTA keeps a STAGES-deep ring of 3-D TMA
//   boxes {64 n, 16 rows, ATOMS} (the K4 B-tile shape) from random row blocks
//   in flight; a consumer warp releases each stage as soon as it lands.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

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

__global__ void ldg_kernel(const int4* __restrict__ buf, size_t nchunks, int iters, int4* sink) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int4 acc = make_int4(0, 0, 0, 0);
  for (int it = 0; it < iters; ++it) {
    // 4 KB chunk = 256 int4 = 8 per lane
    const size_t c = hash32(gw * 7919u + it) % nchunks;
    const int4* p = buf + c * 256 + lane;
    int4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(p + u * 32);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc.x ^= v[u].x;
      acc.y ^= v[u].y;
      acc.z ^= v[u].z;
      acc.w ^= v[u].w;
    }
  }
  if (acc.x == 0x12345678) sink[0] = acc;
}

template <int STAGES>
__global__ void tma_kernel(const __grid_constant__ CUtensorMap tm, int kb_count, int iters,
                           uint32_t box_bytes, int per_stage) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[STAGES], empty[STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint64_t keep = l2_evict_last();
  if (warp == 0 && lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&empty[stage], phase ^ 1);
      mbar_arrive_expect_tx(&full[stage], box_bytes * per_stage);
      for (int b = 0; b < per_stage; ++b) {
        const int kb = hash32(blockIdx.x * 104729u + it * 8 + b) % kb_count;
        tma_load_3d(smem + (stage * per_stage + b) * box_bytes, &tm, &full[stage], 0, kb * 16, 0,
                    keep);
      }
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else if (warp == 1 && lane == 0) {
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&full[stage], phase);
      mbar_arrive(&empty[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1;
      }
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = 8u << 20;  // 8 MB (cfg2's B), L2-resident
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  int4* sink;
  cudaMalloc(&sink, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  printf("{\"sms\": %d, \"ldg\": [", sms);
  bool first = true;
  for (int cps : {1, 2, 4, 8}) {
    for (int threads : {256, 512}) {
      const int iters = 256;
      const int grid = sms * cps;
      ldg_kernel<<<grid, threads>>>(static_cast<int4*>(buf), bytes / 4096, 8, sink);
      cudaEventRecord(e0);
      ldg_kernel<<<grid, threads>>>(static_cast<int4*>(buf), bytes / 4096, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double moved = double(grid) * (threads / 32) * iters * 4096.0;
      printf("%s{\"ctas_per_sm\": %d, \"threads\": %d, \"GBps\": %.1f}", first ? "" : ", ", cps,
             threads, moved / ms / 1e6);
      first = false;
    }
  }
  printf("], \"tma\": [");
  // B viewed as {64 n, 8192 rows, 8 atoms} bf16, row pitch 1024 B
  auto enc = encode();
  first = true;
  for (int atoms : {2, 4, 8}) {
    CUtensorMap tm;
    cuuint64_t dims[3] = {64, 8192, 8};
    cuuint64_t strides[2] = {1024, 128};
    cuuint32_t box[3] = {64, 16, static_cast<cuuint32_t>(atoms)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("encode failed %d\n", r);
      return 1;
    }
    const uint32_t box_bytes = 64 * 16 * atoms * 2;
    for (int cps : {1, 2, 3, 4}) {
      for (int per_stage : {1, 2, 4}) {
        constexpr int S = 4;
        const size_t smem = size_t(S) * per_stage * box_bytes + 1024;
        if (smem > 220 * 1024 / cps) continue;
        cudaFuncSetAttribute(tma_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(smem));
        const int grid = sms * cps;
        const int iters = 2048 / per_stage;
        tma_kernel<S><<<grid, 64, smem>>>(tm, 512, 16, box_bytes, per_stage);
        cudaEventRecord(e0);
        tma_kernel<S><<<grid, 64, smem>>>(tm, 512, iters, box_bytes, per_stage);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        const double moved = double(grid) * iters * per_stage * box_bytes;
        printf("%s{\"box_bytes\": %u, \"ctas_per_sm\": %d, \"boxes_per_stage\": %d, \"GBps\": %.1f, "
               "\"err\": %d}",
               first ? "" : ", ", box_bytes, cps, per_stage, moved / ms / 1e6, int(err));
        first = false;
      }
    }
  }
  printf("]}\n");
  return 0;
}
