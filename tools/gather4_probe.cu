// Probe of TMA tile::gather4 semantics on sm_100a (perf/design experiment for
// K6; not part of the library): which box height the tensor map needs, where
// the 4 rows land under SWIZZLE_128B, and whether out-of-range rows are
// zero-filled. Build: nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17
//   -I ../paper_2510_17505_b200/csrc gather4_probe.cu -o gather4_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstring>

#include "sm100.cuh"

using namespace ixb::sm100;

__global__ void probe(const __grid_constant__ CUtensorMap tm, int r0, int r1, int r2, int r3,
                      uint16_t* out) {
  __shared__ __align__(1024) uint16_t sm[4 * 64];
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) sm[i] = 0xFFFF;
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
    mbar_arrive_expect_tx(&bar, 4 * 64 * 2);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(sm)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bar)), "r"(0), "r"(r0), "r"(r1),
        "r"(r2), "r"(r3)
        : "memory");
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int rows = 16, cols = 64;
  uint16_t h[rows * cols];
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = static_cast<uint16_t>(r * 256 + c);
  uint16_t *d, *o;
  cudaMalloc(&d, sizeof h);
  cudaMalloc(&o, 512);
  cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                          cudaEnableDefault, &q);
  for (int boxh : {1, 4}) {
    for (auto sw : {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_128B}) {
      CUtensorMap tm;
      cuuint64_t dims[2] = {cols, rows};
      cuuint64_t strides[1] = {cols * 2};
      cuuint32_t box[2] = {64, static_cast<cuuint32_t>(boxh)};
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("boxh=%d sw=%d: encode failed %d\n", boxh, (int)sw, (int)r);
        continue;
      }
      cudaMemset(o, 0, 512);
      probe<<<1, 128>>>(tm, 5, 2, 20 /* out of range */, 7, o);
      cudaError_t e = cudaDeviceSynchronize();
      uint16_t ho[256];
      cudaMemcpy(ho, o, 512, cudaMemcpyDeviceToHost);
      printf("boxh=%d sw=%d err=%s\n", boxh, (int)sw, cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
      for (int rr = 0; rr < 4; ++rr) {
        printf("  smem row %d:", rr);
        for (int c = 0; c < 64; c += 8) printf(" %04x", ho[rr * 64 + c]);
        printf("\n");
      }
    }
  }
  return 0;
}
