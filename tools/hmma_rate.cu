// Microbenchmark: throughput of warp-level mma.sync.m16n8k16 (bf16 -> fp32)
// on B200, register operands, independent accumulator chains. Perf
// experiment for the K4 design; not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 hmma_rate.cu -o hmma_rate
#include <cstdio>

__global__ void hmma(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* o;
  cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    hmma<<<148 * 4, warps * 32>>>(o, 16);
    cudaEventRecord(e0);
    hmma<<<148 * 4, warps * 32>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 16 * 8 * 16 * 8 * double(iters) * warps * 148 * 4;
    printf("warps/CTA %2d (4 CTAs/SM): %.1f TFLOP/s (%s)\n", warps, flops / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
