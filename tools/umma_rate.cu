// Microbenchmark: issue rate of tcgen05.mma (kind::f16, M=128, K=16) for small N
// from one thread, with uniform descriptors and with per-lane operands
// (compiler ELECT loop). Perf experiment backing DESIGN.md §K4; not part of
// the library. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I ../paper_2510_17505_b200/csrc umma_rate.cu -o umma_rate
#include <cstdio>

#include "sm100.cuh"

using namespace ixb::sm100;

template <int N>
__global__ void rate(long long* out, int iters, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, 512);
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, true, false);
    const uint64_t ad = smem_desc(smem_u32(sm), 2048, 1024, kLayoutSW128);
    const uint64_t bd = smem_desc(smem_u32(sm + 32768), 16, 256, kLayoutSW32);
    long long t0 = clock64();
    if (mode == 0) {
      if (lane == 0)
        for (int i = 0; i < iters; ++i) umma_f16_acc(tmem + (i & 15) * 16, ad, bd + (i & 7) * 32, idesc);
    } else if (mode >= 2 && mode < 500) {
      // commit to a scratch barrier every `mode` MMAs (mode 2: commits only)
      __shared__ uint64_t cb[4];
      if (lane == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1);
        fence_barrier_init();
        for (int i = 0; i < iters; ++i) {
          if (mode > 2) umma_f16_acc(tmem + (i & 15) * 16, ad, bd + (i & 7) * 32, idesc);
          if (mode == 2 || i % mode == 0) umma_commit(&cb[i & 3]);
        }
      }
      if (mode >= 1000 && lane == 1) {  // commits from another lane of the same warp
        for (int i = 0; i < iters / 11; ++i) umma_commit(&cb[i & 3]);
      }
    } else if (mode >= 1000) {
      __shared__ uint64_t cb[4];
      if (lane == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1);
        fence_barrier_init();
      }
      __syncwarp();
      if (lane == 0)
        for (int i = 0; i < iters; ++i) umma_f16_acc(tmem + (i & 15) * 16, ad, bd + (i & 7) * 32, idesc);
      if (lane == 1)
        for (int i = 0; i < iters / 11; ++i) umma_commit(&cb[i & 3]);
    } else if (mode >= 500 && mode < 1000) {
      // kernel pattern: batches of 11 per-lane MMAs; commit after every batch (mode 501)
      // or every 8th batch (508), or never (500)
      __shared__ uint64_t cb[4];
      if (lane == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&cb[i], 1);
        fence_barrier_init();
      }
      __syncwarp();
      const int every = (mode - 500) % 100;
      const int bsz = mode >= 700 ? 1 : mode >= 600 ? 4 : 11;  // 6xx: batches of 4, 7xx: single-lane
      int b = 0;
      for (int i = 0; i < iters; i += bsz, ++b) {
        if (lane < bsz) umma_f16_acc(tmem + lane * 16, ad + (lane & 3) * 128, bd + lane * 32, idesc);
        __syncwarp();
        if (every && b % every == 0 && lane == 0) umma_commit(&cb[b & 3]);
        __syncwarp();
      }
    } else {
      // per-lane operands: 16 lanes each issue one MMA per round
      for (int i = 0; i < iters; i += 16) {
        if (lane < 16) umma_f16_acc(tmem + lane * 16, ad + (lane & 3) * 128, bd + lane * 32, idesc);
        __syncwarp();
      }
    }
    if (lane == 0) {
      umma_commit(&bar);
      mbar_wait(&bar, 0);
      out[blockIdx.x] = clock64() - t0;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int N>
void run(int mode, long long* d, int iters) {
  cudaFuncSetAttribute(rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  rate<N><<<148, 128, 64 * 1024>>>(d, iters, mode);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double m = 0;
  for (long long x : h) m += x;
  printf("N=%3d mode=%d: %.1f cycles per MMA (err %s)\n", N, mode, m / 148 / iters,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  for (int mode = 0; mode < 2; ++mode) {
    run<16>(mode, d, 4096);
    run<32>(mode, d, 4096);
    run<64>(mode, d, 4096);
    run<128>(mode, d, 4096);
    run<256>(mode, d, 4096);
  }
  for (int mode : {2, 3, 11, 32, 128, 1000})  // commit cost: alone, every k-th MMA, other lane
    run<16>(mode, d, 4096);
  for (int mode : {600, 601, 604, 616, 700, 701, 704, 716, 732})
    run<16>(mode, d, 4096);
  return 0;
}
