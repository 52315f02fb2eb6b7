// Microbenchmark: does a CTA-pair MMA (tcgen05.mma.cta_group::2, M = 256
// over two SMs) cost the same per instruction as a single-SM M = 128 MMA at
// small N? For 16-wide blocks (K4) the tensor pipe is bound by a fixed
// ~50-cycle cost per instruction (tools/umma_rate.cu); if that cost is per
// dispatch, a pair doubles the block-MMA rate. Operand values do not matter
// (timing only). Waits are bounded so a mistake cannot hang the GPU.
// Perf experiment backing DESIGN.md §8; not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I ../paper_2510_17505_b200/csrc umma_pair_rate.cu -o umma_pair_rate
#include <cstdio>

#include "sm100.cuh"

using namespace ixb::sm100;

__device__ __forceinline__ bool wait_bounded(uint64_t* bar, uint32_t parity) {
  const long long t0 = clock64();
  for (;;) {
    uint32_t done;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return true;
    if (clock64() - t0 > (1ll << 31)) return false;  // ~1 s: give up
  }
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) pair_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers and TMEM ready before the leader issues
  tc_fence_after();
  const uint32_t tmem = slot;
  long long dt = -1;
  if (rank == 0 && warp == 0 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(256, N, true, false);
    const uint64_t ad = smem_desc(smem_u32(sm), 2048, 1024, kLayoutSW128);
    const uint64_t bd = smem_desc(smem_u32(sm + 32768), 16, 256, kLayoutSW32);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(
              tmem + (N >= 256 ? 0 : (i & 7) * 32)),
          "l"(ad), "l"(bd + (i & 7) * 32), "r"(idesc), "r"(1u));
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
        "[%0], %1;" ::"r"(smem_u32(&bar)),
        "h"(static_cast<uint16_t>(3)));
    dt = wait_bounded(&bar, 0) ? clock64() - t0 : -2;
  } else if (rank == 1 && warp == 0 && lane == 0) {
    dt = wait_bounded(&bar, 0) ? 0 : -2;  // keep operands and TMEM alive until done
  }
  if (warp == 0 && lane == 0) out[blockIdx.x] = dt;
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

template <int N>
__global__ void single_rate(long long* out, int iters) {
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
  if (warp == 0 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, true, false);
    const uint64_t ad = smem_desc(smem_u32(sm), 2048, 1024, kLayoutSW128);
    const uint64_t bd = smem_desc(smem_u32(sm + 32768), 16, 256, kLayoutSW32);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_f16(tmem + (i & 15) * 16, ad, bd + (i & 7) * 32, idesc, 1u);
    umma_commit(&bar);
    out[blockIdx.x] = wait_bounded(&bar, 0) ? clock64() - t0 : -2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


// k issuing CTAs per SM (128 TMEM columns, 48 KB smem each): does the per-MMA
// cost overlap across issuing streams, or is it tensor-pipe occupancy?
template <int N>
__global__ void multi_rate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, 128);
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, true, false);
    const uint64_t ad = smem_desc(smem_u32(sm), 2048, 1024, kLayoutSW128);
    const uint64_t bd = smem_desc(smem_u32(sm + 32768), 16, 256, kLayoutSW32);
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_f16(tmem + (i & 3) * 16, ad, bd + (i & 7) * 32, idesc, 1u);
    umma_commit(&bar);
    out[blockIdx.x] = wait_bounded(&bar, 0) ? clock64() - t0 : -2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

void report_multi(int per_sm, long long* d, int iters) {
  const int grid = 148 * per_sm;
  cudaFuncSetAttribute(multi_rate<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  multi_rate<16><<<grid, 128, 48 * 1024>>>(d, iters);
  const cudaError_t e = cudaDeviceSynchronize();
  static long long h[148 * 4];
  cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < grid; ++i) m += h[i];
  printf("%d issuing CTAs/SM, M=128 N=16: %.1f cycles per MMA per stream, %.1f per SM (%s)\n",
         per_sm, m / grid / iters, m / grid / iters / per_sm, cudaGetErrorString(e));
}

template <typename K>
void report(const char* name, K kern, long long* d, int iters, int grid, bool pairs) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  kern<<<grid, 128, 64 * 1024>>>(d, iters);
  const cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double m = 0;
  int n = 0, bad = 0;
  for (int i = 0; i < grid; ++i) {
    if (pairs && i % 2) continue;  // leaders carry the time
    if (h[i] < 0) ++bad;
    else m += h[i], ++n;
  }
  printf("%-34s %.1f cycles per MMA instruction (%d timed, %d timeouts, %s)\n", name,
         n ? m / n / iters : -1.0, n, bad, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 4 * 8);
  const int iters = 4096;
  report("cta_group::1 M=128 N=16", single_rate<16>, d, iters, 148, false);
  report("cta_group::1 M=128 N=32", single_rate<32>, d, iters, 148, false);
  report("cta_group::2 M=256 N=16 (pair)", pair_rate<16>, d, iters, 148, true);
  report("cta_group::2 M=256 N=32 (pair)", pair_rate<32>, d, iters, 148, true);
  report("cta_group::2 M=256 N=64 (pair)", pair_rate<64>, d, iters, 148, true);
  report("cta_group::2 M=256 N=256 (pair)", pair_rate<256>, d, iters, 148, true);
  for (int k : {1, 2, 4}) report_multi(k, d, iters);
  return 0;
}
