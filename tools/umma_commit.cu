// Microbenchmark: tensor-pipe cost of K4-shaped MMA streams (M=128, N=16, K=16,
// bf16) when every batch of k MMAs is committed to an mbarrier and the issuer
// waits for the commit of batch b-D before issuing batch b (a D-deep smem
// ring). Variables: k, D, CTAs per SM, issuing warps per CTA (each warp owns its
// own TMEM columns). Perf experiment for DESIGN.md §K4; not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I ../paper_2510_17505_b200/csrc umma_commit.cu -o umma_commit
#include <cstdio>

#include "sm100.cuh"

using namespace ixb::sm100;

__device__ __forceinline__ void umma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc) : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__global__ void commit_rate(long long* out, int batches, int k, int depth, int iw, int ncols,
                            int nsz, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4][8];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < 4; ++w)
      for (int i = 0; i < 8; ++i) mbar_init(&bar[w][i], 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, ncols);
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp < iw && (lane == 0 || mode == 1)) {
    const uint32_t idesc = nsz == 16 ? idesc_bf16_f32(128, 16, true, false)
                                     : idesc_bf16_f32(128, 128, true, false);
    const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
    const uint32_t cols_per_warp = ncols / iw;
    const uint64_t ad0 = smem_desc(a0, 2048, 1024, kLayoutSW128);
    const uint64_t bd0 = smem_desc(b0, 16, 256, kLayoutSW32);
    long long t0 = clock64();
    for (int b = 0; b < batches; ++b) {
      if (b >= depth) mbar_wait(&bar[warp][(b - depth) & 7], ((b - depth) >> 3) & 1);
      for (int i = 0; i < k; ++i) {
        const int j = b * k + i;
        if (mode == 2) {
          umma_f16(tmem + warp * cols_per_warp, ad0, bd0, idesc, 1u);
        } else {
          // descriptor start addresses advance by (bytes >> 4) in the low bits
          const uint64_t ad = ad0 + static_cast<uint64_t>((j & 7) * (4096 >> 4));
          const uint64_t bd = bd0 + static_cast<uint64_t>((j & 15) * (512 >> 4));
          const uint32_t d = tmem + warp * cols_per_warp + ((j * 16) % cols_per_warp);
          if (mode == 1) umma_elect(d, ad, bd, idesc);
          else umma_f16(d, ad, bd, idesc, 1u);
        }
      }
      if (mode == 1) commit_elect(&bar[warp][b & 7]);
      else umma_commit(&bar[warp][b & 7]);
    }
    for (int b = batches - depth; b < batches; ++b)
      if (b >= 0) mbar_wait(&bar[warp][b & 7], (b >> 3) & 1);
    long long t1 = clock64();
    if (warp == 0 && lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, ncols);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8 * 8);
  cudaFuncSetAttribute(commit_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 41 * 1024);
  printf("[");
  bool first = true;
  for (int mode : {0, 1, 2}) {
    for (int cps : {1, 2}) {
      for (int iw : {1, 2}) {
        for (int k : {4, 8, 32}) {
          const int depth = 2, nsz = 16;
          const int ncols = cps == 1 ? 512 : 256;
          const int batches = 4096 / k;
          commit_rate<<<148 * cps, 64, 41 * 1024>>>(d, batches, k, depth, iw, ncols, nsz, mode);
          cudaError_t e = cudaDeviceSynchronize();
          long long h[148 * 4];
          cudaMemcpy(h, d, 148 * cps * 8, cudaMemcpyDeviceToHost);
          double m = 0;
          for (int i = 0; i < 148 * cps; ++i) m += h[i];
          m /= 148 * cps;
          const double per_sm = m / (double(batches) * k * iw * cps);
          printf("%s{\"mode\": %d, \"ctas_per_sm\": %d, \"issuers\": %d, \"k\": %d, "
                 "\"cycles_per_mma_per_sm\": %.1f, \"cycles_per_mma_per_stream\": %.1f, \"err\": %d}\n",
                 first ? "" : ",", mode, cps, iw, k, per_sm, m / (double(batches) * k), int(e));
          first = false;
        }
      }
    }
  }
  printf("]\n");
  return 0;
}
