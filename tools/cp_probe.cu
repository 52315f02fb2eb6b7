// Probe: tcgen05.cp.128x256b (smem -> TMEM) of a K-major SW128 bf16 tile as
// the A operand of a TS MMA (A in TMEM), B = two 64x64 MN-major SW128 tiles
// side by side (N = 128, LBO = 8 KB). Checks the TMEM image of A against the
// source rows and D = A.B against a host product. Design check for the K7
// V-first kernel; not part of the library.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17
//   -I ../paper_2510_17505_b200/csrc cp_probe.cu -o cp_probe
#include <cuda_bf16.h>

#include <cmath>
#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace ixb::sm100;

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// A [128][64] bf16 row-major (global), W [64 u][128 w] bf16 row-major.
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* W, uint32_t* a_img,
                      float* D) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  uint8_t* As = sm;           // 16 KB: 128 rows x 128 B, SW128 K-major
  uint8_t* Ws = sm + 16384;   // 2 x 8 KB: [u][64 w] per tile, SW128 MN-major
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // A: row m, 16-B chunk c -> m*128 + ((c ^ (m & 7)) << 4)
  for (int i = tid; i < 128 * 8; i += blockDim.x) {
    const int m = i >> 3, c = i & 7;
    *reinterpret_cast<uint4*>(As + m * 128 + ((c ^ (m & 7)) << 4)) =
        *reinterpret_cast<const uint4*>(A + m * 64 + c * 8);
  }
  // W tile t (w in [64t, 64t+64)): row u, chunk c (8 w) -> t*8192 + u*128 + ((c ^ (u & 7)) << 4)
  for (int i = tid; i < 2 * 64 * 8; i += blockDim.x) {
    const int t = i >> 9, u = (i >> 3) & 63, c = i & 7;
    *reinterpret_cast<uint4*>(Ws + t * 8192 + u * 128 + ((c ^ (u & 7)) << 4)) =
        *reinterpret_cast<const uint4*>(W + u * 128 + t * 64 + c * 8);
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&slot, 256);
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;  // cols [0,32) A image, [128,256) D
  if (tid == 0) {
    for (int kk = 0; kk < 4; ++kk)
      tmem_cp_128x256b(tmem + 8 * kk, smem_desc(smem_u32(As) + kk * 32, 16, 1024, kLayoutSW128));
    const uint32_t idesc = idesc_bf16_f32(128, 128, false, true);
    for (int kk = 0; kk < 4; ++kk)
      umma_f16_ts(tmem + 128, tmem + 8 * kk,
                  smem_desc(smem_u32(Ws) + kk * 2048, 8192, 1024, kLayoutSW128), idesc,
                  kk > 0 ? 1u : 0u);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int lane_base = (warp & 3) * 32;
  uint32_t r[16];
  for (int c0 = 0; c0 < 32; c0 += 16) {
    tmem_ld_32x32b_x16(tmem + (lane_base << 16) + c0, r);
    tmem_ld_wait();
    for (int q = 0; q < 16; ++q) a_img[(lane_base + (tid & 31)) * 32 + c0 + q] = r[q];
  }
  for (int c0 = 0; c0 < 128; c0 += 16) {
    tmem_ld_32x32b_x16(tmem + (lane_base << 16) + 128 + c0, r);
    tmem_ld_wait();
    for (int q = 0; q < 16; ++q) D[(lane_base + (tid & 31)) * 128 + c0 + q] = __uint_as_float(r[q]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

int main() {
  std::vector<__nv_bfloat16> hA(128 * 64), hW(64 * 128);
  std::vector<float> fA(128 * 64), fW(64 * 128);
  for (int i = 0; i < 128 * 64; ++i) {
    fA[i] = static_cast<float>((i * 7) % 13 - 6);
    hA[i] = __float2bfloat16(fA[i]);
  }
  for (int i = 0; i < 64 * 128; ++i) {
    fW[i] = static_cast<float>((i * 5) % 11 - 5);
    hW[i] = __float2bfloat16(fW[i]);
  }
  __nv_bfloat16 *dA, *dW;
  uint32_t* dimg;
  float* dD;
  cudaMalloc(&dA, hA.size() * 2);
  cudaMalloc(&dW, hW.size() * 2);
  cudaMalloc(&dimg, 128 * 32 * 4);
  cudaMalloc(&dD, 128 * 128 * 4);
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, hW.data(), hW.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  probe<<<1, 128, 40 * 1024>>>(dA, dW, dimg, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));
    return 1;
  }
  std::vector<uint32_t> img(128 * 32);
  std::vector<float> D(128 * 128);
  cudaMemcpy(img.data(), dimg, img.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad_img = 0, bad_d = 0;
  const uint16_t* a16 = reinterpret_cast<const uint16_t*>(hA.data());
  for (int m = 0; m < 128; ++m)
    for (int c = 0; c < 32; ++c) {
      const uint32_t want = a16[m * 64 + 2 * c] | (static_cast<uint32_t>(a16[m * 64 + 2 * c + 1]) << 16);
      if (img[m * 32 + c] != want) {
        if (bad_img < 4) printf("img m=%d c=%d got %08x want %08x\n", m, c, img[m * 32 + c], want);
        ++bad_img;
      }
    }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 128; ++n) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += fA[m * 64 + k] * fW[k * 128 + n];
      if (std::fabs(D[m * 128 + n] - s) > 1e-3) {
        if (bad_d < 4) printf("D m=%d n=%d got %f want %f\n", m, n, D[m * 128 + n], s);
        ++bad_d;
      }
    }
  printf("{\"cp_image_mismatches\": %d, \"ts_mma_mismatches\": %d}\n", bad_img, bad_d);
  return bad_img || bad_d;
}
