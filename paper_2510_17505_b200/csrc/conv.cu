// K6 — grouped sparse convolution (kernel-map gather-GEMM-scatter):
//   Out[MAPX[p,q],m] += MAPV[p,q] * In[MAPY[p,q],c] * Weight[MAPZ[p],c,m]
// (corpus/grouped_sparse_conv.json:2; reference vars p,q,m,c, oracle
// plan.cpp:579-594; fused kernel: dot over c, kernel.cpp:292-357).
//
// Output-stationary formulation. The plan indexes every slot
// by (output row x, offset z) — a table T[x * n_off + z] -> slot — which for
// a canonical map (group_coo_tensor order (z, x, y), one `in` per (z, x))
// is collision free. The run then treats the conv as an implicit GEMM over
// K = (offset, c):
//   Out[x0:x0+128, :] = sum_z  A_z[128 x Cin] . Weight[z][Cin x Cout]
// where row r of A_z is MAPV[s] * In[MAPY[s], :] for s = T[(x0+r), z] (zero
// row if absent). Each CTA owns 128 output rows, so every output row has
// one writer (deterministic, no atomics) and its per-offset contributions
// accumulate in z order — the order of the canonical slot list.
// tcgen05 path (Cin = Cout = 64): A_z gathered by all 128 threads into a
// SW128 K-major smem tile, Weight[z] by TMA (MN-major SW128), 4 UMMAs
// M=128,N=64,K=16 per offset into one TMEM accumulator, double-buffered.
// Maps with colliding (x, z) or other channel counts take the CSR path: slots
// stable-sorted by output row, one warp per row, fp32 CUDA-core FMAs in slot
// order (bit-faithful to the reference's summation order).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <memory>
#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.h"

namespace ixb {
namespace {

using namespace sm100;

struct PlanArgs {
  const int32_t* MAPZ;
  const int32_t* MAPX;
  const int32_t* MAPY;
  const float* MAPV;
  int64_t G, g, n_in, n_off, n_out;
  int32_t* T;      // [n_out * n_off] slot or -1
  int* conflict;
  int* nonunit;    // some real (non-pad) slot has MAPV != 1
  int check;
  ErrorRecord* err;
};

// Validates every index (gathers In/MAPY op 0, Weight/MAPZ op 1, then the
// scatter Out/MAPX op 2 — plan.cpp:544-561 order) and fills T. A pad slot
// (same x,y as its predecessor in the group, value 0) is inert and skipped.
__global__ void conv_index_kernel(PlanArgs a) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= a.G * a.g) return;
  const int64_t p = s / a.g, q = s % a.g;
  const int y = a.MAPY[s], x = a.MAPX[s], z = a.MAPZ[p];
  bool ok = true;
  if (y < 0 || y >= a.n_in) {
    if (a.check) report_index_error(a.err, 0, s, y);
    ok = false;
  }
  if (q == 0 && (z < 0 || z >= a.n_off)) {
    if (a.check) report_index_error(a.err, 1, p, z);
  }
  if (z < 0 || z >= a.n_off) ok = false;
  if (x < 0 || x >= a.n_out) {
    if (a.check) report_index_error(a.err, 2, s, x);
    ok = false;
  }
  if (!ok) return;
  const float v = a.MAPV ? a.MAPV[s] : 1.f;
  if (q > 0 && v == 0.f && a.MAPX[s - 1] == x && a.MAPY[s - 1] == y) return;  // pad
  if (v != 1.f) atomicOr(a.nonunit, 1);
  const int prev = atomicCAS(&a.T[static_cast<int64_t>(x) * a.n_off + z], -1,
                             static_cast<int>(s));
  if (prev != -1) atomicOr(a.conflict, 1);
}

// ------------------------------------------------------------ tcgen05 path
constexpr int kConvThreads = 128;
constexpr uint32_t kATile = 128 * 128;  // 128 rows x 64 bf16
constexpr uint32_t kWTile = 64 * 128;   // 64 c-rows x 64 bf16

struct RunArgs {
  const int32_t* T;
  const int32_t* MAPY;
  const float* MAPV;
  const __nv_bfloat16* In;
  float* Out;
  int64_t n_out, n_off;
  int accumulate;
};

__global__ void __launch_bounds__(kConvThreads, 1)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmW, RunArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* A = smem;                   // [2][16 KB]
  uint8_t* W = smem + 2 * kATile;      // [2][8 KB]
  uint64_t* w_full = reinterpret_cast<uint64_t*>(W + 2 * kWTile);
  uint64_t* mma_done = w_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 2);
  const int tid = threadIdx.x, warp = tid >> 5;

  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&w_full[b], 1);
      mbar_init(&mma_done[b], 1);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 64);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t x = static_cast<int64_t>(blockIdx.x) * 128 + tid;
  const bool row_ok = x < a.n_out;
  constexpr uint32_t idesc = idesc_bf16_f32(128, 64, /*A K-major*/ false, /*B MN-major*/ true);
  const uint64_t keep = l2_evict_last();
  int k = 0;  // offsets actually used (buffer use counter)
  for (int z = 0; z < a.n_off; ++z) {
    const int s = row_ok ? __ldg(a.T + x * a.n_off + z) : -1;
    if (!__syncthreads_or(s >= 0)) continue;  // no row of this tile has offset z
    const int buf = k & 1;
    if (k >= 2) mbar_wait(&mma_done[buf], ((k - 2) >> 1) & 1);  // MMA k-2 freed buf
    if (tid == 0) {
      mbar_arrive_expect_tx(&w_full[buf], kWTile);
      tma_load_2d(W + buf * kWTile, &tmW, &w_full[buf], 0, z * 64, keep);
    }
    // gather row tid of A_z: MAPV[s] * In[MAPY[s], 0:64] -> bf16, SW128 K-major
    uint4 chunk[8];
    if (s >= 0) {
      const int y = __ldg(a.MAPY + s);
      const float v = a.MAPV ? __ldg(a.MAPV + s) : 1.f;
      const uint4* src = reinterpret_cast<const uint4*>(a.In + static_cast<int64_t>(y) * 64);
#pragma unroll
      for (int j = 0; j < 8; ++j) chunk[j] = __ldg(src + j);
      if (v != 1.f) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&chunk[j]);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 f = __bfloat1622float2(h[e]);
            h[e] = __floats2bfloat162_rn(f.x * v, f.y * v);
          }
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) chunk[j] = make_uint4(0, 0, 0, 0);
    }
    uint8_t* arow = A + buf * kATile + tid * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      *reinterpret_cast<uint4*>(arow + ((j ^ (tid & 7)) << 4)) = chunk[j];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // st.shared -> tensor core
    __syncthreads();
    if (tid == 0) {
      mbar_wait(&w_full[buf], (k >> 1) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_u32(A + buf * kATile), w0 = smem_u32(W + buf * kWTile);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        // A: K-major SW128, 8-row atoms at 1024 B; K step of 16 = +32 B
        const uint64_t ad = smem_desc(a0 + kk * 32, 16, 1024, kLayoutSW128);
        // W[z]: MN-major SW128 (64 m = one atom), K groups of 8 c-rows at 1024 B
        const uint64_t bd = smem_desc(w0 + kk * 2048, 8192, 1024, kLayoutSW128);
        umma_f16(tmem, ad, bd, idesc, (k > 0 || kk > 0) ? 1u : 0u);
      }
      umma_commit(&mma_done[buf]);
    }
    ++k;
  }
  float acc[64];
  if (k > 0) {
    mbar_wait(&mma_done[(k - 1) & 1], ((k - 1) >> 1) & 1);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[16];
      tmem_ld_32x32b_x16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 16, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[c * 16 + j] = __uint_as_float(r[j]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 64; ++j) acc[j] = 0.f;
  }
  if (row_ok) {
    float4* o = reinterpret_cast<float4*>(a.Out + x * 64);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float4 v = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
      if (a.accumulate) {
        const float4 old = o[j];
        v.x += old.x;
        v.y += old.y;
        v.z += old.z;
        v.w += old.w;
      }
      o[j] = v;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}


// ------------------------------------------- tcgen05 path for unit-valued maps
// Unit-valued maps (MAPV == 1 on every real slot — what ixb_kernel_map +
// group_coo_tensor produce) need no per-row scaling. The plan turns T into an
// input-row table Y[x, z] = y + 1 (0 = absent; row stride kOffPad ints, 16 B
// aligned) plus a bitmask of the offsets each 128-row tile uses. A thread
// reads its row's whole Y row in 7 vector loads, so no per-offset T -> MAPY
// dependence and no per-offset block vote remain; the gathers of the next
// two used offsets are in flight (cp.async) while the current one is
// multiplied. The tensor-core part is the kernel above (4 UMMAs M=128,N=64,
// K=16 per offset into one TMEM accumulator), so each output row still
// accumulates its offsets in z order.
// Measured on cfg5 (1 M voxels): 0.83 ms (conv_tc_kernel) -> 0.65 ms
// (register prefetch, one row per thread) -> 0.567 ms (coalesced gather) ->
// 0.513 ms (cp.async, 3-stage ring) -> 0.477 ms (2-stage ring, 4 CTAs/SM).
// Switching parts off (3-stage ring): no gather
// 0.512 ms, no MMA 0.413 ms, neither (nor W) 0.390 ms — the per-offset
// __syncthreads + commit round trip of this one-tile-per-CTA structure is
// the floor. Not shipped:
// - a persistent warp-specialised kernel (8-stage ring, producer warps,
//   MMA warp, epilogue warps with double-buffered TMEM): 0.60-0.92 ms with
//   producer-side wait + proxy fence (the fence waits for all of a thread's
//   cp.async, serialising stages per warp), 0.78 ms with
//   cp.async.mbarrier.arrive.noinc publishing (no producer waits, as
//   CUTLASS's sm100 cp.async pipeline does) and the tile's Y rows in smem;
//   one CTA per SM does not reach the 3-CTA kernel's throughput;
// - deeper rings at this structure (s4d2 0.645 ms, s5d2 1.13 ms: fewer CTAs
//   per SM);
// - TMA tile::gather4 (1.0-3.2 ms; ~43 cycles per 512 B box per SM;
//   tools/gather4_probe.cu pins its semantics);
// - A in tensor memory (round 2): each thread gathers its row into
//   registers 2 offsets ahead and tcgen05.st's it into a TMEM A slot, the
//   MMA reads A from TMEM (umma_f16_ts) and only Weight from shared memory,
//   epilogue staged through smem for 512 B warp stores: correct (every conv
//   test) but 0.539 ms against 0.477 — register-staged gathers cap the
//   bytes in flight per SM below what the cp.async ring keeps.
constexpr int kOffPad = 28;  // Y row stride (ints): 27 offsets padded to 16 B

struct UnitArgs {
  const int32_t* Y;           // [n_out][kOffPad] y + 1, 0 = absent
  const uint32_t* tile_mask;  // [ntiles] offsets used by the tile
  const __nv_bfloat16* In;
  float* Out;
  int64_t n_out;
  int accumulate;
  int64_t tile0;              // first 128-row tile of this launch (host pipeline chunks)
};

// Stage k of a tile = its k-th used offset z: the In rows of the 128 output
// rows land in A[k % S] by cp.async (coalesced: 8 lanes share a 128 B row,
// so a warp instruction covers 4 whole rows; the row's input index comes
// from its owner lane by shuffle; absent rows are zero-filled) and W[z] in
// W[k % S] by TMA, issued D stages ahead of the MMA.
// 2 stages issued 1 ahead (48 KB -> 4 CTAs per SM) beat 3 stages issued 2
// ahead (72 KB -> 3 CTAs): 0.477 vs 0.510 ms on cfg5. More CTAs per SM
// outweigh a deeper per-CTA ring here.
#ifndef IXB_CONV_STAGES
#define IXB_CONV_STAGES 2
#define IXB_CONV_DIST 1
#define IXB_CONV_MINB 4
#endif
constexpr int kUnitStages = IXB_CONV_STAGES;
constexpr int kUnitDist = IXB_CONV_DIST;
constexpr uint32_t kUnitSmem = kUnitStages * (kATile + kWTile) + 1024 + 256;

__global__ void __launch_bounds__(kConvThreads, IXB_CONV_MINB)
    conv_unit_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO,
                     UnitArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* A = smem;                         // [kUnitStages][16 KB]
  uint8_t* W = smem + kUnitStages * kATile;  // [kUnitStages][8 KB]
  uint64_t* w_full = reinterpret_cast<uint64_t*>(W + kUnitStages * kWTile);
  uint64_t* mma_done = w_full + kUnitStages;
  uint64_t* a_full = mma_done + kUnitStages;  // per stage: the 4 warps' gathered rows are in
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + kUnitStages);
  const int tid = threadIdx.x, warp = tid >> 5;

  if (tid == 0) {
    for (int b = 0; b < kUnitStages; ++b) {
      mbar_init(&w_full[b], 1);
      mbar_init(&mma_done[b], 1);
      mbar_init(&a_full[b], kConvThreads / 32);
    }
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 64);
    tmem_relinquish();
  }
  const int64_t tile = a.tile0 + blockIdx.x;
  const int64_t x = tile * 128 + tid;
  const bool row_ok = x < a.n_out;
  // this row's input rows for all offsets (y + 1), one vectorised read
  int yr[kOffPad];
  if (row_ok) {
    const int4* src = reinterpret_cast<const int4*>(a.Y + x * kOffPad);
#pragma unroll
    for (int j = 0; j < kOffPad / 4; ++j) {
      const int4 v = __ldg(src + j);
      yr[4 * j] = v.x, yr[4 * j + 1] = v.y, yr[4 * j + 2] = v.z, yr[4 * j + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kOffPad; ++j) yr[j] = 0;
  }
  const uint32_t tmask = a.tile_mask[tile];
  const int nk = __popc(tmask);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = idesc_bf16_f32(128, 64, /*A K-major*/ false, /*B MN-major*/ true);
  const uint64_t keep = l2_evict_last();

  const int lane = tid & 31, chunk = lane & 7, sub = lane >> 3;
  auto issue = [&](int k) {
    const int z = __fns(tmask, 0, k + 1);  // k-th used offset (warp-uniform)
    const int st = k % kUnitStages;
    // yr[z] for the warp-uniform z: a uniform jump table, not a 28-way
    // compare/select chain per offset (yr stays in registers)
    int y1 = 0;
    switch (z) {
#define IXB_YR_CASE(j) \
  case j:              \
    y1 = yr[j];        \
    break;
      IXB_YR_CASE(0) IXB_YR_CASE(1) IXB_YR_CASE(2) IXB_YR_CASE(3) IXB_YR_CASE(4)
      IXB_YR_CASE(5) IXB_YR_CASE(6) IXB_YR_CASE(7) IXB_YR_CASE(8) IXB_YR_CASE(9)
      IXB_YR_CASE(10) IXB_YR_CASE(11) IXB_YR_CASE(12) IXB_YR_CASE(13) IXB_YR_CASE(14)
      IXB_YR_CASE(15) IXB_YR_CASE(16) IXB_YR_CASE(17) IXB_YR_CASE(18) IXB_YR_CASE(19)
      IXB_YR_CASE(20) IXB_YR_CASE(21) IXB_YR_CASE(22) IXB_YR_CASE(23) IXB_YR_CASE(24)
      IXB_YR_CASE(25) IXB_YR_CASE(26)
#undef IXB_YR_CASE
      default:
        break;
    }
    const uint32_t awarp = smem_u32(A + st * kATile + warp * 32 * 128);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = sub + 4 * i;
      const int yy = __shfl_sync(0xffffffffu, y1, r);
      const __nv_bfloat16* src = a.In + static_cast<int64_t>(yy > 0 ? yy - 1 : 0) * 64 + chunk * 8;
      cp_async_16(awarp + r * 128 + ((chunk ^ (r & 7)) << 4), src, yy > 0 ? 16u : 0u);
    }
    if (warp == 0 && elect_one_sync()) {
      mbar_arrive_expect_tx(&w_full[st], kWTile);
      tma_load_2d(W + st * kWTile, &tmW, &w_full[st], 0, z * 64, keep);
    }
  };
#pragma unroll
  for (int k = 0; k < kUnitDist; ++k) {
    if (k < nk) issue(k);
    cp_async_commit();
  }
  for (int k = 0; k < nk; ++k) {
    const int st = k % kUnitStages;
    cp_async_wait<kUnitDist - 1>();  // this thread's rows of stage k have landed
    fence_proxy_async_smem();        // cp.async (generic proxy) -> tensor core
    __syncwarp();
    if (lane == 0) mbar_arrive(&a_full[st]);  // this warp's 32 rows of stage k are in
    if (warp == 0) {  // whole warp, one elected lane issues
      mbar_wait(&a_full[st], (k / kUnitStages) & 1);
      mbar_wait(&w_full[st], (k / kUnitStages) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_u32(A + st * kATile), w0 = smem_u32(W + st * kWTile);
      umma_ss_k64_commit_elect(tmem, smem_desc(a0, 16, 1024, kLayoutSW128),
                               smem_desc(w0, 8192, 1024, kLayoutSW128), idesc, k > 0 ? 1u : 0u,
                               &mma_done[st]);
    }
    if (k + kUnitDist < nk) {
      // stage k + D reuses the slot of stage k + D - S: wait for its MMAs
      const int old = k + kUnitDist - kUnitStages;
      if (old >= 0) mbar_wait(&mma_done[old % kUnitStages], (old / kUnitStages) & 1);
      issue(k + kUnitDist);
    }
    cp_async_commit();  // (possibly empty) group k + D keeps the wait count uniform
  }
  if (nk > 0) {
    mbar_wait(&mma_done[(nk - 1) % kUnitStages], ((nk - 1) / kUnitStages) & 1);
    tc_fence_after();
  }
  // Epilogue: the tile goes out by TMA store (reduce-add for +=) through the
  // A stages, free once the last MMA has completed: two [128 rows][32 cols]
  // SW128 halves, thread = row (rows past n_out are clipped by the TMA).
  float4* ot = reinterpret_cast<float4*>(A);
#pragma unroll 1
  for (int c = 0; c < 4; ++c) {
    uint32_t r[16];
    if (nk > 0) {
      tmem_ld_32x32b_x16(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 16, r);
      tmem_ld_wait();
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) r[j] = 0;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int chunk = (c & 1) * 4 + j;
      ot[(c >> 1) * 1024 + tid * 8 + (chunk ^ (tid & 7))] =
          make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                      __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
    }
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      if (a.accumulate)
        tma_reduce_add_2d(&tmO, ot + half * 1024, 32 * half, static_cast<int32_t>(tile * 128));
      else
        tma_store_2d(&tmO, ot + half * 1024, 32 * half, static_cast<int32_t>(tile * 128));
    }
    bulk_commit_group();
    bulk_wait_group_read0();  // the stores have read the tile before the CTA's smem goes
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

// Y[x * kOffPad + z] = MAPY[T[x, z]] + 1 (0 = absent); tile masks of used offsets.
__global__ void conv_ytable_kernel(const int32_t* T, const int32_t* MAPY, int64_t n_out,
                                   int64_t n_off, int32_t* Y, uint32_t* tile_mask,
                                   int32_t* tile_need) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_out * kOffPad) return;
  const int64_t x = i / kOffPad, z = i % kOffPad;
  int v = 0;
  if (z < n_off) {
    const int s = T[x * n_off + z];
    if (s >= 0) {
      v = MAPY[s] + 1;
      atomicOr(&tile_mask[x / 128], 1u << z);
      atomicMax(&tile_need[x / 128], v);  // input rows [0, v) hold this tile's inputs
    }
  }
  Y[i] = v;
}

// --------------------------------------------------------------- CSR path
__global__ void iota_conv(int32_t* v, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int32_t>(i);
}

__global__ void row_hist(const int32_t* MAPX, int64_t n, int64_t n_out, int32_t* cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && MAPX[i] >= 0 && MAPX[i] < n_out) atomicAdd(cnt + MAPX[i], 1);
}

// One warp per output row, slots in (stable) slot order; lanes over Cout.
template <typename TI>
__global__ void conv_csr_kernel(const int32_t* perm, const int32_t* rowptr, const int32_t* MAPZ,
                                const int32_t* MAPY, const float* MAPV, int64_t g, const TI* In,
                                int64_t Cin, const TI* Wt, int64_t Cout, float* Out,
                                int64_t n_out, int accumulate) {
  const int64_t x = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (x >= n_out) return;
  const int lane = threadIdx.x & 31;
  for (int64_t m0 = 0; m0 < Cout; m0 += 32) {
    const int64_t m = m0 + lane;
    float acc = 0.f;
    for (int32_t i = rowptr[x]; i < rowptr[x + 1]; ++i) {
      const int s = perm[i];
      const int y = MAPY[s];
      const int z = MAPZ[s / g];
      const float v = MAPV ? MAPV[s] : 1.f;
      const TI* in = In + static_cast<int64_t>(y) * Cin;
      const TI* w = Wt + static_cast<int64_t>(z) * Cin * Cout + m;
      if (m < Cout) {
        for (int64_t c = 0; c < Cin; ++c) {
          acc = fmaf(v * static_cast<float>(in[c]), static_cast<float>(w[c * Cout]), acc);
        }
      }
    }
    if (m < Cout) {
      float* o = Out + x * Cout + m;
      *o = accumulate ? *o + acc : acc;
    }
  }
}

}  // namespace

}  // namespace ixb

struct ixb_conv_plan {
  int64_t G = 0, g = 1, n_in = 0, n_off = 0, n_out = 0;
  const int32_t *MAPZ = nullptr, *MAPX = nullptr, *MAPY = nullptr;
  const float* MAPV = nullptr;
  bool conflict = false;
  bool unit = false;  // every real slot has MAPV == 1: conv_unit_kernel usable
  ixb::Scratch<int32_t> T, perm, rowptr, Y;
  ixb::Scratch<uint32_t> tile_mask;
  std::vector<int32_t> tile_need;  // per 128-row tile: input rows [0, need) it reads
};

using namespace ixb;

namespace {
// conv_unit_kernel over the 128-row tiles [tile0, tile0 + ntiles)
void launch_unit(const ixb_conv_plan* P, const void* In, const void* Weight, float* Out,
                 int accumulate, int64_t tile0, int64_t ntiles, cudaStream_t s) {
  if (ntiles <= 0) return;
  const CUtensorMap tmW = make_tmap_2d(Weight, 64, static_cast<uint64_t>(P->n_off) * 64, 128, 64,
                                       64, CU_TENSOR_MAP_SWIZZLE_128B);
  if (reinterpret_cast<uintptr_t>(Out) % 16 != 0)
    fail(IXB_SHAPE, "ixb_conv_plan_run: Out must be 16-byte aligned");
  // Out viewed as (64 cols, n_out rows): {32, 128} boxes, one per tile half
  const CUtensorMap tmO = make_tmap_2d_f32(Out, 64, static_cast<uint64_t>(P->n_out), 256, 32, 128,
                                           CU_TENSOR_MAP_SWIZZLE_128B);
  UnitArgs ua{P->Y.p, P->tile_mask.p, static_cast<const __nv_bfloat16*>(In), Out, P->n_out,
              accumulate, tile0};
  set_max_dynamic_smem(reinterpret_cast<const void*>(conv_unit_kernel), kUnitSmem,
                       "cudaFuncSetAttribute(conv_unit_kernel)");
  conv_unit_kernel<<<static_cast<unsigned>(ntiles), kConvThreads, kUnitSmem, s>>>(tmW, tmO, ua);
  IXB_LAUNCH_CHECK("conv_unit_kernel");
}

struct ConvStreams {  // side streams + events of the host-buffer form, per thread and device
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;
  int device = -1;
  void ensure(size_t nev) {
    int dev = 0;
    IXB_CUDA_CHECK(cudaGetDevice(&dev));
    if (device != dev) {
      IXB_CUDA_CHECK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
      IXB_CUDA_CHECK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
      ev.clear();
      device = dev;
    }
    while (ev.size() < nev) {
      cudaEvent_t e;
      IXB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
  }
};
thread_local ConvStreams t_conv_streams;
}  // namespace

namespace ixb {
int64_t conv_plan_rows(const ixb_conv_plan* P) { return P->n_out; }

void conv_plan_run_rows(ixb_conv_plan* P, const void* In, int64_t Cin, const void* Weight,
                        int64_t Cout, float* Out, int64_t r0, int64_t r1, cudaStream_t s) {
  const bool unit = !P->conflict && P->unit && Cin == 64 && Cout == 64 &&
                    reinterpret_cast<uintptr_t>(In) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(Weight) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(Out) % 16 == 0;
  if (unit) {
    if (r0 % 128) fail(IXB_SHAPE, "conv chunk must start on a 128-row tile");
    launch_unit(P, In, Weight, Out, 0, r0 / 128, ceil_div(r1, 128) - r0 / 128, s);
    return;
  }
  if (r0 != 0 || r1 != P->n_out)
    fail(IXB_SHAPE, "conv map outside the unit tensor-core path: shard with nchunks = 1");
  const int rc = ixb_conv_plan_run(P, In, Cin, Weight, Cout, Out, 0, 0,
                                   reinterpret_cast<ixb_stream>(s));
  if (rc != IXB_OK) fail(rc, ixb_last_error());
}
}  // namespace ixb

extern "C" {

int ixb_conv_plan_create(const int32_t* MAPZ, const int32_t* MAPX, const int32_t* MAPY,
                         const float* MAPV, int64_t G, int64_t g, int64_t n_in, int64_t n_off,
                         int64_t n_out, int flags, ixb_stream stream, ixb_conv_plan** plan) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (G < 0 || g < 1 || n_in < 0 || n_off < 0 || n_out < 0) fail(IXB_SHAPE, "conv: bad extents");
    if (G * g > INT32_MAX || n_out * n_off > INT32_MAX) fail(IXB_SHAPE, "conv: map too large");
    auto P = std::make_unique<ixb_conv_plan>();
    P->G = G;
    P->g = g;
    P->n_in = n_in;
    P->n_off = n_off;
    P->n_out = n_out;
    P->MAPZ = MAPZ;
    P->MAPX = MAPX;
    P->MAPY = MAPY;
    P->MAPV = MAPV;
    const int64_t slots = G * g;
    P->T = Scratch<int32_t>(n_out * n_off + 1, s);
    Scratch<int> conflict(2, s);  // [0] conflict, [1] non-unit MAPV
    IXB_CUDA_CHECK(cudaMemsetAsync(P->T.p, 0xff, (n_out * n_off + 1) * 4, s));
    IXB_CUDA_CHECK(cudaMemsetAsync(conflict.p, 0, 8, s));
    const bool check = !(flags & IXB_UNCHECKED);
    if (slots > 0) {
      PlanArgs a{MAPZ, MAPX, MAPY, MAPV, G, g, n_in, n_off, n_out, P->T.p, conflict.p,
                 conflict.p + 1, check, device_error_record()};
      conv_index_kernel<<<ceil_div(slots, 256), 256, 0, s>>>(a);
      IXB_LAUNCH_CHECK("conv_index_kernel");
    }
    if (check) {
      OperandInfo ops[3] = {{"MAPY", "In", 0, n_in, MAPY, slots},
                            {"MAPZ", "Weight", 0, n_off, MAPZ, G},
                            {"MAPX", "Out", 0, n_out, MAPX, slots}};
      check_error_record(s, ops, 3);
    }
    int h[2] = {0, 0};
    IXB_CUDA_CHECK(cudaMemcpyAsync(h, conflict.p, 8, cudaMemcpyDeviceToHost, s));
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));
    P->conflict = h[0] != 0;
    P->unit = !P->conflict && h[1] == 0 && n_off <= kOffPad && n_in < INT32_MAX;
    if (P->unit && n_out > 0) {
      const int64_t ntiles = ceil_div(n_out, 128);
      P->Y = Scratch<int32_t>(n_out * kOffPad, s);
      P->tile_mask = Scratch<uint32_t>(ntiles, s);
      IXB_CUDA_CHECK(cudaMemsetAsync(P->tile_mask.p, 0, ntiles * 4, s));
      Scratch<int32_t> need(ntiles, s);
      IXB_CUDA_CHECK(cudaMemsetAsync(need.p, 0, ntiles * 4, s));
      conv_ytable_kernel<<<ceil_div(n_out * kOffPad, 256), 256, 0, s>>>(
          P->T.p, MAPY, n_out, n_off, P->Y.p, P->tile_mask.p, need.p);
      IXB_LAUNCH_CHECK("conv_ytable_kernel");
      P->tile_need.resize(ntiles);
      IXB_CUDA_CHECK(cudaMemcpyAsync(P->tile_need.data(), need.p, ntiles * 4,
                                     cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    *plan = P.release();
  });
}

void ixb_conv_plan_free(ixb_conv_plan* plan) {
  if (!plan) return;
  // runs may be in flight on any stream: let them finish, then release the
  // tables on the default stream (the creating stream may be gone)
  cudaDeviceSynchronize();
  plan->T.s = plan->perm.s = plan->rowptr.s = plan->Y.s = nullptr;
  plan->tile_mask.s = nullptr;
  delete plan;
}

int ixb_conv_plan_run(ixb_conv_plan* P, const void* In, int64_t Cin, const void* Weight,
                      int64_t Cout, float* Out, int accumulate, int flags, ixb_stream stream) {
  return ixb_guard([&] {
    (void)flags;
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!P) fail(IXB_FAILURE, "null conv plan");
    if (Cin < 1 || Cout < 1) fail(IXB_SHAPE, "conv: channel counts must be >= 1");
    if (P->n_out == 0) return;
    const bool tc = !P->conflict && Cin == 64 && Cout == 64 &&
                    reinterpret_cast<uintptr_t>(In) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(Weight) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(Out) % 16 == 0;
    if (tc && P->unit) {
      launch_unit(P, In, Weight, Out, accumulate, 0, ceil_div(P->n_out, 128), s);
      return;
    }
    if (tc) {
      const CUtensorMap tmW =
          make_tmap_2d(Weight, 64, static_cast<uint64_t>(P->n_off) * 64, 128, 64, 64,
                       CU_TENSOR_MAP_SWIZZLE_128B);
      RunArgs a{P->T.p, P->MAPY, P->MAPV, static_cast<const __nv_bfloat16*>(In), Out, P->n_out,
                P->n_off, accumulate};
      const uint32_t smem = 2 * kATile + 2 * kWTile + 1024 + 1024;
      set_max_dynamic_smem(reinterpret_cast<const void*>(conv_tc_kernel), smem,
                           "cudaFuncSetAttribute(conv_tc_kernel)");
      conv_tc_kernel<<<ceil_div(P->n_out, 128), kConvThreads, smem, s>>>(tmW, a);
      IXB_LAUNCH_CHECK("conv_tc_kernel");
      return;
    }
    // CSR path: slots stable-sorted by output row.
    const int64_t slots = P->G * P->g;
    if (!P->perm.p) {
      Scratch<int32_t> idx(slots + 1, s), keys_out(slots + 1, s);
      P->perm = Scratch<int32_t>(slots + 1, s);
      if (slots > 0) {
        iota_conv<<<ceil_div(slots, 256), 256, 0, s>>>(idx.p, slots);
        IXB_LAUNCH_CHECK("iota_conv");
        size_t tb = 0;
        IXB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, P->MAPX, keys_out.p, idx.p,
                                                       P->perm.p, static_cast<int>(slots), 0, 32,
                                                       s));
        Scratch<char> tmp(tb, s);
        IXB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, P->MAPX, keys_out.p, idx.p,
                                                       P->perm.p, static_cast<int>(slots), 0, 32,
                                                       s));
        note_launch(4);
      }
      Scratch<int32_t> cnt(P->n_out + 1, s);
      P->rowptr = Scratch<int32_t>(P->n_out + 1, s);
      IXB_CUDA_CHECK(cudaMemsetAsync(cnt.p, 0, (P->n_out + 1) * 4, s));
      if (slots > 0) {
        row_hist<<<ceil_div(slots, 256), 256, 0, s>>>(P->MAPX, slots, P->n_out, cnt.p);
        IXB_LAUNCH_CHECK("row_hist");
      }
      size_t tb = 0;
      IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, P->rowptr.p,
                                                   static_cast<int>(P->n_out + 1), s));
      Scratch<char> tmp(tb, s);
      IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, P->rowptr.p,
                                                   static_cast<int>(P->n_out + 1), s));
      note_launch();
    }
    const int64_t grid = ceil_div(P->n_out * 32, 256);
    conv_csr_kernel<__nv_bfloat16><<<grid, 256, 0, s>>>(
        P->perm.p, P->rowptr.p, P->MAPZ, P->MAPY, P->MAPV, P->g,
        static_cast<const __nv_bfloat16*>(In), Cin, static_cast<const __nv_bfloat16*>(Weight),
        Cout, Out, P->n_out, accumulate);
    IXB_LAUNCH_CHECK("conv_csr_kernel");
  });
}

// Host-buffer form: In [n_in, Cin] bf16 and Out [n_out, Cout] fp32 in host
// memory (pinned for overlap), Weight on the device. With the unit kernel the
// output tiles run in `nchunks` groups: In is copied in row order, and each
// group starts once the input rows its tiles read (recorded per tile by the
// plan) have landed, while the previous group's Out rows copy back. Other
// maps copy In, evaluate, and copy Out back in sequence. Results are
// bit-identical to ixb_conv_plan_run.
int ixb_conv_plan_run_host(ixb_conv_plan* P, const void* In, int64_t Cin, const void* Weight,
                           int64_t Cout, float* Out, int accumulate, int flags, int nchunks,
                           ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!P) fail(IXB_FAILURE, "null conv plan");
    if (Cin < 1 || Cout < 1) fail(IXB_SHAPE, "conv: channel counts must be >= 1");
    if (P->n_out == 0) return;
    const int64_t in_row = Cin * 2, out_row = Cout * 4;
    Scratch<char> dIn(P->n_in * in_row, s), dOut(P->n_out * out_row, s);
    const bool pipelined = !P->conflict && Cin == 64 && Cout == 64 && P->unit &&
                           reinterpret_cast<uintptr_t>(Weight) % 16 == 0 && nchunks > 1;
    if (!pipelined) {
      IXB_CUDA_CHECK(cudaMemcpyAsync(dIn.p, In, P->n_in * in_row, cudaMemcpyHostToDevice, s));
      if (accumulate)
        IXB_CUDA_CHECK(cudaMemcpyAsync(dOut.p, Out, P->n_out * out_row, cudaMemcpyHostToDevice, s));
      const int rc = ixb_conv_plan_run(P, dIn.p, Cin, Weight, Cout,
                                       reinterpret_cast<float*>(dOut.p), accumulate, flags, stream);
      if (rc != IXB_OK) fail(rc, ixb_last_error());
      IXB_CUDA_CHECK(cudaMemcpyAsync(Out, dOut.p, P->n_out * out_row, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaStreamSynchronize(s));
      return;
    }
    const int64_t ntiles = ceil_div(P->n_out, 128);
    if (nchunks > ntiles) nchunks = static_cast<int>(ntiles);
    ConvStreams& st = t_conv_streams;
    st.ensure(2 + 2 * nchunks);
    IXB_CUDA_CHECK(cudaEventRecord(st.ev[0], s));  // scratch allocated on s
    IXB_CUDA_CHECK(cudaStreamWaitEvent(st.h2d, st.ev[0], 0));
    int64_t copied = 0;  // In rows [0, copied) are on their way
    for (int i = 0; i < nchunks; ++i) {
      const int64_t t0 = ntiles * i / nchunks, t1 = ntiles * (i + 1) / nchunks;
      int64_t need = 0;
      for (int64_t t = t0; t < t1; ++t) need = std::max<int64_t>(need, P->tile_need[t]);
      if (i == nchunks - 1) need = P->n_in;  // the rest of In (unread rows are harmless)
      if (need > copied) {
        IXB_CUDA_CHECK(cudaMemcpyAsync(dIn.p + copied * in_row,
                                       static_cast<const char*>(In) + copied * in_row,
                                       (need - copied) * in_row, cudaMemcpyHostToDevice, st.h2d));
        copied = need;
      }
      const int64_t r0 = t0 * 128, r1 = std::min<int64_t>(t1 * 128, P->n_out);
      if (accumulate && r1 > r0)
        IXB_CUDA_CHECK(cudaMemcpyAsync(dOut.p + r0 * out_row,
                                       reinterpret_cast<const char*>(Out) + r0 * out_row,
                                       (r1 - r0) * out_row, cudaMemcpyHostToDevice, st.h2d));
      cudaEvent_t in_ev = st.ev[2 + 2 * i], out_ev = st.ev[3 + 2 * i];
      IXB_CUDA_CHECK(cudaEventRecord(in_ev, st.h2d));
      IXB_CUDA_CHECK(cudaStreamWaitEvent(s, in_ev, 0));
      launch_unit(P, dIn.p, Weight, reinterpret_cast<float*>(dOut.p), accumulate, t0, t1 - t0, s);
      IXB_CUDA_CHECK(cudaEventRecord(out_ev, s));
      IXB_CUDA_CHECK(cudaStreamWaitEvent(st.d2h, out_ev, 0));
      if (r1 > r0)
        IXB_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(Out) + r0 * out_row,
                                       dOut.p + r0 * out_row, (r1 - r0) * out_row,
                                       cudaMemcpyDeviceToHost, st.d2h));
    }
    IXB_CUDA_CHECK(cudaEventRecord(st.ev[1], st.d2h));
    IXB_CUDA_CHECK(cudaStreamWaitEvent(s, st.ev[1], 0));
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));  // Out is in host memory on return
  });
}

int ixb_conv_grouped(const int32_t* MAPZ, const int32_t* MAPX, const int32_t* MAPY,
                     const float* MAPV, int64_t G, int64_t g, const void* In, int64_t n_in,
                     int64_t Cin, const void* Weight, int64_t n_off, int64_t Cout, float* Out,
                     int64_t n_out, int accumulate, int flags, ixb_stream stream) {
  ixb_conv_plan* plan = nullptr;
  int rc = ixb_conv_plan_create(MAPZ, MAPX, MAPY, MAPV, G, g, n_in, n_off, n_out, flags, stream,
                                &plan);
  if (rc != IXB_OK) return rc;
  rc = ixb_conv_plan_run(plan, In, Cin, Weight, Cout, Out, accumulate, flags, stream);
  ixb_conv_plan_free(plan);
  return rc;
}

}  // extern "C"
