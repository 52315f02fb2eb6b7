// K7 — grouped Clebsch–Gordan tensor product:
//   Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[(b,)CGL[p],u,w]
// (corpus/grouped_tensor_product.json:2; reference vars b,p,q,w,u; oracle
// plan.cpp:579-594; fused: dot over u, batch [b,p], kernel.cpp:292-357).
//
// tcgen05 path (shared W[l,u,w], U = W = 64, <= 16 irrep components;
// BASELINE configs[3]): see tp_tc_kernel. U is split hi + lo bf16 (a single
// bf16 U loses ~3e-2 to cancellation across paths on the l_max = 3 table).
// Any other shape, and the per-edge W[b,l,u,w] form, run a CUDA-core kernel
// that follows the reference's summation order exactly.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.h"

namespace ixb {
namespace {

using namespace sm100;

constexpr int kEdges = 64;          // edges per tile: UMMA M = 128 = 2 input rows x 64 edges
constexpr int kMaxPairs = 8;        // input-row pairs (nj <= 16): TMEM columns [0, 256)
constexpr int kNWs = 3;             // W ring: slots of two W[l] tiles (a path pair)
constexpr int kConsumerWarps = 16;  // 4 warpgroups, one output row of the pass each
constexpr int kTpThreads = (2 + kConsumerWarps) * 32;  // TMA, MMA + consumers
constexpr uint32_t kXPair = 2 * kEdges * 128;          // [2 rows][64 edges][128 B], SW128
constexpr uint32_t kWTile = 64 * 128;                  // W[l] [64 u][64 w], SW128 MN-major
constexpr uint32_t kWSlot = 2 * kWTile;
constexpr uint32_t kVBase = 256;                       // V ring: 2 x 128 TMEM columns
constexpr uint32_t kYwgElems = 16 * kEdges;            // per warpgroup: Y [16 k][64 edges] bf16
constexpr uint32_t kExchF4 = 2 * 4 * kEdges;           // per warpgroup: [half][chunk][edge] float4
constexpr uint32_t kTpSmem = kMaxPairs * kXPair + kNWs * kWSlot + 2 * 4 * kYwgElems * 2 +
                             4 * kExchF4 * 16 + 512 + 1024;

// acc(2 lanes) += coef * x(2 lanes): one FFMA2.
__device__ __forceinline__ float2 ffma2(float coef, float2 x, float2 acc) {
  unsigned long long d, xv, cv, av;
  asm("mov.b64 %0, {%1, %2};" : "=l"(xv) : "f"(x.x), "f"(x.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cv) : "f"(acc.x), "f"(acc.y));
  asm("mov.b64 %0, {%1, %1};" : "=l"(av) : "f"(coef));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(av), "l"(xv), "l"(cv));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(d));
  return r;
}

// Schedule of one 64-edge tile, built once per CG table (ixb_tp_plan_create).
//  pass  {first group, groups, out rows of warpgroups 0,1 (int16 each), 2,3}
//  group {jp | mask << 4 | first use of pair jp << 6 | first group of its W
//         slot << 7 | last group of its W slot << 8}: one UMMA chain
//         V = X[rows 2jp, 2jp+1] . [W[la] | W[lb]] (mask: which of the slot's
//         two paths; both -> N = 128)
//  refs  [group][path 0/1][warpgroup][half]: CG terms of (l, out row, j =
//         2jp + half) as offset | count << 24 into terms {k (int bits), v}
//  wseq  {la, lb or -1}: the W tiles of each W slot, in group order
struct TpArgs {
  const int4* pass;
  const int4* grp;
  const uint32_t* refs;
  const float2* terms;
  const int2* wseq;
  const __nv_bfloat16* Y;  // [B, nk]
  float* Z;                // [B, ni, 64]
  int64_t batch;
  int nk, ni, npasses, ngroups, nwseq, pair_mask, y_vec, accumulate;
};

// V-first factorisation:
//   V[b,l,j,:] = X[b,j,:] . W[l]                          (tcgen05, exact bf16 products)
//   Z[b,i,:]  += sum_{l,j} (sum_k v * Y[b,k]) * V[b,l,j,:] (CUDA cores, fp32)
// A tile is 64 edges; UMMA rows m < 64 are (edge m, row 2jp), m >= 64 (edge
// m - 64, row 2jp + 1), so one M = 128 MMA chain covers a pair of input rows.
// X pairs arrive by TMA ({64 u, 64 edges, 2 rows} boxes, SW128) and are
// copied into TMEM columns [32 jp, 32 jp + 32) by tcgen05.cp on first use in
// the tile: the A operand then comes from TMEM and shared memory only feeds W.
// Output rows are processed four at a time ("passes"); warpgroup h owns
// output row h of the pass for all 64 columns, so every consumer thread
// keeps one (edge, row-of-the-pair, out row) accumulator of 64 floats in
// registers and computes each CG coefficient once. The two rows of a pair
// sit in different warps (TMEM lanes m and m + 64), so their partial sums
// meet once per pass through shared memory (each half finalises 32 columns).
// Warps: 0 TMA (X pairs one tile ahead, W slots paced by the MMA), 1 TMEM
// alloc + MMA issuer, 2..17 consumers (576 threads: 112 registers each).
__global__ void __launch_bounds__(kTpThreads, 1)
    tp_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                 TpArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* Xs = smem;                                               // [8 pairs][16 KB]
  uint8_t* Ws = Xs + kMaxPairs * kXPair;                            // [3][2 tiles][8 KB]
  uint16_t* Yw = reinterpret_cast<uint16_t*>(Ws + kNWs * kWSlot);   // [4 wg][16 k][64 e]
  uint16_t* Yr = Yw + 4 * kYwgElems;                                // [4 wg][64 e][16 k] raw
  float4* Ex = reinterpret_cast<float4*>(Yr + 4 * kYwgElems);       // [4 wg][2][4][64]
  uint64_t* x_full = reinterpret_cast<uint64_t*>(Ex + 4 * kExchF4);
  uint64_t* x_empty = x_full + kMaxPairs;
  uint64_t* w_full = x_empty + kMaxPairs;
  uint64_t* w_empty = w_full + kNWs;
  uint64_t* v_full = w_empty + kNWs;
  uint64_t* v_empty = v_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int p = 0; p < kMaxPairs; ++p) {
      mbar_init(&x_full[p], 1);
      mbar_init(&x_empty[p], 1);
    }
    for (int s = 0; s < kNWs; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], kConsumerWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (a.batch + kEdges - 1) / kEdges;
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // W slots are paced by the MMA (3-deep ring); the X pairs of the next tile
    // are issued as soon as the current tile has copied each pair into TMEM
    // (polled between W loads), so X streams one tile ahead of the MMAs.
    if (lane == 0) {
      tma_prefetch_desc(&tmX);
      tma_prefetch_desc(&tmW);
      const uint64_t stream = l2_evict_first(), keep = l2_evict_last();
      uint32_t wc = 0;
      int64_t xt = blockIdx.x;  // tile of the next X load
      int xtl = 0, xp = 0;      // its tile ordinal and pair
      // issue X loads in (tile, pair) order up to tile ordinal `upto`; without
      // `block`, stop at the first staging slot not yet copied out
      auto x_next = [&](int upto, bool block) {
        while (xt < ntiles && xtl <= upto) {
          if (!((a.pair_mask >> xp) & 1)) {
            if (++xp == kMaxPairs) xp = 0, xt += gridDim.x, ++xtl;
            continue;
          }
          const uint32_t par = (xtl & 1) ^ 1;  // previous tile's copy of this pair done
          if (!block && !mbar_test(&x_empty[xp], par)) return;
          mbar_wait(&x_empty[xp], par);
          mbar_arrive_expect_tx(&x_full[xp], kXPair);
          tma_load_3d(Xs + xp * kXPair, &tmX, &x_full[xp], 0, static_cast<int32_t>(xt * kEdges),
                      2 * xp, stream);
          if (++xp == kMaxPairs) xp = 0, xt += gridDim.x, ++xtl;
        }
      };
      int tl = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
        // this tile's X must be in flight before its W (the MMA needs both)
        x_next(tl, true);
        for (int n = 0; n < a.nwseq; ++n, ++wc) {
          const int2 w = __ldg(&a.wseq[n]);
          const uint32_t ws = wc % kNWs;
          while (!mbar_test(&w_empty[ws], ((wc / kNWs) & 1) ^ 1)) x_next(tl + 1, false);
          mbar_arrive_expect_tx(&w_full[ws], w.y >= 0 ? kWSlot : kWTile);
          tma_load_2d(Ws + ws * kWSlot, &tmW, &w_full[ws], 0, w.x * 64, keep);
          if (w.y >= 0) tma_load_2d(Ws + ws * kWSlot + kWTile, &tmW, &w_full[ws], 0, w.y * 64, keep);
          x_next(tl + 1, false);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc64 = idesc_bf16_f32(128, 64, false, /*B MN-major*/ true);
      constexpr uint32_t idesc128 = idesc_bf16_f32(128, 128, false, true);
      uint32_t gc = 0, wc = 0;
      int tl = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
        for (int gi = 0; gi < a.ngroups; ++gi, ++gc) {
          const int f = __ldg(&a.grp[gi].x);
          const int jp = f & 15, mask = (f >> 4) & 3;
          const uint32_t ws = wc % kNWs;
          if ((f >> 7) & 1) mbar_wait(&w_full[ws], (wc / kNWs) & 1);
          const uint32_t vs = gc & 1;
          mbar_wait(&v_empty[vs], ((gc >> 1) & 1) ^ 1);
          if ((f >> 6) & 1) {  // first use of this pair in the tile: stage it into TMEM
            mbar_wait(&x_full[jp], tl & 1);
            tc_fence_after();
            const uint32_t x0 = smem_u32(Xs + jp * kXPair);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tmem_cp_128x256b(tmem + 32 * jp + 8 * kk,
                               smem_desc(x0 + kk * 32, 16, 1024, kLayoutSW128));
            umma_commit(&x_empty[jp]);  // staging slot reusable once copied
          }
          tc_fence_after();
          const uint32_t d = tmem + kVBase + 128 * vs + (mask == 2 ? 64 : 0);
          const uint32_t w0 = smem_u32(Ws + ws * kWSlot) + (mask == 2 ? kWTile : 0);
          const uint32_t idesc = mask == 3 ? idesc128 : idesc64;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_f16_ts(d, tmem + 32 * jp + 8 * kk,
                        smem_desc(w0 + kk * 2048, kWTile, 1024, kLayoutSW128), idesc,
                        kk > 0 ? 1u : 0u);
          umma_commit(&v_full[vs]);
          if ((f >> 8) & 1) {
            umma_commit(&w_empty[ws]);
            ++wc;
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ consumers
    const int cw = warp - 2, h = cw >> 2, q = warp & 3, hf = q >> 1;
    const int e = ((q & 1) << 5) | lane;          // edge of TMEM lane 32q + lane
    const int t = (cw & 3) * 32 + lane;           // thread in the warpgroup
    const int ey = t >> 1, kh = t & 1;            // Y staging: edge ey, k in [8kh, 8kh + 8)
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + kVBase;
    uint16_t* yw = Yw + h * kYwgElems;
    float4* ex = Ex + h * kExchF4;
    // Y rows of the next tile are prefetched by cp.async into this thread's own
    // 16-byte chunk of a raw [edge][16] staging row (no registers held across
    // the tile), then transposed to [k][edge] at the tile start.
    uint16_t* yraw = Yr + h * kYwgElems + ey * 16 + 8 * kh;
    auto fetch_y = [&](int64_t tile) {
      const int64_t b = tile * kEdges + ey;
      if (tile >= ntiles) return;
      if (a.y_vec) {
        cp_async_16(smem_u32(yraw), a.Y + (b < a.batch ? b : 0) * 16 + 8 * kh, b < a.batch ? 16 : 0);
        cp_async_commit();
      } else {
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
          const int k = 8 * kh + qq;
          yraw[qq] = (b < a.batch && k < a.nk)
                         ? __ldg(reinterpret_cast<const uint16_t*>(a.Y) + b * a.nk + k)
                         : static_cast<uint16_t>(0);
        }
      }
    };
    fetch_y(blockIdx.x);
    uint32_t gc = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      {  // publish this tile's Y as [k][edge] (conflict-free per-lane reads)
        cp_async_wait<0>();
        const uint4 yv = *reinterpret_cast<const uint4*>(yraw);
        const uint32_t w4[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          yw[(8 * kh + qq) * kEdges + ey] = static_cast<uint16_t>(w4[qq >> 1] >> (16 * (qq & 1)));
      }
      named_bar_sync(1 + h, 128);
      fetch_y(tile + gridDim.x);
      const int64_t b = tile * kEdges + e;
      for (int P = 0; P < a.npasses; ++P) {
        const int4 ps = __ldg(&a.pass[P]);
        const int out_i = static_cast<int16_t>(((h < 2 ? ps.z : ps.w) >> (16 * (h & 1))) & 0xFFFF);
        float2 acc[4][8];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int qq = 0; qq < 8; ++qq) acc[c][qq] = make_float2(0.f, 0.f);
        for (int gi = ps.x; gi < ps.x + ps.y; ++gi, ++gc) {
          const uint32_t vs = gc & 1;
          const uint32_t r0 = __ldg(&a.refs[gi * 16 + h * 2 + hf]);
          const uint32_t r1 = __ldg(&a.refs[gi * 16 + 8 + h * 2 + hf]);
          mbar_wait(&v_full[vs], (gc >> 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int pi = 0; pi < 2; ++pi) {
            const uint32_t ref = pi ? r1 : r0;
            const int cnt = static_cast<int>(ref >> 24);
            if (cnt == 0) continue;  // warp-uniform
            const float2* tm = a.terms + (ref & 0xFFFFFF);
            float coef = 0.f;
            for (int u = 0; u < cnt; ++u) {
              const float2 term = __ldg(&tm[u]);
              const int k = __float_as_int(term.x);
              coef = fmaf(term.y,
                          __uint_as_float(static_cast<uint32_t>(yw[k * kEdges + e]) << 16), coef);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t r[16];
              tmem_ld_32x32b_x16(trow + 128 * vs + 64 * pi + 16 * c, r);
              tmem_ld_wait();
#pragma unroll
              for (int qq = 0; qq < 8; ++qq)
                acc[c][qq] = ffma2(coef, make_float2(__uint_as_float(r[2 * qq]),
                                                     __uint_as_float(r[2 * qq + 1])),
                                   acc[c][qq]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&v_empty[vs]);
        }
        if (out_i < 0) continue;  // uniform over the warpgroup
        // the two rows of the pair meet: half 0 finalises columns [0, 32),
        // half 1 [32, 64), one 16-column chunk per round
#pragma unroll
        for (int r = 0; r < 2; ++r) {
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            const float2 g0 = hf ? acc[r][2 * qq] : acc[2 + r][2 * qq];
            const float2 g1 = hf ? acc[r][2 * qq + 1] : acc[2 + r][2 * qq + 1];
            ex[(hf * 4 + qq) * kEdges + e] = make_float4(g0.x, g0.y, g1.x, g1.y);
          }
          named_bar_sync(1 + h, 128);
          if (b < a.batch) {
            float4* z = reinterpret_cast<float4*>(a.Z + (b * a.ni + out_i) * 64 + 16 * (hf ? 2 + r : r));
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) {
              const float4 o = ex[((1 - hf) * 4 + qq) * kEdges + e];
              const float2 k0 = hf ? acc[2 + r][2 * qq] : acc[r][2 * qq];
              const float2 k1 = hf ? acc[2 + r][2 * qq + 1] : acc[r][2 * qq + 1];
              float4 v = make_float4(k0.x + o.x, k0.y + o.y, k1.x + o.z, k1.y + o.w);
              if (a.accumulate) {
                const float4 old = z[qq];
                v.x += old.x;
                v.y += old.y;
                v.z += old.z;
                v.w += old.w;
              }
              z[qq] = v;
            }
          }
          named_bar_sync(1 + h, 128);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}


// CUDA-core path: thread per (b, i, w); slots of component i in slot order,
// u innermost, prod = ((CGV * X) * Y) * W as plan.cpp:588-592.
__global__ void tp_simt_kernel(const int32_t* rowptr, const int32_t* slots, const int32_t* CGL,
                               const int32_t* CGJ, const int32_t* CGK, const float* CGV,
                               int64_t g, const __nv_bfloat16* X, const __nv_bfloat16* Y,
                               const __nv_bfloat16* W, int w_per_batch, int64_t batch,
                               int64_t ni, int64_t nj, int64_t nk, int64_t nl, int64_t U,
                               int64_t Wd, float* Z, int accumulate) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= batch * ni * Wd) return;
  const int64_t w = t % Wd, i = (t / Wd) % ni, b = t / (Wd * ni);
  float acc = 0.f;
  for (int e = rowptr[i]; e < rowptr[i + 1]; ++e) {
    const int s = slots[e];
    const int j = CGJ[s], k = CGK[s], l = CGL[s / g];
    const float v = CGV[s];
    const float y = __bfloat162float(Y[b * nk + k]);
    const __nv_bfloat16* x = X + (b * nj + j) * U;
    const __nv_bfloat16* wp = W + ((w_per_batch ? b * nl : 0) + l) * U * Wd + w;
    for (int64_t u = 0; u < U; ++u) {
      acc += ((v * __bfloat162float(x[u])) * y) * __bfloat162float(wp[u * Wd]);
    }
  }
  float* z = Z + (b * ni + i) * Wd + w;
  *z = accumulate ? *z + acc : acc;
}

}  // namespace
}  // namespace ixb

using namespace ixb;

// ------------------------------------------------------------ host side
// Inspector/executor split (like ixb_conv_plan): the CG table is tiny and
// fixed across calls, so it is validated and reshaped (job table for the
// tensor-core path, per-component slot lists for the CUDA-core path) once.
struct ixb_tp_plan {
  int64_t G = 0, g = 1, ni = 0, nj = 0, nk = 0, nl = 0, U = 0, Wd = 0;
  int w_per_batch = 0;
  const int32_t *CGL = nullptr, *CGJ = nullptr, *CGK = nullptr;
  const float* CGV = nullptr;
  bool tc = false;  // shape admits the tensor-core path
  // tensor-core schedule (TpArgs): one device blob, the counts by value
  void* d_sched = nullptr;
  const int4 *pass = nullptr, *grp = nullptr;
  const uint32_t* refs = nullptr;
  const float2* terms = nullptr;
  const int2* wseq = nullptr;
  int npasses = 0, ngroups = 0, nwseq = 0, pair_mask = 0;
  int32_t* d_rowptr = nullptr;  // CUDA-core path: slots per output component
  int32_t* d_slots = nullptr;
};

extern "C" int ixb_tp_plan_create(const int32_t* CGL, const int32_t* CGI, const int32_t* CGJ,
                                  const int32_t* CGK, const float* CGV, int64_t G, int64_t g,
                                  int w_per_batch, int64_t ni, int64_t nj, int64_t nk, int64_t nl,
                                  int64_t U, int64_t Wd, int flags, ixb_stream stream,
                                  ixb_tp_plan** out) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!out) fail(IXB_SHAPE, "ixb_tp_plan_create: null plan pointer");
    *out = nullptr;
    if (G < 0 || g < 1 || ni < 0 || nj < 0 || nk < 0 || nl < 0 || U < 1 || Wd < 1)
      fail(IXB_SHAPE, "ixb_tp_grouped: bad extents");
    // bring the table to the host and validate it like the plan executor
    // (gathers X/CGJ, Y/CGK, W/CGL, then scatter Z/CGI; plan.cpp:544-561)
    const int64_t slots = G * g;
    std::vector<int32_t> hl(G), hi(slots), hj(slots), hk(slots);
    std::vector<float> hv(slots);
    if (slots) {
      IXB_CUDA_CHECK(cudaMemcpyAsync(hl.data(), CGL, G * 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaMemcpyAsync(hi.data(), CGI, slots * 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaMemcpyAsync(hj.data(), CGJ, slots * 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaMemcpyAsync(hk.data(), CGK, slots * 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaMemcpyAsync(hv.data(), CGV, slots * 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaStreamSynchronize(s));
    }
    if (!(flags & IXB_UNCHECKED)) {
      auto bad = [](const char* idx, const char* tgt, int dim, int64_t ext,
                    const std::vector<int32_t>& v) {
        for (size_t p = 0; p < v.size(); ++p) {
          if (v[p] < 0 || v[p] >= ext) {
            fail(IXB_INDEX_RANGE, std::string("index tensor ") + idx + " value " +
                                      std::to_string(v[p]) + " at position [" +
                                      std::to_string(p) + "] out of range for dim " +
                                      std::to_string(dim) + " of " + tgt + " (extent " +
                                      std::to_string(ext) + ")");
          }
        }
      };
      bad("CGJ", "X", 1, nj, hj);
      bad("CGK", "Y", 1, nk, hk);
      bad("CGL", "W", w_per_batch ? 1 : 0, nl, hl);
      bad("CGI", "Z", 1, ni, hi);
    }
    auto plan = std::make_unique<ixb_tp_plan>();
    plan->G = G, plan->g = g, plan->ni = ni, plan->nj = nj, plan->nk = nk, plan->nl = nl;
    plan->U = U, plan->Wd = Wd, plan->w_per_batch = w_per_batch;
    plan->CGL = CGL, plan->CGJ = CGJ, plan->CGK = CGK, plan->CGV = CGV;
    // CUDA-core path: slots per output component, in slot order (pads are inert)
    std::vector<std::vector<int32_t>> by_i(ni);
    for (int64_t sl = 0; sl < slots; ++sl) by_i[hi[sl]].push_back(static_cast<int32_t>(sl));
    std::vector<int32_t> rowptr(ni + 1, 0), flat;
    for (int64_t i = 0; i < ni; ++i) {
      rowptr[i + 1] = rowptr[i] + static_cast<int32_t>(by_i[i].size());
      flat.insert(flat.end(), by_i[i].begin(), by_i[i].end());
    }
    IXB_CUDA_CHECK(cudaMalloc(&plan->d_rowptr, (ni + 1) * 4));
    IXB_CUDA_CHECK(cudaMalloc(&plan->d_slots, (flat.size() + 1) * 4));
    IXB_CUDA_CHECK(cudaMemcpyAsync(plan->d_rowptr, rowptr.data(), (ni + 1) * 4,
                                   cudaMemcpyHostToDevice, s));
    if (!flat.empty())
      IXB_CUDA_CHECK(cudaMemcpyAsync(plan->d_slots, flat.data(), flat.size() * 4,
                                     cudaMemcpyHostToDevice, s));
    // tensor-core path: the V-first schedule of one 64-edge tile (tp_tc_kernel)
    bool tc = !w_per_batch && U == 64 && Wd == 64 && nj <= 2 * kMaxPairs && nk <= 16 &&
              nl >= 1 && ni <= 32767;
    if (tc) {
      // (l, i, j) -> CG terms (k, v) in slot order; pads (v == 0) dropped
      std::map<std::tuple<int, int, int>, std::vector<std::pair<int, float>>> ent;
      for (int64_t sl = 0; sl < slots; ++sl) {
        if (hv[sl] == 0.f) continue;
        ent[std::make_tuple(hl[sl / g], hi[sl], hj[sl])].emplace_back(hk[sl], hv[sl]);
      }
      std::vector<int4> pass, grp;
      std::vector<uint32_t> refs;
      std::vector<float2> terms;
      std::vector<int2> wseq;
      uint32_t seen = 0;  // pairs already staged in this tile
      for (int64_t i0 = 0; i0 < ni && tc; i0 += 4) {
        int outs[4];
        for (int h = 0; h < 4; ++h) outs[h] = i0 + h < ni ? static_cast<int>(i0 + h) : -1;
        // paths feeding this pass and the input-row pairs each needs
        std::map<int, uint32_t> need;
        for (const auto& kv : ent) {
          const int l = std::get<0>(kv.first), i = std::get<1>(kv.first), j = std::get<2>(kv.first);
          if (i >= i0 && i < i0 + 4) need[l] |= 1u << (j / 2);
        }
        // paths with the same pair set side by side, then paired into W slots
        std::vector<std::pair<uint32_t, int>> order;
        for (const auto& kv : need) order.emplace_back(kv.second, kv.first);
        std::sort(order.begin(), order.end());
        const int g0 = static_cast<int>(grp.size());
        for (size_t o = 0; o < order.size(); o += 2) {
          const int la = order[o].second;
          const int lb = o + 1 < order.size() ? order[o + 1].second : -1;
          const uint32_t ma = order[o].first, mb = lb >= 0 ? order[o + 1].first : 0u;
          wseq.push_back(make_int2(la, lb));
          const int first = static_cast<int>(grp.size());
          for (int jp = 0; jp < kMaxPairs; ++jp) {
            const int mask = static_cast<int>(((ma >> jp) & 1) | (((mb >> jp) & 1) << 1));
            if (!mask) continue;
            int f = jp | (mask << 4);
            if (!((seen >> jp) & 1)) f |= 1 << 6;
            seen |= 1u << jp;
            grp.push_back(make_int4(f, 0, 0, 0));
            for (int pi = 0; pi < 2; ++pi)
              for (int h = 0; h < 4; ++h)
                for (int hf = 0; hf < 2; ++hf) {
                  const int l = pi ? lb : la, j = 2 * jp + hf;
                  uint32_t ref = 0;
                  if (l >= 0 && outs[h] >= 0 && ((mask >> pi) & 1)) {
                    auto it = ent.find(std::make_tuple(l, outs[h], j));
                    if (it != ent.end()) {
                      if (it->second.size() > 255 || terms.size() >= (1u << 24)) tc = false;
                      ref = static_cast<uint32_t>(terms.size()) |
                            (static_cast<uint32_t>(it->second.size()) << 24);
                      for (const auto& kvp : it->second) {
                        float kf;
                        std::memcpy(&kf, &kvp.first, sizeof kf);
                        terms.push_back(make_float2(kf, kvp.second));
                      }
                    }
                  }
                  refs.push_back(ref);
                }
          }
          grp[first].x |= 1 << 7;
          grp.back().x |= 1 << 8;
        }
        auto pk = [](int x, int y) {
          return static_cast<int>((static_cast<uint32_t>(x) & 0xFFFF) |
                                  ((static_cast<uint32_t>(y) & 0xFFFF) << 16));
        };
        pass.push_back(make_int4(g0, static_cast<int>(grp.size()) - g0, pk(outs[0], outs[1]),
                                 pk(outs[2], outs[3])));
      }
      if (tc) {
        if (terms.empty()) terms.push_back(make_float2(0.f, 0.f));
        if (wseq.empty()) wseq.push_back(make_int2(0, -1));
        const size_t bp = 0, bg = bp + pass.size() * sizeof(int4),
                     br = bg + grp.size() * sizeof(int4) + 16,
                     bt = (br + refs.size() * 4 + 15) / 16 * 16,
                     bw = bt + terms.size() * sizeof(float2), total = bw + wseq.size() * sizeof(int2);
        std::vector<char> blob(total, 0);
        std::memcpy(blob.data() + bp, pass.data(), pass.size() * sizeof(int4));
        std::memcpy(blob.data() + bg, grp.data(), grp.size() * sizeof(int4));
        std::memcpy(blob.data() + br, refs.data(), refs.size() * 4);
        std::memcpy(blob.data() + bt, terms.data(), terms.size() * sizeof(float2));
        std::memcpy(blob.data() + bw, wseq.data(), wseq.size() * sizeof(int2));
        IXB_CUDA_CHECK(cudaMalloc(&plan->d_sched, total));
        IXB_CUDA_CHECK(cudaMemcpyAsync(plan->d_sched, blob.data(), total, cudaMemcpyHostToDevice, s));
        IXB_CUDA_CHECK(cudaStreamSynchronize(s));  // blob is a host temporary
        char* d = static_cast<char*>(plan->d_sched);
        plan->pass = reinterpret_cast<const int4*>(d + bp);
        plan->grp = reinterpret_cast<const int4*>(d + bg);
        plan->refs = reinterpret_cast<const uint32_t*>(d + br);
        plan->terms = reinterpret_cast<const float2*>(d + bt);
        plan->wseq = reinterpret_cast<const int2*>(d + bw);
        plan->npasses = static_cast<int>(pass.size());
        plan->ngroups = static_cast<int>(grp.size());
        plan->nwseq = static_cast<int>(wseq.size());
        plan->pair_mask = static_cast<int>(seen);
        if (grp.empty()) plan->nwseq = 0;
      }
    }
    plan->tc = tc;
    *out = plan.release();
  });
}

extern "C" int ixb_tp_plan_run(ixb_tp_plan* plan, const void* X, const void* Y, const void* W,
                               int64_t batch, float* Z, int accumulate, int flags,
                               ixb_stream stream) {
  (void)flags;
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!plan) fail(IXB_SHAPE, "ixb_tp_plan_run: null plan");
    if (batch < 0) fail(IXB_SHAPE, "ixb_tp_grouped: bad extents");
    const ixb_tp_plan& p = *plan;
    if (batch == 0 || p.ni == 0) return;
    const bool aligned = reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
                         reinterpret_cast<uintptr_t>(W) % 16 == 0 &&
                         reinterpret_cast<uintptr_t>(Z) % 16 == 0;
    if (p.tc && aligned) {
      const CUtensorMap tmW = make_tmap_2d(W, 64, static_cast<uint64_t>(p.nl) * 64, 128, 64, 64,
                                           CU_TENSOR_MAP_SWIZZLE_128B);
      // X viewed as (u, edge, row): a {64, 64, 2} box lands as [row][edge][u]
      const CUtensorMap tmX = make_tmap_3d(X, 64, static_cast<uint64_t>(batch),
                                           static_cast<uint64_t>(p.nj), p.nj * 128, 128, 64,
                                           kEdges, 2, CU_TENSOR_MAP_SWIZZLE_128B);
      TpArgs args{p.pass, p.grp, p.refs, p.terms, p.wseq, static_cast<const __nv_bfloat16*>(Y), Z,
                  batch, static_cast<int>(p.nk), static_cast<int>(p.ni), p.npasses, p.ngroups,
                  p.nwseq, p.pair_mask,
                  p.nk == 16 && reinterpret_cast<uintptr_t>(Y) % 16 == 0 ? 1 : 0, accumulate};
      set_max_dynamic_smem(reinterpret_cast<const void*>(tp_tc_kernel), kTpSmem,
                           "cudaFuncSetAttribute(tp_tc_kernel)");
      int64_t grid = ceil_div(batch, kEdges);
      if (grid > sm_count()) grid = sm_count();
      tp_tc_kernel<<<static_cast<unsigned>(grid), kTpThreads, kTpSmem, s>>>(tmX, tmW, args);
      IXB_LAUNCH_CHECK("tp_tc_kernel");
      return;
    }
    const int64_t n = batch * p.ni * p.Wd;
    tp_simt_kernel<<<ceil_div(n, 256), 256, 0, s>>>(
        p.d_rowptr, p.d_slots, p.CGL, p.CGJ, p.CGK, p.CGV, p.g,
        static_cast<const __nv_bfloat16*>(X), static_cast<const __nv_bfloat16*>(Y),
        static_cast<const __nv_bfloat16*>(W), p.w_per_batch, batch, p.ni, p.nj, p.nk, p.nl, p.U,
        p.Wd, Z, accumulate);
    IXB_LAUNCH_CHECK("tp_simt_kernel");
  });
}

namespace {
// Side streams and events for the host-buffer form, created once per thread
// and device (as in pipeline.cpp).
struct TpStreams {
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
thread_local TpStreams t_tp_streams;
}  // namespace

// Host-buffer form: X, Y and Z in host memory (pinned for overlap), W on the
// device. Edges are independent, so the batch is cut into chunks of whole
// 64-edge tiles; chunk i's X/Y copy in, its evaluation and its Z copy out
// run on three streams, so both PCIe directions and the kernels overlap.
// Each edge is evaluated exactly as by ixb_tp_plan_run (bit-identical).
extern "C" int ixb_tp_plan_run_host(ixb_tp_plan* plan, const void* X, const void* Y,
                                    const void* W, int64_t batch, float* Z, int accumulate,
                                    int flags, int nchunks, ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!plan) fail(IXB_SHAPE, "ixb_tp_plan_run: null plan");
    if (batch < 0) fail(IXB_SHAPE, "ixb_tp_grouped: bad extents");
    const ixb_tp_plan& p = *plan;
    if (batch == 0 || p.ni == 0) return;
    const int64_t xrow = p.nj * p.U * 2, yrow = p.nk * 2, zrow = p.ni * p.Wd * 4;
    const int64_t wrow = p.w_per_batch ? p.nl * p.U * p.Wd * 2 : 0;  // per-edge W offset
    if (nchunks < 1) nchunks = 1;
    int64_t chunk = (batch + nchunks - 1) / nchunks;
    chunk = (chunk + kEdges - 1) / kEdges * kEdges;
    nchunks = static_cast<int>((batch + chunk - 1) / chunk);
    Scratch<char> dX(batch * xrow, s), dY(batch * yrow, s), dZ(batch * zrow, s);
    TpStreams& st = t_tp_streams;
    st.ensure(2 + 2 * nchunks);
    IXB_CUDA_CHECK(cudaEventRecord(st.ev[0], s));  // scratch allocated on s
    IXB_CUDA_CHECK(cudaStreamWaitEvent(st.h2d, st.ev[0], 0));
    for (int i = 0; i < nchunks; ++i) {
      const int64_t b0 = i * chunk, n = batch - b0 < chunk ? batch - b0 : chunk;
      cudaEvent_t in = st.ev[2 + 2 * i], out = st.ev[3 + 2 * i];
      IXB_CUDA_CHECK(cudaMemcpyAsync(dX.p + b0 * xrow, static_cast<const char*>(X) + b0 * xrow,
                                     n * xrow, cudaMemcpyHostToDevice, st.h2d));
      IXB_CUDA_CHECK(cudaMemcpyAsync(dY.p + b0 * yrow, static_cast<const char*>(Y) + b0 * yrow,
                                     n * yrow, cudaMemcpyHostToDevice, st.h2d));
      if (accumulate)
        IXB_CUDA_CHECK(cudaMemcpyAsync(dZ.p + b0 * zrow,
                                       reinterpret_cast<const char*>(Z) + b0 * zrow, n * zrow,
                                       cudaMemcpyHostToDevice, st.h2d));
      IXB_CUDA_CHECK(cudaEventRecord(in, st.h2d));
      IXB_CUDA_CHECK(cudaStreamWaitEvent(s, in, 0));
      const int rc = ixb_tp_plan_run(plan, dX.p + b0 * xrow, dY.p + b0 * yrow,
                                     static_cast<const char*>(W) + b0 * wrow, n,
                                     reinterpret_cast<float*>(dZ.p + b0 * zrow), accumulate,
                                     flags, stream);
      if (rc != IXB_OK) fail(rc, ixb_last_error());
      IXB_CUDA_CHECK(cudaEventRecord(out, s));
      IXB_CUDA_CHECK(cudaStreamWaitEvent(st.d2h, out, 0));
      IXB_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(Z) + b0 * zrow, dZ.p + b0 * zrow,
                                     n * zrow, cudaMemcpyDeviceToHost, st.d2h));
    }
    IXB_CUDA_CHECK(cudaEventRecord(st.ev[1], st.d2h));
    IXB_CUDA_CHECK(cudaStreamWaitEvent(s, st.ev[1], 0));
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));  // Z is in host memory on return
  });
}

extern "C" void ixb_tp_plan_free(ixb_tp_plan* plan) {
  if (!plan) return;
  cudaFree(plan->d_rowptr);  // synchronous: in-flight runs finish first
  cudaFree(plan->d_slots);
  cudaFree(plan->d_sched);
  delete plan;
}

extern "C" int ixb_tp_grouped(const int32_t* CGL, const int32_t* CGI, const int32_t* CGJ,
                              const int32_t* CGK, const float* CGV, int64_t G, int64_t g,
                              const void* X, const void* Y, const void* W, int w_per_batch,
                              int64_t batch, int64_t ni, int64_t nj, int64_t nk, int64_t nl,
                              int64_t U, int64_t Wd, float* Z, int accumulate, int flags,
                              ixb_stream stream) {
  if (G < 0 || g < 1 || batch < 0 || ni < 0 || nj < 0 || nk < 0 || nl < 0 || U < 1 || Wd < 1)
    return ixb_guard([] { fail(IXB_SHAPE, "ixb_tp_grouped: bad extents"); });
  if (batch == 0 || ni == 0) return ixb_guard([] {});
  ixb_tp_plan* plan = nullptr;
  int rc = ixb_tp_plan_create(CGL, CGI, CGJ, CGK, CGV, G, g, w_per_batch, ni, nj, nk, nl, U, Wd,
                              flags, stream, &plan);
  if (rc != IXB_OK) return rc;
  rc = ixb_tp_plan_run(plan, X, Y, W, batch, Z, accumulate, flags, stream);
  ixb_tp_plan_free(plan);
  return rc;
}
