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
#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.h"

namespace ixb {
namespace {

using namespace sm100;

constexpr int kEdges = 64;                         // edges per tile
constexpr int kMathWarps = 16;                     // 64 edges x 8 u-slices
constexpr int kMathThreads = kMathWarps * 32;
constexpr int kEpiWarps = 4;                        // one per TMEM lane quarter
constexpr int kTpThreads = kMathThreads + 64 + kEpiWarps * 32;  // + UMMA, TMA, epilogue warps
constexpr int kPairs = 8;                           // component pairs (16 components)
constexpr int kMaxJobs = 192;
constexpr int kMaxJSteps = 512;
constexpr int kMaxPathSeq = 64;
constexpr int kNU = 2;                              // U ring (job operands, hi + lo)
constexpr int kNW = 2;                              // W ring (one path each)
constexpr int kGroupWarps = kMathWarps / 2;         // math warps per job group
#ifndef IXB_TP_JUNROLL
#define IXB_TP_JUNROLL 1
#endif
constexpr int kJUnroll = IXB_TP_JUNROLL;            // j-step loop unroll
constexpr uint32_t kUHalf = 128 * 128;              // 128 rows (2 comps x 64 edges) x 64 bf16
constexpr uint32_t kUSlot = 2 * kUHalf;             // hi, lo
constexpr uint32_t kWTileTp = 64 * 128;             // 64 u-rows x 64 bf16
constexpr uint32_t kXTile = kEdges * 16 * 128;      // 64 edges x 16 irrep rows x 64 bf16

// CG table reshaped for the tensor-core path, passed by value (constant bank:
// every lane reads the same entry, which the constant cache broadcasts).
// A job's entries are regrouped by input row j ("j-steps"): each X row is
// loaded and converted once per job and feeds both components of the pair,
// with coef_h(j) = sum_k v * Y[k] over the component's entries at that j.
struct TpMeta {
  int njobs, npaths, ni, present;  // present: bit i = component i receives a job
  int ncp;                         // component pairs that receive a job
  int cp_order[kPairs];            // drain order: the ncp pairs with jobs by their last job, then the rest
  // job: {l | first-touch-of-cp << 8 | last-job-of-path << 9 | first-job-of-path << 10 |
  //       last-touch-of-cp << 11, cp | path-seq << 8, first j-step | j-step count << 16, 0}
  int4 job[kMaxJobs];
  // j-step: {j | n0 << 4 | n1 << 6 | k00 << 8 | k01 << 12 | k10 << 16 | k11 << 20,
  //          v00, v01, v10 (float bits)} and v11 in jv11: component 2cp has n0 <= 2
  //          terms (k0t, v0t) at this j, component 2cp+1 has n1 <= 2 (a (component, j)
  //          with more terms takes several steps)
  int4 jstep[kMaxJSteps];
  float jv11[kMaxJSteps];
  int path_l[kMaxPathSeq];  // W index of each path in job order
};

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

struct TpArgs {
  const __nv_bfloat16* Y;  // [B, nk]
  float* Z;                // [B, ni, 64]
  int64_t batch;
  int nj, nk, ni;
  int accumulate;
};

// Output-side factorisation, batched two output components at
// a time so every UMMA has M = 128:
//   U_{l,i}[b,u] = sum_{(j,k,v) in (l,i)} v * Y[b,k] * X[b,j,u]   (CUDA cores)
//   Z[b,i,:]    += U_{l,i}[b,:] . W[l]                           (tcgen05)
// A job = (path l, component pair cp): A rows 0..63 = U_{l,2cp}, rows 64..127
// = U_{l,2cp+1} (zero when the path has no such component), B = W[l], D =
// TMEM columns [64 cp, 64 cp + 64) (lanes 0..63 component 2cp, 64..127
// component 2cp+1): 8 pairs x 64 = all 512 columns.
// Warps 0..15 compute U for job n into a kNU-deep ring (mbarrier handoff,
// no block-wide barrier per job), warp 16 issues 4 UMMAs (K = 64) per job and
// commits the slot back, warp 17 streams X tiles and W[l] (kNW ring) by TMA,
// warps 18..21 drain TMEM into Z. TMEM is handed over per component pair:
// the issuer commits acc_full[cp] after the pair's last job of the tile and
// waits on acc_empty[cp] before its first job of the next tile. Paths run
// in order of their output irrep, so pairs complete one after another and
// draining overlaps the remaining jobs and the next tile's start.
__global__ void __launch_bounds__(kTpThreads, 1)
    tp_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ TpMeta meta, TpArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // align by offset (not through an integer cast) so every derived pointer
  // stays in the shared space: LDS/STS instead of generic loads
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* Xs = smem;                   // [64 edges * nj rows][128 B]
  uint8_t* Us = Xs + kXTile;            // [kNU][128 rows][128 B]  (SW128 K-major)
  uint8_t* Ws = Us + kNU * kUSlot;      // [kNW][64 rows][128 B]   (SW128 MN-major)
  float* Ys = reinterpret_cast<float*>(Ws + kNW * kWTileTp);  // [2 groups][64][16]
  uint64_t* x_full = reinterpret_cast<uint64_t*>(Ys + 2 * kEdges * 16);
  uint64_t* x_empty = x_full + 1;
  uint64_t* w_full = x_empty + 1;
  uint64_t* w_empty = w_full + kNW;
  uint64_t* u_full = w_empty + kNW;
  uint64_t* u_empty = u_full + kNU;
  uint64_t* acc_full = u_empty + kNU;      // [kPairs]
  uint64_t* acc_empty = acc_full + kPairs;  // [kPairs]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kPairs);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(x_full, 1);
    mbar_init(x_empty, kMathWarps);
    for (int s = 0; s < kNW; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < kNU; ++s) {
      mbar_init(&u_full[s], kGroupWarps);  // slot s is written by job group s
      mbar_init(&u_empty[s], 1);
    }
    for (int c = 0; c < kPairs; ++c) {
      mbar_init(&acc_full[c], 1);
      mbar_init(&acc_empty[c], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == kMathWarps) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (a.batch + kEdges - 1) / kEdges;
  const int njobs = meta.njobs, npaths = meta.npaths;

  if (warp == kMathWarps + 1) {
    // ---------------------------------------------------------- TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmW);
      tma_prefetch_desc(&tmX);
      const uint64_t keep = l2_evict_last(), stream = l2_evict_first();
      // whole 256-row boxes land (out-of-range rows zero-filled), so expect them all
      const uint32_t x_bytes = static_cast<uint32_t>(((kEdges * a.nj + 255) / 256) * 256 * 128);
      int64_t wc = 0;  // W loads issued
      int tl = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
        mbar_wait_backoff(x_empty, (tl & 1) ^ 1, 128);  // previous tile's X fully consumed
        mbar_arrive_expect_tx(x_full, x_bytes);
        for (int r0 = 0; r0 < kEdges * a.nj; r0 += 256)
          tma_load_2d(Xs + r0 * 128, &tmX, x_full, 0,
                      static_cast<int32_t>(tile * kEdges * a.nj + r0), stream);
        for (int ps = 0; ps < npaths; ++ps, ++wc) {
          const int slot = static_cast<int>(wc % kNW);
          mbar_wait_backoff(&w_empty[slot], ((wc / kNW) & 1) ^ 1, 64);
          mbar_arrive_expect_tx(&w_full[slot], kWTileTp);
          tma_load_2d(Ws + slot * kWTileTp, &tmW, &w_full[slot], 0, meta.path_l[ps] * 64, keep);
        }
      }
    }
  } else if (warp == kMathWarps) {
    // ---------------------------------------------------------- UMMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, 64, /*A K-major*/ false, /*B MN-major*/ true);
      int tl = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
        const int64_t jc0 = static_cast<int64_t>(tl) * njobs;
        const int64_t wc0 = static_cast<int64_t>(tl) * npaths;
        for (int n = 0; n < njobs; ++n) {
          const int4 job = meta.job[n];
          const int cp = job.y & 0xFF, ps = job.y >> 8;
          const int64_t wc = wc0 + ps;
          const int wslot = static_cast<int>(wc % kNW);
          if ((job.x >> 10) & 1) mbar_wait(&w_full[wslot], (wc / kNW) & 1);
          const int64_t jc = jc0 + n;
          const int us = static_cast<int>(jc % kNU);
          mbar_wait(&u_full[us], (jc / kNU) & 1);
          tc_fence_after();
          const uint32_t u0 = smem_u32(Us + us * kUSlot);
          const uint32_t w0 = smem_u32(Ws + wslot * kWTileTp);
          const bool first = (job.x >> 8) & 1;
          if (first) {  // this pair's columns drained from the previous tile
            mbar_wait(&acc_empty[cp], (tl & 1) ^ 1);
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t bd = smem_desc(w0 + kk * 2048, 8192, 1024, kLayoutSW128);
            umma_f16(tmem + cp * 64, smem_desc(u0 + kk * 32, 16, 1024, kLayoutSW128), bd, idesc,
                     (!first || kk > 0) ? 1u : 0u);
            umma_f16(tmem + cp * 64, smem_desc(u0 + kUHalf + kk * 32, 16, 1024, kLayoutSW128), bd,
                     idesc, 1u);
          }
          umma_commit(&u_empty[us]);                         // U slot reusable
          if ((job.x >> 9) & 1) umma_commit(&w_empty[wslot]);  // last job of this path
          if ((job.x >> 11) & 1) umma_commit(&acc_full[cp]);   // pair complete for this tile
        }
      }
    }
  } else if (warp < kMathWarps) {
    // ---------------------------------------------------------- math warps
    // Two groups of 8 warps take alternate jobs (job jc -> group jc % 2 -> U
    // slot jc % 2, the issuer's ring order): one group computes while the
    // other group's slot is being consumed, so the handoff round trip hides
    // behind math. A thread owns one edge and 16 u of both components.
    const int grp = warp / kGroupWarps;
    const int gt = tid - grp * kGroupWarps * 32;
    const int b_loc = gt >> 2, slice = gt & 3;  // edge in tile, u chunks {slice, slice + 4}
    // A thread owns the 8-u chunks cA, cB = {slice, slice + 4}, odd edges in
    // swapped order: each X load of a warp (8 edges x 4 lanes, edge rows 2 KB
    // apart) then covers both 64 B halves of the banks, conflict-free.
    const int cA = slice + 4 * (b_loc & 1), cB = slice + 4 * (~b_loc & 1);
    uint32_t rowo[2][2];  // [component][chunk A/B] in the SW128 U tile
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int r = h * 64 + b_loc, ch = c ? cB : cA;
        rowo[h][c] = r * 128 + ((ch ^ (r & 7)) << 4);
      }
    const uint8_t* xrow = Xs + b_loc * a.nj * 128;
    float* yrow = Ys + (grp * kEdges + b_loc) * 16;
    int tl = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
      const int64_t b = tile * kEdges + b_loc;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 4 * slice + q;
        yrow[k] = (b < a.batch && k < a.nk) ? __bfloat162float(a.Y[b * a.nk + k]) : 0.f;
      }
      __syncwarp();  // an edge's 4 threads share one warp
      mbar_wait(x_full, tl & 1);
      const int64_t jc0 = static_cast<int64_t>(tl) * njobs;
      for (int n = 0; n < njobs; ++n) {
        const int64_t jc = jc0 + n;
        if (static_cast<int>(jc & 1) != grp) continue;
        const int4 job = meta.job[n];
        float2 a2[2][8];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 8; ++q) a2[h][q] = make_float2(0.f, 0.f);
        const int s0 = job.z & 0xFFFF, ns = job.z >> 16;
        int4 js_next = ns > 0 ? meta.jstep[s0] : make_int4(0, 0, 0, 0);
#pragma unroll kJUnroll
        for (int st = s0; st < s0 + ns; ++st) {
          const int4 js = js_next;
          if (st + 1 < s0 + ns) js_next = meta.jstep[st + 1];  // next entry in flight
          const int n0 = (js.x >> 4) & 3, n1 = (js.x >> 6) & 3;
          const uint8_t* xp = xrow + (js.x & 15) * 128;
          const uint4 xv0 = *reinterpret_cast<const uint4*>(xp + cA * 16);
          const uint4 xv1 = *reinterpret_cast<const uint4*>(xp + cB * 16);
          float c0 = __int_as_float(js.y) * yrow[(js.x >> 8) & 15];
          float c1 = __int_as_float(js.w) * yrow[(js.x >> 16) & 15];
          if (n0 > 1) c0 = fmaf(__int_as_float(js.z), yrow[(js.x >> 12) & 15], c0);
          if (n1 > 1) c1 = fmaf(meta.jv11[st], yrow[(js.x >> 20) & 15], c1);
          float2 xf[8];
          const __nv_bfloat162* xh0 = reinterpret_cast<const __nv_bfloat162*>(&xv0);
          const __nv_bfloat162* xh1 = reinterpret_cast<const __nv_bfloat162*>(&xv1);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            xf[q] = __bfloat1622float2(xh0[q]);
            xf[4 + q] = __bfloat1622float2(xh1[q]);
          }
          if (n0) {  // uniform: every lane runs the same job
#pragma unroll
            for (int q = 0; q < 8; ++q) a2[0][q] = ffma2(c0, xf[q], a2[0][q]);
          }
          if (n1) {
#pragma unroll
            for (int q = 0; q < 8; ++q) a2[1][q] = ffma2(c1, xf[q], a2[1][q]);
          }
        }
        // U = hi + lo, both bf16 (the UMMA pair sees U to ~2^-16 relative, so
        // the only bf16 roundings are the operands X, Y, W)
        mbar_wait(&u_empty[grp], static_cast<uint32_t>((jc >> 1) & 1) ^ 1);
        uint8_t* U = Us + grp * kUSlot;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint4 hi, lo;
            __nv_bfloat162* ph = reinterpret_cast<__nv_bfloat162*>(&hi);
            __nv_bfloat162* pl = reinterpret_cast<__nv_bfloat162*>(&lo);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float2 v = a2[h][4 * c + q];
              ph[q] = __floats2bfloat162_rn(v.x, v.y);
              const float2 back = __bfloat1622float2(ph[q]);
              pl[q] = __floats2bfloat162_rn(v.x - back.x, v.y - back.y);
            }
            *reinterpret_cast<uint4*>(U + rowo[h][c]) = hi;
            *reinterpret_cast<uint4*>(U + kUHalf + rowo[h][c]) = lo;
          }
        fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&u_full[grp]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(x_empty);  // X of this tile no longer read
    }
  } else {
    // ---------------------------------------------------------- epilogue warps
    // TMEM lane quarter q = warp % 4: component parity q >> 1, edges (q & 1) * 32 + lane
    const int quarter = warp & 3;
    int tl = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
      const int64_t be = tile * kEdges + (quarter & 1) * 32 + lane;
#pragma unroll 1
      for (int oc = 0; oc < kPairs; ++oc) {
        const bool touched = oc < meta.ncp;
        const int cp = meta.cp_order[oc];
        const int comp = 2 * cp + (quarter >> 1);
        if (2 * cp >= a.ni) continue;
        const bool row_ok = be < a.batch && comp < a.ni;
        float4* z = reinterpret_cast<float4*>(a.Z + (be * a.ni + comp) * 64);
        if (!touched) {  // no job writes this pair: `=` stores zeros, `+=` leaves Z
          if (row_ok && !a.accumulate)
            for (int c = 0; c < 16; ++c) z[c] = make_float4(0.f, 0.f, 0.f, 0.f);
          continue;
        }
        mbar_wait_backoff(&acc_full[cp], tl & 1, 256);  // idle polls would steal math issue slots
        tc_fence_after();
        const bool has = comp < a.ni && ((meta.present >> comp) & 1);
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {  // 16 columns at a time keeps register pressure low
          uint32_t r[16];
          tmem_ld_32x32b_x16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cp * 64 + c * 16,
                             r);
          tmem_ld_wait();
          if (row_ok) {
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              float4 v = has ? make_float4(__uint_as_float(r[4 * e]), __uint_as_float(r[4 * e + 1]),
                                           __uint_as_float(r[4 * e + 2]),
                                           __uint_as_float(r[4 * e + 3]))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
              if (a.accumulate) {
                const float4 o = z[c * 4 + e];
                v.x += o.x;
                v.y += o.y;
                v.z += o.z;
                v.w += o.w;
              }
              z[c * 4 + e] = v;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[cp]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMathWarps) {
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
  TpMeta meta{};
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
    // tensor-core path: jobs (l, component pair) in (l, cp) order; entries
    // (j, k, v) of each component in slot order, pads (v == 0) dropped
    bool tc = !w_per_batch && U == 64 && Wd == 64 && ni <= 16 && nj <= 16 && nk <= 16 && nl >= 1;
    if (tc) {
      TpMeta& meta = plan->meta;
      meta.ni = static_cast<int>(ni);
      std::vector<std::vector<std::vector<int32_t>>> li(nl, std::vector<std::vector<int32_t>>(ni));
      for (int64_t sl = 0; sl < slots; ++sl) {
        if (hv[sl] == 0.f) continue;
        li[hl[sl / g]][hi[sl]].push_back(static_cast<int32_t>(sl));
      }
      int njob = 0, nst = 0, nps = 0;
      std::vector<bool> touched((ni + 1) / 2, false);
      // paths in order of the highest output component they write (stable):
      // component pairs then complete one after another within a tile
      std::vector<int> lorder(nl);
      std::vector<int> top(nl, -1);
      for (int l = 0; l < nl; ++l) {
        lorder[l] = l;
        for (int i = 0; i < ni; ++i)
          if (!li[l][i].empty()) top[l] = i;
      }
      std::stable_sort(lorder.begin(), lorder.end(), [&](int x, int y) { return top[x] < top[y]; });
      for (int lo = 0; lo < nl && tc; ++lo) {
        const int l = lorder[lo];
        const int first_job = njob;
        for (int cp = 0; cp < (ni + 1) / 2 && tc; ++cp) {
          // j-steps: distinct input rows j of the pair (ascending); per step the
          // k-terms of component 2cp, then of 2cp+1, each in slot order
          const std::vector<int32_t> none;
          const std::vector<int32_t>& c0 = 2 * cp < ni ? li[l][2 * cp] : none;
          const std::vector<int32_t>& c1 = 2 * cp + 1 < ni ? li[l][2 * cp + 1] : none;
          if (c0.empty() && c1.empty()) continue;
          if (!c0.empty()) meta.present |= 1 << (2 * cp);
          if (!c1.empty()) meta.present |= 1 << (2 * cp + 1);
          const int st0 = nst;
          for (int j = 0; j < nj && tc; ++j) {
            std::vector<int32_t> t[2];
            for (int h = 0; h < 2; ++h)
              for (int32_t sl : h ? c1 : c0)
                if (hj[sl] == j) t[h].push_back(sl);
            for (size_t r = 0; r < t[0].size() || r < t[1].size(); r += 2) {
              if (nst >= kMaxJSteps) {
                tc = false;
                break;
              }
              int n[2], kk[2][2] = {{0, 0}, {0, 0}};
              float vv[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
              for (int h = 0; h < 2; ++h) {
                n[h] = static_cast<int>(std::min<size_t>(2, t[h].size() > r ? t[h].size() - r : 0));
                for (int q = 0; q < n[h]; ++q) {
                  kk[h][q] = hk[t[h][r + q]];
                  vv[h][q] = hv[t[h][r + q]];
                }
              }
              auto bits = [](float f) {
                int b;
                std::memcpy(&b, &f, sizeof b);
                return b;
              };
              meta.jstep[nst] = make_int4(j | (n[0] << 4) | (n[1] << 6) | (kk[0][0] << 8) |
                                              (kk[0][1] << 12) | (kk[1][0] << 16) | (kk[1][1] << 20),
                                          bits(vv[0][0]), bits(vv[0][1]), bits(vv[1][0]));
              meta.jv11[nst++] = vv[1][1];
            }
          }
          if (!tc) break;
          if (njob >= kMaxJobs || nps >= kMaxPathSeq) {
            tc = false;
            break;
          }
          const int ft = touched[cp] ? 0 : 1;
          touched[cp] = true;
          const int fp = njob == first_job ? 1 : 0;
          meta.job[njob] = make_int4(l | (ft << 8) | (fp << 10), cp | (nps << 8),
                                     st0 | ((nst - st0) << 16), 0);
          ++njob;
        }
        if (tc && njob > first_job) {
          meta.job[njob - 1].x |= 1 << 9;  // last job of this path
          meta.path_l[nps++] = l;
        }
      }
      meta.njobs = njob;
      meta.npaths = nps;
      // last job of each pair -> commit flag; drain order = order of last jobs
      int last[kPairs];
      for (int c = 0; c < kPairs; ++c) last[c] = -1;
      for (int n = 0; n < njob; ++n) last[meta.job[n].y & 0xFF] = n;
      meta.ncp = 0;
      for (int n = 0; n < njob; ++n) {
        const int c = meta.job[n].y & 0xFF;
        if (last[c] == n) {
          meta.job[n].x |= 1 << 11;
          meta.cp_order[meta.ncp++] = c;
        }
      }
      int k = meta.ncp;
      for (int c = 0; c < kPairs; ++c)
        if (last[c] < 0) meta.cp_order[k++] = c;
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
      const CUtensorMap tmX = make_tmap_2d(X, 64, static_cast<uint64_t>(batch) * p.nj, 128, 64,
                                           256, CU_TENSOR_MAP_SWIZZLE_NONE);
      TpArgs args{static_cast<const __nv_bfloat16*>(Y), Z, batch, static_cast<int>(p.nj),
                  static_cast<int>(p.nk), static_cast<int>(p.ni), accumulate};
      const uint32_t smem =
          kXTile + kNU * kUSlot + kNW * kWTileTp + 2 * kEdges * 16 * 4 + 256 + 1024;
      set_max_dynamic_smem(reinterpret_cast<const void*>(tp_tc_kernel), smem,
                           "cudaFuncSetAttribute(tp_tc_kernel)");
      int64_t grid = ceil_div(batch, kEdges);
      if (grid > sm_count()) grid = sm_count();
      tp_tc_kernel<<<static_cast<unsigned>(grid), kTpThreads, smem, s>>>(tmW, tmX, p.meta, args);
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
