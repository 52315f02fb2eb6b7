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
constexpr int kXSlots = 4;          // X staging ring (pairs in first-use order)
constexpr int kNWs = 3;             // W ring: slots of two W[l] tiles (a path pair)
constexpr int kConsumerWarps = 16;  // 4 warpgroups, one 16-column quarter of V each
constexpr int kTpThreads = (4 + kConsumerWarps) * 32;  // TMA, MMA, 2 spare + consumers
constexpr uint32_t kXPair = 2 * kEdges * 128;          // [2 rows][64 edges][128 B], SW128
constexpr uint32_t kWTile = 64 * 128;                  // W[l] [64 u][64 w], SW128 MN-major
constexpr uint32_t kWSlot = 2 * kWTile;
constexpr uint32_t kVBase = 256;                       // V ring: 2 x 128 TMEM columns
constexpr int kMaxWgCoefs = 32;                        // CG coefficients per (pass, out row), [c][edge]
constexpr uint32_t kExchF4 = 16 * kEdges;              // per warpgroup: Z tiles [2][edge][32 cols] fp32
constexpr int kMaxSchedBytes = 12288;                  // schedule, staged in shared memory
constexpr uint32_t kTpSmem = kXSlots * kXPair + kNWs * kWSlot + 16 * kEdges * 4 +
                             4 * kMaxWgCoefs * kEdges * 4 + 4 * kExchF4 * 16 + kMaxSchedBytes + 512 +
                             1024;

#ifdef IXB_TP_TRACE
// timeline of CTA 0 (tools/tp_trace.py): [role][event][n] clock64 stamps
__device__ long long g_tp_trace[4][4][512];
#define TPT(role, ev, n)                                                         \
  do {                                                                           \
    if (blockIdx.x == 0 && (n) < 512) g_tp_trace[role][ev][(n)] = clock64();     \
  } while (0)
#else
#define TPT(role, ev, n) \
  do {                   \
  } while (0)
#endif

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

// Schedule of one 64-edge tile, built once per CG table (ixb_tp_plan_create)
// and passed by value (constant bank: every lane of a warp reads the same
// entry).
//  pass  {first group, groups, out rows 0,1 (int16 each), out rows 2,3}
//  pwg   [pass][out row h] {first coefficient, n0 | n1 << 16}: warpgroup
//        h's coefficients for the pass, n0 for rows 2jp of the pairs, then n1
//        for rows 2jp + 1
//  grp   jp | mask << 4 | first use of pair jp << 6 | first group of its W
//        slot << 7 | last group of its W slot << 8 | entries of half 0 << 16
//        | entries of half 1 << 24; one UMMA chain V = X[rows 2jp, 2jp+1] .
//        [W[la] | W[lb]] (mask: which of the slot's two paths; both -> N =
//        128); entry bit 4 pi + s: path pi feeds out row s of the pass
//  cref  coefficient -> CG terms (offset | count << 24), in (group, path)
//        order per list
//  terms {k (int bits), v}
//  wseq  {la, lb or -1}: the W tiles of each W slot, in group order
struct TpSched {
  int npasses, ngroups, nwseq, nx;
  int xorder[kMaxPairs];  // pairs in first-use order (the X staging sequence)
  // byte offsets of pass (int4), pwg (int2), grp (int), cref
  // (uint32), terms (float2), wseq (int2) in blob; blob is copied to shared
  // memory at kernel start (dynamically indexed constant-bank reads miss)
  int o_pass, o_pwg, o_grp, o_cref, o_terms, o_wseq, o_crec, nbytes;
  int two_terms;  // every coefficient has <= 2 CG terms: crec {k0, v0, k1, v1} per coefficient
  uint4 blob[kMaxSchedBytes / 16];
};

struct TpArgs {
  const __nv_bfloat16* Y;  // [B, nk]
  float* Z;                // [B, ni, 64]
  int64_t batch;
  int nk, ni, y_pair, accumulate;
};

// V-first factorisation:
//   V[b,l,j,:] = X[b,j,:] . W[l]                          (tcgen05, exact bf16 products)
//   Z[b,i,:]  += sum_{l,j} (sum_k v * Y[b,k]) * V[b,l,j,:] (CUDA cores, fp32)
// A tile is 64 edges; UMMA rows m < 64 are (edge m, row 2jp), m >= 64 (edge
// m - 64, row 2jp + 1), so one M = 128 MMA chain covers a pair of input rows.
// X pairs arrive by TMA ({64 u, 64 edges, 2 rows} boxes, SW128) and are
// copied into TMEM columns [32 jp, 32 jp + 32) by tcgen05.cp on first use in
// the tile: the A operand then comes from TMEM and shared memory only feeds W.
// Output rows are processed four at a time ("passes"). At the start of a
// pass the 512 consumer threads compute its CG coefficients sum_k v * Y[b,k]
// (one per (edge, CG entry)) into shared memory; warpgroup h then owns V
// columns [16h, 16h + 16) of every group for the pass's four output rows,
// so a group costs each consumer warp one 16-column TMEM load per path plus
// one shared load and 8 FFMA2 per CG entry. The two rows of a pair sit in
// different warps (TMEM lanes m and m + 64): their partial sums meet once per
// pass through shared memory (each half finalises two of the four rows).
// Warps: 0 TMA (X pairs one tile ahead, W slots paced by the MMA), 1 TMEM
// alloc + MMA issuer, 2-3 spare, 4..19 consumers. Warpgroup 0 drops to 56
// registers (setmaxnreg) so the consumers get 104 (the pool must cover the
// increase or setmaxnreg.inc waits forever): each SM sub-partition holds one
// warpgroup-0 warp and four consumer warps.
__global__ void __launch_bounds__(kTpThreads, 1)
    tp_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                 const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ TpSched sc,
                 TpArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* Xs = smem;                                         // [4 slots][16 KB]
  uint8_t* Ws = Xs + kXSlots * kXPair;                        // [6][2 tiles][8 KB]
  float* Yk = reinterpret_cast<float*>(Ws + kNWs * kWSlot);   // [16 k][64 e]
  float* Cf = Yk + 16 * kEdges;                               // [4 wg][coef][64 e]
  float4* Ex = reinterpret_cast<float4*>(Cf + 4 * kMaxWgCoefs * kEdges);  // [4 wg][2][64][8]
  uint8_t* Sb = reinterpret_cast<uint8_t*>(Ex + 4 * kExchF4);           // schedule blob
  uint64_t* x_full = reinterpret_cast<uint64_t*>(Sb + kMaxSchedBytes);
  uint64_t* x_empty = x_full + kXSlots;
  uint64_t* w_full = x_empty + kMaxPairs;
  uint64_t* w_empty = w_full + kNWs;
  uint64_t* v_full = w_empty + kNWs;
  uint64_t* v_empty = v_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < sc.nbytes / 16; i += blockDim.x) reinterpret_cast<uint4*>(Sb)[i] = sc.blob[i];
  const int4* s_pass = reinterpret_cast<const int4*>(Sb + sc.o_pass);
  const int2* s_pwg = reinterpret_cast<const int2*>(Sb + sc.o_pwg);
  const int* s_grp = reinterpret_cast<const int*>(Sb + sc.o_grp);
  const uint32_t* s_cref = reinterpret_cast<const uint32_t*>(Sb + sc.o_cref);
  const float2* s_terms = reinterpret_cast<const float2*>(Sb + sc.o_terms);
  const int2* s_wseq = reinterpret_cast<const int2*>(Sb + sc.o_wseq);
  const float4* s_crec = reinterpret_cast<const float4*>(Sb + sc.o_crec);
  if (tid == 0) {
    for (int p = 0; p < kXSlots; ++p) {
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
  if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // W slots are paced by the MMA; X pairs go through a 4-slot staging ring
    // in first-use order, each issued as soon as its slot has been copied into
    // TMEM (polled while waiting for W slots), up to one tile ahead. The warp
    // runs converged; one elected lane issues.
    {
      tma_prefetch_desc(&tmX);
      tma_prefetch_desc(&tmW);
      const uint64_t stream = l2_evict_first(), keep = l2_evict_last();
      uint32_t wc = 0;
      int64_t xt = blockIdx.x;  // tile of the next X load
      int xtl = 0, xi = 0;      // its tile ordinal and position in xorder
      uint32_t xc = 0;          // X loads issued (staging ring position)
      // issue X loads in (tile, first use) order up to tile ordinal `upto`;
      // without `block`, stop at the first staging slot not yet copied out
      auto x_next = [&](int upto, bool block) {
        while (xt < ntiles && xtl <= upto) {
          const uint32_t xs = xc % kXSlots, par = ((xc / kXSlots) & 1) ^ 1;
          if (!block && !mbar_test(&x_empty[xs], par)) return;
          mbar_wait(&x_empty[xs], par);
          tma_load_3d_elect(Xs + xs * kXPair, &tmX, &x_full[xs], kXPair, 0,
                            static_cast<int32_t>(xt * kEdges), 2 * sc.xorder[xi], stream);
          ++xc;
          if (++xi == sc.nx) xi = 0, xt += gridDim.x, ++xtl;
        }
      };
      int tl = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tl) {
        x_next(tl, false);
        for (int n = 0; n < sc.nwseq; ++n, ++wc) {
          const int2 w = s_wseq[n];
          const uint32_t ws = wc % kNWs;
          while (!mbar_test(&w_empty[ws], ((wc / kNWs) & 1) ^ 1)) x_next(tl + 1, false);
          TPT(0, 0, wc);
          tma_load_2d_pair_elect(Ws + ws * kWSlot, kWTile, &tmW, &w_full[ws],
                                 w.y >= 0 ? kWSlot : kWTile, w.x * 64, w.y >= 0 ? w.y * 64 : -1,
                                 keep);
          x_next(tl + 1, false);
        }
      }
      // X loads are only polled above (a blocking wait there could hold back
      // the W loads the MMA needs to free the slot); the rest go out now
      x_next(tl, true);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (whole warp, converged; elected lanes issue)
    {
      constexpr uint32_t idesc64 = idesc_bf16_f32(128, 64, false, /*B MN-major*/ true);
      constexpr uint32_t idesc128 = idesc_bf16_f32(128, 128, false, true);
      uint32_t gc = 0, wc = 0, xc = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (int gi = 0; gi < sc.ngroups; ++gi, ++gc) {
          const int f = s_grp[gi];
          const int jp = f & 15, mask = (f >> 4) & 3;
          const uint32_t ws = wc % kNWs;
          TPT(1, 0, gc);
          if ((f >> 7) & 1) mbar_wait(&w_full[ws], (wc / kNWs) & 1);
          TPT(1, 1, gc);
          const uint32_t vs = gc & 1;
          mbar_wait(&v_empty[vs], ((gc >> 1) & 1) ^ 1);
          TPT(1, 2, gc);
          if ((f >> 6) & 1) {  // first use of this pair in the tile: stage it into TMEM
            const uint32_t xs = xc % kXSlots;
            mbar_wait(&x_full[xs], (xc / kXSlots) & 1);
            tc_fence_after();
            const uint32_t x0 = smem_u32(Xs + xs * kXPair);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              tmem_cp_128x256b_elect(tmem + 32 * jp + 8 * kk,
                                     smem_desc(x0 + kk * 32, 16, 1024, kLayoutSW128));
            umma_commit_elect(&x_empty[xs]);  // staging slot reusable once copied
            ++xc;
          }
          tc_fence_after();
          const uint32_t d = tmem + kVBase + 128 * vs + (mask == 2 ? 64 : 0);
          const uint32_t w0 = smem_u32(Ws + ws * kWSlot) + (mask == 2 ? kWTile : 0);
          const uint32_t idesc = mask == 3 ? idesc128 : idesc64;
          const uint64_t bd = smem_desc(w0, kWTile, 1024, kLayoutSW128);
          umma_ts_k64_commit_elect(d, tmem + 32 * jp, bd, idesc, &v_full[vs]);
          TPT(1, 3, gc);
          if ((f >> 8) & 1) {
            umma_commit_elect(&w_empty[ws]);
            ++wc;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ consumers
    asm volatile("setmaxnreg.inc.sync.aligned.u32 104;");
    const int cw = warp - 4, h = cw >> 2, q = warp & 3, hf = q >> 1;
    const int ct = cw * 32 + lane;                  // consumer thread 0..511
    const int e = ((q & 1) << 5) | lane;            // edge of TMEM lane 32q + lane
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16) + kVBase;
    float4* zt = Ex + h * kExchF4;  // this warpgroup's Z staging tiles (2 x SW128, 8 KB each)
    const bool issuer = (cw & 3) == 0 && lane == 0;
    // Y: thread ct stages (edge ct % 64, k = 2 (ct / 64) + {0, 1}) of each tile,
    // loaded one tile ahead into one register
    const int ye = ct & (kEdges - 1), yk = (ct >> 6) * 2;
    auto ld_y = [&](int64_t tile) -> uint32_t {
      const int64_t b = tile * kEdges + ye;
      if (tile >= ntiles || b >= a.batch) return 0u;
      const uint16_t* yr = reinterpret_cast<const uint16_t*>(a.Y) + b * a.nk + yk;
      if (a.y_pair) return __ldg(reinterpret_cast<const uint32_t*>(yr));
      const uint32_t lo = yk < a.nk ? __ldg(yr) : 0u;
      const uint32_t hi = yk + 1 < a.nk ? __ldg(yr + 1) : 0u;
      return lo | (hi << 16);
    };
    uint32_t ynext = ld_y(blockIdx.x);
    uint32_t gc = 0;
    const int sh0 = 16 + 8 * hf + h;  // entry bit of (path 0, this half, this out row)
    int pcnt = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      named_bar_sync(1, 512);  // every warpgroup is done with the previous tile's Yk
      Yk[yk * kEdges + ye] = __uint_as_float(ynext << 16);
      Yk[(yk + 1) * kEdges + ye] = __uint_as_float(ynext & 0xFFFF0000u);
      ynext = ld_y(tile + gridDim.x);
      // This warpgroup's CG coefficients for pass Pn (its out row, both rows
      // of the pairs): Cf_h[c][edge] = sum_k v * Y[edge, k], computed by the
      // warpgroup alone (no cross-warpgroup barrier). Records of at most two
      // terms take the unrolled path, four coefficients in flight per thread.
      float* cfw = Cf + h * kMaxWgCoefs * kEdges;
      const int wt = (cw & 3) * 32 + lane, wte = wt & 63;
      auto coefs = [&](int Pn) {
        const int2 pw = s_pwg[Pn * 4 + h];
        const int n = (pw.y & 0xFFFF) + (pw.y >> 16);
        if (sc.two_terms) {
          for (int cb = wt >> 6; cb < n; cb += 8) {
            float4 rec[4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
              rec[u] = cb + 2 * u < n ? s_crec[pw.x + cb + 2 * u] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float y0 = Yk[__float_as_int(rec[u].x) * kEdges + wte];
              const float y1 = Yk[__float_as_int(rec[u].z) * kEdges + wte];
              if (cb + 2 * u < n) cfw[(cb + 2 * u) * kEdges + wte] = fmaf(rec[u].w, y1, rec[u].y * y0);
            }
          }
          return;
        }
        for (int c = wt >> 6; c < n; c += 2) {
          const uint32_t ref = s_cref[pw.x + c];
          float v = 0.f;
          for (int t = 0; t < static_cast<int>(ref >> 24); ++t) {
            const float2 term = s_terms[(ref & 0xFFFFFF) + t];
            v = fmaf(term.y, Yk[__float_as_int(term.x) * kEdges + wte], v);
          }
          cfw[c * kEdges + wte] = v;
        }
      };
      named_bar_sync(1, 512);  // Yk written (read only by coefficient passes of this tile)
      coefs(0);
      named_bar_sync(2 + h, 128);
      for (int P = 0; P < sc.npasses; ++P) {
        const int4 ps = s_pass[P];
        ++pcnt;
        const int2 pw = s_pwg[P * 4 + h];
        const float* cfp = cfw + (hf ? (pw.y & 0xFFFF) : 0) * kEdges + e;
        float2 acc[4][8];  // 64 columns of this (edge, row of the pair, out row) as pairs
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int qq = 0; qq < 8; ++qq) acc[c][qq] = make_float2(0.f, 0.f);
        for (int gi = ps.x; gi < ps.x + ps.y; ++gi, ++gc) {
          const int f = s_grp[gi];
          const int m = ((f >> sh0) & 1) | (((f >> (sh0 + 4)) & 1) << 1);  // paths with an entry
          const uint32_t vs = gc & 1;
          if (warp == 4 && lane == 0) TPT(2, 0, gc);
          mbar_wait(&v_full[vs], (gc >> 1) & 1);
          if (warp == 4 && lane == 0) TPT(2, 1, gc);
          tc_fence_after();
#pragma unroll
          for (int pi = 0; pi < 2; ++pi) {
            if (!((m >> pi) & 1)) continue;  // warp-uniform
            const float cf = *cfp;
            cfp += kEdges;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t v[16];
              tmem_ld_32x32b_x16(trow + 128 * vs + 64 * pi + 16 * c, v);
              tmem_ld_wait();
#pragma unroll
              for (int qq = 0; qq < 8; ++qq)
                acc[c][qq] = ffma2(cf, make_float2(__uint_as_float(v[2 * qq]),
                                                   __uint_as_float(v[2 * qq + 1])),
                                   acc[c][qq]);
            }
          }
          tc_fence_before();
          __syncwarp();
          if (warp == 4 && lane == 0) TPT(2, 2, gc);
          if (lane == 0) mbar_arrive(&v_empty[vs]);
        }
        const int out_i = static_cast<int16_t>(((h < 2 ? ps.z : ps.w) >> (16 * (h & 1))) & 0xFFFF);
        // The two rows of the pair meet in two [64 edges][32 columns] SW128
        // tiles (half 1 writes, half 0 adds), which one thread stores (or,
        // for +=, reduce-adds) to Z by TMA. The tiles were read by the
        // previous pass's stores long ago; the next pass's coefficients are
        // computed while these stores read them.
        if (out_i >= 0) {
          if (issuer) bulk_wait_group_read0();
          named_bar_sync(2 + h, 128);
          if (hf) {
#pragma unroll
            for (int c16 = 0; c16 < 16; ++c16) {  // 16-byte chunk c16 of the 64 columns
              const float2 x0 = acc[c16 >> 2][2 * (c16 & 3)];
              const float2 x1 = acc[c16 >> 2][2 * (c16 & 3) + 1];
              zt[(c16 >> 3) * 512 + e * 8 + ((c16 & 7) ^ (e & 7))] =
                  make_float4(x0.x, x0.y, x1.x, x1.y);
            }
          }
          named_bar_sync(2 + h, 128);
          if (!hf) {
#pragma unroll
            for (int c16 = 0; c16 < 16; ++c16) {
              const float2 x0 = acc[c16 >> 2][2 * (c16 & 3)];
              const float2 x1 = acc[c16 >> 2][2 * (c16 & 3) + 1];
              float4* t = zt + (c16 >> 3) * 512 + e * 8 + ((c16 & 7) ^ (e & 7));
              const float4 o = *t;
              *t = make_float4(x0.x + o.x, x0.y + o.y, x1.x + o.z, x1.y + o.w);
            }
          }
          fence_proxy_async_smem();
          named_bar_sync(2 + h, 128);
          if (issuer) {
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              if (a.accumulate)
                tma_reduce_add_3d(&tmZ, zt + half * 512, 32 * half, out_i,
                                  static_cast<int32_t>(tile * kEdges));
              else
                tma_store_3d(&tmZ, zt + half * 512, 32 * half, out_i,
                             static_cast<int32_t>(tile * kEdges));
            }
            bulk_commit_group();
          }
        }
        if (P + 1 < sc.npasses) {
          if (out_i < 0) named_bar_sync(2 + h, 128);  // (the exchange's barriers order it otherwise)
          coefs(P + 1);
          named_bar_sync(2 + h, 128);
        }
      }
    }
    if (issuer) bulk_wait_group0();
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
  std::unique_ptr<TpSched> sched;  // tensor-core schedule (kernel parameter)
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
      auto sc = std::make_unique<TpSched>();
      std::memset(sc.get(), 0, sizeof(TpSched));
      std::vector<int> grp;
      std::vector<uint32_t> cref;
      std::vector<float2> terms;
      std::vector<int2> wseq, pwg;
      std::vector<int4> pass;
      std::vector<int> xorder;
      uint32_t seen = 0;  // pairs already staged in this tile
      for (int64_t i0 = 0; i0 < ni && tc;) {
        // up to four output rows per pass, fewer if their coefficients overflow smem
        const int64_t ns = std::min<int64_t>(4, ni - i0);  // one out row per warpgroup
        int outs[4];
        for (int h = 0; h < 4; ++h) outs[h] = h < ns ? static_cast<int>(i0 + h) : -1;
        // paths feeding this pass and the input-row pairs each needs
        std::map<int, uint32_t> need;
        for (const auto& kv : ent) {
          const int l = std::get<0>(kv.first), i = std::get<1>(kv.first), j = std::get<2>(kv.first);
          if (i >= i0 && i < i0 + ns) need[l] |= 1u << (j / 2);
        }
        // paths with the same pair set side by side, then paired into W slots
        std::vector<std::pair<uint32_t, int>> order;
        for (const auto& kv : need) order.emplace_back(kv.second, kv.first);
        std::sort(order.begin(), order.end());
        const int g0 = static_cast<int>(grp.size());
        std::vector<uint32_t> crefh[8];  // this pass's coefficients, per (half, out row)
        const size_t step = std::getenv("IXB_TP_NOMERGE") ? 1 : 2;  // perf experiment
        for (size_t o = 0; o < order.size(); o += step) {
          const int la = order[o].second;
          const int lb = step == 2 && o + 1 < order.size() ? order[o + 1].second : -1;
          const uint32_t ma = order[o].first, mb = lb >= 0 ? order[o + 1].first : 0u;
          wseq.push_back(make_int2(la, lb));
          const int first = static_cast<int>(grp.size());
          for (int jp = 0; jp < kMaxPairs; ++jp) {
            const int mask = static_cast<int>(((ma >> jp) & 1) | (((mb >> jp) & 1) << 1));
            if (!mask) continue;
            int f = jp | (mask << 4);
            if (!((seen >> jp) & 1)) {
              f |= 1 << 6;
              xorder.push_back(jp);
            }
            seen |= 1u << jp;
            for (int hf = 0; hf < 2; ++hf)
              for (int pi = 0; pi < 2; ++pi)
                for (int sl4 = 0; sl4 < 4; ++sl4) {
                  const int l = pi ? lb : la, j = 2 * jp + hf;
                  if (l < 0 || outs[sl4] < 0 || !((mask >> pi) & 1)) continue;
                  auto it = ent.find(std::make_tuple(l, outs[sl4], j));
                  if (it == ent.end()) continue;
                  f |= 1 << (16 + 8 * hf + 4 * pi + sl4);
                  if (it->second.size() > 255) tc = false;
                  crefh[4 * hf + sl4].push_back(static_cast<uint32_t>(terms.size()) |
                                      (static_cast<uint32_t>(it->second.size()) << 24));
                  for (const auto& kvp : it->second) {
                    float kf;
                    std::memcpy(&kf, &kvp.first, sizeof kf);
                    terms.push_back(make_float2(kf, kvp.second));
                  }
                }
            grp.push_back(f);
          }
          grp[first] |= 1 << 7;
          grp.back() |= 1 << 8;
        }
        auto pk = [](int x, int y) {
          return static_cast<int>((static_cast<uint32_t>(x) & 0xFFFF) |
                                  ((static_cast<uint32_t>(y) & 0xFFFF) << 16));
        };
        pass.push_back(make_int4(g0, static_cast<int>(grp.size()) - g0, pk(outs[0], outs[1]),
                                 pk(outs[2], outs[3])));
        for (int h = 0; h < 4; ++h) {  // warpgroup h: its out row's lists, half 0 then half 1
          const size_t n0 = crefh[h].size(), n1 = crefh[4 + h].size();
          if (n0 + n1 > static_cast<size_t>(kMaxWgCoefs)) tc = false;
          pwg.push_back(make_int2(static_cast<int>(cref.size()),
                                  static_cast<int>(n0 | (n1 << 16))));
          cref.insert(cref.end(), crefh[h].begin(), crefh[h].end());
          cref.insert(cref.end(), crefh[4 + h].begin(), crefh[4 + h].end());
        }
        i0 += ns;
      }
      if (tc) {
        sc->npasses = static_cast<int>(pass.size());
        sc->ngroups = static_cast<int>(grp.size());
        sc->nwseq = grp.empty() ? 0 : static_cast<int>(wseq.size());
        sc->nx = static_cast<int>(xorder.size());
        std::copy(xorder.begin(), xorder.end(), sc->xorder);
        std::vector<char> blob;
        auto put = [&](const void* p, size_t n) {
          const int o = static_cast<int>(blob.size());
          blob.insert(blob.end(), static_cast<const char*>(p), static_cast<const char*>(p) + n);
          blob.resize((blob.size() + 15) / 16 * 16, 0);
          return o;
        };
        sc->o_pass = put(pass.data(), pass.size() * sizeof(int4));
        sc->o_pwg = put(pwg.data(), pwg.size() * sizeof(int2));
        sc->o_grp = put(grp.data(), grp.size() * sizeof(int));
        sc->o_cref = put(cref.data(), cref.size() * sizeof(uint32_t));
        sc->o_terms = put(terms.data(), terms.size() * sizeof(float2));
        sc->o_wseq = put(wseq.data(), wseq.size() * sizeof(int2));
        // fixed two-term records for the unrolled coefficient path
        std::vector<float4> crec(cref.size());
        sc->two_terms = 1;
        for (size_t c = 0; c < cref.size(); ++c) {
          const uint32_t cnt = cref[c] >> 24, off = cref[c] & 0xFFFFFF;
          if (cnt > 2) sc->two_terms = 0;
          float4 r = make_float4(terms[off].x, terms[off].y, terms[off].x, 0.f);
          if (cnt > 1) r.z = terms[off + 1].x, r.w = terms[off + 1].y;
          crec[c] = r;
        }
        sc->o_crec = put(crec.data(), crec.size() * sizeof(float4));
        sc->nbytes = static_cast<int>(blob.size());
        if (blob.size() > sizeof(sc->blob)) tc = false;  // larger tables: CUDA-core path
        else std::memcpy(sc->blob, blob.data(), blob.size());
      }
      if (tc) {
        plan->sched = std::move(sc);
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
      // Z viewed as (w, row, edge): a {32, 1, 64} box is one pass row's half
      const CUtensorMap tmZ = make_tmap_3d(Z, 64, static_cast<uint64_t>(p.ni),
                                           static_cast<uint64_t>(batch), 256, p.ni * 256, 32, 1,
                                           kEdges, CU_TENSOR_MAP_SWIZZLE_128B, /*f32=*/true);
      TpArgs args{static_cast<const __nv_bfloat16*>(Y), Z, batch, static_cast<int>(p.nk),
                  static_cast<int>(p.ni),
                  p.nk % 2 == 0 && reinterpret_cast<uintptr_t>(Y) % 4 == 0 ? 1 : 0, accumulate};
      set_max_dynamic_smem(reinterpret_cast<const void*>(tp_tc_kernel), kTpSmem,
                           "cudaFuncSetAttribute(tp_tc_kernel)");
      int64_t grid = ceil_div(batch, kEdges);
      if (grid > sm_count()) grid = sm_count();
      tp_tc_kernel<<<static_cast<unsigned>(grid), kTpThreads, kTpSmem, s>>>(tmX, tmW, tmZ, *p.sched,
                                                                             args);
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

#ifdef IXB_TP_TRACE
extern "C" int ixb_tp_trace_copy(void* host) {
  return cudaMemcpyFromSymbol(host, g_tp_trace, sizeof(g_tp_trace)) == cudaSuccess ? 0 : 1;
}
#endif

extern "C" int ixb_tp_plan_uses_tensor_cores(const ixb_tp_plan* plan) {
  return plan && plan->tc ? 1 : 0;
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
