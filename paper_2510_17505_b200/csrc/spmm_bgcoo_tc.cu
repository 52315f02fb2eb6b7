// K4 — BlockGroupCOO SpMM on tcgen05 / TMEM / TMA (sm_100a):
//   C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]   (corpus/structured_spmm.json:2)
// bf16 operands, fp32 accumulation in TMEM. Reference semantics: oracle
// plan.cpp:579-594 (vars p,bm,n,q,bk), plan executor plan.cpp:383-534.
//
// Formulation. bM = 16 is below the smallest UMMA M, so the
// block product is computed transposed, with the dense operand as the M side:
//     D^T[n, bm] += B_tile^T[n, bk] . AV_blk^T[bk, bm]
//   A operand = B[AK*16 : +16, n0 : n0+128]   (128 x 16, MN-major, SW128, TMA)
//   B operand = AV[p,q]                        (16 x 16,  K-major,  SW32,  TMA)
//   D         = TMEM, 128 lanes (n) x 16 columns (bm) per 128-wide n subtile.
// One UMMA M=128,N=16,K=16 per stored block and n subtile.
//
// Work split: static and balanced. CTA c of NC owns the group positions
// [G*c/NC, G*(c+1)/NC) (equal slot counts, so equal B-tile bytes and MMAs
// per CTA); rows crossing a range boundary are summed from per-CTA partials
// in CTA order by the last CTA to finish its part (no float atomics;
// deterministic for a given grid). Whole rows are written from TMEM.
// Warp roles (TcRoles): 4 epilogue warps (TMEM -> registers -> coalesced
// fp32 stores along n), a scheduler warp (range walk -> segment queue),
// NPROD TMA producer warps (stage batches round-robin) and NSUB UMMA issuer
// warps (one per 128-wide n subtile). A STAGES-deep full/empty mbarrier ring
// feeds the tensor core; accumulators are double buffered in TMEM so the
// epilogue of segment j overlaps the main loop of segment j+1.
#include <cudaTypedefs.h>

#include <climits>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.h"

namespace ixb {
namespace {

using namespace sm100;

#ifndef IXB_K4_SPS
#define IXB_K4_SPS 2
#endif
#ifndef IXB_K4_STAGES
#define IXB_K4_STAGES 3
#endif
#ifndef IXB_K4_NPROD
#define IXB_K4_NPROD 2
#endif
#ifndef IXB_K4_MINB
#define IXB_K4_MINB 2
#endif
constexpr int kSps = IXB_K4_SPS;

#ifdef IXB_K4_TRACE
// perf experiment: per-CTA globaltimer stamps of the pipeline's milestones
__device__ long long g_k4_trace[4096 * 16];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define K4TR(slot) (g_k4_trace[blockIdx.x * 16 + (slot)] = gtimer())
#define K4TR_FIRST(slot) \
  do { if (!g_k4_trace[blockIdx.x * 16 + (slot)]) K4TR(slot); } while (0)
#define K4TR_SET(slot, v) (g_k4_trace[blockIdx.x * 16 + (slot)] = (v))
#else
#define K4TR(slot) ((void)0)
#define K4TR_FIRST(slot) ((void)0)
#define K4TR_SET(slot, v) ((void)0)
#endif

constexpr uint32_t kAvBytes = 16 * 16 * 2;
constexpr uint32_t kSubBytes = 16 * 128 * 2;  // one 128-wide n subtile of a B tile

struct TcArgs {
  const int32_t* AM;
  const int32_t* AK;
  float* C;
  int64_t G, g, KB, N, MB;
  int ntiles;   // n tiles of 128*NSUB columns
  int accumulate;
  int check;
  int epi_sleep_ns;  // epilogue warps back off instead of spinning on acc_full
  float* part;       // [grid][2][16][N] partial block-rows of rows split across CTAs
  unsigned* rowctr;  // [grid * ntiles] arrival counters of split rows (zero, self-resetting)
  ErrorRecord* err;
};

// Warp roles. Issue cost on sm_100a is per issuing warp (a UMMA or TMA
// occupies its warp for ~130-240 cycles however small it is,
// profiles/k4_diag_r2.md §1), so the small M=128, N=16 block MMAs are spread
// over NSUB issuer warps (one per 128-wide n subtile) and the TMA boxes over
// NPROD producer warps; the tensor pipe saturates from ~4 issue streams/SM.
template <int NSUB, int NPROD>
struct TcRoles {
  static constexpr int kEpi = 4;              // warps 0..3: epilogue (TMEM lane quarters)
  static constexpr int kSched = 4;            // segment scheduler
  static constexpr int kProd0 = 5;            // producers kProd0 .. kProd0+NPROD-1
  static constexpr int kIss0 = 5 + NPROD;     // issuers (sub) kIss0 .. kIss0+NSUB-1
  static constexpr int kWarps = 5 + NPROD + NSUB;
  static constexpr int kThreads = kWarps * 32;
};

// A stage carries up to SPS consecutive slots of one row segment: SPS B tiles
// (the whole 128*NSUB-column n tile of 16 rows, one TMA box each), then the
// SPS AV blocks (one TMA box for all of them: a segment's slots are
// contiguous in AV).
template <int NSUB, int STAGES, int SPS>
struct TcSmem {
  static constexpr uint32_t kBBytes = NSUB * kSubBytes;
  static constexpr uint32_t kStageBytes = ((SPS * (kBBytes + kAvBytes) + 1023) / 1024) * 1024;
  static constexpr uint32_t kTileBytes = STAGES * kStageBytes;
  static constexpr uint32_t kTotal = kTileBytes + 1024 /*barriers+queue*/ + 1024 /*align*/;
};

// Static balanced schedule. CTA c owns the group positions
// [G*c/NC, G*(c+1)/NC) of the (row-sorted) format — equal slot counts, so
// equal B-tile bytes and MMAs per CTA and per SM. A row (run of equal AM)
// that crosses a range boundary is split: each CTA accumulates its part in
// TMEM, stores it as a partial block-row, and the last CTA to arrive sums
// the partials in CTA order (fixed order: deterministic for a given grid).
// Whole rows — the common case — are written straight from TMEM.
__device__ __forceinline__ int64_t range_lo(int64_t G, int64_t nc, int64_t c) {
  return G * c / nc;
}
// CTA whose range holds group position p
__device__ __forceinline__ int owner_cta(int64_t G, int64_t nc, int64_t p) {
  return static_cast<int>(((p + 1) * nc + G - 1) / G - 1);
}
// First position >= p (< lim) whose AM differs from `row` (warp-collective).
__device__ __forceinline__ int64_t run_end(const int32_t* AM, int64_t p, int64_t lim, int row) {
  const int lane = threadIdx.x & 31;
  for (;; p += 32) {
    const int64_t q = p + lane;
    const unsigned m = __ballot_sync(0xffffffffu, q >= lim || __ldg(AM + q) != row);
    if (m) return p + __ffs(m) - 1;
  }
}
// First position of the run of `row` that contains position p (warp-collective).
__device__ __forceinline__ int64_t run_start(const int32_t* AM, int64_t p, int row) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const int64_t q = p - 1 - lane;  // p-1, p-2, ...
    const unsigned m = __ballot_sync(0xffffffffu, q < 0 || __ldg(AM + q) != row);
    if (m) return p - (__ffs(m) - 1);
    p -= 32;
  }
}

constexpr int kQN = 16;  // segment queue depth (scheduler -> roles)

template <int NSUB, int STAGES, int NACC, int SPS, int NPROD, int MINB = 1>
__global__ void __launch_bounds__(TcRoles<NSUB, NPROD>::kThreads, MINB)
    bgcoo_tc_kernel(const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmAV, TcArgs a) {
  using L = TcSmem<NSUB, STAGES, SPS>;
  using R = TcRoles<NSUB, NPROD>;
  static_assert(32 % SPS == 0, "a stage batch never straddles a 32-slot AK chunk");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* tiles = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kTileBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + NACC;
  uint64_t* seg_full = acc_empty + NACC;
  uint64_t* seg_empty = seg_full + kQN;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(seg_empty + kQN);
  int4* segq = reinterpret_cast<int4*>(tmem_base_slot + 4);  // {s, e, row, prev}
  int4* segq2 = segq + kQN;                                   // {tile, c0, c1, split}
  int* epi_flag = reinterpret_cast<int*>(segq2 + kQN);        // split-row combine: last arriver

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) K4TR(0);
  constexpr uint32_t kAccCols = 16 * NSUB;  // one accumulator buffer
  constexpr uint32_t kTmemCols = NACC * kAccCols <= 32    ? 32
                                 : NACC * kAccCols <= 64  ? 64
                                 : NACC * kAccCols <= 128 ? 128
                                 : NACC * kAccCols <= 256 ? 256
                                                          : 512;

  if (warp == R::kSched) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], NSUB);  // every issuer commits the stage
      }
      for (int b = 0; b < NACC; ++b) {
        mbar_init(&acc_full[b], NSUB);
        mbar_init(&acc_empty[b], R::kEpi);
      }
      for (int q = 0; q < kQN; ++q) {
        mbar_init(&seg_full[q], 1);
        mbar_init(&seg_empty[q], NPROD + NSUB + R::kEpi);
      }
      fence_barrier_init();
    }
  } else if (warp == R::kIss0) {
    tmem_alloc(tmem_base_slot, kTmemCols);
    tmem_relinquish();
  } else if (warp == R::kProd0 && lane == 0) {
    tma_prefetch_desc(&tmB);
    tma_prefetch_desc(&tmAV);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;
  if (threadIdx.x == 0) K4TR(1);

  // Segment queue consumers: entry q holds {s, e, row, prev} + {n tile, c0,
  // c1, split}; s < 0 ends.
  int4 sg2;
  auto pop = [&](int j, int4& sg, int& tile) {
    const int q = j % kQN;
    mbar_wait(&seg_full[q], (j / kQN) & 1);
    sg = segq[q];
    sg2 = segq2[q];
    tile = sg2.x;
  };
  auto release = [&](int j) { mbar_arrive(&seg_empty[j % kQN]); };

  if (warp == R::kSched) {
    // ---------------------------------------------------------- scheduler
    // Walks this CTA's range and queues its segments (row runs clipped to
    // the range) ahead of the pipeline, so no role stalls on the dependent
    // AM loads between segments.
    const int64_t nc = gridDim.x;
    const int64_t lo = range_lo(a.G, nc, blockIdx.x), hi = range_lo(a.G, nc, blockIdx.x + 1);
    int j = 0;
    auto push = [&](int4 v, int4 v2) {
      const int q = j % kQN;
      if (lane == 0) {
        mbar_wait(&seg_empty[q], ((j / kQN) & 1) ^ 1);
        segq[q] = v;
        segq2[q] = v2;
        mbar_arrive(&seg_full[q]);
        if (v.x >= 0) K4TR_FIRST(2); else K4TR(3);
      }
      __syncwarp();
      ++j;
    };
    // Order: the segment at lo, then the trailing segment when its row
    // continues past hi, then the whole rows between. Both split rows of
    // the range are thus finished (partials stored, combined by whichever
    // CTA arrives last) early, behind the MMAs of the whole rows, instead of
    // at the end of the kernel.
    auto seg = [&](int tile, int64_t s, int64_t e, int row, int64_t rs, int64_t re) {
      const int prev = rs == s ? (s > 0 ? __ldg(a.AM + s - 1) : -1) : row;
      push(make_int4(static_cast<int>(s), static_cast<int>(e), row, prev),
           make_int4(tile, owner_cta(a.G, nc, rs), owner_cta(a.G, nc, re - 1),
                     rs < lo || re > hi));
    };
    // The two boundary segments come from 32-position windows around lo and
    // hi, loaded together (one dependent round trip instead of a chain of
    // ballot scans; the scans remain the fallback for longer runs).
    const int64_t w0 = lo - 32 + lane, w1 = lo + lane, w2 = hi - 32 + lane, w3 = hi + lane;
    const int a0 = w0 >= 0 ? __ldg(a.AM + w0) : INT_MIN;
    const int a1 = w1 < a.G ? __ldg(a.AM + w1) : INT_MAX;
    const int a2 = w2 >= 0 ? __ldg(a.AM + w2) : INT_MIN;
    const int a3 = w3 < a.G ? __ldg(a.AM + w3) : INT_MAX;
    const int row0 = __shfl_sync(0xffffffffu, a1, 0);
    int64_t rs0, re0;
    {
      const unsigned mb = __ballot_sync(0xffffffffu, a0 != row0);
      rs0 = mb ? lo - 32 + (32 - __clz(mb)) : run_start(a.AM, lo - 32, row0);
      const unsigned ma = __ballot_sync(0xffffffffu, lane >= 1 && a1 != row0);
      re0 = ma ? lo + __ffs(ma) - 1 : run_end(a.AM, lo + 32, a.G, row0);
    }
    const int64_t e0 = re0 < hi ? re0 : hi;
    int64_t ts = -1, te = -1;  // trailing segment [ts, hi) of a row continuing past hi
    const int rowt = __shfl_sync(0xffffffffu, a2, 31);
    if (e0 < hi && hi < a.G && __shfl_sync(0xffffffffu, a3, 0) == rowt) {
      const unsigned mb = __ballot_sync(0xffffffffu, a2 != rowt);
      ts = mb ? hi - 32 + (32 - __clz(mb)) : run_start(a.AM, hi - 32, rowt);
      const unsigned ma = __ballot_sync(0xffffffffu, lane >= 1 && a3 != rowt);
      te = ma ? hi + __ffs(ma) - 1 : run_end(a.AM, hi + 32, a.G, rowt);
    }
    for (int tile = 0; tile < a.ntiles; ++tile) {
      seg(tile, lo, e0, row0, rs0, re0);
      int64_t mid_end = hi;
      if (ts >= 0) {
        seg(tile, ts, hi, rowt, ts, te);
        mid_end = ts;
      }
      for (int64_t p = e0; p < mid_end;) {
        const int row = __ldg(a.AM + p);
        const int64_t re = run_end(a.AM, p + 1, mid_end, row);
        seg(tile, p, re, row, p, re);
        p = re;
      }
    }
    push(make_int4(-1, -1, 0, 0), make_int4(0, 0, 0, 0));
  } else if (warp >= R::kProd0 && warp < R::kProd0 + NPROD) {
    // ---------------------------------------------------------- TMA producers
    // Producer p issues the stage batches bc with bc % NPROD == p.
    const int p = warp - R::kProd0;
    const uint64_t keep = l2_evict_last();    // dense operand: re-read by many blocks
    const uint64_t stream = l2_evict_first();  // format: read once
    int64_t bc = 0;                            // stage batches walked (all producers)
    // Early start: the first segment always begins at this CTA's range start
    // lo (tile 0), and a group holds g >= (NPROD + 1) * SPS slots, so batch p
    // (slots lo*g + p*SPS ...) is known before the scheduler's first push.
    const int64_t lo0 = range_lo(a.G, gridDim.x, blockIdx.x);
    const bool early = a.g >= static_cast<int64_t>((NPROD + 1) * SPS) &&
                       lo0 < range_lo(a.G, gridDim.x, blockIdx.x + 1);
    if (early) {
      const int64_t slot0 = lo0 * a.g + static_cast<int64_t>(p) * SPS;
      int k = 0;
      if (lane < SPS) {
        k = __ldg(a.AK + slot0 + lane);
        if (k < 0 || static_cast<int64_t>(k) >= a.KB) {
          if (a.check) report_index_error(a.err, 0, slot0 + lane, k);
          k = 0;
        }
      }
      int kk[SPS];
#pragma unroll
      for (int b = 0; b < SPS; ++b) kk[b] = __shfl_sync(0xffffffffu, k, b);
      const int stage = p % STAGES;  // batch p, first use of its stage
      if (elect_one_sync()) {
        uint8_t* st = tiles + stage * L::kStageBytes;
        mbar_arrive_expect_tx(&full[stage], SPS * L::kBBytes + SPS * kAvBytes);
#pragma unroll
        for (int b = 0; b < SPS; ++b)
          tma_load_3d(st + b * L::kBBytes, &tmB, &full[stage], 0, kk[b] * 16, 0, keep);
        tma_load_2d(st + SPS * L::kBBytes, &tmAV, &full[stage], 0,
                    static_cast<int32_t>(slot0 * 16), stream);
      }
    }
    for (int j = 0;; ++j) {
      int4 sg;
      int tile;
      pop(j, sg, tile);
      if (sg.x < 0) break;
      const int n0 = tile * 128 * NSUB;
      const int64_t s0 = static_cast<int64_t>(sg.x) * a.g, s1 = static_cast<int64_t>(sg.y) * a.g;
      auto load_k = [&](int64_t i0) {
        const int64_t slot = i0 + lane;
        int k = 0;
        if (slot < s1) {
          k = __ldg(a.AK + slot);
          if (k < 0 || static_cast<int64_t>(k) >= a.KB) {
            if (a.check) report_index_error(a.err, 0, slot, k);
            k = 0;
          }
        }
        return k;
      };
      int k = load_k(s0);
      for (int64_t i0 = s0; i0 < s1; i0 += 32) {
        const int k_next = load_k(i0 + 32);  // prefetch the next 32 member coords
        const int cnt = static_cast<int>(s1 - i0 < 32 ? s1 - i0 : 32);
        for (int t = 0; t < cnt; t += SPS, ++bc) {
          if (static_cast<int>(bc % NPROD) != p) continue;
          if (early && bc < NPROD) continue;  // issued before the first pop
          const int nb = cnt - t < SPS ? cnt - t : SPS;
          int kk[SPS];
#pragma unroll
          for (int b = 0; b < SPS; ++b) kk[b] = __shfl_sync(0xffffffffu, k, (t + b) & 31);
          const int stage = static_cast<int>(bc % STAGES);
          const uint32_t phase = static_cast<uint32_t>((bc / STAGES) & 1);
          mbar_wait(&empty[stage], phase ^ 1);
          if (elect_one_sync()) {
            uint8_t* st = tiles + stage * L::kStageBytes;
            mbar_arrive_expect_tx(&full[stage], nb * L::kBBytes + SPS * kAvBytes);
#pragma unroll
            for (int b = 0; b < SPS; ++b) {
              if (b >= nb) break;
              // one 3-D box {64 n, 16 rows, 2*NSUB atoms} lands as [atom][row][64]
              tma_load_3d(st + b * L::kBBytes, &tmB, &full[stage], 0, kk[b] * 16, n0 / 64, keep);
            }
            // the SPS AV blocks in one box (rows past the format are zero-filled)
            tma_load_2d(st + SPS * L::kBBytes, &tmAV, &full[stage], 0,
                        static_cast<int32_t>((i0 + t) * 16), stream);
            if (p == 0) { K4TR_FIRST(4); K4TR(5); }
          }
        }
        k = k_next;
      }
      __syncwarp();
      if (lane == 0) release(j);
    }
  } else if (warp >= R::kIss0) {
    // ---------------------------------------------------------- UMMA issuers
    // Issuer `sub` owns n subtile sub of every block: D columns sub*16.
    const int sub = warp - R::kIss0;
    constexpr uint32_t idesc = idesc_bf16_f32(128, 16, /*A MN-major*/ true, /*B K-major*/ false);
    int64_t bc = 0;  // stage batches consumed (lane 0)
    // Early start (the producers' first NPROD batches, see there): the first
    // segment's first batches go to accumulator 0 before the first pop.
    const bool early = a.g >= static_cast<int64_t>((NPROD + 1) * SPS) &&
                       range_lo(a.G, gridDim.x, blockIdx.x) <
                           range_lo(a.G, gridDim.x, blockIdx.x + 1);
    if (early) {
      mbar_wait(&acc_empty[0], 1);  // fresh barrier: passes
      tc_fence_after();
      const uint32_t d = tmem_base + sub * 16;
      for (int e = 0; e < NPROD; ++e) {
        const int stage = e % STAGES;
        mbar_wait(&full[stage], 0);
        tc_fence_after();
        const uint32_t st = smem_u32(tiles + stage * L::kStageBytes);
#pragma unroll
        for (int b = 0; b < SPS; ++b) {
          const uint64_t bdesc =
              smem_desc(st + SPS * L::kBBytes + b * kAvBytes, 16, 256, kLayoutSW32);
          const uint64_t adesc =
              smem_desc(st + b * L::kBBytes + sub * kSubBytes, 2048, 1024, kLayoutSW128);
          umma_f16_elect(d, adesc, bdesc, idesc, (e > 0 || b > 0) ? 1u : 0u);
        }
        umma_commit_elect(&empty[stage]);
      }
    }
    for (int j = 0;; ++j) {
      int4 sg;
      int tile;
      pop(j, sg, tile);
      if (sg.x < 0) break;
      const int buf = j % NACC;
      // the whole warp walks the batches; one elected lane issues
      if (!(early && j == 0)) mbar_wait(&acc_empty[buf], ((j / NACC) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + buf * kAccCols + sub * 16;
      const int64_t nslots = (static_cast<int64_t>(sg.y) - sg.x) * a.g;
      // same (32-slot chunk, SPS batch) partition as the producers
      for (int64_t i0 = 0; i0 < nslots; i0 += 32) {
        const int cnt = static_cast<int>(nslots - i0 < 32 ? nslots - i0 : 32);
        for (int t = 0; t < cnt; t += SPS, ++bc) {
          if (early && bc < NPROD) continue;  // issued before the first pop
          const int nb = cnt - t < SPS ? cnt - t : SPS;
          const int stage = static_cast<int>(bc % STAGES);
          mbar_wait(&full[stage], static_cast<uint32_t>((bc / STAGES) & 1));
          tc_fence_after();
          const uint32_t st = smem_u32(tiles + stage * L::kStageBytes);
#pragma unroll
          for (int b = 0; b < SPS; ++b) {
            if (b >= nb) break;
            const uint64_t bdesc =
                smem_desc(st + SPS * L::kBBytes + b * kAvBytes, 16, 256, kLayoutSW32);
            // A: MN atoms (64 n) at +2048, K groups of 8 rows at +1024
            const uint64_t adesc =
                smem_desc(st + b * L::kBBytes + sub * kSubBytes, 2048, 1024, kLayoutSW128);
            umma_f16_elect(d, adesc, bdesc, idesc, (i0 + t + b) > 0 ? 1u : 0u);
          }
          umma_commit_elect(&empty[stage]);  // stage reusable once these UMMAs retire
          if (i0 + t + nb == nslots) umma_commit_elect(&acc_full[buf]);
          if (sub == 0 && lane == 0) { K4TR_FIRST(6); K4TR(7); K4TR_SET(12, bc + 1); }
        }
      }
      __syncwarp();
      if (lane == 0) release(j);
    }
  } else {
    // ---------------------------------------------------------- epilogue
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
    const int nloc = quarter * 32 + lane;
    for (int j = 0;; ++j) {
      int4 sg;
      int tile;
      pop(j, sg, tile);
      if (sg.x < 0) break;
      const int buf = j % NACC;
      const int row = sg.z;
      const int n0 = tile * 128 * NSUB;
      const bool row_ok = row >= 0 && static_cast<int64_t>(row) < a.MB;
      const bool split = sg2.w && row_ok;
      const int c0 = sg2.y, c1 = sg2.z;
      // a split row's partial: slot 1 for the row's first CTA (its last row), else 0
      float* mypart = a.part + (static_cast<int64_t>(blockIdx.x) * 2 +
                                (static_cast<int>(blockIdx.x) == c0 ? 1 : 0)) * 16 * a.N;
      mbar_wait_backoff(&acc_full[buf], (j / NACC) & 1, a.epi_sleep_ns);
      tc_fence_after();
#pragma unroll 1
      for (int sub = 0; sub < NSUB; ++sub) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                               buf * kAccCols + sub * 16,
                           r);
        tmem_ld_wait();
        if (sub == NSUB - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[buf]);  // TMEM buffer free for segment j+NACC
        }
        const int64_t col = n0 + sub * 128 + nloc;
        if (split) {
#pragma unroll
          for (int bm = 0; bm < 16; ++bm) __stcg(mypart + bm * a.N + col, __uint_as_float(r[bm]));
        } else if (row_ok) {
          float* c = a.C + static_cast<int64_t>(row) * 16 * a.N + col;
#pragma unroll
          for (int bm = 0; bm < 16; ++bm) {
            float v = __uint_as_float(r[bm]);
            if (a.accumulate) v += c[static_cast<int64_t>(bm) * a.N];
            __stcs(c + static_cast<int64_t>(bm) * a.N, v);
          }
        }
      }
      if (split) {
        // arrive on the row's counter; the last of the c1-c0+1 CTAs sums the
        // partials in CTA order: C = (C or 0) + P[c0] + ... + P[c1]
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 0 && lane == 0) {
          unsigned* ctr = a.rowctr + static_cast<int64_t>(c0) * a.ntiles + tile;
          const unsigned old = atomicAdd(ctr, 1u);
          const int last = old == static_cast<unsigned>(c1 - c0);
          if (last) *ctr = 0;  // reset for the next launch
          *epi_flag = last;
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (*epi_flag) {
          __threadfence();
#pragma unroll 1
          for (int sub = 0; sub < NSUB; ++sub) {
            const int64_t col = n0 + sub * 128 + nloc;
            float* c = a.C + static_cast<int64_t>(row) * 16 * a.N + col;
            float v[16];
#pragma unroll
            for (int bm = 0; bm < 16; ++bm) v[bm] = a.accumulate ? c[bm * a.N] : 0.f;
            auto part_at = [&](int cc) {
              return a.part + (static_cast<int64_t>(cc) * 2 + (cc == c0 ? 1 : 0)) * 16 * a.N + col;
            };
            int cc = c0;
            for (; cc + 1 <= c1; cc += 2) {  // two partials' loads in flight, adds in CTA order
              const float* p0 = part_at(cc);
              const float* p1 = part_at(cc + 1);
              float x0[16], x1[16];
#pragma unroll
              for (int bm = 0; bm < 16; ++bm) x0[bm] = __ldcg(p0 + bm * a.N);
#pragma unroll
              for (int bm = 0; bm < 16; ++bm) x1[bm] = __ldcg(p1 + bm * a.N);
#pragma unroll
              for (int bm = 0; bm < 16; ++bm) v[bm] = (v[bm] + x0[bm]) + x1[bm];
            }
            if (cc == c1) {
              const float* p0 = part_at(cc);
#pragma unroll
              for (int bm = 0; bm < 16; ++bm) v[bm] += __ldcg(p0 + bm * a.N);
            }
#pragma unroll
            for (int bm = 0; bm < 16; ++bm) __stcs(c + bm * a.N, v[bm]);
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");  // epi_flag reused by the next split row
      }
      if (warp == 0 && lane == 0) { K4TR_FIRST(8); K4TR(9); K4TR_SET(11, j + 1); }
      if (!row_ok && a.check && warp == 0 && lane == 0 && tile == 0) {
        report_index_error(a.err, 1, sg.x, row);
      }
      if (!a.accumulate) {
        // `=`: zero the empty block-rows before this segment (and after the last)
        const int64_t z0 = sg.w + 1 < 0 ? 0 : sg.w + 1;
        const int64_t z1 = row < 0 ? 0 : (row > a.MB ? a.MB : row);
        const bool last = sg.y == a.G;
        for (int pass = 0; pass < 2; ++pass) {
          const int64_t r0 = pass == 0 ? z0 : (row + 1 < 0 ? 0 : row + 1);
          const int64_t r1 = pass == 0 ? z1 : (last ? a.MB : 0);
          for (int64_t br = r0; br < r1; ++br) {
            for (int sub = 0; sub < NSUB; ++sub) {
              float* c = a.C + br * 16 * a.N + n0 + sub * 128 + nloc;
#pragma unroll
              for (int bm = 0; bm < 16; ++bm) c[static_cast<int64_t>(bm) * a.N] = 0.f;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) release(j);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == R::kIss0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
  if (threadIdx.x == 0) K4TR(10);
}

// ----------------------------------------------------- CUDA-core fallback
// Any bm/bk/N: CTA per (group position chunk of 1) handles segment starts;
// thread (bm, n) accumulates over the segment's blocks in slot order.
__global__ void bgcoo_simt_kernel(const int32_t* AM, const int32_t* AK,
                                  const __nv_bfloat16* AV, const __nv_bfloat16* B, float* C,
                                  int64_t G, int64_t g, int64_t bm, int64_t bk, int64_t KB,
                                  int64_t N, int64_t MB, int accumulate, int check,
                                  ErrorRecord* err) {
  const int64_t p = blockIdx.x;
  if (p >= G) return;
  const int row = AM[p];
  if (p > 0 && AM[p - 1] == row) return;  // not a segment start
  int64_t e = p + 1;
  while (e < G && AM[e] == row) ++e;
  const int prev = p > 0 ? AM[p - 1] : -1;
  const bool row_ok = row >= 0 && row < MB;
  if (!accumulate) {
    const int64_t z0 = prev + 1 < 0 ? 0 : prev + 1;
    const int64_t z1 = row < 0 ? 0 : (row > MB ? MB : row);
    for (int64_t i = z0 * bm * N + threadIdx.x; i < z1 * bm * N; i += blockDim.x) C[i] = 0.f;
    if (e == G) {
      const int64_t r0 = row + 1 < 0 ? 0 : row + 1;
      for (int64_t i = r0 * bm * N + threadIdx.x; i < MB * bm * N; i += blockDim.x) C[i] = 0.f;
    }
  }
  if (!row_ok) {
    if (check && threadIdx.x == 0) report_index_error(err, 1, p, row);
  }
  for (int64_t o = threadIdx.x; o < bm * N; o += blockDim.x) {
    const int64_t i = o / N, n = o % N;
    float acc = 0.f;
    for (int64_t slot = p * g; slot < e * g; ++slot) {
      const int k = AK[slot];
      if (k < 0 || k >= KB) {
        if (check) report_index_error(err, 0, slot, k);
        continue;
      }
      const __nv_bfloat16* av = AV + slot * bm * bk + i * bk;
      const __nv_bfloat16* b = B + static_cast<int64_t>(k) * bk * N + n;
      for (int64_t t = 0; t < bk; ++t) {
        acc = fmaf(__bfloat162float(av[t]), __bfloat162float(b[t * N]), acc);
      }
    }
    if (row_ok) {
      float* c = C + (static_cast<int64_t>(row) * bm + i) * N + n;
      *c = accumulate ? *c + acc : acc;
    }
  }
}

// ------------------------------------------------------------ host side
template <int NSUB, int STAGES, int NACC, int SPS, int NPROD, int MINB = 1>
void launch_tc(const CUtensorMap& tmB, const CUtensorMap& tmAV, TcArgs a, cudaStream_t s) {
  using L = TcSmem<NSUB, STAGES, SPS>;
  using R = TcRoles<NSUB, NPROD>;
  auto kern = bgcoo_tc_kernel<NSUB, STAGES, NACC, SPS, NPROD, MINB>;
  set_max_dynamic_smem(reinterpret_cast<const void*>(kern), L::kTotal,
                       "cudaFuncSetAttribute(bgcoo_tc_kernel)");
  // resident CTAs per SM (registers, smem and TMEM columns): a property of the
  // compiled kernel, the same on every sm_100a device
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncAttributes fa;
    IXB_CUDA_CHECK(cudaFuncGetAttributes(&fa, kern));
    const int by_regs = 65536 / (((fa.numRegs * 32 + 255) / 256) * 256 * R::kWarps);
    int n = static_cast<int>((220u * 1024u) / L::kTotal);
    if (n > by_regs) n = by_regs;
    if (n > 2048 / R::kThreads) n = 2048 / R::kThreads;
    constexpr int kCols = NACC * 16 * NSUB <= 32 ? 32 : NACC * 16 * NSUB <= 64 ? 64
                          : NACC * 16 * NSUB <= 128 ? 128 : NACC * 16 * NSUB <= 256 ? 256 : 512;
    if (n > 512 / kCols) n = 512 / kCols;  // a CTA must not wait in tcgen05.alloc
    per_sm = n < 1 ? 1 : n;
  }
  a.ntiles = static_cast<int>(a.N / (128 * NSUB));
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;  // every CTA resident
  if (const char* w = std::getenv("IXB_K4_WAVES")) grid *= std::atoi(w);  // perf experiment
  if (grid > a.G) grid = a.G;
  a.rowctr = work_counters(s, static_cast<size_t>(grid) * a.ntiles);
  const size_t part_n = static_cast<size_t>(grid) * 2 * 16 * a.N;
  a.part = static_cast<float*>(stream_buffer(s, part_n * sizeof(float), kBufK4Partials));
  Scratch<float> part_graph;  // first use inside a graph capture
  if (!a.part) {
    part_graph = Scratch<float>(part_n, s);
    a.part = part_graph.p;
  }
  kern<<<static_cast<unsigned>(grid), R::kThreads, L::kTotal, s>>>(tmB, tmAV, a);
  IXB_LAUNCH_CHECK("bgcoo_tc_kernel");
}

}  // namespace

void spmm_blockgroupcoo(const int32_t* AM, const int32_t* AK, const void* AV, int64_t G,
                        int64_t g, int64_t bm, int64_t bk, const void* B, int64_t KB, int64_t N,
                        float* C, int64_t MB, int accumulate, int flags, cudaStream_t s) {
  if (G < 0 || g < 1 || bm < 1 || bk < 1 || KB < 0 || N < 0 || MB < 0)
    fail(IXB_SHAPE, "ixb_spmm_blockgroupcoo: bad extents");
  const bool check = !(flags & IXB_UNCHECKED);
  if (N == 0 || MB == 0) return;
  if (G == 0) {
    if (!accumulate) IXB_CUDA_CHECK(cudaMemsetAsync(C, 0, MB * bm * N * sizeof(float), s));
    return;
  }
  if (G * g * bk > INT32_MAX || KB * bk > INT32_MAX) fail(IXB_SHAPE, "format exceeds 2^31 rows");
  // Unsorted group coordinates: validate the original arrays (K8), then
  // evaluate over a stably sorted copy of the format (rows of AK/AV gathered
  // by the permutation), which keeps every output row's summation order.
  Scratch<int32_t> am_sorted, perm, ak_sorted;
  Scratch<__nv_bfloat16> av_sorted;
  if (!(flags & IXB_GROUPS_SORTED) && !groups_sorted(AM, G, s)) {
    if (check) {
      validate_range(AK, G * g, KB, 0, s);
      validate_range(AM, G, MB, 1, s);
      OperandInfo ops[2] = {{"AK", "B", 0, KB, AK, G * g}, {"AM", "C", 0, MB, AM, G}};
      check_error_record(s, ops, 2);
    }
    sort_groups(AM, G, s, am_sorted, perm);
    ak_sorted = Scratch<int32_t>(G * g, s);
    av_sorted = Scratch<__nv_bfloat16>(G * g * bm * bk, s);
    gather_rows(perm.p, AK, ak_sorted.p, G, g * 4, s);
    gather_rows(perm.p, AV, av_sorted.p, G, g * bm * bk * 2, s);
    AM = am_sorted.p;
    AK = ak_sorted.p;
    AV = av_sorted.p;
    flags |= IXB_UNCHECKED;
  }
  const bool check2 = !(flags & IXB_UNCHECKED);
  ErrorRecord* err = device_error_record();
  const bool tc_ok = bm == 16 && bk == 16 && N % 128 == 0 &&
                     reinterpret_cast<uintptr_t>(B) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(AV) % 16 == 0;
  if (tc_ok) {
    TcArgs a;
    a.AM = AM;
    a.AK = AK;
    a.C = C;
    a.G = G;
    a.g = g;
    a.KB = KB;
    a.N = N;
    a.MB = MB;
    a.accumulate = accumulate;
    a.check = check2;
    a.err = err;
#ifndef IXB_K4_NSUB
#define IXB_K4_NSUB 4
#endif
    const int nsub = N % (128 * IXB_K4_NSUB) == 0 ? IXB_K4_NSUB : N % 256 == 0 ? 2 : 1;
    // B viewed as {64 n, rows, N/64 atoms}: one TMA box = the whole n tile of
    // 16 rows, landing as [atom][row][64] (the MN-major SW128 canonical layout)
    const CUtensorMap tmB = make_tmap_3d(B, 64, KB * 16, N / 64, N * 2, 128, 64, 16, 2 * nsub,
                                        CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tmAV = make_tmap_2d(AV, 16, G * g * 16, 32, 16, 16 * kSps,
                                         CU_TENSOR_MAP_SWIZZLE_32B);
    a.epi_sleep_ns = 256;  // back-off of the idle epilogue warps' barrier polls
    // 2 slots per stage, 4 stages: ~68 KB -> 3 CTAs (3 independent issue
    // streams) per SM; measured against 1, 4, 8, 12 slots per stage and
    // 1-5 CTAs/SM on cfg2 (profiles/k4_diag_r1.md), and against a panel
    // kernel with B-tile reuse across block rows (profiles/k4_diag_r2.md)
    if (nsub == 1) launch_tc<1, 8, 4, kSps, 1>(tmB, tmAV, a, s);
    else if (nsub == 2) launch_tc<2, 4, 4, kSps, 2>(tmB, tmAV, a, s);
    else launch_tc<IXB_K4_NSUB, IXB_K4_STAGES, 2, kSps, IXB_K4_NPROD, IXB_K4_MINB>(tmB, tmAV, a, s);
  } else {
    const int threads = 256;
    bgcoo_simt_kernel<<<static_cast<unsigned>(G), threads, 0, s>>>(
        AM, AK, static_cast<const __nv_bfloat16*>(AV), static_cast<const __nv_bfloat16*>(B), C,
        G, g, bm, bk, KB, N, MB, accumulate, check2, err);
    IXB_LAUNCH_CHECK("bgcoo_simt_kernel");
  }
  if (check2 && !(flags & IXB_ASYNC)) {
    OperandInfo ops[2] = {{"AK", "B", 0, KB, AK, G * g}, {"AM", "C", 0, MB, AM, G}};
    check_error_record(s, ops, 2);
  }
}

}  // namespace ixb

#ifdef IXB_K4_TRACE
extern "C" int ixb_debug_k4_trace(long long* host, int clear) {
  if (clear) {
    static long long zero[4096 * 16];
    return cudaMemcpyToSymbol(ixb::g_k4_trace, zero, sizeof zero);
  }
  return cudaMemcpyFromSymbol(host, ixb::g_k4_trace, sizeof(long long) * 4096 * 16);
}
#endif

extern "C" int ixb_spmm_blockgroupcoo(const int32_t* AM, const int32_t* AK, const void* AV,
                                      int64_t G, int64_t g, int64_t bm, int64_t bk, const void* B,
                                      int64_t KB, int64_t N, float* C, int64_t MB, int accumulate,
                                      int flags, ixb_stream stream) {
  return ixb_guard([&] {
    ixb::spmm_blockgroupcoo(AM, AK, AV, G, g, bm, bk, B, KB, N, C, MB, accumulate, flags,
                            reinterpret_cast<cudaStream_t>(stream));
  });
}
