// K4 — BlockGroupCOO SpMM on tcgen05 / TMEM / TMA (sm_100a), panel form:
//   C[AM[p],bm,n] += AV[p,q,bm,bk] * B[AK[p,q],bk,n]   (corpus/structured_spmm.json:2)
// bf16 operands, fp32 accumulation in TMEM. Reference semantics: oracle
// plan.cpp:579-594 (vars p,bm,n,q,bk), plan executor plan.cpp:383-534.
//
// bM = 16 is below the smallest UMMA M, so each block product is computed
// transposed with the dense operand on the M side:
//     D^T[n, bm] += B_tile^T[n, bk] . AV_blk^T[bk, bm]
//   A = B[kb*16 : +16, n0 : n0+128]  (128 x 16, MN-major SW128, one TMA box)
//   B = AV[p,q]                       (16 x 16, K-major SW32, one TMA box)
//   D = TMEM, 128 lanes (n) x 16 columns (bm)
//
// Work item = (panel of R consecutive block rows, 128*NSUB columns of n).
// The R accumulators sit side by side in TMEM, so a B tile that several
// rows of the panel use (same block column kb) is fetched from L2 once per
// item instead of once per block: the per-panel op list is sorted by
// (kb, slot) once by the plan kernel (bgcoo_panel_plan_kernel). Each row's
// blocks are still summed in slot order — the canonical format stores a
// row's blocks by ascending kb (formats.cpp:124-129, pads repeat the last
// kb) — so every output row keeps the reference's summation order and has
// exactly one writer (deterministic, no atomics, shard-invariant).
//
// Warp roles (192 threads): warp 0 = TMA producer (walks the op list and
// packs whole stages: <= TMAX distinct B tiles and <= QMAX AV blocks, one
// arrival + byte count per stage, the stage's op table written to smem),
// warp 1 = TMEM allocator + single-thread UMMA issuer (one commit per
// stage), warps 2..5 = epilogue (TMEM -> registers -> coalesced fp32 rows).
// Accumulators are double buffered in TMEM so an item's epilogue overlaps
// the next item's MMAs.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "bgcoo_panel.h"
#include "common.cuh"
#include "sm100.cuh"
#include "tmap.h"

namespace ixb {

namespace {

using namespace sm100;

constexpr int kProducerWarps = 4;
constexpr int kEpiWarps = 4;
constexpr uint32_t kAvBytes = 16 * 16 * 2;
constexpr uint32_t kSubBytes = 16 * 128 * 2;  // 16 rows x 128 n: two SW128 atoms

template <int NSUB>
constexpr int panel_threads() {
  return 32 * (kProducerWarps + NSUB + kEpiWarps);  // producers, one issuer per n subtile, epilogue
}

template <int NSUB, int STAGES, int TMAX, int QMAX>
struct PanelSmem {
  static constexpr uint32_t kTile = NSUB * kSubBytes;  // a B tile: 16 rows x 128*NSUB n
  static constexpr uint32_t kStage = TMAX * kTile + QMAX * kAvBytes;
  static constexpr uint32_t kRing = STAGES * kStage;
  static constexpr uint32_t kTotal = kRing + 1024 /*barriers*/ + 1024 /*align*/;
};

// A stage record (32 ints, built by the plan): [0] nops | ntiles << 8 | last << 16,
// [1..4] one byte per op: tile index | row << 4, [8..15] block column kb of each
// tile, [16..31] AV slot of each op. A stage holds at most kTmaxCap distinct B
// tiles and kQmaxCap ops. Stage records of panel P start at record index
// rowptr[P*R]*g + P (a panel has at most one stage per op).
constexpr int kRecInts = 32;
constexpr int kTmaxCap = 8, kQmaxCap = 16;

struct PanelArgs {
  const int32_t* rec;
  const int32_t* nstages;  // [npanels]
  const int32_t* rowptr;
  const __nv_bfloat16* AV;
  const __nv_bfloat16* B;
  float* C;
  int64_t g, N, MB;
  int nchunks, items;
  int accumulate;
  int epi_sleep_ns;
};

// rowptr[r] = first group p with AM[p] >= r, r in [0, MB] (AM sorted). Out-of-range
// group coordinates are clamped out of every row and reported (operand 1 = AM).
__global__ void bgcoo_rowptr_kernel(const int32_t* AM, int64_t G, int64_t MB, int32_t* rowptr,
                                    int check, ErrorRecord* err) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p > G) return;
  auto clampv = [&](int64_t a) { return a < -1 ? -1 : (a > MB ? MB : a); };
  int64_t a = MB;
  if (p < G) {
    const int64_t v = AM[p];
    if (check && (v < 0 || v >= MB)) report_index_error(err, 1, p, v);
    a = clampv(v);
  }
  const int64_t ap = p > 0 ? clampv(AM[p - 1]) : -1;
  const int64_t lo = ap + 1 < 0 ? 0 : ap + 1;
  for (int64_t r = lo; r <= a && r <= MB; ++r) rowptr[r] = static_cast<int32_t>(p);
}

// One CTA per panel of R block rows. (1) The panel's slots are one contiguous
// range [rowptr[r0]*g, rowptr[r1]*g); each slot's place in the panel's op list
// is its rank under (kb, row, position): position in its own row + elements of
// lower rows with kb' <= kb + elements of higher rows with kb' < kb (binary
// searches over the per-row ascending kb lists). A row whose kb do not ascend
// in slot order (a non-canonical format) keeps plain slot order for the whole
// panel, so each row's summation order is its slot order either way.
// (2) Warp 0 packs the op list into stage records: a stage closes when it holds
// qmax ops or would need a (tmax+1)-th distinct B tile.
template <int R>
__global__ void __launch_bounds__(256)
    bgcoo_panel_plan_kernel(const int32_t* AK, const int32_t* perm, const int32_t* rowptr,
                            int64_t g, int64_t KB, int64_t MB, int2* ops, int32_t* rec,
                            int32_t* nstages, int tmax, int qmax, int check, ErrorRecord* err) {
  constexpr int kCap = 8192;  // slots staged in smem; larger panels search global memory
  __shared__ int32_t sk[kCap];
  __shared__ int64_t rs[R + 1];
  const int P = blockIdx.x;
  const int64_t r0 = static_cast<int64_t>(P) * R;
  const int nr = static_cast<int>(MB - r0 < R ? MB - r0 : R);
  if (threadIdx.x <= R) {
    const int64_t r = r0 + (threadIdx.x < nr ? threadIdx.x : nr);
    rs[threadIdx.x] = static_cast<int64_t>(rowptr[r]) * g;
  }
  __syncthreads();
  const int64_t base = rs[0];
  const int64_t n = rs[nr] - base;
  const bool staged = n <= kCap;
  auto key_at = [&](int64_t i) -> int32_t {  // kb of panel slot i, clamped into range
    int32_t k = staged ? sk[i] : AK[base + i];
    return (k < 0 || k >= KB) ? 0 : k;
  };
  int bad = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int32_t k = AK[base + i];
    if (k < 0 || k >= KB) {
      if (check) {
        const int64_t sl = base + i;
        const int64_t orig = perm ? static_cast<int64_t>(perm[sl / g]) * g + sl % g : sl;
        report_index_error(err, 0, orig, k);
      }
    }
    if (staged) sk[i] = k;
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (i == 0) continue;
    int r = 0;
    while (r + 1 < nr && rs[r + 1] - base <= i) ++r;
    if (rs[r] - base < i && key_at(i) < key_at(i - 1)) bad = 1;
  }
  const int nonmono = __syncthreads_or(bad);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    int r = 0;
    while (r + 1 < nr && rs[r + 1] - base <= i) ++r;
    const int32_t k = key_at(i);
    int64_t dest = i;
    if (!nonmono) {
      dest = i - (rs[r] - base);
      for (int rr = 0; rr < nr; ++rr) {
        if (rr == r) continue;
        // count of row rr's keys < k (rr > r) or <= k (rr < r)
        int64_t lo = rs[rr] - base, hi = rs[rr + 1] - base;
        const int64_t start = lo;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          const int32_t km = key_at(mid);
          if (rr < r ? km <= k : km < k) lo = mid + 1;
          else hi = mid;
        }
        dest += lo - start;
      }
    }
    const int64_t sl = base + i;
    const int64_t orig = perm ? static_cast<int64_t>(perm[sl / g]) * g + sl % g : sl;
    ops[base + dest] = make_int2(static_cast<int32_t>(orig), k | (r << 28));
  }
  __syncthreads();  // the op list (global) is complete and visible to the block
  if (threadIdx.x >= 32) return;
  // (2) warp 0, 32 ops per window: lane 0 runs the greedy stage split on the
  // window's "new block column" bits (registers only) and leaves each op's
  // (stage, position, tile) in smem; every lane then writes its op's record
  // fields. Records start zeroed; the header is the atomicMax over the stage's
  // ops of (q+1) | (t+1) << 8 | last << 16, i.e. the stage's last op.
  __shared__ int s_stage[32], s_q[32], s_t[32];
  const int lane = threadIdx.x;
  int32_t* out = rec + (base + P) * kRecInts;
  int ns = 0, t = 0, q = 0, carry = -1;  // lane 0's running state; carry = previous kb
  for (int64_t b0 = 0; b0 < n; b0 += 32) {
    const int cnt = static_cast<int>(n - b0 < 32 ? n - b0 : 32);
    const int2 mine = lane < cnt ? ops[base + b0 + lane] : make_int2(0, 0);
    const int kb = mine.y & 0x0fffffff;
    int kb_prev = __shfl_up_sync(0xffffffffu, kb, 1);
    if (lane == 0) kb_prev = carry;
    const uint32_t nk = __ballot_sync(0xffffffffu, lane < cnt && kb != kb_prev);
    if (lane == 0) {
      for (int j = 0; j < cnt; ++j) {
        bool nt = (nk >> j) & 1u;
        if (b0 + j > 0 && (q == qmax || (nt && t == tmax))) {
          ++ns;
          t = q = 0;
          nt = true;
        }
        if (nt || b0 + j == 0) ++t;
        s_stage[j] = ns;
        s_q[j] = q++;
        s_t[j] = t - 1;
      }
    }
    __syncwarp();
    if (lane < cnt) {
      const int st = s_stage[lane], qq = s_q[lane], tt = s_t[lane];
      const int r = (mine.y >> 28) & 7;
      int32_t* o = out + static_cast<int64_t>(st) * kRecInts;
      o[16 + qq] = mine.x;
      reinterpret_cast<uint8_t*>(o)[4 + qq] = static_cast<uint8_t>(tt | (r << 4));
      if (qq == 0 || kb != kb_prev) o[8 + tt] = kb;
      const int last = b0 + lane == n - 1 ? 1 << 16 : 0;
      atomicMax(o, (qq + 1) | ((tt + 1) << 8) | last);
    }
    carry = __shfl_sync(0xffffffffu, kb, cnt - 1);
    __syncwarp();
  }
  if (lane == 0) nstages[P] = n > 0 ? ns + 1 : 0;
}

// 16-byte global -> shared copies (LDGSTS) that skip L1; B tiles keep their
// lines in L2 (re-read by other panels), AV streams through.
__device__ __forceinline__ void cp_async_16_hint(uint32_t dst, const void* src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "l"(pol)
               : "memory");
}

template <int R, int NSUB, int STAGES, int NACC, int TMAX, int QMAX>
__global__ void __launch_bounds__(panel_threads<NSUB>(), 1) bgcoo_panel_kernel(PanelArgs a) {
  using L = PanelSmem<NSUB, STAGES, TMAX, QMAX>;
  static_assert(TMAX <= kTmaxCap && QMAX <= kQmaxCap && QMAX % 4 == 0, "stage record limits");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kRing);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;  // NACC
  uint64_t* acc_empty = acc_full + 4;   // NACC (<= 4)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr int kMmaWarp = kProducerWarps;              // issuers: kMmaWarp .. + NSUB - 1
  constexpr int kEpiWarp0 = kProducerWarps + NSUB;
  constexpr uint32_t kSubAcc = R * 16;                  // columns of one n subtile's accumulators
  constexpr uint32_t kAcc = NSUB * kSubAcc;             // columns of one accumulator buffer
  constexpr uint32_t kTmemCols = NACC * kAcc <= 32    ? 32
                                 : NACC * kAcc <= 64  ? 64
                                 : NACC * kAcc <= 128 ? 128
                                 : NACC * kAcc <= 256 ? 256
                                                      : 512;
  static_assert(NACC * kAcc <= 512, "TMEM holds 512 columns");
  static_assert(NACC <= 4 && R <= 8 && (R & (R - 1)) == 0, "panel kernel limits");

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 32 * kProducerWarps);  // one cp.async arrival per producer thread
      mbar_init(&empty[s], NSUB);                // one commit per issuer
    }
    for (int b = 0; b < NACC; ++b) {
      mbar_init(&acc_full[b], NSUB);
      mbar_init(&acc_empty[b], kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // stage records of work item `it` and its panel geometry
  auto item = [&](int it, int64_t& r0, int& nr, int& n0, const int32_t*& rec, int& ns) {
    const int P = it / a.nchunks;
    n0 = (it - P * a.nchunks) * 128 * NSUB;
    r0 = static_cast<int64_t>(P) * R;
    nr = static_cast<int>(a.MB - r0 < R ? a.MB - r0 : R);
    const int64_t o0 = static_cast<int64_t>(__ldg(a.rowptr + r0)) * a.g;
    rec = a.rec + (o0 + P) * kRecInts;
    ns = __ldg(a.nstages + P);
  };

  if (warp < kProducerWarps) {
    // --------------------------------------------------------------- producers
    // 128 threads gather each stage with 16-byte cp.async, applying the UMMA
    // swizzles in the smem address: B tiles MN-major SW128 ([atom][row][64 n],
    // 16-byte chunk c of row k at c ^ (k & 7)), AV blocks K-major SW32 (the two
    // 16-byte halves of rows 4..7 of each 8-row atom swapped).
    const int ptid = threadIdx.x;
    const uint64_t keep = l2_evict_last();
    const uint64_t stream = l2_evict_first();
    int stage = 0;
    uint32_t phase = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x) {
      int64_t r0;
      int nr, n0, ns;
      const int32_t* rec;
      item(it, r0, nr, n0, rec, ns);
      // stage metadata is prefetched two stages ahead (L2 latency is exposed
      // otherwise: a stage's copies cannot be addressed before it lands)
      const int wq = ptid >> 5;  // ops wq, wq + 4, ... carry this thread's AV chunks
      struct Meta {
        int hdr;
        int kb[TMAX];
        int slot[QMAX / 4];
      };
      auto fetch = [&](int s2) {
        Meta m;
        const int32_t* r2 = rec + static_cast<int64_t>(s2) * kRecInts;
        m.hdr = __ldg(r2);
#pragma unroll
        for (int t = 0; t < TMAX; ++t) m.kb[t] = __ldg(r2 + 8 + t);
#pragma unroll
        for (int i = 0; i < QMAX / 4; ++i) m.slot[i] = __ldg(r2 + 16 + wq + 4 * i);
        return m;
      };
      Meta m0 = ns > 0 ? fetch(0) : Meta{}, m1 = ns > 1 ? fetch(1) : Meta{};
      for (int s = 0; s < ns; ++s) {
        const Meta cur = m0;
        m0 = m1;
        if (s + 2 < ns) m1 = fetch(s + 2);
        const int nops = cur.hdr & 0xff, ntiles = (cur.hdr >> 8) & 0xff;
        mbar_wait(&empty[stage], phase ^ 1);
        const uint32_t st = smem_u32(smem + stage * L::kStage);
        // a tile row is 16*NSUB chunks of 16 B (8 n each); 128 threads cover
        // 128 / (16*NSUB) rows per pass, 16 rows per tile
        constexpr int kRowChunks = 16 * NSUB;
#pragma unroll
        for (int i = 0; i < 2 * NSUB * TMAX; ++i) {
          const int t = i / (2 * NSUB);
          if (t < ntiles) {
            const int cc = ptid + 128 * (i % (2 * NSUB));
            const int k = cc / kRowChunks, j = cc % kRowChunks, atom = j >> 3, c8 = j & 7;
            const int kbt = cur.kb[t];
            const __nv_bfloat16* src =
                a.B + (static_cast<int64_t>(kbt) * 16 + k) * a.N + n0 + atom * 64 + c8 * 8;
            cp_async_16_hint(st + t * L::kTile + atom * 2048 + k * 128 + ((c8 ^ (k & 7)) << 4),
                             src, keep);
          }
        }
#pragma unroll
        for (int i = 0; i < QMAX / 4; ++i) {
          const int q = wq + 4 * i;
          if (q < nops) {
            const int row = lane >> 1, h = lane & 1;
            const __nv_bfloat16* src =
                a.AV + static_cast<int64_t>(cur.slot[i]) * 256 + row * 16 + h * 8;
            cp_async_16_hint(st + TMAX * L::kTile + q * kAvBytes + row * 32 +
                                 ((h ^ ((row >> 2) & 1)) << 4),
                             src, stream);
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                         smem_u32(&full[stage]))
                     : "memory");
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp < kEpiWarp0) {
    // ------------------------------------------------------------ UMMA issuers
    // Issuer `sub` owns n subtile sub (A = columns [128*sub, 128*sub+128) of each
    // B tile) and its own accumulator columns: NSUB independent MMA streams
    // over the same stages, each committing its own release of the stage.
    const int sub = warp - kMmaWarp;
    constexpr uint32_t idesc = idesc_bf16_f32(128, 16, /*A MN-major*/ true, /*B K-major*/ false);
    int stage = 0;
    uint32_t phase = 0;
    int j = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x, ++j) {
      int64_t r0;
      int nr, n0, ns;
      const int32_t* rec;
      item(it, r0, nr, n0, rec, ns);
      const int buf = j % NACC;
      if (lane == 0) {
        mbar_wait(&acc_empty[buf], ((j / NACC) & 1) ^ 1);
        tc_fence_after();
        uint32_t mask = 0;
        int4 hdr = ns > 0 ? __ldg(reinterpret_cast<const int4*>(rec)) : make_int4(0, 0, 0, 0);
        int m3 = ns > 0 ? __ldg(rec + 4) : 0;
        for (int s = 0; s < ns; ++s) {
          const int4 cur = hdr;
          const int meta3 = m3;
          if (s + 1 < ns) {  // next stage's header, loaded while this one lands
            hdr = __ldg(reinterpret_cast<const int4*>(rec + static_cast<int64_t>(s + 1) * kRecInts));
            m3 = __ldg(rec + static_cast<int64_t>(s + 1) * kRecInts + 4);
          }
          mbar_wait(&full[stage], phase);
          fence_proxy_async_smem();  // cp.async (generic proxy) writes -> tensor core reads
          tc_fence_after();
          const int nops = cur.x & 0xff;
          const uint32_t st = smem_u32(smem + stage * L::kStage);
          const uint32_t mw[4] = {static_cast<uint32_t>(cur.y), static_cast<uint32_t>(cur.z),
                                  static_cast<uint32_t>(cur.w), static_cast<uint32_t>(meta3)};
          for (int q = 0; q < nops; ++q) {
            const uint32_t m = (mw[q >> 2] >> ((q & 3) * 8)) & 0xff;
            const uint32_t t = m & 15, r = (m >> 4) & (R - 1);
            const uint64_t bdesc =
                smem_desc(st + TMAX * L::kTile + q * kAvBytes, 16, 256, kLayoutSW32);
            // A: MN atoms (64 n) at +2048, K groups of 8 rows at +1024
            const uint64_t adesc =
                smem_desc(st + t * L::kTile + sub * kSubBytes, 2048, 1024, kLayoutSW128);
            umma_f16(tmem + buf * kAcc + sub * kSubAcc + r * 16, adesc, bdesc, idesc,
                     (mask >> r) & 1u);
            mask |= 1u << r;
          }
          umma_commit(&empty[stage]);  // stage reusable once these UMMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&acc_full[buf]);
      }
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int quarter = warp & 3;  // TMEM lanes [32*quarter, 32*quarter+32)
    const int nloc = quarter * 32 + lane;
    int j = 0;
    for (int it = blockIdx.x; it < a.items; it += gridDim.x, ++j) {
      const int P = it / a.nchunks;
      const int n0 = (it - P * a.nchunks) * 128 * NSUB;
      const int64_t r0 = static_cast<int64_t>(P) * R;
      const int nr = static_cast<int>(a.MB - r0 < R ? a.MB - r0 : R);
      // rows of the panel that hold at least one group
      const int rp = lane <= nr ? __ldg(a.rowptr + r0 + lane) : 0;
      const int rpn = __shfl_down_sync(0xffffffffu, rp, 1);
      const uint32_t present = __ballot_sync(0xffffffffu, lane < nr && rpn > rp);
      const int buf = j % NACC;
      mbar_wait_backoff(&acc_full[buf], (j / NACC) & 1, a.epi_sleep_ns);
      tc_fence_after();
      for (int r = 0; r < nr; ++r) {
        const bool has = (present >> r) & 1u;
        if (!has && a.accumulate) continue;
#pragma unroll
        for (int sb = 0; sb < NSUB; ++sb) {
          uint32_t v[16];
          if (has) {
            tmem_ld_32x32b_x16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + buf * kAcc +
                                   sb * kSubAcc + r * 16,
                               v);
            tmem_ld_wait();
          }
          float* c = a.C + (r0 + r) * 16 * a.N + n0 + sb * 128 + nloc;
#pragma unroll
          for (int bm = 0; bm < 16; ++bm) {
            float x = has ? __uint_as_float(v[bm]) : 0.f;
            if (a.accumulate) x += c[static_cast<int64_t>(bm) * a.N];
            c[static_cast<int64_t>(bm) * a.N] = x;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);  // buffer free for item j + NACC
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, kTmemCols);
  }
}

template <int R, int NSUB, int STAGES, int NACC, int TMAX, int QMAX>
void launch_panel(const BgPanelPlan& P, const void* AV, const void* B, int64_t N, float* C,
                  int accumulate, cudaStream_t s) {
  using L = PanelSmem<NSUB, STAGES, TMAX, QMAX>;
  auto kern = bgcoo_panel_kernel<R, NSUB, STAGES, NACC, TMAX, QMAX>;
  set_max_dynamic_smem(reinterpret_cast<const void*>(kern), L::kTotal,
                       "cudaFuncSetAttribute(bgcoo_panel_kernel)");
  // resident CTAs per SM (smem and TMEM columns): a property of the compiled
  // kernel, the same on every sm_100a device
  constexpr int acc = NACC * NSUB * R * 16;
  constexpr int cols = acc <= 32 ? 32 : acc <= 64 ? 64 : acc <= 128 ? 128 : acc <= 256 ? 256 : 512;
  int per_sm = static_cast<int>((227u * 1024u) / (L::kTotal + 1024));
  if (per_sm > 512 / cols) per_sm = 512 / cols;  // a CTA must not wait in tcgen05.alloc
  if (per_sm > 2048 / panel_threads<NSUB>()) per_sm = 2048 / panel_threads<NSUB>();
  if (per_sm < 1) per_sm = 1;
  PanelArgs a;
  a.rec = P.rec.p;
  a.nstages = P.nstages.p;
  a.rowptr = P.rowptr.p;
  a.AV = static_cast<const __nv_bfloat16*>(AV);
  a.B = static_cast<const __nv_bfloat16*>(B);
  a.C = C;
  a.g = P.g;
  a.N = N;
  a.MB = P.MB;
  a.nchunks = static_cast<int>(N / (128 * NSUB));
  a.items = static_cast<int>(ceil_div(P.MB, R)) * a.nchunks;
  a.accumulate = accumulate;
  a.epi_sleep_ns = 128;
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;
  if (grid > a.items) grid = a.items;
  kern<<<static_cast<unsigned>(grid), panel_threads<NSUB>(), L::kTotal, s>>>(a);
  IXB_LAUNCH_CHECK("bgcoo_panel_kernel");
}

// Kernel shapes (panel rows R, ring stages, accumulator buffers, tiles and ops
// per stage); variant 0 is the default.
struct PanelCfg {
  int R, nsub, stages, nacc, tmax, qmax;
};
constexpr PanelCfg kPanelCfgs[] = {
    {4, 2, 2, 2, 6, 8}, {4, 2, 3, 2, 4, 8}, {8, 1, 4, 2, 4, 8}, {4, 2, 2, 2, 5, 12},
    {2, 4, 2, 2, 3, 8}, {2, 4, 3, 2, 2, 4}, {4, 2, 2, 2, 6, 12}, {4, 2, 2, 1, 4, 8},
    {2, 2, 2, 2, 4, 8}, {2, 4, 2, 1, 2, 8}, {4, 2, 3, 1, 4, 8}};
int panel_variant() {
  static int v = [] {
    const char* e = getenv("IXB_K4_VARIANT");
    int x = e ? atoi(e) : 0;
    return (x < 0 || x >= static_cast<int>(sizeof(kPanelCfgs) / sizeof(kPanelCfgs[0]))) ? 0 : x;
  }();
  return v;
}
}  // namespace

void bgcoo_panel_plan(const int32_t* AM, const int32_t* AK, const int32_t* perm, int64_t G,
                      int64_t g, int64_t KB, int64_t MB, bool check, cudaStream_t s,
                      BgPanelPlan& P) {
  P.G = G;
  P.g = g;
  P.KB = KB;
  P.MB = MB;
  const PanelCfg c = kPanelCfgs[panel_variant()];
  P.R = c.R;
  P.variant = panel_variant();
  P.nslots = G * g;
  const int64_t npanels = ceil_div(MB, c.R);
  P.rowptr = Scratch<int32_t>(MB + 1, s);
  Scratch<int2> ops(G * g > 0 ? G * g : 1, s);
  P.rec = Scratch<int32_t>((G * g + npanels + 1) * kRecInts, s);
  P.nstages = Scratch<int32_t>(npanels + 1, s);
  ErrorRecord* err = device_error_record();
  bgcoo_rowptr_kernel<<<static_cast<unsigned>(ceil_div(G + 1, 256)), 256, 0, s>>>(
      AM, G, MB, P.rowptr.p, check && !perm, err);
  IXB_LAUNCH_CHECK("bgcoo_rowptr_kernel");
  if (npanels > 0) {
    IXB_CUDA_CHECK(cudaMemsetAsync(P.rec.p, 0, (G * g + npanels + 1) * kRecInts * 4, s));
    if (c.R == 2)
      bgcoo_panel_plan_kernel<2><<<static_cast<unsigned>(npanels), 256, 0, s>>>(
          AK, perm, P.rowptr.p, g, KB, MB, ops.p, P.rec.p, P.nstages.p, c.tmax, c.qmax,
          check && !perm, err);
    else if (c.R == 8)
      bgcoo_panel_plan_kernel<8><<<static_cast<unsigned>(npanels), 256, 0, s>>>(
          AK, perm, P.rowptr.p, g, KB, MB, ops.p, P.rec.p, P.nstages.p, c.tmax, c.qmax,
          check && !perm, err);
    else
      bgcoo_panel_plan_kernel<4><<<static_cast<unsigned>(npanels), 256, 0, s>>>(
          AK, perm, P.rowptr.p, g, KB, MB, ops.p, P.rec.p, P.nstages.p, c.tmax, c.qmax,
          check && !perm, err);
    IXB_LAUNCH_CHECK("bgcoo_panel_plan_kernel");
  }
}

bool bgcoo_panel_ok(int64_t bm, int64_t bk, int64_t N, const void* AV, const void* B) {
  return bm == 16 && bk == 16 && N % 128 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(AV) % 16 == 0;
}

void bgcoo_panel_run(const BgPanelPlan& P, const void* AV, const void* B, int64_t N, float* C,
                     int accumulate, cudaStream_t s) {
  if (P.MB == 0 || N == 0) return;
  switch (P.variant) {
    case 1: launch_panel<4, 2, 3, 2, 4, 8>(P, AV, B, N, C, accumulate, s); break;
    case 2: launch_panel<8, 1, 4, 2, 4, 8>(P, AV, B, N, C, accumulate, s); break;
    case 3: launch_panel<4, 2, 2, 2, 5, 12>(P, AV, B, N, C, accumulate, s); break;
    case 4: launch_panel<2, 4, 2, 2, 3, 8>(P, AV, B, N, C, accumulate, s); break;
    case 5: launch_panel<2, 4, 3, 2, 2, 4>(P, AV, B, N, C, accumulate, s); break;
    case 6: launch_panel<4, 2, 2, 2, 6, 12>(P, AV, B, N, C, accumulate, s); break;
    case 7: launch_panel<4, 2, 2, 1, 4, 8>(P, AV, B, N, C, accumulate, s); break;
    case 8: launch_panel<2, 2, 2, 2, 4, 8>(P, AV, B, N, C, accumulate, s); break;
    case 9: launch_panel<2, 4, 2, 1, 2, 8>(P, AV, B, N, C, accumulate, s); break;
    case 10: launch_panel<4, 2, 3, 1, 4, 8>(P, AV, B, N, C, accumulate, s); break;
    default: launch_panel<4, 2, 2, 2, 6, 8>(P, AV, B, N, C, accumulate, s); break;
  }
}

}  // namespace ixb
