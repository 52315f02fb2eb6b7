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
// Work split: CTA (chunk of CH group positions, n tile of 128*NSUB columns)
// owns every row segment (run of equal AM) that starts in its chunk, so each
// C block-row slice has exactly one writer (deterministic, no atomics).
// Warp roles: warp 0 = segment scan + TMA producer, warp 1 = TMEM allocator +
// single-thread UMMA issuer, warps 2..5 = epilogue (TMEM -> registers ->
// coalesced fp32 stores along n). A STAGES-deep full/empty mbarrier ring
// feeds the tensor core; accumulators are double buffered in TMEM so the
// epilogue of segment j overlaps the main loop of segment j+1.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.h"

namespace ixb {
namespace {

using namespace sm100;

constexpr int kThreadsTC = 224;  // 7 warps
constexpr uint32_t kAvBytes = 16 * 16 * 2;
constexpr uint32_t kSubBytes = 16 * 128 * 2;  // one 128-wide n subtile of a B tile

struct TcArgs {
  const int32_t* AM;
  const int32_t* AK;
  float* C;
  int64_t G, g, KB, N, MB;
  int chunk;    // group positions scanned per work item
  int nchunks;  // ceil(G / chunk)
  int ntiles;   // n tiles of 128*NSUB columns
  int accumulate;
  int check;
  int epi_sleep_ns;  // epilogue warps back off instead of spinning on acc_full
  ErrorRecord* err;
};

// A stage carries SPS consecutive slots of one row segment: SPS B tiles
// (1024-aligned), then SPS AV blocks. One full/empty round trip and one
// tcgen05.commit per 2*SPS UMMAs: commits interleaved with tiny MMA batches
// roughly double the tensor pipe's per-MMA cost (profiles/k4_diag_r1.md).
template <int NSUB, int STAGES, int SPS>
struct TcSmem {
  static constexpr uint32_t kBBytes = NSUB * kSubBytes;
  static constexpr uint32_t kStageBytes = ((SPS * (kBBytes + kAvBytes) + 1023) / 1024) * 1024;
  static constexpr uint32_t kTileBytes = STAGES * kStageBytes;
  static constexpr uint32_t kTotal = kTileBytes + 1024 /*barriers+queue*/ + 1024 /*align*/;
};

// A row segment (run of equal AM) owned by a work item.
struct Seg {
  int64_t s, e;   // group range [s, e)
  int row, prev;  // AM value, AM[s-1] (or -1)
  int ntile;      // n tile index
};

// Walks this CTA's work items (chunk, n tile), round-robin over the grid,
// and yields every segment that starts inside the chunk. Warp-collective;
// each role warp runs its own copy and sees the identical sequence.
struct SegIter {
  int64_t w;        // current work item
  int64_t base;     // first group position of the chunk
  unsigned starts;  // pending segment starts (lane bits) in the chunk
  int am, amp;      // this lane's AM[base+lane], AM[base+lane-1]
  int ntile;

  __device__ __forceinline__ void load(const TcArgs& a) {
    const int lane = threadIdx.x & 31;
    const int64_t chunk_id = w / a.ntiles;
    ntile = static_cast<int>(w % a.ntiles);
    base = chunk_id * a.chunk;
    const int64_t p = base + lane;
    const bool in = lane < a.chunk && p < a.G;
    am = in ? __ldg(a.AM + p) : 0;
    amp = (in && p > 0) ? __ldg(a.AM + p - 1) : -1;
    starts = __ballot_sync(0xffffffffu, in && (p == 0 || am != amp));
  }
  __device__ __forceinline__ void init(const TcArgs& a) {
    w = blockIdx.x;
    if (w < static_cast<int64_t>(a.nchunks) * a.ntiles) load(a);
    else starts = 0;
  }
  __device__ __forceinline__ bool next(const TcArgs& a, Seg& out) {
    const int64_t total = static_cast<int64_t>(a.nchunks) * a.ntiles;
    while (starts == 0) {
      w += gridDim.x;
      if (w >= total) return false;
      load(a);
    }
    const int lane = threadIdx.x & 31;
    const int sl = __ffs(starts) - 1;
    starts &= starts - 1;
    out.s = base + sl;
    out.row = __shfl_sync(0xffffffffu, am, sl);
    out.prev = __shfl_sync(0xffffffffu, amp, sl);
    out.ntile = ntile;
    int64_t e = out.s + 1;
    for (;;) {
      const int64_t pp = e + lane;
      const bool diff = pp >= a.G || __ldg(a.AM + pp) != out.row;
      const unsigned m = __ballot_sync(0xffffffffu, diff);
      if (m) {
        e += __ffs(m) - 1;
        break;
      }
      e += 32;
    }
    out.e = e;
    return true;
  }
};

constexpr int kQN = 16;  // segment queue depth (scheduler -> roles)

template <int NSUB, int STAGES, int NACC, int SPS, int MINB = 1>
__global__ void __launch_bounds__(kThreadsTC, MINB)
    bgcoo_tc_kernel(const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmAV, TcArgs a) {
  using L = TcSmem<NSUB, STAGES, SPS>;
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
  int* segq_tile = reinterpret_cast<int*>(segq + kQN);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  constexpr uint32_t kAccCols = 16 * NSUB;  // one accumulator buffer
  constexpr uint32_t kTmemCols = NACC * kAccCols <= 32    ? 32
                                 : NACC * kAccCols <= 64  ? 64
                                 : NACC * kAccCols <= 128 ? 128
                                 : NACC * kAccCols <= 256 ? 256
                                                          : 512;

  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&full[s], 1);
        mbar_init(&empty[s], 1);
      }
      for (int b = 0; b < NACC; ++b) {
        mbar_init(&acc_full[b], 1);
        mbar_init(&acc_empty[b], 4);
      }
      for (int q = 0; q < kQN; ++q) {
        mbar_init(&seg_full[q], 1);
        mbar_init(&seg_empty[q], 6);  // producer, UMMA issuer, 4 epilogue warps
      }
      fence_barrier_init();
      tma_prefetch_desc(&tmB);
      tma_prefetch_desc(&tmAV);
    }
  } else if (warp == 1) {
    tmem_alloc(tmem_base_slot, kTmemCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_base_slot;

  // Segment queue consumers: entry q holds {s, e, row, prev} + n tile; s < 0 ends.
  auto pop = [&](int j, int4& sg, int& tile) {
    const int q = j % kQN;
    mbar_wait(&seg_full[q], (j / kQN) & 1);
    sg = segq[q];
    tile = segq_tile[q];
  };
  auto release = [&](int j) { mbar_arrive(&seg_empty[j % kQN]); };

  if (warp == 6) {
    // ---------------------------------------------------------- scheduler
    // Discovers segments ahead of the pipeline so no role stalls on the
    // dependent AM loads between segments.
    SegIter it;
    it.init(a);
    Seg sg;
    int j = 0;
    bool more = true;
    while (more) {
      more = it.next(a, sg);
      const int q = j % kQN;
      if (lane == 0) {
        mbar_wait(&seg_empty[q], ((j / kQN) & 1) ^ 1);
        segq[q] = more ? make_int4(static_cast<int>(sg.s), static_cast<int>(sg.e), sg.row, sg.prev)
                       : make_int4(-1, -1, 0, 0);
        segq_tile[q] = more ? sg.ntile : 0;
        mbar_arrive(&seg_full[q]);
      }
      __syncwarp();
      ++j;
    }
  } else if (warp == 0) {
    // ---------------------------------------------------------- TMA producer
    const uint64_t keep = l2_evict_last();    // dense operand: re-read by many blocks
    const uint64_t stream = l2_evict_first();  // format: read once
    int stage = 0;
    uint32_t phase = 0;
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
        for (int t = 0; t < cnt; t += SPS) {
          const int nb = cnt - t < SPS ? cnt - t : SPS;
          int kk[SPS];
#pragma unroll
          for (int b = 0; b < SPS; ++b) kk[b] = __shfl_sync(0xffffffffu, k, (t + b) & 31);
          if (lane == 0) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* st = tiles + stage * L::kStageBytes;
            mbar_arrive_expect_tx(&full[stage], nb * (L::kBBytes + kAvBytes));
#pragma unroll
            for (int b = 0; b < SPS; ++b) {
              if (b >= nb) break;
              // one 3-D box {64 n, 16 rows, 2*NSUB atoms} lands as [atom][row][64]
              tma_load_3d(st + b * L::kBBytes, &tmB, &full[stage], 0, kk[b] * 16, n0 / 64, keep);
              tma_load_2d(st + SPS * L::kBBytes + b * kAvBytes, &tmAV, &full[stage], 0,
                          static_cast<int32_t>((i0 + t + b) * 16), stream);
            }
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        k = k_next;
      }
      __syncwarp();
      if (lane == 0) release(j);
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- UMMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(128, 16, /*A MN-major*/ true, /*B K-major*/ false);
    int stage = 0;
    uint32_t phase = 0;
    for (int j = 0;; ++j) {
      int4 sg;
      int tile;
      pop(j, sg, tile);
      if (sg.x < 0) break;
      const int buf = j % NACC;
      mbar_wait(&acc_empty[buf], ((j / NACC) & 1) ^ 1);
      tc_fence_after();
      const int64_t nslots = (static_cast<int64_t>(sg.y) - sg.x) * a.g;
      // same (32-slot chunk, SPS batch) partition as the producer
      for (int64_t i0 = 0; i0 < nslots; i0 += 32) {
        const int cnt = static_cast<int>(nslots - i0 < 32 ? nslots - i0 : 32);
        for (int t = 0; t < cnt; t += SPS) {
          const int nb = cnt - t < SPS ? cnt - t : SPS;
          if (lane == 0) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t st = smem_u32(tiles + stage * L::kStageBytes);
#pragma unroll
            for (int b = 0; b < SPS; ++b) {
              if (b >= nb) break;
              const uint64_t bdesc =
                  smem_desc(st + SPS * L::kBBytes + b * kAvBytes, 16, 256, kLayoutSW32);
#pragma unroll
              for (int sub = 0; sub < NSUB; ++sub) {
                // A: MN atoms (64 n) at +2048, K groups of 8 rows at +1024
                const uint64_t adesc =
                    smem_desc(st + b * L::kBBytes + sub * kSubBytes, 2048, 1024, kLayoutSW128);
                umma_f16(tmem_base + buf * kAccCols + sub * 16, adesc, bdesc, idesc,
                         (i0 + t + b) > 0 ? 1u : 0u);
              }
            }
            umma_commit(&empty[stage]);  // stage reusable once these UMMAs retire
            if (i0 + t + nb == nslots) umma_commit(&acc_full[buf]);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
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
      mbar_wait_backoff(&acc_full[buf], (j / NACC) & 1, a.epi_sleep_ns);
      tc_fence_after();
      uint32_t r[NSUB][16];
#pragma unroll
      for (int sub = 0; sub < NSUB; ++sub) {
        tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) +
                               buf * kAccCols + sub * 16,
                           r[sub]);
      }
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);  // TMEM buffer free for segment j+NACC
      if (row_ok) {
#pragma unroll
        for (int sub = 0; sub < NSUB; ++sub) {
          float* c = a.C + static_cast<int64_t>(row) * 16 * a.N + n0 + sub * 128 + nloc;
#pragma unroll
          for (int bm = 0; bm < 16; ++bm) {
            float v = __uint_as_float(r[sub][bm]);
            if (a.accumulate) v += c[static_cast<int64_t>(bm) * a.N];
            c[static_cast<int64_t>(bm) * a.N] = v;
          }
        }
      } else if (a.check && warp == 2 && lane == 0 && tile == 0) {
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
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
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
template <int NSUB, int STAGES, int NACC, int SPS, int MINB = 1>
void launch_tc(const CUtensorMap& tmB, const CUtensorMap& tmAV, TcArgs a, cudaStream_t s) {
  using L = TcSmem<NSUB, STAGES, SPS>;
  auto kern = bgcoo_tc_kernel<NSUB, STAGES, NACC, SPS, MINB>;
  set_max_dynamic_smem(reinterpret_cast<const void*>(kern), L::kTotal,
                       "cudaFuncSetAttribute(bgcoo_tc_kernel)");
  // resident CTAs per SM (registers, smem and TMEM columns): a property of the
  // compiled kernel, the same on every sm_100a device
  static int per_sm = 0;
  if (!per_sm) {
    cudaFuncAttributes fa;
    IXB_CUDA_CHECK(cudaFuncGetAttributes(&fa, kern));
    const int by_regs = 65536 / (((fa.numRegs * 32 + 255) / 256) * 256 * (kThreadsTC / 32));
    per_sm = static_cast<int>((220u * 1024u) / L::kTotal);
    if (per_sm > by_regs) per_sm = by_regs;
    constexpr int kCols = NACC * 16 * NSUB <= 32 ? 32 : NACC * 16 * NSUB <= 64 ? 64
                          : NACC * 16 * NSUB <= 128 ? 128 : NACC * 16 * NSUB <= 256 ? 256 : 512;
    if (per_sm > 512 / kCols) per_sm = 512 / kCols;  // a CTA must not wait in tcgen05.alloc
    if (per_sm < 1) per_sm = 1;
  }
  a.ntiles = static_cast<int>(a.N / (128 * NSUB));
  const int64_t items = static_cast<int64_t>(a.nchunks) * a.ntiles;
  int64_t grid = static_cast<int64_t>(sm_count()) * per_sm;  // persistent CTAs
  if (grid > items) grid = items;
  kern<<<static_cast<unsigned>(grid), kThreadsTC, L::kTotal, s>>>(tmB, tmAV, a);
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
    int64_t ch = MB > 0 ? G / MB : 1;
    a.chunk = static_cast<int>(ch < 1 ? 1 : (ch > 32 ? 32 : ch));
    a.accumulate = accumulate;
    a.check = check2;
    a.err = err;
    a.nchunks = static_cast<int>(ceil_div(G, a.chunk));
    const int nsub = N % 256 == 0 ? 2 : 1;
    // B viewed as {64 n, rows, N/64 atoms}: one TMA box = the whole n tile of
    // 16 rows, landing as [atom][row][64] (the MN-major SW128 canonical layout)
    const CUtensorMap tmB = make_tmap_3d(B, 64, KB * 16, N / 64, N * 2, 128, 64, 16, 2 * nsub,
                                        CU_TENSOR_MAP_SWIZZLE_128B);
    const CUtensorMap tmAV = make_tmap_2d(AV, 16, G * g * 16, 32, 16, 16,
                                         CU_TENSOR_MAP_SWIZZLE_32B);
    a.epi_sleep_ns = 256;  // back-off of the idle epilogue warps' barrier polls
    // 2 slots per stage, 4 stages: ~68 KB -> 3 CTAs (3 independent issue
    // streams) per SM; measured against 1, 4, 8, 12 slots per stage and
    // 1-5 CTAs/SM on cfg2 (profiles/k4_diag_r1.md), and against a panel
    // kernel with B-tile reuse across block rows (profiles/k4_diag_r2.md)
    if (nsub == 1) launch_tc<1, 8, 4, 2>(tmB, tmAV, a, s);
    else launch_tc<2, 4, 4, 2>(tmB, tmAV, a, s);
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

extern "C" int ixb_spmm_blockgroupcoo(const int32_t* AM, const int32_t* AK, const void* AV,
                                      int64_t G, int64_t g, int64_t bm, int64_t bk, const void* B,
                                      int64_t KB, int64_t N, float* C, int64_t MB, int accumulate,
                                      int flags, ixb_stream stream) {
  return ixb_guard([&] {
    ixb::spmm_blockgroupcoo(AM, AK, AV, G, g, bm, bk, B, KB, N, C, MB, accumulate, flags,
                            reinterpret_cast<cudaStream_t>(stream));
  });
}
