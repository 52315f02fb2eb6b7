// K3 — GroupCOO SpMM on sm_100a:  C[AM[p],n] += AV[p,q] * B[AK[p,q],n]
// (corpus/unstructured_spmm.json:2; reference evaluators plan.cpp:383-534,
// oracle plan.cpp:579-594, fused kernel kernel.cpp:461-473).
//
// HBM/L2-gather bound. Design:
//  * Row-segment ownership instead of atomics: groups are sorted by AM (the
//    builders guarantee it), so the groups of one output row are contiguous.
//    Each warp scans a chunk of CH group positions for segment starts
//    (AM[p] != AM[p-1]) and owns every segment that starts there, summing
//    its groups in group order and writing the C row once. The result is
//    run-to-run deterministic and independent of CH / grid / sharding.
//  * The dense operand row B[k, :] is gathered with 128-bit
//    ld.global.nc.L1::no_allocate loads under an L2 evict_last policy (B is
//    re-read by every group that names k), the format (AK/AV) is streamed
//    under evict_first. Group metadata is loaded coalesced (one slot per
//    lane) and broadcast by shuffles; the q loop is unrolled by 8 so every
//    lane keeps 8×T independent 16-byte gathers in flight.
//  * `=` writes every row of C exactly once: the owner of a segment also
//    zero-fills the empty rows between the previous segment's row and its
//    own (and the tail after the last segment), so no memset pass is needed.
//  * Long rows (skewed / power-law matrices: more than kSplitSlots slots)
//    would leave one warp serially summing the whole row while the rest of
//    the GPU idles. Their owner cuts the row's slot stream into pieces of
//    kSplitSlots at fixed offsets from the row start, keeps piece 0 and
//    publishes the rest on a device work queue that every warp drains when
//    its own chunk is done. Each piece is summed into a partial row; the
//    last piece to finish adds the partials to C in piece order. Piece
//    boundaries depend only on the row, so results stay deterministic and
//    independent of the grid and of sharding.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"

namespace ixb {
namespace {

constexpr int kThreads = 256;

template <int VEC>
struct VecT;
template <>
struct VecT<4> {
  using T = float4;
};
template <>
struct VecT<1> {
  using T = float;
};

__device__ __forceinline__ void vzero(float4& a) { a = make_float4(0.f, 0.f, 0.f, 0.f); }
__device__ __forceinline__ void vzero(float& a) { a = 0.f; }
__device__ __forceinline__ void vfma(float4& a, float s, const float4& b) {
  a.x = fmaf(s, b.x, a.x);
  a.y = fmaf(s, b.y, a.y);
  a.z = fmaf(s, b.z, a.z);
  a.w = fmaf(s, b.w, a.w);
}
__device__ __forceinline__ void vfma(float& a, float s, const float& b) { a = fmaf(s, b, a); }
// Compensated (Kahan) accumulation: each unrolled batch of terms is summed in
// order into a short partial, then the partial is added to the running sum
// with its rounding error carried in c. Long fp32 rows (cfg3: ~5000 terms)
// then stay within ~4e-6 of the fp64 reference instead of ~1e-4, at
// ~1.5 ALU ops per term (exact sums keep c == 0: integer data unaffected).
// add a partial sum p into (a, c) with compensation
__device__ __forceinline__ void kadd1(float& a, float& c, float p) {
  const float y = p - c;
  const float t = a + y;
  c = (t - a) - y;
  a = t;
}
__device__ __forceinline__ void kadd(float4& a, float4& c, const float4& p) {
  kadd1(a.x, c.x, p.x);
  kadd1(a.y, c.y, p.y);
  kadd1(a.z, c.z, p.z);
  kadd1(a.w, c.w, p.w);
}
__device__ __forceinline__ void kadd(float& a, float& c, const float& p) { kadd1(a, c, p); }
__device__ __forceinline__ void vadd(float4& a, const float4& b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}
__device__ __forceinline__ void vadd(float& a, const float& b) { a += b; }

template <int VEC>
__device__ __forceinline__ typename VecT<VEC>::T ld_b(const float* p, uint64_t pol);
template <>
__device__ __forceinline__ float4 ld_b<4>(const float* p, uint64_t pol) {
  return ldg_f4_keep(p, pol);
}
template <>
__device__ __forceinline__ float ld_b<1>(const float* p, uint64_t pol) {
  return ldg_f_keep(p, pol);
}

struct SpmmArgs {
  const int32_t* AM;    // [G] (sorted copy when perm != null)
  const int32_t* perm;  // [G] original group index per sorted position, or null
  const int32_t* AK;    // [G, g]
  const float* AV;      // [G, g]
  const float* B;       // [K, N]
  float* C;             // [M, N]
  int64_t G, g, K, N, M;
  int chunk;            // CH: group positions scanned per warp (<= 32)
  int accumulate;
  int check;
  ErrorRecord* err;
  // long-row split queue (self-resetting): ctr = {head, tail, long rows,
  // CTAs done}, then lrctr[cap] (pieces finished per long row)
  unsigned* ctr;
  int4* rec;     // [cap][2] {s, i0, i1, row}, {long row id, pieces, first task, piece}
  float* part;   // [cap][N] piece partial rows
  int64_t cap;   // task capacity
  int64_t split; // slots per piece; 0: no row can be longer (no queue protocol)
};

// Zero rows [r0, r1) of C, cooperatively by one warp.
__device__ __forceinline__ void zero_rows(float* C, int64_t N, int64_t r0, int64_t r1) {
  if (r1 <= r0) return;
  int64_t total = (r1 - r0) * N;
  float* base = C + r0 * N;
  if ((N & 3) == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0) {
    float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t i = lane_id(); i < total / 4; i += 32) reinterpret_cast<float4*>(base)[i] = z;
  } else {
    for (int64_t i = lane_id(); i < total; i += 32) base[i] = 0.f;
  }
}

// Residency over gathers in flight: T = 1 (N <= 128) runs 4 CTAs (32 warps)
// per SM with 8 gathers per lane (cfg1 24.0 -> 20.9 us against 2 CTAs x 16);
// wider passes run 3 CTAs per SM (cfg3 d0.02 349 -> 336 us) without spills.
#ifndef IXB_K3_U1
#define IXB_K3_U1 8
#endif
#ifndef IXB_K3_MINB_WIDE
#define IXB_K3_MINB_WIDE 3
#endif
template <int T>
constexpr int k3_min_blocks() {
  return T == 1 ? 4 : IXB_K3_MINB_WIDE;
}
// Sums the slots [i_beg, i_end) of the segment that starts at group s (slot
// i is slot i % g of group s + i / g, in (p, q) order) into the row `dst`:
// dst = acc (add: dst += acc). Warp-collective.
template <int VEC, int T, bool PERM>
__device__ __forceinline__ void sum_range(const SpmmArgs& a, int64_t s, int64_t i_beg,
                                          int64_t i_end, float* dst, bool add, uint64_t keep,
                                          uint64_t stream) {
  using V = typename VecT<VEC>::T;
  constexpr int kColsPerPass = 32 * VEC * T;
  constexpr int kUnroll = T >= 4 ? 4 : (T == 2 ? 8 : IXB_K3_U1);  // gathers in flight per lane
  const int lane = lane_id();
  for (int64_t c0 = 0; c0 < a.N; c0 += kColsPerPass) {
    V acc[T];
    V comp[T];  // compensation of acc
#pragma unroll
    for (int t = 0; t < T; ++t) vzero(comp[t]);
#pragma unroll
    for (int t = 0; t < T; ++t) vzero(acc[t]);
    int64_t col[T];
    bool col_ok[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      col[t] = c0 + (t * 32 + lane) * VEC;
      col_ok[t] = col[t] < a.N;
    }
    // The slots as one stream: 32 slots of metadata per coalesced load, the
    // next chunk prefetched while the current one's gathers are in flight.
    auto load_meta = [&](int64_t i0, int& k, float& v) {
      k = 0;
      v = 0.f;
      const int64_t i = i0 + lane;
      if (i < i_end) {
        const int64_t grp = s + i / a.g;
        const int64_t gp = PERM ? __ldg(a.perm + grp) : grp;
        const int64_t slot = gp * a.g + i % a.g;
        k = ldg_i_stream(a.AK + slot, stream);
        v = ldg_f_stream(a.AV + slot, stream);
        if (k < 0 || static_cast<int64_t>(k) >= a.K) {
          if (a.check) report_index_error(a.err, 0, slot, k);
          k = 0;
          v = 0.f;
        }
      }
    };
    int nk, my_k;
    float nv, my_v;
    load_meta(i_beg, my_k, my_v);
    for (int64_t i0 = i_beg; i0 < i_end; i0 += 32) {
      load_meta(i0 + 32, nk, nv);  // prefetch next chunk
      const int qn = static_cast<int>(i_end - i0 < 32 ? i_end - i0 : 32);
      for (int q = 0; q < qn; q += kUnroll) {
        int kk[kUnroll];
        float vv[kUnroll];
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
          kk[j] = __shfl_sync(0xffffffffu, my_k, (q + j) & 31);
          vv[j] = __shfl_sync(0xffffffffu, my_v, (q + j) & 31);
        }
        V bv[kUnroll][T];
#pragma unroll
        for (int j = 0; j < kUnroll; ++j) {
          const float* brow = a.B + static_cast<int64_t>(kk[j]) * a.N;
#pragma unroll
          for (int t = 0; t < T; ++t) {
            if (q + j < qn && col_ok[t]) bv[j][t] = ld_b<VEC>(brow + col[t], keep);
            else vzero(bv[j][t]);
          }
        }
        // the batch's terms summed in (p, q) order, then folded in with
        // compensation (see kadd)
#pragma unroll
        for (int t = 0; t < T; ++t) {
          V part;
          vzero(part);
#pragma unroll
          for (int j = 0; j < kUnroll; ++j) vfma(part, vv[j], bv[j][t]);
          kadd(acc[t], comp[t], part);
        }
      }
      my_k = nk;
      my_v = nv;
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      if (!col_ok[t]) continue;
      V* d = reinterpret_cast<V*>(dst + col[t]);
      if (add) {
        V old = *d;
        vadd(old, acc[t]);
        *d = old;
      } else {
        *d = acc[t];
      }
    }
  }
}

// One piece (queue task `pos`) of a long row: partial row, then the last
// piece of the row to finish sums the partials into C in piece order.
template <int VEC, int T, bool PERM>
__device__ __forceinline__ void run_piece(const SpmmArgs& a, int64_t pos, uint64_t keep,
                                          uint64_t stream) {
  const int lane = lane_id();
  const int4 r0 = __ldcg(a.rec + 2 * pos), r1 = __ldcg(a.rec + 2 * pos + 1);
  const int64_t s = r0.x, row = r0.w;
  float* mine = a.part + pos * a.N;
  sum_range<VEC, T, PERM>(a, s, r0.y, r0.z, mine, false, keep, stream);
  __threadfence();
  __syncwarp();
  unsigned last = 0;
  if (lane == 0) {
    unsigned* done = a.ctr + 4 + r1.x;
    last = atomicAdd(done, 1u) == static_cast<unsigned>(r1.y - 1);
    if (last) *done = 0;  // reset for the next launch
  }
  if (!__shfl_sync(0xffffffffu, last, 0)) return;
  __threadfence();
  float* crow = a.C + row * a.N;
  const float* p0 = a.part + static_cast<int64_t>(r1.z) * a.N;
  for (int64_t c = lane; c < a.N; c += 32) {
    float v = a.accumulate ? crow[c] : 0.f;
    for (int k = 0; k < r1.y; ++k) v += __ldcg(p0 + k * a.N + c);
    crow[c] = v;
  }
}

// A long row's pieces [k*split, (k+1)*split) go on the queue for
// spmm_groupcoo_pieces_kernel (launched after the main kernel).
__device__ __noinline__ void publish_long_row(const SpmmArgs& a, int64_t s, int64_t nslots,
                                              int row) {
  const int lane = lane_id();
  const int64_t np = (nslots + a.split - 1) / a.split;
  unsigned pos0 = 0, lr = 0;
  if (lane == 0) {
    pos0 = atomicAdd(a.ctr + 1, static_cast<unsigned>(np));
    lr = atomicAdd(a.ctr + 2, 1u);
  }
  pos0 = __shfl_sync(0xffffffffu, pos0, 0);
  lr = __shfl_sync(0xffffffffu, lr, 0);
  for (int64_t k = lane; k < np; k += 32) {
    const int64_t i0 = k * a.split, i1 = i0 + a.split < nslots ? i0 + a.split : nslots;
    a.rec[2 * (pos0 + k)] = make_int4(static_cast<int>(s), static_cast<int>(i0),
                                      static_cast<int>(i1), row);
    a.rec[2 * (pos0 + k) + 1] = make_int4(static_cast<int>(lr), static_cast<int>(np),
                                          static_cast<int>(pos0), static_cast<int>(k));
  }
}

template <int VEC, int T, bool PERM, bool SPLIT>
__device__ __forceinline__ void k3_body(const SpmmArgs& a) {
  using V = typename VecT<VEC>::T;
  constexpr int kColsPerPass = 32 * VEC * T;
  constexpr int kUnroll = T >= 4 ? 4 : (T == 2 ? 8 : IXB_K3_U1);  // gathers in flight per lane
  const int lane = lane_id();
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5;
  const int64_t base = warp * a.chunk;
  if (base >= a.G) return;
  const uint64_t keep = policy_evict_last();
  const uint64_t stream = policy_evict_first();

  // Segment starts inside this warp's chunk.
  const int64_t p_lane = base + lane;
  const bool in_chunk = lane < a.chunk && p_lane < a.G;
  int am_here = in_chunk ? __ldg(a.AM + p_lane) : 0;
  int am_prev = (in_chunk && p_lane > 0) ? __ldg(a.AM + p_lane - 1) : -1;
  unsigned starts = __ballot_sync(0xffffffffu, in_chunk && (p_lane == 0 || am_here != am_prev));

  while (starts) {
    const int sl = __ffs(starts) - 1;
    starts &= starts - 1;
    const int64_t s = base + sl;
    const int row = __shfl_sync(0xffffffffu, am_here, sl);
    const int prev_row = __shfl_sync(0xffffffffu, am_prev, sl);
    // Segment end: first p > s with AM[p] != row (windows of 32, coalesced).
    int64_t e = s + 1;
    for (;;) {
      const int64_t pp = e + lane;
      const bool diff = pp >= a.G || __ldg(a.AM + pp) != row;
      const unsigned m = __ballot_sync(0xffffffffu, diff);
      if (m) {
        e += __ffs(m) - 1;
        break;
      }
      e += 32;
    }
    const bool row_ok = row >= 0 && static_cast<int64_t>(row) < a.M;
    if (!a.accumulate) {
      // Empty rows between the previous segment and this one; the tail.
      int64_t z0 = prev_row + 1 < 0 ? 0 : prev_row + 1;
      int64_t z1 = row < 0 ? 0 : (row > a.M ? a.M : row);
      zero_rows(a.C, a.N, z0, z1);
      if (e == a.G) zero_rows(a.C, a.N, row + 1 < 0 ? 0 : row + 1, a.M);
    }
    if (!row_ok) {
      if (a.check) {
        // First offending AM position of this value is the segment start.
        if (lane == 0) report_index_error(a.err, 1, PERM ? __ldg(a.perm + s) : s, row);
        // Gathers are checked before scatters (plan.cpp:544-561): still
        // validate this segment's AK so a gather error keeps priority.
        for (int64_t p = s; p < e; ++p) {
          const int64_t gp = PERM ? __ldg(a.perm + p) : p;
          for (int64_t q = lane; q < a.g; q += 32) {
            const int k = __ldg(a.AK + gp * a.g + q);
            if (k < 0 || static_cast<int64_t>(k) >= a.K) report_index_error(a.err, 0, gp * a.g + q, k);
          }
        }
      }
      continue;
    }
    if constexpr (SPLIT) {
      const int64_t ns = (e - s) * a.g;
      if (ns > a.split) {  // long row: its pieces go on the queue
        publish_long_row(a, s, ns, row);
        continue;
      }
    }
    float* crow = a.C + static_cast<int64_t>(row) * a.N;
    for (int64_t c0 = 0; c0 < a.N; c0 += kColsPerPass) {
      V acc[T];
      V comp[T];  // compensation of acc
#pragma unroll
      for (int t = 0; t < T; ++t) vzero(comp[t]);
#pragma unroll
      for (int t = 0; t < T; ++t) vzero(acc[t]);
      int64_t col[T];
      bool col_ok[T];
#pragma unroll
      for (int t = 0; t < T; ++t) {
        col[t] = c0 + (t * 32 + lane) * VEC;
        col_ok[t] = col[t] < a.N;
      }
      // The segment's slots as one stream (group order, then q): 32 slots of
      // metadata per coalesced load, the next chunk prefetched while the
      // current one's gathers are in flight. Summation order = (p, q) order.
      const int64_t nslots = (e - s) * a.g;
      auto load_meta = [&](int64_t i0, int& k, float& v) {
        k = 0;
        v = 0.f;
        const int64_t i = i0 + lane;
        if (i < nslots) {
          const int64_t grp = s + i / a.g;
          const int64_t gp = PERM ? __ldg(a.perm + grp) : grp;
          const int64_t slot = gp * a.g + i % a.g;
          k = ldg_i_stream(a.AK + slot, stream);
          v = ldg_f_stream(a.AV + slot, stream);
          if (k < 0 || static_cast<int64_t>(k) >= a.K) {
            if (a.check) report_index_error(a.err, 0, slot, k);
            k = 0;
            v = 0.f;
          }
        }
      };
      int nk, my_k;
      float nv, my_v;
      load_meta(0, my_k, my_v);
      for (int64_t i0 = 0; i0 < nslots; i0 += 32) {
        load_meta(i0 + 32, nk, nv);  // prefetch next chunk
        const int qn = static_cast<int>(nslots - i0 < 32 ? nslots - i0 : 32);
        for (int q = 0; q < qn; q += kUnroll) {
          int kk[kUnroll];
          float vv[kUnroll];
#pragma unroll
          for (int j = 0; j < kUnroll; ++j) {
            kk[j] = __shfl_sync(0xffffffffu, my_k, (q + j) & 31);
            vv[j] = __shfl_sync(0xffffffffu, my_v, (q + j) & 31);
          }
          V bv[kUnroll][T];
#pragma unroll
          for (int j = 0; j < kUnroll; ++j) {
            const float* brow = a.B + static_cast<int64_t>(kk[j]) * a.N;
#pragma unroll
            for (int t = 0; t < T; ++t) {
              if (q + j < qn && col_ok[t]) bv[j][t] = ld_b<VEC>(brow + col[t], keep);
              else vzero(bv[j][t]);
            }
          }
          // the batch's terms summed in (p, q) order, then folded in with
          // compensation (see kadd)
#pragma unroll
          for (int t = 0; t < T; ++t) {
            V part;
            vzero(part);
#pragma unroll
            for (int j = 0; j < kUnroll; ++j) vfma(part, vv[j], bv[j][t]);
            kadd(acc[t], comp[t], part);
          }
        }
        my_k = nk;
        my_v = nv;
      }
#pragma unroll
      for (int t = 0; t < T; ++t) {
        if (!col_ok[t]) continue;
        V* dst = reinterpret_cast<V*>(crow + col[t]);
        if (a.accumulate) {
          V old = *dst;
          vadd(old, acc[t]);
          *dst = old;
        } else {
          *dst = acc[t];
        }
      }
    }
  }
}

// Matrices whose rows cannot exceed the piece length (canonical rows hold at
// most K nonzeros): the plain kernel.
template <int VEC, int T, bool PERM>
__global__ void __launch_bounds__(kThreads, k3_min_blocks<T>()) spmm_groupcoo_kernel(SpmmArgs a) {
  k3_body<VEC, T, PERM, false>(a);
}

// Long rows possible: the same, queueing long rows for the pieces kernel.
template <int VEC, int T, bool PERM>
__global__ void __launch_bounds__(kThreads, k3_min_blocks<T>())
    spmm_groupcoo_split_kernel(const __grid_constant__ SpmmArgs a) {
  k3_body<VEC, T, PERM, true>(a);
}

// The long-row pieces queued by spmm_groupcoo_kernel: persistent warps claim
// tasks [0, tail) (all published: stream order) and sum them; the last piece
// of a row combines. The last CTA out resets the queue counters.
template <int VEC, int T, bool PERM>
__global__ void __launch_bounds__(kThreads, k3_min_blocks<T>())
    spmm_groupcoo_pieces_kernel(const __grid_constant__ SpmmArgs a) {
  __shared__ unsigned warps_out;
  if (threadIdx.x == 0) warps_out = 0;
  __syncthreads();
  const int lane = lane_id();
  const uint64_t keep = policy_evict_last();
  const uint64_t stream = policy_evict_first();
  const unsigned ntasks = *reinterpret_cast<volatile unsigned*>(a.ctr + 1);
  for (;;) {
    unsigned t = 0;
    if (lane == 0) t = atomicAdd(a.ctr, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= ntasks) break;
    run_piece<VEC, T, PERM>(a, t, keep, stream);
  }
  if (lane == 0 && atomicAdd(&warps_out, 1u) == kThreads / 32 - 1) {
    __threadfence();
    if (atomicAdd(a.ctr + 3, 1u) == gridDim.x - 1) {
      a.ctr[0] = 0;
      a.ctr[1] = 0;
      a.ctr[2] = 0;
      a.ctr[3] = 0;
      __threadfence();
    }
  }
}

__global__ void not_sorted_kernel(const int32_t* AM, int64_t G, int* flag) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i > 0 && i < G && AM[i] < AM[i - 1]) *flag = 1;
}

__global__ void iota_kernel(int32_t* x, int64_t n) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = static_cast<int32_t>(i);
}

template <int VEC, int T, bool PERM>
void launch_t(const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  if (a.split <= 0) {
    spmm_groupcoo_kernel<VEC, T, PERM><<<grid, kThreads, 0, s>>>(a);
    IXB_LAUNCH_CHECK("spmm_groupcoo_kernel");
  } else {  // long rows possible: queue them, then drain the queue
    spmm_groupcoo_split_kernel<VEC, T, PERM><<<grid, kThreads, 0, s>>>(a);
    IXB_LAUNCH_CHECK("spmm_groupcoo_split_kernel");
    spmm_groupcoo_pieces_kernel<VEC, T, PERM>
        <<<sm_count() * k3_min_blocks<T>(), kThreads, 0, s>>>(a);
    IXB_LAUNCH_CHECK("spmm_groupcoo_pieces_kernel");
  }
}

template <int VEC, bool PERM>
void launch_vec(const SpmmArgs& a, int64_t grid, cudaStream_t s) {
  const int64_t passes = ceil_div(a.N, 32 * VEC);
  if (passes >= 4) launch_t<VEC, 4, PERM>(a, grid, s);
  else if (passes >= 2) launch_t<VEC, 2, PERM>(a, grid, s);
  else launch_t<VEC, 1, PERM>(a, grid, s);
}

}  // namespace

// Returns true when AM is non-decreasing (one pass + sync).
bool groups_sorted(const int32_t* AM, int64_t G, cudaStream_t s) {
  if (G < 2) return true;
  Scratch<int> flag(1, s);
  IXB_CUDA_CHECK(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
  not_sorted_kernel<<<ceil_div(G, 256), 256, 0, s>>>(AM, G, flag.p);
  IXB_LAUNCH_CHECK("not_sorted_kernel");
  int h = 0;
  IXB_CUDA_CHECK(cudaMemcpyAsync(&h, flag.p, sizeof h, cudaMemcpyDeviceToHost, s));
  IXB_CUDA_CHECK(cudaStreamSynchronize(s));
  return h == 0;
}

// Stable permutation of groups by AM (CUB LSD radix sort is stable).
void sort_groups(const int32_t* AM, int64_t G, cudaStream_t s, Scratch<int32_t>& am_sorted,
                 Scratch<int32_t>& perm) {
  Scratch<int32_t> iota(G, s);
  am_sorted = Scratch<int32_t>(G, s);
  perm = Scratch<int32_t>(G, s);
  iota_kernel<<<ceil_div(G, 256), 256, 0, s>>>(iota.p, G);
  IXB_LAUNCH_CHECK("iota_kernel");
  size_t tmp_bytes = 0;
  IXB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, AM, am_sorted.p, iota.p,
                                                 perm.p, static_cast<int>(G), 0, 32, s));
  Scratch<char> tmp(tmp_bytes, s);
  // CUB orders signed int32 keys correctly (negative = invalid rows first).
  IXB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, AM, am_sorted.p, iota.p,
                                                 perm.p, static_cast<int>(G), 0, 32, s));
  note_launch(4);
}

void spmm_groupcoo(const int32_t* AM, const int32_t* AK, const float* AV, int64_t G, int64_t g,
                   const float* B, int64_t K, int64_t N, float* C, int64_t M, int accumulate,
                   int flags, cudaStream_t s) {
  if (G < 0 || g < 1 || K < 0 || N < 0 || M < 0) fail(IXB_SHAPE, "ixb_spmm_groupcoo: bad extents");
  if (G > INT32_MAX) fail(IXB_SHAPE, "ixb_spmm_groupcoo: more than 2^31 groups");
  const bool check = !(flags & IXB_UNCHECKED);
  if (N == 0 || M == 0) return;
  if (G == 0) {
    if (!accumulate) IXB_CUDA_CHECK(cudaMemsetAsync(C, 0, M * N * sizeof(float), s));
    return;
  }
  Scratch<int32_t> am_sorted, perm;
  bool use_perm = false;
  if (!(flags & IXB_GROUPS_SORTED) && !groups_sorted(AM, G, s)) {
    sort_groups(AM, G, s, am_sorted, perm);
    use_perm = true;
  }
  SpmmArgs a;
  a.AM = use_perm ? am_sorted.p : AM;
  a.perm = use_perm ? perm.p : nullptr;
  a.AK = AK;
  a.AV = AV;
  a.B = B;
  a.C = C;
  a.G = G;
  a.g = g;
  a.K = K;
  a.N = N;
  a.M = M;
  int64_t ch = M > 0 ? G / M : 1;
  a.chunk = static_cast<int>(ch < 1 ? 1 : (ch > 32 ? 32 : ch));
  a.accumulate = accumulate;
  a.check = check;
  a.err = device_error_record();
  // long rows: pieces of kSplitSlots slots (a constant: pieces depend only on
  // the row, so results do not depend on the grid or on sharding); the
  // capacity bounds the tasks of any matrix (sum over long rows of ceil(n/L)
  // <= 2 * slots / L); matrices beyond ~1e8 slots per piece budget use
  // longer pieces
  const int64_t slots = G * g;
  constexpr int64_t kSplitSlots = 8192;
  constexpr int64_t kMaxTasks = 65536 - 4;
  a.split = kSplitSlots;
  while (2 * slots / a.split + 1 > kMaxTasks) a.split *= 2;
  // a canonical row holds at most K nonzeros, padded to a multiple of g: when
  // that cannot exceed the piece length the queue protocol is skipped (a row
  // longer only through duplicate coordinates is still summed, by its owner)
  const int64_t split_len = a.split;
  if (K + g - 1 <= a.split) a.split = 0;
  a.cap = 2 * slots / split_len + 1;
  a.ctr = work_counters(s, static_cast<size_t>(4 + a.cap));
  const size_t qbytes = a.cap * 2 * sizeof(int4) + a.cap * N * sizeof(float);
  Scratch<char> q_graph;  // first use inside a graph capture
  char* q = static_cast<char*>(stream_buffer(s, qbytes, kBufK3Split));
  if (!q) {
    q_graph = Scratch<char>(qbytes, s);
    q = q_graph.p;
  }
  a.rec = reinterpret_cast<int4*>(q);
  a.part = reinterpret_cast<float*>(q + a.cap * 2 * sizeof(int4));
  const int64_t warps = ceil_div(G, a.chunk);
  const int64_t grid = ceil_div(warps * 32, kThreads);
  const bool vec_ok = (N % 4 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0) &&
                      (reinterpret_cast<uintptr_t>(C) % 16 == 0);
  if (vec_ok) {
    use_perm ? launch_vec<4, true>(a, grid, s) : launch_vec<4, false>(a, grid, s);
  } else {
    use_perm ? launch_vec<1, true>(a, grid, s) : launch_vec<1, false>(a, grid, s);
  }
  if (check && !(flags & IXB_ASYNC)) {
    OperandInfo ops[2] = {{"AK", "B", 0, K, AK, G * g}, {"AM", "C", 0, M, AM, G}};
    check_error_record(s, ops, 2);
  }
}

}  // namespace ixb

extern "C" int ixb_spmm_groupcoo(const int32_t* AM, const int32_t* AK, const float* AV, int64_t G,
                                 int64_t g, const float* B, int64_t K, int64_t N, float* C,
                                 int64_t M, int accumulate, int flags, ixb_stream stream) {
  return ixb_guard([&] {
    ixb::spmm_groupcoo(AM, AK, AV, G, g, B, K, N, C, M, accumulate, flags,
                       reinterpret_cast<cudaStream_t>(stream));
  });
}
