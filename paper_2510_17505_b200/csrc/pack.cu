// Device-side format builders (K1 GroupCOO, K2 BlockGroupCOO, rank-n
// grouping) and the group-size tuner. Outputs reproduce the reference
// builders bit-for-bit (formats.cpp:24-46, 115-174, 224-292, 417-479;
// tuner.cpp:31-118).
//
// Two grouping engines, both HBM-bound integer work:
//  * dense-row engine (dense source, group_dim 0): one warp per row counts
//    the row's nonzeros with 16-byte loads (occ), two scans give row and
//    group offsets, and a second warp-per-row pass compacts the nonzeros in
//    column order straight into their (group, slot) — the sort of
//    formats.cpp:124-129 is the identity for a row-major scan.
//  * sorted-run engine (COO / rank-n sources): stable LSD radix sort of a
//    permutation over the key dims (CUB, stable per pass ⇒ lexicographic and
//    stable like std::stable_sort), head flags + scans for the runs of equal
//    group coordinate, then element-parallel slot writes.
// Padding repeats the last real member and stores value 0 / mask 0
// (formats.cpp:155-160, 454-468).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <cmath>
#include <memory>
#include <vector>

#include "common.cuh"

namespace ixb {

// ------------------------------------------------------------------ tuner
struct OccStats {
  unsigned long long S = 0, nonzero = 0, maxocc = 0;
  unsigned long long groups_pow2[32] = {};  // sum_r ceil(occ_r / 2^i)
};

namespace {

constexpr int kTB = 256;

// One pass over the occupancy counts: S, non-empty rows, max, and
// sum_r ceil(occ_r / 2^i) for every i (all candidate F(g) at once). Each
// thread reduces its rows in registers, warps reduce by shuffles, one smem
// atomic per warp per statistic, one global atomic per CTA per statistic.
__global__ void occ_stats_kernel(const int32_t* occ, int64_t n, OccStats* out) {
  __shared__ unsigned long long part[kTB / 32][35];
  // 32-bit per-thread partials (a warp's rows hold < 2^32 nonzeros: int32
  // coordinates), warp sums by REDUX (__reduce_*_sync: one instruction per
  // statistic instead of five 64-bit shuffle rounds), 64-bit from smem on;
  // grp[i] is warp-uniform after the reduction: lane i stores it
  unsigned S = 0, nz = 0, mx = 0, grp[32] = {};
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < n;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned o = static_cast<unsigned>(occ[r]);
    S += o;
    nz += o > 0;
    mx = o > mx ? o : mx;
#pragma unroll
    for (int i = 0; i < 32; ++i) grp[i] += static_cast<unsigned>(
        (static_cast<unsigned long long>(o) + (1ull << i) - 1) >> i);
  }
  S = __reduce_add_sync(0xffffffffu, S);
  nz = __reduce_add_sync(0xffffffffu, nz);
  mx = __reduce_max_sync(0xffffffffu, mx);
#pragma unroll
  for (int i = 0; i < 32; ++i) grp[i] = __reduce_add_sync(0xffffffffu, grp[i]);
  // per-warp partials to smem, then 35 threads each sum one statistic over
  // the CTA's warps (no shared-memory atomics) and do one global atomic
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    part[w][0] = S;
    part[w][1] = nz;
    part[w][2] = mx;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (lane == i) part[w][3 + i] = grp[i];
  __syncthreads();
  const int nw = blockDim.x >> 5;
  if (threadIdx.x < 35) {
    unsigned long long v = 0;
    for (int k = 0; k < nw; ++k) {
      const unsigned long long x = part[k][threadIdx.x];
      v = threadIdx.x == 2 ? (x > v ? x : v) : v + x;
    }
    if (threadIdx.x == 2) atomicMax(&out->maxocc, v);
    else if (v) atomicAdd(threadIdx.x < 2 ? (threadIdx.x == 0 ? &out->S : &out->nonzero)
                                          : &out->groups_pow2[threadIdx.x - 3], v);
  }
}

}  // namespace

// select() of tuner.cpp:100-118 from the occupancy statistics (host or
// device: IEEE double sqrt/division, the same result either side).
// g_star (tuner.cpp:60-65) and candidate_group_sizes (tuner.cpp:67-84): the
// power-of-two candidates lo <= hi around g_star, capped by the largest
// occupancy; S == 0 gives {1}.
__host__ __device__ void tuner_candidates(unsigned long long S, unsigned long long nonzero,
                                          unsigned long long maxocc, int64_t extent,
                                          int count_empty_rows, double* gs_out, int64_t* lo_out,
                                          int64_t* hi_out) {
  double gs = 1.0;
  if (S > 0) {
    double nn = count_empty_rows ? static_cast<double>(extent) : static_cast<double>(nonzero);
    gs = nn <= 0 ? 1.0 : sqrt(static_cast<double>(S) / nn);
  }
  *gs_out = gs;
  if (S == 0) {
    *lo_out = *hi_out = 1;
    return;
  }
  int64_t lo = 1;
  while (lo * 2 <= static_cast<int64_t>(gs)) lo *= 2;
  int64_t hi = lo;
  while (static_cast<double>(hi) < gs) hi *= 2;
  int64_t cap = 1;
  while (cap * 2 <= static_cast<int64_t>(maxocc)) cap *= 2;
  *lo_out = lo < 1 ? 1 : (lo > cap ? cap : lo);
  *hi_out = hi < 1 ? 1 : (hi > cap ? cap : hi);
}

__host__ __device__ int64_t choose_group_size(const OccStats& h, int64_t extent,
                                              int count_empty_rows, double* gstar_out,
                                              int64_t* cand_g, double* cand_score, int* ncand) {
  double gs;
  int64_t lo, hi;
  tuner_candidates(h.S, h.nonzero, h.maxocc, extent, count_empty_rows, &gs, &lo, &hi);
  if (gstar_out) *gstar_out = gs;
  if (h.S == 0) {  // candidate_group_sizes: {1}
    if (ncand) {
      *ncand = 1;
      cand_g[0] = 1;
      cand_score[0] = 2.0 * static_cast<double>(h.groups_pow2[0]);
    }
    return 1;
  }
  auto cost = [&](int64_t g) {  // cost_exact (tuner.cpp:31-36), g a power of two
    int sh = 0;
    while ((1ll << sh) < g) ++sh;
    return static_cast<double>((g + 1) * static_cast<int64_t>(h.groups_pow2[sh]));
  };
  int64_t chosen = lo;
  double best = cost(lo);
  if (hi != lo && cost(hi) < best) chosen = hi;
  if (ncand) {
    *ncand = hi == lo ? 1 : 2;
    cand_g[0] = lo;
    cand_score[0] = cost(lo);
    if (hi != lo) {
      cand_g[1] = hi;
      cand_score[1] = cost(hi);
    }
  }
  return chosen;
}


// select() of tuner.cpp:100-118 over device occupancy counts.
int64_t tune_from_occ(const int32_t* occ, int64_t n, int64_t extent, int count_empty_rows,
                      cudaStream_t s, double* gstar_out, int64_t* cand_g = nullptr,
                      double* cand_score = nullptr, int* ncand = nullptr,
                      int64_t* total_out = nullptr, int64_t* maxocc_out = nullptr) {
  Scratch<OccStats> d(1, s);
  IXB_CUDA_CHECK(cudaMemsetAsync(d.p, 0, sizeof(OccStats), s));
  if (n > 0) {
    // one row per thread up to two CTAs per SM (latency-bound for short
    // profiles), grid-stride beyond; one global atomic per statistic per CTA
    int64_t grid = ceil_div(n, kTB);
    if (grid > 2 * sm_count()) grid = 2 * sm_count();
    occ_stats_kernel<<<grid, kTB, 0, s>>>(occ, n, d.p);
    IXB_LAUNCH_CHECK("occ_stats_kernel");
  }
  OccStats h;
  HostReads rd(s);
  rd.add(&h, d.p, sizeof h);
  rd.wait();
  if (total_out) *total_out = static_cast<int64_t>(h.S);
  if (maxocc_out) *maxocc_out = static_cast<int64_t>(h.maxocc);
  return choose_group_size(h, extent, count_empty_rows, gstar_out, cand_g, cand_score, ncand);
}

namespace {

// ------------------------------------------------------------ elem helpers
template <typename T>
__device__ __forceinline__ bool nz(T v);
template <>
__device__ __forceinline__ bool nz<float>(float v) { return v != 0.0f; }
template <>
__device__ __forceinline__ bool nz<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v) != 0.0f;
}
template <>
__device__ __forceinline__ bool nz<uint8_t>(uint8_t v) { return v != 0; }
template <>
__device__ __forceinline__ bool nz<double>(double v) { return v != 0.0; }
template <>
__device__ __forceinline__ bool nz<int64_t>(int64_t v) { return v != 0; }

// Dense-source element types: fp32, bf16, fp64 (u8 for block flags).
template <typename F>
void dispatch_dense(int dtype, F&& f) {
  if (dtype == IXB_F32) f(float{});
  else if (dtype == IXB_BF16) f(__nv_bfloat16{});
  else if (dtype == IXB_F64) f(double{});
  else if (dtype == IXB_I64) f(int64_t{});
  else f(uint8_t{});
}
void check_dense_dtype(int dtype) {
  if (dtype != IXB_F32 && dtype != IXB_BF16 && dtype != IXB_F64 && dtype != IXB_I64)
    fail(IXB_FAILURE, "unsupported dtype");
}
int dense_bytes(int dtype) {
  return dtype == IXB_BF16 ? 2 : (dtype == IXB_F64 || dtype == IXB_I64) ? 8 : 4;
}

template <typename T>
struct alignas(16) Vec16 {
  static constexpr int V = 16 / sizeof(T);
  T x[V];
};

// occ[row] = number of nonzeros of row `row` (formats.cpp:33-41 scan order).
// Long rows are cut into nseg segments of seg columns, one warp each: the
// segment's count goes to occ_seg[row * nseg + seg] and is added to occ[row]
// (zeroed by the caller); nseg == 1 stores occ[row] directly.
template <typename T, int V>
__global__ void row_count_kernel(const T* __restrict__ dense, int64_t rows, int64_t cols,
                                 int64_t nseg, int64_t seg, int32_t* occ, int32_t* occ_seg) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= rows * nseg) return;
  const int64_t row = w / nseg, c0 = (w % nseg) * seg;
  const int64_t c1 = c0 + seg < cols ? c0 + seg : cols;
  const int lane = lane_id();
  const T* p = dense + row * cols;
  int cnt = 0;
#pragma unroll 4
  for (int64_t c = c0 + static_cast<int64_t>(lane) * V; c < c1; c += 32 * V) {
    if (V > 1) {
      Vec16<T> v = *reinterpret_cast<const Vec16<T>*>(p + c);
#pragma unroll
      for (int j = 0; j < (V > 1 ? V : 1); ++j) cnt += nz<T>(v.x[j]);
    } else {
      cnt += nz<T>(p[c]);
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) {
    if (nseg == 1) {
      occ[row] = cnt;
    } else {
      occ_seg[w] = cnt;
      if (cnt) atomicAdd(&occ[row], cnt);
    }
  }
}

// Dense-row pack. mode 0: GroupCOO slots (gofs, g); mode 1: plain COO at rowptr.
// One warp per (row, segment) as in row_count_kernel: the segment's first
// entry index in the row is the sum of the earlier segments' counts; the
// warp of the row's last non-empty segment also writes AM and the padding.
template <typename T, int V>
__global__ void __launch_bounds__(256, 4) row_pack_kernel(const T* __restrict__ dense, int64_t rows, int64_t cols,
                                int64_t nseg, int64_t seg, const int32_t* __restrict__ occ,
                                const int32_t* __restrict__ occ_seg,
                                const int32_t* __restrict__ offs,  // gofs (mode 0) / rowptr (1)
                                int64_t g, int mode, int32_t* AM, int32_t* AK, T* AV,
                                uint8_t* mask) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= rows * nseg) return;
  const int64_t row = w / nseg;
  const int sg = static_cast<int>(w % nseg);
  const int lane = lane_id();
  const int64_t c_lo = static_cast<int64_t>(sg) * seg;
  const int64_t c_hi = c_lo + seg < cols ? c_lo + seg : cols;
  const T* p = dense + row * cols;
  // batches of kB chunks of 32 * V columns: the kB 16-byte loads of a lane
  // are in flight together; the first batch is issued before the row's
  // metadata arrives
  constexpr int kB = 4;
  static_assert(32 * V < 65536, "16-bit count fields");
  auto load_batch = [&](T (&vals)[kB][V], int64_t cb) {
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int64_t c = cb + u * 32 * V;
      if (V > 1) {
        if (c < c_hi) {
          Vec16<T> v = *reinterpret_cast<const Vec16<T>*>(p + c);
#pragma unroll
          for (int j = 0; j < V; ++j) vals[u][j] = v.x[j];
        } else {
#pragma unroll
          for (int j = 0; j < V; ++j) vals[u][j] = T(0);
        }
      } else {
        vals[u][0] = c < c_hi ? p[c] : T(0);
      }
    }
  };
  T vals[kB][V];
  int64_t cb = c_lo + static_cast<int64_t>(lane) * V;
  load_batch(vals, cb);
  const int n = occ[row];
  const int cs = nseg > 1 && lane < nseg ? occ_seg[row * nseg + lane] : 0;
  const int64_t base = offs[row];
  if (n == 0) return;
  int64_t k0 = 0;
  bool last_seg = true;
  if (nseg > 1) {  // nseg <= 32: one count per lane
    if (__shfl_sync(0xffffffffu, cs, sg) == 0) return;
    k0 = __reduce_add_sync(0xffffffffu, lane < sg ? cs : 0);
    last_seg = __ballot_sync(0xffffffffu, lane > sg && cs > 0) == 0;
  }
  int last_col = 0;
  // The compacted entries go through a per-warp shared staging buffer and
  // leave as contiguous runs (each lane-level store a whole sector's worth
  // per warp): scattered per-lane stores made the pack L2-store-bound.
  constexpr int kPerBatch = kB * 32 * V;
  constexpr bool kChunkFlush = kPerBatch > 512;
  constexpr int kStage = kChunkFlush ? 32 * V : kPerBatch;
  __shared__ int32_t s_col[kTB / 32][kStage];
  __shared__ T s_val[kTB / 32][kStage];
  const int wib = threadIdx.x >> 5;
  int32_t* st_col = s_col[wib];
  T* st_val = s_val[wib];
  auto flush = [&](int& staged) {
    __syncwarp();
    for (int r = lane; r < staged; r += 32) {
      const int64_t k = k0 + r;
      if (mode == 0) {  // slot (base + k / g) * g + k % g = base * g + k
        const int64_t slot = base * g + k;
        AK[slot] = st_col[r];
        if (AV) AV[slot] = st_val[r];
        if (mask) mask[slot] = 1;
      } else {
        AM[base + k] = static_cast<int32_t>(row);
        AK[base + k] = st_col[r];
        if (AV) AV[base + k] = st_val[r];
      }
    }
    __syncwarp();
    k0 += staged;
    staged = 0;
  };
  for (bool first = true; cb - lane * V < c_hi; cb += kB * 32 * V, first = false) {
    if (!first) load_batch(vals, cb);
    // one warp scan for the kB chunks: their per-lane counts packed as
    // 16-bit fields (chunks 0, 1 in lo; 2, 3 in hi)
    int cnt[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      cnt[u] = 0;
#pragma unroll
      for (int j = 0; j < V; ++j) cnt[u] += nz<T>(vals[u][j]);
    }
    const uint32_t plo = static_cast<uint32_t>(cnt[0]) | (static_cast<uint32_t>(cnt[1]) << 16);
    const uint32_t phi = static_cast<uint32_t>(cnt[2]) | (static_cast<uint32_t>(cnt[3]) << 16);
    if (!__any_sync(0xffffffffu, (plo | phi) != 0)) continue;  // an all-zero batch
    uint32_t ilo = plo, ihi = phi;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t tl = __shfl_up_sync(0xffffffffu, ilo, o);
      const uint32_t th = __shfl_up_sync(0xffffffffu, ihi, o);
      if (lane >= o) {
        ilo += tl;
        ihi += th;
      }
    }
    const uint32_t tlo = __shfl_sync(0xffffffffu, ilo, 31), thi = __shfl_sync(0xffffffffu, ihi, 31);
    const uint32_t elo = ilo - plo, ehi = ihi - phi;  // exclusive
    int my_last = -1;
    int staged = 0;  // entries staged since the last flush (warp-uniform)
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const uint32_t tot_f = u < 2 ? tlo : thi, ex_f = u < 2 ? elo : ehi;
      const int sh = 16 * (u & 1);
      const int total = static_cast<int>((tot_f >> sh) & 0xFFFFu);
      if (total == 0) continue;  // warp-uniform
      int r = staged + static_cast<int>((ex_f >> sh) & 0xFFFFu);
      const int64_t c = cb + u * 32 * V;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (!nz<T>(vals[u][j])) continue;
        const int col = static_cast<int>(c + j);
        st_col[r] = col;
        st_val[r] = vals[u][j];
        my_last = col;
        ++r;
      }
      staged += total;
      if (kChunkFlush || u == kB - 1) flush(staged);
    }
    if (!kChunkFlush && staged) flush(staged);
    // the row's last nonzero so far: the largest column any lane wrote
    const int bl = __reduce_max_sync(0xffffffffu, my_last);
    if (bl >= 0) last_col = bl;
  }
  if (mode == 0 && last_seg) {
    const int64_t ng = (n + g - 1) / g;
    for (int64_t j = lane; j < ng; j += 32) AM[base + j] = static_cast<int32_t>(row);
    const int64_t real_last = n - (ng - 1) * g;  // real entries in the last group
    const int64_t lastg = base + ng - 1;
    for (int64_t q = real_last + lane; q < g; q += 32) {
      const int64_t slot = lastg * g + q;
      AK[slot] = last_col;
      if (AV) AV[slot] = T(0);
      if (mask) mask[slot] = 0;
    }
  }
}

// occupancy() (formats.cpp:96-103): histogram of a coordinate array. Small
// extents (the 27 kernel offsets of a conv map, the paths of a CG table) are
// counted in a per-CTA shared-memory histogram, grid-stride, and merged with
// one global atomic per non-empty bin per CTA; large extents (matrix rows)
// have little contention and count straight into global memory.
constexpr int kOccSmemBins = 8192;
__global__ void occupancy_kernel(const int32_t* c, int64_t n, int64_t ext, int32_t* o) {
  __shared__ int32_t h[kOccSmemBins];
  const bool small = ext <= kOccSmemBins;
  if (small) {
    for (int64_t b = threadIdx.x; b < ext; b += blockDim.x) h[b] = 0;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  auto add = [&](int32_t v, int cnt) {
    if (v < 0 || v >= ext) return;
    if (small) atomicAdd(h + v, cnt);
    else atomicAdd(o + v, cnt);
  };
  int64_t done = 0;
  if (small && (reinterpret_cast<uintptr_t>(c) & 15) == 0) {
    // 16-byte loads, whole warps (the lanes stay converged): a warp whose
    // 128 values are all equal (sorted input: nearly every warp) adds once,
    // a lane whose 4 values are equal adds once
    const int64_t n4 = n / 4;
    for (int64_t base = (tid >> 5) * 32; base < n4; base += (nthreads >> 5) * 32) {
      const int64_t q = base + lane;
      const int4 x = q < n4 ? reinterpret_cast<const int4*>(c)[q] : make_int4(-1, -1, -1, -1);
      const int32_t v0 = __shfl_sync(0xffffffffu, x.x, 0);
      const bool eq = x.x == x.y && x.y == x.z && x.z == x.w;  // the lane's four values
      if (__all_sync(0xffffffffu, eq && x.x == v0 && q < n4)) {
        if (lane == 0) add(v0, 128);
      } else if (q < n4) {
        if (eq) {
          add(x.x, 4);
        } else {
          add(x.x, 1);
          add(x.y, 1);
          add(x.z, 1);
          add(x.w, 1);
        }
      }
    }
    done = n4 * 4;
  }
  for (int64_t i = done + tid; i < n; i += nthreads) add(c[i], 1);
  if (small) {
    __syncthreads();
    for (int64_t b = threadIdx.x; b < ext; b += blockDim.x)
      if (h[b]) atomicAdd(o + b, h[b]);
  }
}
// brute_force_optimal (tuner.cpp:86-97): F(g) = (g+1) * sum_i ceil(occ_i / g)
// for every g in [1, maxocc]; a CTA per g (grid-stride), threads over rows.
__global__ void brute_cost_kernel(const int32_t* occ, int64_t n, int64_t maxocc,
                                  unsigned long long* F) {
  __shared__ unsigned long long red[kWarp];
  for (int64_t g = blockIdx.x + 1; g <= maxocc; g += gridDim.x) {
    unsigned long long sum = 0;
    for (int64_t r = threadIdx.x; r < n; r += blockDim.x)
      sum += (static_cast<unsigned long long>(occ[r]) + g - 1) / g;
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
      F[g - 1] = static_cast<unsigned long long>(g + 1) * t;
    }
    __syncthreads();
  }
}

void launch_occupancy(const int32_t* coord, int64_t nnz, int64_t extent, int32_t* occ,
                      cudaStream_t s) {
  int64_t grid = ceil_div(nnz, kTB);
  if (extent <= kOccSmemBins && grid > 6 * sm_count()) grid = 6 * sm_count();
  occupancy_kernel<<<static_cast<unsigned>(grid), kTB, 0, s>>>(coord, nnz, extent, occ);
  IXB_LAUNCH_CHECK("occupancy_kernel");
}

// ---------------------------------------------------------- sorted runs
__global__ void iota32(int32_t* x, int64_t n) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = static_cast<int32_t>(i);
}

__global__ void gather_key(const int32_t* coord, const int32_t* perm, int64_t n, int32_t* key) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) key[i] = coord[perm[i]];
}

// Head flag of sorted position i (a run of equal group coordinate starts
// there), computed inside the scan's input iterator: no flag array.
struct HeadFlag {
  const int32_t* gcoord;
  const int32_t* perm;
  __host__ __device__ int operator()(int64_t i) const {
    if (i == 0) return 1;
    return gcoord[perm ? perm[i] : i] != gcoord[perm ? perm[i - 1] : i - 1] ? 1 : 0;
  }
};

__global__ void run_starts(const int32_t* run_incl, int64_t n, int32_t* start) {
  int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && (i == 0 || run_incl[i] != run_incl[i - 1]))
    start[run_incl[i] - 1] = static_cast<int32_t>(i);
}

__global__ void run_lengths(const int32_t* start, int64_t R, int64_t n, int32_t* len) {
  int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < R) len[r] = (r + 1 < R ? start[r + 1] : static_cast<int32_t>(n)) - start[r];
}

struct RunPackArgs {
  const int32_t* perm;      // sorted pos -> source (null = identity)
  const int32_t* run_incl;  // inclusive run count per sorted pos (run id + 1); null:
                            // runs indexed by group coordinate value
  const int32_t* start;     // [R]
  const int32_t* len;       // [R]
  const int32_t* gofs;      // [R] exclusive group offsets
  const int32_t* gcoord;    // source group coordinates
  const int32_t* mcoord[8]; // source member coordinates
  int32_t* mout[8];         // member outputs [G, g]
  int nm;
  int64_t n, R, g;
  const void* vals;
  void* vout;
  int vbytes;  // 0 (no values), 2 (bf16), 4 (f32) or 8 (f64 / i64, copied bitwise)
  uint8_t* mask;
  int32_t* gout;  // group coordinate output [G]
};

// kPackElems consecutive-by-stride entries per thread, in two phases: every
// load of the thread's entries is issued before any store (the outputs may
// alias the inputs as far as the compiler knows, so interleaved load/store
// pairs would serialise each entry's loads behind the previous stores).
constexpr int kPackElems = 4;
constexpr int kMaxMembers = 8;
__global__ void __launch_bounds__(kTB) run_pack_elems(RunPackArgs a) {
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * kTB * kPackElems + threadIdx.x;
  int64_t slot[kPackElems];
  int32_t mc[kPackElems][kMaxMembers];
  unsigned long long v[kPackElems];
#pragma unroll
  for (int u = 0; u < kPackElems; ++u) {
    const int64_t i = i0 + u * kTB;
    slot[u] = -1;
    if (i < a.n) {
      // runs by rank (run_incl) or, for canonical small-extent input, by value
      const int64_t r = a.run_incl ? a.run_incl[i] - 1 : a.gcoord[i];
      const int64_t k = i - a.start[r];
      slot[u] = static_cast<int64_t>(a.gofs[r]) * a.g + k;  // = (gofs + k / g) * g + k % g
      const int64_t src = a.perm ? a.perm[i] : i;
#pragma unroll
      for (int m = 0; m < kMaxMembers; ++m)
        if (m < a.nm) mc[u][m] = a.mcoord[m][src];
      if (a.vbytes == 8) v[u] = static_cast<const unsigned long long*>(a.vals)[src];
      else if (a.vbytes == 4) v[u] = __float_as_uint(static_cast<const float*>(a.vals)[src]);
      else if (a.vbytes == 2)
        v[u] = static_cast<const unsigned short*>(a.vals)[src];  // bf16 bits
    }
  }
#pragma unroll
  for (int u = 0; u < kPackElems; ++u) {
    if (slot[u] < 0) continue;
    const int64_t sl = slot[u];
#pragma unroll
    for (int m = 0; m < kMaxMembers; ++m)
      if (m < a.nm) a.mout[m][sl] = mc[u][m];
    if (a.vbytes == 8) static_cast<unsigned long long*>(a.vout)[sl] = v[u];
    else if (a.vbytes == 4) static_cast<unsigned*>(a.vout)[sl] = static_cast<unsigned>(v[u]);
    else if (a.vbytes == 2)
      static_cast<unsigned short*>(a.vout)[sl] = static_cast<unsigned short>(v[u]);
    if (a.mask) a.mask[sl] = 1;
  }
}

// Per run: its group coordinates and the pad slots of its last group.
// `cta`: one CTA per run, threads striding the run's groups and pads (few
// long runs, e.g. the 27 offsets of a kernel map); otherwise one thread per
// run (many short runs).
__global__ void run_pack_runs(RunPackArgs a, int cta) {
  const int64_t r = cta ? blockIdx.x : static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= a.R) return;
  const int64_t t0 = cta ? threadIdx.x : 0, dt = cta ? blockDim.x : 1;
  const int64_t len = a.len[r];
  if (len == 0) return;  // a value with no entries (value-indexed runs)
  const int64_t ng = (len + a.g - 1) / a.g;
  const int64_t g0 = a.gofs[r];
  const int64_t first = a.start[r], last = first + len - 1;
  const int64_t src0 = a.perm ? a.perm[first] : first;
  const int64_t srcl = a.perm ? a.perm[last] : last;
  const int32_t gc = a.gcoord[src0];
  for (int64_t j = t0; j < ng; j += dt) a.gout[g0 + j] = gc;
  const int64_t real_last = len - (ng - 1) * a.g;
  for (int64_t q = real_last + t0; q < a.g; q += dt) {
    const int64_t slot = (g0 + ng - 1) * a.g + q;
    for (int m = 0; m < a.nm; ++m) a.mout[m][slot] = a.mcoord[m][srcl];
    if (a.vbytes == 8) static_cast<unsigned long long*>(a.vout)[slot] = 0ull;  // 0.0 / 0
    else if (a.vbytes == 4) static_cast<float*>(a.vout)[slot] = 0.f;
    else if (a.vbytes == 2)
      static_cast<__nv_bfloat16*>(a.vout)[slot] = __float2bfloat16(0.f);
    if (a.mask) a.mask[slot] = 0;
  }
}

// ------------------------------------------------------------- blocks (K2)
template <typename T>
__global__ void block_flags_kernel(const T* __restrict__ dense, int64_t rows, int64_t cols,
                                   int64_t bm, int64_t bk, int64_t gr, int64_t gcn,
                                   uint8_t* flags) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= gr * gcn) return;
  const int64_t br = b / gcn, bc = b % gcn;
  const int64_t ie = (br + 1) * bm < rows ? (br + 1) * bm : rows;
  const int64_t je = (bc + 1) * bk < cols ? (bc + 1) * bk : cols;
  bool any = false;
  for (int64_t i = br * bm; i < ie && !any; ++i) {
    const T* p = dense + i * cols;
    for (int64_t j = bc * bk; j < je; ++j) any |= nz<T>(p[j]);
  }
  flags[b] = any ? 1 : 0;
}

// Vectorised block flags: a warp covers one block row and 32 16-byte column
// chunks (32 * 16 / (bk * sizeof(T)) consecutive blocks), walking the block's
// bm rows with coalesced 512-byte loads; the lanes of one block OR their
// "any nonzero" bits by shuffles. Needs bk * sizeof(T) to divide 512 and 16-byte
// aligned rows (the shape check is on the host); ragged edges are masked.
// With `occ`, the warp also adds its nonzero-block count to occ[block row]
// (the block row occupancy the grouping needs: no separate count pass).
template <typename T>
__global__ void block_flags_vec_kernel(const T* __restrict__ dense, int64_t rows, int64_t cols,
                                       int64_t bm, int64_t bk, int64_t gr, int64_t gcn,
                                       uint8_t* flags, int32_t* occ) {
  constexpr int V = 16 / sizeof(T);  // elements per chunk
  const int lane = lane_id();
  const int cpb = static_cast<int>(bk / V);  // chunks per block row segment
  const int bpw = 32 / cpb;                  // blocks per warp
  const int64_t warps_per_row = (gcn + bpw - 1) / bpw;
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (w >= gr * warps_per_row) return;
  const int64_t br = w / warps_per_row;
  const int64_t bc = (w % warps_per_row) * bpw + lane / cpb;
  const int64_t c0 = bc * bk + static_cast<int64_t>(lane % cpb) * V;
  const bool in = bc < gcn && c0 < cols;
  const int64_t ie = (br + 1) * bm < rows ? (br + 1) * bm : rows;
  bool any = false;
  if (in) {
    if (c0 + V <= cols) {
#pragma unroll 4
      for (int64_t i = br * bm; i < ie; ++i) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(dense + i * cols + c0));
        const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int j = 0; j < V; ++j) any |= nz<T>(e[j]);
      }
    } else {
      for (int64_t i = br * bm; i < ie; ++i)
        for (int64_t j = c0; j < cols; ++j) any |= nz<T>(dense[i * cols + j]);
    }
  }
  unsigned m = __ballot_sync(0xffffffffu, any);
  const int first = (lane / cpb) * cpb;
  const unsigned mine = (m >> first) & ((cpb == 32 ? 0u : (1u << cpb)) - 1u);
  const bool f = (cpb == 32 ? m : mine) != 0;
  if (in && lane % cpb == 0) flags[br * gcn + bc] = f ? 1 : 0;
  if (occ) {
    const unsigned nzb = __ballot_sync(0xffffffffu, in && lane % cpb == 0 && f);
    if (lane == 0 && nzb) atomicAdd(&occ[br], __popc(nzb));
  }
}

// Fused block-row pack (group_dim 0, 16-byte vector rows): one CTA per
// block row. Per tile of 16 * kTB block flags the CTA lists the row's
// nonzero blocks in column order (block scan) into shared memory, writes
// their AK/mask slots and copies their bm x bk values into AV with all
// threads (independent 16-byte loads, several in flight per thread); then
// AM and the padded tail of the row's last group. Replaces row_pack over
// the flags + a warp-per-slot block copy.
template <typename T>
__global__ void __launch_bounds__(kTB) block_row_pack_kernel(
    const T* __restrict__ dense, int64_t rows, int64_t cols, int64_t bm, int64_t bk, int64_t gcn,
    const uint8_t* __restrict__ flags, const int32_t* __restrict__ occ,
    const int32_t* __restrict__ gofs, int64_t g, int32_t* AM, int32_t* AK, T* AV, uint8_t* mask) {
  constexpr int V = 16 / sizeof(T);
  constexpr int kTile = 16 * kTB;
  __shared__ int32_t list[kTile];
  __shared__ int wsum[kTB / 32];
  __shared__ int last_col_s;
  const int64_t br = blockIdx.x;
  const int n = occ[br];
  if (n == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = gofs[br];
  const uint8_t* frow = flags + br * gcn;
  const int cpr = static_cast<int>(bk / V);             // 16-byte chunks per block row
  const int cpb = static_cast<int>(bm) * cpr;           // chunks per block
  const int64_t blk = bm * bk;                          // elements per block
  int64_t k0 = 0;
  for (int64_t t0 = 0; t0 < gcn; t0 += kTile) {
    // 16 flags per thread (byte loads: rows of flags need not be aligned)
    uint32_t bits = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int64_t c = t0 + tid * 16 + q;
      if (c < gcn && frow[c]) bits |= 1u << q;
    }
    const int mine = __popc(bits);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int wbase = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kTB / 32; ++w) {
      const int v = wsum[w];
      if (w < warp) wbase += v;
      tot += v;
    }
    int k = wbase + incl - mine;
    for (uint32_t b = bits; b; b &= b - 1) list[k++] = static_cast<int32_t>(t0 + tid * 16 + __ffs(b) - 1);
    __syncthreads();
    for (int i = tid; i < tot; i += kTB) {
      const int64_t kk = k0 + i;
      const int64_t slot = base * g + kk;  // = (base + kk / g) * g + kk % g
      AK[slot] = list[i];
      if (mask) mask[slot] = 1;
    }
    if (tot > 0 && tid == 0) last_col_s = list[tot - 1];
    if (AV) {
      // 4 independent 16-byte loads in flight per thread before their stores
      const int nchunks = tot * cpb;
      for (int e0 = tid; e0 < nchunks; e0 += 4 * kTB) {
        uint4 v[4];
        T* dst[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * kTB;
          v[u] = make_uint4(0, 0, 0, 0);
          dst[u] = nullptr;
          if (e < nchunks) {
            const int i = e / cpb, c = e - i * cpb;
            const int r = c / cpr, j = (c - r * cpr) * V;
            const int kk = static_cast<int>(k0) + i;
            const int64_t slot = base * g + kk;  // = (base + kk / g) * g + kk % g
            const int64_t si = br * bm + r, sj = static_cast<int64_t>(list[i]) * bk + j;
            if (si < rows && sj < cols)
              v[u] = __ldg(reinterpret_cast<const uint4*>(dense + si * cols + sj));
            dst[u] = AV + slot * blk + r * bk + j;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (dst[u]) *reinterpret_cast<uint4*>(dst[u]) = v[u];
      }
    }
    k0 += tot;
    __syncthreads();  // list and wsum reused by the next tile
  }
  const int64_t ng = (n + g - 1) / g;
  for (int64_t j = tid; j < ng; j += kTB) AM[base + j] = static_cast<int32_t>(br);
  const int64_t real_last = n - (ng - 1) * g;  // real entries in the last group
  const int64_t lastg = base + ng - 1;
  const int lc = last_col_s;
  for (int64_t q = real_last + tid; q < g; q += kTB) {
    const int64_t slot = lastg * g + q;
    AK[slot] = lc;
    if (mask) mask[slot] = 0;
  }
  if (AV) {
    const int64_t z0 = (lastg * g + real_last) * blk, z1 = (lastg + 1) * g * blk;  // pad values
    for (int64_t e = z0 + static_cast<int64_t>(tid) * V; e < z1; e += static_cast<int64_t>(kTB) * V)
      *reinterpret_cast<uint4*>(AV + e) = make_uint4(0, 0, 0, 0);
  }
}

// Block copy: one warp per slot, 16-byte chunks (bk * sizeof(T) a multiple of
// 16, 16-byte aligned rows); pad slots and ragged edges are zero-filled.
template <typename T>
__global__ void block_copy_kernel(const T* __restrict__ dense, int64_t rows, int64_t cols,
                                  int64_t bm, int64_t bk, int group_dim, const int32_t* AM,
                                  const int32_t* AK, const uint8_t* mask, int64_t slots, int64_t g,
                                  T* AV, int vec) {
  const int64_t slot = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (slot >= slots) return;
  const int lane = lane_id();
  T* dst = AV + slot * bm * bk;
  const bool real = mask[slot] != 0;
  const int64_t p = slot / g;
  const int64_t rb = group_dim == 0 ? AM[p] : AK[slot];
  const int64_t cb = group_dim == 0 ? AK[slot] : AM[p];
  if (vec) {
    constexpr int V = 16 / sizeof(T);
    const int64_t cpr = bk / V;  // chunks per block row
    for (int64_t e = lane; e < bm * cpr; e += 32) {
      const int64_t i = e / cpr, j = (e % cpr) * V;
      const int64_t si = rb * bm + i, sj = cb * bk + j;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (real && si < rows) {
        if (sj + V <= cols) {
          v = __ldg(reinterpret_cast<const uint4*>(dense + si * cols + sj));
        } else {
          T* t = reinterpret_cast<T*>(&v);
          for (int k = 0; k < V; ++k)
            if (sj + k < cols) t[k] = dense[si * cols + sj + k];
        }
      }
      *reinterpret_cast<uint4*>(dst + i * bk + j) = v;
    }
    return;
  }
  for (int64_t e = lane; e < bm * bk; e += 32) {
    const int64_t i = e / bk, j = e % bk;
    const int64_t si = rb * bm + i, sj = cb * bk + j;
    T v = T(0);
    if (real && si < rows && sj < cols) v = dense[si * cols + sj];
    dst[e] = v;
  }
}

}  // namespace
}  // namespace ixb

// =========================================================== the plan object
struct ixb_pack {
  int type = 0;  // 1 dense-row grouping, 2 dense_to_coo, 3 sorted-run grouping, 4 blocks, 5 kmap
  cudaStream_t s = nullptr;
  int64_t nnz = 0, G = 0, g = 1, R = 0;
  int group_dim = 0, rank = 2, dtype = IXB_F32;
  // dense sources
  const void* dense = nullptr;
  int64_t rows = 0, cols = 0;
  ixb::Scratch<int32_t> occ, offs;  // per row: occupancy, group/row offsets
  ixb::Scratch<int32_t> occ_seg;    // per (row, column segment) counts when nseg > 1
  int64_t nseg = 1, seg = 0;
  // sorted-run engine
  std::vector<const int32_t*> coords;  // rank source coordinate arrays
  ixb::Scratch<int32_t> perm, run_incl, start, len, gofs;
  // blocks
  int64_t bm = 1, bk = 1, gr = 0, gcn = 0, nblocks = 0;
  ixb::Scratch<uint8_t> flags;
  std::unique_ptr<ixb_pack> inner;
  ixb::Scratch<int32_t> coo_r, coo_c;  // block COO when grouping by columns
  // kernel map
  ixb::Scratch<int32_t> kmap_out, kmap_in, kmap_off;
};

namespace ixb {
namespace {

// Segment width of the count/pack warps: whole chunks of 32 * V columns,
// at least 8 of them, and at most 32 segments per row.
void row_segments(int64_t cols, int V, int64_t* nseg, int64_t* seg) {
  const int64_t chunk = 32 * static_cast<int64_t>(V);
  int64_t sc = 8 * chunk;
  const int64_t need = ceil_div(ceil_div(cols, 32), chunk) * chunk;
  if (need > sc) sc = need;
  *seg = sc;
  *nseg = cols > 0 ? ceil_div(cols, sc) : 1;
}

template <typename T>
void launch_row_count(const T* d, ixb_pack* P) {
  constexpr int V = 16 / sizeof(T);
  const bool vec = P->cols % V == 0 && reinterpret_cast<uintptr_t>(d) % 16 == 0;
  row_segments(P->cols, vec ? V : 1, &P->nseg, &P->seg);
  if (P->rows == 0) return;
  if (P->nseg > 1) {
    P->occ_seg = Scratch<int32_t>(P->rows * P->nseg, P->s);
    IXB_CUDA_CHECK(cudaMemsetAsync(P->occ.p, 0, P->rows * sizeof(int32_t), P->s));
  }
  const int64_t grid = ceil_div(P->rows * P->nseg * 32, kTB);
  if (vec)
    row_count_kernel<T, V><<<grid, kTB, 0, P->s>>>(d, P->rows, P->cols, P->nseg, P->seg, P->occ.p,
                                                   P->occ_seg.p);
  else
    row_count_kernel<T, 1><<<grid, kTB, 0, P->s>>>(d, P->rows, P->cols, P->nseg, P->seg, P->occ.p,
                                                   P->occ_seg.p);
  IXB_LAUNCH_CHECK("row_count_kernel");
}

// P's occupancy (and segments, when count_rows made them) over rows x cols of d.
template <typename T>
void launch_row_pack(const T* d, const ixb_pack* P, const int32_t* offs, int64_t g, int mode,
                     int32_t* AM, int32_t* AK, T* AV, uint8_t* mask, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T);
  if (P->rows == 0) return;
  const bool vec = P->cols % V == 0 && reinterpret_cast<uintptr_t>(d) % 16 == 0;
  // a plan whose occupancy came from elsewhere (block flags) has one segment
  int64_t nseg = P->occ_seg.p ? P->nseg : 1, seg = P->occ_seg.p ? P->seg : P->cols;
  if (seg < 1) seg = 1;
  const int64_t grid = ceil_div(P->rows * nseg * 32, kTB);
  if (vec)
    row_pack_kernel<T, V><<<grid, kTB, 0, s>>>(d, P->rows, P->cols, nseg, seg, P->occ.p,
                                               P->occ_seg.p, offs, g, mode, AM, AK, AV, mask);
  else
    row_pack_kernel<T, 1><<<grid, kTB, 0, s>>>(d, P->rows, P->cols, nseg, seg, P->occ.p,
                                               P->occ_seg.p, offs, g, mode, AM, AK, AV, mask);
  IXB_LAUNCH_CHECK("row_pack_kernel");
}

// Exclusive scan of n counts into out[0..n), with the total in out[n], all on
// the device (no host round trip): out[0] = 0, then an inclusive scan into
// out + 1.
template <typename It>
void exclusive_scan_dev(It in, int64_t n, int32_t* out, cudaStream_t s) {
  IXB_CUDA_CHECK(cudaMemsetAsync(out, 0, 4, s));
  if (n == 0) return;
  size_t tb = 0;
  IXB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tb, in, out + 1, static_cast<int>(n), s));
  Scratch<char> tmp(tb, s);
  IXB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.p, tb, in, out + 1, static_cast<int>(n), s));
  note_launch();
}

// ceil(occ / g): groups of a run (the scan input of the group offsets)
struct GroupsOf {
  int64_t g;
  __host__ __device__ int32_t operator()(int32_t occ) const {
    return static_cast<int32_t>((static_cast<int64_t>(occ) + g - 1) / g);
  }
};

// Short profiles (block rows, matrix rows up to kSmallScan): one CTA scans
// ceil(in / g) (g = 1: the counts themselves) in tiles of 8 per thread and
// writes the total to out[n] — one launch instead of cub's init + scan.
constexpr int kSmallScan = 1 << 16;
__device__ __forceinline__ int groups_of(int occ, int64_t g) {
  // ceil(occ / g), 32-bit: occ < 2^31
  if (g > INT32_MAX) return occ > 0;
  return static_cast<int>((static_cast<uint32_t>(occ) + static_cast<uint32_t>(g) - 1u) /
                          static_cast<uint32_t>(g));
}

__device__ void block_scan_groups(const int32_t* in, int64_t n, int64_t g, int32_t* out,
                                  int* wsum /* smem [32] */) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = blockDim.x >> 5;
  int carry = 0;
  for (int64_t t0 = 0; t0 < n; t0 += 8 * blockDim.x) {
    int v[8], mine = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t i = t0 + tid * 8 + q;
      v[q] = i < n ? groups_of(in[i], g) : 0;
      mine += v[q];
    }
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    int wbase = 0, tot = 0;
    for (int w = 0; w < nw; ++w) {
      const int x = wsum[w];
      wbase += w < warp ? x : 0;
      tot += x;
    }
    int run = carry + wbase + incl - mine;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t i = t0 + tid * 8 + q;
      if (i < n) out[i] = run;
      run += v[q];
    }
    carry += tot;
    __syncthreads();
  }
  if (tid == 0) out[n] = carry;
}

__global__ void __launch_bounds__(1024) small_scan_kernel(const int32_t* in, int64_t n, int64_t g,
                                                          int32_t* out) {
  __shared__ int wsum[32];
  block_scan_groups(in, n, g, out, wsum);
}

// Sum over the CTA of a per-thread unsigned partial (REDUX per warp, then
// warp 0 over the warps' sums in 64 bits); the result is valid in thread 0.
__device__ unsigned long long block_sum(unsigned v, unsigned long long* part /* smem [32] */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = __reduce_add_sync(0xffffffffu, v);
  if (lane == 0) part[w] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (w == 0) {
    t = lane < static_cast<int>(blockDim.x >> 5) ? part[lane] : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;
}

// Short profiles, one launch and one host read for the whole plan step:
// S, the non-empty count and the maximum occupancy; with g_req = 0 the
// tuner's candidates (tuner_candidates, the host's function) and, when they
// differ, F(lo) and F(hi) = sum ceil(occ / g) for just those two (select():
// cost (g + 1) F(g), the smaller wins, lo on a tie — tuner.cpp:100-118);
// then the group offsets ceil(occ / g) scanned into out[0..n]. res = {g, S}.
__global__ void __launch_bounds__(1024) tune_scan_kernel(const int32_t* occ, int64_t n,
                                                         int64_t extent, int count_empty_rows,
                                                         int64_t g_req, int32_t* out,
                                                         int64_t* res) {
  __shared__ unsigned long long part[32];
  __shared__ int wsum[32];
  __shared__ int64_t cand[2];
  __shared__ int64_t g_s;
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned S = 0, nz = 0, mx = 0;
  for (int64_t r = tid; r < n; r += blockDim.x) {
    const unsigned o = static_cast<unsigned>(occ[r]);
    S += o;
    nz += o > 0;
    mx = o > mx ? o : mx;
  }
  const unsigned long long tS = block_sum(S, part);
  const unsigned long long tnz = block_sum(nz, part);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if (lane == 0) part[tid >> 5] = mx;
  __syncthreads();
  if (tid == 0) {
    unsigned long long m = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) m = part[w] > m ? part[w] : m;
    int64_t lo = g_req, hi = g_req;
    if (g_req == 0) {
      double gs;
      tuner_candidates(tS, tnz, m, extent, count_empty_rows, &gs, &lo, &hi);
    }
    cand[0] = lo;
    cand[1] = hi;
    g_s = lo;
    res[1] = static_cast<int64_t>(tS);
  }
  __syncthreads();
  const int64_t lo = cand[0], hi = cand[1];
  if (lo != hi) {  // the tuner's two candidates (powers of two)
    const int sl = __ffsll(lo) - 1, shh = __ffsll(hi) - 1;
    unsigned fl = 0, fh = 0;
    for (int64_t r = tid; r < n; r += blockDim.x) {
      const unsigned long long o = static_cast<unsigned>(occ[r]);
      fl += static_cast<unsigned>((o + static_cast<unsigned long long>(lo) - 1) >> sl);
      fh += static_cast<unsigned>((o + static_cast<unsigned long long>(hi) - 1) >> shh);
    }
    const unsigned long long Fl = block_sum(fl, part);
    const unsigned long long Fh = block_sum(fh, part);
    if (tid == 0) {
      const double cl = static_cast<double>((lo + 1) * static_cast<int64_t>(Fl));
      const double ch = static_cast<double>((hi + 1) * static_cast<int64_t>(Fh));
      g_s = ch < cl ? hi : lo;
    }
    __syncthreads();
  }
  if (tid == 0) res[0] = g_s;
  block_scan_groups(occ, n, g_s, out, wsum);
}

int64_t read_scan_total(const int32_t* out, int64_t n, cudaStream_t s) {
  int32_t total = 0;
  HostReads rd(s);
  rd.add(&total, out + n, 4);
  rd.wait();
  // counts are non-negative, so a negative int32 total means it wrapped past 2^31
  if (total < 0) fail(IXB_SHAPE, "format exceeds 2^31 entries");
  return total;
}

// Tuner (g_req = 0) + group offsets of short profiles in one launch and one
// host read: returns false (nothing done) when n is too long for one CTA.
bool tune_and_scan(const int32_t* counts, int64_t n, int64_t extent, int count_empty_rows,
                   int64_t g_req, int32_t* out, cudaStream_t s, int64_t* g, int64_t* S,
                   int64_t* G) {
  if (n == 0 || n > kSmallScan) return false;
  Scratch<int64_t> res(2, s);
  tune_scan_kernel<<<1, 1024, 0, s>>>(counts, n, extent, count_empty_rows, g_req, out, res.p);
  IXB_LAUNCH_CHECK("tune_scan_kernel");
  int64_t h[2];
  int32_t total = 0;
  HostReads rd(s);
  rd.add(h, res.p, sizeof h);
  rd.add(&total, out + n, 4);
  rd.wait();
  if (total < 0 || h[1] > INT32_MAX) fail(IXB_SHAPE, "format exceeds 2^31 entries");
  *g = h[0];
  if (S) *S = h[1];
  *G = total;
  return true;
}

// ceil(counts / g) scanned (exclusive, total in out[n]) and the total read back.
int64_t groups_scan_total(const int32_t* counts, int64_t n, int64_t g, int32_t* out,
                          cudaStream_t s) {
  if (n == 0) return 0;
  if (n <= kSmallScan) {
    small_scan_kernel<<<1, 1024, 0, s>>>(counts, n, g, out);
    IXB_LAUNCH_CHECK("small_scan_kernel");
  } else {
    exclusive_scan_dev(thrust::make_transform_iterator(counts, GroupsOf{g}), n, out, s);
  }
  return read_scan_total(out, n, s);
}

void count_rows(ixb_pack* P) {
  P->occ = Scratch<int32_t>(P->rows + 1, P->s);
  dispatch_dense(P->dtype, [&](auto tag) {
    using T = decltype(tag);
    launch_row_count(static_cast<const T*>(P->dense), P);
  });
}

// Dense-row grouping plan (group_dim 0): occ -> tuner -> groups per row -> gofs.
void plan_dense_rows(ixb_pack* P, int64_t g_req, int64_t* g_out, bool have_occ = false) {
  if (!have_occ) count_rows(P);
  P->offs = Scratch<int32_t>(P->rows + 1, P->s);
  if (tune_and_scan(P->occ.p, P->rows, P->rows, 0, g_req, P->offs.p, P->s, &P->g, &P->nnz,
                    &P->G)) {
    if (g_out) *g_out = P->g;
    return;
  }
  int64_t g = g_req;
  if (g == 0) {
    // the tuner's one read-back also returns S = nnz
    g = tune_from_occ(P->occ.p, P->rows, P->rows, 0, P->s, nullptr, nullptr, nullptr, nullptr,
                      &P->nnz);
    if (P->nnz > INT32_MAX) fail(IXB_SHAPE, "format exceeds 2^31 entries");
  } else {
    Scratch<int32_t> tmp(P->rows + 1, P->s);
    P->nnz = groups_scan_total(P->occ.p, P->rows, 1, tmp.p, P->s);
  }
  P->g = g;
  if (g_out) *g_out = g;
  P->G = groups_scan_total(P->occ.p, P->rows, g, P->offs.p, P->s);
}

template <typename T>
void pack_dense_rows_t(ixb_pack* P, int32_t* AM, int32_t* AK, void* AV, uint8_t* mask) {
  launch_row_pack(static_cast<const T*>(P->dense), P, P->offs.p, P->g, 0, AM, AK,
                  static_cast<T*>(AV), mask, P->s);
}

void pack_dense_rows(ixb_pack* P, int32_t* AM, int32_t* AK, void* AV, uint8_t* mask) {
  dispatch_dense(P->dtype, [&](auto tag) { pack_dense_rows_t<decltype(tag)>(P, AM, AK, AV, mask); });
}

// Sorted-run plan over rank coordinate arrays; key order: group_dim, then
// the other dims ascending (formats.cpp:124-129, 423-434).
void plan_sorted_runs(ixb_pack* P, bool identity_order, int64_t g_req, int64_t extent,
                      int count_empty_rows, int64_t* g_out) {
  const int64_t n = P->nnz;
  cudaStream_t s = P->s;
  if (n > INT32_MAX) fail(IXB_SHAPE, "more than 2^31 nonzeros");
  if (!identity_order && n > 0) {
    P->perm = Scratch<int32_t>(n, s);
    iota32<<<ceil_div(n, kTB), kTB, 0, s>>>(P->perm.p, n);
    IXB_LAUNCH_CHECK("iota32");
    std::vector<int> order;  // most significant first
    order.push_back(P->group_dim);
    for (int d = 0; d < P->rank; ++d) {
      if (d != P->group_dim) order.push_back(d);
    }
    Scratch<int32_t> key(n, s), key_out(n, s), perm_out(n, s);
    size_t tb = 0;
    IXB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_out.p, P->perm.p,
                                                   perm_out.p, static_cast<int>(n), 0, 32, s));
    Scratch<char> tmp(tb, s);
    for (int i = static_cast<int>(order.size()) - 1; i >= 0; --i) {  // LSD over keys
      gather_key<<<ceil_div(n, kTB), kTB, 0, s>>>(P->coords[order[i]], P->perm.p, n, key.p);
      IXB_LAUNCH_CHECK("gather_key");
      IXB_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key_out.p, P->perm.p,
                                                     perm_out.p, static_cast<int>(n), 0, 32, s));
      note_launch(4);
      std::swap(P->perm.p, perm_out.p);
    }
  }
  const int32_t* gcoord = P->coords[P->group_dim];
  if (identity_order && n > 0 && extent > 0 && extent <= kOccSmemBins) {
    // Canonical input over a small extent (the 27 offsets of a kernel map,
    // the paths of a CG table): the runs are the values in order, so their
    // lengths are the value histogram and their starts its exclusive scan —
    // no pass over the entries beyond the histogram. Runs are indexed by
    // value (empty values give no groups); tune_scan's S = the in-range
    // count proves every coordinate was in [0, extent).
    P->len = Scratch<int32_t>(extent + 1, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(P->len.p, 0, (extent + 1) * sizeof(int32_t), s));
    launch_occupancy(gcoord, n, extent, P->len.p, s);
    P->start = Scratch<int32_t>(extent + 1, s);
    small_scan_kernel<<<1, 1024, 0, s>>>(P->len.p, extent, 1, P->start.p);
    IXB_LAUNCH_CHECK("small_scan_kernel");
    P->gofs = Scratch<int32_t>(extent + 1, s);
    int64_t S = 0;
    if (tune_and_scan(P->len.p, extent, extent, count_empty_rows, g_req, P->gofs.p, s, &P->g, &S,
                      &P->G) &&
        S == n) {
      P->R = extent;
      if (g_out) *g_out = P->g;
      return;
    }
    P->len = Scratch<int32_t>();  // out-of-range coordinates: the general path
    P->start = Scratch<int32_t>();
    P->gofs = Scratch<int32_t>();
  }
  P->run_incl = Scratch<int32_t>(n + 1, s);
  if (n > 0) {
    auto flags = thrust::make_transform_iterator(thrust::counting_iterator<int64_t>(0),
                                                 HeadFlag{gcoord, P->perm.p});
    size_t tb = 0;
    IXB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(nullptr, tb, flags, P->run_incl.p,
                                                 static_cast<int>(n), s));
    Scratch<char> tmp(tb, s);
    IXB_CUDA_CHECK(cub::DeviceScan::InclusiveSum(tmp.p, tb, flags, P->run_incl.p,
                                                 static_cast<int>(n), s));
    note_launch();
    int32_t R = 0;
    HostReads rd(s);
    rd.add(&R, P->run_incl.p + n - 1, 4);
    rd.wait();
    P->R = R;
  }
  const int64_t R = P->R;
  P->start = Scratch<int32_t>(R + 1, s);
  P->len = Scratch<int32_t>(R + 1, s);
  if (n > 0) {
    run_starts<<<ceil_div(n, kTB), kTB, 0, s>>>(P->run_incl.p, n, P->start.p);
    IXB_LAUNCH_CHECK("run_starts");
    run_lengths<<<ceil_div(R, kTB), kTB, 0, s>>>(P->start.p, R, n, P->len.p);
    IXB_LAUNCH_CHECK("run_lengths");
  }
  P->gofs = Scratch<int32_t>(R + 1, s);
  if (tune_and_scan(P->len.p, R, extent, count_empty_rows, g_req, P->gofs.p, s, &P->g, nullptr,
                    &P->G)) {
    if (g_out) *g_out = P->g;
    return;
  }
  int64_t g = g_req;
  if (g == 0) g = tune_from_occ(P->len.p, R, extent, count_empty_rows, s, nullptr);
  P->g = g;
  if (g_out) *g_out = g;
  P->G = groups_scan_total(P->len.p, R, g, P->gofs.p, s);
}

void pack_sorted_runs(ixb_pack* P, const void* vals, int dtype, int32_t* gout,
                      int32_t* const* mout, void* vout, uint8_t* mask) {
  RunPackArgs a{};
  a.perm = P->perm.p;
  a.run_incl = P->run_incl.p;
  a.start = P->start.p;
  a.len = P->len.p;
  a.gofs = P->gofs.p;
  a.gcoord = P->coords[P->group_dim];
  int m = 0;
  for (int d = 0; d < P->rank; ++d) {
    if (d == P->group_dim) continue;
    a.mcoord[m] = P->coords[d];
    a.mout[m] = mout[m];
    ++m;
  }
  a.nm = m;
  a.n = P->nnz;
  a.R = P->R;
  a.g = P->g;
  a.vals = vals;
  a.vout = vout;
  a.vbytes = (vals && vout) ? (dtype == IXB_BF16 ? 2 : (dtype == IXB_F64 || dtype == IXB_I64) ? 8 : 4)
                            : 0;
  a.mask = mask;
  a.gout = gout;
  if (a.n > 0) {
    run_pack_elems<<<ceil_div(a.n, kTB * kPackElems), kTB, 0, P->s>>>(a);
    IXB_LAUNCH_CHECK("run_pack_elems");
    if (a.R <= 4 * sm_count()) run_pack_runs<<<a.R, 128, 0, P->s>>>(a, 1);
    else run_pack_runs<<<ceil_div(a.R, kTB), kTB, 0, P->s>>>(a, 0);
    IXB_LAUNCH_CHECK("run_pack_runs");
  }
}

// Sorted-run packs only move values: 8-byte payloads pass through unchanged.
void check_run_dtype(int dtype) {
  if (dtype != IXB_F32 && dtype != IXB_BF16 && dtype != IXB_F64 && dtype != IXB_I64)
    fail(IXB_FAILURE, "unsupported dtype");
}

}  // namespace
}  // namespace ixb

using namespace ixb;

extern "C" {

void ixb_pack_free(ixb_pack* plan) { delete plan; }

int ixb_dense_to_coo_plan(const void* dense, int dtype, int64_t rows, int64_t cols,
                          ixb_stream stream, ixb_pack** plan, int64_t* nnz) {
  return ixb_guard([&] {
    check_dense_dtype(dtype);
    if (rows < 0 || cols < 0) fail(IXB_SHAPE, "dense_to_coo expects a rank-2 tensor");
    auto P = std::make_unique<ixb_pack>();
    P->type = 2;
    P->s = reinterpret_cast<cudaStream_t>(stream);
    P->dense = dense;
    P->dtype = dtype;
    P->rows = rows;
    P->cols = cols;
    count_rows(P.get());
    P->offs = Scratch<int32_t>(rows + 1, P->s);
    P->nnz = groups_scan_total(P->occ.p, rows, 1, P->offs.p, P->s);
    *nnz = P->nnz;
    *plan = P.release();
  });
}

int ixb_dense_to_coo_pack(ixb_pack* P, int32_t* row_coord, int32_t* col_coord, void* values,
                          ixb_stream stream) {
  return ixb_guard([&] {
    if (!P || P->type != 2) fail(IXB_FAILURE, "not a dense_to_coo plan");
    P->s = reinterpret_cast<cudaStream_t>(stream);
    dispatch_dense(P->dtype, [&](auto tag) {
      using T = decltype(tag);
      launch_row_pack(static_cast<const T*>(P->dense), P, P->offs.p, 1, 1, row_coord, col_coord,
                      static_cast<T*>(values), nullptr, P->s);
    });
  });
}

int ixb_groupcoo_plan(const int32_t* row_coord, const int32_t* col_coord, int64_t nnz,
                      int64_t rows, int64_t cols, int canonical, int group_dim, int64_t g,
                      ixb_stream stream, ixb_pack** plan, int64_t* num_groups, int64_t* g_out) {
  return ixb_guard([&] {
    if (g < 0) fail(IXB_SHAPE, "group size must be >= 1, got " + std::to_string(g));
    if (group_dim != 0 && group_dim != 1) fail(IXB_SHAPE, "group_dim must be 0 or 1");
    auto P = std::make_unique<ixb_pack>();
    P->type = 3;
    P->s = reinterpret_cast<cudaStream_t>(stream);
    P->nnz = nnz;
    P->rank = 2;
    P->group_dim = group_dim;
    P->coords = {row_coord, col_coord};
    plan_sorted_runs(P.get(), canonical && group_dim == 0, g, group_dim == 0 ? rows : cols, 0,
                     g_out);
    *num_groups = P->G;
    *plan = P.release();
  });
}

int ixb_groupcoo_pack(ixb_pack* P, const void* values, int dtype, int32_t* AM, int32_t* AK,
                      void* AV, uint8_t* mask, ixb_stream stream) {
  return ixb_guard([&] {
    if (!P || P->type != 3 || P->rank != 2) fail(IXB_FAILURE, "not a groupcoo plan");
    if (values) check_run_dtype(dtype);
    P->s = reinterpret_cast<cudaStream_t>(stream);
    int32_t* mo[1] = {AK};
    pack_sorted_runs(P, values, dtype, AM, mo, AV, mask);
  });
}

int ixb_dense_groupcoo_plan(const void* dense, int dtype, int64_t rows, int64_t cols,
                            int group_dim, int64_t g, ixb_stream stream, ixb_pack** plan,
                            int64_t* num_groups, int64_t* g_out, int64_t* nnz) {
  return ixb_guard([&] {
    check_dense_dtype(dtype);
    if (g < 0) fail(IXB_SHAPE, "group size must be >= 1, got " + std::to_string(g));
    if (group_dim != 0 && group_dim != 1) fail(IXB_SHAPE, "group_dim must be 0 or 1");
    auto P = std::make_unique<ixb_pack>();
    P->s = reinterpret_cast<cudaStream_t>(stream);
    P->dense = dense;
    P->dtype = dtype;
    P->rows = rows;
    P->cols = cols;
    P->group_dim = group_dim;
    if (group_dim == 0) {
      P->type = 1;
      plan_dense_rows(P.get(), g, g_out);
    } else {
      // columns: dense_to_coo, then the sorted-run engine keyed (col, row)
      count_rows(P.get());
      P->offs = Scratch<int32_t>(rows + 1, P->s);
      P->nnz = groups_scan_total(P->occ.p, rows, 1, P->offs.p, P->s);
      P->coo_r = Scratch<int32_t>(P->nnz, P->s);
      P->coo_c = Scratch<int32_t>(P->nnz, P->s);
      dispatch_dense(dtype, [&](auto tag) {
        using T = decltype(tag);
        launch_row_pack(static_cast<const T*>(dense), P.get(), P->offs.p, 1, 1, P->coo_r.p,
                        P->coo_c.p, static_cast<T*>(nullptr), nullptr, P->s);
      });
      P->type = 3;
      P->rank = 2;
      P->coords = {P->coo_r.p, P->coo_c.p};
      plan_sorted_runs(P.get(), false, g, cols, 0, g_out);
    }
    *num_groups = P->G;
    if (nnz) *nnz = P->nnz;
    *plan = P.release();
  });
}

int ixb_dense_groupcoo_pack(ixb_pack* P, int32_t* AM, int32_t* AK, void* AV, uint8_t* mask,
                            ixb_stream stream) {
  return ixb_guard([&] {
    if (!P || (P->type != 1 && P->type != 3) || !P->dense) fail(IXB_FAILURE, "not a dense groupcoo plan");
    P->s = reinterpret_cast<cudaStream_t>(stream);
    if (P->type == 1) {
      pack_dense_rows(P, AM, AK, AV, mask);
    } else {
      // values in dense_to_coo order = row-major positions; gather by (r, c)
      Scratch<char> vals(P->nnz * dense_bytes(P->dtype), P->s);
      dispatch_dense(P->dtype, [&](auto tag) {
        using T = decltype(tag);
        launch_row_pack(static_cast<const T*>(P->dense), P, P->offs.p, 1, 1, P->coo_r.p,
                        P->coo_c.p, reinterpret_cast<T*>(vals.p), nullptr, P->s);
      });
      int32_t* mo[1] = {AK};
      pack_sorted_runs(P, vals.p, P->dtype, AM, mo, AV, mask);
    }
  });
}

int ixb_blockgroupcoo_plan(const void* dense, int dtype, int64_t rows, int64_t cols, int64_t bm,
                           int64_t bk, int64_t g, int group_dim, ixb_stream stream,
                           ixb_pack** plan, int64_t* num_groups, int64_t* g_out,
                           int64_t* num_blocks) {
  return ixb_guard([&] {
    check_dense_dtype(dtype);
    if (bm < 1 || bk < 1) fail(IXB_SHAPE, "block dims must be >= 1");
    if (g < 0) fail(IXB_SHAPE, "group size must be >= 1");
    if (group_dim != 0 && group_dim != 1) fail(IXB_SHAPE, "group_dim must be 0 or 1");
    auto P = std::make_unique<ixb_pack>();
    P->type = 4;
    P->s = reinterpret_cast<cudaStream_t>(stream);
    P->dense = dense;
    P->dtype = dtype;
    P->rows = rows;
    P->cols = cols;
    P->bm = bm;
    P->bk = bk;
    P->group_dim = group_dim;
    P->gr = ceil_div(rows, bm);
    P->gcn = ceil_div(cols, bk);
    const int64_t nb = P->gr * P->gcn;
    P->flags = Scratch<uint8_t>(nb + 16, P->s);
    auto I = std::make_unique<ixb_pack>();
    bool fused = false;  // flags kernel also counted the block rows (I->occ)
    if (nb) {
      dispatch_dense(dtype, [&](auto tag) {
        using T = decltype(tag);
        const int64_t rowb = bk * static_cast<int64_t>(sizeof(T));
        const bool vec = rowb % 16 == 0 && 512 % rowb == 0 &&
                         (cols * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
                         reinterpret_cast<uintptr_t>(dense) % 16 == 0;
        if (vec) {
          const int64_t bpw = 512 / rowb;
          const int64_t warps = P->gr * ceil_div(P->gcn, bpw);
          fused = group_dim == 0;
          if (fused) {
            I->occ = Scratch<int32_t>(P->gr + 1, P->s);
            IXB_CUDA_CHECK(cudaMemsetAsync(I->occ.p, 0, (P->gr + 1) * 4, P->s));
          }
          block_flags_vec_kernel<<<ceil_div(warps * 32, kTB), kTB, 0, P->s>>>(
              static_cast<const T*>(dense), rows, cols, bm, bk, P->gr, P->gcn, P->flags.p,
              fused ? I->occ.p : nullptr);
        } else {
          block_flags_kernel<<<ceil_div(nb, kTB), kTB, 0, P->s>>>(
              static_cast<const T*>(dense), rows, cols, bm, bk, P->gr, P->gcn, P->flags.p);
        }
      });
      IXB_LAUNCH_CHECK("block_flags_kernel");
    }
    // group the block-level COO like coo_to_groupcoo (formats.cpp:265)
    I->s = P->s;
    I->dense = P->flags.p;
    I->dtype = IXB_U8;  // block flags
    I->rows = P->gr;
    I->cols = P->gcn;
    I->group_dim = group_dim;
    if (group_dim == 0) {
      I->type = 1;
      plan_dense_rows(I.get(), g, g_out, fused);
    } else {
      count_rows(I.get());
      I->offs = Scratch<int32_t>(I->rows + 1, I->s);
      I->nnz = groups_scan_total(I->occ.p, I->rows, 1, I->offs.p, I->s);
      I->coo_r = Scratch<int32_t>(I->nnz, I->s);
      I->coo_c = Scratch<int32_t>(I->nnz, I->s);
      launch_row_pack(static_cast<const uint8_t*>(I->dense), I.get(), I->offs.p, 1, 1,
                      I->coo_r.p, I->coo_c.p, static_cast<uint8_t*>(nullptr), nullptr, I->s);
      I->type = 3;
      I->rank = 2;
      I->coords = {I->coo_r.p, I->coo_c.p};
      plan_sorted_runs(I.get(), false, g, I->cols, 0, g_out);
    }
    P->G = I->G;
    P->g = I->g;
    P->nblocks = I->nnz;
    *num_groups = P->G;
    if (num_blocks) *num_blocks = P->nblocks;
    P->inner = std::move(I);
    *plan = P.release();
  });
}

int ixb_blockgroupcoo_pack(ixb_pack* P, int32_t* AM, int32_t* AK, void* AV, uint8_t* mask,
                           ixb_stream stream) {
  return ixb_guard([&] {
    if (!P || P->type != 4) fail(IXB_FAILURE, "not a blockgroupcoo plan");
    P->s = reinterpret_cast<cudaStream_t>(stream);
    ixb_pack* I = P->inner.get();
    I->s = P->s;
    const int64_t slots = P->G * P->g;
    Scratch<uint8_t> own_mask;
    uint8_t* m = mask;
    if (!m) {
      own_mask = Scratch<uint8_t>(slots + 16, P->s);
      m = own_mask.p;
    }
    const bool vec_rows = (P->bk * static_cast<int64_t>(dense_bytes(P->dtype))) % 16 == 0 &&
                          (P->cols * static_cast<int64_t>(dense_bytes(P->dtype))) % 16 == 0 &&
                          reinterpret_cast<uintptr_t>(P->dense) % 16 == 0 &&
                          reinterpret_cast<uintptr_t>(AV) % 16 == 0;
    if (I->type == 1 && vec_rows) {
      // fused: AM/AK/mask and the AV blocks in one pass per block row
      if (P->gr && slots) {
        dispatch_dense(P->dtype, [&](auto tag) {
          using T = decltype(tag);
          block_row_pack_kernel<T><<<static_cast<unsigned>(P->gr), kTB, 0, P->s>>>(
              static_cast<const T*>(P->dense), P->rows, P->cols, P->bm, P->bk, P->gcn, P->flags.p,
              I->occ.p, I->offs.p, P->g, AM, AK, static_cast<T*>(AV), m);
        });
        IXB_LAUNCH_CHECK("block_row_pack_kernel");
      }
      return;
    }
    if (I->type == 1) {
      pack_dense_rows(I, AM, AK, nullptr, m);
    } else {
      int32_t* mo[1] = {AK};
      pack_sorted_runs(I, nullptr, IXB_F32, AM, mo, nullptr, m);
    }
    if (AV && slots) {
      const int64_t grid = ceil_div(slots * 32, kTB);
      dispatch_dense(P->dtype, [&](auto tag) {
        using T = decltype(tag);
        const int vec = (P->bk * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
                        (P->cols * static_cast<int64_t>(sizeof(T))) % 16 == 0 &&
                        reinterpret_cast<uintptr_t>(P->dense) % 16 == 0 &&
                        reinterpret_cast<uintptr_t>(AV) % 16 == 0;
        block_copy_kernel<<<grid, kTB, 0, P->s>>>(static_cast<const T*>(P->dense), P->rows,
                                                 P->cols, P->bm, P->bk, P->group_dim, AM, AK, m,
                                                 slots, P->g, static_cast<T*>(AV), vec);
      });
      IXB_LAUNCH_CHECK("block_copy_kernel");
    }
  });
}

int ixb_group_coo_tensor_plan(int rank, const int64_t* shape, const int32_t* const* coords,
                              int64_t nnz, int group_dim, int64_t g, int canonical,
                              ixb_stream stream, ixb_pack** plan, int64_t* num_groups) {
  return ixb_guard([&] {
    if (g < 1) fail(IXB_SHAPE, "group size must be >= 1");
    if (group_dim < 0 || group_dim >= rank) fail(IXB_SHAPE, "group_dim out of range");
    if (rank > 9) fail(IXB_SHAPE, "rank > 9 not supported");
    auto P = std::make_unique<ixb_pack>();
    P->type = 3;
    P->s = reinterpret_cast<cudaStream_t>(stream);
    P->nnz = nnz;
    P->rank = rank;
    P->group_dim = group_dim;
    P->coords.assign(coords, coords + rank);
    plan_sorted_runs(P.get(), canonical != 0, g, shape ? shape[group_dim] : 0, 0, nullptr);
    *num_groups = P->G;
    *plan = P.release();
  });
}

int ixb_group_coo_tensor_pack(ixb_pack* P, const void* values, int dtype, int32_t* group_coord,
                              int32_t* const* member_coords, void* out_values, uint8_t* mask,
                              ixb_stream stream) {
  return ixb_guard([&] {
    if (!P || P->type != 3) fail(IXB_FAILURE, "not a group_coo_tensor plan");
    if (values) check_run_dtype(dtype);
    P->s = reinterpret_cast<cudaStream_t>(stream);
    pack_sorted_runs(P, values, dtype, group_coord, member_coords, out_values, mask);
  });
}

int ixb_tune_report(const int32_t* coord, int64_t nnz, int64_t extent, int count_empty_rows,
                    ixb_stream stream, int64_t* g_out, double* gstar_out, int64_t* cand_g,
                    double* cand_score, int* ncand) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!cand_g || !cand_score || !ncand) fail(IXB_SHAPE, "ixb_tune_report: null output");
    Scratch<int32_t> occ(extent + 1, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(occ.p, 0, (extent + 1) * 4, s));
    if (nnz) {
      launch_occupancy(coord, nnz, extent, occ.p, s);
    }
    *g_out = tune_from_occ(occ.p, extent, extent, count_empty_rows, s, gstar_out, cand_g,
                           cand_score, ncand);
  });
}

int ixb_tune_group_size(const int32_t* coord, int64_t nnz, int64_t extent, int count_empty_rows,
                        ixb_stream stream, int64_t* g_out, double* gstar_out) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    // occupancy histogram (occupancy(), formats.cpp:96-103): integer atomics
    Scratch<int32_t> occ(extent + 1, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(occ.p, 0, (extent + 1) * 4, s));
    if (nnz) {
      launch_occupancy(coord, nnz, extent, occ.p, s);
    }
    *g_out = tune_from_occ(occ.p, extent, extent, count_empty_rows, s, gstar_out);
  });
}

int ixb_tune_brute(const int32_t* coord, int64_t nnz, int64_t extent, ixb_stream stream,
                   int64_t* g_out, int64_t* f_out) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!g_out || !f_out) fail(IXB_SHAPE, "ixb_tune_brute: null output");
    *g_out = 0;
    *f_out = 0;
    if (nnz == 0 || extent == 0) return;  // empty profile: nullopt (g_out = 0)
    Scratch<int32_t> occ(extent + 1, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(occ.p, 0, (extent + 1) * 4, s));
    launch_occupancy(coord, nnz, extent, occ.p, s);
    int64_t maxocc = 0;
    {
      // max occupancy from the tuner's one-pass statistics
      int64_t total = 0;
      tune_from_occ(occ.p, extent, extent, 0, s, nullptr, nullptr, nullptr, nullptr, &total,
                    &maxocc);
    }
    if (maxocc < 1) return;
    Scratch<unsigned long long> F(maxocc, s);
    const int64_t grid = maxocc < 4 * sm_count() ? maxocc : 4 * sm_count();
    brute_cost_kernel<<<static_cast<unsigned>(grid), 256, 0, s>>>(occ.p, extent, maxocc, F.p);
    IXB_LAUNCH_CHECK("brute_cost_kernel");
    std::vector<unsigned long long> h(static_cast<size_t>(maxocc));
    IXB_CUDA_CHECK(cudaMemcpyAsync(h.data(), F.p, maxocc * 8, cudaMemcpyDeviceToHost, s));
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));
    int64_t best_g = 1;
    unsigned long long best_f = h[0];
    for (int64_t g = 2; g <= maxocc; ++g) {  // strict < : ties keep the smaller g
      if (h[static_cast<size_t>(g - 1)] < best_f) {
        best_f = h[static_cast<size_t>(g - 1)];
        best_g = g;
      }
    }
    *g_out = best_g;
    *f_out = static_cast<int64_t>(best_f);
  });
}

}  // extern "C"
