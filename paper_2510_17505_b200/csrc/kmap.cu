// K5 — submanifold 3x3x3 kernel map on the device (no reference
// implementation, oracle: ixo_kernel_map).
//
// Two passes over the voxels in blocks of 256: the count pass finds all 27
// neighbours of each voxel, keeps a 27-bit hit mask per voxel and the hit
// count per (offset, block); an exclusive scan of those counts in (offset,
// block) order gives every (offset, block) its first output position; the
// emit pass resolves only the hits and writes the pairs in (z, i) order —
// the canonical order of group_coo_tensor(MAP, group_dim=2, g) (sort key
// (z, out, in); each (z, out) has at most one `in`), so grouping is a run
// split with no sort.
//
// Neighbour lookups: a bounding-box pass (min/max + order check, one host
// read) picks the structure. A dense enough box gets an occupancy bitmap
// (bit ((x-x0)·Y + (y-y0))·Z + (z-z0)): the count pass reads nine 64-bit
// windows per voxel (the three z-neighbours of a column are adjacent bits),
// and voxels given in strictly increasing (x, y, z) order — the bitmap's
// order — take a neighbour's index as its rank (word popcount prefix +
// popcount below it): no hash at all. Otherwise an open-addressing hash
// (16-byte slots {64-bit packed key, index}, one 128-bit load per probe,
// duplicate detection) serves the count (sparse boxes) and the emit
// (unsorted voxels). Integer work; no 27·n-sized flag arrays.
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <climits>
#include <memory>

#include "common.cuh"

namespace ixb {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr int kBias = 1 << 20;
constexpr int kKmBlock = 256;  // voxels per count/emit block
constexpr int kKmWarps = kKmBlock / 32;

struct __align__(16) Slot {
  unsigned long long key;
  int32_t val;
  int32_t pad;
};

__device__ __forceinline__ unsigned long long vox_key(int x, int y, int z) {
  return (static_cast<unsigned long long>(x + kBias) << 42) |
         (static_cast<unsigned long long>(y + kBias) << 21) |
         static_cast<unsigned long long>(z + kBias);
}

__device__ __forceinline__ uint32_t vox_hash(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return static_cast<uint32_t>(k);
}

__global__ void hash_insert(const int32_t* coords, int64_t n, Slot* table, uint32_t mask,
                            int* flags /*0 dup,1 range*/) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
  if (x < -kBias + 1 || x >= kBias - 1 || y < -kBias + 1 || y >= kBias - 1 || z < -kBias + 1 ||
      z >= kBias - 1) {
    atomicOr(&flags[1], 1);
    return;
  }
  const unsigned long long k = vox_key(x, y, z);
  uint32_t h = vox_hash(k) & mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(&table[h].key, kEmpty, k);
    if (prev == kEmpty) {
      table[h].val = static_cast<int32_t>(i);
      return;
    }
    if (prev == k) {
      atomicOr(&flags[0], 1);  // duplicate voxel
      return;
    }
    h = (h + 1) & mask;
  }
}

// Bounding box of the voxels: bb = {min x, min y, min z, max x, max y, max z}
// (pre-set to INT_MAX / INT_MIN).
// bb[6] != 0: the voxels are not in strictly increasing (x, y, z) order.
__global__ void bbox_kernel(const int32_t* coords, int64_t n, int* bb) {
  int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
  bool unsorted = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int v[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      v[d] = coords[3 * i + d];
      lo[d] = min(lo[d], v[d]);
      hi[d] = max(hi[d], v[d]);
    }
    if (i + 1 < n) {
      const int a = coords[3 * i + 3], b = coords[3 * i + 4], c = coords[3 * i + 5];
      const bool less = v[0] < a || (v[0] == a && (v[1] < b || (v[1] == b && v[2] < c)));
      unsorted |= !less;
    }
  }
  // warp (REDUX), then CTA (shared memory), then 7 global atomics per CTA:
  // per-warp atomics on the same 7 words serialised at the L2
  __shared__ int red[7][8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool uns = __any_sync(0xffffffffu, unsorted);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    lo[d] = __reduce_min_sync(0xffffffffu, lo[d]);
    hi[d] = __reduce_max_sync(0xffffffffu, hi[d]);
  }
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      red[d][w] = lo[d];
      red[3 + d][w] = hi[d];
    }
    red[6][w] = uns ? 1 : 0;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    const int k = threadIdx.x;
    int v = red[k][0];
    for (int j = 1; j < static_cast<int>(blockDim.x >> 5); ++j)
      v = k < 3 ? min(v, red[k][j]) : k < 6 ? max(v, red[k][j]) : (v | red[k][j]);
    if (k < 3) atomicMin(&bb[k], v);
    else if (k < 6) atomicMax(&bb[k], v);
    else if (v) atomicOr(&bb[6], 1);
  }
}

// Occupancy bitmap over the bounding box, bit ((x-x0) * Y + (y-y0)) * Z + (z-z0).
struct Bitmap {
  uint32_t* bits;
  int x0, y0, z0, X, Y, Z;
};

__global__ void bitmap_set(const int32_t* coords, int64_t n, Bitmap bm) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t b = ((static_cast<int64_t>(coords[3 * i] - bm.x0) * bm.Y + (coords[3 * i + 1] - bm.y0)) *
                         bm.Z + (coords[3 * i + 2] - bm.z0));
  atomicOr(&bm.bits[b >> 5], 1u << (b & 31));
}

__device__ __forceinline__ unsigned long long neighbour_key(int x, int y, int z, int off) {
  return vox_key(x + off / 9 - 1, y + (off / 3) % 3 - 1, z + off % 3 - 1);
}

// Index of the voxel with key k, or -1 (the table was filled by an earlier
// kernel). One 128-bit load per probe. (Batching nine lookups per thread
// raised registers to 97 and measured 1.5x slower: the lookups are bound by
// the L2's random-sector rate, not by latency.)
__device__ __forceinline__ int hash_find(const Slot* table, uint32_t mask, unsigned long long k) {
  uint32_t h = vox_hash(k) & mask;
  for (;;) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(table + h));
    const unsigned long long cur = static_cast<unsigned long long>(v.x) |
                                   (static_cast<unsigned long long>(v.y) << 32);
    if (cur == k) return static_cast<int>(v.z);
    if (cur == kEmpty) return -1;
    h = (h + 1) & mask;
  }
}

// Count pass: hit mask per voxel, hits per (offset, block) -> cnt[off * nb + block].
__global__ void __launch_bounds__(kKmBlock) km_count(const int32_t* coords, int64_t n,
                                                     const Slot* table, uint32_t mask,
                                                     uint32_t* masks, int32_t* cnt) {
  __shared__ int wc[kKmWarps][27];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kKmBlock + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t m = 0;
  if (i < n) {
    const int x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
#pragma unroll 3
    for (int off = 0; off < 27; ++off)
      if (hash_find(table, mask, neighbour_key(x, y, z, off)) >= 0) m |= 1u << off;
    masks[i] = m;
  }
#pragma unroll
  for (int off = 0; off < 27; ++off) {
    const unsigned b = __ballot_sync(0xffffffffu, (m >> off) & 1);
    if (lane == 0) wc[warp][off] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x < 27) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kKmWarps; ++w) s += wc[w][threadIdx.x];
    cnt[static_cast<int64_t>(threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
}

// Count pass over the occupancy bitmap (dense bounding boxes): the three
// z-neighbours of each (dx, dy) column are adjacent bits, so a voxel costs
// nine 64-bit windows instead of 27 hash probes, and neighbouring voxels
// share their words in L1/L2. Same outputs as km_count.
__global__ void __launch_bounds__(kKmBlock) km_count_bitmap(const int32_t* coords, int64_t n,
                                                            Bitmap bm, uint32_t* masks,
                                                            int32_t* cnt) {
  __shared__ int wc[kKmWarps][27];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kKmBlock + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t m = 0;
  if (i < n) {
    const int x = coords[3 * i] - bm.x0, y = coords[3 * i + 1] - bm.y0,
              z = coords[3 * i + 2] - bm.z0;
#pragma unroll
    for (int dx = -1; dx <= 1; ++dx) {
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy) {
        const int xx = x + dx, yy = y + dy;
        if (xx < 0 || xx >= bm.X || yy < 0 || yy >= bm.Y) continue;
        // bits z-1, z, z+1 of the (xx, yy) column: a 64-bit window from the
        // word holding bit z-1 (z-1 >= -1: start one bit early, clamp below)
        const int64_t b = (static_cast<int64_t>(xx) * bm.Y + yy) * bm.Z + z - 1;
        const int64_t bb = b < 0 ? 0 : b;
        const int64_t w = bb >> 5;
        const unsigned long long win =
            static_cast<unsigned long long>(__ldg(bm.bits + w)) |
            (static_cast<unsigned long long>(__ldg(bm.bits + w + 1)) << 32);
        uint32_t three = static_cast<uint32_t>(win >> (bb & 31)) & 7u;
        if (b < 0) three = (three << 1) & 7u;  // only reachable when z = 0 at the first row
        if (z == 0) three &= ~1u;              // z - 1 is outside the box (previous column)
        if (z + 1 >= bm.Z) three &= ~4u;       // z + 1 is outside (next column)
        m |= three << ((dx + 1) * 9 + (dy + 1) * 3);
      }
    }
    masks[i] = m;
  }
#pragma unroll
  for (int off = 0; off < 27; ++off) {
    const unsigned b = __ballot_sync(0xffffffffu, (m >> off) & 1);
    if (lane == 0) wc[warp][off] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x < 27) {
    int s = 0;
#pragma unroll
    for (int w = 0; w < kKmWarps; ++w) s += wc[w][threadIdx.x];
    cnt[static_cast<int64_t>(threadIdx.x) * gridDim.x + blockIdx.x] = s;
  }
}

// Emit pass: pair (z, i) of block b goes to base[z * nb + b] + (hits of
// offset z before voxel i in the block); only the hits are re-probed.
// Neighbour index by hash probe (any voxel order).
struct HashFind {
  const Slot* table;
  uint32_t mask;
  __device__ int operator()(int x, int y, int z, int off) const {
    return hash_find(table, mask, neighbour_key(x, y, z, off));
  }
};
// Neighbour index by rank in the occupancy bitmap (voxels in strictly
// increasing (x, y, z) order = bitmap order): words before it + bits below
// it in its word.
struct RankFind {
  Bitmap bm;
  const int32_t* pre;  // exclusive scan of the words' popcounts
  __device__ int operator()(int x, int y, int z, int off) const {
    const int64_t b = (static_cast<int64_t>(x + off / 9 - 1 - bm.x0) * bm.Y +
                       (y + (off / 3) % 3 - 1 - bm.y0)) * bm.Z + (z + off % 3 - 1 - bm.z0);
    const int64_t w = b >> 5;
    return __ldg(pre + w) + __popc(__ldg(bm.bits + w) & ((1u << (b & 31)) - 1u));
  }
};

template <class Find>
__global__ void __launch_bounds__(kKmBlock) km_emit(const int32_t* coords, int64_t n, Find find,
                                                    const uint32_t* masks, const int32_t* base,
                                                    int32_t* mo, int32_t* mi, int32_t* mz) {
  __shared__ int wb[kKmWarps][27];
  __shared__ unsigned bal[kKmWarps][27];  // per warp and offset: lanes with a hit
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kKmBlock + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t m = i < n ? masks[i] : 0u;
#pragma unroll
  for (int off = 0; off < 27; ++off) {
    const unsigned b = __ballot_sync(0xffffffffu, (m >> off) & 1);
    if (lane == 0) {
      bal[warp][off] = b;
      wb[warp][off] = __popc(b);
    }
  }
  __syncthreads();
  if (threadIdx.x < 27) {  // per-warp starts: block base + earlier warps' hits
    int s = base[static_cast<int64_t>(threadIdx.x) * gridDim.x + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kKmWarps; ++w) {
      const int c = wb[w][threadIdx.x];
      wb[w][threadIdx.x] = s;
      s += c;
    }
  }
  __syncthreads();
  if (!m) return;
  const int x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
  const unsigned lt = (1u << lane) - 1u;
#pragma unroll
  for (int off = 0; off < 27; ++off) {
    if (!((m >> off) & 1)) continue;
    const int64_t p = wb[warp][off] + __popc(bal[warp][off] & lt);
    mo[p] = static_cast<int32_t>(i);
    mi[p] = find(x, y, z, off);
    mz[p] = off;
  }
}

}  // namespace

struct KmapPlan {
  cudaStream_t s = nullptr;
  int64_t n = 0, pairs = 0, nb = 0;
  uint32_t mask = 0;
  const int32_t* coords = nullptr;
  bool rank = false;        // neighbour indices by bitmap rank (sorted voxels) or by hash
  Scratch<Slot> table;      // hash mode
  Scratch<uint32_t> bits;   // occupancy bitmap (bitmap count pass / rank mode)
  Scratch<int32_t> pre;     // rank mode: word popcount prefix
  Bitmap bm{};
  Scratch<uint32_t> masks;
  Scratch<int32_t> base;
};

struct Popc {
  __host__ __device__ int32_t operator()(uint32_t w) const {
#ifdef __CUDA_ARCH__
    return __popc(w);
#else
    return __builtin_popcount(w);
#endif
  }
};

}  // namespace ixb

struct ixb_kmap {
  ixb::KmapPlan p;
};

extern "C" {

int ixb_kernel_map_plan(const int32_t* coords, int64_t n, ixb_stream stream, ixb_kmap** plan,
                        int64_t* num_pairs) {
  return ixb_guard([&] {
    using namespace ixb;
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (n < 0) fail(IXB_SHAPE, "kernel map: negative voxel count");
    if (27 * n > INT32_MAX) fail(IXB_SHAPE, "kernel map: too many voxels for int32 pairs");
    auto H = std::make_unique<ixb_kmap>();
    KmapPlan& P = H->p;
    P.s = s;
    P.n = n;
    P.coords = coords;
    Scratch<int> flags(2, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int), s));
    P.nb = ceil_div(n, kKmBlock);
    const int64_t T = 27 * P.nb;  // (offset, block) counts
    Scratch<int32_t> cnt(T + 1, s);
    P.base = Scratch<int32_t>(T + 1, s);
    P.masks = Scratch<uint32_t>(n + 1, s);
    if (n > 0) {
      // bounding box + order check (one host read). A dense enough box
      // (<= 256 bits per voxel, the hash table's own footprint; < 2^31
      // bits) gets an occupancy bitmap for the count pass; voxels in
      // strictly increasing (x, y, z) order (no duplicates possible) also
      // take their neighbour indices from bitmap ranks and skip the hash.
      Scratch<int> bbd(7, s);
      const int init[7] = {INT_MAX, INT_MAX, INT_MAX, INT_MIN, INT_MIN, INT_MIN, 0};
      IXB_CUDA_CHECK(cudaMemcpyAsync(bbd.p, init, sizeof init, cudaMemcpyHostToDevice, s));
      bbox_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(n, 256), 8 * sm_count())),
                    256, 0, s>>>(coords, n, bbd.p);
      IXB_LAUNCH_CHECK("bbox_kernel");
      int bb[7];
      HostReads rd(s);
      rd.add(bb, bbd.p, sizeof bb);
      rd.wait();
      for (int d = 0; d < 3; ++d)  // the hash key's range (hash_insert checks the same)
        if (bb[d] < -kBias + 1 || bb[3 + d] >= kBias - 1)
          fail(IXB_SHAPE, "kernel map: voxel coordinate outside [-2^20, 2^20)");
      const int64_t X = static_cast<int64_t>(bb[3]) - bb[0] + 1,
                    Y = static_cast<int64_t>(bb[4]) - bb[1] + 1,
                    Z = static_cast<int64_t>(bb[5]) - bb[2] + 1;
      const double vol = static_cast<double>(X) * static_cast<double>(Y) * static_cast<double>(Z);
      const bool use_bitmap = vol <= 256.0 * static_cast<double>(n) && vol < 2147483648.0;
      P.rank = use_bitmap && !bb[6];
      if (!P.rank) {
        uint32_t cap = 64;
        while (cap < 2 * n) cap <<= 1;
        P.mask = cap - 1;
        P.table = Scratch<Slot>(cap, s);
        IXB_CUDA_CHECK(cudaMemsetAsync(P.table.p, 0xff, cap * sizeof(Slot), s));
        hash_insert<<<ceil_div(n, 256), 256, 0, s>>>(coords, n, P.table.p, P.mask, flags.p);
        IXB_LAUNCH_CHECK("hash_insert");
      }
      if (use_bitmap) {
        const int64_t words = ceil_div(static_cast<int64_t>(vol), 32) + 2;
        P.bits = Scratch<uint32_t>(words, s);
        IXB_CUDA_CHECK(cudaMemsetAsync(P.bits.p, 0, words * sizeof(uint32_t), s));
        P.bm = Bitmap{P.bits.p, bb[0], bb[1], bb[2], static_cast<int>(X), static_cast<int>(Y),
                      static_cast<int>(Z)};
        bitmap_set<<<ceil_div(n, 256), 256, 0, s>>>(coords, n, P.bm);
        IXB_LAUNCH_CHECK("bitmap_set");
        km_count_bitmap<<<static_cast<unsigned>(P.nb), kKmBlock, 0, s>>>(coords, n, P.bm,
                                                                          P.masks.p, cnt.p);
        IXB_LAUNCH_CHECK("km_count_bitmap");
        if (P.rank) {
          P.pre = Scratch<int32_t>(words, s);
          auto pc = thrust::make_transform_iterator(P.bits.p, Popc{});
          size_t tb = 0;
          IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, pc, P.pre.p,
                                                       static_cast<int>(words), s));
          Scratch<char> tmp(tb, s);
          IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, pc, P.pre.p,
                                                       static_cast<int>(words), s));
          note_launch();
        }
      } else {
        km_count<<<static_cast<unsigned>(P.nb), kKmBlock, 0, s>>>(coords, n, P.table.p, P.mask,
                                                                  P.masks.p, cnt.p);
        IXB_LAUNCH_CHECK("km_count");
      }
      size_t tb = 0;
      IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, P.base.p,
                                                   static_cast<int>(T), s));
      Scratch<char> tmp(tb, s);
      IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, P.base.p,
                                                   static_cast<int>(T), s));
      note_launch();
    }
    int hflags[2] = {0, 0};
    int32_t last_base = 0, last_cnt = 0;
    HostReads rd(s);
    rd.add(hflags, flags.p, sizeof hflags);
    if (n > 0) {
      rd.add(&last_base, P.base.p + T - 1, 4);
      rd.add(&last_cnt, cnt.p + T - 1, 4);
    }
    rd.wait();
    if (hflags[1]) fail(IXB_SHAPE, "kernel map: voxel coordinate outside [-2^20, 2^20)");
    if (hflags[0]) fail(IXB_SHAPE, "kernel map: duplicate voxel coordinates");
    P.pairs = static_cast<int64_t>(last_base) + last_cnt;
    *num_pairs = P.pairs;
    *plan = H.release();
  });
}

int ixb_kernel_map_pack(ixb_kmap* plan, int32_t* map_out, int32_t* map_in, int32_t* map_off,
                        ixb_stream stream) {
  return ixb_guard([&] {
    using namespace ixb;
    auto* H = plan;
    if (!H) fail(IXB_FAILURE, "null kernel map plan");
    auto s = reinterpret_cast<cudaStream_t>(stream);
    const KmapPlan& P = H->p;
    if (P.n > 0) {
      if (P.rank)
        km_emit<<<static_cast<unsigned>(P.nb), kKmBlock, 0, s>>>(
            P.coords, P.n, RankFind{P.bm, P.pre.p}, P.masks.p, P.base.p, map_out, map_in,
            map_off);
      else
        km_emit<<<static_cast<unsigned>(P.nb), kKmBlock, 0, s>>>(
            P.coords, P.n, HashFind{P.table.p, P.mask}, P.masks.p, P.base.p, map_out, map_in,
            map_off);
      IXB_LAUNCH_CHECK("km_emit");
    }
  });
}

void ixb_kernel_map_free(ixb_kmap* plan) { delete plan; }

}  // extern "C"
