// K5 — submanifold 3x3x3 kernel map on the device (no reference
// implementation, oracle: ixo_kernel_map).
//
// Voxel hash (open addressing, 16-byte slots {64-bit packed key, index}:
// one 128-bit load per probe), then two passes over the voxels in blocks of
// 256: the count pass probes all 27 neighbours of each voxel, keeps a 27-bit
// hit mask per voxel and the hit count per (offset, block); an exclusive scan
// of those counts in (offset, block) order gives every (offset, block) its
// first output position; the emit pass re-probes only the hits and writes
// the pairs in (z, i) order — the canonical order of
// group_coo_tensor(MAP, group_dim=2, g) (sort key (z, out, in); each (z, out)
// has at most one `in`), so grouping is a run split with no sort.
// Integer work, bound by the random L2 lookups: no 27·n-sized flag arrays.
#include <cub/device/device_scan.cuh>

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

// Emit pass: pair (z, i) of block b goes to base[z * nb + b] + (hits of
// offset z before voxel i in the block); only the hits are re-probed.
__global__ void __launch_bounds__(kKmBlock) km_emit(const int32_t* coords, int64_t n,
                                                    const Slot* table, uint32_t mask,
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
    mi[p] = hash_find(table, mask, neighbour_key(x, y, z, off));
    mz[p] = off;
  }
}

}  // namespace

struct KmapPlan {
  cudaStream_t s = nullptr;
  int64_t n = 0, pairs = 0, nb = 0;
  uint32_t mask = 0;
  const int32_t* coords = nullptr;
  Scratch<Slot> table;
  Scratch<uint32_t> masks;
  Scratch<int32_t> base;
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
    uint32_t cap = 64;
    while (cap < 2 * n) cap <<= 1;
    P.mask = cap - 1;
    P.table = Scratch<Slot>(cap, s);
    Scratch<int> flags(2, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(P.table.p, 0xff, cap * sizeof(Slot), s));
    IXB_CUDA_CHECK(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int), s));
    P.nb = ceil_div(n, kKmBlock);
    const int64_t T = 27 * P.nb;  // (offset, block) counts
    Scratch<int32_t> cnt(T + 1, s);
    P.base = Scratch<int32_t>(T + 1, s);
    P.masks = Scratch<uint32_t>(n + 1, s);
    if (n > 0) {
      hash_insert<<<ceil_div(n, 256), 256, 0, s>>>(coords, n, P.table.p, P.mask, flags.p);
      IXB_LAUNCH_CHECK("hash_insert");
      km_count<<<static_cast<unsigned>(P.nb), kKmBlock, 0, s>>>(coords, n, P.table.p, P.mask,
                                                                P.masks.p, cnt.p);
      IXB_LAUNCH_CHECK("km_count");
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
    IXB_CUDA_CHECK(cudaMemcpyAsync(hflags, flags.p, sizeof hflags, cudaMemcpyDeviceToHost, s));
    if (n > 0) {
      IXB_CUDA_CHECK(cudaMemcpyAsync(&last_base, P.base.p + T - 1, 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaMemcpyAsync(&last_cnt, cnt.p + T - 1, 4, cudaMemcpyDeviceToHost, s));
    }
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));
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
      km_emit<<<static_cast<unsigned>(P.nb), kKmBlock, 0, s>>>(P.coords, P.n, P.table.p, P.mask,
                                                               P.masks.p, P.base.p, map_out,
                                                               map_in, map_off);
      IXB_LAUNCH_CHECK("km_emit");
    }
  });
}

void ixb_kernel_map_free(ixb_kmap* plan) { delete plan; }

}  // extern "C"
