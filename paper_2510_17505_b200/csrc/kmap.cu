// K5 — submanifold 3x3x3 kernel map on the device (no reference
// implementation, oracle: ixo_kernel_map).
//
// Voxel hash (open addressing, 64-bit packed keys, atomicCAS insert) ->
// one probe per (offset z, voxel i) -> hit flags -> exclusive scan -> pairs
// written in (z, i) order, i.e. already in the canonical order of
// group_coo_tensor(MAP, group_dim=2, g) (sort key (z, out, in); each (z, out)
// has at most one `in`). Integer/byte work, HBM/L2 bound.
#include <cub/device/device_scan.cuh>

#include <memory>

#include "common.cuh"

namespace ixb {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr int kBias = 1 << 20;

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

__global__ void hash_insert(const int32_t* coords, int64_t n, unsigned long long* keys,
                            int32_t* vals, uint32_t mask, int* flags /*0 dup,1 range*/) {
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
    const unsigned long long prev = atomicCAS(&keys[h], kEmpty, k);
    if (prev == kEmpty) {
      vals[h] = static_cast<int32_t>(i);
      return;
    }
    if (prev == k) {
      atomicOr(&flags[0], 1);  // duplicate voxel
      return;
    }
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ int hash_find(const unsigned long long* keys, const int32_t* vals,
                                         uint32_t mask, unsigned long long k) {
  uint32_t h = vox_hash(k) & mask;
  for (;;) {
    const unsigned long long cur = keys[h];
    if (cur == k) {
      // vals[h] is written right after the CAS in hash_insert (previous kernel)
      return vals[h];
    }
    if (cur == kEmpty) return -1;
    h = (h + 1) & mask;
  }
}

// hit[z*n + i] = neighbour index (or -1); cnt[z*n + i] = hit >= 0.
__global__ void probe_kernel(const int32_t* coords, int64_t n, const unsigned long long* keys,
                             const int32_t* vals, uint32_t mask, int32_t* hit, int32_t* cnt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= 27 * n) return;
  const int z = static_cast<int>(t / n);
  const int64_t i = t % n;
  const int dx = z / 9 - 1, dy = (z / 3) % 3 - 1, dz = z % 3 - 1;
  const int j = hash_find(keys, vals, mask,
                          vox_key(coords[3 * i] + dx, coords[3 * i + 1] + dy, coords[3 * i + 2] + dz));
  hit[t] = j;
  cnt[t] = j >= 0 ? 1 : 0;
}

__global__ void emit_pairs(const int32_t* hit, const int32_t* pos, int64_t n, int32_t* mo,
                           int32_t* mi, int32_t* mz) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= 27 * n) return;
  const int j = hit[t];
  if (j < 0) return;
  const int64_t p = pos[t];
  mo[p] = static_cast<int32_t>(t % n);
  mi[p] = j;
  mz[p] = static_cast<int32_t>(t / n);
}

}  // namespace

struct KmapPlan {
  cudaStream_t s = nullptr;
  int64_t n = 0, pairs = 0;
  Scratch<int32_t> hit, pos;
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
    H->p.s = s;
    H->p.n = n;
    uint32_t cap = 64;
    while (cap < 2 * n) cap <<= 1;
    Scratch<unsigned long long> keys(cap, s);
    Scratch<int32_t> vals(cap, s);
    Scratch<int> flags(2, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(keys.p, 0xff, cap * sizeof(unsigned long long), s));
    IXB_CUDA_CHECK(cudaMemsetAsync(flags.p, 0, 2 * sizeof(int), s));
    if (n > 0) {
      hash_insert<<<ceil_div(n, 256), 256, 0, s>>>(coords, n, keys.p, vals.p, cap - 1, flags.p);
      IXB_LAUNCH_CHECK("hash_insert");
    }
    const int64_t T = 27 * n;
    H->p.hit = Scratch<int32_t>(T + 1, s);
    H->p.pos = Scratch<int32_t>(T + 1, s);
    Scratch<int32_t> cnt(T + 1, s);
    if (n > 0) {
      probe_kernel<<<ceil_div(T, 256), 256, 0, s>>>(coords, n, keys.p, vals.p, cap - 1,
                                                      H->p.hit.p, cnt.p);
      IXB_LAUNCH_CHECK("probe_kernel");
      size_t tb = 0;
      IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, H->p.pos.p,
                                                   static_cast<int>(T), s));
      Scratch<char> tmp(tb, s);
      IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, H->p.pos.p,
                                                   static_cast<int>(T), s));
      note_launch();
    }
    int hflags[2] = {0, 0};
    int32_t last_pos = 0, last_cnt = 0;
    IXB_CUDA_CHECK(cudaMemcpyAsync(hflags, flags.p, sizeof hflags, cudaMemcpyDeviceToHost, s));
    if (n > 0) {
      IXB_CUDA_CHECK(cudaMemcpyAsync(&last_pos, H->p.pos.p + T - 1, 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaMemcpyAsync(&last_cnt, cnt.p + T - 1, 4, cudaMemcpyDeviceToHost, s));
    }
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));
    if (hflags[1]) fail(IXB_SHAPE, "kernel map: voxel coordinate outside [-2^20, 2^20)");
    if (hflags[0]) fail(IXB_SHAPE, "kernel map: duplicate voxel coordinates");
    H->p.pairs = static_cast<int64_t>(last_pos) + last_cnt;
    *num_pairs = H->p.pairs;
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
    const int64_t T = 27 * H->p.n;
    if (T > 0) {
      emit_pairs<<<ceil_div(T, 256), 256, 0, s>>>(H->p.hit.p, H->p.pos.p, H->p.n, map_out, map_in,
                                                  map_off);
      IXB_LAUNCH_CHECK("emit_pairs");
    }
  });
}

void ixb_kernel_map_free(ixb_kmap* plan) { delete plan; }

}  // extern "C"
