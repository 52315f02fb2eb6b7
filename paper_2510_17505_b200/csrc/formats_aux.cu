// GroupCOO helpers around the builders, on the
// device: real_count / pad_count (formats.cpp:105-113), is_ell
// (formats.cpp:202-208), the occupancy maximum that ell_view uses
// (formats.cpp:196-200) and groupcoo_to_coo (formats.cpp:176-194: the
// non-pad slots in slot order; the caller canonicalizes, as the reference
// does, with the g = 1 grouping). Integer/byte work: one pass each.
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/transform_iterator.h>

#include "common.cuh"

namespace ixb {
namespace {

__global__ void mask_count_kernel(const uint8_t* mask, int64_t n, unsigned long long* out) {
  __shared__ unsigned long long part[8];
  unsigned long long s = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    s += mask[i] ? 1u : 0u;
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
    atomicAdd(out, t);
  }
}

__global__ void adjacent_equal_kernel(const int32_t* gc, int64_t G, int* flag) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1;
  if (i < G && gc[i] == gc[i - 1]) *flag = 1;
}

__global__ void occ_hist_kernel(const int32_t* coord, int64_t nnz, int64_t extent, int32_t* occ,
                                int* bad) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const int32_t c = coord[i];
  if (c < 0 || c >= extent) {
    *bad = 1;
    return;
  }
  atomicAdd(&occ[c], 1);
}

__global__ void max_kernel(const int32_t* v, int64_t n, int* out) {
  int m = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = max(m, v[i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

struct MaskToInt {
  __host__ __device__ int operator()(uint8_t m) const { return m ? 1 : 0; }
};

// Slot s (non-pad) -> COO entry pos[s]: (group coord, member coord) in the
// order of group_dim, value bytes copied as is.
__global__ void compact_kernel(const int32_t* AM, const int32_t* AK, const uint8_t* vals,
                               int esize, const uint8_t* mask, const int32_t* pos, int64_t G,
                               int64_t g, int group_dim, int32_t* row_out, int32_t* col_out,
                               uint8_t* val_out) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= G * g || !mask[s]) return;
  const int64_t p = pos[s];
  const int32_t gco = AM[s / g], mco = AK[s];
  row_out[p] = group_dim == 0 ? gco : mco;
  col_out[p] = group_dim == 0 ? mco : gco;
  if (vals)
    for (int b = 0; b < esize; ++b) val_out[p * esize + b] = vals[s * esize + b];
}

int elem_size(int dtype) {
  switch (dtype) {
    case IXB_F32: case IXB_I32: return 4;
    case IXB_BF16: return 2;
    case IXB_F64: case IXB_I64: return 8;
    case IXB_U8: return 1;
    default: fail(IXB_SHAPE, "unknown dtype"); return 0;
  }
}

}  // namespace
}  // namespace ixb

using namespace ixb;

extern "C" int ixb_mask_real_count(const uint8_t* mask, int64_t slots, ixb_stream stream,
                                   int64_t* real) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (slots < 0 || !real) fail(IXB_SHAPE, "ixb_mask_real_count: bad arguments");
    *real = 0;
    if (slots == 0) return;
    Scratch<unsigned long long> acc(1, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(acc.p, 0, 8, s));
    const int64_t blocks = std::min<int64_t>(ceil_div(slots, 256), 4 * sm_count());
    mask_count_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(mask, slots, acc.p);
    IXB_LAUNCH_CHECK("mask_count_kernel");
    unsigned long long h = 0;
    {
      HostReads rd(s);
      rd.add(&h, acc.p, 8);
      rd.wait();
    }
    *real = static_cast<int64_t>(h);
  });
}

extern "C" int ixb_is_ell(const int32_t* group_coord, int64_t G, ixb_stream stream, int* is_ell) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (G < 0 || !is_ell) fail(IXB_SHAPE, "ixb_is_ell: bad arguments");
    *is_ell = 1;
    if (G < 2) return;
    Scratch<int> flag(1, s);
    IXB_CUDA_CHECK(cudaMemsetAsync(flag.p, 0, 4, s));
    adjacent_equal_kernel<<<static_cast<unsigned>(ceil_div(G - 1, 256)), 256, 0, s>>>(
        group_coord, G, flag.p);
    IXB_LAUNCH_CHECK("adjacent_equal_kernel");
    int h = 0;
    {
      HostReads rd(s);
      rd.add(&h, flag.p, 4);
      rd.wait();
    }
    *is_ell = h ? 0 : 1;
  });
}

extern "C" int ixb_max_occupancy(const int32_t* coord, int64_t nnz, int64_t extent,
                                 ixb_stream stream, int64_t* max_occ) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (nnz < 0 || extent < 0 || !max_occ) fail(IXB_SHAPE, "ixb_max_occupancy: bad arguments");
    *max_occ = 0;
    if (nnz == 0 || extent == 0) return;
    Scratch<int32_t> occ(extent, s);
    Scratch<int> res(2, s);  // max, bad coordinate
    IXB_CUDA_CHECK(cudaMemsetAsync(occ.p, 0, extent * 4, s));
    IXB_CUDA_CHECK(cudaMemsetAsync(res.p, 0, 8, s));
    occ_hist_kernel<<<static_cast<unsigned>(ceil_div(nnz, 256)), 256, 0, s>>>(coord, nnz, extent,
                                                                             occ.p, res.p + 1);
    IXB_LAUNCH_CHECK("occ_hist_kernel");
    const int64_t blocks = std::min<int64_t>(ceil_div(extent, 256), 4 * sm_count());
    max_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(occ.p, extent, res.p);
    IXB_LAUNCH_CHECK("max_kernel");
    int h[2] = {0, 0};
    {
      HostReads rd(s);
      rd.add(h, res.p, 8);
      rd.wait();
    }
    if (h[1]) fail(IXB_SHAPE, "occupancy: coordinate out of range");
    *max_occ = h[0];
  });
}

extern "C" int ixb_groupcoo_to_coo(const int32_t* group_coord, const int32_t* member_coord,
                                   const void* values, int dtype, const uint8_t* mask, int64_t G,
                                   int64_t g, int group_dim, int32_t* row_out, int32_t* col_out,
                                   void* val_out, ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (G < 0 || g < 1 || (group_dim != 0 && group_dim != 1))
      fail(IXB_SHAPE, "ixb_groupcoo_to_coo: bad extents");
    const int64_t slots = G * g;
    if (slots == 0) return;
    if (slots > INT32_MAX) fail(IXB_SHAPE, "ixb_groupcoo_to_coo: too many slots");
    const int esize = values ? elem_size(dtype) : 0;
    Scratch<int32_t> pos(slots + 1, s);
    auto in = thrust::make_transform_iterator(mask, MaskToInt());
    size_t tb = 0;
    IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, pos.p, static_cast<int>(slots), s));
    Scratch<char> tmp(tb, s);
    IXB_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, pos.p, static_cast<int>(slots), s));
    note_launch();
    compact_kernel<<<static_cast<unsigned>(ceil_div(slots, 256)), 256, 0, s>>>(
        group_coord, member_coord, static_cast<const uint8_t*>(values), esize, mask, pos.p, G, g,
        group_dim, row_out, col_out, static_cast<uint8_t*>(val_out));
    IXB_LAUNCH_CHECK("compact_kernel");
  });
}
