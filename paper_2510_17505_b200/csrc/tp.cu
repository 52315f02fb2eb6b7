// K7 — grouped Clebsch–Gordan tensor product:
//   Z[b,CGI[p,q],w] += CGV[p,q] * X[b,CGJ[p,q],u] * Y[b,CGK[p,q]] * W[(b,)CGL[p],u,w]
// (corpus/grouped_tensor_product.json:2; reference vars b,p,q,w,u; oracle
// plan.cpp:579-594; fused: dot over u, batch [b,p], kernel.cpp:292-357).
//
// tcgen05 path (shared W[l,u,w], U = W = 64, <= 16 irrep components, <= 23
// paths; BASELINE configs[3]). Output-side factorisation:
//   U_{l,i}[b,u] = sum_{(j,k,v) in path l, output i} v * Y[b,k] * X[b,j,u]
//   Z[b,i,:]     = sum_l U_{l,i}[b,:] . W[l]        (99 GEMMs for l_max = 3)
// A CTA is persistent over tiles of 64 edges: X[tile] (64 x 16 x 64 bf16)
// lands in smem by TMA, Y[tile] as fp32. 512 threads = (edge, 8-wide u
// slice) contract the CG entries of one (path, component) pair per step
// (one LDS.128 of X + 8 FMAs per entry). U is split hi + lo bf16, written as
// K-major SW128 tiles (double-buffered) and fed to UMMA M=64,N=64,K=16
// against W[l] (3-slot TMA ring prefetching the next path's W). Z
// accumulates in TMEM: 16 components x 64 columns as two M=64
// half-subpartition sets (lane offset 16), i.e. the full 512 columns. The
// contraction of pair n+1 overlaps the UMMAs of pair n.
// Any other shape, and the per-edge W[b,l,u,w] form, run a CUDA-core kernel
// that follows the reference's summation order exactly.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "sm100.cuh"
#include "tmap.h"

namespace ixb {
namespace {

using namespace sm100;

constexpr int kEdges = 64;       // edges per tile (UMMA M)
constexpr int kTpThreads = 512;  // 64 edges x 8 u-slices
constexpr int kMaxPairs = 128;
constexpr int kMaxEntries = 480;
constexpr int kMaxPaths = 23;
constexpr uint32_t kUTile = kEdges * 128;  // 64 rows x 64 bf16
constexpr uint32_t kWTileTp = 64 * 128;    // 64 u-rows x 64 bf16
constexpr uint32_t kXTile = kEdges * 16 * 128;  // 64 edges x 16 irrep rows x 64 bf16

struct TpMeta {
  int npairs, nentries, nl, ni;
  int4 pair[kMaxPairs];    // {l, i, first entry, entry count}
  int first[kMaxPairs];    // first pair of component i in the list
  int present[16];         // component i receives at least one pair
  int4 entry[kMaxEntries]; // {j, k, float bits of v, 0}
};

struct TpArgs {
  const __nv_bfloat16* X;  // [B, nj, 64]
  const __nv_bfloat16* Y;  // [B, nk]
  float* Z;                // [B, ni, 64]
  int64_t batch;
  int nj, nk, ni;
  int accumulate;
  const TpMeta* meta;
};

__global__ void __launch_bounds__(kTpThreads, 1)
    tp_tc_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                 TpArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* Us = smem;                        // [2 bufs][hi, lo][8 KB]  (SW128 K-major)
  uint8_t* Ws = Us + 4 * kUTile;             // [3][8 KB]               (SW128 MN-major)
  uint8_t* Xs = Ws + 3 * kWTileTp;           // [64 edges * nj rows][128 B]
  float* Ys = reinterpret_cast<float*>(Xs + kXTile);  // [64][16]
  uint64_t* x_full = reinterpret_cast<uint64_t*>(Ys + kEdges * 16);
  uint64_t* w_full = x_full + 1;  // [3]
  uint64_t* mma_done = w_full + 3;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mma_done + 2);
  __shared__ int4 s_pair[kMaxPairs];  // {l | is_first_of_component << 16, i, entry0, count}
  __shared__ int4 s_entry[kMaxEntries];

  const int tid = threadIdx.x, warp = tid >> 5;
  const int b_loc = tid >> 3, slice = tid & 7;  // edge in tile, u slice [8*slice, +8)
  const int npairs = a.meta->npairs;
  for (int i = tid; i < npairs; i += kTpThreads) {
    int4 pr = a.meta->pair[i];
    pr.x |= (a.meta->first[i] == i) ? (1 << 16) : 0;
    s_pair[i] = pr;
  }
  for (int i = tid; i < a.meta->nentries; i += kTpThreads) s_entry[i] = a.meta->entry[i];
  if (tid == 0) {
    mbar_init(x_full, 1);
    for (int b = 0; b < 3; ++b) mbar_init(&w_full[b], 1);
    mbar_init(&mma_done[0], 1);
    mbar_init(&mma_done[1], 1);
    fence_barrier_init();
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
  }
  if (warp == 0) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = idesc_bf16_f32(64, 64, /*A K-major*/ false, /*B MN-major*/ true);
  // whole 256-row boxes land (out-of-range rows zero-filled), so expect them all
  const uint32_t x_bytes = static_cast<uint32_t>(((kEdges * a.nj + 255) / 256) * 256 * 128);
  const uint64_t keep = l2_evict_last(), stream = l2_evict_first();

  // thread-0 state for the W ring (3 buffers, one per upcoming path)
  uint32_t w_loads[3] = {0, 0, 0};
  int n_global = 0;  // pairs issued by this CTA (U buffer / barrier phase counter)
  int tiles_done = 0;
  const int64_t ntiles = (a.batch + kEdges - 1) / kEdges;
  auto issue_w = [&](int path, int slot) {
    mbar_arrive_expect_tx(&w_full[slot], kWTileTp);
    tma_load_2d(Ws + slot * kWTileTp, &tmW, &w_full[slot], 0, path * 64, keep);
    ++w_loads[slot];
  };
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tiles_done) {
    // ---- stage the tile: X by TMA (rows b*nj + j), Y as fp32, first paths' W
    if (tid == 0) {
      mbar_arrive_expect_tx(x_full, x_bytes);
      const int rows = kEdges * a.nj;
      for (int r0 = 0; r0 < rows; r0 += 256) {
        tma_load_2d(Xs + r0 * 128, &tmX, x_full, 0,
                    static_cast<int32_t>(tile * kEdges * a.nj + r0), stream);
      }
      if (npairs > 0) issue_w(s_pair[0].x & 0xFFFF, 0);
    }
    for (int e = tid; e < kEdges * 16; e += kTpThreads) {
      const int bb = e >> 4, k = e & 15;
      const int64_t b = tile * kEdges + bb;
      Ys[e] = (b < a.batch && k < a.nk) ? __bfloat162float(a.Y[b * a.nk + k]) : 0.f;
    }
    mbar_wait(x_full, tiles_done & 1);
    __syncthreads();
    const uint8_t* xrow = Xs + b_loc * a.nj * 128 + slice * 16;
    const float* yrow = Ys + b_loc * 16;
    int cur_path = -1, path_idx = -1;
    for (int n = 0; n < npairs; ++n, ++n_global) {
      const int4 pr = s_pair[n];
      const int path = pr.x & 0xFFFF;
      const bool new_path = path != cur_path;
      if (new_path) {
        cur_path = path;
        ++path_idx;
        if (tid == 0) {
          // prefetch the next path's W into the slot last used two paths ago
          for (int m = n + 1; m < npairs; ++m) {
            const int pth = s_pair[m].x & 0xFFFF;
            if (pth != path) {
              issue_w(pth, (path_idx + 1) % 3);
              break;
            }
          }
        }
      }
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      for (int e = pr.z; e < pr.z + pr.w; ++e) {
        const int4 en = s_entry[e];
        const float coef = __int_as_float(en.z) * yrow[en.y];
        const uint4 xv = *reinterpret_cast<const uint4*>(xrow + en.x * 128);
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&xv);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = __bfloat1622float2(h[q]);
          acc[2 * q] = fmaf(coef, f.x, acc[2 * q]);
          acc[2 * q + 1] = fmaf(coef, f.y, acc[2 * q + 1]);
        }
      }
      // U = hi + lo, both bf16: the UMMA pair sees U to ~2^-16 relative, so the
      // only bf16 roundings are the operands X, Y, W themselves.
      uint4 hi, lo;
      __nv_bfloat162* ph = reinterpret_cast<__nv_bfloat162*>(&hi);
      __nv_bfloat162* pl = reinterpret_cast<__nv_bfloat162*>(&lo);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ph[q] = __floats2bfloat162_rn(acc[2 * q], acc[2 * q + 1]);
        const float2 back = __bfloat1622float2(ph[q]);
        pl[q] = __floats2bfloat162_rn(acc[2 * q] - back.x, acc[2 * q + 1] - back.y);
      }
      const int buf = n_global & 1;
      if (n_global >= 2) mbar_wait(&mma_done[buf], ((n_global - 2) >> 1) & 1);
      const uint32_t off = b_loc * 128 + ((slice ^ (b_loc & 7)) << 4);
      *reinterpret_cast<uint4*>(Us + (2 * buf) * kUTile + off) = hi;
      *reinterpret_cast<uint4*>(Us + (2 * buf + 1) * kUTile + off) = lo;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        const int wslot = path_idx % 3;
        if (new_path) mbar_wait(&w_full[wslot], (w_loads[wslot] - 1) & 1);
        tc_fence_after();
        const int i = pr.y;
        // component i: columns 64*(i%8), lane set 16*(i/8) (M=64 half subpartitions)
        const uint32_t d = tmem + (static_cast<uint32_t>((i >> 3) * 16) << 16) + (i & 7) * 64;
        const uint32_t u0 = smem_u32(Us + (2 * buf) * kUTile);
        const uint32_t w0 = smem_u32(Ws + wslot * kWTileTp);
        const bool first = (pr.x >> 16) & 1;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc(w0 + kk * 2048, 8192, 1024, kLayoutSW128);
          umma_f16(d, smem_desc(u0 + kk * 32, 16, 1024, kLayoutSW128), bd, idesc,
                   (!first || kk > 0) ? 1u : 0u);
          umma_f16(d, smem_desc(u0 + kUTile + kk * 32, 16, 1024, kLayoutSW128), bd, idesc, 1u);
        }
        umma_commit(&mma_done[buf]);
      }
    }
    // ---- epilogue: all UMMAs of this tile done -> TMEM -> Z
    if (npairs > 0) {
      const int last = n_global - 1;
      mbar_wait(&mma_done[last & 1], (last >> 1) & 1);
    }
    tc_fence_after();
    const int quarter = warp & 3, wg = warp >> 2;  // 4 warps per TMEM lane quarter
    const int t = tid & 31;
    const int row = quarter * 16 + (t & 15);        // edge within tile
    const int64_t be = tile * kEdges + row;
#pragma unroll 1
    for (int cb = 2 * wg; cb < 2 * wg + 2; ++cb) {  // column block: components cb, cb+8
      const int comp = cb + 8 * (t >> 4);
      float outv[64];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[16];
        tmem_ld_32x32b_x16(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + cb * 64 + c * 16,
                           r);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) outv[c * 16 + e] = __uint_as_float(r[e]);
      }
      const bool has = comp < a.ni && a.meta->present[comp];
      if (be < a.batch && comp < a.ni) {
        float4* z = reinterpret_cast<float4*>(a.Z + (be * a.ni + comp) * 64);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          float4 v = has ? make_float4(outv[4 * e], outv[4 * e + 1], outv[4 * e + 2],
                                       outv[4 * e + 3])
                         : make_float4(0.f, 0.f, 0.f, 0.f);
          if (a.accumulate) {
            const float4 o = z[e];
            v.x += o.x;
            v.y += o.y;
            v.z += o.z;
            v.w += o.w;
          }
          z[e] = v;
        }
      }
    }
    tc_fence_before();
    __syncthreads();  // TMEM drained and Xs/Ys free before the next tile
  }
  __syncthreads();
  if (warp == 0) {
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

extern "C" int ixb_tp_grouped(const int32_t* CGL, const int32_t* CGI, const int32_t* CGJ,
                              const int32_t* CGK, const float* CGV, int64_t G, int64_t g,
                              const void* X, const void* Y, const void* W, int w_per_batch,
                              int64_t batch, int64_t ni, int64_t nj, int64_t nk, int64_t nl,
                              int64_t U, int64_t Wd, float* Z, int accumulate, int flags,
                              ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (G < 0 || g < 1 || batch < 0 || ni < 0 || nj < 0 || nk < 0 || nl < 0 || U < 1 || Wd < 1)
      fail(IXB_SHAPE, "ixb_tp_grouped: bad extents");
    if (batch == 0 || ni == 0) return;
    // The CG table is tiny: bring it to the host, validate it like the plan
    // executor (gathers X/CGJ, Y/CGK, W/CGL, then scatter Z/CGI), and build
    // the per-component slot lists.
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
    // slots per output component, in slot order (pads v == 0 are inert)
    std::vector<std::vector<int32_t>> by_i(ni);
    for (int64_t sl = 0; sl < slots; ++sl) by_i[hi[sl]].push_back(static_cast<int32_t>(sl));
    const bool tc = !w_per_batch && U == 64 && Wd == 64 && ni <= 16 && nj <= 16 && nk <= 16 &&
                    nl >= 1 && nl <= kMaxPaths && reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(W) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(Z) % 16 == 0;
    if (tc) {
      // pairs (l, i) in (l, i) order; entries (j, k, v) in slot order, pads dropped
      TpMeta meta{};
      meta.nl = static_cast<int>(nl);
      meta.ni = static_cast<int>(ni);
      std::vector<std::vector<std::vector<int32_t>>> li(nl, std::vector<std::vector<int32_t>>(ni));
      for (int64_t sl = 0; sl < slots; ++sl) {
        if (hv[sl] == 0.f) continue;
        li[hl[sl / g]][hi[sl]].push_back(static_cast<int32_t>(sl));
      }
      int np = 0, ne = 0;
      std::vector<int> first_of_i(ni, -1);
      for (int l = 0; l < nl; ++l) {
        for (int i = 0; i < ni; ++i) {
          if (li[l][i].empty()) continue;
          if (np >= kMaxPairs || ne + static_cast<int>(li[l][i].size()) > kMaxEntries)
            fail(IXB_SHAPE, "ixb_tp_grouped: CG table too large for the tensor-core path");
          if (first_of_i[i] < 0) first_of_i[i] = np;
          meta.pair[np] = make_int4(l, i, ne, static_cast<int>(li[l][i].size()));
          for (int32_t sl : li[l][i]) {
            int vbits;
            std::memcpy(&vbits, &hv[sl], sizeof vbits);
            meta.entry[ne++] = make_int4(hj[sl], hk[sl], vbits, 0);
          }
          ++np;
        }
      }
      meta.npairs = np;
      meta.nentries = ne;
      for (int n = 0; n < np; ++n) meta.first[n] = first_of_i[meta.pair[n].y];
      // components that receive no pair get zeros (`=`) / keep their value (`+=`)
      for (int i = 0; i < 16; ++i) meta.present[i] = (i < ni && first_of_i[i] >= 0) ? 1 : 0;
      Scratch<TpMeta> dmeta(1, s);
      IXB_CUDA_CHECK(cudaMemcpyAsync(dmeta.p, &meta, sizeof meta, cudaMemcpyHostToDevice, s));
      const CUtensorMap tmW = make_tmap_2d(W, 64, static_cast<uint64_t>(nl) * 64, 128, 64, 64,
                                           CU_TENSOR_MAP_SWIZZLE_128B);
      const CUtensorMap tmX = make_tmap_2d(X, 64, static_cast<uint64_t>(batch) * nj, 128, 64, 256,
                                           CU_TENSOR_MAP_SWIZZLE_NONE);
      TpArgs args{static_cast<const __nv_bfloat16*>(X), static_cast<const __nv_bfloat16*>(Y), Z,
                  batch, static_cast<int>(nj), static_cast<int>(nk), static_cast<int>(ni),
                  accumulate, dmeta.p};
      const uint32_t smem = 4 * kUTile + 3 * kWTileTp + kXTile + kEdges * 16 * 4 + 256 + 1024;
      static std::once_flag once;
      std::call_once(once, [&] {
        cuda_check(cudaFuncSetAttribute(tp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        smem),
                   "cudaFuncSetAttribute(tp_tc_kernel)");
      });
      int64_t grid = ceil_div(batch, kEdges);
      if (grid > sm_count()) grid = sm_count();
      tp_tc_kernel<<<static_cast<unsigned>(grid), kTpThreads, smem, s>>>(tmW, tmX, args);
      IXB_LAUNCH_CHECK("tp_tc_kernel");
      IXB_CUDA_CHECK(cudaStreamSynchronize(s));  // host meta buffer lifetime
      return;
    }
    std::vector<int32_t> rowptr(ni + 1, 0), flat;
    for (int64_t i = 0; i < ni; ++i) {
      rowptr[i + 1] = rowptr[i] + static_cast<int32_t>(by_i[i].size());
      flat.insert(flat.end(), by_i[i].begin(), by_i[i].end());
    }
    Scratch<int32_t> drow(ni + 1, s), dslots(flat.size() + 1, s);
    IXB_CUDA_CHECK(cudaMemcpyAsync(drow.p, rowptr.data(), (ni + 1) * 4, cudaMemcpyHostToDevice, s));
    if (!flat.empty()) {
      IXB_CUDA_CHECK(cudaMemcpyAsync(dslots.p, flat.data(), flat.size() * 4,
                                     cudaMemcpyHostToDevice, s));
    }
    const int64_t n = batch * ni * Wd;
    tp_simt_kernel<<<ceil_div(n, 256), 256, 0, s>>>(
        drow.p, dslots.p, CGL, CGJ, CGK, CGV, g, static_cast<const __nv_bfloat16*>(X),
        static_cast<const __nv_bfloat16*>(Y), static_cast<const __nv_bfloat16*>(W), w_per_batch,
        batch, ni, nj, nk, nl, U, Wd, Z, accumulate);
    IXB_LAUNCH_CHECK("tp_simt_kernel");
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));  // host vectors' lifetime
  });
}
