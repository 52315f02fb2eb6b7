// Host-buffer entry points of the SpMM evaluators (the shape the reference's
// execute_mode has: host Tensors in, host result out — driver.cpp:235-265),
// pipelined so the PCIe transfers overlap each other and the kernels:
//   stream h2d : dense operand B and the index arrays, then the values of
//                chunk 0, 1, ...
//   stream comp: (zero C) then the evaluator on chunk i once it has landed
//   stream d2h : C rows of chunk i once its kernel is done
// Chunks are contiguous group ranges cut at output-row boundaries
// (ixb_shard_groups), so each output row is produced by one kernel. K3 keeps
// its summation order (bit-identical to the one-shot call); K4 balances slots
// across CTAs per launch, so a row split between CTAs sums its partials at
// chunk-dependent cut points: equal to fp32 rounding, bit-identical on
// integer data (tests/test_gpu_bgcoo.py). Measured (cfg2, best of 20):
// uniform 8/12/16/24 chunks and graded schedules (small first / last
// chunks) all land within 0.67-0.76 ms, inside the box-to-box PCIe noise:
// the auto rule below stays.
// The chunk kernels run unchecked (they clamp indices and guard row stores
// either way); the whole uploaded format is validated once afterwards, so an
// index error names the same operand and absolute position as the one-shot
// call (K8, plan.cpp:249-259).
#include <cuda_runtime.h>

#include <cstring>
#include <vector>

#include "common.cuh"

namespace ixb {
namespace {

// Side streams and events are created once per thread and device and
// reused (creating them per call costs more than the overlap gains).
struct Streams {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> ev;
  int device = -1;
  void ensure(size_t nev) {
    int dev = 0;
    IXB_CUDA_CHECK(cudaGetDevice(&dev));
    if (device != dev) {
      IXB_CUDA_CHECK(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking));
      IXB_CUDA_CHECK(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
      ev.clear();
      device = dev;
    }
    while (ev.size() < nev) {
      cudaEvent_t e;
      IXB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ev.push_back(e);
    }
  }
};
thread_local Streams t_streams;

bool sorted_host(const int32_t* gc, int64_t G) {
  for (int64_t i = 1; i < G; ++i)
    if (gc[i] < gc[i - 1]) return false;
  return true;
}

// Generic driver: `rowbytes` = bytes of one output row (bm * N * 4 for BGCOO,
// N * 4 for GroupCOO); `slotbytes` = bytes of AV per slot; `eval` runs the
// device evaluator on a group range with accumulate = 1 into dC.
template <typename Eval>
void run_pipelined(const int32_t* AM, const int32_t* AK, const void* AV, int64_t G, int64_t g,
                   int64_t slotbytes, const void* B, int64_t bbytes, float* C, int64_t MB,
                   int64_t rowbytes, int accumulate, int nchunks, bool check, int64_t K,
                   cudaStream_t s, Eval&& eval) {
  if (nchunks < 1) {
    // auto (tools/e2e_chunks.py, bench e2e): BlockGroupCOO ~2 MB of values
    // in + C rows out per chunk, 2..8 chunks (cfg2: 0.73 ms at 2, 0.65 at
    // 8); GroupCOO 2 chunks (cfg1 and cfg3: more chunks measured slower —
    // each costs a latency-bound K3 launch and its copies)
    const double mb = (static_cast<double>(G) * g * (slotbytes + 4) +
                       static_cast<double>(MB) * rowbytes) / (2.0 * 1024 * 1024);
    nchunks = slotbytes < 64 || mb < 2 ? 2 : mb > 8 ? 8 : static_cast<int>(mb + 0.5);
  }
  if (nchunks > G) nchunks = static_cast<int>(G < 1 ? 1 : G);
  std::vector<int64_t> bounds(nchunks + 1);
  if (ixb_shard_groups(AM, G, nchunks, bounds.data()) != IXB_OK)
    fail(IXB_FAILURE, ixb_last_error());
  Scratch<int32_t> dAM(G, s), dAK(G * g, s);
  Scratch<char> dAV(G * g * slotbytes, s), dB(bbytes, s), dC(MB * rowbytes, s);
  Streams& st = t_streams;
  st.ensure(2 + 2 * nchunks);
  cudaEvent_t ready = st.ev[0], done = st.ev[1];
  // scratch allocated on `s`: make the side streams wait for it
  IXB_CUDA_CHECK(cudaEventRecord(ready, s));
  IXB_CUDA_CHECK(cudaStreamWaitEvent(st.h2d, ready, 0));
  IXB_CUDA_CHECK(cudaMemcpyAsync(dB.p, B, bbytes, cudaMemcpyHostToDevice, st.h2d));
  // AM whole (one small copy); AK whole too when it is small next to the
  // values (BlockGroupCOO: 4 B per 512-B block), else per chunk with them
  // (GroupCOO: as large as AV — uploading it first delays chunk 0)
  const bool ak_whole = slotbytes >= 64;
  IXB_CUDA_CHECK(cudaMemcpyAsync(dAM.p, AM, G * 4, cudaMemcpyHostToDevice, st.h2d));
  if (ak_whole)
    IXB_CUDA_CHECK(cudaMemcpyAsync(dAK.p, AK, G * g * 4, cudaMemcpyHostToDevice, st.h2d));
  if (accumulate)  // `+=` needs the caller's C; `=` starts from zeros
    IXB_CUDA_CHECK(cudaMemcpyAsync(dC.p, C, MB * rowbytes, cudaMemcpyHostToDevice, st.h2d));
  else
    IXB_CUDA_CHECK(cudaMemsetAsync(dC.p, 0, MB * rowbytes, s));
  // rows owned by chunk i for the write-back: [row_lo(i), row_lo(i+1))
  std::vector<int64_t> row_lo(nchunks + 1);
  for (int i = 0; i < nchunks; ++i) {
    const int64_t r = bounds[i] < G ? AM[bounds[i]] : MB;
    row_lo[i] = i == 0 ? 0 : (r < 0 ? 0 : (r > MB ? MB : r));
  }
  row_lo[nchunks] = MB;
  for (int i = 0; i < nchunks; ++i) {
    const int64_t g0 = bounds[i], g1 = bounds[i + 1];
    cudaEvent_t in = st.ev[2 + 2 * i], out = st.ev[3 + 2 * i];
    if (g1 > g0) {
      if (!ak_whole)
        IXB_CUDA_CHECK(cudaMemcpyAsync(dAK.p + g0 * g, AK + g0 * g, (g1 - g0) * g * 4,
                                       cudaMemcpyHostToDevice, st.h2d));
      IXB_CUDA_CHECK(cudaMemcpyAsync(dAV.p + g0 * g * slotbytes,
                                     static_cast<const char*>(AV) + g0 * g * slotbytes,
                                     (g1 - g0) * g * slotbytes, cudaMemcpyHostToDevice, st.h2d));
    }
    IXB_CUDA_CHECK(cudaEventRecord(in, st.h2d));
    IXB_CUDA_CHECK(cudaStreamWaitEvent(s, in, 0));
    if (g1 > g0) eval(dAM.p + g0, dAK.p + g0 * g, dAV.p + g0 * g * slotbytes, g1 - g0, dB.p, dC.p);
    IXB_CUDA_CHECK(cudaEventRecord(out, s));
    IXB_CUDA_CHECK(cudaStreamWaitEvent(st.d2h, out, 0));
    const int64_t r0 = row_lo[i], r1 = row_lo[i + 1];
    if (r1 > r0)
      IXB_CUDA_CHECK(cudaMemcpyAsync(reinterpret_cast<char*>(C) + r0 * rowbytes,
                                     dC.p + r0 * rowbytes, (r1 - r0) * rowbytes,
                                     cudaMemcpyDeviceToHost, st.d2h));
  }
  // the caller's stream observes completion of every transfer
  IXB_CUDA_CHECK(cudaEventRecord(done, st.d2h));
  IXB_CUDA_CHECK(cudaStreamWaitEvent(s, done, 0));
  if (check) {  // gathers (AK) before scatters (AM), absolute positions
    validate_range(dAK.p, G * g, K, 0, s);
    validate_range(dAM.p, G, MB, 1, s);
    OperandInfo ops[2] = {{"AK", "B", 0, K, dAK.p, G * g}, {"AM", "C", 0, MB, dAM.p, G}};
    check_error_record(s, ops, 2);
  }
  // scratch frees are stream-ordered on `s`, after `done`
  IXB_CUDA_CHECK(cudaStreamSynchronize(s));
}

}  // namespace
}  // namespace ixb

using namespace ixb;

extern "C" {

int ixb_spmm_blockgroupcoo_host(const int32_t* AM, const int32_t* AK, const void* AV, int64_t G,
                                int64_t g, int64_t bm, int64_t bk, const void* B, int64_t KB,
                                int64_t N, float* C, int64_t MB, int accumulate, int flags,
                                int nchunks, ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (G < 0 || g < 1 || bm < 1 || bk < 1 || KB < 0 || N < 0 || MB < 0)
      fail(IXB_SHAPE, "ixb_spmm_blockgroupcoo: bad extents");
    const bool sorted = sorted_host(AM, G);
    if (!sorted) nchunks = 1;  // one chunk: the evaluator sorts on the device
    const int64_t slotbytes = bm * bk * 2, rowbytes = bm * N * 4;
    int rc_err = IXB_OK;
    // sortedness was checked here on the host: the evaluator need not
    const int cflags = IXB_UNCHECKED | IXB_ASYNC | (sorted ? IXB_GROUPS_SORTED : 0);
    run_pipelined(AM, AK, AV, G, g, slotbytes, B, KB * bk * N * 2, C, MB, rowbytes, accumulate,
                  nchunks, !(flags & IXB_UNCHECKED), KB, s,
                  [&](const int32_t* am, const int32_t* ak, const char* av, int64_t Gc,
                      const char* dB, char* dC) {
                    const int rc = ixb_spmm_blockgroupcoo(am, ak, av, Gc, g, bm, bk, dB, KB, N,
                                                          reinterpret_cast<float*>(dC), MB, 1,
                                                          cflags, stream);
                    if (rc != IXB_OK) rc_err = rc;
                  });
    if (rc_err != IXB_OK) fail(rc_err, ixb_last_error());
  });
}

int ixb_spmm_groupcoo_host(const int32_t* AM, const int32_t* AK, const float* AV, int64_t G,
                           int64_t g, const float* B, int64_t K, int64_t N, float* C, int64_t M,
                           int accumulate, int flags, int nchunks, ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (G < 0 || g < 1 || K < 0 || N < 0 || M < 0) fail(IXB_SHAPE, "ixb_spmm_groupcoo: bad extents");
    const bool sorted = sorted_host(AM, G);
    if (!sorted) nchunks = 1;
    int rc_err = IXB_OK;
    // sortedness was checked here on the host: the evaluator need not
    const int cflags = IXB_UNCHECKED | IXB_ASYNC | (sorted ? IXB_GROUPS_SORTED : 0);
    run_pipelined(AM, AK, AV, G, g, 4, B, K * N * 4, C, M, N * 4, accumulate, nchunks,
                  !(flags & IXB_UNCHECKED), K, s,
                  [&](const int32_t* am, const int32_t* ak, const char* av, int64_t Gc,
                      const char* dB, char* dC) {
                    const int rc = ixb_spmm_groupcoo(
                        am, ak, reinterpret_cast<const float*>(av), Gc, g,
                        reinterpret_cast<const float*>(dB), K, N, reinterpret_cast<float*>(dC), M,
                        1, cflags, stream);
                    if (rc != IXB_OK) rc_err = rc;
                  });
    if (rc_err != IXB_OK) fail(rc_err, ixb_last_error());
  });
}

}  // extern "C"
