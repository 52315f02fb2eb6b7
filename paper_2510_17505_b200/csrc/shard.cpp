// Multi-GPU sharded evaluation behind the C-ABI: one process
// per GPU, the format and the dense operand replicated, each rank evaluating
// its row-group (SpMM) or point-block (conv) shard straight into its rows of
// the FULL output, and NCCL over NVLink used only to all-gather the output.
//
// The gather overlaps the evaluation: a rank's shard is cut into `nchunks`
// row-aligned chunks; as chunk c finishes on the compute stream, one NCCL
// group of broadcasts on a side stream sends every rank's chunk c into place
// (ncclBroadcast root q, in place at q's rows — an all-gather of unequal
// slabs with no padding and no re-layout pass) while chunk c+1 computes.
// Chunk boundaries are cut only where the output row changes, so every row
// keeps one owner and its summation order: the gathered result equals the
// unsharded evaluation bit for bit on GroupCOO (K3) and conv (K6); K4
// balances slots per launch, so its chunks agree to fp32 rounding.
//
// NCCL is loaded at first use (dlopen "libnccl.so.2": under torch that is
// torch's own, already loaded copy), so libixb has no link-time dependency.
#include <dlfcn.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "ixb_internal.h"

namespace ixb {
void spmm_groupcoo(const int32_t* AM, const int32_t* AK, const float* AV, int64_t G, int64_t g,
                   const float* B, int64_t K, int64_t N, float* C, int64_t M, int accumulate,
                   int flags, cudaStream_t s);
void spmm_blockgroupcoo(const int32_t* AM, const int32_t* AK, const void* AV, int64_t G,
                        int64_t g, int64_t bm, int64_t bk, const void* B, int64_t KB, int64_t N,
                        float* C, int64_t MB, int accumulate, int flags, cudaStream_t s);
}  // namespace ixb

namespace {

using namespace ixb;

// ------------------------------------------------------------ NCCL (dlopen)
typedef int nccl_result;  // ncclResult_t: 0 = ncclSuccess
typedef struct nccl_comm* nccl_comm_t;
struct nccl_unique_id {
  char internal[128];
};
constexpr int kNcclInt8 = 0;

struct Nccl {
  void* h = nullptr;
  nccl_result (*get_unique_id)(nccl_unique_id*) = nullptr;
  nccl_result (*comm_init_rank)(nccl_comm_t*, int, nccl_unique_id, int) = nullptr;
  nccl_result (*comm_destroy)(nccl_comm_t) = nullptr;
  nccl_result (*broadcast)(const void*, void*, size_t, int, int, nccl_comm_t,
                           cudaStream_t) = nullptr;
  nccl_result (*group_start)() = nullptr;
  nccl_result (*group_end)() = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
};

Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!n.h) {
      err = dlerror();
      return;
    }
    auto sym = [](const char* name) {
      void* p = dlsym(n.h, name);
      if (!p) err = std::string("missing NCCL symbol ") + name;
      return p;
    };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.broadcast = reinterpret_cast<decltype(n.broadcast)>(sym("ncclBroadcast"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
  });
  if (!n.h || !err.empty()) fail(IXB_FAILURE, "NCCL unavailable: " + err);
  return n;
}

void nccl_check(nccl_result r, const char* what) {
  if (r != 0) fail(IXB_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

// Row-aligned cut of groups [g0, g1) into `parts` ranges of ~equal groups
// (as ixb_shard_groups); bounds get parts+1 entries.
void cut_groups(const int32_t* gc, int64_t g0, int64_t g1, int parts, int64_t* bounds) {
  bounds[0] = g0;
  for (int r = 1; r < parts; ++r) {
    int64_t cut = g0 + ((g1 - g0) * r) / parts;
    if (cut < bounds[r - 1]) cut = bounds[r - 1];
    while (cut > g0 && cut < g1 && gc[cut] == gc[cut - 1]) ++cut;
    bounds[r] = cut;
  }
  bounds[parts] = g1;
}

}  // namespace

struct ixb_comm {
  nccl_comm_t comm = nullptr;
  int world = 1, rank = 0, device = 0;
  cudaStream_t side = nullptr;  // broadcasts run here, overlapping the compute stream
  std::vector<cudaEvent_t> ev;
};

// Every rank's chunks: chunk (q, c) = groups [g[q][c], g[q][c+1]) writing
// rows [r[q][c], r[q][c+1]); the rank's own groups re-based to chunk rows.
struct ixb_shard_plan {
  int world = 1, rank = 0, nchunks = 1;
  int64_t G = 0, rows = 0;
  std::vector<std::vector<int64_t>> gb, rb;  // [world][nchunks + 1]
  int32_t* am_local = nullptr;               // device: AM[p] - chunk row start, own groups
  ~ixb_shard_plan() { cudaFree(am_local); }  // synchronous: in-flight runs finish first
};

extern "C" {

int ixb_comm_unique_id(void* id) {
  return ixb_guard([&] {
    if (!id) fail(IXB_FAILURE, "ixb_comm_unique_id: null id");
    nccl_unique_id u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, sizeof u.internal);
  });
}

int ixb_comm_init(const void* id, int world, int rank, ixb_comm** out) {
  return ixb_guard([&] {
    if (!out) fail(IXB_FAILURE, "ixb_comm_init: null output");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) fail(IXB_SHAPE, "ixb_comm_init: bad rank/world");
    auto c = new ixb_comm;
    c->world = world, c->rank = rank;
    IXB_CUDA_CHECK(cudaGetDevice(&c->device));
    IXB_CUDA_CHECK(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking));
    {  // a 1-rank communicator too: the same code path on a 1-GPU box
      nccl_unique_id u;
      std::memcpy(u.internal, id, sizeof u.internal);
      const nccl_result r = nccl().comm_init_rank(&c->comm, world, u, rank);
      if (r != 0) {
        cudaStreamDestroy(c->side);
        delete c;
        nccl_check(r, "ncclCommInitRank");
      }
    }
    *out = c;
  });
}

void ixb_comm_free(ixb_comm* c) {
  if (!c) return;
  cudaStreamSynchronize(c->side);
  if (c->comm) nccl().comm_destroy(c->comm);
  for (cudaEvent_t e : c->ev) cudaEventDestroy(e);
  cudaStreamDestroy(c->side);
  delete c;
}

int ixb_comm_broadcast(ixb_comm* c, void* buf, int64_t bytes, int root, ixb_stream stream) {
  return ixb_guard([&] {
    if (!c || root < 0 || root >= c->world || bytes < 0)
      fail(IXB_SHAPE, "ixb_comm_broadcast: bad communicator, root or size");
    if (bytes == 0) return;
    nccl_check(nccl().broadcast(buf, buf, static_cast<size_t>(bytes), kNcclInt8, root, c->comm,
                                reinterpret_cast<cudaStream_t>(stream)),
               "ncclBroadcast");
  });
}

int ixb_shard_plan_create(const int32_t* group_coord, int64_t G, int64_t rows, int world,
                          int rank, int nchunks, ixb_stream stream, ixb_shard_plan** out) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!out) fail(IXB_FAILURE, "ixb_shard_plan_create: null output");
    *out = nullptr;
    if (G < 0 || rows < 0 || world < 1 || rank < 0 || rank >= world || nchunks < 1)
      fail(IXB_SHAPE, "ixb_shard_plan_create: bad extents");
    std::vector<int32_t> gc(G);
    if (G) {
      IXB_CUDA_CHECK(cudaMemcpyAsync(gc.data(), group_coord, G * 4, cudaMemcpyDeviceToHost, s));
      IXB_CUDA_CHECK(cudaStreamSynchronize(s));
      for (int64_t p = 1; p < G; ++p)
        if (gc[p] < gc[p - 1]) fail(IXB_SHAPE, "ixb_shard_plan_create: groups not sorted by row");
      if (gc[0] < 0 || gc[G - 1] >= rows)
        fail(IXB_INDEX_RANGE, "ixb_shard_plan_create: group coordinate out of range");
    }
    auto holder = std::make_unique<ixb_shard_plan>();
    ixb_shard_plan* plan = holder.get();
    plan->world = world, plan->rank = rank, plan->nchunks = nchunks, plan->G = G;
    plan->rows = rows;
    std::vector<int64_t> shard(world + 1);
    cut_groups(gc.data(), 0, G, world, shard.data());
    // first output row of a group range: its first group's row (empty rows
    // before it belong to the range before); the tail belongs to the last
    auto row_at = [&](int64_t gpos) { return gpos < G ? static_cast<int64_t>(gc[gpos]) : rows; };
    plan->gb.assign(world, std::vector<int64_t>(nchunks + 1));
    plan->rb.assign(world, std::vector<int64_t>(nchunks + 1));
    for (int q = 0; q < world; ++q) {
      cut_groups(gc.data(), shard[q], shard[q + 1], nchunks, plan->gb[q].data());
      for (int c = 0; c <= nchunks; ++c) plan->rb[q][c] = row_at(plan->gb[q][c]);
      plan->rb[q][0] = q == 0 ? 0 : row_at(shard[q]);
      plan->rb[q][nchunks] = q + 1 == world ? rows : row_at(shard[q + 1]);
      for (int c = 1; c <= nchunks; ++c)  // monotone (a chunk may own no rows)
        if (plan->rb[q][c] < plan->rb[q][c - 1]) plan->rb[q][c] = plan->rb[q][c - 1];
      for (int c = nchunks - 1; c >= 0; --c)
        if (plan->rb[q][c] > plan->rb[q][c + 1]) plan->rb[q][c] = plan->rb[q][c + 1];
    }
    // own groups re-based to their chunk's first row: `=` then zero-fills
    // only inside the chunk's rows of the full output
    const auto& gb = plan->gb[rank];
    const auto& rb = plan->rb[rank];
    const int64_t n = gb[nchunks] - gb[0];
    std::vector<int32_t> loc(n);
    for (int c = 0; c < nchunks; ++c)
      for (int64_t p = gb[c]; p < gb[c + 1]; ++p)
        loc[p - gb[0]] = static_cast<int32_t>(gc[p] - rb[c]);
    IXB_CUDA_CHECK(cudaMalloc(&plan->am_local, (n + 1) * 4));
    if (n)
      IXB_CUDA_CHECK(cudaMemcpyAsync(plan->am_local, loc.data(), n * 4, cudaMemcpyHostToDevice, s));
    IXB_CUDA_CHECK(cudaStreamSynchronize(s));
    *out = holder.release();
  });
}

int ixb_shard_plan_chunk(const ixb_shard_plan* p, int rank, int chunk, int64_t* g0, int64_t* g1,
                         int64_t* r0, int64_t* r1) {
  return ixb_guard([&] {
    if (!p || rank < 0 || rank >= p->world || chunk < 0 || chunk >= p->nchunks)
      fail(IXB_SHAPE, "ixb_shard_plan_chunk: bad rank/chunk");
    *g0 = p->gb[rank][chunk], *g1 = p->gb[rank][chunk + 1];
    *r0 = p->rb[rank][chunk], *r1 = p->rb[rank][chunk + 1];
  });
}

void ixb_shard_plan_free(ixb_shard_plan* p) { delete p; }

}  // extern "C"

namespace {

// Chunked evaluate + overlapped in-place all-gather. eval(c, g0, g1, r0, r1)
// enqueues chunk c of this rank on `s`; row_bytes is one output row.
template <typename Eval>
void run_sharded(int world, int rank, int nchunks, const std::vector<std::vector<int64_t>>& rb,
                 char* out, int64_t row_bytes, int flags, ixb_comm* comm, cudaStream_t s,
                 Eval&& eval) {
  const bool compute = !(flags & IXB_SHARD_COMM_ONLY);
  const bool gather = comm && !(flags & IXB_SHARD_NO_COMM);
  if (world > 1 && !comm && !(flags & IXB_SHARD_NO_COMM))
    fail(IXB_FAILURE, "sharded evaluation: world > 1 needs a communicator");
  if (gather && (comm->world != world || comm->rank != rank))
    fail(IXB_FAILURE, "sharded evaluation: communicator does not match the plan's rank/world");
  if (gather) {
    while (comm->ev.size() < static_cast<size_t>(nchunks) + 1) {
      cudaEvent_t e;
      IXB_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      comm->ev.push_back(e);
    }
  }
  for (int c = 0; c < nchunks; ++c) {
    if (compute) eval(c);
    if (!gather) continue;
    IXB_CUDA_CHECK(cudaEventRecord(comm->ev[c], s));
    IXB_CUDA_CHECK(cudaStreamWaitEvent(comm->side, comm->ev[c], 0));
    Nccl& n = nccl();
    nccl_check(n.group_start(), "ncclGroupStart");
    for (int q = 0; q < world; ++q) {
      const int64_t a = rb[q][c], b = rb[q][c + 1];
      if (b <= a) continue;
      char* p = out + a * row_bytes;
      nccl_check(n.broadcast(p, p, static_cast<size_t>((b - a) * row_bytes), kNcclInt8, q,
                             comm->comm, comm->side),
                 "ncclBroadcast");
    }
    nccl_check(n.group_end(), "ncclGroupEnd");
  }
  if (gather) {
    IXB_CUDA_CHECK(cudaEventRecord(comm->ev[nchunks], comm->side));
    IXB_CUDA_CHECK(cudaStreamWaitEvent(s, comm->ev[nchunks], 0));  // full output on `s`
  }
}

}  // namespace

extern "C" {

int ixb_spmm_groupcoo_sharded(const ixb_shard_plan* p, const int32_t* AK, const float* AV,
                              int64_t g, const float* B, int64_t K, int64_t N, float* C,
                              int flags, ixb_comm* comm, ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!p) fail(IXB_FAILURE, "ixb_spmm_groupcoo_sharded: null plan");
    const auto& gb = p->gb[p->rank];
    const auto& rb = p->rb[p->rank];
    run_sharded(p->world, p->rank, p->nchunks, p->rb, reinterpret_cast<char*>(C), N * 4, flags,
                comm, s, [&](int c) {
                  const int64_t g0 = gb[c], g1 = gb[c + 1], r0 = rb[c], r1 = rb[c + 1];
                  if (r1 <= r0) return;
                  spmm_groupcoo(p->am_local + (g0 - gb[0]), AK + g0 * g, AV + g0 * g, g1 - g0, g,
                                B, K, N, C + r0 * N, r1 - r0, 0,
                                (flags & ~(IXB_SHARD_NO_COMM | IXB_SHARD_COMM_ONLY)) |
                                    IXB_GROUPS_SORTED,
                                s);
                });
  });
}

int ixb_spmm_blockgroupcoo_sharded(const ixb_shard_plan* p, const int32_t* AK, const void* AV,
                                   int64_t g, int64_t bm, int64_t bk, const void* B, int64_t KB,
                                   int64_t N, float* C, int flags, ixb_comm* comm,
                                   ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (!p) fail(IXB_FAILURE, "ixb_spmm_blockgroupcoo_sharded: null plan");
    const auto& gb = p->gb[p->rank];
    const auto& rb = p->rb[p->rank];
    const int64_t blk = bm * bk * 2;  // bytes of one bf16 block
    run_sharded(p->world, p->rank, p->nchunks, p->rb, reinterpret_cast<char*>(C), bm * N * 4,
                flags, comm, s, [&](int c) {
                  const int64_t g0 = gb[c], g1 = gb[c + 1], r0 = rb[c], r1 = rb[c + 1];
                  if (r1 <= r0) return;
                  spmm_blockgroupcoo(p->am_local + (g0 - gb[0]), AK + g0 * g,
                                     static_cast<const char*>(AV) + g0 * g * blk, g1 - g0, g, bm,
                                     bk, B, KB, N, C + r0 * bm * N, r1 - r0, 0,
                                     (flags & ~(IXB_SHARD_NO_COMM | IXB_SHARD_COMM_ONLY)) |
                                         IXB_GROUPS_SORTED,
                                     s);
                });
  });
}

int ixb_conv_plan_run_sharded(ixb_conv_plan* local, const void* In, int64_t Cin,
                              const void* Weight, int64_t Cout, float* Out, int64_t n_total,
                              int world, int rank, int nchunks, int flags, ixb_comm* comm,
                              ixb_stream stream) {
  return ixb_guard([&] {
    auto s = reinterpret_cast<cudaStream_t>(stream);
    if (world < 1 || rank < 0 || rank >= world || nchunks < 1 || n_total < 0)
      fail(IXB_SHAPE, "ixb_conv_plan_run_sharded: bad extents");
    // point blocks [n*q/world, n*(q+1)/world); chunks of whole 128-row tiles
    std::vector<std::vector<int64_t>> rb(world, std::vector<int64_t>(nchunks + 1));
    for (int q = 0; q < world; ++q) {
      const int64_t a = n_total * q / world, b = n_total * (q + 1) / world;
      const int64_t tiles = (b - a + 127) / 128;
      for (int c = 0; c <= nchunks; ++c) {
        const int64_t r = a + tiles * c / nchunks * 128;
        rb[q][c] = r < b ? r : b;
      }
    }
    const int64_t base = rb[rank][0];
    if (local && conv_plan_rows(local) != rb[rank][nchunks] - base)
      fail(IXB_SHAPE, "ixb_conv_plan_run_sharded: plan rows != this rank's point block");
    run_sharded(world, rank, nchunks, rb, reinterpret_cast<char*>(Out), Cout * 4, flags, comm, s,
                [&](int c) {
                  const int64_t r0 = rb[rank][c] - base, r1 = rb[rank][c + 1] - base;
                  if (r1 <= r0 || !local) return;
                  conv_plan_run_rows(local, In, Cin, Weight, Cout, Out + base * Cout, r0, r1, s);
                });
  });
}

}  // extern "C"
