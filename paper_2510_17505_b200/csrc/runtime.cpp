// Host runtime of the C-ABI: error state, per-device error records, scratch
// pool, launch accounting and the multi-GPU shard planner.
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "ixb_internal.h"

namespace {

thread_local std::string t_msg;
thread_local int t_idx_operand = -1;
thread_local int64_t t_idx_pos = 0, t_idx_value = 0, t_idx_extent = 0;
std::atomic<int64_t> g_launches{0};

struct DeviceCtx {
  ixb::ErrorRecord* rec = nullptr;
  int sms = 0;
  std::vector<std::pair<const void*, int>> smem_optin;  // (kernel, bytes) opted in
  // self-resetting work counters of the persistent kernels, one pair per
  // stream (kernels on different streams must not share a counter)
  unsigned* counters = nullptr;
  std::vector<cudaStream_t> counter_streams;
  // per (counter slot, tag): persistent scratch
  std::vector<std::vector<std::pair<void*, size_t>>> stream_bufs;
};
constexpr int kCounterSlots = 64;
constexpr size_t kCountersPerSlot = 65536;
std::mutex g_mu;
std::vector<DeviceCtx> g_dev;

DeviceCtx& ctx() {
  int d = 0;
  ixb::cuda_check(cudaGetDevice(&d), "cudaGetDevice");
  std::lock_guard<std::mutex> lk(g_mu);
  if (static_cast<int>(g_dev.size()) <= d) g_dev.resize(static_cast<size_t>(d) + 1);
  DeviceCtx& c = g_dev[static_cast<size_t>(d)];
  if (!c.rec) {
    ixb::cuda_check(cudaMalloc(&c.rec, sizeof(ixb::ErrorRecord)), "cudaMalloc(error record)");
    ixb::cuda_check(cudaMemset(c.rec, 0xff, sizeof(ixb::ErrorRecord)), "cudaMemset");
    ixb::cuda_check(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, d),
                    "cudaDeviceGetAttribute");
  }
  return c;
}

}  // namespace

namespace ixb {

void fail(int code, const std::string& msg) { throw Error(code, msg); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(IXB_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
}

void note_launch(int n) { g_launches += n; }

int sm_count() { return ctx().sms; }

void set_max_dynamic_smem(const void* func, int bytes, const char* name) {
  DeviceCtx& c = ctx();
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (const auto& e : c.smem_optin)
      if (e.first == func && e.second >= bytes) return;
  }
  cuda_check(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), name);
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& e : c.smem_optin)
    if (e.first == func) {
      if (bytes > e.second) e.second = bytes;
      return;
    }
  c.smem_optin.emplace_back(func, bytes);
}

ErrorRecord* device_error_record() { return ctx().rec; }

unsigned* work_counters(cudaStream_t stream, size_t n) {
  if (n > kCountersPerSlot) fail(IXB_FAILURE, "work_counters: too many counters");
  DeviceCtx& c = ctx();
  std::lock_guard<std::mutex> lk(g_mu);
  if (!c.counters) {
    const size_t bytes = kCounterSlots * kCountersPerSlot * sizeof(unsigned);
    cuda_check(cudaMalloc(&c.counters, bytes), "cudaMalloc(counters)");
    cuda_check(cudaMemset(c.counters, 0, bytes), "cudaMemset");
  }
  size_t i = 0;
  while (i < c.counter_streams.size() && c.counter_streams[i] != stream) ++i;
  if (i == c.counter_streams.size()) {
    if (i == kCounterSlots) fail(IXB_FAILURE, "work_counter: more than 64 streams on one device");
    c.counter_streams.push_back(stream);
  }
  return c.counters + kCountersPerSlot * i;
}

void* stream_buffer(cudaStream_t stream, size_t bytes, int tag) {
  work_counters(stream, 0);  // assigns the stream its slot
  DeviceCtx& c = ctx();
  std::lock_guard<std::mutex> lk(g_mu);
  size_t i = 0;
  while (c.counter_streams[i] != stream) ++i;
  if (c.stream_bufs.size() <= i) c.stream_bufs.resize(i + 1);
  if (c.stream_bufs[i].size() <= static_cast<size_t>(tag))
    c.stream_bufs[i].resize(static_cast<size_t>(tag) + 1, {nullptr, 0});
  auto& b = c.stream_bufs[i][static_cast<size_t>(tag)];
  if (b.second < bytes) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(stream, &cs), "cudaStreamIsCapturing");
    if (cs != cudaStreamCaptureStatusNone) return nullptr;  // caller allocates in the graph
    if (b.first) {
      // a kernel still reading the old buffer must finish before it goes
      cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
      cuda_check(cudaFree(b.first), "cudaFree(stream buffer)");
    }
    cuda_check(cudaMalloc(&b.first, bytes), "cudaMalloc(stream buffer)");
    b.second = bytes;
  }
  return b.first;
}

namespace {
constexpr size_t kPinnedBytes = 4096;
thread_local char* t_pinned = nullptr;
char* pinned_staging() {
  if (!t_pinned) {
    void* p = nullptr;
    cuda_check(cudaMallocHost(&p, kPinnedBytes), "cudaMallocHost(staging)");
    t_pinned = static_cast<char*>(p);
  }
  return t_pinned;
}
}  // namespace

void HostReads::add(void* dst, const void* src, size_t bytes) {
  const size_t off = (used_ + 15) & ~size_t(15);
  if (off + bytes > kPinnedBytes || n_ == 16) {
    IXB_CUDA_CHECK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s_));
    return;
  }
  IXB_CUDA_CHECK(cudaMemcpyAsync(pinned_staging() + off, src, bytes, cudaMemcpyDeviceToHost, s_));
  items_[n_++] = {dst, off, bytes};
  used_ = off + bytes;
}

void HostReads::wait() {
  IXB_CUDA_CHECK(cudaStreamSynchronize(s_));
  for (int i = 0; i < n_; ++i) std::memcpy(items_[i].dst, t_pinned + items_[i].off, items_[i].bytes);
  n_ = 0;
  used_ = 0;
}

void reset_error_record(cudaStream_t stream) {
  IXB_CUDA_CHECK(cudaMemsetAsync(&ctx().rec->key, 0xff, sizeof(unsigned long long), stream));
}

void check_error_record(cudaStream_t stream, const OperandInfo* ops, int nops) {
  unsigned long long key = kNoError;
  HostReads rd(stream);
  rd.add(&key, &ctx().rec->key, sizeof key);
  rd.wait();
  if (key == kNoError) return;
  int op = static_cast<int>(key >> 56);
  int64_t pos = static_cast<int64_t>(key & ((1ull << 56) - 1));
  reset_error_record(stream);
  if (op >= nops || !ops) fail(IXB_INDEX_RANGE, "index out of range");
  const OperandInfo& o = ops[op];
  int32_t v = 0;
  if (o.device_array && pos < o.numel) {
    IXB_CUDA_CHECK(cudaMemcpy(&v, o.device_array + pos, sizeof v, cudaMemcpyDeviceToHost));
  }
  t_idx_operand = op;
  t_idx_pos = pos;
  t_idx_value = v;
  t_idx_extent = o.extent;
  // Message content of checked_index (plan.cpp:253-256).
  fail(IXB_INDEX_RANGE, "index tensor " + std::string(o.index_name) + " value " +
                            std::to_string(v) + " at position [" + std::to_string(pos) +
                            "] out of range for dim " + std::to_string(o.target_dim) + " of " +
                            o.target_name + " (extent " + std::to_string(o.extent) + ")");
}

// Stream-ordered scratch from the device's default memory pool. The pool
// keeps freed memory mapped (release threshold = max) so repeated calls do
// not unmap and remap their temporaries at every synchronisation.
void* scratch_alloc(size_t bytes, cudaStream_t stream) {
  static thread_local int configured = -1;
  int dev = 0;
  IXB_CUDA_CHECK(cudaGetDevice(&dev));
  if (configured != dev) {
    cudaMemPool_t pool;
    IXB_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = ~0ull;
    IXB_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured = dev;
  }
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  IXB_CUDA_CHECK(cudaMallocAsync(&p, bytes, stream));
  return p;
}

void scratch_free(void* p, cudaStream_t stream) {
  if (p) cudaFreeAsync(p, stream);
}

}  // namespace ixb

int ixb_guard_set(int code, const char* msg) {
  if (code != IXB_OK) {
    t_msg = msg;
  }
  return code;
}

extern "C" {

const char* ixb_last_error(void) { return t_msg.c_str(); }

int ixb_version(void) { return 1; }

int ixb_last_index_error(int* operand, int64_t* position, int64_t* value, int64_t* extent) {
  if (operand) *operand = t_idx_operand;
  if (position) *position = t_idx_pos;
  if (value) *value = t_idx_value;
  if (extent) *extent = t_idx_extent;
  return t_idx_operand >= 0 ? IXB_INDEX_RANGE : IXB_OK;
}

int ixb_check_errors(ixb_stream stream) {
  return ixb_guard([&] { ixb::check_error_record(stream, nullptr, 0); });
}

int ixb_sm_count(void) {
  int n = 0;
  ixb_guard([&] { n = ixb::sm_count(); });
  return n;
}

int64_t ixb_launch_count(void) { return g_launches.load(); }

// Shard planner: contiguous group ranges with ~equal slots,
// cut only at group-coordinate changes so no output row spans two ranks.
int ixb_shard_groups(const int32_t* gc, int64_t G, int parts, int64_t* bounds) {
  return ixb_guard([&] {
    if (parts < 1) ixb::fail(IXB_FAILURE, "ixb_shard_groups: parts must be >= 1");
    bounds[0] = 0;
    for (int r = 1; r < parts; ++r) {
      int64_t target = (G * r) / parts;
      int64_t cut = target;
      if (cut < bounds[r - 1]) cut = bounds[r - 1];
      // advance to the next row boundary (never split a row's groups)
      while (cut > 0 && cut < G && gc[cut] == gc[cut - 1]) ++cut;
      bounds[r] = cut;
    }
    bounds[parts] = G;
  });
}

}  // extern "C"
