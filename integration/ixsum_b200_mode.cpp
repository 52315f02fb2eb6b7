// Drop-in "b200" mode for the reference driver (ixsum::execute_mode,
// /root/reference/proj/src/driver.cpp:235-265), built against the
// reference's own headers (proj/include/ixsum) and the C-ABI (include/ixb.h).
//
// A maintainer adds one branch to execute_mode:
//     } else if (mode == "b200") { return ixsum::b200::execute(problem); }
// This file is that branch's implementation: it matches the inferred
// EinsumStmt to one of the hot-path workloads, moves the BoundProblem's
// Tensors to the device in the device formats (int32 indices; fp32 for the
// GroupCOO SpMM, bf16 operands with fp32 accumulation elsewhere), calls the
// sm_100a evaluator and returns a ModeResult with the analytic access
// counters (count_accesses_model, plan.cpp:607-631). Errors come back as the
// reference's exception types with the reference's message content.
#include "ixsum_b200_mode.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "ixb.h"

namespace ixsum::b200 {
namespace {

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) throw std::runtime_error("cudaMalloc");
  }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

void rethrow(int code, const EinsumStmt& stmt) {
  (void)stmt;
  const std::string msg = ixb_last_error();
  switch (code) {
    case IXB_OK: return;
    case IXB_PARSE: throw ParseError(msg, 0);
    case IXB_BIND: throw BindError(msg);
    case IXB_SHAPE: throw ShapeError(msg);
    case IXB_INDEX_RANGE: throw IndexRangeError(msg);
    default: throw std::runtime_error(msg);
  }
}

std::unique_ptr<DevBuf> up_index(const Tensor& t) {
  std::vector<int32_t> h(static_cast<size_t>(t.numel()));
  for (int64_t i = 0; i < t.numel(); ++i) h[i] = static_cast<int32_t>(t.int_at(i));
  auto d = std::make_unique<DevBuf>(h.size() * 4);
  cudaMemcpy(d->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  return d;
}

std::unique_ptr<DevBuf> up_f32(const Tensor& t) {
  std::vector<float> h(static_cast<size_t>(t.numel()));
  for (int64_t i = 0; i < t.numel(); ++i) h[i] = static_cast<float>(t.as_real(i));
  auto d = std::make_unique<DevBuf>(h.size() * 4);
  cudaMemcpy(d->p, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  return d;
}

std::unique_ptr<DevBuf> up_bf16(const Tensor& t) {
  std::vector<__nv_bfloat16> h(static_cast<size_t>(t.numel()));
  for (int64_t i = 0; i < t.numel(); ++i) h[i] = __float2bfloat16_rn(static_cast<float>(t.as_real(i)));
  auto d = std::make_unique<DevBuf>(h.size() * 2);
  cudaMemcpy(d->p, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  return d;
}

Tensor down(const DevBuf& d, const Tensor& like) {
  std::vector<float> h(static_cast<size_t>(like.numel()));
  cudaMemcpy(h.data(), d.p, h.size() * 4, cudaMemcpyDeviceToHost);
  Tensor out = Tensor::zeros(like.kind(), like.shape());
  for (int64_t i = 0; i < like.numel(); ++i) {
    if (out.is_int()) out.int_at(i) = std::llround(h[i]);
    else out.real_at(i) = h[i];
  }
  return out;
}

const std::string& dvar(const IndexExpr& e) { return std::get<DirectIndex>(e).var; }
bool direct(const IndexExpr& e) { return std::holds_alternative<DirectIndex>(e); }
const IndirectIndex& ind(const IndexExpr& e) { return std::get<IndirectIndex>(e); }

}  // namespace

ModeResult execute(const BoundProblem& problem) {
  const auto t0 = std::chrono::steady_clock::now();
  const EinsumStmt& st = problem.stmt;
  const auto& T = problem.tensors;
  const Tensor& out = problem.out;
  const int acc = st.accumulate ? 1 : 0;
  ModeResult mo;
  mo.kernel_count = 1;
  const auto& o = st.output;
  const auto& in = st.inputs;
  // -- GroupCOO / COO SpMM: C[AM[p..],n] (+)= AV[p..] * B[AK[p..],n]
  if (in.size() == 2 && o.indices.size() == 2 && !direct(o.indices[0]) && direct(o.indices[1]) &&
      in[1].indices.size() == 2 && !direct(in[1].indices[0])) {
    const Tensor& AM = T.at(ind(o.indices[0]).tensor);
    const Tensor& AK = T.at(ind(in[1].indices[0]).tensor);
    const Tensor& AV = T.at(in[0].tensor);
    const Tensor& B = T.at(in[1].tensor);
    const int64_t G = AM.numel(), g = G ? AV.numel() / G : 1;
    auto dAM = up_index(AM), dAK = up_index(AK);
    auto dAV = up_f32(AV), dB = up_f32(B), dC = up_f32(out);
    rethrow(ixb_spmm_groupcoo(static_cast<int32_t*>(dAM->p), static_cast<int32_t*>(dAK->p),
                              static_cast<float*>(dAV->p), G, g, static_cast<float*>(dB->p),
                              B.dim(0), B.dim(1), static_cast<float*>(dC->p), out.dim(0), acc, 0,
                              nullptr),
            st);
    mo.result = down(*dC, out);
    mo.counters = {G * g, G, G * B.dim(1)};
  } else if (in.size() == 2 && o.indices.size() == 3 && !direct(o.indices[0])) {
    // -- BlockGroupCOO SpMM: C[AM[p],bm,n] (+)= AV[p,q,bm,bk] * B[AK[p,q],bk,n]
    const Tensor& AM = T.at(ind(o.indices[0]).tensor);
    const Tensor& AK = T.at(ind(in[1].indices[0]).tensor);
    const Tensor& AV = T.at(in[0].tensor);
    const Tensor& B = T.at(in[1].tensor);
    auto dAM = up_index(AM), dAK = up_index(AK), dAV = up_bf16(AV), dB = up_bf16(B);
    auto dC = up_f32(out);
    rethrow(ixb_spmm_blockgroupcoo(static_cast<int32_t*>(dAM->p), static_cast<int32_t*>(dAK->p),
                                   dAV->p, AV.dim(0), AV.dim(1), AV.dim(2), AV.dim(3), dB->p,
                                   B.dim(0), B.dim(2), static_cast<float*>(dC->p), out.dim(0),
                                   acc, 0, nullptr),
            st);
    mo.result = down(*dC, out);
    mo.counters = {AV.dim(0) * AV.dim(1), AV.dim(0), AV.dim(0) * AV.dim(2) * B.dim(2)};
  } else if (in.size() == 3 && o.indices.size() == 2 && !direct(o.indices[0])) {
    // -- (grouped) sparse conv: Out[MAPX[..],m] += MAPV[..] * In[MAPY[..],c] * W[MAPZ[p],c,m]
    const Tensor& MX = T.at(ind(o.indices[0]).tensor);
    const Tensor& MV = T.at(in[0].tensor);
    const Tensor& In = T.at(in[1].tensor);
    const Tensor& MY = T.at(ind(in[1].indices[0]).tensor);
    const Tensor& W = T.at(in[2].tensor);
    const Tensor& MZ = T.at(ind(in[2].indices[0]).tensor);
    const int64_t G = MZ.numel(), g = G ? MX.numel() / G : 1;
    auto dMX = up_index(MX), dMY = up_index(MY), dMZ = up_index(MZ), dMV = up_f32(MV);
    auto dIn = up_bf16(In), dW = up_bf16(W), dO = up_f32(out);
    rethrow(ixb_conv_grouped(static_cast<int32_t*>(dMZ->p), static_cast<int32_t*>(dMX->p),
                             static_cast<int32_t*>(dMY->p), static_cast<float*>(dMV->p), G, g,
                             dIn->p, In.dim(0), In.dim(1), dW->p, W.dim(0), W.dim(2),
                             static_cast<float*>(dO->p), out.dim(0), acc, 0, nullptr),
            st);
    mo.result = down(*dO, out);
    mo.counters = {G * g, G, G * W.dim(2)};
  } else if (in.size() == 4 && o.indices.size() == 3 && direct(o.indices[0])) {
    // -- CG tensor product: Z[b,CGI[p,q],w] += CGV * X[b,CGJ,u] * Y[b,CGK] * W[(b,)CGL[p],u,w]
    const Tensor& CI = T.at(ind(o.indices[1]).tensor);
    const Tensor& CV = T.at(in[0].tensor);
    const Tensor& X = T.at(in[1].tensor);
    const Tensor& CJ = T.at(ind(in[1].indices[1]).tensor);
    const Tensor& Y = T.at(in[2].tensor);
    const Tensor& CK = T.at(ind(in[2].indices[1]).tensor);
    const Tensor& W = T.at(in[3].tensor);
    const bool per_b = W.rank() == 4;
    const Tensor& CL = T.at(ind(in[3].indices[per_b ? 1 : 0]).tensor);
    const int64_t G = CL.numel(), g = G ? CI.numel() / G : 1;
    auto dL = up_index(CL), dI = up_index(CI), dJ = up_index(CJ), dK = up_index(CK);
    auto dV = up_f32(CV), dX = up_bf16(X), dY = up_bf16(Y), dW = up_bf16(W), dZ = up_f32(out);
    rethrow(ixb_tp_grouped(static_cast<int32_t*>(dL->p), static_cast<int32_t*>(dI->p),
                           static_cast<int32_t*>(dJ->p), static_cast<int32_t*>(dK->p),
                           static_cast<float*>(dV->p), G, g, dX->p, dY->p, dW->p, per_b ? 1 : 0,
                           X.dim(0), out.dim(1), X.dim(1), Y.dim(1), W.dim(per_b ? 1 : 0),
                           X.dim(2), W.dim(per_b ? 3 : 2), static_cast<float*>(dZ->p), acc, 0,
                           nullptr),
            st);
    mo.result = down(*dZ, out);
    mo.counters = {G * g, G, G * X.dim(0) * W.dim(per_b ? 3 : 2)};
  } else {
    throw std::invalid_argument("b200 mode: statement outside the hot path: " + to_string(st));
  }
  mo.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                   .count();
  return mo;
}

ModeResult execute_mode(const std::string& mode, const BoundProblem& problem, int threads,
                        const BlockSizeMap& block_sizes) {
  if (mode == "b200") return execute(problem);
  return ixsum::execute_mode(mode, problem, threads, block_sizes);
}

}  // namespace ixsum::b200
