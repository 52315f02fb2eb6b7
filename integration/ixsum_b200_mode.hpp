// "b200" execute_mode for the reference driver (see ixsum_b200_mode.cpp).
#pragma once

#include <string>

#include "ixsum/driver.hpp"

namespace ixsum::b200 {

/// Evaluates the problem's indirect Einsum on the B200 (libixb.so). Throws
/// std::invalid_argument for a statement outside the four hot-path workloads.
ModeResult execute(const BoundProblem& problem);

/// Relative tolerance (max_rel_error, tensor.cpp:124-136) of the device result
/// of `stmt` against the fp64 oracle: 1e-5 for the fp32 GroupCOO/COO SpMM,
/// 1e-2 for the bf16-operand evaluators; 0 (bit-exact) outside the hot path.
double device_tolerance(const EinsumStmt& stmt);

/// ixsum::execute_mode plus the "b200" mode.
ModeResult execute_mode(const std::string& mode, const BoundProblem& problem, int threads = 1,
                        const BlockSizeMap& block_sizes = {});

}  // namespace ixsum::b200
