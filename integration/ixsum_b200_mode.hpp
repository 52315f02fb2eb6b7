// "b200" execute_mode for the reference driver (see ixsum_b200_mode.cpp).
#pragma once

#include <string>

#include "ixsum/driver.hpp"

namespace ixsum::b200 {

/// Evaluates the problem's indirect Einsum on the B200 (libixb.so).
ModeResult execute(const BoundProblem& problem);

/// ixsum::execute_mode plus the "b200" mode.
ModeResult execute_mode(const std::string& mode, const BoundProblem& problem, int threads = 1,
                        const BlockSizeMap& block_sizes = {});

}  // namespace ixsum::b200
