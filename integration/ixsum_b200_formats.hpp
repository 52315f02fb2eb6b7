// Drop-in format builders for the reference toolkit: the reference's C++
// signatures and structs (/root/reference/proj/include/ixsum/formats.hpp),
// computed by the device builders of libixb.so (include/ixb.h, K1/K2/K5
// grouping engines) and returned as the reference's host structs. Results
// are bit-identical to the reference's (b200_mode_check --builders and the
// corpus specs check every one), errors are the reference's exception types
// and messages.
#pragma once

#include <cstdint>

#include "ixsum/driver.hpp"
#include "ixsum/formats.hpp"
#include "ixsum/tuner.hpp"

namespace ixsum::b200 {

/// dense_to_coo (formats.hpp:26, formats.cpp:24-46).
CooMatrix dense_to_coo(const Tensor& t);
/// canonicalize (formats.hpp:28, formats.cpp:68-89): the g = 1 grouping.
CooMatrix canonicalize(const CooMatrix& c);
/// coo_to_groupcoo (formats.hpp:53, formats.cpp:115-174).
GroupCooMatrix coo_to_groupcoo(const CooMatrix& c, int group_dim, int64_t g);
/// dense_to_blockgroupcoo (formats.hpp:81-83, formats.cpp:224-292).
BlockGroupCooMatrix dense_to_blockgroupcoo(const Tensor& t, int64_t block_rows,
                                           int64_t block_cols, int64_t g, int group_dim = 0);
/// GroupCooMatrix::real_count / pad_count (formats.hpp:49-50, formats.cpp:105-113).
int64_t real_count(const GroupCooMatrix& gc);
int64_t pad_count(const GroupCooMatrix& gc);
/// groupcoo_to_coo (formats.hpp:54, formats.cpp:176-194): real slots, canonicalized.
CooMatrix groupcoo_to_coo(const GroupCooMatrix& gc);
/// ell_view (formats.hpp:57, formats.cpp:196-200): g = max occupancy along group_dim.
GroupCooMatrix ell_view(const CooMatrix& c, int group_dim = 0);
/// is_ell (formats.hpp:58, formats.cpp:202-208).
bool is_ell(const GroupCooMatrix& gc);
/// group_coo_tensor (formats.hpp:141, formats.cpp:417-479).
GroupCooTensor group_coo_tensor(const CooTensor& c, int group_dim, int64_t g);
/// select() over the occupancy of c along `dim` (tuner.hpp:63, tuner.cpp:100-118,
/// OccProfile::from_coo), with brute_optimal, on the device.
TuneReport tune(const CooMatrix& c, int dim, bool count_empty_rows = false);

/// materialize (driver.hpp:89, driver.cpp:165-233) with every format
/// directive built on the device: the same synth streams and call order, the
/// same operand names, bytes and tuner reports as the reference's.
BoundProblem materialize(const RunConfig& cfg);

}  // namespace ixsum::b200
