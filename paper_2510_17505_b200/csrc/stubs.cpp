// Entry points whose kernels land in later milestones; they fail loudly.
#include "ixb_internal.h"

extern "C" {

int ixb_tp_grouped(const int32_t*, const int32_t*, const int32_t*, const int32_t*, const float*,
                   int64_t, int64_t, const void*, const void*, const void*, int, int64_t, int64_t,
                   int64_t, int64_t, int64_t, int64_t, int64_t, float*, int, int, ixb_stream) {
  return ixb_guard([] { ixb::fail(IXB_FAILURE, "ixb_tp_grouped: not built yet"); });
}

}  // extern "C"
