// K4 panel form (spmm_bgcoo_panel.cu): plan + run entry points shared with the
// BlockGroupCOO SpMM front end (spmm_bgcoo_tc.cu) and the C-ABI plan object.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ixb_internal.h"

namespace ixb {

// Plan of the panel kernel for one BlockGroupCOO structure (AM, AK): block
// row starts and the per-panel (kb, slot)-sorted op list. Depends on the
// index arrays only; AV and B are read at run time.
struct BgPanelPlan {
  int64_t G = 0, g = 1, KB = 0, MB = 0, nslots = 0;
  int R = 8;
  int variant = 0;  // kernel shape the stage records were packed for
  Scratch<int32_t> rowptr;   // [MB + 1]: first (sorted) group of each block row
  Scratch<int32_t> rec;      // stage records (16 ints each), per panel from rowptr[P*R]*g + P
  Scratch<int32_t> nstages;  // [npanels]
};

// Whether the tensor-core panel kernel takes this shape (16 x 16 blocks,
// N a multiple of 128, 16-byte aligned operands).
bool bgcoo_panel_ok(int64_t bm, int64_t bk, int64_t N, const void* AV, const void* B);
// Builds the plan on `s` without a host sync. AM must be non-decreasing; `perm`
// (optional) maps sorted group positions to the caller's, so the ops address
// the caller's AV directly; AK is then the sorted copy. With `check`, AK/AM
// range errors go to the device error record (reference order).
void bgcoo_panel_plan(const int32_t* AM, const int32_t* AK, const int32_t* perm, int64_t G,
                      int64_t g, int64_t KB, int64_t MB, bool check, cudaStream_t s,
                      BgPanelPlan& P);
void bgcoo_panel_run(const BgPanelPlan& P, const void* AV, const void* B, int64_t N, float* C,
                     int accumulate, cudaStream_t s);

}  // namespace ixb
