"""Runs the K7 tensor-core kernel on the cfg4 shape (1M edges, l_max 3 CG,
64 channels, shared W) with torch-random bf16 inputs: `reps` timed calls
(CUDA events) after 2 warm-ups. For ncu captures and A/B timing of library
builds (IXB_LIB_PATH). Perf experiment, not a bench number."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_17505_b200 as P  # noqa: E402
from paper_2510_17505_b200 import synth as S  # noqa: E402

B = int(os.environ.get("TP_B", 1_000_000))
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn((B, 16, 64), device="cuda", generator=g).to(torch.bfloat16)
Y = torch.randn((B, 16), device="cuda", generator=g).to(torch.bfloat16)
cg = S.cg_table(3)
nl = cg["npaths"]
W = (torch.randn((nl, 64, 64), device="cuda", generator=g) / 8).to(torch.bfloat16)
gt = P.group_coo_tensor([16, 16, 16, nl], [cg[k].cuda() for k in ("i", "j", "k", "l")],
                        cg["v"].cuda(), 3, 4)
plan = P.TpPlan(gt.group_coord, *gt.member_coords, gt.values, 16, 16, 16, nl)
Z = torch.empty((B, 16, 64), device="cuda")
for _ in range(2):
    plan.run(X, Y, W, Z, accumulate=False)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    plan.run(X, Y, W, Z, accumulate=False)
b.record()
torch.cuda.synchronize()
print(f"{os.environ.get('IXB_LIB_PATH', 'libixb.so')}: {a.elapsed_time(b) / max(reps, 1):.3f} ms")
if os.environ.get("TP_TRACE_DUMP"):  # -DIXB_TP_TRACE build: CTA 0 timeline of the last call
    import ctypes

    import numpy as np
    buf = np.zeros(4 * 4 * 512, np.int64)
    P.lib().ixb_tp_trace_copy(ctypes.c_void_p(buf.ctypes.data))
    np.save(os.environ["TP_TRACE_DUMP"], buf)
