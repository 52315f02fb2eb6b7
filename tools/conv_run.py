"""Runs K6 (grouped sparse conv) on the cfg5 shape through bench.py's workload
setup: `reps` timed calls (CUDA events) after 2 warm-ups. For ncu captures and
A/B timing of library builds (IXB_LIB_PATH). Perf experiment."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2510_17505_b200 as P  # noqa: E402
from paper_2510_17505_b200 import synth as S  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
wl = bench.WORKLOADS["cfg5"]()
dev = torch.device("cuda", 0)
wl.setup(torch, P, S, dev, wl.seed)
for _ in range(2):
    wl.step(P)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    wl.step(P)
b.record()
torch.cuda.synchronize()
print(f"{os.environ.get('IXB_LIB_PATH', 'libixb.so')}: {a.elapsed_time(b) / max(reps, 1):.4f} ms")
