"""Is a small workload's bench step inflated by host launch latency? Times
cfg1's K3 step (a) as bench.py does (events around each launch after an L2
flush), (b) with the step captured in a CUDA graph and replayed after the
same flush, (c) 200 launches back to back (L2 warm). Perf experiment."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2510_17505_b200 as P  # noqa: E402
from paper_2510_17505_b200 import synth as S  # noqa: E402

wl = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]()
dev = torch.device("cuda", 0)
wl.setup(torch, P, S, dev, wl.seed)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
s = torch.cuda.current_stream()
for _ in range(5):
    wl.step(P)
torch.cuda.synchronize()


def timed(fn, n=50):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n)]
    for a, b in evs:
        flush.zero_()
        a.record(s)
        fn()
        b.record(s)
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in evs) / n * 1e3


print("per-step events (bench style): %.2f us" % timed(lambda: wl.step(P)))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    wl.step(P)
g.replay()
torch.cuda.synchronize()
print("graph replay after flush:      %.2f us" % timed(g.replay))
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(200):
    wl.step(P)
b.record(s)
torch.cuda.synchronize()
print("back-to-back (L2 warm):        %.2f us" % (a.elapsed_time(b) / 200 * 1e3))
