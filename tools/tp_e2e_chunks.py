"""e2e time of the TP host-buffer pipeline vs chunk count (cfg4). Perf experiment."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import bench, paper_2510_17505_b200 as P
from paper_2510_17505_b200 import synth as S
wl = bench.WORKLOADS["cfg4"](); wl.setup(torch, P, S, torch.device("cuda", 0), 1)
for n in (4, 8, 16, 32):
    for _ in range(2): wl.plan.run_host(wl.h_in[0], wl.h_in[1], wl.W, wl.h_out, accumulate=False, nchunks=n)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3): wl.plan.run_host(wl.h_in[0], wl.h_in[1], wl.W, wl.h_out, accumulate=False, nchunks=n)
    b.record(); torch.cuda.synchronize()
    print("nchunks", n, round(a.elapsed_time(b) / 3, 2), "ms")
