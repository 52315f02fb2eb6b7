import sys, torch
sys.path.insert(0, '.')
import bench, paper_2510_17505_b200 as P
from paper_2510_17505_b200 import synth as S
wl = bench.WORKLOADS["cfg2"]()
wl.setup(torch, P, S, torch.device("cuda", 0), 1)
AM, AK, AV, B = wl.h_in
for nch in (1, 2, 4, 8, 16):
    for _ in range(3):
        P.spmm_blockgroupcoo_host(AM, AK, AV, B, wl.h_out, accumulate=False, nchunks=nch)
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); P.spmm_blockgroupcoo_host(AM, AK, AV, B, wl.h_out, accumulate=False, nchunks=nch); b.record()
        torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    print("nchunks", nch, "e2e ms", round(sorted(ts)[5], 3))
# serial reference: H2D all, kernel, D2H
d = [x.cuda() for x in wl.h_in]
ts = []
for _ in range(10):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for dd, h in zip(d, wl.h_in): dd.copy_(h, non_blocking=True)
    P.spmm_blockgroupcoo(d[0], d[1], d[2], d[3], wl.C, accumulate=False, flags=3)
    wl.h_out.copy_(wl.C, non_blocking=True)
    b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print("serial e2e ms", round(sorted(ts)[5], 3))
# raw copy bandwidths
x = torch.empty(64 << 20, dtype=torch.uint8).pin_memory(); y = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
for name, f in (("h2d", lambda: y.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(y, non_blocking=True))):
    f(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize()
    print(name, "GB/s", round(64 * 2**20 / a.elapsed_time(b) / 1e6, 1))
# concurrent H2D + D2H on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
x2 = torch.empty(64 << 20, dtype=torch.uint8).pin_memory(); y2 = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
with torch.cuda.stream(s1): y.copy_(x, non_blocking=True)
with torch.cuda.stream(s2): x2.copy_(y2, non_blocking=True)
e1 = s1.record_event(); e2 = s2.record_event()
torch.cuda.current_stream().wait_event(e1); torch.cuda.current_stream().wait_event(e2)
b.record(); torch.cuda.synchronize()
print("concurrent h2d+d2h: total GB/s", round(2 * 64 * 2**20 / a.elapsed_time(b) / 1e6, 1), "ms", round(a.elapsed_time(b), 3))
