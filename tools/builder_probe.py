"""Wall-time breakdown of the K1/K2 format builders at cfg1/cfg2 (plan call,
output allocation, pack call) against the device time of their kernels:
perf diagnosis, not a bench number. `python tools/builder_probe.py`"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_17505_b200 as P  # noqa: E402
from paper_2510_17505_b200 import synth as S  # noqa: E402

dev = torch.device("cuda", 0)
P.lib()
out = {}
for name in ("cfg2", "cfg1"):
    rng = S.Rng(1)
    if name == "cfg2":
        Ad = S.synth_block_sparse_matrix(rng, 8192, 8192, 16, 16, 0.10, S.REAL,
                                         torch.bfloat16).to(dev)
    else:
        Ad = S.synth_sparse_matrix(rng, 4096, 4096, 0.01, S.REAL, torch.float32).to(dev)
    fn = ((lambda: P.dense_to_blockgroupcoo(Ad, 16, 16, 0)) if name == "cfg2"
          else (lambda: P.dense_to_groupcoo(Ad, g=0)))
    for _ in range(3):
        fn()
    walls, devs = [], []
    for _ in range(30):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
        devs.append(a.elapsed_time(b))
    out[name] = {"wall_min": min(walls), "wall_med": statistics.median(walls),
                 "wall_best2": min(walls[:2]), "event_min": min(devs),
                 "event_med": statistics.median(devs)}
print(json.dumps(out))
# host floor: one tiny D2H read + sync (what each plan phase pays once)
x = torch.zeros(4, device=dev)
ts = []
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x.cpu()
    ts.append((time.perf_counter() - t0) * 1e3)
print(json.dumps({"d2h_sync_floor_ms": min(ts), "med": statistics.median(ts)}))
