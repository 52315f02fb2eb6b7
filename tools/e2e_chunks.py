"""e2e (host buffers in, host C out) time of the cfg1/cfg2 SpMM host entry
points against the pipeline's chunk count: perf experiment, not a bench
number. `python tools/e2e_chunks.py`"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2510_17505_b200 as P  # noqa: E402
from paper_2510_17505_b200 import synth as S  # noqa: E402

dev = torch.device("cuda", 0)
P.lib()
out = {}
for name in ("cfg2", "cfg1"):
    wl = bench.WORKLOADS[name]()
    wl.setup(torch, P, S, dev, wl.seed)
    AM, AK, AV, B = wl.h_in
    fn = P.spmm_blockgroupcoo_host if name == "cfg2" else P.spmm_groupcoo_host
    res = {}
    for nch in (0, 1, 2, 4, 8):
        for chk in (True, False):
            def step():
                fn(AM, AK, AV, B, wl.h_out, accumulate=False, nchunks=nch,
                   **({} if chk else {"flags": 2}))
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            ts = []
            for _ in range(10):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                step()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            res[f"n{nch}{'' if chk else '_unchecked'}"] = round(min(ts), 4)
    out[name] = res
print(json.dumps(out))
