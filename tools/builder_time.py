"""Wall time of the device builder API calls at their BASELINE sizes (cfg1 K1,
cfg2 K2, cfg5 K5 + grouping), warm, best and median of --reps. Perf tooling,
not part of the library: `python tools/builder_time.py [--reps 10]`."""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
dev = torch.device("cuda", 0)


def wall(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e6)
    return {"best_us": min(ts), "median_us": statistics.median(ts)}


rng = S.Rng(1)
S.synth_dense(rng, (4096, 128), S.REAL, torch.float32)
A1 = S.synth_sparse_matrix(rng, 4096, 4096, 0.01, S.REAL, torch.float32).to(dev)
rng = S.Rng(1)
S.synth_dense(rng, (512, 16, 512), S.REAL, torch.bfloat16)
A2 = S.synth_block_sparse_matrix(rng, 8192, 8192, 16, 16, 0.10, S.REAL, torch.bfloat16).to(dev)
out = {"k1_cfg1": wall(lambda: P.dense_to_groupcoo(A1, g=0)),
       "k2_cfg2": wall(lambda: P.dense_to_blockgroupcoo(A2, 16, 16, 0))}
print(json.dumps(out))
