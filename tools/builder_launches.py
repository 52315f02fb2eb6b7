"""Runs each device builder once at its BASELINE size (cfg1 K1, cfg2 K2, cfg5 K5 +
grouping) so `ncu --metrics gpu__time_duration.sum` can list its launches.
Perf tooling, not part of the library."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2510_17505_b200 as P  # noqa: E402
from paper_2510_17505_b200 import synth as S  # noqa: E402

dev = torch.device("cuda", 0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "k1"):
    rng = S.Rng(1)
    S.synth_dense(rng, (4096, 128), S.REAL, torch.float32)
    A = S.synth_sparse_matrix(rng, 4096, 4096, 0.01, S.REAL, torch.float32).to(dev)
    for _ in range(2):
        P.dense_to_groupcoo(A, g=0)
if which == "k1big":  # cfg3 d = 0.30: 16384^2 fp32
    rng = S.Rng(1)
    S.synth_dense(rng, (16384, 256), S.REAL, torch.float32)
    A = S.synth_sparse_matrix(rng, 16384, 16384, 0.30, S.REAL, torch.float32).to(dev)
    for _ in range(2):
        P.dense_to_groupcoo(A, g=0)
if which in ("all", "k2"):
    rng = S.Rng(1)
    S.synth_dense(rng, (512, 16, 512), S.REAL, torch.bfloat16)
    A = S.synth_block_sparse_matrix(rng, 8192, 8192, 16, 16, 0.10, S.REAL, torch.bfloat16).to(dev)
    for _ in range(2):
        P.dense_to_blockgroupcoo(A, 16, 16, 0)
if which in ("all", "k5"):
    coords = S.synth_voxel_shells(1_000_000).to(dev)
    n = coords.shape[0]
    for _ in range(2):
        mo, mi, mz = P.kernel_map(coords)
        g, _ = P.tune_group_size(mz, 27)
        ones = torch.ones(mo.numel(), dtype=torch.float32, device=dev)
        P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, g, canonical=True)
torch.cuda.synchronize()
