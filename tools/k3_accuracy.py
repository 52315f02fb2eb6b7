"""Max relative error of K3 (fp32) against the fp64 oracle on long rows
(~1200 and ~4900 terms per row). Accuracy experiment for compensated
accumulation; load another build with IXB_LIB_PATH."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_17505_b200 as P  # noqa: E402
from oracle import ixo  # noqa: E402

for M, K, d in ((40, 1500, 0.8), (24, 16384, 0.3)):
    rng = ixo.Rng(23)
    a = ixo.synth_sparse_matrix(rng, M, K, d)
    b = ixo.synth_dense(rng, (K, 256))
    a32, b32 = a.astype(np.float32), b.astype(np.float32)
    fmt = P.dense_to_groupcoo(torch.from_numpy(a32).cuda(), g=0)
    C = torch.zeros((M, 256), device="cuda")
    P.spmm_groupcoo(fmt.AM, fmt.AK, fmt.AV, torch.from_numpy(b32).cuda(), C)
    want = a32.astype(np.float64) @ b32.astype(np.float64)
    print(f"{os.environ.get('TAG', 'main')}: {int(d * K)} terms/row: max_rel_error "
          f"{ixo.max_rel_error(want, C.double().cpu().numpy()):.2e}")
