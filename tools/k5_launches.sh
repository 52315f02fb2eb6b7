ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_k5_r2.csv python - <<'PY'
import torch, sys
sys.path.insert(0, '.')
import paper_2510_17505_b200 as P
from paper_2510_17505_b200 import synth as S
c = S.synth_voxel_shells(1000000).cuda()
n = c.shape[0]
mo, mi, mz = P.kernel_map(c)
g, _ = P.tune_group_size(mz, 27)
ones = torch.ones(mo.numel(), dtype=torch.float32, device='cuda')
gt = P.group_coo_tensor([n, n, 27], [mo, mi, mz], ones, 2, g, canonical=True)
torch.cuda.synchronize()
PY
