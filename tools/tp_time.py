"""Times the K7 tensor-core kernel on the cfg4 shape (1M edges), once per
command-line tag (each in a fresh process; set IXB_LIB_PATH to time another
build of libixb.so). Perf experiment, not a bench number."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2510_17505_b200 as P
    from paper_2510_17505_b200 import synth as S
    B = 1_000_000
    rng = S.Rng(1)
    X = S.synth_dense(rng, (B, 16, 64), S.REAL, torch.bfloat16).cuda()
    Y = S.synth_dense(rng, (B, 16), S.REAL, torch.bfloat16).cuda()
    cg = S.cg_table(3)
    nl = cg["npaths"]
    W = S.synth_dense(rng, (nl, 64, 64), S.REAL, torch.bfloat16).cuda()
    gt = P.group_coo_tensor([16, 16, 16, nl], [cg[k].cuda() for k in ("i", "j", "k", "l")],
                            cg["v"].cuda(), 3, 4)
    plan = P.TpPlan(gt.group_coord, *gt.member_coords, gt.values, 16, 16, 16, nl)
    Z = torch.empty((B, 16, 64), device="cuda")
    for _ in range(3):
        plan.run(X, Y, W, Z, accumulate=False)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        plan.run(X, Y, W, Z, accumulate=False)
    b.record()
    torch.cuda.synchronize()
    print(f"{os.environ.get('TP_TAG', '')}: {a.elapsed_time(b) / 10:.3f} ms")
else:
    for d in sys.argv[1:] or ["0"]:
        subprocess.run([sys.executable, __file__, "--child"], env=dict(os.environ, TP_TAG=d))
