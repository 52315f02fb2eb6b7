"""K4 timing on cfg2 (perf experiment, not part of the library): the shipped
BlockGroupCOO SpMM as a CUDA-graph replay bracketed by events after an L2
flush, median and best of --reps.

  python tools/k4_time.py [--reps 20] [--n 512]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(torch, fn, reps, flush):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):  # queued back to back (as bench.py): no host launch gap inside
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    out = [a.elapsed_time(b) * 1e3 for a, b in evs]
    out.sort()
    return out[len(out) // 2], out[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--n", type=int, default=512)
    args = ap.parse_args()
    import torch

    import paper_2510_17505_b200 as P
    from paper_2510_17505_b200 import synth as S
    dev = torch.device("cuda", 0)
    rng = S.Rng(1)
    B = S.synth_dense(rng, (512, 16, args.n), S.REAL, torch.bfloat16).to(dev)
    A = S.synth_block_sparse_matrix(rng, 8192, 8192, 16, 16, 0.10, S.REAL, torch.bfloat16)
    fmt = P.dense_to_blockgroupcoo(A.to(dev), 16, 16, 0)
    C = torch.empty((512, 16, args.n), dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    res = {"G": fmt.num_groups(), "g": fmt.group_size, "blocks": fmt.num_blocks}
    res["call_us"] = timed(torch, lambda: P.spmm_blockgroupcoo(fmt.AM, fmt.AK, fmt.AV, B, C,
                                                               accumulate=False, flags=1 | 2),
                           args.reps, flush)
    res["TFLOPs"] = 2.0 * fmt.num_blocks * 256 * args.n / (res["call_us"][0] * 1e-6) / 1e12
    print(json.dumps(res))


if __name__ == "__main__":
    main()
