"""K4 pipeline timeline (perf experiment): per-CTA globaltimer stamps from a
build with -DIXB_K4_TRACE (tools/build_variant.sh k4tr spmm_bgcoo_tc.cu
-DIXB_K4_TRACE), one cfg2 call after warm-up, summarised as percentiles
relative to the earliest CTA start (microseconds).

  IXB_LIB_PATH=scratch_libs/k4tr/libixb.so python tools/k4_trace.py
"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {0: "start", 1: "setup_done", 2: "sched_first_push", 3: "sched_end",
         4: "prod_first_tma", 5: "prod_last_tma", 6: "iss_first_stage", 7: "iss_last_stage",
         8: "epi_first_seg", 9: "epi_last_seg", 10: "end"}


def main():
    import torch

    import paper_2510_17505_b200 as P
    from paper_2510_17505_b200 import abi, synth as S
    lib = abi.lib()
    dev = torch.device("cuda", 0)
    rng = S.Rng(1)
    B = S.synth_dense(rng, (512, 16, 512), S.REAL, torch.bfloat16).to(dev)
    A = S.synth_block_sparse_matrix(rng, 8192, 8192, 16, 16, 0.10, S.REAL, torch.bfloat16)
    fmt = P.dense_to_blockgroupcoo(A.to(dev), 16, 16, 0)
    C = torch.empty((512, 16, 512), dtype=torch.float32, device=dev)
    run = lambda: P.spmm_blockgroupcoo(fmt.AM, fmt.AK, fmt.AV, B, C, accumulate=False, flags=1 | 2)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    f = lib.ixb_debug_k4_trace
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    f(None, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    flush.zero_()  # keeps the GPU busy while the host enqueues: no launch gap in the events
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    h = np.zeros(4096 * 16, dtype=np.int64)
    f(h.ctypes.data, 0)
    t = h.reshape(4096, 16)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    out = {"ctas": int(used.sum()), "event_us": e0.elapsed_time(e1) * 1e3}
    for k, n in NAMES.items():
        v = t[:, k]
        v = v[v > 0]
        if len(v) == 0:
            continue
        r = (v - t0) / 1e3
        out[n] = {q: round(float(np.percentile(r, q)), 2) for q in (0, 10, 50, 90, 100)}
    out["segments_per_cta"] = {q: float(np.percentile(t[:, 11], q)) for q in (0, 50, 100)}
    out["stages_per_cta"] = {q: float(np.percentile(t[:, 12], q)) for q in (0, 50, 100)}
    dur = (t[:, 7] - t[:, 6]) / 1e3
    out["iss_active_us"] = {q: round(float(np.percentile(dur, q)), 2) for q in (10, 50, 90, 100)}
    # end time (us) by CTA index (c and c + grid/2 usually share an SM)
    endt = (t[:, 10] - t0) / 1e3
    first = (t[:, 6] - t0) / 1e3
    n = len(endt)
    out["end_by_cta_half"] = [round(float(np.median(endt[: n // 2])), 2),
                              round(float(np.median(endt[n // 2:])), 2)]
    order = np.argsort(endt)
    out["latest_ctas"] = [(int(i), round(float(endt[i]), 2), round(float(first[i]), 2))
                          for i in order[-12:]]
    out["earliest_ctas"] = [(int(i), round(float(endt[i]), 2), round(float(first[i]), 2))
                            for i in order[:6]]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
