"""Timeline of CTA 0 of the K7 kernel (a build with -DIXB_TP_TRACE, loaded via
IXB_LIB_PATH): per group, the MMA issuer's W wait / V-slot wait / commit and
consumer warps' V wait / release, in cycles. Perf experiment."""
import ctypes
import os
import subprocess
import sys

import numpy as np

here = os.path.dirname(os.path.abspath(__file__))
subprocess.run([sys.executable, os.path.join(here, "tp_run.py"), "1"], check=True,
               env=dict(os.environ, TP_TRACE_DUMP="/tmp/tp_trace.npy"))
t = np.load("/tmp/tp_trace.npy").reshape(4, 4, 512).astype(np.int64)
t0 = t[1, 0, 0]
print("group  mma:wW  wW->  vE->  commit   cons4: wait  got  done   cons19 done   wload")
print("pass end (consumer warp 4): start  after-read-wait  after-barA  after-barB  after-barC  coefs-done  after-bar")
for P in range(1, 13):
    print(P, " ".join(f"{t[i, j, P] - t0:8d}" for i, j in ((3, 0), (3, 1), (3, 2), (0, 1), (0, 2), (3, 3), (0, 3))))
for g in range(0, 130):
    r = [t[1, 0, g], t[1, 1, g], t[1, 2, g], t[1, 3, g], t[2, 0, g], t[2, 1, g], t[2, 2, g],
         0, t[0, 0, g]]
    print(f"{g:4d} " + " ".join(f"{(x - t0) if x else 0:7d}" for x in r))
