"""Top SASS lines of an ncu report by stall samples and by instructions
executed: `python tools/ncu_sass_hot.py report.ncu-rep [n]`."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
ci = {k: i for i, k in enumerate(hdr)}
samp = ci["Warp Stall Sampling (All Samples)"]
inst = ci["Instructions Executed"]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot_s = sum(num(r[samp]) for r in data)
tot_i = sum(num(r[inst]) for r in data)
stall_cols = [k for k in hdr if k.startswith("stall_")]
print(f"total samples {tot_s:.0f}, instructions {tot_i:.3e}")
for r in sorted(data, key=lambda r: -num(r[samp]))[:n]:
    top = sorted(((num(r[ci[k]]), k) for k in stall_cols), reverse=True)[:2]
    print(f"{100 * num(r[samp]) / tot_s:5.2f}% {num(r[inst]):12.0f} {r[ci['Address']]:>6} "
          f"{r[ci['Source']][:60]:60s} {top}")
# instruction mix by opcode
mix = {}
for r in data:
    op = r[ci["Source"]].split()[0] if r[ci["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[ci["Source"]].split()[1]
    op = op.split(".")[0]
    mix[op] = mix.get(op, 0) + num(r[inst])
print("instruction mix:", ", ".join(f"{k} {100 * v / tot_i:.1f}%"
                                    for k, v in sorted(mix.items(), key=lambda kv: -kv[1])[:16]))
