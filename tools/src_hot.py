"""Aggregate an ncu source page (--page source --csv --print-source cuda,sass)
by CUDA source line: warp-stall samples and warp instructions executed.

    ncu -i rep --page source --csv --print-source cuda,sass [--launch-skip k
        --launch-count 1] > src.csv ; python tools/src_hot.py src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        si = 4  # Warp Stall Sampling (All Samples)
        ie = 7  # Instructions Executed
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    try:
        s, n = int(r[si]), int(r[ie])
    except ValueError:
        continue
    out.append((s, n, f"{fname}:{r[0]}", r[1].strip()[:90]))
ts = sum(o[0] for o in out) or 1
tn = sum(o[1] for o in out) or 1
print(f"samples {ts}  warp-instructions {tn}")
for s, n, loc, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / ts:5.1f}% {100 * n / tn:5.1f}%i  {loc:22s} {src}")
