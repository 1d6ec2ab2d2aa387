"""Stall samples of one kernel's SASS, split at barrier / mbarrier / TMA instructions.

    ncu -i rep --page source --csv --print-source sass > k.csv
    python tools/ncu_segments.py k.csv
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [dict(zip(h, r)) for r in rows[2:] if len(r) == len(h) and r[0] != h[0]]
S = lambda d: int(d["Warp Stall Sampling (All Samples)"] or 0)
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(S(d) for d in data)
cut = ("BAR.SYNC", "BAR.RED", "SYNCS.ARRIVE", "SYNCS.PHASECHK", "UTMALDG", "EXIT")
last = 0
print(f"total samples {tot}, instructions executed {sum(int(d['Instructions Executed'] or 0) for d in data)/1e6:.1f}M")
for i, d in enumerate(data):
    s = d["Source"].strip()
    if any(k in s for k in cut):
        seg = data[last:i + 1]
        n = sum(S(x) for x in seg)
        if n > tot * 0.005:
            ins = sum(int(x["Instructions Executed"] or 0) for x in seg)
            agg = {r[6:]: sum(int(x[r] or 0) for x in seg) for r in reasons}
            top = ", ".join(f"{k}={100*v/tot:.1f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:5])
            print(f"{last:5d}-{i:5d} {100*n/tot:5.1f}% instr={ins/1e6:6.1f}M  [{s[:40]}]  {top}")
        last = i + 1
