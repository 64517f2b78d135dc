"""Per-source-line instruction and stall-sample shares of one kernel in an
ncu report (captured with -lineinfo + --import-source on).

    python tools/ncu_lines.py REPORT.ncu-rep [TOP]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = {}
for r in csv.reader(out.splitlines()):
    if len(r) < 9 or not r[0].isdigit() or r[2] != "-":
        continue
    ie = float(r[7]) if r[7] not in ("-", "") else 0.0
    st = float(r[4]) if r[4] not in ("-", "") else 0.0
    k = (int(r[0]), r[1].strip()[:100])
    a = agg.setdefault(k, [0.0, 0.0])
    a[0] += ie
    a[1] += st
tot = sum(v[0] for v in agg.values()) or 1.0
tst = sum(v[1] for v in agg.values()) or 1.0
print(f"warp instructions {tot:.0f}, stall samples {tst:.0f} (inlined lines counted at each level)")
print("--- by instructions")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]:5d} {100 * v[0] / tot:5.1f}% inst {100 * v[1] / tst:5.1f}% stall  {k[1]}")
print("--- by stall samples")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]:5d} {100 * v[0] / tot:5.1f}% inst {100 * v[1] / tst:5.1f}% stall  {k[1]}")
