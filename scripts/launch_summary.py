"""Summarise an ncu --csv launch list (gpu__time_duration per launch): time per kernel for the LAST solve."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
idx = [i for i, r in enumerate(rows) if "k_split" in r[4]]
sel = rows[idx[-1]:] if idx else rows
tot = sum(float(r[14]) for r in sel)
agg = {}
for r in sel:
    name = r[4].split("(")[0].replace("void ", "")
    a = agg.setdefault(name, [0.0, 0])
    a[0] += float(r[14])
    a[1] += 1
print(f"{sys.argv[1]}: {len(sel)} launches, {tot / 1e6:.3f} ms total (serialised, cold)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"  {k:55s} {v[1]:6d} launches {v[0] / 1e3:10.1f} us {100 * v[0] / tot:5.1f}%")
