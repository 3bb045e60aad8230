"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py: per
(kernel, grid) the launch count and mean device time, and each one's share of the quick
kernels' total (the share the bench's live CUDA-event timing must agree with)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ki, gi, vi = hdr.index("Kernel Name"), hdr.index("Grid Size"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in data:
    name = r[ki].split("(")[0].replace("void ", "")
    agg[(name, r[gi])].append(float(r[vi]) / 1e3)
quick_total = sum(sum(v) for (n, g), v in agg.items() if "quick" in n)
print("| kernel | grid | launches | mean us | share of quick kernel time |")
print("|---|---|---|---|---|")
for (n, g), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    share = sum(v) / quick_total if "quick" in n else float("nan")
    print(f"| {n} | {g} | {len(v)} | {sum(v) / len(v):.2f} | {share:.3f} |")
