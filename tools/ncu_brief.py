"""Brief of one ncu report: duration, DRAM throughput, issue/pipe utilisation, stall mix and
the instruction-count breakdown (by opcode) from the SASS source page.
usage: python tools/ncu_brief.py report.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
hdr = raw[0]
d = dict(zip(hdr, raw[2]))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "smsp__cycles_active.avg",
        "sm__cycles_elapsed.avg"]
print(d.get("Kernel Name", "")[:90])
for k in keys:
    if k in d:
        print(f"  {k:70s} {d[k]}")
st = {k: float(d[k]) for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio") and d[k]}
print("  stalls/issue:", ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v:.2f}"
                                  for k, v in sorted(st.items(), key=lambda kv: -kv[1]) if v > 0.05))
src = page("source", ["--print-source", "sass"])
h = src[0] if "Source" in src[0] else src[1]
rows = src[src.index(h) + 1:]
ie, si = h.index("Instructions Executed"), h.index("Source")
ws = h.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter()
stall = collections.Counter()
for r in rows:
    s = r[si].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    op = s.split()[0] if s else "?"
    ops[op] += float(r[ie] or 0)
    stall[op] += float(r[ws] or 0)
tot = sum(ops.values())
tots = sum(stall.values()) or 1
print(f"  warp instructions {tot:.0f}")
for op, n in ops.most_common(22):
    print(f"    {op:34s} {n:12.0f} {n / tot * 100:5.1f}%   stall-samples {stall[op] / tots * 100:5.1f}%")
