"""Summarise ncu reports for profiles/: key SOL / memory / pipe / stall metrics per report, plus
the per-launch DRAM traffic map bench.py reads (profiles/ncu_traffic.json).
usage: python tools/ncu_summary.py OUT.md KEY=report.ncu-rep [KEY=report.ncu-rep ...]
KEY is 'workload:N:K:M' (the bench sweep point the report profiles)."""
import csv
import io
import json
import os
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg", "sm__inst_executed_pipe_fma_type_fp16.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "launch__grid_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "smsp__cycles_active.avg"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def main():
    out_md = sys.argv[1]
    traffic = {}
    lines = ["| metric | " + " | ".join(a.split("=")[0] for a in sys.argv[2:]) + " |",
             "|---|" + "---|" * (len(sys.argv) - 2)]
    table = {m: [] for m in WANT + ["kernel"]}
    for arg in sys.argv[2:]:
        key, rep = arg.split("=", 1)
        r = raw(rep)
        name = r.get("Kernel Name", ("?", ""))[0]
        table["kernel"].append(name.split("(")[0].replace("void ", ""))
        for m in WANT:
            v = r.get(m)
            table[m].append(f"{v[0]} {v[1]}".strip() if v else "n/a")
        rd = r.get("dram__bytes_read.sum")
        wr = r.get("dram__bytes_write.sum")
        if rd and wr:
            traffic[key] = int(to_bytes(*rd) + to_bytes(*wr))
    for m, vals in table.items():
        lines.append(f"| {m} | " + " | ".join(vals) + " |")
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
    old = json.load(open(tpath)) if os.path.exists(tpath) else {}
    old.update(traffic)
    json.dump(old, open(tpath, "w"), indent=1, sort_keys=True)
    print(open(out_md).read())
    print(traffic)


if __name__ == "__main__":
    main()
