"""Summarise tools/ncu_kernel.sh captures: headline metrics, top stalls, opcode mix.
    python tools/ncu_report.py TAG [TAG...]"""
import csv
import sys
from collections import Counter

WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Issue Slots Busy", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]
for tag in sys.argv[1:]:
    res = {}
    for r in csv.DictReader(open(f"gpurun_out/{tag}_details.csv")):
        if r["Metric Name"] in WANT and not r["Rule Name"]:
            res[r["Metric Name"]] = r["Metric Value"] + " " + r["Metric Unit"]
    print("==", tag, res)
    rows = list(csv.reader(open(f"gpurun_out/{tag}_raw.csv")))
    d = dict(zip(rows[0], rows[2]))
    st = {k: float(d[k].replace(",", "")) for k in rows[0]
          if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")
          and d[k] not in ("", "n/a")}
    print("  stalls", [(k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                        round(x, 2)) for k, x in sorted(st.items(), key=lambda x: -x[1])[:8]])
    for k in ["dram__bytes_read.sum", "dram__bytes_write.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]:
        print("  ", k, d.get(k))
    src = list(csv.reader(open(f"gpurun_out/{tag}_source.csv")))
    hdr, data = src[1], src[2:]
    iE = hdr.index("Instructions Executed")
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    c, s = Counter(), Counter()
    for r in data:
        t = r[1].strip()
        if not t:
            continue
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        op = op.split(".")[0]
        c[op] += float(r[iE] or 0)
        s[op] += float(r[iS] or 0)
    tot, stot = sum(c.values()), max(sum(s.values()), 1)
    print("  opcodes (% instr, % stall samples)",
          [(k, round(100 * x / tot, 1), round(100 * s[k] / stot, 1)) for k, x in c.most_common(12)])
