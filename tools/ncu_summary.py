"""Summarise an ncu report: key details metrics + top stall reasons + top SASS lines.
usage: python tools/ncu_summary.py report.ncu-rep [n_top]"""
import csv, io, subprocess, sys, collections

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 15
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Executed Instructions", "Issue Slots Busy", "Achieved Occupancy", "DRAM Throughput",
        "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate", "L2 Hit Rate"]
rows = list(csv.reader(io.StringIO(det)))
if rows:
    h = rows[0]
    kn, mn, mu, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    seen = set()
    for r in rows[1:]:
        if r[mn] in want and (r[kn], r[mn]) not in seen:
            seen.add((r[kn], r[mn]))
            print(f"{r[kn][:60]:60s} {r[mn]:40s} {r[mv]:>14s} {r[mu]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
if len(rr) > 2:
    h = rr[0]
    ik = h.index("Kernel Name")
    for v in rr[2:]:
        print(f"== {v[ik][:70]}")
        for key in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]:
            if key in h:
                print(f"   {key:40s} {v[h.index(key)]} {rr[1][h.index(key)]}")
        st = [(n, v[i]) for i, n in enumerate(h)
              if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued")]
        st = sorted(((n.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x.replace(",", "") or 0))
                     for n, x in st), key=lambda t: -t[1])
        tot = sum(x for _, x in st) or 1
        print("   stalls:", ", ".join(f"{n} {100 * x / tot:.1f}%" for n, x in st[:8]))
