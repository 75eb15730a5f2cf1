"""Key details + stall reasons of an ncu report (one kernel)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
run = lambda a: subprocess.run(["ncu", "-i", rep] + a, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = rows[0]
ni, vi, si = h.index("Metric Name"), h.index("Metric Value"), h.index("Section Name")
want = {"Duration", "Grid Size", "Block Size", "Registers Per Thread", "Achieved Occupancy",
        "Theoretical Occupancy", "Executed Ipc Active", "Issued Warp Per Scheduler",
        "Memory Throughput", "L2 Cache Throughput", "DRAM Throughput", "Waves Per SM",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem"}
seen = set()
for r in rows[1:]:
    if r[ni] in want and r[ni] not in seen:
        seen.add(r[ni]); print(f"  {r[ni]:34s} {r[vi]}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
H, V = raw[0], raw[2]
st = [(H[i], V[i]) for i in range(len(H)) if "average_warps_issue_stalled" in H[i] and H[i].endswith("per_issue_active.ratio")]
st = sorted([(float(b), a.split("stalled_")[1].split("_per")[0]) for a, b in st if b.replace('.', '', 1).isdigit()], reverse=True)[:6]
print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in st))
for m in ("sm__inst_executed.sum", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"):
    if m in H: print(f"  {m} {V[H.index(m)]}")
