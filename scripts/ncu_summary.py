"""Summarise an ncu report: key metrics + top source lines by stall samples."""
import csv, io, subprocess, sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy",
        "Registers Per Thread", "Warp Cycles Per Issued Instruction", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Dynamic Shared Memory Per Block")


def run(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def summary(rep, top=12):
    out = []
    rows = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "details", "--csv"]))))
    hdr = rows[0]
    ni, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    seen = set()
    for r in rows[1:]:
        if r[ni] in KEYS and r[ni] not in seen:
            seen.add(r[ni])
            out.append(f"  {r[ni]:36s} {r[vi]:>12s} {r[ui]}")
    raw = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "raw", "--csv"]))))
    h, units, vals = raw[0], raw[1], raw[2]
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        if m in h:
            out.append(f"  {m:36s} {vals[h.index(m)]:>12s} {units[h.index(m)]}")
    src = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "source", "--csv",
                                             "--print-source", "cuda,sass"]))))
    cur, lines = None, []
    for r in src:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) < 10 or not r[0] or r[0] == "Line No":
            continue
        try:
            lines.append((int(r[4]), int(r[7]), cur, r[0], r[1].strip()[:80]))
        except ValueError:
            pass
    ts = sum(x[0] for x in lines) or 1
    ti = sum(x[1] for x in lines) or 1
    out.append("  top source lines (stall samples %, instructions %):")
    for s, i, f, ln, text in sorted(lines, reverse=True)[:top]:
        out.append(f"   {100*s/ts:5.1f}% {100*i/ti:5.1f}%  {f}:{ln}  {text}")
    return "\n".join(out)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        print(rep)
        print(summary(rep))
