"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum CSV launch list
(divided by the number of steps captured)."""
import collections
import csv
import sys

path = sys.argv[1]
rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
# steps: the given count, or "mds" = the number of MDS launches (one per step)
arg = sys.argv[2] if len(sys.argv) > 2 else "1"
steps = float(sum(1 for r in rows if "mds_kernel" in r[4])) if arg == "mds" else float(arg)
d = collections.defaultdict(list)
for r in rows:
    name = r[4].split("(")[0].split("<")[0].replace("void ", "")
    d[name].append(float(r[-1]) / 1e6)
tot = sum(sum(v) for v in d.values())
print(f"{len(rows)} launches, {tot / steps:.3f} ms per step ({steps:g} steps)")
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:44s} n/step={len(v) / steps:7.1f} ms/step={sum(v) / steps:8.3f} avg_us={1e3 * sum(v) / len(v):9.1f}")
