"""DRAM traffic of one sketch pass from ncu captures (--cache-control none,
so the leaf sums read back from L2 count as they do in the real run):
    python scripts/ncu_traffic.py PHASES.ncu-rep BATCHES N TREES [FINAL.ncu-rep]
PHASES holds phase A + phase B of one tree batch; FINAL the per-pass ordered
f64 sum of the batch partials.  sketch_pass bytes = BATCHES x (A + B) + final.
Writes profiles/ncu_traffic.json (bench.py reports it as roofline.traffic
for that workload only)."""
import csv, io, json, subprocess, sys


def kernels(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    cols = [h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")]
    out = []
    for r in rows[2:]:
        b = sum(float(r[c].replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                 "Gbyte": 1e9}.get(units[c], 1) for c in cols)
        out.append((r[ki][:48], b))
    return out


rep, batches, n, trees = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
ph = kernels(rep)
fin = kernels(sys.argv[5]) if len(sys.argv) > 5 else []
per_pass = batches * sum(b for _, b in ph) + sum(b for _, b in fin)
print(ph, fin, "per pass", per_pass)
json.dump({"sketch_pass": per_pass, "n": n, "trees": trees, "batches": batches,
           "phases": ph, "final": fin, "sources": [rep] + sys.argv[5:6],
           "cache_control": "none"}, open("profiles/ncu_traffic.json", "w"), indent=1)
