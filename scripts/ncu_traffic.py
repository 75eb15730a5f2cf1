"""DRAM traffic per launch of the bench's dominant region from ncu --set full
captures: sketch_pass = (phase A + phase B bytes) x tree batches per pass.
Writes profiles/ncu_traffic.json, read by bench.py (roofline.traffic)."""
import csv, io, json, subprocess, sys
rep, batches = sys.argv[1], int(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
ki = h.index("Kernel Name")
cols = [h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")]
units = rows[1]
tot = 0.0
seen = []
for r in rows[2:]:
    b = 0.0
    for c in cols:
        v = float(r[c].replace(",", ""))
        u = units[c]
        b += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    seen.append((r[ki][:40], b))
    tot += b
per_pass = tot * batches
print(seen, "per pass", per_pass)
json.dump({"sketch_pass": per_pass, "source": rep, "kernels": seen, "batches": batches},
          open("profiles/ncu_traffic.json", "w"), indent=1)
