"""DRAM bytes of one whole sketch pass (all 2 x batches phase launches, ncu
--cache-control none, so what L2 keeps between launches counts as in the real
run): python scripts/traffic_pass.py REPORT N TREES BATCHES
Writes profiles/ncu_traffic.json (bench.py reports it as roofline.traffic)."""
import csv, io, json, subprocess, sys

rep, n, trees, batches = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
cols = [h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per_launch = [sum(float(r[c].replace(",", "")) * scale.get(units[c], 1) for c in cols) for r in rows[2:]]
assert len(per_launch) == 2 * batches, (len(per_launch), batches)
total = sum(per_launch)
print("launches", len(per_launch), "pass bytes", total)
json.dump({"sketch_pass": total, "n": n, "trees": trees, "batches": batches,
           "phase_a_mean": sum(per_launch[0::2]) / batches, "phase_b_mean": sum(per_launch[1::2]) / batches,
           "last_phase_b": per_launch[-1], "source": rep, "cache_control": "none",
           "note": "all phase launches of one pass; the last phase B also adds up Y (fused final)"},
          open("profiles/ncu_traffic.json", "w"), indent=1)
