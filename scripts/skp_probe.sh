# Sketch phase timing: correctness tests, pass time, per-phase ncu launch sums.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
python -m pytest tests/test_gpu_sketch.py tests/test_gpu_lowrank.py -q -x 2>&1 | tail -1
echo TESTS; RFXC_SKETCH_TIMING=1 python scripts/path_probe.py 500 2>&1 | grep sketch | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sketch_ --csv --log-file gpurun_out/skp_launches.csv python scripts/path_probe.py 500 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open('gpurun_out/skp_launches.csv')) if len(r) > 10 and r[0].isdigit()]
acc = collections.defaultdict(list)
for r in rows: acc[r[4][:40]].append(float(r[-1]) / 1e3)
for k, x in acc.items(): print(k, len(x), "per pass ms %.3f avg us %.1f" % (sum(x) / 2 / 1e3, sum(x) / len(x)))
PY
