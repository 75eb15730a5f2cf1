# DRAM bytes per sketch batch (phase A + B, warm L2) with two leaf-sum
# buffers (default) and with one (RFX_SKETCH_L2_FRACTION=0.5)
cd "${GRAFT_REPO_ROOT:-.}"
for f in 0.9 0.5; do
  RFX_SKETCH_L2_FRACTION=$f timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:sketch_phase_kernel -s 40 -c 4 --csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary 2>/dev/null | grep -E '"(dram__|gpu__time)' | awk -F'","' -v f=$f '{print "fraction=" f, $5, $(NF-2), $NF}'
done
