# Final-state evidence: smoke, bench (20 steps, CPU baseline, secondary
# configs), ncu launch list of one step, ncu --set full of the traversal.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_bench.out 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv mds > gpurun_out/launches_summary.txt 2>&1; head -6 gpurun_out/launches_summary.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:traverse_kernel -s 2 -c 1 -o gpurun_out/full_traverse_kernel -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
