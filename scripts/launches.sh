# ncu launch list (per-kernel durations) of one bench step; summary printed.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCHARGS} > gpurun_out/ncu_bench.out 2>&1; tail -2 gpurun_out/ncu_bench.out
python scripts/launch_summary.py gpurun_out/launches.csv ${NSTEPS:-5}
