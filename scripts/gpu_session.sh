set -x
export RFX_FOREST_CACHE=/tmp/rfxcache
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -3 gpurun_out/smoke.log
timeout 600 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/gpu_tests.log; tail -15 gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.out 2>&1; tail -3 gpurun_out/ncu_bench.out
