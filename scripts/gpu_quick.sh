# GPU tests (optionally a subset) + a short bench; output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
timeout 900 python -m pytest ${TESTS:-tests} -m gpu -q --timeout 300 -p no:cacheprovider -x 2>&1 | tail -25 > gpurun_out/gpu_tests.log; tail -25 gpurun_out/gpu_tests.log
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py --steps ${STEPS:-5} --warmup 3 ${BENCHARGS:---no-cpu-baseline} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
fi
