# Round evidence: smoke, GPU tests, the reference's own suite with the B200
# path installed, bench (with CPU baseline), reference arm, dense bench, ncu
# launch list of one bench step, ncu --set full of the top kernels.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
NOCOMPAT=1 bash scripts/gpu_refsuite.sh > /dev/null 2>&1; tail -14 gpurun_out/ref_suite_gpu.log
timeout 900 python bench.py --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 1500 python bench.py --impl reference --steps ${REFSTEPS:-3} --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-300
timeout 900 python bench.py --config 50k-dense --steps 5 --warmup 3 > gpurun_out/bench_dense.json 2> gpurun_out/bench_dense.err; tail -1 gpurun_out/bench_dense.json | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.out 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv 8 | head -16 | tee gpurun_out/launches_summary.txt
if [ -z "$NOFULL" ]; then
for k in ${KERNELS:-sketch_phase_kernel mds_kernel traverse_kernel radix_bucket_kernel}; do
  c=1; if [ $k = sketch_phase_kernel ]; then c=2; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c $c -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
python scripts/ncu_traffic.py gpurun_out/full_sketch_phase_kernel.ncu-rep 16 | tail -1
fi
ls gpurun_out/*.ncu-rep
