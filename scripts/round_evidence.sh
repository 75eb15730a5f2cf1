# Round evidence: smoke, GPU tests, the reference's own suite with the B200
# path installed, bench (with CPU baseline + secondary dense config), the
# reference arm, ncu launch list of one bench step, ncu --set full of the top
# kernels, and the sketch pass's DRAM traffic (cache-control none).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -5 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
NOCOMPAT=1 bash scripts/gpu_refsuite.sh > /dev/null 2>&1; tail -14 gpurun_out/ref_suite_gpu.log
timeout 1200 python bench.py --steps ${STEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
timeout 1500 python bench.py --impl reference --steps ${REFSTEPS:-3} --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -1 gpurun_out/bench_ref.json | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_bench.out 2>&1
python scripts/launch_summary.py gpurun_out/launches.csv mds > gpurun_out/launches_summary.txt 2>&1; head -16 gpurun_out/launches_summary.txt
if [ -z "$NOFULL" ]; then
for k in ${KERNELS:-sketch_phase_kernel mds_kernel traverse_kernel radix_bucket_kernel}; do
  c=1; if [ $k = sketch_phase_kernel ]; then c=2; fi
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c $c -o gpurun_out/full_$k -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1
done
RFX_PAIRS_KERNEL=leaf timeout 900 ncu --set full --import-source on --clock-control none -k regex:pair_seg_kernel -s 1 -c 1 -o gpurun_out/full_pair_seg -f python bench.py --config 50k-dense --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
# DRAM bytes of one sketch pass as the real run sees them (no cache flush)
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:sketch_phase_kernel -s 40 -c 2 -o gpurun_out/traffic_phases -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1
timeout 600 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:skp_final_kernel -s 2 -c 1 -o gpurun_out/traffic_final -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-secondary > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/traffic_phases.ncu-rep 16 100000 500 gpurun_out/traffic_final.ncu-rep | tail -1
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
fi
ls gpurun_out/*.ncu-rep
