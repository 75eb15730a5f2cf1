# Dense path check: K3 parity tests (both kernels, full-size SHAs) + the
# configs[2] bench with each kernel.  Output in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
[ -z "$NOTESTS" ] && timeout 1200 python -m pytest ${TESTS:-tests/test_gpu_pairs.py tests/test_gpu_scale.py} -m gpu -q --timeout 900 -p no:cacheprovider -x 2>&1 | tail -25 > gpurun_out/gpu_tests_dense.log; tail -25 gpurun_out/gpu_tests_dense.log
for k in ${KERNELS:-leaf tile}; do
  RFX_PAIRS_KERNEL=$k timeout 900 python bench.py --config 50k-dense --steps ${STEPS:-3} --warmup 3 --no-cpu-baseline > gpurun_out/bench_dense_$k.json 2> gpurun_out/bench_dense_$k.err
  tail -2 gpurun_out/bench_dense_$k.err; cut -c1-400 gpurun_out/bench_dense_$k.json
  python -c "import json;d=json.load(open('gpurun_out/bench_dense_$k.json'));print('$k', d['ms_per_step'], d['kernels_ms_per_step'], d['roofline']['frac'], d['e2e']['ms_per_step'])"
done
if [ -n "$NCU" ]; then
  RFX_PAIRS_KERNEL=leaf timeout 900 ncu --set full --import-source on --clock-control none -k regex:pair_seg_kernel -s 1 -c 1 -o gpurun_out/full_pair_seg -f python bench.py --config 50k-dense --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_dense.out 2>&1
  tail -3 gpurun_out/ncu_dense.out
fi
