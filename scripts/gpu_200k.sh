# configs[4] on one B200 (200k x 200, 1000 trees, QLORA + MDS) and an ncu
# capture of the traversal at that shape (128-tree subset).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
timeout 2400 python bench.py --config 200k --steps 5 --warmup 3 --no-secondary ${BENCHARGS:---no-cpu-baseline} > gpurun_out/bench_200k.json 2> gpurun_out/bench_200k.err; tail -3 gpurun_out/bench_200k.err
python -c "import json;d=json.loads(open('gpurun_out/bench_200k.json').read().strip().splitlines()[-1]);print(d['ms_per_step'], d['kernels_ms_per_step'], d['e2e']['ms_per_step'])"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:traverse_kernel -s 3 -c 1 -o gpurun_out/full_traverse_200k -f python scripts/trav_probe.py 128 200000 200 1000 > /dev/null 2>&1; ls -la gpurun_out/full_traverse_200k.ncu-rep
