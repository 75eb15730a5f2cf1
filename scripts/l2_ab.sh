cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
RFXC_SKETCH_L2PERSIST_DEBUG=1 python scripts/path_probe.py 32 2>&1 | grep "L2 window"
python -m pytest -q -m gpu tests/test_gpu_linalg.py tests/test_gpu_sketch.py tests/test_gpu_lowrank.py 2>&1 | tail -1
B='python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d[\"kernels_ms_per_step\"]; print(round(d[\"ms_per_step\"],3), {a: round(b,3) for a,b in k.items() if b > 0.3}, d[\"e2e\"][\"ms_per_step\"])"'
for i in 1 2; do echo "persist on"; eval $B; echo "persist off"; RFXC_SKETCH_L2PERSIST=0 eval $B; done
for v in 1 0; do RFXC_SKETCH_L2PERSIST=$v timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none --clock-control none -k regex:sketch_phase -s 40 -c 4 --csv python scripts/path_probe.py 500 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print "persist='$v'", $5, $(NF-2), $NF}'; done
