cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 180 -p no:cacheprovider -x 2>&1 | tail -4
timeout 120 python scripts/mds_probe.py 100000 32 5,25,105
for k in traverse_kernel bucket_kernel leaf_sums_kernel leaf_gather_kernel; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k python scripts/path_probe.py 64 > gpurun_out/ncu_$k.log 2>&1; tail -1 gpurun_out/ncu_$k.log
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:mds_kernel -c 1 -o gpurun_out/prof_mds python scripts/mds_probe.py 100000 32 10 > gpurun_out/ncu_mds.log 2>&1; tail -1 gpurun_out/ncu_mds.log
