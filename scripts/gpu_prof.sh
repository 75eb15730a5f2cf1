# ncu --set full captures of the hot kernels (one launch each) on the
# bench-shaped workload subset; reports land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in ${KERNELS:-traverse_kernel bucket_kernel leaf_sums_kernel leaf_gather_kernel}; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$k -s 1 -c 1 \
      -o gpurun_out/prof_$k -f python scripts/path_probe.py ${PROBE_TREES:-64} > gpurun_out/ncu_$k.log 2>&1
  tail -1 gpurun_out/ncu_$k.log
done
if [ -n "$MDS" ]; then
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:mds_kernel -c 1 \
      -o gpurun_out/prof_mds -f python scripts/mds_probe.py 100000 32 10 > gpurun_out/ncu_mds.log 2>&1
  tail -1 gpurun_out/ncu_mds.log
fi
