# Traversal: tree-top shared-memory staging ablation (RFXC_TRAV_TOP) at the
# 100k x 100 and 200k x 200 shapes; same codes required.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cfg in "128 100000 100 500" "128 200000 200 1000"; do
  for top in 0 63 127 255; do
    RFXC_TRAV_TOP=$top python scripts/trav_probe.py $cfg 2>&1 | tail -1 | sed "s/^/top=$top /"
  done
done | tee gpurun_out/trav_top_ablation.txt
