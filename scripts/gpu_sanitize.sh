# compute-sanitizer over scripts/sanitize_probe.py: memcheck, racecheck (shared
# memory hazards), synccheck; logs in gpurun_out/sanitizer_*.log
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_probe.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
