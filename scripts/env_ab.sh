# A/B environment settings on the 100k bench: ENVS="A=1 B=2|A=0" bash scripts/env_ab.sh
cd "${GRAFT_REPO_ROOT:-.}"
B='python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d[\"kernels_ms_per_step\"]; print(round(d[\"ms_per_step\"],3), {a: round(b,3) for a,b in k.items() if b > 0.3}, round(d[\"e2e\"][\"ms_per_step\"],3))"'
IFS='|' read -ra SETS <<< "${ENVS}"
for i in ${ROUNDS:-1 2}; do
  for e in "${SETS[@]}"; do echo "== [$e]"; env $e bash -c "$B"; done
done
