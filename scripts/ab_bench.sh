# A/B the builds in variants/ on the 100k bench (ms/step + kernel split), twice each
cd "${GRAFT_REPO_ROOT:-.}"
CMD='python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d[\"kernels_ms_per_step\"]; print(round(d[\"ms_per_step\"],3), {a: round(b,3) for a,b in k.items() if b > 0.3})"' 
export CMD
for i in ${ROUNDS:-1 2}; do bash scripts/variants.sh; done
