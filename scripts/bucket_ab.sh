cd "${GRAFT_REPO_ROOT:-.}"
export CMD='python -m pytest -q -m gpu tests/test_gpu_pairs.py -k "bucket" 2>&1 | tail -1; python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d[\"kernels_ms_per_step\"]; print(round(d[\"ms_per_step\"],3), {a: round(b,3) for a,b in k.items() if b > 0.3})"'
bash scripts/variants.sh
export CMD='python bench.py --steps 20 --warmup 5 --no-secondary --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d[\"kernels_ms_per_step\"]; print(round(d[\"ms_per_step\"],3), {a: round(b,3) for a,b in k.items() if b > 0.3})"'
bash scripts/variants.sh
