cd "${GRAFT_REPO_ROOT:-.}"
cp variants/j1.so paper_2511_19493_b200/_build/librfxc.so
python -m pytest -q -m gpu tests/test_gpu_sketch.py tests/test_gpu_lowrank.py 2>&1 | tail -1
cp variants/j0.so paper_2511_19493_b200/_build/librfxc.so
ROUNDS="1 2" bash scripts/ab_bench.sh
