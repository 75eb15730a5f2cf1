# The reference's own test suite (baseline/_ref/tests) with the B200 path
# installed (scripts/ref_suite_plugin.py) + the compat GPU tests.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
[ -z "$NOCOMPAT" ] && timeout 1200 python -m pytest tests/test_gpu_compat.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -15 > gpurun_out/gpu_compat.log; tail -15 gpurun_out/gpu_compat.log
cd baseline/_ref
PYTHONPATH=.:../../scripts timeout 1800 python -m pytest -p ref_suite_plugin tests -q -p no:cacheprovider --rootdir . 2>&1 | tail -60 > ../../gpurun_out/ref_suite_gpu.log
tail -40 ../../gpurun_out/ref_suite_gpu.log
