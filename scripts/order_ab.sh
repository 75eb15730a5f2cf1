cd "${GRAFT_REPO_ROOT:-.}"
python -m pytest -q -m gpu tests/test_gpu_membership.py 2>&1 | tail -2
ENVS="RFX_TRAV_ORDER=1|RFX_TRAV_ORDER=0" bash scripts/env_ab.sh
