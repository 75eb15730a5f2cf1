cd "${GRAFT_REPO_ROOT:-.}"
cp variants/m384.so paper_2511_19493_b200/_build/librfxc.so
python -m pytest -q -m gpu tests/test_gpu_mds.py tests/test_gpu_lowrank100k.py 2>&1 | tail -1
export CMD='python scripts/mds_probe.py 100000 32 100 2>&1 | tail -1'
bash scripts/variants.sh; bash scripts/variants.sh
