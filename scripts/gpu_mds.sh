# MDS: tests, per-phase timing, ncu of the kernel on the probe, FP64 probe
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
[ -z "$NOTESTS" ] && timeout 900 python -m pytest tests/test_gpu_mds.py tests/test_gpu_lowrank100k.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
RFXC_MDS_TIMING=1 python scripts/mds_probe.py 100000 32 100 2>&1 | grep "\[mds\]" | head -12
python scripts/mds_probe.py 100000 32 5,100 2>&1 | grep median
RFXC_MDS_F64=1 python scripts/mds_probe.py 100000 32 5,100 2>&1 | grep median
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_fp64 scripts/probe_fp64.cu && /tmp/probe_fp64 | grep DMMA
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mds_kernel -c 1 -o gpurun_out/full_mds -f python scripts/mds_probe.py 100000 32 30 > /dev/null 2>&1; ls -la gpurun_out/full_mds.ncu-rep
fi
