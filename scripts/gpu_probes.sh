# Probes: MDS per-phase timing, L2 gather peak, and a bench run of the new bench.py
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export RFX_FOREST_CACHE=/tmp/rfxcache
RFXC_MDS_TIMING=1 python scripts/mds_probe.py 100000 32 100 > gpurun_out/mds_timing.txt 2>&1; tail -16 gpurun_out/mds_timing.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_gather scripts/probe_gather.cu && /tmp/probe_gather > gpurun_out/l2_gather_probe.txt 2>&1; cat gpurun_out/l2_gather_probe.txt
[ -z "$NOBENCH" ] && timeout 900 python bench.py --steps 5 --warmup 3 ${BENCHARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
