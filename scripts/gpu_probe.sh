cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/probe_sync scripts/probe_sync.cu && timeout 60 /tmp/probe_sync
timeout 120 python scripts/mds_probe.py 100000 32 5,25,105
timeout 300 ncu --set full --import-source on --clock-control none -k regex:mds_kernel -c 1 -o gpurun_out/mds_prof python scripts/mds_probe.py 100000 32 10 > gpurun_out/mds_ncu.log 2>&1; tail -2 gpurun_out/mds_ncu.log
