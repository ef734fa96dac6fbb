#!/bin/bash
mkdir -p gpurun_out/p4
python bench.py --workload crs_small --gathers 32 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p4/crs.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:semblance_scan -c 1 -o gpurun_out/p4/crs_s \
    python bench.py --workload crs_small --gathers 32 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p4/ncu_crs.log 2>&1
echo done
