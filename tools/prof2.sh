#!/bin/bash
# full-set ncu captures of the scan kernel: CMP-large slice and CRS-small slice
mkdir -p gpurun_out/p2
python bench.py --workload crs_small --gathers 32 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p2/crs.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:semblance_scan -c 1 -o gpurun_out/p2/crs_s \
    python bench.py --workload crs_small --gathers 32 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p2/ncu_crs.log 2>&1
python bench.py --workload cmp_large --gathers 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p2/cmp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:semblance_scan -c 1 -o gpurun_out/p2/cmp_l \
    python bench.py --workload cmp_large --gathers 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/p2/ncu_cmp.log 2>&1
echo done
