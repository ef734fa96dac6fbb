#!/bin/bash
# GPU call: one ncu --set full capture of the scan kernel on CRS small (a
# 16-midpoint slice) and CRS large (a 4-midpoint slice), each after the same
# command has exited 0 without ncu
O=gpurun_out/ncrs; mkdir -p $O
for spec in "crs_small 16" "crs_large 4"; do
  set -- $spec
  python bench.py --workload $1 --gathers $2 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/$1.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:semblance_scan -c 1 -o $O/prof_$1 \
      python bench.py --workload $1 --gathers $2 --steps 1 --warmup 1 --no-e2e --no-cpu > $O/ncu_$1.log 2>&1
  echo $1 $?
done
