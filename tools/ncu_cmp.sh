#!/bin/bash
# GPU call: one ncu --set full capture (with SASS source) of the scan kernel
# on a CMP-large slice, after the same command has exited 0 without ncu.
# usage: tools/ncu_cmp.sh OUTDIR [workload] [gathers]
O=${1:-gpurun_out/ncmp}; WL=${2:-cmp_large}; NG=${3:-148}; mkdir -p $O
CMD="python bench.py --workload $WL --gathers $NG --steps 1 --warmup 1 --no-e2e --no-cpu"
$CMD > $O/plain_$WL.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:semblance_scan -c 1 \
    -o $O/prof_$WL $CMD > $O/ncu_$WL.log 2>&1
echo "$WL rc=$?"
