#!/bin/bash
# GPU call: default lib vs the experimental libs under _lib/exp (CMP-large
# 1024-midpoint slice, CRS-small), twice
for rep in 1 2; do
for L in paper_1907_11678_b200/_lib/libvelan_gpu.so $(ls paper_1907_11678_b200/_lib/exp/*.so); do
  n=$(basename $L .so)
  for wl in "cmp_large --gathers 1024" "crs_small"; do
    VELAN_GPU_LIB=$L timeout 300 python bench.py --workload $wl --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', '$wl'.split()[0], round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"
  done
done
done
