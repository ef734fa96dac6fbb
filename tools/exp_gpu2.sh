#!/bin/bash
# default + experimental libraries on all four workloads (CRS-L: 64-midpoint slice)
for L in paper_1907_11678_b200/_lib/libvelan_gpu.so $(ls paper_1907_11678_b200/_lib/exp/*.so 2>/dev/null); do
  for WL in "cmp_large --gathers 1024" "crs_small" "cmp_small" "crs_large --gathers 64"; do
    VELAN_GPU_LIB=$L timeout 300 python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', '$WL', round(d['ms_per_step'],2), round(d['roofline']['frac'],4))" 2>/dev/null || echo "$(basename $L) $WL FAILED"
  done
done
