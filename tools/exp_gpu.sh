#!/bin/bash
# time the default and every experimental library on CMP-L (1024 gathers) and CRS-S
for L in paper_1907_11678_b200/_lib/libvelan_gpu.so $(ls paper_1907_11678_b200/_lib/exp/*.so 2>/dev/null); do
  for WL in "cmp_large --gathers 1024" "crs_small"; do
    VELAN_GPU_LIB=$L timeout 300 python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $L)', '$WL', round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"
  done
done
