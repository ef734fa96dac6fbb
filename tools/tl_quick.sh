#!/bin/bash
# GPU call: TL=1 vs TL=2 timing only (CMP-large 1024-midpoint slice, CRS-small)
O=gpurun_out/tlq; mkdir -p $O
for TL in 1 2 1 2; do
  VELAN_TL=$TL timeout 300 python bench.py --workload cmp_large --gathers 1024 --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null | tail -1 > $O/cmpl_$TL.json
  VELAN_TL=$TL timeout 300 python bench.py --workload crs_small --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null | tail -1 > $O/crss_$TL.json
  for f in cmpl crss; do python -c "import json; d=json.load(open('$O/${f}_$TL.json')); print('TL=$TL $f', round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"; done
done
