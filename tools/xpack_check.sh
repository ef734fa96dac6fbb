#!/bin/bash
# GPU call: EXACT-variant parity tests and timing with the packed EXACT
# library (_lib/exp/libxpack.so) against the default library
L=paper_1907_11678_b200/_lib/exp/libxpack.so
VELAN_GPU_LIB=$L timeout 900 python -m pytest tests -q -m gpu -x -k "exact or known or golden or run_cmp_matches or run_crs_matches or smoke" 2>&1 | tail -2
for rep in 1 2; do
for lib in paper_1907_11678_b200/_lib/libvelan_gpu.so $L; do
  VELAN_GPU_LIB=$lib timeout 300 python bench.py --variant exact --gathers 512 --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', 'cmp_large exact', round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"
  VELAN_GPU_LIB=$lib timeout 300 python bench.py --variant exact --workload crs_small --gathers 32 --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$(basename $lib)', 'crs_small exact', round(d['ms_per_step'],2), round(d['roofline']['frac'],4))"
done
done
