#!/bin/bash
# GPU call: time the default library and every experimental build under
# paper_1907_11678_b200/_lib/exp/ on a CMP-large slice, CRS small and a CRS
# large slice, two interleaved rounds (variants compared inside one call:
# boxes differ by a few percent).  usage: tools/exp_libs.sh [OUT]
OUT=${1:-gpurun_out/exp}; mkdir -p $OUT
LIBS="paper_1907_11678_b200/_lib/libvelan_gpu.so $(ls paper_1907_11678_b200/_lib/exp/*.so 2>/dev/null)"
for R in 1 2; do
  for L in $LIBS; do
    for WL in "cmp_large --gathers 1024" "crs_small" "crs_large --gathers 64"; do
      VELAN_GPU_LIB=$L timeout 600 python bench.py --workload $WL --steps 2 --warmup 2 \
          --no-e2e --no-cpu --no-parity --no-sub 2>>$OUT/err.log | tail -1 | \
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$R', '$(basename $L)', '$WL'.split()[0], round(d['ms_per_step'],2), round(d['roofline']['frac'],4))" \
        | tee -a $OUT/results.txt
    done
  done
done
