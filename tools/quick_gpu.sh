#!/bin/bash
# quick GPU check: tests, CMP-L slice timing for the default + experimental libs
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_q.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_q.log
for L in paper_1907_11678_b200/_lib/libvelan_gpu.so $(ls paper_1907_11678_b200/_lib/exp/*.so 2>/dev/null); do
  VELAN_GPU_LIB=$L timeout 300 python bench.py --workload cmp_large --gathers 1024 --steps 2 --warmup 1 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', d['ms_per_step'], d['roofline']['frac'])"
done
