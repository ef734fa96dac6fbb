#!/bin/bash
# GPU tests + default bench + full-set ncu of the scan kernel (CMP-L slice)
mkdir -p gpurun_out/g2
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/g2/pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/g2/pytest.log
timeout 600 python bench.py > gpurun_out/g2/bench.json 2> gpurun_out/g2/bench.err; echo bench=$?; cat gpurun_out/g2/bench.json
python bench.py --workload cmp_large --gathers 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/g2/cmp.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:semblance_scan -c 1 -o gpurun_out/g2/cmp_l \
    python bench.py --workload cmp_large --gathers 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/g2/ncu_cmp.log 2>&1
echo done
