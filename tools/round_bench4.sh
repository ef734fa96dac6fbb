#!/bin/bash
# One GPU call: the default bench, other workloads, the reference arm, the
# torchrun path, the ncu launch list + DRAM traffic of the default bench
# command and one full-set capture of the scan kernel.
mkdir -p gpurun_out/rb4
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/rb4/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rb4/smoke.log 2>&1; echo smoke=$?
set -x
mkdir -p gpurun_out/rb4
python bench.py > gpurun_out/rb4/bench_default.json 2> gpurun_out/rb4/bench_default.err
python bench.py --workload cmp_small --cpu-seconds 5 > gpurun_out/rb4/bench_cmp_small.json 2> gpurun_out/rb4/bench_cmp_small.err
python bench.py --workload crs_small --steps 2 --warmup 3 --cpu-seconds 10 > gpurun_out/rb4/bench_crs_small.json 2> gpurun_out/rb4/bench_crs_small.err
python bench.py --workload crs_large --gathers 64 --steps 1 --warmup 3 --no-e2e --cpu-seconds 10 > gpurun_out/rb4/bench_crs_large64.json 2> gpurun_out/rb4/bench_crs_large64.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rb4/bench_reference.json 2> gpurun_out/rb4/bench_reference.err
python bench.py --variant exact --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/rb4/bench_exact.json 2> gpurun_out/rb4/bench_exact.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu > gpurun_out/rb4/bench_torchrun1.json 2> gpurun_out/rb4/bench_torchrun1.err
# ncu: launch list (every launch, device time) and DRAM bytes of the default command
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/rb4/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/rb4/launches.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/rb4/ncu_launch.log 2>&1
# one full-set capture of the scan kernel on a CMP-large slice
python bench.py --workload cmp_large --gathers 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/rb4/slice.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:semblance_scan -c 1 -o gpurun_out/rb4/prof_final4 \
    python bench.py --workload cmp_large --gathers 256 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/rb4/ncu_full.log 2>&1
echo done
