#!/bin/bash
# One GPU call: the evidence of a round — the default bench (CMP large +
# the crs_small sub-record), the other workloads, both reference arms, the
# EXACT variant, the --gpus / torchrun paths at N = 1, the ncu launch list
# with DRAM bytes of the bench command, and full-set captures of the scan
# kernel.  usage: tools/round_bench.sh OUT
O=${1:-gpurun_out/round}; mkdir -p $O
set -x
python bench.py --steps 10 --warmup 3 > $O/bench_default.json 2> $O/bench_default.err
python bench.py --workload cmp_small --cpu-seconds 5 > $O/bench_cmp_small.json 2> $O/bench_cmp_small.err
python bench.py --workload crs_large --gathers 256 --steps 1 --warmup 1 > $O/bench_crs_large256.json 2> $O/bench_crs_large256.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
python bench.py --impl reference --workload crs_small --steps 3 --warmup 1 > $O/bench_reference_crs_small.json 2> $O/bench_reference_crs_small.err
python bench.py --variant exact --steps 1 --warmup 3 --no-e2e --no-cpu --no-sub > $O/bench_exact.json 2> $O/bench_exact.err
python bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu --no-sub > $O/bench_gpus1.json 2> $O/bench_gpus1.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu --no-sub > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err
for WL in "cmp_large 8192" "crs_small 256"; do
  set -- $WL
  CMD="python bench.py --workload $1 --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-sub"
  $CMD > $O/plain_$1.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file $O/launches_$1.csv $CMD > $O/ncu_launch_$1.log 2>&1
done
./tools/ncu_cmp.sh $O cmp_large 148
./tools/ncu_cmp.sh $O crs_small 32
./tools/ncu_cmp.sh $O crs_large 12
echo done
