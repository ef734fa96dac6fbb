#!/bin/bash
# GPU call: CRS large on a 1024-midpoint slice (a quarter of the line; the
# per-midpoint work is the full config's), W=3, K=1
O=gpurun_out/crsl; mkdir -p $O
timeout 1800 python bench.py --workload crs_large --gathers 1024 --steps 1 --warmup 3 --no-e2e --cpu-seconds 10 > $O/bench_crs_large1024.json 2> $O/bench_crs_large1024.err
tail -1 $O/bench_crs_large1024.json
