mkdir -p gpurun_out/g1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/g1/pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/g1/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/g1/smoke.log
timeout 600 python bench.py > gpurun_out/g1/bench.json 2> gpurun_out/g1/bench.err; echo bench=$?; cat gpurun_out/g1/bench.json
timeout 600 python bench.py --workload crs_small --steps 2 --warmup 3 --cpu-seconds 5 > gpurun_out/g1/crs_small.json 2>&1; tail -1 gpurun_out/g1/crs_small.json
