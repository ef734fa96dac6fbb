mkdir -p gpurun_out/pw
for L in profw profw512; do VELAN_GPU_LIB=paper_1907_11678_b200/_lib/exp/lib$L.so timeout 300 python bench.py --workload cmp_large --gathers 1024 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/pw/$L.txt 2>&1; done
