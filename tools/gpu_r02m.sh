set -x
O=gpurun_out/r02m
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ldsb tools/lds_gather_bench.cu -lcuda && /tmp/ldsb 1024 > $O/lds_gather.jsonl 2>&1
for c in 1/2 1/1 2/1 7/1; do python bench.py --config random --c $c --steps 20 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json >> $O/c_sweep.txt 2>&1; done
for c in 1/2 1/1 2/1 240/1; do python bench.py --config worst --c $c --steps 5 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json >> $O/c_sweep.txt 2>&1; done
