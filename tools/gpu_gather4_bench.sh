O=gpurun_out/r02x
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/g4bench tools/tma_gather4_bench.cu -lcuda && timeout 300 /tmp/g4bench 1024 > $O/gather4_bench.jsonl 2>&1
cat $O/gather4_bench.jsonl
