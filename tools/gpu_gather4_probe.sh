O=gpurun_out/r02w
mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/g4probe tools/tma_gather4_probe.cu -lcuda && timeout 120 /tmp/g4probe > $O/gather4_probe.jsonl 2>&1
cat $O/gather4_probe.jsonl
