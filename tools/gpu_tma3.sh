O=gpurun_out/tma2
mkdir -p $O
K="python bench.py --config random --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work --opt tma_input=1"
ncu --set full --clock-control none --import-source on -k regex:"lanes_kernel" -s 6 -c 1 -o $O/random_tma_src $K > /dev/null 2>&1
ls -la $O
