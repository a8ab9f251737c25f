# chunk-count (1K-64K) and lanes-per-thread sweeps of the four throughput configs (BASELINE configs[4])
O=gpurun_out/sweeps
mkdir -p $O
for c in worst protein keyword random; do timeout 900 python tools/sweep.py $c > $O/sweep_$c.jsonl 2> $O/sweep_$c.err; done
tail -n 20 $O/sweep_worst.jsonl
