#!/bin/bash
# Round profiling: bench JSON lines, the ncu launch list of the default bench
# command, and one --set full capture per hot kernel (run under gpurun).
set -x
O=gpurun_out/r
mkdir -p $O
python bench.py > $O/bench_random.json 2> $O/bench_random.err
for c in tiny keyword protein; do python bench.py --config $c --steps 50 --e2e-steps 3 --no-cpu-baseline > $O/bench_$c.json 2>&1; done
python bench.py --config worst --steps 5 --e2e-steps 1 --no-cpu-baseline > $O/bench_worst.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json"
$B > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 12 --csv --log-file $O/launches_random.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:lanes_kernel -s 3 -c 1 -o $O/lanes_random $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 3 -c 1 -o $O/tree_random $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fold_rows -s 3 -c 1 -o $O/fold_random $B > /dev/null 2>&1
K="python bench.py --config keyword --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json"
$K > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:lanes_kernel -s 3 -c 1 -o $O/lanes_keyword $K > /dev/null 2>&1
Q="python bench.py --config protein --n 1073741824 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json"
$Q > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"lanes_kernel|converge_kernel" -s 6 -c 2 -o $O/protein $Q > /dev/null 2>&1
W="python bench.py --config worst --n 1073741824 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json"
$W > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"lanes_kernel|converge_kernel" -s 6 -c 2 -o $O/worst $W > /dev/null 2>&1
ls -la $O
