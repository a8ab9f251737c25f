set -x
O=gpurun_out/r02u
mkdir -p $O
B="python bench.py --config protein --n 1073741824 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work"
$B > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -s 20 -c 24 --csv --log-file $O/launches_protein.csv $B > /dev/null 2>&1
cat $O/launches_protein.csv | cut -d, -f5,12- | tail -50
