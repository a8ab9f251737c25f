set -x
O=gpurun_out/r02c
mkdir -p $O
python bench.py --steps 10 > $O/bench_worst.json 2> $O/bench_worst.err
python bench.py --config protein --steps 10 --e2e-steps 1 --no-cpu-baseline --quiet-json > $O/q_protein.txt 2>&1
Q="python bench.py --config worst --n 1073741824 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work"
$Q > $O/plain.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"converge_kernel|lanes_kernel|walk_kernel" -s 6 -c 4 -o $O/worst $Q > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/worst.ncu-rep worst > $O/ncu_worst.txt 2>&1
ncu -i $O/worst.ncu-rep --page source --csv --kernel-name regex:converge_kernel > $O/worst_converge_source.csv 2>/dev/null
gzip -f $O/worst_converge_source.csv
rm -f $O/worst.ncu-rep
