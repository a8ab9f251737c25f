#!/bin/bash
# Round profiling (run under gpurun): bench JSON lines for every config, the
# ncu launch list of the default bench command, and one --set full capture
# per hot kernel.  Then, here: tools/ncu_summary.py / tools/ncu_traffic.py.
set -x
O=gpurun_out/r
mkdir -p $O
python bench.py > $O/bench_random.json 2> $O/bench_random.err
for c in tiny keyword protein; do python bench.py --config $c --steps 50 --e2e-steps 3 --no-cpu-baseline > $O/bench_$c.json 2>&1; done
python bench.py --config worst --steps 5 --e2e-steps 1 --no-cpu-baseline > $O/bench_worst.json 2>&1
for c in random keyword protein; do python bench.py --config $c --steps 20 --e2e-steps 1 --no-cpu-baseline --no-lookahead --alg2 > $O/bench_alg2_$c.json 2>&1; done
for c in random keyword; do python bench.py --config $c --steps 20 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --convergence 0 > $O/bench_noconv_$c.json 2>&1; done
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ldsb tools/lds_gather_bench.cu && /tmp/ldsb 1024 > $O/lds_gather.jsonl 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead"
$B > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 12 --csv --log-file $O/launches_random.csv $B > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"lanes_kernel|compose8" -s 6 -c 2 -o $O/random $B > /dev/null 2>&1
for c in tiny keyword; do
  K="python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead"
  $K > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"lanes_kernel|compose8" -s 6 -c 2 -o $O/$c $K > /dev/null 2>&1
done
for c in protein worst; do
  Q="python bench.py --config $c --n 1073741824 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead"
  $Q > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"lanes_kernel|converge_kernel|walk_kernel" -s 9 -c 3 -o $O/$c $Q > /dev/null 2>&1
done
ls -la $O
# summarise on the box (the .ncu-rep files are too big to bring back all)
for r in random tiny keyword protein worst; do
  [ -f $O/$r.ncu-rep ] && python tools/ncu_summary.py $O/$r.ncu-rep $r > $O/ncu_$r.txt 2>&1
done
python tools/ncu_traffic.py $O/traffic.json random=$O/random.ncu-rep:268435456 tiny=$O/tiny.ncu-rep:1048576 \
  keyword=$O/keyword.ncu-rep:1073741824 protein=$O/protein.ncu-rep:1073741824 worst=$O/worst.ncu-rep:1073741824 > /dev/null 2>&1
for r in $O/*.ncu-rep; do
  ncu -i $r --page source --csv --kernel-name regex:lanes_kernel > ${r%.ncu-rep}_lanes_source.csv 2>/dev/null
  gzip -f ${r%.ncu-rep}_lanes_source.csv
done
rm -f $O/tiny.ncu-rep $O/keyword.ncu-rep $O/protein.ncu-rep $O/worst.ncu-rep
du -sh $O
