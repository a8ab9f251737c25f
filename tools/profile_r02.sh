#!/bin/bash
# Round-2 profiling (run under gpurun): bench JSON lines for every config (the default
# command first), convergence-off and Alg.2 lines, the reference arm, the ncu launch list of
# the default bench command and one --set full capture per config's hot kernels.  Then here:
# tools/ncu_summary.py / tools/ncu_traffic.py output is copied to profiles/r02_*.
set -x
O=gpurun_out/r02p
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench_worst.json 2> $O/bench_worst.err
for c in tiny random keyword protein; do python bench.py --config $c --steps 50 --e2e-steps 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err; done
for c in tiny random keyword protein; do python bench.py --config $c --steps 20 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --convergence 0 > $O/bench_noconv_$c.json 2>&1; done
python bench.py --config worst --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --convergence 0 > $O/bench_noconv_worst.json 2>&1
for c in random keyword protein worst; do python bench.py --config $c --steps 5 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --alg2 > $O/bench_alg2_$c.json 2>&1; done
python bench.py --impl reference --steps 5 --warmup 1 > $O/bench_reference.json 2>&1
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work"
$B > $O/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 40 --csv --log-file $O/launches_worst.csv $B > /dev/null 2>&1
for c in worst protein; do
  Q="python bench.py --config $c --n 1073741824 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work"
  $Q > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"lanes_kernel|converge_kernel|fchunk_kernel|fexpand_kernel|ffold_kernel" -s 15 -c 5 -o $O/$c $Q > /dev/null 2>&1
done
for c in random keyword tiny; do
  K="python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work"
  $K > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:"lanes_kernel|compose8" -s 6 -c 2 -o $O/$c $K > /dev/null 2>&1
done
for r in worst protein random keyword tiny; do
  [ -f $O/$r.ncu-rep ] && python tools/ncu_summary.py $O/$r.ncu-rep $r > $O/ncu_$r.txt 2>&1
done
python tools/ncu_traffic.py $O/traffic.json worst=$O/worst.ncu-rep:1073741824 protein=$O/protein.ncu-rep:1073741824 \
  random=$O/random.ncu-rep:268435456 keyword=$O/keyword.ncu-rep:1073741824 tiny=$O/tiny.ncu-rep:1048576 > /dev/null 2>&1
rm -f $O/*.ncu-rep
ls -la $O
