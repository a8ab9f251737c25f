set -x
O=gpurun_out/r02t
mkdir -p $O
for c in worst protein; do
  Q="python bench.py --config $c --n 1073741824 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work"
  $Q > $O/plain_$c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"converge_kernel" -s 3 -c 1 -o $O/conv_$c $Q > /dev/null 2>&1
done
ls -la $O
