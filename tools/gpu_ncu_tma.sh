O=gpurun_out/tma2
mkdir -p $O
for t in 1 0; do
  K="python bench.py --config random --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work --opt tma_input=$t"
  ncu --set full --clock-control none -k regex:"lanes_kernel" -s 6 -c 1 -o $O/random_tma$t $K > /dev/null 2>&1
  python tools/ncu_summary.py $O/random_tma$t.ncu-rep tma$t > $O/ncu_tma$t.txt 2>&1
done
rm -f $O/*.ncu-rep
cat $O/ncu_tma1.txt
