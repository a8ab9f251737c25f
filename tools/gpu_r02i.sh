set -x
O=gpurun_out/r02i
mkdir -p $O
python tools/phase_timing.py random keyword tiny > $O/phase_fused.txt 2>&1
K="python bench.py --config keyword --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --quiet-json --no-lookahead --no-batch --no-ceiling --no-work"
$K > $O/plain.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"lanes_kernel" -s 6 -c 1 -o $O/kw $K > $O/ncu.log 2>&1
python tools/ncu_summary.py $O/kw.ncu-rep keyword > $O/ncu_kw.txt 2>&1
ncu -i $O/kw.ncu-rep --page source --csv --kernel-name regex:lanes_kernel > $O/kw_source.csv 2>/dev/null; gzip -f $O/kw_source.csv
rm -f $O/kw.ncu-rep
