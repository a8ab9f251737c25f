set -x
O=gpurun_out/r02d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in tiny random keyword; do
  for f in 1 0; do python bench.py --config $c --steps 30 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --opt fused_tail=$f --quiet-json >> $O/q_fused.txt 2>&1; done
done
python tools/phase_timing.py random keyword tiny > $O/phase_fused.txt 2>&1
FUSED=0 python tools/phase_timing.py random tiny > $O/phase_nofused.txt 2>&1
for t in 60000 75776 85000 0; do python bench.py --config worst --steps 5 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --opt subchunk_target=$t --quiet-json >> $O/sweep_worst_target.txt 2>&1; done
