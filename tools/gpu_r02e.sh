set -x
O=gpurun_out/r02h
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "pipelined or fused or config_small or tiny_hard or segment or graph or starts or edge or 2_20" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in tiny random keyword; do
  for f in 1 0; do python bench.py --config $c --steps 30 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --opt fused_tail=$f --quiet-json >> $O/q_fused.txt 2>&1; done
done
python tools/phase_timing.py random keyword tiny > $O/phase_fused.txt 2>&1
