set -x
O=gpurun_out/r02b
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py > $O/bench_worst.json 2> $O/bench_worst.err
for c in tiny random keyword protein; do python bench.py --config $c --steps 20 --e2e-steps 2 --no-cpu-baseline --quiet-json > $O/q_$c.txt 2>&1; done
for P in 1024 2048 4096 8192 16384; do python bench.py --config worst --chunks $P --steps 5 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json >> $O/sweep_worst.txt 2>&1; done
