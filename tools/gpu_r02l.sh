set -x
O=gpurun_out/r02l
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py --steps 10 > $O/bench_worst.json 2> $O/bench_worst.err
for c in tiny random keyword protein; do python bench.py --config $c --steps 20 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json >> $O/q.txt 2>&1; done
for t in 60000 94720 120000 0; do python bench.py --config protein --steps 10 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --opt subchunk_target=$t --quiet-json >> $O/sweep_protein_target.txt 2>&1; done
