set -x
O=gpurun_out/r02r
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
python bench.py > $O/bench_worst.json 2> $O/bench_worst.err; tail -c 3000 $O/bench_worst.json
for c in random keyword protein tiny; do python bench.py --config $c --no-cpu-baseline --quiet-json >> $O/bench_other.jsonl 2>> $O/bench_other.err; done
tools/checked_run.sh $O
