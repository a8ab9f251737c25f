O=gpurun_out/kw
mkdir -p $O
rm -f $O/sweep3.txt
for c in keyword tiny random; do python bench.py --config $c --steps 30 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --quiet-json >> $O/sweep3.txt 2>> $O/err.txt; done
cat $O/sweep3.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not slow" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
