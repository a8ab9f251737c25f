set -x
O=gpurun_out/quick
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "not slow" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
rm -f $O/bench.txt
for c in worst protein keyword random; do python bench.py --config $c --no-cpu-baseline --no-batch --no-lookahead --e2e-steps 1 --quiet-json >> $O/bench.txt 2>> $O/bench.err; done
cat $O/bench.txt
