O=gpurun_out/w16
mkdir -p $O
rm -f $O/sweep3.txt
for c in protein worst; do python bench.py --config $c --steps 20 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --quiet-json >> $O/sweep3.txt 2>> $O/err.txt; done
cat $O/sweep3.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "protein" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
