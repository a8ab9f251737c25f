O=gpurun_out/tma1
mkdir -p $O
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -3 $O/smoke.log
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "random and not slow" > $O/pytest_random.log 2>&1; echo "rc=$?" >> $O/pytest_random.log; tail -5 $O/pytest_random.log
for t in 1 0; do timeout 300 python bench.py --config random --steps 50 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-work --quiet-json --opt tma_input=$t >> $O/bench.txt 2>> $O/bench.err; done
cat $O/bench.txt
