set -x
O=gpurun_out/r02k
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "config_small or max_lanes or rep8_with_converge or subchunk or misaligned or segment or alg2 or worst or protein" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
for c in worst protein; do python bench.py --config $c --steps 10 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json >> $O/q.txt 2>&1; done
python bench.py --config worst --n 1073741824 --steps 10 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json >> $O/q.txt 2>&1
