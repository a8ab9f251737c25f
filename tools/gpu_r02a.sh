set -x
mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02a/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02a/pytest.log
python bench.py --config worst --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02a/bench_worst.json 2> gpurun_out/r02a/bench_worst.err
python bench.py --config protein --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/r02a/bench_protein.json 2> gpurun_out/r02a/bench_protein.err
tools/sanitize.sh gpurun_out/r02a memcheck synccheck racecheck initcheck
