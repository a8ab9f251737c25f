O=gpurun_out/r02z
mkdir -p $O
B="python bench.py --config tiny --steps 50 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --no-work --quiet-json"
for t in 0 1024 2048 4096 8192 16384 65536; do $B --opt subchunk_target=$t >> $O/tiny_sweep.txt 2>> $O/err.txt; done
B="python bench.py --config random --steps 50 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --no-work --quiet-json"
for t in 0 47360 71040 94720; do $B --opt subchunk_target=$t >> $O/tiny_sweep.txt 2>> $O/err.txt; done
cat $O/tiny_sweep.txt
