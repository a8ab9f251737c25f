set -x
O=gpurun_out/r02n
mkdir -p $O
Q="python bench.py --config tiny --steps 100 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json"
$Q >> $O/tiny.txt 2>&1
$Q --opt fused_tail=1 >> $O/tiny.txt 2>&1
$Q --opt fused_tail=1 --opt threads_per_cta=1024 --opt subchunk_target=32768 >> $O/tiny.txt 2>&1
$Q --opt fused_tail=1 --opt threads_per_cta=1024 --opt subchunk_target=16384 >> $O/tiny.txt 2>&1
$Q --opt fused_tail=1 --opt threads_per_cta=512 --opt subchunk_target=16384 >> $O/tiny.txt 2>&1
$Q --opt fused_tail=0 --opt threads_per_cta=1024 --opt subchunk_target=32768 >> $O/tiny.txt 2>&1
$Q --opt fused_tail=0 --opt threads_per_cta=512 --opt subchunk_target=16384 >> $O/tiny.txt 2>&1
$Q --opt fused_tail=0 --opt subchunk_target=8192 >> $O/tiny.txt 2>&1
