O=gpurun_out/kw
mkdir -p $O
rm -f $O/sweep4.txt
B="python bench.py --config random --steps 50 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --no-work --quiet-json"
for t in 73728 81920 86016 90112 94208; do $B --opt subchunk_target=$t >> $O/sweep4.txt 2>> $O/err.txt; done
cat $O/sweep4.txt
