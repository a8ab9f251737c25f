set -x
O=gpurun_out/r02v
mkdir -p $O
B="python bench.py --config worst --steps 10 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --no-work --quiet-json"
run() { DFA_LIB=$PWD/paper_1210_5093_b200/$1 $B ${2:+--opt subchunk_target=$2} >> $O/sweep.txt 2>> $O/sweep.err; echo "   ^ lib=$1 target=${2:-auto}" >> $O/sweep.txt; }
run libdfa.so
run libdfa.so 104192
run libdfa_p768.so 113664
run libdfa_p768.so 104192
run libdfa_p832.so 123136
run libdfa_p1024.so 132608
run libdfa_p1024.so 151552
cat $O/sweep.txt
