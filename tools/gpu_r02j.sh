set -x
O=gpurun_out/r02j
mkdir -p $O
python tools/phase_timing.py random keyword tiny > $O/phase_fused.txt 2>&1
FUSED=0 python tools/phase_timing.py random keyword tiny > $O/phase_nofused.txt 2>&1
