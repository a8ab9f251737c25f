set -x
O=gpurun_out/r02q
mkdir -p $O
python - > $O/h2d.txt 2>&1 <<'PY'
import torch, time
x = torch.empty(1 << 30, dtype=torch.uint8).pin_memory(); y = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10): y.copy_(x, non_blocking=True)
b.record(); torch.cuda.synchronize()
print("pinned H2D GB/s", 10 * (1 << 30) / (a.elapsed_time(b) * 1e-3) / 1e9)
PY
for lib in libdfa.so libdfa_w768.so; do DFA_LIB=$PWD/paper_1210_5093_b200/$lib python bench.py --config protein --steps 10 --e2e-steps 1 --no-cpu-baseline --no-lookahead --no-batch --no-ceiling --quiet-json >> $O/w768.txt 2>&1; done
tools/checked_run.sh $O
