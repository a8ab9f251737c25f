"""Timing experiments on a library variant (results ignored): DFA_LIB=<variant .so>
python tools/exp_time.py [config] [steps].  Prints ms/step and GB/s of dfa_chunk_maps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1210_5093_b200 as D  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "random"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
w = W.get(name)
x = w.input()
dx = torch.from_numpy(x).cuda()
d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
P = w.chunks
for _ in range(5):
    d.chunk_maps(dx, P)
torch.cuda.synchronize()
D.dfa_get_last_device_error(d.h)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    d.chunk_maps(dx, P)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / steps
print(f"{os.path.basename(os.environ.get('DFA_LIB', 'libdfa.so'))} {name}: {ms:.4f} ms/step {x.size / ms / 1e6:.1f} GB/s")
