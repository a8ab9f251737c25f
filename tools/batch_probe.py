"""Probe: one dfa_match_batch call of N x L-byte records (for ncu / timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1210_5093_b200 as D  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "random"
L = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
N = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 18
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
w = W.get(name)
x = w.input(N * L)
dx = torch.from_numpy(x).cuda()
d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
offs = torch.arange(N + 1, dtype=torch.int64, device="cuda") * L
fin = torch.empty(N, dtype=torch.int16, device="cuda")
acc = torch.empty(N, dtype=torch.uint8, device="cuda")
for _ in range(reps):
    D.dfa_match_batch(d.h, dx, offs, fin, acc)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    D.dfa_match_batch(d.h, dx, offs, fin, acc)
b.record()
torch.cuda.synchronize()
print(f"{name} batch {N} x {L}: {a.elapsed_time(b) / 10:.4f} ms/call, stats {D.dfa_get_stats(d.h)}")
