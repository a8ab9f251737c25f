"""Debug experiment: per-level completion times of tree_kernel (build with -DDFA_TREE_TIMING)."""
import ctypes, os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HERE = os.path.dirname(os.path.abspath(__file__))
lib = "/tmp/libdfa_timing.so"
src = os.path.join(HERE, "..", "paper_1210_5093_b200", "csrc")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-DDFA_TREE_TIMING",
                       "-Xcompiler", "-fPIC", "-shared", "-o", lib] + [os.path.join(src, f) for f in ("api.cpp", "prep.cpp", "kernels.cu")])
os.environ["DFA_LIB"] = lib
import numpy as np, torch
import paper_1210_5093_b200 as D
import workloads as W
L = ctypes.CDLL(lib)
buf = (ctypes.c_ulonglong * 32)()
name = sys.argv[1] if len(sys.argv) > 1 else "random"
w = W.get(name)
x = w.input(int(sys.argv[3]) if len(sys.argv) > 3 else w.full_n)
dx = torch.from_numpy(x).cuda()
d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
for P in [int(p) for p in sys.argv[2].split(",")] if len(sys.argv) > 2 else [w.chunks]:
    for F in (8, 32, 64):
        D.dfa_set_option(d.h, D.DFA_OPT_TREE_FANIN, F)
        for rep in range(3):
            L.dfa_debug_tree_timing(buf, 1)
            d.chunk_maps(dx, P)
            torch.cuda.synchronize()
            L.dfa_debug_tree_timing(buf, 0)
        t0 = buf[0]
        lv = [(buf[i] - t0) / 1000 for i in range(1, 32) if buf[i]]
        print(f"{name} P={P} F={F} level done (us after kernel start):", [round(v, 1) for v in lv])
