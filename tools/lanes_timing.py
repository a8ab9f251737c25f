"""Debug experiment: phase times of lanes_kernel and compose8_kernel (build with -DDFA_TREE_TIMING).
usage: python tools/lanes_timing.py [config] [P]"""
import ctypes, os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
HERE = os.path.dirname(os.path.abspath(__file__))
lib = "/tmp/libdfa_timing.so"
src = os.path.join(HERE, "..", "paper_1210_5093_b200", "csrc")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-DDFA_TREE_TIMING",
                       "-Xcompiler", "-fPIC", "-shared", "-o", lib] + [os.path.join(src, f) for f in ("api.cpp", "prep.cpp", "kernels.cu")])
os.environ["DFA_LIB"] = lib
import torch
import paper_1210_5093_b200 as D
import workloads as W
L = ctypes.CDLL(lib)
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
w = W.get(name)
P = int(sys.argv[2]) if len(sys.argv) > 2 else w.chunks
x = w.input(w.full_n if w.full_n <= (1 << 28) else (1 << 28))
dx = torch.from_numpy(x).cuda()
d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
D.dfa_set_option(d.h, D.DFA_OPT_GRAPHS, 0)
buf = (ctypes.c_ulonglong * 32)()
for rep in range(5):
    L.dfa_debug_tree_timing(buf, 1)
    d.chunk_maps(dx, P)
    torch.cuda.synchronize()
    L.dfa_debug_tree_timing(buf, 0)
t0 = buf[25]
us = lambda i: (buf[i] - t0) / 1e3
print(f"{name} n={x.size} P={P} lanes (us after first CTA start): staged {us(26):.2f} run_lanes {us(27):.2f} "
      f"warp_compose {us(28):.2f} end {us(29):.2f}")
print(f"  compose8: first CTA start {us(10):.2f} waited {us(11):.2f} chunks {us(12):.2f} ticket {us(16):.2f} "
      f"done {us(19):.2f}")
