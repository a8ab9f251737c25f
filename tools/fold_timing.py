"""Debug experiment: phase times of fold_rows_kernel (build with -DDFA_TREE_TIMING)."""
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
buf = (ctypes.c_ulonglong * 32)()
w = W.get("random")
x = w.input()
dx = torch.from_numpy(x).cuda()
d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
D.dfa_set_option(d.h, D.DFA_OPT_GRAPHS, 0)
for rep in range(4):
    L.dfa_debug_tree_timing(buf, 1)
    buf2 = (ctypes.c_ulonglong * 32)()
    d.chunk_maps(dx, 4096)
    torch.cuda.synchronize()
    L.dfa_debug_tree_timing(buf, 0)
t1 = buf[10]
if t1 and t1 != 0xFFFFFFFFFFFFFFFF:
    print("compose8 (us after first CTA start): waited", (buf[11]-t1)/1e3, "chunks", (buf[12]-t1)/1e3,
          "cta-fold+ticket", (buf[16]-t1)/1e3, "done", (buf[19]-t1)/1e3)
    print("  per-CTA max durations: cta fold", buf[20]/1e3, "ticket", buf[21]/1e3, "last fold", buf[22]/1e3)
    sys.exit(0)
t0 = buf[20]
print("fold phases (us after first CTA start): staged", (buf[21]-t0)/1e3, "cta-fold", (buf[22]-t0)/1e3,
      "last-start", (buf[23]-t0)/1e3, "done", (buf[24]-t0)/1e3)
print("tree (us after its start):", [(buf[i]-buf[0])/1e3 for i in range(1, 8) if buf[i]])
print("fold start after tree start:", (buf[20]-buf[0])/1e3)
