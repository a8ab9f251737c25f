"""Debug experiment: phase timestamps of one dfa_chunk_maps call (lanes_kernel prologue, match loop,
epilogue; compose8 PDL wait, chunk phase, ticket, last-CTA fold), in microseconds after the first lanes
CTA starts.  Builds the library with -DDFA_TREE_TIMING into /tmp.  usage: tools/phase_timing.py random keyword"""
import ctypes, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import hashlib
_src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1210_5093_b200", "csrc")
_h = hashlib.sha256(b"".join(open(os.path.join(_src, f), "rb").read() for f in sorted(os.listdir(_src)))).hexdigest()[:12]
lib = f"/tmp/libdfa_timing_{_h}.so"  # keyed by the source: /tmp survives between calls on a reused box
src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_1210_5093_b200", "csrc")
if not os.path.exists(lib):
    # one translation unit (DFA_TU_MODE=0: every layout's match kernels beside the composition
    # kernels) so that all kernels write the same g_tree_t
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-DDFA_TREE_TIMING",
                           "-DDFA_TU_MODE=0", "-DDFA_TU_MAIN=1", "-diag-suppress", "177",
                           "-Xcompiler", "-fPIC", "-shared", "-o", lib] +
                          [os.path.join(src, f) for f in ("api.cpp", "prep.cpp", "kernels.cu")])
os.environ["DFA_LIB"] = lib
import torch
import paper_1210_5093_b200 as D
import workloads as W
L = ctypes.CDLL(lib)
buf = (ctypes.c_ulonglong * 32)()
for name in sys.argv[1:]:
    w = W.get(name)
    x = w.input()
    dx = torch.from_numpy(x).cuda()
    d = D.Dfa(w.automaton.table, w.automaton.q0, w.automaton.accept_bitmap)
    D.dfa_set_option(d.h, D.DFA_OPT_FUSED_TAIL, int(os.environ.get("FUSED", "1")))
    for rep in range(6):
        L.dfa_debug_tree_timing(buf, 1)
        d.chunk_maps(dx, w.chunks)
        torch.cuda.synchronize()
        L.dfa_debug_tree_timing(buf, 0)
        t0 = buf[25]
        names = {25: "lanes start", 26: "table loaded", 27: "run_lanes done(max)", 28: "warp_compose done(max)", 29: "lanes end(max)",
                 10: "compose8 start(min)", 11: "pdl_wait passed(max)", 12: "chunk phase done(max)", 16: "ticket(max)", 19: "final written"}
        if rep >= 4 and os.environ.get("FUSED", "1") == "1":
            print("  fused tail per-CTA max durations (us): staging+geometry", round(buf[13] / 1000, 2),
                  "short-segment warp", round(buf[18] / 1000, 2), "chunk phase", round(buf[17] / 1000, 2))
        if rep >= 4:
            print(name, {v: round((buf[k] - t0) / 1000, 2) for k, v in names.items() if buf[k]},
                  "cta_fold_dur", round(buf[20] / 1000, 2), "ticket_dur", round(buf[21] / 1000, 2), "last_fold", round(buf[22] / 1000, 2))
