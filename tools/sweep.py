"""Chunk-count and lanes-per-thread sweep (BASELINE.json configs[4]: "sweep of chunk
counts 1K-64K and of lanes per thread 1-8").  One input, one handle; each point is
K timed dfa_chunk_maps steps (CUDA events on the stream, after warm-up), reported
as matched GB/s.  usage: python tools/sweep.py [config] [n_bytes] > profiles/rNN_sweep_<config>.jsonl"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1210_5093_b200 as D  # noqa: E402
import workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "worst"
    w = W.get(name)
    n = int(sys.argv[2]) if len(sys.argv) > 2 else w.full_n
    x = w.input(n)
    dev = torch.device("cuda", 0)
    dx = torch.from_numpy(x).to(dev)
    del x
    a = w.automaton
    d = D.Dfa(a.table, a.q0, a.accept_bitmap)
    imax = d.info["i_max"]
    s = torch.cuda.current_stream()
    points = [(P, 8) for P in (1024, 2048, 4096, 8192, 16384, 32768, 65536)]
    points += [(w.chunks, c) for c in (1, 2, 4, 6)]
    for P, cap in points:
        D.dfa_set_option(d.h, D.DFA_OPT_MAX_LANES, cap)
        bounds = torch.empty(P + 1, dtype=torch.int64, device=dev)
        e0 = torch.empty(1, dtype=torch.int16, device=dev)
        maps = torch.empty(max(P - 1, 1) * imax, dtype=torch.int16, device=dev)
        final = torch.empty(2, dtype=torch.int16, device=dev)
        steps = 5 if n > (1 << 30) else 20
        for _ in range(3):
            D.dfa_chunk_maps(d.h, dx, P, bounds, e0, maps, None, final, stream=s)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(s)
        for _ in range(steps):
            D.dfa_chunk_maps(d.h, dx, P, bounds, e0, maps, None, final, stream=s)
        t1.record(s)
        torch.cuda.synchronize()
        assert D.dfa_get_last_device_error(d.h) == 0
        ms = t0.elapsed_time(t1) / steps
        fin = int(final.cpu().numpy().view("uint16")[0])
        print(json.dumps({"config": name, "n": n, "chunks": P, "lanes_per_thread": cap, "steps": steps,
                          "ms_per_step": ms, "GB/s": n / (ms * 1e-3) / 1e9, "final_state": fin}), flush=True)


if __name__ == "__main__":
    main()
